set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 600 python bench.py --config papers --steps 5 --warmup 3 --no-e2e > gpurun_out/final_papers_n1.log 2>&1; echo p1=$?
timeout 600 python bench.py --config products --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final_products_n1.log 2>&1; echo pr1=$?
timeout 600 python bench.py --engine coupled --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final_coupled_n1.log 2>&1; echo c1=$?
