mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_propagate.py tests/test_gpu_epoch.py tests/test_gpu_papers.py tests/test_gpu_coupled.py -x -q -m gpu > gpurun_out/vb_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/vb_tests.log
timeout 600 python bench.py --config papers --steps 5 --warmup 3 --no-e2e > gpurun_out/papers_n1.log 2>&1; echo p1=$?
tail -1 gpurun_out/papers_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['phase_ms'], d['roofline']['frac'])"
timeout 600 python bench.py --config products --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/products_n1.log 2>&1; echo pr=$?
tail -1 gpurun_out/products_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'])"
