# c5 papers-shaped epoch at N=1 (memory-lean path) and the products/orkut shapes
mkdir -p gpurun_out
free -g | head -2; nproc
timeout 900 python bench.py --config papers --steps 5 --warmup 3 --no-e2e > gpurun_out/papers_n1.log 2>&1; echo papers=$?
tail -1 gpurun_out/papers_n1.log | cut -c1-2500
timeout 600 python bench.py --config products --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/products_n1.log 2>&1; echo products=$?
tail -1 gpurun_out/products_n1.log | cut -c1-1200
