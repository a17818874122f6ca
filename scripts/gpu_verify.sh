#!/bin/bash
# One gpurun call that reproduces the driver's round-end checks on a B200:
#   /usr/local/graft/bin/gpurun --timeout 3000 -- bash scripts/gpu_verify.sh [pytest-args]
# smoke(), pytest -m gpu, the bench line (N = 1) and the reference arm; logs under gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q ${@} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | cut -c1-1500
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
tail -1 gpurun_out/bench_ref.log | cut -c1-400
