timeout 900 python -m pytest tests/test_gpu_epoch.py -x -q -m gpu -k "head or pack or wgrad" > gpurun_out/hd_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/hd_tests.log
timeout 600 python bench.py --config papers_slice8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s8_hd.log 2>&1
tail -1 gpurun_out/s8_hd.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'])"
