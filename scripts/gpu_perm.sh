timeout 900 python -m pytest tests/test_gpu_epoch.py -x -q -m gpu -k "head or reordered or wgrad or pack" > gpurun_out/perm_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/perm_tests.log; grep -m3 "Error" gpurun_out/perm_tests.log
timeout 600 python bench.py --config papers --steps 5 --warmup 3 --no-e2e > gpurun_out/papers_perm.log 2>&1; echo p=$?
tail -1 gpurun_out/papers_perm.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k: round(v,1) for k,v in d['phase_ms'].items()})"
