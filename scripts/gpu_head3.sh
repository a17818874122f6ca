mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_epoch.py -x -q -m gpu -k "head or chunked or bf16" > gpurun_out/head_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/head_tests.log
timeout 600 python bench.py --config papers_slice8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/slice8_1.log 2>&1; echo s8=$?
tail -1 gpurun_out/slice8_1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:head_fused -s 1 -c 1 -o gpurun_out/head_s8b -f \
    python bench.py --config papers_slice8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_head.log 2>&1; echo nh=$?
