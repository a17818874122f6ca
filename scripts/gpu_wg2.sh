timeout 900 python -m pytest tests/test_gpu_epoch.py -x -q -m gpu -k "wgrad" > gpurun_out/wg_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/wg_tests.log
NTP_WGRAD_FUSED=1 timeout 600 python bench.py --config papers_slice8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s8_wg1.log 2>&1
tail -1 gpurun_out/s8_wg1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms']['mlp_bwd'])"
NTP_WGRAD_FUSED=0 timeout 600 python bench.py --config papers_slice8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s8_wg0.log 2>&1
tail -1 gpurun_out/s8_wg0.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms']['mlp_bwd'])"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:wgrad_kernel -s 1 -c 1 -o gpurun_out/wgrad_s8 -f \
    env NTP_WGRAD_FUSED=1 python bench.py --config papers_slice8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_wg.log 2>&1; echo ncu=$?
