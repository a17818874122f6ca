timeout 900 python -m pytest tests/test_gpu_epoch.py -x -q -m gpu -k "wgrad or head_bf16" > gpurun_out/wg_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/wg_tests.log; grep -m2 "relative" gpurun_out/wg_tests.log
for f in 1 0; do NTP_WGRAD_FUSED=$f timeout 600 python bench.py --config papers_slice8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s8_wg$f.log 2>&1
tail -1 gpurun_out/s8_wg$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms']['mlp_bwd'])"; done
