mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_epoch.py -x -q -m gpu -k "wgrad or head or pack or chunked or bf16" > gpurun_out/wg_tests.log 2>&1; echo tests=$?
tail -25 gpurun_out/wg_tests.log | grep -v "^$" | tail -12
for f in 1 0; do NTP_WGRAD_FUSED=$f timeout 600 python bench.py --config papers --steps 5 --warmup 3 --no-e2e > gpurun_out/papers_wg$f.log 2>&1; echo p=$?
tail -1 gpurun_out/papers_wg$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'])"; done
