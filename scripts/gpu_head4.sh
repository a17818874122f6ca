mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_epoch.py -x -q -m gpu -k "head or chunked or bf16" > gpurun_out/head_tests.log 2>&1; echo htests=$?
tail -2 gpurun_out/head_tests.log
for t in 1 0; do NTP_HEAD_TMA=$t timeout 600 python bench.py --config papers_slice8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/slice8_t$t.log 2>&1; echo s8=$?
tail -1 gpurun_out/slice8_t$t.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'])"; done
