mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_epoch.py -x -q -m gpu -k "pack or head or chunked or bf16" > gpurun_out/pack_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/pack_tests.log
for f in 1 0; do NTP_PACK_FUSED=$f timeout 600 python bench.py --config papers --steps 5 --warmup 3 --no-e2e > gpurun_out/papers_pk$f.log 2>&1; echo p=$?
tail -1 gpurun_out/papers_pk$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'])"; done
