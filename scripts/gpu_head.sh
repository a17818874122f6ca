# fused head: parity tests, then the papers N=1 epoch with and without it, and the epoch launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_epoch.py tests/test_synth.py -x -q -m gpu -k "head or cuda or chunked or bf16" > gpurun_out/head_tests.log 2>&1; echo tests=$?
tail -15 gpurun_out/head_tests.log
timeout 600 python bench.py --config papers --steps 5 --warmup 3 --no-e2e > gpurun_out/papers_fused.log 2>&1; echo fused=$?
tail -1 gpurun_out/papers_fused.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'])"
NTP_HEAD_FUSED=0 timeout 600 python bench.py --config papers --steps 3 --warmup 3 --no-e2e > gpurun_out/papers_unfused.log 2>&1; echo unfused=$?
tail -1 gpurun_out/papers_unfused.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/papers_launches.csv \
    python bench.py --config papers --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/papers_ll.log 2>&1; echo ll=$?
tail -2 gpurun_out/papers_ll.log
