mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_propagate.py -x -q -m gpu -k "pipelined" > gpurun_out/pipe_tests.log 2>&1; echo ptests=$?
tail -3 gpurun_out/pipe_tests.log
timeout 900 python -m pytest tests/test_gpu_epoch.py -x -q -m gpu -k "head or chunked or bf16" > gpurun_out/head_tests.log 2>&1; echo htests=$?
tail -2 gpurun_out/head_tests.log
timeout 600 python bench.py --config papers_slice8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/slice8_1.log 2>&1; echo s8=$?
tail -1 gpurun_out/slice8_1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'])"
for pp in 0 1 2; do NTP_SPMM_PIPE=$pp python scripts/spmm_bench.py --config papers --dtype bf16 --reorder --widths 128,64,32,16 --K 2 --reps 3; done > gpurun_out/papers_pipe.jsonl 2>&1
for pp in 0 1 2; do NTP_SPMM_PIPE=$pp python scripts/spmm_bench.py --config products --reorder --widths 48,24,12,8 --K 2 --reps 5; done >> gpurun_out/papers_pipe.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/papers_pipe.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(r['config'], r['d'], r['ms_per_hop'], r['env'])
PY
