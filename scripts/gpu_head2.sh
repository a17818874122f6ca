mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_epoch.py -x -q -m gpu -k "head or chunked or bf16" > gpurun_out/head_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/head_tests.log
for f in 1 0; do NTP_HEAD_FUSED=$f timeout 600 python bench.py --config papers_slice8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/slice8_$f.log 2>&1; echo s8_$f=$?
tail -1 gpurun_out/slice8_$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'])"; done
for o in 0 1 2; do NTP_SPMM_OCC=$o python scripts/spmm_bench.py --config papers --dtype bf16 --reorder --widths 128,16 --K 2 --reps 3; done > gpurun_out/papers_occ.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/papers_occ.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(r['d'], r['ms_per_hop'], r['env'])
PY
