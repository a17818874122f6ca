mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_propagate.py -x -q -m gpu -k "ring" > gpurun_out/ring_tests.log 2>&1; echo rtests=$?
tail -15 gpurun_out/ring_tests.log
for rr in 0 1; do NTP_SPMM_RING=$rr timeout 300 python scripts/spmm_bench.py --config papers --dtype bf16 --reorder --widths 128,64 --K 2 --reps 3; done > gpurun_out/papers_ring.jsonl 2>&1
for rr in 0 1; do NTP_SPMM_RING=$rr timeout 300 python scripts/spmm_bench.py --config products --reorder --widths 48,32 --K 2 --reps 5; done >> gpurun_out/papers_ring.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/papers_ring.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(r['config'], r['d'], r['ms_per_hop'], r['env'])
PY
