timeout 1200 python -m pytest tests/test_gpu_propagate.py -x -q -m gpu -k "stream or dense" 2>&1 | tail -3
for st in 0 1 3 8; do NTP_SPMM_STREAM=$st python scripts/spmm_bench.py --config reddit --widths 16,12,8 --K 2 --reps 10; done > gpurun_out/stream.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/stream.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l.strip()); continue
    print(r['d'], r['ms_per_hop'], r['env'])
PY
