for vb in 16 32; do NTP_SPMM_VB=$vb timeout 300 python scripts/spmm_bench.py --config reddit --widths 44,24,12,8 --K 2 --reps 10; done > gpurun_out/reddit_vb.jsonl 2>&1
for vb in 16 32; do NTP_SPMM_VB=$vb timeout 300 python scripts/spmm_bench.py --config products --reorder --widths 48,24,12,8 --K 2 --reps 10; done >> gpurun_out/reddit_vb.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/reddit_vb.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(r['config'], r['d'], r['ms_per_hop'], r['env'])
PY
