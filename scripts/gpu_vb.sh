for o in 0 2; do for vb in 16 32; do
  NTP_SPMM_OCC=$o NTP_SPMM_VB=$vb python scripts/spmm_bench.py --config reddit --widths 44,24,16,8 --K 2 --reps 10
done; done > gpurun_out/vb.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/vb.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l.strip()); continue
    print(r['d'], r['ms_per_hop'], r['env'])
PY
