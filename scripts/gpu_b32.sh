timeout 300 python scripts/spmm_bench.py --config papers --dtype bf16 --reorder --widths 128,64,16 --K 2 --reps 3 > gpurun_out/b32.jsonl 2>&1
timeout 300 python scripts/spmm_bench.py --config products --reorder --widths 24 --K 2 --reps 10 >> gpurun_out/b32.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/b32.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(r['config'], r['d'], r['ms_per_hop'])
PY
