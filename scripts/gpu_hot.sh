python -c "
import ctypes, torch
p = torch.cuda.get_device_properties(0)
print('L2', p.L2_cache_size, 'persist max', getattr(p, 'persisting_l2_cache_max_size', None))"
for hm in 0 32 64 96; do NTP_L2_HOT=$hm timeout 300 python scripts/spmm_bench.py --config papers --dtype bf16 --reorder --widths 128,16 --K 2 --reps 3; done > gpurun_out/hot.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/hot.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(r['config'], r['d'], r['ms_per_hop'], r['env'])
PY
