for vb in 16 32; do NTP_SPMM_VB=$vb timeout 300 python scripts/spmm_bench.py --config papers --dtype bf16 --reorder --widths 128,64,32,16 --K 2 --reps 3; done > gpurun_out/papers_vb.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/papers_vb.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(r['config'], r['d'], r['ms_per_hop'], r['env'])
PY
timeout 600 python bench.py --config papers --steps 5 --warmup 3 --no-e2e > gpurun_out/papers_n1.log 2>&1; echo p1=$?
tail -1 gpurun_out/papers_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'])"
