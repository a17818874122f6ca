mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_propagate.py -x -q -m gpu -k "prefetch" > gpurun_out/pf_tests.log 2>&1; echo ptests=$?
tail -2 gpurun_out/pf_tests.log
for pf in 0 64 128 256 512; do NTP_SPMM_PF=$pf python scripts/spmm_bench.py --config papers --dtype bf16 --reorder --widths 128,64,32,16 --K 2 --reps 3; done > gpurun_out/papers_pf.jsonl 2>&1
for pf in 0 128 512; do NTP_SPMM_PF=$pf python scripts/spmm_bench.py --config products --reorder --widths 48,12 --K 2 --reps 5; done >> gpurun_out/papers_pf.jsonl 2>&1
for pf in 0 128; do NTP_SPMM_PF=$pf python scripts/spmm_bench.py --config reddit --widths 44,8 --K 2 --reps 5; done >> gpurun_out/papers_pf.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/papers_pf.jsonl'):
    try: r=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(r['config'], r['d'], r['ms_per_hop'], r['env'])
PY
