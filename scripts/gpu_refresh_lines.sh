#!/bin/bash
# (gpurun --gpus 4) DRAM bytes of the padded Reddit slices (32 / 16 columns), then the Reddit and papers
# lines at N = 2 / 4 again with every roofline on measured traffic; JSON under gpurun_out/refresh/.
O=gpurun_out/refresh
mkdir -p $O gpurun_out/prof
cp profiles/spmm_traffic.json gpurun_out/prof/spmm_traffic.json
ncu --set full --clock-control none -k regex:spmm_hop -o /tmp/rp -f python scripts/spmm_bench.py --K 1 --reps 1 \
    --warmup 0 --config reddit --widths 32,16 > $O/ncu_rp.log 2>&1; echo ncu=$?
python scripts/profile_hops.py --outdir gpurun_out/prof --rep /tmp/rp.ncu-rep --tag r02_hops_reddit_padded \
    --keys reddit/P2/f32/d32,reddit/P4/f32/d16 --widths 32,16 --elem 4 \
    --note "spmm_bench.py --config reddit: the slices bench.py pads at N = 2 / 4 (--slice-align auto)" >> $O/ncu_rp.log 2>&1; echo sum=$?
rm -f /tmp/rp.ncu-rep
cp gpurun_out/prof/spmm_traffic.json profiles/spmm_traffic.json
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  timeout 600 $R --nproc-per-node $N --master-port 2995$N bench.py --gpus $N --steps 10 --warmup 3 > $O/reddit_N$N.log 2>&1; echo reddit$N=$?
  tail -1 $O/reddit_N$N.log > $O/reddit_N$N.json
  timeout 900 $R --nproc-per-node $N --master-port 2996$N bench.py --gpus $N --config papers --steps 3 --warmup 3 --no-e2e --no-hbm-leg > $O/papers_N$N.log 2>&1; echo papers$N=$?
  tail -1 $O/papers_N$N.log > $O/papers_N$N.json
  timeout 900 $R --nproc-per-node $N --master-port 2997$N bench.py --gpus $N --config papers --steps 3 --warmup 3 --no-e2e --no-hbm-leg --overlap --chunks 4 --layouts p2p > $O/papers_ce_N$N.log 2>&1; echo papers_ce$N=$?
  tail -1 $O/papers_ce_N$N.log > $O/papers_ce_N$N.json
done
python - <<'PY'
import json
for f in ("reddit_N2", "reddit_N4", "papers_N2", "papers_N4", "papers_ce_N2", "papers_ce_N4"):
    try:
        d = json.load(open(f"gpurun_out/refresh/{f}.json"))
    except Exception as e:
        print(f, "no line", e); continue
    r = d["roofline"]
    print(f, round(d["ms_per_step"], 2), r.get("bound"), round(r.get("frac") or 0, 3), r.get("traffic"), (r.get("hbm") or {}).get("traffic"))
PY
