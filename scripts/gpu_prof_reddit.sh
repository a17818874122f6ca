#!/bin/bash
# ncu --set full of the Reddit hop at every slice width with the final variants, and the bench's launch list
mkdir -p gpurun_out/prof
cp profiles/spmm_traffic.json gpurun_out/prof/spmm_traffic.json
ncu --set full --clock-control none -k regex:spmm_hop -o /tmp/rr -f python scripts/spmm_bench.py --K 1 --reps 1 \
    --warmup 0 --config reddit --widths 44,24,12,8 > gpurun_out/ncu_rr.log 2>&1; echo ncu=$?
python scripts/profile_hops.py --outdir gpurun_out/prof --rep /tmp/rr.ncu-rep --tag r02_hops_reddit \
    --keys reddit/P1/f32,reddit/P2/f32,reddit/P4/f32,reddit/P8/f32 --widths 44,24,12,8 --elem 4 \
    --note "spmm_bench.py --config reddit (d_s 44: the single-accumulator 4-CTA/SM variant, 64 registers)" >> gpurun_out/ncu_rr.log 2>&1; echo sum=$?
rm -f /tmp/rr.ncu-rep
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/r02_reddit_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-hbm-leg > gpurun_out/ncu_ll.log 2>&1; echo ll=$?
cat gpurun_out/prof/r02_hops_reddit.md
