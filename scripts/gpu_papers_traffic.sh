#!/bin/bash
# ncu DRAM bytes of the papers bf16 hops at the N = 2 / 4 slice widths and the N = 8 backward hop (the
# --set full captures of these launches returned NaN metrics): a short metric list instead.
mkdir -p gpurun_out/prof
cp profiles/spmm_traffic.json gpurun_out/prof/spmm_traffic.json
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,lts__t_sectors.avg.pct_of_peak_sustained_elapsed"
SB="python scripts/spmm_bench.py --K 1 --reps 1 --warmup 0 --config papers --dtype bf16 --reorder"
ncu --metrics $M --clock-control none -k regex:spmm_hop -o /tmp/pp -f $SB --widths 64,32 > gpurun_out/ncu_pp.log 2>&1; echo ncu_fwd=$?
python scripts/profile_hops.py --outdir gpurun_out/prof --rep /tmp/pp.ncu-rep --tag r02_hops_papers_P2P4 \
    --keys papers/P2/bf16,papers/P4/bf16 --widths 64,32 --elem 2 --note "spmm_bench.py --config papers --dtype bf16 --reorder (short metric list)" >> gpurun_out/ncu_pp.log 2>&1; echo sum_fwd=$?
ncu --metrics $M --clock-control none -k regex:spmm_hop -o /tmp/pb -f $SB --widths 16 --bwd > gpurun_out/ncu_pb.log 2>&1; echo ncu_bwd=$?
python scripts/profile_hops.py --outdir gpurun_out/prof --rep /tmp/pb.ncu-rep --tag r02_hops_papers_bwd_P8 \
    --keys papers_bwd/P8/bf16 --widths 16 --elem 2 --note "spmm_bench.py --config papers --dtype bf16 --reorder --bwd (short metric list)" >> gpurun_out/ncu_pb.log 2>&1; echo sum_bwd=$?
rm -f /tmp/pp.ncu-rep /tmp/pb.ncu-rep
cat gpurun_out/prof/r02_hops_papers_P2P4.md gpurun_out/prof/r02_hops_papers_bwd_P8.md
