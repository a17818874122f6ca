#!/bin/bash
# ncu DRAM bytes of the fp32 papers hop (d_s = 128, 512-B rows: the NEXT-3 host-streamed epoch's slice)
mkdir -p gpurun_out/prof
cp profiles/spmm_traffic.json gpurun_out/prof/spmm_traffic.json
ncu --set full --clock-control none -k regex:spmm_hop -o /tmp/r02_hops_papers_f32 -f \
    python scripts/spmm_bench.py --K 1 --reps 1 --warmup 0 --widths 128 --config papers --dtype f32 --reorder \
    > gpurun_out/ncu_papers_f32.log 2>&1; echo ncu=$?
python scripts/profile_hops.py --outdir gpurun_out/prof --rep /tmp/r02_hops_papers_f32.ncu-rep --tag r02_hops_papers_f32 \
    --keys papers/P1/f32 --widths 128 --elem 4 --note "spmm_bench.py --config papers --dtype f32 --reorder" \
    >> gpurun_out/ncu_papers_f32.log 2>&1; echo sum=$?
rm -f /tmp/r02_hops_papers_f32.ncu-rep
cat gpurun_out/prof/r02_hops_papers_f32.md
