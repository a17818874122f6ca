#!/bin/bash
# papers100M shape on one B200: the bf16 epoch, the fp32 epoch with host-resident inputs (NEXT-3), and the
# Orkut bulk-gather hop under ncu (traffic for the bench's HBM leg at N = 1, 2).
#   /usr/local/graft/bin/gpurun --timeout 3000 -- bash scripts/gpu_papers.sh
mkdir -p gpurun_out/prof
cp profiles/spmm_traffic.json gpurun_out/prof/spmm_traffic.json
NCU="ncu --set full --clock-control none -k regex:spmm_hop"
$NCU -o /tmp/r02_hops_orkut_bulk -f python scripts/spmm_bench.py --K 1 --reps 1 --warmup 0 --widths 512,256 --config orkut --reorder > gpurun_out/ncu_orkut_bulk.log 2>&1; echo ncu=$?
python scripts/profile_hops.py --outdir gpurun_out/prof --rep /tmp/r02_hops_orkut_bulk.ncu-rep --tag r02_hops_orkut_bulk --keys orkut/P1/f32,orkut/P2/f32 --widths 512,256 --elem 4 --note "spmm_bench.py --config orkut --reorder: spmm_hop_bulk_kernel (rows >= 1 KB)" >> gpurun_out/ncu_orkut_bulk.log 2>&1; echo sum=$?
rm -f /tmp/r02_hops_orkut_bulk.ncu-rep
python bench.py --config papers --steps 3 --warmup 3 --no-e2e --no-hbm-leg > gpurun_out/papers_bf16.log 2>&1; echo papers_bf16=$?
tail -1 gpurun_out/papers_bf16.log | cut -c1-600
python bench.py --config papers --dtype f32 --host-stream --chunks 32 --steps 2 --warmup 3 --no-hbm-leg --no-cpu-baseline > gpurun_out/papers_f32_hs.log 2>&1; echo papers_f32=$?
tail -1 gpurun_out/papers_f32_hs.log | cut -c1-600
