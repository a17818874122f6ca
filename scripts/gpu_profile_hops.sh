#!/bin/bash
# Round-2 measurement pass (one gpurun call, 1 GPU):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- bash scripts/gpu_profile_hops.sh
# bench line (with the HBM-bound Orkut leg), then one ncu --set full capture of spmm_hop_kernel per slice
# width for the final kernel variants (papers bf16 d_s 128/64/32/16 reordered, Orkut w=512 fp32 at the
# N = 1/2/4/8 slice widths, products, Reddit), and the bench's launch list.
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_r02.log | cut -c1-4000
NCU="ncu --set full --import-source on --clock-control none -k regex:spmm_hop_kernel"
SB="python scripts/spmm_bench.py --K 1 --reps 1 --warmup 0"
$NCU -o gpurun_out/r02_hops_orkut -f $SB --config orkut --widths 512,256,128,64 --reorder > gpurun_out/ncu_orkut.log 2>&1; echo orkut=$?
$NCU -o gpurun_out/r02_hops_reddit -f $SB --config reddit --widths 44,24,12,8 > gpurun_out/ncu_reddit.log 2>&1; echo reddit=$?
$NCU -o gpurun_out/r02_hops_products -f $SB --config products --widths 48,24,12,8 --reorder > gpurun_out/ncu_products.log 2>&1; echo products=$?
$NCU -o gpurun_out/r02_hops_papers -f $SB --config papers --dtype bf16 --widths 128,64,32,16 --reorder > gpurun_out/ncu_papers.log 2>&1; echo papers=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_reddit_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-hbm-leg > gpurun_out/ncu_ll.log 2>&1; echo ll=$?
