#!/bin/bash
# Round-2 measurement pass (one gpurun call, 1 GPU):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- bash scripts/gpu_profile_hops.sh [--bench]
# one ncu --set full capture of spmm_hop_kernel per slice width for the final kernel variants (papers bf16
# d_s 128/64/32/16 reordered, Orkut w=512 fp32 at the N = 1/2/4/8 slice widths, products, Reddit), summarised
# on the box (scripts/profile_hops.py -> gpurun_out/prof/), and the bench's launch list.
mkdir -p gpurun_out/prof
cp profiles/spmm_traffic.json gpurun_out/prof/spmm_traffic.json
if [ "$1" == "--bench" ]; then
  python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02.log 2>&1; echo bench=$?
  tail -1 gpurun_out/bench_r02.log | cut -c1-3000
fi
NCU="ncu --set full --clock-control none -k regex:spmm_hop"
SB="python scripts/spmm_bench.py --K 1 --reps 1 --warmup 0"
SUM="python scripts/profile_hops.py --outdir gpurun_out/prof"
run() {   # tag, keys, widths, elem, spmm_bench args...
  local tag=$1 keys=$2 widths=$3 elem=$4; shift 4
  $NCU -o /tmp/$tag -f $SB --widths $widths "$@" > gpurun_out/ncu_$tag.log 2>&1; echo $tag=$?
  $SUM --rep /tmp/$tag.ncu-rep --tag $tag --keys $keys --widths $widths --elem $elem --note "spmm_bench.py $*" \
      >> gpurun_out/ncu_$tag.log 2>&1; echo sum_$tag=$?
  rm -f /tmp/$tag.ncu-rep
}
run r02_hops_orkut orkut/P1/f32,orkut/P2/f32,orkut/P4/f32,orkut/P8/f32 512,256,128,64 4 --config orkut --reorder
run r02_hops_reddit reddit/P1/f32,reddit/P2/f32,reddit/P4/f32,reddit/P8/f32 44,24,12,8 4 --config reddit
run r02_hops_products products/P1/f32,products/P2/f32,products/P4/f32,products/P8/f32 48,24,12,8 4 --config products --reorder
run r02_hops_papers papers/P1/bf16,papers/P2/bf16,papers/P4/bf16,papers/P8/bf16 128,64,32,16 2 --config papers --dtype bf16 --reorder
run r02_hops_papers_bwd papers_bwd/P1/bf16,papers_bwd/P8/bf16 128,16 2 --config papers --dtype bf16 --reorder --bwd
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/r02_reddit_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-hbm-leg > gpurun_out/ncu_ll.log 2>&1; echo ll=$?
ls -la gpurun_out/prof
