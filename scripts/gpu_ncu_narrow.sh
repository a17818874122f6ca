# ncu --set full of the hop kernel at slice widths 8 and 44 (Reddit graph) and of the pure gather probe
mkdir -p gpurun_out
nvcc -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -o /tmp/l2_probe scripts/l2_probe.cu
python scripts/spmm_bench.py --config reddit --widths 8 --K 1 --reps 2 > /dev/null 2>&1 || echo bench-fail
ncu --set full --import-source on --clock-control none -k regex:spmm_hop -s 3 -c 1 -o gpurun_out/hop_d8 -f \
    python scripts/spmm_bench.py --config reddit --widths 8 --K 1 --reps 2 > gpurun_out/ncu_d8.log 2>&1; echo n1=$?
ncu --set full --import-source on --clock-control none -k regex:spmm_hop -s 3 -c 1 -o gpurun_out/hop_d44 -f \
    python scripts/spmm_bench.py --config reddit --widths 44 --K 1 --reps 2 > gpurun_out/ncu_d44.log 2>&1; echo n2=$?
ncu --set full --import-source on --clock-control none -k regex:gather_kernel -s 1 -c 1 -o gpurun_out/probe_g32 -f \
    /tmp/l2_probe 232965 114082446 32 x > gpurun_out/ncu_probe.log 2>&1; echo n3=$?
ls -la gpurun_out
