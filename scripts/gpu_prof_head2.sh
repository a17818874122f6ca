mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:head_fused -s 2 -c 1 -o gpurun_out/head_s8c -f \
    python bench.py --config papers_slice8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_head.log 2>&1; echo nh=$?
