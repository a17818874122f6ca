mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_ll.log 2>&1; echo ll=$?
ncu --set full --import-source on --clock-control none -k regex:spmm_hop -s 8 -c 2 -o gpurun_out/r01_spmm -f \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo full=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/papers_launches.csv \
    python bench.py --config papers --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/papers_ll.log 2>&1; echo pll=$?
