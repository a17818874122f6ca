ncu --set full --import-source on --clock-control none -k regex:spmm_stream -s 3 -c 1 -o gpurun_out/stream_d8 -f \
    python scripts/spmm_bench.py --config reddit --widths 8 --K 1 --reps 2 > gpurun_out/ncu_st.log 2>&1; echo n1=$?
