mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2_probe scripts/l2_probe.cu
/tmp/l2_probe 232965 114082446 32,48,64,96,176,192 > gpurun_out/l2_probe_reddit.jsonl 2>&1; echo probe1=$?
/tmp/l2_probe 111059956 400000000 32,64 x > gpurun_out/l2_probe_papers.jsonl 2>&1; echo probe2=$?
python scripts/spmm_bench.py --config reddit --widths 44,24,12,8 --K 2 > gpurun_out/spmm_reddit.jsonl 2>&1; echo sb=$?
cat gpurun_out/l2_probe_reddit.jsonl gpurun_out/l2_probe_papers.jsonl gpurun_out/spmm_reddit.jsonl
