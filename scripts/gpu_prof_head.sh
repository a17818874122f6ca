# ncu --set full of the fused head (papers_slice8 proxy at P = 1: 13.9M rows x 128, C = 172) and the
# HBM-resident random-gather probe at 64-256 B rows (111M-row table)
mkdir -p gpurun_out
timeout 600 python bench.py --config papers_slice8 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/slice8.log 2>&1; echo s8=$?
tail -1 gpurun_out/slice8.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:head_fused -s 1 -c 1 -o gpurun_out/head_s8 -f \
    python bench.py --config papers_slice8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_head.log 2>&1; echo nh=$?
nvcc -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -o /tmp/l2_probe scripts/l2_probe.cu && \
  timeout 600 /tmp/l2_probe 111059956 400000000 64,128,256 x > gpurun_out/probe_hbm_wide.jsonl 2>&1; echo pr=$?
cat gpurun_out/probe_hbm_wide.jsonl
