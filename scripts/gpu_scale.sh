#!/bin/bash
# Multi-GPU pass on one node (gpurun --gpus 4): mp_check on 4 GPUs, then the bench at N = 2 and 4 (Reddit
# line with the Orkut HBM leg), the papers epoch at N = 4 and the GAT epoch at N = 4.
mkdir -p gpurun_out/scale
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/scale/multi4.log 2>&1; echo multi=$?
tail -2 gpurun_out/scale/multi4.log; grep -h "MP OK\|MP FAIL" gpurun_out/scale/multi4.log | head
for N in 2 4; do
  timeout 600 $R --nproc-per-node $N --master-port 2960$N bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/scale/bench_N$N.log 2>&1; echo bench$N=$?
  tail -1 gpurun_out/scale/bench_N$N.log | cut -c1-300
done
timeout 900 $R --nproc-per-node 4 --master-port 29611 bench.py --gpus 4 --config papers --steps 3 --warmup 3 --no-e2e --no-hbm-leg > gpurun_out/scale/papers_N4.log 2>&1; echo papers4=$?
tail -1 gpurun_out/scale/papers_N4.log | cut -c1-300
timeout 600 $R --nproc-per-node 4 --master-port 29612 bench.py --gpus 4 --engine gat --steps 5 --warmup 3 > gpurun_out/scale/gat_N4.log 2>&1; echo gat4=$?
tail -1 gpurun_out/scale/gat_N4.log | cut -c1-300
