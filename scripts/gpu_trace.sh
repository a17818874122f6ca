R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $R --nproc-per-node 2 --master-port 29961 tests/mp_check.py head_dir > gpurun_out/mp_trace.log 2>&1; echo mp=$?
grep -h "MP OK\|MP FAIL\|Error\|error" gpurun_out/mp_trace.log | head -5
mkdir -p gpurun_out/trace
timeout 900 $R --nproc-per-node 2 --master-port 29962 bench.py --gpus 2 --config papers --steps 2 --warmup 3 --no-e2e --no-hbm-leg --overlap --chunks 4 --trace gpurun_out/trace/papers_N2_nccl > gpurun_out/trace/b1.log 2>&1; echo b1=$?
tail -1 gpurun_out/trace/b1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('overlap_trace'))"
timeout 900 $R --nproc-per-node 2 --master-port 29963 bench.py --gpus 2 --config papers --steps 2 --warmup 3 --no-e2e --no-hbm-leg --overlap --chunks 4 --layouts p2p --trace gpurun_out/trace/papers_N2_ce > gpurun_out/trace/b2.log 2>&1; echo b2=$?
tail -1 gpurun_out/trace/b2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('overlap_trace'))"
