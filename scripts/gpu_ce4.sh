mkdir -p gpurun_out/ce
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 500 $R --nproc-per-node 4 --master-port 29741 tests/mp_check.py head_dir > gpurun_out/ce/mp4_head_dir.log 2>&1; echo mp4=$?
grep -h "MP OK\|MP FAIL" gpurun_out/ce/mp4_head_dir.log | head -3
for mode in "--overlap --chunks 4 --layouts p2p" "--overlap --chunks 8 --layouts p2p"; do
  timeout 600 $R --nproc-per-node 4 --master-port 29731 bench.py --gpus 4 --config papers --steps 3 --warmup 3 --no-e2e --no-hbm-leg $mode > gpurun_out/ce/papers4.log 2>&1; echo "papers4 [$mode]"=$?
  tail -1 gpurun_out/ce/papers4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config']['layouts'], d['phase_ms'])"
  cp gpurun_out/ce/papers4.log "gpurun_out/ce/papers4_$(echo $mode | tr ' -' '__').log"
done
