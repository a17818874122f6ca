mkdir -p gpurun_out/ce
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for cfgname in head_dir tiny_dir; do
  timeout 500 $R --nproc-per-node 2 --master-port 29717 tests/mp_check.py $cfgname > gpurun_out/ce/mp_$cfgname.log 2>&1; echo mp_$cfgname=$?
  grep -h "MP OK\|MP FAIL" gpurun_out/ce/mp_$cfgname.log | head -3
done
for mode in "" "--overlap --chunks 4" "--overlap --chunks 4 --layouts p2p"; do
  timeout 600 $R --nproc-per-node 2 --master-port 29721 bench.py --gpus 2 --config papers --steps 3 --warmup 3 --no-e2e --no-hbm-leg $mode > gpurun_out/ce/papers.log 2>&1; echo "papers [$mode]"=$?
  tail -1 gpurun_out/ce/papers.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config']['layouts'], d['phase_ms'])"
done
