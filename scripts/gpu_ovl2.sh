mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_epoch.py -x -q -m gpu > gpurun_out/epoch_tests.log 2>&1; echo etests=$?
tail -2 gpurun_out/epoch_tests.log
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/multi_tests.log 2>&1; echo multi=$?
tail -2 gpurun_out/multi_tests.log; grep -m4 "MP FAIL" gpurun_out/multi_tests.log
run() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n "$@"; }
run 2 --config papers --steps 5 --warmup 3 --no-e2e > gpurun_out/papers_n2.log 2>&1; echo p2=$?
tail -1 gpurun_out/papers_n2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'])"
for ch in 4 8; do run 2 --config papers --steps 5 --warmup 3 --no-e2e --overlap --chunks $ch > gpurun_out/papers_n2_ov$ch.log 2>&1; echo p2ov=$?
tail -1 gpurun_out/papers_n2_ov$ch.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'])"; done
