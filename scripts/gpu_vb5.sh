mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_propagate.py tests/test_gpu_epoch.py tests/test_gpu_multi.py tests/test_gpu_coupled.py -x -q -m gpu > gpurun_out/vb5_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/vb5_tests.log; grep -m3 "MP FAIL\|FAILED" gpurun_out/vb5_tests.log
run() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n "$@"; }
run 2 --steps 10 --warmup 3 > gpurun_out/reddit_n2.log 2>&1; echo r2=$?
tail -1 gpurun_out/reddit_n2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e']['ms_per_step'], d['phase_ms'])"
run 2 --config products --steps 10 --warmup 3 --no-e2e > gpurun_out/products_n2.log 2>&1; echo pr2=$?
tail -1 gpurun_out/products_n2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])"
