mkdir -p gpurun_out
nvidia-smi -L | wc -l
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/multi_tests.log 2>&1; echo multi=$?
tail -2 gpurun_out/multi_tests.log; grep -m3 "MP FAIL" gpurun_out/multi_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/final_reddit_n2.log 2>&1; echo r2=$?
tail -1 gpurun_out/final_reddit_n2.log | cut -c1-300
