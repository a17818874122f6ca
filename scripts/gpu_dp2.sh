mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_epoch.py -x -q -m gpu -k "data_parallel or staged or head_bf16" > gpurun_out/dp_tests.log 2>&1; echo t1=$?
tail -3 gpurun_out/dp_tests.log
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/multi_tests.log 2>&1; echo multi=$?
tail -2 gpurun_out/multi_tests.log; grep -m4 "MP FAIL" gpurun_out/multi_tests.log
run() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n "$@"; }
pj() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['engine'], d['ms_per_step'], d['load_balance'], d['phase_ms']['prop_fwd'])"; }
for e in decoupled dp; do run 2 --engine $e --steps 10 --warmup 3 --no-e2e > gpurun_out/reddit2_$e.log 2>&1; echo $e=$?; pj < gpurun_out/reddit2_$e.log; done
python bench.py --engine dp --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/reddit1_dp.log 2>&1; echo dp1=$?; pj < gpurun_out/reddit1_dp.log
