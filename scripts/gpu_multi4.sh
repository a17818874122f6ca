# 4-GPU box: multi-GPU parity (mp_check via pytest), papers and reddit epochs at N = 2 / 4
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name --format=csv
timeout 1800 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/multi_tests.log 2>&1; echo multi=$?
tail -3 gpurun_out/multi_tests.log
run() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n "$@"; }
run 4 --config papers --steps 5 --warmup 3 --no-e2e > gpurun_out/papers_n4.log 2>&1; echo p4=$?
tail -1 gpurun_out/papers_n4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['phase_ms'])"
run 2 --config papers --steps 5 --warmup 3 --no-e2e > gpurun_out/papers_n2.log 2>&1; echo p2=$?
tail -1 gpurun_out/papers_n2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['phase_ms'])"
for n in 2 4; do run $n --steps 10 --warmup 3 > gpurun_out/reddit_n$n.log 2>&1; echo r$n=$?
tail -1 gpurun_out/reddit_n$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e'], d['phase_ms'])"; done
