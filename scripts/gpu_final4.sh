mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/multi_tests.log 2>&1; echo multi=$?
tail -1 gpurun_out/multi_tests.log; grep -m3 "MP FAIL" gpurun_out/multi_tests.log
run() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n "$@"; }
pj() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],2), round(d['value'],1), (d.get('e2e') or {}).get('ms_per_step'), d['load_balance']['max_over_min'], {k: round(v,1) for k,v in d['phase_ms'].items()})"; }
for n in 2 4; do run $n --steps 10 --warmup 3 > gpurun_out/final_reddit_n$n.log 2>&1; echo r$n=$?; pj < gpurun_out/final_reddit_n$n.log; done
for n in 2 4; do run $n --config papers --steps 5 --warmup 3 --no-e2e > gpurun_out/final_papers_n$n.log 2>&1; echo p$n=$?; pj < gpurun_out/final_papers_n$n.log; done
run 4 --config products --steps 10 --warmup 3 --no-e2e > gpurun_out/final_products_n4.log 2>&1; echo pr4=$?; pj < gpurun_out/final_products_n4.log
run 4 --engine dp --steps 10 --warmup 3 --no-e2e > gpurun_out/final_dp_n4.log 2>&1; echo dp4=$?; pj < gpurun_out/final_dp_n4.log
