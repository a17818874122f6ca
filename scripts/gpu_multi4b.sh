mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/multi_tests.log 2>&1; echo multi=$?
tail -2 gpurun_out/multi_tests.log; grep -m4 "MP FAIL" gpurun_out/multi_tests.log
run() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n "$@"; }
python bench.py --engine coupled --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/coupled_n1.log 2>&1; echo c1=$?
tail -1 gpurun_out/coupled_n1.log | cut -c1-1500
for n in 2 4; do run $n --engine coupled --steps 5 --warmup 3 --no-e2e > gpurun_out/coupled_n$n.log 2>&1; echo c$n=$?
tail -1 gpurun_out/coupled_n$n.log | cut -c1-1500; done
timeout 900 python bench.py --config papers --steps 5 --warmup 3 --no-e2e > gpurun_out/papers_n1.log 2>&1; echo p1=$?
tail -1 gpurun_out/papers_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['phase_ms'], d['roofline']['frac'], d['roofline']['bytes_model'])"
run 4 --config papers --steps 5 --warmup 3 --no-e2e > gpurun_out/papers_n4.log 2>&1; echo p4=$?
tail -1 gpurun_out/papers_n4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['phase_ms'], d['roofline']['frac'])"
