mkdir -p gpurun_out
run() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n "$@"; }
pj() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], round(d['value'],1), d['phase_ms'], round(d['roofline']['frac'],3))"; }
for n in 2 4; do
run $n --config papers --steps 5 --warmup 3 --no-e2e > gpurun_out/papers_n$n.log 2>&1; echo p$n=$?; pj < gpurun_out/papers_n$n.log
run $n --config papers --steps 5 --warmup 3 --no-e2e --overlap --chunks 4 > gpurun_out/papers_n${n}_ov.log 2>&1; echo p${n}ov=$?; pj < gpurun_out/papers_n${n}_ov.log
done
for n in 2 4; do run $n --steps 10 --warmup 3 > gpurun_out/reddit_n$n.log 2>&1; echo r$n=$?; pj < gpurun_out/reddit_n$n.log; done
