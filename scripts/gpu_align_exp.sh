#!/bin/bash
# Reddit lines at N = 2 / 4 with the automatic slice padding vs plain 16-byte slices (gpurun --gpus 4)
O=gpurun_out/align
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  for A in auto 16; do
    timeout 600 $R --nproc-per-node $N --master-port 2993$N bench.py --gpus $N --steps 10 --warmup 3 --no-hbm-leg --slice-align $A > $O/reddit_N${N}_$A.log 2>&1
    tail -1 $O/reddit_N${N}_$A.log > $O/reddit_N${N}_$A.json
    python -c "import json; d=json.load(open('$O/reddit_N${N}_$A.json')); print('N=$N align $A', d['config']['d_s'], d['config'].get('slice_align'), round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['phase_ms'])"
  done
done
timeout 600 $R --nproc-per-node 4 --master-port 29939 bench.py --gpus 4 --engine gat --steps 5 --warmup 3 --no-hbm-leg > $O/gat_N4_auto.log 2>&1
tail -1 $O/gat_N4_auto.log > $O/gat_N4_auto.json; python -c "import json; d=json.load(open('$O/gat_N4_auto.json')); print('gat N=4 auto', d['config'].get('slice_align'), d['ms_per_step'])"
