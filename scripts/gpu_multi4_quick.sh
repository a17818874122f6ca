#!/bin/bash
# 4-GPU check after kernel changes: GAT and Reddit lines at N = 4 (JSON under gpurun_out/m4/)
O=gpurun_out/m4
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $R --nproc-per-node 4 --master-port 29811 bench.py --gpus 4 --engine gat --steps 5 --warmup 3 --no-hbm-leg > $O/gat_N4.log 2>&1; echo gat4=$?
tail -1 $O/gat_N4.log > $O/gat_N4.json; python -c "import json; d=json.load(open('$O/gat_N4.json')); print(d['ms_per_step'], d['phase_ms'], d['clocks'])"
timeout 600 $R --nproc-per-node 4 --master-port 29812 bench.py --gpus 4 --steps 10 --warmup 3 > $O/reddit_N4.log 2>&1; echo reddit4=$?
tail -1 $O/reddit_N4.log > $O/reddit_N4.json; python -c "import json; d=json.load(open('$O/reddit_N4.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['clocks'])"
