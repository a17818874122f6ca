#!/bin/bash
# (gpurun --gpus 4) GAT lines at N = 1 / 2 / 4, the dual hop under ncu, mp_check's GAT step on 4 GPUs
O=gpurun_out/gatf
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python bench.py --engine gat --steps 5 --warmup 3 --no-hbm-leg > $O/gat_N1.log 2>&1; echo gat1=$?
tail -1 $O/gat_N1.log > $O/gat_N1.json
for N in 2 4; do
  timeout 600 $R --nproc-per-node $N --master-port 2998$N bench.py --gpus $N --engine gat --steps 5 --warmup 3 --no-hbm-leg > $O/gat_N$N.log 2>&1; echo gat$N=$?
  tail -1 $O/gat_N$N.log > $O/gat_N$N.json
done
python -c "
import json
for n in (1, 2, 4):
    d = json.load(open('$O/gat_N%d.json' % n)); print(n, round(d['ms_per_step'], 3), round(d['hop_ms'], 3), d['phase_ms'])
"
bash scripts/gpu_prof_gat.sh
timeout 900 $R --nproc-per-node 4 --master-port 29989 tests/mp_check.py small_dir > $O/mp4.log 2>&1; echo mp4=$?
grep -h "MP OK\|MP FAIL" $O/mp4.log | head -3
