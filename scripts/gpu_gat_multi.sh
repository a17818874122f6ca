#!/bin/bash
# (gpurun --gpus 4) GAT multi-rank parity (mp_check at 2 and 4 GPUs) and the GAT lines at N = 2 / 4
O=gpurun_out/gatm
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  timeout 900 $R --nproc-per-node $N --master-port 2999$N tests/mp_check.py small_dir > $O/mp$N.log 2>&1; echo mp$N=$?
  grep -h "MP OK\|MP FAIL" $O/mp$N.log | head -3
  timeout 600 $R --nproc-per-node $N --master-port 2990$N bench.py --gpus $N --engine gat --steps 5 --warmup 3 --no-hbm-leg > $O/gat_N$N.log 2>&1; echo gat$N=$?
  tail -1 $O/gat_N$N.log > $O/gat_N$N.json
  python -c "import json; d=json.load(open('$O/gat_N$N.json')); print($N, round(d['ms_per_step'],3), d['phase_ms'])"
done
