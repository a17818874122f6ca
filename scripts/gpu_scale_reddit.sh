#!/bin/bash
# (gpurun --gpus 4) the driver's scaling run on one box: bench.py at N = 1, 2, 4 back to back (default config)
O=gpurun_out/scale_final
mkdir -p $O
python bench.py --steps 10 --warmup 3 > $O/N1.log 2>&1; echo N1=$?
tail -1 $O/N1.log > $O/N1.json
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  timeout 900 $R --nproc-per-node $N --master-port 2987$N bench.py --gpus $N --steps 10 --warmup 3 > $O/N$N.log 2>&1; echo N$N=$?
  tail -1 $O/N$N.log > $O/N$N.json
done
python - <<'PY'
import json
rows = []
for n in (1, 2, 4):
    d = json.load(open(f"gpurun_out/scale_final/N{n}.json"))
    rows.append((n, d["ms_per_step"], d["value"], d["e2e"]["value"], d["roofline"]["frac"], d["clocks"]))
base = rows[0][2]
for n, ms, v, e, f, clk in rows:
    print(n, round(ms, 3), round(v), round(e), round(f, 3), "speedup", round(v / base, 2), clk)
PY
