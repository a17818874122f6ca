#!/bin/bash
# End-of-round multi-GPU pass (gpurun --gpus 4): the multi-rank parity suite, then every bench line at
# N = 2 and 4 (Reddit line + Orkut HBM leg, products, papers with NCCL and with the copy-engine overlap,
# the GAT epoch, the coupled baseline) and the reference arm under torchrun.  JSON lines land in
# gpurun_out/multi_final/.
O=gpurun_out/multi_final
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_multi.py -q > $O/pytest_multi.log 2>&1; echo pytest_multi=$?
tail -2 $O/pytest_multi.log; grep -h "MP OK\|MP FAIL" $O/pytest_multi.log | head -20
run() {   # name nproc port args...
  local name=$1 n=$2 port=$3; shift 3
  timeout 900 $R --nproc-per-node $n --master-port $port bench.py --gpus $n "$@" > $O/$name.log 2>&1
  echo "$name rc=$?"
  tail -1 $O/$name.log > $O/$name.json
  python - "$O/$name.json" <<'EOF'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read())
except Exception as e:
    print("  no JSON line:", e); sys.exit(0)
keys = ("ms_per_step", "value", "unit")
print("  ", {k: d.get(k) for k in keys}, "e2e", (d.get("e2e") or {}).get("value"),
      "clocks", d.get("clocks"), "parity", (d.get("parity") or {}).get("pass"))
if d.get("hbm_leg"):
    h = d["hbm_leg"]
    print("   hbm_leg", h.get("ms_per_step"), h.get("roofline", {}).get("frac"))
if d.get("a2a_standalone"):
    print("   a2a", d["a2a_standalone"])
EOF
}
for N in 2 4; do
  run reddit_N$N $N 2970$N --steps 10 --warmup 3
  run products_N$N $N 2971$N --config products --steps 5 --warmup 3 --no-e2e --no-hbm-leg
  run gat_N$N $N 2972$N --engine gat --steps 5 --warmup 3 --no-hbm-leg
  run papers_N$N $N 2973$N --config papers --steps 3 --warmup 3 --no-e2e --no-hbm-leg
  run papers_ce_N$N $N 2974$N --config papers --steps 3 --warmup 3 --no-e2e --no-hbm-leg --overlap --chunks 4 --layouts p2p
done
run coupled_N4 4 29751 --engine coupled --steps 5 --warmup 3 --no-hbm-leg --no-e2e
run reference_N2 2 29752 --impl reference --steps 2 --warmup 1
run dp_N4 4 29753 --engine dp --steps 5 --warmup 3 --no-hbm-leg --no-e2e
