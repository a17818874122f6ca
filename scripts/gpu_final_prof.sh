#!/bin/bash
# Round-2 final measurement pass (1 GPU): products-shape bench line, then every hop variant under ncu
# (scripts/gpu_profile_hops.sh) and the bench's launch list.
mkdir -p gpurun_out/prof
python bench.py --config products --steps 5 --warmup 3 --no-hbm-leg > gpurun_out/products_N1.log 2>&1; echo products=$?
tail -1 gpurun_out/products_N1.log | cut -c1-400
bash scripts/gpu_profile_hops.sh
