mkdir -p gpurun_out
for o in 0 1 2; do NTP_SPMM_OCC=$o python scripts/spmm_bench.py --config reddit --widths 44,24,12,8 --K 2 --reps 10; done > gpurun_out/occ.jsonl 2>&1
for o in 1 2; do NTP_SPMM_OCC=$o timeout 900 python -m pytest tests/test_gpu_propagate.py -x -q -m gpu 2>&1 | tail -2; done
cat gpurun_out/occ.jsonl | cut -c1-200
