for st in 0 1; do
  export NTP_SPMM_STAGE=$st
  python scripts/spmm_bench.py --config reddit --widths 44,24,12,8 --K 2 --reps 10 | cut -c1-100
  python scripts/spmm_bench.py --config products --reorder --widths 48,12 --K 2 --reps 10 | cut -c1-100
  python scripts/spmm_bench.py --config papers --dtype bf16 --reorder --widths 128,16 --K 1 --reps 3 | cut -c1-100
done
NTP_SPMM_STAGE=1 python -m pytest tests/test_gpu_propagate.py -x -q 2>&1 | tail -2
