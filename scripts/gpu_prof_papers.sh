# ncu evidence for the HBM-bound shapes: launch list of the papers N=1 epoch, --set full of the hop at
# the P=1 / P=8 slice widths (papers, bf16, reordered) and of the products hop (fp32, reordered)
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/papers_launches.csv \
    python bench.py --config papers --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/papers_ll.log 2>&1; echo ll=$?
for w in 128 16; do
ncu --set full --import-source on --clock-control none -k regex:spmm_hop -s 3 -c 1 -o gpurun_out/papers_hop_d$w -f \
    python scripts/spmm_bench.py --config papers --dtype bf16 --reorder --widths $w --K 1 --reps 1 > gpurun_out/ncu_papers_d$w.log 2>&1; echo p$w=$?
done
ncu --set full --import-source on --clock-control none -k regex:spmm_hop -s 3 -c 1 -o gpurun_out/products_hop_d48 -f \
    python scripts/spmm_bench.py --config products --reorder --widths 48 --K 1 --reps 1 > gpurun_out/ncu_products.log 2>&1; echo pr=$?
python scripts/spmm_bench.py --config papers --dtype bf16 --reorder --widths 128,64,32,16 --K 2 --reps 3 > gpurun_out/papers_widths.jsonl 2>&1; echo pw=$?
ls -la gpurun_out
