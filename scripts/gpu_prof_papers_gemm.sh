mkdir -p gpurun_out/gp
ncu --set full --clock-control none -k regex:gemm_tf32x3 --launch-count 2 -o /tmp/gp -f python bench.py --config papers --steps 1 --warmup 1 --no-e2e --no-hbm-leg --no-cpu-baseline > gpurun_out/gp/ncu.log 2>&1; echo ncu=$?
ncu -i /tmp/gp.ncu-rep --page raw --csv > gpurun_out/gp/raw.csv 2>/dev/null
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/gp/raw.csv")))
hdr = rows[0]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size"]
stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled")]
for r in rows[2:]:
    print({k: r[hdr.index(k)][:70] for k in keys if k in hdr})
    st = sorted(((float(r[hdr.index(h)].replace(",", "") or 0), h) for h in stall if r[hdr.index(h)] not in ("", "n/a")), reverse=True)[:8]
    print("  stalls:", [(int(v), h.split("stalled_")[-1]) for v, h in st])
PY
rm -f /tmp/gp.ncu-rep
