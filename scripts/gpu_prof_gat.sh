#!/bin/bash
# ncu --set full of the GAT epoch's dual hops (forward and transposed) and the unweighted Reddit hop, with
# the stall breakdown, summarised on the box into gpurun_out/prof_gat/.
O=gpurun_out/prof_gat
mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:spmm_hop_kernel --launch-skip 4 --launch-count 4 \
    -o /tmp/gat_hops -f python bench.py --engine gat --steps 1 --warmup 1 --no-hbm-leg > $O/ncu.log 2>&1; echo ncu=$?
ncu -i /tmp/gat_hops.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null; echo raw=$?
ncu -i /tmp/gat_hops.ncu-rep --page details --csv > $O/details.csv 2>/dev/null; echo det=$?
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/prof_gat/raw.csv")))
hdr, units = rows[0], rows[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum"]
stall = [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled") or h.startswith("smsp__pcsamp_warps_issue_stalled")]
for r in rows[2:]:
    print({k: r[hdr.index(k)][:60] for k in keys if k in hdr})
    st = sorted(((float(r[hdr.index(h)].replace(",", "") or 0), h) for h in stall if r[hdr.index(h)] not in ("", "n/a")), reverse=True)[:8]
    print("  stalls:", [(round(v, 1), h.split("stalled_")[-1]) for v, h in st])
PY
rm -f /tmp/gat_hops.ncu-rep
