#!/usr/bin/env python
"""Summarise an `ncu --set full` capture of spmm_hop_kernel launches (one per slice width, from
scripts/spmm_bench.py --warmup 0 --reps 1 --K 1) into profiles/<tag>.md and profiles/spmm_traffic.json.

    python scripts/profile_hops.py --rep gpurun_out/r02_hops_papers.ncu-rep --tag r02_hops_papers \
        --keys papers/P1/bf16,papers/P2/bf16,papers/P4/bf16,papers/P8/bf16 --widths 128,64,32,16 --elem 2

Per launch: time, DRAM bytes (read + write), DRAM GB/s and its fraction of the measured copy peak
(MEASURED_PEAKS.json) and of 8 TB/s, L2 hit rate, L2 sector throughput, warps active, registers.
"""
import argparse
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum"]
SCALE = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--tag", required=True)
    ap.add_argument("--keys", required=True)
    ap.add_argument("--widths", required=True)
    ap.add_argument("--elem", type=int, default=4)
    ap.add_argument("--note", default="")
    ap.add_argument("--outdir", default=os.path.join(ROOT, "profiles"))
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        if "spmm_hop" not in r[hdr.index("Kernel Name")]:
            continue
        d = {}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                v = float(r[i].replace(",", "")) if r[i] not in ("", "n/a") else None
                if v is not None and units[i] in SCALE:
                    v *= SCALE[units[i]]
                d[w] = v
        recs.append(d)
    keys = args.keys.split(",")
    widths = [int(x) for x in args.widths.split(",")]
    assert len(recs) == len(keys), (len(recs), keys)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    os.makedirs(args.outdir, exist_ok=True)
    tj = os.path.join(args.outdir, "spmm_traffic.json")
    traffic = json.load(open(tj)) if os.path.exists(tj) else {}
    lines = [f"# {args.tag}: spmm_hop_kernel, ncu --set full --clock-control none (one launch per slice width)", "",
             args.note, "",
             "| key | d_s | row B | ms | DRAM GB/launch | DRAM GB/s | of measured peak | of 8 TB/s | L2 hit % | "
             "L2 sectors % peak | warps active % | LSU wavefronts % | regs |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for k, w, d in zip(keys, widths, recs):
        t = d["gpu__time_duration.sum"]
        b = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        gbs = b / t / 1e9
        traffic[k] = b
        lines.append(f"| {k} | {w} | {w * args.elem} | {t * 1e3:.2f} | {b / 1e9:.2f} | {gbs:.0f} | {gbs / peak:.2f} | "
                     f"{gbs / 8000:.2f} | {d.get('lts__t_sector_hit_rate.pct') or 0:.1f} | "
                     f"{d.get('lts__t_sectors.avg.pct_of_peak_sustained_elapsed') or 0:.1f} | "
                     f"{d.get('sm__warps_active.avg.pct_of_peak_sustained_active') or 0:.1f} | "
                     f"{d.get('l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed') or 0:.1f} | "
                     f"{int(d.get('launch__registers_per_thread') or 0)} |")
    lines.append("")
    lines.append(f"ncu times are cold-cache, serialised replays (compare against bench CUDA-event times for shares "
                 f"only). Measured copy peak {peak} GB/s (MEASURED_PEAKS.json).")
    open(os.path.join(args.outdir, args.tag + ".md"), "w").write("\n".join(lines) + "\n")
    json.dump(dict(sorted(traffic.items())), open(tj, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
