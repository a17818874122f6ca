#!/usr/bin/env python
"""Summarise an ncu launch list (gpu__time_duration per launch) and a --set full capture
into committed profile files.

    python scripts/profile_summary.py --launches gpurun_out/r01_launches.csv \
        --full gpurun_out/r01_spmm.ncu-rep --tag r02_reddit_P1 --steps 2 --key reddit/P1/f32
Writes profiles/<tag>_launches.md and updates profiles/spmm_traffic.json (dram bytes per launch).
The launch list is cold-cache and serialised: compare SHARES of the timed epochs, not absolutes.
"""
import argparse
import collections
import csv
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("ntp::", "").replace("(anonymous namespace)::", "")
    return name[:90]


def launches(path, steps):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    recs = []
    for r in rows[hi + 1:]:
        if len(r) != len(hdr):
            continue
        v = float(r[vi].replace(",", ""))
        if r[ui] == "us":
            v *= 1e3
        elif r[ui] == "ms":
            v *= 1e6
        recs.append((short(r[ki]), v))
    return recs


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum",
            "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
            "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "smsp__inst_executed.sum", "launch__grid_size"]
    res = []
    units = rows[1]
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for w in want:
            if w in hdr:
                i = hdr.index(w)
                val = float(r[i].replace(",", "")) if r[i] else None
                u = units[i]
                if val is not None and u in ("Mbyte", "Gbyte", "Kbyte", "byte"):
                    val *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
                    u = "byte"
                if val is not None and u in ("msecond", "ms", "usecond", "us", "nsecond", "ns"):
                    val *= {"msecond": 1e6, "ms": 1e6, "usecond": 1e3, "us": 1e3, "nsecond": 1, "ns": 1}[u]
                    u = "ns"
                d[w] = val
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--key")
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    md = [f"# {args.tag}\n", args.note + "\n" if args.note else ""]
    if args.launches:
        recs = launches(args.launches, 0)
        tot = collections.Counter()
        cnt = collections.Counter()
        for k, v in recs:
            tot[k] += v
            cnt[k] += 1
        s = sum(tot.values())
        md.append(f"## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`), {len(recs)} launches, "
                  f"{s / 1e6:.3f} ms total (cold-cache, serialised: shares matter)\n")
        md.append("| kernel | launches | total ms | share | avg us |\n|---|---|---|---|---|")
        for k, v in tot.most_common():
            md.append(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {v / s * 100:.1f}% | {v / cnt[k] / 1e3:.1f} |")
        md.append("")
    if args.full:
        fm = full_metrics(args.full)
        md.append("## `ncu --set full` of the dominant kernel (per launch)\n")
        keys = [k for k in fm[0] if k != "kernel"]
        md.append("| kernel | " + " | ".join(keys) + " |")
        md.append("|---" * (len(keys) + 1) + "|")
        for d in fm:
            md.append(f"| `{d['kernel']}` | " + " | ".join(f"{d[k]:.4g}" if isinstance(d[k], float) else str(d[k])
                                                          for k in keys) + " |")
        if args.key:
            path = os.path.join(ROOT, "profiles", "spmm_traffic.json")
            data = json.load(open(path)) if os.path.exists(path) else {}
            tr = [d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in fm
                  if d.get("dram__bytes_read.sum") is not None]
            data[args.key] = sum(tr) / len(tr)
            json.dump(data, open(path, "w"), indent=1, sort_keys=True)
            md.append(f"\nDRAM traffic per launch (read + write), mean of {len(tr)}: {sum(tr) / len(tr) / 1e6:.1f} MB "
                      f"-> profiles/spmm_traffic.json[{args.key!r}]")
    open(os.path.join(ROOT, "profiles", f"{args.tag}.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
