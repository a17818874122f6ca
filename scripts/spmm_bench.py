#!/usr/bin/env python
"""SpMM hop microbenchmark (development tool): times ntp_propagate_fwd/bwd on a config's
graph at several slice widths and prints ms per hop and derived throughputs.

    python scripts/spmm_bench.py --config reddit --widths 44,24,12,8 --K 1 --reps 10
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2412_20379_b200 import ntp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="reddit")
    ap.add_argument("--widths", default="44,24,12,8")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--K", type=int, default=1)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--bwd", action="store_true")
    ap.add_argument("--reorder", action="store_true")
    ap.add_argument("--warmup", type=int, default=3, help="untimed calls per width (0 under ncu: one launch each)")
    ap.add_argument("--pitch", type=int, default=0, help="row pitch in elements (>= width; 0: dense rows)")
    args = ap.parse_args()
    cfg = synth.get_config(args.config)
    ctx = ntp.Context()
    ctx.generate_rmat(cfg.n, cfg.scale, cfg.m_raw, synth.rmat_thresholds(*cfg.abc), cfg.seed, cfg.symmetric,
                      reorder=args.reorder)
    n, nnz, sym = ctx.graph_info()
    tdt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    esz = 2 if args.dtype == "bf16" else 4
    out = []
    for d in [int(x) for x in args.widths.split(",")]:
        ld = max(args.pitch, d)
        H = torch.randn(n, ld, device="cuda").to(tdt)[:, :d]
        Z = torch.empty(n, ld, device="cuda", dtype=tdt)[:, :d]
        f = ctx.propagate_bwd if args.bwd else ctx.propagate_fwd
        for _ in range(args.warmup):
            f(H, Z, args.K, 1.0, 0.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            f(H, Z, args.K, 1.0, 0.0)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps / args.K
        r = d * esz
        rs = -(-r // 32) * 32
        rec = dict(config=args.config, d=d, pitch=ld, dtype=args.dtype, ms_per_hop=round(ms, 4),
                   GE_per_s=round(nnz * d / (ms * 1e-3) / 1e9, 1),
                   gather_TBps=round((nnz + n) * rs / (ms * 1e-3) / 1e12, 2),
                   edges_per_ns=round(nnz / (ms * 1e6), 2), nnz=nnz, n=n, reorder=args.reorder,
                   env={k: v for k, v in os.environ.items() if k.startswith("NTP_")})
        out.append(rec)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
