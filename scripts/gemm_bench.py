#!/usr/bin/env python
"""tcgen05 3xTF32 GEMM timing on the MLP shapes of a workload (development tool), next to cuBLAS
fp32 SGEMM (TF32 off) for context, plus the max relative error against an fp64 product.

    python scripts/gemm_bench.py --config reddit --reps 20
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


def r4(x):
    return (x + 3) // 4 * 4


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="reddit")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    cfg = synth.get_config(args.config)
    V, d, h, C = cfg.n, cfg.d_in, cfg.hid, cfg.C
    torch.backends.cuda.matmul.allow_tf32 = False
    ctx = ntp.Context()
    g = torch.Generator(device="cuda").manual_seed(0)

    def mat(r, c):
        return torch.randn(r, r4(c), device="cuda", generator=g)[:, :c]

    X, W0, H1, W1, dL = mat(V, d), mat(d, h), mat(V, h), mat(h, C), mat(V, C)
    shapes = [  # name, A, B, trans_a, trans_b, M, N, relu
        ("X.W0", X, W0, False, False, V, h, True),
        ("H1.W1", H1, W1, False, False, V, C, False),
        ("H1^T.dL", H1, dL, True, False, h, C, False),
        ("dL.W1^T", dL, W1, False, True, V, h, False),
        ("X^T.dH1", X, H1, True, False, d, h, False),
    ]
    for name, A, B, ta, tb, M, N, relu in shapes:
        Cm = torch.empty(M, r4(N), device="cuda")[:, :N]
        f = lambda: ctx.gemm(A, B, Cm, trans_a=ta, trans_b=tb, relu=relu)  # noqa: E731
        opA = A.t() if ta else A
        opB = B.t() if tb else B
        K = opA.shape[1]
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        e0.record()
        for _ in range(args.reps):
            ref32 = opA @ opB
        e1.record()
        torch.cuda.synchronize()
        ms_cublas = e0.elapsed_time(e1) / args.reps
        rows = torch.arange(0, M, max(1, M // 512), device="cuda")
        ref = opA[rows].double() @ opB.double()
        if relu:
            ref = ref.clamp_min(0)
        err = ((Cm[rows].double() - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item()
        flops = 2.0 * M * N * K
        byts = 4.0 * (M * K + K * N + M * N)
        print(json.dumps(dict(gemm=name, M=M, N=N, K=K, ms=round(ms, 4), cublas_fp32_ms=round(ms_cublas, 4),
                              tflops_3x=round(3 * flops / ms / 1e9, 1), min_GBps=round(byts / ms / 1e6, 1),
                              rel_err=err)), flush=True)
        del ref32


if __name__ == "__main__":
    main()
