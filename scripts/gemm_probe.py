#!/usr/bin/env python
"""Development probe for the tcgen05 GEMM: identity x index-coded operands reveal layout bugs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_20379_b200 import ntp  # noqa: E402

ctx = ntp.Context()
M, N, K = 128, 32, 32
for ta in (False, True):
    for tb in (False, True):
        a = np.zeros((M, K), np.float32)
        a[:K, :K] = np.eye(K)                       # op(A) = [I; 0]
        b = (1000 * np.arange(N)[None, :] + np.arange(K)[:, None]).astype(np.float32)   # op(B)[k][n]
        A = torch.from_numpy(np.ascontiguousarray(a.T if ta else a)).cuda()
        B = torch.from_numpy(np.ascontiguousarray(b.T if tb else b)).cuda()
        C = torch.full((M, N), -1.0, device="cuda")
        ctx.gemm(A, B, C, trans_a=ta, trans_b=tb)
        torch.cuda.synchronize()
        c = C.cpu().numpy()
        ref = a.astype(np.float64) @ b.astype(np.float64)
        ok = np.abs(c - ref).max()
        print(f"ta={ta} tb={tb} maxerr={ok}")
        if ok > 1e-3:
            np.set_printoptions(linewidth=200)
            print(" C[0:10,0:6]=\n", c[0:10, 0:6])
            print(" C[30:34,0:3]=\n", c[30:34, 0:3])
        # random check
        rng = np.random.default_rng(0)
        a2 = rng.standard_normal((M, 64)).astype(np.float32)
        b2 = rng.standard_normal((64, N)).astype(np.float32)
        A2 = torch.from_numpy(np.ascontiguousarray(a2.T if ta else a2)).cuda()
        B2 = torch.from_numpy(np.ascontiguousarray(b2.T if tb else b2)).cuda()
        C2 = torch.zeros((M, N), device="cuda")
        ctx.gemm(A2, B2, C2, trans_a=ta, trans_b=tb)
        torch.cuda.synchronize()
        print(f"   random 128x32x64 maxerr {np.abs(C2.cpu().numpy() - a2.astype(np.float64) @ b2).max():.3e}")
