"""Adversarial graph structures for the hop kernels (a4/a8) vs the oracle, through the C ABI.

The R-MAT configs of the other tests never produce these shapes: a destination row with 150K in-arcs that
spans ~150 merge-path units (one fix-up chain over all of them), every arc gathering the same source row,
hub rows among thousands of empty rows, a triangular degree ramp, and graphs of one to three vertices.
Each runs forward and backward, fp32 (register kernel at 32 / 176 B rows, bulk-copy gather at 1 KB rows)
and bf16, with the APPNP mix on, against oracle/propagate.py under reading R10's bound."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import cond_bound, assert_r10

pytestmark = pytest.mark.gpu


def _arcs(kind):
    rng = np.random.default_rng(7)
    if kind == "star_in":        # row 0 has n-1 in-arcs
        n = 150_001
        src, dst = np.arange(1, n), np.zeros(n - 1, np.int64)
    elif kind == "star_out":     # every row gathers row 0
        n = 60_001
        src, dst = np.zeros(n - 1, np.int64), np.arange(1, n)
    elif kind == "hubs_sparse":  # 5 hubs of 10K in-arcs among mostly empty rows
        n = 20_000
        hubs = np.array([3, 4_999, 5_000, 12_345, 19_999])
        src = [rng.integers(0, n, 10_000) for _ in hubs]
        dst = [np.full(10_000, h) for h in hubs]
        rows = rng.choice(n, 2_000, replace=False)
        src.append(rng.integers(0, n, rows.size * 2))
        dst.append(np.repeat(rows, 2))
        src, dst = np.concatenate(src), np.concatenate(dst)
    elif kind == "ramp":         # row v has v in-arcs (0 .. 1999)
        n = 2_000
        dst = np.repeat(np.arange(n), np.arange(n))
        src = np.concatenate([rng.choice(n, v, replace=False) for v in range(n)])
    elif kind == "one":
        n = 1
        src, dst = np.array([], np.int64), np.array([], np.int64)
    elif kind == "two":
        n = 2
        src, dst = np.array([0]), np.array([1])
    elif kind == "k3":
        n = 3
        src = np.array([0, 0, 1, 1, 2, 2])
        dst = np.array([1, 2, 0, 2, 0, 1])
    else:
        raise ValueError(kind)
    return n, np.asarray(src, np.int64), np.asarray(dst, np.int64)


def _case(kind, d, dtype, transposed, reorder=False, K=2, gamma=0.9, alpha=0.1):
    from paper_2412_20379_b200 import ntp
    n, src, dst = _arcs(kind)
    g = oracle.graph.build_graph(src, dst, n, symmetric=False)
    ctx = ntp.Context()
    ctx.build_graph(src, dst, n, symmetric=False, reorder=reorder)
    rp, col, _ = ctx.copy_csr(False)
    assert np.array_equal(rp, g.row_ptr) and np.array_equal(col, g.col), f"{kind}: CSR mismatch"
    H = synth.features(31 + d, n, d)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    Hd = torch.from_numpy(H).to(tdt).cuda()
    Zd = torch.full_like(Hd, 7.0)
    (ctx.propagate_bwd if transposed else ctx.propagate_fwd)(Hd, Zd, K, gamma, alpha)
    torch.cuda.synchronize()
    Hx = Hd.double().cpu().numpy()                     # the operand the GPU saw (bf16-rounded for bf16)
    f = oracle.propagate.propagate_bwd if transposed else oracle.propagate.propagate_fwd
    ref = f(g, Hx, K, gamma, alpha)
    den = cond_bound(g, Hx, K, gamma, alpha, transposed)
    tol = 2e-2 if dtype == "bf16" else 1e-5
    assert_r10(Zd.double().cpu().numpy(), ref, den, tol, f"{kind} d={d} {dtype} T={transposed} reorder={reorder}")
    ctx.close()


@pytest.mark.parametrize("transposed", [False, True])
@pytest.mark.parametrize("kind", ["star_in", "star_out", "hubs_sparse", "ramp", "one", "two", "k3"])
@pytest.mark.parametrize("d", [8, 44])
def test_adversarial_fp32(kind, d, transposed):
    _case(kind, d, "f32", transposed)


@pytest.mark.parametrize("transposed", [False, True])
@pytest.mark.parametrize("kind", ["star_in", "hubs_sparse", "ramp"])
def test_adversarial_bulk_rows(kind, transposed):
    """1 KB rows: the bulk-copy gather (one CTA per unit, producer warp + shared-memory ring)."""
    _case(kind, 256, "f32", transposed)


@pytest.mark.parametrize("kind", ["star_in", "star_out", "hubs_sparse", "k3"])
def test_adversarial_bf16(kind):
    _case(kind, 16, "bf16", False)


@pytest.mark.parametrize("kind", ["star_in", "hubs_sparse", "ramp"])
def test_adversarial_reordered(kind):
    _case(kind, 44, "f32", False, reorder=True)
