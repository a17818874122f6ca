"""Bulk-copy gather hop (spmm_hop_bulk_kernel: cp.async.bulk of whole row slices into a shared-memory ring,
used for rows of >= 1 KB) against the oracle, and BITWISE equal to the register-staged spmm_hop_kernel
on the same input (same per-column summation order: group (j - eb) mod 8, fixed butterfly), so results
stay independent of the slice width across the two kernels.  The selection switch NTP_SPMM_BULK is read
once per process, so each variant runs in its own subprocess."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth
from gpu_util import oracle_graph, assert_r10, cond_bound

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import synth
from gpu_util import ntp_ctx_for
name, d, dt, tr, K, reorder, out = {args!r}
cfg = synth.get_config(name)
ctx = ntp_ctx_for(name, reorder=reorder)
H = torch.from_numpy(synth.features(17, cfg.n, d)).cuda().to(torch.bfloat16 if dt == "bf16" else torch.float32)
Z = torch.empty_like(H)
(ctx.propagate_bwd if tr else ctx.propagate_fwd)(H, Z, K, cfg.gamma, cfg.alpha)
torch.cuda.synchronize()
np.save(out, Z.float().cpu().numpy())
"""


def _run(tmp_path, bulk, name, d, dt, tr, K, reorder=False, var="NTP_SPMM_BULK"):
    out = str(tmp_path / f"z_{var}_{bulk}_{name}_{d}_{dt}_{int(tr)}_{K}_{int(reorder)}.npy")
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"), args=(name, d, dt, tr, K, reorder, out))
    env = dict(os.environ)
    env[var] = str(bulk)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


@pytest.mark.parametrize("name,d,dt,tr,K,reorder", [
    ("dense_sym", 512, "f32", False, 3, False),     # 2 KB rows, hubs across units, alpha mix
    ("dense_dir", 256, "f32", True, 2, False),      # 1 KB rows, out-CSR
    ("small_dir", 1024, "bf16", False, 2, False),   # 2 KB bf16 rows, low degree
    ("small_appnp", 128, "f32", False, 3, True),    # 512 B rows (forced), reordered graph
])
def test_bulk_gather_bitwise_and_oracle(tmp_path, name, d, dt, tr, K, reorder):
    a = _run(tmp_path, 0, name, d, dt, tr, K, reorder)
    b = _run(tmp_path, 1, name, d, dt, tr, K, reorder)
    assert np.array_equal(a, b), f"bulk != register kernel: max diff {np.abs(a - b).max()}"
    cfg = synth.get_config(name)
    g = oracle_graph(name)
    H = synth.features(17, cfg.n, d)
    if dt == "bf16":
        import torch
        H = torch.from_numpy(H).to(torch.bfloat16).float().numpy()
    f = oracle.propagate.propagate_bwd if tr else oracle.propagate.propagate_fwd
    ref = f(g, H, K, cfg.gamma, cfg.alpha)
    den = cond_bound(g, H, K, cfg.gamma, cfg.alpha, tr)
    assert_r10(b, ref, den, 1e-5 if dt == "f32" else 2e-2, f"{name} bulk")
