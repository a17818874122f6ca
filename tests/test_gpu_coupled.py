"""NEXT-1 on the GPU: the naive (coupled) tensor-parallel epoch (ntp_train_epoch_coupled) against the
coupled-GCN oracle (oracle/coupled.py): per-epoch loss within 1e-4 (fp32 storage) / 2e-2 relative
(bf16), weights after the SGD steps, and the report's layout-change / hop counts."""
import numpy as np
import pytest
import torch

import synth
from oracle import coupled
from gpu_util import oracle_graph, ntp_ctx_for

pytestmark = pytest.mark.gpu


def _weights(cfg, widths):
    return [synth.glorot(cfg.seed, widths[i], widths[i + 1], 100_000 * (i + 1)) for i in range(len(widths) - 1)]


def _run(name, widths, epochs, dtype=0, reorder=False):
    cfg = synth.get_config(name)
    ctx = ntp_ctx_for(name, reorder=reorder)
    X, y, m = synth.config_inputs(cfg)
    Ws = _weights(cfg, widths)
    lr = cfg.lr * 50
    Wd = [torch.from_numpy(W).cuda() for W in Ws]
    Xd, yd, md = (torch.from_numpy(a).cuda() for a in (X, y, m))
    losses, reps = [], []
    for _ in range(epochs):
        rep = ctx.train_epoch_coupled(widths, lr, Xd, yd, md, Wd, dtype=dtype)
        losses.append(rep["loss"])
        reps.append(rep)
    ref_losses, rWs = coupled.train(oracle_graph(name), X, y, m, Ws, lr, epochs)
    ctx.close()
    return losses, [W.cpu().numpy() for W in Wd], reps, ref_losses, rWs


@pytest.mark.parametrize("name,mid", [("tiny_sym", (16,)), ("tiny_dir", (20, 12)), ("small_appnp", (32,)),
                                      ("cora", (64,)), ("head_dir", (40, 24))])
def test_coupled_epoch_parity_fp32(name, mid):
    cfg = synth.get_config(name)
    widths = (cfg.d_in, *mid, cfg.C)
    losses, Ws, reps, ref_losses, rWs = _run(name, widths, 3)
    for e, (a, b) in enumerate(zip(losses, ref_losses)):
        assert abs(a - b) <= 1e-4, f"epoch {e}: gpu {a} oracle {b}"
    for got, ref in zip(Ws, rWs):
        assert np.abs(got - ref).max() <= 1e-4 * max(1.0, np.abs(ref).max())
    L = len(widths) - 1
    assert all(r["layout_changes"] == 0 and r["bytes_sent"] == 0 for r in reps)     # one GPU: local
    assert all(r["hops"] == 2 * L - 1 for r in reps)                                 # L forward, L-1 backward


@pytest.mark.parametrize("name", ["tiny_dir", "small_dir"])
def test_coupled_epoch_bf16_and_reordered(name):
    cfg = synth.get_config(name)
    widths = (cfg.d_in, 24, cfg.C)
    losses, _, _, ref_losses, _ = _run(name, widths, 2, dtype=1, reorder=True)
    for a, b in zip(losses, ref_losses):
        assert abs(a - b) <= 2e-2 * abs(b)
