"""NEXT-3 memory-efficient scheduling with host-resident inputs (NTP_M_HOST_STREAM): X_v stays in
pinned host memory and every vertex-row chunk is streamed through a 2-slot device ring right before the MLP
forward / dW0 kernels that read it.  Forced host chunking (NTP_HEAD_CHUNK) on small configs: the epochs are
bitwise those of the device-resident run with the same kernels (the fused dW0 kernel reads X whole, so the
device run here disables it), and match the oracle."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import oracle_graph, ntp_ctx_for

pytestmark = pytest.mark.gpu


def _epochs(name, dtype, host, epochs=3):
    from paper_2412_20379_b200 import ntp
    cfg = synth.get_config(name)
    ctx = ntp_ctx_for(name)
    X, y, m = synth.config_inputs(cfg)
    ldx = (cfg.d_in + 3) // 4 * 4
    if host:
        Xt = torch.zeros(cfg.n, ldx, dtype=torch.float32).pin_memory()[:, :cfg.d_in]
        Xt.copy_(torch.from_numpy(X))
    else:
        Xt = torch.from_numpy(X).cuda()
    yd, md = torch.from_numpy(y).cuda(), torch.from_numpy(m).cuda()
    W0, W1 = (torch.from_numpy(a).cuda() for a in synth.model_weights(cfg))
    model = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=cfg.K, gamma=cfg.gamma, alpha=cfg.alpha, lr=cfg.lr * 50,
                 dtype=dtype, chunks=1, flags=ntp.NTP_M_W1_AFTER_PROP)
    losses = [ctx.train_epoch(model, Xt, yd, md, W0, W1, host_stream=host)["loss"] for _ in range(epochs)]
    ctx.close()
    return losses, W0.cpu().numpy(), W1.cpu().numpy(), model


@pytest.mark.parametrize("name,dtype,chunk", [("tiny_dir", 0, 700), ("head_dir", 0, 1024), ("head_dir", 1, 999),
                                              ("head_sym", 1, 4096)])
def test_host_stream_epoch(name, dtype, chunk, monkeypatch):
    monkeypatch.setenv("NTP_HEAD_CHUNK", str(chunk))
    monkeypatch.setenv("NTP_WGRAD_FUSED", "0")
    a = _epochs(name, dtype, host=False)
    b = _epochs(name, dtype, host=True)
    assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    cfg = synth.get_config(name)
    X, y, m = synth.config_inputs(cfg)
    W0, W1 = synth.model_weights(cfg)
    ref, _, _ = oracle.model.train(oracle_graph(name), X, y, m, W0, W1, cfg.K, cfg.gamma, cfg.alpha, b[3]["lr"], 3)
    tol = (lambda r: 1e-4) if dtype == 0 else (lambda r: 2e-2 * abs(r))
    for x, r in zip(b[0], ref):
        assert abs(x - r) <= tol(r)


def test_host_stream_refuses_w1_before():
    from paper_2412_20379_b200 import ntp
    cfg = synth.get_config("tiny_sym")
    ctx = ntp_ctx_for("tiny_sym")
    X, y, m = synth.config_inputs(cfg)
    W0, W1 = (torch.from_numpy(a).cuda() for a in synth.model_weights(cfg))
    model = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=cfg.K, gamma=cfg.gamma, alpha=cfg.alpha, lr=0.1,
                 dtype=0, chunks=1, flags=0)
    with pytest.raises(RuntimeError):
        ctx.train_epoch(model, torch.from_numpy(X).pin_memory(), torch.from_numpy(y).cuda(), torch.from_numpy(m).cuda(),
                        W0, W1, host_stream=True)
    ctx.close()
