"""The torch (device) copy of the input formulas equals the numpy one bit for bit (SURVEY §8(d)
synthetic input spec); the bench generates papers-scale inputs with it."""
import numpy as np
import pytest
import torch

import synth


@pytest.mark.parametrize("name,row0,rows", [("cora", 0, 300), ("head_dir", 1000, 700), ("reddit", 232_000, 965),
                                            ("papers", 111_059_000, 956)])
def test_config_inputs_device_matches_numpy(name, row0, rows):
    cfg = synth.get_config(name)
    X, y, m = synth.config_inputs_device(cfg, row0, rows, device="cpu", ld=(cfg.d_in + 3) // 4 * 4)
    Xn, yn, mn = synth.config_inputs(cfg, row0, rows)
    assert np.array_equal(X.numpy(), Xn) and np.array_equal(y.numpy(), yn) and np.array_equal(m.numpy(), mn)


def test_hash_torch_matches_numpy_edge_counters():
    idx = np.array([0, 1, 2**31, 2**40 + 7, 2**62 + 12345], dtype=np.uint64)
    a = synth.hash64(5, 1, idx)
    b = synth.hash64_torch(5, 1, torch.from_numpy(idx.astype(np.int64))).numpy().view(np.uint64)
    assert np.array_equal(a, b)


@pytest.mark.gpu
def test_config_inputs_cuda_matches_numpy():
    cfg = synth.get_config("papers")
    X, y, m = synth.config_inputs_device(cfg, 50_000_000, 4096, device="cuda")
    Xn, yn, mn = synth.config_inputs(cfg, 50_000_000, 4096)
    assert np.array_equal(X.cpu().numpy(), Xn) and np.array_equal(y.cpu().numpy(), yn)
    assert np.array_equal(m.cpu().numpy(), mn)


def test_features_device_matches_numpy():
    a = synth.features_device(27, 10_000, 4, device="cpu", row0=9_000, rows=1000).numpy()
    assert np.array_equal(a, synth.features(27, 10_000, 4, row0=9_000, rows=1000))
