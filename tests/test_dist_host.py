"""World-size-2 gloo tests (CPU) of the host-side multi-rank logic: row ownership,
per-rank input materialisation, id broadcast and max-over-ranks timing."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, out_q, slices=0):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2412_20379_b200 import dist as pd
        cfg = synth.get_config(name)
        X, y, m = pd.rank_inputs(cfg, world, rank, slices=slices)
        parts = [None] * world
        dist.all_gather_object(parts, (X, y, m))
        # id broadcast through the same object channel the bench uses (library not needed)
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        mx = pd.max_over_ranks(dist, float(rank + 1) * 1.5)
        if rank == 0:
            out_q.put((parts, obj[0], mx))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,slices", [("tiny_dir", 0), ("cora", 0), ("tiny_dir", 6), ("cora", 8)])
def test_rank_inputs_tile_the_graph(name, slices):
    """Per-rank vertex rows tile [0, n) exactly, for P = world and for virtual slices (P = slices, P % world
    == 0: each rank owns V_pad / world = (P / world) * ceil(n / P) rows)."""
    import synth
    from paper_2412_20379_b200 import build
    build.build(verbose=False)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q, slices)) for r in range(world)]
    for p in procs:
        p.start()
    parts, uid, mx = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = synth.get_config(name)
    X = np.concatenate([p[0] for p in parts])
    y = np.concatenate([p[1] for p in parts])
    m = np.concatenate([p[2] for p in parts])
    Xf, yf, mf = synth.config_inputs(cfg)
    n = cfg.n
    P = slices or world
    assert X.shape[0] == P * -(-n // P)
    assert np.array_equal(X[:n], Xf) and np.array_equal(y[:n], yf) and np.array_equal(m[:n], mf)
    assert not X[n:].any() and not m[n:].any()
    assert uid == bytes(range(128))
    assert mx == 3.0
