"""Multi-GPU parity check, one rank per GPU (run by tests/test_gpu_multi.py):

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 tests/mp_check.py [config]

Per rank, through the C ABI with the library's own NCCL communicator:
  1. split/gather (v2f/f2v) against the oracle's layout definitions, bitwise (fp32, bf16);
  2. K-hop propagation of this rank's FEATURE slice vs the oracle (R10, 1e-5) and
     bitwise vs the same columns of a single-GPU (P = 1) propagation;
  3. 3 training epochs with the overlap scheduler on and off: losses vs the oracle
     (1e-4), and on == off bitwise (scheduling neutrality);
  4. the same on a degree-reordered graph (NTP_G_REORDER): slice propagation bitwise vs P = 1,
     epochs vs the oracle;
  5.-7. bf16 / fused head, NEXT-4 data-parallel baseline, NEXT-1 coupled epochs;
  8. NEXT-2 decoupled GAT epochs vs the GAT oracle (one and two slices per rank);
  9. virtual slices across ranks (P = 2 * world): layouts and epochs;
 10. a mismatched collective times out (NTP_ERR_TIMEOUT) and aborts the communicator.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2412_20379_b200 import ntp  # noqa: E402
from paper_2412_20379_b200 import dist as pd  # noqa: E402


def _step(k, rank):
    print(f"[mp_check rank {rank}] step {k}", flush=True)


def main(name):
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = pd.broadcast_unique_id(dist, rank)
    cfg = synth.get_config(name)
    ctx = ntp.Context(device=local, rank=rank, world=world, unique_id=uid)
    thr = synth.rmat_thresholds(*cfg.abc)
    ctx.generate_rmat(cfg.n, cfg.scale, cfg.m_raw, thr, cfg.seed, cfg.symmetric)
    g = oracle.graph.graph_from_config(cfg)
    n = g.n

    _step('1', rank)
    # ---- 1. layouts
    for dt, tdt, eb in ((ntp.NTP_F32, torch.float32, 4), (ntp.NTP_BF16, torch.bfloat16, 2)):
        w = 37
        Xfull = synth.features(99, n, w)
        part = oracle.layout.partition(n, w, world, eb)
        Xv = torch.from_numpy(oracle.layout.vertex_part(Xfull, n, w, world, rank, eb)[:, :w].copy()).to(tdt).cuda()
        Hf = torch.empty(part["V_pad"], part["d_s"], dtype=tdt, device="cuda")
        ctx.layout_v2f(Xv, Hf)
        ref_f = oracle.layout.feature_part(torch.from_numpy(Xfull).to(tdt).float().numpy(), n, w, world, rank, eb)
        torch.cuda.synchronize()
        assert np.array_equal(Hf.float().cpu().numpy(), ref_f), f"v2f mismatch rank {rank}"
        back = torch.zeros_like(Xv)
        ctx.layout_f2v(Hf, back)
        torch.cuda.synchronize()
        assert torch.equal(back, Xv), f"f2v(v2f(x)) != x rank {rank}"

    _step('2', rank)
    # ---- 2. propagation of this rank's slice
    w = 41
    part = oracle.layout.partition(n, w, world, 4)
    d_s = part["d_s"]
    H = synth.features(5, n, w)
    Hs = oracle.layout.feature_part(H, n, w, world, rank, 4)       # [V_pad x d_s]
    ctx1 = ntp.Context(device=local)                                 # P = 1 reference on the same GPU
    ctx1.generate_rmat(cfg.n, cfg.scale, cfg.m_raw, thr, cfg.seed, cfg.symmetric)
    full_w = oracle.layout.slice_width(w, 1, 4)
    Hp = np.zeros((n, full_w), np.float32)
    Hp[:, :w] = H
    Hp1 = np.zeros((n, world * d_s), np.float32)
    Hp1[:, :w] = H
    for transposed in (False, True):
        f = ctx.propagate_bwd if transposed else ctx.propagate_fwd
        Ht = torch.from_numpy(Hs).cuda()
        Zt = torch.empty_like(Ht)
        f(Ht, Zt, cfg.K, cfg.gamma, cfg.alpha)
        torch.cuda.synchronize()
        of = oracle.propagate.propagate_bwd if transposed else oracle.propagate.propagate_fwd
        ref = of(g, Hs[:n], cfg.K, cfg.gamma, cfg.alpha)
        den = of(g, np.abs(Hs[:n]), cfg.K, cfg.gamma, cfg.alpha)
        err = np.abs(Zt.double().cpu().numpy()[:n] - ref)
        assert (err <= 1e-5 * den + 1e-30).all(), f"propagation parity rank {rank} T={transposed}"
        # slice invariance across GPUs: same columns of the P=1 run, bitwise
        H1 = torch.from_numpy(Hp1).cuda()
        Z1 = torch.empty_like(H1)
        (ctx1.propagate_bwd if transposed else ctx1.propagate_fwd)(H1, Z1, cfg.K, cfg.gamma, cfg.alpha)
        torch.cuda.synchronize()
        assert torch.equal(Z1[:, rank * d_s:(rank + 1) * d_s], Zt[:n]), f"P-invariance rank {rank}"

    _step('2b', rank)
    # ---- 2b. vertex-layout pipeline (split -> K hops -> gather), overlap off / on: vs the oracle
    # on this rank's rows, and bitwise equal to each other
    wv = 37
    Hfull = synth.features(13, n, wv)
    V_p = part["V_p"]
    Hv = np.zeros((V_p, wv), np.float32)
    lo, hi = rank * V_p, min(n, (rank + 1) * V_p)
    Hv[:hi - lo] = Hfull[lo:hi]
    outs = []
    for transposed in (False, True):
        of = oracle.propagate.propagate_bwd if transposed else oracle.propagate.propagate_fwd
        ref = of(g, Hfull, cfg.K, cfg.gamma, cfg.alpha)[lo:hi]
        den = of(g, np.abs(Hfull), cfg.K, cfg.gamma, cfg.alpha)[lo:hi]
        for overlap in (False, True):
            Zv = torch.zeros(V_p, wv, device="cuda")
            ctx.propagate_pipeline(torch.from_numpy(Hv).cuda(), Zv, cfg.K, cfg.gamma, cfg.alpha,
                                   transposed=transposed, chunks=3, overlap=overlap)
            torch.cuda.synchronize()
            z = Zv.double().cpu().numpy()[:hi - lo]
            assert (np.abs(z - ref) <= 1e-5 * den + 1e-30).all(), f"pipeline parity rank {rank} T={transposed}"
            outs.append(Zv.cpu())
        assert torch.equal(outs[-2], outs[-1]), f"pipeline overlap changed bits rank {rank} T={transposed}"

    _step('3', rank)
    # ---- 3. epochs, overlap off / on
    X, y, m = pd.rank_inputs(cfg, world, rank)
    W0h, W1h = synth.model_weights(cfg)
    lr = cfg.lr * 50
    ref_losses, _, _ = oracle.model.train(g, *synth.config_inputs(cfg), W0h, W1h, cfg.K, cfg.gamma, cfg.alpha, lr, 3)
    results = []
    # peer-direct layouts (producers store into the owners' IPC windows), the NCCL block exchange
    # (default) and the overlapped NCCL gather: all three bitwise equal
    # (W1 after propagation also: "ce", the overlapped schedule with copy-engine peer copies + inbox flags)
    modes = ("p2p", "nccl", "overlap") + (("ce",) if cfg.w_after_prop else ())
    for mode in modes:
        overlap = mode in ("overlap", "ce")
        W0, W1 = torch.from_numpy(W0h).cuda(), torch.from_numpy(W1h).cuda()
        flags = ((ntp.NTP_M_W1_AFTER_PROP if cfg.w_after_prop else 0) | (ntp.NTP_M_OVERLAP if overlap else 0)
                 | (ntp.NTP_M_P2P_LAYOUTS if mode in ("p2p", "ce") else 0))
        model = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=cfg.K, gamma=cfg.gamma, alpha=cfg.alpha, lr=lr,
                     dtype=ntp.NTP_F32, chunks=3, flags=flags)
        losses = []
        for _ in range(3):
            rep = ctx.train_epoch(model, *(torch.from_numpy(a).cuda() for a in (X, y, m)), W0, W1)
            losses.append(rep["loss"])
        for a, b in zip(losses, ref_losses):
            assert abs(a - b) <= 1e-4, f"loss {a} vs oracle {b} (mode={mode})"
        # bytes handed to the transport per layout change (counted where issued) = the closed form
        wire = (world - 1) * V_p * oracle.layout.slice_width(cfg.hid if cfg.w_after_prop else cfg.C, world, 4) * 4
        assert rep["bytes_sent"] == [wire] * 4, f"wire bytes {rep['bytes_sent']} vs {wire} (mode={mode})"
        results.append((losses, W0.cpu(), W1.cpu()))
    for k in range(1, len(modes)):
        assert results[0][0] == results[k][0], f"layout mode {modes[k]} changed the loss"
        assert torch.equal(results[0][1], results[k][1]) and torch.equal(results[0][2], results[k][2])

    # K = 1 with the overlapped gather (W1 before propagation): the last hop is the only hop, so it reads the
    # receive buffer the chunked gather overwrites -- the epoch keeps S^0 in a copy
    if not cfg.w_after_prop:
        ref1, _, _ = oracle.model.train(g, *synth.config_inputs(cfg), W0h, W1h, 1, cfg.gamma, cfg.alpha, lr, 2)
        for overlap in (False, True):
            W0, W1 = torch.from_numpy(W0h).cuda(), torch.from_numpy(W1h).cuda()
            model = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=1, gamma=cfg.gamma, alpha=cfg.alpha, lr=lr,
                         dtype=ntp.NTP_F32, chunks=3, flags=ntp.NTP_M_OVERLAP if overlap else 0)
            for e in range(2):
                rep = ctx.train_epoch(model, *(torch.from_numpy(a).cuda() for a in (X, y, m)), W0, W1)
                assert abs(rep["loss"] - ref1[e]) <= 1e-4, f"K=1 loss {rep['loss']} vs {ref1[e]} (overlap={overlap})"

    _step('4', rank)
    # ---- 4. degree-reordered graph (NTP_G_REORDER): slice propagation bitwise vs P = 1 on the same
    # reordered graph, epochs vs the oracle
    uid2 = pd.broadcast_unique_id(dist, rank)
    ctxr = ntp.Context(device=local, rank=rank, world=world, unique_id=uid2)
    ctxr.generate_rmat(cfg.n, cfg.scale, cfg.m_raw, thr, cfg.seed, cfg.symmetric, reorder=True)
    ctxr1 = ntp.Context(device=local)
    ctxr1.generate_rmat(cfg.n, cfg.scale, cfg.m_raw, thr, cfg.seed, cfg.symmetric, reorder=True)
    Ht = torch.from_numpy(Hs).cuda()
    Zt = torch.empty_like(Ht)
    ctxr.propagate_fwd(Ht, Zt, cfg.K, cfg.gamma, cfg.alpha)
    H1 = torch.from_numpy(Hp1).cuda()
    Z1 = torch.empty_like(H1)
    ctxr1.propagate_fwd(H1, Z1, cfg.K, cfg.gamma, cfg.alpha)
    torch.cuda.synchronize()
    assert torch.equal(Z1[:, rank * d_s:(rank + 1) * d_s], Zt[:n]), f"reordered P-invariance rank {rank}"
    W0, W1 = torch.from_numpy(W0h).cuda(), torch.from_numpy(W1h).cuda()
    model = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=cfg.K, gamma=cfg.gamma, alpha=cfg.alpha, lr=lr,
                 dtype=ntp.NTP_F32, chunks=1,
                 flags=(ntp.NTP_M_W1_AFTER_PROP if cfg.w_after_prop else 0) | ntp.NTP_M_P2P_LAYOUTS)
    for e in range(3):
        rep = ctxr.train_epoch(model, *(torch.from_numpy(a).cuda() for a in (X, y, m)), W0, W1)
        assert abs(rep["loss"] - ref_losses[e]) <= 1e-4, f"reordered loss {rep['loss']} vs {ref_losses[e]}"
    ctxr.close()
    ctxr1.close()

    _step('5', rank)
    # ---- 5. bf16 storage epochs (the fused tcgen05 head where P*d_s = 128, e.g. head_dir): losses vs
    # the oracle within 2e-2 relative; peer-direct and NCCL layouts bitwise equal
    bres = []
    # (the W1-after-propagation epoch's overlap runs every layout change per row chunk on the comm stream)
    bmodes = ("nccl", "p2p", "overlap") + (("ce",) if cfg.w_after_prop else ())
    for mode in bmodes:
        W0, W1 = torch.from_numpy(W0h).cuda(), torch.from_numpy(W1h).cuda()
        model = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=cfg.K, gamma=cfg.gamma, alpha=cfg.alpha, lr=lr,
                     dtype=ntp.NTP_BF16, chunks=3,
                     flags=(ntp.NTP_M_W1_AFTER_PROP if cfg.w_after_prop else 0)
                     | (ntp.NTP_M_P2P_LAYOUTS if mode in ("p2p", "ce") else 0)
                     | (ntp.NTP_M_OVERLAP if mode in ("overlap", "ce") else 0))
        losses = []
        for e in range(2):
            rep = ctx.train_epoch(model, *(torch.from_numpy(a).cuda() for a in (X, y, m)), W0, W1)
            losses.append(rep["loss"])
            assert abs(rep["loss"] - ref_losses[e]) <= 2e-2 * abs(ref_losses[e]), \
                f"bf16 loss {rep['loss']} vs oracle {ref_losses[e]} (mode={mode})"
        bres.append((losses, W0.cpu(), W1.cpu()))
    for k in range(1, len(bmodes)):
        assert bres[0][0] == bres[k][0] and torch.equal(bres[0][1], bres[k][1]) and torch.equal(bres[0][2], bres[k][2]), \
            f"bf16 mode {bmodes[k]} changed the bits"
    if cfg.w_after_prop:   # overlap trace (ntp_set_trace): per-chunk intervals on both streams, causality, same bits
        for mode in ("overlap", "ce"):
            W0, W1 = torch.from_numpy(W0h).cuda(), torch.from_numpy(W1h).cuda()
            model = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=cfg.K, gamma=cfg.gamma, alpha=cfg.alpha, lr=lr,
                         dtype=ntp.NTP_BF16, chunks=3, flags=ntp.NTP_M_W1_AFTER_PROP | ntp.NTP_M_OVERLAP
                         | (ntp.NTP_M_P2P_LAYOUTS if mode == "ce" else 0))
            ctx.set_trace(True)
            rep = ctx.train_epoch(model, *(torch.from_numpy(a).cuda() for a in (X, y, m)), W0, W1)
            tr = ctx.trace()
            ctx.set_trace(False)
            assert rep["loss"] == bres[0][0][0], f"traced epoch changed the loss ({mode})"
            recs = {}
            for r in tr:
                assert r["end_ms"] >= r["begin_ms"] >= 0.0, r
                recs.setdefault((r["stream"], r["phase"]), {})[r["chunk"]] = (r["begin_ms"], r["end_ms"])
            nch = len(recs[("comm", 0)])
            assert nch >= 2, recs.keys()
            for key in [("comm", q) for q in range(4)] + [("compute", 0), ("compute", 1), ("compute", 3)]:
                assert sorted(recs[key]) == list(range(nch)), (mode, key, sorted(recs[key]))
            assert list(recs[("compute", 4)]) == [-1] and list(recs[("compute", 5)]) == [-1]
            eps = 0.01
            for ch in range(nch):   # every transfer waits for its producer, every consumer for its transfer
                assert recs[("comm", 0)][ch][0] >= recs[("compute", 0)][ch][1] - eps, (mode, "split", ch)
                assert recs[("comm", 1)][ch][0] >= recs[("compute", 4)][-1][1] - eps, (mode, "gather", ch)
                assert recs[("compute", 1)][ch][0] >= recs[("comm", 1)][ch][1] - eps, (mode, "head", ch)
                assert recs[("comm", 2)][ch][0] >= recs[("compute", 1)][ch][1] - eps, (mode, "gsplit", ch)
                assert recs[("compute", 3)][ch][0] >= recs[("comm", 3)][ch][1] - eps, (mode, "mlp bwd", ch)
            # the first chunk's split starts before the last chunk's MLP forward ends: the transfer overlaps
            assert recs[("comm", 0)][0][0] < recs[("compute", 0)][nch - 1][1], (mode, "no overlap")
    if cfg.w_after_prop:   # overlap on a degree-reordered graph (the papers configuration): vs the oracle
        W0, W1 = torch.from_numpy(W0h).cuda(), torch.from_numpy(W1h).cuda()
        ctxo = ntp.Context(device=local, rank=rank, world=world, unique_id=pd.broadcast_unique_id(dist, rank))
        ctxo.generate_rmat(cfg.n, cfg.scale, cfg.m_raw, thr, cfg.seed, cfg.symmetric, reorder=True)
        model = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=cfg.K, gamma=cfg.gamma, alpha=cfg.alpha, lr=lr,
                     dtype=ntp.NTP_BF16, chunks=4, flags=ntp.NTP_M_W1_AFTER_PROP | ntp.NTP_M_OVERLAP)
        for e in range(2):
            rep = ctxo.train_epoch(model, *(torch.from_numpy(a).cuda() for a in (X, y, m)), W0, W1)
            assert abs(rep["loss"] - ref_losses[e]) <= 2e-2 * abs(ref_losses[e]), f"reordered overlap loss {rep['loss']}"
        ctxo.close()

    _step('7', rank)
    # ---- 7. NEXT-4: the data-parallel baseline (full-width rows, all-gather before every hop) trains the
    # same model: losses vs the oracle (fp32 1e-4, bf16 2e-2), traffic = 2K all-gathers of full rows
    if not cfg.w_after_prop:
        for dtype, tol in ((ntp.NTP_F32, 1e-4), (ntp.NTP_BF16, 2e-2)):
            W0, W1 = torch.from_numpy(W0h).cuda(), torch.from_numpy(W1h).cuda()
            model = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=cfg.K, gamma=cfg.gamma, alpha=cfg.alpha, lr=lr,
                         dtype=dtype, chunks=1, flags=ntp.NTP_M_DATA_PARALLEL)
            for e in range(3):
                rep = ctx.train_epoch(model, *(torch.from_numpy(a).cuda() for a in (X, y, m)), W0, W1)
                bound = tol if dtype == ntp.NTP_F32 else tol * abs(ref_losses[e])
                assert abs(rep["loss"] - ref_losses[e]) <= bound, f"DP loss {rep['loss']} vs {ref_losses[e]} ({dtype})"
            eb = 4 if dtype == ntp.NTP_F32 else 2
            assert rep["bytes_sent"][0] == 2 * cfg.K * (world - 1) * V_p * oracle.layout.slice_width(cfg.C, 1, eb) * eb

    _step('6', rank)
    # ---- 6. NEXT-1: naive (coupled) TP epochs, 2 and 3 layers: losses vs the coupled oracle, and the
    # communication ledger: 4L - 2 layout changes moving the closed-form bytes
    from oracle import coupled
    for mid in ((24,), (24, 16)):
        widths = (cfg.d_in, *mid, cfg.C)
        L = len(widths) - 1
        Ws = [synth.glorot(cfg.seed, widths[i], widths[i + 1], 100_000 * (i + 1)) for i in range(L)]
        ref_c, _ = coupled.train(g, *synth.config_inputs(cfg), Ws, lr, 2)
        Wd = [torch.from_numpy(W).cuda() for W in Ws]
        for e in range(2):
            rep = ctx.train_epoch_coupled(widths, lr, *(torch.from_numpy(a).cuda() for a in (X, y, m)), Wd)
            assert abs(rep["loss"] - ref_c[e]) <= 1e-4, f"coupled loss {rep['loss']} vs {ref_c[e]} (L={L})"
            assert rep["layout_changes"] == coupled.layout_changes(L, world)
            ds = lambda w: oracle.layout.slice_width(w, world, 4)
            assert rep["bytes_sent"] == coupled.layout_bytes(widths, V_p, ds, world, 4)
    _step('8', rank)
    # ---- 8. NEXT-2: decoupled GAT (score halves all-gathered, coefficients recomputed per rank, dalpha
    # allreduced): losses and every parameter vs the GAT oracle; then with 2 virtual slices per rank
    if not cfg.w_after_prop:
        from oracle import gat
        a0 = synth.glorot(cfg.seed, 2, cfg.C, 7_000_000)
        gmodel = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=2, gamma=0.9, alpha=0.0, lr=lr, dtype=ntp.NTP_F32,
                      chunks=1, flags=0)
        rl, rW0, rW1, ras, rad = gat.train(g, *synth.config_inputs(cfg), W0h, W1h, a0[0], a0[1], 2, 0.9, lr, 2)
        for vsl in (1, 2):
            ctxg = ntp.Context(device=local, rank=rank, world=world, unique_id=pd.broadcast_unique_id(dist, rank))
            ctxg.generate_rmat(cfg.n, cfg.scale, cfg.m_raw, thr, cfg.seed, cfg.symmetric)
            ctxg.set_slices(world * vsl)
            Xg, yg, mg = pd.rank_inputs(cfg, world, rank, slices=world * vsl)
            W0, W1, A = (torch.from_numpy(a).cuda() for a in (W0h, W1h, a0))
            for e in range(2):
                rep = ctxg.train_epoch_gat(gmodel, *(torch.from_numpy(a).cuda() for a in (Xg, yg, mg)), W0, W1, A)
                assert abs(rep["loss"] - rl[e]) <= 1e-4, f"GAT loss {rep['loss']} vs {rl[e]} (vs={vsl})"
            for got, ref in ((W0, rW0), (W1, rW1), (A, np.stack([ras, rad]))):
                got = got.cpu().numpy()
                assert np.abs(got - ref).max() <= 1e-4 * max(1.0, np.abs(ref).max()), f"GAT weights (vs={vsl})"
            ctxg.close()

    _step('9', rank)
    # ---- 9. virtual slices across ranks (P = 2 * world: two slices per GPU, per-(peer, slice) exchanges):
    # layouts round trip, epochs vs the oracle
    ctxv = ntp.Context(device=local, rank=rank, world=world, unique_id=pd.broadcast_unique_id(dist, rank))
    ctxv.generate_rmat(cfg.n, cfg.scale, cfg.m_raw, thr, cfg.seed, cfg.symmetric)
    Pv = 2 * world
    ctxv.set_slices(Pv)
    partv = oracle.layout.partition(n, 37, Pv, 4)
    Vr = partv["V_pad"] // world
    Xfull = synth.features(99, n, 37)
    Hv_ = np.zeros((Vr, 37), np.float32)
    lo_, hi_ = rank * Vr, min(n, (rank + 1) * Vr)
    Hv_[:max(0, hi_ - lo_)] = Xfull[lo_:hi_]
    Hv_t = torch.from_numpy(Hv_).cuda()
    Hf = torch.empty(2 * partv["V_pad"], partv["d_s"], device="cuda")
    ctxv.layout_v2f(Hv_t, Hf)
    for j in range(2):   # slice j of this rank = global slice rank*2 + j of the matrix
        q = rank * 2 + j
        ref = np.zeros((partv["V_pad"], partv["d_s"]), np.float32)
        c0, c1 = q * partv["d_s"], min(37, (q + 1) * partv["d_s"])
        if c1 > c0:
            ref[:n, :c1 - c0] = Xfull[:, c0:c1]
        torch.cuda.synchronize()
        assert np.array_equal(Hf[j * partv["V_pad"]:(j + 1) * partv["V_pad"]].cpu().numpy(), ref), f"virtual v2f {rank}/{j}"
    back = torch.zeros_like(Hv_t)
    ctxv.layout_f2v(Hf, back)
    ctxv.sync()
    assert torch.equal(back, Hv_t), "virtual f2v(v2f(x)) != x"
    Xv_, yv_, mv_ = pd.rank_inputs(cfg, world, rank, slices=Pv)
    W0, W1 = torch.from_numpy(W0h).cuda(), torch.from_numpy(W1h).cuda()
    model = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=cfg.K, gamma=cfg.gamma, alpha=cfg.alpha, lr=lr,
                 dtype=ntp.NTP_F32, chunks=1, flags=ntp.NTP_M_W1_AFTER_PROP if cfg.w_after_prop else 0)
    for e in range(3):
        rep = ctxv.train_epoch(model, *(torch.from_numpy(a).cuda() for a in (Xv_, yv_, mv_)), W0, W1)
        assert abs(rep["loss"] - ref_losses[e]) <= 1e-4, f"virtual-slice loss {rep['loss']} vs {ref_losses[e]}"
    ctxv.close()

    _step('10', rank)
    # ---- 10. collective timeout: rank 0 issues a layout change the other ranks never join;
    # its synchronising call must abort the communicator and return NTP_ERR_TIMEOUT, not hang
    ctxt = ntp.Context(device=local, rank=rank, world=world, unique_id=pd.broadcast_unique_id(dist, rank))
    ctxt.generate_rmat(cfg.n, cfg.scale, cfg.m_raw, thr, cfg.seed, cfg.symmetric)
    ctxt.set_timeout(3000)
    part1 = oracle.layout.partition(n, 37, world, 4)
    Hv1 = torch.zeros(part1["V_p"], 37, device="cuda")
    Hf1 = torch.empty(part1["V_pad"], part1["d_s"], device="cuda")
    ctxt.layout_v2f(Hv1, Hf1)   # a matched exchange first: NCCL connects peers lazily, inside the enqueueing call
    ctxt.sync()
    dist.barrier()
    if rank == 0:
        ctxt.layout_v2f(Hv1, Hf1)
        import time as _t
        t0 = _t.time()
        try:
            ctxt.sync()
            raise AssertionError("mismatched collective did not time out")
        except ntp.NtpError as ex:
            assert ex.status == ntp.NTP_ERR_TIMEOUT, f"expected NTP_ERR_TIMEOUT, got {ex}"
        assert _t.time() - t0 < 60, "timeout took too long"
        try:   # the aborted communicator refuses further collectives
            ctxt.layout_v2f(Hv1, Hf1)
            raise AssertionError("collective accepted after abort")
        except ntp.NtpError as ex:
            assert ex.status == ntp.NTP_ERR_NCCL
    dist.barrier()
    if rank != 0:
        ctxt.abort()   # the peer gave up: leave without waiting for it
    ctxt.close()

    dist.barrier()
    if rank == 0:
        print(f"MP OK world={world} config={name} losses={results[1][0]}", flush=True)
    ctx.close()
    ctx1.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    try:
        main(sys.argv[1] if len(sys.argv) > 1 else "small_dir")
    except Exception as e:  # the failing assertion on stdout (torchrun's stderr is long)
        import traceback
        print(f"MP FAIL rank {os.environ.get('RANK')}: {type(e).__name__}: {e}\n{traceback.format_exc()[-1500:]}",
              flush=True)
        raise
