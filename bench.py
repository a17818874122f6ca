#!/usr/bin/env python
"""Benchmark: one decoupled-TP training epoch (all SURVEY §8(a) rows) per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config reddit] [--impl ntp|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1: one rank per GPU, NCCL)

Metric (BASELINE.json): epoch time and aggregation GE/s; value = epoch GE/s =
2*K*nnz*w / t_epoch summed over the whole job (strong scaling: the graph is
fixed, its feature columns are split over the N GPUs).  The dominant kernel's
roofline uses the algorithmic bytes of DESIGN.md §6 and CUDA-event durations
recorded by the library on the stream the SpMM kernel runs on.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "epoch time (s) and aggregation GE/s at 1/2/4/8 B200; % of HBM roofline"
WORKLOADS = {
    "reddit": "Reddit-shaped R-MAT graph (232,965 vertices, ~114M arcs, 602 features, 41 classes), "
              "decoupled 2-hop GCN training epoch",
    "products": "ogbn-products-shaped R-MAT graph (2.45M vertices, ~62M arcs, 100 features, 47 classes), "
                "APPNP K=10 training epoch",
    "cora": "Cora-shaped R-MAT graph (2,708 vertices, ~10.6K arcs, 1,433 binary features, 7 classes), "
            "decoupled 2-hop GCN training epoch",
    "orkut": "Orkut-shaped R-MAT graph (3.07M vertices, ~116M arcs), 512-feature decoupled training epoch",
    "papers": "ogbn-papers100M-shaped R-MAT graph (111M vertices, ~1.6B directed arcs, 128 features, 172 classes), "
              "decoupled 2-hop GCN training epoch, bf16 feature slices, W1 after propagation",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ algorithmic bytes
def hop_bytes(n, nnz, d_s, elem, symmetric, alpha, l2_bytes):
    """Algorithmic HBM bytes of one SpMM hop on one GPU, by residency:
    B_lo = col_idx 4*nnz + row_ptr 4*(n+1) + D~^{-1/2} (4n, or 8n directed) + slice rows read once,
           output written once, S^0 once more if alpha > 0 (n*r*(2 + [alpha > 0]));
    slice (n*r) <= L2: B_lo (perfect reuse: the gathered rows are re-read from L2, not HBM);
    slice  >  L2: B_hi = B_lo + nnz*r_s (SURVEY's no-reuse per-edge figure: every arc's row slice,
           sector-rounded r_s = ceil(r/32)*32, comes from HBM).  Returns (bytes, model)."""
    r = d_s * elem
    lo = 4 * nnz + 4 * (n + 1) + (4 if symmetric else 8) * n + n * r * (2 + (1 if alpha > 0 else 0))
    if n * r <= l2_bytes:
        return lo, "perfect reuse (slice fits L2)"
    return lo + nnz * (-(-r // 32) * 32), "no reuse (slice larger than L2)"


def l2_gather_bytes(nnz, n, d_s, elem):
    """Bytes the gather pulls through L2 (no-reuse model): every arc and self row, sector-rounded."""
    r = -(-(d_s * elem) // 32) * 32
    return (nnz + n) * r


def gather_ceiling(n, row_bytes, l2_bytes):
    """Measured random-row-gather ceiling of this B200 (profiles/gather_ceiling.json, written from
    scripts/l2_probe.cu): rows/s for the table's residency (L2 if the slice fits the device's L2, the same
    test as hop_bytes, else HBM) at the smallest probed row size >= row_bytes."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "gather_ceiling.json")))
    except Exception:
        return None
    l2_res = n * row_bytes <= l2_bytes
    tab = d["l2_resident"] if l2_res else d["hbm_resident"]
    sizes = sorted(int(k) for k in tab)
    fit = [k for k in sizes if k >= row_bytes] or sizes[-1:]
    if not fit:
        return None
    k = fit[0]
    return {"rows_per_s": tab[str(k)]["Grows_per_s"] * 1e9, "probe_row_bytes": k,
            "residency": "L2" if l2_res else "HBM", "source": "profiles/gather_ceiling.json"}


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


def load_traffic(config, P, dtype, padded_d_s=None):
    """ncu dram bytes per launch of the SpMM hop kernel, from the committed profile summary (captured at the
    16-byte-rounded slice width; a padded slice (--slice-align) looks up its own key `.../d<d_s>`)."""
    path = os.path.join(ROOT, "profiles", "spmm_traffic.json")
    try:
        d = json.load(open(path))
        key = f"{config}/P{P}/{dtype}" + (f"/d{padded_d_s}" if padded_d_s else "")
        v = d.get(key)
        return v if v == v else None     # NaN (a failed capture) counts as missing
    except Exception:
        return None


# ------------------------------------------------------------------ oracle (cpu baseline / reference arm)
def host_info():
    """nproc, CPU model and RAM of this host (SURVEY §8(d) oracle timing)."""
    info = {"nproc": os.cpu_count(), "cpu_model": None, "ram_GB": None}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                info["ram_GB"] = round(int(line.split()[1]) / 1e6, 1)
                break
    except Exception:
        pass
    return info


def oracle_epoch_time(cfg, epochs=1):
    """Times the fp64 oracle (as it stands) for `epochs` full epochs on this host, from the same initial
    weights the GPU run starts from; returns its per-epoch losses too (the bench line's parity check), and
    a single-thread one-hop timing on a 2% row sample, extrapolated to the whole graph."""
    import oracle
    use_all_host_cores()
    t0 = time.time()
    g = oracle.graph.graph_from_config(cfg)
    t_graph = time.time() - t0
    X, y, m = synth.config_inputs(cfg)
    W0, W1 = synth.model_weights(cfg)
    losses = []
    t0 = time.time()
    for _ in range(epochs):
        loss, W0, W1 = oracle.model.train_epoch(g, X, y, m, W0, W1, cfg.K, cfg.gamma, cfg.alpha, cfg.lr)
        losses.append(loss)
    dt = (time.time() - t0) / epochs
    threads = oracle.lib.oracle_num_threads()
    one = None
    try:
        rng = np.random.default_rng(0)
        rows = np.sort(rng.choice(g.n, size=max(1, g.n // 50), replace=False))
        zin = synth.features(cfg.seed, g.n, cfg.w)
        oracle.lib.oracle_set_num_threads(1)
        t1 = time.time()
        oracle.propagate.hop_rows(g, zin, None, rows, cfg.gamma, 0.0)
        one = (time.time() - t1) * g.n / rows.size
    finally:
        oracle.lib.oracle_set_num_threads(threads)
    return dt, g.nnz, threads, t_graph, losses, one


def oracle_sampled_estimate(cfg, frac=0.01, cols=4):
    """SURVEY §8(d) c5 oracle timing: the full fp64 state of the papers shape is ~1 TB, so the oracle (as it
    stands) propagates a `cols`-column subset over a `frac` row sample -- exact per row and column by column
    separability -- and runs the MLP forward/backward and the loss on the same row sample; the epoch
    time is EXTRAPOLATED linearly (x 1/frac rows, x w/cols columns, x 2K hops)."""
    import oracle
    use_all_host_cores()
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(cfg.n, size=max(1, int(cfg.n * frac)), replace=False)).astype(np.int64)
    t0 = time.time()
    nb = oracle.graph.sampled_rows(cfg, rows, False)       # in-arcs of the sample (arc-stream filter)
    t_filter = time.time() - t0
    rp = np.zeros(cfg.n + 1, np.int64)
    deg = np.zeros(cfg.n, np.int64)
    deg[rows] = [nb[v].size for v in rows.tolist()]
    np.cumsum(deg, out=rp[1:])
    col = np.concatenate([nb[v] for v in rows.tolist()]).astype(np.int32)
    sample_arcs = int(col.size)
    ones = np.ones(cfg.n)
    zin = rng.standard_normal((cfg.n, cols))
    lib = oracle.lib
    out = np.empty((rows.size, cols))
    t0 = time.time()
    lib.oracle_hop_rows(rp.ctypes.data, col.ctypes.data, ones.ctypes.data, ones.ctypes.data, cols, zin.ctypes.data,
                        None, 1.0, 0.0, rows.ctypes.data, rows.size, out.ctypes.data)
    t_hop = time.time() - t0
    del zin, rp, col
    X, y, m = synth.config_inputs(cfg, 0, rows.size)        # a row sample of the same shape
    W0, W1 = synth.model_weights(cfg)
    t0 = time.time()
    A1 = X.astype(np.float64) @ W0
    H1 = np.maximum(A1, 0.0)
    logits = H1 @ W1 if not cfg.w_after_prop else H1 @ W1   # W1 applied after propagation: same GEMM
    loss_sum, n_train, d = oracle.model.softmax_xent(logits, y, m)
    dW1 = H1.T @ d
    dH1 = (d @ W1.T) * (A1 > 0)
    dW0 = X.T.astype(np.float64) @ dH1
    t_mlp = time.time() - t0
    hop_full = t_hop / frac * (cfg.w / cols)
    epoch = 2 * cfg.K * hop_full + t_mlp / frac
    return {"epoch_s": epoch, "hop_s": hop_full, "mlp_s": t_mlp / frac, "filter_s": t_filter,
            "sample_rows": int(rows.size), "sample_arcs": sample_arcs, "cols": cols, "frac": frac}


def auto_slice_align(cfg, world, dt, engine, l2_bytes):
    """Slice-row padding (measured on the L2-resident Reddit shape): slice rows of up to 128 bytes
    hop faster at a power-of-two width (16 fp32 columns 0.91 ms vs 12 at 0.96; 32 at 1.27 vs 24 at 1.36), at
    the price of the padding bytes in the layout changes.  Padded when the slice fits L2 and the padding adds
    at most a third; HBM-resident slices (products: 1-4% slower padded) and wide rows keep 16-byte rounding."""
    from paper_2412_20379_b200 import ntp
    if engine not in ("decoupled", "gat"):
        return 16
    esz = 2 if dt == ntp.NTP_BF16 else 4
    row = ntp.partition(cfg.n, cfg.w, world, dt, 1, 16)["d_s"] * esz
    t = 64 if row <= 64 else 128
    if cfg.n * t > l2_bytes:     # the padded slice must stay L2-resident
        return 16
    return t if row > 32 and row <= 128 and 3 * t <= 4 * row else 16


def use_all_host_cores():
    """The oracle runs on every host core this process may use: torchrun exports OMP_NUM_THREADS=1 to its
    workers, which would otherwise pin the reference arm (rank 0) and its BLAS to one thread."""
    import oracle
    n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    oracle.lib.oracle_set_num_threads(n)
    try:
        import threadpoolctl
        threadpoolctl.threadpool_limits(n)
    except Exception:
        pass
    return n


def run_reference(args, cfg, rank):
    if rank != 0:
        return
    w = cfg.w
    times = []
    import oracle
    use_all_host_cores()
    g = oracle.graph.graph_from_config(cfg)
    X, y, m = synth.config_inputs(cfg)
    W0, W1 = synth.model_weights(cfg)
    for i in range(args.warmup + args.steps):
        t0 = time.time()
        loss, W0, W1 = oracle.model.train_epoch(g, X, y, m, W0, W1, cfg.K, cfg.gamma, cfg.alpha, cfg.lr)
        if i >= args.warmup:
            times.append(time.time() - t0)
    t = sum(times) / len(times)
    ge = 2 * cfg.K * g.nnz * w / t / 1e9
    cores = oracle.lib.oracle_num_threads()
    line = {"impl": "reference", "metric": METRIC, "value": ge, "unit": "GE/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS.get(args.config, args.config), "n": cfg.n, "nnz": g.nnz, "w": w,
                       "K": cfg.K},
            "cpu_baseline": {"value": ge, "unit": "GE/s", "cores": cores, "kind": "oracle", "host": host_info(),
                             "sample": f"{args.steps} full fp64 oracle epochs of the same workload (after "
                                       f"{args.warmup} warm-up), OpenMP rows + numpy BLAS"},
            "e2e": {"value": ge, "unit": "GE/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ NEXT-2: decoupled GAT engine
def run_gat(args, ctx, cfg, X, y, msk, n, nnz, world, rank, dist, barrier, stream, dt, dtype_name, V_p):
    """Times ntp_train_epoch_gat on the config's graph (w = C propagated, K hops with the precomputed attention)."""
    import torch
    W0h, W1h = synth.model_weights(cfg)
    W0, W1 = torch.from_numpy(W0h).cuda(), torch.from_numpy(W1h).cuda()
    A = torch.from_numpy(synth.glorot(cfg.seed, 2, cfg.C, 7_000_000)).cuda()
    model = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=cfg.K, gamma=cfg.gamma, alpha=0.0, lr=cfg.lr, dtype=dt,
                 chunks=1, flags=0)
    for _ in range(args.warmup):
        ctx.train_epoch_gat(model, X, y, msk, W0, W1, A, stream=stream)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = []
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    ev0.record(stream)
    for _ in range(args.steps):
        reps.append(ctx.train_epoch_gat(model, X, y, msk, W0, W1, A, stream=stream))
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    hop = sum(r["spmm_ms"] for r in reps) / max(1, sum(r["spmm_launches"] for r in reps))
    if dist is not None:
        t = torch.tensor([ms, hop], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, hop = float(t[0]), float(t[1])
    if rank != 0:
        return
    w = cfg.C
    line = {"metric": METRIC, "engine": "decoupled GAT (NEXT-2): attention precomputed once per epoch, weighted hops",
            "value": 2 * cfg.K * nnz * w / (ms * 1e-3) / 1e9, "unit": "GE/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": dtype_name, "data": "synthetic", "epoch_s": ms / 1e3,
            "config": {"workload": WORKLOADS.get(args.config, args.config) + "; decoupled GAT (w = C)", "n": n,
                       "nnz": nnz, "w": w, "K": cfg.K, "gamma": cfg.gamma, "P": world,
                       "slice_align": args.slice_align},
            "hop_ms": hop, "loss": reps[-1]["loss"],
            "phase_ms": {k: round(sum(r["ms"][k] for r in reps) / len(reps), 4) for k in reps[0]["ms"]},
            "clocks": clk, "gpu_launches": int(sum(r["kernel_launches"] for r in reps))}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ NEXT-1: coupled (naive TP) engine
def run_coupled(args, ctx, cfg, X, y, msk, n, nnz, world, rank, local, dist, barrier, stream, dt, dtype_name, V_p,
                reorder):
    """Times ntp_train_epoch_coupled (2-layer GCN d_in -> hid -> C, every layer aggregated on feature slices)
    and prints its ledger: layout changes and bytes per epoch vs the decoupled epoch's 4 changes."""
    import torch
    from paper_2412_20379_b200 import ntp
    widths = (cfg.d_in, cfg.hid, cfg.C)
    Ws = [torch.from_numpy(synth.glorot(cfg.seed, widths[i], widths[i + 1], 100_000 * (i + 1))).cuda()
          for i in range(len(widths) - 1)]
    for _ in range(args.warmup):
        ctx.train_epoch_coupled(widths, cfg.lr, X, y, msk, Ws, dtype=dt, stream=stream)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = []
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    ev0.record(stream)
    for _ in range(args.steps):
        reps.append(ctx.train_epoch_coupled(widths, cfg.lr, X, y, msk, Ws, dtype=dt, stream=stream))
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank != 0:
        return
    L = len(widths) - 1
    hop_cols = sum(widths[:L]) + sum(widths[1:L])     # forward hops at w_0..w_{L-1}, backward at w_1..w_{L-1}
    ge = nnz * hop_cols / (ms * 1e-3) / 1e9
    esz = 2 if dt == ntp.NTP_BF16 else 4
    d_s_dec = ntp.partition(n, cfg.w, world, dt, 1, args.slice_align)["d_s"]
    dec_bytes = 0 if world == 1 else 4 * (world - 1) * V_p * d_s_dec * esz
    r = reps[-1]
    line = {"metric": METRIC, "engine": "coupled (naive tensor parallelism, NEXT-1)", "value": ge, "unit": "GE/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": dtype_name, "data": "synthetic", "epoch_s": ms / 1e3,
            "config": {"workload": WORKLOADS.get(args.config, args.config) + "; coupled 2-layer GCN "
                       f"{widths[0]}->{widths[1]}->{widths[2]}", "n": n, "nnz": nnz, "P": world,
                       "vertex_order": "degree-ordered internally (NTP_G_REORDER)" if reorder else "R-MAT ids"},
            "ledger": {"layout_changes_per_epoch": r["layout_changes"], "bytes_sent_per_epoch": r["bytes_sent"],
                       "decoupled_layout_changes_per_epoch": 0 if world == 1 else 4,
                       "decoupled_bytes_sent_per_epoch": dec_bytes,
                       "volume_ratio": (r["bytes_sent"] / dec_bytes) if dec_bytes else None,
                       "note": "naive TP: a split and a gather around every layer's aggregation (4L-2 = 6 for L=2, "
                               "P:696); decoupled: 4 per epoch at the propagated width w"},
            "phase_ms": {"total": r["ms_total"], "aggregation": r["ms_agg"]},
            "clocks": clk, "gpu_launches": int(sum(x["kernel_launches"] for x in reps))}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ HBM-bound propagation leg
def hbm_leg(args, world, rank, local, dist, barrier, allmax, peak, peak_src, l2_size):
    """The Orkut-shaped pipeline of BASELINE configs[3] (3.07M vertices, ~116M arcs, w = 512 fp32, K = 2): this
    rank's rows -> split -> K hops on its d_s = 512/N column slice -> gather, forward and backward
    (ntp_propagate_pipeline), timed with CUDA events; the hop kernel's roofline against HBM (the slice is
    3.07M x d_s x 4 B >= 786 MB at N <= 8, far above L2, so every arc's row slice streams from HBM)."""
    import torch
    from paper_2412_20379_b200 import ntp
    cfg = synth.get_config("orkut")
    w, K = cfg.d_in, cfg.K
    uid = None
    if world > 1:
        obj = [ntp.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    ctx = ntp.Context(device=local, rank=rank, world=world, unique_id=uid)
    t0 = time.time()
    ctx.generate_rmat(cfg.n, cfg.scale, cfg.m_raw, synth.rmat_thresholds(*cfg.abc), cfg.seed, cfg.symmetric,
                      reorder=True)
    n, nnz, sym = ctx.graph_info()
    t_graph = time.time() - t0
    part = ntp.partition(n, w, world, ntp.NTP_F32)
    V_p, d_s = part["V_p"], part["d_s"]
    rows = max(0, min(V_p, n - rank * V_p))
    Hv = synth.features_device(cfg.seed, n, w, device="cuda", row0=rank * V_p, rows=rows) if rows else None
    H = torch.zeros(V_p, w, device="cuda")
    if rows:
        H[:rows] = Hv
    del Hv
    Z = torch.empty_like(H)
    G = torch.empty_like(H)
    stream = torch.cuda.current_stream()

    def step():
        ctx.propagate_pipeline(H, Z, K, cfg.gamma, cfg.alpha, transposed=False, stream=stream)
        a = ctx.hop_timing()
        ctx.propagate_pipeline(Z, G, K, cfg.gamma, cfg.alpha, transposed=True, stream=stream)
        b = ctx.hop_timing()
        return a[0] + b[0], a[1] + b[1]

    for _ in range(2):
        step()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    hop_ms = hops = 0
    ev0.record(stream)
    for _ in range(args.leg_steps):
        a, b = step()
        hop_ms += a
        hops += b
    ev1.record(stream)
    barrier()
    ms = allmax(ev0.elapsed_time(ev1) / args.leg_steps)
    hop_avg = allmax(hop_ms / max(hops, 1))
    ctx.close()
    del H, Z, G
    torch.cuda.empty_cache()
    bh, bmodel = hop_bytes(n, nnz, d_s, 4, sym, cfg.alpha, l2_size)
    b_lo = hop_bytes(n, nnz, d_s, 4, sym, cfg.alpha, float("inf"))[0]
    traffic = load_traffic("orkut", world, "f32")
    # HBM% as SURVEY §8(d) defines it: ncu DRAM bytes of this kernel on this shape / its live launch time.  The
    # two byte models bracket it (compulsory bytes below; "every arc's row slice from HBM" above -- which the
    # L2 beats on this graph, 37-64% hit rate), so neither is reported as the fraction.
    achieved = (traffic if traffic else bh) / (hop_avg * 1e-3) / 1e9
    return {
        "workload": "Orkut-shaped R-MAT graph (3.07M vertices, ~116M arcs), w = 512 fp32, K = 2: split -> K hops "
                    "-> gather, forward + backward (ntp_propagate_pipeline); BASELINE configs[3]",
        "n": n, "nnz": nnz, "w": w, "K": K, "P": world, "d_s": d_s, "graph_setup_s": round(t_graph, 3),
        "ms_per_step": ms, "value": 2 * K * nnz * w / (ms * 1e-3) / 1e9, "unit": "GE/s",
        "steps": args.leg_steps,
        "roofline": {"kernel": "spmm_hop_bulk_kernel" if d_s * 4 >= 1024 else "spmm_hop_kernel", "bound": "hbm",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "bytes_model": ("ncu DRAM read + write bytes per launch of this kernel on this shape "
                                     "(profiles/spmm_traffic.json)") if traffic else bmodel,
                     "algorithmic_bytes_per_launch": b_lo,
                     "algorithmic_note": "compulsory bytes (col_idx, row_ptr, D~^-1/2, each slice row read once, "
                                         "output written once): a lower bound",
                     "no_reuse_bytes_per_launch": bh, "no_reuse_GBps": bh / (hop_avg * 1e-3) / 1e9,
                     "avg_launch_ms": hop_avg,
                     "launches_timed": hops, "peak_source": peak_src,
                     "timed_span": "spmm_hop_kernel + its spmm_fixup_kernel, CUDA events on the hop's stream",
                     "vs_8TBps": achieved / 8000.0},
    }


# ------------------------------------------------------------------ main GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="reddit")
    ap.add_argument("--impl", default="ntp", choices=["ntp", "reference"])
    ap.add_argument("--dtype", default=None, choices=[None, "f32", "bf16"])
    ap.add_argument("--chunks", type=int, default=1)
    ap.add_argument("--overlap", action="store_true",  # a12
                    help="chunked last hop with the gather on the comm stream (a12); off by default: on "
                         "reddit the gather moves ~1-10 MB and chunking costs more than it hides")
    ap.add_argument("--slice-align", default="auto",
                    help="16/32/64/128 bytes, or auto: an L2-resident slice row of 33-64 or 65-128 bytes is padded to "
                         "64 / 128 bytes when that adds at most a third (DESIGN.md §6), else 16")
    ap.add_argument("--layouts", default="nccl", choices=["p2p", "nccl"],
                    help="P > 1 layout changes: the NCCL block all-to-all (default) or peer-direct stores into the "
                         "owners' IPC windows (NTP_M_P2P_LAYOUTS; alone measured no faster); with --overlap on a "
                         "W1-after-propagation config (papers): copy-engine transfers per row chunk (1.08-1.13x)")
    ap.add_argument("--reorder", default="auto", choices=["auto", "on", "off"],
                    help="NTP_G_REORDER (internal degree-class numbering). auto: on when the vertex table is "
                         "far larger than L2 (n >= 1M: products, orkut, papers), off for the L2-resident Reddit "
                         "shape where it measured slower (DESIGN.md §5); not with the W1-before-propagation "
                         "--overlap (its chunked gather runs in original ids)")
    ap.add_argument("--engine", default="decoupled", choices=["decoupled", "coupled", "dp", "gat"],
                    help="coupled: NEXT-1, the naive tensor-parallel 2-layer GCN (d_in -> hid -> C) with its "
                         "communication ledger, the paper's TP-vs-DTP ablation (P:696, P:1125-1128); dp: NEXT-4, the "
                         "data-parallel baseline (full-width rows, all-gather before each hop; load imbalance); gat: "
                         "NEXT-2, the decoupled GAT epoch (attention precomputed once, weighted hops, W1 before "
                         "propagation, alpha = 0)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-epochs", type=int, default=3)
    ap.add_argument("--no-hbm-leg", action="store_true", help="skip the HBM-bound Orkut-shaped propagation leg")
    ap.add_argument("--trace", default=None,
                    help="after the timed steps, one more epoch with the overlap trace on (ntp_set_trace): JSONL of "
                         "per-chunk begin/end on the compute and comm streams to PATH.rank<r>.jsonl, summary in the line")
    ap.add_argument("--host-stream", action="store_true",
                    help="NEXT-3: keep X_v in pinned host memory and stream its row chunks (NTP_M_HOST_STREAM; "
                         "W1-after-propagation configs, e.g. --config papers --dtype f32)")
    ap.add_argument("--leg-steps", type=int, default=3)
    ap.add_argument("--e2e-steps", type=int, default=30,
                    help="steps of the pipelined e2e loop (at least --steps): the loop's fill (the first copy, "
                         "not overlapped) is paid once per loop, as in a training run")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = synth.get_config(args.config)

    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return

    import torch
    from paper_2412_20379_b200 import ntp

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # NCCL bootstrap id for the library's own communicator
    uid = None
    if world > 1:
        obj = [ntp.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    dtype_name = args.dtype or ("bf16" if cfg.name.startswith("papers") else "f32")
    dt = ntp.NTP_BF16 if dtype_name == "bf16" else ntp.NTP_F32
    if args.slice_align == "auto":
        args.slice_align = auto_slice_align(cfg, world, dt, args.engine,
                                            torch.cuda.get_device_properties(local).L2_cache_size)
    args.slice_align = int(args.slice_align)
    ctx = ntp.Context(device=local, rank=rank, world=world, unique_id=uid, slice_align=args.slice_align)

    t0 = time.time()
    # the last-hop chunked gather of --overlap needs original ids; the W1-after-propagation epoch overlaps its
    # layout changes by row chunk instead and keeps the reorder
    reorder = args.engine not in ("dp", "gat") and (args.reorder == "on" or (args.reorder == "auto" and cfg.n >= 1_000_000)) and \
        (not args.overlap or cfg.w_after_prop)
    ctx.generate_rmat(cfg.n, cfg.scale, cfg.m_raw, synth.rmat_thresholds(*cfg.abc), cfg.seed, cfg.symmetric,
                      reorder=reorder)
    n, nnz, sym = ctx.graph_info()
    t_graph = time.time() - t0

    part = ntp.partition(n, cfg.w, world, dt, args.chunks, args.slice_align)
    V_p, d_s = part["V_p"], part["d_s"]
    if args.engine == "dp":   # every rank aggregates full-width rows
        d_s = ntp.partition(n, cfg.w, 1, dt, 1, args.slice_align)["d_s"]
    row0 = rank * V_p
    rows = max(0, min(V_p, n - row0))
    W0h, W1h = synth.model_weights(cfg)
    ldx = (cfg.d_in + 3) // 4 * 4          # 16-byte row pitch: the MLP GEMMs read X_v with TMA, no staging copy
    X = torch.zeros(V_p, ldx, dtype=torch.float32, device="cuda")[:, :cfg.d_in]
    y = torch.zeros(V_p, dtype=torch.int32, device="cuda")
    msk = torch.zeros(V_p, dtype=torch.uint8, device="cuda")
    if rows:
        # the same formulas evaluated on the device (synth.config_inputs_device, pinned bitwise against
        # the numpy version in tests/test_synth.py): papers-scale inputs in seconds instead of minutes
        synth.config_inputs_device(cfg, row0, rows, device="cuda", out=(X, y, msk))
    if args.host_stream:   # NEXT-3: the inputs live in pinned host memory; HBM holds only row chunks of them
        Xp = torch.zeros(V_p, ldx, dtype=torch.float32).pin_memory()[:, :cfg.d_in]
        Xp.copy_(X)
        del X
        torch.cuda.empty_cache()
        X = Xp
        args.no_e2e = True
    Xh = yh = mh = None
    if not args.no_e2e:
        Xh, yh, mh = X.cpu().contiguous().numpy(), y.cpu().numpy(), msk.cpu().numpy()
    x_bytes = V_p * cfg.d_in * 4
    W0 = torch.from_numpy(W0h).cuda()
    W1 = torch.from_numpy(W1h).cuda()
    flags = ((ntp.NTP_M_W1_AFTER_PROP if cfg.w_after_prop else 0) | (ntp.NTP_M_OVERLAP if args.overlap else 0)
             | (ntp.NTP_M_DATA_PARALLEL if args.engine == "dp" else 0)
             | (ntp.NTP_M_P2P_LAYOUTS if args.layouts == "p2p" else 0))
    model = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=cfg.K, gamma=cfg.gamma, alpha=cfg.alpha, lr=cfg.lr,
                 dtype=dt, chunks=args.chunks, flags=flags)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    if args.engine == "gat":
        run_gat(args, ctx, cfg, X, y, msk, n, nnz, world, rank, dist, barrier, stream, dt, dtype_name, V_p)
        ctx.close()
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    if args.engine == "coupled":
        run_coupled(args, ctx, cfg, X, y, msk, n, nnz, world, rank, local, dist, barrier, stream, dt, dtype_name,
                    V_p, reorder)
        ctx.close()
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- warm-up (the first epochs start from the same weights as the oracle leg: parity check below)
    warm_losses = []
    for _ in range(args.warmup):
        warm_losses.append(ctx.train_epoch(model, X, y, msk, W0, W1, stream=stream, host_stream=args.host_stream)["loss"])
    # ---- timed (device events on the caller's stream; the library orders its streams after it)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = []
    ev0.record(stream)
    for _ in range(args.steps):
        reps.append(ctx.train_epoch(model, X, y, msk, W0, W1, stream=stream, host_stream=args.host_stream))
    ev1.record(stream)
    barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    clk = clocks.stop()
    spmm_ms = sum(r["spmm_ms"] for r in reps)
    spmm_n = sum(r["spmm_launches"] for r in reps)
    launches = sum(r["kernel_launches"] for r in reps)
    phase = {k: sum(r["ms"][k] for r in reps) / len(reps) for k in reps[0]["ms"]}

    # ---- overlap trace (outside the timed region): one eager epoch with per-chunk events on both streams
    trace_summary = None
    if args.trace:
        ctx.set_trace(True)
        ctx.train_epoch(model, X, y, msk, W0, W1, stream=stream, host_stream=args.host_stream)
        tr = ctx.trace()
        ctx.set_trace(False)
        path = f"{args.trace}.rank{rank}.jsonl"
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as f:
            for r in tr:
                f.write(json.dumps(dict(r, rank=rank)) + "\n")

        def union(iv):
            out = []
            for b, e in sorted(iv):
                if out and b <= out[-1][1]:
                    out[-1][1] = max(out[-1][1], e)
                else:
                    out.append([b, e])
            return out

        comm = union([(r["begin_ms"], r["end_ms"]) for r in tr if r["stream"] == "comm"])
        comp = union([(r["begin_ms"], r["end_ms"]) for r in tr if r["stream"] == "compute"])
        comm_ms = sum(e - b for b, e in comm)
        hidden = sum(max(0.0, min(e, e2) - max(b, b2)) for b, e in comm for b2, e2 in comp)
        trace_summary = {"file": path, "records": len(tr), "comm_busy_ms": comm_ms,
                         "comm_hidden_under_compute_ms": hidden,
                         "hidden_frac": hidden / comm_ms if comm_ms else None,
                         "note": "rank 0's trace of one eager epoch after the timed steps (ntp_set_trace); compute "
                                 "intervals: per-chunk MLP forward / head / MLP backward and the hops"}

    # ---- e2e: same call with HOST (pinned) inputs copied in every step, loss read back
    e2e_ms = e2e_serial_ms = None
    h2d = V_p * ldx * 4 + V_p * 4 + V_p      # the padded host rows are what crosses PCIe
    if not args.no_e2e:
        # pinned host rows in the 16-byte pitch the GEMMs read (ldx floats), so each step is one plain DMA
        Xp = torch.zeros(V_p, ldx, dtype=torch.float32).pin_memory()[:, :cfg.d_in]
        Xp.copy_(torch.from_numpy(Xh))
        yp = torch.from_numpy(yh).pin_memory()
        mp = torch.from_numpy(mh).pin_memory()
        for _ in range(2):
            ctx.train_epoch(model, Xp, yp, mp, W0, W1, stream=stream, host_inputs=True)
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            ctx.train_epoch(model, Xp, yp, mp, W0, W1, stream=stream, host_inputs=True)
        ev1.record(stream)
        barrier()
        e2e_serial_ms = ev0.elapsed_time(ev1) / args.steps
        # pipelined loop (ntp_stage_inputs): every step still copies its own inputs from pinned host memory
        # and reads its loss back, but the copies of steps i+1 and i+2 run on the copy engine while step i
        # computes (three slots: the copy engine never waits for an epoch to release a slot)
        ns = ntp.NTP_STAGE_SLOTS
        for i in range(2 * ns):   # eager run per slot, then each slot's epoch graph is captured
            ctx.stage_inputs(i % ns, Xp, yp, mp)
            ctx.train_epoch(model, Xp, yp, mp, W0, W1, stream=stream, staged_slot=i % ns)
        barrier()
        e2e_steps = max(args.steps, args.e2e_steps)
        ev0.record(stream)
        for i in range(min(ns - 1, e2e_steps)):
            ctx.stage_inputs(i % ns, Xp, yp, mp)
        for i in range(e2e_steps):
            if i + ns - 1 < e2e_steps:
                ctx.stage_inputs((i + ns - 1) % ns, Xp, yp, mp)
            ctx.train_epoch(model, Xp, yp, mp, W0, W1, stream=stream, staged_slot=i % ns)
        ev1.record(stream)
        barrier()
        e2e_ms = ev0.elapsed_time(ev1) / e2e_steps

    def allmax(v):
        if dist is None or v is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    free_b, total_b = torch.cuda.mem_get_info()
    hbm_used_gb = allmax((total_b - free_b) / 1e9)
    peaks = load_peaks()
    if peaks and peaks.get("hbm_gbs"):
        peak, peak_src = peaks["hbm_gbs"], "measured (MEASURED_PEAKS.json hbm_gbs)"
    else:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    l2_size = torch.cuda.get_device_properties(local).L2_cache_size
    # layout changes timed inside the epoch (CUDA events): bytes handed to NCCL per rank / phase time
    nvlink = None
    if world > 1:
        names = [("v2f_fwd", 0, "pack + all-to-all"), ("f2v_fwd", 1, "all-to-all"), ("v2f_bwd", 2, "all-to-all"),
                 ("f2v_bwd", 3, "all-to-all + unpack")]
        nvlink = {}
        # with --overlap the exchange runs in chunks under the hops (and the data-parallel baseline all-gathers
        # before every hop), so a phase's time is not the transfer's: bytes only, see a2a_standalone for the rate
        confined = not args.overlap and args.engine == "decoupled"
        for ph, i, what in names:
            t_ph = allmax(phase[ph])
            b = reps[-1]["bytes_sent"][i]
            ok = confined and bool(t_ph)
            nvlink[ph] = {"ms": t_ph, "bytes_sent_per_rank": b, "what": what,
                          "GBps_per_direction": (b / (t_ph * 1e-3) / 1e9) if ok else None,
                          "frac_of_900GBps": (b / (t_ph * 1e-3) / 1e9 / 900.0) if ok else None}
            if not confined:
                nvlink[ph]["note"] = "exchange overlapped with other phases: no per-phase rate"
    # the layout change timed on its own (SURVEY §8(d) "measure the a2a separately at the same counts"):
    # ntp_layout_v2f of this rank's [V_p x w] rows (pack + block all-to-all) into the feature slice
    a2a = None
    if world > 1 and args.engine == "decoupled":
        Hv_a = torch.zeros(V_p, w_prop := (cfg.hid if cfg.w_after_prop else cfg.C), dtype=torch.float32 if dt == ntp.NTP_F32
                           else torch.bfloat16, device="cuda")
        Hf_a = torch.empty(V_p * world, d_s, dtype=Hv_a.dtype, device="cuda")
        for _ in range(3):
            ctx.layout_v2f(Hv_a, Hf_a, stream)
        barrier()
        ev0.record(stream)
        for _ in range(10):
            ctx.layout_v2f(Hv_a, Hf_a, stream)
        ev1.record(stream)
        barrier()
        t_a2a = allmax(ev0.elapsed_time(ev1) / 10)
        b_a2a = (world - 1) * V_p * d_s * (2 if dt == ntp.NTP_BF16 else 4)
        a2a = {"ms": t_a2a, "bytes_sent_per_rank": b_a2a, "what": "ntp_layout_v2f: pack + block all-to-all, standalone",
               "GBps_per_direction": b_a2a / (t_a2a * 1e-3) / 1e9,
               "frac_of_900GBps": b_a2a / (t_a2a * 1e-3) / 1e9 / 900.0}
        del Hv_a, Hf_a
    leg = None
    if not args.no_hbm_leg and args.engine == "decoupled" and args.config == "reddit":
        leg = hbm_leg(args, world, rank, local, dist, barrier, allmax, peak, peak_src, l2_size)
    ms = allmax(ms)
    e2e_ms = allmax(e2e_ms)
    e2e_serial_ms = allmax(e2e_serial_ms)
    own_hop = spmm_ms / max(spmm_n, 1)
    spmm_avg = allmax(own_hop)
    hop_min = own_hop if dist is None else -allmax(-own_hop)   # per-rank hop time spread (load balance)
    # items (gathered rows: self + arcs) one hop launch processes: the whole graph on every feature slice; in the
    # data-parallel baseline only this rank's destination rows -- its roofline is the critical (slowest) rank's
    hop_items = nnz + n
    if args.engine == "dp":
        rp = ctx.copy_csr(False)[0]
        lo, hi = min(row0, n), min(row0 + V_p, n)
        own_items = int(rp[hi] - rp[lo]) + (hi - lo)
        if dist is None:
            hop_items = own_items
        else:
            t = torch.tensor([own_hop, float(own_items)], dtype=torch.float64, device="cuda")
            allt = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(allt, t)
            crit = max(allt, key=lambda x: float(x[0]))
            hop_items = int(crit[1])

    if rank == 0:
        w = cfg.w
        esz = 2 if dt == ntp.NTP_BF16 else 4
        ge = 2 * cfg.K * nnz * w / (ms * 1e-3) / 1e9
        bh, bmodel = hop_bytes(n, nnz, d_s, esz, sym, cfg.alpha, l2_size)
        bh = bh * hop_items / (nnz + n)          # dp: the critical rank's share of the arcs
        achieved = bh / (spmm_avg * 1e-3) / 1e9
        d_s16 = ntp.partition(n, cfg.w, world, dt, 1, 16)["d_s"]
        # (the data-parallel baseline gathers full-width rows of part of the graph: no capture matches it)
        traffic = None if args.engine == "dp" else load_traffic(args.config, world, dtype_name,
                                                                d_s if d_s != d_s16 else None)
        l2b = l2_gather_bytes(nnz, n, d_s, esz)
        gc = gather_ceiling(n, d_s * esz, l2_size)
        gather_line = None
        if gc:
            rows_ps = hop_items / (spmm_avg * 1e-3)
            gather_line = dict(gc, achieved_rows_per_s=rows_ps, frac=rows_ps / gc["rows_per_s"],
                               row_bytes=d_s * esz)
        # The hop's roofline by residency: a slice that exceeds L2 is HBM-bound (measured DRAM
        # bytes of this kernel / its live time against the measured copy peak); a slice that fits L2 reads HBM
        # only for its compulsory bytes and is bound by the L2 random-row gather rate: its rows / s against the
        # measured ceiling of the same access pattern (scripts/l2_probe.cu, random rows of the same size from an
        # L2-resident table).  The other resource's numbers stay in the block.
        hbm = {"achieved": (traffic if traffic else bh) / (spmm_avg * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
               "traffic": traffic, "peak_source": peak_src,
               "bytes_model": ("ncu DRAM read + write bytes per launch (profiles/spmm_traffic.json)" if traffic
                               else bmodel),
               "algorithmic_bytes_per_launch": bh, "algorithmic_model": bmodel}
        hbm["frac"] = hbm["achieved"] / peak
        common = {"kernel": "spmm_hop_bulk_kernel" if d_s * esz >= 1024 else "spmm_hop_kernel",
                  "avg_launch_ms": spmm_avg, "launches_timed": spmm_n,
                  "timed_span": "the hop kernel + its spmm_fixup_kernel (cut-row carries, ~1% of the span), CUDA "
                                "events on the hop's stream"}
        if bmodel.startswith("perfect") and gather_line:
            rb = gather_line["probe_row_bytes"]
            roof = dict(common, bound="l2", unit="GB/s",
                        achieved=gather_line["achieved_rows_per_s"] * rb / 1e9,
                        peak=gather_line["rows_per_s"] * rb / 1e9, frac=gather_line["frac"],
                        peak_source="measured: random-row gather ceiling from an L2-resident table, rows of "
                                    f"{rb} B ({gather_line['source']}, scripts/l2_probe.cu); MEASURED_PEAKS.json "
                                    "has no L2 figure",
                        traffic=traffic, bytes_model="gathered rows (self + every arc) x row bytes, per launch",
                        algorithmic_bytes_per_launch=hop_items * rb,
                        l2_gather_GBps=l2b * hop_items / (nnz + n) / (spmm_avg * 1e-3) / 1e9,
                        hbm=hbm, gather=gather_line)
        else:
            roof = dict(common, bound="hbm", **hbm, gather=gather_line)
        line = {
            "metric": METRIC, "value": ge, "unit": "GE/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32" if dt == ntp.NTP_F32 else "bf16", "data": "synthetic",
            "epoch_s": ms / 1e3,
            "engine": {"decoupled": "decoupled tensor parallelism (NeutronTP)",
                       "dp": "data-parallel baseline (NEXT-4): full-width rows, all-gather before every hop"}[args.engine],
            "load_balance": {"hop_ms_max_rank": spmm_avg, "hop_ms_min_rank": hop_min,
                             "max_over_min": spmm_avg / hop_min if hop_min else None},
            "config": {"workload": WORKLOADS.get(args.config, args.config), "n": n, "nnz": nnz, "w": w, "K": cfg.K,
                       "gamma": cfg.gamma, "alpha": cfg.alpha, "P": world, "d_s": d_s, "slice_align": args.slice_align,
                       "V_p": V_p,
                       "chunks": args.chunks, "overlap": bool(args.overlap),
                       "inputs": "pinned host memory, streamed per row chunk (NTP_M_HOST_STREAM)" if args.host_stream
                                 else "device-resident",
                       "vertex_order": "degree-ordered internally (NTP_G_REORDER)" if reorder else "R-MAT ids",
                       "layouts": ("copy-engine peer copies per row chunk (overlapped)"
                                   if args.layouts == "p2p" and args.overlap and cfg.w_after_prop
                                   else "peer-direct IPC stores" if args.layouts == "p2p" and not args.overlap
                                   else "NCCL all-to-all") if world > 1 else "local",
                       "l2": f"inputs larger than L2 (col_idx {4 * nnz / 1e6:.0f} MB streamed per hop; "
                             f"X_v {x_bytes / 1e6:.0f} MB per rank)",
                       "graph_setup_s": round(t_graph, 3), "hbm_used_GB_max_rank": round(hbm_used_gb, 1)},
            "roofline": roof,
            "prop_GE_per_s": 2 * cfg.K * nnz * w / (spmm_ms / len(reps) * 1e-3) / 1e9 * 1.0,
            "phase_ms": {k: round(v, 4) for k, v in phase.items()},
            "nvlink": nvlink,
            "a2a_standalone": a2a,
            "hbm_leg": leg,
            "clocks": clk,
            **({"overlap_trace": trace_summary} if trace_summary else {}),
            "gpu_launches": int(launches),
            "losses": {"warmup": warm_losses, "timed_last": reps[-1]["loss"]},
            "e2e": None if e2e_ms is None else {
                "value": 2 * cfg.K * nnz * w / (e2e_ms * 1e-3) / 1e9, "unit": "GE/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 16,
                "loop": "ntp_stage_inputs: the host->device copies of steps i+1 and i+2 overlap step i (three device slots)",
                "steps": e2e_steps,
                "serial_ms_per_step": e2e_serial_ms,
                "serial_value": 2 * cfg.K * nnz * w / (e2e_serial_ms * 1e-3) / 1e9},
        }
        if world == 1 and not args.no_cpu_baseline and cfg.n > 10_000_000:
            import oracle
            est = oracle_sampled_estimate(cfg)
            line["cpu_baseline"] = {"value": 2 * cfg.K * nnz * w / est["epoch_s"] / 1e9, "unit": "GE/s",
                                    "cores": oracle.lib.oracle_num_threads(), "kind": "oracle", "extrapolated": True,
                                    "epoch_s": est["epoch_s"], "host": host_info(), "detail": est,
                                    "sample": f"EXTRAPOLATED: fp64 oracle hop on {est['cols']} of {cfg.w} columns over a "
                                              f"{est['frac']:.0%} row sample ({est['sample_arcs']} arcs) plus the MLP "
                                              f"and loss on a {est['frac']:.0%} row sample, scaled linearly "
                                              f"(SURVEY §8(d)); the full fp64 state is ~1 TB"}
        elif world == 1 and not args.no_cpu_baseline:
            try:
                t_cpu, nnz_o, cores, _, o_losses, hop1 = oracle_epoch_time(cfg, args.cpu_epochs)
                line["cpu_baseline"] = {"value": 2 * cfg.K * nnz_o * w / t_cpu / 1e9, "unit": "GE/s",
                                        "cores": cores, "kind": "oracle", "epoch_s": t_cpu,
                                        "sample": f"{args.cpu_epochs} full fp64 oracle epochs of the same workload "
                                                  f"(graph build excluded), OpenMP over rows + numpy BLAS",
                                        "host": host_info(),
                                        "hop_1thread_s": hop1,
                                        "hop_1thread_note": "one forward hop on 1 thread, timed on a 2% row sample "
                                                            "and extrapolated linearly to all rows"}
                # parity of the bench workload itself: the GPU's first epochs (warm-up, same initial weights)
                # against the oracle's, loss by loss (R10: 1e-4 for fp32 slices, 2e-2 |loss| for bf16)
                k = min(len(o_losses), len(warm_losses))
                errs = [abs(warm_losses[i] - o_losses[i]) for i in range(k)]
                tol = 1e-4 if dt == ntp.NTP_F32 else 2e-2 * abs(o_losses[0])
                line["parity"] = {"epochs": k, "loss_gpu": warm_losses[:k], "loss_oracle": o_losses[:k],
                                  "abs_err": max(errs) if errs else None, "tol": tol,
                                  "pass": bool(errs) and max(errs) <= tol}
            except Exception as e:  # pragma: no cover
                line["cpu_baseline"] = {"value": None, "unit": "GE/s", "cores": os.cpu_count(), "kind": "oracle",
                                        "sample": f"failed: {e}"}
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
