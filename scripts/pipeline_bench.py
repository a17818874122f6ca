#!/usr/bin/env python
"""Vertex-layout propagation pipeline benchmark (the Orkut shape at
w = 512 run as split -> K hops -> gather and the backward mirror, with and without the chunked
overlap of the last hop with the gather, a12).  One rank per GPU:

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        scripts/pipeline_bench.py --config orkut --steps 5 --warmup 3 --chunks 4

Prints one JSON line per overlap setting (rank 0): ms per step (forward + backward pipeline,
max over ranks, CUDA events) and GE/s = 2*K*nnz*w / t.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="orkut")
    ap.add_argument("--width", type=int, default=None, help="propagated width (default: d_in)")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--chunks", type=int, default=4)
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    uid = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [ntp.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    cfg = synth.get_config(args.config)
    w = args.width or cfg.d_in
    ctx = ntp.Context(device=local, rank=rank, world=world, unique_id=uid)
    # the overlapped gather needs destination blocks in original order: no NTP_G_REORDER here
    ctx.generate_rmat(cfg.n, cfg.scale, cfg.m_raw, synth.rmat_thresholds(*cfg.abc), cfg.seed, cfg.symmetric)
    n, nnz, _ = ctx.graph_info()
    V_p = -(-n // world)
    row0 = rank * V_p
    rows = max(0, min(V_p, n - row0))
    # timing input: seeded uniform [-1, 1) rows drawn on the device (values do not affect the work)
    gen = torch.Generator(device="cuda").manual_seed(cfg.seed * 1000 + rank)
    Hv = torch.rand(V_p, w, device="cuda", generator=gen) * 2 - 1
    Hv[rows:] = 0
    Zv = torch.empty_like(Hv)
    Gv = torch.empty_like(Hv)
    dt = ntp.NTP_BF16 if args.dtype == "bf16" else ntp.NTP_F32
    stream = torch.cuda.current_stream()

    def step(overlap):
        ctx.propagate_pipeline(Hv, Zv, cfg.K, cfg.gamma, cfg.alpha, transposed=False, dtype=dt, chunks=args.chunks,
                               overlap=overlap, stream=stream)
        ctx.propagate_pipeline(Zv, Gv, cfg.K, cfg.gamma, cfg.alpha, transposed=True, dtype=dt, chunks=args.chunks,
                               overlap=overlap, stream=stream)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for overlap in (False, True):
        for _ in range(args.warmup):
            step(overlap)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step(overlap)
        e1.record(stream)
        barrier()
        ms = e0.elapsed_time(e1) / args.steps
        if dist is not None:
            t = torch.tensor([ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        if rank == 0:
            print(json.dumps(dict(workload=f"{args.config} pipeline (split -> {cfg.K} hops -> gather, fwd + bwd)",
                                  n=n, nnz=nnz, w=w, K=cfg.K, P=world, dtype=args.dtype, chunks=args.chunks,
                                  overlap=overlap, ms_per_step=round(ms, 3),
                                  GE_per_s=round(2 * cfg.K * nnz * w / (ms * 1e-3) / 1e9, 1))), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
