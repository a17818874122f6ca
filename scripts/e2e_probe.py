"""Where does the e2e loop lose against max(H2D copy, epoch)?  Hop time and epoch phases with and without the
staged copy of the next step's inputs running concurrently (Reddit shape, N = 1)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth
from paper_2412_20379_b200 import ntp

cfg = synth.get_config("reddit")
ctx = ntp.Context()
ctx.generate_rmat(cfg.n, cfg.scale, cfg.m_raw, synth.rmat_thresholds(*cfg.abc), cfg.seed, cfg.symmetric)
ldx = (cfg.d_in + 3) // 4 * 4
X = torch.zeros(cfg.n, ldx, device="cuda")[:, :cfg.d_in]
y = torch.zeros(cfg.n, dtype=torch.int32, device="cuda")
m = torch.zeros(cfg.n, dtype=torch.uint8, device="cuda")
synth.config_inputs_device(cfg, 0, cfg.n, out=(X, y, m))
Xp = torch.zeros(cfg.n, ldx).pin_memory()[:, :cfg.d_in]
Xp.copy_(X.cpu())
yp, mp = y.cpu().pin_memory(), m.cpu().pin_memory()
W0, W1 = (torch.from_numpy(a).cuda() for a in synth.model_weights(cfg))
model = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=cfg.K, gamma=cfg.gamma, alpha=cfg.alpha, lr=cfg.lr)
for mode in ("device", "staged"):
    reps = []
    for i in range(12):
        if mode == "device":
            r = ctx.train_epoch(model, X, y, m, W0, W1)
        else:
            if i == 0:
                ctx.stage_inputs(0, Xp, yp, mp)
            ctx.stage_inputs((i + 1) % 2, Xp, yp, mp)
            r = ctx.train_epoch(model, Xp, yp, mp, W0, W1, staged_slot=i % 2)
        reps.append(r)
    reps = reps[4:]
    hop = sum(r["spmm_ms"] for r in reps) / sum(r["spmm_launches"] for r in reps)
    ph = {k: round(sum(r["ms"][k] for r in reps) / len(reps), 3) for k in reps[0]["ms"]}
    print(mode, "hop ms", round(hop, 4), ph, flush=True)

# the copy engine's H2D under a running epoch: one 564 MB pinned copy on a side stream while epochs run
src = torch.empty(564_008_265 // 4, dtype=torch.float32).pin_memory()
dst = torch.empty_like(src, device="cuda")
side = torch.cuda.Stream()
for load in (False, True, True):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(side):
        e0.record(side)
        dst.copy_(src, non_blocking=True)
        e1.record(side)
    if load:
        for _ in range(2):
            ctx.train_epoch(model, X, y, m, W0, W1)
    torch.cuda.synchronize()
    print("copy under epochs" if load else "copy alone", round(e0.elapsed_time(e1), 3), "ms", flush=True)
