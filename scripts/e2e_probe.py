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
