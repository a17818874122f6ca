#!/usr/bin/env python
"""Development tool: deduplicated arc count of a config's R-MAT graph built on the GPU for several m_raw."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2412_20379_b200 import ntp  # noqa: E402

cfg = synth.get_config(sys.argv[1])
ctx = ntp.Context()
for m in [int(x) for x in sys.argv[2].split(",")]:
    t = time.time()
    ctx.generate_rmat(cfg.n, cfg.scale, m, synth.rmat_thresholds(*cfg.abc), cfg.seed, cfg.symmetric)
    n, nnz, sym = ctx.graph_info()
    free, total = torch.cuda.mem_get_info()
    print(f"m_raw={m} nnz={nnz} ratio={nnz / m:.4f} build_s={time.time() - t:.2f} "
          f"free_GB={free / 1e9:.1f} peak_alloc_GB={torch.cuda.max_memory_allocated() / 1e9:.1f}", flush=True)
