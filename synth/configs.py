"""Workload recipes (BASELINE.json `configs`).

Each config fixes the synthetic graph (R-MAT size, quadrant probabilities,
raw arc count, symmetry), the model shape and the propagation parameters.
Values only — no arithmetic of the method.

R-MAT raw counts `m_raw` were calibrated with the oracle's generator
(scripts/calibrate_rmat.py) so that the deduplicated arc count lands near the
paper's |E| (Table 1).
"""
from __future__ import annotations

from dataclasses import dataclass, field

GRAPH500 = (0.57, 0.19, 0.19)
REDDIT_ABC = (0.45, 0.22, 0.22)


@dataclass(frozen=True)
class Config:
    name: str
    seed: int
    n: int                 # |V|
    scale: int             # R-MAT levels (ids drawn in [0, 2^scale), rejected if >= n)
    m_raw: int             # raw R-MAT arcs drawn
    abc: tuple             # quadrant probabilities (a, b, c)
    symmetric: bool        # append reverse arcs (undirected graph)
    d_in: int
    hid: int
    C: int
    K: int
    gamma: float
    alpha: float
    binary_density: float | None = None   # Cora-shaped binary features
    w_after_prop: bool = False             # propagate hid and apply W1 after (R3, c5)
    lr: float = 0.01
    note: str = ""

    @property
    def w(self) -> int:
        """Propagated width: min(hid, C)."""
        return self.hid if self.w_after_prop else self.C


CONFIGS: dict[str, Config] = {}


def _add(c: Config):
    CONFIGS[c.name] = c


# c1: Cora-shaped (2,708 vertices, ~10.5K arcs, 1433 binary features, 7 classes), 2-hop decoupled GCN
_add(Config("cora", 1, 2708, 12, 6_800, GRAPH500, True, 1433, 64, 7, 2, 1.0, 0.0,
            binary_density=0.0127, note="BASELINE configs[0]"))
# c2: Reddit-shaped (233K vertices, ~114M arcs, 602 features, 41 classes), K=2
_add(Config("reddit", 2, 232_965, 18, 62_400_000, REDDIT_ABC, True, 602, 256, 41, 2, 1.0, 0.0,
            note="BASELINE configs[1]; bench workload at N=1"))
# c3: ogbn-products-shaped (2.45M vertices, ~62M arcs, 100 features, 47 classes), APPNP K=10
_add(Config("products", 3, 2_449_029, 22, 40_600_000, GRAPH500, True, 100, 64, 47, 10, 0.9, 0.1,
            note="BASELINE configs[2]; APPNP gamma=1-alpha, alpha=0.1 (R2)"))
# c4: Orkut-shaped (3.07M vertices, ~117M arcs, 512-wide pipeline)
_add(Config("orkut", 4, 3_072_441, 22, 69_000_000, GRAPH500, True, 512, 128, 64, 2, 1.0, 0.0,
            note="BASELINE configs[3]; d=512 propagation pipeline"))
# c5: ogbn-papers100M-shaped (111M vertices, ~1.6B arcs, directed, 128 features, 172 classes)
_add(Config("papers", 5, 111_059_956, 27, 1_693_000_000, GRAPH500, False, 128, 128, 172, 2, 1.0, 0.0,
            w_after_prop=True, note="BASELINE configs[4]; bf16 storage"))

# Small parity cases (several tiles, ragged tails, directed + symmetric, hubs)
_add(Config("tiny_sym", 11, 1000, 10, 6_000, GRAPH500, True, 24, 16, 5, 2, 1.0, 0.0))
_add(Config("tiny_dir", 12, 3001, 12, 40_000, GRAPH500, False, 33, 20, 7, 3, 0.9, 0.1,
            w_after_prop=True))
_add(Config("small_appnp", 13, 20_011, 15, 300_000, GRAPH500, True, 50, 32, 13, 10, 0.9, 0.1))
_add(Config("small_dir", 14, 50_000, 16, 800_000, REDDIT_ABC, False, 64, 48, 19, 2, 1.0, 0.0))
# High-degree parity cases (average degree >= 32, like the Reddit shape): the kernels' high-degree
# variants (streaming narrow-row hop) only run on these; hubs span several merge-path units
_add(Config("dense_sym", 16, 8_000, 13, 260_000, REDDIT_ABC, True, 40, 24, 9, 3, 0.9, 0.1))
_add(Config("dense_dir", 17, 6_007, 13, 420_000, REDDIT_ABC, False, 36, 16, 11, 2, 1.0, 0.0))
# W1-after-propagation with the papers head shape (hid 128 = P*d_s at every P, C = 172 over three
# 64-class boxes; C = 41 ragged in one box): the fused tcgen05 head (head.cu) runs on bf16 storage
_add(Config("head_dir", 18, 5_003, 13, 60_000, GRAPH500, False, 32, 128, 172, 2, 1.0, 0.0, w_after_prop=True))
_add(Config("head_sym", 19, 3_001, 12, 30_000, REDDIT_ABC, True, 24, 128, 41, 3, 0.9, 0.1, w_after_prop=True))


def get_config(name: str) -> Config:
    try:
        return CONFIGS[name]
    except KeyError as e:
        raise KeyError(f"unknown config {name!r}; known: {sorted(CONFIGS)}") from e

# Single-GPU proxy for one rank of the papers100M shape at P = 8 (same dims, 1/8 of the vertices and
# arcs, directed): used to profile the W1-after-propagation MLP/loss path, which the full graph only
# runs at P >= 4 (ncu cannot wrap a multi-rank command).
_add(Config("papers_slice8", 15, 13_882_495, 24, 211_625_000, GRAPH500, False, 128, 128, 172, 2, 1.0, 0.0,
            w_after_prop=True, note="profiling proxy; bf16 storage"))
