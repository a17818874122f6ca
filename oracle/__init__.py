"""NeutronTP hot-path ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU (fp64) implementation of what the
feature-sliced decoupled-GNN hot path computes (arXiv 2412.20379; SURVEY.md
§8(c) O1–O10).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product
package ``paper_2412_20379_b200`` never imports it and shares no code with it;
both sides only share the seeded input generators in ``synth/``.

Modules
  graph      O1/O2 + O10: R-MAT arcs (independent counter-based generator),
             CSR / transpose / degrees, D~^{-1/2}
  propagate  O3/O4: K-hop forward / backward (adjoint) propagation
  model      O5–O9: MLP, decoupled model function, loss, gradients, SGD epoch
  layout     a1/a3/a5: partition maps, vertex <-> feature layouts (definitions)
  coupled    NEXT-1: the coupled L-layer GCN that naive tensor parallelism trains (baseline)
  gat        NEXT-2: decoupled GAT (attention precomputed once per epoch, Eq. 5 / §4.1.1)

Parity pins live in tests/test_oracle_*.py.  Functions without a pin say
"parity unpinned" in their docstring (none at present).
"""
from ._lib import lib, build_oracle_lib  # noqa: F401
from . import graph, propagate, model, layout, coupled, gat  # noqa: F401
