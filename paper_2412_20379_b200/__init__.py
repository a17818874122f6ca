"""paper_2412_20379_b200 — B200-native feature-sliced decoupled-GNN propagation (NeutronTP hot path).

The product is the C-ABI library ``libntp.so`` (include/ntp.h); ``paper_2412_20379_b200.ntp``
is its ctypes binding.  Importing ``ntp`` fails loudly if the library is not built.
"""
