"""Host-side logic of bench.py (no GPU): the slice-padding rule, the roofline's residency test and byte
model, and the gather-ceiling lookup against the committed probe table."""
import json
import os

import bench
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L2 = 132_644_864      # B200: cudaDevAttrL2CacheSize


def test_auto_slice_align_rule():
    from paper_2412_20379_b200 import ntp
    F32, BF16 = ntp.NTP_F32, ntp.NTP_BF16
    # Reddit: 176-B rows at N = 1 stay, 96 -> 128 B at N = 2, 48 -> 64 B at N = 4, 32 B at N = 8 stays
    assert [bench.auto_slice_align(synth.get_config("reddit"), w, F32, "decoupled", L2) for w in (1, 2, 4, 8)] \
        == [16, 128, 64, 16]
    # HBM-resident slices (products, papers, orkut) never pad; nor do the coupled / data-parallel engines
    for name, dt in (("products", F32), ("papers", BF16), ("orkut", F32)):
        assert {bench.auto_slice_align(synth.get_config(name), w, dt, "decoupled", L2) for w in (1, 2, 4, 8)} == {16}
    for engine in ("coupled", "dp"):
        assert bench.auto_slice_align(synth.get_config("reddit"), 2, F32, engine, L2) == 16
    # the padded width is a multiple of the chosen alignment and adds at most a third of the bytes
    for w, a in ((2, 128), (4, 64)):
        d16 = ntp.partition(232_965, 41, w, F32, 1, 16)["d_s"]
        da = ntp.partition(232_965, 41, w, F32, 1, a)["d_s"]
        assert da * 4 % a == 0 and 3 * da <= 4 * d16


def test_hop_bytes_by_residency():
    n, nnz = 232_965, 114_082_446
    lo, model = bench.hop_bytes(n, nnz, 44, 4, True, 0.0, L2)            # 41 MB slice: fits L2
    assert model.startswith("perfect") and lo == 4 * nnz + 4 * (n + 1) + 4 * n + n * 176 * 2
    hi, model = bench.hop_bytes(2_449_029, 61_859_140, 48, 4, True, 0.1, L2)   # 470 MB slice
    assert model.startswith("no reuse")
    lo2 = 4 * 61_859_140 + 4 * (2_449_029 + 1) + 4 * 2_449_029 + 2_449_029 * 192 * 3
    assert hi == lo2 + 61_859_140 * 192


def test_gather_ceiling_lookup():
    tab = json.load(open(os.path.join(ROOT, "profiles", "gather_ceiling.json")))["l2_resident"]
    g = bench.gather_ceiling(232_965, 176, L2)
    assert g["residency"] == "L2" and g["probe_row_bytes"] == 176
    assert g["rows_per_s"] == tab["176"]["Grows_per_s"] * 1e9
    assert bench.gather_ceiling(232_965, 128, L2)["probe_row_bytes"] == 128    # the padded N = 2 slice
    assert bench.gather_ceiling(232_965, 44, L2)["probe_row_bytes"] == 48      # smallest probe >= the row
    assert bench.gather_ceiling(111_059_956, 256, L2)["residency"] == "HBM"


def test_traffic_lookup_by_padded_width():
    assert bench.load_traffic("reddit", 2, "f32") != bench.load_traffic("reddit", 2, "f32", 32)
    assert bench.load_traffic("reddit", 2, "f32", 32) is not None
    assert bench.load_traffic("reddit", 2, "f32", 999) is None
    assert bench.load_traffic("nosuch", 1, "f32") is None
