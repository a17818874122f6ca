"""CPU-only checks of the C-ABI library: it loads, exports every symbol the public
header declares, its pure-host partition maps match the oracle's definition, and
it reports errors (not crashes) when no GPU is present."""
import os
import re

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ntp():
    from paper_2412_20379_b200 import build
    build.build(verbose=False)
    from paper_2412_20379_b200 import ntp
    return ntp


def _declared():
    src = open(os.path.join(ROOT, "include", "ntp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ntp_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(ntp):
    decl = _declared()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(ntp._lib, name), name
    assert sorted(ntp.EXPORTED) == decl


def test_abi_version_and_status_strings(ntp):
    assert ntp.abi_version() == 1
    assert ntp._lib.ntp_status_string(ntp.NTP_ERR_GRAPH) == b"NTP_ERR_GRAPH"


@pytest.mark.parametrize("n,w,P,dt,align", [(232_965, 41, 8, 0, 16), (232_965, 41, 1, 0, 32), (17, 10, 3, 0, 16),
                                            (111_059_956, 128, 8, 1, 16), (5, 3, 8, 1, 32), (2708, 7, 1, 0, 16),
                                            (232_965, 41, 2, 0, 128), (232_965, 41, 4, 0, 64), (99, 20, 3, 1, 64)])
def test_partition_matches_oracle(ntp, n, w, P, dt, align):
    eb = 2 if dt == 1 else 4
    got = ntp.partition(n, w, P, dt, chunks=3, slice_align=align)
    ref = oracle.layout.partition(n, w, P, eb, chunks=3, align=align)
    assert got["V_p"] == ref["V_p"] and got["V_pad"] == ref["V_pad"]
    assert got["d_s"] == ref["d_s"] and got["w_pad"] == ref["w_pad"]
    assert got["chunk"] == ref["chunk"]


def test_bad_arguments_are_errors_not_crashes(ntp):
    import ctypes as C
    h = C.c_void_p()
    assert ntp._lib.ntp_create(C.byref(h), 0, 2, 2, None, 16) == ntp.NTP_ERR_ARG   # rank >= world
    assert ntp._lib.ntp_create(C.byref(h), 0, 0, 1, None, 24) == ntp.NTP_ERR_ARG   # bad align
    assert ntp._lib.ntp_create(None, 0, 0, 1, None, 16) == ntp.NTP_ERR_ARG
    assert ntp._lib.ntp_load_graph(None, None, None, 0, 0, 0) == ntp.NTP_ERR_ARG


def test_no_gpu_create_reports_error(ntp):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(ntp.NtpError):
        ntp.Context()


def test_binding_constants_match_header(ntp):
    """Every NTP_* integer macro the binding mirrors has the header's value (include/ntp.h)."""
    hdr = open(os.path.join(ROOT, "include", "ntp.h")).read()
    macros = dict(re.findall(r"^#define\s+(NTP_\w+)\s+\(?(-?\d+)u?\)?", hdr, flags=re.M))
    mirrored = [k for k in dir(ntp) if k.startswith("NTP_") and isinstance(getattr(ntp, k), int) and k in macros]
    assert len(mirrored) >= 10
    for k in mirrored:
        assert getattr(ntp, k) == int(macros[k]), k
    assert ntp.NTP_STAGE_SLOTS == int(macros["NTP_STAGE_SLOTS"])


def test_header_is_plain_c():
    """include/ntp.h is a C ABI: it compiles as C99 and as C++ (no torch / C++ types in the signatures)."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    hdr = os.path.join(ROOT, "include", "ntp.h")
    for lang, std in (("c", "-std=c99"), ("c++", "-std=c++17")):
        r = subprocess.run(["gcc", "-fsyntax-only", "-x", lang, std, "-Wall", "-Werror", hdr], capture_output=True,
                           text=True)
        assert r.returncode == 0, r.stderr
