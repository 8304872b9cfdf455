"""CPU-side checks of the C ABI library: it loads and exports every symbol
include/bpq_b200.h declares (no compute calls without a GPU)."""

import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    txt = (ROOT / "include" / "bpq_b200.h").read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bpq_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_header_symbols():
    from paper_1404_1831_b200 import _lib

    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert lib.bpq_abi_version() == 3


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(ROOT / "paper_1404_1831_b200" / "libbpq_b200.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_invalid_arguments_report_errors():
    """Argument validation happens before any device work."""
    import ctypes

    from paper_1404_1831_b200 import _lib

    lib = _lib.load()
    d = _lib.IndexDesc()
    d.dim, d.num_coarse, d.num_parts, d.codebook_size = 16, 4, 3, 16
    h = ctypes.c_void_p()
    assert lib.bpq_index_create(ctypes.byref(d), 0, ctypes.byref(h)) == _lib.BPQ_ERR_INVALID
    assert b"even" in lib.bpq_last_error()
    assert lib.bpq_search(None, 1, None, 1, 10, 10, None, None, None, None, None, 0, None) == _lib.BPQ_ERR_INVALID
    assert lib.bpq_merge_topk(None, None, None, 0, 1, 1, None, None, None, None) == _lib.BPQ_ERR_INVALID
