"""ctypes binding of libbpq_b200.so (the C ABI declared in include/bpq_b200.h).

The library is the product path: if it is missing the import fails loudly.
There is no CPU fallback anywhere in this package.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["BPQ_LIB"]) if os.environ.get("BPQ_LIB") else _PKG / "libbpq_b200.so"

ENGINE_BASELINE, ENGINE_FBPQ, ENGINE_HBPQ = 0, 1, 2
ENGINES = {"baseline": ENGINE_BASELINE, "fbpq": ENGINE_FBPQ, "hbpq": ENGINE_HBPQ}

BPQ_OK, BPQ_ERR_INVALID, BPQ_ERR_CUDA, BPQ_ERR_UNSUPPORTED, BPQ_ERR_WORKSPACE = range(5)

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
F32 = ctypes.c_float
SZ = ctypes.c_size_t


class IndexDesc(ctypes.Structure):
    _fields_ = [
        ("dim", I32),
        ("num_coarse", I32),
        ("num_parts", I32),
        ("codebook_size", I32),
        ("num_entries", I64),
        ("num_entries_global", I64),
        ("coarse1", P),
        ("coarse2", P),
        ("coarse_norms1", P),
        ("coarse_norms2", P),
        ("cell_offsets", P),
        ("global_offsets", P),
        ("ids", P),
        ("codes", P),
        ("fine_books", P),
        ("fine_norms", P),
        ("cross1", P),
        ("cross2", P),
        ("bank1", P),
        ("bank2", P),
        ("row_ptr", P),
        ("col_ptr", P),
        ("row_cols", P),
        ("col_rows", P),
        ("rotation", P),
        ("rot1", P),
        ("rot2", P),
        ("fbpq_exact", I32),
    ]


# name -> (restype, argtypes)
SIGNATURES = {
    "bpq_last_error": (ctypes.c_char_p, []),
    "bpq_abi_version": (ctypes.c_int, []),
    "bpq_index_create": (ctypes.c_int, [ctypes.POINTER(IndexDesc), ctypes.c_int, ctypes.POINTER(P)]),
    "bpq_index_destroy": (ctypes.c_int, [P]),
    "bpq_search_workspace_size": (SZ, [P, ctypes.c_int, I64, I64, I32]),
    "bpq_search": (ctypes.c_int, [P, ctypes.c_int, P, I64, I64, I32, P, P, P, P, P, SZ, P]),
    "bpq_search_ex": (ctypes.c_int, [P, ctypes.c_int, P, I64, I64, I32, P, P, P, P, P, P, P, SZ, P]),
    "bpq_traverse_workspace_size": (SZ, [I64, I64, I64]),
    "bpq_traverse_cells": (ctypes.c_int, [P, P, P, P, P, I64, I64, I64, P, P, P, P, P, P, SZ, P]),
    "bpq_scan_tables": (ctypes.c_int, [P, P, P, P, I64, I64, P, P, I32, I32, F32, P, P, P, P, P, P, P, P, P, P]),
    "bpq_scan_global": (ctypes.c_int, [P, P, P, P, I64, I64, P, P, I32, I32, I32, P, P, P, P, P, P]),
    "bpq_scan_local": (ctypes.c_int, [P, P, P, P, I64, I64, P, P, I32, I32, I32, P, P, P, P, P, P, P]),
    "bpq_nearest_centroids": (ctypes.c_int, [P, I64, I64, I32, P, P, I32, P, P, P, I64, P]),
    "bpq_coarse_limb_image_bytes": (SZ, [I32]),
    "bpq_coarse_limb_image": (ctypes.c_int, [P, I32, P, P]),
    "bpq_nearest_centroids_tc": (ctypes.c_int, [P, I64, I64, P, P, I32, P, P, P, I64, P]),
    "bpq_encode_residual": (ctypes.c_int, [P, I64, I32, P, P, P, P, P, P, I32, I32, P, P, SZ, P]),
    "bpq_encode_local": (ctypes.c_int, [P, I64, I32, P, P, P, P, P, P, I32, I32, P, P]),
    "bpq_pack_workspace_size": (SZ, [I64, I32]),
    "bpq_pack_cells": (ctypes.c_int, [P, P, I64, I32, ctypes.c_uint32, P, I32, P, P, P, P, SZ, P]),
    "bpq_cell_lists_workspace_size": (SZ, [I32]),
    "bpq_build_cell_lists": (ctypes.c_int, [P, I32, P, P, P, P, P, SZ, P]),
    "bpq_debug_set_phase_buffer": (ctypes.c_int, [P]),
    "bpq_rotate": (ctypes.c_int, [P, I64, I32, P, P, P]),
    "bpq_coarse_dots": (ctypes.c_int, [P, P, I64, P, P, P]),
    "bpq_merge_topk": (ctypes.c_int, [P, P, P, I32, I64, I32, P, P, P, P]),
    "bpq_merge_topk_packed": (ctypes.c_int, [P, I32, I64, I32, P, P, P, P]),
    "bpq_split_visit_cap": (I64, [P, I64]),
    "bpq_search_split_traverse": (ctypes.c_int, [P, P, I64, I64, P, P, I64, P, P, SZ, P]),
    "bpq_split_scan_workspace_size": (SZ, [P, I64, I64]),
    "bpq_search_split_scan": (ctypes.c_int, [P, P, I64, I32, P, P, I64, P, P, P, P, SZ, P]),
}

_lib = None


class BpqError(RuntimeError):
    pass


def load():
    """Load the extension; raises if it was not built (no silent fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')"
            )
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == BPQ_OK:
        return
    msg = (load().bpq_last_error() or b"").decode()
    if rc == BPQ_ERR_INVALID:
        raise ValueError(msg)
    raise BpqError(f"{what}: {msg} (status {rc})")


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def exported_symbols() -> list[str]:
    return sorted(SIGNATURES)


if os.environ.get("BPQ_EAGER_LOAD") == "1":  # pragma: no cover
    load()
