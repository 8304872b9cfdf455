"""paper_1404_1831_b200 -- B200-native batch query engine for bilayer-PQ search.

Drop-in for the search path of the reference package ``bilayerpq``
(Multi-D-ADC / FBPQ / HBPQ over an inverted multi-index, arXiv 1404.1831):

* ``DeviceIndex`` + ``DeviceIndex.search(queries, L, k, engine)`` -- batched
  search through the C ABI (include/bpq_b200.h), hand-written sm_100a kernels.
* ``search_baseline / search_fbpq / search_hbpq`` and ``make_engine`` --
  the reference's per-query API (multi_index.py:358, fbpq.py:188,
  hbpq.py:337, evalbench.py:271-286) on top of the batched engine.
* ``kernels`` -- the reference kernel backend (traverse_cells, scan_*) on
  the GPU, installable into ``bilayerpq.kernels``.
* ``encode`` -- device-side assignment, residual/local PQ encoding, packing.
* ``sharded`` -- database sharded by point id across GPUs, NCCL all-gather
  of per-rank top-k and a device merge.
"""

from __future__ import annotations

from .api import (
    BaselineEngine,
    FbpqEngine,
    HbpqEngine,
    make_engine,
    search_baseline,
    search_fbpq,
    search_hbpq,
)
from .index import DeviceIndex, SearchResult, build_tables_host

__all__ = [
    "DeviceIndex",
    "SearchResult",
    "build_tables_host",
    "search_baseline",
    "search_fbpq",
    "search_hbpq",
    "make_engine",
    "BaselineEngine",
    "FbpqEngine",
    "HbpqEngine",
]
