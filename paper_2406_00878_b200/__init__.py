"""paper_2406_00878_b200 — B200-native (sm_100a, fp64) all-at-once BDF1 Newton ("ParaDIn",
arXiv 2406.00878): C-ABI library ``libpit.so`` (include/pit.h) plus a thin ctypes binding (``pit``) and
the seeded synthetic workloads (``workloads``)."""
from . import workloads  # noqa: F401

__all__ = ["workloads", "pit", "build"]
