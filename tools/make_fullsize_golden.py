"""Write full-horizon oracle golden data for BASELINE c2..c5 (tests/golden/fullsize/).

Imports ONLY ``oracle/`` and the seeded data generators of ``workloads.py`` (no method arithmetic);
nothing here touches the CUDA path.  For config c it runs the sequential oracle (BDF1 + Newton per level,
PAPER.md:76, 505) over the WHOLE horizon n = 1..nt and stores

* ``c{c}_levels.npy``  — the solution at levels {nt/4, nt/2, 3nt/4, nt} (1-based), shape (4, ns) fp64;
* ``c{c}_stats.npy``   — per-level fingerprints of EVERY level: (sum u, sum u^2, max |u|), shape (nt, 3);
* a line in ``MANIFEST.json``: sha256 of both files, the stored level indices, the oracle's wall time,
  per-level Newton iteration totals, the host CPU and the command.

Usage: ``python tools/make_fullsize_golden.py 3 4 5`` (each config in its own process; c3 takes ~1 h).
The converged solutions of ParaDIn equal the sequential ones at every level (§4,
PAPER.md:506 §8.2), which is what the GPU test then checks element-wise at those levels.
"""
from __future__ import annotations

import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O                       # noqa: E402
from paper_2406_00878_b200 import workloads as W      # noqa: E402  (data only)

OUT = os.path.join(ROOT, "tests", "golden", "fullsize")


def stored_levels(nt: int):
    return [nt // 4, nt // 2, 3 * nt // 4, nt]


def sha256(path: str) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as f:
        for blk in iter(lambda: f.read(1 << 20), b""):
            h.update(blk)
    return h.hexdigest()


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def run(c: int) -> dict:
    p = W.config(c)
    t0 = time.time()
    seq = O.solve_sequential(p)
    wall = time.time() - t0
    assert seq.status == 0, seq.status
    U = seq.U
    lv = stored_levels(p.nt)
    os.makedirs(OUT, exist_ok=True)
    f_lv = os.path.join(OUT, f"c{c}_levels.npy")
    f_st = os.path.join(OUT, f"c{c}_stats.npy")
    np.save(f_lv, np.ascontiguousarray(U[[n - 1 for n in lv]]))
    st = np.stack([U.sum(axis=1), (U * U).sum(axis=1), np.abs(U).max(axis=1)], axis=1)
    np.save(f_st, st)
    return {"config": c, "name": p.name, "levels": lv, "nt": p.nt, "ns": p.ns,
            "levels_sha256": sha256(f_lv), "stats_sha256": sha256(f_st),
            "oracle_seconds": round(wall, 1), "newton_iterations_total": int(seq.iters.sum()),
            "max_abs_U": float(np.abs(U).max()), "cpu": cpu_model(),
            "command": f"python tools/make_fullsize_golden.py {c}"}


def main(argv):
    cs = [int(a) for a in argv] or [2, 3, 4, 5]
    man_path = os.path.join(OUT, "MANIFEST.json")
    for c in cs:
        rec = run(c)
        # merge under a lock-free rename: configs run in separate processes and finish at different times
        man = {}
        if os.path.exists(man_path):
            with open(man_path) as f:
                man = json.load(f)
        man[f"c{c}"] = rec
        tmp = man_path + f".tmp{os.getpid()}"
        with open(tmp, "w") as f:
            json.dump(man, f, indent=1, sort_keys=True)
        os.replace(tmp, man_path)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
