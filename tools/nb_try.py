"""Engine-4 bring-up on the GPU: parity against the oracle on prefixes of the BASELINE configs, then device time of
full solves next to engine 3.  usage: python tools/nb_try.py [quick|full]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O                      # noqa: E402
from paper_2406_00878_b200 import pit, workloads as W  # noqa: E402


def run(p, reps=1, **cfg):
    s = pit.Solver(p, **cfg)
    try:
        d_u0 = torch.from_numpy(p.u0).cuda()
        d_ring = None if p.ring is None else torch.from_numpy(p.ring).cuda()
        d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
        d_hist = torch.zeros((s.cfg.newton_max, 4), dtype=torch.float64, device="cuda")
        d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s.solve_device(d_u0, d_ring, None, d_out, d_hist, d_info)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        nit, st = (int(v) for v in d_info.cpu())
        return d_out.cpu().numpy(), d_hist.cpu().numpy()[:nit], nit, st, min(ts), s.engine_info(), s.stats()
    finally:
        s.close()


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "quick"
    cases = [(2, None, None), (5, None, 4), (4, None, 8), (3, None, 4), (1, None, None)] if mode != "trace" else []
    for c, n, nt in cases:
        p = W.config(c, n=n, nt=nt)
        t0 = time.time()
        seq = O.solve_sequential(p)
        for eng in (4, 0):
            try:
                U, hist, nit, st, ms, ei, stt = run(p, engine=eng) if eng else run(p)
            except pit.PitError as e:
                print(f"{p.name} engine {eng}: {e}")
                continue
            err = np.abs(U - seq.U).max() / np.abs(seq.U).max()
            print(f"{p.name} engine {ei['engine']}: status {st} nit {nit} err {err:.2e} {ms:.3f} ms "
                  f"omega {ei['omega']:.5f} sweeps {ei['sweeps']} q {ei['q']:.4f} linres {[f'{a:.1e}' for a, _ in ei['linres']]} "
                  f"steps {stt['steps']} hist {[f'{h:.1e}' for h in hist[:, 3]]}", flush=True)
        print(f"   oracle {time.time() - t0:.1f} s", flush=True)
    if mode == "trace":
        import os
        os.environ["PIT_TRACE"] = "1"
        for c, dd in ((5, 3), (5, 0), (4, 0), (3, 0), (2, 0)):
            p = W.config(c)
            U, hist, nit, st, ms, ei, stt = run(p, reps=2, engine=4, pipeline_depth=dd)
            tm = {k: round(v / 1965.0, 1) for k, v in ei.get("trace_mean", {}).items()}
            tx = {k: round(v / 1965.0, 1) for k, v in ei.get("trace_max", {}).items()}
            gold = f"tests/golden/fullsize/c{c}_levels.npy"
            import os as _os
            par = ""
            if _os.path.exists(gold):
                g = np.load(gold)
                mine = U[[p.nt // 4 - 1, p.nt // 2 - 1, 3 * p.nt // 4 - 1, p.nt - 1]]
                par = f" golden {np.abs(mine - g).max() / np.abs(g).max():.1e}"
            print(f"TRACE {p.name} D={stt['depth']}: {ms:.2f} ms nit {nit} st {st} levels {stt['steps']} sweeps {ei['sweeps']}{par} linres {[f'{a:.0e}' for a, _ in ei['linres']]}\n  mean us {tm}\n  max us  {tx}", flush=True)
        return
    if mode == "full":
        for c in (5, 4, 3):
            p = W.config(c)
            for eng in (4, 3):
                U, hist, nit, st, ms, ei, stt = run(p, reps=3, engine=eng)
                print(f"FULL {p.name} engine {ei['engine']}: status {st} nit {nit} {ms:.2f} ms  sweeps {ei['sweeps']} "
                      f"linres {[f'{a:.1e}' for a, _ in ei['linres']]} hist {[f'{h:.1e}' for h in hist[:, 3]]}", flush=True)
                if eng == 4:
                    np.save(f"/tmp/U_c{c}_e4.npy", U[[p.nt // 4 - 1, p.nt // 2 - 1, 3 * p.nt // 4 - 1, p.nt - 1]])
            gold = np.load(f"tests/golden/fullsize/c{c}_levels.npy") if c != 3 or __import__('os').path.exists(f"tests/golden/fullsize/c{c}_levels.npy") else None
            if gold is not None:
                mine = np.load(f"/tmp/U_c{c}_e4.npy")
                print(f"   golden parity c{c}: {np.abs(mine - gold).max() / np.abs(gold).max():.2e}")


if __name__ == "__main__":
    main()
