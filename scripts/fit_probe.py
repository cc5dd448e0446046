"""NLL calls per second inside real fits (host path included): the C5-style
metric (total NLL calls / total fit wall time) on C1 / C2 models.

    python scripts/fit_probe.py [--n 10000000]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--profile", action="store_true", help="cProfile 20 C1 fits (host time by function)")
    args = ap.parse_args()
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import mcgen
    from paper_1710_08826_b200.fitting import FitManager
    from tests import models

    # C5 unit: C1 model, 10M events, fit start (4.95, 0.52, -0.29, 0.31)
    x, pdf, params = models.c1()
    col = mcgen.device_sumpdf_1d(args.n, 5.0, 0.5, -0.3, 0.3, 0.0, 10.0, 1000)
    ds = pf.UnbinnedDataSet.from_columns([x], [col], copy=False)
    for v, val in zip(params, (4.95, 0.52, -0.29, 0.31)):
        pf.set_value(v, val)
    pf.nll(pdf, ds)
    # bare objective calls (parameter moves, norm recomputation, launch, D2H)
    t0 = time.perf_counter()
    k = 200
    for i in range(k):
        pf.set_value(params[0], 4.95 + 1e-4 * (i % 7))
        pf.nll(pdf, ds)
    dt = time.perf_counter() - t0
    print(json.dumps({"probe": "nll() loop C1", "n": args.n, "calls": k, "us_per_call": 1e6 * dt / k}), flush=True)
    for v, val in zip(params, (4.95, 0.52, -0.29, 0.31)):
        pf.set_value(v, val)
    t0 = time.perf_counter()
    r = FitManager(pdf, ds).fit()
    dt = time.perf_counter() - t0
    print(json.dumps({"probe": "FitManager C1 (C5 unit)", "n": args.n, "calls": r.n_calls, "wall_s": dt,
                      "calls_per_s": r.n_calls / dt, "status": r.status, "values": list(r.values)}), flush=True)
    if args.profile:
        import cProfile
        import pstats

        prof = cProfile.Profile()
        prof.enable()
        for _ in range(20):
            for v, val in zip(params, (4.95, 0.52, -0.29, 0.31)):
                pf.set_value(v, val)
            FitManager(pdf, ds).fit()
        prof.disable()
        pstats.Stats(prof).sort_stats("tottime").print_stats(25)
    (xx, yy), pdf2, p2 = models.c2((4.9, 1.1, -0.35))
    cx, cy = mcgen.device_prod_2d(args.n, 5.0, 1.0, -0.4, 0.0, 10.0, 2)
    ds2 = pf.UnbinnedDataSet.from_columns([xx, yy], [cx, cy], copy=False)
    pf.nll(pdf2, ds2)
    t0 = time.perf_counter()
    r = FitManager(pdf2, ds2).fit()
    dt = time.perf_counter() - t0
    print(json.dumps({"probe": "FitManager C2", "n": args.n, "calls": r.n_calls, "wall_s": dt,
                      "calls_per_s": r.n_calls / dt, "status": r.status}), flush=True)


if __name__ == "__main__":
    main()


def dalitz_fit(n=10_000_000):
    import time

    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import mcgen
    from paper_1710_08826_b200.fitting import FitManager
    from tests import models

    terms = [(p, s, m, w, mag, ph) for (p, m, w, s, mag, ph) in models.C3_TERMS]
    s12, s13 = mcgen.device_dalitz(n, terms, models.D_CHANNEL_T, 3)
    (o12, o13), pdf, rts = models.c3()
    ds = pf.UnbinnedDataSet.from_columns([o12, o13], [s12, s13], copy=False)
    pf.nll(pdf, ds)
    for t in rts[1:]:
        pf.set_value(t.magnitude, t.magnitude.value * 1.05)
        pf.set_value(t.phase, t.phase.value + 0.05)
    t0 = time.perf_counter()
    r = FitManager(pdf, ds).fit()
    dt = time.perf_counter() - t0
    print(json.dumps({"probe": "FitManager C3 Dalitz (6 free)", "n": n, "calls": r.n_calls, "wall_s": dt,
                      "calls_per_s": r.n_calls / dt, "status": r.status, "timing": r.timing}), flush=True)


if __name__ == "__main__" and os.environ.get("PFB_DALITZ_FIT"):
    dalitz_fit()
