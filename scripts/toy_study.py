"""C5 toy pull study end to end on one GPU.

    python scripts/toy_study.py [--toys 256] [--events 10000000] [--out profiles/r2_c5_toy_study.json]

The C1 model (x in [0, 10], gaussian(mu 5, sigma 0.5) + exponential(alpha
-0.3), f = 0.3); toy i is the reference generator's sample for
``GenSpec(events, seed=1000 + i)`` (mcgen.generate_1d: the reference's PCG64
streams and accept-reject, on the device; ``stats["ambiguous"]`` counts
decisions within 2^-47 of their density), fitted from (4.95, 0.52, -0.29,
0.31) by DeviceFitManager (the reference minimiser, objective in C, batched
stencils).  Metric: total NLL calls / total fit wall time;
generation reported separately.  Pulls (value - truth) / error per parameter.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TRUTH = (5.0, 0.5, -0.3, 0.3)
START = (4.95, 0.52, -0.29, 0.31)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--toys", type=int, default=256)
    ap.add_argument("--events", type=int, default=10_000_000)
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import mcgen
    from tests import models

    P = pf.parafit
    x, pdf, params = models.c1(TRUTH)
    calls = 0
    fit_s = gen_s = 0.0
    ambiguous = 0
    pulls, statuses = [], []
    for i in range(args.toys):
        for v, val in zip(params, TRUTH):
            P.set_value(v, val)
        stats = {}
        t0 = time.perf_counter()
        ds = mcgen.generate_1d(pdf, x, P.GenSpec(args.events, seed=1000 + i), stats)
        gen_s += time.perf_counter() - t0
        ambiguous += stats["ambiguous"]
        for v, val in zip(params, START):
            P.set_value(v, val)
        t0 = time.perf_counter()
        r = pf.DeviceFitManager(pdf, ds).fit()
        fit_s += time.perf_counter() - t0
        calls += r.n_calls
        statuses.append(r.status)
        pulls.append([(v - t) / e for v, t, e in zip(r.values, TRUTH, r.errors)])
        del ds
    pulls = np.array(pulls)
    out = {"study": "C5 toy pulls (C1 model), reference toys (GenSpec seeds 1000..), DeviceFitManager",
           "toys": args.toys, "events_per_toy": args.events, "nll_calls": calls, "fit_wall_s": fit_s,
           "nll_calls_per_s": calls / fit_s, "events_per_s": calls * args.events / fit_s,
           "generation_s": gen_s, "generation_s_per_toy": gen_s / args.toys, "ambiguous_decisions": ambiguous,
           "converged": statuses.count("converged"),
           "pull_mean": pulls.mean(axis=0).tolist(), "pull_std": pulls.std(axis=0).tolist(),
           "names": [p.name for p in params]}
    line = json.dumps(out)
    print(line)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(line + "\n")


if __name__ == "__main__":
    main()
