"""C5 toy pull study: toys of the C1 model generated on the GPU
with the reference's own generator semantics (mcgen.generate_1d, seeds
1000..), each fitted from (4.95, 0.52, -0.29, 0.31) with FitManager.
Reports NLL calls / total fit wall time (the C5 metric) and generation time
separately, plus the pulls.

    python scripts/toy_study.py [--toys 8] [--n 10000000]
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
    ap.add_argument("--toys", type=int, default=8)
    ap.add_argument("--n", type=int, default=10_000_000)
    args = ap.parse_args()
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200.fitting import FitManager
    from paper_1710_08826_b200.mcgen import GenSpec, generate_1d
    from tests import models

    truth = (5.0, 0.5, -0.3, 0.3)
    start = (4.95, 0.52, -0.29, 0.31)
    x, pdf, params = models.c1(truth)
    gen_s = fit_s = 0.0
    calls = 0
    pulls = []
    for t in range(args.toys):
        for v, val in zip(params, truth):
            pf.set_value(v, val)
        t0 = time.perf_counter()
        ds = generate_1d(pdf, x, GenSpec(args.n, seed=1000 + t))
        gen_s += time.perf_counter() - t0
        for v, val in zip(params, start):
            pf.set_value(v, val)
        t0 = time.perf_counter()
        r = FitManager(pdf, ds).fit()
        fit_s += time.perf_counter() - t0
        calls += r.n_calls
        pulls.append([(v - tr) / e for v, tr, e in zip(r.values, truth, r.errors)])
    pulls = np.array(pulls)
    print(json.dumps({"study": "C5 toy pulls (C1 model)", "toys": args.toys, "events_per_toy": args.n,
                      "nll_calls": calls, "fit_wall_s": fit_s, "nll_calls_per_s": calls / fit_s,
                      "generation_s": gen_s, "generation_s_per_toy": gen_s / args.toys,
                      "pull_mean": pulls.mean(0).tolist(), "pull_std": pulls.std(0).tolist()}), flush=True)


if __name__ == "__main__":
    main()
