"""SURVEY 8(f) row 4 in numbers: filling a 2-D binning from 10M device-resident
events and evaluating the binned Poisson NLL (C2 model, 100 x 100 bins), next
to the oracle port of the reference's numpy fill and binned NLL on the host.

    python scripts/binned_probe.py [--n 10000000] [--bins 100]
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
    ap.add_argument("--bins", type=int, default=100)
    args = ap.parse_args()
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import mcgen
    from oracle import parafit_oracle as O
    from tests import models

    (x, y), pdf, _ = models.c2()
    cx, cy = mcgen.device_prod_2d(args.n, 5.0, 1.0, -0.4, 0.0, 10.0, 21)
    ds = pf.UnbinnedDataSet.from_columns([x, y], [cx, cy], copy=False)
    b = pf.BinnedDataSet([x, y], [args.bins, args.bins])
    b.fill(ds)  # warm-up (module, plan)
    reps = 20
    t0 = time.perf_counter()
    for _ in range(reps):
        b = pf.BinnedDataSet([x, y], [args.bins, args.bins])
        b.fill(ds)
    fill_s = (time.perf_counter() - t0) / reps
    pf.binned_nll(pdf, b)
    t0 = time.perf_counter()
    for _ in range(200):
        v = pf.binned_nll(pdf, b)
    nll_s = (time.perf_counter() - t0) / 200
    # the oracle port of the reference (numpy, host)
    axes = [("x", 0.0, 10.0, args.bins), ("y", 0.0, 10.0, args.bins)]
    t0 = time.perf_counter()
    counts = O.fill(axes, {"x": np.asarray(cx), "y": np.asarray(cy)})
    ofill_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    onll = O.binned_nll(models.c2_spec((5.0, 1.0, -0.4)), axes, counts)
    onll_s = time.perf_counter() - t0
    print(json.dumps({
        "probe": "binned C2 (gauss x exp), 2-D fill + binned Poisson NLL",
        "events": args.n, "bins": args.bins * args.bins,
        "gpu_fill_ms": 1e3 * fill_s, "gpu_fill_events_per_s": args.n / fill_s,
        "gpu_binned_nll_us_per_call": 1e6 * nll_s, "binned_nll": v,
        "oracle_fill_ms": 1e3 * ofill_s, "oracle_binned_nll_ms": 1e3 * onll_s,
        "fill_counts_equal": bool(np.array_equal(counts, np.asarray(b.contents))),
        "binned_nll_rel_vs_oracle": abs(v - onll) / abs(onll),
    }), flush=True)


if __name__ == "__main__":
    main()
