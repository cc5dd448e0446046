"""Binned row on one GPU: 2-D BinnedDataSet.fill of 10M
events into 100 x 100 bins on the device (pf.bin_fill) and the device binned
Poisson NLL (pf.binned_nll, P/engine.py:246-276), against the reference's own
fill and binned nll on the host.

    python scripts/binned_probe.py [--events 10000000] [--out profiles/r2_binned.json]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--events", type=int, default=10_000_000)
    ap.add_argument("--calls", type=int, default=200)
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import paper_1710_08826_b200 as pf
    from tests import models

    P = pf.parafit
    rng = np.random.default_rng(3)
    n = args.events
    (x, y), pdf, params = models.c2()
    xs = np.clip(rng.normal(5.0, 1.0, n), 0.0, 10.0)
    ys = np.clip(rng.exponential(2.5, n), 0.0, 10.0)
    ds = pf.DeviceDataSet.from_columns([x, y], [xs, ys], device=0)
    dev = P.BinnedDataSet([x, y], [100, 100])
    pf.bin_fill(dev, ds)  # warm
    dev = P.BinnedDataSet([x, y], [100, 100])
    t0 = time.perf_counter()
    pf.bin_fill(dev, ds)
    fill_s = time.perf_counter() - t0
    ref = P.BinnedDataSet([x, y], [100, 100])
    t0 = time.perf_counter()
    ref.fill(ds)  # the reference fill over the same (host) columns
    ref_fill_s = time.perf_counter() - t0
    equal = bool(np.array_equal(np.asarray(dev.contents), np.asarray(ref.contents)))
    pf.binned_nll(pdf, dev)
    t0 = time.perf_counter()
    for _ in range(args.calls):
        got = pf.binned_nll(pdf, dev)
    dev_s = (time.perf_counter() - t0) / args.calls
    with pf.reference_norms():
        t0 = time.perf_counter()
        want = P.binned_nll(pdf, ref)
        ref_s = time.perf_counter() - t0
    out = {"probe": "binned C2 (gauss x exp), 2-D fill + binned Poisson NLL", "events": n, "bins": 10000,
           "gpu_fill_ms": fill_s * 1e3, "reference_fill_ms": ref_fill_s * 1e3, "fill_counts_equal": equal,
           "gpu_binned_nll_us_per_call": dev_s * 1e6, "reference_binned_nll_ms": ref_s * 1e3,
           "binned_nll": got, "reference_binned_nll": want, "rel": abs(got - want) / abs(want)}
    line = json.dumps(out)
    print(line)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(line + "\n")


if __name__ == "__main__":
    main()
