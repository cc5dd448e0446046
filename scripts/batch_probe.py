"""Device time of the batched objective vs the number of parameter points.

    python scripts/batch_probe.py [--n 10000000]

C2 (ProdPdf, 10M events): one pfb_nll_batch launch with M points (L2 flushed,
GPU spin before the launch), kernel time from CUDA events.  Prints one JSON
line per M with the time per point.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()

    import torch

    import bench
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    torch.cuda.set_device(0)
    cols = bench.make_data("c2", args.n, 1000)
    obs, pdf = bench.build_model("c2")
    ds = pf.UnbinnedDataSet.from_columns(obs, cols, copy=False)
    ctx = pf.device_context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    ctx.enable_timing(True)
    names = tuple(sorted(o.name for o in obs))
    plan = ctx.plan_for(pdf, names)
    store = ctx.store_for([ds.column(k) for k in names])
    params = [v for v in pdf.param_closure() if not v.fixed]
    base = np.array([v.value for v in params])
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    store_norm = pf.NormalizationStore()
    for M in (1, 2, 4, 7, 16):
        snaps, norms = [], []
        for m in range(M):
            for k, v in enumerate(params):
                pf.set_value(v, float(base[k] + 1e-3 * ((m + k) % 3 - 1)))
            snap = pf.snapshot(pdf.param_closure())
            snaps.append(snap)
            norms.append(pf.resolve_norms(pdf, snap, store_norm))
        vals, nv = plan.pack_batch(snaps, norms)
        out = np.empty(M)
        errs = (L.PfbErr * M)()
        times = []
        for r in range(3 + args.reps):
            flush.sum()
            torch.cuda._sleep(2_000_000)
            L.check(L.lib().pfb_nll_batch(ctx.handle, plan.handle, store, 0, args.n, 0, L.dptr(vals), M,
                                          vals.shape[1], L.dptr(nv), nv.shape[1], L.dptr(out), errs),
                    "pfb_nll_batch")
            if r >= 3:
                times.append(ctx.last_kernel_ms())
        ms = float(np.median(times))
        print(json.dumps({"config": "c2", "n": args.n, "points": M, "kernel_ms": ms, "ms_per_point": ms / M,
                          "events_per_s_effective": M * args.n / ms * 1e3}), flush=True)


if __name__ == "__main__":
    main()
