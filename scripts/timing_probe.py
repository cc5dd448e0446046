"""Cross-check of kernel timing methods for one NLL configuration.

    python scripts/timing_probe.py [--config c2] [--n 10000000]

(a) CUDA events around a single synchronous pfb_nll (after an L2 flush and a
    GPU spin that hides host launch latency) -- what bench.py reports;
(b) CUDA events around R back-to-back asynchronous partial evaluations
    (fast kernel + fix-up launch each), divided by R;
(c) the same as (b) without L2 flushing (L2-warm, 10M C2 = 160 MB > L2).
Prints one JSON line per method.
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
    ap.add_argument("--config", default="c2")
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--pipeline", type=int, default=1)
    args = ap.parse_args()

    import torch

    import bench
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    torch.cuda.set_device(0)
    cols = bench.make_data(args.config, args.n, 1000)
    obs, pdf = bench.build_model(args.config)
    ds = pf.UnbinnedDataSet(obs)
    ds.extend(cols)
    ctx = pf.device_context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    ctx.enable_timing(True)
    L.check(L.lib().pfb_ctx_set_pipeline(ctx.handle, args.pipeline), "pipeline")
    names = tuple(sorted(o.name for o in obs))
    plan = ctx.plan_for(pdf, names)
    store = ctx.store_for([ds.column(n) for n in names])
    snap = pf.snapshot(pdf.param_closure())
    norms = pf.resolve_norms(pdf, snap, pf.NormalizationStore())
    vals, nv = plan.pack(snap, norms)
    out = ctypes.c_double()
    err = L.PfbErr()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    acc = torch.zeros(L.PFB_ACC_WORDS, dtype=torch.int64, device="cuda")
    n = args.n

    def nll_sync():
        L.check(L.lib().pfb_nll(ctx.handle, plan.handle, store, 0, n, 0, L.dptr(vals), len(vals), L.dptr(nv),
                                len(nv), ctypes.byref(out), ctypes.byref(err)), "pfb_nll")

    def nll_async():
        L.check(L.lib().pfb_nll_partial_async(ctx.handle, plan.handle, store, 0, n, 0, L.dptr(vals), len(vals),
                                              L.dptr(nv), len(nv), ctypes.c_void_p(acc.data_ptr())), "partial")

    for _ in range(5):
        nll_sync()
    # (a)
    ms = []
    for _ in range(args.reps):
        flush.sum()
        torch.cuda._sleep(200_000)
        nll_sync()
        ms.append(ctx.last_kernel_ms())
    print(json.dumps({"method": "events around one pfb_nll (flush + spin)", "ms_median": float(np.median(ms)),
                      "ms_min": float(np.min(ms))}), flush=True)
    # (b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    torch.cuda._sleep(400_000)
    e0.record()
    for _ in range(args.reps):
        flush.sum()
        nll_async()
    e1.record()
    torch.cuda.synchronize()
    tot = e0.elapsed_time(e1)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(400_000)
    f0.record()
    for _ in range(args.reps):
        flush.sum()
    f1.record()
    torch.cuda.synchronize()
    tf = f0.elapsed_time(f1)
    print(json.dumps({"method": "back-to-back async (flush each), minus flush-only loop",
                      "ms_per_call": (tot - tf) / args.reps, "flush_ms": tf / args.reps}), flush=True)
    # (c)
    torch.cuda._sleep(400_000)
    e0.record()
    for _ in range(args.reps):
        nll_async()
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"method": "back-to-back async, no flush", "ms_per_call": e0.elapsed_time(e1) / args.reps}),
          flush=True)


if __name__ == "__main__":
    main()
