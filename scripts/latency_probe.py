"""Host-side latency of one synchronous NLL call (what a minimiser waits for
per step), layer by layer: raw C ABI call, the mirror API's nll(), and a
torch launch+sync floor for comparison.

    python scripts/latency_probe.py
"""

import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def per_call_us(fn, n=400):
    for _ in range(20):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return 1e6 * (time.perf_counter() - t0) / n


def main():
    import torch

    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L
    from paper_1710_08826_b200 import mcgen
    from paper_1710_08826_b200.engine import NormalizationStore, device_context
    from tests import models

    torch.cuda.set_device(0)
    a = torch.zeros(1, device="cuda")

    def torch_floor():
        a.add_(1.0)
        torch.cuda.synchronize()

    print(json.dumps({"probe": "torch add_ + synchronize", "us": per_call_us(torch_floor)}), flush=True)
    ctx = device_context(0)
    for n in (4096, 1_000_000, 10_000_000):
        x, pdf, params = models.c1()
        col = mcgen.device_sumpdf_1d(n, 5.0, 0.5, -0.3, 0.3, 0.0, 10.0, 1)
        ds = pf.UnbinnedDataSet.from_columns([x], [col], copy=False)
        store = NormalizationStore()
        pf.nll(pdf, ds, store=store)
        names = ("x",)
        plan = ctx.plan_for(pdf, names)
        st = ctx.store_for([ds.column(nm) for nm in names])
        snap = pf.snapshot(pdf.param_closure())
        norms = pf.resolve_norms(pdf, snap, NormalizationStore())
        vals, nv = plan.pack(snap, norms)
        out = ctypes.c_double()
        err = L.PfbErr()

        def raw():
            L.check(L.lib().pfb_nll(ctx.handle, plan.handle, st, 0, n, 0, L.dptr(vals), len(vals), L.dptr(nv),
                                    len(nv), ctypes.byref(out), ctypes.byref(err)), "pfb_nll")

        def mirror():
            pf.nll(pdf, ds, store=store)

        print(json.dumps({"probe": "C1 raw pfb_nll", "n": n, "us": per_call_us(raw)}), flush=True)
        print(json.dumps({"probe": "C1 pf.nll (persistent store)", "n": n, "us": per_call_us(mirror)}), flush=True)
        ctx.enable_timing(True)
        raw()
        print(json.dumps({"probe": "C1 kernel (events)", "n": n, "us": 1e3 * ctx.last_kernel_ms()}), flush=True)
        ctx.enable_timing(False)


if __name__ == "__main__":
    main()
