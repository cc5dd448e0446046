"""Host wall clock of one synchronous NLL call -- what a minimiser waits for.

    python scripts/latency_probe.py [--calls 400] [--sizes 4096,1000000,10000000] [--configs c1,c2,c3]

Per config and size, median over `calls` calls after 20 warm-up calls:
* ``raw``: the C ABI ``pfb_nll`` through ctypes with pre-packed values;
* ``reference_nll``: the reference's ``nll`` with ``DeviceBackend`` and a
  persistent norm store, one parameter moved per call (what the reference
  FitManager's objective does: set_value, snapshot, nll);
* ``fast_objective``: ``DeviceFitManager(...).fcn()`` -- the objective in C
  (pfb_objective) through the reference ``FcnHandle``, one parameter moved
  per call;
* ``persistent``: the same with the resident kernel (pfb_objective_set_persistent);
* ``kernel``: CUDA-event time of the fused launch (pfb_ctx timing).
One JSON line per (config, size).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=400)
    ap.add_argument("--sizes", default="4096,1000000,10000000")
    ap.add_argument("--configs", default="c1,c2,c3")
    args = ap.parse_args()

    import bench
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    P = pf.parafit
    ctx = pf.device_context(0)
    for cfg in args.configs.split(","):
        for n in [int(s) for s in args.sizes.split(",")]:
            model = bench.CONFIGS[cfg]["model"]
            cols = bench.events(cfg, n, seed=7)
            obs, pdf, free = bench.build_model(P, model)
            ds = pf.DeviceDataSet.from_columns(obs, cols, device=0)
            names = tuple(sorted(o.name for o in obs))
            arrays = [ds.column(nm) for nm in names]
            plan = ctx.plan_for(pdf, names)
            st = ctx.store_for(arrays)
            store = P.NormalizationStore()
            snap = P.snapshot(pdf.param_closure())
            vals, nv = [a.copy() for a in plan.pack(snap, P.resolve_norms(pdf, snap, store))]
            out, err = ctypes.c_double(), L.PfbErr()

            def raw():
                L.check(L.lib().pfb_nll(ctx.handle, plan.handle, st, 0, n, 0, L.dptr(vals), len(vals), L.dptr(nv),
                                        len(nv), ctypes.byref(out), ctypes.byref(err)), "pfb_nll")

            backend = pf.DeviceBackend()
            v0 = free[0]
            base = v0.value
            flip = [0]

            def ref_call():
                flip[0] ^= 1
                P.set_value(v0, base + 1e-7 * flip[0])
                P.nll(pdf, ds, P.snapshot(pdf.param_closure()), backend, store)

            handle = pf.DeviceFitManager(pdf, ds, persistent=False).fcn()
            phandle = pf.DeviceFitManager(pdf, ds, persistent=True).fcn()
            x0 = np.array([v.value for v in free])
            x1 = x0.copy()
            x1[0] += 1e-7

            def fast_call():
                flip[0] ^= 1
                handle(x1 if flip[0] else x0)

            def persistent_call():
                flip[0] ^= 1
                phandle(x1 if flip[0] else x0)

            res = {"config": cfg, "n": n, "objective": type(handle._objective).__name__}
            for tag, fn in (("raw_us", raw), ("reference_nll_us", ref_call), ("fast_objective_us", fast_call),
                            ("persistent_us", persistent_call)):
                for _ in range(20):
                    fn()
                t = []
                for _ in range(args.calls):
                    t0 = time.perf_counter()
                    fn()
                    t.append(time.perf_counter() - t0)
                res[tag] = 1e6 * float(np.median(t))
            P.set_value(v0, base)
            phandle._objective.release()
            ctx.enable_timing(True)
            km = []
            for _ in range(50):
                raw()
                km.append(ctx.last_kernel_ms())
            ctx.enable_timing(False)
            res["kernel_event_us"] = 1e3 * float(np.median(km))
            res["evaluator"] = plan.evaluator
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
