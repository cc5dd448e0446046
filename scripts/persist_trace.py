"""Where a persistent-kernel call spends its time: host round trip vs the
kernel's %globaltimer stamps (PFB_PERSIST_TRACE=1).

    PFB_PERSIST_TRACE=1 python scripts/persist_trace.py [--n 4096] [--calls 200]
"""
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
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--calls", type=int, default=200)
    ap.add_argument("--config", default="c1")
    args = ap.parse_args()
    import bench
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    P = pf.parafit
    cols = bench.events(args.config, args.n, seed=7)
    obs, pdf, free = bench.build_model(P, bench.CONFIGS[args.config]["model"])
    ds = pf.DeviceDataSet.from_columns(obs, cols, device=0)
    h = pf.DeviceFitManager(pdf, ds, persistent=True).fcn()
    x0 = np.array([v.value for v in free])
    x1 = x0.copy()
    x1[0] += 1e-7
    ctx = pf.device_context(0)
    tr = (ctypes.c_uint64 * 5)()
    rows = []
    for i in range(args.calls + 20):
        t0 = time.perf_counter()
        h(x1 if i & 1 else x0)
        dt = time.perf_counter() - t0
        L.check(L.lib().pfb_ctx_persist_trace(ctx.handle, tr), "trace")
        if i >= 20:
            t = list(tr)
            rows.append([1e6 * dt] + [(t[k] - t[0]) / 1e3 for k in range(1, 5)])
    med = np.median(np.array(rows), axis=0)
    print(json.dumps({"config": args.config, "n": args.n, "host_us": med[0], "released_us": med[1],
                      "last_cta_start_us": med[2], "last_cta_pass_done_us": med[3], "posted_us": med[4]}))
    h._objective.release()


if __name__ == "__main__":
    main()
