"""Cost of the exchange fused into the NLL kernel's epilogue, on one GPU: the
same C2 launch (10M events) with and without the mailbox protocol (world = 1,
the rank's own mailbox: stores, system fence, release flag, acquire wait,
sum), CUDA-event kernel time, L2 evicted before each call.

    python scripts/fused_probe.py [--n 10000000] [--reps 50]
"""

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L
    from paper_1710_08826_b200 import mcgen
    from paper_1710_08826_b200.sharding import PeerGroup
    from tests import models

    torch.cuda.set_device(0)
    ctx = pf.device_context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    ctx.enable_timing(True)
    (x, y), pdf, _ = models.c2()
    cx, cy = mcgen.device_prod_2d(args.n, 5.0, 1.0, -0.4, 0.0, 10.0, 2)
    plan = ctx.plan_for(pdf, ("x", "y"))
    st = ctx.store_for([cx, cy])
    snap = pf.snapshot(pdf.param_closure())
    norms = pf.resolve_norms(pdf, snap, pf.NormalizationStore())
    vals, nv = plan.pack(snap, norms)
    peers = PeerGroup(ctx, 0, 1)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    out, err, slow = ctypes.c_double(), L.PfbErr(), ctypes.c_int32()
    res = {}
    for mode in ("plain", "fused", "plain", "fused"):
        ts = []
        for _ in range(args.reps):
            ctx.spin(1_000_000, flush.data_ptr(), flush.numel() * 4)
            if mode == "plain":
                L.check(L.lib().pfb_nll(ctx.handle, plan.handle, st, 0, args.n, 0, L.dptr(vals), len(vals), L.dptr(nv),
                                        len(nv), ctypes.byref(out), ctypes.byref(err)), "pfb_nll")
            else:
                L.check(L.lib().pfb_nll_peer(ctx.handle, plan.handle, st, 0, args.n, 0, L.dptr(vals), len(vals),
                                             L.dptr(nv), len(nv), 5.0, ctypes.byref(out), ctypes.byref(slow)),
                        "pfb_nll_peer")
                assert slow.value == 0
            ts.append(ctx.last_kernel_ms())
        res.setdefault(mode, []).append(float(np.median(ts)) * 1e3)
        res.setdefault(mode + "_nll", out.value)
    print(json.dumps({"probe": "fused exchange epilogue, world = 1", "n": args.n, "kernel_us_plain": res["plain"],
                      "kernel_us_fused": res["fused"], "same_nll": res["plain_nll"] == res["fused_nll"]}), flush=True)


if __name__ == "__main__":
    main()
