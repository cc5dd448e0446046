"""Diagnostics for large N: pfb_nll of the whole range vs the exact sum of
block sums (whole range and block-aligned pieces)."""
import ctypes, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_08826_b200 as pf
from paper_1710_08826_b200 import _lib as L, mcgen, sharding
from tests import models

ctx = pf.device_context(0)
(x, y), pdf, _ = models.c2()
plan = ctx.plan_for(pdf, ("x", "y"))
snap = pf.snapshot(pdf.param_closure())
norms = pf.resolve_norms(pdf, snap, pf.NormalizationStore())
vals, nv = plan.pack(snap, norms)
for N in [int(a) for a in sys.argv[1:]] or [50_000_000, 150_000_000, 300_000_000, 600_000_000]:
    st = mcgen._device_store(ctx, 2, N)
    L.check(L.lib().pfb_gen_1d(ctx.handle, 1, 5.0, 1.0, -0.4, 0.0, 0.0, 10.0, 77, N, st), "gen")
    err = L.PfbErr()
    res = {"N": N}
    for pipe in (1, 2, 0):
        L.check(L.lib().pfb_ctx_set_pipeline(ctx.handle, pipe), "pipe")
        out = ctypes.c_double()
        L.check(L.lib().pfb_nll(ctx.handle, plan.handle, st, 0, N, 0, L.dptr(vals), len(vals), L.dptr(nv), len(nv),
                                ctypes.byref(out), ctypes.byref(err)), "nll")
        nb = -(-N // 4096)
        bs = np.empty(nb)
        L.check(L.lib().pfb_nll_block_sums(ctx.handle, plan.handle, st, 0, N, 0, L.dptr(vals), len(vals),
                                           L.dptr(nv), len(nv), L.dptr(bs), nb, ctypes.byref(err)), "bs")
        res[f"p{pipe}_nll"] = out.value
        res[f"p{pipe}_bsum"] = sharding.round_acc(sharding.acc_of_values(bs))
        res[f"p{pipe}_nonfinite_blocks"] = int((~np.isfinite(bs)).sum())
        res[f"p{pipe}_zero_blocks"] = int((bs == 0).sum())
    L.check(L.lib().pfb_ctx_set_pipeline(ctx.handle, 1), "pipe")
    print(json.dumps(res), flush=True)
    L.lib().pfb_store_destroy(st)
