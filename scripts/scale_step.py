"""One (N, pipeline, api) step of the scale diagnostics, printing progress."""
import ctypes, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_08826_b200 as pf
from paper_1710_08826_b200 import _lib as L, mcgen, sharding
from tests import models

N, pipe, api = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
ctx = pf.device_context(0)
(x, y), pdf, _ = models.c2()
plan = ctx.plan_for(pdf, ("x", "y"))
snap = pf.snapshot(pdf.param_closure())
norms = pf.resolve_norms(pdf, snap, pf.NormalizationStore())
vals, nv = plan.pack(snap, norms)
st = mcgen._device_store(ctx, 2, N)
L.check(L.lib().pfb_gen_1d(ctx.handle, 1, 5.0, 1.0, -0.4, 0.0, 0.0, 10.0, 77, N, st), "gen")
L.check(L.lib().pfb_ctx_synchronize(ctx.handle), "sync")
print("generated", flush=True)
L.check(L.lib().pfb_ctx_set_pipeline(ctx.handle, pipe), "pipe")
err = L.PfbErr()
t0 = time.time()
if api == "nll":
    out = ctypes.c_double()
    L.check(L.lib().pfb_nll(ctx.handle, plan.handle, st, 0, N, 0, L.dptr(vals), len(vals), L.dptr(nv), len(nv),
                            ctypes.byref(out), ctypes.byref(err)), "nll")
    print(json.dumps({"N": N, "pipe": pipe, "api": api, "value": out.value, "s": time.time() - t0}), flush=True)
else:
    nb = -(-N // 4096)
    bs = np.empty(nb)
    L.check(L.lib().pfb_nll_block_sums(ctx.handle, plan.handle, st, 0, N, 0, L.dptr(vals), len(vals),
                                       L.dptr(nv), len(nv), L.dptr(bs), nb, ctypes.byref(err)), "bs")
    print(json.dumps({"N": N, "pipe": pipe, "api": api, "value": sharding.round_acc(sharding.acc_of_values(bs)),
                      "zero_blocks": int((bs == 0).sum()), "s": time.time() - t0}), flush=True)
