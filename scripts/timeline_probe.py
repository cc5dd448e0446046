"""Per-CTA timeline of one C2 NLL launch (TMA unit kernel), from %globaltimer
stamps the kernel records in PFB_TRACE builds:

    make OUT=build/trace EXTRA=-DPFB_TRACE
    PFB200_LIB=$PWD/build/trace/libpfb200.so python scripts/timeline_probe.py [n]

Prints, in us from the first CTA's entry: CTA start spread, first copy
issued, first stage ready, teams done (min/median/max = the tail), last
finish entry, last ticket, export done; next to the CUDA-event time of the
same launch.
"""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1710_08826_b200 as pf
from paper_1710_08826_b200 import _lib as L, mcgen
from tests import models
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
cfg = sys.argv[2] if len(sys.argv) > 2 else "c2"
fused = len(sys.argv) > 3 and sys.argv[3] == "fused"
ctx = pf.device_context(0)
ctx.enable_timing(True)
if cfg == "c3":
    terms = [(p, s, m, w, mag, ph) for (p, m, w, s, mag, ph) in models.C3_TERMS]
    cx, cy = mcgen.device_dalitz(n, terms, models.D_CHANNEL_T, 3)
    (x, y), pdf, _ = models.c3()
    names = ("s12", "s13")
else:
    cx, cy = mcgen.device_prod_2d(n, 5.0, 1.0, -0.4, 0.0, 10.0, 2)
    (x, y), pdf, _ = models.c2()
    names = ("x", "y")
pf.nll(pdf, pf.UnbinnedDataSet.from_columns([x, y], [cx, cy], copy=False))  # grid / norms for Dalitz
plan = ctx.plan_for(pdf, names); st = ctx.store_for([cx, cy])
snap = pf.snapshot(pdf.param_closure()); norms = pf.resolve_norms(pdf, snap, pf.NormalizationStore())
vals, nv = plan.pack(snap, norms)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
out = ctypes.c_double(); err = L.PfbErr()
lib = L.lib()
if fused:
    from paper_1710_08826_b200.sharding import PeerGroup
    PeerGroup(ctx, 0, 1)
read = lib.pfb_debug_trace_dal if cfg == "c3" else lib.pfb_debug_trace
read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
for rep in range(6):
    ctx.spin(1_000_000, flush.data_ptr(), flush.numel() * 4)
    if fused:
        slow = ctypes.c_int32()
        L.check(lib.pfb_nll_peer(ctx.handle, plan.handle, st, 0, n, 0, L.dptr(vals), len(vals), L.dptr(nv), len(nv), 5.0, ctypes.byref(out), ctypes.byref(slow)), "nll_peer")
    else:
        L.check(lib.pfb_nll(ctx.handle, plan.handle, st, 0, n, 0, L.dptr(vals), len(vals), L.dptr(nv), len(nv), ctypes.byref(out), ctypes.byref(err)), "nll")
    ms = ctx.last_kernel_ms()
    tr = (ctypes.c_ulonglong * (1024 * 16))()
    read(tr, 148)
    full = np.frombuffer(tr, dtype=np.uint64).reshape(1024, 16)[:148].astype(np.int64)
    a = full[:, :8]
    t0 = a[:, 0].min()
    rel = (a - t0) / 1000.0
    rel[a == 0] = np.nan
    last = np.nanargmax(rel[:, 7]) if np.isfinite(rel[:, 7]).any() else -1
    print(json.dumps({"cfg": cfg, "fused": fused, "n": n, "event_us": 1e3 * ms,
        "entry_spread_us": float(np.nanmax(rel[:, 0])),
        "first_issue_us_med": float(np.nanmedian(rel[:, 1] - rel[:, 0])),
        "first_ready_us_med": float(np.nanmedian(rel[:, 2] - rel[:, 0])), "first_ready_us_max": float(np.nanmax(rel[:, 2])),
        "team_done_min": float(np.nanmin(np.fmax(rel[:, 3], rel[:, 4]))), "team_done_med": float(np.nanmedian(np.fmax(rel[:, 3], rel[:, 4]))), "team_done_max": float(np.nanmax(np.fmax(rel[:, 3], rel[:, 4]))),
        "team_gap_med": float(np.nanmedian(np.abs(rel[:, 3] - rel[:, 4]))),
        "finish_entry_max": float(np.nanmax(rel[:, 5])), "ticket_max_nonlast": float(np.nanmax(rel[:, 6])),
        "export_done": float(rel[last, 7]) if last >= 0 else None,
        "steady_wait_us_per_team_med": float(np.median(full[:, 8:10]) / 1000.0),
        "blocks_per_team_med": float(np.median(full[:, 10:12])),
        # fused exchange, last CTA: finish entry -> limbs read, -> all ranks' lines summed, -> exported
        "fused_phases_us": [float((full[last, 12] - full[last, 5]) / 1000.0),
                            float((full[last, 14] - full[last, 12]) / 1000.0),
                            float((full[last, 15] - full[last, 14]) / 1000.0)] if fused and last >= 0 else None}),
        flush=True)
