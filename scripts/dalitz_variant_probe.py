"""Kernel time of Dalitz models other than the C3 D0 -> pi pi pi0 one (K = 2,
3, 5 and K pi pi with unequal masses, tests/models.py DALITZ_VARIANTS) at 10M
events: which evaluator each plan gets and how fast it runs.

    python scripts/dalitz_variant_probe.py [--n 10000000]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    args = ap.parse_args()
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import mcgen
    from tests import models

    ctx = pf.device_context(0)
    ctx.enable_timing(True)
    for name in ["c3"] + sorted(models.DALITZ_VARIANTS):
        if name == "c3":
            (o12, o13), pdf, rts = models.c3()
            ch_t, spec = models.D_CHANNEL_T, [(p, s, m, w, mag, ph) for (p, m, w, s, mag, ph) in models.C3_TERMS]
        else:
            (o12, o13), pdf, rts = models.dalitz_variant(pf, name)
            ch_t, sp, _ = models.DALITZ_VARIANTS[name]
            spec = [(p, s, m, w, mag, ph) for (p, m, w, s, mag, ph) in sp]
        a, b = mcgen.device_dalitz(args.n, spec, ch_t, 5)
        ds = pf.UnbinnedDataSet.from_columns([o12, o13], [a, b], copy=False)
        store = pf.NormalizationStore()
        pf.nll(pdf, ds, store=store)
        ts = []
        for _ in range(10):
            pf.nll(pdf, ds, store=store)
            ts.append(ctx.last_kernel_ms())
        plan = ctx.plan_for(pdf, ("s12", "s13"))
        t = sorted(ts)[len(ts) // 2]
        print(json.dumps({"model": name, "K": len(rts), "n": args.n, "evaluator": plan.evaluator,
                          "kernel_us": 1e3 * t, "events_per_s": args.n / (t * 1e-3)}), flush=True)


if __name__ == "__main__":
    main()
