"""Determinism stress: the barrier-free kernels (mbarrier rings, last-arriver
folds, CTA tickets, self-resetting counters) must give the same bits on every
call.  Repeats the NLL many times per configuration and size -- each kernel
family, ragged and odd sizes, batched points -- and counts any call whose
value differs from the first.

    python scripts/stress_probe.py [--reps 400]
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=400)
    ap.add_argument("--sizes", default="1000003,10000000,37000001")
    ap.add_argument("--batch", action="store_true", help="also the batched objective (16 points per pass)")
    args = ap.parse_args()
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import mcgen
    from tests import models

    ctx = pf.device_context(0)
    bad_total = 0
    for n in [int(v) for v in args.sizes.split(",")]:
        cases = []
        x, pdf1, p1 = models.c1()
        col = mcgen.device_sumpdf_1d(n, 5.0, 0.5, -0.3, 0.3, 0.0, 10.0, 11)
        cases.append(("c1", pdf1, pf.UnbinnedDataSet.from_columns([x], [col], copy=False), p1))
        (xx, yy), pdf2, p2 = models.c2()
        cx, cy = mcgen.device_prod_2d(n, 5.0, 1.0, -0.4, 0.0, 10.0, 12)
        cases.append(("c2", pdf2, pf.UnbinnedDataSet.from_columns([xx, yy], [cx, cy], copy=False), p2))
        terms = [(p, s, m, w, mag, ph) for (p, m, w, s, mag, ph) in models.C3_TERMS]
        a, b = mcgen.device_dalitz(n, terms, models.D_CHANNEL_T, 13)
        (o12, o13), pdf3, rts = models.c3()
        cases.append(("c3", pdf3, pf.UnbinnedDataSet.from_columns([o12, o13], [a, b], copy=False), None))
        for name, pdf, ds, _ in cases:
            for pipeline in (1, 3, 0):
                ctx.set_pipeline(pipeline)
                first = pf.nll(pdf, ds)
                t0 = time.perf_counter()
                diff = sum(1 for _ in range(args.reps) if pf.nll(pdf, ds) != first)
                dt = time.perf_counter() - t0
                bad_total += diff
                print(json.dumps({"cfg": name, "n": n, "pipeline": pipeline, "reps": args.reps, "mismatches": diff,
                                  "nll": first.hex(), "us_per_call": 1e6 * dt / args.reps}), flush=True)
            ctx.set_pipeline(1)
            if args.batch and name != "c3":
                from paper_1710_08826_b200.engine import _needed_columns, default_backend

                be = default_backend()
                cols = _needed_columns(pdf, ds)
                params = [v for v in pdf.param_closure() if not v.fixed]
                snaps, norms_l, singles = [], [], []
                base = [v.value for v in params]
                for k in range(16):
                    for j, v in enumerate(params):
                        pf.set_value(v, base[j] * (1.0 + 1e-3 * ((k + j) % 5 - 2)))
                    snap = pf.snapshot(pdf.param_closure())
                    nm = pf.resolve_norms(pdf, snap, pf.NormalizationStore())
                    snaps.append(snap)
                    norms_l.append(nm)
                    singles.append(pf.nll(pdf, ds))
                for j, v in enumerate(params):
                    pf.set_value(v, base[j])
                diff = 0
                for _ in range(max(1, args.reps // 10)):
                    vals = be.evaluate_batch(pdf, cols, snaps, norms_l, 0, ds.n_events)
                    diff += sum(1 for a, b in zip(vals, singles) if a != b)
                bad_total += diff
                print(json.dumps({"cfg": name, "n": n, "batch": 16, "reps": max(1, args.reps // 10),
                                  "mismatches_vs_single": diff}), flush=True)
    print(json.dumps({"stress": "done", "mismatches": bad_total}), flush=True)
    if bad_total:
        sys.exit(1)


if __name__ == "__main__":
    main()
