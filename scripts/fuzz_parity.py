"""Randomised parity sweep: random PDF trees (gaussian / exponential /
polynomial leaves; sums over shared observables, products over disjoint
ones; 1-3 observables), random parameters, random event counts (1 .. 300k,
ragged), every pipeline mode and a random warps-per-block override -- each
device NLL against the reference's own nll on the same events (<= 1e-10
relative plus the ~n * 2^-53 absolute rounding of an n-term sum, see the
comparison; or the same exception class and index); for valid cases, three perturbed
parameter points evaluated as one batch (pfb_nll_batch) must equal their
single-point values bit for bit.

    python scripts/fuzz_parity.py [--cases 300] [--seed 1] [--out profiles/r2_fuzz.json]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

OBS = {"x": (0.0, 10.0), "y": (-2.0, 3.0), "z": (0.0, 1.0)}


def leaf(P, rng, o, name, hostile=False):
    """A primitive on one observable; `hostile` draws parameters that can make
    the density vanish (narrow gaussians far from the data) or go negative
    (polynomials with sign changes) -- the reference's error paths."""
    lo, hi = OBS[name]
    var = lambda v, a, b: P.Variable(f"p{rng.integers(1 << 30)}", float(v), a, b)
    k = int(rng.integers(3))
    if k == 0:
        sg = (hi - lo) * (rng.uniform(0.002, 0.01) if hostile else rng.uniform(0.05, 0.6))
        return P.gaussian(o, var(rng.uniform(lo, hi), lo - 5, hi + 5), var(sg, 1e-4, 100))
    if k == 1:
        return P.exponential(o, var(rng.uniform(-1.0, 1.0) / (hi - lo) * 3, -50, 50))
    deg = int(rng.integers(1, 4))
    if hostile:
        cs = list(rng.uniform(-1.0, 1.0, deg + 1))
    else:  # positive on the box
        cs = [1.0 + (2.0 if lo < 0 else 0.0)] + list(rng.uniform(0.0, 0.3, deg) / max(hi, 1.0) ** np.arange(1, deg + 1))
    return P.polynomial(o, [var(c, -100, 100) for c in cs])


def random_tree(P, rng, obs, names, depth=0, hostile=False):
    """A tree over exactly `names`: products split the observables, sums share them."""
    if len(names) > 1:
        cut = int(rng.integers(1, len(names)))
        return P.prod_pdf([random_tree(P, rng, obs, names[:cut], depth + 1, hostile),
                           random_tree(P, rng, obs, names[cut:], depth + 1, hostile)])
    if depth < 2 and rng.random() < 0.4:
        n = int(rng.integers(2, 4))
        kids = [random_tree(P, rng, obs, names, depth + 1, hostile) for _ in range(n)]
        fr = rng.dirichlet(np.ones(n))[: n - 1] * 0.9
        return P.add_pdf(kids, [P.Variable(f"f{rng.integers(1 << 30)}", float(f), 0.0, 1.0) for f in fr])
    return leaf(P, rng, obs[names[0]], names[0], hostile)


def outcome(fn):
    try:
        return ("ok", float(fn()))
    except Exception as exc:  # the reference's class and index
        return (type(exc).__name__, getattr(exc, "index", None))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=300)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import paper_1710_08826_b200 as pf

    P = pf.parafit
    ctx = pf.device_context(0)
    rng = np.random.default_rng(args.seed)
    bad, n_ok, n_err, worst, n_batch, n_cond = [], 0, 0, 0.0, 0, 0
    t0 = time.perf_counter()
    for case in range(args.cases):
        obs = {k: P.Variable.observable(k, *OBS[k]) for k in OBS}
        use = list(rng.permutation(list(OBS))[: int(rng.integers(1, 4))])
        pdf = random_tree(P, rng, obs, use, hostile=bool(rng.random() < 0.3))
        names = sorted({n for node in pdf.walk() for n in node.observable_names()})
        n = int(rng.choice([1, 2, 17, 4095, 4097, 9000, 50_001, 300_000]))
        cols = [rng.uniform(*OBS[k], n) for k in names]
        ds = pf.DeviceDataSet.from_columns([obs[k] for k in names], cols, device=None)
        snap = P.snapshot(pdf.param_closure())
        with pf.reference_norms():
            want = outcome(lambda: P.nll(pdf, ds, snap, P.Backend("serial"), P.NormalizationStore()))
        results = {}
        try:
            for mode in (1, 2, 3, 0):
                ctx.set_pipeline(mode)
                results[mode] = outcome(lambda: pf.nll(pdf, ds))
            w = int(rng.choice([1, 2, 4, 8]))
            ctx.set_pipeline(1)
            ctx.set_warps_per_block(w)
            results[f"w{w}"] = outcome(lambda: pf.nll(pdf, ds))
        finally:
            ctx.set_pipeline(1)
            ctx.set_warps_per_block(0)
        for key, got in results.items():
            if want[0] == "ok":
                r = abs(got[1] - want[1]) / max(abs(want[1]), 1e-300) if got[0] == "ok" else math.inf
                worst = max(worst, r)
                # 1e-10 relative, plus the absolute rounding of a sum of n
                # per-event terms (~n * 2^-53: product-mode units, table
                # logarithms, and the reference's own np.dot polynomial norm,
                # BLAS order, vs the device's correctly rounded dot product) --
                # more than 1e-10 relative only when the NLL cancels to far
                # below n (e.g. 0.22 over 300k events of a near-flat density)
                allow = 1e-10 * abs(want[1]) + 8.0 * n * 2.0 ** -53
                if not (got[0] == "ok" and abs(got[1] - want[1]) <= allow):
                    bad.append({"case": case, "mode": key, "n": n, "tree": repr(pdf), "want": want, "got": got})
                elif r > 1e-10:
                    n_cond += 1
            elif got != want:
                bad.append({"case": case, "mode": key, "n": n, "tree": repr(pdf), "want": want, "got": got})
        # batched points (pfb_nll_batch) bitwise their single-point values
        free = [v for v in pdf.param_closure() if not v.fixed]
        if free and want[0] == "ok":
            base = np.array([v.value for v in free])
            pts = [base * (1.0 + 1e-4 * k) for k in range(3)]
            singles, snaps, norms = [], [], []
            store = P.NormalizationStore()
            for pt in pts:
                for v, val in zip(free, pt):
                    P.set_value(v, float(np.clip(val, v.lower, v.upper)))
                singles.append(outcome(lambda: pf.nll(pdf, ds)))
                sn = P.snapshot(pdf.param_closure())
                snaps.append(sn)
                norms.append(P.resolve_norms(pdf, sn, store))
            cols_d = {k: ds.column(k) for k in names}
            got = pf.DeviceBackend().evaluate_batch(pdf, cols_d, snaps, norms, 0, ds.n_events)
            got = [("ok", float(g)) if not isinstance(g, Exception) else (type(g).__name__, getattr(g, "index", None))
                   for g in got]
            if got != singles:
                bad.append({"case": case, "mode": "batch", "n": n, "tree": repr(pdf), "want": singles, "got": got})
            n_batch += 1
        if want[0] == "ok":
            n_ok += 1
        else:
            n_err += 1
    out = {"cases": args.cases, "seed": args.seed, "ok_cases": n_ok, "error_cases": n_err,
           "evaluations": args.cases * 5, "batched_cases": n_batch, "worst_rel": worst,
           "within_sum_rounding_allowance_only": n_cond, "mismatches": bad[:20], "n_mismatches": len(bad),
           "wall_s": time.perf_counter() - t0}
    line = json.dumps(out)
    print(line)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(line + "\n")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
