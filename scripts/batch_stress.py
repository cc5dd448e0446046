"""Batched-point stress: 16 C1 SumPdf parameter points per pass
(EvSum2GE::POINTS in the TMA unit kernel, every stage and fold slot reused
while a block's points are in flight), 20 random stencils x 10 repeats at
3M and 10M events -- each batch must equal its 16 single-point NLLs bit for
bit (the check that caught a miscompiled single-point variant of the kernel).

    python scripts/batch_stress.py [--out profiles/r2_batch_stress.jsonl]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="3000000,10000000")
    ap.add_argument("--stencils", type=int, default=20)
    ap.add_argument("--repeats", type=int, default=10)
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import paper_1710_08826_b200 as pf
    from tests import models
    from tests.test_gpu_batch import outcome, points_eval, single

    lines = []
    for n in (int(s) for s in args.sizes.split(",")):
        rng = np.random.default_rng(17)
        x, pdf, params = models.c1()
        xs = np.clip(np.concatenate([rng.normal(5, 0.5, n // 3), rng.exponential(3.3, n - n // 3)]), 0, 10)
        ds = models.dataset([x], [xs])
        base = np.array([4.9789, 0.5726, -0.3046, 0.3041])
        bad = batches = 0
        t0 = time.perf_counter()
        for _ in range(args.stencils):
            pts = [base + 1e-3 * rng.standard_normal(4) * (k > 0) for k in range(16)]
            want = [outcome(single(pf, pdf, ds, params, p)) for p in pts]
            snaps, norms = points_eval(pf, pdf, ds, params, pts)
            for _ in range(args.repeats):
                got = pf.DeviceBackend().evaluate_batch(pdf, {"x": ds.column("x")}, snaps, norms, 0, ds.n_events)
                bad += [outcome(r) for r in got] != want
                batches += 1
        rec = {"config": "C1 SumPdf, 16 points per pass", "events": n, "batches": batches,
               "mismatching_batches": bad, "wall_s": time.perf_counter() - t0}
        print(json.dumps(rec), flush=True)
        lines.append(rec)
    if args.out:
        with open(args.out, "w") as fh:
            for rec in lines:
                fh.write(json.dumps(rec) + "\n")
    sys.exit(1 if any(r["mismatching_batches"] for r in lines) else 0)


if __name__ == "__main__":
    main()
