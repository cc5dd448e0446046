"""Batched-point stress: 16 parameter points per pass in the TMA unit
kernel (every stage and fold slot reused while a block's points are in
flight) -- C1 SumPdf points (EvSum2GE::POINTS, default), D0 Dalitz
coefficient points (EvDalitzR<4,D0,true>) or gaussian x polynomial points
(EvGaussPoly) -- 20 random stencils x 10 repeats per size: each batch must
equal its 16 single-point NLLs bit for bit (the check that caught a
miscompiled single-point variant of the kernel).

    python scripts/batch_stress.py [--model c1|c3|c2p] [--sizes 3000000,10000000] [--out FILE]
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
    ap.add_argument("--model", default="c1", choices=["c1", "c3", "c2p"],
                    help="c1: EvSum2GE points; c3: D0 Dalitz coefficient points; c2p: gaussian x polynomial")
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import bench
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import mcgen
    from tests import models
    from tests.test_gpu_batch import outcome, points_eval, single

    lines = []
    for n in (int(s) for s in args.sizes.split(",")):
        rng = np.random.default_rng(17)
        if args.model == "c1":
            x, pdf, params = models.c1()
            xs = np.clip(np.concatenate([rng.normal(5, 0.5, n // 3), rng.exponential(3.3, n - n // 3)]), 0, 10)
            ds = models.dataset([x], [xs])
            base = np.array([4.9789, 0.5726, -0.3046, 0.3041])
            label = "C1 SumPdf"
        elif args.model == "c3":
            terms = [(p, s_, m, w, mag, ph) for (p, m, w, s_, mag, ph) in models.C3_TERMS]
            cols = list(mcgen.device_dalitz(n, terms, models.D_CHANNEL_T, 5))
            (o12, o13), pdf, tl = models.c3(grid=(128, 128))
            ds = pf.DeviceDataSet.from_columns([o12, o13], cols, device=None)
            params = [v for t in tl for v in (t.magnitude, t.phase) if not v.fixed]
            base = np.array([v.value for v in params])
            label = "C3 D0 Dalitz (coefficient points)"
        else:
            obs, pdf, params = bench.build_model(pf.parafit, "c2p")
            ds = pf.DeviceDataSet.from_columns(obs, bench.host_events("c2p", n, 5), device=None)
            base = np.array([v.value for v in params])
            label = "C2p gaussian x polynomial"
        names = sorted({o.name for node in pdf.walk() for o in node.observables})
        cols_d = {k: ds.column(k) for k in names}
        bad = batches = 0
        t0 = time.perf_counter()
        for _ in range(args.stencils):
            pts = [base * (1.0 + 1e-3 * rng.standard_normal(len(base)) * (k > 0)) for k in range(16)]
            want = [outcome(single(pf, pdf, ds, params, p)) for p in pts]
            snaps, norms = points_eval(pf, pdf, ds, params, pts)
            for _ in range(args.repeats):
                got = pf.DeviceBackend().evaluate_batch(pdf, cols_d, snaps, norms, 0, ds.n_events)
                bad += [outcome(r) for r in got] != want
                batches += 1
        for v, val in zip(params, base):
            pf.parafit.set_value(v, float(val))
        rec = {"config": f"{label}, 16 points per pass", "events": n, "batches": batches,
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
