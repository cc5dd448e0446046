"""Wall time of the stream-exact device toy generators at benchmark sizes.

    python scripts/toy_probe.py [--n1d 10000000] [--ndal 10000000]
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
    ap.add_argument("--n1d", type=int, default=10_000_000)
    ap.add_argument("--ndal", type=int, default=10_000_000)
    args = ap.parse_args()
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200.mcgen import GenSpec, generate_1d, generate_dalitz
    from tests import models

    x, pdf, _ = models.c1()
    generate_1d(pdf, x, GenSpec(100000, seed=1))  # warm-up (module load, plan)
    for seed in (1000, 1001):
        stats = {}
        t0 = time.perf_counter()
        ds = generate_1d(pdf, x, GenSpec(args.n1d, seed=seed), stats)
        dt = time.perf_counter() - t0
        print(json.dumps({"gen": "generate_1d C1", "n": ds.n_events, "seed": seed, "wall_s": dt,
                          "events_per_s": ds.n_events / dt, "attempts": stats["attempts"]}), flush=True)
    _, _, terms = models.c3()
    ch = pf.DecayChannel(*models.D_CHANNEL_T)
    generate_dalitz(terms, ch, GenSpec(10000, seed=1))
    for seed in (4,):
        stats = {}
        t0 = time.perf_counter()
        ds = generate_dalitz(terms, ch, GenSpec(args.ndal, seed=seed), stats=stats)
        dt = time.perf_counter() - t0
        print(json.dumps({"gen": "generate_dalitz C3", "n": ds.n_events, "seed": seed, "wall_s": dt,
                          "events_per_s": ds.n_events / dt, "box_draws": stats["box_draws"]}), flush=True)


if __name__ == "__main__":
    main()
