"""Determinism under repetition: each config's NLL evaluated
`--calls` times on the same device data must give one bit pattern; the
product-mode configs also across kernel shells (pipelines 1 / 2 / 3).

    python scripts/stress_probe.py [--calls 2000] [--out profiles/r2_stress_determinism.jsonl]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=2000)
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import bench
    import paper_1710_08826_b200 as pf

    P = pf.parafit
    ctx = pf.device_context(0)
    lines = []
    for cfg, shells in (("c1", (1, 2, 3)), ("c5", (1, 2, 3)), ("c2", (1,)), ("c3", (1, 2, 3)), ("c2p", (1, 2, 3))):
        n = bench.CONFIGS[cfg]["n"]
        print("config", cfg, n, file=sys.stderr, flush=True)
        cols = bench.events(cfg, n, 11)
        obs, pdf, _ = bench.build_model(P, bench.CONFIGS[cfg]["model"])
        ds = pf.DeviceDataSet.from_columns(obs, cols, device=0)
        seen = {}
        t0 = time.perf_counter()
        for shell in shells:
            ctx.set_pipeline(shell)
            for _ in range(args.calls // len(shells)):
                v = pf.nll(pdf, ds)
                seen[v.hex()] = seen.get(v.hex(), 0) + 1
        ctx.set_pipeline(1)
        rec = {"config": cfg, "events": n, "calls": sum(seen.values()), "shells": list(shells),
               "distinct_values": len(seen), "value": next(iter(seen)), "wall_s": time.perf_counter() - t0}
        print(json.dumps(rec), flush=True)
        lines.append(json.dumps(rec))
        del ds
    if args.out:
        with open(args.out, "w") as fh:
            fh.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
