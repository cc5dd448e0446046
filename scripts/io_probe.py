"""Throughput of the binary column ingest (pfb_store_load_npy) at 100M rows.

    python scripts/io_probe.py [--n 100000000] [--dir /tmp/pfb_io]
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
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--dir", default="/tmp/pfb_io")
    args = ap.parse_args()
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import dataio
    from tests import models

    os.makedirs(args.dir, exist_ok=True)
    rng = np.random.default_rng(0)
    t0 = time.perf_counter()
    for name in ("s12", "s13"):
        np.save(os.path.join(args.dir, f"{name}.npy"), rng.uniform(0.5, 1.5, args.n))
    t_write = time.perf_counter() - t0
    (s12, s13), pdf, _ = models.c3()
    dataio.load_npy([s12, s13], args.dir, 0, 1000)  # warm-up (context, pinned buffers)
    for rep in range(2):
        t0 = time.perf_counter()
        ds = dataio.load_npy([s12, s13], args.dir)
        dt = time.perf_counter() - t0
        gb = 16 * ds.n_events / 1e9
        print(json.dumps({"rows": ds.n_events, "columns": 2, "bytes": 16 * ds.n_events, "wall_s": dt,
                          "GBps": gb / dt, "rep": rep, "write_s": t_write, "page_cache": rep > 0 or "likely"}),
              flush=True)
        del ds


if __name__ == "__main__":
    main()
