"""Where the host time of one nll() call goes (cProfile over repeated calls)."""

import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import mcgen
    from paper_1710_08826_b200.engine import NormalizationStore
    from tests import models

    x, pdf, params = models.c1()
    col = mcgen.device_sumpdf_1d(1_000_000, 5.0, 0.5, -0.3, 0.3, 0.0, 10.0, 1)
    ds = pf.UnbinnedDataSet.from_columns([x], [col], copy=False)
    store = NormalizationStore()
    for _ in range(5):
        pf.nll(pdf, ds, store=store)
    n = 300
    t0 = time.perf_counter()
    for i in range(n):
        pf.set_value(params[0], 5.0 + 1e-4 * (i % 5))
        pf.nll(pdf, ds, store=store)
    print(f"nll() with a persistent store: {1e6 * (time.perf_counter() - t0) / n:.1f} us/call")
    t0 = time.perf_counter()
    for i in range(n):
        pf.nll(pdf, ds)
    print(f"nll() with a fresh store: {1e6 * (time.perf_counter() - t0) / n:.1f} us/call")
    prof = cProfile.Profile()
    prof.enable()
    for i in range(n):
        pf.set_value(params[0], 5.0 + 1e-4 * (i % 5))
        pf.nll(pdf, ds, store=store)
    prof.disable()
    pstats.Stats(prof).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
