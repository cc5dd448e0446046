"""Where the host time of one Dalitz nll() call goes (C3 model, cProfile over
repeated calls with a free parameter moving, as a fit drives it)."""

import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200.engine import NormalizationStore, device_context
    from paper_1710_08826_b200.mcgen import GenSpec, generate_dalitz
    from tests import models

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    obs, pdf, rts = models.c3()
    ch = pf.DecayChannel(*models.D_CHANNEL_T)
    ds = generate_dalitz(rts, ch, GenSpec(n, seed=7), observables=obs)
    free = [v for v in pdf.param_closure() if not v.fixed]
    store = NormalizationStore()
    for _ in range(5):
        pf.nll(pdf, ds, store=store)
    reps = 300
    t0 = time.perf_counter()
    for i in range(reps):
        pf.set_value(free[0], free[0].value + (1e-6 if i % 2 else -1e-6))
        pf.nll(pdf, ds, store=store)
    dt = (time.perf_counter() - t0) / reps
    ctx = device_context(0)
    ctx.enable_timing(True)
    ks = []
    for i in range(50):
        pf.set_value(free[0], free[0].value + (1e-6 if i % 2 else -1e-6))
        pf.nll(pdf, ds, store=store)
        ks.append(ctx.last_kernel_ms())
    ctx.enable_timing(False)
    k_us = 1e3 * sorted(ks)[len(ks) // 2]
    print(f"events={n} free={len(free)} nll() {1e6 * dt:.1f} us/call, kernel (CUDA events, median) {k_us:.1f} us, "
          f"host + launch {1e6 * dt - k_us:.1f} us")
    prof = cProfile.Profile()
    prof.enable()
    for i in range(reps):
        pf.set_value(free[0], free[0].value + (1e-6 if i % 2 else -1e-6))
        pf.nll(pdf, ds, store=store)
    prof.disable()
    pstats.Stats(prof).sort_stats("tottime").print_stats(22)


if __name__ == "__main__":
    main()
