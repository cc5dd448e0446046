"""Device-time sweep of the NLL kernels: evaluator x warps-per-block.

    python scripts/kernel_sweep.py [--n 10000000] [--configs terms,c1,c2,c2p,c3] [--warps 0,1,2,4,8]

Each measurement: 3 warm-up calls, then `reps` calls each preceded by a
256 MB L2-evicting write; device time of the fused kernel from CUDA events
on its stream (pfb_ctx timing).  Prints one JSON line per point.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--configs", default="terms,c1,c2,c3")
    ap.add_argument("--warps", default="0,1,2,4,8")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--cache", type=int, default=0, help="Dalitz lineshape cache mode")
    ap.add_argument("--pipeline", type=int, default=1, help="1: TMA pipeline, 0: SIMT streaming kernel")
    ap.add_argument("--spin", default="native", choices=["native", "torch"],
                    help="pre-launch flush + spin: pfb_ctx_spin (same carveout) or torch flush.sum + _sleep")
    args = ap.parse_args()

    import torch

    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L
    from paper_1710_08826_b200 import mcgen
    from tests import models

    torch.cuda.set_device(0)
    ctx = pf.device_context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    ctx.enable_timing(True)
    L.check(L.lib().pfb_ctx_set_pipeline(ctx.handle, args.pipeline), "pfb_ctx_set_pipeline")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    print(json.dumps({"fp64_peak_tflops": ctx.fp64_peak_tflops()}), flush=True)

    def pre():
        # L2 eviction + ~0.5 ms of GPU work: the host has enqueued the launch
        # (and its ev0) before the GPU reaches them
        if args.spin == "native":
            ctx.spin(1_000_000, flush.data_ptr(), flush.numel() * 4)
        else:
            flush.sum()
            torch.cuda._sleep(1_000_000)

    n = args.n
    warps_list = [int(w) for w in args.warps.split(",")]

    for cfg in args.configs.split(","):
        t0 = time.perf_counter()
        if cfg == "terms":
            rng = np.random.default_rng(0)
            terms = rng.normal(size=n)
            out = np.empty(-(-n // 4096))
            total = ctypes.c_double()
            for w in warps_list:
                ctx.set_warps_per_block(w)
                times = []
                for r in range(3 + args.reps):
                    pre()
                    L.check(L.lib().pfb_terms_block_sums(ctx.handle, L.dptr(terms), n, L.dptr(out),
                                                         ctypes.byref(total)), "terms")
                    if r >= 3:
                        times.append(ctx.last_kernel_ms())
                ms = float(np.median(times))
                print(json.dumps({"config": "terms", "n": n, "warps": w, "pipeline": args.pipeline, "kernel_ms": ms,
                                  "GBps": 8 * n / ms / 1e6}), flush=True)
            continue
        if cfg == "c1":
            cols = [mcgen.sumpdf_1d(n, 5.0, 0.5, -0.3, 0.3, 0.0, 10.0, 1)]
            obs, pdf, _ = models.c1()
            obs = [obs]
        elif cfg == "c2":
            cols = list(mcgen.prod_2d(n, 5.0, 1.0, -0.4, 0.0, 10.0, 2))
            obs, pdf, _ = models.c2()
        elif cfg == "c2p":  # gaussian(x) x polynomial(y), bench.py's C2p sub-result
            import bench

            obs, pdf, _ = bench.build_model(pf.parafit, "c2p")
            cols = bench.host_events("c2p", n, 5)
        else:
            terms = [(p, s, m, w, mag, ph) for (p, m, w, s, mag, ph) in models.C3_TERMS]
            cols = list(mcgen.device_dalitz(n, terms, models.D_CHANNEL_T, 3))  # Philox on the GPU
            obs, pdf, _ = models.c3()
        gen_s = time.perf_counter() - t0
        ds = pf.DeviceDataSet.from_columns(list(obs), cols, device=None)
        backend = pf.DeviceBackend(lineshape_cache=args.cache if cfg == "c3" else 0)
        for w in warps_list:
            ctx.set_warps_per_block(w)
            times = []
            val = None
            for r in range(3 + args.reps):
                pre()
                val = pf.nll(pdf, ds, backend=backend)
                if r >= 3:
                    times.append(ctx.last_kernel_ms())
            ms = float(np.median(times))
            ms_mean = float(np.mean(times))  # event stamps tick in ~1 us steps: the mean resolves less
            nbytes = 8 * len(cols) * n
            names = tuple(sorted(o.name for o in obs))
            print(json.dumps({"config": cfg, "n": n, "warps": w, "pipeline": args.pipeline, "kernel_ms": ms,
                              "kernel_ms_mean": ms_mean, "GBps": nbytes / ms / 1e6,
                              "Gevents_per_s": n / ms / 1e6, "evaluator": ctx.plan_for(pdf, names).evaluator,
                              "nll": val, "gen_s": gen_s}), flush=True)
    ctx.set_warps_per_block(0)


if __name__ == "__main__":
    main()
