"""Benchmark: NLL evaluations/s and events/s of the B200 engine.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

A step is one NLL evaluation over the configuration's full event set.  The
default workload is BASELINE.json configs[1]: the 2-D ProductPdf
(Gaussian(x) x Exponential(y)), 10M synthetic events per GPU (weak scaling;
at N>1 ranks hold disjoint shards and combine exact partials with one NCCL
all-reduce of the 72-word integer accumulator).

* value   -- events/s with the events resident in HBM: per-step device time
             of the fused NLL kernel (CUDA events on its stream), L2 flushed
             (256 MB read, pfb_ctx_spin) before every step.
* e2e     -- the same metric through the C ABI with host (pinned) columns:
             every step copies the events host->device (chunked, overlapped
             with the kernels) and reads the result back.
* roofline -- algorithmic bytes (8 B per observable per event) / kernel time
             against MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline -- the reference algorithm (oracle port, numpy, all host
             threads) on a bounded sample, rank 0, N=1.

--impl reference times the reference CPU path (the oracle port of the
reference's numpy implementation) on the same config and prints the same line.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np
from paper_1710_08826_b200._reference import parafit as P

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NLL evals/sec & events/sec (1/2/4/8 B200) vs CPU ref; % HBM/FP64 roofline"

CONFIGS = {
    "c1": dict(workload="C1 SumPdf 1-D (gauss+exp), 1M events", n=1_000_000, ncols=1),
    "c2": dict(workload="C2 ProductPdf 2-D (gauss(x) x exp(y)), 10M events", n=10_000_000, ncols=2),
    "c3": dict(workload="C3 Dalitz D0->pi+pi-pi0 (rho+, rho-, rho0, NR), 10M events", n=10_000_000, ncols=2),
    "c4": dict(workload="C4 Dalitz D0->pi+pi-pi0, 100M events sharded over the GPUs (strong scaling)",
               n=100_000_000, ncols=2),
    "c5": dict(workload="C5 toy unit: SumPdf 1-D, 10M events", n=10_000_000, ncols=1),
}


# SURVEY.md 8(d) algorithmic figures (each + - x / = 1 flop, exp/log = 1):
# 4 terms x 20 + s23 2 + |T|^2 3 + /norm 1 + -log 2 + accumulate 1 (rounded to 84)
FLOPS_PER_EVENT = {"c3": 84, "c4": 84}
VENDOR_FP64_TFLOPS = 37.0


def log(msg: str) -> None:
    print(msg, file=sys.stderr, flush=True)


def make_data(cfg: str, n: int, seed: int, device: bool = True):
    """Synthetic events of the configuration's model: generated on the GPU
    (pfb_gen_*) when one is available, else with the host numpy samplers."""
    from paper_1710_08826_b200 import mcgen

    if cfg in ("c1", "c5"):
        if device:
            return [mcgen.device_sumpdf_1d(n, 5.0, 0.5, -0.3, 0.3, 0.0, 10.0, seed)]
        return [mcgen.sumpdf_1d(n, 5.0, 0.5, -0.3, 0.3, 0.0, 10.0, seed)]
    if cfg == "c2":
        if device:
            return list(mcgen.device_prod_2d(n, 5.0, 1.0, -0.4, 0.0, 10.0, seed))
        return list(mcgen.prod_2d(n, 5.0, 1.0, -0.4, 0.0, 10.0, seed))
    if cfg in ("c3", "c4"):
        from tests import models

        terms = [(p, s, m, w, mag, ph) for (p, m, w, s, mag, ph) in models.C3_TERMS]
        if device:
            return list(mcgen.device_dalitz(n, terms, models.D_CHANNEL_T, seed))
        return list(mcgen.dalitz(n, terms, models.D_CHANNEL_T, seed))
    raise ValueError(cfg)


def build_model(cfg: str):
    from tests import models

    if cfg in ("c1", "c5"):
        x, pdf, _ = models.c1()
        return [x], pdf
    if cfg == "c2":
        obs, pdf, _ = models.c2()
        return list(obs), pdf
    obs, pdf, _ = models.c3()
    return list(obs), pdf


def oracle_spec(cfg: str):
    from tests import models

    if cfg in ("c1", "c5"):
        return models.c1_spec((5.0, 0.5, -0.3, 0.3)), ("x",)
    if cfg == "c2":
        return models.c2_spec((5.0, 1.0, -0.4)), ("x", "y")
    return models.c3_spec(), ("s12", "s13")


def cpu_reference_rate(cfg: str, cols, budget_s: float = 12.0, max_calls: int = 200):
    """The reference algorithm (oracle port of parafit's numpy path) with all host threads."""
    from oracle import parafit_oracle as O

    spec, names = oracle_spec(cfg)
    data = dict(zip(names, cols))
    n = len(cols[0])
    threads = os.cpu_count() or 1
    O.nll(spec, data, workers=threads)  # warm-up (norm / grid integrals)
    t0 = time.perf_counter()
    calls = 0
    while calls < max_calls:
        O.nll(spec, data, workers=threads)
        calls += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    return n * calls / dt, threads, f"{calls} NLL calls x {n} events (full {cfg} event set), pool({threads})"


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return None
        rows = [r.split(", ") for r in open(self.path).read().strip().splitlines() if r.strip()]
        rows = [r for r in rows if len(r) >= 9]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=0, help="override events per GPU")
    ap.add_argument("--collective", default="fused", choices=["fused", "nccl", "peer"],
                    help="N > 1: the accumulator exchange fused into the NLL kernel over NVLink peer memory "
                         "(pfb_nll_peer; NCCL if the peer set-up fails or disagrees), an NCCL all-reduce, "
                         "or the separate peer-memory kernel (pfb_peer_allreduce)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = args.config
    n_per = args.n or CONFIGS[cfg]["n"]
    scaling = "weak"
    if cfg == "c4" and not args.n:
        # strong scaling: the 100M events are sharded over the ranks
        # with the reference's shard() bounds
        from paper_1710_08826_b200.sharding import shard_bounds

        b = shard_bounds(CONFIGS[cfg]["n"], world)
        n_per = b[rank + 1] - b[rank]
        scaling = "strong"

    if args.impl == "reference":
        if rank != 0:
            return
        cols = make_data(cfg, n_per, seed=1000, device=False)
        steps = max(1, args.steps)
        rates = []
        from oracle import parafit_oracle as O

        spec, names = oracle_spec(cfg)
        data = dict(zip(names, cols))
        threads = os.cpu_count() or 1
        for _ in range(max(0, args.warmup)):
            O.nll(spec, data, workers=threads)
        t0 = time.perf_counter()
        for _ in range(steps):
            O.nll(spec, data, workers=threads)
        dt = time.perf_counter() - t0
        value = n_per * steps / dt
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIGS[cfg]["workload"], "n_events": n_per},
            "nll_evals_per_s": steps / dt,
            "cpu_baseline": {"value": value, "unit": "events/s", "cores": threads, "kind": "port",
                             "sample": f"{steps} NLL calls x {n_per} events, pool({threads})"},
            "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return

    import torch

    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", init_method="env://")
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()

    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    t_gen = time.perf_counter()
    cols = make_data(cfg, n_per, seed=1000 + rank)
    log(f"[rank {rank}] generated {n_per} events for {cfg} in {time.perf_counter() - t_gen:.1f}s")
    obs, pdf = build_model(cfg)
    ds = P.UnbinnedDataSet.from_columns(obs, cols, copy=False)  # keeps the generated HBM copy
    ctx = pf.device_context(dev)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    ctx.enable_timing(True)
    names = tuple(sorted(o.name for o in obs))
    arrays = [ds.column(nm) for nm in names]
    plan = ctx.plan_for(pdf, names)
    store = ctx.store_for(arrays)
    snap = P.snapshot(pdf.param_closure())
    norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
    vals, nv = plan.pack(snap, norms)
    acc = torch.zeros(L.PFB_ACC_WORDS, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    out = ctypes.c_double()
    err = L.PfbErr()

    peers = None
    collective = args.collective if world > 1 else "none"
    if world > 1 and collective in ("peer", "fused"):
        from paper_1710_08826_b200.sharding import PeerGroup

        try:  # collective on every rank: a failure raises everywhere, nobody hangs
            peers = PeerGroup(ctx, rank, world, timeout_s=5.0)
        except Exception as exc:  # no CUDA IPC / peer access: the NCCL path still measures the step
            log(f"[rank {rank}] peer-memory set-up failed ({exc}); using NCCL")
            collective = "nccl (peer set-up failed)"
    ev_a = torch.cuda.Event(enable_timing=True)
    ev_b = torch.cuda.Event(enable_timing=True)

    def step_local():
        """One NLL over the local events; returns the kernel's device ms."""
        if world == 1:
            code = L.lib().pfb_nll(ctx.handle, plan.handle, store, 0, n_per, 0, L.dptr(vals), len(vals),
                                   L.dptr(nv), len(nv), ctypes.byref(out), ctypes.byref(err))
            L.check(code, "pfb_nll")
            return ctx.last_kernel_ms(), out.value
        if collective == "fused":
            # N > 1, fused: one launch per step, the exchange of the 72-word
            # exact accumulator over NVLink peer memory inside the kernel
            slow = ctypes.c_int32()
            code = L.lib().pfb_nll_peer(ctx.handle, plan.handle, store, 0, n_per, 0, L.dptr(vals), len(vals),
                                        L.dptr(nv), len(nv), peers.timeout_s, ctypes.byref(out), ctypes.byref(slow))
            L.check(code, "pfb_nll_peer")
            if slow.value:
                raise SystemExit("fused step took the slow path (deferred blocks or an error on a rank)")
            return ctx.last_kernel_ms(), out.value
        # N > 1: the step is the fused kernel plus the all-reduce of the 72-word
        # exact accumulator, timed together with CUDA events on this stream
        ev_a.record()
        L.check(L.lib().pfb_nll_partial_async(ctx.handle, plan.handle, store, 0, n_per, 0, L.dptr(vals), len(vals),
                                              L.dptr(nv), len(nv), ctypes.c_void_p(acc.data_ptr())), "partial")
        if peers is not None and collective == "peer":
            peers.allreduce(acc)
        else:
            torch.distributed.all_reduce(acc)
        ev_b.record()
        fails = ctypes.c_int64()
        L.check(L.lib().pfb_finalize(ctx.handle, ctypes.c_void_p(acc.data_ptr()), ctypes.byref(out),
                                     ctypes.byref(fails)), "finalize")
        return ev_a.elapsed_time(ev_b), out.value

    def warm_up():
        for _ in range(max(3, args.warmup)):
            flush.zero_()
            step_local()

    if collective == "fused":
        try:
            warm_up()
            ok = 1
        except Exception as exc:  # a peer timeout or error: decide together, fall back to NCCL
            log(f"[rank {rank}] fused warm-up failed ({exc})")
            ok = 0
        t_ok = torch.tensor([ok], device=dev)
        torch.distributed.all_reduce(t_ok, op=torch.distributed.ReduceOp.MIN)
        if int(t_ok.item()) == 0:
            collective = "nccl (fused exchange failed in warm-up)"
            warm_up()
    else:
        warm_up()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    # cross-check (untimed): the same NLL through the SIMT reference-tree kernel
    # (pipeline 0) must agree with the fast kernel to rounding
    _, fast_nll = step_local()
    L.check(L.lib().pfb_ctx_set_pipeline(ctx.handle, 0), "pfb_ctx_set_pipeline")
    _, simt_nll = step_local()
    L.check(L.lib().pfb_ctx_set_pipeline(ctx.handle, 1), "pfb_ctx_set_pipeline")
    crosscheck = abs(fast_nll - simt_nll) / abs(simt_nll)
    if not crosscheck <= 1e-12:
        raise SystemExit(f"NLL cross-check failed: fast kernel {fast_nll!r} vs SIMT kernel {simt_nll!r}")
    if collective == "fused":
        # the exchange inside the kernel must give the NCCL path's bits (every
        # rank sees the same two global values, so all ranks decide alike)
        _, fused_nll = step_local()
        collective = "nccl"
        _, nccl_nll = step_local()
        collective = "fused" if fused_nll == nccl_nll else "nccl (fused exchange disagreed)"
        if collective != "fused":
            log(f"[rank {rank}] fused exchange {fused_nll!r} != NCCL {nccl_nll!r}; timing the NCCL path")

    launches0 = ctx.launch_count()
    kernel_ms = []
    with ClockSampler(dev) as clocks:
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            # evict L2 (256 MB streaming read > 126 MB L2) and keep every SM
            # busy ~0.5 ms while the host prepares the launch, so the CUDA
            # events around the kernel time the kernel, not launch latency
            # (pfb_ctx_spin: same shared-memory carveout as the NLL kernels,
            # as in a fit loop where only NLL launches reach the GPU)
            if world > 1:  # ranks start each step together (outside the event window)
                torch.distributed.barrier()
            ctx.spin(1_000_000, flush.data_ptr(), flush.numel() * flush.element_size())
            ms, nll_value = step_local()
            kernel_ms.append(ms)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        wall = time.perf_counter() - t0
    launches = ctx.launch_count() - launches0
    dev_s = float(np.sum(kernel_ms)) / 1e3
    if world > 1:
        t = torch.tensor([dev_s], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_s = float(t.item())
    total_events = n_per * world * args.steps
    value = total_events / dev_s
    ms_per_step = 1e3 * dev_s / args.steps

    # ---- end to end through the C ABI with pinned host columns
    pinned = [torch.empty(n_per, dtype=torch.float64, pin_memory=True) for _ in arrays]
    for p, a in zip(pinned, arrays):
        p.numpy()[:] = a
    hcols = (L._DBL_P * len(pinned))(*[ctypes.cast(p.data_ptr(), L._DBL_P) for p in pinned])
    e2e_steps = max(3, min(args.steps, 10))
    L.check(L.lib().pfb_nll_host(ctx.handle, plan.handle, hcols, len(pinned), n_per, L.dptr(vals), len(vals),
                                 L.dptr(nv), len(nv), ctypes.byref(out), ctypes.byref(err)), "pfb_nll_host")
    e2e_value_nll = out.value
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        L.check(L.lib().pfb_nll_host(ctx.handle, plan.handle, hcols, len(pinned), n_per, L.dptr(vals), len(vals),
                                     L.dptr(nv), len(nv), ctypes.byref(out), ctypes.byref(err)), "pfb_nll_host")
    e2e_dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_dt], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_dt = float(t.item())
    e2e = {"value": n_per * world * e2e_steps / e2e_dt, "unit": "events/s",
           "h2d_bytes_per_step": 8 * len(arrays) * n_per, "d2h_bytes_per_step": 8 * 8,
           "steps": e2e_steps, "nll_matches_device": e2e_value_nll == nll_value}

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return

    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        peak, peak_src = float(json.load(open(peaks_path))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    algo_bytes = 8 * len(arrays) * n_per
    achieved = algo_bytes / (ms_per_step * 1e-3) / 1e9
    # DRAM traffic of the dominant kernel from the committed ncu --set full
    # capture (profiles/traffic_<cfg>.json, 10M events), per launch of this
    # run: measured bytes/event x events per launch.  C4 runs the C3 kernel.
    traffic = None
    tcfg = {"c4": "c3", "c5": "c1"}.get(cfg, cfg)
    tpath = os.path.join(ROOT, "profiles", f"traffic_{tcfg}.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        traffic = tj["bytes_per_launch"] / tj["events"] * n_per
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_event": 8 * len(arrays)}
    if cfg in ("c3", "c4"):
        # The Dalitz coherent sum is FP64-bound (~84 flop per
        # event against 16 B).  Denominator: the FP64 DFMA-chain peak measured
        # on this GPU in this run (pfb_fp64_peak; MEASURED_PEAKS.json has none).
        fp64_peak = ctx.fp64_peak_tflops()
        flops = FLOPS_PER_EVENT[cfg] * n_per
        achieved_tf = flops / (ms_per_step * 1e-3) / 1e12
        roofline = {"bound": "fp64", "achieved": achieved_tf, "peak": fp64_peak, "unit": "TFLOP/s",
                    "frac": achieved_tf / fp64_peak, "traffic": traffic,
                    "peak_source": "measured in this run (pfb_fp64_peak: DFMA chains, 2 flop each)",
                    "algorithmic_flops_per_event": FLOPS_PER_EVENT[cfg],
                    # FP64 also against the vendor figure (DGX B200:
                    # 296 TFLOP/s FP64 over 8 GPUs = 37 per GPU)
                    "vendor": {"peak": VENDOR_FP64_TFLOPS, "frac": achieved_tf / VENDOR_FP64_TFLOPS},
                    "hbm": {"achieved_GBps": achieved, "peak_GBps": peak, "frac": achieved / peak}}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        rate, cores, sample = cpu_reference_rate(cfg, arrays)
        cpu = {"value": rate, "unit": "events/s", "cores": cores, "kind": "port", "sample": sample}

    line = {
        "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": CONFIGS[cfg]["workload"], "n_events_per_gpu": n_per,
                   "evaluator": plan.evaluator, "l2": "flushed (256 MB read) before every step",
                   "parallelism": (f"events sharded over {world} GPUs, one exchange of the 72-limb exact "
                                   f"accumulator per call ({collective})" if world > 1 else "one GPU, no exchange")},
        "nll_evals_per_s": args.steps / dev_s,
        "nll": nll_value,
        "nll_crosscheck_rel": crosscheck,
        "wall_s": wall,
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
