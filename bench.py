"""Benchmark: NLL evaluations/s and events/s of the B200 engine vs the
reference's CPU path, with roofline fractions.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]
                    [--sub c1,c5,c3,c4,c2p | --sub none] [--collective nccl|fused|peer]

A step is one NLL evaluation over the configuration's full event set.  The
headline workload is BASELINE.json configs[1]: the 2-D ProductPdf
(Gaussian(x) x Exponential(y)), 10M synthetic events per GPU (weak scaling;
at N > 1 each rank holds its shard and the exact 72-limb partials are
combined by one all-reduce per call, NCCL by default).  The headline events
are drawn by :func:`host_events` (numpy, fixed seeds) in BOTH arms, so the
two arms time identical arrays.

Headline keys:

* ``value`` -- events/s with the events resident in HBM: device time of the
  fused NLL kernel (CUDA events on its stream), L2 evicted (256 MB read)
  before every step.
* ``e2e`` -- the same metric through the C ABI with host (pinned) columns:
  every step copies the events host->device (chunked, overlapped with the
  kernels) and reads the result back (pfb_nll_host).
* ``roofline`` -- algorithmic bytes (8 B per observable per event, SURVEY
  8(d)) / kernel time against MEASURED_PEAKS.json hbm_gbs; Dalitz configs:
  algorithmic FP64 flops (84 per event) against the DFMA-chain peak measured
  in the same run.  ``traffic`` = ncu DRAM bytes per launch
  (profiles/traffic_<cfg>.json).
* ``parity`` -- the reference's own ``nll`` (baseline/_ref, ``Backend("pool")``,
  its own norms) on the same arrays; the run fails unless |rel| <= 1e-10.
* ``cpu_baseline`` -- that reference path timed on this host (all cores).
* ``fit`` -- a complete fit from the config's start point through the
  reference ``FitManager`` over ``DeviceBackend`` and through
  ``DeviceFitManager``: calls, wall time, calls/s.
* ``subresults`` -- the same record for C1 (1M), C5 (the C1 model at 10M),
  C3 (Dalitz, 10M), C4 (Dalitz, 100M) and C2p (C2 with a polynomial factor:
  every step moves a polynomial coefficient, so the device Gauss-Legendre
  normalisation kernel runs inside each timed step).

``--impl reference`` times the UNMODIFIED reference (baseline/_ref) through its
public API -- ``nll(pdf, ds, snap, Backend("pool", workers=os.cpu_count()))``
-- on the same headline arrays and prints the same line with
``"impl": "reference"``.  It imports nothing from this repository's engine.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
REF_PATH = os.path.join(ROOT, "baseline", "_ref")

METRIC = "NLL evals/sec & events/sec (1/2/4/8 B200) vs CPU ref; % HBM/FP64 roofline"

CONFIGS = {
    "c1": dict(workload="C1 SumPdf 1-D (gauss+exp), 1M events", n=1_000_000, ncols=1, model="c1"),
    "c2": dict(workload="C2 ProductPdf 2-D (gauss(x) x exp(y)), 10M events", n=10_000_000, ncols=2, model="c2"),
    "c2p": dict(workload="C2p ProductPdf 2-D (gauss(x) x polynomial(y)), 10M events, device GL norm every step",
                n=10_000_000, ncols=2, model="c2p"),
    "c3": dict(workload="C3 Dalitz D0->pi+pi-pi0 (rho+, rho-, rho0, NR), 10M events", n=10_000_000, ncols=2,
               model="c3"),
    "c4": dict(workload="C4 Dalitz D0->pi+pi-pi0, 100M events", n=100_000_000, ncols=2, model="c3"),
    "c5": dict(workload="C5 toy unit: SumPdf 1-D (gauss+exp), 10M events", n=10_000_000, ncols=1, model="c1"),
}
SUBS_DEFAULT = ("c1", "c5", "c3", "c4", "c2p")

# SURVEY 8(d) algorithmic FP64 flops per Dalitz event (4 terms x 20 + s23 2 +
# |T|^2 3 + /norm 1 + -log 2 + accumulate 1, rounded to 84)
FLOPS_PER_EVENT = {"c3": 84}
VENDOR_FP64_TFLOPS = 37.0
D_CHANNEL = (1.86484, 0.13957, 0.13957, 0.13498)
# (pair, m, width, spin, magnitude, phase): rho+, rho-, rho0, NR stand-in
C3_TERMS = [(13, 0.77511, 0.1491, 1, 1.0, 0.0), (23, 0.77511, 0.1491, 1, 0.73, -0.03),
            (12, 0.77526, 0.1478, 1, 0.55, 0.28), (12, 1.0, 20.0, 0, 20.0, -0.5)]
FIT_STARTS = {"c1": (4.8, 0.6, -0.25, 0.35), "c2": (4.9, 1.1, -0.35), "c2p": (4.9, 1.1, 1.0, 0.28, 0.06),
              "c3": (0.8, 0.0, 0.5, 0.3, 19.0, -0.45)}


def log(msg: str) -> None:
    print(msg, file=sys.stderr, flush=True)


def reference():
    """The unmodified reference package (baseline/_ref)."""
    if REF_PATH not in sys.path:
        sys.path.append(REF_PATH)
    import parafit

    return parafit


# --- models (the reference's own builders) and inputs ------------------------------------


def build_model(P, model: str):
    """(observables, pdf, free params in fit order) with the reference's builders."""
    x = P.Variable.observable("x", 0.0, 10.0)
    if model == "c1":
        mu, sg = P.Variable("mu", 5.0, 0.0, 10.0, step=0.01), P.Variable("sigma", 0.5, 0.01, 5.0, step=1e-3)
        al, f = P.Variable("alpha", -0.3, -5.0, 5.0, step=1e-3), P.Variable("f", 0.3, 0.0, 1.0, step=1e-3)
        return [x], P.add_pdf([P.gaussian(x, mu, sg), P.exponential(x, al)], [f]), [mu, sg, al, f]
    y = P.Variable.observable("y", 0.0, 10.0)
    if model == "c2":
        mu, sg = P.Variable("mu", 5.0, 0.0, 10.0, step=0.01), P.Variable("sigma", 1.0, 0.01, 5.0, step=1e-3)
        al = P.Variable("alpha", -0.4, -5.0, 5.0, step=1e-3)
        return [x, y], P.prod_pdf([P.gaussian(x, mu, sg), P.exponential(y, al)]), [mu, sg, al]
    if model == "c2p":
        mu, sg = P.Variable("mu", 5.0, 0.0, 10.0, step=0.01), P.Variable("sigma", 1.0, 0.01, 5.0, step=1e-3)
        c = [P.Variable("c0", 1.0, 0.05, 10.0, step=1e-3), P.Variable("c1", 0.3, -0.09, 2.0, step=1e-3),
             P.Variable("c2", 0.05, 0.0, 1.0, step=1e-4)]
        return [x, y], P.prod_pdf([P.gaussian(x, mu, sg), P.polynomial(y, c)]), [mu, sg] + c
    ch = P.DecayChannel(*D_CHANNEL)
    terms, free = [], []
    for k, (pair, m, w, spin, mag, ph) in enumerate(C3_TERMS):
        t = P.ResonanceTerm(pair=pair, mass=P.Variable(f"t{k}_m", m, fixed=True),
                            width=P.Variable(f"t{k}_w", w, fixed=True), spin=spin,
                            magnitude=P.Variable(f"t{k}_mag", mag, 0.0, 100.0, step=0.01, fixed=(k == 0)),
                            phase=P.Variable(f"t{k}_ph", ph, -2 * math.pi, 2 * math.pi, step=0.01, fixed=(k == 0)))
        terms.append(t)
        if k:
            free += [t.magnitude, t.phase]
    s12 = P.Variable.observable("s12", *ch.s12_range)
    s13 = P.Variable.observable("s13", *ch.s13_range)
    return [s12, s13], P.dalitz_pdf(terms, ch, s12_obs=s12, s13_obs=s13, grid=(400, 400)), free


def _trunc_normal(rng, n, mu, sigma, lo, hi):
    out = np.empty(n)
    got = 0
    while got < n:
        v = rng.normal(mu, sigma, int((n - got) * 1.1) + 1024)
        v = v[(v >= lo) & (v <= hi)][: n - got]
        out[got:got + len(v)] = v
        got += len(v)
    return out


def _trunc_exp(rng, n, alpha, lo, hi):
    a, b = math.exp(alpha * lo), math.exp(alpha * hi)
    return np.clip(np.log(a + rng.random(n) * (b - a)) / alpha, lo, hi)


def host_events(model: str, n: int, seed: int):
    """Synthetic events of the model's shape, drawn with numpy from fixed seeds
    (identical arrays in both bench arms)."""
    rng = np.random.default_rng(seed)
    if model == "c1":
        ng = int(rng.binomial(n, 0.3))
        x = np.concatenate([_trunc_normal(rng, ng, 5.0, 0.5, 0.0, 10.0), _trunc_exp(rng, n - ng, -0.3, 0.0, 10.0)])
        rng.shuffle(x)
        return [x]
    x = _trunc_normal(rng, n, 5.0, 1.0, 0.0, 10.0)
    if model == "c2":
        return [x, _trunc_exp(rng, n, -0.4, 0.0, 10.0)]
    if model == "c2p":  # y ~ 1 + 0.3 y + 0.05 y^2 by inverse-CDF on a fine table
        g = np.linspace(0.0, 10.0, 20001)
        cdf = g + 0.15 * g * g + 0.05 * g ** 3 / 3.0
        return [x, np.interp(rng.random(n) * cdf[-1], cdf, g)]
    raise ValueError(model)


def events(cfg: str, n: int, seed: int):
    """Inputs of a config: host numpy draws, or (Dalitz) the device sampler."""
    model = CONFIGS[cfg]["model"]
    if model != "c3":
        return host_events(model, n, seed)
    from paper_1710_08826_b200 import mcgen

    terms = [(p, s, m, w, mag, ph) for (p, m, w, s, mag, ph) in C3_TERMS]
    return list(mcgen.device_dalitz(n, terms, D_CHANNEL, seed))


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


# --- the reference arm ----------------------------------------------------------------------


def reference_rate(P, pdf, ds, snap, budget_s: float, max_calls: int):
    """The reference's own nll (P/engine.py:214-243) with Backend("pool",
    os.cpu_count()), its own norms: (value, events/s, calls, seconds)."""
    os.environ.pop("PARAFIT_WORKERS", None)  # it overrides the pool size (P/engine.py:43-47)
    threads = os.cpu_count() or 1
    backend = P.Backend("pool", workers=threads)
    store = P.NormalizationStore()
    value = P.nll(pdf, ds, snap, backend, store)  # warm-up: norm cache, pool threads
    calls, t0 = 0, time.perf_counter()
    while calls < max_calls:
        P.nll(pdf, ds, snap, backend, store)
        calls += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    backend.close()
    return value, ds.n_events * calls / dt, calls, dt, threads


def run_reference(args, cfg: str, rank: int):
    if rank != 0:
        return
    P = reference()
    obs, pdf, _ = build_model(P, CONFIGS[cfg]["model"])
    n = args.n or CONFIGS[cfg]["n"]
    cols = host_events(CONFIGS[cfg]["model"], n, seed=1000)
    ds = P.UnbinnedDataSet(obs)
    ds.extend(cols)
    snap = P.snapshot(pdf.param_closure())
    os.environ.pop("PARAFIT_WORKERS", None)
    threads = os.cpu_count() or 1
    backend = P.Backend("pool", workers=threads)
    store = P.NormalizationStore()
    for _ in range(max(0, args.warmup)):
        P.nll(pdf, ds, snap, backend, store)
    steps = max(1, args.steps)
    t0 = time.perf_counter()
    for _ in range(steps):
        value_nll = P.nll(pdf, ds, snap, backend, store)
    dt = time.perf_counter() - t0
    backend.close()
    value = n * steps / dt
    sample = f"{steps} reference nll calls x {n} events (the full headline event set), Backend('pool', {threads})"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(cfg, n),
        "nll_evals_per_s": steps / dt, "nll": value_nll,
        "cpu_baseline": {"value": value, "unit": "events/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_of(cfg: str, n: int) -> dict:
    return {"workload": CONFIGS[cfg]["workload"], "n_events_per_gpu": n,
            "inputs": ("numpy default_rng(1000 + rank) draws of the model's shape (bench.host_events)"
                       if CONFIGS[cfg]["model"] != "c3" else "device Philox accept-reject sampler (seed 1000 + rank)"),
            "l2": "evicted (256 MB read) before every timed step"}


# --- the B200 arm ---------------------------------------------------------------------------


class Measure:
    """One config on this rank: device-timed NLL, e2e through the C ABI, roofline,
    reference parity + CPU timing, fits."""

    def __init__(self, args, cfg: str, rank: int, world: int, dev: int, collective: str):
        import torch

        import paper_1710_08826_b200 as pf
        from paper_1710_08826_b200 import _lib as L

        self.args, self.cfg, self.rank, self.world, self.dev = args, cfg, rank, world, dev
        self.pf, self.L, self.torch = pf, L, torch
        self.P = pf.parafit
        self.model = CONFIGS[cfg]["model"]
        n_total = args.n or CONFIGS[cfg]["n"]
        self.n = n_total
        t0 = time.perf_counter()
        cols = events(cfg, self.n, seed=1000 + rank)
        self.gen_s = time.perf_counter() - t0
        self.obs, self.pdf, self.free = build_model(self.P, self.model)
        self.ds = pf.DeviceDataSet.from_columns(self.obs, cols, device=dev)
        self.ctx = pf.device_context(dev)
        self.ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        self.ctx.enable_timing(True)
        self.names = tuple(sorted(o.name for o in self.obs))
        self.arrays = [self.ds.column(nm) for nm in self.names]
        self.plan = self.ctx.plan_for(self.pdf, self.names)
        self.store = self.ctx.store_for(self.arrays)
        self.nstore = self.P.NormalizationStore()
        self.collective = collective
        self.out = ctypes.c_double()
        self.err = L.PfbErr()
        self.acc = torch.zeros(L.PFB_ACC_WORDS, dtype=torch.int64, device=dev)
        self.flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
        self.peers = None
        if world > 1 and collective in ("peer", "fused"):
            from paper_1710_08826_b200.sharding import PeerGroup

            self.peers = PeerGroup(self.ctx, rank, world, timeout_s=5.0)
        self.ev_a = torch.cuda.Event(enable_timing=True)
        self.ev_b = torch.cuda.Event(enable_timing=True)
        self.c_move = 0
        self.c2p_fcn = None

    def pack(self):
        snap = self.P.snapshot(self.pdf.param_closure())
        norms = self.P.resolve_norms(self.pdf, snap, self.nstore)
        return self.plan.pack(snap, norms)

    def step(self):
        """One NLL over this rank's events; returns (device ms, value)."""
        L, pf = self.L, self.pf
        if self.model == "c2p":
            # a finite-difference-like move of a polynomial coefficient through
            # the minimiser's objective in C: the device GL normalisation
            # kernel and the NLL kernel both run inside the timed step
            self.c_move += 1
            if self.c2p_fcn is None:
                self.c2p_fcn = self.pf.DeviceFitManager(self.pdf, self.ds).fcn()
                self.c2p_x = np.array([v.value for v in self.free])
            x = self.c2p_x.copy()
            x[3] += 1e-6 * (self.c_move % 2)
            self.ev_a.record()
            value = self.c2p_fcn(x)
            self.ev_b.record()
            self.ev_b.synchronize()
            return self.ev_a.elapsed_time(self.ev_b), value
        vals, nv = self.vals, self.nv
        if self.world == 1:
            code = L.lib().pfb_nll(self.ctx.handle, self.plan.handle, self.store, 0, self.n, 0, L.dptr(vals),
                                   len(vals), L.dptr(nv), len(nv), ctypes.byref(self.out), ctypes.byref(self.err))
            L.check(code, "pfb_nll")
            return self.ctx.last_kernel_ms(), self.out.value
        if self.collective == "fused":
            slow = ctypes.c_int32()
            code = L.lib().pfb_nll_peer(self.ctx.handle, self.plan.handle, self.store, 0, self.n, 0, L.dptr(vals),
                                        len(vals), L.dptr(nv), len(nv), self.peers.timeout_s, ctypes.byref(self.out),
                                        ctypes.byref(slow))
            L.check(code, "pfb_nll_peer")
            if slow.value:
                raise SystemExit("fused step took the slow path (deferred blocks or an error on a rank)")
            return self.ctx.last_kernel_ms(), self.out.value
        self.ev_a.record()
        L.check(L.lib().pfb_nll_partial_async(self.ctx.handle, self.plan.handle, self.store, 0, self.n, 0,
                                              L.dptr(vals), len(vals), L.dptr(nv), len(nv),
                                              ctypes.c_void_p(self.acc.data_ptr())), "pfb_nll_partial_async")
        if self.collective == "peer":
            self.peers.allreduce(self.acc)
        else:
            self.torch.distributed.all_reduce(self.acc)
        self.ev_b.record()
        fails = ctypes.c_int64()
        L.check(L.lib().pfb_finalize(self.ctx.handle, ctypes.c_void_p(self.acc.data_ptr()), ctypes.byref(self.out),
                                     ctypes.byref(fails)), "pfb_finalize")
        return self.ev_a.elapsed_time(self.ev_b), self.out.value

    def device_timed(self, steps: int, warmup: int):
        """K steps on the device: before each, L2 evicted (256 MB read) and the
        SMs kept busy ~0.5 ms while the host enqueues the launch, so CUDA
        events on the launch stream time the kernel, not launch latency.
        (Back-to-back launches between one event pair measured 1-5% slower
        per step for the inputs larger than L2 -- C2 36.0 vs 34.2 us,
        C3 54.3 vs 52.3 us -- so every config uses the isolated launch.)"""
        torch = self.torch
        self.vals, self.nv = [a.copy() for a in self.pack()]
        for _ in range(max(3, warmup)):
            self.step()
        torch.cuda.synchronize()
        if self.world > 1:
            torch.distributed.barrier()
        launches0 = self.ctx.launch_count()
        kernel_ms = []
        with ClockSampler(self.dev) as clocks:
            t0 = time.perf_counter()
            for _ in range(steps):
                if self.world > 1:
                    torch.distributed.barrier()
                self.ctx.spin(1_000_000, self.flush.data_ptr(), self.flush.numel() * 4)
                ms, value = self.step()
                kernel_ms.append(ms)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
        launches = self.ctx.launch_count() - launches0
        dev_s = float(np.sum(kernel_ms)) / 1e3
        if self.world > 1:
            t = torch.tensor([dev_s], dtype=torch.float64, device=self.dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dev_s = float(t.item())
        return {"dev_s": dev_s, "steps": steps, "ms_per_step": 1e3 * dev_s / steps, "wall_s": wall,
                "launches": launches, "nll": value, "clocks": clocks.summary(),
                "kernel_ms_median": float(np.median(kernel_ms))}

    def e2e(self, steps: int):
        """The metric through the C ABI with pinned host columns: H2D of all
        events + the result read-back inside every timed step."""
        torch, L = self.torch, self.L
        pinned = [torch.empty(self.n, dtype=torch.float64, pin_memory=True) for _ in self.arrays]
        for p, a in zip(pinned, self.arrays):
            p.numpy()[:] = a
        hcols = (L._DBL_P * len(pinned))(*[ctypes.cast(p.data_ptr(), L._DBL_P) for p in pinned])
        vals, nv = self.vals, self.nv

        def call():
            L.check(L.lib().pfb_nll_host(self.ctx.handle, self.plan.handle, hcols, len(pinned), self.n, L.dptr(vals),
                                         len(vals), L.dptr(nv), len(nv), ctypes.byref(self.out),
                                         ctypes.byref(self.err)), "pfb_nll_host")
            return self.out.value

        first = call()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            call()
        dt = time.perf_counter() - t0
        if self.world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device=self.dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dt = float(t.item())
        del pinned
        return {"value": self.n * self.world * steps / dt, "unit": "events/s",
                "h2d_bytes_per_step": 8 * len(self.arrays) * self.n, "d2h_bytes_per_step": 8 * 8,
                "steps": steps, "nll": first}

    def roofline(self, ms_per_step: float) -> dict:
        peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
        if os.path.exists(peaks_path):
            peak, peak_src = float(json.load(open(peaks_path))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        algo_bytes = 8 * len(self.arrays) * self.n
        achieved = algo_bytes / (ms_per_step * 1e-3) / 1e9
        traffic = None
        tcfg = {"c4": "c3", "c5": "c1", "c2p": "c2"}.get(self.cfg, self.cfg)
        tpath = os.path.join(ROOT, "profiles", f"traffic_{tcfg}.json")
        if os.path.exists(tpath):
            tj = json.load(open(tpath))
            traffic = tj["bytes_per_launch"] / tj["events"] * self.n
        hbm = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
               "traffic": traffic, "peak_source": peak_src, "algorithmic_bytes_per_event": 8 * len(self.arrays)}
        if self.model != "c3":
            return hbm
        fp64_peak = self.ctx.fp64_peak_tflops()
        achieved_tf = FLOPS_PER_EVENT["c3"] * self.n / (ms_per_step * 1e-3) / 1e12
        return {"bound": "fp64", "achieved": achieved_tf, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved_tf / fp64_peak, "traffic": traffic,
                "peak_source": "measured in this run (pfb_fp64_peak: DFMA chains, 2 flop each)",
                "algorithmic_flops_per_event": FLOPS_PER_EVENT["c3"],
                "vendor": {"peak": VENDOR_FP64_TFLOPS, "frac": achieved_tf / VENDOR_FP64_TFLOPS},
                "hbm": {"achieved_GBps": achieved, "peak_GBps": peak, "frac": achieved / peak}}

    def parity_and_cpu(self, device_nll: float, budget_s: float) -> tuple[dict, dict]:
        """The reference's own nll on the same arrays (its own norms, pool
        backend): parity (<= 1e-10) and the CPU rate on this host."""
        pf, P = self.pf, self.P
        snap = P.snapshot(self.pdf.param_closure())
        with pf.reference_norms():
            value, rate, calls, dt, threads = reference_rate(P, self.pdf, self.ds, snap, budget_s, max_calls=50)
        rel = abs(device_nll - value) / abs(value)
        parity = {"reference_nll": value, "device_nll": device_nll, "rel": rel, "tol": 1e-10,
                  "reference": "baseline/_ref parafit nll, Backend('pool'), reference norms, same arrays"}
        if not rel <= 1e-10:
            raise SystemExit(f"{self.cfg}: device NLL {device_nll!r} vs reference {value!r} (rel {rel:.3e})")
        cpu = {"value": rate, "unit": "events/s", "cores": threads, "kind": "reference",
               "sample": f"{calls} reference nll calls x {self.n} events (the full event set), "
                         f"Backend('pool', {threads}), {dt:.1f} s"}
        return parity, cpu

    def fits(self) -> dict:
        """Complete fits from the config's start: the reference FitManager over
        DeviceBackend, and DeviceFitManager (batched stencils).  Each manager
        fits twice from the same start on a fresh instance: `calls_per_s` is
        the second fit (steady state), `first_wall_s` the first (one-time set-up
        included, e.g. the fast objective's own Dalitz grid)."""
        import gc

        pf, P = self.pf, self.P
        start = FIT_STARTS.get(self.model)
        if start is None:
            return None
        out = {}
        for tag, make in (("reference_fitmanager", lambda: P.FitManager(self.pdf, self.ds, backend=pf.DeviceBackend())),
                          ("device_fitmanager", lambda: pf.DeviceFitManager(self.pdf, self.ds))):
            walls = []
            for _ in range(2):
                for v, val in zip(self.free, start):
                    P.set_value(v, float(val))
                gc.collect()
                fm = make()
                t0 = time.perf_counter()
                r = fm.fit()
                walls.append(time.perf_counter() - t0)
            dt = walls[-1]
            rec = {"status": r.status, "n_calls": r.n_calls, "wall_s": dt, "calls_per_s": r.n_calls / dt,
                   "first_wall_s": walls[0], "nll_min": r.nll_min, "values": [float(v) for v in r.values]}
            if tag == "device_fitmanager":
                rec["device_passes"] = r.n_calls - fm.objective.batched_points + fm.objective.batches
            out[tag] = rec
        for v, val in zip(self.free, start):
            P.set_value(v, float(val))
        return out

    def record(self, steps: int, warmup: int, cpu_budget_s: float, with_fit: bool = True) -> dict:
        t = self.device_timed(steps, warmup)
        e2e = self.e2e(max(3, min(steps, 10)))
        rec = {"workload": CONFIGS[self.cfg]["workload"], "n_events": self.n,
               "value": self.n * self.world * steps / t["dev_s"], "unit": "events/s",
               "ms_per_step": t["ms_per_step"], "nll_evals_per_s": steps / t["dev_s"],
               "evaluator": self.plan.evaluator, "gpu_launches": t["launches"], "nll": t["nll"],
               "roofline": self.roofline(t["ms_per_step"]), "e2e": e2e, "clocks": t["clocks"],
               "wall_s": t["wall_s"], "generate_s": self.gen_s}
        if self.model == "c2p":
            rec["step"] = ("the C objective (DeviceFitManager.fcn) with c1 moved: device GL quadrature kernel "
                           "(the polynomial's norm) + fused NLL kernel; CUDA events around the call")
            rec["e2e_step"] = "the C ABI with host columns at the Variables' point (norms fixed, as every config's e2e)"
        if self.rank == 0 and self.world == 1:
            dev_nll = t["nll"]
            if self.model == "c2p":  # the timed steps alternate c1; parity at the Variables' own point
                dev_nll = float(self.c2p_fcn(self.c2p_x.copy()))
            rec["parity"], rec["cpu_baseline"] = self.parity_and_cpu(dev_nll, cpu_budget_s)
            if with_fit:
                rec["fit"] = self.fits()
        return rec

    def close(self):
        self.ctx.grids.clear()
        self.ds = None


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` without a launcher: run N ranks via torch.distributed.run."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator lines visible on stderr
    # torch.distributed.run resolves abbreviated options over the whole command
    # line: pass --n as --events (its unambiguous spelling)
    fwd = ["--events" if a == "--n" else ("--events=" + a[4:] if a.startswith("--n=") else a) for a in sys.argv[1:]]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + fwd
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", "--events", dest="n", type=int, default=0, help="override events per GPU")
    ap.add_argument("--sub", default=",".join(SUBS_DEFAULT),
                    help="sub-result configs at N=1 ('none' to skip)")
    ap.add_argument("--collective", default="nccl", choices=["nccl", "fused", "peer"],
                    help="N > 1: NCCL all-reduce of the 72-word accumulator (default), the exchange fused into "
                         "the NLL kernel over NVLink peer memory (pfb_nll_peer), or a separate peer kernel")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=6.0, help="seconds of reference CPU timing per config")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = args.config

    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return

    import torch

    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", init_method="env://")
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    # one explicit stream for torch and the engine (the legacy default stream
    # handle 0 would leave the engine on its own stream, unordered with torch's
    # events and copies)
    torch.cuda.set_stream(torch.cuda.Stream(device=dev))

    head = Measure(args, cfg, rank, world, dev, args.collective if world > 1 else "none")
    rec = head.record(args.steps, args.warmup, args.cpu_budget, with_fit=(world == 1))
    if world > 1:
        torch.distributed.barrier()
    subs = {}
    if world == 1 and args.sub != "none":
        head.close()
        for sc in [s for s in args.sub.split(",") if s and s != cfg]:
            t0 = time.perf_counter()
            m = Measure(args, sc, rank, world, dev, "none")
            steps = args.steps if sc != "c4" else max(5, args.steps // 4)
            subs[sc] = m.record(steps, args.warmup, args.cpu_budget if sc != "c4" else 1.0)
            m.close()
            del m
            log(f"sub-result {sc}: {time.perf_counter() - t0:.1f} s")
    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return
    launches = rec["gpu_launches"]
    line = {
        "metric": METRIC, "value": rec["value"], "unit": "events/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": rec["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        # config: the workload only, key for key the reference arm's (same arrays)
        "config": config_of(cfg, head.n), "evaluator": rec["evaluator"],
        "parallelism": (f"events sharded over {world} GPUs (reference shard() bounds), one exchange of "
                        f"the 72-limb exact accumulator per call ({args.collective})"
                        if world > 1 else "one GPU, no exchange"),
        "nll_evals_per_s": rec["nll_evals_per_s"], "nll": rec["nll"],
        "e2e": rec["e2e"], "gpu_launches": launches, "roofline": rec["roofline"],
        "cpu_baseline": rec.get("cpu_baseline"), "parity": rec.get("parity"), "fit": rec.get("fit"),
        "clocks": rec["clocks"], "wall_s": rec["wall_s"], "subresults": subs,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
