"""Device engine: CUDA contexts, HBM event stores and the reference-facing
``Backend``.

The reference's ``nll`` (P/engine.py:214-243) resolves norms through its own
cache, then maps ``nll_block_sums`` over ``backend.chunk_ranges`` and combines
the block sums with ``math.fsum``.  :class:`DeviceBackend` answers that
protocol (``block``, ``chunk_ranges``, ``map``; P/engine.py:229,235-239) with
ONE fused kernel launch (libpfb200.so) over a device-resident copy of the
columns: ``chunk_ranges`` returns one chunk and ``map`` a one-element array
holding the exactly rounded total, so ``math.fsum([total]) == total`` and the
unmodified reference ``nll`` / ``FitManager`` / ``eval-nll`` run on the GPU.

Everything above the backend -- ``Variable``, snapshots, ``PdfNode`` trees,
the normalisation cache and its counters -- is the reference's own code
(``paper_1710_08826_b200._reference``); only the device norm hooks in
:mod:`.norms` plug into its ``register_cached_norm``.
"""

from __future__ import annotations

import ctypes
from typing import Mapping

import numpy as np

from . import _lib as L
from ._reference import engine as ref_engine
from ._reference import errors as ref_errors
from .plan import Plan, layout

DEFAULT_BLOCK = L.PFB_BLOCK


# --- device contexts ------------------------------------------------------------------


class DeviceContext:
    """One CUDA device: a pfb_ctx plus its caches of stores, plans and grids."""

    MAX_STORES = 8

    def __init__(self, device: int = 0):
        handle = ctypes.c_void_p()
        L.check(L.lib().pfb_ctx_create(int(device), ctypes.byref(handle)), f"pfb_ctx_create(device={device})")
        self.device = int(device)
        self.handle = handle
        self._stores: dict[tuple, tuple] = {}  # key -> (store handle, keepalive arrays)
        self._plans: dict[tuple, Plan] = {}
        self.grids: dict[tuple, object] = {}

    # stores: device copies of host columns, keyed by array identity (the
    # cache holds the arrays, so an id cannot be recycled while cached)
    def store_for(self, arrays, begin: int = 0, end: int | None = None):
        n_all = len(arrays[0])
        end = n_all if end is None else end
        key = tuple(id(a) for a in arrays) + (begin, end)
        hit = self._stores.get(key)
        if hit is not None:
            return hit[0]
        n = end - begin
        st = ctypes.c_void_p()
        L.check(L.lib().pfb_store_create(self.handle, len(arrays), n, ctypes.byref(st)), "pfb_store_create")
        for c, a in enumerate(arrays):
            a = np.ascontiguousarray(a, dtype=np.float64)
            if n:
                L.check(L.lib().pfb_store_upload(st, c, L.dptr(a[begin:end]), 0, n), "pfb_store_upload")
        self.adopt(arrays, st, begin, end)
        return st

    def adopt(self, arrays, st, begin: int = 0, end: int | None = None) -> None:
        """Register `st` as the HBM copy of rows [begin, end) of `arrays`
        (bounded cache: the oldest store is dropped first)."""
        end = len(arrays[0]) if end is None else end
        while len(self._stores) >= self.MAX_STORES:
            old_key = next(iter(self._stores))
            L.lib().pfb_store_destroy(self._stores.pop(old_key)[0])
        self._stores[tuple(id(a) for a in arrays) + (begin, end)] = (st, tuple(arrays))

    def has_store(self, arrays, begin: int = 0, end: int | None = None) -> bool:
        end = len(arrays[0]) if end is None else end
        return (tuple(id(a) for a in arrays) + (begin, end)) in self._stores

    def plan_for(self, pdf, column_names) -> Plan:
        key = (id(pdf), tuple(column_names))
        plan = self._plans.get(key)
        if plan is None or plan.tree.nodes[-1] is not pdf:
            plan = Plan(self, layout(pdf, column_names))
            plan._keepalive = pdf
            self._plans[key] = plan
        return plan

    def set_warps_per_block(self, warps: int) -> None:
        L.check(L.lib().pfb_ctx_set_warps_per_block(self.handle, int(warps)), "pfb_ctx_set_warps_per_block")

    def set_pipeline(self, mode: int) -> None:
        """Kernel structure (include/pfb200.h pfb_ctx_set_pipeline): 1 default,
        2 / 3 alternative TMA layouts, 4 as 1 with the C1 warp-task kernel,
        0 the SIMT reference-tree kernels."""
        L.check(L.lib().pfb_ctx_set_pipeline(self.handle, int(mode)), "pfb_ctx_set_pipeline")

    def launch_count(self) -> int:
        out = ctypes.c_int64()
        L.check(L.lib().pfb_ctx_launch_count(self.handle, ctypes.byref(out)), "pfb_ctx_launch_count")
        return out.value

    CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy

    def set_stream(self, stream_ptr: int | None) -> None:
        """Run the engine on `stream_ptr` (e.g. ``torch.cuda.current_stream().cuda_stream``).
        0 -- torch's default stream -- is the legacy default stream, so the
        engine stays ordered with torch's work; None: the context's own stream."""
        ptr = self.CUDA_STREAM_LEGACY if stream_ptr == 0 else stream_ptr
        L.check(L.lib().pfb_ctx_set_stream(self.handle, ctypes.c_void_p(ptr)), "pfb_ctx_set_stream")

    def enable_timing(self, on: bool = True) -> None:
        L.check(L.lib().pfb_ctx_enable_timing(self.handle, 1 if on else 0), "pfb_ctx_enable_timing")

    def last_kernel_ms(self) -> float:
        out = ctypes.c_float()
        L.check(L.lib().pfb_ctx_last_kernel_ms(self.handle, ctypes.byref(out)), "pfb_ctx_last_kernel_ms")
        return float(out.value)

    def fp64_peak_tflops(self) -> float:
        out = ctypes.c_double()
        L.check(L.lib().pfb_fp64_peak(self.handle, ctypes.byref(out)), "pfb_fp64_peak")
        return out.value

    def spin(self, cycles: int, flush_ptr: int = 0, flush_bytes: int = 0) -> None:
        """Timing support: L2-evicting read of a device buffer + an SM-wide spin
        on the context stream (pfb_ctx_spin)."""
        L.check(L.lib().pfb_ctx_spin(self.handle, int(cycles), ctypes.c_void_p(flush_ptr), int(flush_bytes)),
                "pfb_ctx_spin")

    def close(self) -> None:
        for plan in self._plans.values():
            plan.close()
        self._plans.clear()
        for st, _ in self._stores.values():
            L.lib().pfb_store_destroy(st)
        self._stores.clear()
        for g in self.grids.values():
            g.close()
        self.grids.clear()
        if self.handle:
            L.lib().pfb_ctx_destroy(self.handle)
            self.handle = None


_contexts: dict[int, DeviceContext] = {}


def device_context(device: int = 0) -> DeviceContext:
    """The process's context on `device`.  Creating the first one registers
    the device normalisation hooks (:func:`.norms.install`) in the
    reference's registry -- the engine is then active for every norm the
    reference caches; ``norms.uninstall()`` / ``norms.reference_norms()``
    restore the reference's own."""
    ctx = _contexts.get(device)
    if ctx is None:
        from . import norms

        ctx = DeviceContext(device)
        if not _contexts and not norms.installed():
            norms.install(device)
        _contexts[device] = ctx
    return ctx


# --- error translation ------------------------------------------------------------------


def raise_for(err: L.PfbErr, code: int, where: str) -> None:
    """Raise the reference's own exception for a native status (P/errors.py:54-108):
    the reference line search treats any ParafitError as +inf (P/fitting.py:339-342)."""
    if code == L.OK:
        return
    E = ref_errors
    if code == L.E_NONPOSITIVE_DENSITY:
        raise E.NonPositiveDensity(int(err.index), float(err.value))
    if code == L.E_NONFINITE_DENSITY:
        raise E.NonFiniteDensity(int(err.index), "density kernel produced a non-finite value")
    if code == L.E_NEGATIVE_DENSITY:
        raise E.NegativeDensity(int(err.index), float(err.value))
    if code == L.E_FRACTION_OUT_OF_RANGE:
        raise E.FractionOutOfRange("fractions out of range (device check)")
    if code == L.E_EMPTY_DATASET:
        raise E.EmptyDataSet("cannot evaluate an NLL over zero events")
    if code == L.E_INVALID_SUM:
        raise ValueError("-inf + inf in exact NLL sum")
    if code == L.E_NONPOSITIVE_EXPECTATION:
        raise E.NonPositiveExpectation(int(err.index), float(err.value))
    if code == L.E_NONPOSITIVE_NORM:
        raise E.NonPositiveNorm(f"normalization {float(err.value)!r} is not positive and finite")
    raise L.NativeError(code, where)


def evaluate(ctx: DeviceContext, pdf, arrays, names, snap, norms, begin, end, index_offset=0,
             block_sums=False, lineshape_cache=0):
    """One fused NLL launch over rows [begin, end) of `arrays` (device copy cached)."""
    plan = ctx.plan_for(pdf, names)
    if lineshape_cache:
        plan.set_lineshape_cache(lineshape_cache)
    st = ctx.store_for(arrays)
    vals, nv = plan.pack(snap, norms)
    err = L.PfbErr()
    if block_sums:
        nb = -(-(end - begin) // DEFAULT_BLOCK)
        out = np.empty(nb, dtype=np.float64)
        code = L.lib().pfb_nll_block_sums(ctx.handle, plan.handle, st, begin, end, index_offset,
                                          L.dptr(vals), len(vals), L.dptr(nv), len(nv), L.dptr(out),
                                          nb, ctypes.byref(err))
        raise_for(err, code, "pfb_nll_block_sums")
        return out
    total = ctypes.c_double()
    code = L.lib().pfb_nll(ctx.handle, plan.handle, st, begin, end, index_offset, plan.values_ptr, len(vals),
                           plan.norms_ptr, len(nv), ctypes.byref(total), ctypes.byref(err))
    raise_for(err, code, "pfb_nll")
    return total.value


def shard_bounds(n: int, workers: int, block: int = DEFAULT_BLOCK) -> list[int]:
    """[b0=0, b1, ..., bW=n]: the reference shard() integers (P/sharding.py:80-85),
    computed by the native pfb_shard_bounds."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    out = (ctypes.c_int64 * (workers + 1))()
    L.check(L.lib().pfb_shard_bounds(int(n), int(workers), int(block), out), "pfb_shard_bounds")
    return list(out)


def round_acc(acc) -> float:
    """Correctly rounded value of a 72-word exact accumulator (== math.fsum)."""
    a = np.ascontiguousarray(np.asarray(acc, dtype=np.int64))
    out = ctypes.c_double()
    code = L.lib().pfb_acc_round(a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ctypes.byref(out))
    if code == L.E_INVALID_SUM:
        raise ValueError("-inf + inf in exact sum")
    L.check(code, "pfb_acc_round")
    return out.value


# --- the reference-compatible backend ---------------------------------------------------


class DeviceBackend:
    """Duck-typed replacement for the reference ``Backend`` (P/engine.py:32-97).

    ``devices`` lists the CUDA devices used inside this process.  With several,
    the event range is split at the reference ``shard()`` bounds
    (P/sharding.py:80-85), each device produces its exact integer partial,
    and the partials are summed and rounded once: any device count gives the
    single-GPU bits.  (One process per GPU is :class:`.sharding.ShardedNll`.)
    """

    mode = "device"

    def __init__(self, devices=(0,), block: int = DEFAULT_BLOCK, lineshape_cache: int = 0,
                 warps_per_block: int = 0):
        if block != DEFAULT_BLOCK:
            raise ValueError(f"the device reduction block is fixed at {DEFAULT_BLOCK}")
        self.block = DEFAULT_BLOCK
        self.devices = tuple(int(d) for d in devices)
        if not self.devices:
            raise ValueError("need at least one device")
        self.workers = len(self.devices)
        self.lineshape_cache = int(lineshape_cache)
        self.contexts = [device_context(d) for d in self.devices]
        if warps_per_block:
            for c in self.contexts:
                c.set_warps_per_block(warps_per_block)

    def __repr__(self) -> str:
        return f"DeviceBackend(devices={list(self.devices)})"

    def close(self) -> None:
        pass

    # reference protocol (P/engine.py:235-239) ---------------------------------
    def chunk_ranges(self, n_events: int) -> list[tuple[int, int]]:
        return [(0, n_events)] if n_events > 0 else []

    def map(self, fn, args_list: list[tuple]) -> list:
        out = []
        for args in args_list:
            pdf, columns, snap, norms, start, stop, block = args[:7]
            offset = args[7] if len(args) > 7 else 0
            if block != self.block:
                raise ValueError(f"device backend reduces in blocks of {self.block}, got {block}")
            out.append(np.array([self.evaluate(pdf, columns, snap, norms, start, stop, offset)]))
        return out

    # direct API ---------------------------------------------------------------
    def evaluate(self, pdf, columns: Mapping[str, np.ndarray], snap, norms, start: int, stop: int,
                 index_offset: int = 0) -> float:
        names = tuple(columns.keys())
        arrays = [columns[k] for k in names]
        if len(self.contexts) == 1:
            # NonPositiveDensity carries offset + start + i (P/engine.py:177-186)
            return evaluate(self.contexts[0], pdf, arrays, names, snap, norms, start, stop,
                            index_offset + start, lineshape_cache=self.lineshape_cache)
        return self._evaluate_multi(pdf, arrays, names, snap, norms, start, stop, index_offset)

    MAX_BATCH = 16

    def evaluate_batch(self, pdf, columns: Mapping[str, np.ndarray], snaps, norms_list, start: int, stop: int,
                       index_offset: int = 0) -> list:
        """NLL at several parameter points.  Returns one
        entry per point: the float, or the exception that point's own
        evaluation would raise.  HBM-bound plans read the events once per
        group of up to 16 points; each value is bitwise its single-point NLL."""
        names = tuple(columns.keys())
        arrays = [columns[k] for k in names]
        if len(self.contexts) > 1:
            return [self._try(lambda s=s, n=n: self.evaluate(pdf, columns, s, n, start, stop, index_offset))
                    for s, n in zip(snaps, norms_list)]
        ctx = self.contexts[0]
        plan = ctx.plan_for(pdf, names)
        st = ctx.store_for(arrays)
        out: list = []
        for g0 in range(0, len(snaps), self.MAX_BATCH):
            sn, nl = snaps[g0:g0 + self.MAX_BATCH], norms_list[g0:g0 + self.MAX_BATCH]
            vals, nv = plan.pack_batch(sn, nl)
            m = len(sn)
            res = np.empty(m, dtype=np.float64)
            errs = (L.PfbErr * m)()
            code = L.lib().pfb_nll_batch(ctx.handle, plan.handle, st, start, stop, index_offset + start,
                                         L.dptr(vals), m, vals.shape[1], L.dptr(nv), nv.shape[1], L.dptr(res), errs)
            if code >= L.E_INVALID_ARGUMENT:
                raise L.NativeError(code, "pfb_nll_batch")
            for k in range(m):
                if errs[k].code:
                    out.append(self._try(lambda e=errs[k]: raise_for(e, e.code, "pfb_nll_batch")))
                else:
                    out.append(float(res[k]))
        return out

    @staticmethod
    def _try(fn):
        try:
            return fn()
        except Exception as exc:  # returned, raised by the caller in call order
            return exc

    def block_sums(self, pdf, columns, snap, norms, start: int, stop: int, index_offset: int = 0):
        """Per-4096-event block sums (P/engine.py:190-202, P/reduction.py:59-75)."""
        names = tuple(columns.keys())
        arrays = [columns[k] for k in names]
        return evaluate(self.contexts[0], pdf, arrays, names, snap, norms, start, stop,
                        index_offset + start, block_sums=True)

    def _evaluate_multi(self, pdf, arrays, names, snap, norms, start, stop, index_offset):
        import torch  # device buffers for the per-device accumulators (plumbing only)

        bounds = shard_bounds(stop - start, len(self.contexts), self.block)
        launched = []
        for i, ctx in enumerate(self.contexts):
            b, e = start + bounds[i], start + bounds[i + 1]
            plan = ctx.plan_for(pdf, names)
            st = ctx.store_for(arrays, b, e)
            vals, nv = plan.pack(snap, norms)
            acc = torch.zeros(L.PFB_ACC_WORDS, dtype=torch.int64, device=f"cuda:{ctx.device}")
            L.check(L.lib().pfb_nll_partial_async(ctx.handle, plan.handle, st, 0, e - b, index_offset + b,
                                                  L.dptr(vals), len(vals), L.dptr(nv), len(nv),
                                                  ctypes.c_void_p(acc.data_ptr())), "pfb_nll_partial_async")
            launched.append((ctx, acc, b - start))
        total = np.zeros(L.PFB_ACC_WORDS, dtype=np.int64)
        first_err = None
        for ctx, acc, off in launched:  # shards in order: the first failing shard's error wins
            torch.cuda.synchronize(ctx.device)
            a = acc.cpu().numpy()
            total += a
            frac = ctypes.c_int32()
            L.check(L.lib().pfb_ctx_last_fraction_failure(ctx.handle, ctypes.byref(frac)),
                    "pfb_ctx_last_fraction_failure")
            if (a[L.PFB_ACC_FAILS] or frac.value) and first_err is None:
                err = L.PfbErr()
                L.check(L.lib().pfb_last_error(ctx.handle, ctypes.byref(err)), "pfb_last_error")
                if err.code in (L.E_NONFINITE_DENSITY, L.E_NEGATIVE_DENSITY):
                    err.index += off  # chunk-local in the reference: one chunk here
                first_err = err
        if first_err is not None:
            raise_for(first_err, first_err.code, "pfb_nll (multi-device)")
        return round_acc(total)


_default_backend: DeviceBackend | None = None


def default_backend() -> DeviceBackend:
    global _default_backend
    if _default_backend is None:
        _default_backend = DeviceBackend()
    return _default_backend


def nll(pdf, ds, snap=None, backend=None, store=None) -> float:
    """The reference ``nll`` (P/engine.py:214-243) with the device backend as
    its default: norms through the reference's cache (with the device hooks
    of :mod:`.norms`), evaluation + exact reduction on the GPU."""
    return ref_engine.nll(pdf, ds, snap, backend or default_backend(), store)


def nll_block_sums(pdf, columns, snap, norms, start, stop, block=DEFAULT_BLOCK, offset=0, backend=None):
    """Device ``nll_block_sums`` (P/engine.py:190-202): per-block sums of -ln p."""
    backend = backend or default_backend()
    if block != DEFAULT_BLOCK:
        raise ValueError(f"the device reduction block is fixed at {DEFAULT_BLOCK}")
    return backend.block_sums(pdf, columns, snap, norms, start, stop, offset)
