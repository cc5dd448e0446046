"""Device engine: contexts, HBM event stores, the NLL entry point and the
reference-compatible backend.

The reference's ``nll`` (engine.py:214-243) resolves norms on the host, then
maps ``nll_block_sums`` over block-aligned chunks and combines the block sums
with ``math.fsum``.  Here the whole map + reduce is one fused kernel launch
(libpfb200.so) over a device-resident copy of the columns:

* :class:`DeviceBackend` is a drop-in for the reference ``Backend``: it answers
  ``chunk_ranges`` with one chunk and ``map`` with a one-element list holding
  the exact total, so the *unmodified* reference ``nll`` (and therefore its
  FitManager) runs on the GPU and ``math.fsum([total]) == total``.
* :func:`nll` is this package's own entry point with the reference's
  signature and semantics (EmptyDataSet, default snapshot, norm cache).

Normalisation caching (engine.py:103-164) is mirrored verbatim: per-node
values keyed on parameter generations, with the Dalitz hook from
:mod:`.dalitz` computing its overlap integrals on the GPU.
"""

from __future__ import annotations

import ctypes
import math
import os
import weakref
from collections import defaultdict
from typing import Callable, Mapping

import numpy as np

from . import _lib as L
from .errors import EmptyDataSet, error_module_for
from .pdf import NormalizationValue, normalize_value
from .plan import Plan, layout

DEFAULT_BLOCK = L.PFB_BLOCK


# --- normalisation cache (reference engine.py:103-164) -------------------------------


class NormalizationStore:
    """Per-node normalisation cache keyed on parameter generations."""

    def __init__(self):
        self._entries: dict[object, tuple[tuple, object]] = {}
        self.kernel_evals = 0
        self.norm_computations = 0
        self.recompute_counts: dict[int, int] = defaultdict(int)

    def get(self, key):
        return self._entries.get(key)

    def put(self, key, fingerprint: tuple, payload) -> None:
        self._entries[key] = (fingerprint, payload)

    def clear(self) -> None:
        self._entries.clear()


CACHED_NORM_HOOKS: dict[str, Callable] = {}


def register_cached_norm(kind: str, hook: Callable) -> None:
    CACHED_NORM_HOOKS[kind] = hook


def cached_norm(node, snap, store: NormalizationStore) -> NormalizationValue:
    fp = node.fingerprint()
    cached = store.get(node.id)
    if cached is not None and cached[0] == fp:
        return NormalizationValue(cached[1], fp)
    child_norms = {c.id: cached_norm(c, snap, store).value for c in node.children}
    hook = CACHED_NORM_HOOKS.get(node.kind)
    if hook is not None:
        value = float(hook(node, snap, store))
    else:
        value = normalize_value(node, snap, child_norms)
        if not node.children:
            store.kernel_evals += 1
    store.norm_computations += 1
    store.recompute_counts[node.id] += 1
    store.put(node.id, fp, value)
    return NormalizationValue(value, fp)


def resolve_norms(root, snap, store: NormalizationStore) -> dict[int, float]:
    """Every node's norm in post-order (reference engine.py:158-164).  Same
    cache traffic and counters as calling cached_norm per node -- whose
    recursion into children only ever hits the cache here, since children
    precede their parent -- without that second pass."""
    out: dict[int, float] = {}
    for node in root.walk():
        fp = node.fingerprint()
        cached = store.get(node.id)
        if cached is not None and cached[0] == fp:
            out[node.id] = cached[1]
            continue
        hook = CACHED_NORM_HOOKS.get(node.kind)
        if hook is not None:
            value = float(hook(node, snap, store))
        else:
            value = normalize_value(node, snap, {c.id: out[c.id] for c in node.children})
            if not node.children:
                store.kernel_evals += 1
        store.norm_computations += 1
        store.recompute_counts[node.id] += 1
        store.put(node.id, fp, value)
        out[node.id] = NormalizationValue(value, fp).value  # positivity check as cached_norm
    return out


# --- device contexts ------------------------------------------------------------------


class DeviceContext:
    """One CUDA device: a pfb_ctx plus its caches of stores, plans and grids."""

    def __init__(self, device: int = 0):
        handle = ctypes.c_void_p()
        L.check(L.lib().pfb_ctx_create(int(device), ctypes.byref(handle)), f"pfb_ctx_create(device={device})")
        self.device = int(device)
        self.handle = handle
        self._stores: dict[tuple, tuple] = {}  # key -> (store handle, keepalive arrays)
        self._plans: dict[tuple, Plan] = {}
        self.grids: dict[tuple, object] = {}

    # stores: device copies of host columns, keyed by array identity (the
    # arrays are kept alive by the cache, so ids cannot be recycled)
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

    MAX_STORES = 8

    def adopt(self, arrays, st, begin: int = 0, end: int | None = None) -> None:
        """Register `st` as the HBM copy of rows [begin, end) of `arrays`
        (bounded cache: the oldest store is dropped first)."""
        end = len(arrays[0]) if end is None else end
        while len(self._stores) >= self.MAX_STORES:
            old_key = next(iter(self._stores))
            L.lib().pfb_store_destroy(self._stores.pop(old_key)[0])
        self._stores[tuple(id(a) for a in arrays) + (begin, end)] = (st, tuple(arrays))

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
        2 / 3 alternative TMA layouts, 0 the SIMT reference-tree kernels."""
        L.check(L.lib().pfb_ctx_set_pipeline(self.handle, int(mode)), "pfb_ctx_set_pipeline")

    def launch_count(self) -> int:
        out = ctypes.c_int64()
        L.check(L.lib().pfb_ctx_launch_count(self.handle, ctypes.byref(out)), "pfb_ctx_launch_count")
        return out.value

    def set_stream(self, stream_ptr: int | None) -> None:
        L.check(L.lib().pfb_ctx_set_stream(self.handle, ctypes.c_void_p(stream_ptr or 0)), "pfb_ctx_set_stream")

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
    ctx = _contexts.get(device)
    if ctx is None:
        ctx = DeviceContext(device)
        _contexts[device] = ctx
    return ctx


# --- error translation ------------------------------------------------------------------


def raise_for(err: L.PfbErr, code: int, node, where: str) -> None:
    """Map a native status onto the reference exception the caller expects."""
    if code == L.OK:
        return
    E = error_module_for(node)
    if code == L.E_NONPOSITIVE_DENSITY:
        raise E.NonPositiveDensity(int(err.index), float(err.value))
    if code == L.E_NONFINITE_DENSITY:
        kind = "density"
        raise E.NonFiniteDensity(int(err.index), f"{kind} kernel produced a non-finite value")
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
    raise L.NativeError(code, where)


def _evaluate(ctx: DeviceContext, pdf, arrays, names, snap, norms, begin, end, index_offset=0,
              block_sums=False, lineshape_cache=0):
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
        raise_for(err, code, pdf, "pfb_nll_block_sums")
        return out
    total = ctypes.c_double()
    code = L.lib().pfb_nll(ctx.handle, plan.handle, st, begin, end, index_offset, plan.values_ptr, len(vals),
                           plan.norms_ptr, len(nv), ctypes.byref(total), ctypes.byref(err))
    raise_for(err, code, pdf, "pfb_nll")
    return total.value


# --- the reference-compatible backend ---------------------------------------------------


class DeviceBackend:
    """Duck-typed replacement for the reference ``Backend`` (engine.py:32-97).

    ``devices`` lists CUDA devices to use inside this process; the event range
    is split into block-aligned contiguous ranges, one per device, each device
    produces its exact integer partial, and the partials are summed and
    rounded once -- so any device count gives the single-GPU bits.
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

    # reference protocol ------------------------------------------------------
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

    # direct API --------------------------------------------------------------
    def evaluate(self, pdf, columns: Mapping[str, np.ndarray], snap, norms, start: int, stop: int,
                 index_offset: int = 0) -> float:
        names = tuple(columns.keys())
        arrays = [columns[k] for k in names]
        if len(self.contexts) == 1:
            # NonPositiveDensity carries offset + start + i (reference engine.py:177-186)
            return _evaluate(self.contexts[0], pdf, arrays, names, snap, norms, start, stop,
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
                    out.append(self._try(lambda e=errs[k]: raise_for(e, e.code, pdf, "pfb_nll_batch")))
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
        names = tuple(columns.keys())
        arrays = [columns[k] for k in names]
        return _evaluate(self.contexts[0], pdf, arrays, names, snap, norms, start, stop,
                         index_offset + start, block_sums=True)

    def _evaluate_multi(self, pdf, arrays, names, snap, norms, start, stop, index_offset):
        import torch  # device buffers for the per-device accumulators (plumbing only)

        n = stop - start
        nblocks = -(-n // self.block)
        k = min(len(self.contexts), max(nblocks, 1))
        base, extra = divmod(nblocks, k)
        parts = []
        b0 = 0
        for i in range(k):
            b1 = b0 + base + (1 if i < extra else 0)
            parts.append((start + b0 * self.block, min(start + b1 * self.block, stop)))
            b0 = b1
        accs = []
        for ctx, (b, e) in zip(self.contexts, parts):
            plan = ctx.plan_for(pdf, names)
            st = ctx.store_for(arrays, b, e)
            vals, nv = plan.pack(snap, norms)
            acc = torch.zeros(L.PFB_ACC_WORDS, dtype=torch.int64, device=f"cuda:{ctx.device}")
            L.check(L.lib().pfb_nll_partial_async(ctx.handle, plan.handle, st, 0, e - b, index_offset + b,
                                                  L.dptr(vals), len(vals), L.dptr(nv), len(nv),
                                                  ctypes.c_void_p(acc.data_ptr())), "pfb_nll_partial_async")
            accs.append((ctx, acc, b - start))
        total = np.zeros(L.PFB_ACC_WORDS, dtype=np.int64)
        first_err = None
        for ctx, acc, off in accs:
            torch.cuda.synchronize(ctx.device)
            a = acc.cpu().numpy()
            total += a
            if a[L.PFB_ACC_FAILS] and first_err is None:
                err = L.PfbErr()
                L.check(L.lib().pfb_last_error(ctx.handle, ctypes.byref(err)), "pfb_last_error")
                if err.code in (L.E_NONFINITE_DENSITY, L.E_NEGATIVE_DENSITY):
                    err.index += off  # chunk-local in the reference: one chunk here
                first_err = err
        if first_err is not None:
            raise_for(first_err, first_err.code, pdf, "pfb_nll (multi-device)")
        out = ctypes.c_double()
        code = L.lib().pfb_acc_round(total.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ctypes.byref(out))
        if code == L.E_INVALID_SUM:
            raise ValueError("-inf + inf in exact NLL sum")
        return out.value


_default_backend: DeviceBackend | None = None


def default_backend() -> DeviceBackend:
    global _default_backend
    if _default_backend is None:
        _default_backend = DeviceBackend()
    return _default_backend


def _needed_columns(pdf, ds) -> dict[str, np.ndarray]:
    needed = {name for node in pdf.walk() for name in node.observable_names()}
    available = ds.columns()
    missing = needed - set(available)
    if missing:
        raise KeyError(f"dataset lacks observables {sorted(missing)}")
    return {name: available[name] for name in sorted(needed)}


def nll(pdf, ds, snap=None, backend=None, store: NormalizationStore | None = None) -> float:
    """-sum_i ln(eval(x_i)/norm) on the GPU (reference engine.nll, engine.py:214-243)."""
    from .core import snapshot

    if ds.n_events == 0:
        raise EmptyDataSet("cannot evaluate an NLL over zero events")
    backend = backend or default_backend()
    store = store if store is not None else NormalizationStore()
    if snap is None:
        snap = snapshot(pdf.param_closure())
    norms = resolve_norms(pdf, snap, store)
    columns = _needed_columns(pdf, ds)
    if isinstance(backend, DeviceBackend):
        return backend.evaluate(pdf, columns, snap, norms, 0, ds.n_events)
    ranges = backend.chunk_ranges(ds.n_events)
    chunks = backend.map(None, [(pdf, columns, snap, norms, a, b, backend.block) for a, b in ranges])
    return math.fsum(v for c in chunks for v in np.asarray(c).tolist())


def nll_block_sums(pdf, columns, snap, norms, start, stop, block=DEFAULT_BLOCK, offset=0, backend=None):
    """Per-block sums of -ln(p) (reference engine.nll_block_sums, engine.py:190-202)."""
    backend = backend or default_backend()
    if block != DEFAULT_BLOCK:
        raise ValueError(f"the device reduction block is fixed at {DEFAULT_BLOCK}")
    return backend.block_sums(pdf, columns, snap, norms, start, stop, offset)


def binned_nll(pdf, ds, snap=None, backend=None, store: NormalizationStore | None = None) -> float:
    """Poisson NLL over bins, sum_b [nu_b - n_b ln nu_b] (reference engine.binned_nll,
    engine.py:246-276): densities at the bin centres and the exact sum on the GPU
    (pfb_binned_nll), nu_b = total * p_b * bin volume as the reference computes it."""
    from .core import snapshot

    total = ds.total
    if total <= 0:
        raise error_module_for(pdf).EmptyDataSet("binned dataset has no content")
    store = store if store is not None else NormalizationStore()
    if snap is None:
        snap = snapshot(pdf.param_closure())
    norms = resolve_norms(pdf, snap, store)
    device = backend.devices[0] if isinstance(backend, DeviceBackend) else 0
    ctx = device_context(device)
    centers = ds.device_centers()
    needed = sorted({name for node in pdf.walk() for name in node.observable_names()})
    missing = set(needed) - set(centers)
    if missing:
        raise KeyError(f"binned dataset lacks observables {sorted(missing)}")
    arrays = [centers[name] for name in needed]
    plan = ctx.plan_for(pdf, tuple(needed))
    st = ctx.store_for(arrays)
    vals, nv = plan.pack(snap, norms)
    contents = np.ascontiguousarray(ds.contents, dtype=np.float64)
    out = ctypes.c_double()
    err = L.PfbErr()
    code = L.lib().pfb_binned_nll(ctx.handle, plan.handle, st, L.dptr(contents), contents.size, float(total),
                                  float(ds.bin_volume()), L.dptr(vals), len(vals), L.dptr(nv), len(nv),
                                  ctypes.byref(out), ctypes.byref(err))
    raise_for(err, code, pdf, "pfb_binned_nll")
    return out.value
