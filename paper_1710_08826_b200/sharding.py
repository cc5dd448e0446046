"""Event sharding across GPUs and the exact cross-shard reduction.

The shard plan, the ``Shard``/``PartialSum`` records and ``reduce_partials``
are the reference's own (P/sharding.py:43-131); this module supplies the
device side of them:

* :func:`partial_nll` -- one shard's partial on the GPU, returned as the
  reference ``PartialSum`` whose ``components`` are an exact non-overlapping
  expansion of the shard's 72-word integer accumulator
  (:func:`components_from_acc`), so the reference's ``reduce_partials``
  (``math.fsum`` of all components, P/sharding.py:117-131) merges device
  partials -- and device with host partials -- bit for bit;
* :func:`sharded_nll` -- the driver-side convenience (P/sharding.py:134-146)
  with device partials;
* :class:`ShardedNll` -- one process per GPU (torch.distributed): each rank
  keeps its ``shard()`` rows resident in HBM; one NLL call is one fused kernel
  that writes the shard's accumulator, ONE all-reduce of 72 int64 (NCCL over
  NVLink, or the NVLink peer exchange fused into the kernel), one rounding.
  Integer limbs add associatively, so every rank returns the single-GPU bits.
"""

from __future__ import annotations

import ctypes
import math
from typing import Sequence

import numpy as np

from . import _lib as L
from ._reference import engine as ref_engine
from ._reference import sharding as ref_sharding
from .engine import round_acc, shard_bounds  # noqa: F401  (re-exported)

DEFAULT_BLOCK = L.PFB_BLOCK
Shard = ref_sharding.Shard
PartialSum = ref_sharding.PartialSum
shard = ref_sharding.shard
reduce_partials = ref_sharding.reduce_partials


def components_from_acc(acc) -> tuple[float, ...]:
    """An exact expansion of the accumulator's value: non-overlapping doubles
    in increasing magnitude whose real sum is exactly the accumulated sum (the
    contract of the reference ``ExactAccumulator.partials``,
    P/reduction.py:78-118), so ``math.fsum(components)`` is its correctly
    rounded value.  Limb i of the first 68 carries weight 2^(32 i - 1074);
    words 68..70 count +inf / -inf / NaN terms."""
    a = [int(v) for v in np.asarray(acc, dtype=np.int64).tolist()]
    if a[L.PFB_NLIMBS + 2] > 0:
        return (math.nan,)
    pinf, ninf = a[L.PFB_NLIMBS] > 0, a[L.PFB_NLIMBS + 1] > 0
    if pinf or ninf:
        return tuple(([math.inf] if pinf else []) + ([-math.inf] if ninf else []))
    value = 0
    for i in range(L.PFB_NLIMBS - 1, -1, -1):
        value = (value << 32) + a[i]
    sign = -1.0 if value < 0 else 1.0
    mag = -value if value < 0 else value
    out = []
    j = 0
    while mag:
        chunk = mag & ((1 << 53) - 1)
        if chunk:
            out.append(sign * math.ldexp(float(chunk), 53 * j - 1074))
        mag >>= 53
        j += 1
    return tuple(out)


def acc_of_values(values) -> np.ndarray:
    """Host digit split of doubles into an accumulator (same code as the device)."""
    v = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    acc = np.zeros(L.PFB_ACC_WORDS, dtype=np.int64)
    L.check(L.lib().pfb_acc_add_host(acc.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), L.dptr(v), len(v)),
            "pfb_acc_add_host")
    return acc


def partial_accumulator(sh, pdf, snap, norms=None, block: int = DEFAULT_BLOCK, ctx=None) -> np.ndarray:
    """The shard's exact 72-word accumulator of -ln p, on the GPU; errors carry
    global indices (offset = shard begin, P/sharding.py:110-113)."""
    import torch

    from . import engine

    if norms is None:
        norms = ref_engine.resolve_norms(pdf, snap, ref_engine.NormalizationStore())
    if block != DEFAULT_BLOCK:
        raise ValueError(f"the device reduction block is fixed at {DEFAULT_BLOCK}")
    if sh.size == 0:
        return np.zeros(L.PFB_ACC_WORDS, dtype=np.int64)
    ctx = ctx or engine.device_context(0)
    needed = {nm for node in pdf.walk() for nm in node.observable_names()}
    names = tuple(nm for nm in sorted(sh.columns) if nm in needed)
    arrays = [sh.columns[k] for k in names]
    plan = ctx.plan_for(pdf, names)
    st = ctx.store_for(arrays)
    vals, nv = plan.pack(snap, norms)
    acc = torch.zeros(L.PFB_ACC_WORDS, dtype=torch.int64, device=f"cuda:{ctx.device}")
    L.check(L.lib().pfb_nll_partial_async(ctx.handle, plan.handle, st, 0, sh.size, sh.begin, L.dptr(vals),
                                          len(vals), L.dptr(nv), len(nv), ctypes.c_void_p(acc.data_ptr())),
            "pfb_nll_partial_async")
    L.check(L.lib().pfb_ctx_synchronize(ctx.handle), "pfb_ctx_synchronize")
    a = acc.cpu().numpy()
    frac = ctypes.c_int32()
    L.check(L.lib().pfb_ctx_last_fraction_failure(ctx.handle, ctypes.byref(frac)), "pfb_ctx_last_fraction_failure")
    if a[L.PFB_ACC_FAILS] or frac.value:
        err = L.PfbErr()
        L.check(L.lib().pfb_last_error(ctx.handle, ctypes.byref(err)), "pfb_last_error")
        engine.raise_for(err, err.code, "partial_nll")
    return a


def partial_nll(sh, pdf, snap, norms=None, block: int = DEFAULT_BLOCK, ctx=None):
    """Device ``partial_nll`` (P/sharding.py:94-114): the reference
    ``PartialSum`` with an exact expansion of the shard's sum."""
    if sh.size == 0:
        return PartialSum(sh.index, 0, 0.0, ())
    acc = partial_accumulator(sh, pdf, snap, norms, block, ctx)
    return PartialSum.from_components(sh.index, sh.size, components_from_acc(acc))


def sharded_nll(pdf, ds, snap=None, workers: int = 1, store=None, block: int = DEFAULT_BLOCK) -> float:
    """Device ``sharded_nll`` (P/sharding.py:134-146): shard, device partials,
    the reference's ``reduce_partials``."""
    store = store if store is not None else ref_engine.NormalizationStore()
    norms = ref_engine.resolve_norms(pdf, snap, store)
    return reduce_partials([partial_nll(sh, pdf, snap, norms, block) for sh in shard(ds, workers, block)])


# --- one process per GPU ------------------------------------------------------------------


def allreduce_accumulator(acc, group=None):
    """Sum an int64[72] accumulator over all ranks (NCCL on CUDA tensors, gloo on CPU)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    return acc


class PeerGroup:
    """The ranks' accumulator exchange over NVLink peer memory (pfb_peer_*):
    one single-CTA kernel per call instead of an NCCL all-reduce.  Handles are
    exchanged once with torch.distributed; `allreduce(acc)` sums an int64[72]
    CUDA tensor in place, bitwise the NCCL result."""

    def __init__(self, ctx, rank: int, world: int, group=None, timeout_s: float = 10.0):
        self.ctx, self.rank, self.world, self.timeout_s = ctx, int(rank), int(world), float(timeout_s)
        handle = (ctypes.c_uint8 * 64)()
        # every rank takes part in every collective below even if its own
        # step failed, so a failure raises on all ranks instead of hanging one
        code = L.lib().pfb_peer_create(ctx.handle, self.rank, self.world, handle)
        mine = bytes(handle) if code == L.OK else None
        handles = [mine]
        if self.world > 1:
            import torch.distributed as dist

            handles = [None] * self.world
            dist.all_gather_object(handles, mine, group=group)
        if any(h is None for h in handles):
            L.check(code, "pfb_peer_create")
            raise RuntimeError("peer-memory set-up failed on another rank")
        buf = (ctypes.c_uint8 * (64 * self.world)).from_buffer_copy(b"".join(handles))
        code = L.lib().pfb_peer_open(ctx.handle, buf)
        if self.world > 1:
            import torch
            import torch.distributed as dist

            ok = torch.tensor([1 if code == L.OK else 0], dtype=torch.int64)
            if dist.get_backend(group) == "nccl":
                ok = ok.cuda()
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
            if int(ok.item()) == 0:
                L.check(code, "pfb_peer_open")
                raise RuntimeError("peer-memory set-up failed on another rank")
        L.check(code, "pfb_peer_open")

    def allreduce(self, acc) -> None:
        code = L.lib().pfb_peer_allreduce(self.ctx.handle, ctypes.c_void_p(acc.data_ptr()), self.timeout_s)
        if code == L.E_PEER_TIMEOUT:
            raise TimeoutError(f"rank {self.rank}: a peer did not post its accumulator within {self.timeout_s} s")
        L.check(code, "pfb_peer_allreduce")


class ShardedNll:
    """Rank-local shard of a dataset resident in this rank's HBM.

    ``__call__(snap, norms)`` evaluates the full-dataset NLL: fused kernel on
    the local shard -> one all-reduce of the integer accumulator -> rounding.
    Every rank returns the same bits, equal to the single-GPU NLL.
    """

    def __init__(self, pdf, ds, rank: int, world: int, device: int, group=None, collective: str = "nccl"):
        import torch

        from . import engine

        if collective not in ("nccl", "peer", "fused"):
            raise ValueError("collective must be 'nccl', 'peer' or 'fused'")

        self.pdf = pdf
        self.rank, self.world, self.group = int(rank), int(world), group
        self.n = ds.n_events
        b = shard_bounds(self.n, world)
        self.begin, self.end = b[rank], b[rank + 1]
        self.ctx = engine.device_context(device)
        cols = ref_engine._needed_columns(pdf, ds)
        self.names = tuple(cols)
        # the shard only: this rank never holds the other ranks' events
        self.arrays = [np.ascontiguousarray(cols[k][self.begin:self.end]) for k in self.names]
        self.plan = self.ctx.plan_for(pdf, self.names)
        self.store = self.ctx.store_for(self.arrays)
        self.acc = torch.zeros(L.PFB_ACC_WORDS, dtype=torch.int64, device=f"cuda:{device}")
        self.ctx.set_stream(torch.cuda.current_stream(device).cuda_stream)
        # "fused": the exchange runs inside the NLL kernel (pfb_nll_peer), the
        # unfused peer kernel only on the rare slow path
        self.fused = collective == "fused"
        self.peers = PeerGroup(self.ctx, rank, world, group) if collective in ("peer", "fused") else None

    def launch(self, snap, norms):
        """Enqueue the local partial (no host sync)."""
        vals, nv = self.plan.pack(snap, norms)
        L.check(L.lib().pfb_nll_partial_async(self.ctx.handle, self.plan.handle, self.store, 0,
                                              self.end - self.begin, self.begin, L.dptr(vals), len(vals),
                                              L.dptr(nv), len(nv), ctypes.c_void_p(self.acc.data_ptr())),
                "pfb_nll_partial_async")

    def finish(self) -> float:
        from . import engine

        if self.peers is not None:
            self.peers.allreduce(self.acc)
        else:
            allreduce_accumulator(self.acc, self.group)
        out = ctypes.c_double()
        fails = ctypes.c_int64()
        code = L.lib().pfb_finalize(self.ctx.handle, ctypes.c_void_p(self.acc.data_ptr()), ctypes.byref(out),
                                    ctypes.byref(fails))
        if fails.value:
            self._raise_first_error()
        if code == L.E_INVALID_SUM:
            raise ValueError("-inf + inf in exact NLL sum")
        L.check(code, "pfb_finalize")
        return out.value

    def __call__(self, snap, norms) -> float:
        if self.fused:
            vals, nv = self.plan.pack(snap, norms)
            out, slow = ctypes.c_double(), ctypes.c_int32()
            code = L.lib().pfb_nll_peer(self.ctx.handle, self.plan.handle, self.store, 0, self.end - self.begin,
                                        self.begin, L.dptr(vals), len(vals), L.dptr(nv), len(nv),
                                        self.peers.timeout_s, ctypes.byref(out), ctypes.byref(slow))
            if code == L.E_PEER_TIMEOUT:
                raise TimeoutError(f"rank {self.rank}: a peer did not post its accumulator "
                                   f"within {self.peers.timeout_s} s")
            L.check(code, "pfb_nll_peer")
            if not slow.value:
                return out.value
            # some rank deferred blocks or failed: every rank saw the same
            # global status word and redoes the call unfused (fix-up, errors)
        self.launch(snap, norms)
        return self.finish()

    def _raise_first_error(self):
        """Rare path: gather every rank's first failure, raise the global first."""
        from . import engine

        err = L.PfbErr()
        L.check(L.lib().pfb_last_error(self.ctx.handle, ctypes.byref(err)), "pfb_last_error")
        code, index, node, value = first_error_across_ranks(
            self.rank, self.world, (err.code, err.index, err.node, err.value), self.group, self.acc.device)
        e = L.PfbErr()
        e.code, e.index, e.node, e.value = code, index, node, value
        engine.raise_for(e, e.code, "ShardedNll")


def first_error_across_ranks(rank: int, world: int, err: tuple, group=None, device="cpu") -> tuple:
    """The error the reference would raise: shards are evaluated in order
    (sharding.py:145), so the lowest failing rank wins.  err = (code, index,
    node, value); code 0 means this rank had no failure."""
    import torch
    import torch.distributed as dist

    code, index, node, value = err
    mine = torch.tensor([rank if code else world, code, index, node], dtype=torch.int64, device=device)
    val = torch.tensor([value], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and world > 1:
        allk = [torch.empty_like(mine) for _ in range(world)]
        allv = [torch.empty_like(val) for _ in range(world)]
        dist.all_gather(allk, mine, group=group)
        dist.all_gather(allv, val, group=group)
    else:
        allk, allv = [mine], [val]
    best = min(range(len(allk)), key=lambda i: int(allk[i][0]))
    k = allk[best].cpu().tolist()
    return int(k[1]), int(k[2]), int(k[3]), float(allv[best].item())
