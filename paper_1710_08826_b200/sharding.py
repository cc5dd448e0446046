"""Event sharding across GPUs and the exact cross-shard reduction.

Reference semantics (sharding.py:68-146):

* ``shard(ds, W, block)``: contiguous ceil/floor split, interior bounds
  aligned down to the block when N >= W*block -- computed by the native
  ``pfb_shard_bounds`` so the integers are identical.
* ``partial_nll``: one shard's exact partial.  The reference ships a
  Shewchuk expansion; here the partial *is* the 72-word integer accumulator
  of its block sums, which sums associatively.
* ``reduce_partials``: every shard exactly once (MissingShard /
  DuplicateShard), then one rounding -- bitwise the single-process total
  whenever the shards are block-aligned.

Multi-GPU (one process per GPU, torch.distributed): :class:`ShardedNll` keeps
each rank's shard resident in its HBM; one NLL call is one fused kernel that
writes the shard's accumulator, ONE all-reduce of 72 int64 (NCCL over
NVLink), one rounding kernel.  The same code runs over gloo on CPU tensors for
the host-side tests (accumulators produced by the host digit split).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np

from . import _lib as L
from .errors import DuplicateShard, MissingShard

DEFAULT_BLOCK = L.PFB_BLOCK


def shard_bounds(n: int, workers: int, block: int = DEFAULT_BLOCK) -> list[int]:
    """[b0=0, b1, ..., bW=n] exactly as the reference shard() (sharding.py:80-85)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    out = (ctypes.c_int64 * (workers + 1))()
    L.check(L.lib().pfb_shard_bounds(int(n), int(workers), int(block), out), "pfb_shard_bounds")
    return list(out)


@dataclass(frozen=True)
class Shard:
    index: int
    begin: int
    end: int
    columns: Mapping[str, np.ndarray]

    @property
    def size(self) -> int:
        return self.end - self.begin


@dataclass(frozen=True)
class PartialSum:
    """One shard's contribution: rounded sum plus its exact integer accumulator."""

    shard_index: int
    count: int
    sum: float
    acc: tuple[int, ...] = ()


def shard(ds, workers: int, block: int = DEFAULT_BLOCK) -> list[Shard]:
    n = ds.n_events
    columns = ds.columns() if n else {o.name: np.empty(0) for o in ds.observables}
    b = shard_bounds(n, workers, block)
    return [Shard(k, b[k], b[k + 1], {name: col[b[k]:b[k + 1]] for name, col in columns.items()})
            for k in range(workers)]


def round_acc(acc) -> float:
    a = np.ascontiguousarray(np.asarray(acc, dtype=np.int64))
    out = ctypes.c_double()
    code = L.lib().pfb_acc_round(a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ctypes.byref(out))
    if code == L.E_INVALID_SUM:
        raise ValueError("-inf + inf in exact sum")
    L.check(code, "pfb_acc_round")
    return out.value


def acc_of_values(values) -> np.ndarray:
    """Host digit split of doubles into an accumulator (same code as the device)."""
    v = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    acc = np.zeros(L.PFB_ACC_WORDS, dtype=np.int64)
    L.check(L.lib().pfb_acc_add_host(acc.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), L.dptr(v), len(v)),
            "pfb_acc_add_host")
    return acc


def partial_nll(sh: Shard, pdf, snap, norms=None, block: int = DEFAULT_BLOCK, ctx=None) -> PartialSum:
    """Exact partial of one shard on the GPU (reference sharding.py:94-114)."""
    import torch

    from . import engine

    if norms is None:
        norms = engine.resolve_norms(pdf, snap, engine.NormalizationStore())
    if sh.size == 0:
        return PartialSum(sh.index, 0, 0.0, tuple([0] * L.PFB_ACC_WORDS))
    if block != DEFAULT_BLOCK:
        raise ValueError(f"the device reduction block is fixed at {DEFAULT_BLOCK}")
    ctx = ctx or engine.device_context(0)
    names = tuple(sorted(sh.columns))
    needed = {nm for node in pdf.walk() for nm in node.observable_names()}
    names = tuple(nm for nm in names if nm in needed)
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
    if a[L.PFB_ACC_FAILS]:
        err = L.PfbErr()
        L.check(L.lib().pfb_last_error(ctx.handle, ctypes.byref(err)), "pfb_last_error")
        engine.raise_for(err, err.code, pdf, "partial_nll")
    return PartialSum(sh.index, sh.size, round_acc(a), tuple(int(x) for x in a))


def reduce_partials(partials: Sequence[PartialSum]) -> float:
    """Exact merge in shard order (reference sharding.py:117-131)."""
    seen = sorted(partials, key=lambda p: p.shard_index)
    indices = [p.shard_index for p in seen]
    for k, idx in enumerate(indices):
        if indices.count(idx) > 1:
            raise DuplicateShard(f"shard index {idx} appears more than once")
        if idx != k:
            raise MissingShard(f"expected shard index {k}, found {idx}")
    total = np.zeros(L.PFB_ACC_WORDS, dtype=np.int64)
    for p in seen:
        total += np.asarray(p.acc if p.acc else acc_of_values([p.sum]), dtype=np.int64)
    return round_acc(total)


def sharded_nll(pdf, ds, snap=None, workers: int = 1, store=None, block: int = DEFAULT_BLOCK) -> float:
    from . import engine

    store = store if store is not None else engine.NormalizationStore()
    norms = engine.resolve_norms(pdf, snap, store)
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
        cols = engine._needed_columns(pdf, ds)
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
        engine.raise_for(e, e.code, self.pdf, "ShardedNll")


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
