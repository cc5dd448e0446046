"""World-size-2 gloo test of the multi-rank reduction (CPU, no GPU).

Each rank owns the reference shard() slice of the events; its exact partial
(the 72-word integer accumulator of its block sums -- produced here by the
host digit split, the same code the device runs) is all-reduced over gloo and
rounded once.  The result must equal the single-process reference NLL bit for
bit, and the error chosen across ranks must be the lowest failing shard's.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import parafit_oracle as O
        from paper_1710_08826_b200 import sharding
        from tests import models

        rng = np.random.default_rng(77)
        xs = np.clip(rng.normal(5.0, 1.0, n), 0, 10)
        ys = np.clip(rng.exponential(2.5, n), 0, 10)
        spec = models.c2_spec((5.0, 1.0, -0.4))
        b = sharding.shard_bounds(n, world)
        lo, hi = b[rank], b[rank + 1]
        local = {"x": xs[lo:hi], "y": ys[lo:hi]}
        bs = O.nll_block_sums(spec, local)  # stand-in for the device partial
        acc = torch.from_numpy(sharding.acc_of_values(bs))
        sharding.allreduce_accumulator(acc)
        total = sharding.round_acc(acc.numpy())
        # error selection: ranks 1.. fail, rank 1 must win
        err = (1, 1000 + rank, -1, 0.0) if rank >= 1 else (0, -1, -1, float("nan"))
        first = sharding.first_error_across_ranks(rank, world, err)
        q.put((rank, total, first))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_allreduce_of_exact_partials(world):
    from oracle import parafit_oracle as O
    from tests import models

    n = 9 * 4096 + 123  # N >= W*4096: block-aligned shards
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(77)
    xs = np.clip(rng.normal(5.0, 1.0, n), 0, 10)
    ys = np.clip(rng.exponential(2.5, n), 0, 10)
    want = O.nll(models.c2_spec((5.0, 1.0, -0.4)), {"x": xs, "y": ys})
    for rank, total, first in results:
        assert total == want, rank
        assert first[:2] == (1, 1001)


def _peer_setup_worker(rank, world, port, q):
    """PeerGroup set-up where rank 0's mailbox creation 'succeeds' (a stand-in
    that returns OK) and rank 1's fails (no GPU here): every rank must raise,
    none may hang in the handle exchange."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1710_08826_b200 import _lib as L
        from paper_1710_08826_b200 import sharding

        class FakeCtx:
            handle = None

        if rank == 0:
            class Lib:
                def __getattr__(self, name):
                    return getattr(L.lib(), name)

                @staticmethod
                def pfb_peer_create(h, r, w, out):
                    return L.OK

            real = L.lib
            L.lib = lambda: Lib()
        try:
            sharding.PeerGroup(FakeCtx(), rank, world)
            q.put((rank, "no error"))
        except Exception as exc:  # noqa: BLE001
            q.put((rank, type(exc).__name__))
        finally:
            if rank == 0:
                L.lib = real
    finally:
        dist.destroy_process_group()


def test_peer_setup_failure_raises_on_every_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_setup_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results[0] == "RuntimeError"   # "failed on another rank"
    assert results[1] != "no error"       # its own pfb_peer_create error
