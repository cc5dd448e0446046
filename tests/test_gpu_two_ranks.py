"""Two ranks of ShardedNll on one B200 with a gloo exchange: each process
keeps only its reference shard() rows in HBM, runs the fused NLL kernel on
them into its 72-word exact accumulator, and the accumulators are summed
over gloo (host-side, so neither rank's kernels wait on the other's) and
rounded once.  Both ranks must return the same bits, equal to the
single-process NLL of all events (P/sharding.py:134-146 semantics), and a
failure in one rank's shard must raise the reference's error -- with the
global event index -- on every rank.  The NCCL / NVLink exchanges are the
same accumulator arithmetic (tests/test_gpu_sharding.py, test_gpu_peer.py)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = 3_000_000 + 4097


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _columns():
    rng = np.random.default_rng(41)
    xs = np.clip(rng.normal(5.0, 1.0, N), 0.0, 10.0)
    ys = np.clip(rng.exponential(2.5, N), 0.0, 10.0)
    return xs, ys


def _model(bad_index):
    """C2 for the value test; for the error test a narrow gaussian whose
    density underflows to 0 at one event (NonPositiveDensity, P/engine.py:183-186)."""
    from paper_1710_08826_b200._reference import parafit as P
    from tests import models

    if bad_index is None:
        (x, y), pdf, _ = models.c2()
        return [x, y], pdf, list(_columns())
    x = P.Variable.observable("x", 0.0, 10.0)
    pdf = P.gaussian(x, P.Variable("mu", 5.0, 0.0, 10.0), P.Variable("sg", 0.05, 0.01, 1.0))
    xs = np.clip(np.random.default_rng(43).normal(5.0, 0.1, N), 4.0, 6.0)
    xs[bad_index] = 0.0  # z = 100: exp(-5000) = 0
    return [x], pdf, [xs]


def _worker(rank, world, port, bad_index, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1710_08826_b200 as pf
        from paper_1710_08826_b200._reference import parafit as P

        torch.cuda.set_device(0)
        obs, pdf, cols = _model(bad_index)
        ds = pf.DeviceDataSet.from_columns(obs, cols, device=None)
        snap = P.snapshot(pdf.param_closure())
        norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
        sh = pf.ShardedNll(pdf, ds, rank, world, 0, collective="nccl")  # default group = gloo here
        try:
            out = ("ok", float(sh(snap, norms)).hex())
        except Exception as exc:  # the reference's error class and global index
            out = (type(exc).__name__, getattr(exc, "index", None))
        q.put((rank, out, (sh.begin, sh.end)))
    finally:
        dist.destroy_process_group()


def _run(world, bad_index=None):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, bad_index, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(res)


def test_two_ranks_gloo_exchange_bitwise_single_gpu():
    import paper_1710_08826_b200 as pf
    from tests import models

    (x, y), pdf, _ = models.c2()
    xs, ys = _columns()
    want = float(pf.nll(pdf, models.dataset([x, y], [xs, ys]))).hex()
    res = _run(2)
    assert [r[1] for r in res] == [("ok", want), ("ok", want)]
    # the reference shard() bounds: interior bound block-aligned (P/sharding.py:80-85)
    (b0, b1), (c0, c1) = res[0][2], res[1][2]
    assert b0 == 0 and b1 == c0 and c1 == N and b1 % 4096 == 0


def test_two_ranks_error_in_one_shard_raises_on_both():
    """An event whose density underflows to 0 in rank 1's shard: every rank
    raises what the reference's own sharded_nll (P/sharding.py:134-146)
    raises for the same events -- NonPositiveDensity at the global index."""
    from paper_1710_08826_b200._reference import parafit as P
    from tests import models

    bad = N - 5
    res = _run(2, bad_index=bad)
    assert res[0][1] == res[1][1]
    obs, pdf, cols = _model(bad)
    with pytest.raises(P.errors.ParafitError) as want:
        P.sharded_nll(pdf, models.dataset(obs, cols), workers=2)
    assert res[0][1] == (type(want.value).__name__, getattr(want.value, "index", None)) == ("NonPositiveDensity", bad)
