"""Accumulator exchange over peer memory (pfb_peer_*), on one GPU: the
single-rank path, the protocol against a pre-posted peer contribution, and
the bounded wait when a peer never posts (no hung GPU)."""

import ctypes

import numpy as np
import pytest

from tests import models
from paper_1710_08826_b200._reference import parafit as P

pytestmark = pytest.mark.gpu

SLOT = 80      # words per slot (csrc/pfb_peer.cu)
PEERS = 16


def slot_word(par, r):
    return (par * PEERS + r) * SLOT


def flag_word(par, r):
    return 2 * PEERS * SLOT + par * PEERS + r


LINE_BASE = 2 * PEERS * SLOT + 2 * PEERS      # flag-in-line region of the fused exchange
MBOX_WORDS = LINE_BASE + 2 * 2 * PEERS * SLOT  # whole mailbox, 64-bit words


def line_word(par, r, w):
    return LINE_BASE + 2 * ((par * PEERS + r) * SLOT + w)


def put_line(host, par, r, w, value, seq):
    u = int(value) & ((1 << 64) - 1)
    lo, hi = u & 0xFFFFFFFF, u >> 32
    host[line_word(par, r, w)] = np.int64(np.uint64((seq << 32) | lo).astype(np.int64))
    host[line_word(par, r, w) + 1] = np.int64(np.uint64((seq << 32) | hi).astype(np.int64))


def get_line(arr, par, r, w):
    a = int(np.uint64(arr[line_word(par, r, w)].astype(np.uint64)))
    b = int(np.uint64(arr[line_word(par, r, w) + 1].astype(np.uint64)))
    seq1, seq2 = a >> 32, b >> 32
    v = ((b & 0xFFFFFFFF) << 32) | (a & 0xFFFFFFFF)
    return np.int64(np.uint64(v).astype(np.int64)), seq1, seq2


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    return pf


def _copy_d2d(dst: int, src: int, nbytes: int) -> None:
    from cuda.bindings import runtime as rt

    (err,) = rt.cudaMemcpy(dst, src, nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
    assert err == rt.cudaError_t.cudaSuccess


def raw_ctx():
    from paper_1710_08826_b200 import _lib as L

    h = ctypes.c_void_p()
    L.check(L.lib().pfb_ctx_create(0, ctypes.byref(h)), "pfb_ctx_create")
    return h


def test_single_rank_sharded_nll_equals_nll(pf):
    from paper_1710_08826_b200.sharding import ShardedNll

    rng = np.random.default_rng(3)
    (x, y), pdf, _ = models.c2()
    ds = models.dataset([x, y], [np.clip(rng.normal(5, 1, 50000), 0, 10), np.clip(rng.exponential(2.5, 50000), 0, 10)])
    sn = ShardedNll(pdf, ds, 0, 1, 0, collective="peer")
    snap = P.snapshot(pdf.param_closure())
    norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
    assert sn(snap, norms) == pf.nll(pdf, ds)
    assert sn(snap, norms) == pf.nll(pdf, ds)  # parity flips between calls


def test_protocol_with_preposted_peer(pf):
    import torch

    from paper_1710_08826_b200 import _lib as L

    h = raw_ctx()
    try:
        L.check(L.lib().pfb_peer_create(h, 0, 2, None), "pfb_peer_create")
        other = torch.zeros(MBOX_WORDS, dtype=torch.int64, device="cuda")
        ptrs = (ctypes.c_void_p * 2)(None, ctypes.c_void_p(other.data_ptr()))
        L.check(L.lib().pfb_peer_attach(h, ptrs), "pfb_peer_attach")
        mb = ctypes.c_void_p()
        L.check(L.lib().pfb_peer_mailbox(h, ctypes.byref(mb)), "pfb_peer_mailbox")
        mine = np.arange(72, dtype=np.int64) * 3 - 50
        theirs = np.arange(72, dtype=np.int64) * -7 + (1 << 40)
        # rank 1 has already posted call 1 (parity 1) into rank 0's mailbox
        nwords = MBOX_WORDS
        host = np.zeros(nwords, dtype=np.int64)
        host[slot_word(1, 1):slot_word(1, 1) + 72] = theirs
        host[flag_word(1, 1)] = 1
        box = torch.from_numpy(host).cuda()
        torch.cuda.synchronize()
        _copy_d2d(mb.value, box.data_ptr(), nwords * 8)  # into rank 0's mailbox
        acc = torch.from_numpy(mine.copy()).cuda()
        torch.cuda.synchronize()
        code = L.lib().pfb_peer_allreduce(h, ctypes.c_void_p(acc.data_ptr()), 5.0)
        assert code == L.OK
        assert acc.cpu().numpy().tolist() == (mine + theirs).tolist()
        # rank 0 wrote its own limbs into rank 1's mailbox and raised its flag there
        o = other.cpu().numpy()
        assert o[slot_word(1, 0):slot_word(1, 0) + 72].tolist() == mine.tolist()
        assert o[flag_word(1, 0)] == 1
    finally:
        L.lib().pfb_ctx_destroy(h)


def test_missing_peer_times_out(pf):
    import torch

    from paper_1710_08826_b200 import _lib as L

    h = raw_ctx()
    try:
        L.check(L.lib().pfb_peer_create(h, 0, 2, None), "pfb_peer_create")
        other = torch.zeros(MBOX_WORDS, dtype=torch.int64, device="cuda")
        ptrs = (ctypes.c_void_p * 2)(None, ctypes.c_void_p(other.data_ptr()))
        L.check(L.lib().pfb_peer_attach(h, ptrs), "pfb_peer_attach")
        acc = torch.ones(72, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        assert L.lib().pfb_peer_allreduce(h, ctypes.c_void_p(acc.data_ptr()), 0.01) == L.E_PEER_TIMEOUT
    finally:
        L.lib().pfb_ctx_destroy(h)


# ---- the exchange fused into the NLL kernel's epilogue (pfb_nll_peer) ----------------


def test_fused_single_rank_equals_nll(pf):
    from paper_1710_08826_b200.sharding import ShardedNll

    rng = np.random.default_rng(4)
    n = 3 * 4096 * 50 + 777
    (x, y), pdf, _ = models.c2()
    ds = models.dataset([x, y], [np.clip(rng.normal(5, 1, n), 0, 10), np.clip(rng.exponential(2.5, n), 0, 10)])
    sn = ShardedNll(pdf, ds, 0, 1, 0, collective="fused")
    snap = P.snapshot(pdf.param_closure())
    norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
    ref = pf.nll(pdf, ds)
    for _ in range(5):  # parity alternates call to call
        assert sn(snap, norms) == ref


def test_fused_with_preposted_peer(pf):
    """Rank 0 of 2 evaluates its shard with the exchange fused into the NLL
    kernel; rank 1's limbs (the other shard's exact partial) are pre-posted in
    rank 0's mailbox.  The fused call returns the whole dataset's NLL bit for
    bit and leaves rank 0's limbs + status word + flag in rank 1's mailbox."""
    import torch

    from paper_1710_08826_b200 import _lib as L
    from paper_1710_08826_b200 import sharding
    from paper_1710_08826_b200.engine import DeviceContext

    rng = np.random.default_rng(5)
    n = 4096 * 300 + 1001
    (x, y), pdf, _ = models.c2((4.9, 1.05, -0.38))
    cx, cy = np.clip(rng.normal(5, 1, n), 0, 10), np.clip(rng.exponential(2.5, n), 0, 10)
    ds = models.dataset([x, y], [cx, cy])
    whole = pf.nll(pdf, ds)
    b = sharding.shard_bounds(n, 2)
    ctx = DeviceContext(0)
    try:
        plan = ctx.plan_for(pdf, ("x", "y"))
        snap = P.snapshot(pdf.param_closure())
        norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
        vals, nv = plan.pack(snap, norms)
        # rank 1's exact partial over its shard
        st1 = ctx.store_for([np.ascontiguousarray(cx[b[1]:]), np.ascontiguousarray(cy[b[1]:])])
        acc1 = torch.zeros(72, dtype=torch.int64, device="cuda")
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        L.check(L.lib().pfb_nll_partial_async(ctx.handle, plan.handle, st1, 0, n - b[1], b[1], L.dptr(vals),
                                              len(vals), L.dptr(nv), len(nv), ctypes.c_void_p(acc1.data_ptr())),
                "pfb_nll_partial_async")
        torch.cuda.synchronize()
        theirs = acc1.cpu().numpy()
        # wire rank 0 to a stand-in mailbox for rank 1 and pre-post rank 1's call 1
        L.check(L.lib().pfb_peer_create(ctx.handle, 0, 2, None), "pfb_peer_create")
        other = torch.zeros(MBOX_WORDS, dtype=torch.int64, device="cuda")
        ptrs = (ctypes.c_void_p * 2)(None, ctypes.c_void_p(other.data_ptr()))
        L.check(L.lib().pfb_peer_attach(ctx.handle, ptrs), "pfb_peer_attach")
        mb = ctypes.c_void_p()
        L.check(L.lib().pfb_peer_mailbox(ctx.handle, ctypes.byref(mb)), "pfb_peer_mailbox")
        nwords = MBOX_WORDS
        host = np.zeros(nwords, dtype=np.int64)
        for w in range(72):
            put_line(host, 1, 1, w, theirs[w], 1)
        put_line(host, 1, 1, 72, 0, 1)  # rank 1: no deferred blocks, no error
        box = torch.from_numpy(host).cuda()
        torch.cuda.synchronize()
        _copy_d2d(mb.value, box.data_ptr(), nwords * 8)
        st0 = ctx.store_for([np.ascontiguousarray(cx[:b[1]]), np.ascontiguousarray(cy[:b[1]])])
        out, slow = ctypes.c_double(), ctypes.c_int32()
        code = L.lib().pfb_nll_peer(ctx.handle, plan.handle, st0, 0, b[1], 0, L.dptr(vals), len(vals), L.dptr(nv),
                                    len(nv), 5.0, ctypes.byref(out), ctypes.byref(slow))
        assert code == L.OK and slow.value == 0
        assert out.value == whole
        o = other.cpu().numpy()
        lines = [get_line(o, 1, 0, w) for w in range(73)]
        assert all(s1 == 1 and s2 == 1 for _, s1, s2 in lines)
        mine = np.array([v for v, _, _ in lines[:72]], dtype=np.int64)
        assert sharding.round_acc(mine + theirs) == whole
        assert lines[72][0] == 0
        # a peer that never posts call 2: bounded wait, no hung GPU
        code = L.lib().pfb_nll_peer(ctx.handle, plan.handle, st0, 0, b[1], 0, L.dptr(vals), len(vals), L.dptr(nv),
                                    len(nv), 0.01, ctypes.byref(out), ctypes.byref(slow))
        assert code == L.E_PEER_TIMEOUT
    finally:
        ctx.close()


def test_fused_slow_path_reports_the_reference_error(pf):
    """An event with zero density: the fused call flags the slow path and the
    unfused redo raises the reference's NonPositiveDensity (global index)."""
    from paper_1710_08826_b200._reference import errors as E
    from paper_1710_08826_b200.sharding import ShardedNll

    rng = np.random.default_rng(6)
    n = 4096 * 20 + 5
    x = np.clip(rng.normal(5, 0.1, n), 0, 10)
    x[4321] = 9.999  # 50 sigma from the mean of a pure gaussian: the density underflows to 0
    xv, pdf, params = models.c1((5.0, 0.1, -0.3, 1.0))
    ds = models.dataset([xv], [x])
    with pytest.raises(E.NonPositiveDensity) as ref:
        pf.nll(pdf, ds)
    sn = ShardedNll(pdf, ds, 0, 1, 0, collective="fused")
    snap = P.snapshot(pdf.param_closure())
    norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
    with pytest.raises(E.NonPositiveDensity) as got:
        sn(snap, norms)
    assert got.value.index == ref.value.index == 4321


@pytest.mark.parametrize("cfg,n", [("c1", 4096 * 40 + 3), ("c1", 2_000_001), ("c2", 6_000_123), ("c3", 300_007)])
def test_fused_single_rank_every_kernel_family(pf, cfg, n):
    """The fused epilogue sits in both finish paths (finish_launch: bulk /
    SIMT kernels; finish_launch_pts: TMA unit kernels): world = 1 equals the
    plain NLL bit for bit for each family, ragged sizes included."""
    from paper_1710_08826_b200 import mcgen
    from paper_1710_08826_b200.sharding import ShardedNll

    if cfg == "c1":
        x, pdf, _ = models.c1()
        col = mcgen.device_sumpdf_1d(n, 5.0, 0.5, -0.3, 0.3, 0.0, 10.0, 31)
        ds = pf.DeviceDataSet.from_columns([x], [col], device=None)
    elif cfg == "c2":
        (x, y), pdf, _ = models.c2()
        cx, cy = mcgen.device_prod_2d(n, 5.0, 1.0, -0.4, 0.0, 10.0, 32)
        ds = pf.DeviceDataSet.from_columns([x, y], [cx, cy], device=None)
    else:
        terms = [(p, s, m, w, mag, ph) for (p, m, w, s, mag, ph) in models.C3_TERMS]
        a, b = mcgen.device_dalitz(n, terms, models.D_CHANNEL_T, 33)
        (o12, o13), pdf, _ = models.c3()
        ds = pf.DeviceDataSet.from_columns([o12, o13], [a, b], device=None)
    ref = pf.nll(pdf, ds)
    sn = ShardedNll(pdf, ds, 0, 1, 0, collective="fused")
    snap = P.snapshot(pdf.param_closure())
    norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
    for _ in range(3):
        assert sn(snap, norms) == ref
