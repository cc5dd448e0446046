"""Accumulator exchange over peer memory (pfb_peer_*), on one GPU: the
single-rank path, the protocol against a pre-posted peer contribution, and
the bounded wait when a peer never posts (no hung GPU)."""

import ctypes

import numpy as np
import pytest

from tests import models

pytestmark = pytest.mark.gpu

SLOT = 80      # words per slot (csrc/pfb_peer.cu)
PEERS = 16


def slot_word(par, r):
    return (par * PEERS + r) * SLOT


def flag_word(par, r):
    return 2 * PEERS * SLOT + par * PEERS + r


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
    snap = pf.snapshot(pdf.param_closure())
    norms = pf.resolve_norms(pdf, snap, pf.NormalizationStore())
    assert sn(snap, norms) == pf.nll(pdf, ds)
    assert sn(snap, norms) == pf.nll(pdf, ds)  # parity flips between calls


def test_protocol_with_preposted_peer(pf):
    import torch

    from paper_1710_08826_b200 import _lib as L

    h = raw_ctx()
    try:
        L.check(L.lib().pfb_peer_create(h, 0, 2, None), "pfb_peer_create")
        other = torch.zeros(2 * PEERS * SLOT + 2 * PEERS, dtype=torch.int64, device="cuda")
        ptrs = (ctypes.c_void_p * 2)(None, ctypes.c_void_p(other.data_ptr()))
        L.check(L.lib().pfb_peer_attach(h, ptrs), "pfb_peer_attach")
        mb = ctypes.c_void_p()
        L.check(L.lib().pfb_peer_mailbox(h, ctypes.byref(mb)), "pfb_peer_mailbox")
        mine = np.arange(72, dtype=np.int64) * 3 - 50
        theirs = np.arange(72, dtype=np.int64) * -7 + (1 << 40)
        # rank 1 has already posted call 1 (parity 1) into rank 0's mailbox
        nwords = 2 * PEERS * SLOT + 2 * PEERS
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
        other = torch.zeros(2 * PEERS * SLOT + 2 * PEERS, dtype=torch.int64, device="cuda")
        ptrs = (ctypes.c_void_p * 2)(None, ctypes.c_void_p(other.data_ptr()))
        L.check(L.lib().pfb_peer_attach(h, ptrs), "pfb_peer_attach")
        acc = torch.ones(72, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        assert L.lib().pfb_peer_allreduce(h, ctypes.c_void_p(acc.data_ptr()), 0.01) == L.E_PEER_TIMEOUT
    finally:
        L.lib().pfb_ctx_destroy(h)
