"""Device parity against the reference's golden outputs and the CPU oracle.

Bar (north_star): NLL within 1e-10 relative; block sums / totals of given
terms, shard bounds, grid masks and error indices bit-exact.
"""

import ctypes
import json
import math
import os

import numpy as np
import pytest

from oracle import parafit_oracle as O
from tests import models
from paper_1710_08826_b200._reference import parafit as P

pytestmark = pytest.mark.gpu

RTOL = 1e-10


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf
    import paper_1710_08826_b200.dalitz  # noqa: F401
    from paper_1710_08826_b200 import _lib as L

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    return pf


def load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name))


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


# --- reduction known-answer tests ----------------------------------------------------


def test_terms_block_sums_bitwise(pf, golden_dir):
    from paper_1710_08826_b200 import _lib as L

    ctx = pf.device_context(0)
    g = load(golden_dir, "reduction.npz")
    for key in g.files:
        if not key.startswith("terms_"):
            continue
        tag = key[len("terms_"):]
        terms = np.ascontiguousarray(g[key])
        nb = len(g[f"bsums_{tag}"])
        out = np.empty(nb)
        total = ctypes.c_double()
        for warps in (1, 2, 4, 8):
            ctx.set_warps_per_block(warps)
            L.check(L.lib().pfb_terms_block_sums(ctx.handle, L.dptr(terms), len(terms), L.dptr(out),
                                                 ctypes.byref(total)), "terms")
            assert out.tolist() == g[f"bsums_{tag}"].tolist(), (tag, warps)
            assert total.value == g[f"total_{tag}"][0], (tag, warps)
    ctx.set_warps_per_block(0)


# --- C1 / C2 / C3 parity -----------------------------------------------------------------


def test_c1_sumpdf_parity(pf, golden_dir):
    g = load(golden_dir, "c1_sumpdf.npz")
    x, pdf, params = models.c1()
    ds = models.dataset([x], [g["x"]])
    for i, pt in enumerate(g["points"]):
        for v, val in zip(params, pt):
            P.set_value(v, float(val))
        got = pf.nll(pdf, ds)
        assert rel(got, g["nll"][i]) <= RTOL, (i, got, g["nll"][i])
        bs = pf.nll_block_sums(pdf, ds.columns(), P.snapshot(pdf.param_closure()),
                               P.resolve_norms(pdf, None, P.NormalizationStore()), 0, ds.n_events)
        np.testing.assert_allclose(bs, g[f"bsums_{i}"], rtol=1e-12)


def test_c1_random_points_and_far_outliers(pf, golden_dir):
    """The C1 product-mode evaluator (EvSum2GE) against the reference's own
    nll on the same events at 30 random parameter points (<= 1e-12), and with
    events so far from a very narrow gaussian (|x - mu| = 5000 sigma: d ~
    -1.25e7, where the exponential's integer scale index would wrap) that
    their units must fail the |x - mu| certificate and take the exact fix-up."""
    g = load(golden_dir, "c1_sumpdf.npz")
    x, pdf, params = models.c1()
    ds = models.dataset([x], [g["x"]])
    rng = np.random.default_rng(21)
    for _ in range(30):
        pt = [rng.uniform(4.5, 5.5), rng.uniform(0.3, 0.8), rng.uniform(-0.5, -0.1), rng.uniform(0.1, 0.6)]
        for v, val in zip(params, pt):
            P.set_value(v, val)
        snap = P.snapshot(pdf.param_closure())
        dev = pf.nll(pdf, ds)
        with pf.reference_norms():
            want = P.nll(pdf, ds, snap, P.Backend("serial"), P.NormalizationStore())
        assert rel(dev, want) <= 1e-12, (pt, dev, want)
    xv = P.Variable.observable("x", 0.0, 10.0)
    mu, sg = P.Variable("mu", 5.0, 0.0, 10.0), P.Variable("sg", 0.001, 1e-4, 5.0)
    al, f = P.Variable("al", -0.3, -5.0, 5.0), P.Variable("f", 0.3, 0.0, 1.0)
    narrow = P.add_pdf([P.gaussian(xv, mu, sg), P.exponential(xv, al)], [f])
    xs = np.concatenate([rng.normal(5.0, 0.001, 20000), rng.uniform(0.0, 10.0, 20000)])
    xs[::997] = 0.0  # |x - mu| = 5000 sigma
    dsn = models.dataset([xv], [xs])
    snap = P.snapshot(narrow.param_closure())
    with pf.reference_norms():
        want = P.nll(narrow, dsn, snap, P.Backend("serial"), P.NormalizationStore())
    assert rel(pf.nll(narrow, dsn), want) <= 1e-12


def test_c1_product_shells_bitwise(pf):
    """The C1 product evaluator (EvSum2GE) through every shell the pipeline
    modes select -- bulk prefetch (1, 2), TMA unit ring (3; 1 from 24 blocks
    per SM: tests/test_gpu_scale.py), warp tasks (4) -- gives the same bits;
    the log-domain SIMT kernel (0) within 1e-12."""
    x, pdf, params = models.c1()
    rng = np.random.default_rng(8)
    n = 3 * 1_000_000 + 4097
    xs = np.clip(np.concatenate([rng.normal(5, 0.5, n // 3), rng.exponential(3.3, n - n // 3)]), 0, 10)
    ds = models.dataset([x], [xs])
    ctx = pf.device_context(0)
    got = {}
    try:
        for mode in (1, 2, 3, 4, 0):
            ctx.set_pipeline(mode)
            got[mode] = pf.nll(pdf, ds)
    finally:
        ctx.set_pipeline(1)
    assert got[1] == got[2] == got[3] == got[4]
    assert rel(got[0], got[1]) <= 1e-12


def test_c2_prod_parity_and_shards(pf, golden_dir):
    g = load(golden_dir, "c2_prod.npz")
    (x, y), pdf, params = models.c2()
    ds = models.dataset([x, y], [g["x"], g["y"]])
    for i, pt in enumerate(g["points"]):
        for v, val in zip(params, pt):
            P.set_value(v, float(val))
        assert rel(pf.nll(pdf, ds), g["nll"][i]) <= RTOL
    for v, val in zip(params, g["points"][0]):
        P.set_value(v, float(val))
    whole = pf.nll(pdf, ds)
    for w in (2, 3, 4):
        got = pf.sharded_nll(pdf, ds, P.snapshot(pdf.param_closure()), workers=w)
        assert rel(got, g[f"sharded_{w}"][0]) <= RTOL
        # aligned shards (N >= W*4096) reproduce the unsharded device total bit for bit
        assert got == whole


def test_c3_dalitz_parity(pf, golden_dir):
    g = load(golden_dir, "c3_dalitz.npz")
    (s12, s13), pdf, terms = models.c3()
    ds = models.dataset([s12, s13], [g["s12"], g["s13"]])
    got = pf.nll(pdf, ds)
    assert rel(got, g["nll"][0]) <= RTOL, (got, g["nll"][0])
    P.set_value(terms[1].magnitude, 0.9)
    P.set_value(terms[2].phase, 1.1)
    assert rel(pf.nll(pdf, ds), g["nll_b"][0]) <= RTOL


def test_dalitz_grid_mask_and_integrals(pf, golden_dir):
    g = load(golden_dir, "c3_dalitz.npz")
    ch = P.DecayChannel(*models.D_CHANNEL_T)
    for tag, grid in (("64x64", (64, 64)), ("400x400", (400, 400))):
        dg = pf.dalitz.device_grid(ch, grid, owner="mask-test")
        mask = dg.mask()
        assert np.array_equal(np.packbits(mask), g[f"mask_{tag}"]), tag
        assert int(mask.sum()) == int(g[f"ninside_{tag}"][0]) == dg.n_inside
        assert dg.area == g[f"darea_{tag}"][0]
        _, pdf, terms = models.c3(grid=grid)
        cache = pf.dalitz.compute_integrals(terms, ch, grid)
        np.testing.assert_allclose(cache.matrix, g[f"matrix_{tag}"], rtol=1e-12, atol=0)
        assert rel(P.dalitz_norm(terms, cache), g[f"norm_{tag}"][0]) <= 1e-12


def test_dalitz_integral_cache_reuse(pf):
    ch = P.DecayChannel(*models.D_CHANNEL_T)
    _, pdf, terms = models.c3(grid=(64, 64))
    prior = pf.dalitz.compute_integrals(terms, ch, (64, 64))
    P.set_value(terms[1].magnitude, 2.5)
    assert pf.dalitz.compute_integrals(terms, ch, (64, 64), prior=prior) is prior
    m = P.Variable("mfloat", 0.9, 0.5, 1.3, step=0.001)
    terms[3].mass = m
    fresh = pf.dalitz.compute_integrals(terms, ch, (64, 64), prior=prior)
    scratch = pf.dalitz.compute_integrals(terms, ch, (64, 64))
    assert fresh.matrix[0, 0] == prior.matrix[0, 0]
    np.testing.assert_array_equal(fresh.matrix, scratch.matrix)
    spec_terms = [(t.pair, t.spin, t.mass.value, t.width.value, t.magnitude.value, t.phase.value) for t in terms]
    np.testing.assert_allclose(scratch.matrix, O.compute_integrals(spec_terms, models.D_CHANNEL_T, (64, 64)),
                               rtol=1e-12)


# --- invariances ------------------------------------------------------------------------


def test_warps_per_block_and_ranges_bitwise(pf):
    rng = np.random.default_rng(5)
    n = 37 * 4096 + 1111
    xs = np.clip(np.concatenate([rng.normal(5.0, 0.5, n // 2), rng.exponential(3.0, n - n // 2)]), 0, 10)
    x, pdf, _ = models.c1()
    ds = models.dataset([x], [xs])
    ctx = pf.device_context(0)
    ref = None
    for w in (1, 2, 4, 8):
        ctx.set_warps_per_block(w)
        got = pf.nll(pdf, ds)
        ref = got if ref is None else ref
        assert got == ref, w
    ctx.set_warps_per_block(0)
    assert rel(ref, O.nll(models.c1_spec((5.0, 0.5, -0.3, 0.3)), {"x": xs})) <= RTOL
    # multi-device style split of whole blocks reproduces the bits (host limb sum)
    snap = P.snapshot(pdf.param_closure())
    norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
    bs = pf.nll_block_sums(pdf, ds.columns(), snap, norms, 0, n)
    from paper_1710_08826_b200 import sharding

    assert sharding.round_acc(sharding.acc_of_values(bs)) == ref


def test_e2e_host_streaming_equals_device(pf):
    from paper_1710_08826_b200 import _lib as L

    rng = np.random.default_rng(9)
    n = 3_000_000 + 17
    xs = np.clip(rng.normal(5.0, 1.0, n), 0, 10)
    ys = np.clip(rng.exponential(2.5, n), 0, 10)
    (x, y), pdf, _ = models.c2()
    ds = models.dataset([x, y], [xs, ys])
    dev = pf.nll(pdf, ds)
    ctx = pf.device_context(0)
    plan = ctx.plan_for(pdf, ("x", "y"))
    vals, nv = plan.pack(None, P.resolve_norms(pdf, None, P.NormalizationStore()))
    cols = (L._DBL_P * 2)(L.dptr(ds.column("x")), L.dptr(ds.column("y")))
    out = ctypes.c_double()
    err = L.PfbErr()
    L.check(L.lib().pfb_nll_host(ctx.handle, plan.handle, cols, 2, n, L.dptr(vals), len(vals), L.dptr(nv),
                                 len(nv), ctypes.byref(out), ctypes.byref(err)), "pfb_nll_host")
    assert out.value == dev


def test_lineshape_cache_matches_recompute(pf, golden_dir):
    g = load(golden_dir, "c3_dalitz.npz")
    (s12, s13), pdf, terms = models.c3()
    ds = models.dataset([s12, s13], [g["s12"], g["s13"]])
    plain = pf.nll(pdf, ds)
    cached_backend = pf.DeviceBackend(lineshape_cache=1)
    got = pf.nll(pdf, ds, backend=cached_backend)
    assert rel(got, g["nll"][0]) <= RTOL
    assert rel(got, plain) <= 1e-12
    ctx = pf.device_context(0)
    plan = ctx.plan_for(pdf, ("s12", "s13"))
    before = plan.cache_recomputes()
    P.set_value(terms[1].magnitude, 0.8)  # coefficient move: no amplitude rows recomputed
    pf.nll(pdf, ds, backend=cached_backend)
    assert plan.cache_recomputes() == before
    plan.set_lineshape_cache(0)


# --- error semantics (reference engine.py:182-186, pdf.py:112-116,168-178) ----------------


def test_error_indices_match_reference(pf, golden_dir):
    with open(os.path.join(golden_dir, "errors.json")) as fh:
        cases = json.load(fh)
    x = P.Variable.observable("x", 0.0, 1.0)
    vals = np.full(5000, 0.5)
    vals[4321] = 0.0
    ds = models.dataset([x], [vals])
    with pytest.raises(P.errors.NonPositiveDensity) as e:
        pf.nll(P.polynomial(x, [0.0, 1.0]), ds)
    assert [type(e.value).__name__, e.value.index, e.value.value] == cases["poly_zero"]

    kind, idx, val, c, eps = cases["poly_dip_negative"]
    v3 = np.full(7000, 0.9)
    v3[6001] = c
    v3[6500] = c
    with pytest.raises(P.errors.NegativeDensity) as e:
        pf.nll(P.polynomial(x, [c * c - eps, -2.0 * c, 1.0]), models.dataset([x], [v3]))
    assert e.value.index == idx
    assert rel(e.value.value, val) <= 1e-6

    y = P.Variable.observable("y", 0.0, 10.0)
    g_ = P.gaussian(y, P.Variable("m", 5.0, fixed=True), P.Variable("s", 0.05, fixed=True))
    e_ = P.exponential(y, P.Variable("a", -0.2, fixed=True))
    tree = P.add_pdf([g_, e_], [P.Variable("f", 1.0, 0.0, 1.0)])
    v4 = np.full(6000, 5.0)
    v4[5555] = 9.9
    with pytest.raises(P.errors.NonPositiveDensity) as e:
        pf.nll(tree, models.dataset([y], [v4]))
    assert [type(e.value).__name__, e.value.index, e.value.value] == cases["sum_underflow"]

    z = P.Variable.observable("z")
    one = models.dataset([z], [np.array([0.0])])
    got = pf.nll(P.gaussian(z, P.Variable("mu", 0.0, fixed=True), P.Variable("sg", 1.0, fixed=True)), one)
    assert abs(got - 0.5 * math.log(2 * math.pi)) <= 1e-12
    with pytest.raises(P.errors.EmptyDataSet):
        pf.nll(P.gaussian(z, 0.0, 1.0), P.UnbinnedDataSet([z]))


def test_worker_error_index_in_third_block(pf):
    # reference tests/test_engine.py:106-114 (global index 9000)
    x = P.Variable.observable("x", 0.0, 1.0)
    values = np.full(4096 * 3, 0.5)
    values[9000] = 0.0
    with pytest.raises(P.errors.NonPositiveDensity) as err:
        pf.nll(P.polynomial(x, [0.0, 1.0]), models.dataset([x], [values]))
    assert err.value.index == 9000


# --- the reference's Backend protocol ---------------------------------------------------------


def test_backend_protocol_drop_in(pf, golden_dir):
    """Drive DeviceBackend exactly as the reference nll does (engine.py:235-243)."""
    g = load(golden_dir, "c1_sumpdf.npz")
    x, pdf, params = models.c1()
    ds = models.dataset([x], [g["x"]])
    backend = pf.DeviceBackend()
    snap = P.snapshot(pdf.param_closure())
    norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
    columns = {"x": ds.column("x")}
    ranges = backend.chunk_ranges(ds.n_events)
    chunks = backend.map(lambda *a: None, [(pdf, columns, snap, norms, a, b, backend.block) for a, b in ranges])
    sums = []
    for c in chunks:
        sums.extend(c.tolist())
    assert math.fsum(sums) == pf.nll(pdf, ds)
    assert rel(math.fsum(sums), g["nll"][0]) <= RTOL


# --- certification failures: the exact fix-up path behind every fast kernel -------


@pytest.mark.parametrize("alpha", [-40.0, 35.0])
def test_c1_uncertified_blocks_take_the_exact_fixup(pf, alpha):
    """|alpha x| >= 256 cannot be certified by the product-mode C1 evaluator:
    those blocks go to the literal fix-up launch, and the NLL still matches."""
    rng = np.random.default_rng(12)
    n = 9 * 4096 + 99
    xs = np.clip(np.concatenate([rng.normal(5.0, 0.5, n // 2), rng.uniform(0.0, 10.0, n - n // 2)]), 0, 10)
    x = P.Variable.observable("x", 0.0, 10.0)
    pdf = P.add_pdf([P.gaussian(x, P.Variable("mu", 5.0, 0.0, 10.0), P.Variable("sigma", 0.5, 0.01, 5.0)),
                      P.exponential(x, P.Variable("alpha", alpha, -50.0, 50.0))], [P.Variable("f", 0.3, 0.0, 1.0)])
    ds = models.dataset([x], [xs])
    ctx = pf.device_context(0)
    before = ctx.launch_count()
    got = pf.nll(pdf, ds)
    assert ctx.launch_count() - before == 2  # fast kernel + exact fix-up
    want = O.nll(models.c1_spec((5.0, 0.5, alpha, 0.3)), {"x": xs})
    assert rel(got, want) <= RTOL


def test_c2_uncertified_blocks_take_the_exact_fixup(pf):
    rng = np.random.default_rng(13)
    n = 7 * 4096 + 5
    xs = np.clip(rng.normal(5.0, 1.0, n), 0, 10)
    xs[::3000] = 0.05  # u ~ -725 at sigma = 0.13: beyond the log-domain guard (subnormal in the reference)
    ys = np.clip(rng.exponential(2.5, n), 0, 10)
    (x, y), pdf, _ = models.c2((5.0, 0.13, -0.4))
    ds = models.dataset([x, y], [xs, ys])
    ctx = pf.device_context(0)
    before = ctx.launch_count()
    got = pf.nll(pdf, ds)
    assert ctx.launch_count() - before == 2
    assert rel(got, O.nll(models.c2_spec((5.0, 0.13, -0.4)), {"x": xs, "y": ys})) <= RTOL


def test_c1_narrow_pure_gaussian_far_tails(pf):
    """Densities down to ~2^-290 (a narrow pure gaussian, f = 1, over a wide
    range): whichever kernel the plan takes, the NLL equals the reference's."""
    rng = np.random.default_rng(23)
    n = 6 * 4096 + 17
    xs = np.concatenate([rng.normal(5.0, 0.1, n - 2000), rng.uniform(3.0, 7.0, 2000)])
    rng.shuffle(xs)
    xs = np.clip(xs, 0.0, 10.0)
    point = (5.0, 0.1, -0.3, 1.0)
    x, pdf, _ = models.c1(point)
    ds = models.dataset([x], [xs])
    got = pf.nll(pdf, ds)
    want = O.nll(models.c1_spec(point), {"x": xs})
    assert rel(got, want) <= RTOL


def test_c1_product_shells_bitwise_above_the_tma_threshold(pf):
    """C1 at 20M events (above the 24 blocks per SM where pipeline 1 moves
    the one-column SumPdf onto the TMA unit kernel): pipeline 1, bulk
    prefetch (2) and warp tasks (4) give the same bits; the log-domain SIMT
    kernel (0) agrees within 1e-12."""
    x, pdf, params = models.c1()
    rng = np.random.default_rng(12)
    n = 20_000_000 + 333
    xs = np.clip(np.concatenate([rng.normal(5, 0.5, n // 3), rng.exponential(3.3, n - n // 3)]), 0, 10)
    ds = models.dataset([x], [xs])
    ctx = pf.device_context(0)
    got = {}
    try:
        for mode in (1, 2, 4, 0):
            ctx.set_pipeline(mode)
            got[mode] = pf.nll(pdf, ds)
    finally:
        ctx.set_pipeline(1)
    assert got[1] == got[2] == got[4]
    assert rel(got[1], got[0]) <= 1e-12
