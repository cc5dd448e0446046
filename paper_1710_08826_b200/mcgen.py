"""Toy event generation.

* generate_1d / generate_dalitz: the reference's generators (P/mcgen.py:58-257,
  taking the reference's model nodes and ``GenSpec``) on the GPU, stream for
  stream: the same numpy PCG64 streams (SeedSequence spawning), the same
  chunked accept-reject, the same envelope / rescan / budget semantics -> the
  same events (pfb_pcg_*), returned as a :class:`~.datasets.DeviceDataSet`
  whose HBM copy is the generated store.
* device_*: fast Philox-based samplers for benchmark inputs (pfb_gen_*).
* sumpdf_1d / prod_2d / dalitz: host numpy samplers for small test inputs.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from .datasets import DeviceDataSet


def truncated_gaussian(n: int, mu: float, sigma: float, lo: float, hi: float, rng) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    got = 0
    while got < n:
        k = int((n - got) * 1.2) + 1024
        v = rng.normal(mu, sigma, k)
        v = v[(v >= lo) & (v <= hi)]
        take = min(len(v), n - got)
        out[got:got + take] = v[:take]
        got += take
    return out


def truncated_exponential(n: int, alpha: float, lo: float, hi: float, rng) -> np.ndarray:
    """Inverse CDF of exp(alpha x) on [lo, hi]."""
    u = rng.random(n)
    if alpha == 0.0:
        return lo + (hi - lo) * u
    a, b = math.exp(alpha * lo), math.exp(alpha * hi)
    x = np.log(a + u * (b - a)) / alpha
    return np.clip(x, lo, hi)


def sumpdf_1d(n: int, mu: float, sigma: float, alpha: float, f: float, lo: float, hi: float, seed: int):
    """C1 / C5: f * Gauss + (1 - f) * Exp on [lo, hi]."""
    rng = np.random.default_rng(seed)
    ng = int(rng.binomial(n, f))
    x = np.concatenate([truncated_gaussian(ng, mu, sigma, lo, hi, rng),
                        truncated_exponential(n - ng, alpha, lo, hi, rng)])
    rng.shuffle(x)
    return x


def prod_2d(n: int, mu: float, sigma: float, alpha: float, lo: float, hi: float, seed: int):
    """C2: x ~ Gauss(mu, sigma), y ~ Exp(alpha), independent, on [lo, hi]^2."""
    rng = np.random.default_rng(seed)
    return truncated_gaussian(n, mu, sigma, lo, hi, rng), truncated_exponential(n, alpha, lo, hi, rng)


def _boundary(s12, s13, M, m1, m2, m3):
    with np.errstate(invalid="ignore", divide="ignore"):
        rs = np.sqrt(s12)
        e1 = (s12 + m1 * m1 - m2 * m2) / (2.0 * rs)
        e3 = (M * M - s12 - m3 * m3) / (2.0 * rs)
        p1 = np.sqrt(e1 * e1 - m1 * m1)
        p3 = np.sqrt(e3 * e3 - m3 * m3)
        es = (e1 + e3) ** 2
        return (s13 >= es - (p1 + p3) ** 2) & (s13 <= es - (p1 - p3) ** 2)


def _intensity(terms, s12, s13, M, m1, m2, m3):
    mss = M * M + m1 * m1 + m2 * m2 + m3 * m3
    s23 = mss - s12 - s13
    tot = 0j
    for pair, spin, m, w, mag, ph in terms:
        s = s12 if pair == 12 else (s13 if pair == 13 else s23)
        a = 1.0 / (m * m - s - 1j * m * w)
        if spin == 1:
            if pair == 12:
                z = s13 - s23 + (M * M - m3 * m3) * (m2 * m2 - m1 * m1) / s12
            elif pair == 13:
                z = s12 - s23 + (M * M - m2 * m2) * (m3 * m3 - m1 * m1) / s13
            else:
                z = s12 - s13 + (M * M - m1 * m1) * (m3 * m3 - m2 * m2) / s23
            a = a * z
        tot = tot + mag * np.exp(1j * ph) * a
    return (tot * np.conj(tot)).real


def dalitz(n: int, terms, channel, seed: int, chunk: int = 1 << 22):
    """Accept-reject over the (s12, s13) box; terms = [(pair, spin, m, w, mag, phase)]."""
    M, m1, m2, m3 = channel
    lo12, hi12 = (m1 + m2) ** 2, (M - m3) ** 2
    lo13, hi13 = (m1 + m3) ** 2, (M - m2) ** 2
    rng = np.random.default_rng(seed)
    g12 = lo12 + (np.arange(512) + 0.5) * (hi12 - lo12) / 512
    g13 = lo13 + (np.arange(512) + 0.5) * (hi13 - lo13) / 512
    G12, G13 = np.meshgrid(g12, g13, indexing="ij")
    inside = _boundary(G12, G13, M, m1, m2, m3)
    env = 1.2 * float(_intensity(terms, G12[inside], G13[inside], M, m1, m2, m3).max())
    a12, a13 = np.empty(n), np.empty(n)
    got = 0
    while got < n:
        c12 = rng.uniform(lo12, hi12, chunk)
        c13 = rng.uniform(lo13, hi13, chunk)
        ok = _boundary(c12, c13, M, m1, m2, m3)
        c12, c13 = c12[ok], c13[ok]
        keep = rng.uniform(0.0, env, len(c12)) < _intensity(terms, c12, c13, M, m1, m2, m3)
        c12, c13 = c12[keep], c13[keep]
        take = min(len(c12), n - got)
        a12[got:got + take] = c12[:take]
        a13[got:got + take] = c13[:take]
        got += take
    return a12, a13


# --- device generation (libpfb200: pfb_gen_1d / pfb_gen_dalitz) -------------------------


def _device_store(ctx, ncols: int, n: int):
    import ctypes

    from . import _lib as L

    st = ctypes.c_void_p()
    L.check(L.lib().pfb_store_create(ctx.handle, ncols, n, ctypes.byref(st)), "pfb_store_create")
    return st


def _adopt(ctx, st, ncols: int, n: int, observables=None):
    """Download the generated columns and register the device store as the
    HBM copy of those host arrays (no re-upload when the NLL runs).  With
    `observables`, the dataset's strict range check (reference core.py:262-272)
    runs on the device copy first."""
    from . import _lib as L
    from ._reference import errors as E

    OutOfRange = E.OutOfRange

    if observables is not None:
        for c, obs in enumerate(observables):
            bad = ctypes.c_int64()
            val = ctypes.c_double()
            code = L.lib().pfb_store_check_range(st, c, 0, n, float(obs.lower), float(obs.upper),
                                                 ctypes.byref(bad), ctypes.byref(val))
            if code or bad.value >= 0:
                L.lib().pfb_store_destroy(st)
                L.check(code, "pfb_store_check_range")
                raise OutOfRange(c, float(val.value), obs.name)
    cols = []
    for c in range(ncols):
        a = np.empty(n, dtype=np.float64)
        L.check(L.lib().pfb_store_download(st, c, L.dptr(a), 0, n), "pfb_store_download")
        cols.append(a)
    ctx.adopt(cols, st)
    return cols


def device_sumpdf_1d(n, mu, sigma, alpha, f, lo, hi, seed, ctx=None):
    """C1 / C5 events generated on the GPU: f * Gauss + (1 - f) * Exp on [lo, hi]."""
    from . import _lib as L
    from .engine import device_context

    ctx = ctx or device_context(0)
    st = _device_store(ctx, 1, n)
    L.check(L.lib().pfb_gen_1d(ctx.handle, 0, mu, sigma, alpha, f, lo, hi, seed, n, st), "pfb_gen_1d")
    return _adopt(ctx, st, 1, n)[0]


def device_prod_2d(n, mu, sigma, alpha, lo, hi, seed, ctx=None):
    """C2 events generated on the GPU: Gauss(x) x Exp(y) on [lo, hi]^2."""
    from . import _lib as L
    from .engine import device_context

    ctx = ctx or device_context(0)
    st = _device_store(ctx, 2, n)
    L.check(L.lib().pfb_gen_1d(ctx.handle, 1, mu, sigma, alpha, 0.0, lo, hi, seed, n, st), "pfb_gen_1d")
    return tuple(_adopt(ctx, st, 2, n))


def dalitz_envelope(terms, channel, safety: float = 1.2, points: int = 512) -> float:
    """safety x the largest intensity on a points^2 midpoint scan (reference mcgen.py:180-181)."""
    M, m1, m2, m3 = channel
    lo12, hi12 = (m1 + m2) ** 2, (M - m3) ** 2
    lo13, hi13 = (m1 + m3) ** 2, (M - m2) ** 2
    g12 = lo12 + (np.arange(points) + 0.5) * (hi12 - lo12) / points
    g13 = lo13 + (np.arange(points) + 0.5) * (hi13 - lo13) / points
    G12, G13 = np.meshgrid(g12, g13, indexing="ij")
    inside = _boundary(G12, G13, M, m1, m2, m3)
    return safety * float(_intensity(terms, G12[inside], G13[inside], M, m1, m2, m3).max())


def device_dalitz(n, terms, channel, seed, ctx=None, envelope=None):
    """Dalitz events generated on the GPU; terms = [(pair, spin, m, w, mag, phase)]."""
    import ctypes

    from . import _lib as L
    from .engine import device_context

    ctx = ctx or device_context(0)
    d = L.PfbDalitzDesc()
    d.mother_mass, d.m1, d.m2, d.m3 = channel
    d.nterms = len(terms)
    vals = np.zeros(4 * len(terms))
    for k, (pair, spin, m, w, mag, ph) in enumerate(terms):
        d.pair[k], d.spin[k] = int(pair), int(spin)
        vals[4 * k:4 * k + 4] = (m, w, mag, ph)
    env = envelope if envelope is not None else dalitz_envelope(terms, channel)
    st = _device_store(ctx, 2, n)
    cand = ctypes.c_int64()
    L.check(L.lib().pfb_gen_dalitz(ctx.handle, ctypes.byref(d), L.dptr(vals), env, seed, n, st, ctypes.byref(cand)),
            "pfb_gen_dalitz")
    return tuple(_adopt(ctx, st, 2, n))


# --- the reference generators, stream-exact on the GPU ------------

SCAN_POINTS = 4096  # mcgen.py:29-31
RESCAN_POINTS = 4 * SCAN_POINTS
CHUNK = 8192


from ._reference import mcgen as _ref_mcgen  # noqa: E402

GenSpec = _ref_mcgen.GenSpec  # the reference's spec (P/mcgen.py:34-50)


def _stream_states(spec):
    """PCG64 states of SeedSequence(seed).spawn(streams) (mcgen.py:57-59)."""
    from . import _lib as L

    out = []
    for child in np.random.SeedSequence(spec.seed).spawn(spec.streams):
        st = np.random.PCG64(child).state["state"]
        s, inc = int(st["state"]), int(st["inc"])
        p = L.PfbPcg64()
        p.state_hi, p.state_lo = s >> 64, s & ((1 << 64) - 1)
        p.inc_hi, p.inc_lo = inc >> 64, inc & ((1 << 64) - 1)
        out.append(p)
    return out


def _split_counts(total: int, parts: int) -> list[int]:
    base, extra = divmod(total, parts)
    return [base + (1 if k < extra else 0) for k in range(parts)]


class _EnvelopeHit(Exception):
    def __init__(self, observed: float):
        self.observed = observed


def _run_streams(spec, budget, gen_one, stats, dalitz: bool):
    """The per-stream loop of _generate_streams / _dalitz_streams: events of
    stream i follow those of stream i-1."""
    from . import _lib as L
    from ._reference import errors as E

    AttemptsExhausted = E.AttemptsExhausted

    states = _stream_states(spec)
    counts = _split_counts(spec.n_events, spec.streams)
    budgets = _split_counts(budget, spec.streams)
    offset = 0
    for state, cnt, bud in zip(states, counts, budgets):
        if cnt <= 0:
            continue
        gs = L.PfbGenStats()
        code = gen_one(state, cnt, bud, offset, gs)
        if dalitz:
            stats["box_draws"] = stats.get("box_draws", 0) + gs.attempts
            stats["in_boundary_draws"] = stats.get("in_boundary_draws", 0) + gs.in_boundary
        if code == L.E_ENVELOPE_HIT:
            raise _EnvelopeHit(gs.observed)
        if code == L.E_ATTEMPTS_EXHAUSTED:
            if dalitz:
                raise AttemptsExhausted(f"{gs.attempts} draws produced only {gs.produced}/{cnt} events in one stream")
            raise AttemptsExhausted(f"{gs.attempts} draws produced only {gs.produced}/{cnt} events")
        L.check(code, "pfb_pcg_generate")
        if not dalitz:
            stats["attempts"] = stats.get("attempts", 0) + gs.attempts
        stats["accepted"] = stats.get("accepted", 0) + gs.accepted
        # decisions within 2^-47 of the density (0: the reference's sample bit for bit)
        stats["ambiguous"] = stats.get("ambiguous", 0) + gs.ambiguous
        offset += cnt


def generate_1d(pdf, obs, spec, stats: dict | None = None, device: int = 0):
    """Reference generate_1d (mcgen.py:108-153) on the GPU: the same events
    for the same spec (see pfb_pcg.cu for the one caveat)."""
    from . import _lib as L
    from ._reference import errors as E
    from ._reference import pdf as ref_pdf
    from .engine import device_context

    EnvelopeExceeded, UnboundedObservable, normalize = E.EnvelopeExceeded, E.UnboundedObservable, ref_pdf.normalize

    lo, hi = obs.lower, obs.upper
    if not (math.isfinite(lo) and math.isfinite(hi)):
        raise UnboundedObservable(f"{obs.name!r} needs finite bounds for generation")
    norms = {n.id: normalize(n).value for n in pdf.walk() if n is not pdf} if pdf.children else {}
    norms[pdf.id] = 1.0  # eval_batch returns the unnormalised root density
    ctx = device_context(device)
    plan = ctx.plan_for(pdf, (obs.name,))
    vals, nv = plan.pack(None, norms)
    vals, nv = vals.copy(), nv.copy()

    def scan(points):
        out = ctypes.c_double()
        L.check(L.lib().pfb_pcg_scan_1d(ctx.handle, plan.handle, L.dptr(vals), len(vals), L.dptr(nv), len(nv),
                                        lo, hi, points, ctypes.byref(out)), "pfb_pcg_scan_1d")
        return out.value

    envelope = spec.envelope_safety * scan(SCAN_POINTS)
    budget = spec.max_attempts_factor * spec.n_events
    stats = stats if stats is not None else {}
    st = _device_store(ctx, 1, spec.n_events)
    for attempt in range(2):
        try:
            stats.clear()
            stats["envelope"] = envelope

            def one(state, cnt, bud, offset, gs, env=envelope):
                return L.lib().pfb_pcg_generate_1d(ctx.handle, plan.handle, L.dptr(vals), len(vals), L.dptr(nv),
                                                   len(nv), lo, hi, env, ctypes.byref(state), cnt, bud, st, offset,
                                                   ctypes.byref(gs))

            _run_streams(spec, budget, one, stats, dalitz=False)
            break
        except _EnvelopeHit as hit:
            if attempt == 1:
                L.lib().pfb_store_destroy(st)
                raise EnvelopeExceeded(f"density {hit.observed} exceeded envelope {envelope} after a rescan") from None
            envelope = spec.envelope_safety * max(scan(RESCAN_POINTS), hit.observed)
    col = _adopt(ctx, st, 1, spec.n_events, [obs])[0]
    return DeviceDataSet.adopt_store([obs], [col])


def generate_dalitz(terms, ch, spec, observables=None, stats: dict | None = None, device: int = 0):
    """Reference generate_dalitz (mcgen.py:155-199) on the GPU: flat phase
    space over the (s12, s13) box, boundary filter, intensity accept-reject."""
    from . import _lib as L
    from ._reference import core as ref_core
    from ._reference import errors as E
    from .engine import device_context

    EnvelopeExceeded, Variable = E.EnvelopeExceeded, ref_core.Variable

    if not terms:
        raise ValueError("need at least one resonance term")
    if observables is None:
        observables = (Variable.observable("s12", *ch.s12_range), Variable.observable("s13", *ch.s13_range))
    d = L.PfbDalitzDesc()
    d.mother_mass, d.m1, d.m2, d.m3 = ch.mother_mass, ch.m1, ch.m2, ch.m3
    d.nterms = len(terms)
    vals = np.zeros(4 * len(terms))
    for k, t in enumerate(terms):
        d.pair[k], d.spin[k] = int(t.pair), int(t.spin)
        vals[4 * k:4 * k + 4] = (t.mass.value, t.width.value, t.magnitude.value, t.phase.value)
    ctx = device_context(device)

    def scan(n):
        out = ctypes.c_double()
        L.check(L.lib().pfb_pcg_scan_dalitz(ctx.handle, ctypes.byref(d), L.dptr(vals), n, ctypes.byref(out)),
                "pfb_pcg_scan_dalitz")
        return out.value

    envelope = spec.envelope_safety * scan(512)
    budget = spec.max_attempts_factor * spec.n_events
    stats = stats if stats is not None else {}
    st = _device_store(ctx, 2, spec.n_events)
    for attempt in range(2):
        try:
            stats.clear()
            stats["envelope"] = envelope

            def one(state, cnt, bud, offset, gs, env=envelope):
                return L.lib().pfb_pcg_generate_dalitz(ctx.handle, ctypes.byref(d), L.dptr(vals), env,
                                                       ctypes.byref(state), cnt, bud, st, offset, ctypes.byref(gs))

            _run_streams(spec, budget, one, stats, dalitz=True)
            break
        except _EnvelopeHit as hit:
            if attempt == 1:
                L.lib().pfb_store_destroy(st)
                raise EnvelopeExceeded(
                    f"intensity {hit.observed} exceeded envelope {envelope} after a rescan") from None
            envelope = spec.envelope_safety * max(scan(2048), hit.observed)
    s12, s13 = _adopt(ctx, st, 2, spec.n_events, list(observables))
    return DeviceDataSet.adopt_store(list(observables), [s12, s13])
