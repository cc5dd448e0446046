"""Device normalisation integrals behind the reference's norm cache.

The reference caches every node's normalisation on its parameters'
generations (``cached_norm``, P/engine.py:138-159) and lets a kind supply its
own cached strategy through ``register_cached_norm`` (P/engine.py:131-135).
This module registers device hooks there, so the integrals are recomputed on
the GPU -- and only when the node's parameters changed (the reference cache
decides; north_star item 4):

* ``"polynomial"`` -- the composite Gauss-Legendre integral of
  ``_polynomial_norm`` (P/pdf.py:181-199): the reference's own abscissas and
  weights (``gauss_legendre_points``, uploaded once per box and stored next
  to each other in one HBM store), the density by the device's literal
  evaluator (numpy's Horner order), sum_j w_j f(x_j) as the correctly rounded
  dot product (:func:`quadrature`, pfb_quadrature).  Errors as the reference:
  ``UnboundedObservable`` for an infinite box, ``NegativeDensity`` /
  ``NonFiniteDensity`` with the abscissa index.
* ``"dalitz"`` -- the overlap integrals over the midpoint grid (:mod:`.dalitz`).
* optionally (``grid_kinds``) ``"gaussian"`` / ``"exponential"``: the same
  device quadrature over the node's box in place of the closed forms
  (P/pdf.py:130-161); agrees with them to ~1e-15 (tests), but is not the
  reference's arithmetic, so it is opt-in.

Counters follow the reference: a hook recompute of a leaf integral adds 1 to
``store.kernel_evals`` (the reference's ``cached_norm`` does that for
non-hook leaves, P/engine.py:153-154), a Dalitz refresh the number of changed
terms (P/dalitz.py:400-409); ``norm_computations``/``recompute_counts`` are
the reference cache's own.

:func:`install` registers the hooks (globally, like the reference registering
its own at import); :func:`reference_norms` temporarily restores the
reference's hooks (parity checks compute the reference side under it).
"""

from __future__ import annotations

import contextlib
import ctypes
import math

import numpy as np

from . import _lib as L
from ._reference import engine as ref_engine
from ._reference import errors as ref_errors
from ._reference import pdf as ref_pdf

GL_NODES = ref_pdf.GL_NODES_DEFAULT
GL_PANELS = ref_pdf.GL_PANELS_DEFAULT


class _Rule:
    """Abscissas (one column per axis) and weights of a tensor-product rule,
    resident in HBM as one store [x_0, ..., x_{d-1}, w] owned by the context
    (outside its bounded cache of data stores)."""

    def __init__(self, ctx, axes):
        self.ctx = ctx
        pts, wts = [], []
        for lo, hi, nodes, panels in axes:
            x, w = ref_pdf.gauss_legendre_points(lo, hi, nodes, panels)
            pts.append(np.asarray(x, dtype=np.float64))
            wts.append(np.asarray(w, dtype=np.float64))
        if len(axes) == 1:
            cols, weights = [pts[0]], wts[0]
        else:
            mesh = np.meshgrid(*pts, indexing="ij")
            cols = [m.reshape(-1) for m in mesh]
            weights = wts[0]
            for w in wts[1:]:
                weights = np.multiply.outer(weights, w)
            weights = weights.reshape(-1)
        self.n = len(weights)
        self.ncols = len(axes)
        columns = [np.ascontiguousarray(c) for c in cols] + [np.ascontiguousarray(weights)]
        st = ctypes.c_void_p()
        L.check(L.lib().pfb_store_create(ctx.handle, len(columns), self.n, ctypes.byref(st)), "pfb_store_create")
        for c, a in enumerate(columns):
            L.check(L.lib().pfb_store_upload(st, c, L.dptr(a), 0, self.n), "pfb_store_upload")
        self.store = st

    def close(self) -> None:
        if self.store:
            L.lib().pfb_store_destroy(self.store)
            self.store = None


def _rule(ctx, axes) -> _Rule:
    key = ("gl-rule", tuple(axes))
    r = ctx.grids.get(key)
    if r is None:
        r = _Rule(ctx, axes)
        ctx.grids[key] = r
    return r


def quadrature_handles(node, nodes: int = GL_NODES, panels: int = GL_PANELS, ctx=None):
    """(plan, rule) of the device quadrature of `node` alone -- what the C
    objective launches when the node's parameters move (PFB_NORM_QUADRATURE)."""
    from .engine import device_context

    ctx = ctx or device_context(0)
    obs = node.observables
    for o in obs:
        if math.isinf(o.lower) or math.isinf(o.upper):
            raise ref_errors.UnboundedObservable(f"{node.kind} normalization needs finite bounds")
    rule = _rule(ctx, [(o.lower, o.upper, int(nodes), int(panels)) for o in obs])
    plan = ctx.plan_for(node, tuple(o.name for o in obs) + ("__weights__",))
    return plan, rule


def quadrature(node, snap=None, child_norms=None, nodes: int = GL_NODES, panels: int = GL_PANELS, ctx=None) -> float:
    """Integral of `node`'s unnormalised density over its observables' box by
    the composite Gauss-Legendre rule (tensor product over the axes), on the
    GPU.  Children of add/prod nodes enter normalised by `child_norms`
    (node.id -> value; default: the reference's uncached ``normalize``)."""
    from .engine import device_context, raise_for

    ctx = ctx or device_context(0)
    obs = node.observables
    for o in obs:
        if math.isinf(o.lower) or math.isinf(o.upper):
            raise ref_errors.UnboundedObservable(f"{node.kind} normalization needs finite bounds")
    rule = _rule(ctx, [(o.lower, o.upper, int(nodes), int(panels)) for o in obs])
    names = tuple(o.name for o in obs) + ("__weights__",)
    plan = ctx.plan_for(node, names)
    norms = {}
    if node.children:
        if child_norms is None:
            child_norms = {n.id: ref_pdf.normalize(n, snap).value for n in node.walk() if n is not node}
        norms.update(child_norms)
    norms[node.id] = 1.0
    vals, nv = plan.pack(snap, norms)
    out = ctypes.c_double()
    err = L.PfbErr()
    code = L.lib().pfb_quadrature(ctx.handle, plan.handle, rule.store, rule.ncols, L.dptr(vals), len(vals),
                                  L.dptr(nv), len(nv), ctypes.byref(out), ctypes.byref(err))
    raise_for(err, code, "pfb_quadrature")
    return out.value


# --- hooks -------------------------------------------------------------------------------

_device = {"index": 0}


def _ctx():
    from .engine import device_context

    return device_context(_device["index"])


def polynomial_cached_norm(node, snap, store) -> float:
    """Device ``_polynomial_norm`` (P/pdf.py:192-199) as a cached-norm hook."""
    nodes, panels = node.payload
    value = quadrature(node, snap, None, nodes, panels, ctx=_ctx())
    store.kernel_evals += 1
    return value


def leaf_grid_cached_norm(node, snap, store) -> float:
    """Device quadrature for a gaussian / exponential leaf (opt-in grid mode)."""
    value = quadrature(node, snap, None, GL_NODES, GL_PANELS, ctx=_ctx())
    store.kernel_evals += 1
    return value


def dalitz_cached_norm(node, snap, store) -> float:
    from . import dalitz

    return dalitz.dalitz_cached_norm(node, snap, store)


_saved: dict[str, object] = {}
_SENTINEL = object()


def install(device: int = 0, grid_kinds=()) -> None:
    """Register the device hooks in the reference's CACHED_NORM_HOOKS."""
    hooks = {"polynomial": polynomial_cached_norm, "dalitz": dalitz_cached_norm}
    for kind in grid_kinds:
        if kind not in ("gaussian", "exponential"):
            raise ValueError(f"no device grid norm for kind {kind!r}")
        hooks[kind] = leaf_grid_cached_norm
    _device["index"] = int(device)
    for kind, hook in hooks.items():
        if kind not in _saved:
            _saved[kind] = ref_engine.CACHED_NORM_HOOKS.get(kind, _SENTINEL)
        ref_engine.register_cached_norm(kind, hook)


def uninstall() -> None:
    """Restore the reference's own hooks."""
    for kind, hook in _saved.items():
        if hook is _SENTINEL:
            ref_engine.CACHED_NORM_HOOKS.pop(kind, None)
        else:
            ref_engine.register_cached_norm(kind, hook)
    _saved.clear()


def installed() -> bool:
    return bool(_saved)


@contextlib.contextmanager
def _restoring():
    """Restore the registry and this module's bookkeeping on exit."""
    hooks = dict(ref_engine.CACHED_NORM_HOOKS)
    saved = dict(_saved)
    device = _device["index"]
    try:
        yield
    finally:
        ref_engine.CACHED_NORM_HOOKS.clear()
        ref_engine.CACHED_NORM_HOOKS.update(hooks)
        _saved.clear()
        _saved.update(saved)
        _device["index"] = device


@contextlib.contextmanager
def reference_norms():
    """Run a block with the reference's own normalisation hooks."""
    with _restoring():
        uninstall()
        yield


@contextlib.contextmanager
def device_norms(device: int = 0, grid_kinds=()):
    """Run a block with the device hooks installed (plus `grid_kinds`)."""
    with _restoring():
        install(device, grid_kinds)
        yield
