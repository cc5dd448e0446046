"""PDF tree -> flat post-order node table for the device (pfb_plan_compile).

Replaces the reference's recursive KIND_OPS dispatch (pdf.py:234-269) with a
table the CUDA kernel reads from its constant bank.  Works on any duck-typed
tree with the reference's PdfNode shape (kind, observables, parameters,
children, payload), so nodes built by the reference package and by this one
compile alike.  The native compiler then picks an evaluator: the log-domain
sum-of-products fast path for add/prod trees of gaussian/exponential/
polynomial leaves, the Dalitz evaluator for a Dalitz root, else the literal
interpreter.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


class UnsupportedNode(NotImplementedError):
    """A node kind without a device kernel (custom register_kind extensions)."""


@dataclass
class TreeLayout:
    nodes: list                    # post-order node objects
    params: list                   # Variables, concatenated in node order
    column_names: tuple[str, ...]  # store column order
    table: object = None           # ctypes array of PfbNode
    dalitz: object = None          # ctypes array of PfbDalitzDesc
    ndalitz: int = 0
    dalitz_nodes: list = field(default_factory=list)


def layout(pdf, column_names) -> TreeLayout:
    """Post-order node table with store column indices."""
    nodes = list(pdf.walk())
    col_index = {name: i for i, name in enumerate(column_names)}
    table = (L.PfbNode * len(nodes))()
    descs = []
    params = []
    dal_nodes = []
    for i, node in enumerate(nodes):
        code = L.KIND_CODES.get(node.kind)
        if code is None:
            raise UnsupportedNode(f"node kind {node.kind!r} has no device kernel")
        rec = table[i]
        rec.kind = code
        rec.nchild = len(node.children)
        names = [o.name for o in node.observables]
        leaf = node.kind not in ("add", "prod")
        rec.col0 = col_index[names[0]] if leaf else -1
        rec.col1 = col_index[names[1]] if node.kind == "dalitz" else -1
        rec.nparam = len(node.parameters)
        rec.aux = 0
        if node.kind == "dalitz":
            terms, ch, _grid = node.payload
            if len(terms) > L.PFB_MAX_DALITZ_TERMS:
                raise UnsupportedNode(f"dalitz node with {len(terms)} terms (max {L.PFB_MAX_DALITZ_TERMS})")
            d = L.PfbDalitzDesc()
            d.mother_mass, d.m1, d.m2, d.m3 = ch.mother_mass, ch.m1, ch.m2, ch.m3
            d.nterms = len(terms)
            for k, t in enumerate(terms):
                d.pair[k] = int(t.pair)
                d.spin[k] = int(t.spin)
            rec.aux = len(descs)
            descs.append(d)
            dal_nodes.append(node)
        params.extend(node.parameters)
    out = TreeLayout(nodes=nodes, params=params, column_names=tuple(column_names), table=table)
    if descs:
        arr = (L.PfbDalitzDesc * len(descs))(*descs)
        out.dalitz = arr
        out.ndalitz = len(descs)
        out.dalitz_nodes = dal_nodes
    return out


class Plan:
    """A compiled plan bound to one device context."""

    def __init__(self, ctx, tree: TreeLayout):
        self.ctx = ctx
        self.tree = tree
        handle = ctypes.c_void_p()
        dal = tree.dalitz if tree.dalitz is not None else None
        L.check(
            L.lib().pfb_plan_compile(ctx.handle, tree.table, len(tree.nodes), dal, tree.ndalitz,
                                     ctypes.byref(handle)),
            "pfb_plan_compile",
        )
        self.handle = handle
        self.nvalues = len(tree.params)
        self.nnodes = len(tree.nodes)
        self._values = np.empty(self.nvalues, dtype=np.float64)
        self._norms = np.empty(self.nnodes, dtype=np.float64)
        # pointers to the two per-call buffers, made once (a ctypes cast per
        # call costs ~1 us each on the fit's critical path)
        self.values_ptr = L.dptr(self._values)
        self.norms_ptr = L.dptr(self._norms)
        self._slot_names = None
        self._slots: list = []

    @property
    def evaluator(self) -> str:
        out = ctypes.c_int32()
        L.check(L.lib().pfb_plan_evaluator(self.handle, ctypes.byref(out)), "pfb_plan_evaluator")
        return L.EVALUATORS.get(out.value, str(out.value))

    def set_lineshape_cache(self, mode: int) -> None:
        L.check(L.lib().pfb_plan_set_lineshape_cache(self.handle, int(mode)), "pfb_plan_set_lineshape_cache")

    def cache_recomputes(self) -> int:
        out = ctypes.c_int64()
        L.check(L.lib().pfb_plan_cache_recomputes(self.handle, ctypes.byref(out)), "pfb_plan_cache_recomputes")
        return out.value

    def pack(self, snap, norms) -> tuple[np.ndarray, np.ndarray]:
        """This call's raw parameter values and per-node norms (post-order)."""
        vals = self._values
        params = self.tree.params
        if snap is None:
            for i, v in enumerate(params):
                vals[i] = v.value
        else:
            if snap.names != self._slot_names:
                index = {}
                for k, name in enumerate(snap.names):
                    index.setdefault(name, k)
                self._slots = [index.get(v.name) for v in params]
                self._slot_names = snap.names
            svals = snap.values
            for i, k in enumerate(self._slots):
                vals[i] = svals[k] if k is not None else params[i].value
        nv = self._norms
        for i, node in enumerate(self.tree.nodes):
            nv[i] = norms[node.id]
        return vals, nv

    def pack_batch(self, snaps, norms_list) -> tuple[np.ndarray, np.ndarray]:
        """Rows of raw values and norms for several parameter points."""
        vals = np.empty((len(snaps), self.nvalues), dtype=np.float64)
        nv = np.empty((len(snaps), self.nnodes), dtype=np.float64)
        for m, (snap, norms) in enumerate(zip(snaps, norms_list)):
            v, n = self.pack(snap, norms)
            vals[m] = v
            nv[m] = n
        return vals, nv

    def close(self) -> None:
        if self.handle:
            L.lib().pfb_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
