"""Host logic of Plan.pack (no GPU): the cached snapshot-name -> slot map must
give the same values as the reference's ParameterSnapshot.value_of
(P/core.py ParameterSnapshot; first occurrence of a name wins, variables
outside the snapshot read their live value) and must follow a change of the
snapshot's name set instead of reusing a stale map."""

import types

import numpy as np

from paper_1710_08826_b200._reference import core as _core

ParameterSnapshot, Variable = _core.ParameterSnapshot, _core.Variable
from paper_1710_08826_b200.plan import Plan


def _bare_plan(params, node_ids):
    p = Plan.__new__(Plan)
    p.tree = types.SimpleNamespace(params=params, nodes=[types.SimpleNamespace(id=i) for i in node_ids])
    p._values = np.empty(len(params), dtype=np.float64)
    p._norms = np.empty(len(node_ids), dtype=np.float64)
    p._slot_names = None
    p._slots = []
    p.handle = None
    return p


def _expect(params, snap):
    return [snap.value_of(v) if snap is not None else v.value for v in params]


def test_pack_follows_snapshot_name_changes():
    a = Variable("a", 1.0, -10, 10)
    b = Variable("b", 2.0, -10, 10)
    c = Variable("c", 3.0, -10, 10)
    params = [a, b, c]
    plan = _bare_plan(params, [7, 9])
    norms = {7: 0.5, 9: 4.0}
    snaps = [
        ParameterSnapshot(("a", "b", "c"), (1.5, 2.5, 3.5), (1, 1, 1)),
        ParameterSnapshot(("a", "b", "c"), (1.25, 2.25, 3.25), (2, 2, 2)),  # same names: cached map
        ParameterSnapshot(("c", "a"), (30.0, 10.0), (1, 1)),  # new order, b live
        ParameterSnapshot(("b", "b", "a"), (20.0, 21.0, 11.0), (1, 1, 1)),  # duplicate: first wins
        None,
        ParameterSnapshot(("a", "b", "c"), (0.5, 0.25, 0.125), (3, 3, 3)),
    ]
    for snap in snaps:
        vals, nv = plan.pack(snap, norms)
        assert vals.tolist() == _expect(params, snap)
        assert nv.tolist() == [0.5, 4.0]
