"""Host-side plan layout: post-order node table, column slots, parameter order
(reference PdfNode.walk / param order: pdf.py:86-98, dalitz.py:369-371)."""

import pytest

from paper_1710_08826_b200 import _lib as L
from paper_1710_08826_b200.plan import UnsupportedNode, layout
from tests import models


def test_c1_layout():
    x, pdf, (mu, sigma, alpha, f) = models.c1()
    t = layout(pdf, ("x",))
    kinds = [t.table[i].kind for i in range(len(t.nodes))]
    assert kinds == [L.KIND_CODES["gaussian"], L.KIND_CODES["exponential"], L.KIND_CODES["add"]]
    assert [t.table[i].nchild for i in range(3)] == [0, 0, 2]
    assert [t.table[i].col0 for i in range(3)] == [0, 0, -1]
    assert t.params == [mu, sigma, alpha, f]


def test_c2_layout_columns():
    (x, y), pdf, params = models.c2()
    t = layout(pdf, ("x", "y"))
    assert [t.table[i].col0 for i in range(3)] == [0, 1, -1]
    assert t.params == list(params)


def test_c3_layout_dalitz_desc():
    (s12, s13), pdf, terms = models.c3()
    t = layout(pdf, ("s12", "s13"))
    assert t.ndalitz == 1
    d = t.dalitz[0]
    assert d.nterms == 4
    assert [d.pair[k] for k in range(4)] == [13, 23, 12, 12]
    assert [d.spin[k] for k in range(4)] == [1, 1, 1, 0]
    assert t.table[0].col0 == 0 and t.table[0].col1 == 1
    assert len(t.params) == 16
    assert t.params[:4] == [terms[0].mass, terms[0].width, terms[0].magnitude, terms[0].phase]


def test_unknown_kind_is_rejected():
    x, pdf, _ = models.c1()
    pdf.children[0].kind = "custom"
    with pytest.raises(UnsupportedNode):
        layout(pdf, ("x",))
