"""Golden fixtures (tests/golden/, each file cites its source): worked-example values from
SPEC.md's examples for the paper's kernels and textbook closed forms, checked against the oracle."""
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rows(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                yield [[float(t) for t in field.split()] for field in line.split("|")]


@pytest.mark.parametrize("row", list(rows("gll_closed_forms.txt")), ids=lambda r: f"p{int(r[0][0])}")
def test_gll_golden(row):
    (p,), nodes, weights = row
    z, w, D = oracle.gll(int(p))
    np.testing.assert_allclose(z, nodes, rtol=0, atol=1e-15)
    np.testing.assert_allclose(w, weights, rtol=0, atol=1e-15)


def test_dot2_golden():
    for x, y, (d2,), (plain,) in rows("dot2_cancellation.txt"):
        x32, y32 = np.array(x, np.float32), np.array(y, np.float32)
        one = np.ones_like(x32)
        assert oracle.glsc3(x32, one, y32, oracle.FP32_DOT2) == d2
        assert oracle.glsc3(x32, one, y32, oracle.FP32, seqdot=True) == plain


def test_glsc3_golden():
    for a, c, b, (res,) in rows("glsc3_trivial.txt"):
        for pol in (oracle.FP64, oracle.MIXED, oracle.FP32, oracle.FP32_DOT2):
            assert oracle.glsc3(np.array(a), np.array(c), np.array(b), pol) == res
