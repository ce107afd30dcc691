"""Oracle pins for the compensated dot product policy (PAPER.md:434,
Sec. 5.2.1; SPEC.md eft module): TwoSum / TwoProduct exactness, the Dot2 accuracy staircase,
and the paper's finding that compensated fp32 dots do not cure the gather-scatter stagnation."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth


def f32(v):
    return float(np.float32(v))


def test_two_sum_exact():
    z = synth.uniform_by_id(7, 20, np.arange(2000))
    for i in range(0, 2000, 2):
        a = f32(z[i] * 2.0 ** (int(z[i + 1] * 20)))
        b = f32(z[i + 1] * 3.7)
        s, e = oracle.two_sum_f(a, b)
        assert s == f32(a + b)                                  # s = fl(a + b)
        assert Fraction(s) + Fraction(e) == Fraction(a) + Fraction(b)
    assert oracle.two_sum_f(1.0, 2.0) == (3.0, 0.0)
    s, e = oracle.two_sum_f(2.0 ** 24, 1.0)                     # 2^24 + 1 not representable
    assert (s, e) == (2.0 ** 24, 1.0)


def test_two_prod_exact():
    z = synth.uniform_by_id(8, 21, np.arange(2000))
    for i in range(0, 2000, 2):
        a, b = f32(z[i] * 7.0), f32(z[i + 1] * 0.3)
        p, e = oracle.two_prod_f(a, b)
        assert p == f32(a * b)
        assert Fraction(p) + Fraction(e) == Fraction(a) * Fraction(b)
    p, e = oracle.two_prod_f(f32(1 + 2 ** -12), f32(1 + 2 ** -12))
    assert (p, e) == (f32(1 + 2 ** -11), 2.0 ** -24)


def test_dot2_spec_example():
    """SPEC.md eft/dot2: binary32 x=[1e8, 1, -1e8], y=1 -> dot2 = 1 while the plain dot = 0."""
    x = np.array([1e8, 1.0, -1e8], np.float32)
    one = np.ones(3, np.float32)
    assert oracle.glsc3(x, one, one, oracle.FP32_DOT2) == 1.0
    assert oracle.glsc3(x, one, one, oracle.FP32, seqdot=True) == 0.0


@pytest.mark.parametrize("cond", [1e2, 1e4, 1e6])
def test_dot2_accuracy_staircase(cond):
    """Ill-conditioned dot products (cond = sum|x y| / |sum x y|): Dot2 keeps the relative error
    at ~u (SPEC.md: <= 32 * 2^-23 for cond <= 1e6) -- twice the working precision."""
    n = 200
    z = synth.uniform_by_id(9, 22, np.arange(3 * n))
    e = np.round(z[:n] * np.log2(cond) / 2).astype(int)
    x = (z[n:2 * n] * 2.0 ** e).astype(np.float32)
    y = (z[2 * n:] * 2.0 ** e).astype(np.float32)
    # cancel most of the sum in the last half so the condition number approaches cond
    exact = sum(Fraction(float(a)) * Fraction(float(b)) for a, b in zip(x[: n // 2], y[: n // 2]))
    x[n // 2:] *= np.float32(1.0)
    target = -float(exact)
    x[-1] = np.float32(target / float(y[-1])) if y[-1] != 0 else x[-1]
    exact = sum(Fraction(float(a)) * Fraction(float(b)) for a, b in zip(x, y))
    absum = sum(abs(Fraction(float(a)) * Fraction(float(b))) for a, b in zip(x, y))
    c = np.ones(n, np.float32)
    d2 = oracle.glsc3(x, c, y, oracle.FP32_DOT2)
    ref = float(exact)
    achieved = float(absum / abs(exact)) if exact != 0 else float("inf")
    # Dot2 error bound (Ogita-Rump-Oishi, Prop. 5.5): |res - exact| <= u |exact| + g_n^2 sum|x y|
    u = 2.0 ** -24
    gn = n * u / (1 - n * u)
    assert abs(d2 - ref) <= u * abs(ref) + gn * gn * float(absum) * 1.0001, (d2, ref, achieved)
    assert abs(d2 - ref) <= 32 * 2.0 ** -23 * abs(ref) or achieved > 1e6


@pytest.fixture(scope="module")
def box8():
    o = oracle.Mesh(8, 8, 8, 7)
    return o, o.rhs(seed=0)


def test_dot2_cg_consistent_converges(box8):
    """Consistent gather-scatter: fp32 + Dot2 converges to 1e-8 like the mixed policy."""
    o, b = box8
    _, _, r = o.cg(b, oracle.FP32_DOT2, max_iter=1200, rtol=1e-8)
    _, _, rm = o.cg(b, oracle.MIXED, max_iter=1200, rtol=1e-8)
    assert r.status == oracle.CONVERGED
    assert abs(r.iterations - rm.iterations) <= 0.05 * rm.iterations


def test_dot2_does_not_cure_per_copy_stagnation(box8):
    """PAPER.md:434-441 and Table 4 (:457-476): compensated fp32 dots bring "only marginal
    improvement" -- the stagnation comes from the gather-scatter precision, so fp32 + Dot2 under
    the per-copy (pairwise) order still fails while the fp64 gather-scatter (mixed) converges."""
    o, b = box8
    _, _, rd = o.cg(b, oracle.FP32_DOT2, max_iter=1200, rtol=1e-8, gs_order=oracle.GS_PER_COPY)
    _, _, rm = o.cg(b, oracle.MIXED, max_iter=1200, rtol=1e-8, gs_order=oracle.GS_PER_COPY)
    assert rd.status in (oracle.STAGNATED, oracle.BREAKDOWN) and rd.rel_res_min > 1e-8
    assert rm.status == oracle.CONVERGED
