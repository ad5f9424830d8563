"""Device make_reflector / Reflector (reflect.hpp:47-176, module.cpp:48-66) and
the thin compositions USVOperator / SubsampledHaarOperator over device
operators (ensembles.hpp:133-215), checked against the oracle and the
reference's own test expectations (test_reflect.cpp, test_ensembles.cpp)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_reflector_hand_cases(lm):
    # test_reflect.cpp:25-64, test_smoke.py:16-27
    h = lm.make_reflector(np.array([3.0, 4.0]))
    assert (h.dim, h.offset, h.is_identity) == (2, 0, False)
    hp = h.apply(np.array([3.0, 4.0]))
    assert abs(hp[0] - 5.0) < 1e-12 and abs(hp[1]) < 1e-12
    col = h.apply(np.array([1.0, 0.0]))
    assert abs(col[0] - 0.6) <= 1e-12 and abs(col[1] - 0.8) <= 1e-12
    x = np.array([0.25, -1.5])
    assert np.allclose(h.apply(h.apply(x), adjoint=True), h.apply(h.apply(x)))
    assert np.allclose(h.apply(h.apply(x)), x, atol=1e-14)
    e = np.eye(3)
    h = lm.make_reflector(np.array([1.0, 0, 0]))
    assert np.linalg.norm(h.apply(e[0]) - e[0]) <= 1e-14
    assert np.linalg.norm(h.apply(e[1]) + e[1]) <= 1e-14
    h = lm.make_reflector(np.array([5.0, 0, 0]), 1)
    assert h.is_identity
    assert np.array_equal(h.apply(np.array([1.0, 2, 3])), np.array([1.0, 2, 3]))


def test_reflector_matches_oracle_and_properties(orc, lm):
    src = orc.RandomSource(7)
    for _ in range(60):
        n = 1 + int(src.uniform() * 64)
        off = int(src.uniform() * n)
        p = src.normal_vector(n)
        x = src.normal_vector(n)
        h = lm.make_reflector(p, off)
        tail = np.linalg.norm(p[off:])
        if tail == 0:
            assert h.is_identity
            continue
        hp = h.apply(p)
        assert abs(hp[off] - tail) <= 1e-12 * tail
        if off + 1 < n:
            assert np.linalg.norm(hp[off + 1:]) <= 1e-10 * np.linalg.norm(p)
        assert np.array_equal(hp[:off], p[:off])
        hx = h.apply(x)
        assert np.linalg.norm(hx - orc.reflector_apply(p, off, x)) <= 1e-13 * np.linalg.norm(x)
        assert np.linalg.norm(h.apply(hx) - x) <= 1e-12 * np.linalg.norm(x)


def test_reflector_extreme_scales_and_errors(lm):
    # test_reflect.cpp:172-189 (stableNorm branch), 230-245
    for scale in (1e-300, 1e-150, 1.0, 1e150, 1e290):
        p = np.array([3 * scale, 4 * scale])
        hp = lm.make_reflector(p).apply(p)
        assert np.isfinite(hp[0])
        assert abs(hp[0] - 5 * scale) <= 1e-10 * 5 * scale
        assert abs(hp[1]) <= 1e-10 * 5 * scale
    with pytest.raises(ValueError, match="empty vector"):
        lm.make_reflector(np.zeros(0))
    with pytest.raises(ValueError, match="offset out of range"):
        lm.make_reflector(np.ones(3), 3)
    with pytest.raises(ValueError, match="non-finite"):
        lm.make_reflector(np.array([1.0, np.inf]))
    with pytest.raises(ValueError, match="dimension mismatch"):
        lm.make_reflector(np.ones(3)).apply(np.ones(4))


def test_usv_unit_and_zero_spectrum(orc, lm):
    # test_ensembles.cpp:182-199
    n = 12
    op = lm.USVOperator(lm.HaarOperator(n, seed=331), lm.HaarOperator(n, seed=332), np.ones(n))
    assert (op.rows, op.cols) == (n, n)
    x = orc.RandomSource(333).normal_vector(n)
    y = op.probe(x, "right")
    assert abs(np.linalg.norm(y) - np.linalg.norm(x)) <= 1e-10 * np.linalg.norm(x)
    z = lm.USVOperator(lm.HaarOperator(6, seed=334), lm.HaarOperator(6, seed=335), np.zeros(6))
    assert np.linalg.norm(z.probe(orc.RandomSource(336).normal_vector(6), "right")) == 0.0


def test_usv_rectangular_adjoint_and_spectrum(orc, lm):
    # test_ensembles.cpp:201-233
    rows, cols = 10, 6
    op = lm.USVOperator(lm.HaarOperator(rows, seed=337), lm.HaarOperator(cols, seed=338), 0.5 * np.ones(cols))
    aux = orc.RandomSource(339)
    x, w = aux.normal_vector(cols), aux.normal_vector(rows)
    ax = op.probe(x, "right")
    atw = op.probe(w, "left")
    assert ax.shape == (rows,) and atw.shape == (cols,)
    assert abs(w @ ax - atw @ x) <= 1e-10 * np.linalg.norm(x) * np.linalg.norm(w)
    n = 24
    rs = orc.RandomSource(340)
    sv = np.sort(np.array([0.5 + rs.uniform() for _ in range(n)]))[::-1].copy()
    op = lm.USVOperator(lm.HaarOperator(n, seed=341), lm.HaarOperator(n, seed=342), sv)
    a = np.stack([op.probe(np.eye(n)[j], "right") for j in range(n)], axis=1)
    assert op.remaining_probes == 0
    with pytest.raises(lm.BudgetExhausted):
        op.probe(a[:, 0], "right")
    assert np.max(np.abs(np.linalg.svd(a, compute_uv=False) - sv)) <= 1e-8


def test_usv_validation(lm):
    with pytest.raises(ValueError):
        lm.USVOperator(None, lm.HaarOperator(4, seed=1), np.ones(4))
    with pytest.raises(ValueError):
        lm.USVOperator(lm.GinibreOperator(6, 4, seed=343), lm.HaarOperator(4, seed=2), np.ones(4))
    with pytest.raises(ValueError):
        lm.USVOperator(lm.HaarOperator(4, seed=3), lm.HaarOperator(4, seed=4), np.ones(3))


def test_usv_parity_with_composed_oracle(orc, lm):
    n, k = 50, 6
    sv = np.linspace(2.0, 0.5, n)
    u = lm.HaarOperator(n, seed=11, draws="injected")
    v = lm.HaarOperator(n, seed=12, draws="injected")
    u.push_draws(orc.draws_for(11, [n] * k))
    v.push_draws(orc.draws_for(12, [n] * k))
    op = lm.USVOperator(u, v, sv)
    ru, rv = orc.Operator("haar", n=n, seed=11), orc.Operator("haar", n=n, seed=12)
    aux = orc.RandomSource(13)
    for t in range(k):
        x = aux.normal_vector(n)
        side = "right" if t % 2 == 0 else "left"
        if side == "right":  # ensembles.hpp:377-381 restated
            want = ru.probe(np.concatenate([sv * rv.probe(x, "right")]), "right")
        else:
            want = rv.probe(sv * ru.probe(x, "left"), "left")
        got = op.probe(x, side)
        assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)


def test_subsampled_haar_matches_full_operator(orc, lm):
    # test_ensembles.cpp:235-260: row subsampling is bit-identical to the head
    n, rows = 8, 3
    sub = lm.SubsampledHaarOperator(lm.HaarOperator(n, seed=351), rows)
    full = lm.HaarOperator(n, seed=351)
    assert (sub.rows, sub.cols) == (rows, n)
    x = orc.RandomSource(352).normal_vector(n)
    ys, yf = sub.probe(x, "right"), full.probe(x, "right")
    assert np.array_equal(ys, yf[:rows])
    w = orc.RandomSource(353).normal_vector(rows)
    zl = sub.probe(w, "left")
    pad = np.zeros(n)
    pad[:rows] = w
    assert np.array_equal(zl, full.probe(pad, "left"))
    with pytest.raises(ValueError):
        lm.SubsampledHaarOperator(lm.HaarOperator(4, seed=1), 5)
