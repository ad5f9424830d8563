"""Complex-field oracle pinned by the reference's complex
tests: test_reflect.cpp:115-143 (random complex reflectors), :282-293
(complex chains), test_haar.cpp:113-131 (unitary reconstruction, norm
preservation, adjoint identity), test_ginibre.cpp:117-132 (sesquilinear
adjoint identity, repeat probes); and by the real oracle on real input
(reflect.hpp:114-118: the complex formula reduces to the real one)."""
import numpy as np
import pytest


def test_random_complex_reflectors(orc):
    src = orc.RandomSource(8)
    for _ in range(200):
        n = 1 + int(src.uniform() * 48)
        off = int(src.uniform() * n)
        p = src.normal_complex_vector(n)
        tail = np.linalg.norm(p[off:])
        if tail == 0.0:
            continue
        hp = orc.c_reflector_apply(p, off, p)
        assert abs(hp[off] - tail) <= 1e-12 * tail
        if off + 1 < n:
            assert np.linalg.norm(hp[off + 1:]) <= 1e-10 * np.linalg.norm(p)
        x = src.normal_complex_vector(n)
        hx = orc.c_reflector_apply(p, off, x)
        assert abs(np.linalg.norm(hx) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)
        assert np.linalg.norm(orc.c_reflector_apply(p, off, hx, adjoint=True) - x) <= 1e-12 * np.linalg.norm(x)
        e = np.zeros(n, complex)
        e[off] = 1
        want = np.zeros(n, complex)
        want[off:] = p[off:] / tail
        assert np.linalg.norm(orc.c_reflector_apply(p, off, e, adjoint=True) - want) <= 1e-12


def test_complex_chain_inverts_through_reverse_adjoint(orc):
    src = orc.RandomSource(78)
    n = 10
    ps = np.stack([src.normal_complex_vector(n) for _ in range(4)])
    x = src.normal_complex_vector(n)
    y = orc.c_chain_apply(ps, x)
    assert abs(np.linalg.norm(y) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)
    assert np.linalg.norm(orc.c_chain_apply(ps, y, reverse=True, adjoint=True) - x) <= 1e-12 * np.linalg.norm(x)


def test_complex_reflector_reduces_to_the_real_one(orc):
    src = orc.RandomSource(5)
    for _ in range(50):
        n = 1 + int(src.uniform() * 30)
        off = int(src.uniform() * n)
        p = src.normal_vector(n)
        w, c, s, ident = orc.c_make_reflector(p.astype(complex), off)
        wr, cr, sr, identr = orc.make_reflector(p, off)
        assert ident == identr
        if not ident:
            assert np.allclose(w, wr, rtol=0, atol=1e-14) and abs(c - cr) <= 1e-14 and s == sr


def test_complex_haar(orc):
    n = 12
    op = orc.COperator("haar", n=n, seed=92)
    q = np.stack([op.probe(np.eye(n)[j].astype(complex), "right") for j in range(n)], axis=1)
    assert np.max(np.abs(q.conj().T @ q - np.eye(n))) <= 1e-12
    assert op.remaining_probes == 0
    with pytest.raises(orc.BudgetExhausted):
        op.probe(np.ones(n, complex), "right")
    n = 9
    op = orc.COperator("haar", n=n, seed=93)
    aux = orc.RandomSource(94)
    x, w = aux.normal_complex_vector(n), aux.normal_complex_vector(n)
    qx = op.probe(x, "right")
    assert abs(np.linalg.norm(qx) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)
    qhw = op.probe(w, "left")
    assert abs(np.vdot(w, qx) - np.vdot(qhw, x)) <= 1e-10 * np.linalg.norm(x) * np.linalg.norm(w)


def test_complex_ginibre(orc):
    op = orc.COperator("ginibre", m=13, n=10, sigma=1.0, seed=21)
    aux = orc.RandomSource(22)
    x, w = aux.normal_complex_vector(10), aux.normal_complex_vector(13)
    ax, ahw = op.probe(x, "right"), op.probe(w, "left")
    lhs, rhs = np.vdot(w, ax), np.vdot(ahw, x)
    assert abs(lhs - rhs) <= 1e-10 * (abs(lhs) + 1.0)
    op2 = orc.COperator("ginibre", m=13, n=10, sigma=1.0, seed=23)
    z1, z2 = op2.probe(x, "right"), op2.probe(x, "right")
    assert np.linalg.norm(z1 - z2) <= 1e-12 * np.linalg.norm(z1)
    # first probe closed form: y = sigma ||x|| g (complex analogue of test_ginibre.cpp:56-66)
    op3 = orc.COperator("ginibre", m=7, n=5, sigma=0.5, seed=99)
    x = aux.normal_complex_vector(5)
    g = orc.RandomSource(99).normal_complex_vector(7)
    assert np.linalg.norm(op3.probe(x, "right") - 0.5 * np.linalg.norm(x) * g) <= 1e-12 * np.linalg.norm(x)
    with pytest.raises(ValueError, match="input dimension"):
        op3.probe(np.ones(4, complex), "right")
