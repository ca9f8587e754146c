"""GPU parity of the interpolation baseline (h2_options.interp_p; interp.cu) against oracle/interp.py.

PAPER.md Eq. (2.2), section 6.3; readings Q1-Q4.
Structure (tree, lists, k_i, |Xbar_i|) is compared exactly, the Chebyshev nodes and U element by
element (the two sides share the operation order; only cos may differ in the last bit), the matvec
against the oracle's interpolation matvec and against dense K x, and the stored entry counts against
the oracle's memory count.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import interp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_2206_01885_b200")


def _gpu(pts, kid, kp, q, p, storage=None):
    return P.H2Matrix(torch.from_numpy(pts).cuda(), kid, kp, 1e-6, q, 0.5,
                      storage=P.H2_STORE_ALL if storage is None else storage, interp_p=p)


CASES = [
    ("3sphere", lambda: synth.three_spheres(3000, 21), P.H2_KERNEL_GAUSSIAN, (1.0,), 32, 2),
    ("3sphere", lambda: synth.three_spheres(3000, 21), P.H2_KERNEL_GAUSSIAN, (1.0,), 32, 4),
    ("3sphere", lambda: synth.three_spheres(2500, 22), P.H2_KERNEL_COULOMB, (), 40, 3),
    ("3sphere", lambda: synth.three_spheres(2500, 23), P.H2_KERNEL_COSDOT, (), 40, 3),
    ("3sphere", lambda: synth.three_spheres(2500, 24), P.H2_KERNEL_BUMP, (), 40, 3),
    ("mix2d", lambda: synth.clustered(4000, 2, 25), P.H2_KERNEL_MATERN32, (0.1,), 48, 5),
    ("cube1d", lambda: synth.uniform_cube(1500, 1, 26), P.H2_KERNEL_LAPLACE, (0.5,), 16, 7),
]


@pytest.mark.parametrize("name,gen,kid,kp,q,p", CASES)
def test_interp_parity(name, gen, kid, kp, q, p):
    oracle.build()
    pts = gen()
    n, d = pts.shape
    o = oracle.OracleH2(pts, q, 0.5)
    m = interp.InterpH2(o, p, kid, kp[0] if kp else 0.0)
    g = _gpu(pts, kid, kp, q, p)
    info = g.info()
    assert info["r"] == p ** d
    for what, ow in (("PERM", oracle.PERM), ("IL_IDX", oracle.IL_IDX), ("NF_IDX", oracle.NF_IDX)):
        assert np.array_equal(g.export(what), o.export(ow)), what
    k = g.export("K")
    assert np.array_equal(k, m.k.astype(np.int32))
    xb = g.export("XBAR_N")
    Q = g.export("INTERP_Q").reshape(m.nn, m.r, d)
    off = g.export("U_OFF")
    U = g.export("U")
    for i in range(m.nn):
        if m.k[i] == 0:
            assert xb[i] == 0
            continue
        assert xb[i] == m.U[i].shape[0]
        np.testing.assert_allclose(Q[i], m.Q[i], rtol=1e-15, atol=1e-15 * np.abs(m.Q[i]).max())
        Ug = U[off[i]:off[i + 1]].reshape(m.r, xb[i]).T
        np.testing.assert_allclose(Ug, m.U[i], rtol=0, atol=1e-12 * max(1.0, np.abs(m.U[i]).max()))
    mem = m.memory_entries()
    assert info["coupling_entries"] == mem["coupling"]
    assert info["nearfield_entries"] == mem["nearfield"]
    assert off[-1] == mem["u"]
    x = synth.matvec_vector(1, n)
    yg = g.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    yo = m.matvec(x)
    yd = oracle.dense_rows(pts, kid, kp[0] if kp else 0.0, x, np.arange(n))
    eg = np.linalg.norm(yg - yd) / np.linalg.norm(yd)
    eo = np.linalg.norm(yo - yd) / np.linalg.norm(yd)
    assert np.linalg.norm(yg - yo) / np.linalg.norm(yo) <= 1e-12, (eg, eo)
    assert eg <= 2 * eo + 1e-15
    g.close()


def test_interp_fly_equals_stored():
    pts = synth.three_spheres(3000, 27)
    x = torch.from_numpy(synth.matvec_vector(2, 3000)).cuda()
    a = _gpu(pts, P.H2_KERNEL_GAUSSIAN, (1.0,), 32, 3)
    b = _gpu(pts, P.H2_KERNEL_GAUSSIAN, (1.0,), 32, 3, storage=P.H2_STORE_ON_THE_FLY)
    ya, yb = a.matvec(x), b.matvec(x)
    assert torch.allclose(ya, yb, rtol=1e-13, atol=1e-13 * float(ya.abs().max()))
    a.close()
    b.close()


@pytest.mark.parametrize("kw", [dict(p=17), dict(p=6, d=5), dict(p=3, nonsym=True), dict(p=3, kid=7)])
def test_interp_invalid(kw):
    d = kw.get("d", 3)
    pts = torch.from_numpy(synth.uniform_cube(500, d, 3)).cuda()
    kid = kw.get("kid", P.H2_KERNEL_GAUSSIAN)
    kp = (1.0,) if kid != 7 else (1.0,) + (0.0,) * d
    with pytest.raises(P.H2Error):
        P.H2Matrix(pts, kid, kp, 1e-6, 32, 0.5, interp_p=kw["p"], nonsymmetric=kw.get("nonsym", False))
