"""GPU parity of the non-symmetric path (Algorithm 2 with separate row / column sets: both getBasis
calls of line 11; B_ij = K(X^_i^(row), X^_j^(col)) over every ordered admissible pair and
K(X_i, X_j) over every ordered nearfield pair) against the oracle, with the shifted
multiquadric sqrt(1 + c |x - y + a|^2) of P:711-716 on synthetic 2-D data.

Acceptance as for the symmetric path (BASELINE north_star): r, tree, lists and representor sets
bit-exact; row AND column skeletons agree except at pivot near-ties; U and V element-wise on the
agreeing nodes; stored entries equal the kernel at their recorded points; matvec error within 2x of
the oracle's and within 10 id_tol of the oracle's product.  A symmetric kernel run through the
non-symmetric path gives V = U and X^(col) = X^(row) bit for bit.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2206_01885_b200 as P  # noqa: E402

MQ = 7


def _gpu(pts, kp, tol, q, storage=P.H2_STORE_ALL, kid=MQ, nonsym=False):
    X = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
    return P.H2Matrix(X, kid, kp, tol, q, 0.5, storage=storage, timing=True, nonsymmetric=nonsym)


def _agree(gk, gso, gsi, ok, oso, osi):
    nodes = np.flatnonzero((gk > 0) | (ok > 0))
    same = [i for i in nodes if gk[i] == ok[i] and np.array_equal(gsi[gso[i]:gso[i + 1]], osi[oso[i]:oso[i + 1]])]
    return same, len(same) / max(1, len(nodes))


def _u_err(same, k, uo, U, ouo, oU):
    worst = 0.0
    for i in same:
        a = U[uo[i]:uo[i + 1]]
        b = oU[ouo[i]:ouo[i + 1]]
        if len(a):
            worst = max(worst, np.abs(a - b).max() / max(1.0, np.abs(b).max()))
    return worst


@pytest.mark.parametrize("n,q,c,a,tol,data", [
    (20000, 64, 100.0, (0.0, 0.3), 1e-6, "uniform"),
    (30000, 64, 100.0, (0.0, 20.0), 1e-6, "uniform"),       # the paper's a = [0, 20]
    (40000, 128, 30.0, (0.1, -0.2), 1e-8, "clustered"),
])
def test_nonsym_parity(n, q, c, a, tol, data):
    pts = synth.uniform_cube(n, 2, seed=71) if data == "uniform" else synth.clustered(n, 2, seed=72, k=5, sigma=0.08)
    kp = [c, *a]
    oracle.set_kernel_shift(np.array(a))
    o = oracle.OracleH2(pts, q, 0.5, nonsym=True)
    r = o.build(MQ, c, tol)
    g = _gpu(pts, kp, tol, q)
    info = g.info()
    assert info["nonsymmetric"] == 1 and info["r"] == r
    for gname, oname in [("PERM", oracle.PERM), ("IL_OFF", oracle.IL_OFF), ("IL_IDX", oracle.IL_IDX),
                         ("NF_OFF", oracle.NF_OFF), ("NF_IDX", oracle.NF_IDX), ("XS_IDX", oracle.XS_IDX),
                         ("YS_OFF", oracle.YS_OFF), ("YS_IDX", oracle.YS_IDX)]:
        assert np.array_equal(g.export(gname), o.export(oname)), gname
    same_r, fr = _agree(g.export("K"), g.export("SK_OFF"), g.export("SK_IDX"), o.export(oracle.K),
                        *o.skeletons())
    same_c, fc = _agree(g.export("K_COL"), g.export("SKC_OFF"), g.export("SKC_IDX"), o.export(oracle.K_COL),
                        *o.skeletons_col())
    tol_u = max(1e-10, 2e-15 / tol)
    eu = _u_err(same_r, None, g.export("U_OFF"), g.export("U"), o.export(oracle.U_OFF), o.export(oracle.U))
    ev = _u_err(same_c, None, g.export("V_OFF"), g.export("V"), o.export(oracle.V_OFF), o.export(oracle.V))
    x = synth.matvec_vector(2, n)
    rows = synth.sample_rows(2, n)
    yg = g.matvec(torch.from_numpy(x).cuda()).cpu().numpy()[rows]
    yo = o.matvec(x, rows)
    yd = oracle.dense_rows(pts, MQ, c, x, rows)
    eg = np.linalg.norm(yg - yd) / np.linalg.norm(yd)
    eo = np.linalg.norm(yo - yd) / np.linalg.norm(yd)
    ag = np.linalg.norm(yg - yo) / np.linalg.norm(yo)
    print(f"nonsym n={n} a={a}: r={r} row-agree={fr:.4f} col-agree={fc:.4f} U={eu:.2e} V={ev:.2e} "
          f"err_gpu={eg:.3e} err_oracle={eo:.3e} gpu-vs-oracle={ag:.3e} kmax={info['kmax']}/{info['kmax_col']}")
    assert fr >= 0.99 and fc >= 0.99
    assert eu <= tol_u and ev <= tol_u
    assert eg <= 2.0 * eo + 1e-15
    assert ag <= 10 * tol
    # every ordered pair stored: the entry counts of the oracle's ordered-pair fill
    no, _ = o.fill()
    assert info["coupling_entries"] + info["nearfield_entries"] == no
    # sampled stored entries against the oracle's kernel at the recorded points
    Xt = g.export("TREE_X").reshape(-1, 2)
    rng = np.random.default_rng(3)
    il_off, il_idx = g.export("IL_OFF"), g.export("IL_IDX")
    nf_off, nf_idx = g.export("NF_OFF"), g.export("NF_IDX")
    k, kc = g.export("K"), g.export("K_COL")
    nodes = g.export("NODES").reshape(-1, 7)
    cp = [(i, j) for i in range(len(k)) for j in il_idx[il_off[i]:il_off[i + 1]] if k[i] > 0 and kc[j] > 0]
    nfp = [(i, j) for i in range(len(k)) for j in nf_idx[nf_off[i]:nf_off[i + 1]]]
    kinds, pairs, entries = [], [], []
    for _ in range(1000):
        if rng.random() < 0.5:
            p = int(rng.integers(len(cp)))
            i, j = cp[p]
            kinds.append(0), pairs.append(p), entries.append(int(rng.integers(k[i] * kc[j])))
        else:
            p = int(rng.integers(len(nfp)))
            i, j = nfp[p]
            kinds.append(1), pairs.append(p)
            entries.append(int(rng.integers((nodes[i, 2] - nodes[i, 1]) * (nodes[j, 2] - nodes[j, 1]))))
    val, rp, colp = P.h2_sample_blocks(g.h, kinds, pairs, entries)
    ref = np.array([oracle.kernel(MQ, c, Xt[u], Xt[v]) for u, v in zip(rp, colp)])
    np.testing.assert_allclose(val, ref, rtol=1e-13)
    sk_idx, sk_off = g.export("SK_IDX"), g.export("SK_OFF")
    skc_idx, skc_off = g.export("SKC_IDX"), g.export("SKC_OFF")
    for kd, p, rr, cc in zip(kinds, pairs, rp, colp):
        if kd == 0:
            i, j = cp[p]
            assert rr in sk_idx[sk_off[i]:sk_off[i + 1]] and cc in skc_idx[skc_off[j]:skc_off[j + 1]]
    g.close()


@pytest.mark.parametrize("kid,kp", [(1, []), (2, [0.5]), (3, [0.1])])
def test_symmetric_kernel_through_nonsym_path(kid, kp):
    pts = synth.points(1, 8192)
    a = _gpu(pts, kp, 1e-6, 64, kid=kid)
    b = _gpu(pts, kp, 1e-6, 64, kid=kid, nonsym=True)
    assert b.info()["nonsymmetric"] == 1 and a.info()["nonsymmetric"] == 0
    for nm, nc in [("K", "K_COL"), ("SK_IDX", "SKC_IDX"), ("U", "V"), ("XBAR_N", "XBARC_N")]:
        assert np.array_equal(b.export(nm), b.export(nc)), nm
        assert np.array_equal(a.export(nm), b.export(nm)), nm
    x = torch.from_numpy(synth.matvec_vector(1, 8192)).cuda()
    ya, yb = a.matvec(x), b.matvec(x)
    assert torch.linalg.norm(ya - yb) <= 1e-13 * torch.linalg.norm(ya)
    ia, ib = a.info(), b.info()
    assert ib["nearfield_entries"] > ia["nearfield_entries"]   # every ordered pair stored


def test_nonsym_on_the_fly_equals_stored_and_single_leaf():
    kp = [100.0, 0.0, 0.3]
    oracle.set_kernel_shift(np.array(kp[1:]))
    pts = synth.uniform_cube(12000, 2, seed=73)
    a = _gpu(pts, kp, 1e-6, 64)
    b = _gpu(pts, kp, 1e-6, 64, storage=P.H2_STORE_ON_THE_FLY)
    x = torch.from_numpy(synth.matvec_vector(2, 12000)).cuda()
    ya, yb = a.matvec(x), b.matvec(x)
    assert torch.linalg.norm(ya - yb) <= 1e-12 * torch.linalg.norm(ya)
    small = synth.uniform_cube(50, 2, seed=74)
    g = _gpu(small, kp, 1e-6, 64)
    assert g.info()["nnodes"] == 1
    xs = synth.matvec_vector(2, 50)
    y = g.matvec(torch.from_numpy(xs).cuda()).cpu().numpy()
    yd = oracle.dense_rows(small, MQ, kp[0], xs, np.arange(50))
    np.testing.assert_allclose(y, yd, rtol=1e-12)
