"""HiDR once for all (§6.1.3): h2_rebuild_ex reuses a
base handle's tree, lists and representor sets for another kernel.  The rebuilt handle must equal a
fresh build of the new kernel at the base's r in every index set (bit for bit) and numerically in
its bases and matvec, and must match the oracle run at that r (skeleton agreement, matvec error
within 2x, GPU vs oracle within 10 id_tol) -- the paper's claim that one HiDR serves many kernels."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2206_01885_b200 as P  # noqa: E402

INDEX_SETS = ["PERM", "NODES", "IL_OFF", "IL_IDX", "NF_OFF", "NF_IDX", "XS_OFF", "XS_IDX", "YS_OFF", "YS_IDX",
              "K", "SK_OFF", "SK_IDX", "XBAR_N", "U_OFF"]


@pytest.mark.parametrize("cfg,n,new_kid,new_kp,new_tol", [
    (1, 8192, 2, [0.5], 1e-6),      # Coulomb geometry -> Gaussian
    (4, 60000, 2, [0.05], 1e-6),    # Matern geometry -> Gaussian
    (3, 30000, 3, [0.3], 1e-5),     # Gaussian geometry -> Matern, another tolerance
    (3, 30000, 6, [], 1e-6),        # Gaussian geometry -> Table 1 kappa_3 = cos(x . y)
])
def test_rebuild_equals_fresh_build_at_base_r(cfg, n, new_kid, new_kp, new_tol):
    c = synth.CONFIGS[cfg]
    pts = synth.points(cfg, n)
    X = torch.from_numpy(pts).cuda()
    base = P.H2Matrix(X, c["kernel"], list(c["params"]), c["id_tol"], c["q"], c["tau"], storage=P.H2_STORE_ALL)
    r = base.info()["r"]
    rb = base.rebuild(new_kid, new_kp, new_tol, storage=P.H2_STORE_ALL, timing=True)
    fresh = P.H2Matrix(X, new_kid, new_kp, new_tol, c["q"], c["tau"], r=r, storage=P.H2_STORE_ALL)
    ri, fi = rb.info(), fresh.info()
    assert ri["r"] == r and ri["nnodes"] == fi["nnodes"]
    assert ri["stage_ms"]["tree"] >= 0 and ri["hidr_dist_evals"] == 0  # HiDR did not run again
    for name in INDEX_SETS:
        assert np.array_equal(rb.export(name), fresh.export(name)), name
    np.testing.assert_array_equal(rb.export("U"), fresh.export("U"))
    x = torch.from_numpy(synth.matvec_vector(cfg, n)).cuda()
    ya, yb = rb.matvec(x), fresh.matvec(x)
    assert torch.linalg.norm(ya - yb) <= 1e-12 * torch.linalg.norm(yb)
    # the base handle is untouched and still usable
    yb0 = base.matvec(x)
    assert torch.isfinite(yb0).all()
    # oracle at the same r: the paper's "HiDR once for all" accuracy
    o = oracle.OracleH2(pts, c["q"], c["tau"])
    o.build(new_kid, new_kp[0] if new_kp else 0.0, new_tol, r)
    rows = synth.sample_rows(cfg, n)
    yd = oracle.dense_rows(pts, new_kid, new_kp[0] if new_kp else 0.0, synth.matvec_vector(cfg, n), rows)
    yo = o.matvec(synth.matvec_vector(cfg, n), None if n <= 16384 else rows)
    yo = yo[rows] if n <= 16384 else yo
    yg = ya.cpu().numpy()[rows]
    eg = np.linalg.norm(yg - yd) / np.linalg.norm(yd)
    eo = np.linalg.norm(yo - yd) / np.linalg.norm(yd)
    print(f"cfg{cfg} -> kernel {new_kid}{new_kp}: r={r} err_gpu={eg:.3e} err_oracle={eo:.3e}")
    assert eg <= 2.0 * eo + 1e-15
    assert np.linalg.norm(yg - yo) / np.linalg.norm(yo) <= 10 * new_tol
    for g in (rb, fresh, base):
        g.close()


def test_rebuild_rejects_a_foreign_comm_and_null_base():
    pts = synth.points(1, 2000)
    g = P.H2Matrix(torch.from_numpy(pts).cuda(), 1, [], 1e-6, 64)
    comm = P.H2Comm.local(1, 0, 987654)
    o = P.h2_options_default()
    o.comm = comm.ptr
    import ctypes as C
    kp = (C.c_double * 1)(0.5)
    assert not P.lib().h2_rebuild_ex(C.c_void_p(g.h), 2, kp, 1e-6, C.byref(o))
    assert P.last_error()[0] == -1
    assert not P.lib().h2_rebuild_ex(None, 2, kp, 1e-6, None)
    comm.close()
    g.close()


@pytest.mark.parametrize("reduct", [1, 2])
def test_rebuild_keeps_the_reduction_of_the_base(reduct):
    """HiDR once for all from a base built with FPS / the surface reduction: the rebuild reuses those
    representor sets -- equal to a fresh build of the new kernel with the same reduction and r."""
    c = synth.CONFIGS[4]
    pts = synth.points(4, 40000)
    X = torch.from_numpy(pts).cuda()
    base = P.H2Matrix(X, c["kernel"], list(c["params"]), c["id_tol"], c["q"], c["tau"], storage=P.H2_STORE_ALL,
                      reduct=reduct)
    r = base.info()["r"]
    rb = base.rebuild(2, [0.05], 1e-6, storage=P.H2_STORE_ALL)
    fresh = P.H2Matrix(X, 2, [0.05], 1e-6, c["q"], c["tau"], r=r, storage=P.H2_STORE_ALL, reduct=reduct)
    for name in ("XS_OFF", "XS_IDX", "YS_OFF", "YS_IDX", "K", "SK_IDX"):
        assert np.array_equal(rb.export(name), fresh.export(name)), name
    x = torch.from_numpy(synth.matvec_vector(4, 40000)).cuda()
    ya, yb = rb.matvec(x), fresh.matvec(x)
    assert torch.linalg.norm(ya - yb) <= 1e-12 * torch.linalg.norm(yb)
    for g in (rb, fresh, base):
        g.close()
