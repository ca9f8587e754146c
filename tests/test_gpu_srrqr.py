"""GPU SRRQR refinement (h2_options.srrqr_f, srrqr.cu; PAPER Eq.(4.1), ||G||_max bounded)
against the oracle's (orc_srrqr_swaps): the same skeletons except at near-ties, every U_i entry
bounded by f, swaps made, the matvec error within 2x of the oracle's."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2206_01885_b200 as P  # noqa: E402


@pytest.mark.parametrize("cfg,n,f", [(1, 8192, 1.2), (4, 60000, 1.5), (3, 20000, 1.1)])
def test_srrqr_parity(cfg, n, f):
    c = synth.CONFIGS[cfg]
    pts = synth.points(cfg, n)
    kp = list(c["params"])
    o = oracle.OracleH2(pts, c["q"], c["tau"], srrqr_f=f)
    r = o.build(c["kernel"], kp[0] if kp else 0.0, c["id_tol"])
    g = P.H2Matrix(torch.from_numpy(pts).cuda(), c["kernel"], kp, c["id_tol"], c["q"], c["tau"],
                   storage=P.H2_STORE_ALL, timing=True, srrqr_f=f)
    info = g.info()
    assert info["r"] == r
    gk, ok = g.export("K"), o.export(oracle.K)
    go, gi = g.export("SK_OFF"), g.export("SK_IDX")
    oo, oi = o.skeletons()
    nodes = np.flatnonzero((gk > 0) | (ok > 0))
    same = sum(1 for i in nodes if gk[i] == ok[i] and np.array_equal(gi[go[i]:go[i + 1]], oi[oo[i]:oo[i + 1]]))
    frac = same / max(1, len(nodes))
    U = g.export("U")
    x = synth.matvec_vector(cfg, n)
    rows = synth.sample_rows(cfg, n)
    yg = g.matvec(torch.from_numpy(x).cuda()).cpu().numpy()[rows]
    yo = o.matvec(x, rows)
    yd = oracle.dense_rows(pts, c["kernel"], kp[0] if kp else 0.0, x, rows)
    eg = np.linalg.norm(yg - yd) / np.linalg.norm(yd)
    eo = np.linalg.norm(yo - yd) / np.linalg.norm(yd)
    print(f"srrqr cfg{cfg} f={f}: swaps gpu {info['srrqr_swaps']} oracle {o.srrqr_swaps()} skel-agree={frac:.4f} "
          f"max|U|={np.abs(U).max():.3f} err_gpu={eg:.3e} err_oracle={eo:.3e}")
    assert info["srrqr_swaps"] > 0 and o.srrqr_swaps() > 0
    assert np.abs(U).max() <= f * (1 + 1e-9)
    assert frac >= 0.99
    assert eg <= 2.0 * eo + 1e-15
    g.close()


def test_srrqr_option_validated():
    pts = synth.uniform_cube(1000, 3, seed=1)
    for bad in (-1.0, 0.5, float("inf")):
        with pytest.raises(P.H2Error):
            P.H2Matrix(torch.from_numpy(pts).cuda(), 1, [], 1e-6, 32, srrqr_f=bad)
