"""a8 parity per code path: every ID path of the CUDA sweep against the fp64 oracle, element by
element on U / stacked R_c (Eq.(4.1): K_{X Y*} = P [I; G] K_{X^ Y*}).

The sweep picks a path per node by block size (H2_EXPORT_ID_PATH): the staged shared-memory
classes 0..5, the mid class 6 (lean layout, 256 threads, two CTAs per SM), the lean shared-memory class 7, the global-memory CTA 8 / 9, the thread-block
cluster 10, and (H2_ID_WARP_MIN) one warp per node 11.  Each case runs the GPU build in a subprocess (the path thresholds are read once per
process from the environment) and compares it with the oracle on the same seeded points:
  * r, tree, lists, X^*, Y^* bit-exact;
  * skeleton agreement (same k and the same pivot sequence) >= 0.99 -- pivots may differ only at
    near-ties (BASELINE north_star);
  * on the nodes whose skeleton sequence agrees, U_i equals the oracle's element by element
    (rows matched by point index, columns in pivot order) within max(1e-10, 2e-15 / id_tol)
    max(1, max|U_i|): U = (R11^-1 R12)^T amplifies the O(1e-16) rounding differences of the two
    factorisations by the condition of R11, which the stop rule |R_kk| >= id_tol |R11| bounds by
    ~1 / id_tol (times a modest growth factor);
  * the matvec error within 2x the oracle's, GPU and oracle matvec within 10 id_tol.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_DUMP = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2206_01885_b200 as P, synth
cfg, n, q, out = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
c = synth.CONFIGS[cfg]
X = torch.from_numpy(synth.points(cfg, n)).cuda()
g = P.H2Matrix(X, c["kernel"], list(c["params"]), c["id_tol"], q, c["tau"], storage=P.H2_STORE_ALL, timing=True)
x = torch.from_numpy(synth.matvec_vector(cfg, n)).cuda()
names = ("PERM", "NODES", "IL_OFF", "IL_IDX", "NF_OFF", "NF_IDX", "XS_OFF", "XS_IDX", "YS_OFF", "YS_IDX", "K",
         "SK_OFF", "SK_IDX", "U_OFF", "U", "XBAR_N", "ID_PATH")
np.savez(out, r=g.info()["r"], id_ms=g.info()["stage_ms"]["id_sweep"], y=g.matvec(x).cpu().numpy(),
         **{k: g.export(k) for k in names})
"""

STRUCT = [("PERM", oracle.PERM), ("IL_OFF", oracle.IL_OFF), ("IL_IDX", oracle.IL_IDX), ("NF_OFF", oracle.NF_OFF),
          ("NF_IDX", oracle.NF_IDX), ("XS_OFF", oracle.XS_OFF), ("XS_IDX", oracle.XS_IDX),
          ("YS_OFF", oracle.YS_OFF), ("YS_IDX", oracle.YS_IDX)]


def _xbar(nodes, k, so, si, i):
    """Xbar_i as tree-order point indices: the leaf's points, or the children's skeletons in child
    order (Alg. 2 line 11)."""
    lvl, b, e, par, fc, nc, leaf = nodes[i]
    if leaf:
        return np.arange(b, e)
    return np.concatenate([si[so[c]:so[c + 1]] for c in range(fc, fc + nc)] or [np.zeros(0, np.int64)])


CASES = [  # name, config, n, q, environment, {path: minimum node count}
    ("cfg1_staged", 1, 8192, 64, {"H2_ID_WARP_MIN": "0"}, {"staged": 100}),
    ("cfg4_staged", 4, 60000, 256, {"H2_ID_WARP_MIN": "0"}, {"staged": 200}),
    ("cfg3_lean_global", 3, 30000, 128, {"H2_ID_WARP_MIN": "0"}, {"lean": 20}),
    ("cfg2_tol1e-8", 2, 60000, 200, {"H2_ID_WARP_MIN": "0"}, {"staged": 20, "mid": 20}),
    ("cfg5_cluster", 5, 32768, 256, {"H2_ID_CLMIN": "1", "H2_ID_WARP_MIN": "0"}, {"cluster": 50, "lean": 50}),
    ("cfg5_global", 5, 32768, 256, {"H2_ID_CLUSTER": "0", "H2_ID_WARP_MIN": "0"}, {"global": 50}),
    # the warp-per-node path (off by default: measured slower; here every level)
    ("cfg1_warp", 1, 8192, 64, {"H2_ID_WARP_MIN": "1"}, {"warp": 500}),
    ("cfg4_warp", 4, 60000, 256, {"H2_ID_WARP_MIN": "1"}, {"warp": 700}),
    ("cfg2_warp", 2, 60000, 200, {"H2_ID_WARP_MIN": "1"}, {"warp": 500}),
    ("cfg3_warp", 3, 30000, 128, {"H2_ID_WARP_MIN": "1"}, {"warp": 500}),
    ("cfg5_warp", 5, 32768, 256, {"H2_ID_WARP_MIN": "1"}, {"warp": 500}),
    # the unblocked CPQR (H2_ID_PANEL=0) on the same shapes: both factorisations meet the same bar
    ("cfg3_unblocked", 3, 30000, 128, {"H2_ID_PANEL": "0", "H2_ID_WARP_MIN": "0"}, {"lean": 20}),
    ("cfg2_unblocked", 2, 60000, 200, {"H2_ID_PANEL": "0", "H2_ID_WARP_MIN": "0"}, {"staged": 20, "mid": 20}),
]

PATHS = {"staged": range(0, 6), "mid": (6,), "lean": (7,), "global": (8, 9), "cluster": (10,), "warp": (11,)}


@pytest.mark.parametrize("name,cfg,n,q,env,need", CASES)
def test_id_path_parity_elementwise(name, cfg, n, q, env, need, tmp_path):
    c = synth.CONFIGS[cfg]
    out = str(tmp_path / "g.npz")
    subprocess.run([sys.executable, "-c", _DUMP, ROOT, str(cfg), str(n), str(q), out],
                   env=dict(os.environ, **env), check=True, timeout=900)
    g = np.load(out)
    pts = synth.points(cfg, n)
    kp = c["params"][0] if c["params"] else 0.0
    o = oracle.OracleH2(pts, q, c["tau"])
    r = o.build(c["kernel"], kp, c["id_tol"])
    assert int(g["r"]) == r
    for gname, oname in STRUCT:
        assert np.array_equal(g[gname], o.export(oname)), gname
    nodes = g["NODES"].reshape(-1, 7)
    assert np.array_equal(nodes, o.export(oracle.NODES).reshape(-1, 7))
    path = g["ID_PATH"]
    counts = {p: int(np.isin(path, PATHS[p]).sum()) for p in PATHS}
    for p, m in need.items():
        assert counts[p] >= m, (p, counts)
    gk, ok = g["K"], o.export(oracle.K)
    gso, gsi = g["SK_OFF"], g["SK_IDX"]
    oso, osi = o.skeletons()
    guo, gU = g["U_OFF"], g["U"]
    ouo, oU = o.export(oracle.U_OFF), o.export(oracle.U)
    nodes_b = np.flatnonzero((gk > 0) | (ok > 0))
    agree = [i for i in nodes_b if gk[i] == ok[i] and np.array_equal(gsi[gso[i]:gso[i + 1]], osi[oso[i]:oso[i + 1]])]
    frac = len(agree) / max(1, len(nodes_b))
    worst = {p: 0.0 for p in PATHS}
    compared = {p: 0 for p in PATHS}
    for i in agree:
        k = int(gk[i])
        xg = _xbar(nodes, gk, gso, gsi, i)
        xo = _xbar(nodes, ok, oso, osi, i)
        assert len(xg) == len(xo) == len(set(xg.tolist())) and set(xg.tolist()) == set(xo.tolist())
        Ug = gU[guo[i]:guo[i + 1]].reshape(k, len(xg)).T          # nx x k, rows in GPU Xbar order
        Uo = oU[ouo[i]:ouo[i + 1]].reshape(k, len(xo)).T
        order = np.argsort(xg)
        Ug = Ug[order]
        Uo = Uo[np.argsort(xo)]
        err = np.abs(Ug - Uo).max() / max(1.0, np.abs(Uo).max())
        pname = next(p for p in PATHS if path[i] in PATHS[p])
        worst[pname] = max(worst[pname], err)
        compared[pname] += 1
    # the matvec on the 1024 seeded rows (all rows when n <= 16384)
    x = synth.matvec_vector(cfg, n)
    rows = synth.sample_rows(cfg, n)
    yd = oracle.dense_rows(pts, c["kernel"], kp, x, rows)
    yo = o.matvec(x, rows)
    yg = g["y"][rows]
    eg = np.linalg.norm(yg - yd) / np.linalg.norm(yd)
    eo = np.linalg.norm(yo - yd) / np.linalg.norm(yd)
    ag = np.linalg.norm(yg - yo) / np.linalg.norm(yo)
    print(f"{name}: r={r} paths={counts} skel-agree={frac:.4f} U-compared={compared} worst={worst} "
          f"err_gpu={eg:.3e} err_oracle={eo:.3e} gpu-vs-oracle={ag:.3e} id_ms={float(g['id_ms']):.2f}")
    assert frac >= 0.99
    for p, m in need.items():
        assert compared[p] >= min(m, counts[p]) // 2, (p, compared)
    tol_u = max(1e-10, 2e-15 / c["id_tol"])
    for p in PATHS:
        assert worst[p] <= tol_u, (p, worst[p], tol_u)
    assert eg <= 2.0 * eo + 1e-15
    assert ag <= 10 * c["id_tol"]


def test_nonfinite_points_rejected():
    """H2_ERR_NONFINITE: a NaN or an Inf coordinate fails the build, nothing is returned."""
    import paper_2206_01885_b200 as P
    for bad in (np.nan, np.inf, -np.inf):
        pts = synth.uniform_cube(1000, 3, seed=1)
        pts[517, 1] = bad
        with pytest.raises(P.H2Error):
            P.H2Matrix(torch.from_numpy(pts).cuda(), 1, [], 1e-6, 32)
        assert P.last_error()[0] == -2, P.last_error()


def test_matvec_rejects_bad_vectors():
    """h2_matvec_ex: a length mismatch is H2_ERR_DIM_MISMATCH; the binding refuses
    non-float64 / non-contiguous / host vectors before any device work."""
    import paper_2206_01885_b200 as P
    pts = synth.uniform_cube(2000, 3, seed=2)
    g = P.H2Matrix(torch.from_numpy(pts).cuda(), 1, [], 1e-6, 32)
    x = torch.zeros(2001, dtype=torch.float64, device="cuda")
    y = torch.zeros(2001, dtype=torch.float64, device="cuda")
    with pytest.raises(P.H2Error):
        P.h2_matvec(g.h, x.data_ptr(), y.data_ptr(), x.numel())
    assert P.last_error()[0] == -6
    for bad in (torch.zeros(2000, dtype=torch.float32, device="cuda"), torch.zeros(4000, dtype=torch.float64,
                                                                                     device="cuda")[::2],
                torch.zeros(2000, dtype=torch.float64)):
        with pytest.raises(P.H2Error):
            g.matvec(bad)
    y = g.matvec(torch.ones(2000, dtype=torch.float64, device="cuda"))
    assert torch.isfinite(y).all()
    g.close()
