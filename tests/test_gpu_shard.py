"""Sharded build on one GPU: R virtual ranks are host threads of this process,
joined by the LOCAL transport (host barrier + device copies; no kernel waits on another rank).
Every rank's results must be bit-identical to the single-GPU build on the nodes it computed, the
exchanged X^* and skeletons must be complete, the ranks' stored blocks must partition the
single-GPU block set, and the collective matvec must equal the single-GPU matvec."""
import itertools
import threading

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2206_01885_b200 as P  # noqa: E402

_key = itertools.count(1000)


def build_sharded(pts, R, kid, kp, id_tol, q, tau=0.5, storage=P.H2_STORE_ALL, reduct=P.H2_REDUCT_VOLUME):
    key = next(_key)
    X = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
    out, errs = [None] * R, []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            comm = P.H2Comm.local(R, rank, key)
            st = torch.cuda.Stream()
            out[rank] = P.H2Matrix(X, kid, kp, id_tol, q, tau, storage=storage, stream=st, timing=True, comm=comm,
                                   reduct=reduct)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return out


def collective_matvec(hs, x):
    ys, errs = [None] * len(hs), []

    def run(r):
        try:
            with torch.cuda.stream(hs[r].stream):
                ys[r] = hs[r].matvec(x).cpu().numpy()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(len(hs))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return ys


def slots(g, name):
    off, idx = g.export(name + "_OFF"), g.export(name + "_IDX")
    return [idx[off[i]:off[i + 1]] for i in range(len(off) - 1)]


def u_blocks(g):
    off, U = g.export("U_OFF"), g.export("U")
    return [U[off[i]:off[i + 1]] for i in range(len(off) - 1)]


CASES = [  # cfg, n, q override, ranks
    (1, 8192, None, 2),
    (1, 8192, None, 3),
    (4, 60000, None, 4),
    (3, 30000, None, 2),
    (2, 40000, 64, 8),
]


@pytest.mark.parametrize("R", [2, 4, 8])
def test_sharded_lists_work_falls_as_one_over_ranks(R):
    """a4 sharded: every rank builds the lists of its own rows only, so the largest per-rank pair
    count falls roughly as 1/R (the top levels above the cut are the only redundant rows)."""
    c = synth.CONFIGS[4]
    pts = synth.points(4, 1 << 19)
    kp = list(c["params"])
    ref = P.H2Matrix(torch.from_numpy(pts).cuda(), c["kernel"], kp, c["id_tol"], c["q"], c["tau"],
                     storage=P.H2_STORE_ON_THE_FLY, timing=True)
    total = ref.info()["n_il"] + ref.info()["n_nf"]
    hs = build_sharded(pts, R, c["kernel"], kp, c["id_tol"], c["q"], c["tau"], storage=P.H2_STORE_ON_THE_FLY)
    per = [g.info()["n_il"] + g.info()["n_nf"] for g in hs]
    # the redundant rows: the interaction lists of the nodes above the cut (every rank's HiDR-down
    # of the top levels needs them); everything else is split over the ranks
    cut = hs[0].export("SHARD")[2]
    lv = ref.export("NODES").reshape(-1, 7)[:, 0]
    il_off = ref.export("IL_OFF")
    top = int(sum(il_off[i + 1] - il_off[i] for i in np.flatnonzero(lv < cut)))
    print(f"R={R}: pairs per rank {per} of {total} (max {max(per) / total:.3f} of the total, 1/R = {1 / R:.3f}, "
          f"redundant top rows {top}); lists ms {[round(g.info()['stage_ms']['lists'], 2) for g in hs]}")
    assert sum(per) == total + (R - 1) * top
    assert max(per) <= 1.2 * (total - top) / R + top
    for g in hs:
        g.close()


@pytest.mark.parametrize("cfg,n,q,R", CASES)
def test_sharded_equals_single_gpu(cfg, n, q, R):
    c = synth.CONFIGS[cfg]
    q = q or c["q"]
    kp = list(c["params"])
    pts = synth.points(cfg, n)
    X = torch.from_numpy(pts).cuda()
    ref = P.H2Matrix(X, c["kernel"], kp, c["id_tol"], q, c["tau"], storage=P.H2_STORE_ALL, timing=True)
    hs = build_sharded(pts, R, c["kernel"], kp, c["id_tol"], q, c["tau"])
    info = ref.info()
    depth = info["depth"]
    xs_ref, ys_ref, sk_ref, u_ref = slots(ref, "XS"), slots(ref, "YS"), slots(ref, "SK"), u_blocks(ref)
    k_ref = ref.export("K")
    plo, computed = [], np.zeros(info["nnodes"], int)
    cut = None
    for r, g in enumerate(hs):
        sh = g.export("SHARD")
        assert sh[0] == R and sh[1] == r
        cut = sh[2] if cut is None else cut
        assert sh[2] == cut
        plo.append((sh[3], sh[4]))
        rng = sh[5:].reshape(depth + 1, 2)
        gi = g.info()
        assert gi["r"] == info["r"] and gi["nnodes"] == info["nnodes"]
        # exchanged: X^* and the skeletons of EVERY node equal the single-GPU build
        assert all(np.array_equal(a, b) for a, b in zip(slots(g, "XS"), xs_ref))
        assert np.array_equal(g.export("K"), k_ref)
        assert all(np.array_equal(a, b) for a, b in zip(slots(g, "SK"), sk_ref))
        ys, U = slots(g, "YS"), u_blocks(g)
        # a4 sharded: the rank's lists are the single-GPU lists restricted to the rows it needs
        # (interaction lists: every node above the cut and its own range below; nearfield lists: the
        # leaves whose first point lies in its point range); the other rows are empty
        nodes_ = ref.export("NODES").reshape(-1, 7)
        for nm in ("IL", "NF"):
            mine, full = slots(g, nm), slots(ref, nm)
            need = np.zeros(info["nnodes"], bool)
            for lvl in range(depth + 1):
                lo, hi = rng[lvl]
                need[lo:hi] = True
            if nm == "NF":
                need = (nodes_[:, 1] >= sh[3]) & (nodes_[:, 1] < sh[4])
            for i in range(info["nnodes"]):
                assert np.array_equal(mine[i], full[i] if need[i] else full[i][:0]), (nm, r, i)
        for lvl in range(depth + 1):
            lo, hi = rng[lvl]
            for i in range(lo, hi):  # the nodes this rank computed: Y^* and U bit for bit
                computed[i] += 1
                assert np.array_equal(ys[i], ys_ref[i]), (r, i)
                assert np.array_equal(U[i], u_ref[i]), (r, i)
    # levels >= cut: every node computed by exactly one rank; above: by all
    nodes = ref.export("NODES").reshape(-1, 7)
    lv = nodes[:, 0]
    assert np.all(computed[lv >= cut] == 1) and np.all(computed[lv < cut] == R)
    # block rows: the point ranges tile [0, n); the stored blocks partition the single-GPU set
    plo.sort()
    assert plo[0][0] == 0 and plo[-1][1] == n and all(plo[t][1] == plo[t + 1][0] for t in range(R - 1))
    assert sum(g.info()["coupling_entries"] for g in hs) == info["coupling_entries"]
    assert sum(g.info()["nearfield_entries"] for g in hs) == info["nearfield_entries"]
    # collective matvec == single-GPU matvec (summation order differs only)
    x = torch.from_numpy(synth.matvec_vector(cfg, n)).cuda()
    y_ref = ref.matvec(x).cpu().numpy()
    for y in collective_matvec(hs, x):
        assert np.linalg.norm(y - y_ref) <= 1e-12 * np.linalg.norm(y_ref)
    print(f"cfg{cfg} n={n} R={R}: cut={cut} ranges={plo} "
          f"build ms={[round(g.info()['stage_ms']['build'], 2) for g in hs]}")
    for g in hs:
        g.close()
    ref.close()


def test_sharded_on_the_fly_and_single_leaf():
    pts = synth.uniform_cube(40, 3, seed=5)  # one leaf: rank 0 owns it, rank 1 has nothing
    hs = build_sharded(pts, 2, 1, [], 1e-6, 64, storage=P.H2_STORE_ON_THE_FLY)
    x = torch.from_numpy(synth.matvec_vector(1, 40)).cuda()
    ref = P.H2Matrix(torch.from_numpy(pts).cuda(), 1, [], 1e-6, 64, storage=P.H2_STORE_ON_THE_FLY)
    y_ref = ref.matvec(x).cpu().numpy()
    for y in collective_matvec(hs, x):
        np.testing.assert_allclose(y, y_ref, rtol=1e-13, atol=1e-13 * np.abs(y_ref).max())


def test_sharded_rebuild_equals_single_gpu_rebuild():
    """HiDR once for all on a sharded handle: every rank rebuilds for another kernel (collective)."""
    c = synth.CONFIGS[1]
    pts = synth.points(1, 8192)
    X = torch.from_numpy(pts).cuda()
    ref = P.H2Matrix(X, 1, [], 1e-6, c["q"], storage=P.H2_STORE_ALL).rebuild(2, [0.5], 1e-6, P.H2_STORE_ALL)
    hs = build_sharded(pts, 2, 1, [], 1e-6, c["q"])
    out, errs = [None, None], []

    def run(r):
        try:
            with torch.cuda.stream(hs[r].stream):
                out[r] = hs[r].rebuild(2, [0.5], 1e-6, P.H2_STORE_ALL)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    assert all(np.array_equal(g.export("SK_IDX"), ref.export("SK_IDX")) for g in out)
    x = torch.from_numpy(synth.matvec_vector(1, 8192)).cuda()
    y_ref = ref.matvec(x).cpu().numpy()
    for y in collective_matvec(out, x):
        assert np.linalg.norm(y - y_ref) <= 1e-12 * np.linalg.norm(y_ref)


@pytest.mark.parametrize("reduct", [1, 2])
def test_sharded_fps_equals_single_gpu_fps(reduct):
    """Farthest point sampling (reading C6) and the surface reduction (C7) on a sharded build: every
    rank's X^* / Y^* and skeletons equal the single-GPU build, and the collective matvec equals its
    matvec."""
    c = synth.CONFIGS[4]
    pts = synth.points(4, 30000)
    X = torch.from_numpy(pts).cuda()
    kp = list(c["params"])
    ref = P.H2Matrix(X, c["kernel"], kp, c["id_tol"], c["q"], c["tau"], storage=P.H2_STORE_ALL, reduct=reduct)
    hs = build_sharded(pts, 3, c["kernel"], kp, c["id_tol"], c["q"], c["tau"], reduct=reduct)
    depth = ref.info()["depth"]
    xs_ref, ys_ref, sk_ref = slots(ref, "XS"), slots(ref, "YS"), slots(ref, "SK")
    for g in hs:  # exchanged: X^* and skeletons of every node; Y^* of the nodes the rank computed
        assert all(np.array_equal(a, b) for a, b in zip(slots(g, "XS"), xs_ref))
        assert all(np.array_equal(a, b) for a, b in zip(slots(g, "SK"), sk_ref))
        ys, rng = slots(g, "YS"), g.export("SHARD")[5:].reshape(depth + 1, 2)
        for lo, hi in rng:
            assert all(np.array_equal(ys[i], ys_ref[i]) for i in range(lo, hi))
    x = torch.from_numpy(synth.matvec_vector(4, 30000)).cuda()
    y_ref = ref.matvec(x).cpu().numpy()
    for y in collective_matvec(hs, x):
        assert np.linalg.norm(y - y_ref) <= 1e-12 * np.linalg.norm(y_ref)
