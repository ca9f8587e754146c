"""Diagnostic: the shape of the top-down HiDR work of one config -- per level: nodes, |T_i|
distribution, grid size, algorithmic vs evaluated distances (not a bench)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_01885_b200 as P  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
c = synth.CONFIGS[cfg]
X = torch.from_numpy(synth.points(cfg)).cuda()
g = P.H2Matrix(X, c["kernel"], list(c["params"]), c["id_tol"], c["q"], c["tau"], storage=P.H2_STORE_ON_THE_FLY,
               timing=True)
inf = g.info()
print({k: v for k, v in inf.items()})
nodes = g.export("NODES").reshape(-1, 7)
lvl, par = nodes[:, 0], nodes[:, 3]
ilo, ili = g.export("IL_OFF"), g.export("IL_IDX")
xo, yo = g.export("XS_OFF"), g.export("YS_OFF")
xc, yc = np.diff(xo), np.diff(yo)
r = inf["r"]
for L in range(int(lvl.max()) + 1):
    ids = np.nonzero(lvl == L)[0]
    tot = []
    nil = []
    for i in ids:
        t = yc[par[i]] if par[i] >= 0 else 0
        js = ili[ilo[i]:ilo[i + 1]]
        t += int(xc[js].sum())
        tot.append(t)
        nil.append(len(js))
    tot = np.array(tot)
    nil = np.array(nil)
    big = tot > r
    print(f"L{L}: nodes {len(ids)} |IL| mean {nil.mean():.1f} max {nil.max()} |T| mean {tot.mean():.0f} "
          f"max {tot.max()} >r {big.sum()} alg(G*T>r) {float((tot[big]).sum()) * r:.3e}")
# the ID sweep's blocks per level: |Y*| x |Xbar| and rank k
yc_all = np.diff(g.export("YS_OFF"))
xb = g.export("XBAR_N")
kk = g.export("K")
for L in range(int(lvl.max()) + 1):
    ids = np.nonzero(lvl == L)[0]
    e = yc_all[ids].astype(np.int64) * xb[ids]
    ek = e * kk[ids]
    big = e * 8 > 100 * 1024
    print(f"ID L{L}: nodes {len(ids)} entries {e.sum():.3e} max {e.max()} |Y*| mean {yc_all[ids].mean():.0f} "
          f"|Xbar| mean {xb[ids].mean():.0f} max {xb[ids].max()} k mean {kk[ids].mean():.1f} max {kk[ids].max()} "
          f"sum k*entries {ek.sum():.3e} global-path nodes {big.sum()} their k*entries {ek[big].sum():.3e}")
    if e.sum() > 0:
        for lim in (12800, 28000, 100000, 200000, 400000, 800000):
            sel = e <= lim
            print(f"    entries <= {lim}: nodes {sel.sum()} share of k*entries {ek[sel].sum() / max(1, ek.sum()):.3f}")
