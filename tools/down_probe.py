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
