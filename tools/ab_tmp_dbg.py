import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import synth, paper_2206_01885_b200 as P
from test_gpu_shard import build_sharded, slots
c = synth.CONFIGS[3]; n = 30000; R = 2
pts = synth.points(3, n)
ref = P.H2Matrix(torch.from_numpy(pts).cuda(), c["kernel"], list(c["params"]), c["id_tol"], c["q"], 0.5, storage=P.H2_STORE_ALL, timing=True)
hs = build_sharded(pts, R, c["kernel"], list(c["params"]), c["id_tol"], c["q"], 0.5)
nodes = ref.export("NODES").reshape(-1, 7)
for r, g in enumerate(hs):
    sh = g.export("SHARD"); depth = ref.info()["depth"]; rng = sh[5:].reshape(depth + 1, 2)
    print("rank", r, "cut", sh[2], "p", sh[3], sh[4], "ranges", rng.tolist())
    for nm in ("IL", "NF", "YS", "XS", "SK"):
        a, b = slots(g, nm), slots(ref, nm)
        bad = [i for i in range(len(a)) if not np.array_equal(a[i], b[i])]
        own = np.zeros(len(a), bool)
        for l in range(depth + 1): own[rng[l][0]:rng[l][1]] = True
        badown = [i for i in bad if own[i]]
        print(nm, "mismatch", len(bad), "of which owned", len(badown), badown[:10], [int(nodes[i,0]) for i in badown[:10]])
    k, kr = g.export("K"), ref.export("K")
    bad = np.flatnonzero(k != kr)
    print("K mismatch", len(bad), bad[:10], nodes[bad[:10], 0])
for r, g in enumerate(hs):
    a, b = slots(g, "IL"), slots(ref, "IL")
    an, bn = slots(g, "NF"), slots(ref, "NF")
    for i in ([40, 48, 197] if r == 0 else [9, 198, 688]):
        print("rank", r, "node", i, "level", nodes[i, 0], "leaf", nodes[i, 6], "begin", nodes[i, 1], "parent", nodes[i, 3])
        print("   IL rank", a[i].tolist()[:20], "ref", b[i].tolist()[:20])
        print("   NF rank", an[i].tolist()[:20], "ref", bn[i].tolist()[:20])
