"""One build of a config + a few matvecs (for per-kernel launch lists of the matvec under ncu)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_01885_b200 as P  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = synth.CONFIGS[cfg]
X = torch.from_numpy(synth.points(cfg)).cuda()
g = P.H2Matrix(X, c["kernel"], list(c["params"]), c["id_tol"], c["q"], c["tau"], storage=P.H2_STORE_ALL)
x = torch.randn(len(X), dtype=torch.float64, device="cuda")
for _ in range(3):
    y = g.matvec(x)
torch.cuda.synchronize()
print("ok", float(y.norm()))
