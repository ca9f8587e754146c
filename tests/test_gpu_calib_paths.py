"""a5 calibration (Algorithm 2 line 2; readings E1-E6) on every code path of the
CUDA trials against the fp64 oracle: the calibrated r must equal the oracle's bit for bit.

Paths (each read once per process, so every case runs the GPU build in a subprocess):
  * default: the trial CPQR on an 8-CTA thread-block cluster (calib_cpqr_cluster_kernel), for d >= 3 the
    speculative phase 1 concurrent with phase 0 and cancelled on the device once phase 0 passed a level;
  * H2_CAL_CLUSTER=0: one CTA per trial (panel CPQR on the block in global memory);
  * H2_CAL_MERGE=0: phase 1 after phase 0 on one stream (no cancellation needed).
Shapes: the five BASELINE configs at reduced n (the same point recipes), so levels with and without a
passing phase-0 trial, d = 2, 3, 5, and a pass-through budget (configs[2]: r = 7^3) all occur.
"""
import os
import subprocess
import sys

import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_R = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2206_01885_b200 as P, synth
cfg, n = int(sys.argv[2]), int(sys.argv[3])
c = synth.CONFIGS[cfg]
X = torch.from_numpy(synth.points(cfg, n)).cuda()
rs = []
for _ in range(3):  # repeated builds: an earlier build's cancelled phase 1 must not disturb the next
    g = P.H2Matrix(X, c["kernel"], list(c["params"]), c["id_tol"], c["q"], c["tau"], storage=P.H2_STORE_ON_THE_FLY)
    rs.append(g.info()["r"])
print("R", *rs)
"""

SHAPES = [(1, 8192), (2, 60000), (3, 40000), (4, 60000), (5, 32768)]
ENVS = [("cluster", {}), ("one_cta", {"H2_CAL_CLUSTER": "0"}), ("sequential", {"H2_CAL_MERGE": "0"})]


@pytest.mark.parametrize("cfg,n", SHAPES)
def test_calibrated_r_every_path(cfg, n):
    c = synth.CONFIGS[cfg]
    pts = synth.points(cfg, n)
    kp = c["params"][0] if c["params"] else 0.0
    o = oracle.OracleH2(pts, c["q"], c["tau"])
    r_oracle = o.calibrate(c["kernel"], kp, c["id_tol"])
    o.close()
    for name, env in ENVS:
        out = subprocess.run([sys.executable, "-c", _R, ROOT, str(cfg), str(n)], env=dict(os.environ, **env),
                             capture_output=True, text=True, timeout=600, check=True).stdout
        rs = [int(v) for v in next(l for l in out.splitlines() if l.startswith("R ")).split()[1:]]
        print(f"cfg{cfg} n={n} {name}: r={rs} oracle={r_oracle}")
        assert rs == [r_oracle] * len(rs), (name, rs, r_oracle)
