"""Diagnostic: repeated builds of one config printing the per-stage device times (not a bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("ALT_PKG"): sys.path.insert(0, os.environ["ALT_PKG"])
import torch, numpy as np, synth
import paper_2206_01885_b200 as P
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] not in ("", "0") else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
c = synth.CONFIGS[cfg]
pts = torch.from_numpy(synth.points(cfg, n)).cuda()
n = pts.shape[0]
st = torch.cuda.Stream()
for i in range(reps):
    o = P.h2_options_default(); o.storage = int(os.environ.get("H2_STORAGE", P.H2_STORE_ALL)); o.timing = 1; o.stream = st.cuda_stream
    t0 = time.perf_counter()
    h = P.h2_build(pts.data_ptr(), n, c["d"], c["kernel"], list(c["params"]), c["id_tol"], c["q"], c["tau"], o)
    t1 = time.perf_counter()
    inf = P.h2_info(h)
    print(f"rep {i} wall {1e3*(t1-t0):.1f} ms", {k: round(v, 2) for k, v in inf["stage_ms"].items()}, flush=True)
    P.h2_free(h)
print(P.__file__)
