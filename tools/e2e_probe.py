"""Where the end-to-end (host points) build time goes: device-resident build vs host build vs the
plain H2D copy of the same bytes (A/B only)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2206_01885_b200 as P  # noqa: E402
import synth  # noqa: E402

cfg = 4
c = synth.CONFIGS[cfg]
pts = synth.points(cfg)
n = len(pts)
X = torch.from_numpy(pts).cuda()
pinned = torch.from_numpy(pts).pin_memory()
st = torch.cuda.Stream()


def build(host):
    o = P.h2_options_default()
    o.storage = P.H2_STORE_ALL
    o.stream = st.cuda_stream
    o.points_on_host = 1 if host else 0
    o.timing = 1
    ptr = pinned.data_ptr() if host else X.data_ptr()
    t0 = time.perf_counter()
    h = P.h2_build(ptr, n, c["d"], c["kernel"], list(c["params"]), c["id_tol"], c["q"], c["tau"], o)
    t1 = time.perf_counter()
    k = P.h2_export(h, "K")
    t2 = time.perf_counter()
    info = P.h2_info(h)
    P.h2_free(h)
    return (t1 - t0) * 1e3, (t2 - t1) * 1e3, info["stage_ms"]["build"]


for host in (False, True, False, True, False, True):
    print("host" if host else "dev ", ["%.2f" % v for v in build(host)])
dst = torch.empty_like(X)
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dst.copy_(pinned, non_blocking=True)
    torch.cuda.synchronize()
    print("h2d copy %.2f ms" % ((time.perf_counter() - t0) * 1e3))
