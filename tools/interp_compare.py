"""PAPER section 6.3 on the GPU: approximation error vs memory of the data-driven H^2
(id_tol swept) and the interpolation-based H^2 (h2_options.interp_p swept, Eq. (2.2)) for the four
kernels of Table 1 on the 3-sphere dataset with n = 20000.

Memory = 8 bytes x the stored entries of U (leaves + transfers), the coupling blocks and the
nearfield blocks, symmetric blocks once.  Error = ||K~x - Kx|| / ||Kx|| on 1024 seeded
rows, dense K x by the oracle (test infrastructure; the builds are the CUDA path).
Usage: python tools/interp_compare.py [out.md]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2206_01885_b200 as P  # noqa: E402
import synth  # noqa: E402

N, Q, SEED = 20000, 64, 2206
KERNELS = [("kappa1 1/|x-y|", P.H2_KERNEL_COULOMB, ()), ("kappa2 exp(-|x-y|^2)", P.H2_KERNEL_GAUSSIAN, (1.0,)),
           ("kappa3 cos(x.y)", P.H2_KERNEL_COSDOT, ()), ("kappa4 bump", P.H2_KERNEL_BUMP, ())]
TOLS = [1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 1e-7, 1e-8, 1e-10]
PS = [2, 3, 4, 5, 6, 7]


def main(out):
    oracle.build()
    pts = synth.three_spheres(N, SEED)
    rows = np.sort(np.random.default_rng(SEED + 1).choice(N, 1024, replace=False)).astype(np.int64)
    x = np.random.default_rng(SEED + 2).standard_normal(N)
    xg = torch.from_numpy(x).cuda()
    dpts = torch.from_numpy(pts).cuda()
    recs = []
    for name, kid, kp in KERNELS:
        yd = oracle.dense_rows(pts, kid, kp[0] if kp else 0.0, x, rows)
        runs = [("data-driven", dict(id_tol=t)) for t in TOLS] + [("interpolation", dict(interp_p=p)) for p in PS]
        for method, kw in runs:
            t0 = time.perf_counter()
            g = P.H2Matrix(dpts, kid, kp, kw.get("id_tol", 1e-6), Q, 0.5, storage=P.H2_STORE_ALL, timing=True,
                           interp_p=kw.get("interp_p", 0))
            info = g.info()
            u = int(g.export("U_OFF")[-1])
            y = g.matvec(xg).cpu().numpy()[rows]
            err = float(np.linalg.norm(y - yd) / np.linalg.norm(yd))
            mem = 8 * (u + info["coupling_entries"] + info["nearfield_entries"])
            rec = dict(kernel=name, method=method, **kw, r=info["r"], kmax=info["kmax"], err=err, mem_mb=mem / 2 ** 20,
                       u_mb=8 * u / 2 ** 20, coupling_mb=8 * info["coupling_entries"] / 2 ** 20,
                       nearfield_mb=8 * info["nearfield_entries"] / 2 ** 20, build_ms=info["stage_ms"]["build"],
                       wall_s=time.perf_counter() - t0)
            g.close()
            recs.append(rec)
            print(json.dumps(rec), flush=True)
    with open(out, "w") as f:
        f.write("# Section 6.3 on B200: error vs memory, data-driven vs interpolation (3-sphere, n = 20000)\n\n")
        f.write(f"`python tools/interp_compare.py` (q = {Q}, tau = 0.5, every block stored; error on 1024 seeded rows "
                "against the oracle's dense K x; memory = 8 B x stored entries of U + coupling + nearfield, symmetric "
                "blocks once). PAPER section 6.3 (P:1069-1098), Fig. mem; kernels of Table 1 (P:914-926).\n\n")
        for name, _, _ in KERNELS:
            f.write(f"## {name}\n\n| method | id_tol / p | r | k_max | rel. error | memory MB | U MB | coupling MB | "
                    "nearfield MB | build ms |\n|---|---|---|---|---|---|---|---|---|---|\n")
            for r in recs:
                if r["kernel"] != name:
                    continue
                par = f"id_tol {r['id_tol']:.0e}" if "id_tol" in r else f"p = {r['interp_p']}"
                f.write(f"| {r['method']} | {par} | {r['r']} | {r['kmax']} | {r['err']:.3e} | {r['mem_mb']:.1f} | "
                        f"{r['u_mb']:.1f} | {r['coupling_mb']:.1f} | {r['nearfield_mb']:.1f} | {r['build_ms']:.2f} |\n")
            f.write("\n")
        f.write("```\n" + "\n".join(json.dumps(r) for r in recs) + "\n```\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/interp_vs_dd.md")
