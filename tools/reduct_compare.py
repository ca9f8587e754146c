"""The paper's DataReduct comparison (§5.2: FPS / volume / surface), on synthetic data
instead of the unavailable Dino set: for each reduction, the H^2 matvec relative error (1024
sampled rows against dense K x computed here with numpy) and the HiDR stage times, at the
calibrated r.

usage: python tools/reduct_compare.py [config ...]   (configs with d = 2 or 3; default 1 3 4)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_01885_b200 as P  # noqa: E402
import synth  # noqa: E402

NAMES = {P.H2_REDUCT_VOLUME: "volume", P.H2_REDUCT_FPS: "FPS", P.H2_REDUCT_SURFACE: "surface"}


def dense_rows(pts, kid, p, x, rows):
    """(K x)[rows] by direct numpy evaluation (Coulomb / Gaussian / Matern-3/2)."""
    out = np.empty(len(rows))
    for t, i in enumerate(rows):
        r = np.sqrt(((pts - pts[i]) ** 2).sum(1))
        if kid == 1:
            k = np.where(r > 0, 1.0 / np.where(r > 0, r, 1.0), 0.0)
        elif kid == 2:
            k = np.exp(-(r / p) ** 2)
        else:
            a = np.sqrt(3.0) * r / p
            k = (1.0 + a) * np.exp(-a)
        out[t] = k @ x
    return out


def main(cfgs):
    print("| config | n | reduct | r | mean \\|Y*\\| | HiDR up ms | HiDR down ms | matvec rel. error |")
    print("|---|---|---|---|---|---|---|---|")
    for cfg in cfgs:
        c = synth.CONFIGS[cfg]
        n = min(c["n"], 262144)
        pts = synth.points(cfg, n)
        X = torch.from_numpy(pts).cuda()
        kp = list(c["params"])
        x = synth.matvec_vector(cfg, n)
        rows = synth.sample_rows(cfg, n)
        yd = dense_rows(pts, c["kernel"], kp[0] if kp else 0.0, x, rows)
        for red in (P.H2_REDUCT_VOLUME, P.H2_REDUCT_FPS, P.H2_REDUCT_SURFACE):
            g = P.H2Matrix(X, c["kernel"], kp, c["id_tol"], c["q"], c["tau"], storage=P.H2_STORE_ON_THE_FLY,
                           timing=True, reduct=red)
            g2 = P.H2Matrix(X, c["kernel"], kp, c["id_tol"], c["q"], c["tau"], storage=P.H2_STORE_ON_THE_FLY,
                            timing=True, reduct=red)  # second build: warm timings
            info = g2.info()
            y = g2.matvec(torch.from_numpy(x).cuda()).cpu().numpy()[rows]
            err = np.linalg.norm(y - yd) / np.linalg.norm(yd)
            ys = np.diff(g2.export("YS_OFF"))
            print(f"| {cfg} | {n} | {NAMES[red]} | {info['r']} | {ys[ys > 0].mean():.0f} | "
                  f"{info['stage_ms']['hidr_up']:.2f} | {info['stage_ms']['hidr_down']:.2f} | {err:.2e} |", flush=True)
            g.close()
            g2.close()


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 3, 4])
