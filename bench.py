#!/usr/bin/env python
"""Benchmark of the B200 data-driven H^2 construction (arxiv 2206.01885).

One step = one complete h2_build (a1-a10: tree, lists, r calibration, HiDR up/down, ID sweep,
coupling + nearfield fill, every block stored) of BASELINE.json configs[3] (the largest
configuration whose stored H^2 fits one B200: n = 4,194,304 points, 2-D 16-Gaussian mixture,
Matern-3/2 l = 0.1, q = 256, id_tol 1e-6, tau 0.5).  configs[1] (1M cube, 1e-8) needs ~178 GB of
blocks and configs[4] ~198 GB, so neither fits; they are parity cases, not bench lines.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

Timing: W untimed warm-up builds, then K timed builds, each bracketed by CUDA events on the
library's stream with a barrier + synchronize on both sides of the timed region; L2 is flushed
(512 MiB write) before every timed build; max over ranks.  value = total points built by all
ranks / time (Mpoints/s).  Multi-GPU (torchrun, N > 1): ONE problem of the same config built by the
sharded path (subtree sharding below a cut level, X^* / skeleton allgathers over
NCCL, row-owned block fill; include/h2.h "sharded build") -- strong scaling, value = n / time.
--impl reference times the fp64 CPU oracle (the reference for this tier) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "H² construction Mpoints/s at fixed matvec rel. error; % of FP64/HBM roofline"
UNIT = "Mpoints/s"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "traffic.json")
FALLBACK_HBM_GBS = 6650.0
# FP64 vector peak of B200: 148 SMs x 64 FP64 lanes (DFMA = 2 flops) x clock; see DESIGN.md
FP64_LANES_PER_SM = 64


def workload_desc(cfg: int) -> str:
    c = synth.CONFIGS[cfg]
    kname = {1: "Coulomb", 2: "Gaussian", 3: "Matern-3/2", 7: "shifted multiquadric (non-symmetric)"}[c["kernel"]]
    par = f" param {c['params'][0]}" if c["params"] else ""
    src = f"BASELINE configs[{cfg - 1}]" if cfg <= 5 else "non-BASELINE extra config"
    return (f"{src}: {c['name']} n={c['n']} d={c['d']} {kname}{par} q={c['q']} "
            f"id_tol={c['id_tol']} tau={c['tau']}; full build a1-a10, all blocks stored symmetric-once")


FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "r02_fp64_peak.json")
# FP64 instructions per kernel evaluation (fill / ID block generation) and per
# squared distance + compare (HiDR, 3d - 1 DADD/DMUL + a compare)
KERNEL_FP64_INSTR = {1: 18, 2: 23, 3: 17, 4: 22, 5: 26, 6: 30, 7: 7}


def fp64_peak() -> dict:
    """Measured FP64 instruction rate (tools/micro/fp64_peak.cu, profiles/r02_fp64_peak.json), else
    the 148 SMs x 64 FP64 lanes x 1.965 GHz datasheet figure, saying which."""
    if os.path.exists(FP64_PEAK_FILE):
        try:
            j = json.load(open(FP64_PEAK_FILE))
            return {"instr_per_s": float(j["dfma_per_s"]), "tflops": float(j["fp64_tflops"]),
                    "source": "measured: tools/micro/fp64_peak.cu (profiles/r02_fp64_peak.json)"}
        except Exception:
            pass
    r = 148 * FP64_LANES_PER_SM * 1.965e9
    return {"instr_per_s": r, "tflops": 2 * r / 1e12, "source": "datasheet 148 SMs x 64 lanes x 1.965 GHz"}


def host_cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def build_roofline(c, info, k, xbar, ys_cnt, t_ms, hbm_gbs, fp64):
    """SURVEY §8(d) whole-build roofline: T_roof = sum over steps of max(B_s / BW_HBM, I_s / P_FP64)
    with the algorithmic bytes B_s and FP64 instructions I_s of each step (the top-down HiDR counted
    at the distances the exact pruned search evaluates), against the measured build time."""
    n, d = info["n"], c["d"]
    ck = KERNEL_FP64_INSTR.get(c["kernel"], 20) + (3 * d - 1)
    bw, P = hbm_gbs * 1e9, fp64["instr_per_s"]
    down = info["hidr_dist_done"] or max(0, info["hidr_dist_evals"] - info["hidr_up_evals"])
    cpqr = float(np.sum(2.0 * ys_cnt.astype(np.float64) * xbar.astype(np.float64) * k.astype(np.float64)))
    steps = {  # name: (bytes, fp64 instructions)
        "a1-a3 tree": (8.0 * n * d * 2 + 8 * 24.0 * n, 0.0),
        "a4 lists": (12.0 * (info["n_il"] + info["n_nf"]), 0.0),
        "a6 HiDR up": (0.0, 3.0 * d * info["hidr_up_evals"]),
        "a7 HiDR down": (0.0, 3.0 * d * down),
        "a8 ID": (8.0 * float(np.sum(xbar.astype(np.float64) * k)), ck * info["id_kernel_evals"] + cpqr),
        "a9 coupling": (8.0 * info["coupling_entries"], ck * info["coupling_entries"]),
        "a10 nearfield": (8.0 * info["nearfield_entries"], ck * info["nearfield_entries"]),
    }
    per = {nm: round(1e3 * max(b / bw, i / P), 4) for nm, (b, i) in steps.items()}
    t_roof = sum(per.values())
    return {"t_roof_ms": round(t_roof, 3), "t_measured_ms": round(t_ms, 3), "frac": round(t_roof / t_ms, 4),
            "per_step_floor_ms": per, "hbm_gbs": hbm_gbs, "fp64_instr_per_s": P,
            "note": "algorithmic bytes / FP64 instructions per step (kernel eval %d instr incl. distance, CPQR "
                    "2 DFMA per entry per pivot, HiDR 3d per distance; down = distances evaluated by the exact "
                    "pruned search); floors of concurrent steps are summed" % ck}


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        self.f.seek(0)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            p = [x.strip() for x in line.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                smax.append(float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[3:7]):
                if v.lower() in ("active", "1", "yes"):
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------ dist
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v: float, ws: int) -> float:
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------------------------------ oracle
def oracle_for(cfg: int, pts):
    """The oracle handle of a config (the non-symmetric path and the kernel shift for kernel 7)."""
    import oracle
    c = synth.CONFIGS[cfg]
    ns = c["kernel"] == synth.KERNEL_MQSHIFT
    if ns:
        oracle.set_kernel_shift(np.array(c["params"][1:]))
    return oracle.OracleH2(pts, c["q"], c["tau"], nonsym=ns)


def oracle_sample_run(cfg: int, n_sample: int):
    """The fp64 oracle, as it stands, on a bounded sample of the workload (same distribution,
    n_sample points): a1-a8 plus an evaluate-only pass over every a9/a10 block."""
    c = synth.CONFIGS[cfg]
    pts = synth.points(cfg, n_sample)
    kp = c["params"][0] if c["params"] else 0.0
    t0 = time.perf_counter()
    h = oracle_for(cfg, pts)
    h.build(c["kernel"], kp, c["id_tol"])
    entries, _ = h.fill(store=False)
    dt = time.perf_counter() - t0
    h.close()
    return dt, entries


def cpu_baseline(cfg: int, n_sample: int, y_gpu_rows=None) -> tuple[dict, dict | None]:
    """The oracle timed on the host cores (a1-a8 + evaluate-only a9/a10 on n_sample points), and,
    outside that timing, the accuracy of the timed GPU build: the relative matvec error of the GPU
    H^2 on the 1024 seeded rows against the exact dense K x, next to the oracle's own error on the
    same rows (when the oracle ran on the whole workload)."""
    import oracle
    c = synth.CONFIGS[cfg]
    pts = synth.points(cfg, n_sample)
    kp = c["params"][0] if c["params"] else 0.0
    t0 = time.perf_counter()
    h = oracle_for(cfg, pts)
    r = h.build(c["kernel"], kp, c["id_tol"])
    entries, _ = h.fill(store=False)
    dt = time.perf_counter() - t0
    whole = n_sample == c["n"]
    what = "the whole workload" if whole else "points of the same distribution as the workload"
    base = {"value": round(n_sample / dt / 1e6, 6), "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
            "cpu_model": host_cpu_model(),
            "sample": f"oracle a1-a8 + evaluate-only a9/a10 ({entries} block entries) on n={n_sample} ({what}); "
                      f"wall {dt:.2f} s"}
    acc = None
    if y_gpu_rows is not None:
        n = c["n"]
        x = synth.matvec_vector(cfg, n)
        rows = synth.sample_rows(cfg, n)
        yd = oracle.dense_rows(synth.points(cfg), c["kernel"], kp, x, rows)
        eg = float(np.linalg.norm(y_gpu_rows - yd) / np.linalg.norm(yd))
        acc = {"matvec_rel_err": eg, "rows": int(len(rows)), "id_tol": c["id_tol"],
               "definition": "||K~x - Kx|| / ||Kx|| on the seeded sampled rows (all rows if n <= 16384), "
                             "x = synth.matvec_vector, dense K x by the oracle"}
        if whole:
            yo = h.matvec(x, rows)
            eo = float(np.linalg.norm(yo - yd) / np.linalg.norm(yd))
            acc.update({"oracle_matvec_rel_err": eo, "oracle_r": r, "ratio_to_oracle": round(eg / eo, 4),
                        "gpu_vs_oracle": float(np.linalg.norm(y_gpu_rows - yo) / np.linalg.norm(yo))})
    h.close()
    return base, acc


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    cfg = args.config
    n_s = args.ref_sample
    for _ in range(args.warmup):
        oracle_sample_run(cfg, n_s // 4)
    times = []
    for _ in range(args.steps):
        dt, entries = oracle_sample_run(cfg, n_s)
        times.append(dt)
    t = float(np.mean(times))
    v = n_s / t / 1e6
    line = {"metric": METRIC, "value": round(v, 6), "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": workload_desc(cfg), "sample_n": n_s,
                       "note": "reference = the fp64 CPU oracle (oracle/h2_oracle.c) on the host cores"},
            "cpu_baseline": {"value": round(v, 6), "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": f"n={n_s} points of the workload distribution per step, a1-a8 + "
                                       f"evaluate-only a9/a10"},
            "e2e": {"value": round(v, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------ ours
def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    import paper_2206_01885_b200 as P

    cfg = args.config
    c = synth.CONFIGS[cfg]
    n = c["n"] if args.n is None else args.n
    # N > 1: every rank holds the same points (replicated) and builds its share of one H^2
    pts_np = synth.points(cfg, n)
    pts = torch.from_numpy(pts_np).cuda()
    comm = None
    if ws > 1:
        import torch.distributed as dist
        uid = [P.H2Comm.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = P.H2Comm.nccl(ws, rank, uid[0], device=local)
    stream = torch.cuda.Stream()
    kp = list(c["params"])
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def opts(host=False, serial=False):
        o = P.h2_options_default()
        o.storage = {"all": P.H2_STORE_ALL, "fly": P.H2_STORE_ON_THE_FLY, "auto": P.H2_STORE_AUTO}[args.storage]
        o.timing = 1
        o.stream = stream.cuda_stream
        o.points_on_host = 1 if host else 0
        o.serial_fill = 1 if serial else 0
        if comm is not None:
            o.comm = comm.ptr
        return o

    def one(host=False, src=None, serial=False):
        ptr = src if src is not None else pts.data_ptr()
        return P.h2_build(ptr, n, c["d"], c["kernel"], kp, c["id_tol"], c["q"], c["tau"], opts(host, serial))

    # the first build of the process, timed (cold: lazy module loading of every kernel, first
    # driver allocations of the block store and the caching allocator's pool); not a bench value
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tc0 = time.perf_counter()
    c0.record(stream)
    h = one()
    c1.record(stream)
    c1.synchronize()
    cold = {"device_ms": round(c0.elapsed_time(c1), 3), "wall_ms": round(1e3 * (time.perf_counter() - tc0), 3)}
    P.h2_free(h)
    for _ in range(args.warmup):
        h = one()
        P.h2_free(h)
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    times, fill_ms, cfill_ms, stages, launches = [], [], [], [], 0
    info = None
    barrier(ws)
    torch.cuda.synchronize()
    sampler.start()
    t_wall0 = time.perf_counter()
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h = one()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        info = P.h2_info(h)
        fill_ms.append(info["stage_ms"]["nearfield_fill"])
        cfill_ms.append(info["stage_ms"]["coupling_fill"])
        stages.append(info["stage_ms"])
        launches = info["gpu_launches"]
        P.h2_free(h)
    torch.cuda.synchronize()
    barrier(ws)
    t_wall = time.perf_counter() - t_wall0
    clocks = sampler.stop()

    t_step = max_over_ranks(float(np.mean(times)), ws)
    value = n / (t_step * 1e-3) / 1e6

    # e2e: same build through the C ABI from pinned HOST memory (H2D inside the call) plus the
    # device->host read of the step's result (the skeleton ranks k_i of every node)
    pinned = torch.from_numpy(pts_np).pin_memory()
    P.h2_free(one(host=True, src=pinned.data_ptr()))  # untimed: the host path's first staging allocation
    e2e_times = []
    h2d = n * c["d"] * 8
    d2h = 0
    for _ in range(max(1, min(args.steps, 3))):
        with torch.cuda.stream(stream):
            flush.fill_(2)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = one(host=True, src=pinned.data_ptr())
        kvec = P.h2_export(h, "K")
        t1 = time.perf_counter()
        d2h = kvec.nbytes
        e2e_times.append(t1 - t0)
        P.h2_free(h)
    e2e_t = max_over_ranks(float(np.mean(e2e_times)), ws)
    e2e = {"value": round(n / e2e_t / 1e6, 4), "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": int(d2h)}

    # H^2 matvec on one stored build: y = K~ x, every pass on the GPU; the
    # stored blocks are read once (the nearfield pass dominates: 8 B per stored entry)
    stored = args.storage == "all"
    h = one()
    # accuracy of the benched configuration (outside every timed region): y = K~ x for the seeded x
    xv = torch.from_numpy(synth.matvec_vector(cfg, n)).cuda()
    yv = torch.empty_like(xv)
    P.h2_matvec(h, xv.data_ptr(), yv.data_ptr(), n)
    y_rows = yv.cpu().numpy()[synth.sample_rows(cfg, n)]
    ex = {nm: P.h2_export(h, nm) for nm in ("K", "XBAR_N", "YS_OFF")}
    torch.cuda.synchronize()
    for _ in range(2 if stored else 0):
        P.h2_matvec(h, xv.data_ptr(), yv.data_ptr())
    mv_ms = []
    for _ in range(5 if stored else 0):
        with torch.cuda.stream(stream):
            flush.fill_(4)
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record(stream)
        P.h2_matvec(h, xv.data_ptr(), yv.data_ptr())
        m1.record(stream)
        m1.synchronize()
        mv_ms.append(m0.elapsed_time(m1))
    if stored:
        mv_info = P.h2_info(h)
        mv_t = float(np.median(mv_ms))
        mv_bytes = 8 * (mv_info["nearfield_entries"] + mv_info["coupling_entries"])
    P.h2_free(h)

    # the same build with the nearfield fill run alone (serial_fill): the kernel's own roofline
    iso_ms = []
    for _ in range(2 if stored else 0):
        with torch.cuda.stream(stream):
            flush.fill_(3)
        h = one(serial=True)
        iso_ms.append(P.h2_info(h)["stage_ms"]["nearfield_fill"])
        P.h2_free(h)

    # roofline of the dominant kernel (nearfield fill, a10): algorithmic bytes = 8 B per stored entry
    peaks = json.load(open(PEAKS_FILE)) if os.path.exists(PEAKS_FILE) else {}
    hbm = float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS))
    nf_bytes = 8 * info["nearfield_entries"]
    nf_ms = float(np.mean(fill_ms)) if stored else 0.0
    achieved = nf_bytes / (nf_ms * 1e-3) / 1e9 if stored else 0.0
    traffic = None
    if os.path.exists(TRAFFIC_FILE):
        try:
            tr = json.load(open(TRAFFIC_FILE))
            if tr.get("workload") == c["name"]:
                traffic = tr.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    fp64 = fp64_peak()
    whole = build_roofline(c, info, ex["K"], ex["XBAR_N"], np.diff(ex["YS_OFF"]), t_step, hbm, fp64)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": traffic,
                "kernel": f"nf_fill_kernel<D={c['d']},kernel {c['kernel']}> (a10, nearfield fill)",
                "kernel_ms": round(nf_ms, 3),
                "step_share": round(nf_ms / t_step, 4),
                "note": "live: the kernel runs concurrently with a5-a9 (side stream), sharing the SMs",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if peaks else "fallback 6650 GB/s",
                "fp64_peak_tflops": round(fp64["tflops"], 2), "fp64_peak_source": fp64["source"]}
    iso = float(np.mean(iso_ms)) if stored else 1.0
    roofline_isolated = {"bound": "hbm", "achieved": round(nf_bytes / (iso * 1e-3) / 1e9, 1), "peak": hbm,
                         "unit": "GB/s", "frac": round(nf_bytes / (iso * 1e-3) / 1e9 / hbm, 4),
                         "kernel_ms": round(iso, 3), "traffic": traffic,
                         "note": "same kernel, same build, fill run alone after a9 (h2_options.serial_fill = 1); "
                                 "2 builds after the timed region, L2 flushed before each"}

    if rank == 0:
        mean_stages = {k: round(float(np.mean([s[k] for s in stages])), 3) for k in stages[0]}
        line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(t_step, 3), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_desc(cfg), "n_per_gpu": n, "r": info["r"], "nnodes": info["nnodes"],
                           "stored_bytes": info["stored_bytes"], "coupling_entries": info["coupling_entries"],
                           "nearfield_entries": info["nearfield_entries"],
                           "parallelism": "single GPU" if ws == 1 else
                           f"sharded over {ws} GPUs (subtrees below the cut level; NCCL allgathers)",
                           "l2": "flushed (512 MiB write) before every timed step",
                           "wall_s_timed_region": round(t_wall, 3)},
                "stages_ms": mean_stages, "clocks": clocks, "e2e": e2e, "gpu_launches": launches,
                "cold_first_build": cold, "roofline_whole_build": whole,
                "roofline": roofline if stored else None,
                "roofline_isolated": roofline_isolated if stored else None,
                "matvec": {"ms": round(mv_t, 3), "stored_bytes_read": mv_bytes,
                           "achieved_gbs": round(mv_bytes / (mv_t * 1e-3) / 1e9, 1),
                           "frac_of_hbm": round(mv_bytes / (mv_t * 1e-3) / 1e9 / hbm, 4),
                           "note": "h2_matvec (all four passes, permutations, host sync) on one stored build; "
                                   "median of 5, L2 flushed; not part of the construction metric"} if stored
                else None}
        if not stored:
            line["config"]["storage"] = "blocks not stored (skeleton build a1-a8; a9/a10 evaluated in the matvec)"
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"], line["accuracy"] = cpu_baseline(cfg, args.cpu_sample, y_rows)
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        comm.close()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=4, help="BASELINE configs[C-1] (1..5); 6 = the non-symmetric "
                                                             "extra config (not a bench line)")
    ap.add_argument("--n", type=int, default=None, help="override n (not a bench line)")
    ap.add_argument("--storage", choices=["all", "fly", "auto"], default="all",
                    help="block storage (fly: skeleton build a1-a8, blocks evaluated in the matvec; for "
                         "configs whose blocks exceed one GPU)")
    ap.add_argument("--cpu-sample", type=int, default=None,
                    help="points of the oracle's cpu_baseline run (default: the whole workload, ~6 s for "
                         "configs[3]; configs[4]: 65536 points, ~20 s -- its 5-D HiDR is quadratic in the oracle)")
    ap.add_argument("--ref-sample", type=int, default=None,
                    help="points per step of --impl reference (default: as --cpu-sample)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    default_sample = min(synth.CONFIGS[args.config]["n"], 65536 if args.config == 5 else 1 << 22)
    if args.cpu_sample is None:
        args.cpu_sample = default_sample
    if args.ref_sample is None:
        args.ref_sample = default_sample
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # --gpus N without a launcher: start the N ranks ourselves (one process per GPU, the same
        # torch.distributed.run launch the driver uses), so n_gpus is never silently 1
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
