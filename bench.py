#!/usr/bin/env python3
"""bench.py -- B200 benchmark of the window-based off-diagonal update path.

Workload: the configuration BASELINE.json's metric is quoted on --
eigenvalue reordering of the synthetic standardized Schur form of SURVEY.md
8d at n = 40000 fp64 (configs[3], "C4"; it fits one B200: S + Q = 25.6 GB),
35 % of the diagonal blocks selected (select_fraction seed 99), Q accumulated
(Q_in = I), window size = the reference default (tile size 128).  One step =
one full ``reorder_schur`` of that matrix.  Inputs are generated directly in
HBM by the library's Philox generator (bit-identical to the reference's
generator) and restored from a pristine device copy before every step
(outside the per-step events).  Inputs >> L2 (126 MB): no flush needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--n 40000] [--ws 0]
  python bench.py --impl reference ...   # the reference CPU path, host cores

N = 1: the single-GPU path.  N > 1 (torchrun, one rank per GPU): the
distributed path (S column slabs, Q row slabs, NCCL all-reduce of the
packed Q_w per wavefront, halo transfers; csrc/dist_reorder.cpp) on the SAME
n = 40000 problem: "scaling": "strong", value = max time over ranks.  The
line also carries C2 (n = 10000, configs[1]) and C3 (Schur reduction,
configs[2]) sections at N = 1.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

# More hardware work queues than the default 8 (read once, at CUDA
# initialisation, so before torch touches the device): the library runs a
# level's window kernels, bulk updates and factor updates on three streams
# beside the caller's; with 8 queues two of them can share one and pick up
# false dependencies (C2 calls 100 vs 106 ms depending on stream-creation
# order).  INTEGRATION.md recommends the same for applications.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "reorder/Schur time-to-solution (s) at n=40k; update FP64 TFLOP/s vs peak, 1-8 GPU"
FP64_DMMA_PEAK_TFLOPS = 37.1  # profiles/r01_fp64_peak.txt (MEASURED_PEAKS.json has no FP64 entry)
FILL_SEED_BASE = 1            # fill seed = generate()'s known_spectrum convention of seed 1
SEL_SEED = 99
FRACTION = 0.35


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", type=int, default=40000)
    ap.add_argument("--c2-n", type=int, default=10000, help="size of the C2 section (0: skip)")
    ap.add_argument("--ws", type=int, default=0, help="window size (0: reference default = tile 128)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="reorder", choices=["reorder", "schur"],
                    help="reorder: C2 (headline); schur: C3 multishift QR + AED of random Hessenberg")
    ap.add_argument("--no-schur", action="store_true", help="skip the C3 section of the default line")
    ap.add_argument("--schur-n", type=int, default=10000)
    ap.add_argument("--c5-n", type=int, default=20000, help="size of the C5 (generalized pair) section (0: skip)")
    ap.add_argument("--force-dist", action="store_true", help="use the NCCL distributed path even at N=1 (plumbing test)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.k0 = 0

    def mark(self):
        """Start of the timed region: samples before it are dropped.  The
        sampler is started before the warm-up so that nvidia-smi's own start-up
        (NVML init, ~1 s of driver work) is not inside the timed steps."""
        t0 = time.time()
        while self.proc is not None and not self.samples and time.time() - t0 < 10:
            time.sleep(0.05)
        self.k0 = len(self.samples)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = []
        mx = None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for p in self.samples[self.k0:]:
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_problem(T, n, dev):
    import torch
    S0 = T.gen_schur_input(n, T.known_spectrum_seed(FILL_SEED_BASE), device=dev)
    sel = T.select_fraction(S0, FRACTION, SEL_SEED)
    torch.cuda.synchronize()
    return S0, sel


def synthetic_selection(T, n):
    """select_fraction on the synthetic Schur form's block pattern (reals
    first, then floor(n/4) 2x2 blocks: generate.cpp:68-91, 115-150) without
    materialising the matrix -- what every rank of the distributed run uses."""
    import ctypes as C
    npairs = n // 4
    nreal = n - 2 * npairs
    sizes = np.array([1] * nreal + [2] * npairs, dtype=np.uint8)
    flags = np.zeros(len(sizes), dtype=np.uint8)
    T._native.check(T._native.lib().teig_select_fraction(len(sizes), FRACTION, SEL_SEED,
                                                         flags.ctypes.data_as(C.c_void_p)))
    starts = np.concatenate([[0], np.cumsum(sizes.astype(np.int64))])
    blocks = [T.Block(int(starts[i]), int(sizes[i]), 0j) for i in range(len(sizes))]
    return T.Selection(blocks, [bool(f) for f in flags])


def _band(M):
    """(diagonal, superdiagonal, subdiagonal) of a device matrix, on the host."""
    import torch
    return (torch.diagonal(M, 0).cpu().numpy(), torch.diagonal(M, 1).cpu().numpy(),
            torch.diagonal(M, -1).cpu().numpy())


def _read_off(d, u, l):
    """Eigenvalues read off a standardized quasi-triangular form's diagonal
    blocks (2x2 [[a, b], [c, a]]: a +- sqrt|b| sqrt|c| i; schur.cpp:888-904),
    O(n) from the band."""
    n = len(d)
    ev = d.astype(complex)
    r = 0
    while r < n:
        if r + 1 < n and l[r] != 0.0:
            im = np.sqrt(abs(u[r])) * np.sqrt(abs(l[r]))
            ev[r] = complex(d[r], im)
            ev[r + 1] = complex(d[r + 1], -im)
            r += 2
        else:
            r += 1
    return ev


def _predicted(ev_in, sel):
    """Eigenvalues in the order a clean reorder leaves them: selected blocks
    first, then unselected, both in original order."""
    sizes = sel.sizes_array().astype(np.int64)
    starts = np.concatenate([[0], np.cumsum(sizes)])
    fl = np.asarray(sel.flags, dtype=bool)
    order = np.concatenate([np.nonzero(fl)[0], np.nonzero(~fl)[0]])
    return np.concatenate([ev_in[starts[i]:starts[i + 1]] for i in order])


def positional_eigs(S0, S, sel, tol=1e-10):
    """O(n) positional eigenvalue parity at full size: every diagonal block of
    the output carries exactly the eigenvalue the predicted order puts there,
    to relative tol -- the north_star's "eigenvalues match the reference to
    relative 1e-10" with the reference's (deterministic) final order."""
    ev = _read_off(*_band(S))
    want = _predicted(_read_off(*_band(S0)), sel)
    err = float(np.max(np.abs(ev - want) / np.maximum(1.0, np.abs(want))))
    k = int(sum(b.size for b, f in zip(sel.blocks, sel.flags) if f))
    return {"max_rel_err": err, "tol": tol, "pass": err <= tol, "selected_rows_leading": k}


def positional_eigs_pencil(S0, T0, S, Tm, sel, tol=1e-10):
    """Generalized: the pencil's eigenvalues of every diagonal block (1x1:
    s/t; 2x2: eig(T_blk^-1 S_blk)) in the predicted order, O(n)."""
    def blocks(Sx, Tx):
        sd, su, sl = _band(Sx)
        td, tu, _ = _band(Tx)
        n = len(sd)
        ev = np.empty(n, dtype=complex)
        r = 0
        while r < n:
            if r + 1 < n and sl[r] != 0.0:
                sb = np.array([[sd[r], su[r]], [sl[r], sd[r + 1]]])
                tb = np.array([[td[r], tu[r]], [0.0, td[r + 1]]])
                e = np.linalg.eigvals(np.linalg.solve(tb, sb))
                e = sorted(e, key=lambda z: -z.imag)
                ev[r], ev[r + 1] = e[0], e[1]
                r += 2
            else:
                ev[r] = sd[r] / td[r]
                r += 1
        return ev
    ev = blocks(S, Tm)
    want = _predicted(blocks(S0, T0), sel)
    err = float(np.max(np.abs(ev - want) / np.maximum(1.0, np.abs(want))))
    return {"max_rel_err": err, "tol": tol, "pass": err <= tol}


def run_ours(args, rank, world, local):
    import torch
    import paper_2002_05024_b200 as T

    # serving configuration: the library keeps its device pool and host-path
    # staging between calls (teig_set_memory_retention; off by default)
    T.set_memory_retention(True)
    if world > 1 or args.force_dist:
        return run_ours_dist(args, rank, world, local)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    n = args.n
    S0, sel = make_problem(T, n, dev)
    S = T.colmajor_empty(n, dev)
    Q = T.colmajor_empty(n, dev)
    Q0 = T.identity(n, dev)
    stream = torch.cuda.current_stream(dev)

    def reset():
        S.copy_(S0)
        Q.copy_(Q0)

    opts = T.ReorderOptions(window_size=args.ws)
    # ---------------- e2e: host buffers through the C ABI, copies inside ----------------
    # (first, after one untimed device run whose result the e2e must
    # reproduce: the host path's device staging is then mapped while HBM is
    # unfragmented -- staged after the cuBLAS parity temporaries it ran 10-40 %
    # slower -- and no nvidia-smi sampler runs beside it)
    reset()
    res = T.reorder_schur(S, Q, sel, opts)
    torch.cuda.synchronize()
    e2e = None
    if not args.no_e2e and world == 1:
        e2e = e2e_reorder(T, S0, S, sel, opts, n, 5)

    sampler = ClockSampler(local)
    sampler.start()
    # the timed steps run exactly as a user's call (no per-launch events); the
    # kernel-level numbers come from one extra serialised, profiled step below
    for k in range(max(args.warmup, 0)):
        reset()
        res = T.reorder_schur(S, Q, sel, opts)
    torch.cuda.synchronize()

    # ---------------- timed region (device events per step) ----------------
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.mark()
    t_wall0 = time.perf_counter()
    infos = []
    for k in range(args.steps):
        reset()
        ev[k][0].record(stream)
        res = T.reorder_schur(S, Q, sel, opts)
        ev[k][1].record(stream)
        infos.append(res.info)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall0
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms_step = sum(step_ms) / len(step_ms)
    if world > 1:
        t = torch.tensor([ms_step], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    info = infos[-1]

    # ---------------- parity spot check of the last step (GPU cuBLAS, independent) ----------------
    S0d = S0.to(torch.float64)
    R = S0d - Q @ S @ Q.t()
    resid = float(torch.linalg.norm(R) / torch.linalg.norm(S0d))
    orth = float(torch.linalg.norm(Q.t() @ Q - torch.eye(n, dtype=torch.float64, device=dev)))
    del R
    eig_pos = positional_eigs(S0, S, sel)

    # ---------------- one extra, untimed, SERIALISED step: every launch on one
    # stream (overlap_factor=0), so the per-class event durations are
    # non-overlapped kernel time -- the dominant kernel's rate ----------------
    reset()
    ser = T.reorder_schur(S, Q, sel, T.ReorderOptions(window_size=args.ws, profile=True, overlap_factor=False)).info
    torch.cuda.synchronize()
    # executed flops of a step (the plan is deterministic: the serialised step
    # runs the same windows): DMMA instructions counted on the device
    exec_flops = ser["flops_dmma"] if ser.get("flops_dmma") else (
        ser["flops_left"] + ser["flops_right"] + ser["flops_factor_exec"])

    # ---------------- roofline of the dominant kernel class ----------------
    # achieved: update flops / summed update-kernel durations of the
    # serialised step (non-overlapped); the timed steps' event sums overlap on
    # two streams and are reported separately (two_stream_event_sum)
    # executed flops: the DMMA instructions the update kernels issued, counted
    # on the device (512 flops each) -- the factor updates skip Q's exactly-zero
    # rows (plan.h FactorSupport) and the bulk kernels Q_w's all-zero 8x4
    # fragments, so neither the reference's count (2 d^2 (2n - d) per window)
    # nor the row-skipped count is what the tensor pipe executed
    k_ms = ser["ms_left"] + ser["ms_right"] + ser["ms_factor"]
    k_flops = ser["flops_dmma"] if ser.get("flops_dmma") else (
        ser["flops_left"] + ser["flops_right"] + ser["flops_factor_exec"])
    achieved = k_flops / (k_ms * 1e-3) / 1e12 if k_ms > 0 else 0.0
    steps = args.steps
    roof = {"bound": "tensor", "kernel": "update_left/right DMMA kernels (all launches of one serialised step)",
            "achieved": round(achieved, 3), "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": round(achieved / FP64_DMMA_PEAK_TFLOPS, 4),
            "measurement": "CUDA events around every update launch of one extra step with all launches on one "
                           "stream (overlap_factor=0): non-overlapped kernel time",
            "serialised_step_ms": {"window": round(ser["ms_window"], 2), "left": round(ser["ms_left"], 2),
                                   "right": round(ser["ms_right"], 2), "factor": round(ser["ms_factor"], 2)},

            "peak_source": "FP64 DMMA.8x8x4 issue peak measured on this pool's B200 "
                           "(tools/microbench/fp64_peak.cu, profiles/r01_fp64_peak.txt); "
                           "MEASURED_PEAKS.json has no FP64 entry",
            "traffic": measured_traffic(),
            "aggregate": {"achieved": round(exec_flops / (ms_step * 1e-3) / 1e12, 3),
                          "frac": round(exec_flops / (ms_step * 1e-3) / 1e12 / FP64_DMMA_PEAK_TFLOPS, 4),
                          "note": "executed update flops / step time (both streams, window kernels included)"},
            "executed_vs_reference_flops": {"executed_dmma": exec_flops, "reference_count": info["update_flops"],
                                            "row_skipped_count": info["flops_left"] + info["flops_right"]
                                            + info["flops_factor_exec"],
                                            "note": "executed = DMMA instructions issued x 512 (device counters); "
                                                    "the reference updates Q over all n rows per window and multiplies "
                                                    "Q_w's zero blocks too: the kernels skip Q's exactly-zero rows "
                                                    "and Q_w's all-zero 8x4 fragments, bitwise-identical result"},
            "flops_per_step": k_flops,
            "update_ms_serialised_step": k_ms,
            "window_ms_serialised_step": ser["ms_window"],
            "algorithmic_bytes_per_step": info["update_bytes"]}

    out = {
        "metric": METRIC,
        "value": round(ms_step / 1e3, 6),
        "unit": "s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 3),
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (SURVEY.md 8d Schur form generated in HBM by the library's Philox generator)",
        "config": {"workload": f"{workload_name(n)}: reorder_schur n={n}, 35% selected (select_fraction seed "
                               f"{SEL_SEED}), Q accumulated, window {args.ws or 128}",
                   "n": n, "window_size": args.ws or 128, "fraction": FRACTION,
                   "parallelism": "single-gpu", "memory_retention": True,
                   "l2": f"inputs {2 * n * n * 8 / 1e9:.1f} GB > 126 MB L2, no flush needed"},
        "update_tflops": round(info["update_flops"] / (ms_step * 1e-3) / 1e12, 3),
        "update_tflops_note": "the reference's flop count (Q updated over all n rows) / step time",
        "update_flops": info["update_flops"],
        "update_flops_executed": exec_flops,
        "windows": info["n_windows"], "levels": info["n_levels"], "groups": info["n_groups"],
        "clean": info["clean"] == 1,
        "parity": {"backward_error": resid, "orthogonality": orth, "tol_10neps": 10 * n * 2.220446049250313e-16,
                   "eig_positional": eig_pos,
                   "pass": resid <= 10 * n * 2.220446049250313e-16 and orth <= 10 * n * 2.220446049250313e-16
                   and eig_pos["pass"]},
        "roofline": roof,
        "e2e": e2e,
        "gpu_launches": int(info["n_launches"]),
        "clocks": clocks,
        "wall_s_timed_region": round(t_wall, 3),
        "step_ms": [round(x, 3) for x in step_ms],
    }
    if rank == 0 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(args, n)
    del S0, S, Q, Q0
    torch.cuda.empty_cache()
    if args.c2_n:
        out["c2_n10000"] = run_c2(args, dev)
    if args.c5_n:
        out["greorder_c5"] = run_c5(args, dev)
    if not args.no_schur:
        out["schur_c3"] = run_schur(args, dev, with_cpu=(rank == 0 and not args.no_cpu), with_e2e=not args.no_e2e)
        out["schur_c3"]["gpu_launches_counted_in_line"] = False
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()



def workload_name(n):
    return {10000: "C2", 40000: "C4"}.get(n, "reorder")


def measured_traffic():
    """DRAM bytes of one captured launch of the dominant kernel (ncu --set full,
    profiles/r03_traffic.json) -- per launch, next to that launch's algorithmic
    bytes; None when the capture file is absent."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r03_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return None
    return {"dram_bytes_per_launch": t["dram_bytes"], "algorithmic_bytes_per_launch": t["algorithmic_bytes"],
            "ratio": round(t["dram_bytes"] / t["algorithmic_bytes"], 3), "launch": f'{t["kernel"]}, {t["launch"]}',
            "source": t["source"]}


def e2e_reorder(T, S0, S_dev_result, sel, opts, n, steps):
    """The same reorder through the C ABI's host entry point: pinned host S,Q
    (column-major), H2D + D2H inside the timed call."""
    import torch
    try:
        Sh = torch.empty((n, n), dtype=torch.float64).pin_memory()
        Qh = torch.empty((n, n), dtype=torch.float64).pin_memory()
    except RuntimeError as e:  # host RAM
        return {"value": None, "unit": "s", "skipped": f"pinned host buffers: {e}"[:200]}
    e2e_ms = []
    for k in range(max(1, steps) + 1):
        Sh.copy_(S0.t())  # row-major of S^T == column-major of S
        Qh.zero_()
        Qh.diagonal().fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        T.reorder.reorder_schur_host_buffers(Sh.numpy(), Qh.numpy(), n, sel, opts)
        dt = (time.perf_counter() - t0) * 1e3
        if k > 0:  # first call warms the pinned path
            e2e_ms.append(dt)
    ok = bool(torch.equal(Sh.cuda().t(), S_dev_result))
    h2d, d2h = T.host_transfer_bytes()  # what the last call moved (library counters)
    del Sh, Qh
    return {"value": round(statistics.median(e2e_ms) / 1e3, 6), "unit": "s", "calls_s": [round(x / 1e3, 4) for x in e2e_ms],
            "statistic": "median of the timed calls",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "host_buffer_bytes": 2 * n * n * 8,
            "transfer_note": ("S moves as its upper Hessenberg part (nothing below the first subdiagonal is read "
                              "or written on the path), Q as the row hull of its nonzeros per 512-column block "
                              "(Q_in = I); counted by the library (teig_host_transfer_bytes)"),
            "steps": len(e2e_ms), "matches_device_result": ok,
            "api": "teig_reorder_schur_host (C ABI, pinned host S,Q column-major)"}


def run_c2(args, dev, steps=3, warmup=2):
    """C2 (configs[1]): reorder n=10000 on one GPU, device time + parity + the
    CPU reference sample (kept for continuity with the round-1 profiles)."""
    import torch
    import paper_2002_05024_b200 as T
    n = args.c2_n
    S0, sel = make_problem(T, n, dev)
    S, Q = T.colmajor_empty(n, dev), T.colmajor_empty(n, dev)
    Q0 = T.identity(n, dev)
    opts = T.ReorderOptions(window_size=args.ws)
    for _ in range(warmup):
        S.copy_(S0)
        Q.copy_(Q0)
        T.reorder_schur(S, Q, sel, opts)
    ms = []
    stream = torch.cuda.current_stream(dev)
    for _ in range(steps):
        S.copy_(S0)
        Q.copy_(Q0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = T.reorder_schur(S, Q, sel, opts)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    back = float(torch.linalg.norm(S0 - Q @ S @ Q.t()) / torch.linalg.norm(S0))
    orth = float(torch.linalg.norm(Q.t() @ Q - torch.eye(n, dtype=torch.float64, device=dev)))
    tol = 10 * n * 2.220446049250313e-16
    eig_pos = positional_eigs(S0, S, sel)
    out = {"workload": f"C2: reorder_schur n={n}, 35% selected (seed {SEL_SEED}), Q accumulated, window "
                       f"{args.ws or 128}", "value": round(statistics.mean(ms) / 1e3, 5), "unit": "s",
           "step_ms": [round(x, 2) for x in ms], "update_tflops": round(res.info["update_flops"] / (statistics.mean(ms) * 1e-3) / 1e12, 3),
           "windows": res.info["n_windows"], "levels": res.info["n_levels"], "clean": res.clean,
           "parity": {"backward_error": back, "orthogonality": orth, "tol_10neps": tol, "eig_positional": eig_pos,
                      "pass": back <= tol and orth <= tol and eig_pos["pass"]}}
    if not args.no_e2e:
        out["e2e"] = e2e_reorder(T, S0, S, sel, opts, n, 5)
    if not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(args, n)
    return out


def run_ours_dist(args, rank, world, local):
    """N > 1: one rank per GPU, the distributed path on the same n problem."""
    import torch
    import torch.distributed as dist
    import paper_2002_05024_b200 as T
    from paper_2002_05024_b200 import dist as D

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    n = args.n
    sel = synthetic_selection(T, n)
    cb, rb = D.balance(n, sel, world, args.ws)
    c0, c1, r0, r1 = int(cb[rank]), int(cb[rank + 1]), int(rb[rank]), int(rb[rank + 1])
    comm = D.nccl_comm(rank, world)
    seed = T.known_spectrum_seed(FILL_SEED_BASE)
    S0 = D.gen_schur_input_slab(n, seed, c0, c1, dev)
    Q0 = D.identity_rows_slab(n, r0, r1, dev)
    S = D.s_slab_empty(n, c0, c1, dev)
    Q = D.q_slab_empty(n, r0, r1, dev)
    opts = T.ReorderOptions(window_size=args.ws)

    def reset():
        S.copy_(S0)
        Q.copy_(Q0)

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(max(args.warmup, 0)):
        reset()
        res = D.reorder_schur_dist(S, Q, sel, cb, rb, rank, world, comm, opts)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    sampler.mark()
    t0 = time.perf_counter()
    for k in range(args.steps):
        reset()
        ev[k][0].record(stream)
        res = D.reorder_schur_dist(S, Q, sel, cb, rb, rank, world, comm, opts)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t0
    dist.barrier()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t = torch.tensor([statistics.mean(step_ms)], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item())
    info = res.info
    # parity: the distributed result must equal the single-GPU result bit for
    # bit -- gather both slabs to rank 0, rerun single-GPU there, compare
    parity = None
    if n <= 40000:
        wc = c1 - c0
        s_loc = S[:, :wc].contiguous()
        q_loc = Q.contiguous()
        sizes_s = [int(cb[g + 1] - cb[g]) for g in range(world)]
        sizes_q = [int(rb[g + 1] - rb[g]) for g in range(world)]
        if rank == 0:
            s_parts = [torch.empty((n, w), dtype=torch.float64, device=dev) for w in sizes_s]
            q_parts = [torch.empty((h, n), dtype=torch.float64, device=dev) for h in sizes_q]
        for g in range(world):  # point-to-point gather (unequal slab sizes)
            if rank == 0 and g == 0:
                s_parts[0].copy_(s_loc)
                q_parts[0].copy_(q_loc)
            elif rank == 0:
                dist.recv(s_parts[g], src=g)
                dist.recv(q_parts[g], src=g)
            elif rank == g:
                dist.send(s_loc, dst=0)
                dist.send(q_loc, dst=0)
        del s_loc, q_loc
        if rank == 0:
            Sd = torch.cat(s_parts, dim=1)
            Qd = torch.cat(q_parts, dim=0)
            del s_parts, q_parts
            S1 = T.gen_schur_input(n, seed, device=dev)
            Q1 = T.identity(n, dev)
            T.reorder_schur(S1, Q1, sel, opts)
            parity = {"bitwise_equal_to_single_gpu": bool(torch.equal(Sd, S1) and torch.equal(Qd, Q1))}
            del Sd, Qd, S1, Q1
        dist.barrier()
    # e2e: the same distributed call on slabs held in pinned HOST memory, the
    # H2D of the inputs and D2H of the results inside the timed region
    e2e = None
    if not args.no_e2e:
        hs = torch.empty(S0.shape[::-1], dtype=torch.float64).pin_memory().t()  # column-major host slab
        hq = torch.empty(Q0.shape[::-1], dtype=torch.float64).pin_memory().t()
        hs.copy_(S0)
        hq.copy_(Q0)
        e2e_ms = []
        for k in range(2):
            hs.copy_(S0)
            hq.copy_(Q0)
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            S.copy_(hs, non_blocking=True)
            Q.copy_(hq, non_blocking=True)
            D.reorder_schur_dist(S, Q, sel, cb, rb, rank, world, comm, opts)
            hs.copy_(S, non_blocking=True)
            hq.copy_(Q, non_blocking=True)
            torch.cuda.synchronize()
            dt = torch.tensor([(time.perf_counter() - t0) * 1e3], device=dev, dtype=torch.float64)
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            e2e_ms.append(float(dt.item()))
        hb = (S0.numel() + Q0.numel()) * 8
        tot = torch.tensor([hb], device=dev, dtype=torch.float64)
        dist.all_reduce(tot)
        e2e = {"value": round(min(e2e_ms) / 1e3, 6), "unit": "s", "h2d_bytes_per_step": int(tot.item()),
               "d2h_bytes_per_step": int(tot.item()),
               "api": "teig_dist_reorder_schur (C ABI) on slabs copied from/to pinned host memory on every rank; "
                      "max over ranks"}
        del hs, hq
    D.nccl_comm_destroy(comm)
    # executed update flops of every rank (its slabs; factor rows skipped where
    # Q is exactly zero), summed over ranks
    fl = torch.tensor([info["flops_left"] + info["flops_right"] + info["flops_factor_exec"]], device=dev,
                      dtype=torch.float64)
    dist.all_reduce(fl)
    if rank == 0:
        agg = float(fl.item()) / (ms_step * 1e-3) / 1e12
        roof = {"bound": "tensor", "kernel": "all DMMA update kernels of the step, all ranks (aggregate)",
                "achieved": round(agg / world, 3), "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": round(agg / world / FP64_DMMA_PEAK_TFLOPS, 4), "traffic": None,
                "executed_flops_all_ranks": float(fl.item()), "reference_flop_count": info["update_flops"],
                "note": "per-GPU share of the executed update flops / step time (max over ranks)"}
        out = {"metric": METRIC, "value": round(ms_step / 1e3, 6), "unit": "s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": False,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (SURVEY.md 8d Schur form, each rank generates its slabs in HBM)",
               "config": {"workload": f"{workload_name(n)}: reorder_schur n={n}, 35% selected (select_fraction seed "
                                      f"{SEL_SEED}), Q accumulated, window {args.ws or 128}", "n": n,
                          "window_size": args.ws or 128, "fraction": FRACTION,
                          "parallelism": f"dist{world}: S column slabs {list(map(int, cb))}, Q row slabs, "
                                         "owners' Q_w broadcast (grouped NCCL) per wavefront + halo send/recv",
                          "l2": "inputs >> 126 MB L2"},
               "update_tflops": round(info["update_flops"] / (ms_step * 1e-3) / 1e12, 3),
               "update_flops": info["update_flops"], "windows": info["n_windows"], "levels": info["n_levels"],
               "clean": info["clean"] == 1, "parity": parity, "gpu_launches": info["n_launches"],
               "roofline": roof, "e2e": e2e, "clocks": clocks, "wall_s_timed_region": round(t_wall, 3), "step_ms": [round(x, 3) for x in step_ms]}
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


def run_c5(args, dev, steps=2, warmup=1, ws=64):
    """C5 (configs[4]): generalized (S, T) Schur-pair reordering with Q and Z,
    n=20000, 35% selected, one GPU.  T from the library's C5 generator
    (SURVEY.md 8d); the reference has no generalized path: the CPU baseline
    is LAPACK DTGSEN (third party, scipy-openblas) on a bounded sample."""
    import torch
    import paper_2002_05024_b200 as T
    n = args.c5_n
    S0 = T.gen_schur_input(n, T.known_spectrum_seed(FILL_SEED_BASE), device=dev)
    T0 = T.gen_pair_t(n, 7, device=dev)
    sel = T.select_fraction(S0, FRACTION, SEL_SEED)
    S, Tm, Q, Z = (T.colmajor_empty(n, dev) for _ in range(4))
    I = T.identity(n, dev)
    opts = T.ReorderOptions(window_size=ws)

    def reset():
        S.copy_(S0)
        Tm.copy_(T0)
        Q.copy_(I)
        Z.copy_(I)

    for _ in range(warmup):
        reset()
        T.greorder_schur(S, Tm, Q, Z, sel, opts)
    stream = torch.cuda.current_stream(dev)
    ms = []
    for _ in range(steps):
        reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = T.greorder_schur(S, Tm, Q, Z, sel, opts)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = statistics.mean(ms) / 1e3
    bs = float(torch.linalg.norm(S0 - Q @ S @ Z.t()) / torch.linalg.norm(S0))
    bt = float(torch.linalg.norm(T0 - Q @ Tm @ Z.t()) / torch.linalg.norm(T0))
    oq = float(torch.linalg.norm(Q.t() @ Q - I.t() @ I))
    oz = float(torch.linalg.norm(Z.t() @ Z - I.t() @ I))
    tol = 10 * n * 2.220446049250313e-16
    eig_pos = positional_eigs_pencil(S0, T0, S, Tm, sel)
    out = {"workload": f"C5: generalized (S,T) reorder n={n}, 35% selected (seed {SEL_SEED}), Q and Z accumulated, "
                       f"window {ws}", "value": round(t, 4), "unit": "s", "step_ms": [round(x, 1) for x in ms],
           "update_flops": res.info["update_flops"], "update_tflops": round(res.info["update_flops"] / t / 1e12, 3),
           "windows": res.info["n_windows"], "levels": res.info["n_levels"], "clean": res.clean,
           "parity": {"backward_error_S": bs, "backward_error_T": bt, "orthogonality_Q": oq, "orthogonality_Z": oz,
                      "tol_10neps": tol, "eig_positional": eig_pos,
                      "pass": max(bs, bt, oq, oz) <= tol and eig_pos["pass"],
                      "eigenvalues": "positional at n=20000 (eig_positional, predicted order); position-by-position "
                                     "vs LAPACK DTGSEN to 1e-10 up to n=2000 in tests/test_greorder_gpu.py"}}
    del S, Tm, Q, Z, I, S0, T0
    torch.cuda.empty_cache()
    if not args.no_cpu:
        out["cpu_baseline"] = c5_cpu_baseline(n)
    return out


def c5_cpu_baseline(n_full, n_sample=1500):
    """LAPACK DTGSEN (scipy-openblas; the reference has no generalized path)
    on the same construction at n_sample, extrapolated by (n/n_sample)^3."""
    from oracle import oracle as O
    S = O.schur_input(n_sample, O.known_spectrum_seed(FILL_SEED_BASE))
    Tt = O.pair_t(n_sample, 7)
    sizes = O.scan_blocks(S).astype(np.int64)
    flags = O.select_fraction(len(sizes), FRACTION, SEL_SEED)
    starts = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
    rows = np.zeros(n_sample, dtype=np.int32)
    for i, f in enumerate(flags):
        if f:
            rows[starts[i]:starts[i + 1]] = 1
    t0 = time.perf_counter()
    O.lapack_tgsen(S, Tt, rows)
    secs = time.perf_counter() - t0
    return {"value": round(secs * (n_full / n_sample) ** 3, 1), "unit": "s", "cores": os.cpu_count() or 1,
            "kind": "third-party (LAPACK DTGSEN via scipy-openblas; no reference implementation exists)",
            "sample": f"dtgsen of the n={n_sample} C5 pencil with Q and Z in {secs:.2f} s, extrapolated to "
                      f"n={n_full} by (n/{n_sample})^3", "sample_seconds": round(secs, 3)}

# ---------------------------------------------------------------------------
# C3: Schur reduction (multishift QR + AED) of a random upper Hessenberg matrix

SCHUR_SEED = 1
SCHUR_CPU_N = 0     # 0: the full C3 matrix (~30 s of the reference on 16 host threads)


def run_schur(args, dev, steps=2, warmup=1, with_cpu=True, with_e2e=True):
    """One step = one full schur_reduce (Q accumulated, Q_in = I) of
    generate(hessenberg_random, n, seed 1), generated in HBM (bit-identical
    to the reference generator), restored before every step."""
    import torch
    import paper_2002_05024_b200 as T
    n = args.schur_n
    H0 = T.gen_hessenberg(n, SCHUR_SEED, device=dev)
    H = T.colmajor_empty(n, dev)
    Q = T.colmajor_empty(n, dev)
    Q0 = T.identity(n, dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(warmup):
        H.copy_(H0)
        Q.copy_(Q0)
        T.schur_reduce(H, Q)
    torch.cuda.synchronize()
    ms, infos = [], []
    for _ in range(steps):
        H.copy_(H0)
        Q.copy_(Q0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = T.schur_reduce(H, Q, T.SchurOptions(profile=True))
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        infos.append(res.info)
    info = infos[-1]
    back = float(torch.linalg.norm(H0 - Q @ H @ Q.t()) / torch.linalg.norm(H0))
    orth = float(torch.linalg.norm(Q.t() @ Q - torch.eye(n, dtype=torch.float64, device=dev)))
    from oracle import oracle as O
    std = bool(O.is_standardized(H.cpu().numpy())) if n <= 12000 else None
    t = statistics.mean(ms) / 1e3
    tol = 10 * n * 2.220446049250313e-16
    upd_ms = sum(i["ms_update"] for i in infos) / len(infos)
    win_ms = sum(i["ms_window"] for i in infos) / len(infos)
    ach = info["update_flops"] / (upd_ms * 1e-3) / 1e12 if upd_ms > 0 else 0.0
    out = {"workload": f"C3: schur_reduce of generate(hessenberg_random, n={n}, seed {SCHUR_SEED}), Q accumulated, "
                       f"SchurOptions defaults (norm-stable, 64 shifts, AED window 96, chase window 128)",
           "value": round(t, 4), "unit": "s", "steps": steps, "warmup": warmup,
           "step_ms": [round(x, 2) for x in ms], "converged": bool(info["converged"]), "sweeps": info["sweeps"],
           "rounds": info["rounds"], "aed_windows": info["aed_windows"], "chase_windows": info["chase_windows"],
           "update_flops": info["update_flops"], "gpu_launches": info["n_launches"],
           "parity": {"backward_error": back, "orthogonality": orth, "tol_10neps": tol, "standardized": std,
                      "pass": back <= tol and orth <= tol and std is not False},
           "time_split_ms": {"window_kernels": round(win_ms, 2), "update_kernels_both_streams": round(upd_ms, 2)},
           "roofline": {"bound": "tensor", "kernel": "update_left/right DMMA kernels of the Schur rounds",
                        "achieved": round(ach, 3), "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                        "frac": round(ach / FP64_DMMA_PEAK_TFLOPS, 4), "traffic": None,
                        "note": "the step is bound by the single-CTA AED window kernel (latency, no roofline): "
                                "see time_split_ms"}}
    if with_e2e:
        Hh = H0.t().contiguous().cpu().numpy().copy()  # row-major of H^T == column-major of H
        Qh = np.eye(n)
        e2e = []
        for _ in range(2):
            hh, qh = Hh.copy(), Qh.copy()
            t0 = time.perf_counter()
            T.schur.schur_reduce_host_buffers(hh, qh, n)
            e2e.append(time.perf_counter() - t0)
        out["e2e"] = {"value": round(min(e2e), 4), "unit": "s", "h2d_bytes_per_step": 2 * n * n * 8,
                      "d2h_bytes_per_step": 2 * n * n * 8, "api": "teig_schur_reduce_host (C ABI, host H,Q)"}
    if with_cpu:
        out["cpu_baseline"] = schur_cpu_baseline()
    return out


def schur_cpu_baseline(n_sample=SCHUR_CPU_N, n_full=None):
    from oracle import oracle as O
    n_full = n_full or 10000
    n_sample = n_sample or n_full
    cores = os.cpu_count() or 1
    h = O.hessenberg_random(n_sample, SCHUR_SEED)
    if O.ref_available():
        r = O.ref_schur_reduce(np.ascontiguousarray(h), np.eye(n_sample), workers=cores)
        secs, kind = r["seconds"], "reference"
    else:
        hf, qf = np.asfortranarray(h.copy()), np.asfortranarray(np.eye(n_sample))
        t0 = time.perf_counter()
        O.schur_reduce(hf, qf)
        secs, kind, cores = time.perf_counter() - t0, "port", 1
    full = secs * (n_full / n_sample) ** 3
    return {"value": round(full, 2), "unit": "s", "cores": cores, "kind": kind,
            "sample": (f"the full workload: schur_reduce of generate(hessenberg_random, n={n_sample}, seed {SCHUR_SEED}) "
                       f"with Q, {cores} threads" if n_sample == n_full else
                       f"schur_reduce of generate(hessenberg_random, n={n_sample}, seed {SCHUR_SEED}) with Q timed in "
                       f"{secs:.2f} s with {cores} threads, extrapolated to n={n_full} by (n/{n_sample})^3"),
            "sample_seconds": round(secs, 3)}


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the unmodified reference built from its sources,
# else the C restatement), bounded sample of the same workload.

def _cpu_problem(n):
    from oracle import oracle as O
    S = O.schur_input(n, O.known_spectrum_seed(FILL_SEED_BASE))
    sizes = O.scan_blocks(S)
    flags = O.select_fraction(len(sizes), FRACTION, SEL_SEED)
    return O, S, sizes, flags


def _group_members(sizes, flags, ws):
    """Selected blocks of each group, in order (reorder.cpp:259-267); group
    membership only depends on the original arrangement because earlier groups
    move up from above later ones."""
    starts = np.concatenate([[0], np.cumsum(sizes.astype(np.int64))])
    sel_idx = np.nonzero(flags)[0]
    groups, i = [], 0
    while i < len(sel_idx):
        fs = sel_idx[i]
        rows = int(sizes[fs])
        g = [fs]
        i += 1
        while i < len(sel_idx):
            gi = sel_idx[i]
            if rows + sizes[gi] > ws // 2 or starts[gi + 1] - starts[fs] > ws:
                break
            rows += int(sizes[gi])
            g.append(gi)
            i += 1
        groups.append(g)
    return groups


def _group_targets(sizes, flags, ws):
    """Groups (selected members) and the target row of each: the rows of the
    selected blocks of all earlier groups (reorder.cpp:248-257)."""
    groups = _group_members(sizes, flags, ws)
    tgt, acc = [], 0
    for g in groups:
        tgt.append(acc)
        acc += int(sizes[g].sum())
    return groups, tgt


def _sample_keep(sizes, groups, tgt, g0, m):
    """A bounded sample of the full reorder: groups g0 .. g0+m-1 run EXACTLY
    the window chains they run in the full problem (same targets, so the same
    window positions and orders) because every block in the leading tgt[g0]
    rows is marked selected -- already in place, the reference skips them
    (reorder.cpp:244-246) -- and everything else is unselected."""
    starts = np.concatenate([[0], np.cumsum(sizes.astype(np.int64))])
    keep = np.zeros(len(sizes), dtype=np.uint8)
    k = int(np.searchsorted(starts, tgt[g0]))  # first block starting at/after the target row
    keep[:k] = 1
    for g in groups[g0:g0 + m]:
        keep[g] = 1
    return keep


class RefSampler:
    """Times the reference's reorder_schur (oracle/_ref: the unmodified
    reference, all host threads) on stratified samples of the full workload:
    each sample is a run of consecutive groups at a position spread over the
    diagonal (_sample_keep), extrapolated to the full problem by update flops
    (F_total / F_sample, both from the planner).  The input is generated and
    converted to the reference's TiledMatrix once (RefProblem); a sample times
    reorder_schur alone.  Without oracle/_ref (never on the driver's box) the
    C restatement runs the same samples single-threaded ("port")."""

    def __init__(self, n, ws):
        from oracle import oracle as O
        self.O, self.n, self.ws = O, n, ws
        S = O.schur_input(n, O.known_spectrum_seed(FILL_SEED_BASE))
        self.sizes = O.scan_blocks(S)
        self.flags = O.select_fraction(len(self.sizes), FRACTION, SEL_SEED)
        plan, self.F_total, ng = O.plan_reorder(self.sizes, self.flags, ws, n)
        d = (plan[:, 1] - plan[:, 0]).astype(np.float64)
        fw = 2 * d * d * (n - plan[:, 1]) + 2 * d * d * plan[:, 0] + 2 * d * d * n
        self.per_group = np.bincount(plan[:, 4], weights=fw, minlength=ng)
        self.groups, self.tgt = _group_targets(self.sizes, self.flags, ws)
        assert len(self.groups) == ng
        self.use_ref = O.ref_available()
        self.cores = os.cpu_count() or 1
        if self.use_ref:
            self.prob = O.RefProblem(S)
            self.S = None
        else:
            self.prob = None
            self.S = S
        del S

    def sample(self, pos, flops):
        """pos in [0, 1): where along the group sequence; flops: sample size."""
        ng = len(self.groups)
        g0 = min(ng - 1, int(pos * ng))
        m, f = 0, 0.0
        while g0 + m < ng and (m == 0 or f < flops):
            f += self.per_group[g0 + m]
            m += 1
        keep = _sample_keep(self.sizes, self.groups, self.tgt, g0, m)
        _, F_sample, _ = self.O.plan_reorder(self.sizes, keep, self.ws, self.n)
        if self.use_ref:
            r = self.prob.run(keep, window_size=self.ws, workers=self.cores, with_q=True)
            t = r["seconds"]
        else:
            s = self.S.copy(order="F")
            q = np.asfortranarray(np.eye(self.n))
            t0 = time.perf_counter()
            self.O.reorder_schur(s, q, self.sizes, keep, self.ws)
            t = time.perf_counter() - t0
        return {"groups": (g0, m), "seconds": t, "flops": F_sample, "extrapolated_s": t * self.F_total / F_sample}

    def describe(self, samples):
        t = sum(x["seconds"] for x in samples)
        f = sum(x["flops"] for x in samples)
        ng = len(self.groups)
        return (f"{len(samples)} stratified samples of the same n={self.n} workload, each a run of consecutive "
                f"window chains (groups {', '.join(f'{g}-{g + m - 1}' for (g, m) in (x['groups'] for x in samples))}"
                f" of {ng}) with the chains' true targets (leading rows selected in place), "
                f"{100 * f / self.F_total:.2f}% of the update flops, timed {t:.1f} s with "
                f"{self.cores if self.use_ref else 1} threads, each extrapolated to the full workload by update flops")


def cpu_baseline(args, n, positions=(0.1, 0.45, 0.8), sample_flops=3.0e11):
    """~1e12 update flops of the same workload (3 stratified samples), about
    20 s of the reference on the box's host threads."""
    rs = RefSampler(n, args.ws or 128)
    samples = [rs.sample(p, sample_flops) for p in positions]
    v = statistics.mean(x["extrapolated_s"] for x in samples)
    out = {"value": round(v, 3), "unit": "s", "cores": rs.cores if rs.use_ref else 1,
           "kind": "reference" if rs.use_ref else "port", "sample": rs.describe(samples),
           "sample_seconds": round(sum(x["seconds"] for x in samples), 3),
           "flops_fraction": round(sum(x["flops"] for x in samples) / rs.F_total, 5),
           "per_sample_extrapolated_s": [round(x["extrapolated_s"], 1) for x in samples]}
    del rs
    return out


def run_reference(args, rank, world, local):
    """The reference arm: the unmodified reference's reorder_schur on the host
    cores, one stratified sample per step (positions spread over the
    diagonal), the line's value = the mean extrapolated full-workload time."""
    if rank != 0:
        return
    n = args.n
    rs = RefSampler(n, args.ws or 128)
    total = args.warmup + args.steps
    t = []
    samples = []
    for k in range(total):
        pos = ((k - args.warmup) + 0.5) / max(args.steps, 1) if k >= args.warmup else (k + 0.25) / max(total, 1)
        x = rs.sample(pos, 1.5e11)
        if k >= args.warmup:
            t.append(x["extrapolated_s"])
            samples.append(x)
    v = statistics.mean(t)
    res = {"value": round(v, 3), "unit": "s", "cores": rs.cores if rs.use_ref else 1,
           "kind": "reference" if rs.use_ref else "port", "sample": rs.describe(samples),
           "per_step_extrapolated_s": [round(x, 1) for x in t]}
    out = {"metric": METRIC, "impl": "reference", "value": round(v, 3), "unit": "s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v * 1e3, 1),
           "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (SURVEY.md 8d Schur form, reference Philox generator)",
           "config": {"workload": f"{workload_name(n)}: reorder_schur n={n}, 35% selected (select_fraction seed "
                                  f"{SEL_SEED}), Q accumulated, window {args.ws or 128}", "n": n,
                      "window_size": args.ws or 128, "fraction": FRACTION},
           "cpu_baseline": res,
           "e2e": {"value": round(v, 3), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_schur_line(args, rank, world, local):
    """--workload schur: the C3 measurement as the line's headline."""
    import torch
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if args.impl == "reference":
        if rank != 0:
            return
        vals = [schur_cpu_baseline(n_full=args.schur_n) for _ in range(max(1, args.steps))]
        v = statistics.mean(x["value"] for x in vals)
        out = {"metric": METRIC, "impl": "reference", "value": round(v, 3), "unit": "s", "n_gpus": world,
               "steps": args.steps, "warmup": 0, "higher_is_better": False, "scaling": "weak",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference hessenberg_random generator)",
               "config": {"workload": f"C3: schur_reduce n={args.schur_n}"}, "cpu_baseline": vals[-1],
               "e2e": {"value": round(v, 3), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out), flush=True)
        return
    import paper_2002_05024_b200 as T
    T.set_memory_retention(True)
    sampler = ClockSampler(local)
    sampler.start()
    r = run_schur(args, dev, steps=args.steps, warmup=max(args.warmup, 1), with_cpu=(rank == 0 and not args.no_cpu),
                  with_e2e=not args.no_e2e)
    clocks = sampler.stop()
    if rank != 0:
        return
    out = {"metric": METRIC, "value": r["value"], "unit": "s", "n_gpus": world, "steps": args.steps,
           "warmup": max(args.warmup, 1), "ms_per_step": round(r["value"] * 1e3, 2), "higher_is_better": False,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (reference hessenberg_random generator, in HBM)",
           "config": {"workload": r["workload"], "n": args.schur_n, "parallelism": "single-gpu",
                      "l2": "H + Q = 1.6 GB > 126 MB L2"},
           "roofline": r["roofline"], "e2e": r.get("e2e"), "gpu_launches": r["gpu_launches"], "clocks": clocks,
           "parity": r["parity"], "cpu_baseline": r.get("cpu_baseline"), "schur": r}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.workload == "schur":
        run_schur_line(args, rank, world, local)
    elif args.impl == "reference":
        run_reference(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
