"""Command-line harness over the B200 path (the reference's
CLI is a stub, proj/tools/taskeig.cpp:1 -- this follows its specification,
SPEC.md "[MODULE] cli"): generate problems, run the phases, verify, emit JSON
reports with residuals, eigenvalues, timings and optional execution traces.

  python -m paper_2002_05024_b200.cli <command> [flags]

  generate   --kind {schur,hessenberg,dense,pair-t} --n N --seed S --out PATH
             (schur: the synthetic standardized Schur form of SURVEY 8d, with
             a sidecar PATH.json listing its spectrum; hessenberg: the
             reference's generate(hessenberg_random); dense: uniform [-1, 1)
             entries; pair-t: the C5 T factor)
  reorder    --s S [--q Q] --select SPEC [--window-size W] [--strict]
             --out-s S2 [--out-q Q2] [--report R.json] [--trace T.json]
  hessenberg --a A --out-h H [--out-q Q] [--panel-width B] [--report R.json]
  schur      --h H [--q Q] [--deflation {classic,norm-stable}] [--shift-count M]
             [--aed-window W] --out-s S [--out-q Q] [--report R.json]
  pipeline   (--a A | --h H) [--select SPEC] --out-s S --out-q Q [--report R.json]
             (hessenberg_reduce for --a, schur_reduce, reorder_schur if
             --select, then verify against the input)
  verify     --a A --q Q --s S [--tol-backward T] [--tol-orth T] [--report R.json]
  trace-dump --trace T.json   (per-kind launch counts and device time)

  SPEC: frac=F[,seed=S] | pred=NAME[,k=K] (left-half-plane, inside-unit-disk,
  largest-magnitude-k) | file=PATH (one 0/1 flag per diagonal block)
  --format {teig,matrixmarket} for every matrix file (default teig).

Exit codes: 0 pass, 1 verification failure, 2 non-convergence,
64 usage error.  Every report carries the full run configuration.  All
computation runs on cuda:0 through the C ABI (no CPU fallback); verification
uses cuBLAS (torch) -- independent of the kernels under test.
"""
from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

EPS = 2.220446049250313e-16
EXIT_PASS, EXIT_FAIL, EXIT_NOCONV, EXIT_USAGE = 0, 1, 2, 64


class UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # argparse exits 2 by default; the spec says 64
        raise UsageError(message)


def _parser():
    p = _Parser(prog="taskeig_b200", description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = p.add_subparsers(dest="command")
    g = sub.add_parser("generate")
    g.add_argument("--kind", required=True, choices=["schur", "hessenberg", "dense", "pair-t"])
    g.add_argument("--n", type=int, required=True)
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--out", required=True)
    r = sub.add_parser("reorder")
    r.add_argument("--s", required=True)
    r.add_argument("--q")
    r.add_argument("--select", required=True)
    r.add_argument("--window-size", type=int, default=0)
    r.add_argument("--strict", action="store_true")
    r.add_argument("--out-s", required=True)
    r.add_argument("--out-q")
    r.add_argument("--trace")
    hs = sub.add_parser("hessenberg")
    hs.add_argument("--a", required=True)
    hs.add_argument("--out-h", required=True)
    hs.add_argument("--out-q")
    hs.add_argument("--panel-width", type=int, default=0)
    s = sub.add_parser("schur")
    s.add_argument("--h", required=True)
    s.add_argument("--q")
    s.add_argument("--deflation", choices=["classic", "norm-stable"], default="norm-stable")
    s.add_argument("--shift-count", type=int, default=0)
    s.add_argument("--aed-window", type=int, default=0)
    s.add_argument("--out-s", required=True)
    s.add_argument("--out-q")
    pl = sub.add_parser("pipeline")
    src = pl.add_mutually_exclusive_group(required=True)
    src.add_argument("--a")
    src.add_argument("--h")
    pl.add_argument("--select")
    pl.add_argument("--deflation", choices=["classic", "norm-stable"], default="norm-stable")
    pl.add_argument("--window-size", type=int, default=0)
    pl.add_argument("--out-s", required=True)
    pl.add_argument("--out-q", required=True)
    pl.add_argument("--tol-backward", type=float, default=None)
    pl.add_argument("--tol-orth", type=float, default=None)
    v = sub.add_parser("verify")
    v.add_argument("--a", required=True)
    v.add_argument("--q", required=True)
    v.add_argument("--s", required=True)
    v.add_argument("--tol-backward", type=float, default=None)
    v.add_argument("--tol-orth", type=float, default=None)
    t = sub.add_parser("trace-dump")
    t.add_argument("--trace", required=True)
    for sp in (g, r, hs, s, pl, v):
        sp.add_argument("--format", choices=["teig", "matrixmarket"], default="teig")
    for sp in (r, hs, s, pl, v):
        sp.add_argument("--report")
    return p


# --------------------------------------------------------------------------

def _dev():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 path has no CPU fallback")
    return torch.device("cuda", 0)


def _load(path, fmt):
    import torch
    from . import io
    a = io.read_matrix_file(path, fmt)
    if a.shape[0] != a.shape[1]:
        raise UsageError(f"{path}: a square matrix is required, got {a.shape}")
    t = torch.empty((a.shape[0], a.shape[0]), dtype=torch.float64, device=_dev()).t()  # column-major
    t.copy_(torch.as_tensor(a))
    return t


def _save(path, t, fmt):
    from . import io
    io.write_matrix_file(path, t.cpu().numpy(), fmt)


def _selection(T, s, spec: str):
    kind, _, rest = spec.partition("=")
    if kind == "frac":
        parts = rest.split(",")
        frac = float(parts[0])
        seed = 0
        for p in parts[1:]:
            k, _, val = p.partition("=")
            if k != "seed":
                raise UsageError(f"--select frac: unknown key {k!r}")
            seed = int(val)
        return T.select_fraction(s, frac, seed)
    if kind == "pred":
        parts = rest.split(",")
        k = 0
        for p in parts[1:]:
            key, _, val = p.partition("=")
            if key != "k":
                raise UsageError(f"--select pred: unknown key {key!r}")
            k = int(val)
        return T.select_by_name(s, parts[0], k)
    if kind == "file":
        flags = [int(x) != 0 for x in open(rest).read().split()]
        return T.select_eigenvalues(s, flags)
    raise UsageError("--select must be frac=F[,seed=S] | pred=NAME[,k=K] | file=PATH")


def _residuals(A, Q, S):
    import torch
    n = A.shape[0]
    nrm = float(torch.linalg.norm(A))
    back = float(torch.linalg.norm(A - Q @ S @ Q.t())) / (nrm if nrm > 0 else 1.0)
    orth = float(torch.linalg.norm(Q.t() @ Q - torch.eye(n, dtype=torch.float64, device=A.device)))
    return back, orth


def _eigs(s):
    """Eigenvalues read off the standardized quasi-triangular form (O(n))."""
    d = s.diagonal(0).cpu().numpy()
    u = s.diagonal(1).cpu().numpy()
    lo = s.diagonal(-1).cpu().numpy()
    ev = d.astype(complex)
    r = 0
    while r < len(d):
        if r + 1 < len(d) and lo[r] != 0.0:
            im = np.sqrt(abs(u[r])) * np.sqrt(abs(lo[r]))
            ev[r], ev[r + 1] = complex(d[r], im), complex(d[r + 1], -im)
            r += 2
        else:
            r += 1
    return [[float(z.real), float(z.imag)] for z in ev]


def _write_report(path, rep):
    if path:
        with open(path, "w") as f:
            json.dump(rep, f, indent=1)
    else:
        json.dump(rep, sys.stdout)
        sys.stdout.write("\n")


def _verdict(rep, back, orth, n, tol_b, tol_o):
    tol_b = 10 * n * EPS if tol_b is None else tol_b
    tol_o = 10 * n * EPS if tol_o is None else tol_o
    failing = [m for m, v, t in (("backward_error", back, tol_b), ("orthogonality", orth, tol_o)) if not v <= t]
    rep.update({"backward_error": back, "orthogonality": orth, "tol_backward": tol_b, "tol_orth": tol_o,
                "pass": not failing, "failing": failing})
    return EXIT_PASS if not failing else EXIT_FAIL


# --------------------------------------------------------------------------

def cmd_generate(a, T):
    import torch
    dev = _dev()
    if a.n < 1:
        raise UsageError("--n must be >= 1")
    if a.kind == "schur":
        m = T.gen_schur_input(a.n, T.known_spectrum_seed(a.seed), device=dev)
    elif a.kind == "hessenberg":
        m = T.gen_hessenberg(a.n, a.seed, device=dev)
    elif a.kind == "dense":
        g = torch.Generator(device=dev).manual_seed(a.seed)
        m = (torch.rand(a.n, a.n, dtype=torch.float64, device=dev, generator=g) * 2 - 1).t().contiguous().t()
    else:
        m = T.gen_pair_t(a.n, a.seed, device=dev)
    torch.cuda.synchronize()
    _save(a.out, m, a.format)
    side = {"kind": a.kind, "n": a.n, "seed": a.seed, "format": a.format}
    if a.kind == "schur":
        side["spectrum"] = _eigs(m)
    with open(a.out + ".json", "w") as f:
        json.dump(side, f)
    return EXIT_PASS


def cmd_reorder(a, T):
    s = _load(a.s, a.format)
    n = s.shape[0]
    s0 = s.clone()
    q = _load(a.q, a.format) if a.q else T.identity(n)
    q0 = q.clone()
    sel = _selection(T, s, a.select)
    if a.trace:
        T.trace_enable(True)
    t0 = time.perf_counter()
    try:
        r = T.reorder_schur(s, q, sel, T.ReorderOptions(window_size=a.window_size, strict=a.strict))
    except RuntimeError as e:  # strict-mode rejection
        _write_report(a.report, {"config": vars(a), "error": str(e), "pass": False})
        return EXIT_FAIL
    wall = time.perf_counter() - t0
    if a.trace:
        with open(a.trace, "w") as f:
            f.write(T.trace_json())
        T.trace_enable(False)
    _save(a.out_s, s, a.format)
    if a.out_q:
        _save(a.out_q, q, a.format)
    A = q0 @ s0 @ q0.t()
    back, orth = _residuals(A, q, s)
    rep = {"config": vars(a), "n": n, "phase_seconds": {"reorder": wall}, "clean": r.clean,
           "rejected_blocks": r.rejected_blocks, "permutation": r.permutation, "windows": r.info["n_windows"],
           "passes": r.info["n_passes"], "eigenvalues": _eigs(s)}
    code = _verdict(rep, back, orth, n, None, None)
    _write_report(a.report, rep)
    return code


def cmd_hessenberg(a, T):
    A = _load(a.a, a.format)
    n = A.shape[0]
    A0 = A.clone()
    t0 = time.perf_counter()
    r = T.hessenberg_reduce(A, True, T.HessenbergOptions(panel_width=a.panel_width))
    wall = time.perf_counter() - t0
    _save(a.out_h, r.h, a.format)
    if a.out_q:
        _save(a.out_q, r.q, a.format)
    back, orth = _residuals(A0, r.q, r.h)
    rep = {"config": vars(a), "n": n, "phase_seconds": {"hessenberg": wall}, "panels": r.info["panels"]}
    code = _verdict(rep, back, orth, n, None, None)
    _write_report(a.report, rep)
    return code


def _schur(T, h, q, deflation, shift_count=0, aed_window=0):
    d = T.DeflationCondition.classic if deflation == "classic" else T.DeflationCondition.norm_stable
    opts = T.SchurOptions(deflation=d, shift_count=shift_count, aed_window=aed_window)
    t0 = time.perf_counter()
    sd = T.schur_reduce(h, q, opts)
    return sd, time.perf_counter() - t0


def cmd_schur(a, T):
    h = _load(a.h, a.format)
    n = h.shape[0]
    h0 = h.clone()
    q = _load(a.q, a.format) if a.q else T.identity(n)
    q0 = q.clone()
    sd, wall = _schur(T, h, q, a.deflation, a.shift_count, a.aed_window)
    _save(a.out_s, h, a.format)
    if a.out_q:
        _save(a.out_q, q, a.format)
    back, orth = _residuals(q0 @ h0 @ q0.t(), q, h)
    rep = {"config": vars(a), "n": n, "phase_seconds": {"schur": wall}, "converged": sd.converged,
           "sweeps": sd.sweeps, "eigenvalues": [[float(z.real), float(z.imag)] for z in sd.eigenvalues]}
    code = _verdict(rep, back, orth, n, None, None)
    if not sd.converged:
        rep["converged_trailing"] = sd.converged_trailing
        code = EXIT_NOCONV
    _write_report(a.report, rep)
    return code


def cmd_pipeline(a, T):
    phases = {}
    if a.a:  # general matrix: Hessenberg reduction first, on the device
        h = _load(a.a, a.format)
        h0 = h.clone()
        t0 = time.perf_counter()
        hr = T.hessenberg_reduce(h, True)
        phases["hessenberg"] = time.perf_counter() - t0
        q = hr.q
    else:
        h = _load(a.h, a.format)
        h0 = h.clone()
        q = T.identity(h.shape[0])
    n = h.shape[0]
    sd, phases["schur"] = _schur(T, h, q, a.deflation)
    rep = {"config": vars(a), "n": n, "phase_seconds": phases, "converged": sd.converged,
           "sweeps": sd.sweeps}
    if not sd.converged:
        rep["converged_trailing"] = sd.converged_trailing
        _write_report(a.report, rep)
        return EXIT_NOCONV
    if a.select:
        sel = _selection(T, h, a.select)
        t0 = time.perf_counter()
        r = T.reorder_schur(h, q, sel, T.ReorderOptions(window_size=a.window_size))
        rep["phase_seconds"]["reorder"] = time.perf_counter() - t0
        rep["clean"] = r.clean
        rep["rejected_blocks"] = r.rejected_blocks
        rep["selected_rows"] = sel.selected_rows()
    _save(a.out_s, h, a.format)
    _save(a.out_q, q, a.format)
    rep["eigenvalues"] = _eigs(h)
    back, orth = _residuals(h0, q, h)
    code = _verdict(rep, back, orth, n, a.tol_backward, a.tol_orth)
    _write_report(a.report, rep)
    return code


def cmd_verify(a, T):
    A = _load(a.a, a.format)
    Q = _load(a.q, a.format)
    S = _load(a.s, a.format)
    n = A.shape[0]
    if Q.shape[0] != n or S.shape[0] != n:
        raise UsageError("verify: A, Q and S must have the same order")
    back, orth = _residuals(A, Q, S)
    rep = {"config": vars(a), "n": n}
    code = _verdict(rep, back, orth, n, a.tol_backward, a.tol_orth)
    import torch
    rep["quasi_triangular"] = bool(float(torch.tril(S, -2).abs().max()) == 0.0) if n > 2 else True
    if not rep["quasi_triangular"]:
        rep["pass"] = False
        rep["failing"].append("quasi_triangular")
        code = EXIT_FAIL
    _write_report(a.report, rep)
    return code


def cmd_trace_dump(a, T):
    tr = json.load(open(a.trace))
    kinds = {}
    for t in tr.get("tasks", []):
        k = t["label"].split(":")[1] if ":" in t["label"] else t["label"]
        e = kinds.setdefault(k, {"launches": 0, "device_ms": 0.0})
        e["launches"] += 1
        e["device_ms"] += (t["end_ns"] - t["start_ns"]) / 1e6
    st = {}
    for w in tr.get("windows", []):
        st[w["status"]] = st.get(w["status"], 0) + 1
    json.dump({"kinds": kinds, "windows": len(tr.get("windows", [])), "window_status": st}, sys.stdout)
    sys.stdout.write("\n")
    return EXIT_PASS


def main(argv=None) -> int:
    try:
        a = _parser().parse_args(argv)
        if not a.command:
            raise UsageError("a command is required (generate, reorder, hessenberg, schur, pipeline, verify, "
                             "trace-dump)")
        import paper_2002_05024_b200 as T
        fn = {"generate": cmd_generate, "reorder": cmd_reorder, "hessenberg": cmd_hessenberg, "schur": cmd_schur,
              "pipeline": cmd_pipeline, "verify": cmd_verify, "trace-dump": cmd_trace_dump}[a.command]
        return fn(a, T)
    except UsageError as e:
        sys.stderr.write(f"usage error: {e}\n")
        return EXIT_USAGE
    except (ValueError, OSError) as e:
        sys.stderr.write(f"error: {e}\n")
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
