"""CLI on the B200 (SPEC.md "[MODULE] cli" examples): generate -> reorder /
schur / pipeline -> verify, JSON reports, exit codes, traces, determinism."""
import json
import os

import numpy as np
import pytest

from paper_2002_05024_b200 import cli

pytestmark = pytest.mark.gpu


def test_generate_is_deterministic_and_sidecar_lists_spectrum(cuda, tmp_path):
    a, b = str(tmp_path / "a.teig"), str(tmp_path / "b.teig")
    assert cli.main(["generate", "--kind", "schur", "--n", "50", "--seed", "7", "--out", a]) == 0
    assert cli.main(["generate", "--kind", "schur", "--n", "50", "--seed", "7", "--out", b]) == 0
    assert open(a, "rb").read() == open(b, "rb").read()
    side = json.load(open(a + ".json"))
    assert len(side["spectrum"]) == 50


@pytest.mark.parametrize("fmt", ["teig", "matrixmarket"])
def test_reorder_then_verify(cuda, tmp_path, fmt):
    s = str(tmp_path / f"s.{fmt}")
    assert cli.main(["generate", "--kind", "schur", "--n", "400", "--seed", "3", "--out", s, "--format", fmt]) == 0
    s2, q2, rep, tr = (str(tmp_path / x) for x in ("s2", "q2", "r.json", "t.json"))
    assert cli.main(["reorder", "--s", s, "--select", "frac=0.35,seed=99", "--window-size", "64", "--out-s", s2,
                     "--out-q", q2, "--report", rep, "--trace", tr, "--format", fmt]) == 0
    r = json.load(open(rep))
    assert r["pass"] and r["clean"] and r["config"]["select"] == "frac=0.35,seed=99"
    assert r["backward_error"] <= 10 * 400 * 2.22e-16
    # independent verification of the files (A = S_in since Q_in = I)
    assert cli.main(["verify", "--a", s, "--q", q2, "--s", s2, "--format", fmt,
                     "--report", str(tmp_path / "v.json")]) == 0
    # a corrupted S fails, naming the metric
    from paper_2002_05024_b200 import io
    bad = io.read_matrix_file(s2, fmt)
    bad[5, 5] += 1e-3
    io.write_matrix_file(s2, bad, fmt)
    assert cli.main(["verify", "--a", s, "--q", q2, "--s", s2, "--format", fmt,
                     "--report", str(tmp_path / "v2.json")]) == 1
    assert "backward_error" in json.load(open(tmp_path / "v2.json"))["failing"]
    # zero tolerances on nontrivial data fail
    assert cli.main(["verify", "--a", s, "--q", q2, "--s", s2, "--format", fmt, "--tol-backward", "0",
                     "--tol-orth", "0", "--report", str(tmp_path / "v3.json")]) == 1
    t = json.load(open(tr))
    assert t["tasks"] and t["windows"] and all(w["status"] == "executed" for w in t["windows"])
    assert {x["label"].split(":")[1] for x in t["tasks"]} >= {"W", "L", "Q"}
    assert cli.main(["trace-dump", "--trace", tr]) == 0


def test_schur_and_pipeline(cuda, tmp_path):
    h = str(tmp_path / "h.teig")
    assert cli.main(["generate", "--kind", "hessenberg", "--n", "300", "--seed", "1", "--out", h]) == 0
    s, q, rep = str(tmp_path / "s"), str(tmp_path / "q"), str(tmp_path / "r.json")
    assert cli.main(["schur", "--h", h, "--out-s", s, "--out-q", q, "--report", rep]) == 0
    r = json.load(open(rep))
    assert r["converged"] and r["pass"] and len(r["eigenvalues"]) == 300
    rep2 = str(tmp_path / "p.json")
    assert cli.main(["pipeline", "--h", h, "--select", "pred=left-half-plane", "--out-s", s, "--out-q", q,
                     "--report", rep2]) == 0
    p = json.load(open(rep2))
    assert p["pass"] and p["clean"] and set(p["phase_seconds"]) == {"schur", "reorder"}
    ev = np.array(p["eigenvalues"])
    k = p["selected_rows"]
    assert np.all(ev[:k, 0] < 0) and np.all(ev[k:, 0] >= 0)


def test_one_by_one(cuda, tmp_path):
    from paper_2002_05024_b200 import io
    h = str(tmp_path / "h.teig")
    io.write_matrix_file(h, np.array([[5.0]]), "teig")
    rep = str(tmp_path / "r.json")
    assert cli.main(["pipeline", "--h", h, "--out-s", str(tmp_path / "s"), "--out-q", str(tmp_path / "q"),
                     "--report", rep]) == 0
    r = json.load(open(rep))
    assert r["eigenvalues"] == [[5.0, 0.0]] and r["backward_error"] == 0.0 and r["orthogonality"] == 0.0


def test_full_pipeline_from_a_general_matrix(cuda, tmp_path):
    """SPEC cmd_pipeline: hessenberg -> schur -> reorder on a general matrix,
    report passes, verify of the written files passes (A = Q S Q^T)."""
    a = str(tmp_path / "a.teig")
    assert cli.main(["generate", "--kind", "dense", "--n", "500", "--seed", "2", "--out", a]) == 0
    s, q, rep = str(tmp_path / "s"), str(tmp_path / "q"), str(tmp_path / "r.json")
    assert cli.main(["pipeline", "--a", a, "--select", "frac=0.35,seed=99", "--out-s", s, "--out-q", q,
                     "--report", rep]) == 0
    r = json.load(open(rep))
    assert r["pass"] and r["converged"] and set(r["phase_seconds"]) == {"hessenberg", "schur", "reorder"}
    assert cli.main(["verify", "--a", a, "--q", q, "--s", s, "--report", str(tmp_path / "v.json")]) == 0
    h, hq = str(tmp_path / "h"), str(tmp_path / "hq")
    assert cli.main(["hessenberg", "--a", a, "--out-h", h, "--out-q", hq, "--report", str(tmp_path / "h.json")]) == 0
    from paper_2002_05024_b200 import io
    H = io.read_matrix_file(h, "teig")
    assert np.all(np.tril(H, -2) == 0.0)
