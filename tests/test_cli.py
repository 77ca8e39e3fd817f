"""plnmf-gpu, the C++ front end (csrc/cli/plnmf_gpu.cpp): the reference CLI's
factorize / sweep-tiles / compare / model commands (proj/tools/plnmf.cpp) on the
engine.  CPU: the model command's tile choices match the reference's cost model
(SURVEY.md 8(d) T_auto values).  GPU: the report has report_to_json's schema
(proj/src/run_report.cpp:40-66) plus the "gpu" object, reference-order runs
reproduce the compiled reference's trace bit for bit, compare prints the
lockstep table and its "max factor deviation" line."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from _helpers import bits_equal
from oracle import oracle as O
from paper_1904_07935_b200 import build as B
from paper_1904_07935_b200 import plnmf as P

CLI = B.CLI


def run(*args, check=True):
    res = subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, timeout=900)
    if check:
        assert res.returncode == 0, res.stderr
    return res


@pytest.mark.parametrize("k,t_auto", [(80, 9), (240, 16), (480, 22), (160, 13)])
def test_model_tile_matches_the_reference_cost_model(k, t_auto):
    out = run("model", "--k", k, "--v", 26214, "--d", 11314).stdout
    assert f"best integer tile: {t_auto}" in out


def test_cli_errors_are_reported():
    res = run("factorize", "--k", "4", "--synthetic", "10,10,0.5,1", "--algorithm", "nmf", check=False)
    assert res.returncode == 1 and "error:" in res.stderr
    res = run("factorize", "--k", "0", check=False)
    assert res.returncode == 1


def _mm(tmp_path, m):
    p = tmp_path / "a.mtx"
    rows, cols = m.rows, m.cols
    lines = ["%%MatrixMarket matrix coordinate real general", f"{rows} {cols} {m.nnz()}"]
    for r in range(rows):
        for e in range(m.row_ptr[r], m.row_ptr[r + 1]):
            lines.append(f"{r + 1} {m.col_idx[e] + 1} {float(m.values[e])!r}")
    p.write_text("\n".join(lines) + "\n")
    return p


@pytest.mark.gpu
def test_factorize_report_schema_and_reference_order_bitwise(gpu, tmp_path):
    m = P.synth_csr(600, 400, 0.03, 9)
    path = _mm(tmp_path, m)
    out = tmp_path / "r.json"
    nth = O.ref().ref_max_threads() if O.have_ref() else 1
    run("factorize", "--input", path, "--k", 12, "--algorithm", "pl-nmf", "--tile", 5, "--max-iters", 8,
        "--tol", 0, "--math", "reference-order", "--threads", nth, "--output", out)
    rep = json.loads(out.read_text())
    for key in ("problem", "algorithm", "tile", "config", "initial_rel_error", "final_rel_error", "total_seconds",
                "phase_seconds", "cost_model", "trace", "gpu"):
        assert key in rep
    assert rep["problem"] == {"v": 600, "d": 400, "k": 12, "nnz": m.nnz(), "sparsity": 1.0 - m.nnz() / 240000}
    assert rep["tile"] == {"size": 5, "provenance": "explicit"} and len(rep["trace"]) == 8
    assert rep["gpu"]["kernel_launches"] > 0 and rep["gpu"]["math"] == "reference-order"
    if O.have_ref():
        a = O.RefInput(m.rows, m.cols, m.row_ptr, m.col_idx, m.values)
        w, ht = O.ref_init_factors(m.rows, m.cols, 12)
        prev = O.ref().ref_max_threads()
        O.ref().ref_set_threads(nth)
        _, _, tr = O.ref_iterate(a, w, ht, 12, max_iters=8, rel_tol=0.0, tile=5, tiled=True)
        O.ref().ref_set_threads(prev)
        assert bits_equal([r["rel_error"] for r in rep["trace"]], tr["records"][:, 1])
        assert rep["initial_rel_error"] == tr["initial_error"]


@pytest.mark.gpu
def test_factorize_synthetic_csv_and_auto_tile(gpu, tmp_path):
    res = run("factorize", "--synthetic", "2000,900,0.02,20", "--k", 30, "--max-iters", 5, "--tol", 0,
              "--format", "csv-trace")
    lines = res.stdout.strip().splitlines()
    assert lines[0] == "iteration,rel_error,elapsed_s" and len(lines) == 6
    out = tmp_path / "g.json"
    run("factorize", "--synthetic", "2000,900,0.02,20", "--k", 30, "--max-iters", 3, "--tile", "gpu",
        "--output", out)
    rep = json.loads(out.read_text())
    assert rep["tile"]["provenance"] == "gpu-measured" and 1 <= rep["tile"]["size"] <= 30


@pytest.mark.gpu
def test_compare_and_sweep(gpu, tmp_path):
    res = run("compare", "--synthetic", "1500,900,0.02,20", "--k", 16, "--tile", 5, "--max-iters", 3)
    lines = res.stdout.strip().splitlines()
    assert lines[0].startswith("initial rel error:") and "fast-hals" in lines[1] and "pl-nmf(T=5)" in lines[1]
    assert len(lines) == 6 and lines[-1].startswith("max factor deviation:")
    dev1 = float(lines[2].split()[3])
    assert dev1 <= 1e-10  # iteration 1: the two paths agree to rounding
    csv = tmp_path / "s.csv"
    res = run("sweep-tiles", "--synthetic", "1500,900,0.02,20", "--k", 16, "--max-iters", 2, "--grid", "1,4,16",
              "--output", csv)
    assert "fastest on this GPU" in res.stdout
    assert csv.read_text().splitlines()[0] == "tile,seconds,predicted_vol,model_recommended"
