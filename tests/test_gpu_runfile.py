"""`python -m paper_2004_00546_b200 run --config file.json`: run files in the reference's JSON
layout (its `configs/burgers_hybrid.json` / `linear_d1.json` shapes, written here) on the GPU."""

import csv
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _write(tmp_path, doc):
    p = tmp_path / "run.json"
    p.write_text(json.dumps(doc))
    return str(p)


def test_burgers_hybrid_run_file(cuda_ok, tmp_path):
    """The reference's hybrid run-file shape (32×32 two-field Burgers, D = 1, ω = 1, T = 1,
    f_true = sin x·sin y, f_init = ones): serial and hybrid loops for N = 1, 4, 16, a descent."""
    from paper_2004_00546_b200.__main__ import main
    doc = {"problem": {"kind": "burgers", "nx": 32, "ny": 32, "D": 1.0, "omega": 1.0, "T": 1.0,
                       "f_true": "sin_product", "f_init": "ones"},
           "algorithm": "hybrid", "workers": [1, 4, 16], "rtol": 1e-3, "repeats": 2, "seed": 0,
           "descent": {"steps": 4, "lr": 0.5}}
    out = tmp_path / "res"
    assert main(["run", "--config", _write(tmp_path, doc), "--output", str(out)]) == 0
    rows = list(csv.DictReader(open(out / "results.csv")))
    assert [int(r["N"]) for r in rows] == [1, 4, 16] and all(r["algorithm"] == "hybrid" for r in rows)
    summary = json.load(open(out / "summary.json"))
    assert summary["backend"] == "cuda" and summary["grid"] == [32, 32] and summary["k"] > 0
    # the frozen-span adjoint changes the gradient with N, the direct sweep (hence J) does not
    J = [float(r["J"]) for r in rows]
    assert max(J) - min(J) <= 1e-12 * abs(J[0]) and abs(J[0] - summary["J_serial"]) <= 1e-12 * abs(J[0])
    d = list(csv.DictReader(open(out / "descent.csv")))
    assert len(d) == 4 and float(d[-1]["J"]) < float(d[0]["J"])   # descent from f_init towards f_true
    assert np.load(out / "f_final.npy").shape == (2048,)


def test_linear_run_file_and_errors(cuda_ok, tmp_path):
    from paper_2004_00546_b200.__main__ import main
    doc = {"problem": {"kind": "advection_diffusion", "nx": 32, "ny": 32, "a": 1.0, "D": 1.0, "omega": 1.0, "T": 2.0,
                       "f_true": "sin_product", "f_init": "ones"},
           "algorithm": "linear", "workers": [1, 2, 8], "repeats": 1}
    out = tmp_path / "lin"
    assert main(["run", "--config", _write(tmp_path, doc), "--output", str(out)]) == 0
    rows = list(csv.DictReader(open(out / "results.csv")))
    J = [float(r["J"]) for r in rows]
    g = [float(r["grad_norm"]) for r in rows]
    # Paraexp is exact for the linear problem: J and the gradient do not depend on N beyond the step size
    assert max(J) - min(J) <= 1e-6 * abs(J[0]) and max(g) - min(g) <= 1e-6 * g[0]
    bad = dict(doc, algorithm="hybrid")   # the hybrid needs the nonlinear testbed
    assert main(["run", "--config", _write(tmp_path, bad), "--output", str(out)]) == 1
    assert main(["run", "--config", str(tmp_path / "missing.json")]) == 1


def test_burgers_iterative_run_file(cuda_ok, tmp_path):
    """The reference's `configs/burgers_iterative.json` shape: algorithm "nonlinear" (Algorithm 2), eps 1e-3."""
    from paper_2004_00546_b200.__main__ import main
    doc = {"problem": {"kind": "burgers", "nx": 32, "ny": 32, "D": 1.0, "omega": 1.0, "T": 1.0,
                       "f_true": "sin_product", "f_init": "ones"},
           "algorithm": "nonlinear", "workers": [2, 4, 8], "rtol": 1e-3, "eps": 1e-3, "repeats": 2, "seed": 0}
    out = tmp_path / "it"
    assert main(["run", "--config", _write(tmp_path, doc), "--output", str(out)]) == 0
    rows = list(csv.DictReader(open(out / "results.csv")))
    assert [int(r["N"]) for r in rows] == [2, 4, 8] and all(int(r["K"]) >= 2 for r in rows)
    summary = json.load(open(out / "summary.json"))
    J = [float(r["J"]) for r in rows]
    # the converged iterate is the serial trajectory up to eps and the step size
    assert all(abs(j - summary["J_serial"]) <= 1e-3 * abs(summary["J_serial"]) for j in J)


def test_numbered_baseline_configs_through_the_cli(cuda_ok, tmp_path, capsys):
    """`run --config K` (BASELINE configs), the checkpointed run and `predict` still answer."""
    from paper_2004_00546_b200.__main__ import main
    out = tmp_path / "c1"
    assert main(["run", "--config", "1", "--repeats", "1", "--output", str(out)]) == 0
    s = json.load(open(out / "summary.json"))
    assert s["backend"] == "cuda" and s["timing"]["gradient_evals_per_s"] > 0
    assert main(["run", "--config", "3", "--repeats", "1", "--checkpoints", "3", "--output", str(tmp_path / "c3")]) == 0
    assert json.load(open(tmp_path / "c3" / "summary.json"))["checkpoints"] == 3
    capsys.readouterr()
    assert main(["predict", "--config", "2", "--repeats", "1", "--gpus", "1", "2"]) == 0
    pred = json.loads(capsys.readouterr().out)
    assert [p["gpus"] for p in pred["prediction"]] == [1, 2]
    assert main(["run", "--config", "9"]) == 1   # unknown config number


def test_checkpointed_hybrid_run_file(cuda_ok, tmp_path):
    """`checkpoints` in a run file (`cli.py:155-162`): the hybrid loop segment by segment; the direct
    sweep, hence J, is the serial one whatever the segmentation."""
    from paper_2004_00546_b200.__main__ import main
    doc = {"problem": {"kind": "burgers", "nx": 16, "ny": 16, "D": 0.5, "omega": 2.0, "T": 0.5,
                       "f_true": "sin_product", "f_init": "ones"},
           "algorithm": "hybrid", "workers": [2, 4], "checkpoints": 1, "repeats": 1}
    out = tmp_path / "ck"
    assert main(["run", "--config", _write(tmp_path, doc), "--output", str(out), "--dt", "2.5e-3"]) == 0
    rows = list(csv.DictReader(open(out / "results.csv")))
    summary = json.load(open(out / "summary.json"))
    assert summary["checkpoints"] == 1 and [int(r["N"]) for r in rows] == [2, 4]
    assert all(abs(float(r["J"]) - summary["J_serial"]) <= 1e-11 * abs(summary["J_serial"]) for r in rows)
