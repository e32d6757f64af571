"""Run files in the reference's JSON layout (`config.py:28-175`): parsing and validation (the
GPU run is tests/test_gpu_runfile.py)."""

import numpy as np
import pytest

from paper_2004_00546_b200.errors import ConfigError
from paper_2004_00546_b200.runfile import default_dt, parse_run_file


def _doc(**over):
    d = {"problem": {"kind": "burgers", "nx": 8, "ny": 6, "D": 1.0, "omega": 1.0, "T": 1.0,
                     "f_true": "sin_product", "f_init": "ones"},
         "algorithm": "hybrid", "workers": [1, 2, 4], "rtol": 1e-3, "repeats": 2, "seed": 0, "output": "results/x"}
    d.update(over)
    return d


def test_parse_fields_and_shapes():
    rf = parse_run_file(_doc())
    assert (rf.kind, rf.nx, rf.ny, rf.algorithm, rf.workers, rf.repeats) == ("burgers", 8, 6, "hybrid", (1, 2, 4), 2)
    x = np.arange(8) * 2 * np.pi / 8
    y = np.arange(6) * 2 * np.pi / 6
    one = (np.sin(y)[:, None] * np.sin(x)[None, :]).ravel()
    assert np.allclose(rf.f_true, np.tile(one, 2)) and np.all(rf.f_init == 1.0) and rf.f_init.shape == (96,)
    lin = parse_run_file(_doc(problem={"kind": "advection_diffusion", "D": 1, "T": 10, "a": 1.0}, algorithm="linear",
                              workers=4, descent={"steps": 3, "lr": 0.25}))
    assert (lin.nx, lin.ny, lin.workers, lin.descent_steps, lin.descent_lr) == (32, 32, (4,), 3, 0.25)
    assert lin.f_true.shape == (1024,) and lin.T == 10.0
    lst = parse_run_file(_doc(problem={"kind": "advection_diffusion", "nx": 3, "ny": 3, "D": 0.5, "T": 1.0,
                                       "f_init": list(range(9))}, algorithm="linear"))
    assert np.array_equal(lst.f_init, np.arange(9.0))
    assert 0 < default_dt(rf) <= rf.T / 200


@pytest.mark.parametrize("doc, text", [
    ({"algorithm": "hybrid"}, "problem"),
    (_doc(algorithm="fast"), "algorithm"),
    (_doc(problem={"kind": "burgers", "D": -1.0, "T": 1.0}), "positive"),
    (_doc(problem={"kind": "heat", "D": 1.0, "T": 1.0}), "problem.kind"),
    (_doc(problem={"kind": "burgers", "D": 1.0, "T": 1.0}, algorithm="linear"), "linear"),
    (_doc(workers=[0]), "workers"),
    (_doc(workers=[]), "workers"),
    (_doc(repeats=0), "repeats"),
    (_doc(pilot_fraction=0.5), "pilot_fraction"),
    (_doc(problem={"kind": "burgers", "nx": 4, "ny": 4, "D": 1.0, "T": 1.0, "f_init": [1.0, 2.0]}), "expected 32 values"),
    (_doc(problem={"kind": "burgers", "nx": 2, "ny": 4, "D": 1.0, "T": 1.0}), "at least 3"),
    (_doc(problem={"kind": "burgers", "D": "one", "T": 1.0}), "problem.D"),
    (_doc(descent={"steps": -1}), "descent"),
])
def test_invalid_run_files_name_the_field(doc, text):
    with pytest.raises(ConfigError, match=text):
        parse_run_file(doc)


def test_unsupported_parts_are_refused_before_any_gpu_work():
    from paper_2004_00546_b200.runfile import run_file
    lin = _doc(algorithm="hybrid")
    lin["problem"] = dict(lin["problem"], kind="advection_diffusion")
    with pytest.raises(ConfigError, match="Burgers"):
        run_file(parse_run_file(lin))
    with pytest.raises(ConfigError, match="checkpoints"):
        run_file(parse_run_file(_doc(checkpoints=2, algorithm="nonlinear")))
