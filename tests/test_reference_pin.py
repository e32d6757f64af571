"""Pin the oracle to the reference: restated numerics vs golden vectors that
`oracle/gen_golden.py` produced by running the reference (`paradjoint`) itself.

These tie the config-mode oracle (which checks the GPU) to the reference:
the stencil and Burgers operators are the same functions, and the Paraexp
neighbour-chain structure (`chains_direct`/`chains_adjoint`, reused by the
config-mode "chains" formulation) reproduces `solve_direct_linear` /
`solve_adjoint_linear` piece by piece.
"""

import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import config_mode as C
from oracle import reference_mode as R
from paper_2004_00546_b200.problems import Grid, advdiff_stencil
from tests.conftest import ROOT, rel_l2

GOLD = os.path.join(ROOT, "tests", "golden")


def load(name):
    return np.load(os.path.join(GOLD, f"reference_{name}.npz"))


def csr_of(st, nx, ny):
    """CSR of the matrix-free stencil (columns of the identity)."""
    n = nx * ny
    cols = [C.stencil_apply(st, e, nx, ny) for e in np.eye(n)]
    m = sp.csr_matrix(np.stack(cols, axis=1))
    m.sort_indices()
    return m


def test_stencil_operator_2d_and_transpose():
    f = load("stencil")
    nx, ny = int(f["nx2"]), int(f["ny2"])
    st = advdiff_stencil(Grid(nx, ny), (float(f["a2"]), float(f["a2"])), float(f["D2"]))
    assert np.max(np.abs(C.stencil_apply(st.as_tuple(), f["x2"], nx, ny) - f["Ax2"])) <= 1e-12
    assert np.max(np.abs(C.stencil_apply(st.transpose().as_tuple(), f["x2"], nx, ny) - f["ATx2"])) <= 1e-12


def test_stencil_operator_1d_embedding():
    f = load("stencil")
    nx = int(f["nx1"])
    st = advdiff_stencil(Grid(nx), (float(f["a1"]), 0.0), float(f["D1"]))
    assert np.max(np.abs(C.stencil_apply(st.as_tuple(), f["x1"], nx, 1) - f["Ax1"])) <= 1e-11
    assert np.max(np.abs(C.stencil_apply(st.transpose().as_tuple(), f["x1"], nx, 1) - f["ATx1"])) <= 1e-11


def test_burgers_rhs_and_adjoint_match_reference():
    f = load("burgers")
    nx, D = int(f["nx"]), float(f["D"])
    h = 2 * np.pi / nx
    assert np.max(np.abs(C.burgers_rhs(f["U"], f["f"], D, h) - f["rhs"])) <= 1e-12
    assert np.max(np.abs(f["rhs_V"])) == 0.0  # V stays identically zero
    assert np.max(np.abs(C.burgers_adjoint_apply(f["U"], f["y"], D, h) - f["adj"])) <= 1e-12
    assert np.max(np.abs(f["adj_b"])) <= 1e-14


def test_frozen_operator_is_jacobian_transpose_at_trapezoid_mean():
    """`average_jacobian` then transpose == J(ū)ᵀ with ū the trapezoid mean (the
    GPU's frozen-slice operator)."""
    f = load("burgers")
    nx, D = int(f["nx"]), float(f["D"])
    ub = R.trapezoid_mean(f["tnodes"], f["tstates"])
    got = C.burgers_adjoint_apply(ub, f["y"], D, 2 * np.pi / nx)
    assert np.max(np.abs(got - f["frozenT_y"])) <= 1e-12


def test_linear_interpolation_midpoints_are_means():
    f = load("burgers")
    got = R.linear_interp(f["tnodes"], f["tstates"], f["mids"])
    assert np.max(np.abs(got - f["interp"])) <= 1e-14
    mean = 0.5 * f["tstates"][:-1] + 0.5 * f["tstates"][1:]
    assert np.max(np.abs(mean - f["interp"])) <= 1e-14


def _A(nx, ny, a, D):
    st = advdiff_stencil(Grid(nx, ny), (a, a), D)
    return csr_of(st.as_tuple(), nx, ny)


def test_dopri5_nodes_and_states():
    f = load("dopri5")
    A = _A(4, 4, 1.0, 0.5)
    nodes, states = R.dopri5(lambda t, y: A @ y + f["f"] * np.sin(1.3 * t), f["y0"], 0.0, 0.7,
                             R.DP5Settings(rtol=float(f["rtol"])), f["wps"])
    assert nodes.shape == f["nodes"].shape  # same accepted-step sequence
    assert np.max(np.abs(nodes - f["nodes"])) <= 1e-15
    assert rel_l2(states, f["states"]) <= 1e-13


def test_leja_points_interval_and_propagation():
    f = load("leja")
    assert np.array_equal(R.leja_points(12), f["leja12"])
    A = _A(6, 6, 1.0, 1.0)
    iv = R.gershgorin_interval(A)
    assert abs(iv[0] - f["interval"][0]) <= 1e-12 and abs(iv[1] - f["interval"][1]) <= 1e-12
    end, rec = R.leja_propagate(A, f["v"], float(f["dt"]), R.LejaSettings(tol=float(f["tol"])), record=3)
    assert rel_l2(end, f["end"]) <= 1e-12
    assert rel_l2(rec, f["rec"]) <= 1e-12


@pytest.mark.parametrize("N", [1, 2, 3])
def test_paraexp_direct_and_adjoint_pieces(N):
    f = load("paraexp")
    A = _A(6, 6, 1.0, 1.0)
    T = float(f["T"])
    b = T * np.arange(N + 1) / N
    dp = R.DP5Settings(rtol=float(f["rtol"]))
    lj = R.LejaSettings(tol=float(f["tol"]))
    d = R.reference_direct_linear(A, f["q0"], lambda t: f["f0"] * np.sin(1.3 * t), b, dp, lj)
    a = R.reference_adjoint_linear(A, f["qT"], lambda t: f["s0"] * np.cos(2.0 * t), b, dp, lj)
    for p in range(N):
        nodes, states = d[p]
        assert nodes.shape == f[f"d{N}_{p}_nodes"].shape
        assert np.max(np.abs(nodes - f[f"d{N}_{p}_nodes"])) <= 1e-14
        assert rel_l2(states, f[f"d{N}_{p}_states"]) <= 1e-12
        nodes, states = a[p]
        assert nodes.shape == f[f"a{N}_{p}_nodes"].shape
        assert np.max(np.abs(nodes - f[f"a{N}_{p}_nodes"])) <= 1e-14
        assert rel_l2(states, f[f"a{N}_{p}_states"]) <= 1e-12


def test_config_mode_chains_use_the_pinned_structure():
    """The config-mode 'chains' formulation runs reference_mode.chains_direct /
    chains_adjoint with RK4 + Chebyshev (and tests/test_oracle.py shows it equals
    the summed-chain scan that the GPU executes)."""
    import inspect
    src = inspect.getsource(C.linear_gradient)
    assert "chains_direct" in src and "chains_adjoint" in src


def test_hybrid_frozen_span_matches_solve_hybrid():
    """The frozen-span adjoint (the product's `solve_hybrid(..., adjoint="frozen_span")`,
    config-mode oracle `burgers_gradient(..., adjoint="frozen_span")`) has the structure of
    the reference's `solve_hybrid` with a final condition and no adjoint source
    (`hybrid.py:194-237`): zero inhomogeneous solves, q†_T carried back slice by slice through
    exp((T_{m+1} − T_m)·J(ū_m)ᵀ) (`propagate_span`). Restated here with exact dense
    exponentials of the oracle's Jᵀ at the reference's own slice means ū_m."""
    from scipy.linalg import expm
    f = load("hybrid")
    nx, D = int(f["nx"]), float(f["D"])
    h = 2.0 * np.pi / nx
    bnd, ubar = f["boundaries"], f["ubar"]
    assert float(f["vmax"]) <= 1e-15  # the V component stays zero (y-invariant, V ≡ 0)
    q = f["qT"].copy()
    N = len(bnd) - 1
    for m in range(N - 1, -1, -1):
        JT = np.stack([C.burgers_adjoint_apply(ubar[m], e, D, h) for e in np.eye(nx)], axis=1)
        assert rel_l2(f["qend"][m], q) <= 1e-13     # q† entering slice m from above
        q = expm((bnd[m + 1] - bnd[m]) * JT) @ q
        assert rel_l2(f["qstart"][m], q) <= 1e-13   # q†(T_m)
