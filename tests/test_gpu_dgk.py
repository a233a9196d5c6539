"""General DG degree (K = 0, 2, 3, 4) on the GPU: the sweep and the
streaming operator, which the reference runs for any K
(proj/src/sweep.cpp:10-57, operators.cpp:283-288;
proj/tests/test_sweep.cpp:142-155 sweeps quadratic elements), against the
CPU oracle (its general-K restatement of operators.cpp / sweep.cpp).
Bars: sweeps per direction rel. L2 <= 1e-12 (as the K = 1 tests); the
reference's own residual bar ||op.apply(psi) - rhs|| <= 1e-12 ||rhs||."""
import numpy as np
import pytest

import _oracle as O
import paper_2603_25233_b200 as P

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


CASES = [
    ("pin_cell", {"nx": 12, "ny": 12, "n_theta": 8, "n_omega_z": 4}),       # heterogeneous
    ("C4", {"nx": 24, "ny": 20, "n_theta": 4, "n_omega_z": 4}),             # log-normal medium, ragged
    ("homogeneous(1,1)", {"nx": 7, "ny": 5, "n_theta": 4, "n_omega_z": 2}),  # tiny, ragged
    ("C1", {"nx": 40, "ny": 40, "n_theta": 4, "n_omega_z": 2}),             # diagonals longer than a CTA
]


@pytest.mark.parametrize("degree", [0, 2, 3, 4])
@pytest.mark.parametrize("name,ov", CASES)
def test_sweep_general_degree_matches_oracle(name, ov, degree):
    o = O.Problem(name, use_dsa=0, degree=degree, **ov)
    g = P.Problem(name, use_dsa=0, degree=degree, **ov)
    assert (g.degree, g.dofs_per_cell, g.n) == (degree, (degree + 1) ** 2, o.n)
    rng = np.random.default_rng(3 + degree)
    d = g.get("dirs")
    n = g.n_omega
    rhs = rng.standard_normal((g.n, n))
    psi = g.sweep(np.arange(n), rhs)
    for j in range(n):
        ref = o.sweep(d[j, 0], d[j, 1], rhs[:, j])
        assert rel(psi[:, j], ref) <= 1e-12, (j, rel(psi[:, j], ref))
    src = g.get("source")  # shared right-hand side
    psi2 = g.sweep(np.arange(n), src)
    for j in range(0, n, max(1, n // 4)):
        assert rel(psi2[:, j], o.sweep(d[j, 0], d[j, 1], src)) <= 1e-12


@pytest.mark.parametrize("degree", [0, 2, 3])
def test_apply_general_degree_matches_oracle(degree):
    ov = {"nx": 9, "ny": 11, "n_theta": 4, "n_omega_z": 2}
    o = O.Problem("pin_cell", use_dsa=0, degree=degree, **ov)
    g = P.Problem("pin_cell", use_dsa=0, degree=degree, **ov)
    v = np.random.default_rng(9).standard_normal(g.n)
    for ox, oy in ((0.6, 0.8), (-0.6, 0.8), (0.6, -0.8), (-0.28, -0.96), (1.0, 0.0), (0.0, -1.0)):
        assert rel(g.apply(ox, oy, v), o.apply(ox, oy, v)) <= 1e-14


def test_quadratic_elements_sweep_exactly():  # test_sweep.cpp:142-155
    fields = {"sigma_s": lambda x, y: 2.0 + x + 0.5 * y, "sigma_a": lambda x, y: 0.1}
    g = P.Problem("homogeneous(1,1)", nx=4, ny=4, n_theta=4, n_omega_z=2, degree=2, use_dsa=0, fields=fields)
    assert g.degree == 2
    rng = np.random.default_rng(29)
    rhs = rng.standard_normal((g.n, g.n_omega))
    psi = g.sweep(np.arange(g.n_omega), rhs)
    d = g.get("dirs")
    for j in range(g.n_omega):
        r = g.apply(d[j, 0], d[j, 1], psi[:, j]) - rhs[:, j]
        assert np.linalg.norm(r) <= 1e-12 * np.linalg.norm(rhs[:, j])


@pytest.mark.parametrize("degree", [0, 2])
def test_uniform_inflow_streams_through_general_degree(degree):  # test_sweep.cpp:126-140 at K != 1
    fields = {"sigma_s": lambda x, y: 0.0, "sigma_a": lambda x, y: 0.0, "source": lambda x, y: 0.0,
              "boundary": lambda x, y: 1.0}
    g = P.Problem("homogeneous(1,1)", nx=5, ny=5, x_min=0, x_max=1, y_min=0, y_max=1, degree=degree,
                  use_dsa=0, fields=fields)
    dirs = np.array([[1.0, 0.0], [0.0, -1.0], [np.sqrt(0.5), np.sqrt(0.5)], [-0.6, 0.8]])
    s = g.dofs_per_cell
    o = O.Problem("homogeneous(1,1)", nx=5, ny=5, x_min=0, x_max=1, y_min=0, y_max=1, degree=degree,
                  use_dsa=0, fields=fields)
    for ox, oy in dirs:
        rhs = o.boundary_vector(ox, oy)
        psi = g.sweep_dirs(np.array([[ox, oy]]), rhs[:, None])[:, 0]
        mean = psi[::s] / np.sqrt(0.2 * 0.2)  # DGSpace::cell_mean (dg_space.cpp:39-42)
        assert np.allclose(mean, 1.0, rtol=0, atol=1e-12)


def test_degree_one_through_general_kernel_matches_hot_path():
    """sweep_kernel = 6 runs K = 1 through the general-degree kernel: the same
    sweeps as the K = 1 kernels to rounding."""
    g = P.Problem("pin_cell", nx=16, ny=12, n_theta=4, n_omega_z=4, use_dsa=0)
    rng = np.random.default_rng(2)
    rhs = rng.standard_normal((g.n, g.n_omega))
    a = g.sweep(np.arange(g.n_omega), rhs)
    g.set_option("sweep_kernel", 6)
    b = g.sweep(np.arange(g.n_omega), rhs)
    for j in range(g.n_omega):
        assert rel(b[:, j], a[:, j]) <= 1e-13


def test_general_degree_inflow_matches_oracle():
    ov = {"nx": 10, "ny": 8, "n_theta": 4, "n_omega_z": 2, "boundary_const": 0.75}
    o = O.Problem("homogeneous(1,1)", use_dsa=0, degree=2, **ov)
    g = P.Problem("homogeneous(1,1)", use_dsa=0, degree=2, **ov)
    d = g.get("dirs")
    rhs = np.random.default_rng(4).standard_normal((g.n, g.n_omega))
    psi = g.sweep(np.arange(g.n_omega), rhs)
    for j in range(g.n_omega):
        ref = o.sweep(d[j, 0], d[j, 1], rhs[:, j] + o.boundary_vector(d[j, 0], d[j, 1]))
        assert rel(psi[:, j], ref) <= 1e-12


def test_general_degree_singular_block_raises():  # sweep.cpp:49-52
    g = P.Problem("homogeneous(0,1)", nx=4, ny=4, sigma_a_const=0.0, use_dsa=0, degree=2)
    with pytest.raises(P.RtlrError, match="singular local block"):
        g.sweep_dirs(np.array([[0.0, 0.0]]), np.ones(g.n))


def test_general_degree_solvers_rejected():
    g = P.Problem("homogeneous(1,1)", nx=4, ny=4, n_theta=4, n_omega_z=2, degree=2, use_dsa=0)
    with pytest.raises(P.InvalidArgument, match="degree"):
        g.solve_full_rank()
    with pytest.raises(P.InvalidArgument, match="degree"):
        g.solve_low_rank()
    with pytest.raises(P.InvalidArgument, match="degree"):
        g.rhs_core(np.zeros(g.n))
