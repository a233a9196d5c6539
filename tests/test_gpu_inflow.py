"""Solver-level parity with inflow boundary data against the
CPU oracle on identical inputs.

The reference feeds an inflow datum g through build_boundary_data
(proj/src/full_rank.cpp:11-39): every sweep's right-hand side gains the
angle's boundary vector g_j (full rank: full_rank.cpp:86,94; low rank: the
sampled sweeps and residuals, low_rank.cpp:206,213,302) and every Galerkin
system's right-hand side gains X^T g_j (reduced_rhs, low_rank.cpp:185-190).
Here whole FR and LR SI-DSA solves run with (a) a constant inflow
(boundary_const, a reference config key) and (b) a space-varying inflow given
as a ScalarField callback (rtlr_cu_config_set_field; the oracle takes the
same callable).  Bars (north star): scalar flux rel. L2 <= 1e-10 (FR) and
<= 1e-8 (LR), outer iterations +-1, low-rank ranks reported side by side.
"""
import math

import numpy as np
import pytest

import _oracle as O
import paper_2603_25233_b200 as P

pytestmark = pytest.mark.gpu


def g_varying(x, y):
    # smooth, positive, different on every edge of [-1,1]^2
    return 1.0 + 0.5 * math.sin(1.3 * x + 0.4) * math.cos(0.7 * y - 0.2) + 0.25 * x * y


CASES = [
    # thick medium: the rank adapts (oracle ranks 62 -> 48 of 64)
    ("homogeneous(100,1)", {"n_theta": 16, "n_omega_z": 8, "boundary_const": 1.0}, None),
    # heterogeneous, full rank
    ("pin_cell", {"nx": 24, "ny": 24, "n_theta": 16, "n_omega_z": 8, "boundary_const": 0.5}, None),
    ("variable_scattering", {"nx": 20, "ny": 20, "n_theta": 16, "n_omega_z": 8}, {"boundary": g_varying}),
    # diffusive C2 medium and source on a 32^2 mesh with a varying inflow
    ("C2", {"nx": 32, "ny": 32, "n_theta": 16, "n_omega_z": 8}, {"boundary": g_varying}),
    # thick medium, varying inflow (oracle ranks 83 -> 54 of 96)
    ("homogeneous(100,1)", {"n_theta": 24, "n_omega_z": 8}, {"boundary": g_varying}),
]
IDS = ["thick-const", "pincell-const", "varscat-callback", "C2-callback", "thick-callback"]


def _pair(name, ov, fields):
    o = O.Problem(name, fields=fields, **ov)
    g = P.Problem(name, fields=fields, **ov)
    return o, g


@pytest.mark.parametrize("name,ov,fields", CASES, ids=IDS)
def test_full_rank_with_inflow(name, ov, fields):
    o, g = _pair(name, ov, fields)
    ro = o.solve("full")
    rg = g.solve_full_rank(store_psi=0)
    ref = ro.get("phi", o.n)
    err = np.linalg.norm(rg.phi - ref) / np.linalg.norm(ref)
    print(f"{name} FR inflow: it {rg.iterations}/{ro.iterations} rel {err:.2e}")
    assert rg.converged and ro.converged
    assert abs(rg.iterations - ro.iterations) <= 1
    assert err <= 1e-10


@pytest.mark.parametrize("name,ov,fields", CASES, ids=IDS)
def test_low_rank_with_inflow(name, ov, fields):
    o, g = _pair(name, ov, fields)
    ro = o.solve("lowrank")
    rg = g.solve_low_rank()
    ref = ro.get("phi", o.n)
    err = np.linalg.norm(rg.phi - ref) / np.linalg.norm(ref)
    ranks_g = [int(v) for v in rg.history("rank")]
    ranks_o = [int(v) for v in ro.history("rank")]
    print(f"{name} LR inflow: it {rg.iterations}/{ro.iterations} rel {err:.2e} ranks GPU {ranks_g} oracle {ranks_o}")
    assert rg.converged and ro.converged
    assert abs(rg.iterations - ro.iterations) <= 1
    assert err <= 1e-8
    assert abs(ranks_g[-1] - ranks_o[-1]) <= 2


def test_inflow_si_step_and_boundary_data():
    """One si_step with a callback inflow: the swept angular fluxes carry
    g_j (full_rank.cpp:86) — compared angle by angle, and a nonzero datum
    must change them (the path is live)."""
    name, ov = "pin_cell", {"nx": 16, "ny": 16, "n_theta": 4, "n_omega_z": 2}
    o, g = _pair(name, ov, {"boundary": g_varying})
    phi0 = np.linspace(0.0, 1.0, o.n)
    so, psio = o.si_step(phi0, want_psi=True)
    sg, psig = g.si_step(phi0, want_psi=True)
    assert np.linalg.norm(sg - so) / np.linalg.norm(so) <= 1e-12
    for j in range(o.n_omega):
        assert np.linalg.norm(psig[:, j] - psio[:, j]) / np.linalg.norm(psio[:, j]) <= 1e-12
    vac = P.Problem(name, **ov)
    sv = vac.si_step(phi0)
    assert np.linalg.norm(sv - sg) > 1e-3 * np.linalg.norm(sg)
