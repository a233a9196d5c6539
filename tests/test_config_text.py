"""The reference's config text format (proj/src/problem.cpp:288-459) through
rtlr_cu_config_parse, on the host (device = -1: assembly only, no GPU).
Parity is bitwise on the assembled inputs: a config file describing a preset
assembles exactly what the preset does; field keys modify a preset's
FieldSpecs as in the reference; errors carry the reference's messages."""
import os
import subprocess

import numpy as np
import pytest

import paper_2603_25233_b200 as P

INPUTS = ("dirs", "weights", "source", "sigma_t_blocks", "sigma_s_blocks", "sigma_a_blocks", "sip_bsr")


def same_inputs(a, b):
    return all(np.array_equal(a.get(w), b.get(w)) for w in INPUTS)


@pytest.mark.parametrize("preset", ["homogeneous(1,1)", "variable_scattering", "pin_cell", "lattice", "C1"])
def test_preset_line_assembles_the_preset(preset):
    text = f"# a comment line\npreset = {preset}   # trailing comment\n\n"
    assert same_inputs(P.Problem(config_text=text, device=-1), P.Problem(preset, device=-1))


def test_full_description_without_preset():
    """Every key written out (serialize_config's layout, problem.cpp:288-321)
    reproduces homogeneous(1,1) bit for bit."""
    text = """
domain.x_min = -1
domain.x_max = 1
domain.y_min = -1
domain.y_max = 1
mesh.nx = 16
mesh.ny = 16
quadrature.n_theta = 8
quadrature.n_omega_z = 4
space.degree = 1
sigma_s.kind = constant
sigma_s.value = 1
sigma_a.kind = constant
sigma_a.value = 0
source.kind = gaussian
source.value = 1
source.decay = 100
source.center_x = 0
source.center_y = 0
boundary.kind = constant
boundary.value = 0
solver.eps_si_sa = 9.9999999999999995e-07
solver.p = 2
solver.q = 8
run.mode = both
"""
    assert same_inputs(P.Problem(config_text=text, device=-1), P.Problem("homogeneous(1,1)", device=-1))


def test_field_keys_modify_the_preset_fields():
    # homogeneous(3,1) differs from homogeneous(1,1) only in the constant sigma_s
    a = P.Problem(config_text="preset = homogeneous(1,1)\nsigma_s.value = 3\n", device=-1)
    assert same_inputs(a, P.Problem("homogeneous(3,1)", device=-1))
    # pin_cell's box: the inside value changes, the box and the outside stay
    b = P.Problem(config_text="preset = pin_cell\nsigma_s.value = 0.2\n", device=-1)
    ref = P.Problem("pin_cell", device=-1)
    sb, sr = b.get("sigma_s_blocks"), ref.get("sigma_s_blocks")
    inside = sr[:, 0, 0] < 1.0
    assert np.allclose(sb[inside, 0, 0], 2 * sr[inside, 0, 0], rtol=1e-12)
    assert np.array_equal(sb[~inside], sr[~inside])
    # a later preset line resets the fields (last preset wins)
    c = P.Problem(config_text="preset = pin_cell\nsigma_s.value = 0.2\npreset = pin_cell\n", device=-1)
    assert same_inputs(c, ref)


def test_overrides_after_the_preset():
    a = P.Problem(config_text="preset = pin_cell\nmesh.nx = 20\nmesh.ny = 12\nquadrature.n_theta = 4\n", device=-1)
    assert same_inputs(a, P.Problem("pin_cell", device=-1, nx=20, ny=12, n_theta=4))


@pytest.mark.parametrize("text,msg", [
    ("mesh.nz = 4", "config: unknown key 'mesh.nz'"),
    ("mesh.nx = 4.5", "config: bad integer '4.5' for mesh.nx"),
    ("domain.x_max = one", "config: bad number 'one' for domain.x_max"),
    ("mesh.nx 4", "config line 1: expected key = value"),
    ("\n\npreset = nowhere", "unknown preset 'nowhere'"),
    ("sigma_s.kind = spiral", "unknown field kind 'spiral'"),
    ("solver.p = 9", "config: need 1 <= p <= q"),
    ("run.mode = sideways", "unknown run mode 'sideways'"),
    ("domain.x_max = -2", "config: empty domain"),
    ("preset = C3\nsigma_s.value = 2", "take no field keys"),
])
def test_config_errors(text, msg):
    with pytest.raises(P.ConfigError) as e:
        P.Problem(config_text=text, device=-1)
    assert msg in str(e.value)


def test_cli_reports_config_errors(tmp_path):
    """rtlr_cu_bench (the rtlr_bench driver): exit code 3 on config errors,
    the preset catalogue without a GPU."""
    from paper_2603_25233_b200 import build as B
    cli = B.CLI
    if not os.path.exists(cli):
        B.build()
    cfg = tmp_path / "bad.cfg"
    cfg.write_text("preset = pin_cell\nsolver.q = 0\n")
    r = subprocess.run([cli, "run", "--config", str(cfg)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 3 and "config error: config: need 1 <= p <= q" in r.stderr
    r = subprocess.run([cli, "run"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 3
    r = subprocess.run([cli, "presets"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "pin_cell" in r.stdout and "C4" in r.stdout


def test_degree_key_assembles_a_general_degree_problem():
    """`space.degree = 2` in a config file (the reference's DG degree key,
    problem.cpp) assembles the quadratic-element problem the keyword
    override does (host_dgk.cpp)."""
    text = "preset = pin_cell\nmesh.nx = 6\nmesh.ny = 5\nspace.degree = 2\n"
    a = P.Problem(config_text=text, device=-1)
    b = P.Problem("pin_cell", device=-1, nx=6, ny=5, degree=2)
    assert (a.degree, a.dofs_per_cell, a.n) == (2, 9, 9 * 30)
    for w in ("dirs", "weights", "source", "sigma_t_blocks", "sigma_s_blocks", "sigma_a_blocks", "stream_blocks"):
        assert np.array_equal(a.get(w), b.get(w)), w
