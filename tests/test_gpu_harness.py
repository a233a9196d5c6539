"""The run harness on the GPU: run / write_outputs (proj/src/report.cpp:60-195)
and the rtlr_bench driver (proj/tools/rtlr_bench.cpp) through rtlr_cu_run and
lib/rtlr_cu_bench.  Restates proj/tests/test_harness.cpp's output checks
(file shapes, determinism apart from the timing columns, unclamped negative
cell means) and checks the written numbers against the Python API on the
same problem."""
import os
import subprocess

import numpy as np
import pytest

import paper_2603_25233_b200 as P

pytestmark = pytest.mark.gpu

HEADER = ("run_id,preset,mode,seed,fr_iterations,lr_iterations,rank,compression_ratio,oversampling_ratio,"
          "phi_diff_two_norm,psi_diff_two_norm,fr_converged,lr_converged,speedup,fr_solve_seconds,"
          "lr_solve_seconds,assembly_seconds")


def strip_timing(text):  # test_harness.cpp:199-214: everything before the 14th column
    return "\n".join(",".join(l.split(",")[:13]) for l in text.splitlines())


def test_outputs_shapes_determinism_and_values(tmp_path):
    # (pin_cell: a preset name without the comma of homogeneous(s,L), which
    # the reference writes into the csv unquoted as well)
    text = "preset = pin_cell\nmesh.nx = 20\nmesh.ny = 20\nsolver.seed = 9\n"
    d1, d2 = tmp_path / "o1", tmp_path / "o2"
    s1, ok1 = P.run(config_text=text, out_dir=str(d1), log_flux=True)
    s2, ok2 = P.run(config_text=text, out_dir=str(d2), log_flux=True)
    assert ok1 and ok2 and s1.startswith("run pin_cell-seed9\n") and "compare   : speedup" in s1
    metrics = (d1 / "metrics.csv").read_text()
    lines = metrics.splitlines()
    assert lines[0] == HEADER and len(lines) == 2
    row = dict(zip(HEADER.split(","), lines[1].split(",")))
    assert row["run_id"] == "pin_cell-seed9" and row["mode"] == "both" and row["seed"] == "9"
    for name in ("history.csv", "flux_fr.txt", "flux_lr.txt", "flux_fr_log.txt", "flux_lr_log.txt"):
        assert (d1 / name).read_text() == (d2 / name).read_text(), name
    assert strip_timing(metrics) == strip_timing((d2 / "metrics.csv").read_text())

    # the numbers, against the same solves through the Python API
    g = P.Problem("pin_cell", nx=20, ny=20, seed=9)
    fr, lr = g.solve_full_rank(), g.solve_low_rank()
    assert int(row["fr_iterations"]) == fr.iterations and int(row["lr_iterations"]) == lr.iterations
    assert int(row["rank"]) == int(lr.history("rank")[-1])
    diff = np.linalg.norm(lr.phi - fr.phi)
    assert abs(float(row["phi_diff_two_norm"]) - diff) <= 1e-10 * diff
    assert float(row["psi_diff_two_norm"]) > 0.0  # psi stored (FR) and factors built (LR) by default
    n_x, n_om = g.n, g.n_omega
    r = int(row["rank"])
    assert float(row["compression_ratio"]) == pytest.approx(r * (n_x + n_om) / (n_x * n_om), rel=1e-15)
    assert len((d1 / "history.csv").read_text().splitlines()) == 1 + fr.iterations + lr.iterations
    flux = np.loadtxt(d1 / "flux_fr.txt")
    assert flux.shape == (g.nx * g.ny, 3)
    dx = dy = 2.0 / g.nx
    assert np.allclose(flux[:, 2], fr.phi[0::4] / np.sqrt(dx * dy), rtol=1e-15, atol=0)
    assert flux[0, 0] == pytest.approx(-1 + dx / 2) and flux[g.nx, 1] == pytest.approx(-1 + 3 * dy / 2)


def test_negative_cell_means_stored_unclamped(tmp_path):  # test_harness.cpp:230-262
    text = "preset = lattice\nmesh.nx = 20\nmesh.ny = 20\nquadrature.n_theta = 8\nquadrature.n_omega_z = 4\nrun.mode = full\n"
    _, ok = P.run(config_text=text, out_dir=str(tmp_path), log_flux=True)
    flux = np.loadtxt(tmp_path / "flux_fr.txt")
    flux_log = np.loadtxt(tmp_path / "flux_fr_log.txt")
    assert not (tmp_path / "flux_lr.txt").exists()
    if flux[:, 2].min() < 0.0:
        assert flux_log[:, 2].min() >= 1e-16
    assert np.array_equal(np.maximum(flux[:, 2], 1e-16), flux_log[:, 2])


def test_cli_run_and_batch(tmp_path):
    from paper_2603_25233_b200 import build as B
    cli = B.CLI
    out = tmp_path / "run"
    r = subprocess.run([cli, "run", "--preset", "homogeneous(1,1)", "--mode", "lowrank", "--seed", "3", "--p", "2",
                        "--out", str(out)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert "low-rank  : iterations" in r.stdout and f"outputs written to {out}" in r.stdout
    row = (out / "metrics.csv").read_text().splitlines()[1]
    assert row.startswith("homogeneous(1,1)-seed3,homogeneous(1,1),lowrank,3,,")
    cfg = tmp_path / "c.cfg"
    cfg.write_text("preset = homogeneous(1,1)\nsolver.p = 2\n")
    out2 = tmp_path / "batch"
    r = subprocess.run([cli, "batch", "--config", str(cfg), "--seeds", "1,2", "--out", str(out2)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert "batch: 2 low-rank runs, rank" in r.stdout
    assert len((out2 / "metrics.csv").read_text().splitlines()) == 3
    assert (out2 / "flux_lr_homogeneous(1,1)-seed1.txt").exists()
    assert (out2 / "flux_fr_homogeneous(1,1)-seed2.txt").exists()
    # a driver at its iteration cap: exit code 2
    r = subprocess.run([cli, "run", "--preset", "homogeneous(1,1)", "--mode", "full", "--max-iterations", "1",
                        "--out", str(tmp_path / "cap")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 2 and "(not converged)" in r.stdout
