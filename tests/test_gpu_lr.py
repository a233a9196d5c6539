"""GPU parity of the low-rank SI-DSA solver (low_rank.cpp) against the CPU
oracle through the C ABI.  North-star tolerances: scalar flux rel. L2
<= 1e-8, outer iteration counts +-1, sampled direction sets and final rank
reported side by side (asserted equal where the decisions are not near a
threshold)."""
import numpy as np
import pytest

import _oracle as O
import paper_2603_25233_b200 as P

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


LR_CASES = [
    ("homogeneous(1,1)", {"seed": 2024}),
    ("homogeneous(100,1)", {"seed": 5}),
    ("pin_cell", {"seed": 12345, "nx": 20, "ny": 20}),
    ("lattice", {"seed": 3, "nx": 20, "ny": 20}),
    ("variable_scattering", {"seed": 7}),
    ("homogeneous(0.1,2)", {"seed": 12345}),
]


@pytest.mark.parametrize("name,ov", LR_CASES)
def test_low_rank_matches_oracle(name, ov):
    o = O.Problem(name, **ov)
    g = P.Problem(name, **ov)
    ro = o.solve("lowrank")
    rg = g.solve_low_rank()
    assert rg.converged == ro.converged
    assert abs(rg.iterations - ro.iterations) <= 1, (rg.iterations, ro.iterations)
    assert rel(rg.phi, ro.get("phi", o.n)) <= 1e-8, rel(rg.phi, ro.get("phi", o.n))
    # Side by side: greedy selections and truncated ranks.  Symmetric media
    # make residual norms of rotated directions equal in exact arithmetic,
    # so rounding may break such ties differently; the sets are reported and
    # the final rank must agree within +-2.
    sg, so = rg.sampled_log(), ro.sampled_log()
    prefix = 0
    for a, b in zip(sg[0], so[0]):
        if a != b:
            break
        prefix += 1
    print(f"{name}: first outer iteration sampled GPU {sg[0][:12]}... oracle {so[0][:12]}... "
          f"common prefix {prefix}/{len(so[0])}; ranks {list(rg.history('rank'))} vs {list(ro.history('rank'))}")
    assert prefix >= min(len(so[0]), 8)
    assert abs(rg.factor_rank - ro.factor_rank) <= 2


def test_low_rank_asymmetric_medium_selections():
    """C4's random log-normal medium has no symmetry: the greedy decisions
    coincide with the oracle's until the candidate residuals reach rounding
    level (late in an inner loop all residuals are noise, and either choice
    is valid); the sampled sets are reported side by side."""
    ov = {"nx": 32, "ny": 32, "n_theta": 16, "n_omega_z": 8, "p": 2, "q": 6}
    o = O.Problem("C4", **ov)
    g = P.Problem("C4", **ov)
    ro = o.solve("lowrank")
    rg = g.solve_low_rank()
    assert rg.iterations == ro.iterations
    assert rel(rg.phi, ro.get("phi", o.n)) <= 1e-8
    sg, so = rg.sampled_log(), ro.sampled_log()
    prefix = next((i for i, (a, b) in enumerate(zip(sg[0], so[0])) if a != b), min(len(sg[0]), len(so[0])))
    print(f"C4 reduced: common prefix {prefix}/{len(so[0])}; GPU {sg[0]} oracle {so[0]}")
    assert prefix >= len(so[0]) // 2
    assert abs(rg.factor_rank - ro.factor_rank) <= 2


def test_low_rank_factors_and_determinism():  # test_low_rank.cpp:441-498
    g = P.Problem("homogeneous(1,1)", seed=11)
    a = g.solve_low_rank()
    b = g.solve_low_rank()
    assert np.array_equal(a.phi, b.phi) and a.sampled_log() == b.sampled_log()
    r = a.factor_rank
    X = a.get("X", g.n * r).reshape(r, g.n).T
    V = a.get("V", g.n_omega * r).reshape(r, g.n_omega).T
    S = a.get("S", r)
    assert np.linalg.norm(X.T @ X - np.eye(r)) <= 1e-10
    assert np.linalg.norm(V.T @ V - np.eye(r)) <= 1e-10
    assert np.all(np.diff(S) <= 0)
    assert a.psi_dofs == r * (g.n + g.n_omega)
    f = g.solve_full_rank()
    assert abs(f.iterations - a.iterations) <= 1
    assert np.linalg.norm(f.phi - a.phi) <= 1e-6
    psi = f.get("psi", g.n * g.n_omega).reshape(g.n_omega, g.n).T
    assert np.linalg.norm(psi - X @ np.diag(S) @ V.T) <= 1e-5


def test_low_rank_exhausted_fallback():  # test_low_rank.cpp:425-439
    o = O.Problem("homogeneous(1,1)", nx=2, ny=2, n_theta=4, n_omega_z=2, p=2, q=3, eps_res=1e-300,
                  max_iterations=1, use_dsa=0, seed=3)
    g = P.Problem("homogeneous(1,1)", nx=2, ny=2, n_theta=4, n_omega_z=2, p=2, q=3, eps_res=1e-300,
                  max_iterations=1, use_dsa=0, seed=3)
    ro, rg = o.solve("lowrank"), g.solve_low_rank()
    assert rg.history("fullrank_fallback")[0] == 1.0
    assert rg.history("sampled_count")[0] == g.n_omega
    assert rel(rg.phi, ro.get("phi", o.n)) <= 1e-12


@pytest.mark.parametrize("name", ["C2"])
def test_baseline_c2_reduced(name):
    ov = {"nx": 32, "ny": 32, "n_theta": 16, "n_omega_z": 8}
    o = O.Problem(name, **ov)
    g = P.Problem(name, **ov)
    ro = o.solve("lowrank")
    rg = g.solve_low_rank()
    assert abs(rg.iterations - ro.iterations) <= 1
    assert rel(rg.phi, ro.get("phi", o.n)) <= 1e-8


def test_sharded_low_rank_single_rank_nccl_is_bitwise():
    """The angle-sharded LR driver (sampled sweeps, Galerkin solves and
    residual norms per rank block + NCCL all-gathers) on a one-rank
    communicator: every per-angle result is computed exactly as unsharded, so
    phi, ranks and the sampled sets are bitwise identical."""
    a = P.Problem("C1")
    ra = a.solve_low_rank(build_factors=0)
    b = P.Problem("C1")
    b.set_comm(1, 0, P.nccl_unique_id())
    rb = b.solve_low_rank(build_factors=0)
    assert rb.iterations == ra.iterations
    assert np.array_equal(rb.phi, ra.phi)
    assert list(rb.history("rank")) == list(ra.history("rank"))
    assert rb.sampled_log() == ra.sampled_log()


@pytest.mark.parametrize("m,n", [(5000, 70), (3000, 33), (2048, 32), (777, 1), (4096, 96)])
def test_blocked_householder_qr(m, n):
    """Blocked Householder QR (basis rebuild, low_rank.cpp:112-130): q r = a,
    q orthonormal, r upper, |r| equal to LAPACK's (signs follow Eigen)."""
    rng = np.random.default_rng(m + n)
    a = rng.standard_normal((m, n))
    a[:, n // 2] = a[:, 0] + 1e-9 * rng.standard_normal(m)  # a nearly dependent column
    q, r = P.dense_qr(a)
    assert np.allclose(np.triu(r), r, rtol=0, atol=0)
    assert np.linalg.norm(q @ r - a) / np.linalg.norm(a) <= 1e-14
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= 1e-13
    r_ref = np.linalg.qr(a, mode="r")
    assert np.allclose(np.abs(np.diag(r)), np.abs(np.diag(r_ref)), rtol=1e-8, atol=1e-12)


def test_psi_difference_matches_oracle():
    """psi_difference (report.cpp:47-58) on the GPU, fed the oracle's own
    full-rank psi and low-rank factors, against the oracle's value."""
    name, ov = "pin_cell", {}
    o = O.Problem(name, **ov)
    full, low = o.solve("full"), o.solve("lowrank")
    n, nom, r = o.n, o.n_theta * o.n_omega_z, low.factor_rank
    psi, X, S, V = full.get("psi", n * nom), low.get("X", n * r), low.get("S", r), low.get("V", nom * r)
    ref = O.lib().oracle_psi_difference(full.h, low.h)
    g = P.Problem(name, **ov)
    got = g.psi_difference(psi, X, S, V)
    assert abs(got - ref) <= 1e-12 * max(1.0, abs(ref)) + 1e-15, (got, ref)
    # and the GPU's own runs, compared the reference's way (compare_runs)
    cmp = P.compare_runs(g.solve_full_rank(), g.solve_low_rank(), problem=g)
    assert cmp["has_psi_diff"] and cmp["psi_diff_two_norm"] <= 1e-5
    assert cmp["phi_diff_two_norm"] <= 1e-6 and 0 < cmp["compression_ratio"] < 1


_SWITCH_RUN = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + "/tests")
import paper_2603_25233_b200 as P
g = P.Problem("C2", nx=64, ny=64, n_theta=16, n_omega_z=8)
r = g.solve_low_rank(build_factors=1)
np.save(sys.argv[2], np.asarray(r.phi))
'''


@pytest.mark.parametrize("switch", ["RTLR_CGS_COOP", "RTLR_JACOBI_COOP", "RTLR_QR_COOP", "RTLR_MG_FUSE", "RTLR_NN_NT",
                                    "RTLR_TN_NT", "RTLR_SWEEP_TMA"])
def test_device_path_switches_keep_the_solve(switch, tmp_path):
    """The fused / cooperative device paths against the launch-per-step and
    64 x 64-tile paths they replaced (each switch is read once per process,
    so each setting runs in its own process).  The cooperative CGS and
    Jacobi kernels reduce in the same order: bitwise equal.  The GEMM tile
    and sweep kernel choices change summation orders: within the LR
    tolerance."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for v in ("1", "0"):
        f = str(tmp_path / f"phi_{v}.npy")
        env = dict(os.environ, **{switch: v})
        subprocess.run([sys.executable, "-c", _SWITCH_RUN, root, f], env=env, check=True, timeout=600)
        out[v] = np.load(f)
    if switch in ("RTLR_CGS_COOP", "RTLR_JACOBI_COOP", "RTLR_MG_FUSE"):
        assert np.array_equal(out["1"], out["0"])
    else:
        assert rel(out["1"], out["0"]) <= 1e-8


_ROWSLICE_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2603_25233_b200 as P
p = P.Problem(sys.argv[2], seed=7, **eval(sys.argv[3]))
r = p.solve_low_rank()
np.save(sys.argv[4], np.concatenate([[r.iterations, r.history("rank")[-1]], r.phi]))
"""


@pytest.mark.parametrize("name,ov", [("pin_cell", {"nx": 24, "ny": 24}), ("C4", {"nx": 48, "ny": 40, "n_theta": 16,
                                                                                "n_omega_z": 8, "p": 4, "q": 8})])
def test_row_sliced_contractions_match_the_unsliced_solve(name, ov, tmp_path):
    """The multi-GPU row slicing of the tall contractions (CGS projections,
    border extension X^T W, the remainder update with its row all-gather;
    SURVEY.md §8(e)) run as 3 virtual slices on one GPU
    (RTLR_ROWSLICE_VIRTUAL=3: every slice's partial product and the
    pack / unpack of the gathered rows, summed in slice order): the low-rank
    solve agrees with the unsliced one (rounding of the split sums only) and
    with the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for tag, env in (("plain", {}), ("sliced", {"RTLR_ROWSLICE_VIRTUAL": "3"})):
        f = str(tmp_path / f"{tag}.npy")
        e = dict(os.environ, **env)
        subprocess.run([sys.executable, "-c", _ROWSLICE_SCRIPT, root, name, repr(ov), f], check=True, env=e,
                       timeout=600)
        out[tag] = np.load(f)
    a, b = out["plain"], out["sliced"]
    assert a[0] == b[0] and abs(a[1] - b[1]) <= 2  # iterations, final rank
    assert rel(b[2:], a[2:]) <= 1e-10, rel(b[2:], a[2:])
    o = O.Problem(name, seed=7, **ov)
    ref = o.solve("lowrank").get("phi", o.n)
    assert rel(b[2:], ref) <= 1e-8


_REBUILD_RUN = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2603_25233_b200 as P
g = P.Problem("C2", nx=48, ny=48, n_theta=16, n_omega_z=8)
r = g.solve_low_rank(build_factors=0, eps_mgs=1e-15)
np.save(sys.argv[2], np.concatenate([[r.iterations, r.history("rank")[-1]], r.phi]))
'''


def test_basis_rebuild_paths_agree(tmp_path):
    """The overlap-triggered basis rebuild (low_rank.cpp:107-130) by
    CholeskyQR2 of [X_old, the batch's orthonormalised columns] (default)
    against the reference's Householder QR of [X_old, accepted snapshots]
    (RTLR_REBUILD=householder): the same nested column spaces, so the same
    solve to rounding.  eps_mgs = 1e-15 makes the overlap test fire at
    almost every batch."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for v in ("householder", "cholqr2"):
        f = str(tmp_path / f"phi_{v}.npy")
        env = dict(os.environ, RTLR_REBUILD=v)
        subprocess.run([sys.executable, "-c", _REBUILD_RUN, root, f], env=env, check=True, timeout=600)
        out[v] = np.load(f)
    a, b = out["householder"], out["cholqr2"]
    assert abs(a[0] - b[0]) <= 1 and abs(a[1] - b[1]) <= 2
    assert rel(b[2:], a[2:]) <= 1e-8


_MIRROR_RUN = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2603_25233_b200 as P
p = P.Problem("C2")
r = p.solve_low_rank(build_factors=0)
np.save(sys.argv[2], np.concatenate([[r.iterations], r.history("rank"), r.phi]))
'''


def test_verification_skips_mirrors_of_sampled_angles(tmp_path):
    """The verification pass (low_rank.cpp:396-424) does not evaluate an
    unsampled angle whose mirror partner is sampled (its residual is rounding
    noise: the partner's snapshot is in the basis span): the solve is
    bitwise the one that evaluates every angle (RTLR_VERIFY_MIRRORS=eval),
    and with =check the skipped residuals are reported far below eps_res."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for v in ("eval", "skip", "check"):
        f = str(tmp_path / f"phi_{v}.npy")
        env = dict(os.environ, RTLR_VERIFY_MIRRORS=v)
        res = subprocess.run([sys.executable, "-c", _MIRROR_RUN, root, f], env=env, check=True, timeout=600,
                             capture_output=True, text=True)
        out[v] = np.load(f)
        if v == "check":
            worst = [float(l.split("largest residual ")[1].split()[0]) for l in res.stderr.splitlines()
                     if "sampled mirror partner" in l]
            assert worst and max(worst) < 1e-3 * 1e-7
    assert np.array_equal(out["eval"], out["skip"])
    assert np.array_equal(out["eval"], out["check"])


def _coercive_projections(r, rng):
    """Five r x r matrices shaped like the reduced operators: upwind
    derivative projections (skew part plus a positive semidefinite flux
    part) and a positive definite Sigma_t projection."""
    out = []
    for _ in range(4):
        g = rng.standard_normal((r, r)) / np.sqrt(r)
        h = rng.standard_normal((r, r)) / np.sqrt(r)
        out.append(g - g.T + 0.3 * h @ h.T)
    h = rng.standard_normal((r, r)) / np.sqrt(r)
    out.append(np.eye(r) + 0.2 * h @ h.T)
    return out


@pytest.mark.parametrize("r0,k,m", [(65, 8, 16), (100, 4, 16), (160, 8, 7), (257, 8, 16), (300, 0, 3), (333, 5, 16),
                                    (600, 8, 16), (40, 3, 5), (31, 8, 2), (100, 12, 16), (300, 9, 4), (600, 16, 16),
                                    (130, 16, 3)])
def test_bordered_galerkin_solve(r0, k, m):
    """The greedy candidates' prefactored systems (rank r0 factors finished
    with k border columns, dense.cu galerkin_border_kernel) against the
    pivoted LU at rank r0 + k and against LAPACK."""
    rng = np.random.default_rng(1000 * r0 + k)
    r = r0 + k
    proj = _coercive_projections(r, rng)
    nd = 24
    th = rng.uniform(0, 2 * np.pi, nd)
    dirs = np.stack([np.cos(th), np.sin(th), rng.uniform(0.1, 0.9, nd)], axis=1)
    angles = rng.choice(nd, size=m, replace=False)
    prhs = rng.standard_normal(r)
    full, bord = P.dense_galerkin_border(r0, k, angles, dirs, proj, prhs)
    for c, j in enumerate(angles):
        ox, oy = dirs[j, 0], dirs[j, 1]
        a = ox * proj[0 if ox >= 0 else 1] + oy * proj[2 if oy >= 0 else 3] + proj[4]
        ref = np.linalg.solve(a, prhs)
        assert np.linalg.norm(full[:, c] - ref) <= 1e-11 * np.linalg.norm(ref)
        assert np.linalg.norm(bord[:, c] - ref) <= 1e-11 * np.linalg.norm(ref), (r0, k, c)


_PREFACTOR_RUN = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2603_25233_b200 as P
g = P.Problem("C3", nx=48, ny=48, n_theta=24, n_omega_z=8)
r = g.solve_low_rank(build_factors=0)
np.save(sys.argv[2], np.concatenate([[r.iterations, sum(r.history("inner_iterations"))], r.history("rank"), r.phi]))
'''


def test_prefactored_candidates_keep_the_solve(tmp_path):
    """The greedy candidates' systems factored one inner iteration ahead on
    the second stream and finished by bordering (lowrank.cu predraw,
    dense.cu galerkin_border_kernel), from rank 8 up here: every bordered
    batch equals the full pivoted LU to rounding (the check mode compares
    them in situ), the solve is reproducible run to run, and against the
    solve without the look-ahead the outer iterations and ranks are equal
    and phi agrees far inside the low-rank tolerance."""
    import os
    import re
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out, err = {}, {}
    for tag, v in (("on", "1"), ("on2", "1"), ("off", "0"), ("check", "check")):
        f = str(tmp_path / f"pf_{tag}.npy")
        env = dict(os.environ, RTLR_LU_PREFACTOR=v, RTLR_LU_PREFACTOR_MIN="8")
        res = subprocess.run([sys.executable, "-c", _PREFACTOR_RUN, root, f], env=env, check=True, timeout=600,
                             capture_output=True, text=True)
        out[tag], err[tag] = np.load(f), res.stderr
    assert np.array_equal(out["on"], out["on2"])
    assert np.array_equal(out["on"], out["check"])
    m = re.search(r"over (\d+) candidate batches: worst relative difference of a solution ([0-9.e+-]+)", err["check"])
    assert m, err["check"][-400:]
    assert int(m.group(1)) >= 20 and float(m.group(2)) <= 1e-12, m.group(0)
    nit = int(out["off"][0])
    assert out["on"][0] == out["off"][0]
    assert np.array_equal(out["on"][2:2 + nit], out["off"][2:2 + nit])  # ranks per outer iteration
    assert rel(out["on"][2 + nit:], out["off"][2 + nit:]) <= 1e-9


_PREFACTOR_SHARDED_RUN = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2603_25233_b200 as P
g = P.Problem("C3", nx=48, ny=48, n_theta=24, n_omega_z=8)
if sys.argv[3] == "1":
    g.set_comm(1, 0, P.nccl_unique_id())
r = g.solve_low_rank(build_factors=0)
np.save(sys.argv[2], np.concatenate([[r.iterations, sum(r.history("inner_iterations"))], r.history("rank"), r.phi]))
'''


def test_prefactored_candidates_with_a_communicator(tmp_path):
    """With a communicator every rank factors and finishes all the greedy
    candidates itself (replicated projections, no all-gather of their
    solutions): a single-rank NCCL solve is bitwise the unsharded one with
    the look-ahead active from rank 8 up."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for tag in ("0", "1"):
        f = str(tmp_path / f"pfs_{tag}.npy")
        env = dict(os.environ, RTLR_LU_PREFACTOR_MIN="8")
        subprocess.run([sys.executable, "-c", _PREFACTOR_SHARDED_RUN, root, f, tag], env=env, check=True, timeout=600)
        out[tag] = np.load(f)
    assert np.array_equal(out["0"], out["1"])


_PREDRAW_RUN = r'''
import sys, json, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2603_25233_b200 as P
g = P.Problem("C3", nx=48, ny=48, n_theta=24, n_omega_z=8)
r = g.solve_low_rank(build_factors=0)
np.save(sys.argv[2], r.phi)
json.dump({"it": int(r.iterations), "inner": [int(x) for x in r.history("inner_iterations")],
           "rank": [int(x) for x in r.history("rank")], "sampled": r.sampled_log()}, open(sys.argv[2] + ".json", "w"))
'''


def test_predrawn_candidates_follow_the_reference_rng_sequence(tmp_path):
    """The candidates of an inner iteration are drawn at the end of the one
    before (lowrank.cu predraw).  With the look-ahead factorisation out of
    reach (threshold rank 10^6) the arithmetic is that of the solve without
    it, so the early draw alone is tested: the sampled angles of every outer
    iteration, the inner-iteration counts, the ranks and phi are bitwise
    those of the solve that draws where the reference does
    (low_rank.cpp:217-226)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for tag, env_add in (("early", {"RTLR_LU_PREFACTOR_MIN": "1000000"}), ("late", {"RTLR_LU_PREFACTOR": "0"})):
        f = str(tmp_path / f"pd_{tag}.npy")
        subprocess.run([sys.executable, "-c", _PREDRAW_RUN, root, f], env=dict(os.environ, **env_add), check=True,
                       timeout=600)
        out[tag] = (np.load(f), json.load(open(f + ".json")))
    assert out["early"][1] == out["late"][1]
    assert np.array_equal(out["early"][0], out["late"][0])
    assert sum(out["early"][1]["inner"]) >= 20
