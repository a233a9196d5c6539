"""GPU solvers at the BASELINE configs' full size against golden fixtures
produced by the CPU oracle (tests/golden/make_golden.py).  Bars from the
north star: scalar flux rel. L2 <= 1e-10 (full rank) / 1e-8 (low rank),
outer iterations +-1, final rank reported side by side (+-2)."""
import os

import numpy as np
import pytest

import paper_2603_25233_b200 as P

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def split_log(counts, flat):
    out, k = [], 0
    for c in counts:
        out.append([int(v) for v in flat[k:k + int(c)]])
        k += int(c)
    return out


def sampled_side_by_side(gpu_log, ref_log):
    """Per outer iteration: common prefix of the sampled orders and the Jaccard
    index of the sampled sets (GPU vs oracle)."""
    rows = []
    for a, b in zip(gpu_log, ref_log):
        prefix = next((i for i, (x, y) in enumerate(zip(a, b)) if x != y), min(len(a), len(b)))
        sa, sb = set(a), set(b)
        jac = len(sa & sb) / max(1, len(sa | sb))
        rows.append((len(a), len(b), prefix, jac))
    return rows


def load(tag):
    path = os.path.join(GOLD, tag + ".npz")
    if not os.path.exists(path):
        pytest.skip(f"no golden fixture {tag}")
    return np.load(path)


# C4r: BASELINE C4's medium and source (the same ScalarFields) on 128^2 cells
# with CL(32, 16) = 512 directions, p = 8, q = 16: C4's low-rank oracle run
# at full size takes days on one core, this one 371 s, so the low-rank GPU
# solve of C4's medium is held to the oracle's own low-rank run (ranks,
# iterations, sampled sets side by side) as well as to its full-rank run.
C4R = {"nx": 128, "ny": 128, "n_theta": 32, "n_omega_z": 16}
C4R_TAG = "C4_n_omega_z16_n_theta32_nx128_ny128"
# C4m: the same medium at 256^2 cells (262,144 DOFs, rank ~229 of the 256
# distinct directions): the largest low-rank oracle run of C4's medium that
# fits a session (tests/golden/make_golden.py, one core).
C4M = {"nx": 256, "ny": 256, "n_theta": 32, "n_omega_z": 16}
C4M_TAG = "C4_n_omega_z16_n_theta32_nx256_ny256"
# C4l: 384^2 cells (589,824 DOFs), the oracle's low-rank run ~1 h.
C4L = {"nx": 384, "ny": 384, "n_theta": 32, "n_omega_z": 16}
C4L_TAG = "C4_n_omega_z16_n_theta32_nx384_ny384"
TAGS = {128: C4R_TAG, 256: C4M_TAG, 384: C4L_TAG}


@pytest.mark.parametrize("name,method,ov", [("C1", "full", {}), ("C2", "full", {}), ("C2", "lowrank", {}),
                                            ("C3", "full", {}), ("C3", "lowrank", {}), ("C4", "full", {}),
                                            ("C4", "full", C4R), ("C4", "lowrank", C4R),
                                            ("C4", "full", C4M), ("C4", "lowrank", C4M),
                                            ("C4", "full", C4L), ("C4", "lowrank", C4L)],
                         ids=["C1-full", "C2-full", "C2-lowrank", "C3-full", "C3-lowrank", "C4-full",
                              "C4r-full", "C4r-lowrank", "C4m-full", "C4m-lowrank", "C4l-full", "C4l-lowrank"])
def test_baseline_config_matches_oracle(name, method, ov):
    g = load((TAGS[ov["nx"]] if ov else name) + f"_{method}")
    p = P.Problem(name, **ov)
    r = p.solve_full_rank(store_psi=0) if method == "full" else p.solve_low_rank(build_factors=0)
    ref = g["phi"]
    err = np.linalg.norm(r.phi - ref) / np.linalg.norm(ref)
    tol = 1e-10 if method == "full" else 1e-8
    print(f"{name} {method}: it {r.iterations} vs {int(g['iterations'])}, rel {err:.2e}")
    assert r.converged and bool(g["converged"])
    assert abs(r.iterations - int(g["iterations"])) <= 1
    assert err <= tol
    if method == "lowrank":
        ranks, ref_ranks = r.history("rank"), g["rank"]
        print(f"  ranks GPU {list(map(int, ranks))} oracle {list(map(int, ref_ranks))}")
        assert abs(int(ranks[-1]) - int(ref_ranks[-1])) <= 2
        # The greedily selected direction sets side by side with the oracle's
        # (north star).  The greedy picks agree until the candidate residuals
        # reach rounding level, where either pick is valid and the two
        # summation orders break near-ties differently; asserted: the first
        # 8 picks of the first outer iteration are identical and the first
        # outer iteration's sets overlap by at least half (Jaccard >= 0.5).
        rows = sampled_side_by_side(r.sampled_log(), split_log(g["sampled_counts"], g["sampled_flat"]))
        for k, (na, nb, prefix, jac) in enumerate(rows):
            print(f"  outer {k + 1}: sampled GPU {na} oracle {nb}, common prefix {prefix}, Jaccard {jac:.2f}")
        assert len(rows) >= 1
        assert rows[0][2] >= min(8, rows[0][1])
        assert rows[0][3] >= 0.5


def test_c4_low_rank_against_oracle_full_rank():
    """C4's low-rank oracle run takes days on one core, so the GPU low-rank
    solve is held to the oracle's full-rank flux: the low-rank iteration
    converges to the same SI-DSA fixed point (the reference's LR-vs-FR bar is
    1e-6 absolute, proj/tests/test_low_rank.cpp:472-498); asserted here at the
    low-rank parity bar, 1e-8 relative, and iterations +-1."""
    g = load("C4_full")
    p = P.Problem("C4")
    r = p.solve_low_rank(build_factors=0)
    ref = g["phi"]
    err = np.linalg.norm(r.phi - ref) / np.linalg.norm(ref)
    print(f"C4 lowrank vs oracle full: it {r.iterations} vs {int(g['iterations'])}, rel {err:.2e}, "
          f"abs {np.linalg.norm(r.phi - ref):.2e}, rank {int(r.history('rank')[-1])}")
    assert r.converged and abs(r.iterations - int(g["iterations"])) <= 1
    assert np.linalg.norm(r.phi - ref) <= 1e-6 and err <= 1e-8
