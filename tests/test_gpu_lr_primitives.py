"""The reference's low-rank unit tests (proj/tests/test_low_rank.cpp:84-423)
and acceptance criterion 3 (proj/tests/acceptance.cpp:143-236), restated on
the GPU through the exported primitives (rtlr_cu_lr_*: LowRankBasis,
greedy_subsample, truncation_rank / truncate_factors, low_rank_si).

The tiny problems are make_tiny's (test_low_rank.cpp:25-41): [-1,1]^2,
sigma_s = 1 or the pin-cell field, sigma_a = 0, a Gaussian source — the
"homogeneous(1,1)" preset with overrides.  Direct products X^T A X use the
oracle's assembled CSR operators (the same matrices as the reference's
ops).  Bars are the reference's own.
"""
import numpy as np
import pytest

import _oracle as O
import paper_2603_25233_b200 as P

pytestmark = pytest.mark.gpu


def pin(x, y):
    return 0.1 if (abs(x) <= 0.5 and abs(y) <= 0.5) else 100.0


def tiny(nx, n_theta, n_omega_z, pin_cell=False):
    fields = {"sigma_s": pin} if pin_cell else None
    ov = dict(nx=nx, ny=nx, n_theta=n_theta, n_omega_z=n_omega_z, use_dsa=0)
    return P.Problem("homogeneous(1,1)", fields=fields, **ov), O.Problem("homogeneous(1,1)", fields=fields, **ov)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def upwind(o, omx, omy):  # operators.cpp:298-308: Omega >= 0 -> "minus"
    a = o.csr("sigma_t").toarray()
    a = a + omx * o.csr("d_x_minus" if omx >= 0 else "d_x_plus").toarray()
    a = a + omy * o.csr("d_y_minus" if omy >= 0 else "d_y_plus").toarray()
    return a


def test_orthogonal_snapshots_into_empty_basis():  # test_low_rank.cpp:84-98
    g, _ = tiny(5, 4, 2)
    b = P.LowRankBasis(g, np.zeros(g.n))
    snaps = np.zeros((g.n, 3))
    snaps[0, 0], snaps[1, 1], snaps[2, 2] = 2.0, -3.0, 0.5
    assert not b.mgs_ro_update(snaps, [0, 1, 2], 1e-10)
    assert b.rank() == 3
    x, rec = b.basis(), b.coefficient_record()
    assert np.linalg.norm(x.T @ x - np.eye(3)) < 1e-14
    assert all(rec[i, i] > 0 for i in range(3))
    assert np.linalg.norm(x @ rec - snaps) < 1e-14


def test_dependent_snapshot_dropped_keeps_coefficients():  # :100-115
    g, _ = tiny(5, 4, 2)
    rng = np.random.default_rng(3)
    b = P.LowRankBasis(g, np.zeros(g.n))
    first = rng.standard_normal((g.n, 2))
    b.mgs_ro_update(first, [0, 1], 1e-10)
    assert b.rank() == 2
    dup = (0.25 * first[:, 0] - 2.0 * first[:, 1])[:, None]
    b.mgs_ro_update(dup, [2], 1e-10)
    assert b.rank() == 2 and b.snapshot_count() == 3
    rec = b.coefficient_record()
    assert np.linalg.norm(b.basis() @ rec[:, 2] - dup[:, 0]) <= 1e-10 * np.linalg.norm(dup)


def test_300_random_steps_track_qr():  # :117-147 (rank 300 > N_Omega: the record and projections grow)
    g, _ = tiny(10, 4, 2)  # N_x = 400
    rng = np.random.default_rng(77)
    b = P.LowRankBasis(g, np.zeros(g.n))
    acc, step = [], 0
    while sum(a.shape[1] for a in acc) < 300:
        p = min(1 + step % 3, 300 - sum(a.shape[1] for a in acc))
        s = rng.standard_normal((g.n, p))
        b.mgs_ro_update(s, [0] * p, 1e-10)
        acc.append(s)
        step += 1
    A = np.hstack(acc)
    assert b.rank() == 300
    x = b.basis()
    assert np.linalg.norm(x.T @ x - np.eye(300)) <= 1e-10
    assert np.linalg.norm(x @ b.coefficient_record() - A) <= 1e-9 * np.linalg.norm(A)
    q, _ = np.linalg.qr(A)
    d = np.minimum(np.linalg.norm(x - q, axis=0), np.linalg.norm(x + q, axis=0))
    assert d.max() <= 1e-10, d.max()


def test_forced_reorthogonalization_keeps_invariants():  # :149-178
    g, o = tiny(5, 8, 4, pin_cell=True)
    rng = np.random.default_rng(11)
    b = P.LowRankBasis(g, rng.standard_normal(g.n))
    st = o.csr("sigma_t").toarray()
    acc, reorth = [], 0
    for _ in range(12):
        s = rng.standard_normal((g.n, 2))
        ro = b.mgs_ro_update(s, [0, 1], 0.0)  # eps_mgs = 0 forces the Householder rebuild
        reorth += ro
        b.update_projections(ro)
        acc.append(s)
        A = np.hstack(acc)
        r, x = b.rank(), b.basis()
        assert np.linalg.norm(x.T @ x - np.eye(r)) <= 1e-12
        assert np.linalg.norm(x @ b.coefficient_record() - A) <= 1e-9 * np.linalg.norm(A)
        assert rel(b.projected("sigma_t"), x.T @ st @ x) <= 1e-11
    assert reorth > 0


def test_incremental_projections_match_direct_products():  # :180-206
    g, o = tiny(4, 4, 2, pin_cell=True)
    rng = np.random.default_rng(5)
    phi_prev = rng.standard_normal(g.n)
    rhs_core = o.rhs_core(phi_prev)
    b = P.LowRankBasis(g, rhs_core)
    mats = {k: o.csr(m).toarray() for k, m in (("dx_minus", "d_x_minus"), ("dx_plus", "d_x_plus"),
                                                ("dy_minus", "d_y_minus"), ("dy_plus", "d_y_plus"),
                                                ("sigma_t", "sigma_t"))}
    for start in range(0, g.n_omega - 1, 2):
        ang = [start, start + 1]
        snaps = g.sweep(ang, np.column_stack([rhs_core, rhs_core]))
        ro = b.mgs_ro_update(snaps, ang, 1e-10)
        b.update_projections(ro)
        x = b.basis()
        for k, a in mats.items():
            assert rel(b.projected(k), x.T @ a @ x) <= 1e-11, k
        assert rel(b.prhs(), x.T @ rhs_core) <= 1e-11


def test_projected_sigma_t_is_identity_for_constant_cross_section():  # :208-216
    g, _ = tiny(4, 4, 2)
    rng = np.random.default_rng(19)
    b = P.LowRankBasis(g, np.zeros(g.n))
    ro = b.mgs_ro_update(rng.standard_normal((g.n, 5)), [0, 1, 2, 3, 4], 1e-10)
    b.update_projections(ro)
    assert np.linalg.norm(b.projected("sigma_t") - np.eye(5)) <= 1e-11 * np.sqrt(5.0)


def test_galerkin_reproduces_snapshots_and_matches_dense_oracle():  # :237-270 and :218-235
    g, o = tiny(4, 4, 2)
    rhs_core = o.rhs_core(np.zeros(g.n))
    b = P.LowRankBasis(g, rhs_core)
    angles = [0, 3, 5, 6]
    snaps = g.sweep(angles, np.column_stack([rhs_core] * 4))
    b.update_projections(b.mgs_ro_update(snaps, angles, 1e-10))
    rec, x = b.coefficient_record(), b.basis()
    c = b.galerkin_solve(angles)
    for i in range(4):
        assert np.linalg.norm(x @ c[:, i] - snaps[:, i]) <= 1e-9 * np.linalg.norm(snaps[:, i])
        assert np.linalg.norm(c[:, i] - rec[:, i]) <= 1e-8 * np.linalg.norm(rec[:, i])
    d = o.get("dirs")
    cu = b.galerkin_solve([1, 2, 4, 7])
    for k, j in enumerate([1, 2, 4, 7]):
        red = x.T @ upwind(o, d[j, 0], d[j, 1]) @ x  # reduced_streaming (low_rank.cpp:176-183)
        expect = np.linalg.solve(red, x.T @ rhs_core)
        assert np.linalg.norm(cu[:, k] - expect) <= 1e-10 * max(1.0, np.linalg.norm(expect))


def test_galerkin_exact_once_the_basis_spans_the_space():  # :272-293
    g, o = tiny(1, 8, 1)  # N_x = 4 < N_Omega = 8
    rhs_core = o.get("source")
    b = P.LowRankBasis(g, rhs_core)
    snaps = g.sweep(list(range(5)), np.column_stack([rhs_core] * 5))
    b.update_projections(b.mgs_ro_update(snaps, list(range(5)), 1e-10))
    assert b.rank() == g.n
    d = o.get("dirs")
    c = b.galerkin_solve(list(range(g.n_omega)))
    for j in range(g.n_omega):
        direct = np.linalg.solve(upwind(o, d[j, 0], d[j, 1]), rhs_core)
        assert np.linalg.norm(b.basis() @ c[:, j] - direct) <= 1e-10 * np.linalg.norm(direct)


def test_greedy_subsampling_selection_and_determinism():  # :295-328
    g, o = tiny(1, 8, 1)
    rhs_core = o.get("source")
    b = P.LowRankBasis(g, rhs_core)
    snaps = g.sweep(list(range(4)), np.column_stack([rhs_core] * 4))
    b.update_projections(b.mgs_ro_update(snaps, list(range(4)), 1e-10))
    assert b.rank() == g.n
    mask = [1, 1, 1, 1, 0, 0, 0, 0]
    s1 = P.greedy_subsample(b, mask, 2, 4, P.SubsampleRng(42))
    s2 = P.greedy_subsample(b, mask, 2, 4, P.SubsampleRng(42))
    assert s1["selected"] == s2["selected"] and len(s1["selected"]) == 2
    assert s1["max_residual"] < 1e-10
    assert all(not mask[j] for j in s1["selected"])
    norms = dict(zip(s1["candidates"], s1["residual_norms"]))
    max_sel = max(norms[j] for j in s1["selected"])
    for j, v in norms.items():
        if j not in s1["selected"]:
            assert v <= max_sel + 1e-18


def test_greedy_subsample_scores_match_full_space_residuals():
    """The greedy scores are residual_norm(angle, c) = ||rhs_j - A_j X c||
    (low_rank.cpp:202-208, 236-238), checked against dense products."""
    g, o = tiny(4, 8, 4, pin_cell=True)
    rhs_core = o.rhs_core(np.linspace(0, 1, g.n))
    b = P.LowRankBasis(g, rhs_core)
    ang = [0, 9, 17]
    b.update_projections(b.mgs_ro_update(g.sweep(ang, np.column_stack([rhs_core] * 3)), ang, 1e-10))
    mask = np.zeros(g.n_omega, dtype=np.uint8)
    mask[ang] = 1
    out = P.greedy_subsample(b, mask, 3, 8, P.SubsampleRng(5))
    d, x = o.get("dirs"), b.basis()
    for k, j in enumerate(out["candidates"]):
        r = rhs_core - upwind(o, d[j, 0], d[j, 1]) @ (x @ out["candidate_solutions"][:, k])
        assert abs(out["residual_norms"][k] - np.linalg.norm(r)) <= 1e-12 * max(1.0, np.linalg.norm(r))
    # the sampled candidates follow the reference RNG: the same draws as SubsampleRng(5) on the pool
    pool = [j for j in range(g.n_omega) if not mask[j]]
    assert out["candidates"] == P.SubsampleRng(5).sample_without_replacement(pool, 8)


def test_truncation_rank_and_factors():  # :330-378
    assert P.truncation_rank([1.0, 1e-4, 1e-12], 1e-8) == 2
    assert P.truncation_rank([1.0, 1e-4, 1e-12], 1e-2) == 1
    assert P.truncation_rank([1.0, 1e-4, 1e-12], 1e-18) == 3
    assert P.truncation_rank([0.0] * 4, 1e-8) == 1
    g = P.Problem("homogeneous(1,1)", nx=3, ny=3, n_theta=10, n_omega_z=1, use_dsa=0)  # N_x = 36, N_Omega = 10
    rng = np.random.default_rng(2)
    u, v = rng.standard_normal((6, 1)), rng.standard_normal((10, 1))
    c1 = u @ v.T
    bx, _ = np.linalg.qr(rng.standard_normal((g.n, 6)))
    X1, S1, V1 = P.truncate_factors(g, c1, bx, 1e-8)
    assert len(S1) == 1
    assert np.linalg.norm(X1 @ np.diag(S1) @ V1.T - bx @ c1) <= 1e-12 * np.linalg.norm(c1)
    uu, _ = np.linalg.qr(rng.standard_normal((6, 3)))
    vv, _ = np.linalg.qr(rng.standard_normal((10, 3)))
    c2 = uu @ np.diag([1.0, 1e-4, 1e-12]) @ vv.T
    bx2, _ = np.linalg.qr(rng.standard_normal((g.n, 6)))
    X2, S2, V2 = P.truncate_factors(g, c2, bx2, 1e-8)
    assert len(S2) == 2
    assert np.linalg.norm(X2.T @ X2 - np.eye(2)) < 1e-13
    assert np.linalg.norm(V2.T @ V2 - np.eye(2)) < 1e-13
    assert S2[0] >= S2[1]
    assert np.linalg.norm(X2 @ np.diag(S2) @ V2.T - bx2 @ c2) <= 1e-10
    sv = P.svd_values(g, c2, bx2)
    assert np.allclose(sv[:3], [1.0, 1e-4, 1e-12], rtol=1e-8, atol=1e-15)


def test_inner_loop_matches_one_si_step():  # :390-412
    g, _ = tiny(4, 4, 2)
    prm = P.lr_params(p=1, q=4)
    phi0 = np.zeros(g.n)
    inner = P.low_rank_si(g, phi0, prm, P.SubsampleRng(7))
    full = g.si_step(phi0)
    assert np.linalg.norm(inner.phi_star - full) <= 1e-7
    assert inner.rank <= min(g.n, g.n_omega)
    assert inner.sampled_count >= inner.rank
    C, X = inner.coefficients, inner.basis
    assert C.shape == (inner.rank, g.n_omega)
    w = g.get("weights")
    acc = sum(w[j] * (X @ C[:, j]) for j in range(g.n_omega))
    assert np.linalg.norm(acc - inner.phi_star) <= 1e-12 * max(1.0, np.linalg.norm(inner.phi_star))


def test_termination_every_angle_meets_the_residual_gate():  # :414-437
    g, o = tiny(6, 8, 4, pin_cell=True)
    rng = np.random.default_rng(13)
    d = o.get("dirs")
    for seed in (1, 2, 3):
        phi_prev = 0.05 * rng.standard_normal(g.n)
        prm = P.lr_params()
        inner = P.low_rank_si(g, phi_prev, prm, P.SubsampleRng(seed))
        rhs_core = o.rhs_core(phi_prev)
        X, C = inner.basis, inner.coefficients
        worst = max(np.linalg.norm(rhs_core - o.apply(d[j, 0], d[j, 1], X @ C[:, j])) for j in range(g.n_omega))
        assert worst < prm.eps_res, (seed, worst)


def test_unreachable_tolerance_falls_back_to_full_rank():  # :439-455
    g, _ = tiny(2, 4, 2)
    prm = P.lr_params(p=2, q=3, eps_res=1e-300)
    phi0 = np.zeros(g.n)
    inner = P.low_rank_si(g, phi0, prm, P.SubsampleRng(3))
    assert inner.exhausted_all_angles
    assert inner.sampled_count == g.n_omega
    full = g.si_step(phi0)
    assert np.linalg.norm(inner.phi_star - full) <= 1e-12 * np.linalg.norm(full)


def test_acceptance_criterion_3_machinery_invariants():
    """acceptance.cpp:143-236: 200 randomized mgs_ro_update steps on sweep
    snapshots of a 4x4 pin cell with CL(8,4), fresh bases with random
    frozen fluxes: orth <= 1e-10, projections <= 1e-11, Galerkin
    reproduction of a sampled angle <= 1e-8, record <= 1e-9."""
    g, o = tiny(4, 8, 4, pin_cell=True)
    rng = np.random.default_rng(777)
    srng = P.SubsampleRng(777)
    st, dxm = o.csr("sigma_t").toarray(), o.csr("d_x_minus").toarray()
    worst = dict(orth=0.0, proj=0.0, galerkin=0.0, record=0.0)
    steps = 0
    while steps < 200:
        phi_prev = 0.2 * rng.standard_normal(g.n)
        rhs_core = o.rhs_core(phi_prev)
        b = P.LowRankBasis(g, rhs_core)
        acc = []
        remaining = list(range(g.n_omega))
        while remaining and steps < 200:
            p = min(1 + srng.draw_below(3), len(remaining))
            chosen = srng.sample_without_replacement(remaining, p)
            for c in chosen:
                remaining.remove(c)
            snaps = g.sweep(chosen, np.column_stack([rhs_core] * p))
            b.update_projections(b.mgs_ro_update(snaps, chosen, 1e-10))
            acc.append(snaps)
            steps += 1
            A = np.hstack(acc)
            r, x = b.rank(), b.basis()
            worst["orth"] = max(worst["orth"], np.linalg.norm(x.T @ x - np.eye(r)))
            worst["record"] = max(worst["record"], rel(x @ b.coefficient_record(), A))
            worst["proj"] = max(worst["proj"], rel(b.projected("sigma_t"), x.T @ st @ x),
                                rel(b.projected("dx_minus"), x.T @ dxm @ x))
            sampled = b.sampled_angles()
            probe = sampled[srng.draw_below(len(sampled))]
            k = sampled.index(probe)
            c = b.galerkin_solve([probe])[:, 0]
            worst["galerkin"] = max(worst["galerkin"], rel(x @ c, A[:, k]))
    print("criterion 3 worst:", worst)
    assert worst["orth"] <= 1e-10 and worst["proj"] <= 1e-11
    assert worst["galerkin"] <= 1e-8 and worst["record"] <= 1e-9


def test_uploaded_problem_matches_preset_solves():
    """rtlr_cu_problem_upload with the arrays of an assembled preset (host
    copies) solves exactly as the preset problem does: full rank and low
    rank, bitwise."""
    name, ov = "pin_cell", dict(nx=16, ny=16, n_theta=8, n_omega_z=4, seed=3)
    a = P.Problem(name, **ov)
    u = P.upload_problem(a.nx, a.ny, a.get("dirs"), a.get("weights"), a.get("sigma_t_blocks"),
                         a.get("sigma_s_blocks"), a.get("source"), domain=(-1.0, 1.0, -1.0, 1.0),
                         n_theta=8, n_omega_z=4, sigma_a_blocks=a.get("sigma_a_blocks"))
    assert np.array_equal(u.get("sip_bsr"), a.get("sip_bsr"))
    fa, fu = a.solve_full_rank(), u.solve_full_rank()
    assert np.array_equal(fa.phi, fu.phi) and fa.iterations == fu.iterations
    la, lu = a.solve_low_rank(seed=3), u.solve_low_rank(seed=3)
    assert np.array_equal(la.phi, lu.phi) and la.sampled_log() == lu.sampled_log()


def test_cpp_facade_consumer_on_gpu():
    """The C++ façade consumer (tests/cpp/facade_test.cpp) with its GPU checks:
    solve_full_rank / solve_low_rank / LowRankBasis / greedy_subsample /
    low_rank_si / DiffusionSystem through include/rtlr_cu.hpp."""
    import subprocess
    from paper_2603_25233_b200 import build as B
    r = subprocess.run([B.FACADE], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("r,n_omega", [(40, 96), (300, 1100), (560, 540)])
def test_singular_values_bidiagonal_path(r, n_omega, monkeypatch):
    """The per-outer-iteration singular values (low_rank.cpp:457) of factors
    with >= 3e5 entries come from a Golub-Kahan bidiagonalisation + bisection
    (no vectors needed; smaller ones from QR + Jacobi); against
    numpy's SVD and the one-sided Jacobi path (RTLR_SVD=jacobi is read once
    per process, so the Jacobi values come from truncate_factors with
    vectors): absolute error <= 1e-13 sigma_max (n eps: backward error of the
    bidiagonalisation) over singular values graded
    from 1 to 1e-13, so the truncation rank (tail sum vs eps_svd * total)
    cannot move."""
    g = P.Problem("homogeneous(1,1)", nx=12, ny=12, n_theta=n_omega, n_omega_z=1, use_dsa=0)
    rng = np.random.default_rng(r)
    k = min(r, n_omega)
    uu, _ = np.linalg.qr(rng.standard_normal((r, k)))
    vv, _ = np.linalg.qr(rng.standard_normal((n_omega, k)))
    s_true = np.logspace(0, -13, k)
    C = uu @ np.diag(s_true) @ vv.T
    bx, _ = np.linalg.qr(rng.standard_normal((g.n, r)))
    sv = P.svd_values(g, C, bx)
    ref = np.linalg.svd(C, compute_uv=False)
    assert len(sv) == k
    assert np.max(np.abs(sv - ref)) <= 1e-13 * ref[0]
    for eps in (1e-8, 1e-10, 1e-6):
        assert P.truncation_rank(sv, eps) == P.truncation_rank(ref, eps)
    _, S2, _ = P.truncate_factors(g, C, bx, 1e-12)  # the vectors path (QR + Jacobi)
    kk = len(S2)
    assert np.max(np.abs(np.asarray(S2) - sv[:kk])) <= 1e-13 * ref[0]
