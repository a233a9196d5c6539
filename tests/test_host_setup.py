"""Product host setup vs the oracle, bit for bit (north star: bit-exact
quadrature and mesh indexing; identical assembled inputs), plus the C-ABI
surface and the angle partition.  CPU only: problems are assembled with
device = -1 (host-only)."""
import os
import re

import numpy as np
import pytest

import _oracle as O
import paper_2603_25233_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [
    ("C1", {}),
    ("C2", {}),
    ("C3", {"nx": 98, "ny": 77}),
    ("C4", {}),
    ("C5", {"nx": 64, "ny": 48}),
    ("homogeneous(100,2)", {}),
    ("pin_cell", {}),
    ("variable_scattering", {}),
    ("lattice", {}),
]


def _pair(name, ov):
    o = O.Problem(name, assemble=False, **ov)
    o.set("dsa_factor", 0)
    o.assemble()
    p = P.Problem(name, device=-1, **ov)
    return o, p


@pytest.mark.parametrize("name,ov", CASES)
def test_inputs_bitwise(name, ov):
    o, p = _pair(name, ov)
    assert (p.n, p.n_omega) == (o.n, o.n_omega)
    assert np.array_equal(p.get("dirs"), o.get("dirs"))
    assert np.array_equal(p.get("weights"), o.get("weights"))
    assert np.array_equal(p.get("source"), o.get("source"))
    for blk in ("sigma_t_blocks", "sigma_s_blocks", "sigma_a_blocks"):
        assert np.array_equal(p.get(blk), o.get(blk)), blk
    assert np.array_equal(p.get("stream_blocks"), o.get("stream_blocks"))


def _bsr_to_dense_rows(p, sip):
    """Scatter the product's 5-block BSR into a scipy matrix."""
    import scipy.sparse as sp
    nx, ny = p.nx, p.ny
    rows, cols, vals = [], [], []
    for c in range(p.ncell):
        a, b = c % nx, c // nx
        nbr = [c, c - 1 if a > 0 else -1, c + 1 if a + 1 < nx else -1,
               c - nx if b > 0 else -1, c + nx if b + 1 < ny else -1]
        for s, cc in enumerate(nbr):
            if cc < 0:
                assert not sip[c, s].any()
                continue
            blk = sip[c, s]
            for i in range(4):
                for j in range(4):
                    if blk[i, j] != 0.0:
                        rows.append(4 * c + i)
                        cols.append(4 * cc + j)
                        vals.append(blk[i, j])
    return sp.csr_matrix((vals, (rows, cols)), shape=(p.n, p.n))


@pytest.mark.parametrize("name,ov", [("C1", {}), ("C3", {"nx": 49, "ny": 35}),
                                     ("C4", {"nx": 64, "ny": 64}), ("lattice", {"nx": 20, "ny": 20}),
                                     ("pin_cell", {})])
def test_sip_matrix_bitwise(name, ov):
    o, p = _pair(name, ov)
    ref = o.csr("sip").tocoo()
    mine = _bsr_to_dense_rows(p, p.get("sip_bsr")).tocsr()
    got = np.asarray(mine[ref.row, ref.col]).ravel()
    assert np.array_equal(got, ref.data)
    # the reference CSR also keeps duplicate sums that cancel to exactly 0
    assert mine.nnz == np.count_nonzero(ref.data)


def test_quadrature_bitwise_all_baseline_rules():
    for nt, nz in ((16, 8), (32, 16), (48, 24), (64, 32), (32, 8), (64, 16), (128, 32)):
        p = P.Problem("C5", device=-1, nx=4, ny=4, n_theta=nt, n_omega_z=nz)
        d, w = O.quadrature(nt, nz)
        assert np.array_equal(p.get("dirs"), d) and np.array_equal(p.get("weights"), w)
        assert p.n_unique == nt * nz // 2  # mirror pairs collapse


@pytest.mark.parametrize("degree", [0, 2, 3, 4])
@pytest.mark.parametrize("name,ov", [("pin_cell", {"nx": 9, "ny": 7}), ("C4", {"nx": 24, "ny": 20}),
                                     ("homogeneous(1,1)", {"nx": 5, "ny": 6, "boundary_const": 0.5})])
def test_general_degree_inputs_bitwise(name, ov, degree):
    """K != 1 assembly (host_dgk.cpp): streaming blocks, (K+2)^2-point cross
    sections and source projection bitwise equal to the oracle's general-K
    restatement of operators.cpp."""
    o = O.Problem(name, degree=degree, use_dsa=0, **ov)
    p = P.Problem(name, device=-1, degree=degree, use_dsa=0, **ov)
    assert (p.degree, p.dofs_per_cell, p.n) == (degree, (degree + 1) ** 2, o.n)
    assert np.array_equal(p.get("source"), o.get("source"))
    for blk in ("sigma_t_blocks", "sigma_s_blocks", "sigma_a_blocks"):
        assert np.array_equal(p.get(blk), o.get(blk)), blk
    assert np.array_equal(p.get("stream_blocks"), o.get("stream_blocks"))


def test_degree_above_four_rejected():
    with pytest.raises(P.InvalidArgument, match="degree"):
        P.Problem("homogeneous(1,1)", device=-1, degree=5)


def test_config_errors_map_to_config_error():  # problem.cpp:95-107
    with pytest.raises(P.ConfigError):
        P.Problem("no_such_preset", device=-1)
    with pytest.raises(P.ConfigError, match="p <= q"):
        P.Problem("C1", device=-1, p=9, q=8)


def test_host_only_problem_rejects_gpu_calls():
    p = P.Problem("C1", device=-1)
    with pytest.raises(P.InvalidArgument, match="host-only"):
        p.sweep([0], p.get("source"))


def test_c_abi_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "rtlr_cu.h")).read()
    declared = set(re.findall(r"\b(rtlr_cu_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(P.EXPORTS)
    lib = P.load_library()
    for sym in declared:
        assert hasattr(lib, sym), sym


@pytest.mark.parametrize("nt,nz,n", [(16, 8, 1), (16, 8, 2), (32, 16, 4), (64, 32, 8), (7, 3, 3)])
def test_partition_angles(nt, nz, n):
    parts = [P.partition_angles(nt, nz, n, r) for r in range(n)]
    allv = np.concatenate(parts)
    assert sorted(allv.tolist()) == list(range(nt * nz))
    sizes = [len(x) for x in parts]
    assert max(sizes) - min(sizes) <= 2
    for x in parts:  # mirror pairs never split
        s = set(x.tolist())
        for a in x:
            j1, j2 = divmod(int(a), nz)
            assert j1 * nz + (nz - 1 - j2) in s


def test_c5_uniform_matches_oracle():
    # host restatement of the device generator (paper_2603_25233_b200/csrc/host.hpp)
    vals = [O.c5_uniform(12345, c) for c in (0, 1, 2, 10**9, 2**40 + 7)]
    assert all(0.0 <= v < 1.0 for v in vals)
    assert len(set(vals)) == len(vals)


@pytest.mark.parametrize("name,ov", [("pin_cell", {"nx": 12, "ny": 10}), ("C4", {"nx": 32, "ny": 32, "n_theta": 8,
                                                                                "n_omega_z": 4})])
def test_uploaded_arrays_assemble_like_the_preset(name, ov):
    """rtlr_cu_problem_upload on the host (device < 0) with a preset's own
    arrays: the completed problem (SIP matrix built from the blocks, streaming
    blocks from the mesh) is bitwise the preset's."""
    a = P.Problem(name, device=-1, **ov)
    dom = {"pin_cell": (-1.0, 1.0, -1.0, 1.0), "C4": (0.0, 1.0, 0.0, 1.0)}[name]
    u = P.upload_problem(a.nx, a.ny, a.get("dirs"), a.get("weights"), a.get("sigma_t_blocks"),
                         a.get("sigma_s_blocks"), a.get("source"), domain=dom, n_theta=a.n_theta,
                         n_omega_z=a.n_omega_z, sigma_a_blocks=a.get("sigma_a_blocks"), device=-1)
    for what in ("dirs", "weights", "source", "sigma_t_blocks", "sigma_s_blocks", "sigma_a_blocks", "sip_bsr",
                 "stream_blocks"):
        assert np.array_equal(u.get(what), a.get(what)), what
    assert (u.n_unique, u.sigma_t_uniform) == (a.n_unique, a.sigma_t_uniform)


def test_upload_rejects_bad_descriptions():
    a = P.Problem("homogeneous(1,1)", device=-1, nx=4, ny=4)
    args = (a.nx, a.ny, a.get("dirs"), a.get("weights"), a.get("sigma_t_blocks"), a.get("sigma_s_blocks"),
            a.get("source"))
    with pytest.raises(P.InvalidArgument):
        P.upload_problem(*args, n_theta=3, n_omega_z=3, device=-1)  # 9 != 32 directions
    with pytest.raises(P.InvalidArgument):
        P.upload_problem(0, 4, *args[2:], device=-1)
    bad = a.get("sigma_t_blocks").copy()
    bad[0, 0, 0] = 0.0
    with pytest.raises(P.RtlrError, match="sigma_t must be positive"):
        P.upload_problem(a.nx, a.ny, a.get("dirs"), a.get("weights"), bad, a.get("sigma_s_blocks"), a.get("source"),
                         device=-1)


def test_host_low_rank_helpers():
    """SubsampleRng / truncation_rank through the ABI (host logic, no GPU):
    the reference's known answers (test_low_rank.cpp:57-82, 330-336)."""
    a, b = P.SubsampleRng(1234), P.SubsampleRng(1234)
    for _ in range(50):
        sa, sb = a.sample_without_replacement(list(range(128)), 3), b.sample_without_replacement(list(range(128)), 3)
        assert sa == sb and len(set(sa)) == 3
    c = P.SubsampleRng(99)
    for _ in range(2000):
        s = c.sample_without_replacement(list(range(10)), 3)
        assert len(set(s)) == 3 and all(0 <= v < 10 for v in s)
    assert sorted(P.SubsampleRng(5).sample_without_replacement(list(range(10)), 64)) == list(range(10))
    assert P.truncation_rank([1.0, 1e-4, 1e-12], 1e-8) == 2
    assert P.truncation_rank([1.0, 1e-4, 1e-12], 1e-2) == 1
    assert P.truncation_rank([1.0, 1e-4, 1e-12], 1e-18) == 3
    assert P.truncation_rank([0.0, 0.0, 0.0, 0.0], 1e-8) == 1
    p = P.lr_params()
    assert (p.p, p.q, p.eps_res, p.eps_diff, p.eps_svd, p.eps_mgs) == (1, 8, 1e-7, 1e-7, 1e-8, 1e-10)


def test_cpp_facade_consumer_builds_and_runs_host_only():
    """include/rtlr_cu.hpp (the rtlr::cuda façade of INTEGRATION.md §1) compiled
    into a C++ consumer (tests/cpp/facade_test.cpp) that links only the
    library; its host-only checks run without a GPU."""
    import subprocess
    from paper_2603_25233_b200 import build as B
    B._build_facade_test()
    r = subprocess.run([B.FACADE, "--no-gpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
