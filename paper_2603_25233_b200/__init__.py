"""B200-native compute core of the rank-adaptive low-rank SI-DSA transport
solver (arXiv 2603.25233), behind the reference's solver API.

This module is a thin ctypes mirror of the C ABI in include/rtlr_cu.h; the
host drivers and every kernel live in the sm_100a shared library
lib/librtlr_cu.so (built by build.py).  There is no CPU fallback: loading
fails loudly when the library is missing, and every solver call runs on a
GPU.  Names follow the reference (proj/include/rtlr/*.hpp): sweep,
si_step, solve_full_rank, solve_low_rank, DiffusionSystem.solve/correct,
StreamingOperator.apply.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "librtlr_cu.so")

HOST, DEVICE = 0, 1
_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int)
_I64 = ctypes.POINTER(ctypes.c_int64)
# rtlr_cu_field_fn: double f(void* user, double x, double y) (ScalarField, dg_space.hpp:10)
FIELD_FN = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_void_p, ctypes.c_double, ctypes.c_double)
_lib = None

# Every symbol include/rtlr_cu.h declares.
EXPORTS = [
    "rtlr_cu_last_error", "rtlr_cu_version", "rtlr_cu_device_count", "rtlr_cu_config_create",
    "rtlr_cu_config_set", "rtlr_cu_config_set_field", "rtlr_cu_config_destroy",
    "rtlr_cu_problem_create", "rtlr_cu_problem_destroy", "rtlr_cu_problem_info",
    "rtlr_cu_problem_get", "rtlr_cu_problem_degree", "rtlr_cu_problem_set_stream", "rtlr_cu_problem_set_option",
    "rtlr_cu_synchronize", "rtlr_cu_sweep", "rtlr_cu_sweep_dirs", "rtlr_cu_apply",
    "rtlr_cu_rhs_core", "rtlr_cu_si_step", "rtlr_cu_dsa_solve", "rtlr_cu_dsa_correct",
    "rtlr_cu_c5_fill", "rtlr_cu_fr_options_default", "rtlr_cu_lr_options_default",
    "rtlr_cu_solve_full_rank", "rtlr_cu_solve_low_rank", "rtlr_cu_report_info",
    "rtlr_cu_report_get", "rtlr_cu_report_sampled", "rtlr_cu_report_destroy",
    "rtlr_cu_partition_angles", "rtlr_cu_problem_fr_options", "rtlr_cu_problem_lr_options",
    "rtlr_cu_sweep_async", "rtlr_cu_check", "rtlr_cu_nccl_unique_id", "rtlr_cu_problem_set_comm",
    "rtlr_cu_shard_block", "rtlr_cu_dense_qr", "rtlr_cu_dense_galerkin_border", "rtlr_cu_psi_difference",
    "rtlr_cu_config_parse", "rtlr_cu_config_load", "rtlr_cu_config_set_mode", "rtlr_cu_run",
    "rtlr_cu_problem_upload", "rtlr_cu_lr_params_default", "rtlr_cu_rng_create", "rtlr_cu_rng_destroy",
    "rtlr_cu_rng_draw_below", "rtlr_cu_rng_sample", "rtlr_cu_lr_basis_create", "rtlr_cu_lr_basis_destroy",
    "rtlr_cu_lr_basis_info", "rtlr_cu_lr_basis_get", "rtlr_cu_lr_basis_sampled", "rtlr_cu_lr_mgs_ro_update",
    "rtlr_cu_lr_update_projections", "rtlr_cu_lr_galerkin_solve", "rtlr_cu_lr_residual_norms",
    "rtlr_cu_lr_greedy_subsample", "rtlr_cu_lr_build_coefficients", "rtlr_cu_truncation_rank",
    "rtlr_cu_truncate_factors", "rtlr_cu_low_rank_si", "rtlr_cu_inner_info", "rtlr_cu_inner_get",
    "rtlr_cu_inner_sampled", "rtlr_cu_inner_destroy",
]


class FrOptions(ctypes.Structure):
    _fields_ = [("eps_si_sa", ctypes.c_double), ("max_iterations", ctypes.c_int),
                ("use_dsa", ctypes.c_int), ("store_psi", ctypes.c_int)]


class LrOptions(ctypes.Structure):
    _fields_ = [("p", ctypes.c_int), ("q", ctypes.c_int), ("eps_res", ctypes.c_double),
                ("eps_diff", ctypes.c_double), ("eps_svd", ctypes.c_double),
                ("eps_mgs", ctypes.c_double), ("eps_si_sa", ctypes.c_double),
                ("max_iterations", ctypes.c_int), ("use_dsa", ctypes.c_int),
                ("seed", ctypes.c_uint64), ("build_factors", ctypes.c_int)]


class LrParams(ctypes.Structure):
    """LowRankParams (low_rank.hpp:29-36)."""
    _fields_ = [("p", ctypes.c_int), ("q", ctypes.c_int), ("eps_res", ctypes.c_double),
                ("eps_diff", ctypes.c_double), ("eps_svd", ctypes.c_double), ("eps_mgs", ctypes.c_double)]


class ProblemDesc(ctypes.Structure):
    """rtlr_cu_problem_desc: a caller-assembled problem."""
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("x_min", ctypes.c_double),
                ("x_max", ctypes.c_double), ("y_min", ctypes.c_double), ("y_max", ctypes.c_double),
                ("n_theta", ctypes.c_int), ("n_omega_z", ctypes.c_int), ("n_omega", ctypes.c_int),
                ("dirs", ctypes.c_void_p), ("weights", ctypes.c_void_p), ("sigma_t_blocks", ctypes.c_void_p),
                ("sigma_s_blocks", ctypes.c_void_p), ("sigma_a_blocks", ctypes.c_void_p),
                ("source", ctypes.c_void_p), ("boundary", ctypes.c_void_p), ("sip_bsr", ctypes.c_void_p),
                ("use_dsa", ctypes.c_int)]


class RtlrError(RuntimeError):
    """Base of the reference's exception classes as seen through the ABI."""


class InvalidArgument(RtlrError, ValueError):
    pass


class ConfigError(RtlrError):
    pass


class CudaError(RtlrError):
    pass


_ERR = {1: InvalidArgument, 2: RtlrError, 3: ConfigError, 4: CudaError}


def load_library(path: str = LIB_PATH):
    """Loads lib/librtlr_cu.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run paper_2603_25233_b200/build.py (no CPU fallback)")
    L = ctypes.CDLL(path)
    L.rtlr_cu_last_error.restype = ctypes.c_char_p
    L.rtlr_cu_config_create.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    L.rtlr_cu_config_set.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_double]
    L.rtlr_cu_config_destroy.argtypes = [ctypes.c_void_p]
    L.rtlr_cu_config_set_field.argtypes = [ctypes.c_void_p, ctypes.c_char_p, FIELD_FN, ctypes.c_void_p]
    L.rtlr_cu_config_parse.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    L.rtlr_cu_config_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    L.rtlr_cu_config_set_mode.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
    L.rtlr_cu_run.argtypes = [ctypes.c_void_p, ctypes.c_int, _I64, ctypes.c_int, ctypes.c_char_p, ctypes.c_int,
                              ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_int)]
    L.rtlr_cu_problem_create.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    L.rtlr_cu_problem_destroy.argtypes = [ctypes.c_void_p]
    L.rtlr_cu_problem_info.argtypes = [ctypes.c_void_p, _I64]
    L.rtlr_cu_problem_get.argtypes = [ctypes.c_void_p, ctypes.c_char_p, _D]
    L.rtlr_cu_problem_degree.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
    L.rtlr_cu_problem_set_stream.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    L.rtlr_cu_problem_set_option.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_double]
    L.rtlr_cu_synchronize.argtypes = [ctypes.c_void_p]
    L.rtlr_cu_sweep.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
    L.rtlr_cu_sweep_async.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                      ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64]
    L.rtlr_cu_check.argtypes = [ctypes.c_void_p]
    L.rtlr_cu_nccl_unique_id.argtypes = [ctypes.c_char_p]
    L.rtlr_cu_problem_set_comm.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_char_p]
    L.rtlr_cu_sweep_dirs.argtypes =[ctypes.c_void_p, _D, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
    L.rtlr_cu_apply.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_int]
    L.rtlr_cu_rhs_core.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    L.rtlr_cu_si_step.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_int]
    L.rtlr_cu_dsa_solve.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, _I]
    L.rtlr_cu_psi_difference.argtypes = [ctypes.c_void_p] + [ctypes.c_void_p] * 4 + [ctypes.c_int, _D, ctypes.c_int]
    L.rtlr_cu_dsa_correct.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_int]
    L.rtlr_cu_c5_fill.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                  ctypes.c_uint64]
    L.rtlr_cu_fr_options_default.argtypes = [ctypes.POINTER(FrOptions)]
    L.rtlr_cu_lr_options_default.argtypes = [ctypes.POINTER(LrOptions)]
    L.rtlr_cu_problem_fr_options.argtypes = [ctypes.c_void_p, ctypes.POINTER(FrOptions)]
    L.rtlr_cu_problem_lr_options.argtypes = [ctypes.c_void_p, ctypes.POINTER(LrOptions)]
    L.rtlr_cu_solve_full_rank.argtypes = [ctypes.c_void_p, ctypes.POINTER(FrOptions),
                                          ctypes.POINTER(ctypes.c_void_p)]
    L.rtlr_cu_solve_low_rank.argtypes = [ctypes.c_void_p, ctypes.POINTER(LrOptions),
                                         ctypes.POINTER(ctypes.c_void_p)]
    L.rtlr_cu_report_info.argtypes = [ctypes.c_void_p, _I64]
    L.rtlr_cu_report_get.argtypes = [ctypes.c_void_p, ctypes.c_char_p, _D]
    L.rtlr_cu_report_sampled.argtypes = [ctypes.c_void_p, _I, _I]
    L.rtlr_cu_report_destroy.argtypes = [ctypes.c_void_p]
    L.rtlr_cu_partition_angles.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _I, _I]
    _ip = ctypes.POINTER(ctypes.c_int)
    L.rtlr_cu_shard_block.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _ip, _ip, _ip]
    L.rtlr_cu_dense_galerkin_border.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                                ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_void_p, ctypes.c_void_p]
    L.rtlr_cu_dense_qr.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p]
    V, Vp, Dp = ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p), _D
    L.rtlr_cu_problem_upload.argtypes = [ctypes.POINTER(ProblemDesc), ctypes.c_int, Vp]
    L.rtlr_cu_lr_params_default.argtypes = [ctypes.POINTER(LrParams)]
    L.rtlr_cu_lr_params_default.restype = None
    L.rtlr_cu_rng_create.argtypes = [ctypes.c_uint64, Vp]
    L.rtlr_cu_rng_destroy.argtypes = [V]
    L.rtlr_cu_rng_destroy.restype = None
    L.rtlr_cu_rng_draw_below.argtypes = [V, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
    L.rtlr_cu_rng_sample.argtypes = [V, _ip, ctypes.c_int, ctypes.c_int, _ip, _ip]
    L.rtlr_cu_lr_basis_create.argtypes = [V, ctypes.POINTER(LrParams), V, ctypes.c_int, Vp]
    L.rtlr_cu_lr_basis_destroy.argtypes = [V]
    L.rtlr_cu_lr_basis_destroy.restype = None
    L.rtlr_cu_lr_basis_info.argtypes = [V, _I64]
    L.rtlr_cu_lr_basis_get.argtypes = [V, ctypes.c_char_p, V, ctypes.c_int]
    L.rtlr_cu_lr_basis_sampled.argtypes = [V, _ip]
    L.rtlr_cu_lr_mgs_ro_update.argtypes = [V, V, _ip, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                           _ip]
    L.rtlr_cu_lr_update_projections.argtypes = [V, ctypes.c_int]
    L.rtlr_cu_lr_galerkin_solve.argtypes = [V, _ip, ctypes.c_int, V, ctypes.c_int]
    L.rtlr_cu_lr_residual_norms.argtypes = [V, _ip, ctypes.c_int, V, V, ctypes.c_int]
    L.rtlr_cu_lr_greedy_subsample.argtypes = [V, ctypes.c_char_p, ctypes.c_int, ctypes.c_int, V, _ip, _ip, Dp, _ip,
                                              _ip, V, V, ctypes.c_int]
    L.rtlr_cu_lr_build_coefficients.argtypes = [V, _ip, ctypes.c_int, V, V, V, ctypes.c_int]
    L.rtlr_cu_truncation_rank.argtypes = [Dp, ctypes.c_int, ctypes.c_double, _ip]
    L.rtlr_cu_truncate_factors.argtypes = [V, V, V, ctypes.c_int, ctypes.c_double, ctypes.c_int, _ip, V, V, V]
    L.rtlr_cu_low_rank_si.argtypes = [V, V, ctypes.POINTER(LrParams), V, ctypes.c_int, Vp]
    L.rtlr_cu_inner_info.argtypes = [V, _I64]
    L.rtlr_cu_inner_get.argtypes = [V, ctypes.c_char_p, V, ctypes.c_int]
    L.rtlr_cu_inner_sampled.argtypes = [V, _ip]
    L.rtlr_cu_inner_destroy.argtypes = [V]
    L.rtlr_cu_inner_destroy.restype = None
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        msg = load_library().rtlr_cu_last_error().decode()
        raise _ERR.get(rc, RtlrError)(msg)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def device_count() -> int:
    return load_library().rtlr_cu_device_count()


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (create on rank 0, broadcast to the others)."""
    buf = ctypes.create_string_buffer(128)
    _check(load_library().rtlr_cu_nccl_unique_id(buf))
    return buf.raw


def partition_angles(n_theta: int, n_omega_z: int, nranks: int, rank: int) -> np.ndarray:
    """Angles owned by `rank` of `nranks` (mirror pairs kept together)."""
    L = load_library()
    cnt = ctypes.c_int(0)
    _check(L.rtlr_cu_partition_angles(n_theta, n_omega_z, nranks, rank, ctypes.byref(cnt), None))
    out = np.zeros(max(1, cnt.value), dtype=np.int32)
    _check(L.rtlr_cu_partition_angles(n_theta, n_omega_z, nranks, rank, ctypes.byref(cnt),
                                      out.ctypes.data_as(_I)))
    return out[:cnt.value]


def shard_block(m: int, nranks: int, rank: int) -> tuple[int, int, int]:
    """(begin, end, bsz): rank's contiguous block of an m-item low-rank phase."""
    L = load_library()
    b, e, z = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    _check(L.rtlr_cu_shard_block(m, nranks, rank, ctypes.byref(b), ctypes.byref(e), ctypes.byref(z)))
    return b.value, e.value, z.value


def dense_qr(a: np.ndarray, device: int = 0):
    """(q, r) of the GPU blocked Householder QR (the basis-rebuild kernel)."""
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    q = np.zeros((m, n), dtype=np.float64, order="F")
    r = np.zeros((n, n), dtype=np.float64, order="F")
    _check(load_library().rtlr_cu_dense_qr(device, m, n, _dp(a), _dp(q), _dp(r)))
    return q, r


def dense_galerkin_border(r0: int, k: int, angles, dirs: np.ndarray, proj: np.ndarray, prhs: np.ndarray,
                          device: int = 0):
    """(sol_full, sol_border): the Galerkin systems of `angles` solved at rank
    r0 + k by the pivoted LU and by the rank-r0 factors plus the k border
    columns.  proj: (5, r, r) with proj[q][:, :] the q-th projection (stored
    column-major on the device), dirs (n_omega, 3), prhs (r,)."""
    angles = np.ascontiguousarray(angles, dtype=np.int32)
    dirs = np.ascontiguousarray(dirs, dtype=np.float64)
    r = r0 + k
    pj = np.ascontiguousarray(np.stack([np.asfortranarray(proj[q]).T for q in range(5)]), dtype=np.float64)
    prhs = np.ascontiguousarray(prhs, dtype=np.float64)
    m = len(angles)
    s1 = np.zeros((r, m), dtype=np.float64, order="F")
    s2 = np.zeros((r, m), dtype=np.float64, order="F")
    _check(load_library().rtlr_cu_dense_galerkin_border(device, r0, k, m, angles.ctypes.data_as(ctypes.c_void_p),
                                                        dirs.shape[0], _dp(dirs), _dp(pj), _dp(prhs), _dp(s1), _dp(s2)))
    return s1, s2


def compare_runs(full, low, problem=None) -> dict:
    """compare_runs (report.cpp:60-74): speedup, compression ratio, ||phi_LR -
    phi_FR||_2 and, when the full-rank report holds psi and the low-rank one
    its factors, ||psi_FR - X S V^T||_F (computed on the problem's GPU)."""
    if full.phi.size != low.phi.size:
        raise RtlrError("compare_runs: reports come from different discretizations")
    fs, ls = float(full.get("solve_seconds", 1)[0]), float(low.get("solve_seconds", 1)[0])
    n_x = full.phi.size
    n_omega = problem.n_omega if problem is not None else None
    out = {"speedup": fs / ls if ls > 0 else 0.0,
           "compression_ratio": low.psi_dofs / (n_x * n_omega) if n_omega else None,
           "phi_diff_two_norm": float(np.linalg.norm(low.phi - full.phi)), "has_psi_diff": False}
    if problem is not None and full.has_psi and low.factor_rank > 0:
        r = low.factor_rank
        out["psi_diff_two_norm"] = problem.psi_difference(
            full.get("psi", n_x * n_omega), low.get("X", n_x * r), low.get("S", r), low.get("V", n_omega * r))
        out["has_psi_diff"] = True
    return out


class Report:
    """SolveReport (proj/include/rtlr/report.hpp:33-44)."""

    def __init__(self, h):
        self.h = h
        info = np.zeros(8, dtype=np.int64)
        _check(load_library().rtlr_cu_report_info(h, info.ctypes.data_as(_I64)))
        self.iterations = int(info[0])
        self.converged = bool(info[1])
        self.n_history = int(info[2])
        self.has_psi = bool(info[3])
        self.factor_rank = int(info[4])
        self._sampled_total = int(info[5])
        self.psi_dofs = int(info[6])
        self.n = int(info[7])

    def get(self, what: str, n: int) -> np.ndarray:
        out = np.zeros(max(1, n))
        _check(load_library().rtlr_cu_report_get(self.h, what.encode(), out.ctypes.data_as(_D)))
        return out[:n]

    @property
    def phi(self) -> np.ndarray:
        return self.get("phi", self.n)

    def history(self, what: str) -> np.ndarray:
        return self.get(what, self.n_history)

    PHASES = ("sweep", "cgs", "projections", "galerkin_q", "residual_q", "build_C", "verify", "svd", "dsa")

    def phase_work(self) -> dict:
        """Low-rank phases: {name: {"seconds" (None unless profile_phases),
        "bytes" (algorithmic HBM bytes), "flops", "calls"}}."""
        w = self.get("phase_work", 4 * len(self.PHASES)).reshape(-1, 4)
        return {name: {"seconds": None if row[0] < 0 else float(row[0]), "bytes": float(row[1]),
                       "flops": float(row[2]), "calls": int(row[3])} for name, row in zip(self.PHASES, w)}

    def sampled_log(self):
        counts = np.zeros(max(1, self.n_history), dtype=np.int32)
        flat = np.zeros(max(1, self._sampled_total), dtype=np.int32)
        _check(load_library().rtlr_cu_report_sampled(self.h, counts.ctypes.data_as(_I),
                                                     flat.ctypes.data_as(_I)))
        out, k = [], 0
        for c in counts[:self.n_history]:
            out.append([int(v) for v in flat[k:k + c]])
            k += c
        return out

    def __del__(self):
        if getattr(self, "h", None):
            try:
                load_library().rtlr_cu_report_destroy(self.h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self.h = None


def _make_config(L, name, config_text=None, config_path=None):
    cfg = ctypes.c_void_p()
    if config_text is not None:
        _check(L.rtlr_cu_config_parse(config_text.encode(), ctypes.byref(cfg)))
    elif config_path is not None:
        _check(L.rtlr_cu_config_load(os.fsencode(config_path), ctypes.byref(cfg)))
    else:
        _check(L.rtlr_cu_config_create(name.encode(), ctypes.byref(cfg)))
    return cfg


def run(preset: str = None, config_text: str = None, config_path: str = None, mode: str = None, seeds=None,
        out_dir: str = None, device: int = 0, log_flux: bool = False, **overrides):
    """The reference's run / rtlr_bench driver (report.cpp:60-195,
    tools/rtlr_bench.cpp): FR and/or LR per run mode (the config's run.mode,
    or `mode`), compared when both ran, for the config's seed or each of
    `seeds`; writes metrics.csv, history.csv and the flux grids into out_dir
    when given.  Returns (summary text, all drivers converged)."""
    L = load_library()
    cfg = _make_config(L, preset, config_text, config_path)
    try:
        for k, v in overrides.items():
            _check(L.rtlr_cu_config_set(cfg, k.encode(), float(v)))
        if mode is not None:
            _check(L.rtlr_cu_config_set_mode(cfg, mode.encode()))
        sd = np.ascontiguousarray(seeds if seeds is not None else [], dtype=np.int64)
        buf = ctypes.create_string_buffer(1 << 16)
        ok = ctypes.c_int(0)
        _check(L.rtlr_cu_run(cfg, device, sd.ctypes.data_as(_I64) if len(sd) else None, len(sd),
                             os.fsencode(out_dir) if out_dir else None, int(log_flux), buf, len(buf),
                             ctypes.byref(ok)))
    finally:
        L.rtlr_cu_config_destroy(cfg)
    return buf.value.decode(), bool(ok.value)


class Problem:
    """An assembled problem resident on one GPU (AssembledProblem,
    proj/include/rtlr/problem.hpp:98-106).  `name` is a reference preset
    ("homogeneous(1,2)", "pin_cell", ...) or a BASELINE config "C1".."C5";
    keyword overrides use the reference's config keys.  device < 0 assembles
    on the host only (inputs inspectable, no GPU calls)."""

    def __init__(self, name: str = None, device: int = 0, config_text: str = None, fields=None, **overrides):
        """config_text: a reference config file's contents (key = value lines,
        parse_config_text) instead of a preset name.  fields: {"sigma_s" |
        "sigma_a" | "source" | "boundary": f(x, y)} — arbitrary ScalarField
        callables (rtlr_cu_config_set_field), evaluated during assembly."""
        L = load_library()
        cfg = _make_config(L, name, config_text)
        self._fields = []
        try:
            for k, v in overrides.items():
                _check(L.rtlr_cu_config_set(cfg, k.encode(), float(v)))
            for which, f in (fields or {}).items():
                cb = FIELD_FN(lambda _u, x, y, f=f: float(f(x, y)))
                self._fields.append(cb)
                _check(L.rtlr_cu_config_set_field(cfg, which.encode(), cb, None))
            h = ctypes.c_void_p()
            _check(L.rtlr_cu_problem_create(cfg, device, ctypes.byref(h)))
            self.h = h
        finally:
            L.rtlr_cu_config_destroy(cfg)
        info = np.zeros(8, dtype=np.int64)
        _check(L.rtlr_cu_problem_info(self.h, info.ctypes.data_as(_I64)))
        self.nx, self.ny, self.n_theta, self.n_omega_z, self.n, self.n_omega = (int(v) for v in info[:6])
        self.n_unique = int(info[6])
        self.sigma_t_uniform = bool(info[7])
        k, spc = ctypes.c_int(), ctypes.c_int()
        _check(L.rtlr_cu_problem_degree(self.h, ctypes.byref(k), ctypes.byref(spc)))
        self.degree, self.dofs_per_cell = k.value, spc.value  # DG degree K, (K+1)^2
        self.ncell = self.n // self.dofs_per_cell

    # ---- inputs (host copies) ----
    def get(self, what: str) -> np.ndarray:
        s = self.dofs_per_cell
        sizes = {"dirs": 3 * self.n_omega, "weights": self.n_omega, "source": self.n,
                 "sigma_t_blocks": s * s * self.ncell, "sigma_s_blocks": s * s * self.ncell,
                 "sigma_a_blocks": s * s * self.ncell, "sip_bsr": 80 * self.ncell, "stream_blocks": 8 * s * s}
        out = np.zeros(sizes[what])
        _check(load_library().rtlr_cu_problem_get(self.h, what.encode(), out.ctypes.data_as(_D)))
        if what == "dirs":
            return out.reshape(self.n_omega, 3)
        if what.endswith("_blocks") and what != "stream_blocks":
            return out.reshape(self.ncell, s, s).transpose(0, 2, 1).copy()
        if what == "sip_bsr":
            return out.reshape(self.ncell, 5, 4, 4).transpose(0, 1, 3, 2).copy()
        return out

    def set_stream(self, cuda_stream: int):
        _check(load_library().rtlr_cu_problem_set_stream(self.h, ctypes.c_void_p(cuda_stream)))

    def set_comm(self, nranks: int, rank: int, nccl_id: bytes | None):
        """Attach an NCCL communicator: the drivers then shard directions."""
        _check(load_library().rtlr_cu_problem_set_comm(self.h, nranks, rank, nccl_id))

    def set_option(self, key: str, value: float):
        _check(load_library().rtlr_cu_problem_set_option(self.h, key.encode(), float(value)))

    def synchronize(self):
        _check(load_library().rtlr_cu_synchronize(self.h))

    # ---- kernels (host numpy in, host numpy out) ----
    def sweep(self, angles, rhs: np.ndarray) -> np.ndarray:
        """psi[:, k] = sweep(angle k, rhs[:, k] or shared rhs) (sweep.hpp:14-15)."""
        angles = np.ascontiguousarray(np.atleast_1d(angles), dtype=np.int32)
        n = len(angles)
        rhs = np.asfortranarray(rhs, dtype=np.float64)
        stride = 0 if rhs.ndim == 1 else self.n
        psi = np.zeros((self.n, n), order="F")
        _check(load_library().rtlr_cu_sweep(self.h, angles.ctypes.data_as(ctypes.c_void_p), n, _dp(rhs),
                                            stride, _dp(psi), self.n, HOST))
        return psi

    def sweep_dirs(self, omega_xy, rhs: np.ndarray) -> np.ndarray:
        om = np.ascontiguousarray(np.atleast_2d(omega_xy), dtype=np.float64)
        n = om.shape[0]
        rhs = np.asfortranarray(rhs, dtype=np.float64)
        stride = 0 if rhs.ndim == 1 else self.n
        psi = np.zeros((self.n, n), order="F")
        _check(load_library().rtlr_cu_sweep_dirs(self.h, om.ctypes.data_as(_D), n, _dp(rhs), stride,
                                                 _dp(psi), self.n, HOST))
        return psi

    def sweep_device(self, angles_ptr: int, n: int, rhs_ptr: int, rhs_stride: int, psi_ptr: int,
                     psi_stride: int):
        """Device-pointer sweep (torch tensors' data_ptr()); angles on the host."""
        _check(load_library().rtlr_cu_sweep(self.h, ctypes.c_void_p(angles_ptr), n, ctypes.c_void_p(rhs_ptr),
                                            rhs_stride, ctypes.c_void_p(psi_ptr), psi_stride, DEVICE))

    def sweep_async(self, d_angles_ptr: int, n: int, rhs_ptr: int, rhs_stride: int, psi_ptr: int,
                    psi_stride: int):
        """Enqueue a batched sweep on the problem's stream (all device pointers)."""
        _check(load_library().rtlr_cu_sweep_async(self.h, ctypes.c_void_p(d_angles_ptr), n,
                                                  ctypes.c_void_p(rhs_ptr), rhs_stride,
                                                  ctypes.c_void_p(psi_ptr), psi_stride))

    def check(self):
        _check(load_library().rtlr_cu_check(self.h))

    def sweep_host_ptr(self, angles: np.ndarray, rhs_ptr: int, rhs_stride: int, psi_ptr: int,
                       psi_stride: int):
        """Sweep with HOST rhs/psi pointers (e.g. pinned buffers); copies inside the call."""
        angles = np.ascontiguousarray(angles, dtype=np.int32)
        _check(load_library().rtlr_cu_sweep(self.h, angles.ctypes.data_as(ctypes.c_void_p), len(angles),
                                            ctypes.c_void_p(rhs_ptr), rhs_stride, ctypes.c_void_p(psi_ptr),
                                            psi_stride, HOST))

    def c5_fill(self, rhs_ptr: int, n_dirs: int, dir0: int, seed: int):
        _check(load_library().rtlr_cu_c5_fill(self.h, ctypes.c_void_p(rhs_ptr), n_dirs, dir0, seed))

    def apply(self, omx: float, omy: float, v: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros(self.n)
        _check(load_library().rtlr_cu_apply(self.h, omx, omy, _dp(v), _dp(out), HOST))
        return out

    def rhs_core(self, phi: np.ndarray) -> np.ndarray:
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        out = np.zeros(self.n)
        _check(load_library().rtlr_cu_rhs_core(self.h, _dp(phi), _dp(out), HOST))
        return out

    def si_step(self, phi_prev: np.ndarray, want_psi: bool = False):
        phi_prev = np.ascontiguousarray(phi_prev, dtype=np.float64)
        phi_star = np.zeros(self.n)
        psi = np.zeros((self.n, self.n_omega), order="F") if want_psi else None
        _check(load_library().rtlr_cu_si_step(self.h, _dp(phi_prev), _dp(phi_star),
                                              _dp(psi) if want_psi else None, HOST))
        return (phi_star, psi) if want_psi else phi_star

    def dsa_solve(self, rhs: np.ndarray, return_iterations: bool = False):
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        out = np.zeros(self.n)
        it = ctypes.c_int(0)
        _check(load_library().rtlr_cu_dsa_solve(self.h, _dp(rhs), _dp(out), HOST, ctypes.byref(it)))
        return (out, it.value) if return_iterations else out

    def dsa_correct(self, phi_star: np.ndarray, phi_prev: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(phi_star, dtype=np.float64)
        b = np.ascontiguousarray(phi_prev, dtype=np.float64)
        out = np.zeros(self.n)
        _check(load_library().rtlr_cu_dsa_correct(self.h, _dp(a), _dp(b), _dp(out), HOST))
        return out

    def psi_difference(self, psi_full: np.ndarray, X: np.ndarray, S: np.ndarray, V: np.ndarray) -> float:
        """psi_difference (report.cpp:47-58): ||psi_full - X diag(S) V^T||_F on the GPU."""
        r = int(np.asarray(S).size)
        ps = np.asfortranarray(np.reshape(psi_full, (self.n, self.n_omega), order="F"), dtype=np.float64)
        x = np.asfortranarray(np.reshape(X, (self.n, r), order="F"), dtype=np.float64)
        v = np.asfortranarray(np.reshape(V, (self.n_omega, r), order="F"), dtype=np.float64)
        sv = np.ascontiguousarray(S, dtype=np.float64)
        out = ctypes.c_double(0.0)
        _check(load_library().rtlr_cu_psi_difference(self.h, _dp(ps), _dp(x), _dp(sv), _dp(v), r,
                                                      ctypes.byref(out), HOST))
        return out.value

    # ---- drivers ----
    def solve_full_rank(self, **opts) -> Report:
        o = FrOptions()
        _check(load_library().rtlr_cu_problem_fr_options(self.h, ctypes.byref(o)))
        for k, v in opts.items():
            setattr(o, k, v)
        r = ctypes.c_void_p()
        _check(load_library().rtlr_cu_solve_full_rank(self.h, ctypes.byref(o), ctypes.byref(r)))
        return Report(r)

    def solve_low_rank(self, **opts) -> Report:
        o = LrOptions()
        _check(load_library().rtlr_cu_problem_lr_options(self.h, ctypes.byref(o)))
        for k, v in opts.items():
            setattr(o, k, v)
        r = ctypes.c_void_p()
        _check(load_library().rtlr_cu_solve_low_rank(self.h, ctypes.byref(o), ctypes.byref(r)))
        return Report(r)

    def __del__(self):
        if getattr(self, "h", None):
            try:
                load_library().rtlr_cu_problem_destroy(self.h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self.h = None


# ---------------------------------------------------------------- caller-assembled problems
def upload_problem(nx: int, ny: int, dirs, weights, sigma_t_blocks, sigma_s_blocks, source,
                   domain=(0.0, 1.0, 0.0, 1.0), n_theta: int = 0, n_omega_z: int = 0, sigma_a_blocks=None,
                   boundary=None, sip_bsr=None, use_dsa: bool = True, device: int = 0) -> "Problem":
    """rtlr_cu_problem_upload: a Problem from the arrays the reference's
    solvers take (solve_full_rank(ops, quad, bc, source, dsa, opts),
    full_rank.hpp:41-43).  Blocks are (ncell, 4, 4) arrays (row, column);
    dirs (n_omega, 3); boundary (n_omega, N_x) per-angle inflow vectors;
    sip_bsr (ncell, 5, 4, 4) in the order self, west, east, south, north."""
    def blocks(b):  # (ncell, 4, 4) -> ncell x 16 column-major blocks
        b = np.asarray(b, dtype=np.float64)
        return np.ascontiguousarray(b.reshape(-1, 4, 4).transpose(0, 2, 1)).ravel()

    keep = []

    def ptr(a):
        if a is None:
            return None
        a = np.ascontiguousarray(a, dtype=np.float64)
        keep.append(a)
        return a.ctypes.data

    dirs = np.asarray(dirs, dtype=np.float64).reshape(-1, 3)
    d = ProblemDesc()
    d.nx, d.ny = nx, ny
    d.x_min, d.x_max, d.y_min, d.y_max = domain
    d.n_theta, d.n_omega_z, d.n_omega = n_theta, n_omega_z, dirs.shape[0]
    d.dirs, d.weights = ptr(dirs), ptr(weights)
    d.sigma_t_blocks, d.sigma_s_blocks = ptr(blocks(sigma_t_blocks)), ptr(blocks(sigma_s_blocks))
    d.sigma_a_blocks = ptr(None if sigma_a_blocks is None else blocks(sigma_a_blocks))
    d.source = ptr(source)
    d.boundary = ptr(boundary)
    if sip_bsr is not None:
        sip_bsr = np.ascontiguousarray(np.asarray(sip_bsr, dtype=np.float64).reshape(-1, 5, 4, 4)
                                       .transpose(0, 1, 3, 2)).ravel()
    d.sip_bsr = ptr(sip_bsr)
    d.use_dsa = int(bool(use_dsa))
    h = ctypes.c_void_p()
    _check(load_library().rtlr_cu_problem_upload(ctypes.byref(d), device, ctypes.byref(h)))
    return Problem._from_handle(h)


def _problem_from_handle(cls, h):
    self = cls.__new__(cls)
    self.h = h
    self._fields = []
    info = np.zeros(8, dtype=np.int64)
    _check(load_library().rtlr_cu_problem_info(self.h, info.ctypes.data_as(_I64)))
    self.nx, self.ny, self.n_theta, self.n_omega_z, self.n, self.n_omega = (int(v) for v in info[:6])
    self.n_unique = int(info[6])
    self.sigma_t_uniform = bool(info[7])
    self.degree, self.dofs_per_cell = 1, 4  # caller-assembled problems are K = 1
    self.ncell = self.n // 4
    return self


Problem._from_handle = classmethod(_problem_from_handle)


# ---------------------------------------------------------------- low-rank primitives
def lr_params(**kw) -> LrParams:
    """LowRankParams with the reference's defaults (low_rank.hpp:29-36)."""
    o = LrParams()
    load_library().rtlr_cu_lr_params_default(ctypes.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def _ints(a):
    return np.ascontiguousarray(np.atleast_1d(np.asarray(a, dtype=np.int32)))


class SubsampleRng:
    """SubsampleRng (low_rank.hpp:18-27): mt19937_64, masked rejection."""

    def __init__(self, seed: int):
        h = ctypes.c_void_p()
        _check(load_library().rtlr_cu_rng_create(seed, ctypes.byref(h)))
        self.h = h

    def draw_below(self, n: int) -> int:
        out = ctypes.c_uint64(0)
        _check(load_library().rtlr_cu_rng_draw_below(self.h, n, ctypes.byref(out)))
        return out.value

    def sample_without_replacement(self, pool, count: int) -> list:
        pool = _ints(pool) if len(pool) else np.zeros(0, dtype=np.int32)
        out = np.zeros(max(1, min(count, len(pool))), dtype=np.int32)
        n = ctypes.c_int(0)
        _check(load_library().rtlr_cu_rng_sample(self.h, pool.ctypes.data_as(_I), len(pool), count,
                                                 out.ctypes.data_as(_I), ctypes.byref(n)))
        return [int(v) for v in out[:n.value]]

    def __del__(self):
        if getattr(self, "h", None):
            try:
                load_library().rtlr_cu_rng_destroy(self.h)
            except TypeError:
                pass
            self.h = None


class LowRankBasis:
    """LowRankBasis(ops, quad, bc, rhs_core) (low_rank.hpp:42-102) on the
    problem's GPU: mgs_ro_update, update_projections, galerkin_solve,
    residual norms and the projected operators, host numpy in and out."""

    def __init__(self, problem: "Problem", rhs_core, params: LrParams = None):
        self.problem = problem
        rhs = np.ascontiguousarray(rhs_core, dtype=np.float64)
        self.params = params or lr_params()
        h = ctypes.c_void_p()
        _check(load_library().rtlr_cu_lr_basis_create(problem.h, ctypes.byref(self.params), rhs.ctypes.data, HOST,
                                                      ctypes.byref(h)))
        self.h = h

    def _info(self):
        info = np.zeros(4, dtype=np.int64)
        _check(load_library().rtlr_cu_lr_basis_info(self.h, info.ctypes.data_as(_I64)))
        return [int(v) for v in info]

    def rank(self) -> int:
        return self._info()[0]

    def snapshot_count(self) -> int:
        return self._info()[1]

    def _get(self, what, shape):
        out = np.zeros(int(np.prod(shape)) or 1)
        _check(load_library().rtlr_cu_lr_basis_get(self.h, what.encode(), out.ctypes.data, HOST))
        return out[:int(np.prod(shape))].reshape(shape, order="F")

    def basis(self) -> np.ndarray:
        r, _, n, _ = self._info()
        return self._get("basis", (n, r))

    def coefficient_record(self) -> np.ndarray:
        r, m, _, _ = self._info()
        return self._get("record", (r, m))

    def projected(self, which: str) -> np.ndarray:
        """which: dx_minus | dx_plus | dy_minus | dy_plus | sigma_t"""
        r = self.rank()
        return self._get(which, (r, r))

    def prhs(self) -> np.ndarray:
        return self._get("prhs", (self.rank(),))

    def sampled_angles(self) -> list:
        m = self.snapshot_count()
        out = np.zeros(max(1, m), dtype=np.int32)
        _check(load_library().rtlr_cu_lr_basis_sampled(self.h, out.ctypes.data_as(_I)))
        return [int(v) for v in out[:m]]

    def mgs_ro_update(self, snapshots, angles, eps_mgs: float = 1e-10, drop_tol: float = 1e-12) -> bool:
        snaps = np.asfortranarray(np.reshape(snapshots, (self.problem.n, -1), order="F"), dtype=np.float64)
        ang = _ints(angles)
        ro = ctypes.c_int(0)
        _check(load_library().rtlr_cu_lr_mgs_ro_update(self.h, snaps.ctypes.data, ang.ctypes.data_as(_I), len(ang),
                                                       eps_mgs, drop_tol, HOST, ctypes.byref(ro)))
        return bool(ro.value)

    def update_projections(self, reorthogonalized: bool):
        _check(load_library().rtlr_cu_lr_update_projections(self.h, int(bool(reorthogonalized))))

    def galerkin_solve(self, angles) -> np.ndarray:
        """Reduced solutions, one column per angle (rank x m)."""
        ang = _ints(angles)
        r = self.rank()
        out = np.zeros((r, len(ang)), order="F")
        _check(load_library().rtlr_cu_lr_galerkin_solve(self.h, ang.ctypes.data_as(_I), len(ang), out.ctypes.data,
                                                        HOST))
        return out

    def residual_norms(self, angles, coeffs) -> np.ndarray:
        ang = _ints(angles)
        c = np.asfortranarray(np.reshape(coeffs, (self.rank(), len(ang)), order="F"), dtype=np.float64)
        out = np.zeros(len(ang))
        _check(load_library().rtlr_cu_lr_residual_norms(self.h, ang.ctypes.data_as(_I), len(ang), c.ctypes.data,
                                                        out.ctypes.data, HOST))
        return out

    def build_full_coefficients(self, candidates=(), candidate_solutions=None):
        """(C, phi): C rank x N_Omega (record / candidates / Galerkin solves), phi = X (C w)."""
        cand = _ints(candidates) if len(candidates) else np.zeros(0, dtype=np.int32)
        r = self.rank()
        cs = None
        if len(cand):
            cs = np.asfortranarray(np.reshape(candidate_solutions, (r, len(cand)), order="F"), dtype=np.float64)
        C = np.zeros((r, self.problem.n_omega), order="F")
        phi = np.zeros(self.problem.n)
        _check(load_library().rtlr_cu_lr_build_coefficients(
            self.h, cand.ctypes.data_as(_I), len(cand), None if cs is None else cs.ctypes.data, C.ctypes.data,
            phi.ctypes.data, HOST))
        return C, phi

    def __del__(self):
        if getattr(self, "h", None):
            try:
                load_library().rtlr_cu_lr_basis_destroy(self.h)
            except TypeError:
                pass
            self.h = None


def greedy_subsample(basis: LowRankBasis, sampled_mask, p: int, q: int, rng: SubsampleRng) -> dict:
    """greedy_subsample (low_rank.hpp:114-116) -> SubsampleOutcome fields."""
    mask = np.ascontiguousarray(np.asarray(sampled_mask, dtype=np.uint8))
    r = basis.rank()
    sel = np.zeros(max(1, p), dtype=np.int32)
    cand = np.zeros(max(1, q), dtype=np.int32)
    ns, nc = ctypes.c_int(0), ctypes.c_int(0)
    mx = ctypes.c_double(0.0)
    sols = np.zeros((r, q), order="F")
    norms = np.zeros(q)
    _check(load_library().rtlr_cu_lr_greedy_subsample(
        basis.h, mask.tobytes(), p, q, rng.h, sel.ctypes.data_as(_I), ctypes.byref(ns), ctypes.byref(mx),
        cand.ctypes.data_as(_I), ctypes.byref(nc), sols.ctypes.data, norms.ctypes.data, HOST))
    m = nc.value
    return {"selected": [int(v) for v in sel[:ns.value]], "max_residual": mx.value,
            "candidates": [int(v) for v in cand[:m]], "candidate_solutions": sols[:, :m],
            "residual_norms": norms[:m]}


def truncation_rank(s, eps_svd: float) -> int:
    """truncation_rank (low_rank.cpp:254-266)."""
    s = np.ascontiguousarray(s, dtype=np.float64)
    out = ctypes.c_int(0)
    _check(load_library().rtlr_cu_truncation_rank(s.ctypes.data_as(_D), len(s), eps_svd, ctypes.byref(out)))
    return out.value


def truncate_factors(problem: "Problem", C, X, eps_svd: float):
    """truncate_factors(C, X, eps_svd) (low_rank.cpp:268-277) on the GPU ->
    (X_out, S, V) with X_out N_x x r', V N_Omega x r'."""
    C = np.asfortranarray(C, dtype=np.float64)
    X = np.asfortranarray(X, dtype=np.float64)
    r = C.shape[0]
    n, nom = X.shape[0], C.shape[1]
    Xo = np.zeros((n, r), order="F")
    S = np.zeros(r)
    Vo = np.zeros((nom, r), order="F")
    ro = ctypes.c_int(0)
    _check(load_library().rtlr_cu_truncate_factors(problem.h, C.ctypes.data, X.ctypes.data, r, eps_svd, HOST,
                                                   ctypes.byref(ro), Xo.ctypes.data, S.ctypes.data, Vo.ctypes.data))
    k = ro.value
    return Xo[:, :k].copy(order="F"), S[:k].copy(), Vo[:, :k].copy(order="F")


def svd_values(problem: "Problem", C, X) -> np.ndarray:
    """The per-outer-iteration singular values of C (low_rank.cpp:457)."""
    C = np.asfortranarray(C, dtype=np.float64)
    X = np.asfortranarray(X, dtype=np.float64)
    r = C.shape[0]
    S = np.zeros(r)
    ro = ctypes.c_int(0)
    _check(load_library().rtlr_cu_truncate_factors(problem.h, C.ctypes.data, X.ctypes.data, r, 0.0, HOST,
                                                   ctypes.byref(ro), None, S.ctypes.data, None))
    return S[:ro.value]


class InnerLoopResult:
    """InnerLoopResult (low_rank.hpp:125-136) of low_rank_si."""

    def __init__(self, h, problem):
        self.h = h
        self.problem = problem  # the engine borrows the problem: keep it alive
        info = np.zeros(8, dtype=np.int64)
        _check(load_library().rtlr_cu_inner_info(h, info.ctypes.data_as(_I64)))
        (self.iterations, self.rank, self.sampled_count, self.reorthogonalizations, self.verification_rejections,
         ex, self.n, self.n_omega) = (int(v) for v in info)
        self.exhausted_all_angles = bool(ex)

    def _get(self, what, shape):
        out = np.zeros(int(np.prod(shape)) or 1)
        _check(load_library().rtlr_cu_inner_get(self.h, what.encode(), out.ctypes.data, HOST))
        return out[:int(np.prod(shape))].reshape(shape, order="F")

    @property
    def phi_star(self):
        return self._get("phi_star", (self.n,))

    @property
    def coefficients(self):
        return self._get("coefficients", (self.rank, self.n_omega))

    @property
    def basis(self):
        return self._get("basis", (self.n, self.rank))

    @property
    def sampled_order(self):
        out = np.zeros(max(1, self.sampled_count), dtype=np.int32)
        _check(load_library().rtlr_cu_inner_sampled(self.h, out.ctypes.data_as(_I)))
        return [int(v) for v in out[:self.sampled_count]]

    def __del__(self):
        if getattr(self, "h", None):
            try:
                load_library().rtlr_cu_inner_destroy(self.h)
            except TypeError:
                pass
            self.h = None


def low_rank_si(problem: "Problem", phi_prev, params: LrParams, rng: SubsampleRng) -> InnerLoopResult:
    """low_rank_si(ops, quad, bc, source, phi_prev, params, rng) (low_rank.hpp:141-144)."""
    phi = np.ascontiguousarray(phi_prev, dtype=np.float64)
    h = ctypes.c_void_p()
    _check(load_library().rtlr_cu_low_rank_si(problem.h, phi.ctypes.data, ctypes.byref(params), rng.h, HOST,
                                              ctypes.byref(h)))
    return InnerLoopResult(h, problem)
