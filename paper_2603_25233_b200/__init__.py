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
    "rtlr_cu_problem_get", "rtlr_cu_problem_set_stream", "rtlr_cu_problem_set_option",
    "rtlr_cu_synchronize", "rtlr_cu_sweep", "rtlr_cu_sweep_dirs", "rtlr_cu_apply",
    "rtlr_cu_rhs_core", "rtlr_cu_si_step", "rtlr_cu_dsa_solve", "rtlr_cu_dsa_correct",
    "rtlr_cu_c5_fill", "rtlr_cu_fr_options_default", "rtlr_cu_lr_options_default",
    "rtlr_cu_solve_full_rank", "rtlr_cu_solve_low_rank", "rtlr_cu_report_info",
    "rtlr_cu_report_get", "rtlr_cu_report_sampled", "rtlr_cu_report_destroy",
    "rtlr_cu_partition_angles", "rtlr_cu_problem_fr_options", "rtlr_cu_problem_lr_options",
    "rtlr_cu_sweep_async", "rtlr_cu_check", "rtlr_cu_nccl_unique_id", "rtlr_cu_problem_set_comm",
    "rtlr_cu_shard_block", "rtlr_cu_dense_qr", "rtlr_cu_psi_difference",
    "rtlr_cu_config_parse", "rtlr_cu_config_load", "rtlr_cu_config_set_mode", "rtlr_cu_run",
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
    L.rtlr_cu_dense_qr.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p]
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
        self.ncell = self.n // 4

    # ---- inputs (host copies) ----
    def get(self, what: str) -> np.ndarray:
        sizes = {"dirs": 3 * self.n_omega, "weights": self.n_omega, "source": self.n,
                 "sigma_t_blocks": 16 * self.ncell, "sigma_s_blocks": 16 * self.ncell,
                 "sigma_a_blocks": 16 * self.ncell, "sip_bsr": 80 * self.ncell, "stream_blocks": 128}
        out = np.zeros(sizes[what])
        _check(load_library().rtlr_cu_problem_get(self.h, what.encode(), out.ctypes.data_as(_D)))
        if what == "dirs":
            return out.reshape(self.n_omega, 3)
        if what.endswith("_blocks") and what != "stream_blocks":
            return out.reshape(self.ncell, 4, 4).transpose(0, 2, 1).copy()
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
