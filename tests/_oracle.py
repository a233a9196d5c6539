"""ctypes binding of the CPU oracle (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE ONLY: the oracle is the checker, never the product.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs use it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB_PATH = os.path.join(ORACLE_DIR, "_build", "liboracle.so")

_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int)
_LL = ctypes.POINTER(ctypes.c_longlong)
# ScalarField callback: double f(void* user, double x, double y)
FIELD_FN = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_void_p, ctypes.c_double, ctypes.c_double)


def build() -> None:
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_last_error.restype = ctypes.c_char_p
        L.oracle_problem_new.restype = ctypes.c_void_p
        L.oracle_problem_new.argtypes = [ctypes.c_char_p]
        L.oracle_problem_free.argtypes = [ctypes.c_void_p]
        L.oracle_problem_set.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_double]
        L.oracle_problem_assemble.argtypes = [ctypes.c_void_p]
        L.oracle_problem_set_field.argtypes = [ctypes.c_void_p, ctypes.c_char_p, FIELD_FN, ctypes.c_void_p]
        L.oracle_problem_info.argtypes = [ctypes.c_void_p, _LL]
        L.oracle_problem_get.argtypes = [ctypes.c_void_p, ctypes.c_char_p, _D]
        L.oracle_problem_nnz.restype = ctypes.c_longlong
        L.oracle_problem_nnz.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
        L.oracle_problem_csr.argtypes = [ctypes.c_void_p, ctypes.c_char_p, _I, _I, _D]
        L.oracle_sweep.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, _D, _D]
        L.oracle_apply.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, _D, _D]
        L.oracle_rhs_core.argtypes = [ctypes.c_void_p, _D, _D]
        L.oracle_boundary_vector.argtypes = [ctypes.c_void_p, ctypes.c_int, _D]
        L.oracle_boundary_vector_dir.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, _D]
        L.oracle_dsa_solve.argtypes = [ctypes.c_void_p, _D, _D]
        L.oracle_dsa_correct.argtypes = [ctypes.c_void_p, _D, _D, _D]
        L.oracle_si_step.argtypes = [ctypes.c_void_p, _D, _D, _D]
        L.oracle_solve.restype = ctypes.c_void_p
        L.oracle_solve.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
        L.oracle_result_free.argtypes = [ctypes.c_void_p]
        L.oracle_result_info.argtypes = [ctypes.c_void_p, _LL]
        L.oracle_result_get.argtypes = [ctypes.c_void_p, ctypes.c_char_p, _D]
        L.oracle_result_sampled.argtypes = [ctypes.c_void_p, _I, _I]
        L.oracle_psi_difference.restype = ctypes.c_double
        L.oracle_psi_difference.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_c5_uniform.restype = ctypes.c_double
        L.oracle_c5_uniform.argtypes = [ctypes.c_ulonglong, ctypes.c_ulonglong]
        L.oracle_c5_fill.argtypes = [ctypes.c_ulonglong, ctypes.c_longlong, ctypes.c_longlong,
                                     ctypes.c_longlong, _D]
        L.oracle_truncation_rank.argtypes = [_D, ctypes.c_int, ctypes.c_double]
        L.oracle_svd_values.argtypes = [_D, ctypes.c_int, ctypes.c_int, _D]
        L.oracle_gauss_legendre.argtypes = [ctypes.c_int, _D, _D]
        L.oracle_quadrature.argtypes = [ctypes.c_int, ctypes.c_int, _D, _D]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_D)


class OracleError(RuntimeError):
    pass


def _check(rc):
    if rc != 0:
        raise OracleError(lib().oracle_last_error().decode())


def gauss_legendre(n):
    x = np.zeros(n)
    w = np.zeros(n)
    _check(lib().oracle_gauss_legendre(n, _p(x), _p(w)))
    return x, w


def quadrature(n_theta, n_z):
    n = n_theta * n_z
    d = np.zeros((n, 3))
    w = np.zeros(n)
    _check(lib().oracle_quadrature(n_theta, n_z, _p(d), _p(w)))
    return d, w


def truncation_rank(s, eps):
    s = np.ascontiguousarray(s, dtype=np.float64)
    return lib().oracle_truncation_rank(_p(s), len(s), eps)


def svd_values(a):
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    s = np.zeros(min(m, n))
    _check(lib().oracle_svd_values(_p(a), m, n, _p(s)))
    return s


def c5_uniform(seed, counter):
    return lib().oracle_c5_uniform(seed, counter)


def c5_fill(seed, dir0, ndirs, ndof):
    out = np.zeros((ndirs, ndof))
    lib().oracle_c5_fill(seed, dir0, ndirs, ndof, _p(out))
    return out


class Result:
    def __init__(self, h):
        self.h = h
        info = np.zeros(8, dtype=np.int64)
        _check(lib().oracle_result_info(h, info.ctypes.data_as(_LL)))
        self.iterations = int(info[0])
        self.converged = bool(info[1])
        self.n_history = int(info[2])
        self.has_psi = bool(info[3])
        self.factor_rank = int(info[4])
        self.psi_dofs = int(info[6])
        self._sampled_total = int(info[5])

    def get(self, what, n):
        out = np.zeros(n)
        _check(lib().oracle_result_get(self.h, what.encode(), _p(out)))
        return out

    def history(self, what):
        return self.get(what, self.n_history)

    def sampled_log(self):
        counts = np.zeros(self.n_history, dtype=np.int32)
        flat = np.zeros(max(1, self._sampled_total), dtype=np.int32)
        _check(lib().oracle_result_sampled(self.h, counts.ctypes.data_as(_I), flat.ctypes.data_as(_I)))
        out, k = [], 0
        for c in counts:
            out.append([int(v) for v in flat[k:k + c]])
            k += c
        return out

    def __del__(self):
        if self.h:
            lib().oracle_result_free(self.h)
            self.h = None


class Problem:
    """An assembled oracle problem (preset name or C1..C5 plus overrides)."""

    def __init__(self, name: str, assemble: bool = True, fields=None, **overrides):
        """fields: {"sigma_s" | "sigma_a" | "source" | "boundary": f(x, y)}
        (arbitrary ScalarField callables, as the reference's assembly takes)."""
        self.h = lib().oracle_problem_new(name.encode())
        if not self.h:
            raise OracleError(lib().oracle_last_error().decode())
        for k, v in overrides.items():
            _check(lib().oracle_problem_set(self.h, k.encode(), float(v)))
        self._fields = []
        for which, f in (fields or {}).items():
            cb = FIELD_FN(lambda _u, x, y, f=f: float(f(x, y)))
            self._fields.append(cb)
            _check(lib().oracle_problem_set_field(self.h, which.encode(), cb, None))
        if assemble:
            self.assemble()

    def set(self, key, value):
        _check(lib().oracle_problem_set(self.h, key.encode(), float(value)))

    def assemble(self):
        _check(lib().oracle_problem_assemble(self.h))
        info = np.zeros(8, dtype=np.int64)
        _check(lib().oracle_problem_info(self.h, info.ctypes.data_as(_LL)))
        self.nx, self.ny, self.n_theta, self.n_omega_z = (int(v) for v in info[:4])
        self.n = int(info[4])
        self.n_omega = int(info[5])
        self.degree = int(info[6])
        self.s = (self.degree + 1) ** 2

    def get(self, what):
        sizes = {
            "source": self.n,
            "dirs": 3 * self.n_omega,
            "weights": self.n_omega,
            "sigma_t_blocks": self.n * self.s,
            "sigma_s_blocks": self.n * self.s,
            "sigma_a_blocks": self.n * self.s,
            "stream_blocks": 8 * self.s * self.s,
        }
        out = np.zeros(sizes[what])
        _check(lib().oracle_problem_get(self.h, what.encode(), _p(out)))
        if what == "dirs":
            out = out.reshape(self.n_omega, 3)
        elif what.endswith("_blocks") and what != "stream_blocks":
            # per-cell s x s blocks, column-major inside each block
            out = out.reshape(-1, self.s, self.s).transpose(0, 2, 1).copy()
        return out

    def csr(self, which):
        import scipy.sparse as sp
        nnz = lib().oracle_problem_nnz(self.h, which.encode())
        if nnz < 0:
            raise OracleError(lib().oracle_last_error().decode())
        rp = np.zeros(self.n + 1, dtype=np.int32)
        ci = np.zeros(nnz, dtype=np.int32)
        v = np.zeros(nnz)
        _check(lib().oracle_problem_csr(self.h, which.encode(), rp.ctypes.data_as(_I), ci.ctypes.data_as(_I), _p(v)))
        return sp.csr_matrix((v, ci, rp), shape=(self.n, self.n))

    def sweep(self, omx, omy, rhs):
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        out = np.zeros(self.n)
        _check(lib().oracle_sweep(self.h, omx, omy, _p(rhs), _p(out)))
        return out

    def apply(self, omx, omy, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros(self.n)
        _check(lib().oracle_apply(self.h, omx, omy, _p(v), _p(out)))
        return out

    def rhs_core(self, phi):
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        out = np.zeros(self.n)
        _check(lib().oracle_rhs_core(self.h, _p(phi), _p(out)))
        return out

    def boundary_vector(self, omx, omy):
        out = np.zeros(self.n)
        _check(lib().oracle_boundary_vector_dir(self.h, omx, omy, _p(out)))
        return out

    def dsa_solve(self, rhs):
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        out = np.zeros(self.n)
        _check(lib().oracle_dsa_solve(self.h, _p(rhs), _p(out)))
        return out

    def dsa_correct(self, phi_star, phi_prev):
        a = np.ascontiguousarray(phi_star, dtype=np.float64)
        b = np.ascontiguousarray(phi_prev, dtype=np.float64)
        out = np.zeros(self.n)
        _check(lib().oracle_dsa_correct(self.h, _p(a), _p(b), _p(out)))
        return out

    def si_step(self, phi_prev, want_psi=False):
        phi_prev = np.ascontiguousarray(phi_prev, dtype=np.float64)
        phi_star = np.zeros(self.n)
        psi = np.zeros((self.n_omega, self.n)) if want_psi else None
        _check(lib().oracle_si_step(self.h, _p(phi_prev), _p(phi_star), _p(psi) if want_psi else None))
        return (phi_star, psi.T) if want_psi else phi_star

    def solve(self, method):
        h = lib().oracle_solve(self.h, method.encode())
        if not h:
            raise OracleError(lib().oracle_last_error().decode())
        return Result(h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_problem_free(self.h)
            self.h = None
