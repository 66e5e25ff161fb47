"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU checkers.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs import this module, and only as the checker.  The
product package (paper_2407_11349_b200) never imports it.

Two libraries:
  * liboracle.so        — oracle/hawkes_oracle.c, the C restatement of the
                          reference's hot path (+ long-double gradient).
  * _ref/libhawkes_ref.so — the reference's own headers compiled unmodified
                          (oracle/ref_shim.cpp; built where /root/reference
                          exists and shipped as a binary).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_sz = C.c_size_t


def _params(p) -> np.ndarray:
    """(mu0, tau_t, xi0, sigma_x, sigma_t, area) from a dict/sequence/object."""
    if isinstance(p, dict):
        v = [p["mu0"], p["tau_t"], p["xi0"], p["sigma_x"], p["sigma_t"], p["area"]]
    elif hasattr(p, "mu0"):
        v = [p.mu0, p.tau_t, p.xi0, p.sigma_x, p.sigma_t, p.area]
    else:
        v = list(p)[:6]
    return np.ascontiguousarray(v, dtype=np.float64)


def _arr(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    """The C restatement (always available once `make -C oracle` ran)."""

    def __init__(self, path: Path | None = None):
        path = path or HERE / "liboracle.so"
        if not path.exists():
            raise FileNotFoundError(f"{path} missing; run `make -C oracle`")
        L = C.CDLL(str(path))
        L.orc_log_likelihood.argtypes = [_dp, _dp, _dp, _dp, _sz, _dp, C.c_int, _sz, C.POINTER(C.c_double)]
        L.orc_naive_log_likelihood.argtypes = [_dp, _dp, _dp, _dp, _sz, _dp, C.c_int, C.POINTER(C.c_double)]
        L.orc_rows_ld.argtypes = [_dp, _dp, _dp, _dp, _sz, _dp, C.c_int, _up, _sz, _sz, _dp, C.c_void_p]
        L.orc_ll_grad.argtypes = [_dp, _dp, _dp, _dp, _sz, _dp, C.c_int, _sz, C.POINTER(C.c_double), _dp]
        L.orc_grad_scale.argtypes = [_dp, _dp, _dp, _dp, _sz, _dp, C.c_int, _sz, C.POINTER(C.c_double), _dp]
        L.orc_ll_grad_dbl.argtypes = [_dp, _dp, _dp, _dp, _sz, _dp, C.c_int, _sz, C.POINTER(C.c_double),
                                      _dp, _dp]
        L.orc_rows_lanes.argtypes = [_dp, _dp, _dp, _dp, _sz, _dp, C.c_int, _up, _sz, _sz, _dp]
        L.orc_integral_term.argtypes = [_dp, C.c_double, C.c_double]
        L.orc_integral_term.restype = C.c_double
        L.orc_pair_rate.argtypes = [_dp, C.c_int, _dp, _dp]
        L.orc_pair_rate.restype = C.c_double
        L.orc_gaussian_pdf.argtypes = [C.c_double]
        L.orc_gaussian_pdf.restype = C.c_double
        L.orc_gaussian_cdf.argtypes = [C.c_double]
        L.orc_gaussian_cdf.restype = C.c_double
        self.L = L

    @staticmethod
    def _cat(cat):
        t, x, y, d = (_arr(a) for a in cat)
        return t, x, y, d, len(t)

    def log_likelihood(self, cat, p, variant: int, workers: int = 1) -> float:
        t, x, y, d, n = self._cat(cat)
        out = C.c_double()
        if self.L.orc_log_likelihood(t, x, y, d, n, _params(p), variant, workers, C.byref(out)):
            raise ValueError("orc_log_likelihood: invalid arguments")
        return out.value

    def naive_log_likelihood(self, cat, p, variant: int) -> float:
        t, x, y, d, n = self._cat(cat)
        out = C.c_double()
        if self.L.orc_naive_log_likelihood(t, x, y, d, n, _params(p), variant, C.byref(out)):
            raise ValueError("orc_naive_log_likelihood: invalid arguments")
        return out.value

    def ll_grad(self, cat, p, variant: int, threads: int = 0):
        t, x, y, d, n = self._cat(cat)
        out = C.c_double()
        g = np.zeros(5)
        if self.L.orc_ll_grad(t, x, y, d, n, _params(p), variant, threads or os.cpu_count() or 1,
                              C.byref(out), g):
            raise ValueError("orc_ll_grad: invalid arguments")
        return out.value, g

    def grad_scale(self, cat, p, variant: int, threads: int = 0):
        t, x, y, d, n = self._cat(cat)
        out = C.c_double()
        g = np.zeros(5)
        if self.L.orc_grad_scale(t, x, y, d, n, _params(p), variant, threads or os.cpu_count() or 1,
                                 C.byref(out), g):
            raise ValueError("orc_grad_scale: invalid arguments")
        return out.value, g

    def ll_grad_dbl(self, cat, p, variant: int, threads: int = 0):
        """Double-precision LL, gradient and conditioning scale (sum_n
        |d ell_n / d theta|) with compensated row sums: the checker for
        catalogs too large for the long-double path (N = 1e6)."""
        t, x, y, d, n = self._cat(cat)
        out = C.c_double()
        g, sc = np.zeros(5), np.zeros(5)
        if self.L.orc_ll_grad_dbl(t, x, y, d, n, _params(p), variant, threads or os.cpu_count() or 1,
                                  C.byref(out), g, sc):
            raise ValueError("orc_ll_grad_dbl: invalid arguments")
        return out.value, g, sc

    def rows_ld(self, cat, p, variant: int, rows, threads: int = 0, grad: bool = True):
        t, x, y, d, n = self._cat(cat)
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        ell = np.zeros(len(rows))
        g = np.zeros((len(rows), 5)) if grad else None
        rc = self.L.orc_rows_ld(t, x, y, d, n, _params(p), variant, rows, len(rows),
                                threads or os.cpu_count() or 1, ell,
                                g.ctypes.data_as(C.c_void_p) if grad else None)
        if rc:
            raise ValueError("orc_rows_ld: invalid arguments")
        return (ell, g) if grad else ell

    def rows_lanes(self, cat, p, variant: int, rows, threads: int = 0) -> np.ndarray:
        """The lane evaluator (reference algorithm, double) on a row list."""
        t, x, y, d, n = self._cat(cat)
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        out = np.zeros(len(rows))
        if self.L.orc_rows_lanes(t, x, y, d, n, _params(p), variant, rows, len(rows),
                                 threads or os.cpu_count() or 1, out):
            raise ValueError("orc_rows_lanes: invalid arguments")
        return out

    def integral_term(self, p, t_n, t_end) -> float:
        return self.L.orc_integral_term(_params(p), t_n, t_end)

    def pair_rate(self, p, variant, source, target) -> float:
        return self.L.orc_pair_rate(_params(p), variant, _arr(source), _arr(target))


def _has_avx512() -> bool:
    try:
        return " avx512f " in (" " + Path("/proc/cpuinfo").read_text().replace("\n", " ") + " ")
    except OSError:
        return False


def ref_available() -> bool:
    return (HERE / "_ref" / "libhawkes_ref.so").exists()


class Reference:
    """The reference's own CPU path (oracle/_ref, compiled from the unmodified
    reference headers)."""

    def __init__(self):
        name = "libhawkes_ref.so" if _has_avx512() else "libhawkes_ref_v3.so"
        path = HERE / "_ref" / name
        if not path.exists():
            raise FileNotFoundError(f"{path} missing; run `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(str(path))
        L.ref_last_error.restype = C.c_char_p
        L.ref_benchmark_catalog.argtypes = [_sz, C.c_uint64, _dp, _dp, _dp, _dp]
        L.ref_log_likelihood.argtypes = [_dp, _dp, _dp, _dp, _sz, _dp, C.c_int, _sz, C.c_int, C.POINTER(C.c_double)]
        L.ref_naive_log_likelihood.argtypes = [_dp, _dp, _dp, _dp, _sz, _dp, C.c_int, C.POINTER(C.c_double)]
        L.ref_event_contribution.argtypes = [_dp, _dp, _dp, _dp, _sz, _dp, C.c_int, _sz, C.POINTER(C.c_double)]
        L.ref_rows.argtypes = [_dp, _dp, _dp, _dp, _sz, _dp, C.c_int, _up, _sz, _sz, _dp]
        L.ref_pair_rate.argtypes = [_dp, C.c_int, _dp, _dp, C.POINTER(C.c_double)]
        L.ref_integral_term.argtypes = [_dp, C.c_double, C.c_double, C.POINTER(C.c_double)]
        L.ref_gaussian_pdf.argtypes = [C.c_double]
        L.ref_gaussian_pdf.restype = C.c_double
        L.ref_gaussian_cdf.argtypes = [C.c_double]
        L.ref_gaussian_cdf.restype = C.c_double
        L.ref_partition.argtypes = [_sz, _sz, np.ctypeslib.ndpointer(dtype=np.uintp, flags="C_CONTIGUOUS")]
        L.ref_workspace_script.argtypes = [_dp, _dp, _dp, _dp, _sz, C.c_int, _sz,
                                           np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS"),
                                           _dp, _sz, _dp]
        L.ref_county_densities.argtypes = [C.c_int, C.c_uint64, _dp]
        self.L = L
        self.path = path

    def _check(self, rc):
        if rc:
            msg = self.L.ref_last_error().decode()
            raise {1: ValueError, 2: IndexError}.get(rc, RuntimeError)(msg)

    def benchmark_catalog(self, n: int, seed: int = 42):
        t, x, y, d = (np.zeros(n) for _ in range(4))
        self._check(self.L.ref_benchmark_catalog(n, seed, t, x, y, d))
        return t, x, y, d

    def county_densities(self, grid: int = 60, seed: int = 1) -> np.ndarray:
        out = np.zeros(grid * grid)
        self._check(self.L.ref_county_densities(grid, seed, out))
        return out

    def log_likelihood(self, cat, p, variant: int, workers: int = 1, single: bool = False) -> float:
        t, x, y, d = (_arr(a) for a in cat)
        out = C.c_double()
        self._check(self.L.ref_log_likelihood(t, x, y, d, len(t), _params(p), variant, workers,
                                               int(single), C.byref(out)))
        return out.value

    def naive_log_likelihood(self, cat, p, variant: int) -> float:
        t, x, y, d = (_arr(a) for a in cat)
        out = C.c_double()
        self._check(self.L.ref_naive_log_likelihood(t, x, y, d, len(t), _params(p), variant, C.byref(out)))
        return out.value

    def event_contribution(self, cat, p, variant: int, row: int) -> float:
        t, x, y, d = (_arr(a) for a in cat)
        out = C.c_double()
        self._check(self.L.ref_event_contribution(t, x, y, d, len(t), _params(p), variant, row, C.byref(out)))
        return out.value

    def rows(self, cat, p, variant: int, rows, threads: int = 0) -> np.ndarray:
        t, x, y, d = (_arr(a) for a in cat)
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        out = np.zeros(len(rows))
        self._check(self.L.ref_rows(t, x, y, d, len(t), _params(p), variant, rows, len(rows),
                                    threads or os.cpu_count() or 1, out))
        return out

    def pair_rate(self, p, variant, source, target) -> float:
        out = C.c_double()
        self._check(self.L.ref_pair_rate(_params(p), variant, _arr(source), _arr(target), C.byref(out)))
        return out.value

    def integral_term(self, p, t_n, t_end) -> float:
        out = C.c_double()
        self._check(self.L.ref_integral_term(_params(p), t_n, t_end, C.byref(out)))
        return out.value

    def partition(self, n: int, g: int) -> np.ndarray:
        b = np.zeros(g + 1, dtype=np.uintp)
        self._check(self.L.ref_partition(n, g, b))
        return b

    def workspace_script(self, cat, variant: int, workers: int, ops, params_seq) -> np.ndarray:
        t, x, y, d = (_arr(a) for a in cat)
        ops = np.ascontiguousarray(ops, dtype=np.int32)
        ps = np.ascontiguousarray(np.concatenate([_params(p) for p in params_seq]), dtype=np.float64)
        out = np.zeros(len(ops))
        self._check(self.L.ref_workspace_script(t, x, y, d, len(t), variant, workers, ops, ps, len(ops), out))
        return out


def county_index(x, y, grid: int = 60) -> np.ndarray:
    """County of each event in BASELINE config 5's fixture:
    grid x grid squares over [-5, 5]^2 in row-major order, the square
    containing (x, y), clamped to the grid (tools/cpp/cut_posterior_bench.cpp
    uses the same arithmetic: int((lon + 5) / (10 / grid)))."""
    cell = 10.0 / grid
    gx = np.minimum(((np.asarray(x) + 5.0) / cell).astype(np.int64), grid - 1)
    gy = np.minimum(((np.asarray(y) + 5.0) / cell).astype(np.int64), grid - 1)
    return gx + grid * gy
