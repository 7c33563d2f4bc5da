"""ctypes binding of the C table-analysis oracle (oracle/lscat_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "lscat_oracle.c")

COUNTERS = [
    "n_rows", "n_ok", "n_nan", "n_invalid",
    "n_groups", "n_defined", "n_all_nan", "n_complete", "n_incomplete",
    "n_largest_missing", "n_ratio_defined",
    "n_largest_is_best", "n_largest_strictly_slower", "n_gain_gt", "n_perf_lt", "n_perf_band",
    "perf_fx_hi", "perf_fx_lo", "gain_fx_hi", "gain_fx_lo",
]


OMP_LIB_PATH = os.path.join(HERE, "liboracle_omp.so")
OMP_SRC = os.path.join(HERE, "lscat_oracle_omp.c")


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (-O2, no FMA contraction, no fast-math), and its
    all-cores variant (the same oracle over group-aligned chunks, OpenMP; baseline timing)."""
    deps = [SRC, OMP_SRC, os.path.join(HERE, "oracle.h")]
    flags = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(d) for d in deps):
        subprocess.check_call(["gcc"] + flags + ["-o", LIB_PATH, SRC, "-lm"])
    if force or not os.path.exists(OMP_LIB_PATH) or os.path.getmtime(OMP_LIB_PATH) < max(
            os.path.getmtime(d) for d in deps):
        subprocess.check_call(["gcc"] + flags + ["-fopenmp", "-o", OMP_LIB_PATH, SRC, OMP_SRC,
                                                 "-lm"])
    return LIB_PATH


class _Table(C.Structure):
    _fields_ = [("runtime_ms", C.c_void_p), ("block_id", C.c_void_p), ("n_rows", C.c_uint64),
                ("group_offset", C.c_void_p), ("n_groups", C.c_uint64),
                ("rows_per_group", C.c_uint32), ("group_matrix", C.c_void_p),
                ("first_group", C.c_uint64)]


class _Opts(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in (
        "n_blocks", "largest_block_id", "n_matrices", "nan_policy", "bins_per_unit", "gain_cap",
        "gain_gt_num", "gain_gt_den", "perf_lt_num", "perf_lt_den", "band_lo_num",
        "band_lo_den")]


class _Result(C.Structure):
    _fields_ = [("counters", C.c_uint64 * len(COUNTERS)), ("perf_hist", C.c_void_p),
                ("gain_hist", C.c_void_p), ("best_block_hist", C.c_void_p),
                ("profile_sum", C.c_void_p), ("profile_count", C.c_void_p)]


class _GroupOut(C.Structure):
    _fields_ = [("best_block", C.c_void_p), ("best_runtime", C.c_void_p), ("perf", C.c_void_p),
                ("gain", C.c_void_p), ("flags", C.c_void_p)]


ROLLUP = ["n_kernels", "n_kernels_not_best", "n_kernels_perf_lt", "n_kernels_perf_band",
          "kernel_mean_fx_hi", "kernel_mean_fx_lo"]


class _Rollup(C.Structure):
    _fields_ = [("counters", C.c_uint64 * len(ROLLUP)), ("perf_hist", C.c_void_p)]


class _Derived(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "frac_nonnan", "frac_largest_not_best", "frac_gain_gt", "frac_perf_lt",
        "frac_perf_band", "mean_perf", "mean_gain")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.oracle_reduce_table.argtypes = [C.POINTER(_Table), C.POINTER(_Opts),
                                             C.POINTER(_Result), C.POINTER(_GroupOut)]
        _lib.oracle_reduce_table.restype = C.c_int
        _lib.oracle_finalize.argtypes = [C.POINTER(_Result), C.POINTER(_Derived)]
        _lib.oracle_finalize.restype = None
        _lib.oracle_kernel_rollup.argtypes = [C.POINTER(_Table), C.c_void_p, C.POINTER(_Opts),
                                              C.POINTER(_GroupOut), C.POINTER(_Rollup)]
        _lib.oracle_kernel_rollup.restype = C.c_int
        _lib.oracle_percentile.argtypes = [C.c_void_p, C.c_uint64, C.c_double]
        _lib.oracle_percentile.restype = C.c_double
    return _lib


@dataclass
class Opts:
    """Analysis options.  Defaults = the paper's thresholds."""
    n_blocks: int = 32
    largest_block_id: int | None = None
    n_matrices: int = 8
    nan_policy: int = 0          # 0 = skipna (pandas), 1 = complete-only
    bins_per_unit: int = 100
    gain_cap: int = 10
    gain_gt: tuple = (1, 5)      # "more than 20 %"
    perf_lt: tuple = (17, 20)    # "less than 85 %"
    band_lo: tuple = (2, 5)      # "from 40 to 85 %"
    block_profile: bool = False  # Figs. 2/4 block profile (R-22)

    def ell(self):
        return self.n_blocks - 1 if self.largest_block_id is None else self.largest_block_id


@dataclass
class Result:
    counters: dict
    perf_hist: np.ndarray
    gain_hist: np.ndarray
    best_block_hist: np.ndarray
    derived: dict
    best_block: np.ndarray
    best_runtime: np.ndarray
    perf: np.ndarray
    gain: np.ndarray
    flags: np.ndarray
    percentiles: dict = field(default_factory=dict)
    rollup: dict | None = None
    profile_sum: np.ndarray | None = None
    profile_count: np.ndarray | None = None
    profile_mean: np.ndarray | None = None


class OracleError(RuntimeError):
    pass


def reduce_table(runtime_ms, block_id, group_offset=None, rows_per_group=0, group_matrix=None,
                 first_group=0, opts: Opts | None = None, percentiles=(), group_kernel=None,
                 kernel_rollup=False) -> Result:
    """Run the oracle on one table (host numpy arrays).  kernel_rollup: also the per-kernel
    roll-up (R-26) with group_kernel (None -> (first_group + g) // n_matrices)."""
    o = opts or Opts()
    rt = np.ascontiguousarray(runtime_ms, dtype=np.float32)
    bid = np.ascontiguousarray(block_id, dtype=np.uint16)
    n = rt.size
    if rows_per_group:
        G = -(-n // rows_per_group)
        off = None
    else:
        off = np.ascontiguousarray(group_offset, dtype=np.int64)
        G = off.size - 1
    gm = None if group_matrix is None else np.ascontiguousarray(group_matrix, dtype=np.uint32)
    T = _Table(rt.ctypes.data, bid.ctypes.data, n, None if off is None else off.ctypes.data, G,
               rows_per_group, None if gm is None else gm.ctypes.data, first_group)
    op = _Opts(o.n_blocks, o.ell(), o.n_matrices, o.nan_policy, o.bins_per_unit, o.gain_cap,
               o.gain_gt[0], o.gain_gt[1], o.perf_lt[0], o.perf_lt[1], o.band_lo[0], o.band_lo[1])
    ph = np.zeros(o.bins_per_unit + 1, np.uint64)
    gh = np.zeros(o.gain_cap * o.bins_per_unit + 1, np.uint64)
    bh = np.zeros(o.n_matrices * o.n_blocks, np.uint64)
    R = _Result()
    R.perf_hist, R.gain_hist, R.best_block_hist = ph.ctypes.data, gh.ctypes.data, bh.ctypes.data
    psum = pcnt = None
    if o.block_profile:
        psum = np.zeros(o.n_matrices * o.n_blocks, np.uint64)
        pcnt = np.zeros(o.n_matrices * o.n_blocks, np.uint64)
        R.profile_sum, R.profile_count = psum.ctypes.data, pcnt.ctypes.data
    bb = np.zeros(G, np.uint16)
    br = np.zeros(G, np.float32)
    pf = np.zeros(G, np.float64)
    gn = np.zeros(G, np.float64)
    fl = np.zeros(G, np.uint32)
    GO = _GroupOut(bb.ctypes.data, br.ctypes.data, pf.ctypes.data, gn.ctypes.data, fl.ctypes.data)
    rc = lib().oracle_reduce_table(C.byref(T), C.byref(op), C.byref(R), C.byref(GO))
    if rc != 0:
        raise OracleError(f"oracle_reduce_table failed: code {rc}")
    D = _Derived()
    lib().oracle_finalize(C.byref(R), C.byref(D))
    counters = {k: int(R.counters[i]) for i, k in enumerate(COUNTERS)}
    derived = {k: getattr(D, k) for k, _ in _Derived._fields_}
    res = Result(counters, ph, gh, bh.reshape(o.n_matrices, o.n_blocks), derived, bb, br, pf, gn,
                 fl)
    if o.block_profile:
        res.profile_sum = psum.reshape(o.n_matrices, o.n_blocks)
        res.profile_count = pcnt.reshape(o.n_matrices, o.n_blocks)
        with np.errstate(invalid="ignore", divide="ignore"):
            res.profile_mean = (psum.astype(np.float64) * 2.0 ** -31 / pcnt).reshape(
                o.n_matrices, o.n_blocks)
    if kernel_rollup:
        gk = None if group_kernel is None else np.ascontiguousarray(group_kernel, dtype=np.uint32)
        kh = np.zeros(o.bins_per_unit + 1, np.uint64)
        K = _Rollup()
        K.perf_hist = kh.ctypes.data
        rc = lib().oracle_kernel_rollup(C.byref(T), None if gk is None else gk.ctypes.data,
                                        C.byref(op), C.byref(GO), C.byref(K))
        if rc != 0:
            raise OracleError(f"oracle_kernel_rollup failed: code {rc}")
        kc = {k: int(K.counters[i]) for i, k in enumerate(ROLLUP)}
        nk = kc["n_kernels"]
        tot = (kc["kernel_mean_fx_hi"] << 21) + kc["kernel_mean_fx_lo"]
        res.rollup = dict(kc, perf_hist=kh,
                          frac_kernels_not_best=kc["n_kernels_not_best"] / nk if nk else float("nan"),
                          frac_kernels_perf_lt=kc["n_kernels_perf_lt"] / nk if nk else float("nan"),
                          frac_kernels_perf_band=kc["n_kernels_perf_band"] / nk if nk else float("nan"),
                          mean_kernel_perf=(float(tot) * 2.0 ** -52) / nk if nk else float("nan"))
    if percentiles:
        rd = (fl & 0x008) != 0
        res.percentiles = {
            "perf": [percentile(pf[rd], p) for p in percentiles],
            "gain": [percentile(gn[rd], p) for p in percentiles],
        }
    return res


_omp = None


def omp_lib():
    global _omp
    if _omp is None:
        build()
        _omp = C.CDLL(OMP_LIB_PATH)
        _omp.oracle_reduce_table_omp.argtypes = [C.POINTER(_Table), C.POINTER(_Opts),
                                                 C.POINTER(_Result), C.c_void_p, C.c_int]
        _omp.oracle_reduce_table_omp.restype = C.c_int
    return _omp


def reduce_table_parallel(runtime_ms, block_id, group_offset=None, rows_per_group=0,
                          group_matrix=None, first_group=0, opts: Opts | None = None,
                          threads: int = 0):
    """The same oracle on all host cores (group-aligned chunks, integer partials summed):
    counters and histograms only.  Baseline timing (bench.py cpu_baseline)."""
    o = opts or Opts()
    rt = np.ascontiguousarray(runtime_ms, dtype=np.float32)
    bid = np.ascontiguousarray(block_id, dtype=np.uint16)
    n = rt.size
    if rows_per_group:
        G = -(-n // rows_per_group)
        off = None
    else:
        off = np.ascontiguousarray(group_offset, dtype=np.int64)
        G = off.size - 1
    gm = None if group_matrix is None else np.ascontiguousarray(group_matrix, dtype=np.uint32)
    T = _Table(rt.ctypes.data, bid.ctypes.data, n, None if off is None else off.ctypes.data, G,
               rows_per_group, None if gm is None else gm.ctypes.data, first_group)
    op = _Opts(o.n_blocks, o.ell(), o.n_matrices, o.nan_policy, o.bins_per_unit, o.gain_cap,
               o.gain_gt[0], o.gain_gt[1], o.perf_lt[0], o.perf_lt[1], o.band_lo[0], o.band_lo[1])
    ph = np.zeros(o.bins_per_unit + 1, np.uint64)
    gh = np.zeros(o.gain_cap * o.bins_per_unit + 1, np.uint64)
    bh = np.zeros(o.n_matrices * o.n_blocks, np.uint64)
    R = _Result()
    R.perf_hist, R.gain_hist, R.best_block_hist = ph.ctypes.data, gh.ctypes.data, bh.ctypes.data
    rc = omp_lib().oracle_reduce_table_omp(C.byref(T), C.byref(op), C.byref(R), None, threads)
    if rc != 0:
        raise OracleError(f"oracle_reduce_table_omp failed: code {rc}")
    return ({k: int(R.counters[i]) for i, k in enumerate(COUNTERS)}, ph, gh,
            bh.reshape(o.n_matrices, o.n_blocks))


def percentile(values, p: float) -> float:
    v = np.ascontiguousarray(values, dtype=np.float64)
    return float(lib().oracle_percentile(v.ctypes.data, v.size, float(p)))
