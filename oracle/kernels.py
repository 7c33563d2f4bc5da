"""fp64 CPU oracle of the suite kernels' outputs.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by the product package.

The paper times scraped linear-algebra kernels and names only
`euclidean_kernel`; the suite is this build's own (BASELINE.json north_star), so
each definition below is the textbook formula of the operation, written out in float64 over
the float32 (bf16 for the GEMM) inputs the device generated.  Scalars follow the paper's
naming roles ("w for width ... n for total size"): width = height = N for matrix
kernels, size = N*N for axpy, k = width for the GEMM.

Each function also has an *_abs_scale companion giving, per output element, the sum of the
absolute values of the terms that are added (the error-bound scale of DESIGN.md §9: an
fp32 sum of m terms in any order is within about m*eps*sum|terms| of the exact value).
"""
from __future__ import annotations

import numpy as np

ALPHA = 0.5           # axpy alpha (R-17)
C0, C1 = 0.5, 0.125   # stencil weights: centre, each of the 4 neighbours (c0 + 4 c1 = 1)


def _f64(a):
    return np.asarray(a, dtype=np.float64)


# --- euclidean_kernel: d[i] = sqrt(sum_j (A[i][j] - q[j])^2)   (reading R-14)
def euclid(A, q):
    D = _f64(A) - _f64(q)[None, :]
    return np.sqrt(np.sum(D * D, axis=1))


def euclid_abs_scale(A, q):
    return euclid(A, q)   # all terms are >= 0: the scale is the value itself


# --- matvec: y[i] = sum_j A[i][j] x[j]
def matvec(A, x):
    return _f64(A) @ _f64(x)


def matvec_abs_scale(A, x):
    return np.abs(_f64(A)) @ np.abs(_f64(x))


# --- row / column reductions: r[i] = sum_j A[i][j], c[j] = sum_i A[i][j]
def rowsum(A):
    return np.sum(_f64(A), axis=1)


def rowsum_abs_scale(A):
    return np.sum(np.abs(_f64(A)), axis=1)


def colsum(A):
    return np.sum(_f64(A), axis=0)


def colsum_abs_scale(A):
    return np.sum(np.abs(_f64(A)), axis=0)


# --- transpose: B[j][i] = A[i][j]
def transpose(A):
    return np.ascontiguousarray(np.asarray(A).T)


# --- axpy over N*N elements: z[t] = alpha x[t] + y[t] (out of place, so repeats are idempotent)
def axpy(x, y, alpha=ALPHA):
    return alpha * _f64(x) + _f64(y)


def axpy_abs_scale(x, y, alpha=ALPHA):
    return np.abs(alpha * _f64(x)) + np.abs(_f64(y))


# --- 5-point stencil: interior c0*A[i][j] + c1*(4 neighbours); border cells copied (R-17)
def stencil5(A):
    A = _f64(A)
    out = A.copy()
    if A.shape[0] >= 3 and A.shape[1] >= 3:
        out[1:-1, 1:-1] = C0 * A[1:-1, 1:-1] + C1 * (A[:-2, 1:-1] + A[2:, 1:-1] + A[1:-1, :-2]
                                                      + A[1:-1, 2:])
    return out


def stencil5_abs_scale(A):
    A = np.abs(_f64(A))
    out = A.copy()
    if A.shape[0] >= 3 and A.shape[1] >= 3:
        out[1:-1, 1:-1] = C0 * A[1:-1, 1:-1] + C1 * (A[:-2, 1:-1] + A[2:, 1:-1] + A[1:-1, :-2]
                                                      + A[1:-1, 2:])
    return out


# --- GEMM: C[i][j] = sum_k A[i][k] Bt[j][k]  (A, Bt: N x K row-major = K-major, K = N)
def gemm(A, Bt):
    return _f64(A) @ _f64(Bt).T


def gemm_abs_scale(A, Bt):
    return np.abs(_f64(A)) @ np.abs(_f64(Bt)).T
