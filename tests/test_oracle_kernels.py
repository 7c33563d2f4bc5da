"""Pins of the fp64 suite-kernel oracle (oracle/kernels.py) against closed forms, invariants
and brute-force loops written here."""
import numpy as np

from oracle import kernels as K


def _loops_matvec(A, x):
    return [sum(float(A[i][j]) * float(x[j]) for j in range(len(x))) for i in range(len(A))]


def test_euclid_closed_forms():
    N = 64
    s = 0.375
    A = np.zeros((N, N), np.float32)
    A[:, 0], A[:, 1] = 3 * s, 4 * s
    assert (K.euclid(A, np.zeros(N, np.float32)) == 5 * s).all()      # 3-4-5 triangle
    for m in (1, 2, 3):
        n = 4 ** m
        A = np.full((n, n), -0.5, np.float32)
        assert (K.euclid(A, np.zeros(n, np.float32)) == 0.5 * 2 ** m).all()
    rng = np.random.default_rng(0)
    A = rng.uniform(-1, 1, (7, 5)).astype(np.float32)
    q = rng.uniform(-1, 1, 5).astype(np.float32)
    ref = [np.sqrt(sum((float(A[i][j]) - float(q[j])) ** 2 for j in range(5))) for i in range(7)]
    np.testing.assert_allclose(K.euclid(A, q), ref, rtol=1e-15)


def test_matvec_closed_forms():
    N = 96
    x = np.random.default_rng(1).uniform(-1, 1, N).astype(np.float32)
    assert (K.matvec(np.eye(N, dtype=np.float32), x) == x.astype(np.float64)).all()
    assert (K.matvec(np.ones((N, N), np.float32), np.ones(N, np.float32)) == N).all()
    A = np.random.default_rng(2).uniform(-1, 1, (5, 6)).astype(np.float32)
    np.testing.assert_allclose(K.matvec(A, x[:6]), _loops_matvec(A, x[:6]), rtol=1e-14)
    assert (K.matvec_abs_scale(A, x[:6]) >= np.abs(K.matvec(A, x[:6]))).all()


def test_reductions():
    N = 128
    assert (K.rowsum(np.ones((N, N), np.float32)) == N).all()
    assert (K.colsum(np.ones((N, N), np.float32)) == N).all()
    alt = np.tile((-1.0) ** np.arange(N), (N, 1)).astype(np.float32)     # (-1)^j
    assert (K.rowsum(alt) == 0).all()
    assert (K.colsum(alt.T) == 0).all()
    A = np.random.default_rng(3).uniform(-1, 1, (6, 9)).astype(np.float32)
    np.testing.assert_allclose(K.rowsum(A), [sum(map(float, r)) for r in A], rtol=1e-14)
    np.testing.assert_allclose(K.colsum(A), [sum(float(A[i][j]) for i in range(6))
                                             for j in range(9)], rtol=1e-14)


def test_transpose():
    N = 64
    A = (np.arange(N)[:, None] * N + np.arange(N)[None, :]).astype(np.float32)  # exact ints
    T = K.transpose(A)
    assert all(T[j][i] == i * N + j for i in range(0, N, 7) for j in range(0, N, 5))
    assert (K.transpose(T) == A).all()


def test_axpy():
    x = np.full(100, 2.0, np.float32)
    y = np.ones(100, np.float32)
    assert (K.axpy(x, y) == 2.0).all()                                      # 0.5*2 + 1
    assert K.ALPHA == 0.5


def test_stencil5():
    N = 40
    c = np.full((N, N), 0.75, np.float32)
    assert (K.stencil5(c) == 0.75).all()                                   # c0 + 4 c1 = 1
    i, j = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    lin = (i + 2 * j).astype(np.float32)
    assert (K.stencil5(lin) == lin).all()                                  # linear -> unchanged
    A = np.random.default_rng(4).uniform(-1, 1, (5, 6)).astype(np.float32)
    S = K.stencil5(A)
    for r in range(5):
        for s in range(6):
            if r in (0, 4) or s in (0, 5):
                assert S[r][s] == A[r][s]
            else:
                ref = 0.5 * float(A[r][s]) + 0.125 * (float(A[r - 1][s]) + float(A[r + 1][s])
                                                     + float(A[r][s - 1]) + float(A[r][s + 1]))
                assert abs(S[r][s] - ref) < 1e-15


def test_gemm():
    N = 48
    A = np.random.default_rng(5).uniform(-1, 1, (N, N)).astype(np.float32)
    assert (K.gemm(A, np.eye(N, dtype=np.float32)) == A).all()              # Bt = I -> C = A
    assert (K.gemm(np.ones((N, N)), np.ones((N, N))) == N).all()
    B = np.random.default_rng(6).uniform(-1, 1, (4, 5))
    A4 = A[:3, :5]
    ref = [[sum(float(A4[i][k]) * float(B[j][k]) for k in range(5)) for j in range(4)]
           for i in range(3)]
    np.testing.assert_allclose(K.gemm(A4, B), ref, rtol=1e-14)
