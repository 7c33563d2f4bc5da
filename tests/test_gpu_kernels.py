"""a3 parity: every suite kernel at every block size against the fp64 oracle (DESIGN.md §9
tolerances: fp32 results within 1e-5 of the sum of |terms|, data movement bit-exact; the
bf16 GEMM within 1e-2).  Sizes span several tiles, vector and scalar paths and ragged tails;
N = 8192 (the bench configuration) is checked on sampled rows."""
import numpy as np
import pytest

from oracle import kernels as OK
from tests.gpu_util import ctx, require_gpu, to_np

pytestmark = pytest.mark.gpu

BLOCKS = list(range(32, 1025, 32))
SIZES = [64, 96, 100, 257, 512]
TOL = 1e-5


def _setup(kernel, sizes):
    c = ctx()
    c.register_suite([kernel], sizes)
    return c


def _run(c, kernel, n, block):
    import torch
    out = c.suite_tensor(kernel, n, 2)
    out.fill_(float("nan")) if out.dtype != torch.bfloat16 else out.fill_(0)
    c.launch(kernel, n, block)
    torch.cuda.synchronize()
    return to_np(out)


def _inputs(c, kernel, n):
    A = to_np(c.suite_tensor(kernel, n, 0))
    try:
        v = to_np(c.suite_tensor(kernel, n, 1))
    except Exception:
        v = None
    return A, v


def _check_rel(out, ref, scale, tol=TOL):
    err = np.abs(out.astype(np.float64) - ref)
    bad = err > tol * scale
    assert not bad.any(), f"{bad.sum()} elements off; worst {np.max(err / np.maximum(scale, 1e-300))}"


@pytest.mark.parametrize("name", ["euclid", "matvec", "rowsum", "colsum"])
def test_vector_outputs(name):
    from paper_2103_14409_b200 import KERNELS
    k = KERNELS[name]
    c = _setup(k, SIZES)
    for n in SIZES:
        A, v = _inputs(c, k, n)
        A = A.reshape(n, n)
        ref, scale = {
            "euclid": lambda: (OK.euclid(A, v), OK.euclid_abs_scale(A, v)),
            "matvec": lambda: (OK.matvec(A, v), OK.matvec_abs_scale(A, v)),
            "rowsum": lambda: (OK.rowsum(A), OK.rowsum_abs_scale(A)),
            "colsum": lambda: (OK.colsum(A), OK.colsum_abs_scale(A)),
        }[name]()
        for b in BLOCKS:
            out = _run(c, k, n, b)
            assert np.isfinite(out).all(), (name, n, b)
            _check_rel(out, ref, scale)


def test_transpose_bit_exact():
    from paper_2103_14409_b200 import K_TRANSPOSE
    c = _setup(K_TRANSPOSE, SIZES)
    for n in SIZES:
        A, _ = _inputs(c, K_TRANSPOSE, n)
        ref = OK.transpose(A.reshape(n, n))
        for b in BLOCKS:
            out = _run(c, K_TRANSPOSE, n, b).reshape(n, n)
            assert (out.view(np.uint32) == ref.view(np.uint32)).all(), (n, b)


def test_axpy():
    from paper_2103_14409_b200 import K_AXPY
    sizes = SIZES + [33]          # n = 1089 elements: scalar path
    c = _setup(K_AXPY, sizes)
    for n in sizes:
        x, y = _inputs(c, K_AXPY, n)
        ref, scale = OK.axpy(x, y), OK.axpy_abs_scale(x, y)
        for b in BLOCKS:
            _check_rel(_run(c, K_AXPY, n, b), ref, scale)


def test_stencil5():
    from paper_2103_14409_b200 import K_STENCIL5
    c = _setup(K_STENCIL5, SIZES)
    for n in SIZES:
        A, _ = _inputs(c, K_STENCIL5, n)
        A = A.reshape(n, n)
        ref, scale = OK.stencil5(A), OK.stencil5_abs_scale(A)
        border = np.zeros((n, n), bool)
        border[0, :] = border[-1, :] = border[:, 0] = border[:, -1] = True
        for b in BLOCKS:
            out = _run(c, K_STENCIL5, n, b).reshape(n, n)
            assert (out[border].view(np.uint32) == A[border].view(np.uint32)).all(), (n, b)
            _check_rel(out[~border], ref[~border], scale[~border])


def test_euclid_full_size_sampled():
    """BASELINE configs[1] size N = 8192, the launch configuration bench.py times."""
    import torch
    from paper_2103_14409_b200 import K_EUCLID
    n = 8192
    c = _setup(K_EUCLID, [n])
    A = c.suite_tensor(K_EUCLID, n, 0).view(n, n)
    q = to_np(c.suite_tensor(K_EUCLID, n, 1))
    rows = np.r_[0:8, np.random.default_rng(0).choice(n, 56, replace=False), n - 8:n]
    Ar = A[torch.as_tensor(rows, device=A.device)].cpu().numpy()
    ref = OK.euclid(Ar, q)
    for b in (32, 128, 256, 512, 1024):
        out = _run(c, K_EUCLID, n, b)[rows]
        _check_rel(out, ref, ref)


@pytest.mark.parametrize("n", [2048, 8192])
def test_data_movement_full_size_sampled(n):
    """transpose (bit-exact) and stencil5 at the sizes the sweep times, where the warp-unit
    loops run several iterations per warp: sampled output rows vs the oracle."""
    import torch
    from paper_2103_14409_b200 import K_STENCIL5, K_TRANSPOSE
    rng = np.random.default_rng(n)
    rows = np.unique(np.r_[1:5, rng.choice(np.arange(1, n - 1), 40, replace=False), n - 5:n - 1])
    c = _setup(K_TRANSPOSE, [n])
    A = c.suite_tensor(K_TRANSPOSE, n, 0).view(n, n)
    cols = to_np(A[:, torch.as_tensor(rows, device=A.device)])          # A[:, rows]
    ref_t = OK.transpose(cols)                                          # = T[rows, :]
    for b in (32, 96, 256, 1024):
        out = c.suite_tensor(K_TRANSPOSE, n, 2)
        out.fill_(float("nan"))
        c.launch(K_TRANSPOSE, n, b)
        torch.cuda.synchronize()
        got = to_np(out.view(n, n)[torch.as_tensor(rows, device=A.device)])
        assert (got.view(np.uint32) == ref_t.view(np.uint32)).all(), (n, b)
    c2 = _setup(K_STENCIL5, [n])
    S = c2.suite_tensor(K_STENCIL5, n, 0).view(n, n)
    Sh = to_np(S)
    for b in (32, 160, 1024):
        out = c2.suite_tensor(K_STENCIL5, n, 2)
        out.fill_(float("nan"))
        c2.launch(K_STENCIL5, n, b)
        torch.cuda.synchronize()
        O = to_np(out.view(n, n))
        for i in (0, n - 1):                                            # border rows: copies
            assert (O[i].view(np.uint32) == Sh[i].view(np.uint32)).all(), (n, b, i)
        for i in rows:                                                  # interior rows
            band = Sh[i - 1:i + 2]
            ref = OK.stencil5(band)[1]
            scale = OK.stencil5_abs_scale(band)[1]
            assert (O[i, [0, n - 1]].view(np.uint32) == Sh[i, [0, n - 1]].view(np.uint32)).all()
            _check_rel(O[i, 1:-1], ref[1:-1], scale[1:-1])


def test_launch_rejects_illegal_blocks():
    from paper_2103_14409_b200 import K_EUCLID, LscatError
    c = _setup(K_EUCLID, [64])
    for b in (0, 16, 33, 1056, 2048):
        with pytest.raises(LscatError):
            c.launch(K_EUCLID, 64, b)


GEMM_SIZES = [64, 200, 520]      # multiples of 8 (TMA pitch); ragged 128 x 256 tiles


def test_gemm_bf16_all_blocks():
    import torch
    from paper_2103_14409_b200 import K_GEMM_BF16, LscatError
    c = _setup(K_GEMM_BF16, GEMM_SIZES)
    for n in GEMM_SIZES:
        A, Bt = _inputs(c, K_GEMM_BF16, n)
        A, Bt = A.reshape(n, n), Bt.reshape(n, n)
        ref, scale = OK.gemm(A, Bt), OK.gemm_abs_scale(A, Bt)
        for b in BLOCKS:
            if b < 128:
                with pytest.raises(LscatError):
                    c.launch(K_GEMM_BF16, n, b)
                continue
            out = _run(c, K_GEMM_BF16, n, b).reshape(n, n)
            _check_rel(out, ref, scale, tol=1e-2)


def test_gemm_persistent_multi_tile():
    """N = 2056: 17 x 9 = 153 output tiles > 148 SMs, so persistent CTAs (B >= 192) run two
    tiles through both TMEM accumulator buffers; ragged 8-row / 8-column edge tiles."""
    from paper_2103_14409_b200 import K_GEMM_BF16
    n = 2056
    c = _setup(K_GEMM_BF16, [n])
    A, Bt = _inputs(c, K_GEMM_BF16, n)
    A, Bt = A.reshape(n, n), Bt.reshape(n, n)
    ref, scale = OK.gemm(A, Bt), OK.gemm_abs_scale(A, Bt)
    for b in (128, 192, 224, 256, 1024):
        out = _run(c, K_GEMM_BF16, n, b).reshape(n, n)
        _check_rel(out, ref, scale, tol=1e-2)


def test_gemm_identity_bit_exact():
    """Bt = I -> C = A exactly (one non-zero product per output, bf16 A exact)."""
    import torch
    from paper_2103_14409_b200 import K_GEMM_BF16
    n = 256
    c = _setup(K_GEMM_BF16, [n])
    eye = torch.eye(n, dtype=torch.bfloat16, device="cuda").contiguous()
    c.suite_upload(K_GEMM_BF16, n, 1, eye.view(-1))
    A = c.suite_tensor(K_GEMM_BF16, n, 0).view(n, n).clone()
    for b in (128, 256, 1024):
        out = c.suite_tensor(K_GEMM_BF16, n, 2)
        out.zero_()
        c.launch(K_GEMM_BF16, n, b)
        torch.cuda.synchronize()
        assert torch.equal(out.view(n, n), A)


def _check_gemm(got, ref, scale):
    """|C - C^| <= 2^-8 |C^| + 1e-5 sum_k |A_ik Bt_jk| (the bf16 output rounding is
    <= 2^-9 relative, fp32 accumulation of K products is far below 1e-5 of the absolute sum;
    a dropped 64-wide k-block (~sqrt(64)/3 ~ 2.7 at |C| ~ 30) fails it)."""
    err = np.abs(got.astype(np.float64) - ref)
    bound = 2.0 ** -8 * np.abs(ref) + 1e-5 * scale
    bad = err > bound
    assert not bad.any(), f"{bad.sum()} elements off; worst {np.max(err / bound)}"


@pytest.mark.parametrize("n", [520, 2056])
def test_gemm_tight_bound(n):
    """The tight GEMM bound at the ragged one-tile-row size and the multi-tile size."""
    from paper_2103_14409_b200 import K_GEMM_BF16
    c = _setup(K_GEMM_BF16, [n])
    A, Bt = _inputs(c, K_GEMM_BF16, n)
    A, Bt = A.reshape(n, n), Bt.reshape(n, n)
    ref, scale = OK.gemm(A, Bt), OK.gemm_abs_scale(A, Bt)
    for b in (128, 160, 192, 256, 1024):
        _check_gemm(_run(c, K_GEMM_BF16, n, b).reshape(n, n), ref, scale)


def test_gemm_full_size_sampled():
    """N = 8192: 32 x 32 tiles of 256 x 256 over 74 CTA pairs, so every pair runs ~14 tiles and
    each TMEM accumulator buffer is reused (flipped tmem_empty phase).  256 sampled rows (every
    tile row, each row crossing every tile column) cover every tile, including those a pair
    processes third or later; checked with the tight bound."""
    import torch
    from paper_2103_14409_b200 import K_GEMM_BF16
    n = 8192
    c = _setup(K_GEMM_BF16, [n])
    A = c.suite_tensor(K_GEMM_BF16, n, 0).view(n, n)
    Bt = c.suite_tensor(K_GEMM_BF16, n, 1).view(n, n)
    rng = np.random.default_rng(8192)
    rows_np = np.unique(np.r_[0:4, 127:131, 4090:4100, n - 4:n,
                              np.arange(0, n, 256) + rng.integers(0, 256, n // 256),
                              rng.choice(n, 240, replace=False)])
    assert len(rows_np) >= 256 and len(np.unique(rows_np // 256)) == n // 256
    rows = torch.as_tensor(rows_np, device="cuda")
    Ar = A[rows].float().cpu().numpy()
    Bn = Bt.float().cpu().numpy()
    ref, scale = OK.gemm(Ar, Bn), OK.gemm_abs_scale(Ar, Bn)
    for b in (128, 256, 1024):
        out = c.suite_tensor(K_GEMM_BF16, n, 2)
        out.zero_()
        c.launch(K_GEMM_BF16, n, b)
        torch.cuda.synchronize()
        got = out.view(n, n)[rows].float().cpu().numpy()
        _check_gemm(got, ref, scale)


@pytest.mark.parametrize("name", ["matvec", "rowsum", "colsum", "euclid"])
def test_vector_outputs_full_size(name):
    """N = 8192 (the suite roofline / bench size), every output element: the row kernels'
    persistent grid for B > 512, colsum's 64 row chunks + last-CTA ticket."""
    from paper_2103_14409_b200 import KERNELS
    k = KERNELS[name]
    n = 8192
    c = _setup(k, [n])
    A, v = _inputs(c, k, n)
    A = A.reshape(n, n)
    ref, scale = {
        "euclid": lambda: (OK.euclid(A, v), OK.euclid_abs_scale(A, v)),
        "matvec": lambda: (OK.matvec(A, v), OK.matvec_abs_scale(A, v)),
        "rowsum": lambda: (OK.rowsum(A), OK.rowsum_abs_scale(A)),
        "colsum": lambda: (OK.colsum(A), OK.colsum_abs_scale(A)),
    }[name]()
    for b in (32, 128, 256, 512, 544, 1024):
        out = _run(c, k, n, b)
        assert np.isfinite(out).all(), (name, b)
        _check_rel(out, ref, scale)


@pytest.mark.parametrize("name", ["euclid", "matvec", "rowsum"])
def test_row_kernels_mid_sizes(name):
    """The row kernels between the parity sizes and N = 8192, at every block size, each launch
    twice: a ragged float4 tail (N = 1028, 4100, 6000: 257, 1025, 1500 float4 per row), a scalar
    row (N % 4 != 0), grids above one wave (one row per warp) and the persistent grid (B > 512)."""
    from paper_2103_14409_b200 import KERNELS
    k = KERNELS[name]
    sizes = [1028, 2050, 4100, 6000]
    c = _setup(k, sizes)
    for n in sizes:
        A, v = _inputs(c, k, n)
        A = A.reshape(n, n)
        ref, scale = {
            "euclid": lambda: (OK.euclid(A, v), OK.euclid_abs_scale(A, v)),
            "matvec": lambda: (OK.matvec(A, v), OK.matvec_abs_scale(A, v)),
            "rowsum": lambda: (OK.rowsum(A), OK.rowsum_abs_scale(A)),
        }[name]()
        for b in BLOCKS:
            for _ in range(2):
                out = _run(c, k, n, b)
                assert np.isfinite(out).all(), (name, n, b)
                _check_rel(out, ref, scale)


def test_axpy_full_size():
    from paper_2103_14409_b200 import K_AXPY
    n = 8192
    c = _setup(K_AXPY, [n])
    x, y = _inputs(c, K_AXPY, n)
    ref, scale = OK.axpy(x, y), OK.axpy_abs_scale(x, y)
    for b in (32, 256, 1024):
        _check_rel(_run(c, K_AXPY, n, b), ref, scale)


def test_suite_inputs_non_degenerate():
    """a1 inputs (reading R-15): uniform on [-1, 1) -- range, mean ~ 0, sd ~ 1/sqrt(3), many
    distinct values, in0 != in1, and different (kernel, N, slot) buffers differ.  A broken
    generator (all zeros, one constant, a repeated stream) fails here, not silently in the
    closed-form checks."""
    import torch
    from paper_2103_14409_b200 import KERNELS
    c = ctx()
    ks = [KERNELS[k] for k in ("euclid", "matvec", "gemm_bf16", "transpose", "axpy", "rowsum",
                               "colsum", "stencil5")]
    sizes = [64, 512, 2048]
    c.register_suite(ks, sizes)
    seen = {}
    for k in ks:
        for n in sizes:
            for slot in (0, 1):
                try:
                    t = c.suite_tensor(k, n, slot)
                except Exception:
                    continue
                x = t.float().cpu().numpy().astype(np.float64)
                assert x.min() >= -1.0 and x.max() < 1.0, (k, n, slot)
                # the grid's own mean: -2^-8 on the bf16 grid (256 points), -2^-24 on fp32's
                mu = -2.0 ** -8 if t.dtype == torch.bfloat16 else -2.0 ** -24
                assert abs(x.mean() - mu) < 6.0 / np.sqrt(3 * x.size), (k, n, slot, x.mean())
                assert abs(x.std() - 1 / np.sqrt(3)) < 6 * np.sqrt(0.8 / (4 * x.size)) / np.sqrt(3) + 1e-3, \
                    (k, n, slot, x.std())
                distinct = np.unique(x).size
                grid = 256 if t.dtype == torch.bfloat16 else 2 ** 24
                assert distinct >= min(x.size, grid) * 0.5, (k, n, slot, distinct)
                head = x[:64].tobytes()
                assert head not in seen, (k, n, slot, seen.get(head))
                seen[head] = (k, n, slot)


def test_gemm_one_cta_persistent_path():
    """The one-CTA persistent GEMM (LSCAT_GEMM_2CTA=0; the CTA-pair kernel is the default for
    B >= 192) on the multi-tile size, in a child process (the switch is read once)."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, torch\n"
        "from oracle import kernels as OK\n"
        "import paper_2103_14409_b200 as L\n"
        "c = L.Ctx(0, seed=0x15CA7); n = 2056\n"
        "c.register_suite([L.K_GEMM_BF16], [n])\n"
        "A = c.suite_tensor(L.K_GEMM_BF16, n, 0).float().cpu().numpy().reshape(n, n)\n"
        "Bt = c.suite_tensor(L.K_GEMM_BF16, n, 1).float().cpu().numpy().reshape(n, n)\n"
        "ref, scale = OK.gemm(A, Bt), OK.gemm_abs_scale(A, Bt)\n"
        "for b in (192, 512):\n"
        "    c.launch(L.K_GEMM_BF16, n, b); torch.cuda.synchronize()\n"
        "    out = c.suite_tensor(L.K_GEMM_BF16, n, 2).float().cpu().numpy().reshape(n, n)\n"
        "    assert (np.abs(out - ref) <= 1e-2 * scale).all(), b\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LSCAT_GEMM_2CTA="0")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
