"""a2-a5: the sweep engine end to end on the device (BASELINE configs[0]), its timeout /
invalid-config / launch-mode behaviour, and stats of the swept table against the oracle."""
import time

import numpy as np
import pytest

from oracle import table as OT
from tests.gpu_util import ctx

pytestmark = pytest.mark.gpu

TINY_K = None


def _tiny():
    from paper_2103_14409_b200 import K_EUCLID, K_MATVEC, K_AXPY
    return [K_EUCLID, K_MATVEC, K_AXPY], [64, 128, 256, 512], [32, 64, 128, 256, 512, 1024]


def test_tiny_sweep_and_stats():
    """configs[0]: 3 kernels x 6 blocks x 4 matrices = 72 rows, 12 groups; stats bit-exact."""
    from paper_2103_14409_b200 import reduce_opts, ROW_OK
    c = ctx()
    ks, ns, bs = _tiny()
    c.register_suite(ks, ns)
    tab = c.sweep(ks, ns, bs, warmup=1, brackets=10, launches=100, with_brackets=True)
    t = tab.to_numpy()
    assert t["n_rows"] == 72 and t["n_groups"] == 12                  # S:538 totality
    assert (np.diff(t["group_offset"]) == 6).all()
    assert (t["status"] == ROW_OK).all()
    rt = t["runtime_ms"]
    assert np.isfinite(rt).all() and (rt > 0).all()
    assert (t["block_id"] == np.tile(np.arange(6), 12)).all()
    assert (t["group_kernel"] == np.repeat(ks, 4)).all()
    assert (t["group_matrix"] == np.tile(np.arange(4), 3)).all()
    med = np.median(tab.brackets.astype(np.float64), axis=1).astype(np.float32)
    assert np.allclose(med, rt, rtol=1e-6)                               # median of K
    o = reduce_opts(6, 4)
    c.reduce_table(tab, o, per_group=False)
    st = c.stats(o, percentiles=[0.5, 0.9])
    ref = OT.reduce_table(rt, t["block_id"], t["group_offset"], group_matrix=t["group_matrix"],
                          opts=OT.Opts(n_blocks=6, n_matrices=4), percentiles=[0.5, 0.9])
    for k, v in ref.counters.items():
        assert st[k] == v, k
    assert (st["best_block_hist"] == ref.best_block_hist).all()
    assert st["pct_perf"] == ref.percentiles["perf"]


def test_runtime_grows_with_n():
    """Sanity: at fixed block the per-launch time does not shrink as the data grows 64x."""
    from paper_2103_14409_b200 import K_AXPY
    c = ctx()
    c.register_suite([K_AXPY], [256, 2048])
    t = c.sweep([K_AXPY], [256, 2048], [256], warmup=1, brackets=5, launches=50).to_numpy()
    assert t["runtime_ms"][1] > t["runtime_ms"][0]


def test_timeout_marks_nan_quickly():
    """P:228 timeout -> NaN row (bounded wall time)."""
    from paper_2103_14409_b200 import K_SPIN, ROW_TIMEOUT, ROW_OK, LAUNCH_STREAM
    c = ctx()
    t0 = time.time()
    tab = c.sweep([K_SPIN], [1], [32, 64], warmup=1, brackets=10, launches=100, timeout_s=1.0,
                  spin_ns=5_000_000, launch_mode=LAUNCH_STREAM)
    wall = time.time() - t0
    t = tab.to_numpy()
    assert (t["status"] == ROW_TIMEOUT).all() and np.isnan(t["runtime_ms"]).all()
    assert wall < 3.0
    tab = c.sweep([K_SPIN], [1], [32], warmup=1, brackets=3, launches=2, timeout_s=1.0,
                  spin_ns=100_000)
    t = tab.to_numpy()
    assert t["status"][0] == ROW_OK
    assert 0.09 < t["runtime_ms"][0] < 0.5                                # ~0.1 ms per launch


def test_gemm_small_blocks_invalid_config():
    from paper_2103_14409_b200 import K_GEMM_BF16, ROW_INVALID_CONFIG
    c = ctx()
    c.register_suite([K_GEMM_BF16], [256])
    t = c.sweep([K_GEMM_BF16], [256], [32, 64, 96], warmup=1, brackets=2, launches=2).to_numpy()
    assert (t["status"] == ROW_INVALID_CONFIG).all() and np.isnan(t["runtime_ms"]).all()


def test_stream_mode_and_host_table():
    from paper_2103_14409_b200 import K_EUCLID, LAUNCH_STREAM, Table, ROW_OK
    c = ctx()
    c.register_suite([K_EUCLID], [128])
    host = Table.empty(4, 1, device="cpu", pin=True)
    t = c.sweep([K_EUCLID], [128], [32, 64, 128, 1024], brackets=3, launches=20,
                launch_mode=LAUNCH_STREAM, table=host)
    assert t.n_rows == 4
    assert (t.status.numpy()[:4] == ROW_OK).all()
    assert np.isfinite(t.runtime_ms.numpy()[:4]).all()


def test_sweep_argument_errors():
    from paper_2103_14409_b200 import K_EUCLID, LscatError
    c = ctx()
    c.register_suite([K_EUCLID], [64])
    for bad in ([33], [32, 32], [1056], [64, 32]):
        with pytest.raises(LscatError):
            c.sweep([K_EUCLID], [64], bad, brackets=1, launches=1)
    with pytest.raises(LscatError):
        c.sweep([K_EUCLID], [128], [32], brackets=1, launches=1)       # not registered


def test_full_suite_small_sweep_stats():
    """All eight suite kernels swept at small N (GEMM rows < 128 threads are INVALID_CONFIG
    NaN rows); the stats of the swept table match the oracle bit for bit."""
    from paper_2103_14409_b200 import reduce_opts, ROW_OK, ROW_INVALID_CONFIG, KERNELS
    c = ctx()
    ks = [KERNELS[k] for k in ("euclid", "matvec", "gemm_bf16", "transpose", "axpy", "rowsum",
                               "colsum", "stencil5")]
    ns = [64, 256]
    bs = [32, 64, 96, 128, 256, 512, 1024]
    c.register_suite(ks, ns)
    t = c.sweep(ks, ns, bs, warmup=1, brackets=3, launches=20).to_numpy()
    assert t["n_rows"] == len(ks) * len(ns) * len(bs)
    gemm_rows = np.repeat(t["group_kernel"], np.diff(t["group_offset"])) == KERNELS["gemm_bf16"]
    small = np.tile(np.array(bs) < 128, len(ks) * len(ns))
    assert (t["status"][gemm_rows & small] == ROW_INVALID_CONFIG).all()
    assert (t["status"][~(gemm_rows & small)] == ROW_OK).all()
    o = reduce_opts(len(bs), len(ns))
    c.reduce_table(c.sweep(ks, ns, bs, warmup=1, brackets=3, launches=20), o, per_group=False)
    st = c.stats(o)
    assert st["n_rows"] == t["n_rows"] and st["n_nan"] == 3 * len(ns)


@pytest.mark.parametrize("n", [100, 512, 2048])
def test_pdl_graph_mode_outputs(n):
    """LAUNCH_GRAPH_PDL: back-to-back launches overlap their prologues/loads with the previous
    launch's drain; every kernel waits for its predecessor before storing, so after a PDL
    sweep each output still equals the oracle (colsum's partials/tickets are the sensitive
    case), and the table is complete."""
    import torch
    from oracle import kernels as OK
    from paper_2103_14409_b200 import KERNELS, LAUNCH_GRAPH_PDL, ROW_OK
    c = ctx()
    names = ("euclid", "matvec", "rowsum", "colsum", "transpose", "axpy", "stencil5")
    ks = [KERNELS[k] for k in names]
    bs = [32, 96, 256, 1024]
    c.register_suite(ks, [n])
    for k in ks:                                       # poison the outputs first
        c.suite_tensor(k, n, 2).fill_(float("nan"))
    t = c.sweep(ks, [n], bs, warmup=1, brackets=3, launches=200,
                launch_mode=LAUNCH_GRAPH_PDL).to_numpy()
    assert t["n_rows"] == len(ks) * len(bs) and (t["status"] == ROW_OK).all()
    assert np.isfinite(t["runtime_ms"]).all()
    torch.cuda.synchronize()
    f = lambda k, s: c.suite_tensor(KERNELS[k], n, s).cpu().numpy().astype(np.float64)
    A = f("euclid", 0).reshape(n, n)
    checks = {
        "euclid": (OK.euclid(A, f("euclid", 1)), OK.euclid_abs_scale(A, f("euclid", 1))),
    }
    for name, (ref, scale) in checks.items():
        out = f(name, 2)
        assert (np.abs(out - ref) <= 1e-5 * scale).all(), name
    Am = f("matvec", 0).reshape(n, n)
    assert (np.abs(f("matvec", 2) - OK.matvec(Am, f("matvec", 1)))
            <= 1e-5 * OK.matvec_abs_scale(Am, f("matvec", 1))).all()
    Ar = f("rowsum", 0).reshape(n, n)
    assert (np.abs(f("rowsum", 2) - OK.rowsum(Ar)) <= 1e-5 * OK.rowsum_abs_scale(Ar)).all()
    Ac = f("colsum", 0).reshape(n, n)
    assert (np.abs(f("colsum", 2) - OK.colsum(Ac)) <= 1e-5 * OK.colsum_abs_scale(Ac)).all()
    At = c.suite_tensor(KERNELS["transpose"], n, 0).cpu().numpy().reshape(n, n)
    Tt = c.suite_tensor(KERNELS["transpose"], n, 2).cpu().numpy().reshape(n, n)
    assert (Tt.view(np.uint32) == OK.transpose(At).view(np.uint32)).all()
    x, y = f("axpy", 0), f("axpy", 1)
    assert (np.abs(f("axpy", 2) - OK.axpy(x, y)) <= 1e-5 * OK.axpy_abs_scale(x, y)).all()
    As = f("stencil5", 0).reshape(n, n)
    Os = f("stencil5", 2).reshape(n, n)
    assert (np.abs(Os - OK.stencil5(As)) <= 1e-5 * OK.stencil5_abs_scale(As)).all()


def test_bench_launch_configuration_n8192():
    """The configuration bench.py times: euclidean_kernel at N = 8192 swept in PDL graph
    brackets of R = 1000 launches (7 graphs of 128 + one of 104) with the fractional L2 policy
    on A; afterwards the output equals the oracle on sampled rows (fp32 vs fp64, 1e-5 of the
    row's distance), and the measured per-launch time is physically plausible (no faster than
    the non-L2-resident part of A at 10 TB/s)."""
    import torch
    from oracle import kernels as OK
    from paper_2103_14409_b200 import K_EUCLID, LAUNCH_GRAPH_PDL, ROW_OK
    n = 8192
    c = ctx()
    c.register_suite([K_EUCLID], [n])
    out = c.suite_tensor(K_EUCLID, n, 2)
    out.fill_(float("nan"))
    t = c.sweep([K_EUCLID], [n], [32, 352, 1024], warmup=1, brackets=2, launches=1000,
                launch_mode=LAUNCH_GRAPH_PDL).to_numpy()
    assert (t["status"] == ROW_OK).all() and np.isfinite(t["runtime_ms"]).all()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    nbytes = 4 * n * n
    resident = min(1.0, 0.45 * l2 / nbytes)
    assert (t["runtime_ms"] * 1e-3 > (1 - resident) * nbytes / 10e12).all()
    torch.cuda.synchronize()
    A = c.suite_tensor(K_EUCLID, n, 0).view(n, n)
    q = c.suite_tensor(K_EUCLID, n, 1).cpu().numpy()
    rows = np.r_[0:4, np.random.default_rng(3).choice(n, 60, replace=False), n - 4:n]
    ref = OK.euclid(A[torch.as_tensor(rows, device=A.device)].cpu().numpy(), q)
    got = out.cpu().numpy()[rows]
    assert (np.abs(got - ref) <= 1e-5 * ref).all()


def test_tiny_sweep_every_point_output_checked():
    """configs[0] with verify: the output of the last timed launch of all 72 points (3 kernels
    x 6 blocks x 4 N) is copied back by the sweep and checked against the fp64 oracle."""
    from oracle import kernels as OK
    from paper_2103_14409_b200 import K_EUCLID, K_MATVEC, K_AXPY
    c = ctx()
    ks, ns, bs = _tiny()
    c.register_suite(ks, ns)
    cap = sum(len(bs) * (n * n * 4 if k == K_AXPY else n * 4) for k in ks for n in ns)
    tab = c.sweep(ks, ns, bs, warmup=1, brackets=10, launches=100, verify_bytes=cap)
    t = tab.to_numpy()
    assert t["n_rows"] == 72 and len(tab.verify) == 72
    row = 0
    for k in ks:
        for n in ns:
            A = c.suite_tensor(k, n, 0).cpu().numpy()
            v = c.suite_tensor(k, n, 1).cpu().numpy()
            if k == K_EUCLID:
                ref, scale = OK.euclid(A.reshape(n, n), v), OK.euclid_abs_scale(A.reshape(n, n), v)
            elif k == K_MATVEC:
                ref, scale = OK.matvec(A.reshape(n, n), v), OK.matvec_abs_scale(A.reshape(n, n), v)
            else:
                ref, scale = OK.axpy(A, v), OK.axpy_abs_scale(A, v)
            for _ in bs:
                out = np.frombuffer(tab.verify[row], np.float32).astype(np.float64)
                assert out.size == ref.size, (k, n)
                assert (np.abs(out - ref) <= 1e-5 * scale).all(), (k, n, row)
                row += 1


def test_globaltimer_agrees_with_events():
    """timer = GLOBALTIMER: the %globaltimer stamp brackets agree with the CUDA-event clock of
    the same brackets within a few percent."""
    from paper_2103_14409_b200 import K_EUCLID, TIMER_GLOBALTIMER, ROW_OK
    c = ctx()
    c.register_suite([K_EUCLID], [4096, 8192])
    tab = c.sweep([K_EUCLID], [4096, 8192], [128, 256, 1024], warmup=1, brackets=5, launches=200,
                  timer=TIMER_GLOBALTIMER, with_brackets=True, with_event_brackets=True)
    t = tab.to_numpy()
    assert (t["status"] == ROW_OK).all()
    gt, ev = tab.brackets.astype(np.float64), tab.brackets_event.astype(np.float64)
    assert np.isfinite(gt).all() and np.isfinite(ev).all()
    rel = np.abs(gt - ev) / ev
    assert rel.max() < 0.03, rel
    med = np.median(gt, axis=1).astype(np.float32)
    assert np.allclose(med, t["runtime_ms"], rtol=1e-6)                 # runtime from the stamps


def test_rotate_mode_cold_l2():
    """l2_mode = ROTATE: outputs still exact, the per-launch time at N = 2048 (A = 16.8 MB,
    L2-resident in WARM mode) does not shrink, and at N = 8192 the cold launch cannot beat HBM: algorithmic
    bytes / time <= 8 TB/s (nominal B200 HBM3e)."""
    from oracle import kernels as OK
    from paper_2103_14409_b200 import K_EUCLID, L2_ROTATE, ROW_OK, kernel_work
    c = ctx()
    ns, bs = [2048, 8192], [256, 1024]
    c.register_suite([K_EUCLID], ns)
    warm = c.sweep([K_EUCLID], ns, bs, warmup=1, brackets=5, launches=200).to_numpy()
    cap = sum(len(bs) * n * 4 for n in ns)
    tab = c.sweep([K_EUCLID], ns, bs, warmup=1, brackets=5, launches=200, l2_mode=L2_ROTATE,
                  verify_bytes=cap)
    cold = tab.to_numpy()
    assert (cold["status"] == ROW_OK).all()
    assert (cold["runtime_ms"][:2] >= warm["runtime_ms"][:2]).all(), (cold["runtime_ms"], warm["runtime_ms"])
    nbytes, _ = kernel_work(K_EUCLID, 8192)
    assert (nbytes / (cold["runtime_ms"][2:] * 1e-3) <= 8.0e12).all()
    row = 0
    for n in ns:
        A = c.suite_tensor(K_EUCLID, n, 0).cpu().numpy().reshape(n, n)
        q = c.suite_tensor(K_EUCLID, n, 1).cpu().numpy()
        ref = OK.euclid(A, q)
        for _ in bs:
            out = np.frombuffer(tab.verify[row], np.float32).astype(np.float64)
            assert (np.abs(out - ref) <= 1e-5 * ref).all(), (n, row)
            row += 1


def test_rotate_mode_every_kernel():
    """ROTATE runs every suite kernel (the GEMM with per-copy tensor maps, colsum sharing its
    scratch) with outputs equal to the WARM outputs' oracle."""
    from oracle import kernels as OK
    from paper_2103_14409_b200 import KERNELS, L2_ROTATE, ROW_OK
    c = ctx()
    n = 512
    names = ["euclid", "matvec", "gemm_bf16", "transpose", "axpy", "rowsum", "colsum", "stencil5"]
    ks = [KERNELS[k] for k in names]
    c.register_suite(ks, [n])
    bs = [128, 1024]
    tab = c.sweep(ks, [n], bs, warmup=1, brackets=3, launches=20, l2_mode=L2_ROTATE,
                  verify_bytes=len(ks) * len(bs) * n * n * 4)
    t = tab.to_numpy()
    assert (t["status"] == ROW_OK).all()
    row = 0
    for name, k in zip(names, ks):
        A = c.suite_tensor(k, n, 0).float().cpu().numpy()
        try:
            v = c.suite_tensor(k, n, 1).float().cpu().numpy()
        except Exception:
            v = None
        for _ in bs:
            raw = tab.verify[row]
            row += 1
            if name == "gemm_bf16":
                import torch
                out = torch.frombuffer(bytearray(raw), dtype=torch.bfloat16).float().numpy().reshape(n, n)
                ref, sc = OK.gemm(A.reshape(n, n), v.reshape(n, n)), OK.gemm_abs_scale(A.reshape(n, n), v.reshape(n, n))
                assert (np.abs(out - ref) <= 2.0 ** -8 * np.abs(ref) + 1e-5 * sc).all()
                continue
            out = np.frombuffer(raw, np.float32)
            if name == "transpose":
                assert (out.reshape(n, n) == OK.transpose(A.reshape(n, n))).all()
                continue
            ref, sc = {
                "euclid": lambda: (OK.euclid(A.reshape(n, n), v), OK.euclid_abs_scale(A.reshape(n, n), v)),
                "matvec": lambda: (OK.matvec(A.reshape(n, n), v), OK.matvec_abs_scale(A.reshape(n, n), v)),
                "rowsum": lambda: (OK.rowsum(A.reshape(n, n)), OK.rowsum_abs_scale(A.reshape(n, n))),
                "colsum": lambda: (OK.colsum(A.reshape(n, n)), OK.colsum_abs_scale(A.reshape(n, n))),
                "axpy": lambda: (OK.axpy(A, v), OK.axpy_abs_scale(A, v)),
                "stencil5": lambda: (OK.stencil5(A.reshape(n, n)).ravel(), OK.stencil5_abs_scale(A.reshape(n, n)).ravel()),
            }[name]()
            assert (np.abs(out.astype(np.float64) - ref) <= 1e-5 * sc).all(), name


def test_budget_checked_after_every_bracket():
    """A-18 / P:228: without a warm-up prediction (warmup = 0) the brackets run one at a time
    and the point stops as soon as the budget is exceeded: 10 brackets of 0.4 s against a 1 s
    budget stop after 2 (the second was already queued), not after 4 s."""
    from paper_2103_14409_b200 import K_SPIN, ROW_TIMEOUT, ROW_OK
    c = ctx()
    t0 = time.time()
    tab = c.sweep([K_SPIN], [1], [32], warmup=0, brackets=10, launches=2, timeout_s=1.0,
                  spin_ns=200_000_000, with_brackets=True)
    wall = time.time() - t0
    t = tab.to_numpy()
    assert t["status"][0] == ROW_TIMEOUT and np.isnan(t["runtime_ms"][0])
    ran = np.isfinite(tab.brackets[0]).sum()
    assert ran == 2, tab.brackets[0]
    assert wall < 2.0, wall
    # the same point with a budget that fits runs all brackets one at a time
    tab = c.sweep([K_SPIN], [1], [32], warmup=0, brackets=4, launches=1, timeout_s=1.0,
                  spin_ns=100_000_000, with_brackets=True)
    t = tab.to_numpy()
    assert t["status"][0] == ROW_OK and np.isfinite(tab.brackets[0]).all()
