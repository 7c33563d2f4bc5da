"""CPU-side checks of the C ABI (no GPU needed): the library loads, exports every function
include/lscat.h declares, the host-only helpers behave, and compute calls fail loudly (no
CPU fallback) when no device is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2103_14409_b200 import build as _b  # noqa: F401
    import importlib
    b = importlib.import_module("paper_2103_14409_b200.build")
    b.build()
    from paper_2103_14409_b200 import lscat
    return lscat


def header_functions():
    src = open(os.path.join(ROOT, "include", "lscat.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lscat_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    L = lib.load()
    declared = header_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(lib.EXPORTS) == declared
    assert L.lscat_abi_version() == 2
    assert L.lscat_status_string(1) == b"invalid argument"


def test_no_cpu_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(lib.LscatError) as e:
        lib.Ctx(0)
    assert e.value.status == lib.ERR_CUDA if hasattr(lib, "ERR_CUDA") else 2


def test_kernel_work(lib):
    N = 8192
    assert lib.kernel_work(lib.K_EUCLID, N) == (4 * N * N + 8 * N, 3 * N * N)
    assert lib.kernel_work(lib.K_AXPY, N)[0] == 12 * N * N
    assert lib.kernel_work(lib.K_TRANSPOSE, N)[0] == 8 * N * N
    assert lib.kernel_work(lib.K_GEMM_BF16, N) == (6 * N * N, 2 * N ** 3)
    assert round(lib.kernel_work(lib.K_EUCLID, N)[0] / 1e6, 1) == 268.5


def test_plan_partition_and_lpt(lib):
    ks = [lib.K_EUCLID, lib.K_MATVEC, lib.K_AXPY]
    sizes = [64, 128, 256, 512, 1024, 2048, 4096, 8192]
    blocks = list(range(32, 1025, 32))
    npts = len(ks) * len(sizes) * len(blocks)
    for world in (1, 2, 3, 8):
        parts = [lib.plan(ks, sizes, blocks, r, world) for r in range(world)]
        allp = np.sort(np.concatenate(parts))
        assert (allp == np.arange(npts)).all()                  # every point exactly once
        for p in parts:
            assert (np.diff(p) > 0).all()                        # ascending ids
        # LPT load balance: max load <= mean + max single point cost
        cost = np.zeros(npts)
        for p in range(npts):
            k = ks[p // (len(sizes) * 32)]
            n = sizes[(p // 32) % len(sizes)]
            by, fl = lib.kernel_work(k, n)
            cost[p] = 10001 * max(by / 6.55e12, fl / 75e12, 2e-6)
        loads = [cost[p].sum() for p in parts]
        assert max(loads) <= cost.sum() / world + cost.max() + 1e-12
    # group sharding keeps whole groups together
    parts = [lib.plan(ks, sizes, blocks, r, 4, shard=lib.SHARD_GROUP) for r in range(4)]
    for p in parts:
        groups = np.unique(p // 32)
        assert len(p) == 32 * len(groups)
    # deterministic
    assert (lib.plan(ks, sizes, blocks, 1, 4) == lib.plan(ks, sizes, blocks, 1, 4)).all()


def test_plan_rejects_illegal_blocks(lib):
    # block legality (<= 1024, multiple of 32); ids need a unique ascending list
    for bad in ([33], [1056], [64, 32], [32, 32], [0]):
        with pytest.raises(lib.LscatError):
            lib.plan([lib.K_EUCLID], [64], bad, 0, 1)
    with pytest.raises(lib.LscatError):
        lib.plan([lib.K_EUCLID], [128, 64], [32], 0, 1)      # sizes must ascend


def test_reduce_opts_and_partials(lib):
    o = lib.reduce_opts(32, 8)
    assert (o.largest_block_id, o.bins_per_unit, o.gain_cap) == (31, 100, 10)
    assert (o.gain_gt_num, o.gain_gt_den, o.perf_lt_num, o.perf_lt_den) == (1, 5, 17, 20)
    assert lib.partials_len(o) == 24 + 101 + 1001 + 8 * 32


def test_reduce_opts_percentiles(lib):
    """R-27: the percentile list in the reduce options (struct layout = the header's: 16 u32,
    n_percentiles, pad, a pointer); the defaults leave it off and the library's option check
    (lscat_partials_len returns 0 for rejected options) accepts <= 64 values in [0, 1]."""
    o = lib.reduce_opts(32, 8)
    assert C.sizeof(o) == 16 * 4 + 8 + 8 and (o.n_percentiles, o.percentiles) == (0, None)
    good = lib.reduce_opts(32, 8, percentiles=[0.0, 0.5, 0.99, 1.0])
    assert good.n_percentiles == 4 and lib.partials_len(good) == lib.partials_len(o)
    assert list(np.ctypeslib.as_array(C.cast(good.percentiles, C.POINTER(C.c_double)), (4,))) == [0.0, 0.5, 0.99, 1.0]
    for bad in ([0.5, 1.5], [-0.1], [float("nan")], [0.5] * 65):
        assert lib.partials_len(lib.reduce_opts(32, 8, percentiles=bad)) == 0, bad
    o.n_percentiles = 3  # a count without an array
    assert lib.partials_len(o) == 0


def test_gen_shape(lib):
    L = lib.load()
    o = lib.lscat.GenOpts(2140796, 8363, 32, 31, 8, 1, 0.03, 980, 0, 0, 1, 0) \
        if hasattr(lib, "lscat") else None
    from paper_2103_14409_b200.lscat import GenOpts
    o = GenOpts(2140796, 8363, 32, 31, 8, 1, 0.03, 980, 0, 0, 1, 0)
    nr, ng = C.c_uint64(), C.c_uint64()
    assert L.lscat_gen_table_shape(C.byref(o), C.byref(nr), C.byref(ng)) == 0
    assert (nr.value, ng.value) == (2140796, 66900)
    o = GenOpts(5028536, 19683, 32, 31, 8, 0, 0.03, 4, 0, 0, 4, 1)       # point shard 1 of 4
    assert L.lscat_gen_table_shape(C.byref(o), C.byref(nr), C.byref(ng)) == 0
    assert ng.value == 157142 and nr.value == 157141 * 8 + 6             # last group: 24 rows


def test_table_c_view_cache():
    """The binding's cached C view of a table (reduce calls take a const table): reused while
    nothing changes, rebuilt after any attribute assignment, and equal to a fresh one."""
    import torch
    from paper_2103_14409_b200 import Table
    n, G = 100, 4
    t = Table(torch.zeros(n), torch.zeros(n, dtype=torch.int16), None,
              torch.arange(0, n + 1, n // G, dtype=torch.int64), None, torch.zeros(G, dtype=torch.int32),
              n_rows=n, n_groups=G)
    a = t.c_input()
    assert t.c_input() is a
    fresh = t.c()
    for f, _ in fresh._fields_:
        assert getattr(a, f) == getattr(fresh, f), f
    t.n_rows = 50
    b = t.c_input()
    assert b is not a and b.n_rows == 50
    t.runtime_ms = torch.zeros(n)
    c = t.c_input()
    assert c is not b and c.runtime_ms == t.runtime_ms.data_ptr()
    assert t.c_input(with_groups=False).group_offset is None
