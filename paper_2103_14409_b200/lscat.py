"""Thin ctypes binding of liblscat.so (include/lscat.h).

Argument marshalling only: every step of the hot path runs in the library's CUDA kernels.
Torch is used for device memory and streams (tensors own the table buffers).  There is no
CPU fallback: if the shared library is missing or no GPU is present the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblscat.so")

# ---- enums (include/lscat.h)
OK, ERR_INVALID_ARG, ERR_CUDA, ERR_OOM, ERR_NCCL, ERR_STATE, ERR_UNSUPPORTED = range(7)
ROW_OK, ROW_TIMEOUT, ROW_LAUNCH_ERROR, ROW_INVALID_CONFIG = range(4)
K_EUCLID, K_MATVEC, K_GEMM_BF16, K_TRANSPOSE, K_AXPY, K_ROWSUM, K_COLSUM, K_STENCIL5 = range(8)
K_SPIN = 100
KERNELS = {"euclid": K_EUCLID, "matvec": K_MATVEC, "gemm_bf16": K_GEMM_BF16,
           "transpose": K_TRANSPOSE, "axpy": K_AXPY, "rowsum": K_ROWSUM, "colsum": K_COLSUM,
           "stencil5": K_STENCIL5, "spin": K_SPIN}
SLOT_IN0, SLOT_IN1, SLOT_OUT = 0, 1, 2
MEM_DEVICE, MEM_HOST = 0, 1
LAUNCH_GRAPH, LAUNCH_STREAM, LAUNCH_GRAPH_PDL = 0, 1, 2
SHARD_POINT_LPT, SHARD_GROUP = 0, 1
TIMER_EVENT, TIMER_GLOBALTIMER = 0, 1
L2_WARM, L2_ROTATE = 0, 1
SKIPNA, COMPLETE_ONLY = 0, 1
PRESET_T4, PRESET_GTX980 = 0, 1
GF = dict(defined=0x1, complete=0x2, all_nan=0x4, ratio_defined=0x8, largest_is_best=0x10,
          largest_slower=0x20, gain_gt=0x40, perf_lt=0x80, perf_band=0x100,
          largest_missing=0x200)
P_NCOUNTERS = 24
COUNTERS = ["n_rows", "n_ok", "n_nan", "n_invalid", "n_groups", "n_defined", "n_all_nan",
            "n_complete", "n_incomplete", "n_largest_missing", "n_ratio_defined",
            "n_largest_is_best", "n_largest_strictly_slower", "n_gain_gt", "n_perf_lt",
            "n_perf_band", "perf_fx_hi", "perf_fx_lo", "gain_fx_hi", "gain_fx_lo"]
ROLLUP = ["n_kernels", "n_kernels_largest_not_best", "n_kernels_perf_lt", "n_kernels_perf_band",
          "kernel_mean_fx_hi", "kernel_mean_fx_lo"]
ROLLUP_DERIVED = ["frac_kernels_largest_not_best", "frac_kernels_perf_lt", "frac_kernels_perf_band",
                  "mean_kernel_perf"]
DERIVED = ["frac_nonnan", "frac_largest_not_best", "frac_gain_gt", "frac_perf_lt",
           "frac_perf_band", "mean_perf", "mean_gain"]


class LscatError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"lscat status {status}: {msg}")
        self.status = status


# ---- structs
u8p, u16p, u32p, u64p = (C.c_void_p,) * 4


class PlanOpts(C.Structure):
    _fields_ = [("kernels", C.c_void_p), ("n_kernels", C.c_uint32),
                ("sizes", C.c_void_p), ("n_sizes", C.c_uint32),
                ("blocks", C.c_void_p), ("n_blocks", C.c_uint32),
                ("warmup", C.c_uint32), ("brackets", C.c_uint32),
                ("launches_per_bracket", C.c_uint32), ("shard", C.c_uint32),
                ("launch_overhead_s", C.c_double), ("hbm_bytes_per_s", C.c_double),
                ("tensor_flops_per_s", C.c_double)]


class SweepOpts(C.Structure):
    _fields_ = [("blocks", C.c_void_p), ("n_blocks", C.c_uint32), ("warmup", C.c_uint32),
                ("brackets", C.c_uint32), ("launches_per_bracket", C.c_uint32),
                ("timeout_s", C.c_double), ("launch_mode", C.c_uint32), ("shard", C.c_uint32),
                ("launch_overhead_s", C.c_double), ("spin_ns", C.c_uint64),
                ("bracket_ms_host", C.c_void_p), ("timer", C.c_uint32), ("l2_mode", C.c_uint32),
                ("bracket_ms_event_host", C.c_void_p), ("verify", C.c_uint32),
                ("verify_host", C.c_void_p), ("verify_cap_bytes", C.c_uint64),
                ("verify_offsets", C.c_void_p)]


class TableC(C.Structure):
    _fields_ = [("runtime_ms", C.c_void_p), ("block_id", C.c_void_p), ("status", C.c_void_p),
                ("group_offset", C.c_void_p), ("group_kernel", C.c_void_p),
                ("group_matrix", C.c_void_p), ("cap_rows", C.c_uint64),
                ("cap_groups", C.c_uint64), ("n_rows", C.c_uint64), ("n_groups", C.c_uint64),
                ("rows_per_group", C.c_uint32), ("mem", C.c_uint32),
                ("first_group", C.c_uint64)]


class ReduceOpts(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in (
        "n_blocks", "largest_block_id", "n_matrices", "nan_policy", "bins_per_unit", "gain_cap",
        "gain_gt_num", "gain_gt_den", "perf_lt_num", "perf_lt_den", "band_lo_num",
        "band_lo_den", "point_sharded", "keep_values", "block_profile", "kernel_rollup",
        "n_percentiles", "pad0")] + [("percentiles", C.c_void_p)]


class ReduceOutC(C.Structure):
    _fields_ = [("best_block_id", C.c_void_p), ("best_runtime", C.c_void_p),
                ("perf", C.c_void_p), ("gain", C.c_void_p), ("flags", C.c_void_p),
                ("partials", C.c_void_p)]


class StatsOutC(C.Structure):
    _fields_ = ([(n, C.c_uint64) for n in COUNTERS] + [(n, C.c_double) for n in DERIVED] +
                [("perf_hist", C.c_void_p), ("gain_hist", C.c_void_p),
                 ("best_block_hist", C.c_void_p), ("percentiles", C.c_void_p),
                 ("n_percentiles", C.c_uint32), ("pct_perf", C.c_void_p),
                 ("pct_gain", C.c_void_p), ("profile_mean", C.c_void_p),
                 ("profile_count", C.c_void_p)] +
                [(n, C.c_uint64) for n in ROLLUP] + [(n, C.c_double) for n in ROLLUP_DERIVED] +
                [("kernel_perf_hist", C.c_void_p)])


class OccInfo(C.Structure):
    _fields_ = [("threads", C.c_uint32)] + [(n, C.c_int32) for n in (
        "regs_per_thread", "static_smem", "dynamic_smem", "max_threads_per_block",
        "blocks_per_sm", "warps_per_sm", "api_block", "api_min_grid")]


class GenOpts(C.Structure):
    _fields_ = [("n_rows_global", C.c_uint64), ("n_kernels", C.c_uint32),
                ("n_blocks", C.c_uint32), ("largest_block_id", C.c_uint32),
                ("n_matrices", C.c_uint32), ("preset", C.c_uint32), ("nan_rate", C.c_double),
                ("seed", C.c_uint64), ("group_begin", C.c_uint64), ("group_end", C.c_uint64),
                ("block_mod", C.c_uint32), ("block_rem", C.c_uint32)]


_lib = None

EXPORTS = [
    "lscat_abi_version", "lscat_status_string", "lscat_ctx_create", "lscat_ctx_destroy",
    "lscat_last_error", "lscat_launch_count", "lscat_comm_unique_id", "lscat_comm_init",
    "lscat_comm_init_local", "lscat_register_suite",
    "lscat_suite_buffer", "lscat_suite_upload", "lscat_launch", "lscat_kernel_work",
    "lscat_plan", "lscat_sweep", "lscat_reduce_opts_default", "lscat_partials_len",
    "lscat_reduce_table", "lscat_stats", "lscat_gen_table", "lscat_gen_table_shape",
    "lscat_aggregation_experiment", "lscat_occupancy_block", "lscat_timeout_curve",
    "lscat_ingest",
]


def load(path: str = LIB_PATH):
    """Load liblscat.so; raises (no fallback) if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python __graft_entry__.py build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(path)
    vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
    sig = {
        "lscat_abi_version": ([], C.c_int),
        "lscat_status_string": ([i32], C.c_char_p),
        "lscat_ctx_create": ([i32, u64, C.POINTER(vp)], i32),
        "lscat_ctx_destroy": ([vp], None),
        "lscat_last_error": ([vp], C.c_char_p),
        "lscat_launch_count": ([vp, C.POINTER(u64)], i32),
        "lscat_comm_unique_id": ([vp], i32),
        "lscat_comm_init": ([vp, vp, i32, i32], i32),
        "lscat_comm_init_local": ([vp, C.c_char_p, i32, i32], i32),
        "lscat_register_suite": ([vp, vp, u32, vp, u32, vp], i32),
        "lscat_suite_buffer": ([vp, u32, u32, u32, C.POINTER(vp), C.POINTER(u64)], i32),
        "lscat_suite_upload": ([vp, u32, u32, u32, vp, u64, u32, vp], i32),
        "lscat_launch": ([vp, u32, u32, u32, vp], i32),
        "lscat_kernel_work": ([u32, u32, C.POINTER(u64), C.POINTER(u64)], i32),
        "lscat_plan": ([C.POINTER(PlanOpts), i32, i32, vp, u64, C.POINTER(u64)], i32),
        "lscat_sweep": ([vp, vp, u32, vp, u32, C.POINTER(SweepOpts), C.POINTER(TableC), vp], i32),
        "lscat_reduce_opts_default": ([C.POINTER(ReduceOpts), u32, u32], None),
        "lscat_partials_len": ([C.POINTER(ReduceOpts)], C.c_size_t),
        "lscat_reduce_table": ([vp, C.POINTER(TableC), C.POINTER(ReduceOpts),
                                C.POINTER(ReduceOutC), vp], i32),
        "lscat_stats": ([vp, C.POINTER(ReduceOpts), C.POINTER(StatsOutC), vp], i32),
        "lscat_gen_table": ([vp, C.POINTER(GenOpts), C.POINTER(TableC), vp], i32),
        "lscat_gen_table_shape": ([C.POINTER(GenOpts), C.POINTER(u64), C.POINTER(u64)], i32),
        "lscat_aggregation_experiment": ([vp, vp, u64, u32, u32, u64, vp, vp, vp, vp], i32),
        "lscat_occupancy_block": ([vp, u32, vp, u32, C.POINTER(u32), C.POINTER(OccInfo)], i32),
        "lscat_timeout_curve": ([vp, C.POINTER(TableC), u32, u32, u32, vp, u32, vp, vp], i32),
        "lscat_ingest": ([vp, vp, vp, vp, vp, vp, u64, C.POINTER(TableC), C.POINTER(u64), vp], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    if L.lscat_abi_version() != 2:
        raise ImportError("liblscat ABI version mismatch")
    _lib = L
    return L


def _arr(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data


# ---------------------------------------------------------------- host-only helpers -------
def kernel_work(kernel: int, n: int):
    """Algorithmic (bytes, flops) of one launch."""
    b, f = C.c_uint64(), C.c_uint64()
    st = load().lscat_kernel_work(kernel, n, C.byref(b), C.byref(f))
    if st:
        raise LscatError(st, "kernel_work")
    return b.value, f.value


def plan(kernels, sizes, blocks, rank, world, warmup=1, brackets=10, launches=1000,
         shard=SHARD_POINT_LPT, launch_overhead_s=0.0):
    """Point ids owned by `rank` (a2).  Host-only."""
    k, kp = _arr(kernels, np.uint32)
    s, sp = _arr(sizes, np.uint32)
    b, bp = _arr(blocks, np.uint16)
    o = PlanOpts(kp, k.size, sp, s.size, bp, b.size, warmup, brackets, launches, shard,
                 launch_overhead_s, 0.0, 0.0)
    n = C.c_uint64()
    st = load().lscat_plan(C.byref(o), rank, world, None, 0, C.byref(n))
    if st:
        raise LscatError(st, "plan")
    out = np.zeros(n.value, np.uint32)
    st = load().lscat_plan(C.byref(o), rank, world, out.ctypes.data, out.size, C.byref(n))
    if st:
        raise LscatError(st, "plan")
    return out


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = load().lscat_comm_unique_id(buf)
    if st:
        raise LscatError(st, "comm_unique_id")
    return buf.raw


def reduce_opts(n_blocks=32, n_matrices=8, **kw) -> ReduceOpts:
    o = ReduceOpts()
    load().lscat_reduce_opts_default(C.byref(o), n_blocks, n_matrices)
    for k, v in kw.items():
        if k in ("gain_gt", "perf_lt", "band_lo"):
            setattr(o, k + "_num", v[0])
            setattr(o, k + "_den", v[1])
        elif k == "percentiles":  # R-27: selection enqueued by reduce_table (host array kept)
            o._pct = np.ascontiguousarray(v, dtype=np.float64)
            o.n_percentiles = o._pct.size
            o.percentiles = o._pct.ctypes.data if o._pct.size else None
        else:
            setattr(o, k, v)
    return o


def partials_len(o: ReduceOpts) -> int:
    return int(load().lscat_partials_len(C.byref(o)))


# ---------------------------------------------------------------- device-side objects -----
class _CAI:
    """__cuda_array_interface__ view of a library-owned device buffer (zero copy)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


@dataclass
class Table:
    """Runtime table (a5): torch tensors on the device (or pinned host tensors)."""
    runtime_ms: object
    block_id: object          # int16 storage of uint16 ids
    status: object
    group_offset: object
    group_kernel: object      # int32 storage of uint32
    group_matrix: object
    n_rows: int = 0
    n_groups: int = 0
    rows_per_group: int = 0
    first_group: int = 0
    mem: int = MEM_DEVICE

    @staticmethod
    def empty(cap_rows, cap_groups, device="cuda", pin=False):
        import torch
        kw = dict(device=device) if device != "cpu" else dict(pin_memory=pin)
        return Table(torch.empty(max(cap_rows, 1), dtype=torch.float32, **kw),
                     torch.empty(max(cap_rows, 1), dtype=torch.int16, **kw),
                     torch.empty(max(cap_rows, 1), dtype=torch.uint8, **kw),
                     torch.zeros(cap_groups + 1, dtype=torch.int64, **kw),
                     torch.empty(max(cap_groups, 1), dtype=torch.int32, **kw),
                     torch.empty(max(cap_groups, 1), dtype=torch.int32, **kw),
                     mem=MEM_DEVICE if device != "cpu" else MEM_HOST)

    def __setattr__(self, k, v):  # any attribute change drops the cached C view
        object.__setattr__(self, k, v)
        if k != "_cview":
            object.__setattr__(self, "_cview", None)

    def c_input(self, with_groups=True) -> TableC:
        """c() for calls that only read the table (lscat_reduce_table takes a const table):
        built once and reused until an attribute changes (building it costs ~4 us per call on
        the small tables' critical path)."""
        cv = getattr(self, "_cview", None)
        if cv is None or cv[0] != with_groups:
            cv = (with_groups, self.c(with_groups))
            object.__setattr__(self, "_cview", cv)
        return cv[1]

    def c(self, with_groups=True) -> TableC:
        def p(t):
            return None if t is None else t.data_ptr()
        return TableC(p(self.runtime_ms), p(self.block_id), p(self.status),
                      p(self.group_offset) if with_groups else None,
                      p(self.group_kernel) if with_groups else None,
                      p(self.group_matrix) if with_groups else None,
                      self.runtime_ms.numel(), max(self.group_offset.numel() - 1, 0)
                      if self.group_offset is not None else 0,
                      self.n_rows, self.n_groups, self.rows_per_group, self.mem, self.first_group)

    def to_numpy(self):
        """Host copies (for the oracle and tests)."""
        n, G = self.n_rows, self.n_groups
        d = dict(runtime_ms=self.runtime_ms[:n].cpu().numpy(),
                 block_id=self.block_id[:n].cpu().numpy().view(np.uint16),
                 status=self.status[:n].cpu().numpy() if self.status is not None else None,
                 n_rows=n, n_groups=G, rows_per_group=self.rows_per_group,
                 first_group=self.first_group)
        if self.group_offset is not None:
            d["group_offset"] = self.group_offset[:G + 1].cpu().numpy()
        if self.group_kernel is not None:
            d["group_kernel"] = self.group_kernel[:G].cpu().numpy().view(np.uint32)
        if self.group_matrix is not None:
            d["group_matrix"] = self.group_matrix[:G].cpu().numpy().view(np.uint32)
        return d


_raw_stream = None


def _stream(stream, device=None):
    """The cudaStream_t of `stream` (None: torch's current stream on `device`).  The current
    stream is read with torch's raw-pointer accessor when available (constructing a Stream
    object costs ~3 us per call on the small tables' critical path)."""
    global _raw_stream
    if stream is None:
        import torch
        if device is not None:
            if _raw_stream is None:
                _raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", False)
            if _raw_stream:
                return C.c_void_p(_raw_stream(device))
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


class Ctx:
    """One lscat context per process/rank and device."""

    def __init__(self, device: int = 0, seed: int = 0x15CA7):
        self._lib = load()
        h = C.c_void_p()
        st = self._lib.lscat_ctx_create(device, seed, C.byref(h))
        if st:
            raise LscatError(st, f"ctx_create(device={device}) failed (no CUDA device?)")
        self.h = h
        self.device = device
        self._stats_bufs = {}  # stats(): output struct + host arrays per shape

    def close(self):
        self._reduce_keep = None
        if getattr(self, "h", None):
            self._lib.lscat_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, st, what):
        if st:
            msg = self._lib.lscat_last_error(self.h)
            raise LscatError(st, f"{what}: {msg.decode() if msg else ''}")

    def launch_count(self) -> int:
        n = C.c_uint64()
        self._ck(self._lib.lscat_launch_count(self.h, C.byref(n)), "launch_count")
        return n.value

    # a9 plumbing
    def comm_init(self, unique_id: bytes, rank: int, world: int):
        buf = C.create_string_buffer(unique_id, 128) if unique_id else None
        self._ck(self._lib.lscat_comm_init(self.h, buf, rank, world), "comm_init")

    def comm_init_local(self, name: str, rank: int, world: int):
        """Test transport: ranks are threads of this process (see include/lscat.h)."""
        self._ck(self._lib.lscat_comm_init_local(self.h, name.encode(), rank, world),
                 "comm_init_local")

    # a1
    def register_suite(self, kernels, sizes, stream=None):
        k, kp = _arr(kernels, np.uint32)
        s, sp = _arr(sizes, np.uint32)
        self._ck(self._lib.lscat_register_suite(self.h, kp, k.size, sp, s.size, _stream(stream)),
                 "register_suite")

    def suite_buffer(self, kernel, n, slot):
        p, b = C.c_void_p(), C.c_uint64()
        self._ck(self._lib.lscat_suite_buffer(self.h, kernel, n, slot, C.byref(p), C.byref(b)),
                 "suite_buffer")
        return p.value, b.value

    def suite_tensor(self, kernel, n, slot):
        """Zero-copy torch view of a suite buffer (fp32, or bf16 for the GEMM)."""
        import torch
        p, b = self.suite_buffer(kernel, n, slot)
        if kernel == K_GEMM_BF16:
            t = torch.as_tensor(_CAI(p, (b // 2,), "<i2"), device=f"cuda:{self.device}")
            return t.view(torch.bfloat16)
        return torch.as_tensor(_CAI(p, (b // 4,), "<f4"), device=f"cuda:{self.device}")

    def suite_upload(self, kernel, n, slot, src, stream=None):
        mem = MEM_DEVICE if src.is_cuda else MEM_HOST
        nbytes = src.numel() * src.element_size()
        self._ck(self._lib.lscat_suite_upload(self.h, kernel, n, slot, src.data_ptr(), nbytes,
                                              mem, _stream(stream)), "suite_upload")

    # a3
    def launch(self, kernel, n, block, stream=None):
        self._ck(self._lib.lscat_launch(self.h, kernel, n, block, _stream(stream)), "launch")

    # a4/a5
    def sweep(self, kernels, sizes, blocks, warmup=1, brackets=10, launches=1000,
              timeout_s=30.0, launch_mode=LAUNCH_GRAPH, shard=SHARD_POINT_LPT, spin_ns=0,
              table: Table | None = None, with_brackets=False, stream=None, timer=TIMER_EVENT,
              l2_mode=L2_WARM, with_event_brackets=False, verify_bytes=0) -> Table:
        """a2-a5.  with_brackets -> table.brackets [rows, K] (per-launch ms by `timer`);
        with_event_brackets -> table.brackets_event (the CUDA-event clock of the same brackets);
        verify_bytes > 0 -> table.verify = list of per-row output byte strings (None if NaN)."""
        k, kp = _arr(kernels, np.uint32)
        s, sp = _arr(sizes, np.uint32)
        b, bp = _arr(blocks, np.uint16)
        npts = k.size * s.size * b.size
        if table is None:
            table = Table.empty(npts, k.size * s.size)
        brk = np.full(npts * brackets, np.nan, np.float32) if with_brackets else None
        brk_ev = np.full(npts * brackets, np.nan, np.float32) if with_event_brackets else None
        vbuf = np.zeros(verify_bytes, np.uint8) if verify_bytes else None
        voff = np.zeros(npts + 1, np.uint64) if verify_bytes else None
        o = SweepOpts(bp, b.size, warmup, brackets, launches, timeout_s, launch_mode, shard,
                      0.0, spin_ns, None if brk is None else brk.ctypes.data, timer, l2_mode,
                      None if brk_ev is None else brk_ev.ctypes.data, 1 if verify_bytes else 0,
                      None if vbuf is None else vbuf.ctypes.data, verify_bytes,
                      None if voff is None else voff.ctypes.data)
        tc = table.c()
        self._ck(self._lib.lscat_sweep(self.h, kp, k.size, sp, s.size, C.byref(o), C.byref(tc),
                                       _stream(stream)), "sweep")
        table.n_rows, table.n_groups = tc.n_rows, tc.n_groups
        table.rows_per_group, table.first_group = tc.rows_per_group, tc.first_group
        if with_brackets:
            table.brackets = brk[:tc.n_rows * brackets].reshape(tc.n_rows, brackets)
        if with_event_brackets:
            table.brackets_event = brk_ev[:tc.n_rows * brackets].reshape(tc.n_rows, brackets)
        if verify_bytes:
            table.verify = [bytes(vbuf[int(voff[i]):int(voff[i + 1])]) for i in range(tc.n_rows)]
        return table

    # a6-a9
    def reduce_table(self, table: Table, opts: ReduceOpts, per_group=True, partials=False,
                     stream=None):
        G = table.n_groups
        out = {}
        oc = ReduceOutC()
        if per_group:
            import torch
            dev = f"cuda:{self.device}"
            out = dict(best_block_id=torch.empty(max(G, 1), dtype=torch.int16, device=dev),
                       best_runtime=torch.empty(max(G, 1), dtype=torch.float32, device=dev),
                       perf=torch.empty(max(G, 1), dtype=torch.float64, device=dev),
                       gain=torch.empty(max(G, 1), dtype=torch.float64, device=dev),
                       flags=torch.empty(max(G, 1), dtype=torch.int32, device=dev))
            for k, v in out.items():
                setattr(oc, k, v.data_ptr())
        if partials:
            import torch
            out["partials"] = torch.zeros(partials_len(opts), dtype=torch.int64, device=f"cuda:{self.device}")
            oc.partials = out["partials"].data_ptr()
        tc = table.c_input(with_groups=not table.rows_per_group or table.group_offset is not None)
        self._ck(self._lib.lscat_reduce_table(self.h, C.byref(tc), C.byref(opts), C.byref(oc),
                                              _stream(stream, self.device)), "reduce_table")
        # the library reads the per-group perf/gain again in lscat_stats (keep_values): hold
        # the tensors until the next reduce_table or close, even if the caller drops `out`
        self._reduce_keep = out
        return out

    # a8/a10
    def stats(self, opts: ReduceOpts, percentiles=(), hist=True, stream=None) -> dict:
        pcs = np.ascontiguousarray(percentiles, dtype=np.float64).ravel()
        ML = opts.n_matrices * opts.n_blocks
        nb, cap = opts.bins_per_unit, opts.gain_cap
        # the output struct and its host arrays are cached per shape (argument marshalling is
        # on the small tables' critical path); results are returned as copies
        key = (nb, cap, ML, pcs.size, bool(hist), bool(opts.block_profile), bool(opts.kernel_rollup))
        bufs = self._stats_bufs.get(key)
        if bufs is None:
            so = StatsOutC()
            ph, gh, bh = (np.zeros(nb + 1, np.uint64), np.zeros(cap * nb + 1, np.uint64),
                          np.zeros(ML, np.uint64))
            pc, pp, pg = np.zeros(pcs.size), np.zeros(pcs.size), np.zeros(pcs.size)
            pm, pn, kh = np.zeros(ML), np.zeros(ML, np.uint64), np.zeros(nb + 1, np.uint64)
            if hist:
                so.perf_hist, so.gain_hist, so.best_block_hist = (ph.ctypes.data, gh.ctypes.data,
                                                                  bh.ctypes.data)
            if pcs.size:
                so.percentiles, so.n_percentiles = pc.ctypes.data, pcs.size
                so.pct_perf, so.pct_gain = pp.ctypes.data, pg.ctypes.data
            if opts.block_profile:
                so.profile_mean, so.profile_count = pm.ctypes.data, pn.ctypes.data
            if opts.kernel_rollup:
                so.kernel_perf_hist = kh.ctypes.data
            # views over the struct's counters and derived doubles (no per-call bytes() copy)
            cv = np.frombuffer(so, np.uint64, len(COUNTERS))
            dv = np.frombuffer(so, np.float64, len(DERIVED), 8 * len(COUNTERS))
            bufs = (so, ph, gh, bh, pc, pp, pg, pm, pn, kh, cv, dv)
            self._stats_bufs[key] = bufs
        so, ph, gh, bh, pc, pp, pg, pm, pn, kh, cv, dv = bufs
        pc[:] = pcs
        pp.fill(np.nan)
        pg.fill(np.nan)
        self._ck(self._lib.lscat_stats(self.h, C.byref(opts), C.byref(so), _stream(stream, self.device)),
                 "stats")
        # counters (u64) then the derived doubles, in COUNTERS / DERIVED order
        res = dict(zip(COUNTERS, cv.tolist()))
        res.update(zip(DERIVED, dv.tolist()))
        if hist:
            res["perf_hist"], res["gain_hist"] = ph.copy(), gh.copy()
            res["best_block_hist"] = bh.reshape(opts.n_matrices, opts.n_blocks).copy()
        if pcs.size:
            res["pct_perf"], res["pct_gain"] = pp.tolist(), pg.tolist()
        if opts.kernel_rollup:
            res.update({k: int(getattr(so, k)) for k in ROLLUP})
            res.update({k: float(getattr(so, k)) for k in ROLLUP_DERIVED})
            res["kernel_perf_hist"] = kh.copy()
        if opts.block_profile:
            res["profile_mean"] = pm.reshape(opts.n_matrices, opts.n_blocks).copy()
            res["profile_count"] = pn.reshape(opts.n_matrices, opts.n_blocks).copy()
        return res

    # group an unordered dataframe into a table
    def ingest(self, kernel, matrix, block_id, runtime, status=None, stream=None) -> Table:
        """CUDA tensors [n]: kernel (int32/uint32), matrix (int32), block_id (int16), runtime
        (float32), status (uint8, optional).  Returns the grouped Table."""
        n = runtime.numel()
        table = Table.empty(n, n)
        tc = table.c()
        dups = C.c_uint64()
        st = self._lib.lscat_ingest(self.h, kernel.data_ptr(), matrix.data_ptr(),
                                    block_id.data_ptr(), runtime.data_ptr(),
                                    None if status is None else status.data_ptr(), n,
                                    C.byref(tc), C.byref(dups), _stream(stream))
        table.n_rows, table.n_groups = tc.n_rows, tc.n_groups
        table.duplicates = dups.value
        self._ck(st, "ingest")
        return table

    # occupancy-API block and timeout economics
    def occupancy_block(self, kernel, blocks):
        """{'block_id': index into blocks of the occupancy calculator's choice, 'min_grid': the
        API's minGridSize at that block, 'info': per-candidate dicts (lscat_occupancy_info)}."""
        b, bp = _arr(blocks, np.uint16)
        info = (OccInfo * b.size)()
        out = C.c_uint32()
        self._ck(self._lib.lscat_occupancy_block(self.h, kernel, bp, b.size, C.byref(out), info),
                 "occupancy_block")
        rows = [{f: getattr(x, f) for f, _ in OccInfo._fields_} for x in info]
        return {"block_id": out.value, "min_grid": rows[out.value]["api_min_grid"], "info": rows}

    def timeout_curve(self, table: Table, taus, warmup=1, brackets=10, launches=1000,
                      stream=None):
        t, tp = _arr(taus, np.float64)
        cnt = np.zeros(t.size, np.uint64)
        tc = table.c()
        self._ck(self._lib.lscat_timeout_curve(self.h, C.byref(tc), warmup, brackets, launches,
                                               tp, t.size, cnt.ctypes.data, _stream(stream)),
                 "timeout_curve")
        return cnt

    # the paper's aggregation experiment
    AGG_METHODS = ("mean", "median", "min", "max", "trimmed_mean_20")

    def aggregation_experiment(self, pool, k=10, reps=10_000, seed=0, aggregates=False,
                               stream=None):
        """pool: 1-D float32 CUDA tensor.  Returns {method: spread} (+ per-rep aggregates)."""
        import torch
        sp = np.zeros(5)
        mn = np.zeros(5)
        agg = torch.empty(5 * reps, dtype=torch.float64, device=pool.device) if aggregates else None
        self._ck(self._lib.lscat_aggregation_experiment(
            self.h, pool.data_ptr(), pool.numel(), k, reps, seed, sp.ctypes.data, mn.ctypes.data,
            None if agg is None else agg.data_ptr(), _stream(stream)), "aggregation_experiment")
        out = {"spread": dict(zip(self.AGG_METHODS, sp.tolist())),
               "mean": dict(zip(self.AGG_METHODS, mn.tolist()))}
        if aggregates:
            out["aggregates"] = agg.view(5, reps).cpu().numpy()
        return out

    # synthetic tables
    def gen_table(self, n_rows_global, n_kernels, n_blocks=32, largest_block_id=None,
                  n_matrices=8, preset=PRESET_T4, nan_rate=0.03, seed=0, group_begin=0,
                  group_end=0, block_mod=1, block_rem=0, offsets=True, stream=None) -> Table:
        import torch
        o = GenOpts(n_rows_global, n_kernels, n_blocks,
                    n_blocks - 1 if largest_block_id is None else largest_block_id, n_matrices,
                    preset, nan_rate, seed, group_begin, group_end, block_mod, block_rem)
        nr, ng = C.c_uint64(), C.c_uint64()
        st = self._lib.lscat_gen_table_shape(C.byref(o), C.byref(nr), C.byref(ng))
        if st:
            raise LscatError(st, "gen_table_shape")
        dev = f"cuda:{self.device}"
        t = Table(torch.empty(max(nr.value, 1), dtype=torch.float32, device=dev),
                  torch.empty(max(nr.value, 1), dtype=torch.int16, device=dev),
                  torch.empty(max(nr.value, 1), dtype=torch.uint8, device=dev),
                  torch.empty(ng.value + 1, dtype=torch.int64, device=dev) if offsets else None,
                  torch.empty(max(ng.value, 1), dtype=torch.int32, device=dev) if offsets else None,
                  torch.empty(max(ng.value, 1), dtype=torch.int32, device=dev) if offsets else None)
        tc = TableC(t.runtime_ms.data_ptr(), t.block_id.data_ptr(), t.status.data_ptr(),
                    t.group_offset.data_ptr() if offsets else None,
                    t.group_kernel.data_ptr() if offsets else None,
                    t.group_matrix.data_ptr() if offsets else None,
                    t.runtime_ms.numel(), ng.value, 0, 0, 0, MEM_DEVICE, 0)
        self._ck(self._lib.lscat_gen_table(self.h, C.byref(o), C.byref(tc), _stream(stream)),
                 "gen_table")
        t.n_rows, t.n_groups = tc.n_rows, tc.n_groups
        t.rows_per_group, t.first_group = tc.rows_per_group, tc.first_group
        if not offsets and not t.rows_per_group:
            raise LscatError(ERR_INVALID_ARG, "gen_table: ragged table needs offsets")
        return t
