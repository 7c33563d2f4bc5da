"""B200-native LS-CAT hot path (arXiv 2103.14409): thread-block-size sweep + runtime-table
statistics, behind the C ABI of include/lscat.h.  See DESIGN.md.

The package holds only the path: csrc/ (CUDA for sm_100a + the C ABI), the ctypes binding
(lscat.py) and its build script.  It never imports oracle/ (test infrastructure).
"""
from .lscat import (  # noqa: F401
    Ctx, Table, LscatError, load, plan, kernel_work, reduce_opts, partials_len, comm_unique_id,
    KERNELS, K_EUCLID, K_MATVEC, K_GEMM_BF16, K_TRANSPOSE, K_AXPY, K_ROWSUM, K_COLSUM,
    K_STENCIL5, K_SPIN, SLOT_IN0, SLOT_IN1, SLOT_OUT, MEM_DEVICE, MEM_HOST, LAUNCH_GRAPH, LAUNCH_GRAPH_PDL,
    LAUNCH_STREAM, SHARD_POINT_LPT, SHARD_GROUP, SKIPNA, COMPLETE_ONLY, PRESET_T4,
    PRESET_GTX980, ROW_OK, ROW_TIMEOUT, ROW_LAUNCH_ERROR, ROW_INVALID_CONFIG, GF, COUNTERS,
    EXPORTS, OK, ERR_INVALID_ARG, ERR_CUDA, ERR_STATE, ERR_UNSUPPORTED, TIMER_EVENT,
    TIMER_GLOBALTIMER, L2_WARM, L2_ROTATE,
)
