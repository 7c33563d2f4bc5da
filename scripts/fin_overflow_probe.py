"""Dense-sub-bin table on the sampled selection path (test_percentiles_sampled_finish_overflow)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from tests.test_gpu_reduce import _compare  # noqa: E402

rng = np.random.default_rng(5)
G = 2_500_000
b = rng.uniform(0.5, 2.0, G).astype(np.float32)
dense = rng.random(G) < 0.4
j = rng.integers(1, 5, G).astype(np.float32)
t = np.where(dense, b * (np.float32(1) + j * np.float32(2.0 ** -22)),
             b * rng.uniform(1.0, 4.0, G).astype(np.float32)).astype(np.float32)
rt = np.empty(2 * G, np.float32)
rt[0::2], rt[1::2] = b, t
tab = dict(runtime_ms=rt, block_id=np.tile(np.array([0, 1], np.uint16), G),
           group_offset=np.arange(0, 2 * G + 1, 2, dtype=np.int64), group_matrix=np.zeros(G, np.uint32))
_compare(tab, L=2, M=1, ell=1, pcts=[0.05, 0.3, 0.5, 0.7, 0.95])
print("ok")
