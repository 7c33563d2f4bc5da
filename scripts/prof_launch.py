"""Launch one suite kernel `count` times (for ncu / compute-sanitizer captures).

    python scripts/prof_launch.py <kernel name> <N> <block> <count>
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

name, n, block, count = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
c = L.Ctx(0)
k = L.KERNELS[name]
c.register_suite([k], [n])
for _ in range(count):
    c.launch(k, n, block)
torch.cuda.synchronize()
print("launched", name, n, block, count)
c.close()
