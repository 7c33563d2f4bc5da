"""Per-(N, block) runtime matrix of one suite kernel's sweep (probe, not a bench line).

    python scripts/sweep_dump.py [kernel=0] [brackets=3] [launches=1000]

Prints one line per N: min / median / max us per launch over the blocks, the sum of
(W + K*R) * runtime over the blocks (that N's share of a sweep step), and the full row.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402

kern = int(sys.argv[1]) if len(sys.argv) > 1 else L.K_EUCLID
K = int(sys.argv[2]) if len(sys.argv) > 2 else 3
R = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
ns = [64 << i for i in range(8)]
bs = list(range(32, 1025, 32))
c = L.Ctx(0)
c.register_suite([kern], ns)
tab = c.sweep([kern], ns, bs, warmup=1, brackets=K, launches=R).to_numpy()
rt = tab["runtime_ms"][: tab["n_rows"]].reshape(len(ns), len(bs)) * 1e3
tot = 0.0
for i, n in enumerate(ns):
    r = rt[i]
    s = float(np.nansum(r)) * (1 + 10 * 1000) * 1e-6
    tot += s
    print(f"N={n:5d} min {np.nanmin(r):8.2f} med {np.nanmedian(r):8.2f} max {np.nanmax(r):8.2f} us"
          f"  paper-policy s {s:6.2f}  best block {bs[int(np.nanargmin(r))]}")
    print("   ", " ".join(f"{x:.1f}" for x in r))
print(f"paper-policy step estimate {tot:.2f} s -> {len(ns) * len(bs) / tot:.2f} points/s")
