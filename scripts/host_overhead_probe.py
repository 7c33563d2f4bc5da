"""Host-side cost of the binding's table calls on a small table (configs[2] shape): the
Python marshalling pieces against the raw C-ABI call (graph-replayed reduce_table)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402
from paper_2103_14409_b200 import lscat as M  # noqa: E402

PCTS = [0.01, 0.05, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99]
c = L.Ctx(0)
tab = c.gen_table(2_140_796, 8363, preset=L.PRESET_GTX980, seed=980)
o = L.reduce_opts(32, 8, percentiles=PCTS)
for _ in range(5):
    c.reduce_table(tab, o, per_group=False)
    c.stats(o, percentiles=PCTS)
torch.cuda.synchronize()


def t(f, n=2000):
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    return (time.perf_counter() - t0) / n * 1e6


res = {}
res["current_stream"] = t(lambda: torch.cuda.current_stream())
res["_stream(None)"] = t(lambda: M._stream(None))
res["table.c"] = t(lambda: tab.c(with_groups=True))
res["table.c_input"] = t(lambda: tab.c_input(with_groups=True))
tc = tab.c(with_groups=True)
oc = M.ReduceOutC()
sp = M._stream(None)
lib = c._lib


def raw():
    lib.lscat_reduce_table(c.h, C.byref(tc), C.byref(o), C.byref(oc), sp)


res["raw reduce_table (graph replay)"] = t(raw, 500)
torch.cuda.synchronize()
res["binding reduce_table"] = t(lambda: c.reduce_table(tab, o, per_group=False), 500)
torch.cuda.synchronize()


def both():
    c.reduce_table(tab, o, per_group=False)
    c.stats(o, percentiles=PCTS)


res["reduce_table + stats (incl. GPU)"] = t(both, 300)
print({k: round(v, 2) for k, v in res.items()})
