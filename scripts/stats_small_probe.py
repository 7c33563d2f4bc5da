import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2103_14409_b200 as L
c = L.Ctx(0)
tab = c.gen_table(n_rows_global=2_140_796, n_kernels=8363, preset=L.PRESET_GTX980, seed=980)
o = L.reduce_opts(32, 8)
for i in range(3):
    c.reduce_table(tab, o, per_group=False)
    c.stats(o, percentiles=[0.01, 0.05, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99])
torch.cuda.synchronize()
