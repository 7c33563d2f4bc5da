#!/bin/bash
# A/B of the small-N row-kernel variant (LSCAT_ROW_SMALL=0: the 8-deep kernel at every N),
# interleaved, plain graph brackets, euclid at N = 64..2048 over the 32 blocks.
cat > /tmp/ab_small.py <<'PY'
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2103_14409_b200 as L
c = L.Ctx(0)
ns = [64, 128, 256, 512, 1024, 2048]
bs = list(range(32, 1025, 32))
c.register_suite([L.K_EUCLID], ns)
c.sweep([L.K_EUCLID], ns, bs, warmup=1, brackets=2, launches=50)
t = c.sweep([L.K_EUCLID], ns, bs, warmup=1, brackets=5, launches=500).to_numpy()
rt = t["runtime_ms"] * 1e3
print(json.dumps({"tag": sys.argv[1], **{str(n): [round(float(rt[i*32:(i+1)*32].min()), 3), round(float(rt[i*32:(i+1)*32].mean()), 3), round(float(rt[i*32:(i+1)*32].max()), 3)] for i, n in enumerate(ns)}}))
PY
for i in 1 2; do
  LSCAT_ROW_SMALL=0 python /tmp/ab_small.py deep8
  python /tmp/ab_small.py default_small2_to256_small4_to1024
  LSCAT_ROW_SMALL4_MAX=2048 python /tmp/ab_small.py small4_to2048
done
