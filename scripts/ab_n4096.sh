#!/bin/bash
# A/B at N = 4096 (A = 67 MB, L2-resident in WARM mode): load depth / register budget and the
# L2 keep share, interleaved, plain graph brackets, euclid over the 32 blocks.
cat > /tmp/ab_4096.py <<'PY'
import json, os, sys
sys.path.insert(0, os.getcwd())
import paper_2103_14409_b200 as L
c = L.Ctx(0)
ns = [4096, 8192]
bs = list(range(32, 1025, 32))
c.register_suite([L.K_EUCLID], ns)
c.sweep([L.K_EUCLID], ns, bs, warmup=1, brackets=2, launches=50)
t = c.sweep([L.K_EUCLID], ns, bs, warmup=1, brackets=5, launches=500).to_numpy()
rt = t["runtime_ms"] * 1e3
print(json.dumps({"tag": sys.argv[1], **{str(n): [round(float(rt[i*32:(i+1)*32].min()), 3), round(float(rt[i*32:(i+1)*32].mean()), 3), round(float(rt[i*32:(i+1)*32].max()), 3)] for i, n in enumerate(ns)}}))
PY
for i in 1 2; do
  python /tmp/ab_4096.py default
  LSCAT_ROW_SMALL4_MAX=4096 python /tmp/ab_4096.py small4_to4096
  LSCAT_ROW_L2FRAC=0.6 python /tmp/ab_4096.py l2share0.6
  LSCAT_ROW_SMALL4_MAX=4096 LSCAT_ROW_L2FRAC=0.6 python /tmp/ab_4096.py both
done
