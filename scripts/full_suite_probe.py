import os, sys, json
sys.path.insert(0, os.getcwd())
import bench
import paper_2103_14409_b200 as L
c = L.Ctx(0, seed=0x15CA7)
print(json.dumps(bench.full_suite_sweep(c, L, L.LAUNCH_GRAPH_PDL)))
