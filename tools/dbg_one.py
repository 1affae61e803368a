import sys, os; sys.path.insert(0, ".")
from paper_1911_06895_b200 import DeviceGraph, graphs
sc = int(sys.argv[1])
g = DeviceGraph.rmat(sc, 16, 1, 2)
ip = g.download_indptr()
s = graphs.pick_sources(ip, 1, seed=7)[0]
try:
    st = g.solve(s, 0.1); print(os.environ.get("DS_LEX"), sc, "ok", st.inner_phases, flush=True)
except Exception as e:
    print(os.environ.get("DS_LEX"), sc, "FAIL", e, flush=True)
