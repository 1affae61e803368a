"""Repeated solves across lex / classic prepares: time, work and barriers."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_06895_b200 import DeviceGraph, graphs
g = DeviceGraph.rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 24, 16, 1, 2)
ip = g.download_indptr()
pool = graphs.pick_sources(ip, 64, seed=7)
for env in ("0", None, "0", None):
    if env is None:
        os.environ.pop("DS_LEX", None)
    else:
        os.environ["DS_LEX"] = env
    info = g.prepare(0.1)
    for s in [pool[1], pool[1], pool[2]]:
        st = g.solve(s, 0.1)
        print(f"DS_LEX={env} ksub={info.sub_buckets} src={s} ms={st.kernel_ms:.2f} scanned={st.edges_scanned} "
              f"barriers={st.grid_barriers} pulls={st.pull_steps} phases={st.inner_phases}", flush=True)
