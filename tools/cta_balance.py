"""Load balance of every grid step of one solve (DS_TRACE=2): per step the
spread of the CTAs' finish times.  For each step kind: time, the mean CTA
idle share (waiting for the slowest CTA) and the barrier latency (last CTA
finished -> barrier released)."""
import collections, os, sys, ctypes
os.environ["DS_TRACE"] = "2"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1911_06895_b200 import DeviceGraph, graphs, _lib

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
delta = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
L = _lib.lib()
L.ds_debug_cta_times.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
L.ds_debug_cta_times.restype = ctypes.c_int64
g = DeviceGraph.rmat(scale, 16, 1, 2)
ip = g.download_indptr()
s = graphs.pick_sources(ip, 64, seed=7)[0]
g.solve(s, delta)
st = g.solve(s, delta)
cap = 1 << 16
buf = np.zeros(1 + 2 * cap, dtype=np.uint64)
m = L.ds_debug_trace(g._handle(), buf.ctypes.data, cap)
t0 = int(buf[0]); ts = buf[1::2][:m].astype(np.int64); info = buf[2::2][:m]
kinds = (info >> np.uint64(56)).astype(int)
cbuf = np.zeros(1 + m * 200, dtype=np.uint64)
w = L.ds_debug_cta_times(g._handle(), cbuf.ctypes.data, cbuf.size)
grid = int(cbuf[0])
done = cbuf[1:1 + w].astype(np.int64).reshape(-1, grid)[:m]
names = ["scan", "l_relax", "l_capt", "h_capt", "h_relax", "l_pull", "l_commit", "h_pull", "h_commit",
         "l_local", "h_local", "u_capt", "h_gather"]
starts = np.concatenate([[t0], ts[:-1]])
agg = collections.defaultdict(lambda: np.zeros(4))
for i in range(m):
    dur = ts[i] - starts[i]
    last = done[i].max()
    idle = (last - done[i]).mean()
    a = agg[names[kinds[i]]]
    a += [1, dur, idle, ts[i] - last]
print(f"R-MAT {scale} delta {delta}: kernel {st.kernel_ms:.3f} ms, {m} steps, grid {grid}")
print(f"{'kind':10s} {'n':>4s} {'time ms':>8s} {'CTA idle ms':>12s} {'barrier ms':>11s}")
for k, (n, dur, idle, bar) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:10s} {int(n):4d} {dur/1e6:8.3f} {idle/1e6:12.3f} {bar/1e6:11.3f}")
tot = sum(a[1] for a in agg.values()); idl = sum(a[2] for a in agg.values()); br = sum(a[3] for a in agg.values())
print(f"total {tot/1e6:.3f} ms: mean CTA idle {idl/1e6:.3f} ms ({100*idl/tot:.0f}%), barrier {br/1e6:.3f} ms ({100*br/tot:.0f}%)")
print("largest steps: kind, work, time us, CTA idle us, barrier us")
order = np.argsort(-(ts - starts))[:14]
for i in sorted(order):
    dur = ts[i] - starts[i]
    last = done[i].max()
    print(f"  {i:4d} {names[kinds[i]]:9s} {int(info[i] & np.uint64((1 << 56) - 1)):11d} {dur/1e3:8.1f} "
          f"{(last - done[i]).mean()/1e3:8.1f} {(ts[i]-last)/1e3:6.1f}")
small = (ts - starts) < 15000
print(f"steps < 15 us: {int(small.sum())}, their total {((ts - starts)[small]).sum()/1e6:.3f} ms")
