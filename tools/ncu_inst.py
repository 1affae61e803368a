"""Instructions executed and L1 tag requests per CUDA source line of an ncu report
(source page), top N lines by warp-level instructions.
usage: python tools/ncu_inst.py report.ncu-rep [topN]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None; hdr = None; out = []
for r in csv.reader(io.StringIO(txt)):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; col = {c: i for i, c in enumerate(hdr)}; continue
    if hdr and len(r) > 4 and r[2] == "-":
        def f(name):
            try: return float(r[col[name]] or 0)
            except (KeyError, ValueError): return 0.0
        out.append((f("Instructions Executed"), f("L1 Tag Requests Global"), f("# Samples"), cur, r[0], r[1][:90]))
ti = sum(o[0] for o in out) or 1; tt = sum(o[1] for o in out) or 1; ts = sum(o[2] for o in out) or 1
print(f"total warp instructions {ti:.3e}, L1 tag requests (global) {tt:.3e}, samples {ts:.0f}")
for i, t, s, f_, l, src in sorted(out, key=lambda x: -x[0])[:top]:
    print(f"inst {100*i/ti:5.1f}%  tags {100*t/tt:5.1f}%  samples {100*s/ts:5.1f}%  {f_}:{l:5s} {src}")
print("--- by L1 tag requests")
for i, t, s, f_, l, src in sorted(out, key=lambda x: -x[1])[:20]:
    print(f"inst {100*i/ti:5.1f}%  tags {100*t/tt:5.1f}%  samples {100*s/ts:5.1f}%  {f_}:{l:5s} {src}")
