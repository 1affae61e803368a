"""Aggregate ncu source-page warp-stall samples per CUDA source line.
usage: python tools_ncu_lines.py report.ncu-rep [topN]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None; hdr = None; out = []
for r in csv.reader(io.StringIO(txt)):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; continue
    if hdr and len(r) > 4 and r[2] == "-":  # cuda line rows carry aggregated metrics
        try: s = float(r[4] or 0)
        except ValueError: continue
        stalls = {}
        for i, c in enumerate(hdr):
            if c.startswith("stall_") and "Not Issued" not in c:
                try: stalls[c] = float(r[i] or 0)
                except ValueError: pass
        best = sorted(stalls.items(), key=lambda x: -x[1])[:2]
        out.append((s, cur, r[0], r[1][:80], best))
tot = sum(o[0] for o in out) or 1
for s, f, l, t, b in sorted(out, key=lambda x: -x[0])[:top]:
    print(f"{100*s/tot:5.1f}% {f}:{l:5s} {t:80s} {[(k[6:], int(v)) for k, v in b]}")
