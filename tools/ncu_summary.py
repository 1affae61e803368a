"""Summarise an `ncu --page raw --csv` export of the solver launches of one
source into profiles/<round>_ncu_summary.json (bench.py reads
traffic_bytes_per_launch from the newest one)."""
import csv, json, sys

raw, out, command = sys.argv[1], sys.argv[2], sys.argv[3]
workload = sys.argv[4] if len(sys.argv) > 4 else "rmat24_ef16_delta0.1, bench pool source 0 (tools/one_source.py)"
rows = list(csv.reader(open(raw)))
hdr, data = rows[0], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


def f(r, k):
    try:
        return float(r[col[k]].replace(",", ""))
    except (KeyError, ValueError):
        return None


launches = []
for r in data:
    name = r[col["Kernel Name"]]
    ms = f(r, "gpu__time_duration.sum")
    unit = rows[1][col["gpu__time_duration.sum"]]
    if unit == "ns":
        ms /= 1e6
    elif unit == "us":
        ms /= 1e3
    launches.append({
        "kernel": name.split("(")[0],
        "ms": ms,
        "dram_read": f(r, "dram__bytes_read.sum"),
        "dram_write": f(r, "dram__bytes_write.sum"),
        "l2_hit_pct": f(r, "lts__t_sector_hit_rate.pct"),
        "dram_pct": f(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "warps_active_pct": f(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": f(r, "launch__registers_per_thread"),
    })
# dram byte units
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
    u = rows[1][col[k]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
    for L in launches:
        key = "dram_read" if "read" in k else "dram_write"
        if L[key] is not None:
            L[key] *= scale
tot = sum((L["dram_read"] or 0) + (L["dram_write"] or 0) for L in launches)
json.dump({
    "workload": workload,
    "command": command,
    "launches_of_one_source": launches,
    "gpu_time_ms": sum(L["ms"] for L in launches),
    "traffic_bytes_per_launch": tot,
    "note": "one solve = the persistent kernel segments plus the handed-off giant pushes; "
            "traffic_bytes_per_launch sums them (bytes per source solve, cold caches under ncu)",
}, open(out, "w"), indent=1)
print(json.dumps({"launches": len(launches), "gpu_time_ms": sum(L["ms"] for L in launches), "traffic": tot}))
