"""Launch list (ncu --csv with gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum)
-> markdown table per kernel and the per-class DRAM traffic json bench.py reads.

usage: python tools/launch_summary.py <launches.csv> <out.md> [traffic.json]
"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
H = rows[h]
ki, mi, vi, ui = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value"), H.index("Metric Unit")
idi = H.index("ID")
per = collections.OrderedDict()
for r in rows[h + 1:]:
    if len(r) <= vi or not r[idi].isdigit():
        continue
    d = per.setdefault(r[idi], {"name": r[ki]})
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    if r[mi] == "gpu__time_duration.sum":
        d["us"] = v / 1e3 if unit in ("ns", "nsecond") else (v if unit.startswith("us") else v * 1e3)
    elif r[mi].startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        d["dram"] = d.get("dram", 0.0) + v * scale
agg = collections.OrderedDict()
for d in per.values():
    a = agg.setdefault(d["name"], {"n": 0, "us": 0.0, "dram": 0.0, "max_us": 0.0, "dram_at_max": 0.0})
    a["n"] += 1
    a["us"] += d.get("us", 0.0)
    a["dram"] += d.get("dram", 0.0)
    if d.get("us", 0.0) > a["max_us"]:
        a["max_us"], a["dram_at_max"] = d["us"], d.get("dram", 0.0)
tot = sum(a["us"] for a in agg.values())
with open(sys.argv[2], "w") as f:
    f.write(f"{len(per)} launches, total {tot / 1e3:.2f} ms (ncu serialised, cold)\n\n")
    f.write("| share | launches | us / launch | longest launch us | DRAM GB/s | kernel |\n|---:|---:|---:|---:|---:|---|\n")
    for name, a in sorted(agg.items(), key=lambda x: -x[1]["us"]):
        if a["us"] / tot < 0.001:
            continue
        gbs = a["dram"] / (a["us"] * 1e-6) / 1e9 if a["us"] else 0.0
        f.write(f"| {a['us'] / tot:.3f} | {a['n']} | {a['us'] / a['n']:.1f} | {a['max_us']:.1f} | "
                f"{gbs:.0f} | `{name[:70]}` |\n")
print(open(sys.argv[2]).read())
if len(sys.argv) > 3:
    # full-batch launches (the longest of each fine kernel) against their algorithmic bytes
    nodes, inst = 63 ** 3, 1024
    classes = {"fine_cg_update": ("cgp_kernel<64>", 42.0), "fine_cg_update_separate": ("fine_kernel<4, 64", 40.0),
               "fine_p_update_apply_dot": ("fine_kernel<5, 64", 24.0),
               "fine_prolong_post_smooth": ("fine_kernel<6, 64", 25.0),
               "fine_pre_residual": ("fine_kernel<7, 64", 10.0), "fine_resid": ("fine_kernel<1, 64", 16.0)}
    out = {"source": f"{sys.argv[1]}: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                     "dram__bytes_write.sum, the longest (full-batch, 1024 active instances, 64^3) "
                     "launch of each kernel"}
    for cls, (pat, bpn) in classes.items():
        for name, a in agg.items():
            if pat in name and a["dram_at_max"] > 0:
                out[cls] = {"dram_bytes": int(a["dram_at_max"]), "algorithmic_bytes": int(bpn * nodes * inst),
                            "us": a["max_us"]}
    json.dump(out, open(sys.argv[3], "w"), indent=1)
    print(json.dumps(out, indent=1))
