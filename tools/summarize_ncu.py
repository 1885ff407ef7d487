"""Summarise ncu CSV exports (launch list + raw pages) into markdown for profiles/.

usage: python tools/summarize_ncu.py <launches.csv> <raw.csv> [<raw.csv> ...] > profiles/rNN_x.md
"""
import collections
import csv
import io
import re
import sys


def _rows(path):
    text = open(path).read().splitlines()
    start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
    return list(csv.reader(io.StringIO("\n".join(text[start:]))))


def short(name):
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"\(.*$", "", name)
    return name.replace("rbws::", "")


def launch_list(path):
    rows = _rows(path)
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    per = collections.OrderedDict()
    total = 0.0
    n = 0
    for r in rows[1:]:
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue
        ns = float(r[vi].replace(",", ""))
        k = short(r[ki])
        t, c = per.get(k, (0.0, 0))
        per[k] = (t + ns, c + 1)
        total += ns
        n += 1
    out = [f"launches in the timed region: {n}, summed device time {total/1e6:.3f} ms "
           "(cold-cache, serialised under ncu)\n",
           "| kernel | launches | ms total | us/launch | share |", "|---|---:|---:|---:|---:|"]
    for k, (t, c) in sorted(per.items(), key=lambda kv: -kv[1][0]):
        out.append(f"| `{k}` | {c} | {t/1e6:.3f} | {t/c/1e3:.1f} | {t/total:.3f} |")
    return "\n".join(out)


WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %"),
    ("sm__inst_executed.sum", "inst"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "fp64 cycles %"),
]


def raw(path):
    rows = _rows(path)
    h = rows[0]
    units = rows[1] if rows[1][0] == "" else None
    body = rows[2:] if units else rows[1:]
    ki = h.index("Kernel Name")
    cols = [(h.index(m), lab) for m, lab in WANT if m in h]
    out = ["| kernel | grid | " + " | ".join(l for _, l in cols) + " |",
           "|---|---|" + "---:|" * len(cols)]
    gi = h.index("Grid Size") if "Grid Size" in h else None
    for r in body:
        vals = []
        for i, lab in cols:
            v = r[i]
            u = units[i] if units else ""
            try:
                x = float(v.replace(",", ""))
                if lab.startswith("dram r") or lab.startswith("dram w"):
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
                    v = f"{x*scale/1e6:.1f} MB"
                elif lab == "time":
                    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3,
                             "ms": 1e3}.get(u, 1)
                    v = f"{x*scale:.1f} us"
                elif lab == "inst":
                    v = f"{x/1e6:.1f} M"
                else:
                    v = f"{x:.1f}" if x != int(x) else f"{int(x)}"
            except ValueError:
                pass
            vals.append(v)
        out.append(f"| `{short(r[ki])}` | {r[gi] if gi is not None else ''} | " + " | ".join(vals) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    print("## launch list\n")
    print(launch_list(sys.argv[1]))
    for p in sys.argv[2:]:
        print(f"\n## full capture: {p.split('/')[-1]}\n")
        print(raw(p))
