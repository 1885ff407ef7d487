"""Per-kernel SASS opcode mix and stall reasons from an `ncu --page source --csv` export.

usage: python tools/ncu_source_summary.py <source.csv> <nodes per launch> [top_lines]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
nodes = float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 0
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and r:
        cur["rows"].append(r)
for b in blocks:
    h = b["hdr"]
    si, ie = h.index("Source"), h.index("Instructions Executed")
    sa = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    ops, st, tot, lines = collections.Counter(), collections.Counter(), 0, []
    for r in b["rows"]:
        try:
            n = int(r[ie].replace(",", ""))
        except ValueError:
            continue
        toks = r[si].split()
        op = (toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")).split(".")[0]
        ops[op] += n
        tot += n
        for c in stall_cols:
            try:
                st[c] += int(r[h.index(c)].replace(",", ""))
            except ValueError:
                pass
        try:
            lines.append((int(r[sa].replace(",", "")), r[0], r[si]))
        except ValueError:
            pass
    print(b["name"][:90])
    print("  thread-instructions per node:", round(tot * 32 / nodes, 1))
    print("  ", [(k, round(v * 32 / nodes, 1)) for k, v in ops.most_common(16)])
    s = sum(st.values()) or 1
    print("   stalls:", [(k[6:], round(v / s, 3)) for k, v in st.most_common(8)])
    for smp, addr, src in sorted(lines, reverse=True)[:top]:
        print(f"     {smp:7d} {addr} {src}")
