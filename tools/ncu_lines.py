"""Per-source-line / per-region / per-opcode breakdown of an ncu source export.

    ncu -i rep --page source --csv --print-source cuda,sass > /tmp/src_cs.csv
    python tools/ncu_lines.py /tmp/src_cs.csv [top]
"""
import collections
import csv
import re
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
cur = None
line = None
agg = {}
ops = collections.Counter()
opsamp = collections.Counter()
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if not r or r[0] in ("Line No", "Function Name"):
        continue
    if r[0] != "":
        try:
            line = (cur, int(r[0]))
            agg[line] = [int(r[4]), int(r[7]), r[1][:100].strip()]
        except ValueError:
            pass
        continue
    try:
        ie = int(r[7])
        s = int(r[4])
    except ValueError:
        continue
    src = re.sub(r"^@!?U?P\w+\s+", "", r[3].strip())
    op = src.split()[0].split(".")[0] if src else "?"
    ops[op] += ie
    opsamp[op] += s
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total samples {ts}, warp instructions {ti}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / ts * 100:5.1f}% smp {v[1] / ti * 100:5.1f}% ins  {k[0]}:{k[1]} {v[2]}")
print("opcodes:")
to = sum(ops.values()) or 1
so = sum(opsamp.values()) or 1
for o, c in ops.most_common(25):
    print(f"  {o:10s} {c / to * 100:5.1f}% ins {opsamp[o] / so * 100:5.1f}% smp")
