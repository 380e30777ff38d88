"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel name:
total us, launches, share.   python tools/ncu_launch_summary.py launches.csv"""
import csv
import re
import sys
from collections import defaultdict


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("<unnamed>::", "")
        v = float(r[vi].replace(",", ""))
        unit = r[h.index("Metric Unit")] if "Metric Unit" in h else "ns"
        us = v / 1000.0 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1000.0)
        tot[name] += us
        cnt[name] += 1
    T = sum(tot.values())
    print(f"total {T:.1f} us over {sum(cnt.values())} launches")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{v:12.1f} us {100 * v / T:6.2f}%  {cnt[k]:6d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
