"""Summarise an ncu launch list (--metrics gpu__time_duration.sum[,dram bytes] --csv)
into per-kernel share of the step: python tools/launch_summary.py file.csv"""
import collections
import csv
import gzip
import re
import sys


def short(name: str) -> str:
    n = re.sub(r"\(.*", "", name)
    n = re.sub(r"<.*", "", n)
    n = n.replace("void ", "").replace("tim::", "")
    if "nvjet" in n or "gemm" in n.lower() or "cutlass" in n:
        n = "cuBLAS " + n.split("_")[0] if "nvjet" in n else n
    return n


def main(path):
    opener = gzip.open if path.endswith(".gz") else open
    rows = [r for r in csv.reader(line for line in opener(path, "rt") if line.startswith('"'))]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = short(r[ki])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for i, m in per.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a = agg[names[i]]
        a[0] += 1
        a[1] += t
        a[2] += b
        tot += t
    print(f"{len(per)} launches, {tot / 1e3:.1f} us serialised")
    print("| kernel | launches | share | avg us / launch | avg DRAM MB / launch |")
    print("|---|---|---|---|---|")
    for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {n} | {c} | {100 * t / tot:.1f} % | {t / c / 1e3:.1f} | {b / c / 1e6:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1])
