"""From an ncu launch list of bench.py's value window (TIMRUN_PROFILE_TIMED=1,
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum),
write profiles/attention_traffic.json: measured DRAM bytes per attention launch
(decode-only launches = attn_tiles_kernel, mixed launches = attn_step_kernel),
which bench.py reports as roofline.traffic.
usage: python tools/attention_traffic.py launches.csv[.gz] [label]"""
import collections
import csv
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main(path, label):
    opener = gzip.open if path.endswith(".gz") else open
    rows = [r for r in csv.reader(line for line in opener(path, "rt") if line.startswith('"'))]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki]
    cls = {"decode": [], "mixed": []}
    for i, m in per.items():
        n = names[i]
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        t = m.get("gpu__time_duration.sum", 0.0)
        if "attn_tiles_kernel" in n:
            cls["decode"].append((b, t))
        elif "attn_step_kernel" in n:
            cls["mixed"].append((b, t))
    out = {"source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                     f"--clock-control none of `TIMRUN_PROFILE_TIMED=1 python bench.py` ({label}), "
                     "every attention launch of the timed steps (serialised, cold-L2 replays)"}
    allb = []
    for k, v in cls.items():
        if v:
            out[k] = {"launches": len(v), "bytes_per_launch": sum(b for b, _ in v) / len(v),
                      "ns_per_launch": sum(t for _, t in v) / len(v)}
            allb += [b for b, _ in v]
    out["bytes_per_launch"] = sum(allb) / len(allb) if allb else None
    (ROOT / "profiles" / "attention_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
