python tools/gemm_microbench.py
TIMRUN_GRAPHS=0 ncu --metrics gpu__time_duration.sum --clock-control none -s 120000 -c 800 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 5 --warmup 3 --skip 600 --cpu-budget 0 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/launches_r1.csv")))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[hdr["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[hdr["Kernel Name"]][:80]
    v = float(r[hdr["Metric Value"]].replace(",", ""))
    unit = r[hdr["Metric Unit"]]
    v = v / 1000 if unit == "nsecond" else v
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{t:10.1f} us {100*t/tot:5.1f}%  n={n:4d}  {k}")
print("total us", tot)
PY
