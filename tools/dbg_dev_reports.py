import sys, gzip, json
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from pathlib import Path
import test_engine_gpu as T
golden = Path("/root/repo/tests/golden")
scens = T._load(golden, "engine_runs.json.gz")
scen = next(s for s in scens if s["name"] == "deep32_T0")
eng, rids = T._engine_for(scen)
for gs in scen["steps"]:
    rep = eng.step()
    if 76 <= rep.step <= 81:
        dev = eng.device_step_report()
        recs = [r for r in eng.runtime.device_reports() if r["serial"] > eng._step_serials[0] - 3]
        print(rep.step, eng._step_serials, "host", gs["report"], rep.decoded, "dev", dev["flops_units"], dev["pages_free"],
              [(r["serial"], r["flops_units"], r["pages_free"]) for r in recs])
