import cProfile, pstats, sys, time
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import torch
import bench_configs as bc
class A: steps = 120
pr = cProfile.Profile()
pr.enable()
r = bc.run_c2u(A())
pr.disable()
print(r["ms_per_step"], r["tokens_per_s"])
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(18)
