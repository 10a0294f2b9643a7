import sys, time
sys.path.insert(0,'/root/repo')
import paper_2105_00039_b200 as cg
from paper_2105_00039_b200 import workloads
pool = workloads.c4()
cfg = cg.SimulationConfig(strategy=cg.Gpu(summation="stencil"), steps=5)
cg.run(pool.copy(), cfg)
cfg = cg.SimulationConfig(strategy=cg.Gpu(summation="stencil"), steps=100)
p = pool.copy()
t0 = time.perf_counter(); rep = cg.run(p, cfg); t1 = time.perf_counter()
dev = sum(s.t_total for s in rep.steps)
print("engine.run 100 steps: wall %.1f ms (incl. upload + download), device %.1f ms = %.3f ms/step; hash %s" % ((t1-t0)*1e3, dev*1e3, dev*10, rep.final_state_hash[:16]))
