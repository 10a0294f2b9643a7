"""Times the UNMODIFIED reference (cellgrid AgentParallel, numba) on C4 in the build
container (the reference does not travel to the GPU box), for comparison with the
C oracle port that bench.py --impl reference times on the GPU box. Build container only."""
import os, sys, time, json
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, "/root/repo")
import numpy as np
import cellgrid
from cellgrid import engine, pool as cpool
from paper_2105_00039_b200.workloads import jittered_lattice_positions
pos = jittered_lattice_positions(256)
n = pos.shape[0]
p = cpool.AgentPool(position_x=pos[:,0].copy(), position_y=pos[:,1].copy(), position_z=pos[:,2].copy(),
                    diameter=np.full(n, 10.0), adherence=np.full(n, 0.4), uid=np.arange(n, dtype=np.uint64))
threads = os.cpu_count()
cfg = engine.SimulationConfig(strategy=engine.AgentParallel(thread_count=threads), steps=1)
t0 = time.perf_counter(); st = engine.step(p, cfg, 0); t1 = time.perf_counter()
times = []
for k in range(1, 3):
    a = time.perf_counter(); s = engine.step(p, cfg, k); times.append(time.perf_counter() - a)
print(json.dumps({"impl": "cellgrid AgentParallel (numba, the unmodified reference)", "agents": n, "threads": threads,
                  "first_step_s_incl_jit": t1 - t0, "step_s": times, "force_evals_step0": st.force_evals,
                  "candidates_step0": st.candidates, "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ")}))
