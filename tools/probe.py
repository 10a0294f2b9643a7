"""Quick device timing probe: per-phase CUDA-event times of cg_step on a config."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2105_00039_b200 import _native, workloads
from paper_2105_00039_b200.pool import PrecisionMode

def probe(name, pool, summation, order, flags, steps=5, warm=3, sweep=1):
    N = _native
    ctx = N.Context(0, pool.dtype)
    ctx.set_option(N.CG_OPT_SWEEP, sweep)
    ctx.set_option(N.CG_OPT_SUMMATION, summation)
    ctx.set_option(N.CG_OPT_RELAYOUT_EVERY, order)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
    p = np.array([2.0, 1.0, 0.01, 3.0, 1.0])
    for _ in range(warm):
        ctx.step(p, None, 1 << 24, flags)
    ctx.synchronize()
    t0 = time.perf_counter()
    sts = [ctx.step(p, None, 1 << 24, flags) for _ in range(steps)]
    wall = (time.perf_counter() - t0) / steps
    st = sts[-1]
    tot = np.median([s.t_total_ms for s in sts])
    print("%-10s sweep=%d sum=%d relayout=%d flags=%d n=%d grid=%.3f sort=%.3f force=%.3f total=%.3f ms wall=%.3f ms  "
          "-> %.2f G agent-upd/s (dev) evals/agent=%.2f cands/agent=%.2f" % (
          name, sweep, summation, order, flags, pool.count, st.t_grid_ms, st.t_sort_ms, st.t_force_ms, tot,
          wall * 1e3, pool.count / tot * 1e-6, st.force_evals / pool.count, st.candidates / pool.count))
    sys.stdout.flush()
    ctx.close()

if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2", "c4"]
    for w in which:
        if w == "c1": pool = workloads.c1()
        elif w == "c2": pool = workloads.c2()
        elif w == "c2f": pool = workloads.c2(PrecisionMode.FP32)
        elif w == "c4": pool = workloads.c4()
        elif w == "c4f": pool = workloads.c4(PrecisionMode.FP32)
        elif w.startswith("c3_"): pool = workloads.c3(float(w[3:]))
        for summ in [int(x) for x in os.environ.get("SUMS", "0,1").split(",")]:
            for order in [int(x) for x in os.environ.get("RELAYOUT", "1").split(",")]:
                probe(w, pool, summ, order, int(os.environ.get("FLAGS", "1")),
                      sweep=int(os.environ.get("SWEEP", "1")))
