"""Behaviour phase (growth then division, reference engine.py:191-232) against
fixtures made by the reference itself (tests/golden/make_golden_growth.py):
the host grow_and_divide bit for bit (CPU), and engine.run with growth on the
GPU step (same per-step counters, divisions, agent counts and final state
hash as the reference's Serial run)."""

import glob
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
BEHAVIOUR = sorted(p for p in glob.glob(os.path.join(GOLD, "growth_*.npz")) if str(np.load(p)["kind"]) == "behaviour")
RUNS = sorted(p for p in glob.glob(os.path.join(GOLD, "growth_*.npz")) if str(np.load(p)["kind"]) == "run")


def _pool(g, prefix="in_"):
    from paper_2105_00039_b200.pool import AgentPool
    return AgentPool(position_x=g[prefix + "px"].copy(), position_y=g[prefix + "py"].copy(),
                     position_z=g[prefix + "pz"].copy(), diameter=g[prefix + "diam"].copy(),
                     adherence=g[prefix + "adh"].copy(), uid=g[prefix + "uid"].copy(),
                     next_uid=int(g[prefix + "next_uid"]))


def _growth(g):
    from paper_2105_00039_b200 import GrowthParams
    return GrowthParams(volume_growth_rate=float(g["rate"]), division_diameter=float(g["div"]),
                        division_enabled=bool(g["enabled"]))


@pytest.mark.parametrize("path", BEHAVIOUR, ids=[os.path.basename(p)[7:-4] for p in BEHAVIOUR])
def test_grow_and_divide_matches_reference(path):
    from paper_2105_00039_b200 import grow_and_divide
    g = np.load(path)
    pool = _pool(g)
    k = grow_and_divide(pool, _growth(g), int(g["step_index"]))
    assert k == int(g["divisions"])
    for c, attr in (("px", "position_x"), ("py", "position_y"), ("pz", "position_z"), ("diam", "diameter"),
                    ("adh", "adherence"), ("uid", "uid")):
        assert np.array_equal(getattr(pool, attr), g["out_" + c]), c
    assert pool.next_uid == int(g["out_next_uid"])
    assert pool.state_hash() == str(g["state_hash"])


def test_pool_append_and_remove():
    from paper_2105_00039_b200.pool import AgentPool
    pool = AgentPool.from_arrays(np.arange(12, dtype=np.float64).reshape(4, 3), 10.0, 0.4)
    u = pool.append([1.0, 2.0, 3.0], 9.0, 0.5)
    assert u == 4 and pool.count == 5 and pool.next_uid == 5
    assert pool.diameter[-1] == 9.0 and pool.displacement_x[-1] == 0.0
    new = pool.append_many(np.ones((2, 3)), [8.0, 7.0], [0.1, 0.2])
    assert list(new) == [5, 6] and pool.count == 7
    pool.remove(0)
    assert pool.count == 6 and pool.uid[0] == 6 and 0 not in set(pool.uid.tolist())
    pool.validate()


@pytest.mark.gpu
@pytest.mark.parametrize("path", RUNS, ids=[os.path.basename(p)[7:-4] for p in RUNS])
def test_run_with_growth_matches_reference(cuda_required, path):
    import paper_2105_00039_b200 as P
    g = np.load(path)
    pool = P.AgentPool(position_x=g["in_px"].copy(), position_y=g["in_py"].copy(), position_z=g["in_pz"].copy(),
                       diameter=g["in_diam"].copy(), adherence=g["in_adh"].copy(), uid=g["in_uid"].copy(),
                       next_uid=int(g["in_next_uid"]))
    cfg = P.SimulationConfig(strategy=P.Gpu(), growth=_growth(g), steps=int(g["steps"]),
                             morton_sort_every=int(g["sort_every"]))
    rep = P.run(pool, cfg)
    assert [s.divisions for s in rep.steps] == list(g["divisions"])
    assert [s.agent_count for s in rep.steps] == list(g["counts"])
    assert [s.force_evals for s in rep.steps] == list(g["evals"])
    assert [s.candidates for s in rep.steps] == list(g["cands"])
    assert np.array_equal(pool.uid, g["out_uid"])
    assert np.array_equal(pool.position_x, g["out_px"])
    assert rep.final_state_hash == str(g["state_hash"])
