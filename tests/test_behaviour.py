"""Behaviour phase (growth then division, reference engine.py:191-232) against
fixtures made by the reference itself (tests/golden/make_golden_growth.py):
the oracle's host restatement (CPU) and the device phase cg_behavior bit for
bit, the device unit vectors against the reference's rng.unit_vector, and
engine.run with growth (resident on the GPU: same per-step counters,
divisions, agent counts and final state hash as the reference's Serial run)."""

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


def _check_pool(pool, g, k):
    assert k == int(g["divisions"])
    for c, attr in (("px", "position_x"), ("py", "position_y"), ("pz", "position_z"), ("diam", "diameter"),
                    ("adh", "adherence"), ("uid", "uid")):
        assert np.array_equal(getattr(pool, attr), g["out_" + c]), c
    assert pool.next_uid == int(g["out_next_uid"])
    assert pool.state_hash() == str(g["state_hash"])


@pytest.mark.parametrize("path", BEHAVIOUR, ids=[os.path.basename(p)[7:-4] for p in BEHAVIOUR])
def test_oracle_grow_and_divide_matches_reference(path):
    import oracle
    if not oracle.behavior.numpy_cbrt_is_svml():
        pytest.skip("numpy's np.cbrt is libm's on this CPU (the fixtures were written with SVML)")
    g = np.load(path)
    pool = _pool(g)
    k = oracle.behavior.grow_and_divide(pool, _growth(g), int(g["step_index"]))
    _check_pool(pool, g, k)


@pytest.mark.gpu
@pytest.mark.parametrize("path", BEHAVIOUR, ids=[os.path.basename(p)[7:-4] for p in BEHAVIOUR])
def test_device_grow_and_divide_matches_reference(cuda_required, path):
    from paper_2105_00039_b200 import grow_and_divide
    g = np.load(path)
    pool = _pool(g)
    k = grow_and_divide(pool, _growth(g), int(g["step_index"]))
    _check_pool(pool, g, k)


@pytest.mark.gpu
def test_device_unit_vectors_match_reference(cuda_required):
    from paper_2105_00039_b200 import _native
    g = np.load(os.path.join(GOLD, "growth_unitvec.npz"))
    ctx = _native.Context(0, np.float64)
    try:
        for s in np.unique(g["step"])[:40]:          # the small-step block: many uids per step
            sel = g["step"] == s
            assert np.array_equal(ctx.unit_vectors(g["uid"][sel], int(s)), g["vec"][sel]), int(s)
        big = np.flatnonzero(g["step"] >= 50)[:4000]   # wide uids and steps, one call each
        got = np.array([ctx.unit_vectors(g["uid"][i:i + 1], int(g["step"][i]))[0] for i in big])
        assert np.array_equal(got, g["vec"][big])
    finally:
        ctx.close()


@pytest.mark.gpu
def test_device_growth_large_pool_matches_oracle(cuda_required):
    """200,000 agents, several thousand divisions in one phase (the radix sort of
    the ripe mothers spans many tiles): device == oracle, bit for bit."""
    import oracle
    if not oracle.behavior.numpy_cbrt_is_svml():
        pytest.skip("numpy's np.cbrt is libm's on this CPU")
    from paper_2105_00039_b200 import GrowthParams, grow_and_divide
    from paper_2105_00039_b200.pool import AgentPool, PrecisionMode
    rng = np.random.default_rng(21)
    n = 200_000
    for pm in (PrecisionMode.FP64, PrecisionMode.FP32):
        pos = rng.uniform(0, 600.0, (n, 3))
        pool = AgentPool.from_arrays(pos, rng.uniform(8.0, 11.2, n), rng.uniform(0, 1, n), pm)
        perm = rng.permutation(n)                      # uids not in storage order
        pool.uid = pool.uid[perm] * np.uint64(3) + np.uint64(7)
        pool.next_uid = int(pool.uid.max()) + 1
        ref = pool.copy()
        gp = GrowthParams(volume_growth_rate=30.0, division_diameter=11.0)
        k = grow_and_divide(pool, gp, 9)
        kr = oracle.behavior.grow_and_divide(ref, gp, 9)
        assert k == kr and k > 1000
        for attr in ("position_x", "position_y", "position_z", "diameter", "adherence", "uid"):
            assert np.array_equal(getattr(pool, attr), getattr(ref, attr)), (pm, attr)
        assert pool.next_uid == ref.next_uid


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
@pytest.mark.parametrize("api", ["run", "step"])
@pytest.mark.parametrize("path", RUNS, ids=[os.path.basename(p)[7:-4] for p in RUNS])
def test_run_with_growth_matches_reference(cuda_required, path, api):
    """engine.run (pool resident, behaviour phase on the device every step) and
    the same steps through engine.step (upload / step / download each step)."""
    import paper_2105_00039_b200 as P
    g = np.load(path)
    pool = P.AgentPool(position_x=g["in_px"].copy(), position_y=g["in_py"].copy(), position_z=g["in_pz"].copy(),
                       diameter=g["in_diam"].copy(), adherence=g["in_adh"].copy(), uid=g["in_uid"].copy(),
                       next_uid=int(g["in_next_uid"]))
    prec = P.PrecisionMode.FP64 if pool.dtype == np.float64 else P.PrecisionMode.FP32
    cfg = P.SimulationConfig(strategy=P.Gpu(), growth=_growth(g), steps=int(g["steps"]), precision=prec,
                             morton_sort_every=int(g["sort_every"]))
    if api == "run":
        rep = P.run(pool, cfg)
        steps, final_hash = rep.steps, rep.final_state_hash
    else:
        steps = [P.step(pool, cfg, k) for k in range(cfg.steps)]
        final_hash = pool.state_hash()
    assert [s.divisions for s in steps] == list(g["divisions"])
    assert [s.agent_count for s in steps] == list(g["counts"])
    assert [s.force_evals for s in steps] == list(g["evals"])
    assert [s.candidates for s in steps] == list(g["cands"])
    assert np.array_equal(pool.uid, g["out_uid"])
    assert np.array_equal(pool.position_x, g["out_px"])
    assert final_hash == str(g["state_hash"])
