"""uids at or above 2^32 on a single context.  With every uid < 2^32 the
sparse sweeps sort survivors by 32-bit keys taken from the proxies (KEY32);
above that they fall back to 64-bit keys, and the dense warp sweep to its
64-bit sort.  These pools carry uids scrambled over the whole 64-bit range
(a bijection, so still unique and in a different order than their spawn
order) and are stepped with neighbour lists on -- grid sweeps, list builds
and list sweeps -- against the C oracle, bit for bit (kernels.py:206-225
sums each agent's pairs in uid order, so the order is observable)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

PARAMS5 = np.array([2.0, 1.0, 0.01, 3.0, 1.0])


def _scramble(uid):
    """odd multiplier mod 2^62 (a bijection there), lifted above 2^33"""
    u = ((uid.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)) & np.uint64((1 << 62) - 1)) + np.uint64(1 << 33)
    assert len(np.unique(u)) == len(u)
    return u


def _pools():
    from paper_2105_00039_b200.pool import AgentPool
    from paper_2105_00039_b200.workloads import jittered_lattice_positions
    p = AgentPool.from_arrays(jittered_lattice_positions(20, 8.0, 1.0, 5), 10.0, 0.4)
    yield "lattice", p
    rng = np.random.default_rng(12)
    yield "moderate", AgentPool.from_arrays(rng.uniform(0.0, 150.0, (15000, 3)), 10.0, 0.4)    # ~16 survivors/agent
    yield "dense", AgentPool.from_arrays(rng.uniform(0.0, 110.0, (20000, 3)), 10.0, 0.4)       # warp sweep


@pytest.mark.parametrize("name,pool", list(_pools()), ids=lambda v: v if isinstance(v, str) else "")
def test_uid64_matches_oracle(cuda_required, name, pool):
    from paper_2105_00039_b200 import _native as N
    from paper_2105_00039_b200.mechanics import ForceParams
    pool = pool.copy()
    pool.uid = _scramble(pool.uid)
    pool.next_uid = int(pool.uid.max()) + 1
    assert int(pool.uid.max()) >= 1 << 32
    ref = pool.copy()
    ctx = N.Context(0, pool.dtype)
    ctx.set_option(N.CG_OPT_SUMMATION, 0)
    ctx.set_option(N.CG_OPT_LIST_SKIN, -1)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
    kinds = []
    for k in range(8):
        flags = N.CG_STEP_SORT | (N.CG_STEP_FREEZE if name != "lattice" else 0)
        st = ctx.step(PARAMS5, None, 1 << 24, flags)
        kinds.append(int(st.sweep_kind))
        r = oracle.step(ref, ForceParams(), sort=True, freeze=name != "lattice", threads=8)
        assert (st.force_evals, st.candidates, st.degenerate_pairs) == (
            r.force_evals, r.candidates, r.degenerate_pairs), (name, k)
        cols = ctx.download()
        assert np.array_equal(cols["uid"], ref.uid), (name, k)
        for a, b in (("px", "position_x"), ("py", "position_y"), ("pz", "position_z"),
                     ("dx", "displacement_x"), ("dy", "displacement_y"), ("dz", "displacement_z")):
            assert np.array_equal(cols[a], getattr(ref, b)), (name, k, a)
    ctx.close()
    assert 1 in kinds and 2 in kinds, kinds     # a list build and list sweeps ran
