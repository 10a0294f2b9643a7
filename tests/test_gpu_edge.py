"""Edge cases of the device step against the C oracle (pinned to the
reference, tests/test_oracle.py): one agent, a single crowded box (the
warp-cooperative dense kernel and the overflow kernel), far-from-origin and
negative coordinates (the fp32 prefilter margin), heterogeneous diameters
(the largest-radius reach bound), and a zero-adherence / zero-cap parameter
set.  uid summation: counters, storage order, m / nk and every output column
bit-exact; stencil summation: counters exact, displacements within 1e-12
(per-agent vector norm)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _pool(pos, diam, adh, prec="fp64"):
    from paper_2105_00039_b200.pool import AgentPool, PrecisionMode
    pm = PrecisionMode.FP64 if prec == "fp64" else PrecisionMode.FP32
    return AgentPool.from_arrays(np.asarray(pos, np.float64), diam, adh, pm)


def _cases():
    rng = np.random.default_rng(42)
    yield "single", _pool([[1.0, 2.0, 3.0]], 10.0, 0.4), None
    yield "pair_touching", _pool([[0, 0, 0], [10.0, 0, 0]], 10.0, 0.4), None
    yield "crowded_box", _pool(rng.uniform(0, 12.0, (600, 3)), 10.0, 0.4), None
    yield "crowded_cluster", _pool(rng.uniform(0, 30.0, (4000, 3)), 10.0, 0.4), None
    yield "far_offset", _pool(rng.uniform(0, 300.0, (20000, 3)) + np.array([1e6, -3e5, 7.5e5]), 10.0, 0.4), None
    yield "negative", _pool(rng.uniform(-500, -100.0, (20000, 3)), 10.0, 0.4), None
    yield "hetero_diam", _pool(rng.uniform(0, 200.0, (20000, 3)), rng.uniform(2.0, 20.0, 20000),
                               rng.uniform(0.0, 2.0, 20000)), 22.0
    yield "far_offset_f32", _pool(rng.uniform(0, 300.0, (20000, 3)) + np.array([3e3, -2e3, 1e3]), 10.0, 0.4,
                                  "fp32"), None


CASES = list(_cases())


@pytest.mark.parametrize("summation", [0, 1])
@pytest.mark.parametrize("name,pool,ir", CASES, ids=[c[0] for c in CASES])
def test_edge_step_matches_oracle(cuda_required, name, pool, ir, summation):
    from paper_2105_00039_b200 import _native as N
    from paper_2105_00039_b200.mechanics import ForceParams
    params = (ForceParams(), ForceParams(kappa=5.0, gamma=0.2, timestep=0.1, max_displacement=0.05,
                                         adherence_scale=0.0))
    ref = pool.copy()
    ctx = N.Context(0, pool.dtype)
    ctx.set_option(N.CG_OPT_SUMMATION, summation)
    try:
        ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
        for k, fp in enumerate(params * 2):
            if summation == 1 and k > 0:       # stencil order: restart from the reference state
                ctx.upload(ref.position_x, ref.position_y, ref.position_z, ref.diameter, ref.adherence, ref.uid)
            p5 = np.array([fp.kappa, fp.gamma, fp.timestep, fp.max_displacement, fp.adherence_scale])
            st = ctx.step(p5, ir, 1 << 24, N.CG_STEP_SORT | N.CG_STEP_RECORD)
            r = oracle.step(ref, fp, sort=True, interaction_radius=ir, threads=8)
            assert (st.force_evals, st.candidates, st.degenerate_pairs) == (
                r.force_evals, r.candidates, r.degenerate_pairs), (name, k)
            assert st.grid_max_occupancy == int(r.box_count.max())
            cols = ctx.download()
            assert np.array_equal(cols["uid"], ref.uid)
            m, nk = ctx.record_export()
            assert np.array_equal(m, r.m) and np.array_equal(nk, r.nk)
            mine = np.stack([cols[c].astype(np.float64) for c in ("dx", "dy", "dz")], 1)
            want = np.stack([getattr(ref, c).astype(np.float64) for c in
                             ("displacement_x", "displacement_y", "displacement_z")], 1)
            if summation == 0 and r.degenerate_pairs == 0:
                assert np.array_equal(mine, want), (name, k)
                for a, b in (("px", "position_x"), ("py", "position_y"), ("pz", "position_z")):
                    assert np.array_equal(cols[a], getattr(ref, b)), (name, k, a)
            else:
                tol = 1e-12 if pool.dtype == np.float64 else 1e-4
                err = np.linalg.norm(mine - want, axis=1)
                assert np.all(err <= tol * np.linalg.norm(want, axis=1) + 1e-300), (name, k, float(err.max()))
    finally:
        ctx.close()
