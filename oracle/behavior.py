"""Host restatement of the reference behaviour phase -- TEST INFRASTRUCTURE.

``grow_and_divide`` follows /root/reference/pkg/src/cellgrid/engine.py:191-232
line by line with numpy (np.cbrt, and rng.unit_vector = numpy's
Generator(Philox(key=(uid, step))).standard_normal, rng.py:41-54), so on the
CPUs the reference runs on it reproduces the reference's pools bit for bit
(tests/test_behaviour.py pins it to fixtures the reference wrote).  The
product computes the same phase on the device (cg_behavior); this module is
the checker the GPU tests compare it with.
"""

from __future__ import annotations

import math

import numpy as np

_SIXTH_PI = np.pi / 6.0      # engine.py:41


def unit_vector(uid, step):
    """rng.py:47-54."""
    gen = np.random.Generator(np.random.Philox(key=np.array([int(uid) & (2**64 - 1), int(step) & (2**64 - 1)],
                                                            dtype=np.uint64)))
    while True:
        v = gen.standard_normal(3)
        n = math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])
        if n > 1e-12:
            return v / n


def grow_and_divide(pool, growth, step_index=0):
    """engine.py:191-232 on an AgentPool-like object (mutated in place)."""
    if pool.count == 0:
        return 0
    T = pool.dtype.type
    k6 = T(_SIXTH_PI)
    d = pool.diameter
    vol = k6 * (d * d * d)
    vol = vol + T(growth.volume_growth_rate)
    pool.diameter = np.cbrt(vol / k6)
    if not growth.division_enabled:
        return 0
    ripe = np.flatnonzero(pool.diameter >= T(growth.division_diameter))
    if ripe.shape[0] == 0:
        return 0
    ripe = ripe[np.argsort(pool.uid[ripe])]
    k = ripe.shape[0]
    where = np.empty((k, 3), np.float64)
    half_d = np.empty(k, np.float64)
    adh = np.empty(k, np.float64)
    for row, i in enumerate(ripe):
        dm = pool.diameter[i]
        dh = np.cbrt((T(0.5) * (k6 * (dm * dm * dm))) / k6)
        shift = unit_vector(int(pool.uid[i]), step_index) * (float(dm) * 0.5 / 4.0)
        where[row] = (float(pool.position_x[i]) + shift[0], float(pool.position_y[i]) + shift[1],
                      float(pool.position_z[i]) + shift[2])
        half_d[row] = float(dh)
        adh[row] = float(pool.adherence[i])
        pool.diameter[i] = dh
    pool.append_many(where, half_d, adh)
    return k


def numpy_cbrt_is_svml():
    """numpy evaluates np.cbrt with Intel SVML on AVX512_SKX CPUs (the routine
    csrc/behavior_math.h restates); elsewhere it calls libm."""
    try:
        from numpy._core._multiarray_umath import __cpu_features__ as feats
    except ImportError:   # numpy < 2
        from numpy.core._multiarray_umath import __cpu_features__ as feats
    return bool(feats.get("AVX512_SKX"))
