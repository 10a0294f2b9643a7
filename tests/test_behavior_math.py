"""The behaviour-phase arithmetic of csrc/behavior_math.h, built for the host
(gcc -ffp-contract=off, tests/behavior_math_host.c) and compared with what the
reference computes through numpy / libm: np.cbrt in both precisions (SVML on
AVX512_SKX CPUs -- skipped elsewhere, numpy uses libm there), glibc log1p,
numpy's Philox4x64 stream and standard normals, and the reference's
rng.unit_vector fixture.  The device build of the same header is checked
against the same fixtures in tests/test_behaviour.py."""

import ctypes
import math
import os
import shutil
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
P = ctypes.c_void_p


@pytest.fixture(scope="module")
def bm(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("bm") / "bm.so")
    cxx = shutil.which("g++") or "g++"
    subprocess.run([cxx, "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-x", "c++", "-o", out,
                    os.path.join(HERE, "behavior_math_host.c"), "-lm"], check=True)
    return ctypes.CDLL(out)


def _svml():
    import oracle
    return oracle.behavior.numpy_cbrt_is_svml()


def test_cbrt_matches_numpy(bm):
    if not _svml():
        pytest.skip("numpy's np.cbrt is libm's on this CPU")
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.uniform(0.5, 5000, 400_000), 10.0 ** rng.uniform(-300, 300, 200_000),
                        -rng.uniform(1e-3, 1e6, 50_000), 2.0 ** rng.integers(-1074, 1023, 20_000)])
    y = np.empty_like(x)
    bm.bm_cbrt64(ctypes.c_long(x.size), x.ctypes.data_as(P), y.ctypes.data_as(P))
    assert np.array_equal(y, np.cbrt(x))
    x32 = np.concatenate([rng.uniform(0.5, 5000, 400_000), 10.0 ** rng.uniform(-37, 37, 200_000)]).astype(np.float32)
    y32 = np.empty_like(x32)
    bm.bm_cbrt32(ctypes.c_long(x32.size), x32.ctypes.data_as(P), y32.ctypes.data_as(P))
    assert np.array_equal(y32, np.cbrt(x32))


def test_log1p_matches_libm(bm):
    rng = np.random.default_rng(4)
    u = np.concatenate([-(rng.integers(0, 2 ** 53, 400_000) * (1.0 / 9007199254740992.0)),
                        rng.uniform(-0.99, 30.0, 50_000), -10.0 ** rng.uniform(-20, -5, 20_000),
                        -1 + 10.0 ** rng.uniform(-16, -1, 20_000)])
    y = np.empty_like(u)
    bm.bm_log1p(ctypes.c_long(u.size), u.ctypes.data_as(P), y.ctypes.data_as(P))
    assert np.array_equal(y, np.array([math.log1p(v) for v in u]))


def test_philox_and_normals_match_numpy(bm):
    for key in ((0, 0), (123456789, 42), (2 ** 63 + 5, 2 ** 40)):
        raw = np.empty(4001, np.uint64)
        bm.bm_philox_raw(ctypes.c_uint64(key[0]), ctypes.c_uint64(key[1]), ctypes.c_long(raw.size),
                         raw.ctypes.data_as(P))
        assert np.array_equal(raw, np.random.Philox(key=np.array(key, np.uint64)).random_raw(raw.size))
    nrm = np.empty(600_000)
    bm.bm_normals(ctypes.c_uint64(7), ctypes.c_uint64(99), ctypes.c_long(nrm.size), nrm.ctypes.data_as(P))
    ref = np.random.Generator(np.random.Philox(key=np.array([7, 99], np.uint64))).standard_normal(nrm.size)
    assert np.count_nonzero(np.abs(ref) > 3.6541528853610088) > 50     # the tail path ran
    assert np.array_equal(nrm, ref)


def test_unit_vectors_match_reference_fixture(bm):
    g = np.load(os.path.join(HERE, "golden", "growth_unitvec.npz"))
    out = np.empty((g["uid"].size, 3))
    uid = np.ascontiguousarray(g["uid"], np.uint64)
    step = g["step"]
    for s in np.unique(step[:20000]):
        sel = np.flatnonzero(step == s)
        o = np.empty((sel.size, 3))
        u = np.ascontiguousarray(uid[sel])
        bm.bm_unit_vectors(ctypes.c_long(sel.size), u.ctypes.data_as(P), ctypes.c_uint64(int(s)), o.ctypes.data_as(P))
        out[sel] = o
    for i in range(20000, uid.size):
        o = np.empty(3)
        u = uid[i:i + 1].copy()
        bm.bm_unit_vectors(ctypes.c_long(1), u.ctypes.data_as(P), ctypes.c_uint64(int(step[i])), o.ctypes.data_as(P))
        out[i] = o
    assert np.array_equal(out, g["vec"])
