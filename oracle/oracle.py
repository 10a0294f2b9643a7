"""ctypes driver for the C oracle (oracle/cg_oracle.c) -- TEST INFRASTRUCTURE.

``step`` restates the orchestration of reference engine.step
(/root/reference/pkg/src/cellgrid/engine.py:279-341): optional Z-order
re-sort on a pre-grid, grid rebuild, force phase, apply -- with every numeric
kernel executed by the C restatement.  It mutates the pool exactly as the
reference does (storage permutation, displacement columns, positions).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libcg_oracle.so")
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double


class OracleError(ValueError):
    pass


class OracleGridOverflow(RuntimeError):
    pass


def build():
    """Compile the oracle (gcc, -ffp-contract=off) into oracle/_build/."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        for sfx in ("f64", "f32"):
            getattr(L, "cgo_geometry_" + sfx).argtypes = [_I64, _P, _P, _P, _P, _D, _I64, _P, _P, _P, _P]
            getattr(L, "cgo_geometry_" + sfx).restype = ctypes.c_int
            getattr(L, "cgo_box_ids_" + sfx).argtypes = [_I64, _P, _P, _P, _D, _P, _P, _P]
            getattr(L, "cgo_force_phase_" + sfx).argtypes = [
                _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _P, ctypes.c_int,
                _P, _P, _P, _P, _P, _P]
            getattr(L, "cgo_all_pairs_" + sfx).argtypes = [_I64, _P, _P, _P, _P, _P, _P, _P,
                                                          _P, _P, _P, _P]
        L.cgo_csr.argtypes = [_I64, _P, _I64, _P, _P, _P]
        L.cgo_morton_perm.argtypes = [_I64, _P, _P, _P, _P, _P]
        L.cgo_morton_encode.argtypes = [ctypes.c_uint64] * 3
        L.cgo_morton_encode.restype = ctypes.c_uint64
        L.cgo_degenerate_dir.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _P]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_P) if a is not None else None


def _sfx(dtype):
    return "f64" if np.dtype(dtype) == np.float64 else "f32"


def geometry(pool, interaction_radius=None, box_cap=1 << 24):
    """(box_length, origin f64[3], dims i64[3], num_boxes) -- spatial.py:99-116."""
    L = np.zeros(1, np.float64)
    origin = np.zeros(3, np.float64)
    dims = np.zeros(3, np.int64)
    nb = np.zeros(1, np.int64)
    ir = float("nan") if interaction_radius is None else float(interaction_radius)
    rc = getattr(lib(), "cgo_geometry_" + _sfx(pool.dtype))(
        pool.count, _p(pool.position_x), _p(pool.position_y), _p(pool.position_z),
        _p(pool.diameter), ir, int(box_cap), _p(L), _p(origin), _p(dims), _p(nb))
    if rc == 1:
        raise OracleError("cannot build a grid over an empty pool")
    if rc == 2:
        raise OracleError("interaction_radius must be positive, got %r" % (interaction_radius,))
    if rc == 3:
        raise OracleGridOverflow("grid of %s boxes exceeds cap %d" % (dims.tolist(), box_cap))
    return float(L[0]), origin, dims, int(nb[0])


def box_ids(pool, box_length, origin, dims):
    out = np.empty(pool.count, np.int64)
    getattr(lib(), "cgo_box_ids_" + _sfx(pool.dtype))(
        pool.count, _p(pool.position_x), _p(pool.position_y), _p(pool.position_z),
        float(box_length), _p(np.ascontiguousarray(origin, np.float64)),
        _p(np.ascontiguousarray(dims, np.int64)), _p(out))
    return out


def csr(box_index, num_boxes):
    """(count, start[nb+1], members) -- CSR form of link_chains (kernels.py:132-145)."""
    box_index = np.ascontiguousarray(box_index, np.int64)
    count = np.empty(num_boxes, np.int64)
    start = np.empty(num_boxes + 1, np.int64)
    members = np.empty(box_index.shape[0], np.int64)
    lib().cgo_csr(box_index.shape[0], _p(box_index), num_boxes, _p(count), _p(start), _p(members))
    return count, start, members


def morton_encode(ix, iy, iz):
    return int(lib().cgo_morton_encode(int(ix), int(iy), int(iz)))


def morton_perm(box_index, dims, uid):
    n = box_index.shape[0]
    perm = np.empty(n, np.int64)
    lib().cgo_morton_perm(n, _p(np.ascontiguousarray(box_index, np.int64)),
                          _p(np.ascontiguousarray(dims, np.int64)),
                          _p(np.ascontiguousarray(uid, np.uint64)), _p(perm), None)
    return perm


def force_phase(pool, box_index, dims, start, members, params, threads=1):
    """Displacements + per-agent m/nk + (evals, cands, ndeg) -- kernels.py:280-333."""
    n = pool.count
    dt = pool.dtype
    radii = pool.radii()
    out = [np.zeros(n, dt) for _ in range(3)]
    m = np.zeros(n, np.int32)
    nk = np.zeros(n, np.int32)
    counters = np.zeros(3, np.int64)
    occ = np.diff(start)
    cap = 27 * int(occ.max()) if occ.size else 1
    getattr(lib(), "cgo_force_phase_" + _sfx(dt))(
        n, _p(pool.position_x), _p(pool.position_y), _p(pool.position_z), _p(radii),
        _p(pool.adherence), _p(pool.uid), _p(np.ascontiguousarray(box_index, np.int64)),
        _p(np.ascontiguousarray(dims, np.int64)), _p(start), _p(members), cap,
        _p(np.ascontiguousarray(params, np.float64)), int(threads),
        _p(out[0]), _p(out[1]), _p(out[2]), _p(m), _p(nk), _p(counters))
    return out, m, nk, counters


def all_pairs(pool, params):
    """O(n^2) displacements and counters -- mechanics.py:186-233."""
    n = pool.count
    dt = pool.dtype
    out = [np.zeros(n, dt) for _ in range(3)]
    counters = np.zeros(3, np.int64)
    if not isinstance(params, np.ndarray):
        params = _params_vec(params)
    getattr(lib(), "cgo_all_pairs_" + _sfx(dt))(
        n, _p(pool.position_x), _p(pool.position_y), _p(pool.position_z), _p(pool.radii()),
        _p(pool.adherence), _p(pool.uid), _p(np.ascontiguousarray(params, np.float64)),
        _p(out[0]), _p(out[1]), _p(out[2]), _p(counters))
    return out, counters


@dataclass
class OracleStep:
    force_evals: int
    candidates: int
    degenerate_pairs: int
    box_length: float
    origin: np.ndarray
    dims: np.ndarray
    box_index: np.ndarray      # per storage index (after the sort), flat box id
    box_count: np.ndarray      # flat box order
    box_offsets: np.ndarray    # exclusive prefix sum of box_count, nb+1 slots
    m: np.ndarray              # per storage index: stencil candidates
    nk: np.ndarray             # per storage index: colliding pairs
    perm: np.ndarray           # storage permutation applied by the sort (or None)


def _params_vec(params):
    return np.asarray([params.kappa, params.gamma, params.timestep, params.max_displacement,
                       params.adherence_scale, 0.0, 1.0], np.float64)


def step(pool, params, sort=True, freeze=False, interaction_radius=None, threads=1,
         box_cap=1 << 24):
    """One reference step (engine.py:279-341) on ``pool``; mutates it in place."""
    n = pool.count
    perm = None
    if sort and n > 1:                                   # engine.py:305-309
        L, origin, dims, nb = geometry(pool, interaction_radius, box_cap)
        perm = morton_perm(box_ids(pool, L, origin, dims), dims, pool.uid)
        for name in ("position_x", "position_y", "position_z", "diameter", "adherence",
                     "displacement_x", "displacement_y", "displacement_z", "uid"):
            setattr(pool, name, getattr(pool, name)[perm])
    L, origin, dims, nb = geometry(pool, interaction_radius, box_cap)   # engine.py:313
    bidx = box_ids(pool, L, origin, dims)
    count, start, members = csr(bidx, nb)
    disp, m, nk, counters = force_phase(pool, bidx, dims, start, members,
                                        _params_vec(params), threads)
    pool.displacement_x, pool.displacement_y, pool.displacement_z = disp
    if not freeze:                                       # engine.py:323-327
        pool.position_x = pool.position_x + pool.displacement_x
        pool.position_y = pool.position_y + pool.displacement_y
        pool.position_z = pool.position_z + pool.displacement_z
    return OracleStep(force_evals=int(counters[0]), candidates=int(counters[1]),
                      degenerate_pairs=int(counters[2]), box_length=L, origin=origin,
                      dims=dims, box_index=bidx, box_count=count, box_offsets=start,
                      m=m, nk=nk, perm=perm)


def neighbor_csr(px, py, pz, uid, radius, block=1024):
    """Radius-query table by brute force -- the predicate of reference
    kernels._grid_count_one / grid_neighbor_fill (kernels.py:427-520): widen to
    f64, dx = p_j - p_i per axis, d2 = (dx*dx + dy*dy) + dz*dz, keep j != i
    with d2 <= radius^2 (closed ball); each row ascends by neighbour uid
    (kernels._sort_row_by_uid, kernels.py:471-480).  The grid only restricts
    candidates to the 27-box stencil, which holds every agent within
    radius <= box_length, so the all-pairs table is the same table.
    Returns (indptr, indices) in storage order (numpy, O(n^2) in blocks)."""
    x = np.asarray(px).astype(np.float64)
    y = np.asarray(py).astype(np.float64)
    z = np.asarray(pz).astype(np.float64)
    uid = np.asarray(uid)
    n = x.shape[0]
    r2 = float(radius) * float(radius)
    by_uid = np.argsort(uid, kind="stable")
    rows = []
    for a in range(0, n, block):
        b = min(n, a + block)
        dx = x[by_uid][None, :] - x[a:b, None]
        dy = y[by_uid][None, :] - y[a:b, None]
        dz = z[by_uid][None, :] - z[a:b, None]
        hit = (dx * dx + dy * dy) + dz * dz <= r2
        hit[np.arange(b - a), np.searchsorted(uid[by_uid], uid[a:b])] = False
        for r in range(b - a):
            rows.append(by_uid[hit[r]])
    counts = np.array([len(r) for r in rows], np.int64)
    indptr = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=indptr[1:])
    indices = np.concatenate(rows).astype(np.int64) if n else np.zeros(0, np.int64)
    return indptr, indices
