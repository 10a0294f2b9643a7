"""ctypes binding of libcellgrid_b200.so (C ABI: include/cellgrid_b200.h).

There is no CPU fallback: if the library is missing or no sm_100 device is
present, every entry point raises.  Status codes are re-raised as the
reference's exception classes (cellgrid spatial.py:35-40, pool.py:30).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .pool import PoolCapacityError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CG_LIB") or os.path.join(_HERE, "libcellgrid_b200.so")

CG_OK, CG_ERR_VALUE, CG_ERR_GRID_OVERFLOW, CG_ERR_STENCIL = 0, 1, 2, 3
CG_ERR_POOL_CAPACITY, CG_ERR_CUDA, CG_ERR_NO_DEVICE, CG_ERR_STATE = 4, 5, 6, 7
CG_FP64, CG_FP32 = 0, 1
CG_STEP_SORT, CG_STEP_FREEZE, CG_STEP_RECORD = 1, 2, 4
CG_OPT_SUMMATION, CG_OPT_SWEEP, CG_OPT_RELAYOUT_EVERY, CG_OPT_PATH, CG_OPT_LIST_SKIN = 1, 3, 4, 5, 6
CG_OPT_INNER_LIST, CG_OPT_MID_LIST = 7, 8

# every symbol include/cellgrid_b200.h declares (checked by tests/test_abi.py)
EXPORTED = ("cg_abi_version", "cg_device_count", "cg_create", "cg_destroy", "cg_last_error",
            "cg_set_option", "cg_stream", "cg_upload", "cg_download", "cg_count", "cg_step",
            "cg_fetch_stats", "cg_build_grid", "cg_synchronize", "cg_grid_export",
            "cg_record_export", "cg_box_ids", "cg_force_phase", "cg_launch_count",
            "cg_host_alloc", "cg_host_free", "cg_record_bytes", "cg_reserve", "cg_local_bbox",
            "cg_slab_plan", "cg_slab_pack", "cg_slab_unpack",
            "cg_slab_step", "cg_slab_step_interior", "cg_neighbor_counts", "cg_neighbor_fill",
            "cg_list_stats", "cg_slab_list_epoch", "cg_step_download", "cg_behavior",
            "cg_unit_vectors")


class GridOverflowError(RuntimeError):
    """Grid would allocate more boxes than the configured cap (spatial.py:35)."""


class StencilTooSmallError(ValueError):
    """Search radius exceeds box_length (spatial.py:39)."""


class CudaError(RuntimeError):
    """CUDA runtime failure inside the native path."""


class NativeUnavailable(RuntimeError):
    """libcellgrid_b200.so missing or no sm_100 device: the path refuses to run."""


class StepStatsC(ctypes.Structure):
    _fields_ = [("step_id", ctypes.c_int64), ("agent_count", ctypes.c_int64),
                ("force_evals", ctypes.c_int64), ("candidates", ctypes.c_int64),
                ("degenerate_pairs", ctypes.c_int64), ("grid_dims", ctypes.c_int64 * 3),
                ("grid_occupied_boxes", ctypes.c_int64), ("grid_max_occupancy", ctypes.c_int64),
                ("box_length", ctypes.c_double), ("origin", ctypes.c_double * 3),
                ("t_sort_ms", ctypes.c_float), ("t_grid_ms", ctypes.c_float),
                ("t_force_ms", ctypes.c_float), ("t_total_ms", ctypes.c_float),
                ("sweep_kind", ctypes.c_int32), ("reserved", ctypes.c_int32)]


_lib = None
_P = ctypes.c_void_p
_I64 = ctypes.c_int64


def load():
    """Load the shared library (raises NativeUnavailable if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable("%s is not built; run __graft_entry__.build()" % LIB_PATH)
    L = ctypes.CDLL(LIB_PATH)
    sig = {
        "cg_abi_version": ([], ctypes.c_int),
        "cg_device_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
        "cg_create": ([ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)], ctypes.c_int),
        "cg_destroy": ([_P], None),
        "cg_last_error": ([_P], ctypes.c_char_p),
        "cg_set_option": ([_P, ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "cg_stream": ([_P], _P),
        "cg_upload": ([_P, _I64, _P, _P, _P, _P, _P, _P], ctypes.c_int),
        "cg_download": ([_P] + [_P] * 9, ctypes.c_int),
        "cg_count": ([_P], _I64),
        "cg_launch_count": ([_P], _I64),
        "cg_host_alloc": ([_I64], _P),
        "cg_host_free": ([_P], None),
        "cg_step": ([_P, _P, ctypes.c_double, _I64, ctypes.c_int, ctypes.POINTER(StepStatsC)],
                    ctypes.c_int),
        "cg_fetch_stats": ([_P, _I64, ctypes.POINTER(StepStatsC)], ctypes.c_int),
        "cg_build_grid": ([_P, ctypes.c_double, _I64, ctypes.POINTER(StepStatsC)], ctypes.c_int),
        "cg_synchronize": ([_P], ctypes.c_int),
        "cg_grid_export": ([_P, _P, _P], ctypes.c_int),
        "cg_record_export": ([_P, _P, _P], ctypes.c_int),
        "cg_box_ids": ([_P, _I64, _P, _P, _P] + [ctypes.c_double] * 4 + [_I64] * 3 + [_P],
                       ctypes.c_int),
        "cg_force_phase": ([_P, _I64] + [_P] * 7 + [_I64] * 3 + [_P] * 5, ctypes.c_int),
        "cg_neighbor_counts": ([_P, ctypes.c_double, _P], ctypes.c_int),
        "cg_list_stats": ([_P, _P], ctypes.c_int),
        "cg_behavior": ([_P, _I64, ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_uint64, _P],
                        ctypes.c_int),
        "cg_unit_vectors": ([_P, _I64, _P, _I64, _P], ctypes.c_int),
        "cg_step_download": ([_P, _P, ctypes.c_double, _I64, ctypes.c_int, ctypes.POINTER(StepStatsC)]
                             + [_P] * 9, ctypes.c_int),
        "cg_slab_list_epoch": ([_P], _I64),
        "cg_neighbor_fill": ([_P, ctypes.c_double, _P, _P], ctypes.c_int),
        "cg_record_bytes": ([_P], _I64),
        "cg_reserve": ([_P, _I64], ctypes.c_int),
        "cg_local_bbox": ([_P, _P], ctypes.c_int),
        "cg_slab_plan": ([_P, _P, ctypes.c_double, _I64, ctypes.c_int, ctypes.c_int, _P, _P],
                         ctypes.c_int),
        "cg_slab_pack": ([_P, _P], ctypes.c_int),
        "cg_slab_unpack": ([_P, _P, _P], ctypes.c_int),
        "cg_slab_step": ([_P, _P, ctypes.c_int, ctypes.POINTER(StepStatsC)], ctypes.c_int),
        "cg_slab_step_interior": ([_P, _P, ctypes.c_int], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    if L.cg_abi_version() != 6:
        raise NativeUnavailable("ABI version mismatch")
    _lib = L
    return L


def ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def check(rc, ctx=None):
    if rc == CG_OK:
        return
    msg = load().cg_last_error(ctx).decode() if ctx else ""
    if rc == CG_ERR_VALUE:
        raise ValueError(msg or "invalid argument")
    if rc == CG_ERR_GRID_OVERFLOW:
        raise GridOverflowError(msg)
    if rc == CG_ERR_STENCIL:
        raise StencilTooSmallError(msg)
    if rc == CG_ERR_POOL_CAPACITY:
        raise PoolCapacityError(msg)
    if rc == CG_ERR_NO_DEVICE:
        raise NativeUnavailable("no sm_100 CUDA device available")
    if rc == CG_ERR_STATE:
        raise RuntimeError(msg)
    raise CudaError(msg or "CUDA failure (status %d)" % rc)


class Context:
    """Owns one cg_context: an agent population resident on one GPU."""

    def __init__(self, device=0, dtype=np.float64):
        lib = load()
        self._lib = lib          # kept for close() at interpreter shutdown
        self.dtype = np.dtype(dtype)
        self.device = int(device)
        h = _P()
        rc = lib.cg_create(self.device, CG_FP64 if self.dtype == np.float64 else CG_FP32,
                           ctypes.byref(h))
        check(rc)
        self.h = h
        self.n = 0
        self.steps = 0          # successful cg_step calls == device step ids issued

    def close(self):
        if getattr(self, "h", None):
            self._lib.cg_destroy(self.h)
            self.h = None

    __del__ = close

    @property
    def launches(self):
        return int(load().cg_launch_count(self.h))

    def set_option(self, key, value):
        check(load().cg_set_option(self.h, key, value), self.h)

    @property
    def stream(self):
        return load().cg_stream(self.h)

    def upload(self, px, py, pz, diameter, adherence, uid):
        cols = [np.ascontiguousarray(c, self.dtype) for c in (px, py, pz, diameter, adherence)]
        uid = np.ascontiguousarray(uid, np.uint64)
        n = cols[0].shape[0]
        check(load().cg_upload(self.h, n, *(ptr(c) for c in cols), ptr(uid)), self.h)
        self.n = n

    def download(self, columns=("px", "py", "pz", "diameter", "adherence", "uid", "dx", "dy", "dz"),
                 into=None):
        """Copy columns back; ``into`` may supply destination arrays (e.g. pinned)."""
        out = {}
        args = []
        for name in ("px", "py", "pz", "diameter", "adherence", "uid", "dx", "dy", "dz"):
            if name in columns:
                dst = None if into is None else into.get(name)
                if dst is None or dst.shape[0] != self.n:
                    dst = np.empty(self.n, np.uint64 if name == "uid" else self.dtype)
                out[name] = dst
                args.append(ptr(dst))
            else:
                args.append(None)
        check(load().cg_download(self.h, *args), self.h)
        return out

    def step_download(self, params5, interaction_radius=None, box_cap=1 << 24, flags=0, into=None,
                      columns=("px", "py", "pz", "diameter", "adherence", "uid", "dx", "dy", "dz")):
        """step + download with the unchanged columns copied during the sweep
        (cg_step_download); returns (stats, the requested columns)."""
        p = np.ascontiguousarray(params5, np.float64)
        ir = float("nan") if interaction_radius is None else float(interaction_radius)
        out, args = {}, []
        for name in ("px", "py", "pz", "diameter", "adherence", "uid", "dx", "dy", "dz"):
            if name not in columns:
                args.append(None)
                continue
            dst = None if into is None else into.get(name)
            if dst is None or dst.shape[0] != self.n:
                dst = np.empty(self.n, np.uint64 if name == "uid" else self.dtype)
            out[name] = dst
            args.append(ptr(dst))
        st = StepStatsC()
        check(load().cg_step_download(self.h, ptr(p), ir, int(box_cap), int(flags), ctypes.byref(st), *args),
              self.h)
        self.steps += 1
        return st, out

    def step(self, params5, interaction_radius=None, box_cap=1 << 24, flags=0, wait=True):
        p = np.ascontiguousarray(params5, np.float64)
        ir = float("nan") if interaction_radius is None else float(interaction_radius)
        st = StepStatsC() if wait else None
        rc = load().cg_step(self.h, ptr(p), ir, int(box_cap), int(flags),
                            ctypes.byref(st) if wait else None)
        check(rc, self.h)
        self.steps += 1
        return st if wait else self.steps - 1

    def fetch_stats(self, step_id):
        st = StepStatsC()
        check(load().cg_fetch_stats(self.h, int(step_id), ctypes.byref(st)), self.h)
        return st

    def build_grid(self, interaction_radius=None, box_cap=1 << 24):
        st = StepStatsC()
        ir = float("nan") if interaction_radius is None else float(interaction_radius)
        check(load().cg_build_grid(self.h, ir, int(box_cap), ctypes.byref(st)), self.h)
        return st

    def synchronize(self):
        check(load().cg_synchronize(self.h), self.h)

    def grid_export(self, num_boxes):
        bi = np.empty(self.n, np.int64)
        bc = np.empty(num_boxes, np.int64)
        check(load().cg_grid_export(self.h, ptr(bi), ptr(bc)), self.h)
        return bi, bc

    def behavior(self, step_index, volume_growth_rate, division_diameter, division_enabled, next_uid):
        """cg_behavior: grow (and divide) the resident pool; returns the number
        of divisions (the caller's next_uid advances by it)."""
        out = ctypes.c_int64(0)
        check(load().cg_behavior(self.h, int(step_index), float(volume_growth_rate), float(division_diameter),
                                 1 if division_enabled else 0, int(next_uid), ctypes.byref(out)), self.h)
        self.n += int(out.value)
        return int(out.value)

    def unit_vectors(self, uid, step):
        """rng.unit_vector(uid[i], step) for every uid, on the device: (n, 3) f64."""
        uid = np.ascontiguousarray(uid, np.uint64)
        out = np.empty((uid.shape[0], 3), np.float64)
        check(load().cg_unit_vectors(self.h, uid.shape[0], ptr(uid), int(step), ptr(out)), self.h)
        return out

    def list_stats(self):
        """(builds, list steps, valid, skin, slab list steps with the interior
        sweep overlapping the ghost refresh, list steps that swept the
        sub-list) of the neighbour-list reuse."""
        out = np.zeros(6, np.int64)
        check(load().cg_list_stats(self.h, ptr(out)), self.h)
        return {"builds": int(out[0]), "list_steps": int(out[1]), "valid": bool(out[2]),
                "skin": out[3] * 1e-6, "overlapped": int(out[4]), "inner_steps": int(out[5])}

    # ---- radius queries (spatial.neighbor_counts / neighbor_csr)
    def neighbor_counts(self, radius):
        out = np.empty(self.n, np.int64)
        check(load().cg_neighbor_counts(self.h, float(radius), ptr(out)), self.h)
        return out

    def neighbor_csr(self, radius):
        counts = self.neighbor_counts(radius)
        indptr = np.zeros(self.n + 1, np.int64)
        np.cumsum(counts, out=indptr[1:])
        indices = np.empty(int(indptr[-1]), np.int64)
        check(load().cg_neighbor_fill(self.h, float(radius), ptr(indptr), ptr(indices)), self.h)
        return indptr, indices

    # ---- x-slab decomposition (see include/cellgrid_b200.h and distributed.py)
    @property
    def record_bytes(self):
        return int(load().cg_record_bytes(self.h))

    def reserve(self, capacity):
        check(load().cg_reserve(self.h, int(capacity)), self.h)

    def local_bbox(self):
        """min xyz, max xyz, max diameter, last step's largest squared
        displacement, last step's neighbour-list overflows, -min diameter,
        max uid (cg_local_bbox)."""
        out = np.empty(11, np.float64)
        check(load().cg_local_bbox(self.h, ptr(out)), self.h)
        return out

    def slab_plan(self, bbox, world, rank, interaction_radius=None, box_cap=1 << 24):
        """-> (counts[3 * world], planes[2]); see cg_slab_plan."""
        bb = np.ascontiguousarray(bbox, np.float64)
        counts = np.zeros(3 * world, np.int64)
        planes = np.zeros(2, np.int64)
        ir = float("nan") if interaction_radius is None else float(interaction_radius)
        check(load().cg_slab_plan(self.h, ptr(bb), ir, int(box_cap), int(world), int(rank),
                                  ptr(counts), ptr(planes)), self.h)
        return counts, planes

    def slab_list_epoch(self):
        """-1 for a rebuild step, else the list epoch of the planned refresh step."""
        return int(load().cg_slab_list_epoch(self.h))

    def slab_pack(self, send_ptr):
        check(load().cg_slab_pack(self.h, send_ptr), self.h)
        self.n = int(load().cg_count(self.h))

    def slab_unpack(self, recv_ptr, recv_counts):
        rc = np.ascontiguousarray(recv_counts, np.int64)
        check(load().cg_slab_unpack(self.h, recv_ptr, ptr(rc)), self.h)
        self.n = int(load().cg_count(self.h))

    def slab_step_interior(self, params5, flags=0):
        """cg_slab_step_interior: the interior rows' list sweep, enqueued before
        the ghost refresh is unpacked (a no-op on rebuild steps)."""
        p = np.ascontiguousarray(params5, np.float64)
        check(load().cg_slab_step_interior(self.h, ptr(p), int(flags)), self.h)

    def slab_step(self, params5, flags=0, wait=True):
        p = np.ascontiguousarray(params5, np.float64)
        st = StepStatsC() if wait else None
        check(load().cg_slab_step(self.h, ptr(p), int(flags), ctypes.byref(st) if wait else None),
              self.h)
        self.steps += 1
        self.n = int(load().cg_count(self.h))
        return st if wait else self.steps - 1

    def record_export(self):
        m = np.empty(self.n, np.int32)
        nk = np.empty(self.n, np.int32)
        check(load().cg_record_export(self.h, ptr(m), ptr(nk)), self.h)
        return m, nk


class PinnedArray:
    """numpy view of page-locked host memory (cg_host_alloc); freed on drop."""

    @classmethod
    def empty(cls, n, dtype):
        dtype = np.dtype(dtype)
        nbytes = max(1, int(n) * dtype.itemsize)
        p = load().cg_host_alloc(nbytes)
        if not p:
            raise MemoryError("cg_host_alloc(%d) failed" % nbytes)
        buf = (ctypes.c_char * nbytes).from_address(p)
        arr = np.frombuffer(buf, dtype=dtype, count=int(n))
        import weakref
        weakref.finalize(buf, lambda q=p: load().cg_host_free(q))
        return arr

    @classmethod
    def copy_of(cls, a):
        out = cls.empty(a.shape[0], a.dtype)
        out[:] = a
        return out
