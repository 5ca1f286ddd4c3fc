"""Drop-in replacement for the reference kernel module `lumenwave.core._kernels`.

Same names, argument meaning and error behaviour as `_kernels.py`; every call
runs an sm_100a kernel of liblw_b200.so through its C ABI (include/lw_b200.h).
There is no interpreted or CPU fallback: importing this module without the
built library raises ImportError.

Divergence (documented in DESIGN.md §2): `intersect_batch` takes an optional
`mode` ("corrected" by default, "compat" for the pristine reference including
defects D1/D2, "brute" for the exhaustive oracle).  The reference's own tests
(test_accel.py:75-145) specify the corrected behaviour.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from paper_1705_01263_b200 import _abi
from paper_1705_01263_b200._abi import check, ptr

_lib = _abi.lib()  # fail loudly at import if the CUDA library is missing

PI = 3.141592653589793
TWO_PI = 6.283185307179586
FOUR_PI = 12.566370614359172
INV_PI = 0.3183098861837907
INF = 1e308

# Path stages (_kernels.py:42-48)
STAGE_GENERATE = 0
STAGE_TRACE = 1
STAGE_MATERIAL = 2
STAGE_NEE = 3
STAGE_ENVMATTE = 4
STAGE_TERMINATED = 5
STAGE_COUNT = 6

_MODES = {
    "compat": _abi.LW_TRAVERSE_COMPAT,
    "corrected": _abi.LW_TRAVERSE_CORRECTED,
    "brute": _abi.LW_TRAVERSE_BRUTE,
}
default_traversal_mode = "corrected"


def is_compiled() -> bool:
    """_kernels.py:30 -- the B200 module is always native."""
    return True


def _i64(a):
    a = np.asarray(a)
    if a.dtype != np.int64 or not a.flags["C_CONTIGUOUS"]:
        raise ValueError("expected a C-contiguous int64 array")
    return a


def _f64(a):
    a = np.asarray(a)
    if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
        raise ValueError("expected a C-contiguous float64 array")
    return a


def halton_batch(bases, perm_flat, perm_offset, dim, indices, out):
    """Evaluate one Halton dimension for many indices (_kernels.py:211-222)."""
    bases = _i64(bases)
    perm_flat = _i64(perm_flat)
    perm_offset = _i64(perm_offset)
    idx = _i64(indices)
    res = _f64(out)
    n = idx.shape[0]
    if res.shape[0] < n:
        raise ValueError("out is shorter than indices")
    check(_lib.lw_halton_batch(ptr(bases, C.c_int64), len(bases), ptr(perm_flat, C.c_int64), len(perm_flat),
                               ptr(perm_offset, C.c_int64), int(dim), ptr(idx, C.c_int64), n, ptr(res, C.c_double)))


def sample_pixel_offset(u1: float, u2: float) -> tuple:
    """Filter-importance-sampled anti-aliasing offset in pixels (_kernels.py:132-134)."""
    u = np.array([u1, u2], dtype=np.float64)
    out = np.empty(2)
    check(_lib.lw_pixel_offset_batch(ptr(u, C.c_double), 1, ptr(out, C.c_double)))
    return (float(out[0]), float(out[1]))


def pixel_offset_batch(u):
    """Batched `sample_pixel_offset`: u [n, 2] -> offsets [n, 2]."""
    u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1, 2)
    out = np.empty_like(u)
    check(_lib.lw_pixel_offset_batch(ptr(u, C.c_double), len(u), ptr(out, C.c_double)))
    return out


def compress_unit_vector(x: float, y: float, z: float) -> int:
    """Pack a unit vector into 2x16 bits (_kernels.py:302-307)."""
    if math.sqrt(x * x + y * y + z * z) == 0.0:
        raise ValueError("zero vector cannot be compressed")
    v = np.array([x, y, z], dtype=np.float64)
    out = np.empty(1, dtype=np.int64)
    check(_lib.lw_oct_encode_batch(ptr(v, C.c_double), 1, ptr(out, C.c_int64)))
    return int(out[0])


def decompress_unit_vector(packed: int) -> tuple:
    """Inverse of compress_unit_vector, renormalised (_kernels.py:310-318)."""
    p = np.array([int(packed)], dtype=np.int64)
    d = np.empty(3)
    check(_lib.lw_oct_decode_batch(ptr(p, C.c_int64), 1, ptr(d, C.c_double)))
    x, y, z = (float(d[0]), float(d[1]), float(d[2]))
    n = math.sqrt(x * x + y * y + z * z)
    if n == 0.0:
        return (0.0, 0.0, 1.0)
    return (x / n, y / n, z / n)


def oct_roundtrip_batch(vecs, out):
    """Compress+decompress rows of `vecs` into `out` (_kernels.py:321-342)."""
    v = _f64(vecs)
    o = _f64(out)
    if v.ndim != 2 or v.shape[1] != 3 or o.shape != v.shape:
        raise ValueError("vecs and out must both be (n, 3)")
    check(_lib.lw_oct_roundtrip_batch(ptr(v, C.c_double), v.shape[0], ptr(o, C.c_double)))


def intersect_batch(bounds, children, order, verts, instances, origins, dirs, tmaxs, out_t, out_tri, out_bary,
                    mode: str | None = None):
    """Closest-hit query for a batch of rays (_kernels.py:548-585)."""
    b = _f64(bounds)
    ch = _i64(children)
    od = _i64(order)
    tv = _f64(verts)
    o = _f64(origins)
    d = _f64(dirs)
    tm = _f64(tmaxs)
    ot = _f64(out_t)
    otri = _i64(out_tri)
    ob = _f64(out_bary)
    n = o.shape[0]
    m = _MODES[mode or default_traversal_mode]
    check(_lib.lw_intersect_batch(m, ptr(b, C.c_double), ptr(ch, C.c_int64), b.shape[0], ptr(od, C.c_int64),
                                  ptr(tv, C.c_double), tv.shape[0], ptr(o, C.c_double), ptr(d, C.c_double),
                                  ptr(tm, C.c_double), n, ptr(ot, C.c_double), ptr(otri, C.c_int64),
                                  ptr(ob, C.c_double)))
