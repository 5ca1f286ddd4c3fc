"""ctypes wrapper of the C restatement oracle and loader for the reference kernels.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg.  The product never imports it.

- `liblw_oracle.so` (oracle/lw_oracle.c): CPU restatement of every hot-path row.
- `ref_kernels(variant)`: the reference's own `_kernels` module compiled from
  /root/reference by oracle/Makefile into oracle/_ref/{pristine,corrected}/.
  Returns None when it has not been built (e.g. a box without the reference).
"""

from __future__ import annotations

import ctypes as C
import glob
import importlib.util
import os
import subprocess

import numpy as np

from paper_1705_01263_b200 import _abi
from paper_1705_01263_b200._abi import LwRenderParams, LwRenderStats, LwSceneDesc, ptr

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liblw_oracle.so")

_pd = C.POINTER(C.c_double)
_pi64 = C.POINTER(C.c_int64)
_pi32 = C.POINTER(C.c_int32)
_V = C.c_void_p

_SIG = {
    "lwo_halton_batch": (None, [_pi64, _pi64, _pi64, C.c_int64, _pi64, C.c_int64, _pd]),
    "lwo_gauss_filter_offset": (C.c_double, [C.c_double]),
    "lwo_pixel_offset_batch": (None, [_pd, C.c_int64, _pd]),
    "lwo_oct_encode": (C.c_int64, [C.c_double, C.c_double, C.c_double]),
    "lwo_oct_decode": (None, [C.c_int64, _pd]),
    "lwo_oct_roundtrip_batch": (None, [_pd, C.c_int64, _pd]),
    "lwo_intersect_batch": (None, [C.c_int, _pd, _pi64, _pi64, _pd, C.c_int64, _pd, _pd, _pd, C.c_int64, _pd, _pi64, _pd]),
    "lwo_build_bvh": (C.c_int64, [_pd, C.c_int64, _pd, _pi64, _pi64]),
    "lwo_alias_build": (C.c_int, [_pd, C.c_int64, _pd, _pi32, _pd]),
    "lwo_scene_create": (_V, [C.POINTER(LwSceneDesc)]),
    "lwo_scene_destroy": (None, [_V]),
    "lwo_trace_closest_batch": (None, [_V, _pd, _pd, _pd, C.c_int64, _pd, _pi64, _pd]),
    "lwo_trace_any_batch": (None, [_V, _pd, _pd, _pd, C.c_int64, _pi32]),
    "lwo_camera_rays": (None, [_V, C.POINTER(LwRenderParams), _pi64, C.c_int64, _pd, _pd]),
    "lwo_light_tree": (C.c_int64, [_V, _pd, _pi32, C.POINTER(C.c_uint64), _pi32]),
    "lwo_light_sample_batch": (None, [_V, _pd, _pd, _pd, C.c_int64, _pi64, _pd, _pd]),
    "lwo_light_pdf_batch": (None, [_V, _pi64, _pd, _pd, C.c_int64, _pd]),
    "lwo_env_pyramid_info": (C.c_int, [_V, _pi32]),
    "lwo_env_sample_batch": (None, [_V, _pi64, _pd, C.c_int64, _pi64, _pd, _pd]),
    "lwo_env_pdf_batch": (None, [_V, _pi64, _pi64, C.c_int64, _pd]),
    "lwo_render": (None, [_V, C.POINTER(LwRenderParams), C.c_int64, C.c_int64, C.c_int64, C.c_int64, _pi64, C.c_int, C.POINTER(LwRenderStats)]),
    "lwo_render_lpe": (None, [_V, C.POINTER(LwRenderParams), C.c_int64, C.c_int64, C.c_int64, C.c_int64, _pi64,
                               C.c_int, C.c_int, C.POINTER(C.c_int16), C.POINTER(C.c_uint8), C.c_int, _pi64, C.c_int,
                               C.POINTER(LwRenderStats)]),
    "lwo_sincos2pi": (None, [C.c_double, _pd, _pd]),
    "lwo_bsdf_eval_batch": (None, [C.POINTER(_abi.LwMaterial), _pd, _pd, C.c_int64, _pd, _pd]),
    "lwo_bsdf_sample_batch": (None, [C.POINTER(_abi.LwMaterial), _pd, _pi32, _pd, C.c_int64, _pd, _pd, _pd, _pi32]),
    "lwo_nee_light_sample_batch": (None, [_V, _pd, _pd, _pd, C.c_int64, _pd, _pd, _pd, _pd, _pi64]),
    "lwo_emission_pdf_batch": (None, [_V, _pd, _pd, _pi32, C.c_int64, _pd, _pd, _pi64]),
    "lwo_atan2": (C.c_double, [C.c_double, C.c_double]),
}

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        h = C.CDLL(LIB)
        for name, (res, args) in _SIG.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib = h
    return _lib


def ref_kernels(variant: str = "pristine"):
    """The reference's compiled `_kernels` module (oracle/_ref), or None."""
    hits = glob.glob(os.path.join(HERE, "_ref", variant, "_kernels*.so"))
    if not hits:
        return None
    spec = importlib.util.spec_from_file_location("_kernels", hits[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


# ---- thin numpy wrappers ------------------------------------------------------------


def halton_batch(bases, perm_flat, perm_offset, dim, indices):
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    out = np.empty(len(idx))
    lib().lwo_halton_batch(ptr(np.ascontiguousarray(bases, np.int64), C.c_int64),
                           ptr(np.ascontiguousarray(perm_flat, np.int64), C.c_int64),
                           ptr(np.ascontiguousarray(perm_offset, np.int64), C.c_int64),
                           int(dim), ptr(idx, C.c_int64), len(idx), ptr(out, C.c_double))
    return out


def pixel_offset_batch(u):
    u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1, 2)
    out = np.empty_like(u)
    lib().lwo_pixel_offset_batch(ptr(u, C.c_double), len(u), ptr(out, C.c_double))
    return out


def oct_encode(v):
    return int(lib().lwo_oct_encode(float(v[0]), float(v[1]), float(v[2])))


def oct_roundtrip_batch(vecs):
    v = np.ascontiguousarray(vecs, dtype=np.float64).reshape(-1, 3)
    out = np.zeros_like(v)
    lib().lwo_oct_roundtrip_batch(ptr(v, C.c_double), len(v), ptr(out, C.c_double))
    return out


def intersect_batch(mode, bounds, children, order, verts, origins, dirs, tmaxs):
    o = np.ascontiguousarray(origins, np.float64)
    d = np.ascontiguousarray(dirs, np.float64)
    tm = np.ascontiguousarray(tmaxs, np.float64)
    n = len(o)
    out_t = np.empty(n)
    out_tri = np.empty(n, np.int64)
    out_b = np.empty((n, 2))
    verts = np.ascontiguousarray(verts, np.float64)
    lib().lwo_intersect_batch(int(mode), ptr(np.ascontiguousarray(bounds, np.float64), C.c_double),
                              ptr(np.ascontiguousarray(children, np.int64), C.c_int64),
                              ptr(np.ascontiguousarray(order, np.int64), C.c_int64),
                              ptr(verts, C.c_double), len(verts), ptr(o, C.c_double), ptr(d, C.c_double),
                              ptr(tm, C.c_double), n, ptr(out_t, C.c_double), ptr(out_tri, C.c_int64),
                              ptr(out_b, C.c_double))
    return out_t, out_tri, out_b


def build_bvh(verts):
    v = np.ascontiguousarray(verts, np.float64).reshape(-1, 9)
    n = len(v)
    cap = max(2 * n, 1)
    bounds = np.zeros((cap, 6))
    children = np.zeros((cap, 2), np.int64)
    order = np.zeros(max(n, 1), np.int64)
    nn = lib().lwo_build_bvh(ptr(v, C.c_double), n, ptr(bounds, C.c_double), ptr(children, C.c_int64),
                             ptr(order, C.c_int64))
    return bounds[:nn].copy(), children[:nn].copy(), order[:n].copy()


def alias_build(weights):
    w = np.ascontiguousarray(weights, np.float64)
    prob = np.zeros(len(w))
    alias = np.zeros(len(w), np.int32)
    pdf = np.zeros(len(w))
    rc = lib().lwo_alias_build(ptr(w, C.c_double), len(w), ptr(prob, C.c_double), ptr(alias, C.c_int32),
                               ptr(pdf, C.c_double))
    if rc:
        raise ValueError("alias build rejected the weights")
    return prob, alias, pdf


def sincos2pi(u):
    s = C.c_double()
    c = C.c_double()
    lib().lwo_sincos2pi(float(u), C.byref(s), C.byref(c))
    return s.value, c.value


def atan2(y, x):
    return lib().lwo_atan2(float(y), float(x))


def bsdf_evaluate(m, wo, wi):
    """Oracle bsdf_eval (lw_oracle.c) with the semantics of paper_1705_01263_b200.bsdf.bsdf_evaluate."""
    wo = np.ascontiguousarray(wo, np.float64).reshape(-1, 3)
    wi = np.ascontiguousarray(wi, np.float64).reshape(-1, 3)
    n = max(len(wo), len(wi))
    wo = np.ascontiguousarray(np.broadcast_to(wo, (n, 3)))
    wi = np.ascontiguousarray(np.broadcast_to(wi, (n, 3)))
    f, pdf = np.empty((n, 3)), np.empty(n)
    lib().lwo_bsdf_eval_batch(C.byref(m), ptr(wo, C.c_double), ptr(wi, C.c_double), n, ptr(f, C.c_double),
                              ptr(pdf, C.c_double))
    return f, pdf


def bsdf_sample(m, wo, uv, front=True):
    uv = np.ascontiguousarray(uv, np.float64).reshape(-1, 2)
    n = len(uv)
    wo = np.ascontiguousarray(np.broadcast_to(np.asarray(wo, np.float64).reshape(-1, 3), (n, 3)))
    fr = np.ascontiguousarray(np.broadcast_to(np.asarray(front, np.int32), (n,)))
    wi, w, pdf, fl = np.empty((n, 3)), np.empty((n, 3)), np.empty(n), np.empty(n, np.int32)
    lib().lwo_bsdf_sample_batch(C.byref(m), ptr(wo, C.c_double), ptr(fr, C.c_int32), ptr(uv, C.c_double), n,
                                ptr(wi, C.c_double), ptr(w, C.c_double), ptr(pdf, C.c_double), ptr(fl, C.c_int32))
    return {"wi": wi, "weight": w, "pdf": pdf, "sampled": (fl & 1) != 0, "delta": (fl & 2) != 0,
            "transmit": (fl & 4) != 0, "event": fl >> 8}


class OracleScene:
    """Oracle-side scene built from the same packed description the GPU receives."""

    def __init__(self, packed):
        self.packed = packed  # keeps numpy buffers alive
        self.h = lib().lwo_scene_create(C.byref(packed.desc))

    def close(self):
        if self.h:
            lib().lwo_scene_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def trace_closest(self, origins, dirs, tmaxs=None):
        o = np.ascontiguousarray(origins, np.float64)
        d = np.ascontiguousarray(dirs, np.float64)
        n = len(o)
        tm = np.full(n, np.inf) if tmaxs is None else np.ascontiguousarray(tmaxs, np.float64)
        t = np.empty(n)
        tri = np.empty(n, np.int64)
        b = np.empty((n, 2))
        lib().lwo_trace_closest_batch(self.h, ptr(o, C.c_double), ptr(d, C.c_double), ptr(tm, C.c_double), n,
                                      ptr(t, C.c_double), ptr(tri, C.c_int64), ptr(b, C.c_double))
        return t, tri, b

    def trace_any(self, origins, dirs, tmaxs):
        o = np.ascontiguousarray(origins, np.float64)
        d = np.ascontiguousarray(dirs, np.float64)
        tm = np.ascontiguousarray(tmaxs, np.float64)
        n = len(o)
        occ = np.empty(n, np.int32)
        lib().lwo_trace_any_batch(self.h, ptr(o, C.c_double), ptr(d, C.c_double), ptr(tm, C.c_double), n,
                                  ptr(occ, C.c_int32))
        return occ

    def light_tree(self):
        """Light hierarchy (oracle lt_build): (nodes [n,15], right [n], path, depth) or None."""
        n = lib().lwo_light_tree(self.h, None, None, None, None)
        if n == 0:
            return None
        ne = self.packed.nemit
        nodes = np.empty((n, 15))
        right = np.empty(n, np.int32)
        path = np.empty(max(ne, 1), np.uint64)
        depth = np.empty(max(ne, 1), np.int32)
        lib().lwo_light_tree(self.h, ptr(nodes, C.c_double), ptr(right, C.c_int32), ptr(path, C.c_uint64),
                             ptr(depth, C.c_int32))
        return nodes, right, path[:ne], depth[:ne]

    def light_sample(self, x, nrm, u):
        x = np.ascontiguousarray(x, np.float64)
        nrm = np.ascontiguousarray(nrm, np.float64)
        u = np.ascontiguousarray(u, np.float64)
        n = len(u)
        e, p, uo = np.empty(n, np.int64), np.empty(n), np.empty(n)
        lib().lwo_light_sample_batch(self.h, ptr(x, C.c_double), ptr(nrm, C.c_double), ptr(u, C.c_double), n,
                                     ptr(e, C.c_int64), ptr(p, C.c_double), ptr(uo, C.c_double))
        return e, p, uo

    def light_pdf(self, e, x, nrm):
        e = np.ascontiguousarray(e, np.int64)
        x = np.ascontiguousarray(x, np.float64)
        nrm = np.ascontiguousarray(nrm, np.float64)
        p = np.empty(len(e))
        lib().lwo_light_pdf_batch(self.h, ptr(e, C.c_int64), ptr(x, C.c_double), ptr(nrm, C.c_double), len(e),
                                  ptr(p, C.c_double))
        return p

    def env_pyramid_levels(self):
        n = C.c_int32()
        lib().lwo_env_pyramid_info(self.h, C.byref(n))
        return n.value

    def env_sample(self, packed_normal, uv):
        pk = np.ascontiguousarray(packed_normal, np.int64)
        uv = np.ascontiguousarray(uv, np.float64)
        n = len(pk)
        t, p, o = np.empty(n, np.int64), np.empty(n), np.empty((n, 2))
        lib().lwo_env_sample_batch(self.h, ptr(pk, C.c_int64), ptr(uv, C.c_double), n, ptr(t, C.c_int64),
                                   ptr(p, C.c_double), ptr(o, C.c_double))
        return t, p, o

    def env_pdf(self, packed_normal, texel):
        pk = np.ascontiguousarray(packed_normal, np.int64)
        tx = np.ascontiguousarray(texel, np.int64)
        p = np.empty(len(pk))
        lib().lwo_env_pdf_batch(self.h, ptr(pk, C.c_int64), ptr(tx, C.c_int64), len(pk), ptr(p, C.c_double))
        return p

    def nee_light_sample(self, points, facing_normals, uv):
        uv = np.ascontiguousarray(uv, np.float64).reshape(-1, 2)
        n = len(uv)
        p = np.ascontiguousarray(np.broadcast_to(np.asarray(points, np.float64).reshape(-1, 3), (n, 3)))
        nrm = np.ascontiguousarray(np.broadcast_to(np.asarray(facing_normals, np.float64).reshape(-1, 3), (n, 3)))
        wi, le, pdf, tm, e = np.empty((n, 3)), np.empty((n, 3)), np.empty(n), np.empty(n), np.empty(n, np.int64)
        lib().lwo_nee_light_sample_batch(self.h, ptr(p, C.c_double), ptr(nrm, C.c_double), ptr(uv, C.c_double), n,
                                         ptr(wi, C.c_double), ptr(le, C.c_double), ptr(pdf, C.c_double),
                                         ptr(tm, C.c_double), ptr(e, C.c_int64))
        return {"wi": wi, "radiance": le, "pdf": pdf, "tmax": tm, "emitter": e}

    def emission_pdf(self, origins, dirs, nprev=None):
        d = np.ascontiguousarray(dirs, np.float64).reshape(-1, 3)
        n = len(d)
        o = np.ascontiguousarray(np.broadcast_to(np.asarray(origins, np.float64).reshape(-1, 3), (n, 3)))
        npv = np.zeros(n, np.int32) if nprev is None else np.ascontiguousarray(  # packed normals are 32-bit patterns
            np.broadcast_to((np.asarray(nprev, np.int64) & 0xFFFFFFFF).astype(np.uint32).view(np.int32), (n,)))
        le, pdf, e = np.empty((n, 3)), np.empty(n), np.empty(n, np.int64)
        lib().lwo_emission_pdf_batch(self.h, ptr(o, C.c_double), ptr(d, C.c_double), ptr(npv, C.c_int32), n,
                                     ptr(le, C.c_double), ptr(pdf, C.c_double), ptr(e, C.c_int64))
        return {"radiance": le, "pdf": pdf, "emitter": e}

    def camera_rays(self, params, sample_index):
        idx = np.ascontiguousarray(sample_index, np.int64)
        o = np.empty((len(idx), 3))
        d = np.empty((len(idx), 3))
        lib().lwo_camera_rays(self.h, C.byref(params.struct), ptr(idx, C.c_int64), len(idx), ptr(o, C.c_double),
                              ptr(d, C.c_double))
        return o, d

    def render_lpe(self, params, it_begin, it_end, tables, pix_begin=0, pix_end=None, nthreads=0):
        """render() plus LPE layers (tables = lpe.compile_layers(...)): (fb, {name: layer fb}, stats)."""
        W, H = params.width, params.height
        if pix_end is None:
            pix_end = W * H
        fb = np.zeros((H * W, 3), np.int64)
        nl = len(tables.names)
        lfb = np.zeros((nl, H * W, 3), np.int64)
        tr = np.ascontiguousarray(tables.trans, np.int16)
        ac = np.ascontiguousarray(tables.accept, np.uint8)
        st = LwRenderStats()
        lib().lwo_render_lpe(self.h, C.byref(params.struct), int(pix_begin), int(pix_end), int(it_begin), int(it_end),
                             ptr(fb, C.c_int64), nl, len(tr), ptr(tr, C.c_int16), ptr(ac, C.c_uint8),
                             int(tables.start), ptr(lfb, C.c_int64), int(nthreads), C.byref(st))
        return fb, {n: lfb[k] for k, n in enumerate(tables.names)}, st.as_dict()

    def render(self, params, it_begin, it_end, pix_begin=0, pix_end=None, nthreads=0):
        W, H = params.width, params.height
        if pix_end is None:
            pix_end = W * H
        fb = np.zeros((H * W, 3), np.int64)
        st = LwRenderStats()
        lib().lwo_render(self.h, C.byref(params.struct), int(pix_begin), int(pix_end), int(it_begin), int(it_end),
                         ptr(fb, C.c_int64), int(nthreads), C.byref(st))
        return fb, st.as_dict()
