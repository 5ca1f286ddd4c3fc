"""BSDF evaluate / sample and the MIS weight on the GPU.

The same device functions the render engines call (`lw_integrator.cuh`: lw_layer_weights,
lw_bsdf_eval, lw_bsdf_sample, lw_mis_balance), exposed as batch entries of liblw_b200.so so the
SPEC known answers can be checked directly: Lambert rho/pi with pdf cos/pi, Fresnel 0.04 at normal
incidence for ior 1.5, the sample -> evaluate pdf round trip, the hemisphere integral of the pdf,
and the balance-heuristic weight 0.5 for equal pdfs.

Directions are in the local shading frame (z = shading normal); `wo` points away from the surface
towards the previous vertex.  Materials are `scene.Material` records (packed with the renderer's
own rules) or already packed `LwMaterial` structs.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from paper_1705_01263_b200 import _abi
from paper_1705_01263_b200._abi import LwMaterial, check, ptr

EVENTS = {1: "RD", 2: "RG", 3: "RS", 4: "TS"}  # LW_EV_* of a sampled lobe


def _material(m) -> LwMaterial:
    if isinstance(m, LwMaterial):
        return m
    from paper_1705_01263_b200.scene import _pack_material

    return _pack_material(m)


def _dirs(v, n=None):
    a = np.ascontiguousarray(v, np.float64).reshape(-1, 3)
    if n is not None and len(a) == 1 and n > 1:
        a = np.ascontiguousarray(np.repeat(a, n, axis=0))
    return a


def bsdf_evaluate(material, wo, wi):
    """(f [n,3], pdf [n]) for local directions wo, wi (either may be a single direction)."""
    wo, wi = np.asarray(wo, np.float64).reshape(-1, 3), np.asarray(wi, np.float64).reshape(-1, 3)
    n = max(len(wo), len(wi))
    wo, wi = _dirs(wo, n), _dirs(wi, n)
    f, pdf = np.empty((n, 3)), np.empty(n)
    m = _material(material)
    check(_abi.lib().lw_bsdf_eval_batch(C.byref(m), ptr(wo, C.c_double), ptr(wi, C.c_double), n,
                                        ptr(f, C.c_double), ptr(pdf, C.c_double)))
    return f, pdf


def bsdf_sample(material, wo, uv, front=True):
    """Sample the layered BSDF for local wo and uniforms uv [n,2]: dict of wi [n,3], weight [n,3]
    (f*cos/pdf; delta lobes carry their throughput), pdf [n] (0 for delta lobes), sampled / delta /
    transmit flags and the LPE event code."""
    uv = np.ascontiguousarray(uv, np.float64).reshape(-1, 2)
    n = len(uv)
    wo = _dirs(wo, n)
    fr = np.ascontiguousarray(np.broadcast_to(np.asarray(front, np.int32), (n,)))
    wi, w, pdf, fl = np.empty((n, 3)), np.empty((n, 3)), np.empty(n), np.empty(n, np.int32)
    m = _material(material)
    check(_abi.lib().lw_bsdf_sample_batch(C.byref(m), ptr(wo, C.c_double), ptr(fr, C.c_int32), ptr(uv, C.c_double), n,
                                          ptr(wi, C.c_double), ptr(w, C.c_double), ptr(pdf, C.c_double),
                                          ptr(fl, C.c_int32)))
    return {"wi": wi, "weight": w, "pdf": pdf, "sampled": (fl & 1) != 0, "delta": (fl & 2) != 0,
            "transmit": (fl & 4) != 0, "event": fl >> 8}


def mis_weight(pdf_a, pdf_b):
    """Balance-heuristic weight of strategy a against b, as the engines compute it."""
    a = np.ascontiguousarray(pdf_a, np.float64).reshape(-1)
    b = np.ascontiguousarray(np.broadcast_to(np.asarray(pdf_b, np.float64), a.shape))
    out = np.empty(len(a))
    check(_abi.lib().lw_mis_weight_batch(ptr(a, C.c_double), ptr(b, C.c_double), len(a), ptr(out, C.c_double)))
    return out
