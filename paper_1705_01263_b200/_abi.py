"""ctypes mirror of include/lw_b200.h and the loader for liblw_b200.so.

The library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a) into
``paper_1705_01263_b200/csrc/build/liblw_b200.so``.  There is no CPU fallback:
if the library is missing, :func:`lib` raises instead of degrading.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LW_B200_LIB") or os.path.join(_HERE, "csrc", "build", "liblw_b200.so")

LW_OK = 0
LW_ERR_INVALID = 1
LW_ERR_CUDA = 2
LW_ERR_NOMEM = 3
LW_ERR_STATE = 4
LW_ERR_OVERFLOW = 5

LW_TRAVERSE_COMPAT = 0
LW_TRAVERSE_CORRECTED = 1
LW_TRAVERSE_BRUTE = 2

LW_BSDF_DIFFUSE = 0
LW_BSDF_GLOSSY = 1
LW_BSDF_SPECULAR_REFLECT = 2
LW_BSDF_SPECULAR_TRANSMIT = 3
LW_MAX_LAYERS = 4

LW_ENV_NONE = 0
LW_ENV_CONSTANT = 1
LW_ENV_IMAGE = 2

LW_EST_MIS = 0
LW_EST_NEE = 1
LW_EST_BSDF = 2

LW_ENGINE_WAVEFRONT = 0
LW_ENGINE_MEGAKERNEL = 1

LW_COMM_ID_BYTES = 128

LW_FB_FRAC_BITS = 20
LW_FB_SAMPLE_CLAMP = 4294967296.0

_pd = C.POINTER(C.c_double)
_pi64 = C.POINTER(C.c_int64)
_pi32 = C.POINTER(C.c_int32)
_pf = C.POINTER(C.c_float)


class LwLayer(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("coat", C.c_int32),
        ("tint", C.c_double * 3),
        ("weight", C.c_double),
        ("roughness", C.c_double),
    ]


class LwMaterial(C.Structure):
    _fields_ = [
        ("nlayers", C.c_int32),
        ("thin_walled", C.c_int32),
        ("layers", LwLayer * LW_MAX_LAYERS),
        ("ior", C.c_double),
    ]


class LwSceneDesc(C.Structure):
    _fields_ = [
        ("ntris", C.c_int64),
        ("verts", _pd),
        ("normals", _pd),
        ("material", _pi32),
        ("nmaterials", C.c_int32),
        ("env_kind", C.c_int32),
        ("materials", C.POINTER(LwMaterial)),
        ("nemit", C.c_int64),
        ("emit_tri", _pi64),
        ("emit_radiance", _pd),
        ("emit_twosided", _pi32),
        ("emit_weight", _pd),
        ("env_constant", C.c_double * 3),
        ("env_scale", C.c_double),
        ("env_width", C.c_int32),
        ("env_height", C.c_int32),
        ("env_image", _pf),
        ("env_weight", _pd),
        ("p_env", C.c_double),
        ("cam_pos", C.c_double * 3),
        ("cam_fwd", C.c_double * 3),
        ("cam_right", C.c_double * 3),
        ("cam_up", C.c_double * 3),
        ("tan_half_fov", C.c_double),
        ("bvh_kind", C.c_int32),
        ("light_sampler", C.c_int32),
    ]


LW_LIGHTS_ALIAS = 0
LW_LIGHTS_TREE = 1
LW_LIGHTS_ENV_PYRAMID = 2
LW_BVH_SAH = 0
LW_BVH_MEDIAN = 1


class LwRenderParams(C.Structure):
    _fields_ = [
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("max_depth", C.c_int32),
        ("rr_start", C.c_int32),
        ("ndims", C.c_int64),
        ("bases", _pi64),
        ("perm_flat", _pi64),
        ("perm_len", C.c_int64),
        ("perm_offset", _pi64),
        ("engine", C.c_int32),
        ("pool_log2", C.c_int32),
        ("regen_fraction", C.c_double),
        ("megakernel_tail", C.c_int64),
        ("estimator", C.c_int32),
        ("compact_state", C.c_int32),
    ]


class LwRenderStats(C.Structure):
    _fields_ = [
        ("paths", C.c_int64),
        ("rays_extension", C.c_int64),
        ("rays_shadow", C.c_int64),
        ("waves", C.c_int64),
        ("regenerations", C.c_int64),
        ("nonfinite", C.c_int64),
    ]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class LwKernelProfile(C.Structure):
    _fields_ = [
        ("trace_ext_ms", C.c_double),
        ("trace_shadow_ms", C.c_double),
        ("total_ms", C.c_double),
        ("trace_ext_launches", C.c_int64),
        ("trace_shadow_launches", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("ext_rays", C.c_int64),
        ("ext_nodes", C.c_int64),
        ("ext_tris", C.c_int64),
        ("shadow_rays", C.c_int64),
        ("shadow_nodes", C.c_int64),
        ("shadow_tris", C.c_int64),
        ("stage_ms", C.c_double * 6),
        ("stage_launches", C.c_int64 * 6),
        ("pool_slots", C.c_int64),
        ("waves", C.c_int64),
        ("paths", C.c_int64),
        ("shadow_unoccluded", C.c_int64),
    ]

    def as_dict(self):
        out = {}
        for k, t in self._fields_:
            v = getattr(self, k)
            if k == "stage_ms":
                out[k] = {n: float(v[i]) for i, n in enumerate(PROF_STAGES)}
            elif k == "stage_launches":
                out[k] = {n: int(v[i]) for i, n in enumerate(PROF_STAGES)}
            else:
                out[k] = float(v) if t is C.c_double else int(v)
        return out


LW_INSTR_TIME = 1
LW_INSTR_COUNT = 2

PROF_STAGES = ("generate", "trace_ext", "shade_nee", "shade", "trace_shadow", "other")  # LW_PROF_*


def ptr(a: np.ndarray | None, ctype):
    """Pointer to a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return C.cast(None, C.POINTER(ctype))
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data_as(C.POINTER(ctype))


# Every exported symbol of include/lw_b200.h with its ctypes signature.
_V = C.c_void_p
SIGNATURES = {
    "lw_last_error": (C.c_char_p, []),
    "lw_abi_version": (C.c_int, []),
    "lw_device_count": (C.c_int, [_pi32]),
    "lw_set_device": (C.c_int, [C.c_int]),
    "lw_halton_batch": (C.c_int, [_pi64, C.c_int64, _pi64, C.c_int64, _pi64, C.c_int64, _pi64, C.c_int64, _pd]),
    "lw_halton_batch_device": (C.c_int, [_pi64, C.c_int64, _pi64, C.c_int64, _pi64, C.c_int64, _V, C.c_int64, _V]),
    "lw_pixel_offset_batch": (C.c_int, [_pd, C.c_int64, _pd]),
    "lw_oct_roundtrip_batch": (C.c_int, [_pd, C.c_int64, _pd]),
    "lw_oct_encode_batch": (C.c_int, [_pd, C.c_int64, _pi64]),
    "lw_oct_decode_batch": (C.c_int, [_pi64, C.c_int64, _pd]),
    "lw_intersect_batch": (
        C.c_int,
        [C.c_int, _pd, _pi64, C.c_int64, _pi64, _pd, C.c_int64, _pd, _pd, _pd, C.c_int64, _pd, _pi64, _pd],
    ),
    "lw_intersect_batch_device": (
        C.c_int,
        [C.c_int, _V, _V, C.c_int64, _V, _V, C.c_int64, _V, _V, _V, C.c_int64, _V, _V, _V],
    ),
    "lw_bvh_build": (C.c_int, [_pd, C.c_int64, _pd, _pi64, _pi64, _pi64]),
    "lw_alias_build": (C.c_int, [_pd, C.c_int64, _pd, _pi32, _pd]),
    "lw_ctx_create": (C.c_int, [C.c_int, C.POINTER(_V)]),
    "lw_ctx_destroy": (C.c_int, [_V]),
    "lw_ctx_set_stream": (C.c_int, [_V, _V]),
    "lw_ctx_set_instrumentation": (C.c_int, [_V, C.c_int]),
    "lw_ctx_kernel_profile": (C.c_int, [_V, C.POINTER(LwKernelProfile)]),
    "lw_scene_upload": (C.c_int, [_V, C.POINTER(LwSceneDesc)]),
    "lw_render_configure": (C.c_int, [_V, C.POINTER(LwRenderParams)]),
    "lw_framebuffer_clear": (C.c_int, [_V]),
    "lw_render_pass": (C.c_int, [_V, C.c_int64, C.c_int64]),
    "lw_render_pass_pixels": (C.c_int, [_V, C.c_int64, C.c_int64, C.c_int64, C.c_int64]),
    "lw_ctx_synchronize": (C.c_int, [_V]),
    "lw_framebuffer_download": (C.c_int, [_V, _pi64]),
    "lw_framebuffer_resolve": (C.c_int, [_V, C.c_double, _pf]),
    "lw_framebuffer_copy_device": (C.c_int, [_V, _V]),
    "lw_framebuffer_load_device": (C.c_int, [_V, _V]),
    "lw_get_stats": (C.c_int, [_V, C.POINTER(LwRenderStats)]),
    "lw_ctx_trace_closest": (C.c_int, [_V, _pd, _pd, _pd, C.c_int64, _pd, _pi64, _pd]),
    "lw_ctx_trace_any": (C.c_int, [_V, _pd, _pd, _pd, C.c_int64, _pi32]),
    "lw_ctx_camera_rays": (C.c_int, [_V, _pi64, C.c_int64, _pd, _pd]),
    "lw_ctx_light_tree_info": (C.c_int, [_V, _pi64]),
    "lw_ctx_light_tree_download": (C.c_int, [_V, _pd, _pi32, C.POINTER(C.c_uint64), _pi32]),
    "lw_ctx_light_sample": (C.c_int, [_V, _pd, _pd, _pd, C.c_int64, _pi64, _pd, _pd]),
    "lw_ctx_light_pdf": (C.c_int, [_V, _pi64, _pd, _pd, C.c_int64, _pd]),
    "lw_framebuffer_upload": (C.c_int, [_V, _pi64]),
    "lw_ctx_set_lpe": (C.c_int, [_V, C.c_int32, C.c_int32, C.POINTER(C.c_int16), C.POINTER(C.c_uint8), C.c_int32]),
    "lw_ctx_lpe_download": (C.c_int, [_V, C.c_int32, _pi64]),
    "lw_ctx_lpe_upload": (C.c_int, [_V, C.c_int32, _pi64]),
    "lw_framebuffer_accumulate": (C.c_int, [_V, _V, C.c_int]),
    "lw_bsdf_eval_batch": (C.c_int, [C.POINTER(LwMaterial), _pd, _pd, C.c_int64, _pd, _pd]),
    "lw_bsdf_sample_batch": (C.c_int, [C.POINTER(LwMaterial), _pd, _pi32, _pd, C.c_int64, _pd, _pd, _pd, _pi32]),
    "lw_mis_weight_batch": (C.c_int, [_pd, _pd, C.c_int64, _pd]),
    "lw_ctx_nee_light_sample": (C.c_int, [_V, _pd, _pd, _pd, C.c_int64, _pd, _pd, _pd, _pd, _pi64]),
    "lw_ctx_emission_pdf": (C.c_int, [_V, _pd, _pd, _pi32, C.c_int64, _pd, _pd, _pi64]),
    "lw_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "lw_ctx_comm_init": (C.c_int, [_V, C.POINTER(C.c_uint8), C.c_int, C.c_int]),
    "lw_framebuffer_reduce": (C.c_int, [_V]),
    "lw_ctx_env_pyramid_info": (C.c_int, [_V, _pi32]),
    "lw_ctx_env_sample": (C.c_int, [_V, _pi64, _pd, C.c_int64, _pi64, _pd, _pd]),
    "lw_ctx_env_pdf": (C.c_int, [_V, _pi64, _pi64, C.c_int64, _pd]),
    "lw_ctx_bvh_info": (C.c_int, [_V, _pi64]),
    "lw_ctx_bvh_download": (C.c_int, [_V, _pd, _pi64, _pi64]),
    "lw_ctx_last_pass_timing": (C.c_int, [_V, _pd, _pd, _pi64]),
}

_lib = None
_lock = threading.Lock()


class LwError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"liblw_b200 error {code}: {msg}")
        self.code = code


def lib():
    """Load liblw_b200.so (raises if it has not been built: no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not found: build the CUDA library with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        handle = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.lw_abi_version() != 1:
            raise ImportError("liblw_b200.so ABI version mismatch")
        _lib = handle
        return _lib


def check(code: int):
    """Raise the reference wrapper's exception type for a non-zero status."""
    if code == LW_OK:
        return
    msg = lib().lw_last_error().decode("utf-8", "replace")
    if code == LW_ERR_INVALID:
        raise ValueError(msg)
    if code == LW_ERR_OVERFLOW:
        raise OverflowError(msg)
    raise LwError(code, msg)
