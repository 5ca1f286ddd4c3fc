"""Scene model and packing into the C-ABI scene description.

The dataclasses mirror the reference's scene model (sceneformat.py:219-358) so
that scenes built here and scenes parsed by the reference's `load_scene` are
interchangeable: `pack_scene` only reads the attributes the reference defines.
Parsing the text format is out of scope; procedural configs
construct `Scene` objects directly (`scenes.py`).

Extension (documented in DESIGN.md §4.5): `Emitter.radiance` may be an
(len(triangles), 3) array for per-triangle (spatially varying) emission.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from paper_1705_01263_b200 import _abi
from paper_1705_01263_b200._abi import LwMaterial, LwSceneDesc, ptr
from paper_1705_01263_b200.geometry import flatten_instances

BSDF_KINDS = ("diffuse", "glossy", "specular_reflect", "specular_transmit")  # sceneformat.py:223
NODE_KINDS = ("constant", "texture", "checker", "mix", "multiply")
MAX_LAYERS = 4


@dataclass
class TextureNode:
    kind: str
    value: tuple = (0.0, 0.0, 0.0)
    operands: tuple = ()
    params: tuple = ()
    image: np.ndarray | None = None


@dataclass
class Layer:
    bsdf: str
    tint: int
    weight: int
    roughness: int = -1
    coat: bool = False
    bump: int = -1
    bump_strength: float = 1.0


@dataclass
class Material:
    name: str
    layers: list
    nodes: list
    cutout: int = -1
    emission: int = -1
    emission_scale: float = 1.0
    ior: float = 1.5
    abbe: float = 0.0
    thin_walled: bool = False
    sigma_a: tuple = (0.0, 0.0, 0.0)
    sigma_s: tuple = (0.0, 0.0, 0.0)
    has_medium: bool = False


@dataclass
class Mesh:
    name: str
    positions: np.ndarray
    normals: np.ndarray
    uvw: np.ndarray
    triangles: np.ndarray


@dataclass
class Instance:
    name: str
    mesh: int
    material: int
    transform: np.ndarray = field(default_factory=lambda: np.eye(4)[:3, :].copy())
    transform_t1: np.ndarray | None = None
    matte: bool = False
    matte_shadow_intensity: float = 1.0
    visible: bool = True


@dataclass
class Emitter:
    instance: int
    triangles: np.ndarray | None
    radiance_node: int = -1
    radiance: tuple | np.ndarray = (1.0, 1.0, 1.0)
    scale: float = 1.0
    flux: float | None = None
    twosided: bool = False


@dataclass
class DomeConfig:
    kind: str = "infinite"
    radius: float = 100.0
    center: tuple = (0.0, 0.0, 0.0)
    height: float = 0.0


@dataclass
class Environment:
    image: np.ndarray | None = None
    constant: tuple | None = None
    scale: float = 1.0
    dome: DomeConfig = field(default_factory=DomeConfig)


@dataclass
class Camera:
    position: np.ndarray
    forward: np.ndarray
    up: np.ndarray
    right: np.ndarray
    fov_y: float
    shutter: tuple = (0.0, 0.0)


@dataclass
class Scene:
    camera: Camera
    meshes: list
    instances: list
    materials: list
    emitters: list
    environment: Environment
    decals: list = field(default_factory=list)
    backplate: np.ndarray | None = None
    material_index: dict = field(default_factory=dict)
    instance_index: dict = field(default_factory=dict)

    @property
    def has_motion(self) -> bool:
        return any(inst.transform_t1 is not None for inst in self.instances)


def make_camera(position, look_at=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0), fov_y=45.0, shutter=(0.0, 0.0)) -> Camera:
    """Camera basis exactly as sceneformat.py:776-801 (block_camera)."""
    position = np.asarray(position, dtype=np.float64)
    forward = np.asarray(look_at, dtype=np.float64) - position
    norm = np.linalg.norm(forward)
    if norm == 0:
        raise ValueError("camera position equals look_at")
    forward = forward / norm
    right = np.cross(forward, np.asarray(up, dtype=np.float64))
    rn = np.linalg.norm(right)
    if rn == 0:
        raise ValueError("camera up is parallel to the view direction")
    right = right / rn
    upv = np.cross(right, forward)
    if not 0 < fov_y < 180:
        raise ValueError("fov_y must be in (0, 180)")
    return Camera(position=position, forward=forward, up=upv, right=right, fov_y=float(fov_y),
                  shutter=(float(shutter[0]), float(shutter[1])))


def diffuse_material(name, rgb, emission=None) -> Material:
    nodes = [TextureNode("constant", value=tuple(float(x) for x in rgb)), TextureNode("constant", value=(1.0, 1.0, 1.0))]
    m = Material(name=name, layers=[Layer("diffuse", tint=0, weight=1)], nodes=nodes)
    if emission is not None:
        nodes.append(TextureNode("constant", value=tuple(float(x) for x in emission)))
        m.emission = len(nodes) - 1
    return m


def layered_material(name, layers, ior=1.5) -> Material:
    """layers: list of dicts {bsdf, tint, weight=1, roughness=0.2, coat=False}."""
    nodes, out = [], []

    def const(v):
        v = (float(v),) * 3 if np.isscalar(v) else tuple(float(x) for x in v)
        nodes.append(TextureNode("constant", value=v))
        return len(nodes) - 1

    for spec in layers:
        rough = const(spec.get("roughness", 0.2)) if spec["bsdf"] == "glossy" else -1
        out.append(Layer(spec["bsdf"], tint=const(spec.get("tint", 1.0)), weight=const(spec.get("weight", 1.0)),
                         roughness=rough, coat=bool(spec.get("coat", False))))
    return Material(name=name, layers=out, nodes=nodes, ior=float(ior))


# ---- packing ------------------------------------------------------------------------------

_LUM = np.array([0.2126, 0.7152, 0.0722])


def _node_value(mat, idx, what):
    """Constant-fold a texturing node to an RGB triple (constant/mix/multiply of constants)."""
    node = mat.nodes[idx]
    if node.kind == "constant":
        return np.asarray(node.value, dtype=np.float64)
    if node.kind == "mix":
        t = node.params[0] if node.params else 0.5
        a = _node_value(mat, node.operands[0], what)
        b = _node_value(mat, node.operands[1], what)
        return (1.0 - t) * a + t * b
    if node.kind == "multiply":
        return _node_value(mat, node.operands[0], what) * _node_value(mat, node.operands[1], what)
    raise NotImplementedError(f"material '{mat.name}': {what} node kind '{node.kind}' (textures are out of scope)")


def _pack_material(mat) -> LwMaterial:
    if len(mat.layers) > MAX_LAYERS:
        raise ValueError(f"material '{mat.name}': at most {MAX_LAYERS} layers supported")
    out = LwMaterial()
    out.nlayers = len(mat.layers)
    out.thin_walled = int(bool(mat.thin_walled))
    out.ior = float(mat.ior)
    for k, layer in enumerate(mat.layers):
        if layer.bsdf not in BSDF_KINDS:
            raise ValueError(f"material '{mat.name}': unknown bsdf '{layer.bsdf}'")
        L = out.layers[k]
        L.kind = BSDF_KINDS.index(layer.bsdf)
        L.coat = int(bool(layer.coat))
        tint = _node_value(mat, layer.tint, "tint")
        for c in range(3):
            L.tint[c] = float(tint[c])
        L.weight = float(np.mean(_node_value(mat, layer.weight, "weight")))
        L.roughness = float(_node_value(mat, layer.roughness, "roughness")[0]) if layer.roughness >= 0 else 0.2
    return out


@dataclass
class PackedScene:
    """Numpy buffers + the LwSceneDesc pointing into them (kept alive together)."""

    desc: LwSceneDesc
    arrays: dict
    geometry: object
    ntris: int
    nemit: int

    @property
    def verts(self):
        return self.arrays["verts"]

    _PIN_FIELDS = {"verts": ("verts", C.c_double), "normals": ("normals", C.c_double),
                   "material": ("material", C.c_int32), "emit_tri": ("emit_tri", C.c_int64),
                   "emit_rad": ("emit_radiance", C.c_double), "emit_two": ("emit_twosided", C.c_int32),
                   "emit_w": ("emit_weight", C.c_double), "env_img": ("env_image", C.c_float),
                   "env_w": ("env_weight", C.c_double)}

    def pinned(self) -> "PackedScene":
        """Copy whose geometry / emitter / environment arrays live in page-locked host memory, so
        lw_scene_upload is a DMA from pinned buffers (torch pinned tensors; torch is plumbing here)."""
        import torch

        arrays = dict(self.arrays)
        desc = type(self.desc).from_buffer_copy(self.desc)
        keep = []
        for key, (field, ctype) in self._PIN_FIELDS.items():
            a = arrays.get(key)
            if not isinstance(a, np.ndarray) or a.size == 0:
                continue
            if key in ("env_img", "env_w") and desc.env_kind != _abi.LW_ENV_IMAGE:
                continue
            t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
            arrays[key] = t.numpy()
            keep.append(t)
            setattr(desc, field, ptr(arrays[key], ctype))
        arrays["_pinned"] = keep
        return PackedScene(desc=desc, arrays=arrays, geometry=self.geometry, ntris=self.ntris, nemit=self.nemit)


def _tri_areas(v):
    p = v.reshape(-1, 3, 3)
    return 0.5 * np.linalg.norm(np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), axis=1)


def pack_scene(scene, time: float = 0.0, p_env: float = 0.5, bvh: str = "sah", lights: str = "alias",
               env_sampling: str = "alias") -> PackedScene:
    """Flatten `scene` (reference or local dataclasses) into the C-ABI scene description.

    bvh: render acceleration structure, "sah" (binned SAH, default) or "median" (the reference's tree).
    lights: NEE emitter selection, "alias" (flat alias table over luminance * area) or "tree" (the
    light hierarchy of PAPER.md:215-253, importance by flux, distance and orientation).
    env_sampling: environment-image sampling, "alias" (alias table over texels) or "pyramid" (PAPER.md:262-276
    image pyramid with normal-binned top levels; needs a 2H x H image, H a power of two).
    """
    if bvh not in ("sah", "median"):
        raise ValueError("bvh must be 'sah' or 'median'")
    if lights not in ("alias", "tree"):
        raise ValueError("lights must be 'alias' or 'tree'")
    if env_sampling not in ("alias", "pyramid"):
        raise ValueError("env_sampling must be 'alias' or 'pyramid'")
    geo = flatten_instances(scene, time)
    ntris = len(geo.verts)
    verts = np.ascontiguousarray(geo.verts, dtype=np.float64)
    normals = np.ascontiguousarray(geo.shading_normals, dtype=np.float64)
    material = np.ascontiguousarray(geo.material, dtype=np.int32)
    mats = (LwMaterial * max(len(scene.materials), 1))()
    for k, m in enumerate(scene.materials):
        mats[k] = _pack_material(m)
    if not scene.materials:
        mats[0].nlayers = 0
        mats[0].ior = 1.5
    # emitters: material emission + emitter blocks, merged per triangle
    rad = {}
    two = {}
    tri_base = {}
    base = 0
    for idx, inst in enumerate(scene.instances):
        tri_base[idx] = base
        nt = len(scene.meshes[inst.mesh].triangles)
        mat = scene.materials[inst.material]
        if getattr(mat, "emission", -1) >= 0:
            le = _node_value(mat, mat.emission, "emission") * float(getattr(mat, "emission_scale", 1.0))
            for t in range(base, base + nt):
                rad[t] = rad.get(t, 0.0) + le
                two.setdefault(t, False)
        base += nt
    areas = _tri_areas(verts) if ntris else np.zeros(0)
    for em in scene.emitters:
        inst = scene.instances[em.instance]
        nt = len(scene.meshes[inst.mesh].triangles)
        local = np.arange(nt) if em.triangles is None else np.asarray(em.triangles, dtype=np.int64)
        glob = tri_base[em.instance] + local
        r = np.asarray(em.radiance, dtype=np.float64)
        if r.ndim == 1:
            r = np.tile(r, (len(glob), 1))
        if em.flux is not None:  # radiance colour scaled so the emitter's flux is pi*L*A = flux
            total = float(np.sum(areas[glob] * (r @ _LUM)))
            r = r * (float(em.flux) / (math.pi * total)) if total > 0 else r * 0.0
        else:
            r = r * float(em.scale)
        for k, t in enumerate(glob.tolist()):
            rad[t] = rad.get(t, 0.0) + r[k]
            two[t] = two.get(t, False) or bool(em.twosided)
    emit_tri = np.array(sorted(rad), dtype=np.int64)
    emit_rad = np.ascontiguousarray(np.array([rad[t] for t in emit_tri.tolist()], dtype=np.float64).reshape(-1, 3))
    emit_two = np.array([int(two[t]) for t in emit_tri.tolist()], dtype=np.int32)
    emit_w = np.ascontiguousarray((emit_rad @ _LUM) * areas[emit_tri] if len(emit_tri) else np.zeros(0))
    keep = emit_w > 0
    emit_tri, emit_rad, emit_two, emit_w = (np.ascontiguousarray(emit_tri[keep]), np.ascontiguousarray(emit_rad[keep]),
                                            np.ascontiguousarray(emit_two[keep]), np.ascontiguousarray(emit_w[keep]))
    env = scene.environment
    env_kind = _abi.LW_ENV_NONE
    env_img = None
    env_w = None
    env_const = (0.0, 0.0, 0.0)
    scale = float(getattr(env, "scale", 1.0)) if env is not None else 1.0
    if env is not None and getattr(env, "image", None) is not None and np.asarray(env.image).size > 3:
        img = np.asarray(env.image, dtype=np.float64)
        h, w = img.shape[:2]
        env_img = np.ascontiguousarray(img.astype(np.float32))
        theta = (np.arange(h) + 0.5) / h * np.pi
        env_w = np.ascontiguousarray(((img @ _LUM) * np.sin(theta)[:, None]).reshape(-1))
        env_kind = _abi.LW_ENV_IMAGE
    elif env is not None and (getattr(env, "constant", None) is not None or getattr(env, "image", None) is not None):
        c = env.constant if env.constant is not None else tuple(np.asarray(env.image).reshape(-1)[:3])
        env_const = tuple(float(x) for x in c)
        if any(x > 0 for x in env_const):
            env_kind = _abi.LW_ENV_CONSTANT
    d = LwSceneDesc()
    arrays = dict(verts=verts, normals=normals, material=material, mats=mats, emit_tri=emit_tri, emit_rad=emit_rad,
                  emit_two=emit_two, emit_w=emit_w, env_img=env_img, env_w=env_w)
    d.ntris = ntris
    d.verts = ptr(verts, C.c_double)
    d.normals = ptr(normals, C.c_double)
    d.material = ptr(material, C.c_int32)
    d.nmaterials = max(len(scene.materials), 1)
    d.materials = C.cast(mats, C.POINTER(LwMaterial))
    d.nemit = len(emit_tri)
    d.emit_tri = ptr(emit_tri, C.c_int64)
    d.emit_radiance = ptr(emit_rad, C.c_double)
    d.emit_twosided = ptr(emit_two, C.c_int32)
    d.emit_weight = ptr(emit_w, C.c_double)
    d.env_kind = env_kind
    for k in range(3):
        d.env_constant[k] = env_const[k]
    d.env_scale = scale
    if env_kind == _abi.LW_ENV_IMAGE:
        d.env_height, d.env_width = env_img.shape[:2]
        d.env_image = ptr(env_img, C.c_float)
        d.env_weight = ptr(env_w, C.c_double)
    d.p_env = float(p_env)
    cam = scene.camera
    for k in range(3):
        d.cam_pos[k] = float(cam.position[k])
        d.cam_fwd[k] = float(cam.forward[k])
        d.cam_right[k] = float(cam.right[k])
        d.cam_up[k] = float(cam.up[k])
    d.tan_half_fov = math.tan(math.radians(float(cam.fov_y)) * 0.5)
    d.bvh_kind = _abi.LW_BVH_SAH if bvh == "sah" else _abi.LW_BVH_MEDIAN
    d.light_sampler = (_abi.LW_LIGHTS_TREE if lights == "tree" else 0) | \
        (_abi.LW_LIGHTS_ENV_PYRAMID if env_sampling == "pyramid" else 0)
    return PackedScene(desc=d, arrays=arrays, geometry=geo, ntris=ntris, nemit=len(emit_tri))
