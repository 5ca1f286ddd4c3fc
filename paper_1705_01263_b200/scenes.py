"""Procedural scenes for the five benchmark configurations (BASELINE.json `configs`).

C1  Cornell box 64x64, 16 spp, depth 4
C2  Cornell box 1024x1024, 1024 spp, depth 8 (the headline bench workload)
C3  ~2^20-triangle random soup, diffuse/glossy materials, constant env + one area light, 1920x1080, 256 spp, depth 8
C4  4096x2048 procedural HDR environment, glossy/layered spheres on a ground quad, 1920x1080
C5  10,000 emissive triangles with position-varying radiance, 1920x1080, 512 spp, depth 12

All scenes are constructed directly as `Scene` objects (no text parsing) and are
deterministic functions of their arguments (seeded numpy generators).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_1705_01263_b200 import meshgen
from paper_1705_01263_b200.scene import (Emitter, Environment, Instance, Mesh, Scene, diffuse_material,
                                         layered_material, make_camera)


def _mesh(name, pos, nrm, uvw, tris):
    return Mesh(name, np.asarray(pos, np.float64), np.asarray(nrm, np.float64), np.asarray(uvw, np.float64),
                np.asarray(tris, np.int64))


def _sub(mesh_tuple, keep):
    pos, nrm, uvw, tris = mesh_tuple
    return pos, nrm, uvw, tris[keep]


WHITE = (0.75, 0.75, 0.75)
RED = (0.63, 0.065, 0.05)
GREEN = (0.14, 0.45, 0.091)


def cornell(light_radiance=10.0) -> Scene:
    """Unit Cornell room open at +z: 36 triangles.

    Triangle ids: 0-1 red left wall (x=0), 2-3 green right wall (x=1), 4-9 white
    floor/ceiling/back, 10-21 short box, 22-33 tall box, 34-35 ceiling light.
    """
    room = meshgen.box((0, 0, 0), (1, 1, 1), inward=True)  # faces -x,+x,-y,+y,-z,+z
    meshes = [
        _mesh("left", *_sub(room, [0, 1])),
        _mesh("right", *_sub(room, [2, 3])),
        _mesh("room", *_sub(room, [4, 5, 6, 7, 8, 9])),  # front face (10, 11) removed
        _mesh("short", *meshgen.box((0.15, 0.0, 0.15), (0.45, 0.3, 0.45))),
        _mesh("tall", *meshgen.box((0.55, 0.0, 0.5), (0.85, 0.6, 0.8))),
        _mesh("light", *meshgen.quad((0.35, 0.999, 0.35), (0.3, 0.0, 0.0), (0.0, 0.0, 0.3))),
    ]
    materials = [diffuse_material("red", RED), diffuse_material("green", GREEN), diffuse_material("white", WHITE),
                 diffuse_material("lamp", (0.0, 0.0, 0.0))]
    mat_of = [0, 1, 2, 2, 2, 3]
    instances = [Instance(m.name, k, mat_of[k]) for k, m in enumerate(meshes)]
    emitters = [Emitter(instance=5, triangles=None, radiance=(light_radiance,) * 3)]
    cam = make_camera((0.5, 0.5, 2.5), (0.5, 0.5, 0.0), fov_y=45.0)
    return Scene(camera=cam, meshes=meshes, instances=instances, materials=materials, emitters=emitters,
                 environment=Environment(),
                 material_index={m.name: k for k, m in enumerate(materials)},
                 instance_index={inst.name: k for k, inst in enumerate(instances)})


def soup(n_tris: int = 1 << 20, n_materials: int = 64, seed: int = 7) -> Scene:
    """Random triangle soup in [0,20)^3 (test_accel.py:121-127 distribution), random diffuse/GGX materials."""
    rng = np.random.default_rng(seed)
    per = -(-n_tris // n_materials)
    meshes, instances, materials = [], [], []
    made = 0
    for k in range(n_materials):
        cnt = min(per, n_tris - made)
        if cnt <= 0:
            break
        base = rng.random((cnt, 3)) * 20.0
        e1 = rng.normal(size=(cnt, 3)) * 0.3
        e2 = rng.normal(size=(cnt, 3)) * 0.3
        pos = np.concatenate([base, base + e1, base + e2])
        tris = np.stack([np.arange(cnt), np.arange(cnt) + cnt, np.arange(cnt) + 2 * cnt], axis=1)
        fn = np.cross(e1, e2)
        ln = np.linalg.norm(fn, axis=1, keepdims=True)
        ln[ln == 0] = 1.0
        fn = fn / ln
        nrm = np.concatenate([fn, fn, fn])
        meshes.append(_mesh(f"soup{k}", pos, nrm, np.zeros_like(pos), tris))
        albedo = tuple(0.2 + 0.7 * rng.random(3))
        if rng.random() < 0.5:
            materials.append(layered_material(f"m{k}", [{"bsdf": "diffuse", "tint": albedo}]))
        else:
            alpha = float(0.05 + 0.45 * rng.random())
            materials.append(layered_material(f"m{k}", [{"bsdf": "glossy", "tint": albedo, "roughness": alpha}]))
        instances.append(Instance(f"soup{k}", k, k))
        made += cnt
    lamp = meshgen.quad((5.0, 24.0, 5.0), (10.0, 0.0, 0.0), (0.0, 0.0, 10.0))  # faces -y (down)
    meshes.append(_mesh("lamp", *lamp))
    materials.append(diffuse_material("lamp", (0.0, 0.0, 0.0)))
    instances.append(Instance("lamp", len(meshes) - 1, len(materials) - 1))
    emitters = [Emitter(instance=len(instances) - 1, triangles=None, radiance=(8.0, 8.0, 8.0))]
    cam = make_camera((10.0, 10.0, -30.0), (10.0, 10.0, 10.0), fov_y=45.0)
    return Scene(camera=cam, meshes=meshes, instances=instances, materials=materials, emitters=emitters,
                 environment=Environment(constant=(0.3, 0.35, 0.45)))


def procedural_sky(width: int = 4096, height: int = 2048, seed: int = 3) -> np.ndarray:
    """Lat-long HDR: vertical sky gradient, dim ground, and a sun disc ~1e4x the sky peak."""
    rng = np.random.default_rng(seed)
    v = (np.arange(height) + 0.5) / height  # 0 = +y pole
    u = (np.arange(width) + 0.5) / width
    theta = v * np.pi
    phi = u * 2 * np.pi
    up = np.cos(theta)[:, None] * np.ones((1, width))
    sky = np.where(up > 0, 0.4 + 0.8 * up, 0.08)
    img = np.stack([sky * 0.55, sky * 0.7, sky * 1.0], axis=2)
    img *= (1.0 + 0.05 * rng.random((height, width, 1)))
    sun_theta, sun_phi = 0.9, 1.3 + rng.random()
    st, ct = np.sin(theta)[:, None], np.cos(theta)[:, None]
    d = np.stack([st * np.cos(phi)[None, :], ct * np.ones((1, width)), st * np.sin(phi)[None, :]], axis=2)
    sd = np.array([np.sin(sun_theta) * np.cos(sun_phi), np.cos(sun_theta), np.sin(sun_theta) * np.sin(sun_phi)])
    cosang = d @ sd
    sun = cosang > np.cos(np.radians(0.6))
    img[sun] = np.array([1.2e4, 1.1e4, 0.95e4])
    return img


def envmap_scene(env_width: int = 4096, env_height: int = 2048, sphere_subdiv: int = 4) -> Scene:
    """C4: glossy / layered (GGX coat over diffuse) spheres on a diffuse ground, lit by the HDR env only."""
    meshes = [
        _mesh("ground", *meshgen.quad((-6.0, 0.0, 6.0), (12.0, 0.0, 0.0), (0.0, 0.0, -12.0))),
        _mesh("s0", *meshgen.icosphere((-1.6, 1.0, 0.0), 1.0, sphere_subdiv)),
        _mesh("s1", *meshgen.icosphere((0.6, 0.8, -0.6), 0.8, sphere_subdiv)),
        _mesh("s2", *meshgen.icosphere((2.2, 0.6, 0.6), 0.6, sphere_subdiv)),
    ]
    materials = [
        layered_material("ground", [{"bsdf": "diffuse", "tint": (0.5, 0.5, 0.5)}]),
        layered_material("coated", [{"bsdf": "glossy", "tint": 1.0, "roughness": 0.05, "coat": True},
                                    {"bsdf": "diffuse", "tint": (0.7, 0.1, 0.08)}], ior=1.5),
        layered_material("metal", [{"bsdf": "glossy", "tint": (0.95, 0.7, 0.3), "roughness": 0.25}]),
        layered_material("mix", [{"bsdf": "glossy", "tint": (0.9, 0.9, 0.9), "roughness": 0.1, "weight": 0.3},
                                 {"bsdf": "diffuse", "tint": (0.1, 0.3, 0.7)}]),
    ]
    instances = [Instance(m.name, k, k) for k, m in enumerate(meshes)]
    env = Environment(image=procedural_sky(env_width, env_height), scale=1.0)
    cam = make_camera((0.0, 2.0, 7.0), (0.0, 0.8, 0.0), fov_y=40.0)
    return Scene(camera=cam, meshes=meshes, instances=instances, materials=materials, emitters=[], environment=env)


def many_lights(n_lights: int = 10000, seed: int = 11) -> Scene:
    """C5: 10k small emissive triangles on the ceiling of a room, radiance varying with position."""
    rng = np.random.default_rng(seed)
    room = meshgen.box((0, 0, 0), (10, 4, 10), inward=True)
    meshes = [_mesh("room", *room), _mesh("block", *meshgen.box((3, 0, 3), (5, 2, 6))),
              _mesh("block2", *meshgen.box((6.5, 0, 5), (8, 3.2, 7.5)))]
    centers = np.stack([rng.random(n_lights) * 9.6 + 0.2, np.full(n_lights, 3.99), rng.random(n_lights) * 9.6 + 0.2], 1)
    s = 0.06
    p0 = centers + np.array([-s, 0, -s])
    p1 = centers + np.array([s, 0, -s])
    p2 = centers + np.array([0, 0, s])
    pos = np.concatenate([p0, p1, p2])
    tris = np.stack([np.arange(n_lights), np.arange(n_lights) + n_lights, np.arange(n_lights) + 2 * n_lights], 1)
    # winding so that the geometric normal faces down (-y)
    nrm = np.tile([0.0, -1.0, 0.0], (3 * n_lights, 1))
    e1 = p1 - p0
    e2 = p2 - p0
    if np.cross(e1[0], e2[0])[1] > 0:
        tris = tris[:, [0, 2, 1]]
    meshes.append(_mesh("lights", pos, nrm, np.zeros_like(pos), tris))
    materials = [diffuse_material("white", (0.7, 0.7, 0.7)), diffuse_material("lamp", (0.0, 0.0, 0.0))]
    instances = [Instance("room", 0, 0), Instance("block", 1, 0), Instance("block2", 2, 0), Instance("lights", 3, 1)]
    x, z = centers[:, 0] / 10.0, centers[:, 2] / 10.0
    radiance = np.stack([20 + 60 * x, 20 + 60 * (1 - x) * z, 30 + 50 * (1 - z)], axis=1)
    emitters = [Emitter(instance=3, triangles=np.arange(n_lights), radiance=radiance)]
    cam = make_camera((5.0, 2.0, 9.8), (5.0, 1.6, 0.0), fov_y=60.0)
    return Scene(camera=cam, meshes=meshes, instances=instances, materials=materials, emitters=emitters,
                 environment=Environment())


@dataclass(frozen=True)
class Config:
    name: str
    builder: object
    width: int
    height: int
    spp: int
    max_depth: int
    description: str


CONFIGS = {
    "C1": Config("C1", cornell, 64, 64, 16, 4, "Cornell box 64x64, 16 spp, depth 4"),
    "C2": Config("C2", cornell, 1024, 1024, 1024, 8, "Cornell box 1024x1024, 1024 spp, depth 8"),
    "C3": Config("C3", soup, 1920, 1080, 256, 8, "2^20-triangle soup 1920x1080, 256 spp, depth 8"),
    "C4": Config("C4", envmap_scene, 1920, 1080, 256, 8, "4Kx2K HDR env + glossy/layered spheres 1920x1080"),
    "C5": Config("C5", many_lights, 1920, 1080, 512, 12, "10k emissive triangles 1920x1080, 512 spp, depth 12"),
}
