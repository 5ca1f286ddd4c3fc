"""Light hierarchy.

CPU: the oracle restatement against the SPEC examples -- one triangle -> selection probability 1;
two identical triangles placed symmetrically about the shading point -> 0.5 each; sample_light and
light_pdf agree exactly; selection probabilities over all emitters sum to 1; no emitter gets 0.
GPU: tree arrays, sampled emitters, probabilities and rescaled uniforms bit-exact vs the oracle;
images rendered with the light tree bit-exact vs the oracle (wavefront and megakernel).
"""

import numpy as np
import pytest

from paper_1705_01263_b200 import scenes
from paper_1705_01263_b200.scene import Emitter, Instance, Scene, make_camera, pack_scene


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def _tri_scene(tris, radiance=5.0):
    """Scene of emissive triangles (each a one-triangle mesh, geometric normal facing -y) over a floor."""
    from paper_1705_01263_b200.scenes import _mesh, diffuse_material

    meshes, inst, ems = [], [], []
    for k, t in enumerate(tris):
        pos = np.asarray(t, np.float64).reshape(3, 3)
        meshes.append(_mesh(f"l{k}", pos, np.tile([0.0, -1.0, 0.0], (3, 1)), np.zeros((3, 3)), [[0, 1, 2]]))
        inst.append(Instance(f"l{k}", k, 1))
        ems.append(Emitter(instance=k, triangles=np.arange(1), radiance=(radiance, radiance, radiance)))
    floor = np.array([[-5, 0, -5], [5, 0, -5], [5, 0, 5], [-5, 0, 5]], np.float64)
    meshes.append(_mesh("floor", floor, np.tile([0.0, 1.0, 0.0], (4, 1)), np.zeros((4, 3)), [[0, 2, 1], [0, 3, 2]]))
    inst.append(Instance("floor", len(tris), 0))
    mats = [diffuse_material("floor", (0.5, 0.5, 0.5)), diffuse_material("lamp", (0.0, 0.0, 0.0))]
    return Scene(camera=make_camera((0, 2, 6), (0, 0, 0)), meshes=meshes, instances=inst, materials=mats,
                 emitters=ems, environment=scenes.Environment())


def test_one_triangle_probability_one(oracle):
    sc = _tri_scene([[(0, 2, 0), (1, 2, 0), (0, 2, 1)]])
    os_ = oracle.OracleScene(pack_scene(sc, lights="tree"))
    x = np.array([[0.2, 0.0, 0.2], [3.0, 1.0, -2.0]])
    nrm = np.array([[0.0, 1.0, 0.0], [0.0, 1.0, 0.0]])
    e, p, _ = os_.light_sample(x, nrm, np.array([0.3, 0.9]))
    assert list(e) == [0, 0] and list(p) == [1.0, 1.0]


def test_symmetric_pair_half_each(oracle):
    # mirror images through the plane x = 0, facing down, shading point on the plane
    a = [(-2, 3, 0), (-1, 3, 0), (-2, 3, 1)]
    b = [(2, 3, 0), (2, 3, 1), (1, 3, 0)]
    os_ = oracle.OracleScene(pack_scene(_tri_scene([a, b]), lights="tree"))
    x = np.array([[0.0, 0.0, 0.4]])
    nrm = np.array([[0.0, 1.0, 0.0]])
    p = os_.light_pdf(np.array([0, 1]), np.repeat(x, 2, 0), np.repeat(nrm, 2, 0))
    assert p[0] == p[1] == 0.5


def test_many_lights_probabilities(oracle):
    packed = pack_scene(scenes.many_lights(2000), lights="tree")
    os_ = oracle.OracleScene(packed)
    nodes, right, path, depth = os_.light_tree()
    ne = packed.nemit
    assert nodes.shape[0] == 2 * int((depth >= 0).sum()) - 1
    assert np.allclose(nodes[0, 6], nodes[1:][right[1:] < 0, 6].sum(), rtol=1e-6)  # FP32 node records
    rng = np.random.default_rng(3)
    v = packed.verts.reshape(-1, 3)
    lo, hi = v.min(0), v.max(0)
    for _ in range(4):
        x = lo + (hi - lo) * rng.random(3)
        nrm = rng.normal(size=3)
        nrm /= np.linalg.norm(nrm)
        pe = os_.light_pdf(np.arange(ne), np.tile(x, (ne, 1)), np.tile(nrm, (ne, 1)))
        assert abs(pe.sum() - 1.0) < 1e-12 and pe.min() > 0.0
        u = rng.random(4000)
        e, ps, uo = os_.light_sample(np.tile(x, (4000, 1)), np.tile(nrm, (4000, 1)), u)
        assert np.array_equal(_bits(ps), _bits(pe[e]))  # sample_light pdf == light_pdf, exactly
        assert uo.min() >= 0.0 and uo.max() < 1.0


def test_light_tree_lowers_error_cpu(oracle):
    """Equal-sample comparison on a C5 crop: the hierarchy's image is closer to a converged one."""
    from paper_1705_01263_b200.render import RenderParams

    c = scenes.CONFIGS["C5"]
    sc = scenes.many_lights(3000)
    prm = RenderParams(48, 27, c.max_depth)
    img = {}
    for lights in ("alias", "tree"):
        fb, _ = oracle.OracleScene(pack_scene(sc, lights=lights)).render(prm, 0, 8)
        img[lights] = fb / (8 * 1048576.0)
    fb, _ = oracle.OracleScene(pack_scene(sc, lights="tree")).render(prm, 1000, 1256)
    ref = fb / (256 * 1048576.0)
    err = {k: np.sqrt(((v - ref) ** 2).mean()) for k, v in img.items()}
    assert err["tree"] < err["alias"], err


@pytest.mark.gpu
def test_light_tree_arrays_bit_exact(gpu, oracle):
    from paper_1705_01263_b200.render import Renderer

    packed = pack_scene(scenes.many_lights(5000), lights="tree")
    with Renderer(None, 16, 16, 4, packed=packed) as r:
        t = r.light_tree()
    t2 = oracle.OracleScene(packed).light_tree()
    assert np.array_equal(_bits(t[0]), _bits(t2[0]))
    for a, b in zip(t[1:], t2[1:]):
        assert np.array_equal(a, b)


@pytest.mark.gpu
def test_light_sample_and_pdf_bit_exact(gpu, oracle):
    from paper_1705_01263_b200.render import Renderer

    packed = pack_scene(scenes.many_lights(5000), lights="tree")
    rng = np.random.default_rng(5)
    n = 50000
    v = packed.verts.reshape(-1, 3)
    lo, hi = v.min(0), v.max(0)
    x = lo - 1.0 + (hi - lo + 2.0) * rng.random((n, 3))
    nrm = rng.normal(size=(n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    u = rng.random(n)
    u[:4] = [0.0, 0.5, 0.9999999999999999, 1e-300]
    os_ = oracle.OracleScene(packed)
    with Renderer(None, 16, 16, 4, packed=packed) as r:
        e, p, uo = r.light_sample(x, nrm, u)
        ee = rng.integers(0, packed.nemit, n)
        q = r.light_pdf(ee, x, nrm)
    e2, p2, uo2 = os_.light_sample(x, nrm, u)
    q2 = os_.light_pdf(ee, x, nrm)
    assert np.array_equal(e, e2) and np.array_equal(_bits(p), _bits(p2)) and np.array_equal(_bits(uo), _bits(uo2))
    assert np.array_equal(_bits(q), _bits(q2))


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["wavefront", "megakernel"])
def test_render_with_light_tree_bit_exact(gpu, oracle, engine):
    from paper_1705_01263_b200.render import Renderer, RenderParams

    c = scenes.CONFIGS["C5"]
    packed = pack_scene(scenes.many_lights(2000), lights="tree")
    W, H = 96, 54
    with Renderer(None, W, H, c.max_depth, packed=packed, engine=engine) as r:
        r.render_pass(0, 3)
        fb = r.framebuffer()
    fb2, _ = oracle.OracleScene(packed).render(RenderParams(W, H, c.max_depth), 0, 3)
    assert np.array_equal(fb, fb2) and fb.sum() > 0


# ---- environment pyramid --------------

def _env_scene(w=256, h=128):
    return scenes.envmap_scene(w, h, sphere_subdiv=3)


def test_env_pyramid_probabilities(oracle):
    packed = pack_scene(_env_scene(), env_sampling="pyramid")
    os_ = oracle.OracleScene(packed)
    assert os_.env_pyramid_levels() == 8
    nt = 256 * 128
    w = packed.arrays["env_w"].reshape(-1)
    rng = np.random.default_rng(2)
    for pk in [0, 0xFFFFFFFF, 0x7FFF7FFF, int(rng.integers(0, 2 ** 32))]:
        pe = os_.env_pdf(np.full(nt, pk), np.arange(nt))
        assert abs(pe.sum() - 1.0) < 1e-12
        assert np.array_equal(pe > 0, w > 0)  # coverage: never zero where there is radiance
        uv = rng.random((4000, 2))
        t, ps, uvo = os_.env_sample(np.full(4000, pk), uv)
        assert np.array_equal(_bits(ps), _bits(os_.env_pdf(np.full(4000, pk), t)))
        assert uvo.min() >= 0.0 and uvo.max() < 1.0


def test_env_pyramid_single_texel(oracle):
    """a single nonzero texel is sampled with probability 1."""
    from paper_1705_01263_b200.scene import Environment

    sc = _env_scene(64, 32)
    img = np.zeros((32, 64, 3))
    img[9, 41] = (5.0, 4.0, 3.0)
    sc.environment = Environment(image=img, scale=1.0)
    os_ = oracle.OracleScene(pack_scene(sc, env_sampling="pyramid"))
    t, p, _ = os_.env_sample(np.zeros(100, np.int64), np.random.default_rng(0).random((100, 2)))
    assert np.all(t == 9 * 64 + 41) and np.all(p == 1.0)


@pytest.mark.gpu
def test_env_sample_and_pdf_bit_exact(gpu, oracle):
    from paper_1705_01263_b200.render import Renderer

    packed = pack_scene(_env_scene(512, 256), env_sampling="pyramid")
    rng = np.random.default_rng(8)
    n = 40000
    pk = rng.integers(0, 2 ** 32, n)
    uv = rng.random((n, 2))
    tx = rng.integers(0, 512 * 256, n)
    os_ = oracle.OracleScene(packed)
    with Renderer(None, 16, 16, 4, packed=packed) as r:
        assert r.env_pyramid_levels() == 9
        t, p, o = r.env_sample(pk, uv)
        q = r.env_pdf(pk, tx)
    t2, p2, o2 = os_.env_sample(pk, uv)
    assert np.array_equal(t, t2) and np.array_equal(_bits(p), _bits(p2)) and np.array_equal(_bits(o), _bits(o2))
    assert np.array_equal(_bits(q), _bits(os_.env_pdf(pk, tx)))


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["wavefront", "megakernel"])
def test_render_with_env_pyramid_bit_exact(gpu, oracle, engine):
    from paper_1705_01263_b200.render import Renderer, RenderParams

    packed = pack_scene(_env_scene(512, 256), env_sampling="pyramid", lights="tree")
    W, H = 96, 54
    with Renderer(None, W, H, 8, packed=packed, engine=engine) as r:
        r.render_pass(0, 3)
        fb = r.framebuffer()
    fb2, _ = oracle.OracleScene(packed).render(RenderParams(W, H, 8), 0, 3)
    assert np.array_equal(fb, fb2) and fb.sum() > 0
