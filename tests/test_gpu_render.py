"""Render path on the GPU vs the CPU oracle (SPEC-only path).

Bars:
  * camera rays, render-traversal hit ids / t / barycentrics, any-hit: bit-exact;
  * framebuffers (int64 fixed point): bit-exact vs the oracle on the same (pixel, iteration) set;
  * execution-strategy invariance: megakernel == wavefront == any pool size, bit for bit;
  * SPEC known answers: constant-env camera rays give L exactly, furnace within 1%.
"""

import numpy as np
import pytest

from paper_1705_01263_b200 import scenes
from paper_1705_01263_b200.scene import Environment, Instance, Scene, layered_material, make_camera, pack_scene

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


@pytest.fixture(scope="module")
def cornell_packed(gpu):
    return pack_scene(scenes.cornell())


def _renderer(packed, w, h, depth, **kw):
    from paper_1705_01263_b200.render import Renderer

    return Renderer(None, w, h, depth, packed=packed, **kw)


def test_scene_bvh_matches_oracle(cornell_packed, oracle):
    with _renderer(cornell_packed, 64, 64, 4) as r:
        b, c, o = r.bvh()
    b2, c2, o2 = oracle.build_bvh(cornell_packed.verts)
    assert np.array_equal(b, b2) and np.array_equal(c, c2) and np.array_equal(o, o2)


def test_camera_rays_bit_exact(cornell_packed, oracle):
    from paper_1705_01263_b200.render import RenderParams

    w, h = 97, 61
    rng = np.random.default_rng(1)
    idx = np.concatenate([np.arange(w * h), rng.integers(0, w * h * 4096, 20000)]).astype(np.int64)
    with _renderer(cornell_packed, w, h, 4) as r:
        o, d = r.camera_rays(idx)
    os_ = oracle.OracleScene(cornell_packed)
    o2, d2 = os_.camera_rays(RenderParams(w, h, 4), idx)
    assert np.array_equal(_bits(o), _bits(o2)) and np.array_equal(_bits(d), _bits(d2))


def _random_rays(n, lo, hi, seed):
    rng = np.random.default_rng(seed)
    o = lo + rng.random((n, 3)) * (hi - lo)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d[:200, 1] = 0.0
    d[200:300, :2] = 0.0
    d[200:300, 2] = 1.0
    return o, d


@pytest.mark.parametrize("which,bvh", [("cornell", "sah"), ("cornell", "median"), ("soup", "sah"), ("soup", "median")])
def test_render_traversal_bit_exact(gpu, oracle, which, bvh):
    if which == "cornell":
        packed = pack_scene(scenes.cornell(), bvh=bvh)
        o, d = _random_rays(50000, np.array([0.0, 0.0, -0.5]), np.array([1.0, 1.0, 3.0]), 3)
    else:
        packed = pack_scene(scenes.soup(1 << 16, n_materials=8), bvh=bvh)
        o, d = _random_rays(50000, np.zeros(3), np.full(3, 20.0), 4)
    tm = np.where(np.arange(len(o)) % 5 == 0, 3.0, np.inf)
    with _renderer(packed, 64, 64, 4) as r:
        t, tri, b = r.trace_closest(o, d, tm)
        occ = r.trace_any(o, d, np.where(np.isinf(tm), 2.0, tm))
    os_ = oracle.OracleScene(packed)
    t2, tri2, b2 = os_.trace_closest(o, d, tm)
    occ2 = os_.trace_any(o, d, np.where(np.isinf(tm), 2.0, tm))
    assert np.array_equal(tri, tri2)
    assert np.array_equal(_bits(t), _bits(t2)) and np.array_equal(_bits(b), _bits(b2))
    assert np.array_equal(occ, occ2)
    # near-first + conservative cull == exhaustive search (brute force) on these rays
    if which == "cornell":
        v = packed.verts
        t3, tri3, _ = oracle.intersect_batch(2, np.zeros((1, 6)), np.zeros((1, 2), np.int64), np.zeros(0, np.int64), v, o, d, tm)
        assert np.array_equal(tri, tri3)


@pytest.mark.parametrize("engine,bvh", [("megakernel", "sah"), ("wavefront", "sah"), ("wavefront", "median")])
def test_c1_framebuffer_bit_exact_vs_oracle(oracle, engine, bvh):
    """C1 (Cornell 64x64, 16 spp, depth 4): the whole accumulated framebuffer, bit for bit."""
    from paper_1705_01263_b200.render import RenderParams

    cornell_packed = pack_scene(scenes.cornell(), bvh=bvh)
    with _renderer(cornell_packed, 64, 64, 4, engine=engine, pool_log2=12) as r:
        r.render_pass(0, 16)
        fb = r.framebuffer()
        st = r.stats()
    fb2, st2 = oracle.OracleScene(cornell_packed).render(RenderParams(64, 64, 4), 0, 16)
    assert np.array_equal(fb, fb2)
    assert st["paths"] == 64 * 64 * 16
    assert st["rays_extension"] == st2["rays_extension"] and st["rays_shadow"] == st2["rays_shadow"]


def test_c2_subset_bit_exact(cornell_packed, oracle):
    """C2 (1024^2, depth 8): a pixel band x 4 iterations bit-exact vs the oracle."""
    from paper_1705_01263_b200.render import RenderParams

    W = H = 1024
    pb, pe = 400 * W, 420 * W
    with _renderer(cornell_packed, W, H, 8) as r:
        r.render_pass(5, 9, pb, pe)
        fb = r.framebuffer()
    fb2, _ = oracle.OracleScene(cornell_packed).render(RenderParams(W, H, 8), 5, 9, pb, pe)
    assert np.array_equal(fb, fb2)


def test_execution_strategy_invariance(cornell_packed):
    """megakernel, wavefront at several pool sizes / regen thresholds / tail switch: identical."""
    outs = []
    cfgs = [dict(engine="megakernel"), dict(engine="wavefront", pool_log2=10), dict(engine="wavefront", pool_log2=14),
            dict(engine="wavefront", pool_log2=16, regen_fraction=0.0),
            dict(engine="wavefront", pool_log2=12, megakernel_tail=3000)]
    for cfg in cfgs:
        with _renderer(cornell_packed, 128, 96, 8, **cfg) as r:
            r.render_pass(0, 8)
            r.render_pass(8, 11)
            outs.append(r.framebuffer())
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)


def _class_scene(name):
    if name == "cornell":  # diffuse + no environment + alias lights
        return pack_scene(scenes.cornell())
    if name == "tree":  # diffuse + no environment (light hierarchy)
        return pack_scene(scenes.many_lights(300), lights="tree")
    if name == "furnace":  # diffuse under a constant environment
        sc = scenes.cornell()
        sc.environment = Environment(constant=(0.3, 0.3, 0.3))
        return pack_scene(sc)
    if name == "soup":  # one-layer diffuse / glossy, constant sky, alias lights, two layers at most
        return pack_scene(scenes.soup(1 << 14, n_materials=8))
    return pack_scene(scenes.envmap_scene(256, 128, sphere_subdiv=2))  # layered, image env, no emitters


@pytest.mark.parametrize("name", ["cornell", "tree", "furnace", "soup", "envmap"])
def test_material_class_instantiations_identical(gpu, oracle, monkeypatch, name):
    """Each scene class runs its specialised shading kernels (constants folded for the
    scene's materials, environment and light selection): identical to the general instantiations
    (LW_MATCLASS=0) and to the oracle."""
    from paper_1705_01263_b200.render import RenderParams

    packed = _class_scene(name)
    W, H, D = 96, 64, 8
    outs = []
    for v in ("1", "0"):
        monkeypatch.setenv("LW_MATCLASS", v)
        with _renderer(packed, W, H, D, pool_log2=12) as r:
            r.render_pass(0, 4)
            outs.append(r.framebuffer())
    fb2, _ = oracle.OracleScene(packed).render(RenderParams(W, H, D), 0, 4)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], fb2) and outs[0].sum() > 0


@pytest.mark.parametrize("cfg", ["C3", "C4", "C5"])
def test_other_configs_subset_bit_exact(gpu, oracle, cfg):
    from paper_1705_01263_b200.render import RenderParams

    c = scenes.CONFIGS[cfg]
    if cfg == "C3":
        sc = scenes.soup(1 << 16, n_materials=16)
    elif cfg == "C4":
        sc = scenes.envmap_scene(512, 256, sphere_subdiv=3)
    else:
        sc = scenes.many_lights(2000)
    packed = pack_scene(sc)
    W, H = 192, 108
    with _renderer(packed, W, H, c.max_depth) as r:
        r.render_pass(0, 3)
        fb = r.framebuffer()
    fb2, _ = oracle.OracleScene(packed).render(RenderParams(W, H, c.max_depth), 0, 3)
    assert np.array_equal(fb, fb2)
    assert fb.sum() > 0


@pytest.mark.parametrize("w,h", [(512, 256), (1000, 37)])
def test_env_alias_tables_block_build_matches_serial(gpu, oracle, monkeypatch, w, h):
    """The environment alias tables built one thread block per row in shared memory equal the
    one-thread-per-row construction (LW_ENV_SERIAL=1) and the oracle: renders bit-exact, including
    rows without weight (a black band) and a ragged width."""
    from paper_1705_01263_b200.render import RenderParams

    sc = scenes.envmap_scene(w, h, sphere_subdiv=2)
    sc.environment.image[h // 3: h // 3 + 4] = 0.0  # rows that are never drawn
    packed = pack_scene(sc)
    W, H = 64, 48
    fbs = []
    for serial in (False, True):
        if serial:
            monkeypatch.setenv("LW_ENV_SERIAL", "1")
        else:
            monkeypatch.delenv("LW_ENV_SERIAL", raising=False)
        with _renderer(packed, W, H, 6) as r:
            r.render_pass(0, 4)
            fbs.append(r.framebuffer())
    fb2, _ = oracle.OracleScene(packed).render(RenderParams(W, H, 6), 0, 4)
    assert np.array_equal(fbs[0], fbs[1]) and np.array_equal(fbs[0], fb2) and fbs[0].sum() > 0


def test_constant_env_camera_rays_return_L(gpu):
    """camera ray straight to a constant environment L returns L (every pixel, exactly)."""
    sc = Scene(camera=make_camera((0, 0, 5), (0, 0, 0)), meshes=[], instances=[],
               materials=[layered_material("m", [{"bsdf": "diffuse", "tint": 0.5}])], emitters=[],
               environment=Environment(constant=(0.25, 0.5, 1.0)))
    packed = pack_scene(sc)
    with _renderer(packed, 32, 32, 4) as r:
        r.render_pass(0, 4)
        img = r.image()
    assert np.all(img == np.array([0.25, 0.5, 1.0], dtype=np.float32))


def test_white_furnace(gpu):
    """unit-albedo diffuse sphere in a constant env converges to the env (1%)."""
    from paper_1705_01263_b200 import meshgen
    from paper_1705_01263_b200.scene import Mesh

    pos, nrm, uvw, tris = meshgen.icosphere((0, 0, 0), 1.0, 3)
    sc = Scene(camera=make_camera((0, 0, 4), (0, 0, 0), fov_y=30.0), meshes=[Mesh("s", pos, nrm, uvw, tris)],
               instances=[Instance("s", 0, 0)], materials=[layered_material("w", [{"bsdf": "diffuse", "tint": 1.0}])],
               emitters=[], environment=Environment(constant=(1.0, 1.0, 1.0)))
    packed = pack_scene(sc)
    with _renderer(packed, 32, 32, 8, rr_start=8) as r:
        r.render_pass(0, 256)
        img = r.image()
    assert abs(float(img.mean()) - 1.0) < 0.01


@pytest.mark.parametrize("n", [1, 5, 8, 100, 4097, 70000])
def test_gpu_sah_tree_traversal_matches_oracle(gpu, oracle, n):
    """The device-built SAH tree and the oracle's sequential restatement give identical hits on
    soups that exercise small-segment, large-segment and coincident-centroid paths."""
    sc = scenes.soup(n, n_materials=1, seed=n)
    if n == 4097:  # coincident centroids force the halving rule
        m = sc.meshes[0]
        m.positions[: len(m.positions) // 2] = m.positions[0]
    packed = pack_scene(sc, bvh="sah")
    o, d = _random_rays(20000, np.zeros(3), np.full(3, 20.0), n)
    with _renderer(packed, 8, 8, 2) as r:
        t, tri, b = r.trace_closest(o, d)
    t2, tri2, b2 = oracle.OracleScene(packed).trace_closest(o, d)
    assert np.array_equal(tri, tri2) and np.array_equal(_bits(t), _bits(t2)) and np.array_equal(_bits(b), _bits(b2))


def test_cli_render_writes_snapshots(gpu, tmp_path):
    from paper_1705_01263_b200 import cli
    from paper_1705_01263_b200.imagefiles import read_pfm

    out = str(tmp_path / "c1")
    assert cli.main(["render", "--config", "C1", "--res", "32x32", "--iterations", "4", "--snapshot-every", "2",
                     "--out", out, "--metrics", str(tmp_path / "m.json")]) == 0
    img = read_pfm(out + "_000004.pfm")
    assert img.shape == (32, 32, 3) and img.sum() > 0
    assert cli.main(["render", "--config", "C1", "--res", "bad"]) == 3


@pytest.mark.parametrize("cfg", ["C3", "C4", "C5"])
def test_full_size_config_band_bit_exact(gpu, oracle, cfg):
    """BASELINE configs at full scene size and resolution (2^20-triangle soup, 4K x 2K environment,
    10k emitters): a band of rows x 2 iterations bit-exact vs the oracle, with the alias samplers
    of the configs and with the light hierarchy / environment pyramid."""
    from paper_1705_01263_b200.render import RenderParams

    c = scenes.CONFIGS[cfg]
    sc = c.builder()
    W, H = c.width, c.height
    pb, pe = 530 * W, 534 * W
    for kw in ({}, {"lights": "tree", "env_sampling": "pyramid"}):
        if kw and cfg == "C3":
            continue
        packed = pack_scene(sc, **kw)
        with _renderer(packed, W, H, c.max_depth) as r:
            r.render_pass(7, 9, pb, pe)
            fb = r.framebuffer()
        fb2, _ = oracle.OracleScene(packed).render(RenderParams(W, H, c.max_depth), 7, 9, pb, pe)
        assert np.array_equal(fb, fb2), (cfg, kw)
        assert fb[pb:pe].sum() > 0


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_full_frame_pass_split_and_pool_invariance(gpu, cfg):
    """Size-independent properties at the full resolution: one pass of 4 iterations equals two
    passes of 2 (int64 accumulation is associative) and does not depend on the pool size."""
    c = scenes.CONFIGS[cfg]
    packed = pack_scene(c.builder())
    outs = []
    for pool, splits in ((22, [(0, 4)]), (22, [(0, 2), (2, 4)]), (18, [(0, 4)])):
        with _renderer(packed, c.width, c.height, c.max_depth, pool_log2=pool) as r:
            for a, b in splits:
                r.render_pass(a, b)
            outs.append(r.framebuffer())
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)


@pytest.mark.parametrize("cfg", ["C2", "C3", "C5"])
def test_persistent_refill_trace_invariance(gpu, cfg, monkeypatch):
    """The persistent lane-refill trace kernels with speculative traversal (the default, for
    shared- and global-memory BVHs) and the one-ray-per-thread kernels give the same full-frame
    framebuffer (same hits), with and without LPE layers (the LPE shadow instantiation)."""
    c = scenes.CONFIGS[cfg]
    packed = pack_scene(c.builder())
    outs = []
    for mask in ("0", "5", "10", "15"):
        monkeypatch.setenv("LW_TRACE_PERSIST", mask)
        with _renderer(packed, c.width, c.height, c.max_depth) as r:
            r.render_pass(0, 2)
            fb = r.framebuffer()
            r.clear()
            r.set_lpe_layers({"direct": "C.?L", "all": "C.*[LE]"})
            r.render_pass(0, 1)
            outs.append((fb, r.layer_framebuffers()))
    for fb, layers in outs[1:]:
        assert np.array_equal(outs[0][0], fb)
        for k in layers:
            assert np.array_equal(outs[0][1][k], layers[k]), k
    assert outs[0][0].sum() > 0


@pytest.mark.parametrize("name", ["cornell", "soup65k", "many_lights", "soup1M"])
def test_warp_sah_decide_builds_the_serial_tree(gpu, name, monkeypatch):
    """The warp-per-segment SAH split decision builds the same render tree as the per-thread one
    (LW_SAH_SERIAL=1): the extension-ray work counters of the one-ray-per-thread trace kernels (a
    function of the tree) agree exactly on a full pass."""
    sc = {"cornell": lambda: scenes.cornell(), "soup65k": lambda: scenes.soup(1 << 16),
          "many_lights": lambda: scenes.many_lights(), "soup1M": lambda: scenes.soup()}[name]()
    packed = pack_scene(sc, bvh="sah")
    monkeypatch.setenv("LW_TRACE_PERSIST", "0")
    prof = []
    for serial in (True, False):
        if serial:
            monkeypatch.setenv("LW_SAH_SERIAL", "1")
        else:
            monkeypatch.delenv("LW_SAH_SERIAL", raising=False)
        with _renderer(packed, 256, 256, 6) as r:
            r.set_instrumentation(count_work=True)
            r.render_pass(0, 1)
            p = r.kernel_profile()
            # extension rays only: the shadow kernels traverse speculatively, and which lanes are
            # converged at a speculation vote is up to the warp scheduler (counts vary, hits do not)
            prof.append({k: p[k] for k in ("ext_nodes", "ext_tris")})
    assert prof[0] == prof[1]
    assert prof[0]["ext_nodes"] > 0


@pytest.mark.parametrize("name", ["cornell", "soup1000", "soup4096", "coincident"])
def test_single_block_sah_build_matches_level_build(gpu, name, monkeypatch):
    """Scenes up to 4096 triangles build their SAH tree in one thread block (k_sah_small); the tree
    is the level-synchronous build's (LW_SAH_LEVELS=1): same hits and same traversal work."""
    if name == "coincident":
        sc = scenes.soup(3000, n_materials=1, seed=7)
        m = sc.meshes[0]
        m.positions[: len(m.positions) // 3] = m.positions[0]
    else:
        sc = {"cornell": lambda: scenes.cornell(), "soup1000": lambda: scenes.soup(1000, n_materials=1, seed=3),
              "soup4096": lambda: scenes.soup(4096, n_materials=1, seed=4)}[name]()
    packed = pack_scene(sc, bvh="sah")
    lo, hi = (np.array([0.0, 0.0, -0.5]), np.array([1.0, 1.0, 3.0])) if name == "cornell" else (np.zeros(3), np.full(3, 20.0))
    o, d = _random_rays(20000, lo, hi, 9)
    monkeypatch.setenv("LW_TRACE_PERSIST", "0")
    outs = []
    for levels in (False, True):
        if levels:
            monkeypatch.setenv("LW_SAH_LEVELS", "1")
        else:
            monkeypatch.delenv("LW_SAH_LEVELS", raising=False)
        with _renderer(packed, 96, 64, 5) as r:
            hits = r.trace_closest(o, d)
            r.set_instrumentation(count_work=True)
            r.render_pass(0, 2)
            p = r.kernel_profile()
            outs.append((hits, {k: p[k] for k in ("ext_nodes", "ext_tris")}, r.framebuffer()))
    (h0, c0, f0), (h1, c1, f1) = outs
    assert all(np.array_equal(_bits(a) if a.dtype == np.float64 else a, _bits(b) if b.dtype == np.float64 else b)
               for a, b in zip(h0, h1))
    assert c0 == c1 and c0["ext_nodes"] > 0
    assert np.array_equal(f0, f1)


def test_degenerate_deep_sah_tree_falls_back_to_median(gpu, oracle):
    """A SAH tree deeper than the traversal stack (exponentially spaced triangles) is replaced by the
    median tree at upload; hits do not depend on the tree, so the image still matches the oracle."""
    from paper_1705_01263_b200.render import RenderParams
    from paper_1705_01263_b200.scenes import _mesh, diffuse_material
    from paper_1705_01263_b200.scene import Instance, Scene, make_camera

    n = 300
    x = np.cumsum(1.5 ** np.arange(n) * 1e-6)  # exponential spacing: SAH peels one triangle per level
    pos = np.concatenate([np.stack([x, np.zeros(n), np.zeros(n)], 1), np.stack([x, np.full(n, 1e-7), np.zeros(n)], 1),
                          np.stack([x, np.zeros(n), np.full(n, 1e-7)], 1)])
    tris = np.stack([np.arange(n), np.arange(n) + n, np.arange(n) + 2 * n], 1)
    sc = Scene(camera=make_camera((0, 0, 5), (0, 0, 0)), meshes=[_mesh("comb", pos, np.zeros_like(pos), np.zeros_like(pos), tris)],
               instances=[Instance("comb", 0, 0)], materials=[diffuse_material("m", (0.5, 0.5, 0.5))], emitters=[],
               environment=scenes.Environment(constant=(1.0, 1.0, 1.0)))
    packed = pack_scene(sc)
    with _renderer(packed, 16, 16, 2) as r:
        r.render_pass(0, 2)
        fb = r.framebuffer()
    fb2, _ = oracle.OracleScene(packed).render(RenderParams(16, 16, 2), 0, 2)
    assert np.array_equal(fb, fb2)


def test_checkpoint_resume_bit_exact(cornell_packed, tmp_path):
    """save after iterations [0, 6), resume in a new context, render [6, 12): identical
    to rendering [0, 12) in one context; a checkpoint of another scene is refused."""
    ck = str(tmp_path / "ck.npz")
    with _renderer(cornell_packed, 48, 32, 5) as r:
        r.render_pass(0, 6)
        r.save_checkpoint(ck)
    with _renderer(cornell_packed, 48, 32, 5) as r:
        r.load_checkpoint(ck)
        assert r.iterations == 6
        r.render_pass(6, 12)
        resumed = r.framebuffer()
    with _renderer(cornell_packed, 48, 32, 5) as r:
        r.render_pass(0, 12)
        assert np.array_equal(r.framebuffer(), resumed)
    with _renderer(pack_scene(scenes.soup(64, seed=1)), 48, 32, 5) as r:
        with pytest.raises(ValueError):
            r.load_checkpoint(ck)


def test_cli_checkpoint_resume(gpu, tmp_path):
    from paper_1705_01263_b200 import cli
    from paper_1705_01263_b200.imagefiles import read_pfm

    a, b, ck = str(tmp_path / "a"), str(tmp_path / "b"), str(tmp_path / "ck.npz")
    base = ["render", "--config", "C1", "--res", "24x16"]
    assert cli.main(base + ["--iterations", "8", "--out", a]) == 0
    assert cli.main(base + ["--iterations", "4", "--out", b, "--checkpoint", ck]) == 0
    assert cli.main(base + ["--iterations", "8", "--out", b, "--resume", ck]) == 0
    assert (read_pfm(a + "_000008.pfm") == read_pfm(b + "_000008.pfm")).all()


# ---- compressed path state ---------------------------------

@pytest.mark.parametrize("cfg", ["C1", "C3", "C4", "C5"])
def test_compact_state_bit_exact_vs_oracle_both_engines(gpu, oracle, cfg):
    """Oct-16 directions and FP32 throughput / radiance / pdf, quantised where produced: the
    wavefront (64-byte pool state), the megakernel (registers) and the oracle agree bit for bit."""
    from paper_1705_01263_b200.render import RenderParams

    c = scenes.CONFIGS[cfg]
    sc = {"C1": scenes.cornell, "C3": lambda: scenes.soup(1 << 16, n_materials=16),
          "C4": lambda: scenes.envmap_scene(512, 256, sphere_subdiv=3), "C5": lambda: scenes.many_lights(2000)}[cfg]()
    packed = pack_scene(sc)
    W, H = (64, 64) if cfg == "C1" else (192, 108)
    fbs = []
    for engine in ("wavefront", "megakernel"):
        with _renderer(packed, W, H, c.max_depth, engine=engine, compact_state=True, pool_log2=14) as r:
            r.render_pass(0, 3)
            fbs.append(r.framebuffer())
    fb2, _ = oracle.OracleScene(packed).render(RenderParams(W, H, c.max_depth, compact_state=True), 0, 3)
    assert np.array_equal(fbs[0], fb2) and np.array_equal(fbs[1], fb2)
    # the compressed state changes bits, not the image: same mean radiance as the FP64 state
    fb64, _ = oracle.OracleScene(packed).render(RenderParams(W, H, c.max_depth), 0, 3)
    m_c, m_64 = fb2.astype(np.float64).mean(), fb64.astype(np.float64).mean()
    assert not np.array_equal(fb2, fb64) and abs(m_c - m_64) <= 0.02 * m_64


def test_compact_state_pool_and_tail_invariance(cornell_packed):
    """Compact state under different pool sizes / regeneration / megakernel tail: identical."""
    outs = []
    for cfg in [dict(engine="megakernel"), dict(pool_log2=10), dict(pool_log2=16, regen_fraction=0.0),
                dict(pool_log2=12, megakernel_tail=3000)]:
        with _renderer(cornell_packed, 128, 96, 8, compact_state=True, **cfg) as r:
            r.render_pass(0, 8)
            outs.append(r.framebuffer())
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)


# ---- asynchronous passes: the CUDA-graph wave loop ------------------------------

def test_queued_passes_equal_one_pass_and_host_loop(cornell_packed, monkeypatch):
    """Passes queued back to back without a host sync (graph path) == one pass == the host-driven
    loop (LW_GRAPH=0), bit for bit; the running statistics count every path."""
    W, H = 96, 64
    with _renderer(cornell_packed, W, H, 8, pool_log2=12) as r:
        for a in range(0, 12, 3):
            r.render_pass(a, a + 3)  # returns once queued
        fb_q = r.framebuffer()
        st = r.stats()
    assert st["paths"] == W * H * 12
    with _renderer(cornell_packed, W, H, 8, pool_log2=12) as r:
        r.render_pass(0, 12)
        fb_1 = r.framebuffer()
    monkeypatch.setenv("LW_GRAPH", "0")
    with _renderer(cornell_packed, W, H, 8, pool_log2=12) as r:
        r.render_pass(0, 12)
        fb_h = r.framebuffer()
    assert np.array_equal(fb_q, fb_1) and np.array_equal(fb_1, fb_h)


def test_stage_timing_inside_the_graph(cornell_packed):
    """LW_INSTR_TIME stamps every stage inside the graph: every stage has time and launches, and
    the stage times add up to at most the pass time."""
    with _renderer(cornell_packed, 256, 256, 8) as r:
        r.set_instrumentation(time_kernels=True)
        r.render_pass(0, 16)
        kp = r.kernel_profile()
    for st in ("generate", "trace_ext", "shade_nee", "shade", "trace_shadow"):
        assert kp["stage_ms"][st] > 0 and kp["stage_launches"][st] >= 1, st
    assert sum(kp["stage_ms"].values()) <= kp["total_ms"] * 1.05
    assert kp["ext_rays"] > 0 and kp["paths"] == 256 * 256 * 16


def test_checkpoint_refuses_other_camera_material_or_environment(cornell_packed, tmp_path):
    """The checkpoint fingerprint covers camera, materials, environment and sampler choices, not
    only the geometry: a checkpoint is refused by a render that would produce a different image."""
    from paper_1705_01263_b200.scene import make_camera

    ck = str(tmp_path / "ck.npz")
    with _renderer(cornell_packed, 32, 32, 4) as r:
        r.render_pass(0, 2)
        r.save_checkpoint(ck)
    base = scenes.cornell()
    moved = scenes.cornell()
    moved.camera = make_camera((0.5, 0.55, 2.5), (0.5, 0.5, 0.0), fov_y=45.0)
    tinted = scenes.cornell()
    tinted.materials[2].nodes[0].value = (0.7, 0.75, 0.75)
    env = scenes.cornell()
    env.environment = Environment(constant=(0.1, 0.1, 0.1))
    for variant in (pack_scene(moved), pack_scene(tinted), pack_scene(env), pack_scene(base, lights="tree")):
        with _renderer(variant, 32, 32, 4) as r:
            with pytest.raises(ValueError):
                r.load_checkpoint(ck)
    with _renderer(pack_scene(base), 32, 32, 4, compact_state=True) as r:  # different state layout
        with pytest.raises(ValueError):
            r.load_checkpoint(ck)
    with _renderer(pack_scene(base), 32, 32, 4, engine="megakernel") as r:  # same image: accepted
        r.load_checkpoint(ck)


def test_checkpoint_resume_with_lpe_layers(cornell_packed, tmp_path):
    """Checkpoints carry the LPE layer framebuffers: a resumed render's layers equal an
    uninterrupted one's; a renderer with different layers refuses the checkpoint."""
    ck = str(tmp_path / "ck.npz")
    layers = {"direct": "C.?L", "all": "C.*[LE]"}
    with _renderer(cornell_packed, 32, 32, 5) as r:
        r.set_lpe_layers(layers)
        r.render_pass(0, 4)
        r.save_checkpoint(ck)
    with _renderer(cornell_packed, 32, 32, 5) as r:  # layers restored from the checkpoint
        r.load_checkpoint(ck)
        r.render_pass(4, 8)
        resumed = r.layer_framebuffers()
        fb_resumed = r.framebuffer()
    with _renderer(cornell_packed, 32, 32, 5) as r:
        r.set_lpe_layers(layers)
        r.render_pass(0, 8)
        ref = r.layer_framebuffers()
        assert np.array_equal(r.framebuffer(), fb_resumed)
    for k in layers:
        assert np.array_equal(resumed[k], ref[k]) and ref[k].sum() > 0
    with _renderer(cornell_packed, 32, 32, 5) as r:
        r.set_lpe_layers({"other": "C.*E"})
        with pytest.raises(ValueError):
            r.load_checkpoint(ck)
