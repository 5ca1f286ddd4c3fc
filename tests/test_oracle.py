"""Pin the CPU oracle: bit-exact against the reference's golden vectors and (when built) the
reference's own compiled kernels.  CPU only."""

import numpy as np
import pytest

from conftest import golden


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def test_halton_all_dims_golden(oracle):
    g = golden("halton.npz")
    t = golden("qmc_tables.npz")
    bases, perm, off = t["d8_bases"], t["d8_perm_flat"], t["d8_perm_offset"]
    for dim in range(len(bases)):
        out = oracle.halton_batch(bases, perm, off, dim, g["indices"])
        assert np.array_equal(_bits(out), _bits(g["values"][dim])), f"dim {dim}"
        big = oracle.halton_batch(bases, perm, off, dim, g["big_indices"])
        assert np.array_equal(_bits(big), _bits(g["big_values"][dim])), f"dim {dim} (index >= 2^53)"


def test_pixel_offset_golden(oracle):
    g = golden("pixel_offset.npz")
    out = oracle.pixel_offset_batch(g["u"])
    assert np.array_equal(_bits(out), _bits(g["offsets"]))


def test_pixel_offset_spec_known_answers(oracle):
    # u=(0.5,0.5) -> (0,0); |offset| <= 1.5
    assert tuple(oracle.pixel_offset_batch([[0.5, 0.5]])[0]) == (0.0, 0.0)
    u = np.random.default_rng(0).random((20000, 2))
    assert np.abs(oracle.pixel_offset_batch(u)).max() <= 1.5


def test_oct_golden(oracle):
    g = golden("oct.npz")
    out = np.full_like(g["vecs"], -7.0)
    got = oracle.oct_roundtrip_batch(g["vecs"])
    ok = np.linalg.norm(g["vecs"], axis=1) > 0
    assert np.array_equal(got[ok], g["roundtrip"][ok])
    for v, e in zip(g["vecs"][ok], g["encoded"][ok]):
        assert oracle.oct_encode(v) == int(e)
    del out


@pytest.mark.parametrize("name", ["tri1", "tri4", "tri5", "rand200", "cornellbox", "ico2", "soup5k", "quad", "coincident"])
def test_bvh_build_golden(oracle, name):
    g = golden("bvh_traversal.npz")
    b, c, o = oracle.build_bvh(g[f"{name}_verts"])
    assert np.array_equal(b, g[f"{name}_bounds"])
    assert np.array_equal(c, g[f"{name}_children"])
    assert np.array_equal(o, g[f"{name}_order"])


@pytest.mark.parametrize("name", ["tri1", "tri5", "rand200", "cornellbox", "ico2", "soup5k", "quad", "coincident"])
@pytest.mark.parametrize("mode", ["compat", "corrected"])
def test_traversal_golden(oracle, name, mode):
    g = golden("bvh_traversal.npz")
    t, tri, bary = oracle.intersect_batch(0 if mode == "compat" else 1, g[f"{name}_bounds"], g[f"{name}_children"],
                                          g[f"{name}_order"], g[f"{name}_verts"], g[f"{name}_origins"],
                                          g[f"{name}_dirs"], g[f"{name}_tmax"])
    assert np.array_equal(tri, g[f"{name}_{mode}_tri"])
    assert np.array_equal(_bits(t), _bits(g[f"{name}_{mode}_t"]))
    assert np.array_equal(_bits(bary), _bits(g[f"{name}_{mode}_bary"]))


def test_corrected_equals_brute_force(oracle):
    g = golden("bvh_traversal.npz")
    for name in ["rand200", "ico2", "soup5k", "cornellbox"]:
        args = (g[f"{name}_bounds"], g[f"{name}_children"], g[f"{name}_order"], g[f"{name}_verts"],
                g[f"{name}_origins"], g[f"{name}_dirs"], g[f"{name}_tmax"])
        t1, tri1, _ = oracle.intersect_batch(1, *args)
        t2, tri2, _ = oracle.intersect_batch(2, *args)
        assert np.array_equal(tri1, tri2) and np.array_equal(t1, t2), name


def test_oracle_matches_compiled_reference_live(oracle, ref_pristine, ref_corrected):
    """Fresh random inputs through the reference's own compiled kernels (oracle/_ref)."""
    rng = np.random.default_rng(99)
    t = golden("qmc_tables.npz")
    idx = rng.integers(0, 2**40, 4096).astype(np.int64)
    out = np.zeros(len(idx))
    for dim in (0, 1, 2, 3, 9, 17, 30, 67, 137):
        ref_pristine.halton_batch(t["d8_bases"], t["d8_perm_flat"], t["d8_perm_offset"], dim, idx, out)
        got = oracle.halton_batch(t["d8_bases"], t["d8_perm_flat"], t["d8_perm_offset"], dim, idx)
        assert np.array_equal(_bits(got), _bits(out))
    n = 3000
    verts = rng.random((n, 9)) * 10
    b, c, o = oracle.build_bvh(verts)
    orig = rng.random((4000, 3)) * 10
    dirs = rng.normal(size=(4000, 3))
    dirs[:300, 2] = 0.0
    tm = np.full(4000, np.inf)
    for mode, mod in ((0, ref_pristine), (1, ref_corrected)):
        rt, rtri, rb = np.empty(4000), np.empty(4000, np.int64), np.empty((4000, 2))
        mod.intersect_batch(b, c, o, verts, np.zeros(n, np.int64), orig, dirs, tm, rt, rtri, rb)
        t2, tri2, b2 = oracle.intersect_batch(mode, b, c, o, verts, orig, dirs, tm)
        assert np.array_equal(rtri, tri2) and np.array_equal(_bits(rt), _bits(t2)) and np.array_equal(_bits(rb), _bits(b2))


def test_deterministic_math(oracle):
    for u in np.linspace(0, 1, 1001):
        s, c = oracle.sincos2pi(u)
        assert abs(s - np.sin(2 * np.pi * u)) < 4e-15 and abs(c - np.cos(2 * np.pi * u)) < 4e-15
    rng = np.random.default_rng(3)
    for y, x in rng.normal(size=(2000, 2)):
        assert abs(oracle.atan2(y, x) - np.arctan2(y, x)) < 4e-15
    assert oracle.atan2(0.0, -1.0) == np.pi and oracle.atan2(0.0, 1.0) == 0.0


def test_alias_table(oracle):
    w = np.random.default_rng(1).random(1000) ** 4
    prob, alias, pdf = oracle.alias_build(w)
    assert np.allclose(pdf, w / w.sum())
    # implied distribution: P(i) = (prob[i] + sum_{j: alias[j]=i} (1-prob[j])) / n
    implied = prob.copy()
    np.add.at(implied, alias, 1.0 - prob)
    assert np.allclose(implied / len(w), pdf, atol=1e-12)
    with pytest.raises(ValueError):
        oracle.alias_build(np.zeros(4))


@pytest.mark.parametrize("bvh", ["sah", "median"])
def test_render_traversal_equals_brute_force(oracle, bvh):
    """Near-first traversal with the conservative cull over either render tree == exhaustive search."""
    from paper_1705_01263_b200 import scenes
    from paper_1705_01263_b200.scene import pack_scene

    for sc, lo, hi in ((scenes.cornell(), np.array([0.0, 0.0, -0.5]), np.array([1.0, 1.0, 3.0])),
                       (scenes.soup(4000, n_materials=4), np.zeros(3), np.full(3, 20.0))):
        packed = pack_scene(sc, bvh=bvh)
        osc = oracle.OracleScene(packed)
        rng = np.random.default_rng(5)
        o = lo + rng.random((6000, 3)) * (hi - lo)
        d = rng.normal(size=(6000, 3))
        d[:300, 1] = 0.0
        tm = np.where(np.arange(6000) % 4 == 0, 2.5, np.inf)
        t, tri, b = osc.trace_closest(o, d, tm)
        t2, tri2, b2 = oracle.intersect_batch(2, np.zeros((1, 6)), np.zeros((1, 2), np.int64), np.zeros(0, np.int64),
                                              packed.verts, o, d, tm)
        assert np.array_equal(tri, tri2) and np.array_equal(t, t2) and np.array_equal(b, b2)
        # any-hit (0 < t < tmax) == "the exhaustive closest hit without a limit is nearer than tmax"
        t3, tri3, _ = oracle.intersect_batch(2, np.zeros((1, 6)), np.zeros((1, 2), np.int64), np.zeros(0, np.int64),
                                             packed.verts, o, d, np.full(len(o), np.inf))
        occ = osc.trace_any(o, d, np.full(len(o), 3.0))
        assert np.array_equal(occ.astype(bool), (tri3 >= 0) & (t3 < 3.0))
