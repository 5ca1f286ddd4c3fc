"""Stateless sm_100a kernels through the C ABI vs the oracle and the reference's golden vectors.

Bar: bit-exact (integer digits, FP64 results compared as bit patterns)."""

import ctypes as C

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def test_halton_golden_all_dims(gpu):
    from paper_1705_01263_b200.core import kernels

    g = golden("halton.npz")
    t = golden("qmc_tables.npz")
    for dim in range(len(t["d8_bases"])):
        out = np.zeros(len(g["indices"]))
        kernels.halton_batch(t["d8_bases"], t["d8_perm_flat"], t["d8_perm_offset"], dim, g["indices"], out)
        assert np.array_equal(_bits(out), _bits(g["values"][dim])), f"dim {dim}"
        out = np.zeros(len(g["big_indices"]))
        kernels.halton_batch(t["d8_bases"], t["d8_perm_flat"], t["d8_perm_offset"], dim, g["big_indices"], out)
        assert np.array_equal(_bits(out), _bits(g["big_values"][dim])), f"dim {dim} big"


def test_halton_reference_kernel_test(gpu):
    """test_qmc.py:59-67 replayed on the device: kernel == exact Python API."""
    from paper_1705_01263_b200 import qmc
    from paper_1705_01263_b200.core import kernels

    table = qmc.DimensionTable(max_depth=4)
    rng = np.random.default_rng(7)
    idx = rng.integers(0, 2**40, 256)
    out = np.zeros(256)
    for dim in [0, 1, 2, 3, 9, 17, 30]:
        kernels.halton_batch(table.bases, table.perm_flat, table.perm_offset, dim, idx, out)
        for k, i in enumerate(idx.tolist()):
            assert out[k] == qmc.radical_inverse(int(table.bases[dim]), i)


@pytest.mark.parametrize("depth", [4, 8, 12])
def test_halton_vs_oracle_at_scale(gpu, oracle, depth):
    """Every eye dimension of every config's table, 2^18 indices up to the configs' max index (~2^30)."""
    from paper_1705_01263_b200 import qmc
    from paper_1705_01263_b200.core import kernels

    t = qmc.DimensionTable(depth)
    rng = np.random.default_rng(depth)
    # dense small indices, the configs' range, the 32-bit digit-block boundary and beyond it
    edge = np.array([(1 << 32) - 2, (1 << 32) - 1, 1 << 32, (1 << 32) + 1, (1 << 40) + 3], np.int64)
    idx = np.concatenate([np.arange(1 << 16), rng.integers(0, 1 << 31, (1 << 18) - (1 << 16) - 4096),
                          rng.integers(1 << 31, 1 << 32, 4096 - len(edge)), edge]).astype(np.int64)
    out = np.zeros(len(idx))
    for dim in range(4 + 8 * depth):
        kernels.halton_batch(t.bases, t.perm_flat, t.perm_offset, dim, idx, out)
        ref = oracle.halton_batch(t.bases, t.perm_flat, t.perm_offset, dim, idx)
        assert np.array_equal(_bits(out), _bits(ref)), f"dim {dim}"


def test_pixel_offset_golden(gpu):
    from paper_1705_01263_b200.core import kernels

    g = golden("pixel_offset.npz")
    out = kernels.pixel_offset_batch(g["u"])
    assert np.array_equal(_bits(out), _bits(g["offsets"]))
    assert kernels.sample_pixel_offset(0.5, 0.5) == (0.0, 0.0)


def test_pixel_offset_glibc_log_tails(gpu, oracle):
    """Device port of glibc's FMA log against the host libm in the filter's tail domain."""
    from paper_1705_01263_b200.core import kernels

    rng = np.random.default_rng(5)
    u = np.concatenate([rng.random(1 << 20) * 0.023, 1.0 - rng.random(1 << 20) * 0.023]).reshape(-1, 2)
    assert np.array_equal(_bits(kernels.pixel_offset_batch(u)), _bits(oracle.pixel_offset_batch(u)))


def test_oct_golden(gpu):
    from paper_1705_01263_b200.core import kernels

    g = golden("oct.npz")
    out = np.full_like(g["vecs"], -7.0)
    kernels.oct_roundtrip_batch(np.ascontiguousarray(g["vecs"]), out)
    assert np.array_equal(out, g["roundtrip"])
    ok = np.linalg.norm(g["vecs"], axis=1) > 0
    for v, e, d in list(zip(g["vecs"][ok], g["encoded"][ok], g["decoded"][ok]))[:500]:
        assert kernels.compress_unit_vector(*v) == int(e)
        assert kernels.decompress_unit_vector(int(e)) == tuple(d)
    with pytest.raises(ValueError):
        kernels.compress_unit_vector(0.0, 0.0, 0.0)


NAMES = ["tri1", "tri4", "tri5", "rand200", "cornellbox", "ico2", "soup5k", "quad", "coincident"]


@pytest.mark.parametrize("name", NAMES)
def test_bvh_build_golden(gpu, name):
    from paper_1705_01263_b200 import geometry

    g = golden("bvh_traversal.npz")
    b, c, o = geometry.build_bvh(g[f"{name}_verts"])
    assert np.array_equal(b, g[f"{name}_bounds"])
    assert np.array_equal(c, g[f"{name}_children"])
    assert np.array_equal(o, g[f"{name}_order"])


@pytest.mark.parametrize("n", [0, 6, 1000, 65537, 1 << 20])
def test_bvh_build_vs_oracle(gpu, oracle, n):
    from paper_1705_01263_b200 import geometry

    rng = np.random.default_rng(n)
    base = rng.random((n, 3)) * 20
    verts = np.concatenate([base, base + rng.normal(size=(n, 3)) * 0.3, base + rng.normal(size=(n, 3)) * 0.3], 1)
    if n >= 1000:
        verts[: n // 7, 1] = 0.0  # duplicate centroid keys exercise the (key, id) tie rule
        verts[: n // 7, 4] = -0.0
        verts[: n // 7, 7] = 0.0
    b, c, o = geometry.build_bvh(verts)
    if n == 0:
        assert b.shape == (1, 6) and c.tolist() == [[-1, 0]] and len(o) == 0
        return
    b2, c2, o2 = oracle.build_bvh(verts)
    assert np.array_equal(c, c2) and np.array_equal(o, o2) and np.array_equal(b, b2)


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("mode", ["compat", "corrected"])
def test_intersect_golden(gpu, name, mode):
    from paper_1705_01263_b200.core import kernels

    g = golden("bvh_traversal.npz")
    n = len(g[f"{name}_origins"])
    t, tri, bary = np.empty(n), np.empty(n, np.int64), np.empty((n, 2))
    kernels.intersect_batch(g[f"{name}_bounds"], g[f"{name}_children"], g[f"{name}_order"], g[f"{name}_verts"], None,
                            g[f"{name}_origins"], g[f"{name}_dirs"], g[f"{name}_tmax"], t, tri, bary, mode=mode)
    assert np.array_equal(tri, g[f"{name}_{mode}_tri"])
    assert np.array_equal(_bits(t), _bits(g[f"{name}_{mode}_t"]))
    assert np.array_equal(_bits(bary), _bits(g[f"{name}_{mode}_bary"]))


def test_intersect_large_soup_vs_oracle(gpu, oracle):
    from paper_1705_01263_b200 import geometry
    from paper_1705_01263_b200.core import kernels

    rng = np.random.default_rng(17)
    n = 200_000
    base = rng.random((n, 3)) * 20
    verts = np.concatenate([base, base + rng.normal(size=(n, 3)) * 0.3, base + rng.normal(size=(n, 3)) * 0.3], 1)
    b, c, o = geometry.build_bvh(verts)
    m = 20000
    orig = rng.random((m, 3)) * 20
    dirs = rng.normal(size=(m, 3))
    tm = np.full(m, np.inf)
    for mode, code in (("compat", 0), ("corrected", 1), ("brute", 2)):
        if mode == "brute":
            orig, dirs, tm = orig[:500], dirs[:500], tm[:500]
        k = len(orig)
        t, tri, bary = np.empty(k), np.empty(k, np.int64), np.empty((k, 2))
        kernels.intersect_batch(b, c, o, verts, None, orig, dirs, tm, t, tri, bary, mode=mode)
        t2, tri2, b2 = oracle.intersect_batch(code, b, c, o, verts, orig, dirs, tm)
        assert np.array_equal(tri, tri2) and np.array_equal(_bits(t), _bits(t2)) and np.array_equal(_bits(bary), _bits(b2))


def test_abi_error_paths(gpu):
    from paper_1705_01263_b200 import _abi

    lib = _abi.lib()
    assert lib.lw_halton_batch(None, 0, None, 0, None, 0, None, 0, None) == _abi.LW_ERR_INVALID
    assert len(lib.lw_last_error()) > 0
    n = C.c_int()
    assert lib.lw_device_count(C.byref(n)) == 0 and n.value >= 1
