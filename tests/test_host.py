"""Host-side logic (CPU only): QMC tables, dividers, meshes, flattening, packing, ABI exports, IO."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden


def test_dimension_tables_match_reference():
    from paper_1705_01263_b200 import qmc

    g = golden("qmc_tables.npz")
    for d in (4, 8, 12):
        t = qmc.DimensionTable(d)
        for k in ("bases", "perm_flat", "perm_offset", "magic", "shift", "add"):
            assert np.array_equal(np.asarray(getattr(t, k)), g[f"d{d}_{k}"]), (d, k)


def test_dimension_layout():
    from paper_1705_01263_b200 import qmc

    t = qmc.DimensionTable(max_depth=8)  # test_qmc.py:200-209
    assert t.bases[0] == 2 and t.bases[1] == 3 and t.bases[2] == 5
    assert t.eye_bounce_dim(0, qmc.OFF_BSDF_U) == 4
    assert t.eye_bounce_dim(1, qmc.OFF_NEE_U) == 4 + 8 + 2
    assert t.light_bounce_dim(0, 0) == t.light_base + qmc.LIGHT_HEAD_DIMS
    assert np.all(t.bases[1:] > t.bases[:-1])
    assert qmc.DimensionTable(2).sample(0, 1) == 0.5


def test_radical_inverse_exact():
    from fractions import Fraction

    from paper_1705_01263_b200 import qmc

    assert qmc.radical_inverse(2, 1) == 0.5 and qmc.radical_inverse(2, 6) == 0.375
    for base in (3, 5, 7, 97):
        perm = qmc.faure_permutation(base)
        for i in [0, 1, 2, 1000, 999999, 2**40 + 7]:
            rev, scale, k = 0, 1, i
            while k:
                k, dgt = divmod(k, base)
                rev = rev * base + int(perm[dgt])
                scale *= base
            assert qmc.radical_inverse(base, i) == float(Fraction(rev, scale))
    with pytest.raises(ValueError):
        qmc.radical_inverse(3, 2**64)
    assert 0.0 <= qmc.radical_inverse(3, 2**64 - 1) < 1.0


def test_permutations():
    from paper_1705_01263_b200 import qmc

    for base in qmc.primes(60).tolist():
        p = qmc.faure_permutation(base)
        assert sorted(p.tolist()) == list(range(base)) and p[0] == 0
    assert qmc.faure_permutation(2).tolist() == [0, 1]
    with pytest.raises(ValueError):
        qmc.ScrambledBase(3, np.array([0, 0, 2]))


def _mulhi(magic, n, bits):
    return (int(magic) * int(n)) >> bits


@pytest.mark.parametrize("bits", [32, 64])
def test_fast_divisor_exhaustive_reduced_width(bits):
    """test_qmc.py:109-115 for both widths: every n < 2^16 and 4096 random n, all primes < 1000."""
    from paper_1705_01263_b200 import qmc

    rng = np.random.default_rng(bits)
    ns = list(range(1 << 16)) + [int(x) for x in rng.integers(0, 2**bits - 1, 4096, dtype=np.uint64)]
    ns += [2**bits - 1, 2**bits - 2, 2**(bits - 1)]
    for p in qmc.primes(168).tolist():
        d = qmc.prepare_fast_divisor(p, bits)
        for n in ns[::7] if p > 100 else ns:
            assert qmc.fast_divide(d, n, bits) == n // p


def test_fast_divisor_vectorised_32bit_full_scan():
    """32-bit magics (the device's fast path) against numpy for 2^22 consecutive values x 30 bases."""
    from paper_1705_01263_b200 import qmc

    n = np.arange(1 << 22, dtype=np.uint64) * np.uint64(1021)  # spans [0, 2^32)
    for p in qmc.primes(30).tolist()[1:]:
        d = qmc.prepare_fast_divisor(p, 32)
        hi = (n * np.uint64(d.magic)) >> np.uint64(32)
        q = ((((n - hi) >> np.uint64(1)) + hi) >> np.uint64(d.shift)) if d.add else (hi >> np.uint64(d.shift))
        assert np.array_equal(q, n // np.uint64(p)), p


def test_global_sample_index():
    from paper_1705_01263_b200 import qmc

    assert qmc.global_sample_index(7, 2, 100) == 207
    with pytest.raises(OverflowError):
        qmc.global_sample_index(0, 2**40, 2**25)
    with pytest.raises(ValueError):
        qmc.global_sample_index(100, 0, 100)


def test_meshgen_matches_reference():
    from paper_1705_01263_b200 import meshgen

    g = golden("meshes.npz")
    box = meshgen.box((0.15, 0, 0.15), (0.45, 0.3, 0.45))
    for a, k in zip(box, ("box_pos", "box_nrm", "box_uvw", "box_tris")):
        assert np.array_equal(a, g[k])
    room = meshgen.box((0, 0, 0), (1, 1, 1), inward=True)
    assert np.array_equal(room[0], g["room_pos"]) and np.array_equal(room[1], g["room_nrm"])
    assert np.array_equal(room[3], g["room_tris"])
    ico = meshgen.icosphere((0.5, -1, 2), 1.5, 3)
    for a, k in zip(ico, ("ico_pos", "ico_nrm", "ico_uvw", "ico_tris")):
        assert np.array_equal(a, g[k])


def test_cornell_flattening_matches_reference():
    from paper_1705_01263_b200 import scenes
    from paper_1705_01263_b200.geometry import flatten_instances

    g = golden("meshes.npz")
    geo = flatten_instances(scenes.cornell(), 0.0)
    assert np.array_equal(geo.verts, g["cornell_verts"])
    assert np.array_equal(geo.shading_normals, g["cornell_normals"])
    assert len(geo.verts) == 36


def test_pack_cornell():
    from paper_1705_01263_b200 import scenes
    from paper_1705_01263_b200.scene import pack_scene

    p = pack_scene(scenes.cornell())
    assert p.ntris == 36 and p.nemit == 2
    assert p.desc.env_kind == 0
    assert list(p.arrays["emit_tri"]) == [34, 35]
    assert np.allclose(p.arrays["emit_rad"], 10.0)


def test_pack_flux_emitter():
    """a diffuse emitter's flux is pi * L * A; flux given -> radiance."""
    from paper_1705_01263_b200 import meshgen
    from paper_1705_01263_b200.scene import Emitter, Environment, Instance, Mesh, Scene, diffuse_material, make_camera, pack_scene

    pos, nrm, uvw, tris = meshgen.quad((0, 0, 0), (2, 0, 0), (0, 3, 0))
    sc = Scene(make_camera((0, 0, 5)), [Mesh("q", pos, nrm, uvw, tris)], [Instance("q", 0, 0)],
               [diffuse_material("m", (0, 0, 0))], [Emitter(0, None, radiance=(1.0, 1.0, 1.0), flux=6.0 * np.pi)],
               Environment())
    p = pack_scene(sc)
    assert np.allclose(p.arrays["emit_rad"], 1.0)


def test_pfm_roundtrip(tmp_path):
    from paper_1705_01263_b200.imagefiles import read_pfm, write_pfm

    img = np.random.default_rng(0).random((7, 5, 3)).astype(np.float32)
    write_pfm(tmp_path / "a.pfm", img)
    assert np.array_equal(read_pfm(tmp_path / "a.pfm"), img)


def test_partition_iterations():
    from paper_1705_01263_b200.distributed import partition_iterations, pass_schedule

    for n in (1, 7, 16, 1024):
        for world in (1, 2, 3, 4, 8):
            blocks = [partition_iterations(10, 10 + n, r, world) for r in range(world)]
            assert blocks[0][0] == 10 and blocks[-1][1] == 10 + n
            assert all(blocks[k][1] == blocks[k + 1][0] for k in range(world - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    assert pass_schedule(10, 4) == [(0, 4), (4, 8), (8, 10)]


def test_abi_library_exports_every_header_symbol():
    """liblw_b200.so loads (no GPU needed) and exports every function include/lw_b200.h declares."""
    from paper_1705_01263_b200 import _abi

    header = open(os.path.join(ROOT, "include", "lw_b200.h")).read()
    names = set(re.findall(r"\b(lw_[a-z0-9_]+)\s*\(", header))
    lib = C.CDLL(_abi.LIB_PATH)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_abi.SIGNATURES) == names
    assert _abi.lib().lw_abi_version() == 1


def test_struct_layouts_match_header():
    """ctypes mirrors have the C layout (sizes computed by the compiler-independent rules)."""
    from paper_1705_01263_b200 import _abi

    assert C.sizeof(_abi.LwLayer) == 48
    assert C.sizeof(_abi.LwMaterial) == 8 + 4 * 48 + 8
    assert C.sizeof(_abi.LwRenderParams) == 4 * 4 + 8 * 5 + 4 * 2 + 8 + 8 + 8  # estimator (+4 padding)


def test_product_never_imports_oracle():
    """Only tests/, __graft_entry__ and bench.py may touch oracle/ (the product fails loudly instead)."""
    pkg = os.path.join(ROOT, "paper_1705_01263_b200")
    pat = re.compile(r"^\s*(from\s+oracle\b|import\s+oracle\b)|liblw_oracle|\blwo_\w+\s*\(", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                code = re.sub(r"(//|#).*", "", open(os.path.join(dirpath, f)).read())
                assert not pat.search(code), f
