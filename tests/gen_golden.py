"""Generate golden vectors from the reference (run in the build container, where /root/reference exists).

    python tests/gen_golden.py

Writes tests/golden/*.npz.  Every array comes from the reference's own code:
  - lumenwave.qmc (DimensionTable, radical_inverse) imported from /root/reference/pkg/src,
  - the reference kernel module compiled from its source by oracle/Makefile
    (oracle/_ref/pristine) and its D1/D2-patched variant (oracle/_ref/corrected),
  - lumenwave.geometry.build_bvh / flatten_instances, lumenwave.meshgen.
The GPU box has no /root/reference; tests read only these committed fixtures.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from lumenwave import geometry as rgeo  # noqa: E402
from lumenwave import meshgen as rmesh  # noqa: E402
from lumenwave import qmc as rqmc  # noqa: E402

from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, name), **arrays)
    print(name, {k: v.shape for k, v in arrays.items()})


def soup_verts(n, seed):
    rng = np.random.default_rng(seed)
    base = rng.random((n, 3)) * 20
    e1 = rng.normal(size=(n, 3)) * 0.3
    e2 = rng.normal(size=(n, 3)) * 0.3
    return np.ascontiguousarray(np.concatenate([base, base + e1, base + e2], axis=1))


def mesh_verts(pos, tris):
    return np.ascontiguousarray(np.concatenate([pos[tris[:, 0]], pos[tris[:, 1]], pos[tris[:, 2]]], axis=1))


def main():
    pr = O.ref_kernels("pristine")
    cr = O.ref_kernels("corrected")
    if pr is None or cr is None:
        sys.exit("build the reference kernels first: make -C oracle ref")
    # 1. dimension tables (qmc.py:274-305)
    tabs = {}
    for d in (4, 8, 12):
        t = rqmc.DimensionTable(d)
        for k in ("bases", "perm_flat", "perm_offset", "magic", "shift", "add"):
            tabs[f"d{d}_{k}"] = np.asarray(getattr(t, k))
    save("qmc_tables.npz", **tabs)

    # 2. Halton points, every dimension of DimensionTable(8), from the reference kernel;
    #    the exact API agrees on every index < 2^53 / base (checked here)
    rng = np.random.default_rng(20240601)
    t = rqmc.DimensionTable(8)
    idx = np.unique(np.concatenate([
        np.arange(0, 257), rng.integers(0, 2**30, 96), rng.integers(0, 2**40, 96), rng.integers(2**40, 2**53, 32),
        [2**31 - 1, 2**31, 2**32 - 1, 2**32, 2**32 + 1, 2**40, 3**19, 3**19 - 1, 5**13, 2**53 - 1],
    ]).astype(np.int64))
    big = np.array([2**53, 2**53 + 1, 2**60 + 12345, 2**63 - 1], dtype=np.int64)
    vals = np.zeros((t.ndims, len(idx)))
    vals_big = np.zeros((t.ndims, len(big)))
    for dim in range(t.ndims):
        pr.halton_batch(t.bases, t.perm_flat, t.perm_offset, dim, idx, vals[dim])
        pr.halton_batch(t.bases, t.perm_flat, t.perm_offset, dim, big, vals_big[dim])
        b = int(t.bases[dim])
        for k, i in enumerate(idx.tolist()):
            if b * i < 2**53:
                assert vals[dim, k] == rqmc.radical_inverse(b, i)
    save("halton.npz", indices=idx, values=vals, big_indices=big, big_values=vals_big)

    # 3. pixel filter (_kernels.py:121-134), tails included
    u = np.concatenate([rng.random(4000), np.linspace(0, 0.03, 600), np.linspace(0.97, 1.0, 600),
                        [0.0, 0.5, 1.0, 1e-300, 0.02296, 0.97704, 1 - 2**-53]])
    u = u[: len(u) // 2 * 2].reshape(-1, 2)
    off = np.array([pr.sample_pixel_offset(a, b) for a, b in u])
    save("pixel_offset.npz", u=u, offsets=off)

    # 4. octahedral compression (_kernels.py:233-342)
    vecs = rng.normal(size=(3000, 3))
    vecs /= np.linalg.norm(vecs, axis=1, keepdims=True)
    axes = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1], [0, 0, 0.0]])
    vecs = np.concatenate([vecs, axes])
    rt = np.full_like(vecs, -7.0)
    pr.oct_roundtrip_batch(vecs, rt)
    enc = np.array([pr.compress_unit_vector(*v) if np.any(v) else -1 for v in vecs], dtype=np.int64)
    dec = np.array([pr.decompress_unit_vector(int(p)) if p >= 0 else (0.0, 0.0, 1.0) for p in enc])
    save("oct.npz", vecs=vecs, roundtrip=rt, encoded=enc, decoded=dec)

    # 5. BVH builds (geometry.py:100-148) + 6. traversal (both semantics) on the same sets
    sets = {
        "tri1": rng.random((1, 9)),
        "tri4": rng.random((4, 9)),
        "tri5": rng.random((5, 9)),
        "rand200": rng.random((200, 9)) * 3,
        "cornellbox": mesh_verts(*[rmesh.box((0, 0, 0), (1, 1, 1), inward=True)[i] for i in (0, 3)]),
        "ico2": mesh_verts(*[rmesh.icosphere((0, 0, 0), 1.0, 2)[i] for i in (0, 3)]),
        "soup5k": soup_verts(5000, 5),
        "quad": mesh_verts(*[rmesh.quad((0, 0, 0), (1, 0, 0), (0, 1, 0))[i] for i in (0, 3)]),
        "coincident": np.array([[0, 0, 0, 1, 0, 0, 0, 1, 0], [0, 0, 0, 1, 0, 0, 0, 1, 0.0]]),
    }
    out = {}
    for name, verts in sets.items():
        verts = np.ascontiguousarray(verts, dtype=np.float64)
        b, c, o = rgeo.build_bvh(verts)
        out[f"{name}_verts"] = verts
        out[f"{name}_bounds"] = b
        out[f"{name}_children"] = c
        out[f"{name}_order"] = o
        lo, hi = verts.reshape(-1, 3).min(0), verts.reshape(-1, 3).max(0)
        n = 1500
        orig = lo - 0.5 + rng.random((n, 3)) * (hi - lo + 1.0)
        tgt = verts.reshape(-1, 3, 3)[rng.integers(0, len(verts), n)]
        w = rng.random((n, 3))
        w /= w.sum(1, keepdims=True)
        dirs = np.einsum("nk,nkj->nj", w, tgt) - orig
        dirs[: n // 10] = rng.normal(size=(n // 10, 3))
        dirs[n // 10: n // 10 + 40, 0] = 0.0  # zero direction components (D2 territory)
        dirs[n // 10 + 40: n // 10 + 80, :2] = 0.0
        dirs[(np.linalg.norm(dirs, axis=1) == 0)] = [0.0, 0.0, 1.0]
        tmax = np.where(rng.random(n) < 0.2, rng.random(n) * 5, np.inf)
        out[f"{name}_origins"] = orig
        out[f"{name}_dirs"] = dirs
        out[f"{name}_tmax"] = tmax
        for tag, mod in (("compat", pr), ("corrected", cr)):
            ot = np.empty(n)
            otri = np.empty(n, np.int64)
            ob = np.empty((n, 2))
            mod.intersect_batch(b, c, o, verts, np.zeros(len(verts), np.int64), orig, dirs, tmax, ot, otri, ob)
            out[f"{name}_{tag}_t"] = ot
            out[f"{name}_{tag}_tri"] = otri
            out[f"{name}_{tag}_bary"] = ob
    out["names"] = np.array(list(sets))
    save("bvh_traversal.npz", **out)

    # 7. meshgen + instance flattening of the Cornell config
    from paper_1705_01263_b200 import scenes

    sc = scenes.cornell()
    geo = rgeo.flatten_instances(sc, 0.0)
    box = rmesh.box((0.15, 0, 0.15), (0.45, 0.3, 0.45))
    room = rmesh.box((0, 0, 0), (1, 1, 1), inward=True)
    ico = rmesh.icosphere((0.5, -1, 2), 1.5, 3)
    save("meshes.npz", cornell_verts=geo.verts, cornell_normals=geo.shading_normals,
         box_pos=box[0], box_nrm=box[1], box_uvw=box[2], box_tris=box[3],
         room_pos=room[0], room_nrm=room[1], room_tris=room[3],
         ico_pos=ico[0], ico_nrm=ico[1], ico_uvw=ico[2], ico_tris=ico[3])


if __name__ == "__main__":
    main()
