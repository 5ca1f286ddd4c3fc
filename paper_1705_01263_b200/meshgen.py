"""Procedural triangle meshes (same outputs as the reference's `lumenwave.meshgen`).

Each generator returns (positions, normals, uvw, triangles).  Vertex and
triangle order match `meshgen.py:10-108` exactly, because triangle ids are
part of the parity contract (hit IDs are compared bit for bit).
"""

from __future__ import annotations

import numpy as np

__all__ = ["quad", "box", "icosphere"]

_QUAD_UVW = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], dtype=np.float64)
_QUAD_TRIS = np.array([[0, 1, 2], [0, 2, 3]], dtype=np.int64)


def _unit(v):
    return v / np.linalg.norm(v)


def quad(corner, edge_u, edge_v):
    """corner + [0,1]^2 spanned by (edge_u, edge_v), as two triangles (meshgen.py:10-21)."""
    c = np.asarray(corner, dtype=np.float64)
    eu = np.asarray(edge_u, dtype=np.float64)
    ev = np.asarray(edge_v, dtype=np.float64)
    pos = np.array([c, c + eu, c + eu + ev, c + ev])
    nrm = np.repeat(_unit(np.cross(eu, ev))[None, :], 4, axis=0)
    return pos, nrm, _QUAD_UVW.copy(), _QUAD_TRIS.copy()


def box(lo, hi, inward: bool = False):
    """Axis-aligned box, 12 triangles, faces ordered -x,+x,-y,+y,-z,+z (meshgen.py:24-60)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    ext = hi - lo
    pos, nrm, uvw, tris = [], [], [], []
    for face in range(6):
        axis, positive = divmod(face, 2)
        a1, a2 = (axis + 1) % 3, (axis + 2) % 3
        origin = lo.copy()
        if positive:
            origin[axis] = hi[axis]
        e1 = np.zeros(3)
        e2 = np.zeros(3)
        e1[a1] = ext[a1]
        e2[a2] = ext[a2]
        # the low face swaps the spanning edges to keep outward winding; `inward` swaps back
        if (not positive) != bool(inward):
            e1, e2 = e2, e1
        base = 4 * face
        pos += [origin, origin + e1, origin + e1 + e2, origin + e2]
        nrm += [_unit(np.cross(e1, e2))] * 4
        uvw.append(_QUAD_UVW)
        tris.append(_QUAD_TRIS + base)
    return (np.asarray(pos, dtype=np.float64), np.asarray(nrm, dtype=np.float64),
            np.concatenate(uvw).astype(np.float64), np.concatenate(tris).astype(np.int64))


_PHI = (1.0 + np.sqrt(5.0)) / 2.0
_ICO_FACES = [
    (0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
    (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
    (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
    (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1),
]


def _icosahedron():
    t = _PHI
    v = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0],
                  [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
                  [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], dtype=np.float64)
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def icosphere(center, radius, subdivisions: int = 3):
    """Geodesic sphere by midpoint subdivision with smooth normals (meshgen.py:63-108)."""
    verts = [tuple(p) for p in _icosahedron()]
    faces = list(_ICO_FACES)
    for _ in range(subdivisions):
        mids = {}

        def mid(i, j):
            key = (i, j) if i < j else (j, i)
            k = mids.get(key)
            if k is None:
                m = np.asarray(verts[i]) + np.asarray(verts[j])
                m /= np.linalg.norm(m)
                k = len(verts)
                mids[key] = k
                verts.append(tuple(m))
            return k

        refined = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            refined.extend([(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)])
        faces = refined
    unit = np.asarray(verts, dtype=np.float64)
    positions = np.asarray(center, dtype=np.float64) + radius * unit
    theta = np.arccos(np.clip(unit[:, 2], -1, 1))
    phi = np.mod(np.arctan2(unit[:, 1], unit[:, 0]), 2 * np.pi)
    uvw = np.stack([phi / (2 * np.pi), theta / np.pi, np.zeros(len(unit))], axis=1)
    return positions, unit.copy(), uvw, np.asarray(faces, dtype=np.int64)
