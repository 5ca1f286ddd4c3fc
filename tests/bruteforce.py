"""Independent brute-force path tracer in numpy ("brute-force reference integrator
(independent straightforward implementation)").  TEST INFRASTRUCTURE ONLY.

Deliberately shares no code and no sampling scheme with the renderer or with oracle/lw_oracle.c:
pseudo-random numbers (numpy PCG64) instead of QMC, exhaustive Moller-Trumbore intersection over
every triangle instead of a BVH and watertight shear test, rejection-sampled truncated Gaussian
pixel filter instead of the inverse-CDF one, BSDF sampling only (no next-event estimation, no MIS,
no Russian roulette), cosine-weighted hemisphere sampling about the facing geometric normal.
Supports the scenes the check uses: diffuse materials (single diffuse layer, tint = albedo),
one-sided / two-sided triangle emitters, no environment.

What it shares with the renderer is only the *definition* of the measured quantity: the camera
model of DESIGN.md §4.1 (pixel centre + Gaussian filter offset, sigma 0.5 px truncated at 3 sigma),
max_depth path segments with emission added on every hit, and the scene arrays of pack_scene.
"""

from __future__ import annotations

import numpy as np


def _intersect(o, d, v0, e1, e2):
    """Closest hit of rays (o, d) [n,3] against all triangles: (t [n], tri [n]) with tri = -1 on miss."""
    n = len(o)
    best_t = np.full(n, np.inf)
    best_k = np.full(n, -1, np.int64)
    for k in range(len(v0)):  # loop over triangles, vectorised over rays
        p = np.cross(d, e2[k])
        det = p @ e1[k]
        ok = np.abs(det) > 1e-14
        inv = np.where(ok, 1.0 / np.where(ok, det, 1.0), 0.0)
        s = o - v0[k]
        u = (s * p).sum(1) * inv
        q = np.cross(s, e1[k])
        v = (d * q).sum(1) * inv
        t = (q @ e2[k]) * inv
        hit = ok & (u >= 0) & (v >= 0) & (u + v <= 1) & (t > 1e-9) & (t < best_t)
        best_t = np.where(hit, t, best_t)
        best_k = np.where(hit, k, best_k)
    return best_t, best_k


def _trunc_gauss(rng, n, sigma=0.5, cut=1.5):
    out = np.empty(n)
    filled = 0
    while filled < n:
        x = rng.normal(0.0, sigma, 2 * (n - filled) + 16)
        x = x[np.abs(x) <= cut]
        take = min(len(x), n - filled)
        out[filled:filled + take] = x[:take]
        filled += take
    return out


def render_crop(packed, width, height, x0, y0, w, h, spp, max_depth, seed=1, chunk=1 << 16):
    """Per-pixel radiance samples of the crop [x0, x0+w) x [y0, y0+h): returns (mean [h,w,3],
    sample variance of the crop-mean estimator [3], number of paths)."""
    a = packed.arrays
    d = packed.desc
    verts = np.asarray(a["verts"], np.float64).reshape(-1, 3, 3)
    v0, e1, e2 = verts[:, 0], verts[:, 1] - verts[:, 0], verts[:, 2] - verts[:, 0]
    ng = np.cross(e1, e2)
    ng /= np.linalg.norm(ng, axis=1)[:, None]
    mats = a["mats"]
    mat_of = np.asarray(a["material"], np.int64)
    albedo = np.array([[mats[m].layers[0].tint[c] * mats[m].layers[0].weight for c in range(3)]
                       if mats[m].nlayers else [0.0, 0.0, 0.0] for m in range(len(mats))])
    for m in range(len(mats)):
        assert mats[m].nlayers <= 1 and (mats[m].nlayers == 0 or mats[m].layers[0].kind == 0), "diffuse only"
    assert d.env_kind == 0, "no environment"
    emit = np.zeros((len(verts), 3))
    two = np.zeros(len(verts), bool)
    emit[np.asarray(a["emit_tri"], np.int64)] = np.asarray(a["emit_rad"], np.float64).reshape(-1, 3)
    two[np.asarray(a["emit_tri"], np.int64)] = np.asarray(a["emit_two"]) != 0
    cam_pos, fwd, right, up = (np.array(x[:3]) for x in (d.cam_pos, d.cam_fwd, d.cam_right, d.cam_up))
    tan_half = d.tan_half_fov
    aspect = width / height
    rng = np.random.default_rng(seed)
    npix = w * h
    total = npix * spp
    acc = np.zeros((npix, 3))
    crop_means = []  # per-chunk crop-mean estimates for the error bar
    done = 0
    while done < total:
        n = min(chunk, total - done)
        pid = (np.arange(done, done + n) % npix)
        px = x0 + pid % w
        py = y0 + pid // w
        sx = ((px + 0.5) + _trunc_gauss(rng, n)) / width * 2.0 - 1.0
        sy = 1.0 - ((py + 0.5) + _trunc_gauss(rng, n)) / height * 2.0
        dirs = fwd + (sx * tan_half * aspect)[:, None] * right + (sy * tan_half)[:, None] * up
        dirs /= np.linalg.norm(dirs, axis=1)[:, None]
        orig = np.repeat(cam_pos[None, :], n, axis=0)
        beta = np.ones((n, 3))
        L = np.zeros((n, 3))
        alive = np.ones(n, bool)
        for seg in range(max_depth):
            idx = np.nonzero(alive)[0]
            if len(idx) == 0:
                break
            t, k = _intersect(orig[idx], dirs[idx], v0, e1, e2)
            miss = k < 0
            alive[idx[miss]] = False
            idx, t, k = idx[~miss], t[~miss], k[~miss]
            dd = dirs[idx]
            n_g = ng[k]
            front = (n_g * dd).sum(1) < 0
            lit = front | two[k]
            L[idx] += np.where(lit[:, None], beta[idx] * emit[k], 0.0)
            if seg == max_depth - 1:
                break
            nf = np.where(front[:, None], n_g, -n_g)
            # cosine-weighted direction about nf: weight f*cos/pdf = albedo
            u1, u2 = rng.random(len(idx)), rng.random(len(idx))
            r, phi = np.sqrt(u1), 2 * np.pi * u2
            lx, ly, lz = r * np.cos(phi), r * np.sin(phi), np.sqrt(np.maximum(0.0, 1 - u1))
            helper = np.where(np.abs(nf[:, 0:1]) > 0.9, np.array([[0.0, 1.0, 0.0]]), np.array([[1.0, 0.0, 0.0]]))
            tx = np.cross(helper, nf)
            tx /= np.linalg.norm(tx, axis=1)[:, None]
            ty = np.cross(nf, tx)
            wi = lx[:, None] * tx + ly[:, None] * ty + lz[:, None] * nf
            p = orig[idx] + t[:, None] * dd
            orig[idx] = p + 1e-7 * nf
            dirs[idx] = wi
            beta[idx] *= albedo[mat_of[k]]
        np.add.at(acc, pid, L)
        crop_means.append((L.sum(0) / n))
        done += n
    mean = acc / spp
    cm = np.array(crop_means)
    # chunks hold whole multiples of the crop (chunk % npix == 0), so every chunk mean estimates the
    # crop mean without bias; their spread gives the error bar of the overall mean
    var = cm.var(axis=0, ddof=1) / len(cm)
    return mean.reshape(h, w, 3), var, total
