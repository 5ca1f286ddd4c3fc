"""Write a D1/D2-corrected variant of the reference kernel module into oracle/_ref/.

TEST INFRASTRUCTURE ONLY (run by oracle/Makefile; output is git-ignored).
It reads /root/reference/pkg/src/lumenwave/core/_kernels.py and applies the two
fixes named in SURVEY.md §0:

  D1 (_kernels.py:378-386, call at 540): `_tri_hit` subtracts the unpermuted
     origin (ox, oy, oz) from permuted vertex components; the fix passes
     (o[kx], o[ky], o[kz]).
  D2 (_kernels.py:479-533): a zero direction component gets inv = +-1e200 and
     a ray lying on a box max face computes 0*1e200 = 0 and is culled; the fix
     tests o in [bmin, bmax] for such axes instead of the slab product.

The result is the "corrected" reference that LW_TRAVERSE_CORRECTED must match
bit for bit.  Usage: python patch_ref_d1d2.py <src _kernels.py> <dst _kernels.py>
"""

import sys

SLAB_START = "        # AABB slab test against current best distance\n"
SLAB_END = "        if tn > tf or tn > res[0] or tf < tmin:\n"
CALL_OLD = "_tri_hit(verts, order[start + i], ox, oy, oz, kx, ky, kz, sx, sy, sz, tmin, res)"
CALL_NEW = (
    "_tri_hit(verts, order[start + i], "
    "(ox if kx == 0 else (oy if kx == 1 else oz)), "
    "(ox if ky == 0 else (oy if ky == 1 else oz)), "
    "(ox if kz == 0 else (oy if kz == 1 else oz)), "
    "kx, ky, kz, sx, sy, sz, tmin, res)"
)


def _axis_block(lo, hi, o, inv):
    # c0 doubles as the cull flag: it is a declared longlong that is
    # reassigned from `children` right after the slab test.
    return (
        f"        if {inv} == 1e200 or {inv} == -1e200:\n"
        f"            if {o} < bounds[node, {lo}] or {o} > bounds[node, {hi}]:\n"
        f"                c0 = 1\n"
        f"        else:\n"
        f"            t0 = (bounds[node, {lo}] - {o}) * {inv}\n"
        f"            t1 = (bounds[node, {hi}] - {o}) * {inv}\n"
        f"            if t0 > t1:\n"
        f"                if t0 < tf:\n"
        f"                    tf = t0\n"
        f"                if t1 > tn:\n"
        f"                    tn = t1\n"
        f"            else:\n"
        f"                if t1 < tf:\n"
        f"                    tf = t1\n"
        f"                if t0 > tn:\n"
        f"                    tn = t0\n"
    )


def main(src, dst):
    text = open(src).read()
    a = text.index(SLAB_START)
    b = text.index(SLAB_END)
    slab = (
        "        # slab test, D2-corrected (zero-direction axes test containment)\n"
        "        c0 = 0\n"
        "        tn = -1e308 * 10.0\n"
        "        tf = 1e308 * 10.0\n"
        + _axis_block(0, 3, "ox", "ix")
        + _axis_block(1, 4, "oy", "iy")
        + _axis_block(2, 5, "oz", "iz")
        + "        if c0 == 1:\n"
        "            continue\n"
    )
    text = text[:a] + slab + text[b:]
    assert text.count(CALL_OLD) == 1
    text = text.replace(CALL_OLD, CALL_NEW)
    open(dst, "w").write(text)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
