"""Light path expressions.

CPU: grammar errors with positions, DFA == regex semantics on every event string up to length 6
(brute force against Python's `re` on an encoded alphabet), dead-state soundness, oracle layer
routing (a partition of path space sums to the beauty image; relight linearity).
GPU: layer framebuffers bit-exact vs the oracle (megakernel engine)."""

import itertools
import re

import numpy as np
import pytest

from paper_1705_01263_b200 import scenes
from paper_1705_01263_b200.lpe import EVENTS, LpeError, compile_layers, composite, parse_lpe
from paper_1705_01263_b200.scene import pack_scene

# one character per event for Python's re: C, RD, RG, RS, TS, L, E
CH = dict(zip(EVENTS, "CdgstLE"))
SYM = {"C": "C", "L": "L", "e": "L", "E": "E", "D": "d", "G": "g", "S": "[st]", "R": "[dgs]", "T": "t",
       ".": "[dgst]"}


def _to_re(expr):
    """Independent translation of the LPE syntax to a Python regex (test oracle)."""
    out, i, s = [], 0, expr.replace(" ", "")
    while i < len(s):
        c = s[i]
        if c == "<":
            typ, mode = s[i + 1], s[i + 2]
            ts = {"R": "R", "T": "T", ".": "RT"}[typ]
            ms = {"D": "D", "G": "G", "S": "S", ".": "DGS"}[mode]
            ev = [CH[t + m] for t in ts for m in ms if t + m in CH]
            out.append("[" + "".join(ev) + "]")
            i += 4
            continue
        if c == "[":
            j = s.index("]", i)
            body = s[i + 1:j]
            neg = body.startswith("^")
            items = "".join(SYM[x].strip("[]") for x in body.lstrip("^"))
            out.append(("[^C" if neg else "[") + items + "]")
            i = j + 1
            continue
        out.append(SYM.get(c, c))
        i += 1
    return re.compile("".join(out) + r"\Z")


CORPUS = ["C.*[LE]", "CD.*L", "CS+DL", "C<R.>L", "C.*E", "C(D|G)*L", "C[^S]*E", "CL", "C<T.>+.*L",
          "C(DD|GG)?[LE]", "C.?.?L", "C[^DE]+L"]


def test_grammar_errors():
    with pytest.raises(LpeError, match="column 2"):
        parse_lpe("C(")
    for bad in ["", "DL", "C)L", "C[]L", "C<RX>L", "CQ", "C<R"]:
        with pytest.raises(LpeError):
            parse_lpe(bad)
    assert parse_lpe("C D* L") == parse_lpe("CD*L")  # whitespace is insignificant


def test_dfa_matches_regex_exhaustively():
    for exprs in (CORPUS[:8], CORPUS[8:]):
        t = compile_layers({f"l{k}": e for k, e in enumerate(exprs)})
        rx = [_to_re(e) for e in exprs]
        for n in range(0, 6):
            for tail in itertools.product(EVENTS[1:], repeat=n):
                evs = ["C", *tail]
                st = t.run(evs)
                text = "".join(CH[e] for e in evs)
                want = {name for name, r in zip(t.names, rx) if r.match(text)}
                assert set(t.layers_of(st)) == want, (evs, want)


def test_dead_state_is_absorbing_and_sound():
    t = compile_layers({"a": "CDL", "b": "CSL"})
    st = t.run(["C", "RG"])  # C then G is dead for {CDL, CSL}
    assert t.dead[st]
    for e in EVENTS:
        assert t.trans[st, EVENTS.index(e)] == st


def test_oracle_layers_partition_beauty(oracle):
    from paper_1705_01263_b200.render import RenderParams

    sc = scenes.envmap_scene(256, 128, sphere_subdiv=3)
    packed = pack_scene(sc)
    t = compile_layers({"diffuse": "CD.*[LE]", "glossy": "CG.*[LE]", "specular": "CS.*[LE]", "direct": "C[LE]"})
    prm = RenderParams(48, 27, 6)
    fb, layers, _ = oracle.OracleScene(packed).render_lpe(prm, 0, 4, t)
    fb0, _ = oracle.OracleScene(packed).render(prm, 0, 4)
    assert np.array_equal(fb, fb0)  # the beauty is untouched by layer routing
    total = sum(v.astype(np.float64) for v in layers.values())
    rel = np.abs(total - fb).max() / max(1.0, np.abs(fb).max())
    assert rel < 1e-5, rel  # per-contribution vs per-path rounding only
    assert all(layers[k].sum() > 0 for k in ("diffuse", "glossy", "direct"))  # the scene has no specular BSDF
    img = composite({k: v.astype(np.float64) for k, v in layers.items()})
    assert np.allclose(img, total)


@pytest.mark.gpu
@pytest.mark.parametrize("which,engine", [("cornell", "megakernel"), ("env", "megakernel"), ("cornell", "wavefront"),
                                          ("env", "wavefront")])
def test_gpu_lpe_layers_bit_exact(gpu, oracle, which, engine):
    from paper_1705_01263_b200.render import Renderer, RenderParams

    if which == "cornell":
        packed, depth = pack_scene(scenes.cornell()), 6
    else:
        packed, depth = pack_scene(scenes.envmap_scene(256, 128, sphere_subdiv=3), lights="alias"), 8
    layers = {"beauty": "C.*[LE]", "diffuse": "CD.*[LE]", "caustic": "C[GS]+D.*L", "direct": "C.?[LE]",
              "env": "C.*E"}
    W, H = 64, 48
    with Renderer(None, W, H, depth, packed=packed, engine=engine, pool_log2=12) as r:
        t = r.set_lpe_layers(layers)
        r.render_pass(0, 4)
        fb = r.framebuffer()
        got = r.layer_framebuffers()
    fb2, want, _ = oracle.OracleScene(packed).render_lpe(RenderParams(W, H, depth), 0, 4, t)
    assert np.array_equal(fb, fb2)
    for k in layers:
        assert np.array_equal(got[k], want[k]), k
    assert got["beauty"].sum() > 0


@pytest.mark.gpu
def test_cli_layers_and_composite(gpu, tmp_path):
    from paper_1705_01263_b200 import cli
    from paper_1705_01263_b200.imagefiles import read_pfm

    out = str(tmp_path / "c1")
    assert cli.main(["render", "--config", "C1", "--res", "32x32", "--iterations", "4", "--out", out,
                     "--layer", "direct=C.?L", "--layer", "indirect=C..+L"]) == 0
    d, i = read_pfm(out + "_direct_000004.pfm"), read_pfm(out + "_indirect_000004.pfm")
    assert d.sum() > 0 and i.sum() > 0
    comp = str(tmp_path / "sum.pfm")
    assert cli.main(["composite", "--layers", out + "_direct_000004.pfm", out + "_indirect_000004.pfm",
                     "--out", comp]) == 0
    beauty = read_pfm(out + "_000004.pfm").astype(np.float64)
    assert np.abs(read_pfm(comp) - beauty).max() <= 1e-4 * max(1.0, beauty.max())
    assert cli.main(["render", "--config", "C1", "--res", "8x8", "--iterations", "1", "--out", out,
                     "--layer", "bad=C("]) == 2
