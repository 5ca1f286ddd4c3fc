"""Light path expressions (§4.1).

A path is the event string C e1 e2 ... ek X: the camera, one event per scattering vertex (the
sampled lobe: RD diffuse reflection, RG glossy reflection, RS specular reflection, TS specular
transmission) and a terminal X = L (emissive triangle, hit or sampled by NEE) or E
(environment).  An NEE contribution at vertex k is split by lobe: its diffuse and glossy parts
carry the events RD L / RG L (or E).  Each output layer is a regular expression over these
events; a contribution is routed to every layer whose expression matches its event string.

Concrete syntax (normative here; SPEC.md:744 DESIGN DECISIONS):
    C L E        camera, light (emissive geometry; `e` is accepted as a synonym), environment
    D G S        diffuse / glossy reflection, specular (reflection or transmission)
    R T          any reflection / the (specular) transmission
    <XY>         detailed symbol: X in R T . (type), Y in D G S . (mode), e.g. <RD>, <T.>, <.S>
    .            any scattering event (not C, L, E)
    [..] [^..]   class / complemented class of single-event symbols (complement within . L E)
    |  *  +  ?  ( )   alternation, repetition, grouping; whitespace is ignored
Expressions are anchored: they must start with C, and a match covers the whole event string.

compile_layers() builds one DFA per expression (Thompson NFA + subset construction), then the
product automaton over all layers with a dense transition table (state x 7 events), a per-state
accepting-layer bit mask and the dead state (no layer can accept any more).  Tables are uploaded
with Renderer.set_lpe_layers(); the device and the oracle advance a 16-bit state per path.
"""

from __future__ import annotations

import numpy as np

EVENTS = ["C", "RD", "RG", "RS", "TS", "L", "E"]
EV = {e: k for k, e in enumerate(EVENTS)}
SCATTER = {EV["RD"], EV["RG"], EV["RS"], EV["TS"]}
MAX_STATES = 4096
MAX_LAYERS = 8


class LpeError(ValueError):
    def __init__(self, msg, pos):
        super().__init__(f"{msg} at column {pos + 1}")
        self.pos = pos


# ---- parser -> tree of ("set", frozenset) / ("cat", a, b) / ("alt", a, b) / ("star"|"plus"|"opt", a)

_SINGLE = {
    "C": {EV["C"]}, "L": {EV["L"]}, "e": {EV["L"]}, "E": {EV["E"]},
    "D": {EV["RD"]}, "G": {EV["RG"]}, "S": {EV["RS"], EV["TS"]},
    "R": {EV["RD"], EV["RG"], EV["RS"]}, "T": {EV["TS"]}, ".": set(SCATTER),
}


def _detailed(typ, mode, pos):
    types = {"R": {"R"}, "T": {"T"}, ".": {"R", "T"}}
    modes = {"D": {"D"}, "G": {"G"}, "S": {"S"}, ".": {"D", "G", "S"}}
    if typ not in types or mode not in modes:
        raise LpeError(f"bad detailed symbol <{typ}{mode}>", pos)
    return {EV[t + m] for t in types[typ] for m in modes[mode] if t + m in EV}


class _Parser:
    def __init__(self, text):
        self.s = text
        self.toks = [(c, k) for k, c in enumerate(text) if not c.isspace()]
        self.i = 0

    def peek(self):
        return self.toks[self.i][0] if self.i < len(self.toks) else None

    def pos(self):
        return self.toks[self.i][1] if self.i < len(self.toks) else len(self.s)

    def take(self):
        t = self.toks[self.i]
        self.i += 1
        return t

    def parse(self):
        if not self.toks:
            raise LpeError("empty expression", 0)
        if self.peek() != "C":
            raise LpeError("expression must start with C (camera)", self.pos())
        t = self.alt()
        if self.i != len(self.toks):
            c, p = self.toks[self.i]
            raise LpeError("unbalanced ')'" if c == ")" else f"unexpected '{c}'", p)
        return t

    def alt(self):
        t = self.cat()
        while self.peek() == "|":
            self.take()
            t = ("alt", t, self.cat())
        return t

    def cat(self):
        items = []
        while self.peek() not in (None, "|", ")"):
            items.append(self.post())
        if not items:
            raise LpeError("empty alternative", self.pos())
        t = items[0]
        for x in items[1:]:
            t = ("cat", t, x)
        return t

    def post(self):
        t = self.atom()
        while self.peek() in ("*", "+", "?"):
            op = self.take()[0]
            t = ({"*": "star", "+": "plus", "?": "opt"}[op], t)
        return t

    def atom(self):
        c, p = self.take()
        if c == "(":
            if self.peek() is None:
                raise LpeError("unbalanced '('", p)
            t = self.alt()
            if self.peek() != ")":
                raise LpeError("unbalanced '('", p)
            self.take()
            return t
        if c == "[":
            neg = self.peek() == "^"
            if neg:
                self.take()
            s = set()
            while self.peek() not in (None, "]"):
                s |= self.symbol()
            if self.peek() != "]":
                raise LpeError("unterminated class", p)
            self.take()
            if neg:
                s = (set(SCATTER) | {EV["L"], EV["E"]}) - s
            if not s:
                raise LpeError("empty class", p)
            return ("set", frozenset(s))
        self.i -= 1
        return ("set", frozenset(self.symbol()))

    def symbol(self):
        c, p = self.take()
        if c == "<":
            if self.i + 3 > len(self.toks):
                raise LpeError("unterminated '<'", p)
            typ = self.take()[0]
            mode = self.take()[0]
            if self.peek() != ">":
                raise LpeError("unterminated '<'", p)
            self.take()
            return _detailed(typ, mode, p)
        if c in _SINGLE:
            return set(_SINGLE[c])
        raise LpeError(f"unknown symbol '{c}'", p)


def parse_lpe(text: str):
    return _Parser(text).parse()


# ---- Thompson NFA -> DFA

def _nfa(tree):
    trans = []   # state -> list of (eventset or None for epsilon, target)

    def new():
        trans.append([])
        return len(trans) - 1

    def build(t):
        kind = t[0]
        if kind == "set":
            a, b = new(), new()
            trans[a].append((t[1], b))
            return a, b
        if kind == "cat":
            a1, b1 = build(t[1])
            a2, b2 = build(t[2])
            trans[b1].append((None, a2))
            return a1, b2
        if kind == "alt":
            a, b = new(), new()
            for sub in (t[1], t[2]):
                s, e = build(sub)
                trans[a].append((None, s))
                trans[e].append((None, b))
            return a, b
        a, b = new(), new()
        s, e = build(t[1])
        trans[a].append((None, s))
        trans[e].append((None, b))
        if kind in ("star", "opt"):
            trans[a].append((None, b))
        if kind in ("star", "plus"):
            trans[e].append((None, s))
        return a, b

    start, accept = build(tree)
    return trans, start, accept


def _closure(trans, states):
    out, stack = set(states), list(states)
    while stack:
        s = stack.pop()
        for ev, t in trans[s]:
            if ev is None and t not in out:
                out.add(t)
                stack.append(t)
    return frozenset(out)


def _dfa(tree):
    trans, start, accept = _nfa(tree)
    s0 = _closure(trans, {start})
    ids, order, table, acc = {s0: 0}, [s0], [], []
    k = 0
    while k < len(order):
        cur = order[k]
        row = []
        for ev in range(len(EVENTS)):
            nxt = _closure(trans, {t for s in cur for e, t in trans[s] if e is not None and ev in e})
            if nxt not in ids:
                ids[nxt] = len(order)
                order.append(nxt)
            row.append(ids[nxt])
        table.append(row)
        acc.append(accept in cur)
        k += 1
    return np.array(table, np.int32), np.array(acc, bool)


class LpeTables:
    """Product automaton of all layers: trans[state, event], accept bit mask per state."""

    def __init__(self, names, trans, accept, start, dead):
        self.names, self.trans, self.accept, self.start, self.dead = names, trans, accept, start, dead

    def run(self, events):
        s = self.start
        for e in events:
            s = int(self.trans[s, EV[e] if isinstance(e, str) else e])
        return s

    def layers_of(self, state):
        m = int(self.accept[state])
        return [n for k, n in enumerate(self.names) if m >> k & 1]


def compile_layers(layers: dict) -> LpeTables:
    """layers: {name: expression} (at most MAX_LAYERS)."""
    if not 1 <= len(layers) <= MAX_LAYERS:
        raise ValueError(f"1..{MAX_LAYERS} LPE layers supported")
    names = list(layers)
    dfas = [_dfa(parse_lpe(layers[n])) for n in names]
    # live[k][s]: can layer k's DFA still reach an accepting state from s
    lives = []
    for tab, acc in dfas:
        live = acc.copy()
        changed = True
        while changed:
            changed = False
            for s in range(len(tab)):
                if not live[s] and live[tab[s]].any():
                    live[s] = changed = True
        lives.append(live)
    start = tuple(0 for _ in dfas)
    ids, order, rows = {start: 0}, [start], []
    k = 0
    while k < len(order):
        cur = order[k]
        row = []
        for ev in range(len(EVENTS)):
            nxt = tuple(int(d[0][s, ev]) for d, s in zip(dfas, cur))
            if nxt not in ids:
                ids[nxt] = len(order)
                order.append(nxt)
                if len(order) > MAX_STATES:
                    raise ValueError("LPE automaton too large")
            row.append(ids[nxt])
        rows.append(row)
        k += 1
    trans = np.array(rows, np.int16)
    accept = np.array([sum(1 << j for j, (d, s) in enumerate(zip(dfas, st)) if d[1][s]) for st in order], np.uint8)
    dead = np.array([not any(lv[s] for lv, s in zip(lives, st)) for st in order], bool)
    return LpeTables(names, trans, accept, 0, dead)


def composite(layers: dict, gains: dict | None = None) -> np.ndarray:
    """Linear recombination of layer images: sum of gain * layer."""
    gains = gains or {}
    out = None
    for name, img in layers.items():
        g = np.asarray(gains.get(name, 1.0), np.float64)
        v = np.asarray(img, np.float64) * g
        out = v if out is None else out + v
    return out
