"""Seeded synthetic netlist generators (INPUT ONLY).

This module is the one thing the oracle (``oracle/``) and the CUDA path
(``paper_2604_03079_b200``) share: it draws topologies, device sizes, model
cards and node voltages from ``numpy.random.Generator(PCG64(seed))`` and holds
none of the method's arithmetic (no device equations, no stamping, no pattern,
no colouring).  The recipe of every config is stated in DESIGN.md §3 and follows
SURVEY.md §8(d) / BASELINE.json ``configs``.

Conventions ("ground excluded, dense ids"):
  * node ids are ``0 .. n_nodes-1``; ground is ``-1``;
  * unknowns ``n = n_nodes + n_extra`` (source branches after nodes);
  * terminals are ``d, g, s, b`` (drain, gate, source, bulk);
  * ``vprev[3][N]`` = (v_gs, v_gd, v_db) of the last accepted step, formed as
    differences of a seeded ``x_prev``;
  * draw order: topology -> polarity -> W -> L -> x -> x_prev.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List

import numpy as np

UM = 1e-6
H_DEFAULT = 1e-12          # h = 1 ps (BASELINE.json configs[0])
VDD_VOLTS = 1.0            # rails at 1.0 V


@dataclasses.dataclass
class Netlist:
    name: str
    n_nodes: int
    n_extra: int
    d: np.ndarray            # int32 [N]
    g: np.ndarray
    s: np.ndarray
    b: np.ndarray
    w: np.ndarray            # float64 [N], metres
    l: np.ndarray            # float64 [N], metres
    model: np.ndarray        # int32 [N]
    models: List[Dict]       # cards: polarity, vt0, kp, lam, cgs, cgd, cdb
    rails: np.ndarray        # int32 [R] nodes held by ideal sources
    extra_row: np.ndarray    # int32 caller-owned linear entries (V-source branch)
    extra_col: np.ndarray
    x: np.ndarray            # float64 [n] current NR iterate
    x_prev: np.ndarray       # float64 [n] last accepted step
    vprev: np.ndarray        # float64 [3, N] (v_gs, v_gd, v_db) at x_prev
    h: float = H_DEFAULT
    gmin: float = 1e-12
    meta: Dict = dataclasses.field(default_factory=dict)

    @property
    def n_dev(self) -> int:
        return int(self.d.shape[0])

    @property
    def n(self) -> int:
        return self.n_nodes + self.n_extra


# --------------------------------------------------------------------------
# model cards (SPEC S:39-41 ModelCard; S:199 example; SURVEY A4 bench card)
# --------------------------------------------------------------------------
def bench_models() -> List[Dict]:
    """SURVEY A4 bench card: kp=2e-5 A/V^2, C=1 fF, |vt0|=0.3 V,
    lambda=0.05 1/V so cutoff/triode/saturation and both modes all occur."""
    c = 1e-15
    return [
        dict(polarity=+1, vt0=+0.3, kp=2e-5, lam=0.05, cgs=c, cgd=c, cdb=c),
        dict(polarity=-1, vt0=-0.3, kp=2e-5, lam=0.05, cgs=c, cgd=c, cdb=c),
    ]


def spec_models() -> List[Dict]:
    """SPEC S:56/S:199 example card (vt0=1, kp=2e-5, lambda=0) and its PMOS
    mirror (SPICE sign convention vt0<0); caps 1 fF."""
    c = 1e-15
    return [
        dict(polarity=+1, vt0=+1.0, kp=2e-5, lam=0.0, cgs=c, cgd=c, cdb=c),
        dict(polarity=-1, vt0=-1.0, kp=2e-5, lam=0.0, cgs=c, cgd=c, cdb=c),
    ]


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _voltages(rng, n_nodes, n_extra, rails):
    n = n_nodes + n_extra
    x = np.zeros(n)
    x[:n_nodes] = rng.uniform(0.0, 1.0, n_nodes)
    xp = np.zeros(n)
    xp[:n_nodes] = rng.uniform(0.0, 1.0, n_nodes)
    if len(rails):
        x[rails] = VDD_VOLTS
        xp[rails] = VDD_VOLTS
    return x, xp


def _vprev(xp, d, g, s, b):
    def v(t):
        out = np.zeros(t.shape[0])
        m = t >= 0
        out[m] = xp[t[m]]
        return out
    vd, vg, vs, vb = v(d), v(g), v(s), v(b)
    return np.stack([vg - vs, vg - vd, vd - vb])


def _finish(name, n_nodes, n_extra, d, g, s, b, w, l, model, models, rails,
            extra_row, extra_col, rng, meta, h=H_DEFAULT):
    d = np.ascontiguousarray(d, dtype=np.int32)
    g = np.ascontiguousarray(g, dtype=np.int32)
    s = np.ascontiguousarray(s, dtype=np.int32)
    b = np.ascontiguousarray(b, dtype=np.int32)
    rails = np.ascontiguousarray(rails, dtype=np.int32)
    x, xp = _voltages(rng, n_nodes, n_extra, rails)
    return Netlist(
        name=name, n_nodes=int(n_nodes), n_extra=int(n_extra), d=d, g=g, s=s, b=b,
        w=np.ascontiguousarray(w, dtype=np.float64),
        l=np.ascontiguousarray(l, dtype=np.float64),
        model=np.ascontiguousarray(model, dtype=np.int32), models=models,
        rails=rails,
        extra_row=np.ascontiguousarray(extra_row, dtype=np.int32),
        extra_col=np.ascontiguousarray(extra_col, dtype=np.int32),
        x=x, x_prev=xp, vprev=np.ascontiguousarray(_vprev(xp, d, g, s, b)),
        h=h, meta=meta)


def _vdd_branch(vdd, br):
    """V-source branch entries A[VDD,br], A[br,VDD] (linear pre-pass
    entries owned by the caller)."""
    return np.array([vdd, br], np.int32), np.array([br, vdd], np.int32)


def _inverters(inp, out, vdd):
    """CMOS inverters, device order per stage N then P; NMOS bulk to GND,
    PMOS source+bulk to VDD (BASELINE configs[0])."""
    k = inp.shape[0]
    d = np.empty(2 * k, np.int64); g = np.empty(2 * k, np.int64)
    s = np.empty(2 * k, np.int64); b = np.empty(2 * k, np.int64)
    d[0::2] = out; g[0::2] = inp; s[0::2] = -1; b[0::2] = -1
    d[1::2] = out; g[1::2] = inp; s[1::2] = vdd; b[1::2] = vdd
    model = np.tile(np.array([0, 1], np.int32), k)
    return d, g, s, b, model


def _wl_uniform(rng, n):
    w = rng.uniform(0.2, 5.0, n) * UM      # BASELINE configs[0]: W U[0.2,5] um
    l = rng.uniform(0.05, 0.5, n) * UM     # L U[0.05,0.5] um
    return w, l


# --------------------------------------------------------------------------
# the five BASELINE configs
# --------------------------------------------------------------------------
def inverter_chain(stages: int = 1000, seed: int = 0, models=None) -> Netlist:
    """configs[0]: chain of CMOS inverters; nodes o0..o_stages, VDD, branch."""
    rng = _rng(seed)
    inp = np.arange(stages); out = inp + 1
    vdd = stages + 1
    d, g, s, b, model = _inverters(inp, out, vdd)
    w, l = _wl_uniform(rng, d.shape[0])
    er, ec = _vdd_branch(vdd, vdd + 1)
    return _finish(f"chain{stages}", stages + 2, 1, d, g, s, b, w, l, model,
                   models or bench_models(), [vdd], er, ec, rng,
                   dict(config=0, stages=stages))


def ring_oscillators(rings: int = 1000, stages: int = 101, seed: int = 1,
                     fanout: int = 0, models=None) -> Netlist:
    """configs[1]: `rings` independent `stages`-stage rings sharing VDD.
    node id = ring*stages + stage.  fanout>0 adds the B1b variant (SURVEY
    A10): each stage output drives `fanout` extra inverters with private
    outputs, placed right after the driving stage in netlist order."""
    rng = _rng(seed)
    r = np.repeat(np.arange(rings), stages)
    k = np.tile(np.arange(stages), rings)
    inp = r * stages + k
    out = r * stages + (k + 1) % stages
    n_ring_nodes = rings * stages
    if fanout:
        m = inp.shape[0]
        load_in = np.repeat(out, fanout)
        load_out = n_ring_nodes + np.arange(m * fanout)
        # interleave: stage, its loads, next stage ...
        grp_in = np.concatenate([inp[:, None], load_in.reshape(m, fanout)], 1).ravel()
        grp_out = np.concatenate([out[:, None], load_out.reshape(m, fanout)], 1).ravel()
        inp, out = grp_in, grp_out
        n_ring_nodes += m * fanout
    vdd = n_ring_nodes
    d, g, s, b, model = _inverters(inp, out, vdd)
    w, l = _wl_uniform(rng, d.shape[0])
    er, ec = _vdd_branch(vdd, vdd + 1)
    return _finish(f"rings{rings}x{stages}" + (f"_fo{fanout}" if fanout else ""),
                   n_ring_nodes + 1, 1, d, g, s, b, w, l, model,
                   models or bench_models(), [vdd], er, ec, rng,
                   dict(config=1, rings=rings, stages=stages, fanout=fanout))


def sram_6t(rows: int = 512, cols: int = 1024, seed: int = 2, models=None) -> Netlist:
    """configs[2]: 6T SRAM array.  Per cell, device order
    PU1 PD1 PU2 PD2 AX1 AX2; cells row-major.  Node ids: (Q,QB) per cell, then
    WL[rows], BL[cols], BLB[cols], VDD, branch."""
    rng = _rng(seed)
    R, C = rows, cols
    cell = np.arange(R * C)
    i = cell // C; j = cell % C
    Q = 2 * cell; QB = Q + 1
    WL = 2 * R * C + i
    BL = 2 * R * C + R + j
    BLB = 2 * R * C + R + C + j
    vdd = 2 * R * C + R + 2 * C
    G = -np.ones_like(cell)
    V = np.full_like(cell, vdd)
    d = np.stack([Q, Q, QB, QB, BL, BLB], 1).ravel()
    g = np.stack([QB, QB, Q, Q, WL, WL], 1).ravel()
    s = np.stack([V, G, V, G, Q, QB], 1).ravel()
    b = np.stack([V, G, V, G, G, G], 1).ravel()
    model = np.tile(np.array([1, 0, 1, 0, 0, 0], np.int32), R * C)
    base_w = np.tile(np.array([0.20, 0.40, 0.20, 0.40, 0.25, 0.25]) * UM, R * C)
    base_l = np.full(6 * R * C, 0.05 * UM)
    w = base_w * rng.uniform(0.9, 1.1, base_w.shape[0])
    l = base_l * rng.uniform(0.9, 1.1, base_l.shape[0])
    er, ec = _vdd_branch(vdd, vdd + 1)
    return _finish(f"sram{R}x{C}", vdd + 1, 1, d, g, s, b, w, l, model,
                   models or bench_models(), [vdd], er, ec, rng,
                   dict(config=2, rows=R, cols=C))


def random_netlist(n_dev: int = 4_000_000, n_nodes: int = 1_000_000,
                   seed: int = 3, models=None) -> Netlist:
    """configs[3]: D,G,S uniform over nodes, bulk grounded, 50/50 polarity
    (SURVEY A13); no rails, no branch."""
    rng = _rng(seed)
    d = rng.integers(0, n_nodes, n_dev)
    g = rng.integers(0, n_nodes, n_dev)
    s = rng.integers(0, n_nodes, n_dev)
    b = -np.ones(n_dev, np.int64)
    model = rng.integers(0, 2, n_dev).astype(np.int32)
    w, l = _wl_uniform(rng, n_dev)
    e = np.zeros(0, np.int32)
    return _finish(f"random{n_dev}_{n_nodes}", n_nodes, 0, d, g, s, b, w, l, model,
                   models or bench_models(), [], e, e, rng,
                   dict(config=3))


def hub_netlist(n_inv: int = 4_000_000, seed: int = 4, f_lo: int = 256,
                f_hi: int = 4096, hub_share: float = 0.5, models=None) -> Netlist:
    """configs[4] under SURVEY A11: `n_inv` CMOS inverters (2*n_inv FETs).
    Hub fanouts f ~ log-uniform[f_lo, f_hi] gates, rounded to even (f/2
    inverter loads), drawn until hubs hold `hub_share` of all gates.  Each hub
    is the output of one chain inverter ("driver"); its loads follow it
    consecutively in netlist order; the chain continues from the last load's
    output.  All other inverters are plain chain stages.  Blocks are shuffled.
    Inverter k drives node k+1; node 0 is the chain input."""
    rng = _rng(seed)
    target = hub_share * 2 * n_inv
    fan = []
    tot = 0
    lo, hi = math.log(f_lo), math.log(f_hi)
    while tot < target:
        f = math.exp(rng.uniform(lo, hi))
        f = max(2, 2 * int(round(f / 2)))
        fan.append(f); tot += f
    fan = np.array(fan, np.int64)
    loads = fan // 2
    n_plain = n_inv - int(loads.sum()) - len(fan)
    if n_plain < 0:
        raise ValueError("hub budget exceeds inverter count")
    # block list: -1 = plain stage, h>=0 = hub block h (driver + loads)
    blocks = np.concatenate([-np.ones(n_plain, np.int64), np.arange(len(fan))])
    blocks = blocks[rng.permutation(blocks.shape[0])]
    size = np.where(blocks < 0, 1, 1 + loads[np.maximum(blocks, 0)])
    start = np.concatenate([[0], np.cumsum(size)[:-1]])
    inp = np.arange(n_inv)                      # default: previous output
    out = np.arange(n_inv) + 1
    hub_pos = np.nonzero(blocks >= 0)[0]
    hub_nodes = np.empty(len(hub_pos), np.int64)
    for t, bi in enumerate(hub_pos):
        s0 = start[bi]; nl = size[bi] - 1
        inp[s0 + 1: s0 + 1 + nl] = s0 + 1       # loads read the hub (driver out)
        hub_nodes[t] = s0 + 1
    vdd = n_inv + 1
    d, g, s, b, model = _inverters(inp, out, vdd)
    w, l = _wl_uniform(rng, d.shape[0])
    er, ec = _vdd_branch(vdd, vdd + 1)
    return _finish(f"hubs{n_inv}", n_inv + 2, 1, d, g, s, b, w, l, model,
                   models or bench_models(), [vdd], er, ec, rng,
                   dict(config=4, n_hubs=int(len(fan)), max_fanout=int(fan.max()),
                        hub_fraction=float(len(fan)) / (n_inv + 2),
                        hub_nodes=hub_nodes))


def gen_synth(n_dev: int, c_target: int, seed: int = 5, models=None) -> Netlist:
    """gen_synth: ceil(N/C) node-disjoint groups of C FETs whose
    drains share one group node (a clique of the conflict graph); each FET
    has a private gate and source node, bulk grounded, 50/50 polarity.
    Greedy first-fit in netlist order yields exactly C colours."""
    rng = _rng(seed)
    n_groups = -(-n_dev // c_target)
    dev = np.arange(n_dev)
    d = dev // c_target
    g = n_groups + 2 * dev
    s = n_groups + 2 * dev + 1
    b = -np.ones(n_dev, np.int64)
    model = rng.integers(0, 2, n_dev).astype(np.int32)
    w, l = _wl_uniform(rng, n_dev)
    e = np.zeros(0, np.int32)
    return _finish(f"synth{n_dev}_C{c_target}", n_groups + 2 * n_dev, 0, d, g, s, b,
                   w, l, model, models or bench_models(), [], e, e, rng,
                   dict(c_target=c_target))


# --------------------------------------------------------------------------
# Benchmark 2: 64-bit ripple-carry adder of 28T CMOS full adders
# (Fig. 6; the figure is missing, so the textbook mirror adder is
# used) and the R14 / R89 series-resistor variants
# --------------------------------------------------------------------------
# One bit, terminals (d, g, s, b) over the bit's local nets; "VDD" and "GND"
# are the supplies.  Carry stage nCo = NOT(AB + C(A+B)), sum stage
# nS = NOT(ABC + nCo(A+B+C)), then inverters Cout = NOT nCo, S = NOT nS.
# 14 PMOS (bulk VDD) then 14 NMOS (bulk GND) -- 28T; its non-ground terminal
# attachments number 89, the paper's "all transistor-to-transistor
# connections" of R89.
_FA28_P = [  # d, g, s
    ("x1", "A", "VDD"), ("x1", "B", "VDD"), ("nCo", "C", "x1"),
    ("x2", "A", "VDD"), ("nCo", "B", "x2"),
    ("x3", "A", "VDD"), ("x3", "B", "VDD"), ("x3", "C", "VDD"), ("nS", "nCo", "x3"),
    ("x4", "A", "VDD"), ("x5", "B", "x4"), ("nS", "C", "x5"),
    ("Co", "nCo", "VDD"), ("S", "nS", "VDD"),
]
_FA28_N = [
    ("y1", "A", "GND"), ("y1", "B", "GND"), ("nCo", "C", "y1"),
    ("nCo", "A", "y2"), ("y2", "B", "GND"),
    ("y3", "A", "GND"), ("y3", "B", "GND"), ("y3", "C", "GND"), ("nS", "nCo", "y3"),
    ("nS", "A", "y4"), ("y4", "B", "y5"), ("y5", "C", "GND"),
    ("Co", "nCo", "GND"), ("S", "nS", "GND"),
]
_FA28_LOCAL = ["x1", "x2", "x3", "x4", "x5", "y1", "y2", "y3", "y4", "y5", "nCo", "nS", "S"]


def full_adder_28t(bits: int = 64, seed: int = 9, models=None) -> Netlist:
    """Benchmark 2 baseline: `bits` cascaded 28T full adders; carry
    out of bit k is the carry in of bit k+1.  Nodes: Cin, then per bit A, B,
    the 13 local nets and Co; VDD (the rail) and its source branch last.
    Primary inputs (A, B, Cin) are ordinary nodes (their sources are linear
    devices outside the hot path).  W ~ U[0.2, 5] um, L ~ U[0.05, 0.5] um."""
    rng = _rng(seed)
    per_bit = 2 + len(_FA28_LOCAL) + 1
    n_nodes = 1 + bits * per_bit + 1
    vdd = n_nodes - 1
    d, g, s, b, model, stage = [], [], [], [], [], []
    cin = 0
    for k in range(bits):
        base = 1 + k * per_bit
        node = {"A": base, "B": base + 1, "C": cin, "VDD": vdd, "GND": -1}
        for j, nm in enumerate(_FA28_LOCAL):
            node[nm] = base + 2 + j
        node["Co"] = base + 2 + len(_FA28_LOCAL)
        for pol, table in ((1, _FA28_P), (0, _FA28_N)):
            for dn, gn, sn in table:
                d.append(node[dn]); g.append(node[gn]); s.append(node[sn])
                b.append(vdd if pol else -1)
                model.append(pol)
                stage.append(k)
        cin = node["Co"]
    N = len(d)
    w, l = _wl_uniform(rng, N)
    er, ec = _vdd_branch(vdd, n_nodes)
    return _finish(f"adder{bits}_28t", n_nodes, 1, np.array(d), np.array(g), np.array(s),
                   np.array(b), w, l, np.array(model, np.int32), models or bench_models(), [vdd],
                   er, ec, rng, dict(stage=np.array(stage, np.int32), bits=bits))


def insert_resistors(nl: Netlist, per_stage, seed: int = 10) -> Netlist:
    """R14 / R89: in every stage, split `per_stage` randomly
    chosen non-ground terminal attachments ("all" = every one, R89) off
    their net: the terminal moves to a fresh node joined to the old one by a
    1 mOhm series resistor.  The resistors are linear devices: only their
    pattern entries (old,old), (old,new), (new,old), (new,new) are added to
    the caller's extra entries; the FETs keep their sizes and cards.  New
    nodes take the old node's voltages (a 1 mOhm resistor carries ~no drop)."""
    rng = _rng(seed)
    T = np.stack([nl.d, nl.g, nl.s, nl.b], 1).astype(np.int64).copy()
    stage = nl.meta["stage"]
    n_old = nl.n_nodes
    new_of = []                     # old node of each new node
    er, ec = [list(nl.extra_row)], [list(nl.extra_col)]
    rows, cols = [], []
    for k in range(int(stage.max()) + 1 if len(stage) else 0):
        fets = np.nonzero(stage == k)[0]
        att = [(i, a) for i in fets for a in range(4) if T[i, a] >= 0]
        if per_stage == "all":
            pick = att
        else:
            idx = rng.choice(len(att), size=min(int(per_stage), len(att)), replace=False)
            pick = [att[j] for j in sorted(idx)]
        for i, a in pick:
            old = int(T[i, a])
            new = n_old + len(new_of)
            new_of.append(old)
            T[i, a] = new
            rows += [old, old, new, new]
            cols += [old, new, old, new]
    n_new = len(new_of)
    n_nodes = n_old + n_new
    # old nodes keep their ids, new nodes follow them, branch unknowns move up
    def remap(v):
        v = np.asarray(v, np.int64)
        return np.where(v >= n_old, v + n_new, v)
    extra_row = np.concatenate([remap(nl.extra_row), np.array(rows, np.int64)]) if rows else remap(nl.extra_row)
    extra_col = np.concatenate([remap(nl.extra_col), np.array(cols, np.int64)]) if cols else remap(nl.extra_col)
    x = np.concatenate([nl.x[:n_old], nl.x[np.array(new_of, np.int64)] if n_new else [], nl.x[n_old:]])
    xp = np.concatenate([nl.x_prev[:n_old], nl.x_prev[np.array(new_of, np.int64)] if n_new else [],
                         nl.x_prev[n_old:]])
    out = Netlist(name=f"{nl.name}_R{per_stage if per_stage != 'all' else 'all'}", n_nodes=n_nodes,
                  n_extra=nl.n_extra, d=T[:, 0].astype(np.int32), g=T[:, 1].astype(np.int32),
                  s=T[:, 2].astype(np.int32), b=T[:, 3].astype(np.int32), w=nl.w.copy(), l=nl.l.copy(),
                  model=nl.model.copy(), models=nl.models, rails=nl.rails.copy(),
                  extra_row=extra_row.astype(np.int32), extra_col=extra_col.astype(np.int32),
                  x=x, x_prev=xp, vprev=nl.vprev.copy(), h=nl.h, gmin=nl.gmin,
                  meta=dict(nl.meta, resistors=n_new, new_of=np.array(new_of, np.int32)))
    return out


# --------------------------------------------------------------------------
# tiny hand circuits (tests)
# --------------------------------------------------------------------------
def custom(name, n_nodes, terms, model, models, w=None, l=None, rails=(),
           n_extra=0, extra=(), x=None, x_prev=None, seed=7, h=H_DEFAULT) -> Netlist:
    """Arbitrary small netlist from explicit terminal tuples (d,g,s,b)."""
    rng = _rng(seed)
    t = np.asarray(terms, np.int64).reshape(-1, 4)
    n = t.shape[0]
    if w is None or l is None:
        w2, l2 = _wl_uniform(rng, n)
        w = w2 if w is None else w
        l = l2 if l is None else l
    er = np.array([e[0] for e in extra], np.int32)
    ec = np.array([e[1] for e in extra], np.int32)
    nl = _finish(name, n_nodes, n_extra, t[:, 0], t[:, 1], t[:, 2], t[:, 3],
                 np.broadcast_to(np.asarray(w, float), (n,)).copy(),
                 np.broadcast_to(np.asarray(l, float), (n,)).copy(),
                 np.broadcast_to(np.asarray(model, np.int32), (n,)).copy(),
                 models, list(rails), er, ec, rng, {}, h=h)
    if x is not None:
        nl.x = np.asarray(x, float).copy()
    if x_prev is not None:
        nl.x_prev = np.asarray(x_prev, float).copy()
        nl.vprev = np.ascontiguousarray(_vprev(nl.x_prev, nl.d, nl.g, nl.s, nl.b))
    return nl


def ota_5t(seed: int = 8, models=None) -> Netlist:
    """5T OTA with current mirror (Fig. 3, re-derived since the figure
    is missing).  Nodes: inp=0 inn=1 out=2 n1=3 tail=4 vbias=5 VDD=6, branch 7.
    M1 (n1,inp,tail,0)  M2 (out,inn,tail,0)  M3 (n1,n1,VDD,VDD)
    M4 (out,n1,VDD,VDD) M5 (tail,vbias,0,0)."""
    terms = [(3, 0, 4, -1), (2, 1, 4, -1), (3, 3, 6, 6), (2, 3, 6, 6), (4, 5, -1, -1)]
    return custom("ota5t", 7, terms, [0, 0, 1, 1, 0], models or bench_models(),
                  rails=[6], n_extra=1, extra=[(6, 7), (7, 6)], seed=seed)


# --------------------------------------------------------------------------
# registry
# --------------------------------------------------------------------------
def config(i: int, scale: float = 1.0) -> Netlist:
    """BASELINE.json configs[i] at full size (scale=1) or a reduced instance
    of the same structure (scale<1) for CPU-time tests."""
    if i == 0:
        return inverter_chain(max(2, int(round(1000 * scale))) if scale < 1 else 1000)
    if i == 1:
        return ring_oscillators(max(1, int(round(1000 * scale))), 101)
    if i == 2:
        if scale >= 1:
            return sram_6t(512, 1024)
        r = max(2, int(round(512 * math.sqrt(scale))))
        c = max(2, int(round(1024 * math.sqrt(scale))))
        return sram_6t(r, c)
    if i == 3:
        return random_netlist(max(8, int(4_000_000 * scale)), max(2, int(1_000_000 * scale)))
    if i == 4:
        if scale >= 1:
            return hub_netlist()
        return hub_netlist(max(64, int(4_000_000 * scale)),
                           f_hi=max(256, min(4096, int(4096 * math.sqrt(scale) * 4))))
    raise ValueError(i)


CONFIG_NAMES = {
    0: "cfg0 inverter chain 1,000 stages (2,000 FETs)",
    1: "cfg1 1,000 x ring-101 (202,000 FETs)",
    2: "cfg2 6T SRAM 512x1024 (3,145,728 FETs)",
    3: "cfg3 random 4M FETs / 1M nodes",
    4: "cfg4 clock/bus hubs 8M FETs",
}


def named(name: str) -> Netlist:
    """Extra workloads by name (bench.py --netlist): Benchmark 2's adder and
    its resistor variants, cfgN[@scale], synth<N>_<C>."""
    if name == "adder64":
        return full_adder_28t(64)
    if name == "adder64_r14":
        return insert_resistors(full_adder_28t(64), 14)
    if name == "adder64_r89":
        return insert_resistors(full_adder_28t(64), "all")
    if name.startswith("synth"):                       # synth<N>_<C>: gen_synth (B5)
        n_dev, c_target = name[5:].split("_")
        return gen_synth(int(n_dev), int(c_target))
    if name.startswith("cfg"):
        i, _, sc = name[3:].partition("@")
        return config(int(i), float(sc) if sc else 1.0)
    raise ValueError(name)
