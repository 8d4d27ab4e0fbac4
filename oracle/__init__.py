"""CPU oracle for the evaluate+stamp hot path -- TEST INFRASTRUCTURE ONLY.

Thin ctypes binding over ``oracle/ees_oracle.c`` (plain C, FP64, no FMA
contraction).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with ``paper_2604_03079_b200`` (the CUDA path); both consume the
seeded inputs of ``netgen``.

Every function cites the PAPER.md / SPEC.md passage it follows (see the C
source).  Parity status: all functions pinned by tests/test_oracle_*.py, except
absolute physics vs BSIM4/Ngspice, which is "parity unpinned" (P:58, P:163:
BSIM4 and Ngspice are not available; SPEC's Level-1 model stands in).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ees_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

NY, NJ = 24, 12


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
               "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Model(C.Structure):
    _fields_ = [("polarity", C.c_int32), ("vt0", C.c_double), ("kp", C.c_double),
                ("lam", C.c_double), ("cgs", C.c_double), ("cgd", C.c_double),
                ("cdb", C.c_double)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            P = C.c_void_p
            i32, i64, f64 = C.c_int32, C.c_int64, C.c_double
            L.orc_channel.argtypes = [i32, f64, f64, f64, f64, f64, f64, P, P]
            L.orc_device_stamps.argtypes = [P, f64, f64, f64, P, P, P, P, P, P, P, P, P]
            L.orc_pattern.argtypes = [i64, i64, P, P, P, P, i64, P, P, P]
            L.orc_pattern.restype = i64
            L.orc_reference.argtypes = [i64, i64, P, i64, P, P, P, P, P, P, P, P, P,
                                        f64, f64, P, P, P, P, P]
            L.orc_reference.restype = i32
            L.orc_greedy_color.argtypes = [i64, i64, P, P, P, P, P, P]
            L.orc_greedy_color.restype = i32
            L.orc_color_violations.argtypes = [i64, i64, P, P, P, P, P, P, i32]
            L.orc_color_violations.restype = i64
            L.orc_plan_create.argtypes = [i64, i64, P, i64, P, P, P, P, P, P, P, P, P, i32,
                                          P, i32, P]
            L.orc_plan_create.restype = P
            L.orc_plan_destroy.argtypes = [P]
            L.orc_loadsingle.argtypes = [P, f64, f64, P, P, P]
            L.orc_loadomp.argtypes = [P, i32, f64, f64, P, P, P]
            L.orc_colorfused.argtypes = [P, i32, f64, f64, P, P, P]
            L.orc_max_threads.restype = i32
            _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _models(cards):
    arr = (_Model * max(1, len(cards)))()
    for i, m in enumerate(cards):
        arr[i] = _Model(int(m["polarity"]), float(m["vt0"]), float(m["kp"]), float(m["lam"]),
                        float(m["cgs"]), float(m["cgd"]), float(m["cdb"]))
    return arr


# ---------------------------------------------------------------- device
def channel(polarity, vt0, lam, beta, VD, VG, VS):
    """Level-1 channel ->
    (I_ch, gm, gds, region, mode); region 0 cutoff / 1 triode / 2 sat."""
    out = np.zeros(3)
    info = np.zeros(2, np.int32)
    lib().orc_channel(int(polarity), float(vt0), float(lam), float(beta),
                      float(VD), float(VG), float(VS), _p(out), _p(info))
    return out[0], out[1], out[2], int(info[0]), int(info[1])


def device_stamps(card, beta, gmin, h, V, v0):
    """Elementary contributions of one device:
    returns (Y list of (a, c, value), J list of (a, value)), terminals
    D=0 G=1 S=2 B=3."""
    m = _models([card])
    V = np.ascontiguousarray(V, float)
    v0 = np.ascontiguousarray(v0, float)
    ya = np.zeros(NY, np.int32); yc = np.zeros(NY, np.int32); yv = np.zeros(NY)
    ja = np.zeros(NJ, np.int32); jv = np.zeros(NJ)
    ny = np.zeros(1, np.int32); nj = np.zeros(1, np.int32)
    lib().orc_device_stamps(C.byref(m[0]), float(beta), float(gmin), float(h), _p(V), _p(v0),
                            _p(ya), _p(yc), _p(yv), _p(ny), _p(ja), _p(jv), _p(nj))
    Y = [(int(ya[e]), int(yc[e]), float(yv[e])) for e in range(int(ny[0]))]
    J = [(int(ja[e]), float(jv[e])) for e in range(int(nj[0]))]
    return Y, J


def local_stamp(card, beta, gmin, h, V, v0):
    """Dense 4x4 Y and 4-vector J summed from the elementary contributions."""
    Y, J = device_stamps(card, beta, gmin, h, V, v0)
    Yd = np.zeros((4, 4)); Jd = np.zeros(4)
    for a, c, v in Y:
        Yd[a, c] += v
    for a, v in J:
        Jd[a] += v
    return Yd, Jd


# ---------------------------------------------------------------- pattern
def pattern(nl):
    """CSR pattern: returns (row_ptr int64[n+1], col_idx int32[nnz])."""
    n = nl.n
    cap = 16 * nl.n_dev + len(nl.extra_row)
    keys = np.empty(max(1, cap), np.int64)
    nnz = lib().orc_pattern(n, nl.n_dev, _p(nl.d), _p(nl.g), _p(nl.s), _p(nl.b),
                            len(nl.extra_row), _p(nl.extra_row), _p(nl.extra_col), _p(keys))
    keys = keys[:nnz].copy()
    rows = keys // n
    cols = (keys % n).astype(np.int32)
    row_ptr = np.zeros(n + 1, np.int64)
    row_ptr[1:] = np.cumsum(np.bincount(rows, minlength=n))
    return row_ptr, cols, keys


def reference(nl, A0=None, b0=None, patt=None):
    """The reference A, b (S:339 loadsingle; Neumaier-compensated) plus the
    per-entry sum of |elementary contributions|.  Returns dict with
    row_ptr, col_idx, keys, A, A_abs, b, b_abs."""
    if patt is None:
        patt = pattern(nl)
    row_ptr, col_idx, keys = patt
    nnz = keys.shape[0]
    A = np.zeros(nnz) if A0 is None else np.array(A0, float, copy=True)
    Aabs = np.abs(A)
    bb = np.zeros(nl.n) if b0 is None else np.array(b0, float, copy=True)
    babs = np.abs(bb)
    m = _models(nl.models)
    rc = lib().orc_reference(nl.n, nnz, _p(keys), nl.n_dev, _p(nl.d), _p(nl.g), _p(nl.s),
                             _p(nl.b), _p(nl.w), _p(nl.l), _p(nl.model), _p(nl.vprev), m,
                             float(nl.gmin), float(nl.h), _p(nl.x), _p(A), _p(Aabs), _p(bb),
                             _p(babs))
    if rc != 0:
        raise RuntimeError("oracle: contribution outside pattern")
    return dict(row_ptr=row_ptr, col_idx=col_idx, keys=keys, A=A, A_abs=Aabs, b=bb, b_abs=babs)


# ---------------------------------------------------------------- colouring
def node_fanout(nl):
    """Distinct FETs incident on each node (a FET with two terminals on one
    node counts once)."""
    T = np.stack([nl.d, nl.g, nl.s, nl.b], axis=1).astype(np.int64)
    deg = np.zeros(max(1, nl.n_nodes), np.int64)
    for a in range(4):
        t = T[:, a]
        first = t >= 0
        for c in range(a):
            first &= T[:, c] != t
        np.add.at(deg, t[first], 1)
    return deg


def excluded_mask(nl, rule="exclude_rails", heavy_degree=64):
    """Nodes removed from the conflict relation: rails under SURVEY A1's
    reading ("exclude_rails"), none under the paper-literal rule ("paper"),
    rails and every node with more than `heavy_degree` incident FETs under
    SURVEY §8(f) NEXT-1's degree-threshold hybrid ("hybrid")."""
    ex = np.zeros(max(1, nl.n_nodes), np.uint8)
    if rule in ("exclude_rails", "hybrid") and len(nl.rails):
        ex[nl.rails] = 1
    if rule == "hybrid":
        ex[node_fanout(nl) > heavy_degree] = 1
    elif rule not in ("exclude_rails", "paper"):
        raise ValueError(rule)
    return ex


def greedy_color(nl, rule="exclude_rails", heavy_degree=64):
    """First-fit greedy in netlist order -> (color int32[N], C)."""
    ex = excluded_mask(nl, rule, heavy_degree)
    color = np.zeros(max(1, nl.n_dev), np.int32)
    Cn = lib().orc_greedy_color(nl.n_nodes, nl.n_dev, _p(nl.d), _p(nl.g), _p(nl.s), _p(nl.b),
                                _p(ex), _p(color))
    return color[:nl.n_dev], int(Cn)


def color_violations(nl, color, n_colors, rule="exclude_rails", heavy_degree=64):
    """Exhaustive validity scan: 0 iff conflict-free."""
    ex = excluded_mask(nl, rule, heavy_degree)
    color = np.ascontiguousarray(color, np.int32)
    return int(lib().orc_color_violations(nl.n_nodes, nl.n_dev, _p(nl.d), _p(nl.g), _p(nl.s),
                                          _p(nl.b), _p(ex), _p(color), int(n_colors)))


# ---------------------------------------------------------------- CPU baselines
class Baseline:
    """The paper's Table I CPU kernels over this oracle, plain FP64,
    for timing (bench.py cpu_baseline / --impl reference).  Not a parity source."""

    def __init__(self, nl, rule="exclude_rails", patt=None):
        self.nl = nl
        self.patt = patt if patt is not None else pattern(nl)
        self.color, self.C = greedy_color(nl, rule)
        rails = np.zeros(max(1, nl.n), np.uint8)
        if rule == "exclude_rails" and len(nl.rails):
            rails[nl.rails] = 1
        self._rails = rails
        self._m = _models(nl.models)
        keys = self.patt[2]
        self.nnz = keys.shape[0]
        self._keys = keys
        self._h = lib().orc_plan_create(nl.n, self.nnz, _p(keys), nl.n_dev, _p(nl.d), _p(nl.g),
                                        _p(nl.s), _p(nl.b), _p(nl.w), _p(nl.l), _p(nl.model),
                                        _p(nl.vprev), self._m, len(nl.models), _p(self.color),
                                        self.C, _p(rails))

    def close(self):
        if self._h:
            lib().orc_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, kind, A, b, threads=1):
        nl = self.nl
        if kind == "loadsingle":
            lib().orc_loadsingle(self._h, nl.gmin, nl.h, _p(nl.x), _p(A), _p(b))
        elif kind == "loadomp":
            lib().orc_loadomp(self._h, int(threads), nl.gmin, nl.h, _p(nl.x), _p(A), _p(b))
        elif kind == "colorfused":
            lib().orc_colorfused(self._h, int(threads), nl.gmin, nl.h, _p(nl.x), _p(A), _p(b))
        else:
            raise ValueError(kind)


def max_threads() -> int:
    return int(lib().orc_max_threads())
