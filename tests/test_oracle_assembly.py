"""Pins of the oracle's pattern and assembly (
SURVEY §8(c) pins table).  CPU only."""
import math

import numpy as np
import pytest
import scipy.sparse as sp

import netgen
import oracle

D, G, S, B = 0, 1, 2, 3


def numpy_pattern(nl):
    """Independent reconstruction: all ordered non-ground terminal
    pairs + extras, unique-sorted by numpy."""
    T = np.stack([nl.d, nl.g, nl.s, nl.b], 1).astype(np.int64)
    r = np.repeat(T, 4, axis=1).ravel()
    c = np.tile(T, (1, 4)).ravel()
    m = (r >= 0) & (c >= 0)
    keys = np.concatenate([r[m] * nl.n + c[m], nl.extra_row.astype(np.int64) * nl.n + nl.extra_col])
    return np.unique(keys)


def test_footprints():
    """FET with d,g,s non-ground + grounded bulk -> 9 entries."""
    nl = netgen.custom("fet", 3, [(0, 1, 2, -1)], 0, netgen.bench_models())
    _, _, keys = oracle.pattern(nl)
    assert keys.shape[0] == 9
    nl = netgen.custom("fet4", 4, [(0, 1, 2, 3)], 0, netgen.bench_models())
    assert oracle.pattern(nl)[2].shape[0] == 16
    nl = netgen.custom("fetg", 2, [(0, 1, -1, -1)], 0, netgen.bench_models())
    assert oracle.pattern(nl)[2].shape[0] == 4


def test_dedup():
    """devices sharing a node share one diagonal entry."""
    nl = netgen.custom("two", 3, [(0, 1, -1, -1), (0, 2, -1, -1)], 0, netgen.bench_models())
    row_ptr, col_idx, keys = oracle.pattern(nl)
    assert list(keys) == [0 * 3 + 0, 0 * 3 + 1, 0 * 3 + 2, 1 * 3 + 0, 1 * 3 + 1, 2 * 3 + 0, 2 * 3 + 2]
    assert list(row_ptr) == [0, 3, 5, 7]


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_pattern_matches_numpy(cfg):
    nl = netgen.config(cfg, 0.01)
    assert np.array_equal(oracle.pattern(nl)[2], numpy_pattern(nl))


@pytest.mark.parametrize("cfg,nnz", [(0, 5006), (1, 505003)])
def test_nnz_full_size(cfg, nnz):
    """SURVEY §8(a) size table (derived by numpy unique, App. A)."""
    nl = netgen.config(cfg)
    assert oracle.pattern(nl)[2].shape[0] == nnz


def dense_A(nl, ref):
    n = nl.n
    A = np.zeros((n, n))
    rows = ref["keys"] // n
    A[rows, ref["keys"] % n] = ref["A"]
    return A


def circuit_current(nl, V):
    """Nodal current function F(V): sum over devices of the currents leaving
    each terminal (channel, gmin, backward-Euler caps), ground dropped."""
    F = np.zeros(nl.n)
    Vg = np.concatenate([V, [0.0]])               # index -1 -> ground
    for i in range(nl.n_dev):
        cd = nl.models[nl.model[i]]
        beta = cd["kp"] * nl.w[i] / nl.l[i]
        T = [nl.d[i], nl.g[i], nl.s[i], nl.b[i]]
        Vt = [Vg[t] for t in T]
        I, *_ = oracle.channel(cd["polarity"], cd["vt0"], cd["lam"], beta, Vt[D], Vt[G], Vt[S])
        cur = np.zeros(4)
        cur[D] += I; cur[S] -= I
        ig = nl.gmin * (Vt[D] - Vt[S]); cur[D] += ig; cur[S] -= ig
        for k, (a, c, C) in enumerate(((G, S, cd["cgs"]), (G, D, cd["cgd"]), (D, B, cd["cdb"]))):
            ic = C / nl.h * ((Vt[a] - Vt[c]) - nl.vprev[k, i])
            cur[a] += ic; cur[c] -= ic
        for a in range(4):
            if T[a] >= 0:
                F[T[a]] += cur[a]
    return F


def _tiny_circuits():
    ms = netgen.bench_models()
    yield netgen.custom("nmos", 3, [(0, 1, 2, -1)], 0, ms, seed=1)
    yield netgen.custom("pmos", 4, [(0, 1, 2, 3)], 1, ms, seed=2)
    yield netgen.custom("inv", 3, [(1, 0, -1, -1), (1, 0, 2, 2)], [0, 1], ms, rails=[2],
                        n_extra=1, extra=[(2, 3), (3, 2)], seed=3)
    yield netgen.ota_5t()
    yield netgen.custom("dstied", 3, [(0, 1, 0, -1), (2, 2, 1, -1), (1, 2, 0, 1)], [0, 1, 0], ms, seed=4)
    yield netgen.inverter_chain(3, seed=5)


@pytest.mark.parametrize("nl", list(_tiny_circuits()), ids=lambda n: n.name)
def test_tiny_circuit_equals_fd_jacobian(nl):
    """Tiny circuits (<=6 FETs): the assembled A is the Jacobian of the
    circuit's nodal current function and b = A V - F(V) (Newton-Raphson
    linearisation), by brute-force central differences."""
    for trial in range(3):
        rng = np.random.Generator(np.random.PCG64(100 + trial))
        nl.x[:nl.n_nodes] = rng.uniform(0, 1, nl.n_nodes)
        nl.x[nl.rails] = 1.0
        ref = oracle.reference(nl)
        A = dense_A(nl, ref)
        V = nl.x.copy()
        eps = 1e-6
        J = np.zeros((nl.n, nl.n))
        for c in range(nl.n_nodes):
            Vp = V.copy(); Vp[c] += eps
            Vm = V.copy(); Vm[c] -= eps
            J[:, c] = (circuit_current(nl, Vp) - circuit_current(nl, Vm)) / (2 * eps)
        scale = np.abs(A).max()
        assert np.abs(A - J).max() <= 1e-6 * scale
        F = circuit_current(nl, V)
        bb = A @ V - F
        assert np.abs(bb - ref["b"]).max() <= 1e-12 * (np.abs(A).max() * 1 + np.abs(F).max())


def test_all_cutoff_is_a_linear_network_laplacian():
    """Special case: with SPEC's card (vt0 = 1 V) and voltages in [0,1] V every
    FET is in cutoff, so A is the weighted graph Laplacian of the linear
    network {gmin on D-S, C/h on G-S, G-D, D-B} (textbook L = B W B^T) and b is
    B (w * v_prev) -- exactly, up to rounding."""
    nl = netgen.inverter_chain(200, seed=12, models=netgen.spec_models())
    ref = oracle.reference(nl)
    n = nl.n
    edges = []   # (a_node, c_node, weight, v0)
    for i in range(nl.n_dev):
        cd = nl.models[nl.model[i]]
        T = [nl.d[i], nl.g[i], nl.s[i], nl.b[i]]
        edges.append((T[D], T[S], nl.gmin, 0.0))
        edges.append((T[G], T[S], cd["cgs"] / nl.h, nl.vprev[0, i]))
        edges.append((T[G], T[D], cd["cgd"] / nl.h, nl.vprev[1, i]))
        edges.append((T[D], T[B], cd["cdb"] / nl.h, nl.vprev[2, i]))
    Bi, Bj, Bv, w, j = [], [], [], [], []
    for e, (a, c, wt, v0) in enumerate(edges):
        for node, sgn in ((a, 1.0), (c, -1.0)):
            if node >= 0:
                Bi.append(node); Bj.append(e); Bv.append(sgn)
        w.append(wt); j.append(wt * v0)
    Bm = sp.csr_matrix((Bv, (Bi, Bj)), shape=(n, len(edges)))
    L = (Bm @ sp.diags(w) @ Bm.T).toarray()
    bb = Bm @ np.array(j)
    A = dense_A(nl, ref)
    Aabs = dense_A(nl, dict(keys=ref["keys"], A=ref["A_abs"]))
    # scipy's plain sums carry <= n*u*sum|c| error (rail diagonal: 400 terms)
    assert np.all(np.abs(A - L) <= 1e-13 * Aabs)
    assert np.all(np.abs(bb - ref["b"]) <= 1e-13 * ref["b_abs"])


def test_reference_is_exactly_rounded_sum():
    """The reference entry is the exactly-rounded sum (math.fsum) of the
    elementary contributions (Neumaier accumulation)."""
    nl = netgen.ota_5t()
    ref = oracle.reference(nl)
    n = nl.n
    contrib = {}
    bcon = {}
    for i in range(nl.n_dev):
        cd = nl.models[nl.model[i]]
        beta = cd["kp"] * nl.w[i] / nl.l[i]
        T = [int(nl.d[i]), int(nl.g[i]), int(nl.s[i]), int(nl.b[i])]
        V = [nl.x[t] if t >= 0 else 0.0 for t in T]
        Y, J = oracle.device_stamps(cd, beta, nl.gmin, nl.h, V, nl.vprev[:, i])
        for a, c, v in Y:
            if T[a] >= 0 and T[c] >= 0:
                contrib.setdefault(T[a] * n + T[c], []).append(v)
        for a, v in J:
            if T[a] >= 0:
                bcon.setdefault(T[a], []).append(v)
    for k, key in enumerate(ref["keys"]):
        vals = contrib.get(int(key), [])
        assert ref["A"][k] == math.fsum(vals)
        assert ref["A_abs"][k] == pytest.approx(sum(abs(v) for v in vals), rel=1e-15)
    for r in range(n):
        assert ref["b"][r] == math.fsum(bcon.get(r, []))


def test_accumulate_semantics():
    """add is +=; the reference starts from the caller's values."""
    nl = netgen.ota_5t()
    r0 = oracle.reference(nl)
    A0 = np.linspace(-1, 1, r0["A"].shape[0])
    b0 = np.linspace(2, 3, nl.n)
    r1 = oracle.reference(nl, A0=A0, b0=b0)
    assert np.allclose(r1["A"], A0 + r0["A"], rtol=0, atol=1e-15)
    assert np.allclose(r1["b"], b0 + r0["b"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("cfg", [0, 1, 2, 4])
def test_cpu_baselines(cfg):
    """loadomp is bitwise equal to loadsingle; ColorFused
    agrees within 1e-12 * sum|c| (north_star tolerance)."""
    nl = netgen.config(cfg, 0.01)
    patt = oracle.pattern(nl)
    ref = oracle.reference(nl, patt=patt)
    bl = oracle.Baseline(nl, patt=patt)
    nnz = patt[2].shape[0]
    A1 = np.zeros(nnz); b1 = np.zeros(nl.n)
    bl.run("loadsingle", A1, b1)
    A2 = np.zeros(nnz); b2 = np.zeros(nl.n)
    bl.run("loadomp", A2, b2, threads=4)
    assert np.array_equal(A1, A2) and np.array_equal(b1, b2)
    A3 = np.zeros(nnz); b3 = np.zeros(nl.n)
    bl.run("colorfused", A3, b3, threads=4)
    for got in (A1, A3):
        assert np.all(np.abs(got - ref["A"]) <= 1e-12 * ref["A_abs"])
    for got in (b1, b3):
        assert np.all(np.abs(got - ref["b"]) <= 1e-12 * ref["b_abs"])
    bl.close()
