"""Pins of the oracle's device function (
SURVEY §8(c) pins table).  CPU only."""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "device_points.json")))
D, G, S, B = 0, 1, 2, 3


def card(p=1, vt0=1.0, lam=0.0, cgs=0.0, cgd=0.0, cdb=0.0):
    return dict(polarity=p, vt0=vt0, kp=2e-5, lam=lam, cgs=cgs, cgd=cgd, cdb=cdb)


@pytest.mark.parametrize("pt", GOLD["points"], ids=lambda p: p["name"])
def test_closed_form_points(pt):
    I, gm, gds, region, _ = oracle.channel(pt["polarity"], pt["vt0"], pt["lam"], pt["beta"],
                                           pt["VD"], pt["VG"], pt["VS"])
    assert region == pt["region"]
    for got, want in ((I, pt["I"]), (gm, pt["gm"]), (gds, pt["gds"])):
        assert got == pytest.approx(want, rel=1e-12, abs=1e-25)
    # Norton term through the assembled stamp (no caps, gmin=0): J[D] = -Ieq, J[S] = +Ieq
    Y, J = oracle.local_stamp(card(pt["polarity"], pt["vt0"], pt["lam"]), pt["beta"], 0.0, 1.0,
                              [pt["VD"], pt["VG"], pt["VS"], 0.0], [0, 0, 0])
    assert J[D] == pytest.approx(-pt["Ieq"], rel=1e-12, abs=1e-25)
    assert J[S] == pytest.approx(pt["Ieq"], rel=1e-12, abs=1e-25)
    # terminal-frame conductances: dI/dVG = gm, dI/dVD = gds, dI/dVS = -(gm+gds)
    assert Y[D, G] == pytest.approx(pt["gm"], rel=1e-12, abs=1e-25)
    assert Y[D, D] == pytest.approx(pt["gds"], rel=1e-12, abs=1e-25)
    assert Y[D, S] == pytest.approx(-(pt["gm"] + pt["gds"]), rel=1e-12, abs=1e-25)


def test_cutoff_stamps_only_gmin_and_caps():
    """in cutoff A gets only gmin (+ caps)."""
    gmin = 1e-12
    Y, J = oracle.local_stamp(card(), 2e-5, gmin, 1.0, [2.0, 0.5, 0.0, 0.0], [0, 0, 0])
    want = np.zeros((4, 4))
    want[D, D] = want[S, S] = gmin
    want[D, S] = want[S, D] = -gmin
    assert np.array_equal(Y, want)
    assert np.array_equal(J, np.zeros(4))


def test_capacitor_companion():
    """1 pF, dt = 1 ns, v_prev = 1 V -> Geq = 1e-3 S, Ieq = -1e-3 A."""
    cap = GOLD["capacitor"]
    Y, J = oracle.local_stamp(card(vt0=100.0, cgs=cap["C"]), 2e-5, 0.0, cap["h"],
                              [0.0, 0.3, 0.1, 0.0], [cap["v0"], 0, 0])
    assert Y[G, G] == pytest.approx(cap["Geq"], rel=1e-15)
    assert Y[S, S] == pytest.approx(cap["Geq"], rel=1e-15)
    assert Y[G, S] == pytest.approx(-cap["Geq"], rel=1e-15)
    assert J[G] == pytest.approx(-cap["Ieq"], rel=1e-15)
    assert J[S] == pytest.approx(cap["Ieq"], rel=1e-15)


def _rand_bias(rng, p):
    V = rng.uniform(-1.5, 1.5, 4) if p > 0 else rng.uniform(-1.5, 1.5, 4)
    return V


def terminal_currents(cd, beta, gmin, h, V, v0):
    """Physics definition of the currents leaving each terminal: channel
    current (leaves D, enters S), gmin resistor D-S, and backward-Euler
    capacitor currents C/h*(v - v0)."""
    I, *_ = oracle.channel(cd["polarity"], cd["vt0"], cd["lam"], beta, V[D], V[G], V[S])
    i = np.zeros(4)
    i[D] += I; i[S] -= I
    ig = gmin * (V[D] - V[S]); i[D] += ig; i[S] -= ig
    for (a, c, C, vp) in ((G, S, cd["cgs"], v0[0]), (G, D, cd["cgd"], v0[1]), (D, B, cd["cdb"], v0[2])):
        ic = C / h * ((V[a] - V[c]) - vp)
        i[a] += ic; i[c] -= ic
    return i


@pytest.mark.parametrize("p", [1, -1])
def test_fd_jacobian_and_norton(p):
    """gm, gds match central finite differences to 1e-6 relative at
    random biases in every region; and the stamp satisfies J = Y V - i(V)
    (the linearised model reproduces the device current at the bias point)."""
    rng = np.random.Generator(np.random.PCG64(11 + p))
    cd = card(p, 0.3 * p, 0.05, 1e-15, 1.3e-15, 0.7e-15)
    h, gmin, beta = 1e-12, 1e-12, 2e-5 * 7.0
    seen_regions = set()
    n_checked = 0
    while n_checked < 300:
        V = _rand_bias(rng, p)
        v0 = rng.uniform(-1, 1, 3)
        I, gm, gds, region, mode = oracle.channel(p, cd["vt0"], cd["lam"], beta, V[D], V[G], V[S])
        # stay away from region boundaries (model is C1, not C2, there)
        vgs, vds = p * (V[G] - V[S]), p * (V[D] - V[S])
        u, v = (vgs, vds) if vds >= 0 else (vgs - vds, -vds)
        uov = u - p * cd["vt0"]
        if min(abs(uov), abs(v - uov), abs(vds)) < 1e-3:
            continue
        seen_regions.add((region, mode))
        Y, J = oracle.local_stamp(cd, beta, gmin, h, V, v0)
        eps = 1e-6
        Yfd = np.zeros((4, 4))
        for c in range(4):
            Vp = V.copy(); Vp[c] += eps
            Vm = V.copy(); Vm[c] -= eps
            Yfd[:, c] = (terminal_currents(cd, beta, gmin, h, Vp, v0)
                         - terminal_currents(cd, beta, gmin, h, Vm, v0)) / (2 * eps)
        scale = np.abs(Y).max()
        assert np.abs(Y - Yfd).max() <= 1e-6 * scale
        # channel-only derivative check at tight relative tolerance
        if region != 0:
            Ip, *_ = oracle.channel(p, cd["vt0"], cd["lam"], beta, V[D], V[G] + eps, V[S])
            Im, *_ = oracle.channel(p, cd["vt0"], cd["lam"], beta, V[D], V[G] - eps, V[S])
            assert (Ip - Im) / (2 * eps) == pytest.approx(gm, rel=1e-6, abs=1e-6 * abs(gds) + 1e-18)
            Ip, *_ = oracle.channel(p, cd["vt0"], cd["lam"], beta, V[D] + eps, V[G], V[S])
            Im, *_ = oracle.channel(p, cd["vt0"], cd["lam"], beta, V[D] - eps, V[G], V[S])
            assert (Ip - Im) / (2 * eps) == pytest.approx(gds, rel=1e-6, abs=1e-6 * abs(gm) + 1e-18)
        i = terminal_currents(cd, beta, gmin, h, V, v0)
        lhs = Y @ V - i
        mag = np.abs(Y).max() * np.abs(V).max() + np.abs(i).max()
        assert np.abs(lhs - J).max() <= 1e-13 * mag
        n_checked += 1
    assert {(0, 1), (1, 1), (2, 1), (0, -1), (1, -1), (2, -1)} <= seen_regions


def test_kcl_row_column_sums():
    """Translation invariance / KCL (north_star): each device's stamped
    currents sum to zero and its Y rows and columns sum to zero."""
    rng = np.random.Generator(np.random.PCG64(5))
    for _ in range(500):
        p = int(rng.choice([1, -1]))
        cd = card(p, 0.3 * p, 0.05, 1e-15, 2e-15, 3e-15)
        V = rng.uniform(-1.2, 1.2, 4)
        Y, J = oracle.local_stamp(cd, 2e-5 * rng.uniform(0.1, 100), 1e-12, 1e-12, V,
                                  rng.uniform(-1, 1, 3))
        m = np.abs(Y).max()
        assert np.abs(Y.sum(0)).max() <= 4e-16 * m
        assert np.abs(Y.sum(1)).max() <= 4e-16 * m
        assert abs(J.sum()) <= 4e-16 * np.abs(J).max() * 8


def test_drain_source_symmetry():
    """swapping D and S (negating Vds) negates the channel current."""
    rng = np.random.Generator(np.random.PCG64(9))
    for _ in range(1000):
        p = int(rng.choice([1, -1]))
        VD, VG, VS = rng.uniform(-1.5, 1.5, 3)
        I1, *_ = oracle.channel(p, 0.3 * p, 0.05, 3e-5, VD, VG, VS)
        I2, *_ = oracle.channel(p, 0.3 * p, 0.05, 3e-5, VS, VG, VD)
        assert I2 == pytest.approx(-I1, rel=1e-13, abs=1e-30)


def test_pmos_is_reflected_nmos():
    """S:196 'PMOS by sign reflection': I_p(V) = -I_n(-V) with vt0 -> -vt0."""
    rng = np.random.Generator(np.random.PCG64(10))
    for _ in range(1000):
        VD, VG, VS = rng.uniform(-1.5, 1.5, 3)
        In, gmn, gdn, rn, mn = oracle.channel(1, 0.4, 0.05, 3e-5, -VD, -VG, -VS)
        Ip, gmp, gdp, rp, mp = oracle.channel(-1, -0.4, 0.05, 3e-5, VD, VG, VS)
        assert (rn, mn) == (rp, mp)
        assert Ip == pytest.approx(-In, rel=1e-15, abs=1e-30)
        assert gmp == pytest.approx(gmn, rel=1e-15, abs=1e-30)
        assert gdp == pytest.approx(gdn, rel=1e-15, abs=1e-30)


@pytest.mark.parametrize("lam", [0.0, 0.05])
def test_c1_continuity_at_boundaries(lam):
    """S:223 continuity of Id and its first derivatives across regions
    (the model is C1, so tie choices only change rounding)."""
    beta, vt = 2e-5, 0.3
    d = 1e-9
    for vgs in (0.6, 1.0, 1.3):
        uov = vgs - vt
        a = oracle.channel(1, vt, lam, beta, uov - d, vgs, 0.0)   # triode side of v = uov
        b = oracle.channel(1, vt, lam, beta, uov + d, vgs, 0.0)   # saturation side
        assert a[3] == 1 and b[3] == 2
        for k in range(3):
            assert a[k] == pytest.approx(b[k], rel=1e-6, abs=10 * beta * d)
    a = oracle.channel(1, vt, lam, beta, 0.5, vt + d, 0.0)         # just on
    b = oracle.channel(1, vt, lam, beta, 0.5, vt - d, 0.0)         # cutoff
    for k in range(3):
        assert abs(a[k] - b[k]) <= 1e-8 * beta
    for vgs in (0.6, 1.0):                                          # vds = 0: both modes agree
        a = oracle.channel(1, vt, lam, beta, +d, vgs, 0.0)
        b = oracle.channel(1, vt, lam, beta, -d, vgs, 0.0)
        assert a[4] == 1 and b[4] == -1
        assert a[0] == pytest.approx(-b[0], rel=1e-6, abs=1e-6 * beta * d)
        assert a[1] == pytest.approx(b[1], rel=1e-6, abs=1e-6 * beta)
        assert a[2] == pytest.approx(b[2], rel=1e-6, abs=1e-6 * beta)


def test_dc_h_infinite_drops_caps():
    """h = +inf (DC): companion conductances C/h vanish."""
    cd = card(1, 0.3, 0.05, 1e-15, 1e-15, 1e-15)
    Y, J = oracle.local_stamp(cd, 2e-5, 0.0, math.inf, [0.8, 0.9, 0.0, 0.0], [0.3, 0.2, 0.1])
    I, gm, gds, *_ = oracle.channel(1, 0.3, 0.05, 2e-5, 0.8, 0.9, 0.0)
    assert Y[G, G] == 0 and Y[B, B] == 0 and Y[D, B] == 0
    assert Y[D, D] == pytest.approx(gds, rel=1e-15)
    assert J[G] == 0 and J[B] == 0
