"""Pins of the oracle's conflict-graph greedy colouring (
SPEC S:266-305; SURVEY §8(c) coloring oracle + App. A).  CPU only."""
import numpy as np
import pytest

import netgen
import oracle


def brute_excluded(nl, rule, K=64):
    """Nodes outside the relation, by plain Python: rails (A1), plus nodes
    with more than K distinct incident FETs under the NEXT-1 hybrid."""
    ex = set(nl.rails.tolist()) if rule in ("exclude_rails", "hybrid") else set()
    if rule == "hybrid":
        fan = {}
        for row in zip(nl.d.tolist(), nl.g.tolist(), nl.s.tolist(), nl.b.tolist()):
            for t in set(row):
                if t >= 0:
                    fan[t] = fan.get(t, 0) + 1
        ex |= {t for t, f in fan.items() if f > K}
    return ex


def brute_first_fit(nl, rule="exclude_rails", K=64):
    """Independent: explicit edge list by pairwise node sharing (P:60 'share
    at least one non-ground node'), then first-fit in index order."""
    ex = brute_excluded(nl, rule, K)
    T = np.stack([nl.d, nl.g, nl.s, nl.b], 1)
    sets = [set(t for t in row if t >= 0 and t not in ex) for row in T.tolist()]
    N = len(sets)
    color = []
    for i in range(N):
        used = {color[j] for j in range(i) if sets[i] & sets[j]}
        c = 0
        while c in used:
            c += 1
        color.append(c)
    return np.array(color, np.int32)


def fets(terms, n_nodes, rails=()):
    return netgen.custom("t", n_nodes, terms, 0, netgen.bench_models(), rails=rails)


def test_edgeless():
    nl = fets([(2 * i, 2 * i + 1, -1, -1) for i in range(50)], 100)
    c, C = oracle.greedy_color(nl)
    assert C == 1 and not c.any()


def test_clique():
    nl = fets([(0, i + 1, -1, -1) for i in range(17)], 18)
    c, C = oracle.greedy_color(nl)
    assert C == 17 and list(c) == list(range(17))


def test_path():
    nl = fets([(0, 1, -1, -1), (1, 2, -1, -1), (2, 3, -1, -1)], 4)
    c, C = oracle.greedy_color(nl)
    assert list(c) == [0, 1, 0] and C == 2


def test_ground_shared_is_no_edge():
    """two FETs sharing only ground -> no edge."""
    nl = fets([(0, 1, -1, -1), (2, 3, -1, -1)], 4)
    assert oracle.greedy_color(nl)[1] == 1


@pytest.mark.parametrize("ct", [1, 2, 26, 334, 1000])
def test_gen_synth_hits_target(ct):
    """gen_synth cliques -> exactly C_target colours."""
    nl = netgen.gen_synth(1000, ct)
    c, C = oracle.greedy_color(nl)
    assert C == ct
    assert oracle.color_violations(nl, c, C) == 0


def test_topology_counts():
    """chain -> 4, ring-101 -> 6, FO4 ring -> 12, SRAM R x Cc
    -> 2 Cc + 4 (rails excluded); paper rule on the chain -> N/2 + 1."""
    assert oracle.greedy_color(netgen.inverter_chain(1000))[1] == 4
    assert oracle.greedy_color(netgen.inverter_chain(1000), "paper")[1] == 1001
    assert oracle.greedy_color(netgen.ring_oscillators(20, 101))[1] == 6
    assert oracle.greedy_color(netgen.ring_oscillators(5, 101, fanout=4))[1] == 12
    for r, cc in ((16, 32), (8, 64)):
        assert oracle.greedy_color(netgen.sram_6t(r, cc))[1] == 2 * cc + 4
        assert oracle.greedy_color(netgen.sram_6t(r, cc), "paper")[1] == 2 * r * cc


def test_ota_5t():
    """P:61 Fig. 3 example re-derived: M1..M5 -> (0,1,1,2,2)."""
    c, C = oracle.greedy_color(netgen.ota_5t())
    assert list(c) == [0, 1, 1, 2, 2] and C == 3


@pytest.mark.parametrize("seed", range(100))
def test_random_graphs_match_brute_force(seed):
    """S:566 acceptance 2: 100 random conflict graphs (<= 200 vertices):
    identical to brute-force first-fit, valid, and C <= max_degree + 1."""
    rng = np.random.Generator(np.random.PCG64(seed))
    N = int(rng.integers(1, 200))
    nn = int(rng.integers(2, 3 * N + 3))
    T = rng.integers(-1, nn, size=(N, 4))
    rails = [int(rng.integers(0, nn))] if seed % 2 else []
    nl = fets([tuple(t) for t in T], nn, rails=rails)
    for rule in ("exclude_rails", "paper"):
        c, C = oracle.greedy_color(nl, rule)
        want = brute_first_fit(nl, rule)
        assert np.array_equal(c, want)
        assert oracle.color_violations(nl, c, C, rule) == 0
        ex = set(rails) if rule == "exclude_rails" else set()
        sets = [set(t for t in row if t >= 0 and t not in ex) for row in T.tolist()]
        deg = max((sum(1 for j in range(N) if j != i and sets[i] & sets[j]) for i in range(N)), default=0)
        assert C <= deg + 1


def test_corrupted_colouring_detected():
    """S:362 negative test: put two adjacent devices in one colour."""
    nl = netgen.ring_oscillators(3, 101)
    c, C = oracle.greedy_color(nl)
    assert oracle.color_violations(nl, c, C) == 0
    bad = c.copy()
    bad[1] = bad[0]            # N0 and P0 share in/out nodes
    assert oracle.color_violations(nl, bad, C) > 0


@pytest.mark.parametrize("cfg", [0, 1, 2, 4])
def test_conflict_iff_shared_slot(cfg):
    """S:299 / acceptance 3: under the paper rule, two devices are adjacent
    iff their stamp plans share an A entry or b row (checked on circuits of
    <= 100 FETs, exhaustively)."""
    nl = netgen.config(cfg, 0.0001)
    nl = netgen.custom("cut", nl.n_nodes, list(zip(nl.d[:100], nl.g[:100], nl.s[:100], nl.b[:100])),
                       nl.model[:100], nl.models, rails=nl.rails)
    _, _, keys = oracle.pattern(nl)
    n = nl.n
    T = np.stack([nl.d, nl.g, nl.s, nl.b], 1).tolist()
    slots = []
    for t in T:
        s = {a * n + c for a in t for c in t if a >= 0 and c >= 0}
        s |= {-1 - a for a in t if a >= 0}
        slots.append(s)
    nodes = [set(x for x in t if x >= 0) for t in T]
    for i in range(len(T)):
        for j in range(i + 1, len(T)):
            assert bool(slots[i] & slots[j]) == bool(nodes[i] & nodes[j])


def test_hybrid_counts():
    """excluding every node with more than 16
    incident FETs collapses SRAM 64x128 from 260 colours to 5 and the hub
    netlist (60k inverters) from its max hub fanout to 4."""
    nl = netgen.sram_6t(64, 128)
    assert oracle.greedy_color(nl)[1] == 260
    c, C = oracle.greedy_color(nl, "hybrid", 16)
    assert C == 5 and oracle.color_violations(nl, c, C, "hybrid", 16) == 0
    nl = netgen.hub_netlist(60000)
    assert oracle.greedy_color(nl)[1] == int(oracle.node_fanout(nl)[np.setdiff1d(
        np.arange(nl.n_nodes), nl.rails)].max())
    c, C = oracle.greedy_color(nl, "hybrid", 16)
    assert C == 4 and oracle.color_violations(nl, c, C, "hybrid", 16) == 0


def test_hybrid_reduces_to_exclude_rails():
    """With K at least the largest non-rail fanout, the hybrid excludes only
    the rails: the colouring is the A1 one."""
    nl = netgen.ring_oscillators(10, 101, fanout=4)
    K = int(oracle.node_fanout(nl)[np.setdiff1d(np.arange(nl.n_nodes), nl.rails)].max())
    assert np.array_equal(oracle.greedy_color(nl, "hybrid", K)[0], oracle.greedy_color(nl)[0])
    assert oracle.greedy_color(nl, "hybrid", K - 1)[1] < oracle.greedy_color(nl)[1]


@pytest.mark.parametrize("seed", range(30))
def test_hybrid_random_graphs_match_brute_force(seed):
    rng = np.random.Generator(np.random.PCG64(500 + seed))
    N = int(rng.integers(1, 200))
    nn = int(rng.integers(2, N // 2 + 3))
    T = rng.integers(-1, nn, size=(N, 4))
    rails = [int(rng.integers(0, nn))] if seed % 2 else []
    nl = fets([tuple(t) for t in T], nn, rails=rails)
    for K in (1, 3, 8):
        c, C = oracle.greedy_color(nl, "hybrid", K)
        assert np.array_equal(c, brute_first_fit(nl, "hybrid", K))
        assert oracle.color_violations(nl, c, C, "hybrid", K) == 0


# ---------------------------------------------------------------- Benchmark 2 (NEXT-3)
def test_adder_28t_matches_paper_counts():
    """P:101-105 / Table II: the 64-bit ripple-carry adder of 28T
    full adders has 1,792 FETs and 89 non-ground terminal attachments per bit
    (R89 = "all transistor-to-transistor connections"); under the paper's
    conflict rule (VDD shared by every PMOS) greedy gives C = 896;
    after R89 every FET is on private nets and C = 1."""
    nl = netgen.full_adder_28t(64)
    assert nl.n_dev == 1792
    T = np.stack([nl.d, nl.g, nl.s, nl.b], 1)
    assert (T >= 0).sum() == 89 * 64
    c, C = oracle.greedy_color(nl, "paper")
    assert C == 896 and oracle.color_violations(nl, c, C, "paper") == 0
    r89 = netgen.insert_resistors(nl, "all")
    assert r89.meta["resistors"] == 89 * 64
    for rule in ("paper", "exclude_rails"):
        assert oracle.greedy_color(r89, rule)[1] == 1


def test_adder_resistor_split_is_topological():
    """A series resistor moves one terminal to a fresh node: per FET the
    multiset of (old) nets is unchanged, and the new node's only other
    attachment is the resistor (linear extra entries)."""
    nl = netgen.full_adder_28t(4)
    r = netgen.insert_resistors(nl, 14, seed=3)
    new_of = r.meta["new_of"]
    assert len(new_of) == 14 * 4
    T0 = np.stack([nl.d, nl.g, nl.s, nl.b], 1)
    T1 = np.stack([r.d, r.g, r.s, r.b], 1).astype(np.int64)
    back = np.where(T1 >= nl.n_nodes, new_of[np.clip(T1 - nl.n_nodes, 0, None)], T1)
    assert np.array_equal(back, T0)
    assert np.array_equal(np.sort(np.unique(T1[T1 >= nl.n_nodes])), np.arange(nl.n_nodes, r.n_nodes))
