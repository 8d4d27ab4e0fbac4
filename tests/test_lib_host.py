"""Host logic of the C-ABI library, no GPU: the exported symbols, argument
validation, and that the library's setup (pattern, colouring) equals the
independent oracle bit for bit.  CPU only."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import netgen
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    from paper_2604_03079_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "ees.h")).read()
    declared = set(re.findall(r"^(?:ees_status|int64_t|const char \*)\s*(ees_\w+)\s*\(", hdr, re.M))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert getattr(_lib.lib, name) is not None


def _ctx(nl, **kw):
    from paper_2604_03079_b200 import Context
    return Context.from_netlist(nl, host_only=True, **kw)


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_pattern_equals_oracle(cfg):
    nl = netgen.config(cfg, 0.01)
    c = _ctx(nl)
    rp, ci = c.pattern()
    orp, oci, _ = oracle.pattern(nl)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    for k in range(0, len(ci), max(1, len(ci) // 50)):
        r = int(np.searchsorted(rp, k, side="right") - 1)
        assert c.find_slot(r, int(ci[k])) == k


@pytest.mark.parametrize("rule", ["exclude_rails", "paper"])
@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_colouring_equals_oracle(cfg, rule):
    nl = netgen.config(cfg, 0.01)
    c = _ctx(nl, rule=rule)
    col, C_ = c.colors()
    ocol, oC = oracle.greedy_color(nl, rule)
    assert C_ == oC
    assert np.array_equal(col, ocol)
    assert oracle.color_violations(nl, col, C_, rule) == 0


@pytest.mark.parametrize("seed", range(40))
def test_colouring_random_small(seed):
    rng = np.random.Generator(np.random.PCG64(1000 + seed))
    N = int(rng.integers(1, 400)); nn = int(rng.integers(2, N + 3))
    T = rng.integers(-1, nn, size=(N, 4))
    rails = sorted(set(int(v) for v in rng.integers(0, nn, int(rng.integers(0, 3)))))
    nl = netgen.custom("r", nn, [tuple(t) for t in T], 0, netgen.bench_models(), rails=rails)
    for rule in ("exclude_rails", "paper"):
        col, C_ = _ctx(nl, rule=rule).colors()
        ocol, oC = oracle.greedy_color(nl, rule)
        assert C_ == oC and np.array_equal(col, ocol)


@pytest.mark.parametrize("K", [4, 16, 64])
@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_hybrid_colouring_equals_oracle(cfg, K):
    """the library's degree-threshold hybrid colouring
    equals the oracle's first-fit over the same excluded set."""
    nl = netgen.config(cfg, 0.01)
    c = _ctx(nl, rule="hybrid", heavy_degree=K)
    col, C_ = c.colors()
    ocol, oC = oracle.greedy_color(nl, "hybrid", K)
    assert C_ == oC and np.array_equal(col, ocol)
    assert oracle.color_violations(nl, col, C_, "hybrid", K) == 0
    st = c.stats()
    assert st["n_excluded_nodes"] == int(oracle.excluded_mask(nl, "hybrid", K)[:nl.n_nodes].sum())


def test_hybrid_side_targets_sram():
    """SRAM R x Cc with K = 16: the bit and word lines leave the relation.
    Side targets are the heavy diagonals and heavy b rows (WL, BL, BLB: 3 per
    column/row group) plus the rail's; the (BL, WL) cross entries have one
    writer each and stay plain."""
    R, Cc = 64, 128
    nl = netgen.sram_6t(R, Cc)
    st = _ctx(nl, rule="hybrid", heavy_degree=16).stats()
    heavy = R + 2 * Cc                       # word lines + bit lines (+ the rail)
    assert st["n_excluded_nodes"] == heavy + 1
    assert st["n_color_side_targets"] == 2 * (heavy + 1)
    assert st["n_colors"] == 5


def test_full_size_colour_counts():
    """C(cfg0..cfg2) = 4, 6, 2052 (rails excluded); the
    library's incidence/bitset first-fit equals the plain oracle at full size."""
    for cfg, want in ((0, 4), (1, 6), (2, 2052)):
        nl = netgen.config(cfg)
        col, C_ = _ctx(nl).colors()
        assert C_ == want
        if cfg < 2:
            assert np.array_equal(col, oracle.greedy_color(nl)[0])


def test_invalid_descriptors():
    from paper_2604_03079_b200 import Context, EESError
    nl = netgen.inverter_chain(4)
    bad = []
    d2 = nl.d.copy(); d2[0] = nl.n_nodes          # node id out of range
    bad.append(dict(d=d2))
    w2 = nl.w.copy(); w2[1] = 0.0                 # W must be > 0
    bad.append(dict(w=w2))
    m2 = nl.model.copy(); m2[0] = 5               # model index out of range
    bad.append(dict(model=m2))
    bad.append(dict(rails=[nl.rails[0], nl.rails[0]]))     # duplicate rail
    bad.append(dict(extra_row=[nl.n], extra_col=[0]))       # extra entry out of range
    bad.append(dict(gmin=-1.0))
    bad.append(dict(models=[dict(polarity=2, vt0=0.3, kp=2e-5, lam=0, cgs=0, cgd=0, cdb=0)]))
    bad.append(dict(models=[dict(polarity=1, vt0=0.3, kp=0.0, lam=0, cgs=0, cgd=0, cdb=0)]))
    base = dict(n_nodes=nl.n_nodes, n_extra=nl.n_extra, d=nl.d, g=nl.g, s=nl.s, b=nl.b, w=nl.w,
                l=nl.l, model=nl.model, vprev=nl.vprev, models=nl.models, rails=nl.rails,
                extra_row=nl.extra_row, extra_col=nl.extra_col, host_only=True)
    Context(**base).close()
    for over in bad:
        kw = dict(base); kw.update(over)
        if "extra_row" in over:
            kw["extra_col"] = over["extra_col"]
        with pytest.raises(EESError) as e:
            Context(**kw)
        assert e.value.status == -1


def test_descriptor_size_limits():
    """n_dev beyond the int32 device lists, and negative sizes, are refused
    before any array is read (the pointers here are deliberately null)."""
    from paper_2604_03079_b200 import _lib
    m = _lib.ees_model(1, 0, 0.3, 2e-5, 0.0, 0.0, 0.0, 0.0)
    for n_dev, n_nodes in ((2 ** 31, 4), (-1, 4), (0, -1)):
        desc = _lib.ees_desc(n_nodes=n_nodes, n_extra=0, n_dev=n_dev, n_models=1,
                             models=C.cast(C.pointer(m), C.c_void_p), flags=_lib.EES_SETUP_HOST_ONLY)
        h = C.c_void_p()
        assert _lib.lib.ees_setup(C.byref(desc), C.byref(h)) == _lib.EES_EINVAL
        assert not h.value


def test_host_only_refuses_eval():
    from paper_2604_03079_b200 import _lib
    c = _ctx(netgen.inverter_chain(4))
    buf = (C.c_double * 64)()
    st = _lib.lib.ees_eval_stamp(c._h, buf, 1e-12, buf, buf, None)
    assert st == _lib.EES_ESTATE
    assert _lib.lib.ees_eval_stamp(c._h, buf, 0.0, buf, buf, None) == _lib.EES_EINVAL
    assert _lib.lib.ees_eval_stamp(c._h, buf, float("nan"), buf, buf, None) == _lib.EES_EINVAL
    assert _lib.lib.ees_eval_stamp(None, buf, 1e-12, buf, buf, None) == _lib.EES_EINVAL
    # NEXT-4 calls: no device state on a host-only context; argument checks first
    assert _lib.lib.ees_accept(c._h, buf, None) == _lib.EES_ESTATE
    assert _lib.lib.ees_accept(None, buf, None) == _lib.EES_EINVAL
    assert _lib.lib.ees_set_work(c._h, 0) == _lib.EES_EINVAL
    assert _lib.lib.ees_set_work(c._h, 50) == _lib.EES_OK
    assert _lib.lib.ees_set_work(None, 2) == _lib.EES_EINVAL
    assert _lib.lib.ees_fp64_peak(None) == _lib.EES_EINVAL
    assert _lib.lib.ees_set_variant(c._h, 6) == _lib.EES_EINVAL
    assert _lib.lib.ees_set_variant(c._h, _lib.EES_COLOR_BUF) == _lib.EES_OK


def test_empty_netlist():
    nl = netgen.custom("empty", 3, np.zeros((0, 4), np.int64), 0, netgen.bench_models())
    c = _ctx(nl)
    st = c.stats()
    assert st["n_dev"] == 0 and st["nnz"] == 0 and st["n_colors"] == 0


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_tile_structure(cfg):
    """EES_TILE setup: every live contribution is listed exactly once (checked
    inside ees_setup, which fails otherwise); heavy nodes and side targets as
    expected from the topology."""
    nl = netgen.config(cfg, 0.01)
    st = _ctx(nl).stats()
    assert st["n_tiles"] >= 1
    assert st["n_tile_items"] >= st["n_dev"]
    if cfg in (0, 1):
        # VDD is the only heavy node; A[VDD,VDD] and b[VDD] are side targets
        # once the FETs span more than one tile
        assert st["n_heavy_nodes"] == 1
        assert st["n_side_targets"] == (2 if st["n_tiles"] > 1 else 0)


@pytest.mark.parametrize("seed", range(30))
def test_tile_structure_random(seed):
    rng = np.random.Generator(np.random.PCG64(77 + seed))
    N = int(rng.integers(1, 3000)); nn = int(rng.integers(2, 200))
    T = rng.integers(-1, nn, size=(N, 4))
    hubs = rng.integers(0, nn, 3)
    T[rng.random(N) < 0.3, 1] = hubs[0]          # a few high-fanout gates -> heavy nodes
    rails = [int(hubs[1])] if seed % 2 else []
    nl = netgen.custom("r", nn, [tuple(t) for t in T], 0, netgen.bench_models(), rails=rails)
    st = _ctx(nl).stats()
    assert st["n_tile_items"] >= N


@pytest.mark.parametrize("split", [None, 14, "all"])
@pytest.mark.parametrize("rule", ["exclude_rails", "paper", "hybrid"])
def test_adder_setup_equals_oracle(split, rule):
    """Benchmark 2 netlists (NEXT-3): pattern (with the resistors'
    extra entries) and colouring equal the oracle's; tiles build even when
    split nets leave rows with no FET."""
    nl = netgen.full_adder_28t(64)
    if split is not None:
        nl = netgen.insert_resistors(nl, split)
    c = _ctx(nl, rule=rule)
    rp, ci = c.pattern()
    orp, oci, _ = oracle.pattern(nl)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    col, C_ = c.colors()
    ocol, oC = oracle.greedy_color(nl, rule)
    assert C_ == oC and np.array_equal(col, ocol)
    assert c.stats()["n_tiles"] >= 1


def test_invalid_hybrid_threshold():
    from paper_2604_03079_b200 import Context, EESError
    nl = netgen.inverter_chain(4)
    with pytest.raises(EESError):
        Context.from_netlist(nl, rule="hybrid", heavy_degree=-1, host_only=True)
    c = Context.from_netlist(nl, rule="hybrid", heavy_degree=0, host_only=True)   # 0 = default 64
    assert c.stats()["n_excluded_nodes"] == 1                                      # the rail


def test_tile_single_giant_node():
    """TILE setup on a star: one light-by-count node would hold every FET;
    it becomes heavy and its entries go to side parts (setup must not fail)."""
    N = 3000
    terms = [(i + 1, 0, -1, -1) for i in range(N)]            # all gates on node 0
    nl = netgen.custom("star", N + 1, terms, 0, netgen.bench_models())
    c = _ctx(nl)
    st = c.stats()
    assert st["n_tiles"] >= N // 128 and st["n_heavy_nodes"] >= 1 and st["n_side_targets"] >= 2


@pytest.mark.parametrize("form,stage", [(0, 11264), (1, 9360)])
def test_tile_forms_build_within_stage(form, stage):
    """Both TILE forms (items in the blob / in HBM arrays) build on every
    structure, each blob within its pipeline stage (the builder's byte bound
    is an upper bound: setup would fail otherwise)."""
    nets = [netgen.config(c, 0.01 if c else 1.0) for c in range(5)]
    nets += [netgen.full_adder_28t(16), netgen.insert_resistors(netgen.full_adder_28t(8), "all"),
             netgen.ring_oscillators(20, 101, fanout=4), netgen.gen_synth(5000, 300)]
    rng = np.random.Generator(np.random.PCG64(77))
    for _ in range(6):
        N = int(rng.integers(50, 3000)); nn = int(rng.integers(5, N))
        T = rng.integers(-1, nn, size=(N, 4))
        nets.append(netgen.custom("r", nn, [tuple(t) for t in T], 0, netgen.bench_models(),
                                  rails=[int(rng.integers(0, nn))]))
    for nl in nets:
        st = _ctx(nl, tile_form=form).stats()
        assert st["tile_form"] == form
        assert st["n_tiles"] >= 1 and st["tile_blob_max"] <= stage, nl.name


def test_tile_builder_independent_of_thread_count():
    """The TILE blobs are emitted in parallel and concatenated in tile order:
    the structure must not depend on the host thread count (setup with 1 and
    with 4 OpenMP threads, in subprocesses)."""
    import json
    import subprocess
    import sys
    code = ("import json, netgen; from paper_2604_03079_b200 import Context\n"
            "out = {}\n"
            "for c in (2, 3, 4):\n"
            "    st = Context.from_netlist(netgen.config(c, 0.02), host_only=True).stats()\n"
            "    out[c] = [st[k] for k in ('n_tiles', 'n_tile_items', 'tile_blob_max', 'n_side_targets',"
            " 'n_heavy_nodes', 'tile_form')]\n"
            "print(json.dumps(out))\n")
    res = []
    for threads in ("1", "4"):
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                           cwd=ROOT, env=dict(os.environ, OMP_NUM_THREADS=threads))
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert res[0] == res[1]


def test_abi_struct_sizes_match_binding():
    """The binding refuses a library built with other struct layouts; the
    library reports its own sizes (0: ees_desc, 1: ees_stats_t, else 0)."""
    from paper_2604_03079_b200 import _lib
    assert _lib.lib.ees_abi_sizeof(0) == C.sizeof(_lib.ees_desc)
    assert _lib.lib.ees_abi_sizeof(1) == C.sizeof(_lib.ees_stats_t)
    assert _lib.lib.ees_abi_sizeof(7) == 0


def test_tile_bank_placement_never_worse():
    """TILE form 1: the builder's bank-aware lane placement and pair
    orientation (hill-climbs from the identity placement on its 16-bank-pair
    model of the evaluation's STS.64) never raise the modelled store
    wavefronts, and lower them where half-warps collide (the SRAM rows)."""
    nets = [netgen.config(c, 0.01 if c else 1.0) for c in range(5)]
    nets += [netgen.full_adder_28t(16), netgen.ring_oscillators(20, 101, fanout=4)]
    gained = 0
    for nl in nets:
        st = _ctx(nl, tile_form=1).stats()
        assert 0 < st["tile_store_waves"] <= st["tile_store_waves_naive"], nl.name
        gained += st["tile_store_waves"] < st["tile_store_waves_naive"]
    assert gained >= 1
    st = _ctx(netgen.config(2, 0.01), tile_form=0).stats()
    assert st["tile_store_waves"] == 0 and st["tile_store_waves_naive"] == 0
