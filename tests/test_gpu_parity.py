"""Parity of the CUDA path (through the C ABI) against the independent CPU
oracle: per entry |A_gpu - A_ref| <= 1e-12 * sum|c| (BASELINE.json
north_star), pattern set-equality, colouring bit-exact and
conflict-free, determinism, race instrument, edge cases."""
import math

import numpy as np
import pytest

import netgen
import oracle

pytestmark = pytest.mark.gpu
TOL = 1e-12
VARIANTS = ["color", "atomic", "gather", "tile", "color_buf"]

_ref_cache = {}


def ctx_for(nl, **kw):
    from paper_2604_03079_b200 import Context
    return Context.from_netlist(nl, **kw)


def reference(nl, key=None, A0=None, b0=None):
    if key is not None and key in _ref_cache:
        return _ref_cache[key]
    r = oracle.reference(nl, A0=A0, b0=b0)
    if key is not None:
        _ref_cache.clear()          # keep at most one full-size reference alive
        _ref_cache[key] = r
    return r


def gpu_run(ctx, nl, variant=None, h=None, A0=None, b0=None, x=None):
    import torch
    if variant is not None:
        ctx.set_variant(variant)
    dev = torch.device("cuda")
    xt = torch.from_numpy(nl.x if x is None else x).to(dev)
    A = (torch.zeros(ctx.nnz, dtype=torch.float64, device=dev) if A0 is None
         else torch.from_numpy(np.array(A0, float)).to(dev))
    b = (torch.zeros(ctx.n, dtype=torch.float64, device=dev) if b0 is None
         else torch.from_numpy(np.array(b0, float)).to(dev))
    ctx.eval_stamp(xt, nl.h if h is None else h, A, b)
    torch.cuda.synchronize()
    return A.cpu().numpy(), b.cpu().numpy()


def assert_parity(ref, A, b, what=""):
    for got, want, mag, name in ((A, ref["A"], ref["A_abs"], "A"), (b, ref["b"], ref["b_abs"], "b")):
        err = np.abs(got - want)
        bad = ~(err <= TOL * mag)          # NaN-safe: NaN counts as bad
        if bad.any():
            k = int(np.argmax(np.where(bad, err / np.maximum(mag, 1e-300), 0)))
            raise AssertionError(f"{what} {name}: {int(bad.sum())} entries out of tolerance; worst k={k} "
                                 f"got={got[k]!r} want={want[k]!r} sum|c|={mag[k]!r}")


def assert_pattern(ctx, ref):
    rp, ci = ctx.pattern()
    assert np.array_equal(rp, ref["row_ptr"]) and np.array_equal(ci, ref["col_idx"])


# ---------------------------------------------------------------- reduced configs
@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("rule", ["exclude_rails", "paper", "hybrid"])
def test_parity_reduced(cuda_ok, cfg, rule):
    nl = netgen.config(cfg, 0.01 if cfg else 1.0)
    if rule == "paper" and cfg in (2, 4):
        nl = netgen.config(cfg, 0.001)
    ref = reference(nl)
    ctx = ctx_for(nl, rule=rule)
    assert_pattern(ctx, ref)
    col, C = ctx.colors()
    assert np.array_equal(col, oracle.greedy_color(nl, rule)[0])
    assert oracle.color_violations(nl, col, C, rule) == 0
    assert ctx.race_probe() == 0
    for v in VARIANTS:
        A, b = gpu_run(ctx, nl, v)
        assert_parity(ref, A, b, f"cfg{cfg} {rule} {v}")
    ctx.close()


# ---------------------------------------------------------------- full size
@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_parity_full_size(cuda_ok, cfg):
    """BASELINE.json configs at full size, every variant, in the launch
    configuration bench.py times; all entries compared."""
    nl = netgen.config(cfg)
    ref = reference(nl, key=("full", cfg))
    ctx = ctx_for(nl, variant="auto")
    assert_pattern(ctx, ref)
    st = ctx.stats()
    col, C = ctx.colors()
    ocol, oC = oracle.greedy_color(nl)
    assert C == oC and np.array_equal(col, ocol)
    assert oracle.color_violations(nl, col, C) == 0
    for v in VARIANTS:
        if v in ("color", "color_buf") and st["n_colors"] > 600:
            continue        # thousands of launches; covered on reduced instances
        A, b = gpu_run(ctx, nl, v)
        assert_parity(ref, A, b, f"cfg{cfg} full {v}")
    ctx.set_variant("auto")
    A, b = gpu_run(ctx, nl)
    assert_parity(ref, A, b, f"cfg{cfg} full auto={st['variant_chosen']}")
    ctx.close()


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [2, 4])
def test_parity_full_size_color_high_c(cuda_ok, cfg):
    """The colour-phased variants at full size where C is in the thousands
    (cfg2 C = 2,052, cfg4 C = 4,088; one launch per colour): COLOR and
    COLOR_BUF under the default rule, every entry against the oracle."""
    nl = netgen.config(cfg)
    ref = reference(nl, key=("full", cfg))
    ctx = ctx_for(nl, variant="color")
    assert ctx.stats()["n_colors"] > 2000
    for v in ("color", "color_buf"):
        A, b = gpu_run(ctx, nl, v)
        assert_parity(ref, A, b, f"cfg{cfg} full {v}")
    ctx.close()


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [0, 1])
def test_parity_full_size_paper_rule(cuda_ok, cfg):
    """The paper-literal conflict rule (every shared non-ground node,
    VDD included) at full size: cfg0 C = 1,001, cfg1 C = 101,001 colour
    phases; colouring bit-equal to the oracle's and conflict-free, every
    variant within tolerance."""
    nl = netgen.config(cfg)
    ref = reference(nl, key=("full", cfg))
    ctx = ctx_for(nl, variant="color", rule="paper")
    col, C = ctx.colors()
    ocol, oC = oracle.greedy_color(nl, "paper")
    assert C == oC and np.array_equal(col, ocol)
    assert oracle.color_violations(nl, col, C, "paper") == 0
    for v in VARIANTS:
        A, b = gpu_run(ctx, nl, v)
        assert_parity(ref, A, b, f"cfg{cfg} full paper-rule {v}")
    ctx.close()


# ---------------------------------------------------------------- colour sweep (B5)
@pytest.mark.parametrize("ct", [1, 2, 7, 64, 333])
def test_parity_synth(cuda_ok, ct):
    nl = netgen.gen_synth(20000 + 37, ct)
    ref = reference(nl)
    ctx = ctx_for(nl)
    assert ctx.stats()["n_colors"] == ct
    for v in VARIANTS:
        assert_parity(ref, *gpu_run(ctx, nl, v), f"synth C={ct} {v}")


# ---------------------------------------------------------------- edge cases
def _tiny():
    ms = netgen.bench_models()
    yield netgen.custom("nmos", 3, [(0, 1, 2, -1)], 0, ms, seed=1)
    yield netgen.custom("allground", 2, [(-1, -1, -1, -1), (0, -1, -1, -1), (-1, 1, -1, -1)], 0, ms)
    yield netgen.custom("coincident", 3, [(0, 0, 0, 0), (1, 2, 1, -1), (2, 1, 2, 2)], [0, 1, 1], ms)
    yield netgen.ota_5t()
    yield netgen.inverter_chain(1)
    yield netgen.ring_oscillators(3, 101, fanout=4)
    yield netgen.custom("rails3", 6, [(0, 3, 4, 5), (3, 4, 5, 5), (1, 4, 3, 3), (2, 5, 0, 4)],
                        [1, 0, 1, 0], ms, rails=[3, 4, 5])


@pytest.mark.parametrize("nl", list(_tiny()), ids=lambda n: n.name)
def test_parity_tiny(cuda_ok, nl):
    ref = reference(nl)
    ctx = ctx_for(nl)
    assert_pattern(ctx, ref)
    for v in VARIANTS:
        assert_parity(ref, *gpu_run(ctx, nl, v), f"{nl.name} {v}")


def test_empty(cuda_ok):
    nl = netgen.custom("empty", 3, np.zeros((0, 4), np.int64), 0, netgen.bench_models())
    ctx = ctx_for(nl)
    for v in VARIANTS:
        A, b = gpu_run(ctx, nl, v, b0=np.arange(3.0))
        assert A.shape == (0,) and np.array_equal(b, np.arange(3.0))


def test_dc_and_accumulate(cuda_ok):
    """h = +inf (DC: caps open) and accumulate semantics with random
    initial A, b (included in sum|c|)."""
    nl = netgen.config(1, 0.02)
    rng = np.random.Generator(np.random.PCG64(3))
    ctx = ctx_for(nl)
    A0 = rng.uniform(-1, 1, ctx.nnz)
    b0 = rng.uniform(-1, 1, ctx.n)
    for h in (nl.h, math.inf):
        nl2 = netgen.Netlist(**{**nl.__dict__, "h": h})
        ref = oracle.reference(nl2, A0=A0, b0=b0)
        for v in VARIANTS:
            assert_parity(ref, *gpu_run(ctx, nl2, v, h=h, A0=A0, b0=b0), f"h={h} {v}")


def test_spec_card_all_cutoff(cuda_ok):
    nl = netgen.inverter_chain(300, models=netgen.spec_models())
    ref = reference(nl)
    ctx = ctx_for(nl)
    for v in VARIANTS:
        assert_parity(ref, *gpu_run(ctx, nl, v), f"spec card {v}")


def test_determinism(cuda_ok):
    """COLOR, COLOR_BUF, GATHER and TILE are bitwise reproducible run to run
    (fixed summation order); ATOMIC within tolerance."""
    nl = netgen.config(2, 0.02)
    ref = reference(nl)
    ctx = ctx_for(nl)
    for v in ("color", "gather", "tile", "color_buf"):
        A1, b1 = gpu_run(ctx, nl, v)
        for _ in range(3):
            A2, b2 = gpu_run(ctx, nl, v)
            assert np.array_equal(A1, A2) and np.array_equal(b1, b2)
    A, b = gpu_run(ctx, nl, "atomic")
    assert_parity(ref, A, b, "atomic")


def test_race_probe_detects_corrupted_schedule(cuda_ok):
    """S:362 negative test: two adjacent devices forced into one colour."""
    nl = netgen.ring_oscillators(4, 101)
    ctx = ctx_for(nl)
    col, C = ctx.colors()
    assert ctx.race_probe() == 0
    bad = col.copy()
    bad[1] = bad[0]
    assert ctx.race_probe(bad) > 0
    assert ctx.race_probe(np.zeros_like(col)) > 0


def test_nan_propagates(cuda_ok):
    """NaN in x is not checked (ees.h): it propagates exactly where the
    oracle's arithmetic propagates it (a NaN bias fails the cutoff test and
    poisons that FET's conductances and Norton terms)."""
    nl = netgen.inverter_chain(10)
    ctx = ctx_for(nl)
    nl.x[3] = np.nan
    ref = oracle.reference(nl)
    assert np.isnan(ref["b"]).any()
    for v in VARIANTS:
        A, b = gpu_run(ctx, nl, v)
        for got, want in ((A, ref["A"]), (b, ref["b"])):
            assert np.array_equal(np.isnan(got), np.isnan(want))
        for got, want, mag in ((A, ref["A"], ref["A_abs"]), (b, ref["b"], ref["b_abs"])):
            ok = ~np.isnan(want)
            assert np.all(np.abs(got[ok] - want[ok]) <= 1e-12 * mag[ok])


def test_host_buffer_call_matches(cuda_ok):
    nl = netgen.config(1, 0.05)
    ref = reference(nl)
    ctx = ctx_for(nl)
    for v in VARIANTS:
        ctx.set_variant(v)
        A = np.zeros(ctx.nnz)
        b = np.zeros(ctx.n)
        ctx.eval_stamp_host(nl.x, nl.h, A, b)
        assert_parity(ref, A, b, f"host {v}")
        A[:] = 7.0                                  # assign form ignores the inputs
        b[:] = -3.0
        ctx.eval_stamp_host(nl.x, nl.h, A, b, assign=True)
        assert_parity(ref, A, b, f"host assign {v}")


def test_abi_errors(cuda_ok):
    import torch
    from paper_2604_03079_b200 import EESError
    nl = netgen.inverter_chain(5)
    ctx = ctx_for(nl)
    x = torch.zeros(ctx.n, dtype=torch.float64, device="cuda")
    A = torch.zeros(ctx.nnz, dtype=torch.float64, device="cuda")
    b = torch.zeros(ctx.n, dtype=torch.float64, device="cuda")
    for h in (0.0, -1e-12, float("nan")):
        with pytest.raises(EESError):
            ctx.eval_stamp(x, h, A, b)
    with pytest.raises(ValueError):
        ctx.eval_stamp(x[:-1], 1e-12, A, b)
    with pytest.raises(ValueError):
        ctx.eval_stamp(x.float(), 1e-12, A, b)


@pytest.mark.parametrize("mode", ["launch", "coop"])
def test_color_forms(cuda_ok, mode):
    """Both COLOR forms: one launch per colour (Table I ColorFused) and
    the persistent cooperative kernel with a grid barrier per colour (Table I
    Color "single parallel region")."""
    for nl in (netgen.config(0), netgen.config(1, 0.05), netgen.gen_synth(5000, 40),
               netgen.ota_5t()):
        ref = reference(nl)
        ctx = ctx_for(nl, variant="color", color_mode=mode)
        A1, b1 = gpu_run(ctx, nl)
        assert_parity(ref, A1, b1, f"{nl.name} color/{mode}")
        A2, b2 = gpu_run(ctx, nl)
        assert np.array_equal(A1, A2) and np.array_equal(b1, b2)
        ctx.close()


# ---------------------------------------------------------------- NEXT-1 hybrid colouring
@pytest.mark.parametrize("cfg,K", [(2, 16), (2, 64), (4, 64), (1, 64), (3, 16)])
def test_hybrid_color_full_size(cuda_ok, cfg, K):
    """SURVEY §8(f) NEXT-1 at full size: COLOR under the degree-threshold
    hybrid (few colours even on the SRAM and hub configs), every entry within
    tolerance, colouring equal to the oracle's, race-free on the device, and
    bitwise reproducible."""
    nl = netgen.config(cfg)
    ref = reference(nl, key=("full", cfg))
    ctx = ctx_for(nl, variant="color", rule="hybrid", heavy_degree=K)
    col, C = ctx.colors()
    ocol, oC = oracle.greedy_color(nl, "hybrid", K)
    assert C == oC and np.array_equal(col, ocol)
    assert C <= 40
    assert ctx.race_probe() == 0
    A1, b1 = gpu_run(ctx, nl)
    assert_parity(ref, A1, b1, f"cfg{cfg} hybrid K={K} color")
    A2, b2 = gpu_run(ctx, nl)
    assert np.array_equal(A1, A2) and np.array_equal(b1, b2)
    ctx.close()


def test_hybrid_race_probe_detects_corruption(cuda_ok):
    nl = netgen.sram_6t(32, 64)
    ctx = ctx_for(nl, variant="color", rule="hybrid", heavy_degree=16)
    col, C = ctx.colors()
    assert C == 5 and ctx.race_probe() == 0
    assert ctx.race_probe(np.zeros_like(col)) > 0


# ---------------------------------------------------------------- Benchmark 2 (NEXT-3)
@pytest.mark.parametrize("variant_of", ["baseline", "R14", "R89"])
@pytest.mark.parametrize("rule", ["exclude_rails", "paper"])
def test_adder_parity(cuda_ok, variant_of, rule):
    """the 64-bit 28T ripple-carry adder and its R14 / R89
    series-resistor variants, every stamping variant, both conflict rules
    (paper rule: C = 896 / 1 for the baseline / R89, Table II)."""
    nl = netgen.full_adder_28t(64)
    if variant_of == "R14":
        nl = netgen.insert_resistors(nl, 14)
    elif variant_of == "R89":
        nl = netgen.insert_resistors(nl, "all")
    ref = reference(nl)
    ctx = ctx_for(nl, rule=rule)
    assert_pattern(ctx, ref)
    col, C = ctx.colors()
    ocol, oC = oracle.greedy_color(nl, rule)
    assert C == oC and np.array_equal(col, ocol)
    if rule == "paper":
        assert C == {"baseline": 896, "R89": 1}.get(variant_of, C)
    assert ctx.race_probe() == 0
    for v in VARIANTS:
        assert_parity(ref, *gpu_run(ctx, nl, v), f"{nl.name} {rule} {v}")
    ctx.close()


# ---------------------------------------------------------------- NEXT-4: accept, work multiplier
def test_accept_updates_state(cuda_ok):
    """S:212 update_state: after ees_accept(x1) the companion state of every
    FET is the branch voltages at x1 -- in every layout (all variants and the
    hybrid COLOR layout) -- checked against the oracle with vprev rebuilt
    from x1."""
    import torch
    nl = netgen.config(2, 0.01)
    rng = np.random.Generator(np.random.PCG64(11))
    x1 = nl.x.copy()
    x1[: nl.n_nodes] = rng.uniform(0, 1, nl.n_nodes)
    x1[nl.rails] = 1.0
    nl1 = netgen.Netlist(**{**nl.__dict__, "vprev": np.ascontiguousarray(netgen._vprev(x1, nl.d, nl.g, nl.s, nl.b))})
    ref0, ref1 = reference(nl), oracle.reference(nl1)
    assert not np.array_equal(ref0["b"], ref1["b"])
    for rule in ("exclude_rails", "hybrid"):
        ctx = ctx_for(nl, rule=rule, heavy_degree=16)
        assert_parity(ref0, *gpu_run(ctx, nl, "tile"), "before accept")
        ctx.accept(torch.from_numpy(x1).cuda())
        for v in VARIANTS:
            assert_parity(ref1, *gpu_run(ctx, nl, v), f"after accept {rule} {v}")
        ctx.close()


def test_work_multiplier_keeps_results(cuda_ok):
    """repeating the evaluation arithmetic k times leaves the result
    within the parity tolerance (the k > 1 kernels are separate
    instantiations, so FMA contraction may round differently), and the
    deterministic variants stay bitwise reproducible run to run."""
    nl = netgen.config(1, 0.02)
    ref = reference(nl)
    ctx = ctx_for(nl)
    ctx.set_work(9)
    for v in VARIANTS:
        A, b = gpu_run(ctx, nl, v)
        assert_parity(ref, A, b, f"{v} work=9")
        if v != "atomic":
            A2, b2 = gpu_run(ctx, nl, v)
            assert np.array_equal(A, A2) and np.array_equal(b, b2)
    from paper_2604_03079_b200 import EESError
    with pytest.raises(EESError):
        ctx.set_work(0)


def test_fp64_peak_plausible(cuda_ok):
    from paper_2604_03079_b200 import fp64_peak
    t = fp64_peak()
    assert 5.0 < t < 200.0


def test_red_throughput_plausible(cuda_ok):
    """K6 microbenchmark: spread REDs beat same-address REDs."""
    from paper_2604_03079_b200 import red_throughput
    spread, same = red_throughput(0), red_throughput(1)
    assert spread > 10.0 and same > 0.1 and spread > same


def test_cuda_graph_capture(cuda_ok):
    """ees_eval_stamp only enqueues work, so an NR loop can capture it in a
    CUDA graph (task: CUDA graphs instead of a tracing compiler): every
    variant captured once and replayed matches the oracle; the TILE ticket
    resets itself between replays."""
    import torch
    nl = netgen.config(1, 0.02)
    ref = reference(nl)
    ctx = ctx_for(nl)
    dev = torch.device("cuda")
    x = torch.from_numpy(nl.x).to(dev)
    A = torch.zeros(ctx.nnz, dtype=torch.float64, device=dev)
    b = torch.zeros(ctx.n, dtype=torch.float64, device=dev)
    for v in VARIANTS:
        ctx.set_variant(v)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):                  # warm up outside the capture
            ctx.eval_stamp(x, nl.h, A, b)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            A.zero_()
            b.zero_()
            ctx.eval_stamp(x, nl.h, A, b)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        assert_parity(ref, A.cpu().numpy(), b.cpu().numpy(), f"graph {v}")


def test_star_giant_node(cuda_ok):
    """Degenerate fanout: 3,000 FETs with every gate on one node (a 3,000-way
    hub: one colour each, a single-entry hot spot for ATOMIC, a heavy side
    target for TILE), both polarities, private drains."""
    N = 3000
    terms = [(i + 1, 0, -1 if i % 2 == 0 else N + 1, -1 if i % 2 == 0 else N + 1) for i in range(N)]
    nl = netgen.custom("star", N + 2, terms, [i % 2 for i in range(N)], netgen.bench_models(),
                       rails=[N + 1])
    ref = reference(nl)
    ctx = ctx_for(nl)
    assert ctx.stats()["n_colors"] == N
    for v in VARIANTS:
        if v in ("color", "color_buf"):
            continue                     # 3,000 colour launches; covered by the hybrid below
        assert_parity(ref, *gpu_run(ctx, nl, v), f"star {v}")
    ctx.close()
    ctx = ctx_for(nl, rule="hybrid", heavy_degree=64, variant="color")
    assert ctx.stats()["n_colors"] == 1
    assert_parity(ref, *gpu_run(ctx, nl), "star hybrid color")
    ctx.set_variant("color_buf")
    assert_parity(ref, *gpu_run(ctx, nl), "star hybrid color_buf")


# ---------------------------------------------------------------- NEXT-4: NR transient loop
def _cpu_transient(nl, sources, x0, h, steps, tol):
    """The same backward-Euler NR loop with every A, b from the oracle and a
    numpy dense solve (Fig. 1)."""
    xs = []
    x = x0.copy()
    vprev = nl.vprev.copy()
    for _ in range(steps):
        for _it in range(50):
            nl2 = netgen.Netlist(**{**nl.__dict__, "x": x, "vprev": vprev})
            ref = oracle.reference(nl2)
            n = nl.n
            A = np.zeros((n, n))
            rows = np.repeat(np.arange(n), np.diff(ref["row_ptr"]))
            np.add.at(A, (rows, ref["col_idx"]), ref["A"])
            b = ref["b"].copy()
            for node, br, v in sources:
                A[node, br] += 1.0
                A[br, node] += 1.0
                b[br] += v
            x_new = np.linalg.solve(A, b)
            done = np.abs(x_new - x).max() <= tol
            x = x_new
            if done:
                break
        vprev = np.ascontiguousarray(netgen._vprev(x, nl.d, nl.g, nl.s, nl.b))
        xs.append(x.copy())
    return xs


def test_transient_nr_loop_matches_oracle(cuda_ok):
    """NEXT-4: a 5-step backward-Euler transient of two 11-stage ring
    oscillators driven through ees_eval_stamp + ees_accept with a dense
    solve equals the same loop run on the oracle (every step, every node)."""
    import torch
    from paper_2604_03079_b200.transient import Transient, rail_sources
    nl = netgen.ring_oscillators(2, 11)
    src = rail_sources(nl)
    want = _cpu_transient(nl, src, nl.x.copy(), nl.h, 5, 1e-13)
    for v in ("tile", "atomic", "color"):
        ctx = ctx_for(nl, variant=v)
        tr = Transient(ctx, src)
        xs, its = tr.run(torch.from_numpy(nl.x.copy()).cuda(), nl.h, 5, abstol=1e-13, reltol=0.0)
        assert max(its) < 50
        for k, (g, w) in enumerate(zip(xs, want)):
            g = g.cpu().numpy()
            assert np.abs(g - w).max() <= 1e-9 * max(1.0, np.abs(w).max()), f"{v} step {k}"
        assert abs(g[nl.rails[0]] - 1.0) < 1e-12       # the rail stays at its source
        ctx.close()


def test_tile_results_independent_of_setup_threads(cuda_ok):
    """TILE is deterministic and its layout must not depend on how many host
    threads built it: A and b bit-identical for setups with 1 and 4 OpenMP
    threads (subprocesses), and within tolerance of the oracle."""
    import hashlib
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import hashlib, torch, netgen; from paper_2604_03079_b200 import Context\n"
            "nl = netgen.config(4, 0.02); ctx = Context.from_netlist(nl, variant='tile')\n"
            "x = torch.from_numpy(nl.x).cuda()\n"
            "A = torch.zeros(ctx.nnz, dtype=torch.float64, device='cuda'); b = torch.zeros(ctx.n, dtype=torch.float64, device='cuda')\n"
            "ctx.eval_stamp(x, nl.h, A, b); torch.cuda.synchronize()\n"
            "print(hashlib.sha256(A.cpu().numpy().tobytes() + b.cpu().numpy().tobytes()).hexdigest())\n")
    digests = []
    for threads in ("1", "4"):
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                           cwd=root, env=dict(os.environ, OMP_NUM_THREADS=threads))
        assert r.returncode == 0, r.stderr[-2000:]
        digests.append(r.stdout.strip().splitlines()[-1])
    assert digests[0] == digests[1]
    nl = netgen.config(4, 0.02)
    ctx = ctx_for(nl, variant="tile")
    A, b = gpu_run(ctx, nl)
    assert_parity(reference(nl), A, b, "cfg4@0.02 tile")
    assert hashlib.sha256(A.tobytes() + b.tobytes()).hexdigest() == digests[0]
    ctx.close()


def _form_nets():
    ms = netgen.bench_models()
    yield netgen.ring_oscillators(20, 101, fanout=4)          # targets of 10 contributions (group classes)
    yield netgen.gen_synth(6000, 300)                           # heavy cliques: side pieces, hot sums
    yield netgen.full_adder_28t(8)
    yield netgen.config(2, 0.01)
    yield netgen.config(3, 0.01)
    yield netgen.config(4, 0.01)
    rng = np.random.Generator(np.random.PCG64(91))
    for k in range(3):
        N = int(rng.integers(500, 4000)); nn = int(rng.integers(20, N // 4))
        T = rng.integers(-1, nn, size=(N, 4))
        yield netgen.custom(f"rand{k}", nn, [tuple(t) for t in T], [int(v) for v in rng.integers(0, 2, N)], ms,
                            rails=[int(rng.integers(0, nn))])


@pytest.mark.parametrize("form", [0, 1])
def test_tile_forms_parity(cuda_ok, form):
    """Both TILE program formats (form 0: op streams over the evaluation's
    p-major slots; form 1: contribution positions into pair rows, group
    area) on structures that exercise short and long owned targets, side
    pieces and hot sums, whatever form setup would choose."""
    for nl in _form_nets():
        ref = reference(nl)
        ctx = ctx_for(nl, variant="tile", tile_form=form)
        assert ctx.stats()["tile_form"] == form
        assert_parity(ref, *gpu_run(ctx, nl), f"{nl.name} tile form {form}")
        A1, b1 = gpu_run(ctx, nl)
        A2, b2 = gpu_run(ctx, nl)
        assert np.array_equal(A1, A2) and np.array_equal(b1, b2), f"{nl.name} form {form} not deterministic"
        ctx.close()
