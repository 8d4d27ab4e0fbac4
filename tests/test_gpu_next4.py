"""NEXT-4: the steps either side of the hot path in the
library -- the linear pre-pass (ees_stamp_linear) and the sparse LU solve
(ees_solver_*, KLU's role in the paper's NR loop) -- checked against
plain numpy on the same matrices, and a transient of a full cfg1-size ring
circuit (202,000 FETs) through them."""
import numpy as np
import pytest

import netgen
import oracle

pytestmark = pytest.mark.gpu


def _ctx(nl, **kw):
    from paper_2604_03079_b200 import Context
    return Context.from_netlist(nl, **kw)


def _dense(rp, ci, vals, n):
    A = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(rp))
    np.add.at(A, (rows, ci), vals)
    return A


def test_stamp_linear_scatter_add(cuda_ok):
    """A[slot] += val, b[row] += bval, repeated slots accumulating."""
    import torch
    nl = netgen.config(1, 0.01)
    ctx = _ctx(nl, variant="atomic")
    rng = np.random.Generator(np.random.PCG64(3))
    slot = rng.integers(0, ctx.nnz, 500)
    val = rng.standard_normal(500)
    row = rng.integers(0, ctx.n, 200).astype(np.int32)
    bval = rng.standard_normal(200)
    A0 = rng.standard_normal(ctx.nnz)
    b0 = rng.standard_normal(ctx.n)
    A = torch.from_numpy(A0.copy()).cuda()
    b = torch.from_numpy(b0.copy()).cuda()
    ctx.stamp_linear(torch.from_numpy(slot).cuda(), torch.from_numpy(val).cuda(),
                     torch.from_numpy(row).cuda(), torch.from_numpy(bval).cuda(), A, b)
    torch.cuda.synchronize()
    wa, wb = A0.copy(), b0.copy()
    np.add.at(wa, slot, val)
    np.add.at(wb, row, bval)
    assert np.allclose(A.cpu().numpy(), wa, rtol=0, atol=1e-12)
    assert np.allclose(b.cpu().numpy(), wb, rtol=0, atol=1e-12)
    ctx.close()


def _system(nl, ctx):
    """The NR matrix of one iteration (oracle stamps + rail sources), as the
    CSR values of the context's pattern, and its right-hand side."""
    ref = oracle.reference(nl)
    rp, ci = ctx.pattern()
    assert np.array_equal(rp, ref["row_ptr"]) and np.array_equal(ci, ref["col_idx"])
    A, b = ref["A"].copy(), ref["b"].copy()
    for k, r in enumerate(nl.rails):
        br = nl.n_nodes + k
        A[ctx.find_slot(int(r), br)] += 1.0
        A[ctx.find_slot(br, int(r))] += 1.0
        b[br] += 1.0
    return rp, ci, A, b


@pytest.mark.parametrize("cfg,scale", [(0, 1.0), (1, 0.02), (2, 0.002), (4, 0.0005)])
def test_solver_matches_dense_solve(cuda_ok, cfg, scale):
    """ees_solver (host ordering + pivoting, GPU refactorisation and solves)
    equals numpy's dense solve of the same system, and refactorising at new
    values (a later NR iterate) still solves exactly."""
    import torch
    from paper_2604_03079_b200 import Solver
    nl = netgen.config(cfg, scale)
    ctx = _ctx(nl, variant="atomic")
    rp, ci, A, b = _system(nl, ctx)
    n = ctx.n
    Ad = _dense(rp, ci, A, n)
    want = np.linalg.solve(Ad, b)
    s = Solver(ctx, A)
    dA, db = torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda()
    x = torch.empty_like(db)
    s.factor(dA)
    s.solve(db, x)
    torch.cuda.synchronize()
    got = x.cpu().numpy()
    scale_x = max(1.0, np.abs(want).max())
    assert np.abs(got - want).max() <= 1e-8 * scale_x
    # a later NR iterate: same pattern, new values, same ordering and pivots
    nl2 = netgen.Netlist(**{**nl.__dict__, "x": want.copy()})
    _, _, A2, b2 = _system(nl2, ctx)
    want2 = np.linalg.solve(_dense(rp, ci, A2, n), b2)
    s.factor(torch.from_numpy(A2).cuda())
    s.solve(torch.from_numpy(b2).cuda(), x)
    torch.cuda.synchronize()
    assert np.abs(x.cpu().numpy() - want2).max() <= 1e-8 * max(1.0, np.abs(want2).max())
    fl, fu = s.fill()
    assert fl >= 0 and fu >= n
    s.close()
    ctx.close()


def test_transient_full_cfg1(cuda_ok):
    """Two backward-Euler steps of the full cfg1 circuit (1,000 rings x 101
    stages, 202,000 FETs, 101,002 unknowns) entirely through the library:
    pre-pass, eval+stamp, sparse refactorisation + solve, accept.  Every NR
    loop converges and the rail sits at its source; then the system
    re-assembled at the final iterate is solved by the library and by
    SciPy's SuperLU (an independent sparse LU): same solution, and each row's
    residual is within rounding of that row's magnitude."""
    import scipy.sparse as sps
    import scipy.sparse.linalg as spla
    import torch
    from paper_2604_03079_b200.transient import Transient, rail_sources
    nl = netgen.config(1)
    ctx = _ctx(nl, variant="auto")
    tr = Transient(ctx, rail_sources(nl))
    xs, its = tr.run(torch.from_numpy(nl.x.copy()).cuda(), nl.h, 2, abstol=1e-10, reltol=1e-9)
    assert max(its) < 50
    x = xs[-1]
    assert abs(x[int(nl.rails[0])].item() - 1.0) < 1e-12
    A, b = tr.assemble(x, nl.h)
    x1 = torch.empty_like(b)
    tr.solve(A, b, x1)
    torch.cuda.synchronize()
    rp, ci = ctx.pattern()
    Ah, bh, xg = A.cpu().numpy(), b.cpu().numpy(), x1.cpu().numpy()
    M = sps.csr_matrix((Ah, ci, rp), shape=(ctx.n, ctx.n))
    xs_ref = spla.spsolve(M.tocsc(), bh)
    assert np.abs(xg - xs_ref).max() <= 1e-8 * max(1.0, np.abs(xs_ref).max())
    r = np.abs(M @ xg - bh)
    mag = abs(M) @ np.abs(xg) + np.abs(bh)
    assert (r <= 1e-10 * mag + 1e-300).all(), float((r / np.maximum(mag, 1e-300)).max())
    tr.close()
    ctx.close()
