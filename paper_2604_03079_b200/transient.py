"""The Newton-Raphson transient loop around the hot path (SURVEY.md §8(f)
NEXT-4, "the steps either side"): the loop of PAPER.md Fig. 1 and
SPEC.md's newton_step / run_transient.

Per NR iteration (S:426 order), every step in libees.so on the GPU: clear A
and b; ``ees_stamp_linear`` -- the caller's linear pre-pass, here the
ideal voltage sources that hold the rails; ``ees_eval_stamp`` -- the hot
path, every MOSFET evaluated and stamped; ``ees_solver_factor`` +
``ees_solver_solve`` -- the sparse LU (KLU's role): ordering and
pivots fixed at the first iteration (host), numeric refactorisation and
triangular solves on the GPU; then the convergence test max|dx| <= abstol +
reltol max|x|.  On convergence ``ees_accept`` stores the converged
branch voltages as the companion-model state of the next step.
This module only sequences those calls (and reads one convergence scalar
back per iteration).
"""
from __future__ import annotations

import torch

from .api import Solver


class Transient:
    """Backward-Euler transient of one netlist (a ``Context`` built from it).

    sources: list of (node, branch, volts): an ideal source holding `node`
    at `volts`, its current the unknown `branch` (rows n_nodes.. of x).  The
    netlist's pattern must hold the entries (node, branch) and (branch, node)
    (ees_desc extra entries)."""

    def __init__(self, ctx, sources, device=None):
        self.ctx = ctx
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        n = ctx.n
        slots, rows, vals = [], [], []
        for node, br, volts in sources:
            k1, k2 = ctx.find_slot(node, br), ctx.find_slot(br, node)
            if k1 < 0 or k2 < 0:
                raise ValueError(f"pattern lacks the source entries of node {node} / branch {br}")
            slots += [k1, k2]                     # KCL: +i_br at the node; branch row: V(node)
            rows.append(br)
            vals.append(float(volts))             # = volts
        self.lin_slot = torch.tensor(slots, dtype=torch.int64, device=self.dev)
        self.lin_val = torch.ones(len(slots), dtype=torch.float64, device=self.dev)
        self.lin_row = torch.tensor(rows, dtype=torch.int32, device=self.dev)
        self.lin_bval = torch.tensor(vals, dtype=torch.float64, device=self.dev)
        self.A = torch.zeros(ctx.nnz, dtype=torch.float64, device=self.dev)
        self.b = torch.zeros(n, dtype=torch.float64, device=self.dev)
        self.solver = None
        self.n = n

    def assemble(self, x, h):
        """A, b of one NR iteration at x (linear pre-pass, then the FET stamps)."""
        self.A.zero_()
        self.b.zero_()
        self.ctx.stamp_linear(self.lin_slot, self.lin_val, self.lin_row, self.lin_bval, self.A, self.b)
        self.ctx.eval_stamp(x, h, self.A, self.b)
        return self.A, self.b

    def solve(self, A, b, x_out):
        """x_out = A^-1 b: the first call orders and pivots (host LU at these
        values), every call refactorises on the GPU and solves."""
        if self.solver is None:
            self.solver = Solver(self.ctx, A.cpu().numpy())
        self.solver.factor(A)
        self.solver.solve(b, x_out)
        return x_out

    def newton(self, x, h, abstol=1e-9, reltol=1e-6, max_iter=50):
        """NR iterations from x at step h until max|dx| <= abstol + reltol
        max|x|; returns (x, iterations)."""
        x = x.clone()
        x_new = torch.empty_like(x)
        for it in range(1, max_iter + 1):
            A, b = self.assemble(x, h)
            self.solve(A, b, x_new)
            dx = (x_new - x).abs().max().item()
            x, x_new = x_new, x
            if dx <= abstol + reltol * x.abs().max().item():
                return x, it
        raise RuntimeError(f"NR did not converge in {max_iter} iterations (last max|dx| = {dx:.3e})")

    def run(self, x0, h, steps, **kw):
        """`steps` backward-Euler steps from x0; returns the list of accepted
        solutions and NR iteration counts (ees_accept after each step)."""
        xs, its = [], []
        x = x0
        for _ in range(steps):
            x, it = self.newton(x, h, **kw)
            self.ctx.accept(x)
            xs.append(x)
            its.append(it)
        return xs, its

    def close(self):
        if self.solver is not None:
            self.solver.close()
            self.solver = None


def rail_sources(nl, volts=1.0):
    """The netgen convention: rail k is held by a source whose branch is
    unknown n_nodes + k."""
    return [(int(r), nl.n_nodes + k, volts) for k, r in enumerate(nl.rails)]
