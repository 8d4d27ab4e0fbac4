"""A minimal Newton-Raphson transient driver around the hot path (SURVEY.md
§8(f) NEXT-4, "the steps either side"): the loop of PAPER.md Fig. 1
 and SPEC.md's newton_step / run_transient, for small
circuits.

Per NR iteration (S:426 order): clear A and b; stamp the linear devices (the
caller's pre-pass, S:302 -- here the ideal voltage sources that hold the
rails); ``ees_eval_stamp`` (the hot path: every MOSFET evaluated and stamped
on the GPU); solve ``A x = b``.  The solve is a dense LU through
``torch.linalg.solve`` -- a library solve, sized for the small circuits this
driver is for; the paper's sparse KLU / a cuDSS solve are out of
scope.  On convergence, ``ees_accept`` stores the converged
branch voltages as the companion-model state of the next step.
"""
from __future__ import annotations

import torch


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
        rp, ci = ctx.pattern()
        rows = torch.repeat_interleave(torch.arange(n), torch.from_numpy(rp[1:] - rp[:-1]).long())
        self.flat = (rows * n + torch.from_numpy(ci).long()).to(self.dev)
        self.src_slots, self.src_rows, self.src_vals = [], [], []
        for node, br, volts in sources:
            k1, k2 = ctx.find_slot(node, br), ctx.find_slot(br, node)
            if k1 < 0 or k2 < 0:
                raise ValueError(f"pattern lacks the source entries of node {node} / branch {br}")
            self.src_slots += [k1, k2]
            self.src_rows.append(br)
            self.src_vals.append(float(volts))
        self.src_slots = torch.tensor(self.src_slots, dtype=torch.long, device=self.dev)
        self.src_rows = torch.tensor(self.src_rows, dtype=torch.long, device=self.dev)
        self.src_vals = torch.tensor(self.src_vals, dtype=torch.float64, device=self.dev)
        self.A = torch.zeros(ctx.nnz, dtype=torch.float64, device=self.dev)
        self.b = torch.zeros(n, dtype=torch.float64, device=self.dev)
        self.dense = torch.zeros(n * n, dtype=torch.float64, device=self.dev)
        self.n = n

    def assemble(self, x, h):
        """A, b of one NR iteration at x (linear pre-pass, then the FET stamps)."""
        self.A.zero_()
        self.b.zero_()
        self.A[self.src_slots] += 1.0                 # KCL: +i_br at the node; branch row: V(node)
        self.b[self.src_rows] += self.src_vals        # = volts
        self.ctx.eval_stamp(x, h, self.A, self.b)
        return self.A, self.b

    def newton(self, x, h, abstol=1e-9, reltol=1e-6, max_iter=50):
        """NR iterations from x at step h until max|dx| <= abstol + reltol
        max|x|; returns (x, iterations)."""
        x = x.clone()
        for it in range(1, max_iter + 1):
            A, b = self.assemble(x, h)
            self.dense.zero_()
            self.dense.index_put_((self.flat,), A, accumulate=True)
            x_new = torch.linalg.solve(self.dense.view(self.n, self.n), b)
            dx = (x_new - x).abs().max().item()
            x = x_new
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


def rail_sources(nl, volts=1.0):
    """The netgen convention: rail k is held by a source whose branch is
    unknown n_nodes + k."""
    return [(int(r), nl.n_nodes + k, volts) for k, r in enumerate(nl.rails)]
