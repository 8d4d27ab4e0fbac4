"""Python binding of the ees C ABI: names follow include/ees.h, and this
module only marshals arguments -- every step of the hot path runs in
libees.so's sm_100a kernels.  PyTorch supplies device memory and streams."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L

VARIANTS = {"auto": L.EES_AUTO, "color": L.EES_COLOR, "atomic": L.EES_ATOMIC,
            "gather": L.EES_GATHER, "tile": L.EES_TILE, "color_buf": L.EES_COLOR_BUF}
VARIANT_NAMES = {v: k for k, v in VARIANTS.items()}
RULES = {"exclude_rails": L.EES_CONFLICT_EXCLUDE_RAILS, "paper": L.EES_CONFLICT_PAPER,
         "hybrid": L.EES_CONFLICT_HYBRID}


class EESError(RuntimeError):
    def __init__(self, status, what):
        super().__init__(f"{what}: {L.lib.ees_strerror(status).decode()} ({status})")
        self.status = status


def _check(status, what):
    if status != L.EES_OK:
        raise EESError(status, what)


def _arr(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a.size else None


def _flags(host_only, tile_form, gather_form, color_mode):
    f = L.EES_SETUP_HOST_ONLY if host_only else 0
    f |= {None: 0, 0: L.EES_SETUP_TILE_FORM0, 1: L.EES_SETUP_TILE_FORM1}[tile_form]
    f |= {None: 0, 0: L.EES_SETUP_GATHER_FORM0, 1: L.EES_SETUP_GATHER_FORM1}[gather_form]
    f |= {None: 0, "launch": L.EES_SETUP_COLOR_LAUNCH, "coop": L.EES_SETUP_COLOR_COOP}[color_mode]
    return f


def fp64_peak():
    """ees_fp64_peak: measured FP64 FMA TFLOP/s of the current CUDA device."""
    t = C.c_double()
    _check(L.lib.ees_fp64_peak(C.byref(t)), "ees_fp64_peak")
    return t.value


def red_throughput(mode=0):
    """ees_red_throughput: FP64 RED G lane-ops/s (0 spread, 1 same address per warp)."""
    t = C.c_double()
    _check(L.lib.ees_red_throughput(int(mode), C.byref(t)), "ees_red_throughput")
    return t.value


def stream_probe(src, read_bytes, dst, write_bytes, sink, stream=None):
    """ees_stream_probe: enqueue one streaming kernel reading read_bytes of
    src and writing write_bytes of dst (CUDA tensors; sink: one float64)."""
    import torch
    for t in (src, dst, sink):
        if not (isinstance(t, torch.Tensor) and t.is_cuda):
            raise ValueError("stream_probe: CUDA tensors expected")
    if read_bytes > src.numel() * src.element_size() or write_bytes > dst.numel() * dst.element_size():
        raise ValueError("stream_probe: byte counts exceed the buffers")
    if stream is None:
        stream = torch.cuda.current_stream()
    sh = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    _check(L.lib.ees_stream_probe(C.c_void_p(src.data_ptr()), int(read_bytes), C.c_void_p(dst.data_ptr()),
                                  int(write_bytes), C.c_void_p(sink.data_ptr()), C.c_void_p(sh)),
           "ees_stream_probe")


class Context:
    """ees_setup / ees_eval_stamp / ees_stats ... on one CUDA device."""

    def __init__(self, *, n_nodes, n_extra, d, g, s, b, w, l, model, vprev, models,
                 rails=(), extra_row=(), extra_col=(), gmin=1e-12, variant="auto",
                 rule="exclude_rails", heavy_degree=0, host_only=False, tile_form=None,
                 gather_form=None, color_mode=None):
        """Layout overrides (experiments, tests): tile_form / gather_form 0 or 1,
        color_mode "launch" or "coop"; None = setup chooses (ees.h flags)."""
        self._keep = dict(d=_arr(d, np.int32), g=_arr(g, np.int32), s=_arr(s, np.int32),
                          b=_arr(b, np.int32), w=_arr(w, np.float64), l=_arr(l, np.float64),
                          model=_arr(model, np.int32), vprev=_arr(vprev, np.float64),
                          rails=_arr(rails, np.int32), er=_arr(extra_row, np.int32),
                          ec=_arr(extra_col, np.int32))
        k = self._keep
        n_dev = k["d"].shape[0]
        ms = (L.ees_model * max(1, len(models)))()
        for i, m in enumerate(models):
            ms[i] = L.ees_model(int(m["polarity"]), 0, float(m["vt0"]), float(m["kp"]),
                                float(m["lam"]), float(m["cgs"]), float(m["cgd"]), float(m["cdb"]))
        desc = L.ees_desc(
            n_nodes=int(n_nodes), n_extra=int(n_extra), n_dev=int(n_dev),
            d=_ptr(k["d"]), g=_ptr(k["g"]), s=_ptr(k["s"]), b=_ptr(k["b"]), w=_ptr(k["w"]),
            l=_ptr(k["l"]), model=_ptr(k["model"]), vprev=_ptr(k["vprev"]),
            n_models=len(models), models=C.cast(ms, C.c_void_p), n_rails=len(k["rails"]),
            rails=_ptr(k["rails"]), n_extra_entries=len(k["er"]), extra_row=_ptr(k["er"]),
            extra_col=_ptr(k["ec"]), gmin=float(gmin),
            variant=VARIANTS[variant] if isinstance(variant, str) else int(variant),
            conflict_rule=RULES[rule] if isinstance(rule, str) else int(rule),
            flags=_flags(host_only, tile_form, gather_form, color_mode), heavy_degree=int(heavy_degree))
        h = C.c_void_p()
        _check(L.lib.ees_setup(C.byref(desc), C.byref(h)), "ees_setup")
        self._h = h
        self._keep = None          # ees_setup copied every input
        st = self.stats()
        self.n, self.nnz, self.n_dev = st["n"], st["nnz"], st["n_dev"]

    @classmethod
    def from_netlist(cls, nl, variant="auto", rule="exclude_rails", gmin=None, host_only=False,
                     heavy_degree=0, **layout):
        return cls(n_nodes=nl.n_nodes, n_extra=nl.n_extra, d=nl.d, g=nl.g, s=nl.s, b=nl.b,
                   w=nl.w, l=nl.l, model=nl.model, vprev=nl.vprev, models=nl.models,
                   rails=nl.rails, extra_row=nl.extra_row, extra_col=nl.extra_col,
                   gmin=nl.gmin if gmin is None else gmin, variant=variant, rule=rule,
                   heavy_degree=heavy_degree, host_only=host_only, **layout)

    # ------------------------------------------------------------ queries
    def pattern(self):
        n = L.i32(); nnz = L.i64(); rp = C.c_void_p(); ci = C.c_void_p()
        _check(L.lib.ees_pattern(self._h, C.byref(n), C.byref(nnz), C.byref(rp), C.byref(ci)),
               "ees_pattern")
        row_ptr = np.ctypeslib.as_array((L.i32 * (n.value + 1)).from_address(rp.value)).copy()
        col_idx = (np.ctypeslib.as_array((L.i32 * nnz.value).from_address(ci.value)).copy()
                   if nnz.value else np.zeros(0, np.int32))
        return row_ptr, col_idx

    def find_slot(self, row, col):
        k = L.i64()
        _check(L.lib.ees_find_slot(self._h, int(row), int(col), C.byref(k)), "ees_find_slot")
        return k.value

    def colors(self):
        p = C.c_void_p(); nc = L.i32()
        _check(L.lib.ees_colors(self._h, C.byref(p), C.byref(nc)), "ees_colors")
        if self.n_dev == 0:
            return np.zeros(0, np.int32), nc.value
        return np.ctypeslib.as_array((L.i32 * self.n_dev).from_address(p.value)).copy(), nc.value

    def stats(self):
        st = L.ees_stats_t()
        _check(L.lib.ees_stats(self._h, C.byref(st)), "ees_stats")
        out = {f: getattr(st, f) for f, _ in L.ees_stats_t._fields_ if f != "tune_ms"}
        out["tune_ms"] = {VARIANT_NAMES[v]: st.tune_ms[v] for v in (1, 2, 3, 4, 5)}
        out["variant_chosen"] = VARIANT_NAMES[st.variant_chosen]
        return out

    def set_variant(self, variant):
        v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
        _check(L.lib.ees_set_variant(self._h, v), "ees_set_variant")

    def set_timing(self, enable=True):
        _check(L.lib.ees_set_timing(self._h, 1 if enable else 0), "ees_set_timing")

    def phase_times(self):
        """(per-phase device ms summed over calls since the last read, calls)."""
        ms = (C.c_double * 4)()
        n = L.i32()
        _check(L.lib.ees_phase_times(self._h, ms, C.byref(n)), "ees_phase_times")
        return list(ms), n.value

    # ------------------------------------------------------------ hot path
    def eval_stamp(self, x, h, A, b, stream=None):
        """A += stamps, b += stamps for node voltages x at step h (device
        tensors: float64, contiguous, on the current CUDA device)."""
        import torch
        for t, n, name in ((x, self.n, "x"), (A, self.nnz, "A"), (b, self.n, "b")):
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
                    and t.is_contiguous() and t.numel() == n):
                raise ValueError(f"{name}: need a contiguous float64 CUDA tensor of {n} elements")
        if stream is None:
            stream = torch.cuda.current_stream()
        sh = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        _check(L.lib.ees_eval_stamp(self._h, C.c_void_p(x.data_ptr()), float(h),
                                    C.c_void_p(A.data_ptr()), C.c_void_p(b.data_ptr()),
                                    C.c_void_p(sh)), "ees_eval_stamp")

    def eval_stamp_host(self, x, h, A, b, stream=None, assign=False):
        """Host-buffer form (numpy float64 or pinned CPU tensors); blocking.
        assign=True: A, b are outputs only (A = stamps, no upload)."""
        def ptr(t, n, name):
            if isinstance(t, np.ndarray):
                if t.dtype != np.float64 or not t.flags.c_contiguous or t.size != n:
                    raise ValueError(name)
                return C.c_void_p(t.ctypes.data)
            import torch
            if t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous() or t.numel() != n:
                raise ValueError(name)
            return C.c_void_p(t.data_ptr())
        sh = 0
        if stream is not None:
            sh = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        _check(L.lib.ees_eval_stamp_host(self._h, ptr(x, self.n, "x"), float(h),
                                         ptr(A, self.nnz, "A"), ptr(b, self.n, "b"),
                                         C.c_void_p(sh), L.EES_HOST_ASSIGN if assign else 0),
               "ees_eval_stamp_host")

    def accept(self, x, stream=None):
        """ees_accept: v_prev of every FET <- the branch voltages at x (a
        contiguous float64 CUDA tensor of n elements)."""
        import torch
        if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64
                and x.is_contiguous() and x.numel() == self.n):
            raise ValueError(f"x: need a contiguous float64 CUDA tensor of {self.n} elements")
        if stream is None:
            stream = torch.cuda.current_stream()
        sh = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        _check(L.lib.ees_accept(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(sh)), "ees_accept")

    def set_work(self, work):
        """ees_set_work: SPEC S:229 work multiplier (>= 1)."""
        _check(L.lib.ees_set_work(self._h, int(work)), "ees_set_work")

    def tile_trace(self, x, h, A, b, stream=None):
        """Debug: one traced EES_TILE call -> uint64 array [n_ctas, 64] of
        %globaltimer stamps (see ees.h)."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream()
        sh = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        cap = 1 << 20
        buf = np.zeros(cap, np.uint64)
        n = L.i32()
        _check(L.lib.ees_tile_trace(self._h, C.c_void_p(x.data_ptr()), float(h), C.c_void_p(A.data_ptr()),
                                    C.c_void_p(b.data_ptr()), C.c_void_p(sh), C.c_void_p(buf.ctypes.data),
                                    cap, C.byref(n)), "ees_tile_trace")
        return buf[: n.value * 64].reshape(n.value, 64)

    def race_probe(self, color=None):
        cp = None
        if color is not None:
            color = np.ascontiguousarray(color, np.int32)
            cp = C.c_void_p(color.ctypes.data)
        n = L.i64()
        _check(L.lib.ees_race_probe(self._h, cp, C.byref(n)), "ees_race_probe")
        return n.value

    def stamp_linear(self, slot, val, row, bval, A, b, stream=None):
        """ees_stamp_linear (the caller's linear pre-pass): A[slot] +=
        val, b[row] += bval (CUDA tensors: slot int64, row int32, values
        float64)."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream()
        sh = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        for t, dt in ((slot, torch.int64), (val, torch.float64), (row, torch.int32), (bval, torch.float64),
                      (A, torch.float64), (b, torch.float64)):
            if not (t.is_cuda and t.dtype == dt and t.is_contiguous()):
                raise ValueError("stamp_linear: contiguous CUDA tensors of the documented dtypes expected")
        if slot.numel() != val.numel() or row.numel() != bval.numel():
            raise ValueError("stamp_linear: slot/val and row/bval lengths differ")
        if A.numel() != self.nnz or b.numel() != self.n:
            raise ValueError("stamp_linear: A must have nnz and b n elements")
        _check(L.lib.ees_stamp_linear(self._h, slot.numel(), C.c_void_p(slot.data_ptr()), C.c_void_p(val.data_ptr()),
                                      row.numel(), C.c_void_p(row.data_ptr()), C.c_void_p(bval.data_ptr()),
                                      C.c_void_p(A.data_ptr()), C.c_void_p(b.data_ptr()), C.c_void_p(sh)),
               "ees_stamp_linear")

    def close(self):
        if getattr(self, "_h", None):
            L.lib.ees_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class Solver:
    """ees_solver_*: sparse LU of the context's pattern (KLU's role):
    ordering + pivoting at construction (host values), GPU refactorisation
    per factor() call, GPU triangular solves per solve() call."""

    def __init__(self, ctx, A_host):
        A_host = np.ascontiguousarray(A_host, np.float64)
        if A_host.size != ctx.nnz:
            raise ValueError("Solver: A_host must have nnz entries")
        h = C.c_void_p()
        _check(L.lib.ees_solver_create(ctx._h, C.c_void_p(A_host.ctypes.data), C.byref(h)), "ees_solver_create")
        self._h, self.n, self.nnz = h, ctx.n, ctx.nnz

    @staticmethod
    def _sh(stream):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream()
        return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))

    def factor(self, A, stream=None):
        if not (A.is_cuda and A.numel() == self.nnz and A.is_contiguous()):
            raise ValueError("factor: a contiguous CUDA float64 tensor of nnz elements")
        _check(L.lib.ees_solver_factor(self._h, C.c_void_p(A.data_ptr()), self._sh(stream)), "ees_solver_factor")

    def solve(self, b, x, stream=None):
        for t in (b, x):
            if not (t.is_cuda and t.numel() == self.n and t.is_contiguous()):
                raise ValueError("solve: contiguous CUDA float64 tensors of n elements")
        _check(L.lib.ees_solver_solve(self._h, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()),
                                      self._sh(stream)), "ees_solver_solve")

    def fill(self):
        a, c = L.i64(), L.i64()
        _check(L.lib.ees_solver_info(self._h, C.byref(a), C.byref(c)), "ees_solver_info")
        return a.value, c.value

    def close(self):
        if getattr(self, "_h", None):
            L.lib.ees_solver_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
