"""ctypes declarations of include/ees.h (argument marshalling only).

Loads the in-tree ``lib/libees.so``; there is no fallback: if the library is
missing this module raises ImportError (build it with
``python -m paper_2604_03079_b200.build`` or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libees.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libees.so not built ({LIB_PATH}); run `python -m paper_2604_03079_b200.build`"
                      " -- the CUDA path has no CPU fallback")

EES_OK, EES_EINVAL, EES_ENOMEM, EES_ECUDA, EES_ESTATE = 0, -1, -2, -3, -4
EES_AUTO, EES_COLOR, EES_ATOMIC, EES_GATHER, EES_TILE, EES_COLOR_BUF = 0, 1, 2, 3, 4, 5
EES_CONFLICT_EXCLUDE_RAILS, EES_CONFLICT_PAPER, EES_CONFLICT_HYBRID = 0, 1, 2
EES_MAX_MODELS, EES_MAX_RAILS = 16, 8
EES_SETUP_HOST_ONLY = 1
EES_SETUP_TILE_FORM0, EES_SETUP_TILE_FORM1 = 2, 4
EES_SETUP_GATHER_FORM0, EES_SETUP_GATHER_FORM1 = 8, 16
EES_SETUP_COLOR_LAUNCH, EES_SETUP_COLOR_COOP = 32, 64
EES_HOST_ASSIGN = 1

P = C.c_void_p
i32, i64, f64 = C.c_int32, C.c_int64, C.c_double


class ees_model(C.Structure):
    _fields_ = [("polarity", i32), ("reserved", i32), ("vt0", f64), ("kp", f64), ("lambda_", f64),
                ("cgs", f64), ("cgd", f64), ("cdb", f64)]


class ees_desc(C.Structure):
    _fields_ = [("n_nodes", i32), ("n_extra", i32), ("n_dev", i64),
                ("d", P), ("g", P), ("s", P), ("b", P), ("w", P), ("l", P), ("model", P),
                ("vprev", P), ("n_models", i32), ("models", P), ("n_rails", i32), ("rails", P),
                ("n_extra_entries", i64), ("extra_row", P), ("extra_col", P), ("gmin", f64),
                ("variant", i32), ("conflict_rule", i32), ("flags", i32), ("heavy_degree", i32)]


class ees_stats_t(C.Structure):
    _fields_ = [("n_dev", i64), ("nnz", i64), ("n_contributions", i64), ("n", i32),
                ("n_colors", i32), ("max_group", i32), ("min_group", i32),
                ("max_conflict_node_degree", i32), ("variant_chosen", i32),
                ("n_rail_entries", i32), ("n_heavy_targets", i32), ("launches_per_call", i32),
                ("setup_s", f64), ("setup_pattern_s", f64), ("setup_color_s", f64),
                ("n_tiles", i32), ("n_heavy_nodes", i32), ("n_side_targets", i32),
                ("tile_blob_max", i32), ("n_tile_items", i64), ("tune_ms", f64 * 6),
                ("n_excluded_nodes", i32), ("tile_form", i32), ("gather_form", i32),
                ("n_color_side_targets", i32),
                ("n_color_side_contributions", i64), ("atomic_form", i32), ("n_tile_programs", i32),
                ("tile_store_waves", i64), ("tile_store_waves_naive", i64)]


lib = C.CDLL(LIB_PATH)
lib.ees_setup.argtypes = [C.POINTER(ees_desc), C.POINTER(P)]
lib.ees_pattern.argtypes = [P, C.POINTER(i32), C.POINTER(i64), C.POINTER(P), C.POINTER(P)]
lib.ees_find_slot.argtypes = [P, i32, i32, C.POINTER(i64)]
lib.ees_colors.argtypes = [P, C.POINTER(P), C.POINTER(i32)]
lib.ees_eval_stamp.argtypes = [P, P, f64, P, P, P]
lib.ees_eval_stamp_host.argtypes = [P, P, f64, P, P, P, i32]
lib.ees_set_variant.argtypes = [P, i32]
lib.ees_stats.argtypes = [P, C.POINTER(ees_stats_t)]
lib.ees_set_timing.argtypes = [P, i32]
lib.ees_phase_times.argtypes = [P, P, C.POINTER(i32)]
lib.ees_tile_trace.argtypes = [P, P, f64, P, P, P, P, i64, C.POINTER(i32)]
lib.ees_race_probe.argtypes = [P, P, C.POINTER(i64)]
lib.ees_accept.argtypes = [P, P, P]
lib.ees_set_work.argtypes = [P, i32]
lib.ees_fp64_peak.argtypes = [C.POINTER(f64)]
lib.ees_red_throughput.argtypes = [i32, C.POINTER(f64)]
lib.ees_stream_probe.argtypes = [P, i64, P, i64, P, P]
lib.ees_stamp_linear.argtypes = [P, i64, P, P, i64, P, P, P, P, P]
lib.ees_solver_create.argtypes = [P, P, C.POINTER(P)]
lib.ees_solver_factor.argtypes = [P, P, P]
lib.ees_solver_solve.argtypes = [P, P, P, P]
lib.ees_solver_info.argtypes = [P, C.POINTER(i64), C.POINTER(i64)]
lib.ees_solver_destroy.argtypes = [P]
lib.ees_destroy.argtypes = [P]
lib.ees_strerror.argtypes = [i32]
lib.ees_strerror.restype = C.c_char_p
for _f in ("ees_setup", "ees_pattern", "ees_find_slot", "ees_colors", "ees_eval_stamp",
           "ees_eval_stamp_host", "ees_set_variant", "ees_stats", "ees_race_probe", "ees_destroy",
           "ees_set_timing", "ees_phase_times", "ees_tile_trace", "ees_accept", "ees_set_work",
           "ees_fp64_peak", "ees_red_throughput", "ees_stream_probe", "ees_stamp_linear",
           "ees_solver_create", "ees_solver_factor", "ees_solver_solve", "ees_solver_info",
           "ees_solver_destroy"):
    getattr(lib, _f).restype = i32

lib.ees_abi_sizeof.argtypes = [i32]
lib.ees_abi_sizeof.restype = i64
for _which, _cls in ((0, ees_desc), (1, ees_stats_t)):
    if lib.ees_abi_sizeof(_which) != C.sizeof(_cls):
        raise ImportError(f"{LIB_PATH} was built with a different {_cls.__name__} layout "
                          f"({lib.ees_abi_sizeof(_which)} vs {C.sizeof(_cls)} bytes): rebuild it")

EXPORTS = ["ees_setup", "ees_pattern", "ees_find_slot", "ees_colors", "ees_eval_stamp",
           "ees_eval_stamp_host", "ees_set_variant", "ees_stats", "ees_set_timing",
           "ees_phase_times", "ees_tile_trace", "ees_race_probe", "ees_accept", "ees_set_work",
           "ees_fp64_peak", "ees_red_throughput", "ees_stream_probe", "ees_stamp_linear", "ees_solver_create",
           "ees_solver_factor", "ees_solver_solve", "ees_solver_info", "ees_solver_destroy", "ees_destroy", "ees_strerror", "ees_abi_sizeof"]
