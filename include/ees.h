/*
 * ees.h -- C ABI of the B200 evaluate+stamp library (libees.so).
 *
 * One call, ees_eval_stamp(), performs the hot path of one Newton-Raphson
 * iteration of EEspice (arxiv 2604.03079): every MOSFET instance is evaluated
 * at the current node-voltage vector x ("Compute Phase") and
 * its linearised contributions are stamped into the shared MNA matrix A (CSR
 * values) and right-hand side b ("Stamp Phase") without write races
 * (P:31).  The device model is SPEC.md's Level-1 MOSFET with gmin and three
 * backward-Euler capacitor companions, read as in
 * SURVEY.md §8(c) / DESIGN.md §2.
 *
 * Conventions
 *  - All calls return ees_status (0 = EES_OK, < 0 = error).  No C++
 *    exception crosses the ABI.  ees_strerror() names a status.
 *  - Nodes are 0 .. n_nodes-1; ground is -1 and is eliminated.
 *    Unknowns n = n_nodes + n_extra: source-branch unknowns follow the nodes
 *    (S:158).  MOSFETs never reference branch unknowns; the caller's linear
 *    devices may, through `extra_row/extra_col` pattern entries.
 *  - Terminals are d, g, s, b = drain, gate, source, bulk.  The bulk
 *    carries only the drain-bulk capacitor (no body effect).
 *  - beta = (kp * W) / L, evaluated in that order in FP64.
 *  - All floating point is IEEE FP64.  Results equal the serial reference
 *    (S:339 loadsingle) up to summation order: per entry within
 *    1e-12 * sum|elementary contributions| (BASELINE.json north_star).
 *
 * Thread-safety: different contexts are independent.  One context must not
 * be used by two calls at once (it owns scratch buffers), and that includes
 * the device side: calls of one context enqueued on different streams must be
 * ordered by the caller (events), or their kernels may overlap and share the
 * context's scratch (TILE side parts and ticket, GATHER buffers).
 */
#ifndef EES_H
#define EES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ees_ctx ees_ctx;          /* opaque; owns all library device memory */
typedef void *ees_stream;                /* a cudaStream_t; NULL = legacy default stream */

typedef enum {
    EES_OK = 0,
    EES_EINVAL = -1,     /* bad argument (null pointer, id out of range, h <= 0 or NaN, ...) */
    EES_ENOMEM = -2,     /* host or device allocation failed */
    EES_ECUDA = -3,      /* a CUDA runtime call or kernel launch failed */
    EES_ESTATE = -4      /* context not usable (e.g. a variant that was not built) */
} ees_status;

/* Stamping variants (north_star subsystem (3)); all fuse evaluation. */
typedef enum {
    EES_AUTO = 0,        /* setup times COLOR/ATOMIC/GATHER on this topology, keeps the fastest */
    EES_COLOR = 1,       /* colour-phased: one phase per colour, plain read-modify-write */
    EES_ATOMIC = 2,      /* one pass, FP64 atomicAdd (RED) into A and b */
    EES_GATHER = 3,      /* deterministic: contributions to scratch, per-entry segmented reduction */
    EES_TILE = 4,        /* deterministic, one launch: per-CTA row tiles; contributions staged in
                            shared memory and gathered per owned entry; entries shared by tiles
                            (heavy x heavy: rails, hubs) reduced from per-tile partials */
    EES_COLOR_BUF = 5    /* the paper's non-fused "Color" (Table I):
                            one parallel compute phase into a contribution buffer, then one
                            plain-RMW stamp phase per colour reading it (EES_GATHER is the
                            "loadomp" analogue: compute to the buffer, ordered stamp) */
} ees_variant;

/* Conflict relation for the colouring (P:60 and SURVEY A1). */
typedef enum {
    EES_CONFLICT_EXCLUDE_RAILS = 0, /* edge iff two FETs share a node that is neither ground nor a rail;
                                       rail x rail entries of A and rail rows of b then take a
                                       deterministic side reduction (DESIGN.md §2 reading R1) */
    EES_CONFLICT_PAPER = 1,         /* paper-literal: edge iff two FETs share any non-ground node */
    EES_CONFLICT_HYBRID = 2         /* degree-threshold hybrid: rails and every
                                       node with more than `heavy_degree` incident FETs leave the
                                       relation; under EES_COLOR, an entry of A whose row and column
                                       both left it (or a b row that left it) and that more than one
                                       FET stamps is written by no colour phase: its contributions go
                                       to fixed scratch slots and a deterministic segmented sum adds
                                       them after the last colour */
} ees_conflict_rule;

enum { EES_MAX_MODELS = 16, EES_MAX_RAILS = 8 };

typedef struct {
    int32_t polarity;        /* +1 NMOS, -1 PMOS */
    int32_t reserved;        /* must be 0 */
    double vt0;              /* V; SPICE sign convention: PMOS vt0 < 0 */
    double kp;               /* A/V^2, > 0 */
    double lambda;           /* 1/V */
    double cgs, cgd, cdb;    /* F, >= 0 */
} ees_model;

typedef struct {
    int32_t n_nodes;         /* non-ground nodes, >= 0 */
    int32_t n_extra;         /* branch unknowns after the nodes, >= 0 */
    int64_t n_dev;           /* MOSFETs, 0 .. 2^31 - 2 (device lists use int32 indices) */
    const int32_t *d, *g, *s, *b;   /* host [n_dev], each in [-1, n_nodes); -1 = ground */
    const double *w, *l;            /* host [n_dev], metres, finite and > 0 */
    const int32_t *model;           /* host [n_dev], in [0, n_models) */
    const double *vprev;            /* host [3][n_dev] SoA: v_gs, v_gd, v_db at the last accepted
                                       step (physical frame) */
    int32_t n_models;               /* 1 .. EES_MAX_MODELS */
    const ees_model *models;        /* host [n_models] */
    int32_t n_rails;                /* 0 .. EES_MAX_RAILS */
    const int32_t *rails;           /* host [n_rails]: distinct nodes held by ideal sources (VDD) */
    int64_t n_extra_entries;        /* caller's linear-device pattern entries */
    const int32_t *extra_row, *extra_col;  /* host [n_extra_entries], each in [0, n) */
    double gmin;                    /* S, >= 0, added drain-source on every FET */
    int32_t variant;                /* ees_variant */
    int32_t conflict_rule;          /* ees_conflict_rule */
    int32_t flags;                  /* 0, or EES_SETUP_* bits (below) */
    int32_t heavy_degree;           /* EES_CONFLICT_HYBRID threshold (incident FETs); 0 = 64 */
} ees_desc;

/* ees_desc.flags:
 *  EES_SETUP_HOST_ONLY: build only the host-side topology (pattern, slots,
 *    colouring, statistics) without touching a GPU; ees_eval_stamp and
 *    ees_race_probe then return EES_ESTATE.  For host-logic tests.
 *  Layout overrides (experiments and tests; by default setup chooses each
 *  from the topology): at most one of each pair.
 *    EES_SETUP_TILE_FORM0 / _FORM1     EES_TILE item data in the tile blobs /
 *                                      in tile-order HBM arrays
 *    EES_SETUP_GATHER_FORM0 / _FORM1   EES_GATHER compact buffer + index lists /
 *                                      target-ordered buffer
 *    EES_SETUP_COLOR_LAUNCH / _COOP    EES_COLOR one launch per colour /
 *                                      one persistent cooperative kernel
 *  Any other bit -> EES_EINVAL. */
enum {
    EES_SETUP_HOST_ONLY = 1,
    EES_SETUP_TILE_FORM0 = 2,
    EES_SETUP_TILE_FORM1 = 4,
    EES_SETUP_GATHER_FORM0 = 8,
    EES_SETUP_GATHER_FORM1 = 16,
    EES_SETUP_COLOR_LAUNCH = 32,
    EES_SETUP_COLOR_COOP = 64
};

typedef struct {
    int64_t n_dev, nnz, n_contributions;   /* contributions = live (entry, device) stamps */
    int32_t n;                              /* unknowns */
    int32_t n_colors;                       /* C under the context's conflict rule */
    int32_t max_group, min_group;           /* colour-group sizes */
    int32_t max_conflict_node_degree;       /* devices on the busiest conflict node */
    int32_t variant_chosen;                 /* the variant ees_eval_stamp runs */
    int32_t n_rail_entries;                 /* rail x rail A entries + rail b rows */
    int32_t n_heavy_targets;                /* GATHER entries reduced by block-chunks */
    int32_t launches_per_call;              /* kernels one ees_eval_stamp enqueues */
    double setup_s;                         /* wall time of ees_setup */
    double setup_pattern_s, setup_color_s;  /* parts of it */
    int32_t n_tiles, n_heavy_nodes, n_side_targets;   /* EES_TILE structure */
    int32_t tile_blob_max;                  /* largest per-tile head + program (bytes) */
    int64_t n_tile_items;                   /* device copies over all tiles (>= n_dev) */
    double tune_ms[6];                      /* EES_AUTO: measured ms per call of
                                               [_, COLOR, ATOMIC, GATHER, TILE, COLOR_BUF] */
    int32_t n_excluded_nodes;               /* nodes outside the conflict relation */
    int32_t tile_form;                      /* EES_TILE: 0 items in the tile blobs, 1 items in HBM arrays */
    int32_t gather_form;                    /* EES_GATHER: 0 compact buffer + index lists, 1 target-ordered */
    int32_t n_color_side_targets;           /* EES_CONFLICT_HYBRID: entries summed after the colours */
    int64_t n_color_side_contributions;     /* their contributions (scratch slots) */
    int32_t atomic_form;                    /* EES_ATOMIC: 0 one RED per contribution, 1 one RED per
                                               run of equal entries in a warp (timed at setup) */
    int32_t n_tile_programs;                /* EES_TILE: distinct reduction programs (tiles of equal
                                               structure share one) */
    int64_t tile_store_waves;               /* EES_TILE form 1: the builder's estimate of the shared-
                                               memory wavefronts of the evaluation's STS.64 per call
                                               (bank model: 16 bank pairs per half-warp store) */
    int64_t tile_store_waves_naive;         /* the same without the bank-aware lane placement */
} ees_stats_t;

/* Build everything that depends only on topology ("constructs the FET
 * conflict graph during setup"): validate, CSR pattern of all ordered
 * non-ground terminal pairs plus extra entries, per-device stamp
 * slots, first-fit greedy colouring in netlist order, colour-
 * major schedule, transposed contributor lists, rail side-reduction tables;
 * upload to the current CUDA device.  Copies every host input: the caller may
 * free them on return.  On error *out is NULL. */
ees_status ees_setup(const ees_desc *desc, ees_ctx **out);

/* The frozen sparsity pattern ("reserve ... finalize: the
 * pattern is immutable, handles stay valid"; S:114-131 every ordered
 * non-ground terminal pair of every device, deduplicated, plus the caller's
 * extra entries): host CSR, rows sorted by column, library-owned until
 * ees_destroy.  A_vals[k] of ees_eval_stamp is the entry (row r, col
 * col_idx[k]) with row_ptr[r] <= k < row_ptr[r+1].
 *   n, nnz, row_ptr, col_idx  outputs; each may be NULL (not written)
 * Errors: EES_EINVAL for a NULL ctx. */
ees_status ees_pattern(const ees_ctx *ctx, int32_t *n, int64_t *nnz,
                       const int32_t **row_ptr, const int32_t **col_idx);

/* EntryHandle lookup (a handle is the stable position of an
 * entry in the frozen pattern; here the CSR index into A_vals): *slot = k
 * with (row, col) at A_vals[k], or -1 if the pattern has no such entry.
 * Errors: EES_EINVAL for a NULL ctx or slot, or row / col outside [0, n). */
ees_status ees_find_slot(const ees_ctx *ctx, int32_t row, int32_t col, int64_t *slot);

/* Host colour of every device (netlist order), library-owned. */
ees_status ees_colors(const ees_ctx *ctx, const int32_t **color, int32_t *n_colors);

/* Evaluate + stamp every MOSFET at x for time step h, ACCUMULATING
 * into the caller's arrays (S:141 add semantics):
 *   A_vals[k] += sum of device stamps on entry k,  b[r] += sum on row r.
 * The caller clears them or pre-loads linear stamps first (S:426 order).
 *   x       device pointer, [n] FP64 (branch entries are never read)
 *   h       time step in seconds, > 0; +INFINITY = DC (capacitors open)
 *   A_vals  device pointer, [nnz] FP64, in/out
 *   b       device pointer, [n] FP64, in/out
 *   stream  the caller's CUDA stream; the call only enqueues work, never
 *           synchronises.  x, A_vals, b must stay valid until it completes.
 * Errors: EES_EINVAL (null pointer, h <= 0 or NaN) before any work is
 * enqueued; EES_ECUDA if a launch fails.  NaN in x propagates. */
ees_status ees_eval_stamp(ees_ctx *ctx, const double *x, double h, double *A_vals, double *b,
                          ees_stream stream);

/* Same with HOST arrays: copies x (and, unless EES_HOST_ASSIGN, A_vals and b)
 * to the device, runs ees_eval_stamp, copies A_vals and b back and
 * synchronises `stream` before returning.
 *   flags = 0                accumulate: A_vals [nnz], b [n] in/out (+=)
 *   flags = EES_HOST_ASSIGN  assign: A_vals = stamps, b = stamps (outputs only;
 *                            the device copies are cleared instead of uploaded)
 * Page-locked host memory gives full copy bandwidth. */
enum { EES_HOST_ASSIGN = 1 };
ees_status ees_eval_stamp_host(ees_ctx *ctx, const double *x, double h, double *A_vals,
                               double *b, ees_stream stream, int32_t flags);

/* Choose the variant later calls run (EES_AUTO = the one setup measured fastest). */
ees_status ees_set_variant(ees_ctx *ctx, int32_t variant);

/* Statistics of the context (SPEC S:285-293 color_stats: colour count, group
 * sizes, busiest conflict node; S:326-329 KernelReport: the variant run and
 * its timings) plus setup times and the TILE / GATHER / hybrid structure
 * sizes, copied into *out (caller-owned).  Host-side only; never syncs the
 * device.  Errors: EES_EINVAL for a NULL ctx or out. */
ees_status ees_stats(const ees_ctx *ctx, ees_stats_t *out);

/* sizeof of the ABI structs this library was built with (0: ees_desc,
 * 1: ees_stats_t; else 0), so a binding can refuse a mismatched build
 * instead of reading past a struct. */
int64_t ees_abi_sizeof(int32_t which);

/* Per-phase device timing (S:326 PhaseTimings).  When enabled, every
 * ees_eval_stamp records CUDA events on the call's stream around each kernel
 * group ("phase"):  COLOR {0: colour kernels, 1: rail finalise or, under
 * EES_CONFLICT_HYBRID, the side segmented sum},  COLOR_BUF {0: compute to
 * the buffer (t_calc), 1: colour stamp kernels + side sum (t_stamp)},
 * ATOMIC {0: k_atomic},  GATHER {0: evaluate to scratch, 1: segmented
 * reduction, 2: heavy-target finalise},  TILE {0: k_tile}. */
ees_status ees_set_timing(ees_ctx *ctx, int32_t enable);

/* Sum of device milliseconds per phase over the calls recorded since the
 * last read; synchronises on those events, then resets.  ms[4] out;
 * *n_calls = number of calls summed. */
ees_status ees_phase_times(ees_ctx *ctx, double ms[4], int32_t *n_calls);

/* Race instrument: replays the COLOR schedule given by
 * `color` (host [n_dev]; NULL = the context's own colouring) on the device,
 * counting per colour how many devices write each A entry and b row that is
 * not rail-reduced.  *n_conflicts = number of (colour, entry) pairs written by
 * more than one device: 0 for a valid colouring.  Synchronous. */
ees_status ees_race_probe(ees_ctx *ctx, const int32_t *color, int64_t *n_conflicts);

/* Debug: one EES_TILE call that also records %globaltimer stamps (ns) per
 * CTA into trace [n_ctas][64] (host, cap entries): slot 0 start, 1 first tile
 * staged, per tile i < 30: 2+2i evaluated (and the next tile's gathers
 * issued), 3+2i reduced and written; 62 past the grid barrier before the side
 * sums (side targets only), 63 end.  Synchronous. */
ees_status ees_tile_trace(ees_ctx *ctx, const double *x, double h, double *A_vals, double *b,
                          ees_stream stream, uint64_t *trace, int64_t cap, int32_t *n_ctas);

/* State update after an accepted time step (S:212 update_state; Fig. 1,
 * P:40-45): every FET's companion state becomes the converged branch
 * voltages at x, v_prev = (VG - VS, VG - VD, VD - VB), replacing the vprev
 * given at setup for all later ees_eval_stamp calls.
 *   x       device pointer, [n] FP64, the converged solution
 *   stream  enqueue only, like ees_eval_stamp; x must stay valid until done.
 * Errors: EES_EINVAL (null x), EES_ESTATE (host-only context), EES_ECUDA. */
ees_status ees_accept(ees_ctx *ctx, const double *x, ees_stream stream);

/* SPEC S:229 work multiplier: evaluation repeats its arithmetic `work`
 * times (>= 1; default 1) to emulate a costlier model such as BSIM4;
 * results are unchanged.  Errors: EES_EINVAL for work < 1. */
ees_status ees_set_work(ees_ctx *ctx, int32_t work);

/* Measures the FP64 FMA throughput of the current device (one resident
 * wave of independent FMA chains; the FP64 roofline denominator).
 * Synchronous.  *tflops out. */
ees_status ees_fp64_peak(double *tflops);

/* Measures FP64 RED (atomicAdd without return) throughput of the current
 * device in G lane-operations/s: mode 0 = every lane its own address
 * (spread), mode 1 = all lanes of a warp on one address per warp.
 * Synchronous.  (the atomic variant's ceiling.) */
ees_status ees_red_throughput(int32_t mode, double *gops);

/* Streaming probe (bench helper, the size calibration of the
 * HBM roofline, §8(d)): enqueues ONE kernel on `stream` that reads
 * `read_bytes` of `src` and writes `write_bytes` of `dst` with 16-byte
 * vector accesses, grid-stride over one resident wave -- the read/write mix
 * of an eval+stamp call's algorithmic bytes, timed by the caller's events.
 *   src, dst  device pointers, 16-byte aligned, distinct; sizes are rounded
 *             down to multiples of 16 bytes
 *   sink      device pointer to one double (written only to keep the loads live)
 * Errors: EES_EINVAL (null pointer, negative or misaligned), EES_ECUDA. */
ees_status ees_stream_probe(const void *src, int64_t read_bytes, void *dst, int64_t write_bytes,
                            double *sink, ees_stream stream);

/* ---------------------------------------------------------------------------
 * The steps either side of the hot path (SPEC.md
 * newton_step S:423-432 "clear -> linear pre-pass -> device stamps -> solve").
 * ------------------------------------------------------------------------- */

/* Linear pre-pass ("linear devices are stamped first, sequentially";
 * S:426): A_vals[slot[k]] += val[k] for k < n_a and b[row[k]] += bval[k] for
 * k < n_b -- the caller's resistors, capacitor companions and ideal-source
 * entries, pre-computed as (CSR index, value) pairs (ees_find_slot).  One
 * kernel on `stream`, enqueue only.  Repeated slots / rows accumulate (FP64
 * atomic adds, so their summation order is not fixed; distinct slots give
 * deterministic results).
 *   slot, val, row, bval, A_vals, b   device pointers
 * Errors: EES_EINVAL (NULL ctx, negative counts, NULL pointer with a count),
 * EES_ECUDA. */
ees_status ees_stamp_linear(const ees_ctx *ctx, int64_t n_a, const int64_t *slot, const double *val,
                            int64_t n_b, const int32_t *row, const double *bval, double *A_vals, double *b,
                            ees_stream stream);

/* Sparse LU solve of A x = b on the context's frozen pattern: the role of
 * KLU in the paper's NR loop, on the GPU.  Symbolic analysis
 * and pivoting once per topology, numeric refactorisation per NR iteration:
 *  ees_solver_create  orders the pattern (symmetric AMD of A + A^T), factors
 *                     A_vals_host (host, [nnz]) with partial pivoting on the
 *                     host and hands ordering, pivots and L/U patterns to
 *                     cuSOLVER's refactorisation (cusolverRf).  Synchronous.
 *                     EES_EINVAL if A is singular at these values.
 *  ees_solver_factor  refactorises at A_vals (device, [nnz]) with the same
 *                     ordering and pivots, on the GPU; EES_EINVAL on a zero
 *                     pivot (re-create the solver at the new values).
 *  ees_solver_solve   x = A^-1 b (device [n]; x may alias b) with the last
 *                     factorisation.
 * factor and solve are ordered after the caller's stream and the stream
 * after them through events (cuSOLVER's refactorisation runs on the legacy
 * stream); no host synchronisation.  ees_solver_info: fill-in of L and U. */
typedef struct ees_solver ees_solver;
ees_status ees_solver_create(const ees_ctx *ctx, const double *A_vals_host, ees_solver **out);
ees_status ees_solver_factor(ees_solver *solver, const double *A_vals, ees_stream stream);
ees_status ees_solver_solve(ees_solver *solver, const double *b, double *x, ees_stream stream);
ees_status ees_solver_info(const ees_solver *solver, int64_t *nnz_L, int64_t *nnz_U);
ees_status ees_solver_destroy(ees_solver *solver);

ees_status ees_destroy(ees_ctx *ctx);

const char *ees_strerror(ees_status status);

#ifdef __cplusplus
}
#endif
#endif /* EES_H */
