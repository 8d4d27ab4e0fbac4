// ees_internal.h -- shared between the host setup (ees_host.cpp) and the
// sm_100a kernels (ees_kernels.cu).  Product code; never includes oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ees.h"

namespace ees {

// Live stamp pairs of the 4-terminal FET (SURVEY §8(a) "12 of 16"; GB, BG,
// SB, BS are structurally zero because the bulk carries only C_db, S:77,
// S:230).  Terminal index D=0 G=1 S=2 B=3.
enum Pair { DD = 0, DG, DS, DB, GD, GG, GS, SD, SG, SS, BD, BB, NPAIR };
constexpr int kPairRow[NPAIR] = {0, 0, 0, 0, 1, 1, 1, 2, 2, 2, 3, 3};
constexpr int kPairCol[NPAIR] = {0, 1, 2, 3, 0, 1, 2, 0, 1, 2, 0, 3};
__host__ __device__ constexpr int pair_row(int p) { return p < 4 ? 0 : p < 7 ? 1 : p < 10 ? 2 : 3; }
__host__ __device__ constexpr int pair_col(int p)
{
    return p < 4 ? p : p < 7 ? p - 4 : p < 10 ? p - 7 : (p == 10 ? 0 : 3);
}

constexpr int kMaxRailEntries = EES_MAX_RAILS * EES_MAX_RAILS + EES_MAX_RAILS;
constexpr int kBlock = 256;          // threads per block of the per-device kernels
constexpr int kHeavyLen = 128;       // GATHER: lists longer than this are chunk-reduced
constexpr int kChunk = 4096;         // GATHER: contributions per heavy chunk (one block)

// Per-call model card: everything h-dependent is folded in on the host
// (Gc = C/h, correctly rounded FP64 division, "Geq = C/dt").
struct CardK {
    double vt;        // p * vt0
    double lam;
    double gcgs, gcgd, gcdb;
    double p;         // +1 / -1
};

struct CallK {
    CardK cards[EES_MAX_MODELS];
    const double *x;
    double *A;
    double *b;
    double gmin;
    int32_t work;                     // S:229 work multiplier (>= 1)
    int32_t n_models;
    int32_t n_rail_nodes;
    int32_t n_rail_a;                 // rail entries [0, n_rail_a) are A slots, the rest b rows
    int32_t n_rail_entries;
    int32_t rail_node[EES_MAX_RAILS];
    int32_t rail_target[kMaxRailEntries];
};

// SoA device arrays of one execution order.
//  term : (d, g, s, b); >= 0 node, -1 ground, <= -2 rail ordinal r = -2 - code
//         (rail-coded layouts only; the GATHER layout holds plain node ids)
//  slot : [NPAIR][N]; >= 0 A index, -1 no entry, <= -2 rail entry e = -2 - code
struct DevK {
    int64_t N;
    const int4 *term;
    const double *beta;
    const double *v0;      // [3][N]: v_gs, v_gd, v_db at the last accepted step
    const uint8_t *model;
    const int32_t *slot;   // [NPAIR][N] (null in the GATHER layout)
    // ATOMIC order: devices [0, cls_a) have source and bulk grounded (codes
    // other than DD DG GD GG are -1), [cls_a, cls_b) have dead bulk pairs
    // (DB BD BB -1 or merged away); 0, 0 in the other layouts
    int64_t cls_a, cls_b;
};

// GATHER layout extras
struct GatherK {
    const int32_t *off;        // [N+1] first compact contribution of each device
    double *buf;               // [n_contrib] contribution values
    const int32_t *tptr;       // [nnz+n+1] light contributor lists per target
    const int32_t *tidx;       // compact contribution indices
    int64_t n_targets;         // nnz + n
    int64_t nnz;
    // heavy targets, chunk-reduced
    int32_t n_chunks;
    const int32_t *chunk_beg;  // [n_chunks+1] into hidx
    const int32_t *hidx;       // compact indices of heavy lists, concatenated
    double *chunk_part;        // [n_chunks]
    int32_t n_heavy;
    const int32_t *heavy_target;   // [n_heavy]
    const int32_t *heavy_chunk;    // [n_heavy+1]
    // form 1 (EES_GATHER, chosen at setup): each contribution is stored at its
    // place in its target's list, so the reduction streams the buffer; form 0:
    // compact per-device buffer (buf) gathered through tidx / hidx
    int32_t form;
    double *tbuf;                  // [n_contrib]: light lists (tptr), then heavy lists (chunk_beg + heavy_base)
    const int32_t *tpos;           // [16][N] position of each live contribution in tbuf, -1 none
    int64_t heavy_base;            // first heavy entry in tbuf
};

// TILE layout (ees_tile.cpp builds it; k_tile consumes it).  Rows are cut
// into tiles of consecutive light rows; a tile's items are the FETs incident
// on its rows (boundary FETs are copied into every tile they touch).  Each
// item's 16 contributions (12 A pairs, 4 b rows) land in shared memory at
// slot p*kTileItems + item.  A tile OWNS every target (A entry or b row) all
// of whose contributors are among its items: the rows' CSR block, their b
// rows, heavy-row slices (h, c) of its light columns c, and heavy x heavy
// targets whose contributors all live in it; a target shared by several
// tiles (heavy x heavy: rails, hub diagonals) is a SIDE target, to which the
// tile contributes one part.  (That slot layout is form 0's; form 1 stores
// each contribution straight into its pair row, TILE v5 below ProgHdr5.)
//
// The tile's reduction program, form 0 (TILE v4).  Short targets (at most kOpMax
// contributions; every owned target on the inverter / SRAM / hub structures)
// are an OP STREAM: each thread runs its own sequence of pair-ops, one u32
// each (two u16 byte offsets of contributions in the tile's shared-memory
// slot buffer; bit 2 of the first = kEmitBit, "emit"): the thread adds both
// entries to its running sum and, on "emit", adds the sum to the next
// destination of its own destination list with ONE reduction (RED.ADD.F64)
// and restarts the sum at 0.  A target of L contributions is ceil(L/2)
// consecutive pair-ops of one thread (odd L: the last pair's second entry is
// the zero slot).  Every owned target is written by exactly one thread of
// exactly one CTA, once per call, so A_vals[k] + sum is formed once -- the
// same IEEE addition as a plain read-modify-write (deterministic; the SM
// loads no old value).  The builder balances the targets over the threads
// (longest first, least-loaded thread) and orders the threads' sequences by
// length (thread 0 the longest), so op step s is stored as one contiguous row
// of the threads that still have an op there (row offsets orow[]): no
// padding, conflict-free 4-byte loads.  Longer targets form GROUP classes
// (one per kind and lane-group size gs = cls_group(L)): gs lanes per target,
// lane j summing the target's entries j, j+gs, ... in four fixed partial
// sums, then a fixed xor-shuffle tree.  A side target's contributions in the
// tile are cut into pieces of at most kSidePiece entries, each a target of
// the tile (a second op stream, thread order reversed so it falls on the
// warps the owned stream loads least; a side group class if longer than
// kOpMax) whose sum is its part (plain store) or, for the hot side targets
// (rails), adds to the CTA's running sum of its piece index in shared memory,
// in tile order.  (Whole side targets in group classes measured slower:
// profiles/r02_ab.md.)
// Everything a tile needs except x (and, in form 1, the item data) is its
// HEAD (per tile) and its PROGRAM (shared by structurally equal tiles), which
// two TMA bulk copies (cp.async.bulk + one mbarrier) bring into one shared-
// memory stage, kStages tiles ahead (program right after the head):
//   head:    TileHdr (96 B: counts, sizes, offsets, kTileBases destination
//            bases)
//            items: form 0: term int4[ni] | beta f64[ni] | v0 f64[3][ni] | model u8[ni]
//                   form 1: term int4[ni]; beta, v0[3], model in tile-order HBM
//                   arrays (kTileItems slots per tile) loaded one tile ahead
//            side:  SideEnt[n_sent]
//   program: ProgHdr (32 B; form 0 -- form 1: ProgHdr5)
//            owned op stream: orow u16[steps] (row offsets) | ops u32[..] |
//                  ostart u16[n_oseq] (per sequence with ops: its first
//                  destination | its step count << kSeqStartBits) |
//                  odst u32[..] (destination codes, per sequence contiguous)
//            side op stream:  srow | sops | sstart | sdst u16[..] (side entries)
//            group classes:   TileCls[n_cls] | dst u32[..] | meta u32[..]
//                  (first entry | length << 16) | ent u16[..] (each target's
//                  entries contiguous)
// A destination code d is base[d >> 28] + (d & 0x0FFFFFFF): the 16 bases are
// global targets (an A index, or nnz + a b row), each the first target of a
// cluster of the tile's owned targets (its rows' CSR block, its b rows, each
// heavy row's slice; a cluster never straddles nnz), so tiles of the same
// structure have byte-identical programs; the builder stores each distinct
// program once (cfg4: the inverter-chain and hub-load tiles).  The kernel
// turns the bases into 16 pointers per tile (A + g, or b + g - nnz), so a
// destination costs a shift, a mask and one shared-memory load.  With more
// than 16 clusters the bases are fixed: 8 chunks of 2^28 entries of A, then 8
// of b.
// Contributions of a FET whose source and bulk are one node (every PMOS of the
// inverter configs) are merged at evaluation (DB into DS, BD into SD, BB into
// SS, J[B] into J[S]) and the merged-away slots are not listed.
#ifndef EES_TILE_ITEMS
#define EES_TILE_ITEMS 128
#endif
constexpr int kTileItems = EES_TILE_ITEMS;   // max items (FET copies) per tile = threads per CTA
constexpr int kTileThreads = kTileItems;
constexpr int kLogTileThreads = kTileThreads == 128 ? 7 : kTileThreads == 64 ? 6 : kTileThreads == 256 ? 8 : -1;
static_assert(kLogTileThreads > 0, "tile width must be 64, 128 or 256 threads");
constexpr int kHeavyDeg = 64;        // nodes with more incident FETs are heavy
#ifndef EES_SIDE_PIECE
#define EES_SIDE_PIECE 4
#endif
constexpr int kSidePiece = EES_SIDE_PIECE;   // side-target entries per piece (one part each)
constexpr uint32_t kEmitBit = 4;     // pair-op word: bit 2 of the first entry = emit after this pair
#ifndef EES_OP_MAX
#define EES_OP_MAX 32
#endif
constexpr int kOpMax = EES_OP_MAX;   // owned targets of up to kOpMax contributions: op stream
constexpr uint32_t kNoEmit = 0xFFFFFFFFu;
#ifndef EES_HOT_PIECES
#define EES_HOT_PIECES 16
#endif
constexpr int kHotPieces = EES_HOT_PIECES;   // pieces of one hot target per tile
// TILE forms (chosen at setup from the FET copy factor, ees_host.cpp):
// stage bytes (one tile blob), item bytes in the blob, shared-memory slot
// buffers (2: one barrier per tile), CTAs per SM
#ifndef EES_STAGE1
#define EES_STAGE1 9360              // about the largest stage that keeps 5 CTAs per SM (228 KB; the
                                     // shared-memory allocation granularity is 256 B)
#endif
__host__ __device__ constexpr int stage_max(int form) { return (form ? EES_STAGE1 : 11264) * kTileItems / 128; }
// bytes per item in the head and program: form 0 the whole item; form 1 the
// terms (head) and the item's 16 contribution positions (program, TILE v5)
__host__ __device__ constexpr int item_blob_bytes(int form) { return form ? 16 + 32 : 49; }
#ifndef EES_TILE_BUF1
#define EES_TILE_BUF1 1
#endif
#ifndef EES_TILE_BUF0
#define EES_TILE_BUF0 1
#endif
__host__ __device__ constexpr int tile_bufs(int form) { return form ? EES_TILE_BUF1 : EES_TILE_BUF0; }
__host__ __device__ constexpr int tile_ctas(int form)
{
#ifndef EES_TILE_CTAS1
#define EES_TILE_CTAS1 5
#endif
    return (form ? (tile_bufs(1) == 2 ? 4 : EES_TILE_CTAS1) : (tile_bufs(0) == 2 ? 3 : 4)) * 128 / kTileItems;
}

#ifndef EES_STAGES
#define EES_STAGES 3
#endif
constexpr int kStages = EES_STAGES;  // TMA pipeline depth (blobs in flight per CTA), form 0
#ifndef EES_STAGES1
#define EES_STAGES1 EES_STAGES
#endif
__host__ __device__ constexpr int tile_stages(int form) { return form ? EES_STAGES1 : kStages; }
// EES_LATE_GATHER: a tile's successor is gathered after B1 (into the same
// registers the evaluation just consumed) and a stage is refilled after B0;
// fewer registers and stages, shorter latency cover for the gathers
#ifndef EES_A_PREFETCH
#define EES_A_PREFETCH 1               // bulk L2 prefetch of the next tile's CSR block of A
#endif
#ifndef EES_TDESC_ASYNC
#define EES_TDESC_ASYNC 1              // the refill's tdesc entry by a bulk copy into shared memory
#endif
#ifndef EES_LATE_GATHER
#define EES_LATE_GATHER 0
#endif
constexpr int kScSlots = 16 * kTileItems + 2;   // form 0: contribution slots per buffer (+16-byte pad)
#ifndef EES_SC_ROWS
#define EES_SC_ROWS 7
#endif
constexpr int kScRows = EES_SC_ROWS;             // form 1: pair rows (of kTileItems pairs) per tile
static_assert(kScRows <= 7, "row masks are 7 bits");
// form 1 sequence word: first destination (11 bits) | emit mask << 11 | side
// mask << 18 | pad mask << 25 (bit s of each: the thread's pair of row s);
// a sequence's rows end with its last emit (every sequence ends a target)
constexpr int kSeqEmit = 11, kSeqSide = 18, kSeqPad = 25;
// contribution slots (doubles) of the form's slot buffer; form 1: kScRows rows
// of kTileItems 16-byte pairs, then the trash slot and a pad
__host__ __device__ constexpr int sc_slots(int form) { return form ? kScRows * 2 * kTileItems + 2 : kScSlots; }
constexpr int kTrashByte1 = 8 * kScRows * 2 * kTileItems;   // form 1: unlisted contributions land here
constexpr int kZeroSlotByte = 8 * 16 * kTileItems; // the pad's first slot holds 0.0 (odd-length targets)
#ifndef EES_MAX_HOT
#define EES_MAX_HOT 16
#endif
constexpr int kMaxHot = EES_MAX_HOT;  // side targets pre-reduced per CTA (rails): parts = CTAs, not tiles
static_assert(8 * kScSlots < 65536, "entry byte offsets must fit 16 bits");

// Owned targets longer than kOpMax form group classes with cls_group(L)
// lanes per target (about four entries per lane, at most a warp).
__host__ __device__ constexpr int cls_group(int L)
{
    return L <= 16 ? 4 : L <= 32 ? 8 : L <= 64 ? 16 : 32;
}

struct TileCls {
    uint16_t len;                    // 0 (group class)
    uint16_t n;                      // targets
    uint16_t ent;                    // u16 index of the class's first entry in ent[]
    uint16_t dst;                    // index of the class's first destination in dst[]
    uint16_t rot;                    // lane groups (of gs lanes) used before the class, mod the
                                     // groups per CTA (kTileThreads / gs)
    uint16_t lg;                     // log2 of the group size gs
    uint16_t meta;                   // index of the first target's meta[] word
    uint16_t side;                   // 1: side targets (dst = side entry index)
};
static_assert(sizeof(TileCls) == 16, "TileCls layout");

// Per-tile head (streamed: one per tile) and the tile's reduction program
// (shared by every tile with the same program bytes).
constexpr int kTileBases = 16;           // dst code: base[code >> 28] + (code & 0x0FFFFFFF)
struct TileHdr {
    uint16_t n_items, n_full, n_sent, pad0;
    uint32_t head_bytes;             // head size (multiple of 16): the program follows it in the stage
    uint32_t prog_bytes;             // program size (multiple of 16)
    uint32_t off_items, off_side;    // byte offsets of the head's sections
    int32_t base[kTileBases];        // destination bases (global target ids)
    int32_t a_lo, a_n;               // the tile rows' CSR block of A: [a_lo, a_lo + a_n) (L2 prefetch)
};
static_assert(sizeof(TileHdr) == 96, "TileHdr layout");

struct ProgHdr {
    uint16_t n_oseq, off_orow, off_ops, off_ostart, off_odst;    // owned op stream
    uint16_t n_sseq, off_srow, off_sops, off_sstart, off_sdst;   // side op stream
    uint16_t n_cls, off_cls, off_dst, off_meta, off_ent;         // group classes
    uint16_t pad;
};
constexpr int kSeqStartBits = 11;        // sequence word: first destination | steps << 11

// TILE v5 (form 1) program: the contribution POSITIONS replace the op words.
// Each item's 16 contributions are stored by the evaluating thread straight
// into their place in the pair rows: thread j's pair of row s is the 16 bytes
// at (s * kTileItems + j) * 16 of the slot buffer (a conflict-free LDS.128 at
// a compile-time offset), so the reduction reads no program entry per pair.
// An odd target's last pair has no second contribution: that half is never
// written and its pad bit tells the reduction to skip it.  Per thread one
// sequence word: first destination (11 bits) | emit mask << 11 (bit s: the
// pair of row s completes a target) | side mask << 18 (that target is a side
// piece, its destination a side entry) | pad mask << 25.  Owned targets longer than kOpMax1 are group
// classes whose entries are contiguous in a group area after the rows.
//   program: ProgHdr5 | pos u16[2][ni][8] (byte offset of each contribution in
//            the slot buffer; kTrashByte1 if not listed) | oseq u32[kTileItems]
//            | odst u32[..] (destination code, or side entry index) |
//            TileCls[n_cls] | dst u32[..] | meta u32[..] (first slot after
//            the group base | length << 16)
struct ProgHdr5 {
    uint16_t n_rows, off_pos, off_oseq, off_odst;
    uint16_t n_cls, off_cls, off_dst, off_meta;
    uint16_t gbase;                      // first slot (double index) of the group area
    uint16_t pad[7];
};
static_assert(sizeof(ProgHdr5) == 32, "ProgHdr5 layout");
constexpr int kOpMax1 = 8;               // form 1: owned targets of <= 8 contributions in the rows
static_assert(sizeof(ProgHdr) == 32, "ProgHdr layout");

struct SideEnt {
    int32_t sid;                     // side target
    int32_t slot;                    // this piece's part slot in `part`, or -1-(h*kHotPieces+q) for
                                     // piece q of hot target h
};

struct TileK {
    int32_t form;                  // 0: whole items in the blob; 1: items' data in HBM arrays
    int32_t n_tiles;
    int64_t nnz;
    const uint4 *tdesc;            // [T] head offset / 16, head bytes, program offset / 16, program bytes
    const uint8_t *blob;           // the heads
    const uint8_t *prog;           // the distinct programs
    int32_t n_side;                // side targets, ordered: cold with > 8 parts | cold <= 8 | hot
    int32_t n_side_big;            // cold side targets with more than 8 parts (summed by a warp each)
    int32_t n_side_cold;           // cold side targets (the rest of them summed by a thread each)
    int32_t n_hot;                 // hot side targets: CTA b's part at part[hot_base + h*grid + b]
    int64_t hot_base;
    const int32_t *sd_gid;         // [n_side] global target
    const int32_t *hot_gid;        // [n_hot] global target of each hot side target
    const int32_t *sd_part;        // [n_side+1] partial ranges
    const double *item_beta;       // [n_tiles * kTileItems]
    const double *item_v0;         // [n_tiles * kTileItems][3]
    const uint8_t *item_model;     // [n_tiles * kTileItems]
    double *hot_pre;               // [n_hot] old values of the hot targets (read by CTA 0)
    double *part;                  // [n_side_entries]
    unsigned int *gbar;            // [2] grid barrier: arrivals, generation (zero at setup)
    unsigned long long *trace;     // debug: [grid][kTraceSlots] %globaltimer stamps, or null
};
constexpr int kTraceSlots = 64;

#ifndef __CUDACC__
}  // namespace ees
#include <vector>
namespace ees {
struct TileHost {
    int32_t n_tiles = 0, n_heavy = 0, n_side = 0, n_side_big = 0, n_side_cold = 0;
    int64_t n_items = 0, n_owned = 0, n_side_entries = 0;
    int64_t n_parts = 0, hot_base = 0;
    int64_t n_listed = 0, n_padded = 0;    // list entries, and with class padding
    int32_t blob_max = 0, n_hot = 0;       // largest head + program
    int32_t grid = 1;                      // persistent CTAs the hot-part layout is made for
    int32_t n_progs = 0;                   // distinct programs
    int64_t st_waves0 = 0, st_waves = 0;   // form 1: estimated evaluation STS wavefronts per call
    std::vector<int64_t> blob_off;         // [T+1] head offsets
    std::vector<uint8_t> blob;             // heads
    std::vector<uint8_t> prog;             // distinct programs
    std::vector<uint32_t> tdesc;           // [T][4] (TileK::tdesc)
    std::vector<double> item_beta, item_v0;
    std::vector<uint8_t> item_model;
    std::vector<int32_t> sd_gid, sd_part, hot_gid;
};
// ees_tile.cpp.  Per-FET data for the item sections: beta (computed by the
// caller exactly as for the other layouts), vprev [3][N], model.
bool build_tile_host(int form, int64_t N, int32_t n_nodes, int32_t n, int64_t nnz, const int32_t *const TT[4],
                     const int32_t *raw_slot, const std::vector<int64_t> &iptr,
                     const std::vector<int32_t> &idev, const std::vector<int32_t> &rails,
                     const std::vector<int32_t> &row_ptr, const std::vector<int32_t> &col_idx,
                     const double *beta, const double *vprev, const int32_t *model, int32_t grid,
                     TileHost &out);
#endif

// COLOR under EES_CONFLICT_HYBRID.  The layout is the
// colour-major DevK with `slot` = [16][N]: 12 A pairs then 4 b rows, each
// >= 0 (a target written with a plain read-modify-write: no two FETs of one
// colour share it), -1 (none), or <= -2 (scratch slot -2-code: the target is
// a side target, summed after the last colour).  Side targets' scratch slots
// are contiguous per target (netlist order, then pair order), cut into
// chunks of at most kChunk contributions.
struct SideK {
    double *buf;                 // [n_contrib] one slot per side contribution
    int32_t n_side, n_chunks;
    int64_t nnz;
    const int64_t *chunk_lo;     // [n_chunks+1] ranges of buf
    const int32_t *side_gid;     // [n_side] global target (A index, or nnz + b row)
    const int32_t *side_chunk;   // [n_side+1] chunks of each side target
    double *chunk_part;          // [n_chunks]
};

// ---- launchers (ees_kernels.cu); all asynchronous on `st` ----
cudaError_t launch_color_h(const DevK &dv16, const CallK &call, int64_t begin, int64_t count,
                           double *side_buf, cudaStream_t st);
cudaError_t launch_side_sum(const SideK &sk, const CallK &call, cudaStream_t st, int *n_launches);
cudaError_t launch_color_stamp(const DevK &dv16, const GatherK &gk, const CallK &call, const int32_t *perm,
                               int64_t begin, int64_t count, double *side_buf, cudaStream_t st);
cudaError_t launch_accept_soa(const int4 *term, int64_t N, const CallK &call, double *v0, cudaStream_t st);
cudaError_t launch_accept_tile(const TileK &tk, const CallK &call, double *item_v0, cudaStream_t st);
cudaError_t measure_fp64_peak(double *tflops);
cudaError_t measure_red_throughput(int mode, double *gops);
cudaError_t launch_stream_probe(const void *src, int64_t read_bytes, void *dst, int64_t write_bytes,
                                double *sink, cudaStream_t st);
int tile_blocks_per_sm(int form);
cudaError_t launch_tile(const TileK &tk, const CallK &call, int grid, cudaStream_t st, int *n_launches);
cudaError_t launch_atomic(const DevK &dv, const CallK &call, int grid, bool agg, cudaStream_t st);
cudaError_t launch_color(const DevK &dv, const CallK &call, int64_t begin, int64_t count,
                         double *partials, cudaStream_t st);
int color_coop_blocks_per_sm();
cudaError_t launch_color_coop(const DevK &dv, const CallK &call, const int64_t *cptr_dev, int32_t C,
                              double *partials, int grid, cudaStream_t st);
cudaError_t launch_rail_finalize(const CallK &call, const double *partials, int64_t n_blocks,
                                 cudaStream_t st);
cudaError_t launch_eval_compact(const DevK &dv, const GatherK &gk, const CallK &call, cudaStream_t st);
cudaError_t launch_gather(const DevK &dv, const GatherK &gk, const CallK &call, cudaStream_t st,
                          int *n_launches);
// one GATHER phase: 0 evaluate, 1 reduce, 2 heavy finalise (for phase timing)
cudaError_t launch_gather_phase(const DevK &dv, const GatherK &gk, const CallK &call, cudaStream_t st,
                                int phase, int *n_launches);
cudaError_t launch_race_probe(const DevK &dv, const int32_t *perm, int64_t begin, int64_t count,
                              int32_t *cnt_a, int32_t *cnt_b, cudaStream_t st);
cudaError_t launch_count_conflicts(const int32_t *cnt, int64_t n, unsigned long long *out,
                                   cudaStream_t st);
int atomic_blocks_per_sm();

}  // namespace ees
