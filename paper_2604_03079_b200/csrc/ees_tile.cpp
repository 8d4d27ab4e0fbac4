// ees_tile.cpp -- host setup of the TILE variant (EES_TILE).
//
// The stamp phase is re-cut by ownership instead of by colour: rows are
// grouped into tiles of consecutive node ids; a tile owns every target (A
// entry or b row) whose contributors are all FETs incident on its rows, so one
// CTA can gather them in shared memory and write them with a plain RMW.
// Heavy nodes (rails and nodes with more than kHeavyDeg incident FETs) never
// own rows: an entry (h, c) with c light belongs to c's tile (its contributors
// all touch c), and only heavy x heavy entries and heavy b rows can have
// contributors in several tiles -- those are "side" targets, summed from
// per-tile parts in a fixed order.  This is the paper's observation (P:31, P:60:
// writers collide only through shared nodes) applied per SM instead of per
// colour.
#include <algorithm>
#include <cstring>
#include <functional>
#include <iterator>
#include <numeric>
#include <unordered_map>
#include <vector>

#include "ees_internal.h"

// build-time A/B knobs of the TILE builder (tools/ab_tree.sh)
#ifndef EES_BANK_ORDER
#define EES_BANK_ORDER 0
#endif
#ifndef EES_PIECE_INTERLEAVE
#define EES_PIECE_INTERLEAVE 1
#endif
#ifndef EES_BANK_GREEDY
#define EES_BANK_GREEDY 0
#endif
#ifndef EES_BANK_SWAP
#define EES_BANK_SWAP 1          // passes of lane swaps (0: none)
#endif

namespace ees {

namespace {
constexpr int32_t kUnset = -1;
constexpr int32_t kSide = -2;
// Upper bound of a tile's blob while it is being formed.  Owned targets are
// counted exactly: a target with L <= kOpMax contributions costs ceil(L/2)
// 4 B pair-ops and a 4 B destination; a longer one a 4 B destination, 2 B per
// entry, a 4 B meta word and, if its lane-group size is new in the tile, a
// 16 B class header.  Items cost item_blob_bytes(form).  Heavy x heavy
// targets (owned by their home tile, or side) are bounded: owned, as above
// (<= 12 + 2c B for c contributions, plus meta and class header); side, at
// pieces of <= kSidePiece entries, each ceil(c'/2) 4 B pair-ops, a 2 B
// destination and an 8 B side entry (<= 2c' + 12 B) if c' <= kOpMax, else a
// group-class target (<= 2c' + 32 B with its class header): with kSidePiece
// = 4, <= 2c + 12 ceil(c/4) <= 12 + 5c B in all: kHHTarget = 12 B per
// distinct target and kHHContrib = 5 B per contribution cover both.  Fixed:
// head and program headers, the two streams' per-sequence start words and row
// offsets (a tile lists at most 16 kTileItems contributions, so a stream has
// at most 16 + ceil(kOpMax/2) steps: balanced, longest first), fourteen section
// paddings.
constexpr int32_t kMaxSteps = 16 + (kOpMax + 1) / 2;
constexpr int64_t kBlobFixed0 = (int64_t)sizeof(TileHdr) + (int64_t)sizeof(ProgHdr) + 14 * 16 +
                               2 * 2 * kTileThreads + 2 * 2 * (kMaxSteps + 1);
constexpr int64_t kHHTarget = 12, kHHContrib0 = 5;
size_t pad16(size_t x) { return (x + 15) & ~(size_t)15; }
}  // namespace

namespace {
// strict: the form-1 row bound is the guaranteed one (longest-first
// balancing: floor(P / kTileItems) + longest chain); otherwise the expected
// one (ceil(P / kTileItems) + 1), and build_tile_host falls back to strict if
// a tile's rows do not fit.
bool build_tile_impl(int form, bool strict, int64_t N, int32_t n_nodes, int32_t n, int64_t nnz,
                     const int32_t *const TT[4], const int32_t *raw_slot, const std::vector<int64_t> &iptr,
                     const std::vector<int32_t> &idev, const std::vector<int32_t> &rails,
                     const std::vector<int32_t> &row_ptr, const std::vector<int32_t> &col_idx,
                     const double *beta, const double *vprev, const int32_t *model, int32_t grid,
                     TileHost &out)
{
    const int64_t kStageMax = stage_max(form), kItemBlobBytes = item_blob_bytes(form);
    // form 1 (v5): a side piece of <= 4 entries costs a 4 B destination and an
    // 8 B side entry (<= 3c + 12 B for c contributions); an owned heavy x heavy
    // target a 4 B destination (+ meta and class header if long, hh_len_bytes)
    const int64_t kHHContrib = form == 1 ? 3 : kHHContrib0;
    // form 1 (v5): head and program headers, the per-thread sequence words,
    // seven section paddings
    const int64_t kBlobFixed = form == 1 ? (int64_t)sizeof(TileHdr) + (int64_t)sizeof(ProgHdr5) + 4 * kTileThreads +
                                               10 * 16
                                         : kBlobFixed0;
    // a device's 12 slots and 4 terminals in one 64-byte record: the builder
    // visits devices in row order (random in netlist order on scattered
    // topologies), so one cache line per visit instead of sixteen
    struct DevRec {
        int32_t s[NPAIR];
        int32_t t[4];
    };
    std::vector<DevRec> rec((size_t)std::max<int64_t>(1, N));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; i++) {
        for (int p = 0; p < NPAIR; p++) rec[i].s[p] = raw_slot[p * N + i];
        for (int a = 0; a < 4; a++) rec[i].t[a] = TT[a][i];
    }
    // source tied to bulk: the kernel merges DB/BD/BB/J[B] into DS/SD/SS/J[S]
    auto merged = [&](int64_t i) { return rec[i].t[2] == rec[i].t[3] && rec[i].t[2] != -1; };
    // is contribution p (12 pairs, then 4 b rows) of FET i in a list?
    auto listed_c = [&](int64_t i, int p) -> bool {
        if (p < NPAIR) return rec[i].s[p] >= 0 && !(merged(i) && (p == DB || p == BD || p == BB));
        return rec[i].t[p - NPAIR] >= 0 && !(p == NPAIR + 3 && merged(i));
    };
    const int32_t NN = std::max(1, n_nodes);
    // A light row whose FETs alone overflow a tile (pathological: many heavy x
    // heavy entries on few FETs) is promoted to heavy and the partition redone.
    std::vector<uint8_t> promoted((size_t)NN, 0);
    std::vector<uint8_t> heavy;
    std::vector<int32_t> hs_ptr, hs_k;
    std::vector<int32_t> tile_of_row, mark, home, cur, tile_rows_ptr, tile_rows, out_item_ptr, item_dev;
    int32_t t = 0;
    int64_t bytes = kBlobFixed;
    int32_t last_row = -2;
    // distinct heavy x heavy targets a FET brings to tile t; marks them, and
    // returns their bytes beyond kHHContrib per contribution (kHHTarget each,
    // plus the class header of their length if it would be new, as owned)
    std::vector<int32_t> hh_seen((size_t)(nnz + n), -1);
    std::function<int64_t(int32_t, int32_t)> hh_len_bytes;      // set below (needs tcnt)
    int64_t hh_nd = 0;                                           // distinct new targets (hh_new)
    auto hh_new = [&](int64_t i, int32_t tile) {
        int64_t k = 0;
        for (int p = 0; p < NPAIR; p++) {
            const int32_t s2 = rec[i].s[p];
            if (s2 >= 0 && heavy[rec[i].t[pair_row(p)]] && heavy[rec[i].t[pair_col(p)]] && hh_seen[s2] != tile) {
                hh_seen[s2] = tile;
                k += kHHTarget + hh_len_bytes(s2, tile);
                hh_nd++;
            }
        }
        for (int a = 0; a < 4; a++) {
            const int32_t r = rec[i].t[a];
            if (r >= 0 && heavy[r] && hh_seen[nnz + r] != tile) {
                hh_seen[nnz + r] = tile;
                k += kHHTarget + hh_len_bytes((int32_t)(nnz + r), tile);
                hh_nd++;
            }
        }
        return k;
    };
    // listed contributions per target (a target nobody stamps is not listed):
    // an owned target's contributors all lie in its tile, so its program bytes
    // are known before the partition
    std::vector<int32_t> tcnt((size_t)(nnz + n), 0);
    for (int64_t i = 0; i < N; i++)
        for (int p = 0; p < NPAIR + 4; p++)
            if (listed_c(i, p)) tcnt[p < NPAIR ? rec[i].s[p] : nnz + rec[i].t[p - NPAIR]]++;
    // lane-group sizes (group classes) of the tile being formed (class headers)
    std::vector<int32_t> len_tile(64, -1);
    auto tgt_bytes = [&](int32_t L, int32_t tile) -> int64_t {
        if (L <= 0) return 0;
        if (form == 1 && L <= kOpMax1) return 4;                     // v5: destination (positions per item)
        if (form == 0 && L <= kOpMax) return 4 + 4 * (int64_t)((L + 1) / 2);     // destination, pair-ops
        int64_t e = 4 + 2 * (int64_t)L + 4;                         // destination, entries, meta
        const int32_t key = cls_group(L);
        if (len_tile[key] != tile) {
            len_tile[key] = tile;
            e += (int64_t)sizeof(TileCls);
        }
        return e;
    };
    hh_len_bytes = [&](int32_t g, int32_t tile) -> int64_t {
        const int32_t L = tcnt[g];
        if (L <= (form == 1 ? kOpMax1 : kOpMax)) return 0;
        const int32_t key = cls_group(L);
        if (len_tile[key] == tile) return 4;                     // group meta word (owned case)
        len_tile[key] = tile;
        return 4 + (int64_t)sizeof(TileCls);
    };
    auto row_bytes = [&](int32_t r, int32_t tile) {       // the row's CSR entries and its b row
        int64_t e = tgt_bytes(tcnt[nnz + r], tile);
        for (int32_t k = row_ptr[r]; k < row_ptr[r + 1]; k++) e += tgt_bytes(tcnt[k], tile);
        return e;
    };
    // heavy x heavy contributions of a FET (owned by its home tile or side)
    auto hh_count = [&](int64_t i) {
        int32_t k = 0;
        for (int p = 0; p < NPAIR; p++)
            if (rec[i].s[p] >= 0 && heavy[rec[i].t[pair_row(p)]] && heavy[rec[i].t[pair_col(p)]]) k++;
        for (int a = 0; a < 4; a++)
            if (rec[i].t[a] >= 0 && heavy[rec[i].t[a]]) k++;
        return k;
    };

    // form 1 (TILE v5): the tile's pair rows.  Owned targets of L <= kOpMax1
    // contributions take ceil(L/2) pairs of one thread (a chain), longer ones
    // L slots of the group area.  A heavy x heavy target with c contributions
    // in the tile takes at most c/2 + 1 pairs (side pieces of <= 4 entries;
    // owned, a chain) or c group slots (< c/2 + 1 pairs' 2 slots each): counted
    // as half a pair per contribution and one pair per distinct target.
    // Longest-first balancing gives at most floor(P / kTileItems) + (longest
    // chain) rows, which with the group area must fit the kScRows rows of the
    // slot buffer.  (P is kept in half pairs.)
    int64_t tP = 0, tG = 0;
    int32_t tPM = 0;
    auto tgt_pairs = [&](int32_t L, int64_t &P, int32_t &PM, int64_t &G) {
        if (L <= 0) return;
        if (L <= kOpMax1) {
            P += 2 * ((L + 1) / 2);
            PM = std::max(PM, (L + 1) / 2);
        } else {
            G += L;
        }
    };
    auto hh_pm = [&](int64_t i) {                // longest chain a heavy x heavy target of FET i can need
        int32_t m = 0;
        auto one = [&](int64_t g) { m = std::max(m, tcnt[g] <= kOpMax1 ? (tcnt[g] + 1) / 2 : 2); };
        for (int p = 0; p < NPAIR; p++)
            if (rec[i].s[p] >= 0 && heavy[rec[i].t[pair_row(p)]] && heavy[rec[i].t[pair_col(p)]]) one(rec[i].s[p]);
        for (int a = 0; a < 4; a++)
            if (rec[i].t[a] >= 0 && heavy[rec[i].t[a]]) one(nnz + rec[i].t[a]);
        return m;
    };
    auto rows_over = [&](int64_t P, int32_t PM, int64_t G) {
        if (form != 1) return false;
        const int64_t pairs = (P + 1) / 2;
        const int64_t rows = strict ? pairs / kTileItems + PM : (pairs + kTileItems - 1) / kTileItems + (PM > 1);
        return rows > kScRows || rows * 2 * kTileItems + G > (int64_t)kScRows * 2 * kTileItems;
    };
    auto close_tile = [&]() {
        std::sort(cur.begin(), cur.end());
        item_dev.insert(item_dev.end(), cur.begin(), cur.end());
        out_item_ptr.push_back((int32_t)item_dev.size());
        tile_rows_ptr.push_back((int32_t)tile_rows.size());
        cur.clear();
        bytes = kBlobFixed;
        tP = tG = 0;
        tPM = 0;
        t++;
    };
    for (bool done = false; !done;) {
    done = true;
    out = TileHost();
    heavy.assign((size_t)NN, 0);
    for (int32_t v = 0; v < n_nodes; v++) heavy[v] = (iptr[v + 1] - iptr[v]) > kHeavyDeg || promoted[v];
    for (int32_t r : rails) heavy[r] = 1;
    for (int32_t v = 0; v < n_nodes; v++) out.n_heavy += heavy[v];

    // heavy-row entries (h, c) with c a light node belong to c's tile
    hs_ptr.assign((size_t)NN + 1, 0);
    hs_k.clear();
    for (int32_t h = 0; h < n_nodes; h++)
        if (heavy[h])
            for (int32_t k = row_ptr[h]; k < row_ptr[h + 1]; k++) {
                const int32_t c = col_idx[k];
                if (c < n_nodes && !heavy[c]) hs_ptr[c + 1]++;
            }
    for (int32_t v = 0; v < n_nodes; v++) hs_ptr[v + 1] += hs_ptr[v];
    hs_k.resize((size_t)hs_ptr[n_nodes]);
    {
        std::vector<int32_t> fill(hs_ptr.begin(), hs_ptr.end() - 1);
        for (int32_t h = 0; h < n_nodes; h++)
            if (heavy[h])
                for (int32_t k = row_ptr[h]; k < row_ptr[h + 1]; k++) {
                    const int32_t c = col_idx[k];
                    if (c < n_nodes && !heavy[c]) hs_k[fill[c]++] = k;
                }
    }
    // ---- tiles of consecutive light rows: <= kTileItems FETs, <= kStageMax blob bytes
    tile_of_row.assign((size_t)NN, -1);
    mark.assign((size_t)std::max<int64_t>(1, N), -1);
    home.assign((size_t)std::max<int64_t>(1, N), -1);
    cur.clear();
    tile_rows_ptr.assign(1, 0);
    tile_rows.clear();
    out_item_ptr.assign(1, 0);
    item_dev.clear();
    t = 0;
    bytes = kBlobFixed;
    tP = tG = 0;
    tPM = 0;
    last_row = -2;
    std::fill(hh_seen.begin(), hh_seen.end(), -1);
    std::fill(len_tile.begin(), len_tile.end(), -1);
    for (int32_t v = 0; v < n_nodes; v++) {
        if (heavy[v]) continue;
        // a tile's rows are consecutive, so its owned entries of A and b are
        // one CSR block and one row range (implicit ids in the blob)
        if ((int32_t)tile_rows.size() > tile_rows_ptr.back() && last_row != v - 1) close_tile();
        for (int pass = 0; pass < 2; pass++) {
            int32_t fresh = 0;
            int64_t add_bytes = row_bytes(v, t);
            int64_t aP = tP, aG = tG;
            int32_t aPM = tPM;
            tgt_pairs(tcnt[nnz + v], aP, aPM, aG);
            for (int32_t k = row_ptr[v]; k < row_ptr[v + 1]; k++) tgt_pairs(tcnt[k], aP, aPM, aG);
            for (int32_t k = hs_ptr[v]; k < hs_ptr[v + 1]; k++) {
                add_bytes += tgt_bytes(tcnt[hs_k[k]], t);
                tgt_pairs(tcnt[hs_k[k]], aP, aPM, aG);
            }
            for (int64_t k = iptr[v]; k < iptr[v + 1]; k++) {
                const int32_t i = idev[k];
                if (mark[i] != t) {
                    fresh++;
                    add_bytes += kItemBlobBytes;
                }
                if (home[i] < 0) {
                    hh_nd = 0;
                    add_bytes += hh_new(i, t) + kHHContrib * hh_count(i);
                    if (form == 1) {
                        aP += hh_count(i) + 2 * hh_nd;
                        aPM = std::max(aPM, hh_pm(i));
                    }
                }
            }
            const bool over = (int64_t)cur.size() + fresh > kTileItems || bytes + add_bytes > kStageMax ||
                              rows_over(aP, aPM, aG);
            if (over && pass == 0 && !cur.empty()) {
                close_tile();
                continue;
            }
            if (over) {                    // a single light row exceeds a tile
                promoted[v] = 1;
                done = false;
            }
            bytes += add_bytes;
            tP = aP;
            tG = aG;
            tPM = aPM;
            break;
        }
        if (!done) break;
        last_row = v;
        tile_of_row[v] = t;
        tile_rows.push_back(v);
        for (int64_t k = iptr[v]; k < iptr[v + 1]; k++) {
            const int32_t i = idev[k];
            if (mark[i] != t) {
                mark[i] = t;
                cur.push_back(i);
            }
            if (home[i] < 0) home[i] = t;
        }
    }
    }   // partition attempt
    if (!cur.empty()) close_tile();
    // FETs with no light terminal (all heavy or ground): orphan tiles
    for (int64_t i = 0; i < N; i++)
        if (home[i] < 0) {
            const int64_t add_bytes = kItemBlobBytes + (kHHTarget + (int64_t)sizeof(TileCls) + kHHContrib) * hh_count(i);
            const int64_t aP = tP + (form == 1 ? 3 * hh_count(i) : 0);      // (each distinct at most once)
            const int32_t aPM = std::max(tPM, form == 1 ? hh_pm(i) : 0);
            if (!cur.empty() && ((int64_t)cur.size() + 1 > kTileItems || bytes + add_bytes > kStageMax ||
                                 rows_over(aP, aPM, tG)))
                close_tile();
            home[i] = t;
            bytes += add_bytes;
            tP += form == 1 ? 3 * hh_count(i) : 0;
            tPM = std::max(tPM, form == 1 ? hh_pm(i) : 0);
            cur.push_back((int32_t)i);
        }
    if (!cur.empty()) close_tile();
    const int32_t T = t;
    out.n_tiles = T;
    if ((int64_t)item_dev.size() > INT32_MAX) return false;

    // heavy x heavy targets: owned by the common home tile of all contributors, else side
    const int64_t NT = nnz + n;
    std::vector<int32_t> hh_owner((size_t)NT, kUnset);
    std::vector<std::vector<int32_t>> hh_of_tile((size_t)T);
    auto note_hh = [&](int64_t g, int32_t h) {
        int32_t &o = hh_owner[g];
        if (o == kUnset) o = h;
        else if (o != h) o = kSide;
    };
    for (int64_t i = 0; i < N; i++) {
        for (int p = 0; p < NPAIR; p++) {
            const int32_t k = rec[i].s[p];
            if (k >= 0 && heavy[rec[i].t[pair_row(p)]] && heavy[rec[i].t[pair_col(p)]]) note_hh(k, home[i]);
        }
        for (int a = 0; a < 4; a++) {
            const int32_t r = rec[i].t[a];
            if (r >= 0 && heavy[r]) note_hh(nnz + r, home[i]);
        }
    }
    for (int64_t g = 0; g < NT; g++)
        if (hh_owner[g] >= 0) hh_of_tile[hh_owner[g]].push_back((int32_t)g);

    // ---- per tile: blob = header + classes | items | side | dst | ent.
    // Tiles are emitted in parallel into their own buffers (side entries carry
    // their global target for now), then concatenated in tile order, where
    // side ids are numbered by first appearance (the serial order).
    struct TileOut {
        std::vector<uint8_t> blob, prog;     // head, program
        uint64_t hash = 0;                   // of the program bytes
        int64_t listed = 0, L = 0, padded = 0;
        int64_t st_waves0 = 0, st_waves = 0;  // form 1: estimated STS wavefronts (identity / placed)
        int32_t n_own = 0, n_sent = 0;
        bool ok = true;
    };
    std::vector<TileOut> tout((size_t)T);
    if (form == 1) {
        out.item_beta.assign((size_t)T * kTileItems, 0.0);
        out.item_v0.assign((size_t)T * kTileItems * 3, 0.0);
        out.item_model.assign((size_t)T * kTileItems, 0);
    }
    bool all_ok = true;
#pragma omp parallel
    {
    std::vector<std::pair<int32_t, uint16_t>> con, side, piece_tmp;
    std::vector<int32_t> gids;
    std::vector<SideEnt> sents;
    // one target of the program: destination, its entries con/side[beg, beg+len)
    struct Tgt {
        int32_t dst;
        int32_t beg, len;
        bool is_side;
    };
    std::vector<Tgt> tg;
    std::vector<TileCls> cls;
    std::vector<int32_t> dsts;
    std::vector<uint16_t> ents;
    std::vector<uint32_t> meta;
    std::vector<int32_t> owned_g;
    auto emit_tile = [&](int32_t tt, TileOut &o) -> bool {
        // owned targets, ascending
        gids.clear();
        for (int32_t q = tile_rows_ptr[tt]; q < tile_rows_ptr[tt + 1]; q++) {
            const int32_t r = tile_rows[q];
            for (int32_t k = row_ptr[r]; k < row_ptr[r + 1]; k++) gids.push_back(k);
            gids.push_back((int32_t)(nnz + r));
            for (int32_t k = hs_ptr[r]; k < hs_ptr[r + 1]; k++) gids.push_back(hs_k[k]);
        }
        gids.insert(gids.end(), hh_of_tile[tt].begin(), hh_of_tile[tt].end());
        std::sort(gids.begin(), gids.end());
        // contributions of this tile's items, (target, shared-memory slot)
        con.clear();
        side.clear();
        const int32_t q0 = out_item_ptr[tt];
        const int32_t ni = out_item_ptr[tt + 1] - q0;
        // the contributions of FET i this tile lists: owned by it, or (heavy x
        // heavy) side contributions of its home tile
        auto in_tile = [&](int32_t i, int p) -> bool {
            if (!listed_c(i, p)) return false;
            const DevRec &dr = rec[i];
            const int32_t r = p < NPAIR ? dr.t[pair_row(p)] : dr.t[p - NPAIR];
            const int32_t c = p < NPAIR ? dr.t[pair_col(p)] : r;
            if (!heavy[r] || !heavy[c]) return (!heavy[r] ? tile_of_row[r] : tile_of_row[c]) == tt;
            return home[i] == tt;
        };
        // gate-row items (every listed contribution in the gate row: GD, GG,
        // GS, J[G] -- capacitor companions only, no channel evaluation, no x)
        // go last, so whole warps take the short path
        int32_t n_full = ni;
        {
            auto gate_only = [&](int32_t i) {
                for (int p = 0; p < NPAIR + 4; p++)
                    if (in_tile(i, p) && p != GD && p != GG && p != GS && p != NPAIR + 1) return false;
                return true;
            };
            int32_t *it0 = item_dev.data() + q0;
            n_full = (int32_t)(std::stable_partition(it0, it0 + ni, [&](int32_t i) { return !gate_only(i); }) - it0);
        }
        for (int32_t q = q0; q < out_item_ptr[tt + 1]; q++) {
            const int32_t i = item_dev[q];
            const int32_t loc = q - q0;
            for (int p = 0; p < NPAIR + 4; p++) {
                if (!listed_c(i, p)) continue;
                int64_t g;
                int32_t r, c;
                const DevRec &dr = rec[i];
                if (p < NPAIR) {
                    g = dr.s[p];
                    r = dr.t[pair_row(p)];
                    c = dr.t[pair_col(p)];
                } else {
                    r = dr.t[p - NPAIR];
                    g = nnz + r;
                    c = r;
                }
                const uint16_t slot = (uint16_t)(p * kTileItems + loc);
                if (!heavy[r] || !heavy[c]) {
                    const int32_t owner = !heavy[r] ? tile_of_row[r] : tile_of_row[c];
                    if (owner == tt) con.emplace_back((int32_t)g, slot);
                } else if (home[i] == tt) {
                    if (hh_owner[g] == tt) con.emplace_back((int32_t)g, slot);
                    else side.emplace_back((int32_t)g, slot);
                }
            }
        }
        // entries of one target in item order, then pair order (stable)
        auto by_target = [](const std::pair<int32_t, uint16_t> &a, const std::pair<int32_t, uint16_t> &b) {
            return a.first < b.first;
        };
        std::stable_sort(con.begin(), con.end(), by_target);
        std::stable_sort(side.begin(), side.end(), by_target);
        // targets: owned (all contributors in this tile; destination = global
        // target), then side pieces (this tile's contributions to a side
        // target in pieces of <= kSidePiece entries, one side entry each)
        tg.clear();
        for (size_t k = 0; k < con.size();) {
            const int64_t g = con[k].first;
            size_t e = k;
            while (e < con.size() && con[e].first == g) e++;
            if (!std::binary_search(gids.begin(), gids.end(), (int32_t)g)) return false;
            tg.push_back(Tgt{(int32_t)g, (int32_t)k, (int32_t)(e - k), false});
            k = e;
        }
        const int32_t n_own = (int32_t)tg.size();
        sents.clear();
        for (size_t k = 0; k < side.size();) {
            const int32_t g = side[k].first;
            size_t e = k;
            while (e < side.size() && side[e].first == g) e++;
#if EES_PIECE_INTERLEAVE
            // piece q takes entries q, q + P, q + 2P, ... (P pieces): a piece's
            // entries come from items far apart, so its two pair rows do not
            // receive stores of the same half-warp into the same bank pair
            {
                const size_t n = e - k, P = (n + kSidePiece - 1) / kSidePiece;
                if (P > 1) {
                    piece_tmp.assign(side.begin() + (std::ptrdiff_t)k, side.begin() + (std::ptrdiff_t)e);
                    size_t at = k;
                    for (size_t q = 0; q < P; q++)
                        for (size_t m = q; m < n; m += P) side[at++] = piece_tmp[m];
                }
            }
            for (size_t p0 = k, q = 0, n = e - k, P = (n + kSidePiece - 1) / kSidePiece; p0 < e; q++) {
                const size_t p1 = p0 + (n - q + P - 1) / P;   // piece q holds ceil((n - q) / P) entries
#else
            for (size_t p0 = k; p0 < e; p0 += kSidePiece) {
                const size_t p1 = std::min(e, p0 + (size_t)kSidePiece);
#endif
                SideEnt se;
                se.sid = g;             // global target; numbered after the concatenation
                se.slot = -1;
                tg.push_back(Tgt{-1 - (int32_t)sents.size(), (int32_t)p0, (int32_t)(p1 - p0), true});
                sents.push_back(se);
#if EES_PIECE_INTERLEAVE
                p0 = p1;
#endif
            }
            k = e;
        }
        const int32_t n_sent = (int32_t)sents.size();
        o.listed += (int64_t)con.size() + (int64_t)side.size();
        auto entry = [&](const Tgt &t2, int32_t p) {
            return (uint16_t)(8 * (t2.is_side ? side[t2.beg + p].second : con[t2.beg + p].second));
        };
        // ---- destination bases: the first target of each cluster of the owned
        // targets (ascending; a new cluster after a gap > kGap and at nnz, so
        // a cluster is all A or all b), so equal tile structures give equal
        // codes; more than kTileBases clusters: fixed bases (8 chunks of A,
        // 8 of b)
        int32_t bases[kTileBases];
        bool fixed = false;
        {
            constexpr int32_t kGap = 4096, kSpan = 1 << 28;
            int nb = 0;
            int32_t prev = -1;
            owned_g.clear();
            for (const Tgt &t2 : tg)
                if (!t2.is_side) owned_g.push_back(t2.dst);
            std::sort(owned_g.begin(), owned_g.end());
            for (const int32_t g : owned_g) {
                if (nb == 0 || g - prev > kGap || g - bases[nb - 1] >= kSpan - 1 ||
                    (g >= nnz && bases[nb - 1] < nnz)) {
                    if (nb == kTileBases) { fixed = true; break; }
                    bases[nb++] = g;
                }
                prev = g;
            }
            if (fixed) {
                for (int q = 0; q < 8; q++) {
                    bases[q] = (int32_t)std::min<int64_t>((int64_t)q * kSpan, INT32_MAX);
                    bases[8 + q] = (int32_t)std::min<int64_t>(nnz + (int64_t)q * kSpan, INT32_MAX);
                }
            } else {
                for (int q = nb; q < kTileBases; q++) bases[q] = INT32_MAX;
            }
        }
        auto code_of = [&](int32_t g) -> uint32_t {
            if (fixed) {
                const int64_t r = g < nnz ? (int64_t)g : (int64_t)g - nnz;
                const int q = (int)(r >> 28) + (g < nnz ? 0 : 8);
                return ((uint32_t)q << 28) | (uint32_t)(r & 0x0FFFFFFF);
            }
            int q = 0;
            while (q + 1 < kTileBases && bases[q + 1] <= g) q++;      // clusters never straddle nnz
            return ((uint32_t)q << 28) | (uint32_t)(g - bases[q]);
        };
        for (int32_t g : owned_g) {             // every owned target must be codable
            const uint32_t c = code_of(g);
            const int q = (int)(c >> 28);
            if ((int64_t)bases[q] + (c & 0x0FFFFFFF) != (int64_t)g) return false;
        }
        if (form == 1) {
            // ---- TILE v5 program (ees_internal.h ProgHdr5): pair rows, positions
            std::vector<int32_t> opt, lng;            // row targets; long owned targets (group area)
            for (int32_t k = 0; k < (int32_t)tg.size(); k++) {
                if (!tg[k].is_side && tg[k].len > kOpMax1) lng.push_back(k);
                else opt.push_back(k);
            }
            std::stable_sort(opt.begin(), opt.end(), [&](int32_t a, int32_t b) { return tg[a].len > tg[b].len; });
            std::vector<std::vector<int32_t>> seq(kTileThreads);
            std::vector<int32_t> load(kTileThreads, 0);
            for (int32_t k : opt) {                    // longest first onto the least-loaded thread
                int best = 0;
                for (int r = 1; r < kTileThreads; r++)
                    if (load[r] < load[best]) best = r;
                seq[best].push_back(k);
                load[best] += (tg[k].len + 1) / 2;
            }
            const int32_t n_rows = *std::max_element(load.begin(), load.end());
            int64_t G = 0;
            for (int32_t k : lng) G += tg[k].len;
            if (n_rows > kScRows || (int64_t)n_rows * 2 * kTileThreads + G > (int64_t)kScRows * 2 * kTileThreads)
                return false;
            const int32_t gbase = n_rows * 2 * kTileThreads;           // first group slot
            // pos: [2][ni] uint4 -- item `it`'s positions of contributions 0-7
            // at 16*it, of 8-15 at 16*(ni + it) (two conflict-free LDS.128)
            std::vector<uint16_t> pos((size_t)ni * 16, (uint16_t)kTrashByte1);
            auto pos_at = [&](int32_t loc, int32_t pc) -> uint16_t & {
                return pos[((size_t)(pc >> 3) * ni + loc) * 8 + (pc & 7)];
            };
            auto code_at = [&](const Tgt &t2, int32_t p) -> uint16_t {
                return t2.is_side ? side[t2.beg + p].second : con[t2.beg + p].second;
            };
            auto place = [&](const Tgt &t2, int32_t p, int32_t slot_index) {
                const uint16_t cs = code_at(t2, p);
                pos_at(cs % kTileItems, cs / kTileItems) = (uint16_t)(8 * slot_index);   // (item, p)
            };
            // ---- bank-aware placement of the evaluation's stores.  Thread j's
            // pair of row s sits at byte 16 (s kTileItems + j): its two halves
            // are the 8-byte bank pairs 2 (j mod 8) and 2 (j mod 8) + 1.  A
            // half-warp's STS.64 of contribution p (items 16w' .. 16w'+15)
            // takes as many shared-memory wavefronts as its busiest bank pair
            // holds distinct addresses.  Within each warp the 32 sequences are
            // permuted onto the lanes (the warp's set of RED addresses, hence
            // their coalescing, is unchanged) and the two halves of each full
            // pair are oriented, greedily, to spread every such store over the
            // 16 bank pairs.  (The order of a target's additions changes with
            // an orientation; it stays fixed per program: deterministic.)
            std::vector<int32_t> perm(kTileThreads);        // thread j runs sequence perm[j]
            std::vector<uint8_t> flip(tg.size(), 0);         // bit q: pair q of the target swapped
            {
                const int32_t n_full_items = n_full;
                auto key_of = [&](uint16_t cs) {              // (half-warp of items, contribution, item kind)
                    const int32_t pc = cs / kTileItems, loc = cs % kTileItems;
                    return ((loc >> 4) * 16 + pc) * 2 + (loc >= n_full_items ? 1 : 0);
                };
                constexpr int kKeys = (kTileItems / 16) * 16 * 2;
                std::vector<uint8_t> in_rows((size_t)ni * 16, 0);      // 1 rows, 2 group area
                for (int32_t k = 0; k < (int32_t)tg.size(); k++)
                    for (int32_t p = 0; p < tg[k].len; p++) {
                        const uint16_t cs = code_at(tg[k], p);
                        in_rows[(size_t)(cs % kTileItems) * 16 + cs / kTileItems] =
                            (!tg[k].is_side && tg[k].len > kOpMax1) ? 2 : 1;
                    }
                // stores that do not go to the rows: the trash slot (bank pair
                // 0, one address) and the group area (ignored here)
                std::vector<uint16_t> base_cnt((size_t)kKeys * 16, 0);
                for (int32_t loc = 0; loc < ni; loc++) {
                    const bool full = loc < n_full_items;
                    for (int pc = 0; pc < 16; pc++) {
                        if (!full && pc != GD && pc != GG && pc != GS && pc != NPAIR + 1) continue;
                        if (in_rows[(size_t)loc * 16 + pc]) continue;
                        const int key = key_of((uint16_t)(pc * kTileItems + loc));
                        base_cnt[(size_t)key * 16] = 1;                          // trash: one address
                    }
                }
                auto waves = [&](const std::vector<uint16_t> &cnt) {
                    int64_t w = 0;
                    for (int key = 0; key < kKeys; key++) {
                        int m = 0;
                        for (int b = 0; b < 16; b++) m = std::max(m, (int)cnt[(size_t)key * 16 + b]);
                        w += m;
                    }
                    return w;
                };
                // identity placement (the estimate without this step)
                {
                    std::vector<uint16_t> cnt = base_cnt;
                    for (int j = 0; j < kTileThreads; j++)
                        for (int32_t k : seq[j])
                            for (int32_t p = 0; p < tg[k].len; p++)
                                cnt[(size_t)key_of(code_at(tg[k], p)) * 16 + 2 * (j & 7) + (p & 1)]++;
                    o.st_waves0 = waves(cnt);
                }
                std::vector<uint16_t> cnt = base_cnt;
                std::vector<uint16_t> mx(kKeys, 0);                 // per key: its busiest bank pair
                for (int key = 0; key < kKeys; key++)
                    for (int b = 0; b < 16; b++) mx[key] = std::max(mx[key], cnt[(size_t)key * 16 + b]);
                // place sequence s in class c: each full pair oriented by the
                // smaller increase of sum-of-max (then of the counts it meets);
                // returns (increase, counts met); commit = keep the increments
                std::vector<std::pair<int, int>> undo;             // (key*16+b, old max of key)
                auto apply = [&](int s, int c, bool commit, int64_t &dmax, int64_t &prox) {
                    dmax = 0;
                    prox = 0;
                    undo.clear();
                    auto inc = [&](int key, int b) {
                        const size_t q = (size_t)key * 16 + b;
                        undo.emplace_back((int)q, (int)mx[key]);
                        prox += cnt[q];
                        if (++cnt[q] > mx[key]) { mx[key] = cnt[q]; dmax++; }
                    };
                    auto gain = [&](int key, int b) { return cnt[(size_t)key * 16 + b] + 1 > mx[key] ? 1 : 0; };
                    for (int32_t k : seq[s]) {
                        const Tgt &t2 = tg[k];
                        for (int32_t p = 0; p < t2.len; p += 2) {
                            const int ka = key_of(code_at(t2, p));
                            if (p + 1 < t2.len) {
                                const int kb = key_of(code_at(t2, p + 1));
                                int keep, swp;
                                if (ka == kb) {
                                    keep = swp = 0;
                                } else {
                                    keep = 2 * (gain(ka, 2 * c) + gain(kb, 2 * c + 1)) * 64 +
                                           cnt[(size_t)ka * 16 + 2 * c] + cnt[(size_t)kb * 16 + 2 * c + 1];
                                    swp = 2 * (gain(ka, 2 * c + 1) + gain(kb, 2 * c)) * 64 +
                                          cnt[(size_t)ka * 16 + 2 * c + 1] + cnt[(size_t)kb * 16 + 2 * c];
                                }
                                if (swp < keep) {
                                    if (commit) flip[(size_t)k] |= (uint8_t)(1u << (p >> 1));
                                    inc(ka, 2 * c + 1);
                                    inc(kb, 2 * c);
                                } else {
                                    inc(ka, 2 * c);
                                    inc(kb, 2 * c + 1);
                                }
                            } else {
                                inc(ka, 2 * c);
                            }
                        }
                    }
                    if (!commit)
                        for (size_t u = undo.size(); u-- > 0;) {
                            cnt[(size_t)undo[u].first]--;
                            mx[undo[u].first / 16] = (uint16_t)undo[u].second;
                        }
                };
#if EES_BANK_GREEDY
                for (int w = 0; w < kTileThreads / 32; w++) {
                    int order[32], cap[8], n_c[32];
                    for (int l = 0; l < 32; l++) {
                        order[l] = 32 * w + l;
                        n_c[l] = 0;
                        for (int32_t k : seq[32 * w + l]) n_c[l] += tg[k].len;
                    }
                    for (int c = 0; c < 8; c++) cap[c] = 4;
                    if (EES_BANK_ORDER) std::stable_sort(order, order + 32, [&](int a, int b) { return n_c[a - 32 * w] > n_c[b - 32 * w]; });
                    int lane_used[32] = {0};
                    for (int oi = 0; oi < 32; oi++) {
                        const int s = order[oi];
                        int best_c = -1;
                        int64_t best_d = INT64_MAX, best_p = INT64_MAX;
                        for (int c0 = 0; c0 < 8; c0++) {
                            const int c = ((s & 7) + c0) & 7;           // ties: the sequence's own class
                            if (!cap[c]) continue;
                            int64_t d, pr;
                            apply(s, c, false, d, pr);
                            if (d < best_d) { best_d = d; best_p = pr; best_c = c; }
                        }
                        int64_t d, pr;
                        apply(s, best_c, true, d, pr);
                        cap[best_c]--;
                        int lane = best_c;
                        while (lane_used[lane]) lane += 8;
                        lane_used[lane] = 1;
                        perm[32 * w + lane] = s;
                    }
                }
#else
                // identity lane placement; then hill-climb the orientation of
                // each full pair (two halves swapped) on the exact sum of maxima
                for (int j = 0; j < kTileThreads; j++) perm[j] = j;
                for (int j = 0; j < kTileThreads; j++)
                    for (int32_t k : seq[j])
                        for (int32_t p = 0; p < tg[k].len; p++)
                            if (p + 1 < tg[k].len || (p & 1)) {
                                const size_t q = (size_t)key_of(code_at(tg[k], p)) * 16 + 2 * (j & 7) + (p & 1);
                                mx[q / 16] = std::max(mx[q / 16], ++cnt[q]);
                            } else {
                                const size_t q = (size_t)key_of(code_at(tg[k], p)) * 16 + 2 * (j & 7);
                                mx[q / 16] = std::max(mx[q / 16], ++cnt[q]);
                            }
                auto kmax = [&](int key) {
                    uint16_t m = 0;
                    for (int b = 0; b < 16; b++) m = std::max(m, cnt[(size_t)key * 16 + b]);
                    return m;
                };
                for (int pass = 0; pass < 4; pass++) {
                    bool any = false;
                    for (int j = 0; j < kTileThreads; j++) {
                        const int c = j & 7;
                        for (int32_t k : seq[j])
                            for (int32_t p = 0; p + 1 < tg[k].len; p += 2) {
                                const int ka = key_of(code_at(tg[k], p)), kb = key_of(code_at(tg[k], p + 1));
                                if (ka == kb) continue;
                                const bool sw = (flip[(size_t)k] >> (p >> 1)) & 1u;
                                const size_t qa = (size_t)ka * 16 + 2 * c + (sw ? 1 : 0);
                                const size_t qb = (size_t)kb * 16 + 2 * c + (sw ? 0 : 1);
                                const size_t ra = (size_t)ka * 16 + 2 * c + (sw ? 0 : 1);
                                const size_t rb = (size_t)kb * 16 + 2 * c + (sw ? 1 : 0);
                                const int before = mx[ka] + mx[kb];
                                cnt[qa]--; cnt[qb]--; cnt[ra]++; cnt[rb]++;
                                const uint16_t na = kmax(ka), nb = kmax(kb);
                                if (na + nb < before) {
                                    mx[ka] = na; mx[kb] = nb;
                                    flip[(size_t)k] ^= (uint8_t)(1u << (p >> 1));
                                    any = true;
                                } else {
                                    cnt[qa]++; cnt[qb]++; cnt[ra]--; cnt[rb]--;
                                }
                            }
                    }
                    if (!any) break;
                }
#if EES_BANK_SWAP
                // lane swaps inside a warp (the warp's RED set is unchanged): a
                // sequence with a store in a key's busiest bank pair tries each
                // lane of another class; the first swap that lowers the sum of
                // maxima over the keys the two touch is kept
                {
                    std::vector<std::vector<int>> skeys(kTileThreads);
                    for (int s = 0; s < kTileThreads; s++) {
                        for (int32_t k : seq[s])
                            for (int32_t p = 0; p < tg[k].len; p++) skeys[s].push_back(key_of(code_at(tg[k], p)));
                        std::sort(skeys[s].begin(), skeys[s].end());
                        skeys[s].erase(std::unique(skeys[s].begin(), skeys[s].end()), skeys[s].end());
                    }
                    auto add_seq = [&](int s, int c, int sign) {
                        for (int32_t k : seq[s]) {
                            const Tgt &t2 = tg[k];
                            for (int32_t p = 0; p < t2.len; p += 2) {
                                const int ka = key_of(code_at(t2, p));
                                const bool sw = (flip[(size_t)k] >> (p >> 1)) & 1u;
                                cnt[(size_t)ka * 16 + 2 * c + (sw ? 1 : 0)] += sign;
                                if (p + 1 < t2.len)
                                    cnt[(size_t)key_of(code_at(t2, p + 1)) * 16 + 2 * c + (sw ? 0 : 1)] += sign;
                            }
                        }
                    };
                    auto conflicted = [&](int s, int c) {
                        for (int32_t k : seq[s]) {
                            const Tgt &t2 = tg[k];
                            for (int32_t p = 0; p < t2.len; p++) {
                                const int key = key_of(code_at(t2, p));
                                const bool sw = (flip[(size_t)k] >> (p >> 1)) & 1u;
                                const int h = (p + 1 < t2.len || (p & 1)) ? ((p & 1) ^ (sw ? 1 : 0)) : 0;
                                const uint16_t v = cnt[(size_t)key * 16 + 2 * c + h];
                                if (v >= 2 && v == mx[key]) return true;
                            }
                        }
                        return false;
                    };
                    std::vector<int> touched;
                    for (int pass = 0; pass < EES_BANK_SWAP; pass++) {
                        bool moved = false;
                        for (int w = 0; w < kTileThreads / 32; w++)
                            for (int la = 0; la < 32; la++) {
                                const int ja = 32 * w + la, ca = la & 7;
                                if (!conflicted(perm[ja], ca)) continue;
                                for (int lb = 0; lb < 32; lb++) {
                                    const int jb = 32 * w + lb, cb = lb & 7;
                                    if (cb == ca) continue;
                                    const int a = perm[ja], b = perm[jb];
                                    touched.clear();
                                    std::set_union(skeys[a].begin(), skeys[a].end(), skeys[b].begin(), skeys[b].end(),
                                                   std::back_inserter(touched));
                                    int before = 0;
                                    for (int key : touched) before += mx[key];
                                    add_seq(a, ca, -1); add_seq(b, cb, -1); add_seq(a, cb, 1); add_seq(b, ca, 1);
                                    int after = 0;
                                    for (int key : touched) after += kmax(key);
                                    if (after < before) {
                                        for (int key : touched) mx[key] = kmax(key);
                                        std::swap(perm[ja], perm[jb]);
                                        moved = true;
                                        break;
                                    }
                                    add_seq(a, cb, -1); add_seq(b, ca, -1); add_seq(a, ca, 1); add_seq(b, cb, 1);
                                }
                            }
                        if (!moved) break;
                    }
                }
#endif
#endif
                o.st_waves = waves(cnt);
            }
            std::vector<uint32_t> oseq(kTileThreads, 0), odst;
            for (int j = 0; j < kTileThreads; j++) {
                const uint32_t start = (uint32_t)odst.size();
                if (start >= (1u << kSeqStartBits)) return false;
                uint32_t em = 0, sm = 0, pm = 0;
                int32_t st = 0;
                for (int32_t k : seq[perm[j]]) {
                    const Tgt &t2 = tg[k];
                    for (int32_t p = 0; p < t2.len; p += 2, st++) {
                        const int32_t slot = 2 * (st * kTileThreads + j);
                        const bool sw = (flip[(size_t)k] >> (p >> 1)) & 1u;
                        place(t2, p, slot + (sw ? 1 : 0));
                        if (p + 1 < t2.len) place(t2, p + 1, sw ? slot : slot + 1);
                        else pm |= 1u << st;                        // odd target: no second half
                        if (p + 2 >= t2.len) {
                            em |= 1u << st;
                            if (t2.is_side) sm |= 1u << st;
                        }
                    }
                    odst.push_back(t2.is_side ? (uint32_t)(-1 - t2.dst) : code_of(t2.dst));
                }
                oseq[j] = start | (em << kSeqEmit) | (sm << kSeqSide) | (pm << kSeqPad);
            }
            // self-check of the pair rows: every listed contribution has its own
            // slot, no slot holds two, and no thread's pairs pass its step count
            {
                std::vector<uint8_t> used((size_t)n_rows * 2 * kTileThreads, 0);
                int64_t placed = 0;
                for (size_t q = 0; q < pos.size(); q++) {
                    if (pos[q] == (uint16_t)kTrashByte1) continue;
                    const int32_t sl = pos[q] / 8;
                    if (sl >= n_rows * 2 * kTileThreads || used[(size_t)sl]++) return false;
                    const int32_t row = sl / (2 * kTileThreads), j = (sl / 2) % kTileThreads;
                    const uint32_t emj = (oseq[(size_t)j] >> kSeqEmit) & 0x7Fu;
                    if (row >= (emj ? 32 - __builtin_clz(emj) : 0)) return false;
                    placed++;
                }
                int64_t in_rows = 0;
                for (int32_t k : opt) in_rows += tg[k].len;
                if (placed != in_rows) return false;
            }
            // group classes (owned targets longer than kOpMax1), entries contiguous
            cls.clear();
            dsts.clear();
            meta.clear();
            {
                std::stable_sort(lng.begin(), lng.end(), [&](int32_t a, int32_t b) {
                    return cls_group(tg[a].len) > cls_group(tg[b].len);
                });
                int64_t cum = 0, off = 0;
                for (size_t k = 0; k < lng.size();) {
                    const int gs = cls_group(tg[lng[k]].len);
                    size_t e = k;
                    while (e < lng.size() && cls_group(tg[lng[e]].len) == gs) e++;
                    TileCls tc;
                    std::memset(&tc, 0, sizeof(tc));
                    tc.n = (uint16_t)(e - k);
                    tc.dst = (uint16_t)dsts.size();
                    int lg = 0;
                    while ((1 << lg) < gs) lg++;
                    tc.lg = (uint16_t)lg;
                    tc.meta = (uint16_t)meta.size();
                    for (size_t q = k; q < e; q++) {
                        const Tgt &t2 = tg[lng[q]];
                        meta.push_back((uint32_t)off | ((uint32_t)t2.len << 16));
                        for (int32_t p = 0; p < t2.len; p++) place(t2, p, gbase + (int32_t)off + p);
                        off += t2.len;
                        dsts.push_back((int32_t)code_of(t2.dst));
                    }
                    tc.rot = (uint16_t)((cum / gs) % (kTileThreads / gs));
                    cls.push_back(tc);
                    cum += (int64_t)tc.n * gs;
                    k = e;
                }
            }
            ProgHdr5 ph;
            std::memset(&ph, 0, sizeof(ph));
            size_t off = sizeof(ProgHdr5);
            auto place_sec = [&](size_t bytes) {
                const size_t at = off;
                off = pad16(off + bytes);
                return at;
            };
            const size_t o_pos = place_sec(2 * pos.size()), o_oseq = place_sec(4 * oseq.size()),
                         o_odst = place_sec(4 * odst.size()), o_cls = place_sec(sizeof(TileCls) * cls.size()),
                         o_dst = place_sec(4 * dsts.size()), o_meta = place_sec(4 * meta.size());
            const size_t pbytes = off;
            if (pbytes > 65535 || gbase > 65535) return false;
            ph.n_rows = (uint16_t)n_rows;
            ph.off_pos = (uint16_t)o_pos;
            ph.off_oseq = (uint16_t)o_oseq;
            ph.off_odst = (uint16_t)o_odst;
            ph.n_cls = (uint16_t)cls.size();
            ph.off_cls = (uint16_t)o_cls;
            ph.off_dst = (uint16_t)o_dst;
            ph.off_meta = (uint16_t)o_meta;
            ph.gbase = (uint16_t)gbase;
            o.prog.assign(pbytes, 0);
            uint8_t *pp = o.prog.data();
            std::memcpy(pp, &ph, sizeof(ph));
            auto put = [&](size_t at, const void *src, size_t bytes) {
                if (bytes) std::memcpy(pp + at, src, bytes);
            };
            put(o_pos, pos.data(), 2 * pos.size());
            put(o_oseq, oseq.data(), 4 * oseq.size());
            put(o_odst, odst.data(), 4 * odst.size());
            put(o_cls, cls.data(), sizeof(TileCls) * cls.size());
            put(o_dst, dsts.data(), 4 * dsts.size());
            put(o_meta, meta.data(), 4 * meta.size());
            uint64_t hsh = 1469598103934665603ull;            // FNV-1a
            for (size_t q = 0; q < pbytes; q++) hsh = (hsh ^ pp[q]) * 1099511628211ull;
            o.hash = hsh;
            o.padded = 2 * (int64_t)n_rows * kTileThreads;
        } else {
            // ---- op streams: owned targets of <= kOpMax entries (and the side
            // pieces, a stream of their own) as per-thread sequences of pair-ops
            struct Stream {
                std::vector<uint16_t> row;           // [n_step] row offsets
                std::vector<uint32_t> ops;           // pair words, step-major rows
                std::vector<uint16_t> start;         // per sequence with ops: first emission | steps << 11
                std::vector<uint32_t> dst;           // destination per emission
                int32_t n_step = 0;
            };
            auto build_stream = [&](const std::vector<int32_t> &tl, Stream &S) -> bool {
                // longest first onto the least-loaded sequence (ties: lower index)
                std::vector<int32_t> order(tl);
                std::stable_sort(order.begin(), order.end(),
                                 [&](int32_t a, int32_t b) { return tg[a].len > tg[b].len; });
                std::vector<std::vector<int32_t>> seq(kTileThreads);
                std::vector<int32_t> load(kTileThreads, 0);
                for (int32_t k : order) {
                    int best = 0;
                    for (int r = 1; r < kTileThreads; r++)
                        if (load[r] < load[best]) best = r;
                    seq[best].push_back(k);
                    load[best] += (tg[k].len + 1) / 2;
                }
                // sequences by length, longest first: step s is a contiguous row
                std::vector<int32_t> perm(kTileThreads);
                std::iota(perm.begin(), perm.end(), 0);
                std::stable_sort(perm.begin(), perm.end(), [&](int32_t a, int32_t b) { return load[a] > load[b]; });
                S.n_step = load[perm[0]];
                if (S.n_step > kMaxSteps) return false;           // the byte bound's row reserve
                std::vector<std::vector<uint32_t>> words(kTileThreads);
                S.start.clear();
                S.dst.clear();
                for (int j = 0; j < kTileThreads; j++) {
                    const int32_t r = perm[j];
                    if (S.dst.size() > 65535) return false;
                    if (load[r] > 0) {                              // sequences with ops
                        if (S.dst.size() >= (1u << kSeqStartBits) || load[r] >= (1 << (16 - kSeqStartBits))) return false;
                        S.start.push_back((uint16_t)(S.dst.size() | ((size_t)load[r] << kSeqStartBits)));
                    }
                    for (int32_t k : seq[r]) {
                        const Tgt &t2 = tg[k];
                        for (int32_t p = 0; p < t2.len; p += 2) {
                            uint16_t ea = entry(t2, p);
                            const uint16_t eb = p + 1 < t2.len ? entry(t2, p + 1) : (uint16_t)kZeroSlotByte;
                            if (p + 2 >= t2.len) ea |= kEmitBit;               // emit after this pair
                            words[j].push_back((uint32_t)ea | ((uint32_t)eb << 16));
                        }
                        S.dst.push_back(t2.is_side ? (uint32_t)(-1 - t2.dst) : code_of(t2.dst));
                    }
                }
                S.row.clear();
                S.ops.clear();
                for (int32_t st = 0; st < S.n_step; st++) {
                    S.row.push_back((uint16_t)S.ops.size());
                    for (int j = 0; j < kTileThreads && (int32_t)words[j].size() > st; j++) S.ops.push_back(words[j][st]);
                    if (S.ops.size() > 65535) return false;
                }
                return true;
            };
            std::vector<int32_t> own_short, own_long, side_tl;     // own_long: owned, then side
            for (int32_t k = 0; k < (int32_t)tg.size(); k++) {
                if (tg[k].len > kOpMax) own_long.push_back(k);
                else if (tg[k].is_side) side_tl.push_back(k);
                else own_short.push_back(k);
            }
            Stream so, ss;
            if (!build_stream(own_short, so) || !build_stream(side_tl, ss)) return false;
            // ---- group classes: targets longer than kOpMax, one class per kind
            // (owned, then side) and lane-group size (largest first), targets in
            // list order
            cls.clear();
            dsts.clear();
            ents.clear();
            meta.clear();
            {
                auto gkey = [&](int32_t k) { return (tg[k].is_side ? 0 : 64) + cls_group(tg[k].len); };
                std::stable_sort(own_long.begin(), own_long.end(), [&](int32_t a, int32_t b) { return gkey(a) > gkey(b); });
                int64_t cum = 0;
                for (size_t k = 0; k < own_long.size();) {
                    const int gs = cls_group(tg[own_long[k]].len);
                    const int key = gkey(own_long[k]);
                    size_t e = k;
                    while (e < own_long.size() && gkey(own_long[e]) == key) e++;
                    if (e - k > 65535 || ents.size() > 65535 || dsts.size() > 65535 || meta.size() > 65535) return false;
                    TileCls tc;
                    std::memset(&tc, 0, sizeof(tc));
                    tc.n = (uint16_t)(e - k);
                    tc.ent = (uint16_t)ents.size();
                    tc.dst = (uint16_t)dsts.size();
                    int lg = 0;
                    while ((1 << lg) < gs) lg++;
                    tc.lg = (uint16_t)lg;
                    tc.meta = (uint16_t)meta.size();
                    tc.side = tg[own_long[k]].is_side ? 1 : 0;
                    for (size_t q = k; q < e; q++) {
                        const Tgt &t2 = tg[own_long[q]];
                        if (ents.size() > 65535 || t2.len > 65535) return false;
                        meta.push_back((uint32_t)ents.size() | ((uint32_t)t2.len << 16));
                        for (int32_t p = 0; p < t2.len; p++) ents.push_back(entry(t2, p));
                        dsts.push_back(t2.is_side ? -1 - t2.dst : (int32_t)code_of(t2.dst));   // side: entry index
                    }
                    const int64_t ng = kTileThreads / gs;
                    tc.rot = (uint16_t)((cum / gs) % ng);
                    cls.push_back(tc);
                    cum += (int64_t)tc.n * gs;
                    k = e;
                }
                if (ents.size() > 65536) return false;
            }
            // emit the head (per tile) and the program (shared by equal tiles)
            ProgHdr ph;
            std::memset(&ph, 0, sizeof(ph));
            size_t off = sizeof(ProgHdr);
            auto place = [&](size_t bytes) {
                const size_t at = off;
                off = pad16(off + bytes);
                return at;
            };
            const size_t o_orow = place(2 * so.row.size()), o_ops = place(4 * so.ops.size()),
                         o_ost = place(2 * so.start.size()), o_odst = place(4 * so.dst.size());
            const size_t o_srow = place(2 * ss.row.size()), o_sops = place(4 * ss.ops.size()),
                         o_sst = place(2 * ss.start.size()), o_sdst = place(2 * ss.dst.size());
            const size_t o_cls = place(sizeof(TileCls) * cls.size()), o_dst = place(4 * dsts.size()),
                         o_meta = place(4 * meta.size()), o_ent = place(2 * ents.size());
            const size_t pbytes = off;
            if (pbytes > 65535) return false;
            ph.n_oseq = (uint16_t)so.start.size();
            ph.off_orow = (uint16_t)o_orow;
            ph.off_ops = (uint16_t)o_ops;
            ph.off_ostart = (uint16_t)o_ost;
            ph.off_odst = (uint16_t)o_odst;
            ph.n_sseq = (uint16_t)ss.start.size();
            ph.off_srow = (uint16_t)o_srow;
            ph.off_sops = (uint16_t)o_sops;
            ph.off_sstart = (uint16_t)o_sst;
            ph.off_sdst = (uint16_t)o_sdst;
            ph.n_cls = (uint16_t)cls.size();
            ph.off_cls = (uint16_t)o_cls;
            ph.off_dst = (uint16_t)o_dst;
            ph.off_meta = (uint16_t)o_meta;
            ph.off_ent = (uint16_t)o_ent;
            o.prog.assign(pbytes, 0);
            uint8_t *pp = o.prog.data();
            std::memcpy(pp, &ph, sizeof(ph));
            auto put = [&](size_t at, const void *src, size_t bytes) {
                if (bytes) std::memcpy(pp + at, src, bytes);
            };
            put(o_orow, so.row.data(), 2 * so.row.size());
            put(o_ops, so.ops.data(), 4 * so.ops.size());
            put(o_ost, so.start.data(), 2 * so.start.size());
            put(o_odst, so.dst.data(), 4 * so.dst.size());
            put(o_srow, ss.row.data(), 2 * ss.row.size());
            put(o_sops, ss.ops.data(), 4 * ss.ops.size());
            put(o_sst, ss.start.data(), 2 * ss.start.size());
            for (size_t q = 0; q < ss.dst.size(); q++) {
                if (ss.dst[q] > 65535) return false;
                const uint16_t v = (uint16_t)ss.dst[q];
                std::memcpy(pp + o_sdst + 2 * q, &v, 2);
            }
            put(o_cls, cls.data(), sizeof(TileCls) * cls.size());
            put(o_dst, dsts.data(), 4 * dsts.size());
            put(o_meta, meta.data(), 4 * meta.size());
            put(o_ent, ents.data(), 2 * ents.size());
            uint64_t hsh = 1469598103934665603ull;            // FNV-1a
            for (size_t q = 0; q < pbytes; q++) hsh = (hsh ^ pp[q]) * 1099511628211ull;
            o.hash = hsh;
            o.padded = 2 * (int64_t)(so.ops.size() + ss.ops.size()) + (int64_t)ents.size();
        }

        TileHdr hdr;
        std::memset(&hdr, 0, sizeof(hdr));
        hdr.n_items = (uint16_t)ni;
        hdr.n_full = (uint16_t)n_full;
        hdr.n_sent = (uint16_t)n_sent;
        for (int q = 0; q < kTileBases; q++) hdr.base[q] = bases[q];
        if (tile_rows_ptr[tt + 1] > tile_rows_ptr[tt]) {
            const int32_t r0 = tile_rows[tile_rows_ptr[tt]], r1 = tile_rows[tile_rows_ptr[tt + 1] - 1];
            hdr.a_lo = row_ptr[r0];
            hdr.a_n = row_ptr[r1 + 1] - row_ptr[r0];
        }
        hdr.off_items = (uint32_t)sizeof(TileHdr);
        const size_t items_bytes = pad16((size_t)ni * (form == 1 ? 16 : kItemBlobBytes));   // form 1: terms
        hdr.off_side = (uint32_t)(hdr.off_items + items_bytes);
        const size_t bytes = pad16(hdr.off_side + sizeof(SideEnt) * sents.size());
        const size_t pbytes = o.prog.size();
        if (bytes + pbytes > (size_t)kStageMax) return false;
        hdr.head_bytes = (uint32_t)bytes;
        hdr.prog_bytes = (uint32_t)pbytes;
        o.blob.assign(bytes, 0);
        uint8_t *bp = o.blob.data();
        std::memcpy(bp, &hdr, sizeof(hdr));
        uint8_t *it = bp + hdr.off_items;
        int4 *term = reinterpret_cast<int4 *>(it);
        // form 0: beta, v0, model follow the terms in the head; form 1: they
        // live in tile-order arrays, kTileItems slots per tile (v0 per item)
        const size_t ib = (size_t)tt * kTileItems;     // form 1 arrays: preallocated, disjoint per tile
        double *bt = form == 1 ? out.item_beta.data() + ib : reinterpret_cast<double *>(it + 16 * (size_t)ni);
        double *v0b = bt + ni;                                     // form 0 only
        uint8_t *md = form == 1 ? out.item_model.data() + ib : reinterpret_cast<uint8_t *>(v0b + 3 * (size_t)ni);
        for (int32_t q = 0; q < ni; q++) {
            const int32_t i = item_dev[q0 + q];
            int4 tv;
            tv.x = rec[i].t[0]; tv.y = rec[i].t[1]; tv.z = rec[i].t[2]; tv.w = rec[i].t[3];
            std::memcpy(term + q, &tv, sizeof(tv));
            bt[q] = beta[i];
            for (int k = 0; k < 3; k++) {
                if (form == 1) out.item_v0[(ib + q) * 3 + k] = vprev[k * N + i];
                else v0b[k * ni + q] = vprev[k * N + i];
            }
            md[q] = (uint8_t)model[i];
        }
        if (!sents.empty()) std::memcpy(bp + hdr.off_side, sents.data(), sizeof(SideEnt) * sents.size());
        o.n_own = n_own;
        o.n_sent = n_sent;
        o.L = (int64_t)con.size() + (int64_t)side.size();
        return true;
    };
#pragma omp for schedule(dynamic, 64)
    for (int32_t tt = 0; tt < T; tt++) {
        TileOut &o = tout[tt];
        o.ok = emit_tile(tt, o);
        if (!o.ok) {
#pragma omp atomic write
            all_ok = false;
        }
    }
    }   // omp parallel
    if (!all_ok) return false;
    // concatenate in tile order; number side targets by first appearance
    std::vector<int32_t> sid_of((size_t)NT, -1);
    std::vector<int32_t> sent_tile_sid;     // side id of each entry, in emission order
    int64_t listed = 0;
    out.blob_off.assign((size_t)T + 1, 0);
    for (int32_t tt = 0; tt < T; tt++) {
        const TileOut &o = tout[tt];
        out.blob_off[tt + 1] = out.blob_off[tt] + (int64_t)o.blob.size();
        out.blob_max = std::max(out.blob_max, (int32_t)(o.blob.size() + o.prog.size()));
        out.n_owned += o.n_own;
        out.n_side_entries += o.n_sent;
        out.n_listed += o.L;
        out.n_padded += o.padded;
        out.st_waves0 += o.st_waves0;
        out.st_waves += o.st_waves;
        listed += o.listed;
    }
    // distinct programs, numbered by first appearance (tile order)
    std::vector<int64_t> prog_off((size_t)T, -1);
    {
        std::unordered_map<uint64_t, std::vector<int32_t>> by_hash;   // hash -> first tiles
        for (int32_t tt = 0; tt < T; tt++) {
            const TileOut &o = tout[tt];
            std::vector<int32_t> &same = by_hash[o.hash];
            for (int32_t u : same)
                if (tout[u].prog == o.prog) { prog_off[tt] = prog_off[u]; break; }
            if (prog_off[tt] >= 0) continue;
            prog_off[tt] = (int64_t)out.prog.size();
            out.prog.insert(out.prog.end(), o.prog.begin(), o.prog.end());
            same.push_back(tt);
            out.n_progs++;
        }
    }
    if (out.blob_off[T] / 16 > (int64_t)UINT32_MAX || (int64_t)out.prog.size() / 16 > (int64_t)UINT32_MAX)
        return false;
    out.tdesc.resize(4 * (size_t)T);
    for (int32_t tt = 0; tt < T; tt++) {
        out.tdesc[4 * tt] = (uint32_t)(out.blob_off[tt] / 16);
        out.tdesc[4 * tt + 1] = (uint32_t)tout[tt].blob.size();
        out.tdesc[4 * tt + 2] = (uint32_t)(prog_off[tt] / 16);
        out.tdesc[4 * tt + 3] = (uint32_t)tout[tt].prog.size();
    }
    out.blob.resize((size_t)out.blob_off[T]);
#pragma omp parallel for schedule(dynamic, 256)
    for (int32_t tt = 0; tt < T; tt++) {
        if (!tout[tt].blob.empty()) std::memcpy(out.blob.data() + out.blob_off[tt], tout[tt].blob.data(), tout[tt].blob.size());
        std::vector<uint8_t>().swap(tout[tt].blob);
        std::vector<uint8_t>().swap(tout[tt].prog);
    }
    for (int32_t tt = 0; tt < T; tt++) {
        uint8_t *bp = out.blob.data() + out.blob_off[tt];
        TileHdr hdr;
        std::memcpy(&hdr, bp, sizeof(hdr));
        SideEnt *se = reinterpret_cast<SideEnt *>(bp + hdr.off_side);
        for (int e = 0; e < hdr.n_sent; e++) {
            SideEnt v;
            std::memcpy(&v, se + e, sizeof(v));
            const int32_t g = v.sid;
            int32_t &sid = sid_of[g];
            if (sid < 0) {
                sid = (int32_t)out.sd_gid.size();
                out.sd_gid.push_back(g);
            }
            v.sid = sid;
            std::memcpy(se + e, &v, sizeof(v));
            sent_tile_sid.push_back(sid);
        }
    }
    // every live contribution is listed exactly once (owned or side)
    {
        int64_t live = 0;
        for (int64_t i = 0; i < N; i++)
            for (int p = 0; p < NPAIR + 4; p++) live += listed_c(i, p);
        if (listed != live) return false;
    }
    // partial slots.  Side targets with parts in far more tiles than there are
    // CTAs (rails) are "hot": each CTA pre-sums its tiles' parts in tile order
    // and stores one part (CTA order), so the final sum has `grid` terms; the
    // kernel runs min(grid, tiles) CTAs, the grid this layout is made for.
    grid = std::max(1, std::min(grid, T));
    out.grid = grid;
    // Every other side target gets one part per contributing tile, in tile order.
    out.n_side = (int32_t)out.sd_gid.size();
    std::vector<int64_t> cnt((size_t)out.n_side, 0);
    for (int32_t sid : sent_tile_sid) cnt[sid]++;
    std::vector<int32_t> order((size_t)out.n_side);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return cnt[a] > cnt[b]; });
    // pieces of one side target in one tile: a hot target keeps one running
    // sum per piece index in the CTA (kHotPieces of them)
    std::vector<int32_t> max_pieces((size_t)out.n_side, 0);
    {
        std::vector<int32_t> seen((size_t)out.n_side, -1), cnt_t((size_t)out.n_side, 0);
        for (int32_t tt = 0; tt < T; tt++) {
            const uint8_t *bp = out.blob.data() + out.blob_off[tt];
            TileHdr hdr;
            std::memcpy(&hdr, bp, sizeof(hdr));
            const SideEnt *se = reinterpret_cast<const SideEnt *>(bp + hdr.off_side);
            for (int e = 0; e < hdr.n_sent; e++) {
                SideEnt v;
                std::memcpy(&v, se + e, sizeof(v));
                if (seen[v.sid] != tt) { seen[v.sid] = tt; cnt_t[v.sid] = 0; }
                max_pieces[v.sid] = std::max(max_pieces[v.sid], ++cnt_t[v.sid]);
            }
        }
    }
    std::vector<int32_t> hot_of((size_t)out.n_side, -1);
    for (int32_t k = 0; k < out.n_side && out.n_hot < kMaxHot; k++)
        if (cnt[order[k]] > (int64_t)grid && max_pieces[order[k]] <= kHotPieces) {
            hot_of[order[k]] = out.n_hot++;
            out.hot_gid.push_back(out.sd_gid[order[k]]);
        }
    out.sd_part.assign((size_t)out.n_side + 1, 0);
    std::vector<int64_t> base((size_t)out.n_side, 0);
    int64_t cold = 0;
    for (int32_t s2 = 0; s2 < out.n_side; s2++)
        if (hot_of[s2] < 0) { base[s2] = cold; cold += cnt[s2]; }
    out.hot_base = cold;
    out.n_parts = cold + (int64_t)out.n_hot * grid;
    if (out.n_parts > INT32_MAX) return false;
    std::vector<int32_t> part_lo((size_t)out.n_side), part_hi((size_t)out.n_side);
    for (int32_t s2 = 0; s2 < out.n_side; s2++) {
        if (hot_of[s2] >= 0) {
            part_lo[s2] = (int32_t)(out.hot_base + (int64_t)hot_of[s2] * grid);
            part_hi[s2] = part_lo[s2] + grid;
        } else {
            part_lo[s2] = (int32_t)base[s2];
            part_hi[s2] = (int32_t)(base[s2] + cnt[s2]);
        }
    }
    // sd_part as (lo, hi) pairs flattened: sd_part[2*sid], sd_part[2*sid+1]
    out.sd_part.resize(2 * (size_t)out.n_side);
    for (int32_t s2 = 0; s2 < out.n_side; s2++) {
        out.sd_part[2 * s2] = part_lo[s2];
        out.sd_part[2 * s2 + 1] = part_hi[s2];
    }
    {
        std::vector<int64_t> fill(base);
        std::vector<int32_t> seen((size_t)out.n_side, -1), q_t((size_t)out.n_side, 0);
        for (int32_t tt = 0; tt < T; tt++) {
            uint8_t *bp = out.blob.data() + out.blob_off[tt];
            TileHdr hdr;
            std::memcpy(&hdr, bp, sizeof(hdr));
            SideEnt *se = reinterpret_cast<SideEnt *>(bp + hdr.off_side);
            for (int e = 0; e < hdr.n_sent; e++) {
                SideEnt v;
                std::memcpy(&v, se + e, sizeof(v));
                if (seen[v.sid] != tt) { seen[v.sid] = tt; q_t[v.sid] = 0; }
                const int32_t q = q_t[v.sid]++;           // piece index of this target in the tile
                v.slot = hot_of[v.sid] >= 0 ? -1 - (hot_of[v.sid] * kHotPieces + q) : (int32_t)fill[v.sid]++;
                std::memcpy(se + e, &v, sizeof(v));
            }
        }
    }
    // side-target order for the finishing phase: cold targets with more than
    // 8 parts, the other cold ones, then the hot ones (the heads' side
    // entries carry part slots, not these ids)
    {
        std::vector<int32_t> ord;
        for (int pass = 0; pass < 3; pass++)
            for (int32_t s2 = 0; s2 < out.n_side; s2++) {
                const bool hot = hot_of[s2] >= 0, big = part_hi[s2] - part_lo[s2] > 8;
                if ((pass == 0 && !hot && big) || (pass == 1 && !hot && !big) || (pass == 2 && hot))
                    ord.push_back(s2);
                if (pass == 0 && !hot && big) out.n_side_big++;
                if (pass < 2 && !hot && (pass == 0) == big) out.n_side_cold++;
            }
        std::vector<int32_t> gid((size_t)out.n_side), part(2 * (size_t)out.n_side);
        for (int32_t k = 0; k < out.n_side; k++) {
            gid[k] = out.sd_gid[ord[k]];
            part[2 * k] = part_lo[ord[k]];
            part[2 * k + 1] = part_hi[ord[k]];
        }
        out.sd_gid.swap(gid);
        out.sd_part.swap(part);
    }
    out.n_items = (int64_t)item_dev.size();
    return true;
}
}  // namespace

bool build_tile_host(int form, int64_t N, int32_t n_nodes, int32_t n, int64_t nnz, const int32_t *const TT[4],
                     const int32_t *raw_slot, const std::vector<int64_t> &iptr,
                     const std::vector<int32_t> &idev, const std::vector<int32_t> &rails,
                     const std::vector<int32_t> &row_ptr, const std::vector<int32_t> &col_idx,
                     const double *beta, const double *vprev, const int32_t *model, int32_t grid,
                     TileHost &out)
{
    if (build_tile_impl(form, false, N, n_nodes, n, nnz, TT, raw_slot, iptr, idev, rails, row_ptr, col_idx, beta,
                        vprev, model, grid, out))
        return true;
    if (form != 1) return false;
    out = TileHost();
    return build_tile_impl(form, true, N, n_nodes, n, nnz, TT, raw_slot, iptr, idev, rails, row_ptr, col_idx, beta,
                           vprev, model, grid, out);
}

}  // namespace ees
