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
#include <numeric>
#include <vector>

#include "ees_internal.h"

namespace ees {

namespace {
constexpr int32_t kUnset = -1;
constexpr int32_t kSide = -2;
// Upper bound of a tile's blob while it is being formed: items (49 B + 2 B
// per listed contribution), one padding entry per owned target nobody stamps
// (2 B), explicit ids of heavy-row slice targets (4 B), heavy x heavy targets
// (4 B id or an 8 B side entry) -- plus the fixed per-tile parts: header,
// thread words (512 B), list padding to whole chunks (< 256 B) and the
// padding of four sections.
constexpr int64_t kBlobFixed = 64 + 512 + 256 + 64;
constexpr int64_t kOwnMax = kSegMax;   // owned targets + side entries (s_seg capacity)
size_t pad16(size_t x) { return (x + 15) & ~(size_t)15; }
}  // namespace

bool build_tile_host(int form, int64_t N, int32_t n_nodes, int32_t n, int64_t nnz, const int32_t *const TT[4],
                     const int32_t *raw_slot, const std::vector<int64_t> &iptr,
                     const std::vector<int32_t> &idev, const std::vector<int32_t> &rails,
                     const std::vector<int32_t> &row_ptr, const std::vector<int32_t> &col_idx,
                     const double *beta, const double *vprev, const int32_t *model, int32_t grid,
                     TileHost &out)
{
    static_assert(kOwnMax > 64, "tile budget too small");
    const int64_t kStageMax = stage_max(form), kItemBlobBytes = item_blob_bytes(form);
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
    int64_t own = 0, bytes = kBlobFixed;
    int32_t last_row = -2;
    // distinct heavy x heavy targets a FET brings to tile t (each costs at most
    // one side entry + one run + one list start); marks them
    std::vector<int32_t> hh_seen((size_t)(nnz + n), -1);
    auto hh_new = [&](int64_t i, int32_t tile) {
        int32_t k = 0;
        for (int p = 0; p < NPAIR; p++) {
            const int32_t s2 = rec[i].s[p];
            if (s2 >= 0 && heavy[rec[i].t[pair_row(p)]] && heavy[rec[i].t[pair_col(p)]] && hh_seen[s2] != tile) {
                hh_seen[s2] = tile;
                k++;
            }
        }
        for (int a = 0; a < 4; a++) {
            const int32_t r = rec[i].t[a];
            if (r >= 0 && heavy[r] && hh_seen[nnz + r] != tile) {
                hh_seen[nnz + r] = tile;
                k++;
            }
        }
        return k;
    };
    auto live_count = [&](int64_t i) {
        int32_t k = 0;
        for (int p = 0; p < NPAIR + 4; p++) k += listed_c(i, p);
        return k;
    };
    // targets some FET stamps (an owned target nobody stamps costs one padding entry)
    std::vector<uint8_t> has_c((size_t)(nnz + n), 0);
    for (int64_t i = 0; i < N; i++)
        for (int p = 0; p < NPAIR + 4; p++)
            if (listed_c(i, p)) has_c[p < NPAIR ? rec[i].s[p] : nnz + rec[i].t[p - NPAIR]] = 1;
    auto empty_in_row = [&](int32_t r) {
        int64_t e = has_c[nnz + r] ? 0 : 1;
        for (int32_t k = row_ptr[r]; k < row_ptr[r + 1]; k++) e += !has_c[k];
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

    auto close_tile = [&]() {
        std::sort(cur.begin(), cur.end());
        item_dev.insert(item_dev.end(), cur.begin(), cur.end());
        out_item_ptr.push_back((int32_t)item_dev.size());
        tile_rows_ptr.push_back((int32_t)tile_rows.size());
        cur.clear();
        own = 0;
        bytes = kBlobFixed;
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
    // ---- tiles of consecutive light rows: <= kTileItems FETs, <= kOwnMax targets
    tile_of_row.assign((size_t)NN, -1);
    mark.assign((size_t)std::max<int64_t>(1, N), -1);
    home.assign((size_t)std::max<int64_t>(1, N), -1);
    cur.clear();
    tile_rows_ptr.assign(1, 0);
    tile_rows.clear();
    out_item_ptr.assign(1, 0);
    item_dev.clear();
    t = 0;
    own = 0;
    bytes = kBlobFixed;
    last_row = -2;
    std::fill(hh_seen.begin(), hh_seen.end(), -1);
    for (int32_t v = 0; v < n_nodes; v++) {
        if (heavy[v]) continue;
        // a tile's rows are consecutive, so its owned entries of A and b are
        // one CSR block and one row range (implicit ids in the blob)
        if ((int32_t)tile_rows.size() > tile_rows_ptr.back() && last_row != v - 1) close_tile();
        for (int pass = 0; pass < 2; pass++) {
            int32_t fresh = 0;
            const int64_t hs = hs_ptr[v + 1] - hs_ptr[v];
            int64_t add_own = (row_ptr[v + 1] - row_ptr[v]) + 1 + hs;
            int64_t add_bytes = 2 * empty_in_row(v) + 4 * hs;
            for (int64_t k = iptr[v]; k < iptr[v + 1]; k++) {
                const int32_t i = idev[k];
                if (mark[i] != t) {
                    fresh++;
                    add_bytes += kItemBlobBytes + 2 * live_count(i);
                }
                if (home[i] < 0) {
                    const int32_t hh = hh_new(i, t);
                    add_own += hh;
                    add_bytes += 12 * hh;
                }
            }
            const bool over = (int64_t)cur.size() + fresh > kTileItems || own + add_own > kOwnMax ||
                              bytes + add_bytes > kStageMax;
            if (over && pass == 0 && !cur.empty()) {
                close_tile();
                continue;
            }
            if (over) {                    // a single light row exceeds a tile
                promoted[v] = 1;
                done = false;
            }
            own += add_own;
            bytes += add_bytes;
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
            const int32_t add = hh_count(i);
            const int64_t add_bytes = kItemBlobBytes + 2 * live_count(i) + 12 * add;
            if (!cur.empty() && ((int64_t)cur.size() + 1 > kTileItems || own + add > kOwnMax ||
                                 bytes + add_bytes > kStageMax))
                close_tile();
            home[i] = t;
            own += add;
            bytes += add_bytes;
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

    // ---- per tile: blob = header | items | owned program | side entries.
    // Tiles are emitted in parallel into their own buffers (side entries carry
    // their global target for now), then concatenated in tile order, where
    // side ids are numbered by first appearance (the serial order).
    struct TileOut {
        std::vector<uint8_t> blob;
        int64_t listed = 0, L = 0, padded = 0;
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
    std::vector<std::pair<int32_t, uint16_t>> con, side, con_all;
    std::vector<int32_t> gids, xg;
    std::vector<uint16_t> ent;
    std::vector<uint32_t> tw;
    std::vector<int32_t> seg_of;
    std::vector<SideEnt> sents;
    std::vector<int64_t> extra_g;
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
        // contributions of this tile's items
        con.clear();
        side.clear();
        const int32_t q0 = out_item_ptr[tt];
        const int32_t ni = out_item_ptr[tt + 1] - q0;
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
        auto by_target = [](const std::pair<int32_t, uint16_t> &a, const std::pair<int32_t, uint16_t> &b) {
            return a.first < b.first;
        };
        std::stable_sort(con.begin(), con.end(), by_target);
        std::stable_sort(side.begin(), side.end(), by_target);
        // segments, in owned order: the tile rows' CSR block [a0, a0+na) and
        // b rows [b0, b0+nb) (implicit ids; an entry nobody stamps gets one
        // padding entry), then the other owned targets (heavy-row slices and
        // heavy x heavy targets; explicit ids, ascending), then side entries
        int32_t a0 = 0, na = 0, b0 = 0, nb = 0;
        if (tile_rows_ptr[tt + 1] > tile_rows_ptr[tt]) {
            const int32_t r0 = tile_rows[tile_rows_ptr[tt]], r1 = tile_rows[tile_rows_ptr[tt + 1] - 1];
            if (r1 - r0 + 1 != tile_rows_ptr[tt + 1] - tile_rows_ptr[tt]) return false;   // rows not consecutive
            a0 = row_ptr[r0];
            na = row_ptr[r1 + 1] - a0;
            b0 = r0;
            nb = r1 - r0 + 1;
        }
        ent.clear();
        xg.clear();
        size_t ci = 0;
        int32_t seg = 0;
        auto take = [&](int64_t g) {      // the segment of target g: its entries, or one pad
            const size_t c0 = ci;
            while (ci < con.size() && con[ci].first == g) ci++;
            if (ci == c0) ent.push_back((uint16_t)(8 * kZeroSlot | kEntEnd));
            for (size_t k = c0; k < ci; k++) ent.push_back((uint16_t)(8 * con[k].second | (k + 1 == ci ? kEntEnd : 0)));
            seg_of.resize(ent.size(), seg);
            seg++;
        };
        seg_of.clear();
        // con is sorted by target: extras below a0, the CSR block, extras up to
        // nnz, then b rows (the tile's range and heavy extras)
        extra_g.clear();
        {
            size_t k = 0;
            while (k < con.size()) {
                const int64_t g = con[k].first;
                const bool mainA = g >= a0 && g < (int64_t)a0 + na;
                const bool mainB = g >= nnz + b0 && g < nnz + b0 + nb;
                if (!mainA && !mainB) {
                    if (!std::binary_search(gids.begin(), gids.end(), (int32_t)g)) return false;
                    extra_g.push_back(g);
                }
                while (k < con.size() && con[k].first == g) k++;
            }
        }
        // walk con once per class (it is sorted; each class is a sorted subset)
        con_all.clear();
        con_all.swap(con);
        auto class_of = [&](int64_t g) {
            if (g >= a0 && g < (int64_t)a0 + na) return 0;
            if (g >= nnz + b0 && g < nnz + b0 + nb) return 1;
            return 2;
        };
        for (int cls = 0; cls < 3; cls++) {
            con.clear();
            for (auto &e2 : con_all)
                if (class_of(e2.first) == cls) con.push_back(e2);
            ci = 0;
            if (cls == 0)
                for (int64_t g = a0; g < (int64_t)a0 + na; g++) take(g);
            else if (cls == 1)
                for (int64_t g = nnz + b0; g < nnz + b0 + nb; g++) take(g);
            else
                for (int64_t g : extra_g) {
                    take(g);
                    xg.push_back((int32_t)g);
                }
            if (ci != con.size()) return false;
        }
        const int32_t n_own = seg;
        o.listed += (int64_t)con_all.size();
        con.swap(con_all);
        // side entries (slot filled below, once every side target's entry count is known)
        sents.clear();
        int32_t n_sent = 0;
        for (size_t k = 0; k < side.size(); k++) {
            const int32_t g = side[k].first;
            if (k == 0 || g != side[k - 1].first) {
                SideEnt se;
                se.sid = g;             // global target; numbered after the concatenation
                se.slot = -1;
                sents.push_back(se);
                n_sent++;
            }
            const bool last = k + 1 == side.size() || side[k + 1].first != g;
            ent.push_back((uint16_t)(8 * side[k].second | (last ? kEntEnd : 0)));
            seg_of.push_back(n_own + n_sent - 1);
        }
        o.listed += (int64_t)side.size();
        if (n_own + n_sent > kSegMax) return false;
        // equal chunks of K entries per thread, thread-interleaved
        const int64_t L = (int64_t)ent.size();
        const int32_t K = (int32_t)((L + kTileThreads - 1) / kTileThreads);
        tw.assign(kTileThreads, 0);
        auto chunk_has_end = [&](int64_t th2) {
            for (int64_t p2 = th2 * K; p2 < std::min<int64_t>(L, (th2 + 1) * K); p2++)
                if (ent[p2] & kEntEnd) return true;
            return false;
        };
        for (int32_t th2 = 0; th2 < kTileThreads; th2++) {
            const int64_t p0 = (int64_t)th2 * K;
            if (p0 >= L) continue;
            uint32_t chain = 0;
            if (p0 > 0 && seg_of[p0 - 1] == seg_of[p0] && chunk_has_end(th2)) {
                // the segment began in earlier chunks: count them (each carries a partial)
                int64_t k2 = th2 - 1;
                chain = 1;
                while (k2 > 0 && seg_of[k2 * K - 1] == seg_of[p0]) {
                    k2--;
                    chain++;
                }
            }
            tw[th2] = (uint32_t)seg_of[p0] | (chain << 16);
        }
        // emit the blob
        TileHdr hdr;
        std::memset(&hdr, 0, sizeof(hdr));
        hdr.n_items = (uint16_t)ni;
        hdr.n_own = (uint16_t)n_own;
        hdr.n_x = (uint16_t)xg.size();
        hdr.n_sent = (uint16_t)n_sent;
        hdr.K = (uint16_t)K;
        hdr.a0 = a0;
        hdr.na = na;
        hdr.b0 = b0;
        hdr.nb = nb;
        const size_t items_bytes = pad16((size_t)ni * kItemBlobBytes);
        hdr.off_x = (uint32_t)(pad16(sizeof(TileHdr)) + items_bytes);
        hdr.off_tw = (uint32_t)(hdr.off_x + 4 * xg.size());
        hdr.off_ent = (uint32_t)(hdr.off_tw + 4 * kTileThreads);
        hdr.off_side = (uint32_t)pad16(hdr.off_ent + 2 * (size_t)K * kTileThreads);
        const size_t bytes = pad16(hdr.off_side + sizeof(SideEnt) * sents.size());
        if (bytes > (size_t)kStageMax || K > 65535) return false;
        hdr.bytes = (uint32_t)bytes;
        o.blob.assign(bytes, 0);
        uint8_t *bp = o.blob.data();
        std::memcpy(bp, &hdr, sizeof(hdr));
        uint8_t *it = bp + pad16(sizeof(TileHdr));
        int4 *term = reinterpret_cast<int4 *>(it);
        // form 0: beta, v0, model follow the terms in the blob; form 1: they
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
        if (!xg.empty()) std::memcpy(bp + hdr.off_x, xg.data(), 4 * xg.size());
        std::memcpy(bp + hdr.off_tw, tw.data(), 4 * tw.size());
        uint16_t *ep = reinterpret_cast<uint16_t *>(bp + hdr.off_ent);
        for (int64_t k = 0; k < (int64_t)K * kTileThreads; k++) {
            const int64_t th2 = k / K, kk = k % K;     // logical position k -> thread th2, step kk
            ep[kk * kTileThreads + th2] = k < L ? ent[k] : (uint16_t)(8 * kZeroSlot);
        }
        if (!sents.empty()) std::memcpy(bp + hdr.off_side, sents.data(), sizeof(SideEnt) * sents.size());
        o.n_own = n_own;
        o.n_sent = n_sent;
        o.L = L;
        o.padded = (int64_t)K * kTileThreads;
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
        out.blob_max = std::max(out.blob_max, (int32_t)o.blob.size());
        out.n_owned += o.n_own;
        out.n_side_entries += o.n_sent;
        out.n_listed += o.L;
        out.n_padded += o.padded;
        listed += o.listed;
    }
    out.blob.resize((size_t)out.blob_off[T]);
#pragma omp parallel for schedule(dynamic, 256)
    for (int32_t tt = 0; tt < T; tt++) {
        if (!tout[tt].blob.empty()) std::memcpy(out.blob.data() + out.blob_off[tt], tout[tt].blob.data(), tout[tt].blob.size());
        std::vector<uint8_t>().swap(tout[tt].blob);
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
    std::vector<int32_t> hot_of((size_t)out.n_side, -1);
    for (int32_t k = 0; k < out.n_side && k < kMaxHot; k++)
        if (cnt[order[k]] > (int64_t)grid) {
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
        for (int32_t tt = 0; tt < T; tt++) {
            uint8_t *bp = out.blob.data() + out.blob_off[tt];
            TileHdr hdr;
            std::memcpy(&hdr, bp, sizeof(hdr));
            SideEnt *se = reinterpret_cast<SideEnt *>(bp + hdr.off_side);
            for (int e = 0; e < hdr.n_sent; e++) {
                SideEnt v;
                std::memcpy(&v, se + e, sizeof(v));
                v.slot = hot_of[v.sid] >= 0 ? -1 - hot_of[v.sid] : (int32_t)fill[v.sid]++;
                std::memcpy(se + e, &v, sizeof(v));
            }
        }
    }
    out.n_items = (int64_t)item_dev.size();
    return true;
}

}  // namespace ees
