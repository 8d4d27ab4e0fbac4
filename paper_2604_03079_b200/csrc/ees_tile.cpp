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
#include <numeric>
#include <vector>

#include "ees_internal.h"

namespace ees {

namespace {
constexpr int32_t kUnset = -1;
constexpr int32_t kSide = -2;
}  // namespace

bool build_tile_host(int64_t N, int32_t n_nodes, int32_t n, int64_t nnz, const int32_t *const TT[4],
                     const int32_t *raw_slot, const std::vector<int64_t> &iptr,
                     const std::vector<int32_t> &idev, const std::vector<int32_t> &rails, TileHost &out)
{
    out = TileHost();
    std::vector<uint8_t> heavy((size_t)std::max(1, n_nodes), 0);
    for (int32_t v = 0; v < n_nodes; v++) heavy[v] = (iptr[v + 1] - iptr[v]) > kHeavyDeg;
    for (int32_t r : rails) heavy[r] = 1;
    out.n_heavy = 0;
    for (int32_t v = 0; v < n_nodes; v++) out.n_heavy += heavy[v];

    // ---- tiles of consecutive light rows, <= kTileItems incident FETs each
    std::vector<int32_t> tile_of_row((size_t)std::max(1, n_nodes), -1);
    std::vector<int32_t> mark((size_t)std::max<int64_t>(1, N), -1);
    std::vector<int32_t> cur;
    out.item_ptr.push_back(0);
    int32_t t = 0;
    auto close_tile = [&]() {
        std::sort(cur.begin(), cur.end());
        out.item_dev.insert(out.item_dev.end(), cur.begin(), cur.end());
        out.item_ptr.push_back((int32_t)out.item_dev.size());
        cur.clear();
        t++;
    };
    for (int32_t v = 0; v < n_nodes; v++) {
        if (heavy[v]) continue;
        int32_t fresh = 0;
        for (int64_t k = iptr[v]; k < iptr[v + 1]; k++) fresh += mark[idev[k]] != t;
        if (!cur.empty() && (int64_t)cur.size() + fresh > kTileItems) close_tile();
        tile_of_row[v] = t;
        for (int64_t k = iptr[v]; k < iptr[v + 1]; k++)
            if (mark[idev[k]] != t) {
                mark[idev[k]] = t;
                cur.push_back(idev[k]);
            }
    }
    if (!cur.empty()) close_tile();
    // FETs with no light terminal (all heavy or ground): orphan tiles
    for (int64_t i = 0; i < N; i++)
        if (mark[i] < 0) {
            cur.push_back((int32_t)i);
            if ((int64_t)cur.size() == kTileItems) close_tile();
        }
    if (!cur.empty()) close_tile();
    const int32_t T = t;
    out.n_tiles = T;
    if ((int64_t)out.item_dev.size() > INT32_MAX) return false;

    // home tile of each FET = first tile holding it (side contributions come from there)
    std::vector<int32_t> home((size_t)std::max<int64_t>(1, N), -1);
    for (int32_t tt = 0; tt < T; tt++)
        for (int32_t q = out.item_ptr[tt]; q < out.item_ptr[tt + 1]; q++)
            if (home[out.item_dev[q]] < 0) home[out.item_dev[q]] = tt;

    // heavy x heavy targets: owned by the common home tile of all contributors, else side
    const int64_t NT = nnz + n;
    std::vector<int32_t> hh_owner((size_t)NT, kUnset);
    auto note_hh = [&](int64_t g, int32_t h) {
        int32_t &o = hh_owner[g];
        if (o == kUnset) o = h;
        else if (o != h) o = kSide;
    };
    for (int64_t i = 0; i < N; i++) {
        for (int p = 0; p < NPAIR; p++) {
            const int32_t k = raw_slot[p * N + i];
            if (k < 0) continue;
            if (heavy[TT[pair_row(p)][i]] && heavy[TT[pair_col(p)][i]]) note_hh(k, home[i]);
        }
        for (int a = 0; a < 4; a++) {
            const int32_t r = TT[a][i];
            if (r >= 0 && heavy[r]) note_hh(nnz + r, home[i]);
        }
    }

    // ---- per tile: owned lists and side entries
    std::vector<int32_t> sid_of((size_t)NT, -1);
    std::vector<std::pair<int32_t, uint16_t>> own, side;
    out.own_ptr.push_back(0);
    out.own_lst.push_back(0);
    out.side_ptr.push_back(0);
    out.side_lst.push_back(0);
    for (int32_t tt = 0; tt < T; tt++) {
        own.clear();
        side.clear();
        const int32_t q0 = out.item_ptr[tt];
        for (int32_t q = q0; q < out.item_ptr[tt + 1]; q++) {
            const int32_t i = out.item_dev[q];
            const int32_t loc = q - q0;
            for (int p = 0; p < NPAIR + 4; p++) {
                int64_t g;
                int32_t r, c;
                if (p < NPAIR) {
                    const int32_t k = raw_slot[p * N + i];
                    if (k < 0) continue;
                    g = k;
                    r = TT[pair_row(p)][i];
                    c = TT[pair_col(p)][i];
                } else {
                    r = TT[p - NPAIR][i];
                    if (r < 0) continue;
                    g = nnz + r;
                    c = r;
                }
                const uint16_t slot = (uint16_t)(p * kTileItems + loc);
                if (!heavy[r] || !heavy[c]) {
                    const int32_t owner = !heavy[r] ? tile_of_row[r] : tile_of_row[c];
                    if (owner == tt) own.emplace_back((int32_t)g, slot);
                } else if (home[i] == tt) {
                    if (hh_owner[g] == tt) own.emplace_back((int32_t)g, slot);
                    else side.emplace_back((int32_t)g, slot);
                }
            }
        }
        auto by_target = [](const std::pair<int32_t, uint16_t> &a, const std::pair<int32_t, uint16_t> &b) {
            return a.first < b.first;
        };
        std::stable_sort(own.begin(), own.end(), by_target);
        std::stable_sort(side.begin(), side.end(), by_target);
        for (size_t k = 0; k < own.size(); k++) {
            if (k == 0 || own[k].first != own[k - 1].first) {
                if (k) out.own_lst.push_back((int32_t)out.lst.size());
                out.own_gid.push_back(own[k].first);
            }
            out.lst.push_back(own[k].second);
        }
        if (!own.empty()) out.own_lst.push_back((int32_t)out.lst.size());
        out.own_ptr.push_back((int32_t)out.own_gid.size());
        for (size_t k = 0; k < side.size(); k++) {
            if (k == 0 || side[k].first != side[k - 1].first) {
                if (k) out.side_lst.push_back((int32_t)out.slst.size());
                int32_t &sid = sid_of[side[k].first];
                if (sid < 0) {
                    sid = (int32_t)out.sd_gid.size();
                    out.sd_gid.push_back(side[k].first);
                }
                out.side_sid.push_back(sid);
            }
            out.slst.push_back(side[k].second);
        }
        if (!side.empty()) out.side_lst.push_back((int32_t)out.slst.size());
        out.side_ptr.push_back((int32_t)out.side_sid.size());
        if (out.lst.size() > (size_t)INT32_MAX || out.slst.size() > (size_t)INT32_MAX) return false;
    }
    // every live contribution is listed exactly once (owned or side)
    {
        int64_t live = 0;
        for (int64_t k = 0; k < NPAIR * N; k++) live += raw_slot[k] >= 0;
        for (int64_t i = 0; i < N; i++)
            for (int a = 0; a < 4; a++) live += TT[a][i] >= 0;
        if ((int64_t)(out.lst.size() + out.slst.size()) != live) return false;
    }
    // partial slots: per side target, its entries in tile order
    out.n_side = (int32_t)out.sd_gid.size();
    out.sd_part.assign((size_t)out.n_side + 1, 0);
    for (int32_t sid : out.side_sid) out.sd_part[sid + 1]++;
    for (int32_t s = 0; s < out.n_side; s++) out.sd_part[s + 1] += out.sd_part[s];
    std::vector<int32_t> fill(out.sd_part.begin(), out.sd_part.end() - 1);
    out.side_slot.resize(out.side_sid.size());
    for (size_t e = 0; e < out.side_sid.size(); e++) out.side_slot[e] = fill[out.side_sid[e]]++;
    return true;
}

}  // namespace ees
