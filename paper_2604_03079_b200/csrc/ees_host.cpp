// ees_host.cpp -- host side of libees: the C ABI (include/ees.h), topology
// setup (pattern, stamp slots, colouring, schedules, contributor lists) and
// per-call dispatch of the sm_100a kernels in ees_kernels.cu.
//
// Setup follows PAPER.md P:36 ("constructs the FET conflict graph during
// setup, partitions instances into color groups") and SPEC.md's mna-core
// reserve/finalize and coloring module.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <type_traits>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "ees_internal.h"

using namespace ees;

namespace {

double now_s()
{
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Layout {
    int64_t N = 0;
    int4 *term = nullptr;
    double *beta = nullptr;
    double *v0 = nullptr;
    uint8_t *model = nullptr;
    int32_t *slot = nullptr;
    int64_t cls_a = 0, cls_b = 0;         // ATOMIC order only (DevK)
    DevK k() const { return DevK{N, term, beta, v0, model, slot, cls_a, cls_b}; }
};

}  // namespace

struct ees_ctx {
    int32_t n_nodes = 0, n_extra = 0, n = 0;
    int64_t n_dev = 0, nnz = 0;
    std::vector<int32_t> row_ptr, col_idx;
    std::vector<int32_t> color;
    std::vector<int32_t> atomic_pos;      // netlist index -> position in the ATOMIC order
    int32_t n_colors = 0;
    std::vector<int64_t> color_ptr;
    std::vector<ees_model> models;
    std::vector<int32_t> rails;
    double gmin = 0.0;
    int32_t rule = 0;
    int32_t n_rail_a = 0, n_rail_entries = 0;
    int32_t rail_target[kMaxRailEntries] = {};
    Layout L_atomic, L_color, L_gather;
    // EES_CONFLICT_HYBRID: colour-major 16-slot layout, side sum, race-probe codes
    bool hybrid = false;
    Layout L_colorh, L_probe;
    SideK sk{};
    int32_t *d_perm = nullptr;            // colour-major position -> netlist index (COLOR_BUF)
    GatherK gk{};
    TileK tk{};
    std::vector<int64_t> color_blk_off;   // [C+1] block offsets of colours into partials
    double *partials = nullptr;
    int color_coop = 0;                   // 1: persistent cooperative COLOR kernel
    int tile_grid = 1;                    // persistent TILE CTAs
    int coop_grid = 0;
    int64_t *d_color_ptr = nullptr;
    double *coop_partials = nullptr;
    int atomic_grid = 1;
    int atomic_agg = 1;                   // ATOMIC: warp run aggregation (timed at setup)
    int32_t variant = EES_ATOMIC;
    int32_t launches = 0;
    int32_t work = 1;                     // S:229 work multiplier
    bool host_only = false;
    int32_t setup_flags = 0;              // ees_desc.flags
    // phase timing
    bool timing = false;
    struct Mark { int phase; cudaEvent_t a, b; };
    std::vector<Mark> marks;
    std::vector<cudaEvent_t> ev_free;
    int32_t timed_calls = 0;
    ees_stats_t st{};
    double *hx = nullptr, *hA = nullptr, *hb = nullptr;   // ees_eval_stamp_host staging
    std::vector<void *> allocs;
};

namespace {

template <typename T>
ees_status dalloc(ees_ctx *c, T **p, size_t count)
{
    *p = nullptr;
    if (count == 0) count = 1;
    void *q = nullptr;
    const cudaError_t e = cudaMalloc(&q, count * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return e == cudaErrorMemoryAllocation ? EES_ENOMEM : EES_ECUDA;
    }
    c->allocs.push_back(q);
    *p = static_cast<T *>(q);
    return EES_OK;
}

template <typename T>
ees_status upload(ees_ctx *c, T **p, const T *src, size_t count)
{
    ees_status s = dalloc(c, p, count);
    if (s != EES_OK) return s;
    if (count && cudaMemcpy(*p, src, count * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
        return EES_ECUDA;
    return EES_OK;
}

#define TRY(expr)                         \
    do {                                  \
        ees_status _s = (expr);           \
        if (_s != EES_OK) return _s;      \
    } while (0)

ees_status validate(const ees_desc *d)
{
    if (!d) return EES_EINVAL;
    if (d->n_nodes < 0 || d->n_extra < 0 || d->n_dev < 0) return EES_EINVAL;
    if (d->n_dev > INT32_MAX - 1) return EES_EINVAL;   // FET indices are int32 in every device list
    if ((int64_t)d->n_nodes + d->n_extra > INT32_MAX - 1) return EES_EINVAL;
    if (d->n_models < 1 || d->n_models > EES_MAX_MODELS || !d->models) return EES_EINVAL;
    if (d->n_rails < 0 || d->n_rails > EES_MAX_RAILS || (d->n_rails && !d->rails)) return EES_EINVAL;
    if (d->n_extra_entries < 0 || (d->n_extra_entries && (!d->extra_row || !d->extra_col)))
        return EES_EINVAL;
    if (!(d->gmin >= 0.0) || !std::isfinite(d->gmin)) return EES_EINVAL;
    if (d->variant < EES_AUTO || d->variant > EES_COLOR_BUF) return EES_EINVAL;
    if (d->conflict_rule != EES_CONFLICT_EXCLUDE_RAILS && d->conflict_rule != EES_CONFLICT_PAPER &&
        d->conflict_rule != EES_CONFLICT_HYBRID)
        return EES_EINVAL;
    if (d->heavy_degree < 0) return EES_EINVAL;
    {
        const int32_t known = EES_SETUP_HOST_ONLY | EES_SETUP_TILE_FORM0 | EES_SETUP_TILE_FORM1 |
                              EES_SETUP_GATHER_FORM0 | EES_SETUP_GATHER_FORM1 | EES_SETUP_COLOR_LAUNCH |
                              EES_SETUP_COLOR_COOP;
        auto both = [&](int32_t a, int32_t b) { return (d->flags & a) && (d->flags & b); };
        if ((d->flags & ~known) || both(EES_SETUP_TILE_FORM0, EES_SETUP_TILE_FORM1) ||
            both(EES_SETUP_GATHER_FORM0, EES_SETUP_GATHER_FORM1) || both(EES_SETUP_COLOR_LAUNCH, EES_SETUP_COLOR_COOP))
            return EES_EINVAL;
    }
    for (int k = 0; k < d->n_models; k++) {
        const ees_model &m = d->models[k];
        if ((m.polarity != 1 && m.polarity != -1) || m.reserved != 0) return EES_EINVAL;
        if (!(m.kp > 0.0) || !std::isfinite(m.kp) || !std::isfinite(m.vt0) || !std::isfinite(m.lambda))
            return EES_EINVAL;
        if (!(m.cgs >= 0.0) || !(m.cgd >= 0.0) || !(m.cdb >= 0.0)) return EES_EINVAL;
        if (!std::isfinite(m.cgs) || !std::isfinite(m.cgd) || !std::isfinite(m.cdb)) return EES_EINVAL;
    }
    if (d->n_dev) {
        if (!d->d || !d->g || !d->s || !d->b || !d->w || !d->l || !d->model || !d->vprev)
            return EES_EINVAL;
        for (int64_t i = 0; i < d->n_dev; i++) {
            const int32_t T[4] = {d->d[i], d->g[i], d->s[i], d->b[i]};
            for (int a = 0; a < 4; a++)
                if (T[a] < -1 || T[a] >= d->n_nodes) return EES_EINVAL;
            if (d->model[i] < 0 || d->model[i] >= d->n_models) return EES_EINVAL;
            if (!(d->w[i] > 0.0) || !(d->l[i] > 0.0) || !std::isfinite(d->w[i]) || !std::isfinite(d->l[i]))
                return EES_EINVAL;
        }
    }
    const int32_t n = d->n_nodes + d->n_extra;
    for (int k = 0; k < d->n_rails; k++) {
        if (d->rails[k] < 0 || d->rails[k] >= d->n_nodes) return EES_EINVAL;
        for (int j = 0; j < k; j++)
            if (d->rails[j] == d->rails[k]) return EES_EINVAL;
    }
    for (int64_t e = 0; e < d->n_extra_entries; e++)
        if (d->extra_row[e] < 0 || d->extra_row[e] >= n || d->extra_col[e] < 0 || d->extra_col[e] >= n)
            return EES_EINVAL;
    return EES_OK;
}

// node -> devices incidence over all non-ground nodes (a device appears once
// per distinct node), devices ascending.
void build_incidence(const ees_desc *d, std::vector<int64_t> &ptr, std::vector<int32_t> &dev)
{
    const int64_t N = d->n_dev;
    ptr.assign((size_t)d->n_nodes + 1, 0);
    for (int64_t i = 0; i < N; i++) {
        const int32_t T[4] = {d->d[i], d->g[i], d->s[i], d->b[i]};
        for (int a = 0; a < 4; a++) {
            bool dup = T[a] < 0;
            for (int c = 0; c < a; c++) dup |= T[c] == T[a];
            if (!dup) ptr[T[a] + 1]++;
        }
    }
    for (int32_t v = 0; v < d->n_nodes; v++) ptr[v + 1] += ptr[v];
    dev.resize((size_t)ptr[d->n_nodes]);
    std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
    for (int64_t i = 0; i < N; i++) {
        const int32_t T[4] = {d->d[i], d->g[i], d->s[i], d->b[i]};
        for (int a = 0; a < 4; a++) {
            bool dup = T[a] < 0;
            for (int c = 0; c < a; c++) dup |= T[c] == T[a];
            if (!dup) dev[fill[T[a]]++] = (int32_t)i;
        }
    }
}

// CSR pattern: row r holds every non-ground terminal of every device on r
// (all ordered pairs) plus the extra entries of row r; sorted unique.
ees_status build_pattern(const ees_desc *d, ees_ctx *c, const std::vector<int64_t> &iptr,
                         const std::vector<int32_t> &idev)
{
    const int32_t n = c->n;
    std::vector<int64_t> eptr((size_t)n + 1, 0);
    for (int64_t e = 0; e < d->n_extra_entries; e++) eptr[d->extra_row[e] + 1]++;
    for (int32_t r = 0; r < n; r++) eptr[r + 1] += eptr[r];
    std::vector<int32_t> ecol((size_t)eptr[n]);
    {
        std::vector<int64_t> fill(eptr.begin(), eptr.end() - 1);
        for (int64_t e = 0; e < d->n_extra_entries; e++) ecol[fill[d->extra_row[e]]++] = d->extra_col[e];
    }
    std::vector<int64_t> cnt((size_t)n + 1, 0);
    const int32_t *TT[4] = {d->d, d->g, d->s, d->b};
    auto collect = [&](int32_t r, std::vector<int32_t> &tmp) {
        tmp.clear();
        if (r < d->n_nodes)
            for (int64_t k = iptr[r]; k < iptr[r + 1]; k++) {
                const int32_t i = idev[k];
                for (int a = 0; a < 4; a++)
                    if (TT[a][i] >= 0) tmp.push_back(TT[a][i]);
            }
        for (int64_t k = eptr[r]; k < eptr[r + 1]; k++) tmp.push_back(ecol[k]);
        std::sort(tmp.begin(), tmp.end());
        tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
    };
#pragma omp parallel
    {
        std::vector<int32_t> tmp;
#pragma omp for schedule(dynamic, 4096)
        for (int32_t r = 0; r < n; r++) {
            collect(r, tmp);
            cnt[r + 1] = (int64_t)tmp.size();
        }
    }
    for (int32_t r = 0; r < n; r++) cnt[r + 1] += cnt[r];
    if (cnt[n] > INT32_MAX) return EES_EINVAL;   // nnz must fit int32 (SURVEY §8(a) layout)
    c->nnz = cnt[n];
    c->row_ptr.resize((size_t)n + 1);
    for (int32_t r = 0; r <= n; r++) c->row_ptr[r] = (int32_t)cnt[r];
    c->col_idx.resize((size_t)c->nnz);
#pragma omp parallel
    {
        std::vector<int32_t> tmp;
#pragma omp for schedule(dynamic, 4096)
        for (int32_t r = 0; r < n; r++) {
            collect(r, tmp);
            std::copy(tmp.begin(), tmp.end(), c->col_idx.begin() + cnt[r]);
        }
    }
    return EES_OK;
}

int32_t find_slot(const ees_ctx *c, int32_t r, int32_t col)
{
    const int32_t *b = c->col_idx.data() + c->row_ptr[r];
    const int32_t *e = c->col_idx.data() + c->row_ptr[r + 1];
    const int32_t *p = std::lower_bound(b, e, col);
    return (p != e && *p == col) ? (int32_t)(p - c->col_idx.data()) : -1;
}

// First-fit greedy colouring in netlist order over the
// conflict nodes (non-ground; rails removed under EES_CONFLICT_EXCLUDE_RAILS).
// Each node keeps the colours of its already-coloured devices: a node with at
// most kListMax incident devices in a list of its own (a slice of one pool
// sized by the incidence counts, so memory is O(sum of degrees) whatever the
// colour count), a busier node in a bitset with a monotone "first non-full
// word" cursor, so a device on a clique of size f costs O(1) amortised
// instead of O(f).
constexpr int32_t kListMax = 64;

int32_t greedy_color(const ees_desc *d, const std::vector<uint8_t> &excluded,
                     std::vector<int32_t> &color, int32_t &max_node_deg)
{
    const int64_t N = d->n_dev;
    const int32_t NN = std::max(1, d->n_nodes);
    color.assign((size_t)N, 0);
    // distinct incident devices per node (capacity of its list)
    std::vector<int32_t> cap((size_t)NN, 0);
    for (int64_t i = 0; i < N; i++) {
        const int32_t T[4] = {d->d[i], d->g[i], d->s[i], d->b[i]};
        for (int a = 0; a < 4; a++) {
            bool dup = T[a] < 0 || excluded[T[a]];
            for (int c = 0; c < a; c++) dup |= T[c] == T[a];
            if (!dup) cap[T[a]]++;
        }
    }
    std::vector<int64_t> lptr((size_t)NN + 1, 0);
    std::vector<int32_t> big((size_t)NN, -1);          // index into bits, or -1 (list)
    for (int32_t v = 0; v < d->n_nodes; v++) lptr[v + 1] = lptr[v] + (cap[v] <= kListMax ? cap[v] : 0);
    std::vector<int32_t> pool((size_t)std::max<int64_t>(1, lptr[d->n_nodes]));
    std::vector<int32_t> cnt((size_t)NN, 0);
    std::vector<std::vector<uint64_t>> bits;
    std::vector<int32_t> first_nonfull;
    for (int32_t v = 0; v < d->n_nodes; v++)
        if (cap[v] > kListMax) {
            big[v] = (int32_t)bits.size();
            bits.emplace_back();
            first_nonfull.push_back(0);
        }
    int32_t C = 0;
    for (int64_t i = 0; i < N; i++) {
        int32_t U[4];
        int nu = 0;
        const int32_t T[4] = {d->d[i], d->g[i], d->s[i], d->b[i]};
        for (int a = 0; a < 4; a++) {
            if (T[a] < 0 || excluded[T[a]]) continue;
            bool dup = false;
            for (int k = 0; k < nu; k++) dup |= U[k] == T[a];
            if (!dup) U[nu++] = T[a];
        }
        int64_t w = 0;
        for (int k = 0; k < nu; k++)
            if (big[U[k]] >= 0) w = std::max<int64_t>(w, first_nonfull[big[U[k]]]);
        int32_t col;
        for (;; w++) {
            uint64_t m = 0;
            for (int k = 0; k < nu; k++) {
                const int32_t v = U[k];
                if (big[v] >= 0) {
                    const std::vector<uint64_t> &bv = bits[big[v]];
                    if (w < (int64_t)bv.size()) m |= bv[w];
                } else {
                    const int32_t *l = pool.data() + lptr[v];
                    for (int32_t q = 0; q < cnt[v]; q++)
                        if ((l[q] >> 6) == w) m |= 1ull << (l[q] & 63);
                }
            }
            if (~m) {
                col = (int32_t)(64 * w + __builtin_ctzll(~m));
                break;
            }
        }
        color[i] = col;
        if (col + 1 > C) C = col + 1;
        for (int k = 0; k < nu; k++) {
            const int32_t v = U[k];
            if (big[v] < 0) {
                pool[lptr[v] + cnt[v]++] = col;
                continue;
            }
            cnt[v]++;
            std::vector<uint64_t> &bv = bits[big[v]];
            if ((int64_t)bv.size() <= (col >> 6)) bv.resize((col >> 6) + 1, 0);
            bv[col >> 6] |= 1ull << (col & 63);
            int32_t &f = first_nonfull[big[v]];
            while (f < (int32_t)bv.size() && bv[f] == ~0ull) f++;
        }
    }
    max_node_deg = 0;
    for (int32_t v = 0; v < d->n_nodes; v++) max_node_deg = std::max(max_node_deg, cnt[v]);
    return N ? C : 0;
}

CallK make_call(const ees_ctx *c, const double *x, double h, double *A, double *b)
{
    CallK k;
    std::memset(&k, 0, sizeof(k));
    for (size_t m = 0; m < c->models.size(); m++) {
        const ees_model &md = c->models[m];
        CardK &cd = k.cards[m];
        cd.p = (double)md.polarity;
        cd.vt = cd.p * md.vt0;
        cd.lam = md.lambda;
        cd.gcgs = md.cgs / h;      // S:196 Geq = C/dt (IEEE division; h = +inf -> 0)
        cd.gcgd = md.cgd / h;
        cd.gcdb = md.cdb / h;
    }
    k.x = x;
    k.A = A;
    k.b = b;
    k.gmin = c->gmin;
    k.work = c->work;
    k.n_models = (int32_t)c->models.size();
    k.n_rail_nodes = (int32_t)c->rails.size();
    for (size_t r = 0; r < c->rails.size(); r++) k.rail_node[r] = c->rails[r];
    k.n_rail_a = c->n_rail_a;
    k.n_rail_entries = c->n_rail_entries;
    std::memcpy(k.rail_target, c->rail_target, sizeof(k.rail_target));
    return k;
}

cudaEvent_t take_event(ees_ctx *c)
{
    if (!c->ev_free.empty()) {
        cudaEvent_t e = c->ev_free.back();
        c->ev_free.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Records an event pair around one phase when timing is enabled.
struct PhaseMark {
    ees_ctx *c;
    cudaStream_t st;
    int phase;
    cudaEvent_t a = nullptr;
    PhaseMark(ees_ctx *c_, cudaStream_t s_, int p_, bool on) : c(c_), st(s_), phase(p_)
    {
        if (on) {
            a = take_event(c);
            cudaEventRecord(a, st);
        }
    }
    ~PhaseMark()
    {
        if (a) {
            cudaEvent_t b = take_event(c);
            cudaEventRecord(b, st);
            c->marks.push_back({phase, a, b});
        }
    }
};

ees_status enqueue(ees_ctx *c, int32_t variant, const double *x, double h, double *A, double *b,
                   cudaStream_t st, int32_t *launches, bool timed = false)
{
    const CallK call = make_call(c, x, h, A, b);
    int nl = 0;
    cudaError_t e = cudaSuccess;
    if (variant == EES_ATOMIC) {
        PhaseMark m(c, st, 0, timed);
        e = launch_atomic(c->L_atomic.k(), call, c->atomic_grid, c->atomic_agg != 0, st);
        nl = c->n_dev ? 1 : 0;
    } else if (variant == EES_COLOR && c->hybrid) {
        const DevK dv = c->L_colorh.k();
        {
            PhaseMark m(c, st, 0, timed);
            for (int32_t col = 0; col < c->n_colors && e == cudaSuccess; col++) {
                e = launch_color_h(dv, call, c->color_ptr[col], c->color_ptr[col + 1] - c->color_ptr[col],
                                   c->sk.buf, st);
                nl++;
            }
        }
        if (e == cudaSuccess && c->sk.n_side) {
            PhaseMark m(c, st, 1, timed);
            int k = 0;
            e = launch_side_sum(c->sk, call, st, &k);
            nl += k;
        }
    } else if (variant == EES_COLOR && c->color_coop) {
        PhaseMark m(c, st, 0, timed);
        e = launch_color_coop(c->L_color.k(), call, c->d_color_ptr, c->n_colors, c->coop_partials,
                              c->coop_grid, st);
        nl = c->n_dev ? 1 : 0;
    } else if (variant == EES_COLOR) {
        const DevK dv = c->L_color.k();
        {
            PhaseMark m(c, st, 0, timed);
            for (int32_t col = 0; col < c->n_colors && e == cudaSuccess; col++) {
                e = launch_color(dv, call, c->color_ptr[col], c->color_ptr[col + 1] - c->color_ptr[col],
                                 c->partials + c->color_blk_off[col] * c->n_rail_entries, st);
                nl++;
            }
        }
        if (e == cudaSuccess && c->n_rail_entries && c->n_dev) {
            PhaseMark m(c, st, 1, timed);
            e = launch_rail_finalize(call, c->partials, c->color_blk_off[c->n_colors], st);
            nl++;
        }
    } else if (variant == EES_COLOR_BUF) {
        {
            PhaseMark m(c, st, 0, timed);
            e = launch_eval_compact(c->L_gather.k(), c->gk, call, st);
            nl += c->n_dev ? 1 : 0;
        }
        {
            PhaseMark m(c, st, 1, timed);
            const DevK dv = c->L_colorh.k();
            for (int32_t col = 0; col < c->n_colors && e == cudaSuccess; col++) {
                e = launch_color_stamp(dv, c->gk, call, c->d_perm, c->color_ptr[col],
                                       c->color_ptr[col + 1] - c->color_ptr[col], c->sk.buf, st);
                nl++;
            }
            if (e == cudaSuccess && c->sk.n_side) {
                int k = 0;
                e = launch_side_sum(c->sk, call, st, &k);
                nl += k;
            }
        }
    } else if (variant == EES_TILE) {
        PhaseMark m(c, st, 0, timed);
        e = launch_tile(c->tk, call, c->tile_grid, st, &nl);
    } else if (variant == EES_GATHER) {
        if (timed) {
            for (int ph = 0; ph < 3 && e == cudaSuccess; ph++) {
                PhaseMark m(c, st, ph, true);
                int k = 0;
                e = launch_gather_phase(c->L_gather.k(), c->gk, call, st, ph, &k);
                nl += k;
            }
        } else {
            e = launch_gather(c->L_gather.k(), c->gk, call, st, &nl);
        }
    } else {
        return EES_ESTATE;
    }
    if (launches) *launches = nl;
    return e == cudaSuccess ? EES_OK : EES_ECUDA;
}

ees_status build_layouts(const ees_desc *d, ees_ctx *c, const std::vector<int32_t> &raw_slot,
                         const std::vector<int32_t> &rail_ord)
{
    const int64_t N = c->n_dev;
    // netlist-order SoA shared by ATOMIC and GATHER
    std::vector<double> beta((size_t)N), v0((size_t)(3 * N));
    std::vector<uint8_t> model((size_t)N);
    std::vector<int4> term_plain((size_t)N), term_rail((size_t)N);
    std::vector<int32_t> slot_rail((size_t)(NPAIR * N));
    auto railcode = [&](int32_t t) { return (t >= 0 && rail_ord[t] >= 0) ? -2 - rail_ord[t] : t; };
    // map raw A slot -> rail entry
    auto slotcode = [&](int32_t k) {
        if (k < 0) return k;
        for (int e = 0; e < c->n_rail_a; e++)
            if (c->rail_target[e] == k) return -2 - e;
        return k;
    };
    std::vector<uint8_t> is_rail_slot;
    if (c->n_rail_a) {
        is_rail_slot.assign((size_t)c->nnz, 0);
        for (int e = 0; e < c->n_rail_a; e++) is_rail_slot[c->rail_target[e]] = 1;
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; i++) {
        const ees_model &m = c->models[d->model[i]];
        beta[i] = (m.kp * d->w[i]) / d->l[i];
        for (int t = 0; t < 3; t++) v0[t * N + i] = d->vprev[t * N + i];
        model[i] = (uint8_t)d->model[i];
        term_plain[i] = make_int4(d->d[i], d->g[i], d->s[i], d->b[i]);
        term_rail[i] = make_int4(railcode(d->d[i]), railcode(d->g[i]), railcode(d->s[i]), railcode(d->b[i]));
        for (int p = 0; p < NPAIR; p++) {
            const int32_t k = raw_slot[p * N + i];
            slot_rail[p * N + i] = (k >= 0 && c->n_rail_a && is_rail_slot[k]) ? slotcode(k) : k;
        }
    }
    // ATOMIC order: devices grouped by which slot codes are dead by structure
    // -- A: source and bulk grounded (only DD DG GD GG can be live), B: bulk
    // pairs dead (bulk grounded, or tied to the source and merged), C: the rest
    // -- so k_atomic skips the dead codes' loads (and their DRAM sectors) from
    // the device index alone (DevK::cls_a / cls_b), without a prior load.
    {
        std::vector<int32_t> aperm((size_t)N);
        int64_t na = 0, nb = 0;
        auto cls = [&](int64_t i) {
            const int4 T = term_rail[i];
            if (T.z == -1 && T.w == -1) return 0;
            return (T.w == -1 || T.z == T.w) ? 1 : 2;
        };
        for (int64_t i = 0; i < N; i++) {
            const int k = cls(i);
            na += k == 0;
            nb += k == 1;
        }
        int64_t fill[3] = {0, na, na + nb};
        for (int64_t i = 0; i < N; i++) aperm[fill[cls(i)]++] = (int32_t)i;
        c->atomic_pos.assign((size_t)N, 0);
        std::vector<int4> term_a((size_t)N);
        std::vector<double> beta_a((size_t)N), v0_a((size_t)(3 * N));
        std::vector<uint8_t> model_a((size_t)N);
        std::vector<int32_t> slot_a((size_t)(NPAIR * N));
#pragma omp parallel for schedule(static)
        for (int64_t q = 0; q < N; q++) {
            const int64_t i = aperm[q];
            c->atomic_pos[i] = (int32_t)q;
            term_a[q] = term_rail[i];
            beta_a[q] = beta[i];
            for (int t = 0; t < 3; t++) v0_a[t * N + q] = v0[t * N + i];
            model_a[q] = model[i];
            for (int p = 0; p < NPAIR; p++) slot_a[p * N + q] = slot_rail[p * N + i];
        }
        Layout &La = c->L_atomic;
        La.N = N;
        La.cls_a = na;
        La.cls_b = na + nb;
        TRY(upload(c, &La.term, term_a.data(), N));
        TRY(upload(c, &La.beta, beta_a.data(), N));
        TRY(upload(c, &La.v0, v0_a.data(), 3 * N));
        TRY(upload(c, &La.model, model_a.data(), N));
        TRY(upload(c, &La.slot, slot_a.data(), NPAIR * N));
    }
    Layout &Lg = c->L_gather;      // netlist order (GATHER's device offsets)
    Lg.N = N;
    TRY(upload(c, &Lg.term, term_plain.data(), N));
    TRY(upload(c, &Lg.beta, beta.data(), N));
    TRY(upload(c, &Lg.v0, v0.data(), 3 * N));
    TRY(upload(c, &Lg.model, model.data(), N));
    // colour-major copy
    {
        std::vector<int32_t> perm((size_t)N);
        std::vector<int64_t> fill(c->color_ptr.begin(), c->color_ptr.end() - 1);
        for (int64_t i = 0; i < N; i++) perm[fill[c->color[i]]++] = (int32_t)i;
        std::vector<double> beta_c((size_t)N), v0_c((size_t)(3 * N));
        std::vector<uint8_t> model_c((size_t)N);
        std::vector<int4> term_c((size_t)N);
        std::vector<int32_t> slot_c((size_t)(NPAIR * N));
#pragma omp parallel for schedule(static)
        for (int64_t q = 0; q < N; q++) {
            const int64_t i = perm[q];
            beta_c[q] = beta[i];
            for (int t = 0; t < 3; t++) v0_c[t * N + q] = v0[t * N + i];
            model_c[q] = model[i];
            term_c[q] = term_rail[i];
            for (int p = 0; p < NPAIR; p++) slot_c[p * N + q] = slot_rail[p * N + i];
        }
        Layout &Lc = c->L_color;
        Lc.N = N;
        TRY(upload(c, &Lc.term, term_c.data(), N));
        TRY(upload(c, &Lc.beta, beta_c.data(), N));
        TRY(upload(c, &Lc.v0, v0_c.data(), 3 * N));
        TRY(upload(c, &Lc.model, model_c.data(), N));
        TRY(upload(c, &Lc.slot, slot_c.data(), NPAIR * N));
    }
    // colour block offsets + rail partials
    c->color_blk_off.assign((size_t)c->n_colors + 1, 0);
    for (int32_t col = 0; col < c->n_colors; col++) {
        const int64_t cnt = c->color_ptr[col + 1] - c->color_ptr[col];
        c->color_blk_off[col + 1] = c->color_blk_off[col] + (cnt + kBlock - 1) / kBlock;
    }
    TRY(dalloc(c, &c->partials, (size_t)(c->color_blk_off[c->n_colors] * std::max(1, c->n_rail_entries))));
    // persistent cooperative form: one CTA set resident on every SM
    {
        int sms = 148, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        int coop = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        const int bps = coop ? color_coop_blocks_per_sm() : 0;
        c->coop_grid = bps * sms;
        TRY(upload(c, &c->d_color_ptr, c->color_ptr.data(), c->color_ptr.size()));
        TRY(dalloc(c, &c->coop_partials, (size_t)std::max(1, c->coop_grid) * std::max(1, c->n_rail_entries)));
    }
    return EES_OK;
}

// COLOR under EES_CONFLICT_HYBRID.  A target can be
// written by two FETs of one colour only if every node it names left the
// conflict relation: an A entry whose row and column are both excluded, or
// the b row of an excluded node.  Such a target stamped by more than one FET
// is a side target: each of its contributions gets its own scratch slot
// (contiguous per target, netlist order, then pair order) and a segmented sum
// adds them after the last colour.  Every other target keeps a plain RMW.
ees_status build_hybrid(const ees_desc *d, ees_ctx *c, const std::vector<int32_t> &raw_slot,
                        const std::vector<uint8_t> &excluded)
{
    const int64_t N = c->n_dev, nnz = c->nnz, NT = nnz + c->n;
    const int32_t *TT[4] = {d->d, d->g, d->s, d->b};
    auto target = [&](int64_t i, int p) -> int64_t {     // p < 12: A pair, else b row p-12
        if (p < NPAIR) return raw_slot[p * N + i];
        const int32_t r = TT[p - NPAIR][i];
        return r >= 0 ? nnz + r : -1;
    };
    // Rails take the side sum under every rule (as the rail partials of
    // COLOR / ATOMIC do): under the paper rule no two FETs of a colour share
    // a rail, but the rail diagonal would otherwise be a sequential sum over
    // all colour phases (10^5 on cfg1), whose rounding can exceed 1e-12 sum|c|.
    std::vector<uint8_t> side_node(excluded);
    for (int32_t r : c->rails) side_node[r] = 1;
    auto candidate = [&](int64_t i, int p) -> bool {
        if (p < NPAIR) return side_node[TT[kPairRow[p]][i]] && side_node[TT[kPairCol[p]][i]];
        return side_node[TT[p - NPAIR][i]] != 0;
    };
    // distinct FETs per candidate target
    std::vector<int32_t> writers((size_t)NT, 0), last((size_t)NT, -1);
    for (int64_t i = 0; i < N; i++)
        for (int p = 0; p < NPAIR + 4; p++) {
            const int64_t g = target(i, p);
            if (g < 0 || !candidate(i, p) || last[g] == (int32_t)i) continue;
            last[g] = (int32_t)i;
            writers[g]++;
        }
    // side ids in target order; contributions per side target
    std::vector<int32_t> sid((size_t)NT, -1), side_gid;
    for (int64_t g = 0; g < NT; g++)
        if (writers[g] >= 2) {
            sid[g] = (int32_t)side_gid.size();
            side_gid.push_back((int32_t)g);
        }
    const int32_t ns = (int32_t)side_gid.size();
    std::vector<int64_t> sptr((size_t)ns + 1, 0);
    for (int64_t i = 0; i < N; i++)
        for (int p = 0; p < NPAIR + 4; p++) {
            const int64_t g = target(i, p);
            if (g >= 0 && candidate(i, p) && sid[g] >= 0) sptr[sid[g] + 1]++;
        }
    for (int32_t k = 0; k < ns; k++) sptr[k + 1] += sptr[k];
    if (sptr[ns] > INT32_MAX - 2) return EES_EINVAL;
    // 16 codes per FET, netlist order
    std::vector<int32_t> code((size_t)(16 * N));
    {
        std::vector<int64_t> fill(sptr.begin(), sptr.end() - 1);
        for (int64_t i = 0; i < N; i++)
            for (int p = 0; p < NPAIR + 4; p++) {
                const int64_t g = target(i, p);
                int32_t v;
                if (g < 0) v = -1;
                else if (candidate(i, p) && sid[g] >= 0) v = (int32_t)(-2 - fill[sid[g]]++);
                else v = (int32_t)(p < NPAIR ? g : g - nnz);
                code[(size_t)p * N + i] = v;
            }
    }
    // chunks
    std::vector<int64_t> chunk_lo(1, 0);
    std::vector<int32_t> side_chunk(1, 0);
    for (int32_t k = 0; k < ns; k++) {
        for (int64_t lo = sptr[k]; lo < sptr[k + 1]; lo += kChunk)
            chunk_lo.push_back(std::min<int64_t>(sptr[k + 1], lo + kChunk));
        side_chunk.push_back((int32_t)chunk_lo.size() - 1);
    }
    c->st.n_color_side_targets = ns;           // side targets of the colour-phased stamps
    c->st.n_color_side_contributions = sptr[ns];
    if (c->host_only) return EES_OK;
    // colour-major copy
    std::vector<int32_t> perm((size_t)N);
    {
        std::vector<int64_t> fill(c->color_ptr.begin(), c->color_ptr.end() - 1);
        for (int64_t i = 0; i < N; i++) perm[fill[c->color[i]]++] = (int32_t)i;
    }
    std::vector<int32_t> code_c((size_t)(16 * N));
    std::vector<double> beta_c((size_t)N), v0_c((size_t)(3 * N));
    std::vector<uint8_t> model_c((size_t)N);
    std::vector<int4> term_c((size_t)N);
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < N; q++) {
        const int64_t i = perm[q];
        const ees_model &m = c->models[d->model[i]];
        beta_c[q] = (m.kp * d->w[i]) / d->l[i];
        for (int t = 0; t < 3; t++) v0_c[t * N + q] = d->vprev[t * N + i];
        model_c[q] = (uint8_t)d->model[i];
        term_c[q] = make_int4(d->d[i], d->g[i], d->s[i], d->b[i]);
        for (int p = 0; p < 16; p++) code_c[(size_t)p * N + q] = code[(size_t)p * N + i];
    }
    TRY(upload(c, &c->d_perm, perm.data(), perm.size()));
    Layout &L = c->L_colorh;
    L.N = N;
    TRY(upload(c, &L.term, term_c.data(), N));
    TRY(upload(c, &L.beta, beta_c.data(), N));
    TRY(upload(c, &L.v0, v0_c.data(), 3 * N));
    TRY(upload(c, &L.model, model_c.data(), N));
    TRY(upload(c, &L.slot, code_c.data(), 16 * N));
    // race-probe codes (netlist order): side targets coded -2, as rails elsewhere
    {
        std::vector<int32_t> pslot((size_t)(NPAIR * N));
        std::vector<int4> pterm((size_t)N);
        for (int64_t i = 0; i < N; i++) {
            for (int p = 0; p < NPAIR; p++) {
                const int32_t v = code[(size_t)p * N + i];
                pslot[(size_t)p * N + i] = v <= -2 ? -2 : v;
            }
            int32_t t4[4];
            for (int a = 0; a < 4; a++) {
                const int32_t v = code[(size_t)(NPAIR + a) * N + i];
                t4[a] = v <= -2 ? -2 : v;
            }
            pterm[i] = make_int4(t4[0], t4[1], t4[2], t4[3]);
        }
        Layout &P = c->L_probe;
        P.N = N;
        TRY(upload(c, &P.term, pterm.data(), N));
        TRY(upload(c, &P.slot, pslot.data(), NPAIR * N));
    }
    SideK &k = c->sk;
    k.n_side = ns;
    k.n_chunks = (int32_t)chunk_lo.size() - 1;
    k.nnz = nnz;
    TRY(dalloc(c, &k.buf, (size_t)sptr[ns]));
    TRY(upload(c, const_cast<int64_t **>(&k.chunk_lo), chunk_lo.data(), chunk_lo.size()));
    TRY(upload(c, const_cast<int32_t **>(&k.side_gid), side_gid.data(), side_gid.size()));
    TRY(upload(c, const_cast<int32_t **>(&k.side_chunk), side_chunk.data(), side_chunk.size()));
    TRY(dalloc(c, &k.chunk_part, (size_t)k.n_chunks));
    return EES_OK;
}

// Locality of the stamp targets in netlist order: a FET whose light
// terminals (fanout <= kHeavyDeg, not rails) lie far apart in node id (> 32)
// is copied into several TILE tiles and scatters GATHER's target-ordered
// stores.  True when that happens more than once per two FETs (cfg3's random
// netlist: ~2 per FET; the inverter, SRAM and hub configs: ~0).
bool scattered_topology(const ees_desc *d, const ees_ctx *c, const std::vector<int64_t> &iptr)
{
    const int64_t N = c->n_dev;
    const int32_t *TT[4] = {d->d, d->g, d->s, d->b};
    const int32_t NN = std::max(1, c->n_nodes);
    std::vector<uint8_t> heavy((size_t)NN, 0);
    for (int32_t v = 0; v < c->n_nodes; v++) heavy[v] = (iptr[v + 1] - iptr[v]) > kHeavyDeg;
    for (int32_t r : c->rails) heavy[r] = 1;
    int64_t extra = 0;
    for (int64_t i = 0; i < N; i++) {
        int32_t lo = INT32_MAX;
        for (int a = 0; a < 4; a++)
            if (TT[a][i] >= 0 && !heavy[TT[a][i]]) lo = std::min(lo, TT[a][i]);
        for (int a = 0; a < 4; a++) {
            const int32_t t = TT[a][i];
            bool dup = false;
            for (int b2 = 0; b2 < a; b2++) dup |= TT[b2][i] == t;
            if (t >= 0 && !heavy[t] && !dup && t - lo > 32) extra++;
        }
    }
    return N && (double)extra / (double)N > 0.5;
}

// GATHER: per-target contributor lists; the target-ordered buffer (form 1) or
// the compact buffer with transposed index lists (form 0).
ees_status build_gather(const ees_desc *d, ees_ctx *c, const std::vector<int32_t> &raw_slot,
                        const std::vector<int64_t> &iptr)
{
    const int64_t N = c->n_dev, nnz = c->nnz;
    const int64_t NT = nnz + c->n;
    const int32_t *TT[4] = {d->d, d->g, d->s, d->b};
    std::vector<int32_t> off((size_t)N + 1, 0);
    std::vector<int64_t> tcnt((size_t)NT + 1, 0);
    for (int64_t i = 0; i < N; i++) {
        int q = 0;
        for (int p = 0; p < NPAIR; p++) {
            const int32_t k = raw_slot[p * N + i];
            if (k >= 0) { q++; tcnt[k]++; }
        }
        for (int a = 0; a < 4; a++)
            if (TT[a][i] >= 0) { q++; tcnt[nnz + TT[a][i]]++; }
        if ((int64_t)off[i] + q > INT32_MAX) return EES_EINVAL;
        off[i + 1] = off[i] + q;
    }
    const int64_t ncontrib = off[N];
    c->st.n_contributions = ncontrib;
    // light / heavy split
    std::vector<int32_t> tptr((size_t)NT + 1, 0);
    std::vector<int32_t> heavy_target;
    std::vector<int32_t> hpos((size_t)NT, -1);
    int64_t hl = 0;
    for (int64_t t = 0; t < NT; t++) {
        const bool heavy = tcnt[t] > kHeavyLen;
        if (heavy) {
            hpos[t] = (int32_t)heavy_target.size();
            heavy_target.push_back((int32_t)t);
            hl += tcnt[t];
        }
        tptr[t + 1] = tptr[t] + (heavy ? 0 : (int32_t)tcnt[t]);
    }
    const int32_t nh = (int32_t)heavy_target.size();
    std::vector<int64_t> hptr((size_t)nh + 1, 0);
    for (int32_t h = 0; h < nh; h++) hptr[h + 1] = hptr[h] + tcnt[heavy_target[h]];
    std::vector<int32_t> tidx((size_t)tptr[NT]), hidx((size_t)hl);
    // target-ordered positions (light lists, then heavy lists) for EES_GATHER
    const int64_t heavy_base = tptr[NT];
    std::vector<int32_t> tpos((size_t)(16 * N), -1);
    {
        std::vector<int32_t> fill(tptr.begin(), tptr.end() - 1);
        std::vector<int64_t> hfill(hptr.begin(), hptr.end() - 1);
        for (int64_t i = 0; i < N; i++) {     // device order -> lists sorted by device
            int32_t q = off[i];
            auto put = [&](int64_t t, int p) {
                if (hpos[t] >= 0) {
                    const int64_t hk = hfill[hpos[t]]++;
                    hidx[hk] = q;
                    tpos[(size_t)p * N + i] = (int32_t)(heavy_base + hk);
                } else {
                    const int32_t lk = fill[t]++;
                    tidx[lk] = q;
                    tpos[(size_t)p * N + i] = lk;
                }
                q++;
            };
            for (int p = 0; p < NPAIR; p++) {
                const int32_t k = raw_slot[p * N + i];
                if (k >= 0) put(k, p);
            }
            for (int a = 0; a < 4; a++)
                if (TT[a][i] >= 0) put(nnz + TT[a][i], NPAIR + a);
        }
    }
    // heavy lists are cut into chunks of kChunk; chunks of one target are
    // consecutive, so chunk c spans [chunk_beg[c], chunk_beg[c+1]).
    std::vector<int32_t> chunk_beg, heavy_chunk((size_t)nh + 1, 0);
    for (int32_t h = 0; h < nh; h++) {
        heavy_chunk[h] = (int32_t)chunk_beg.size();
        for (int64_t b0 = hptr[h]; b0 < hptr[h + 1]; b0 += kChunk) chunk_beg.push_back((int32_t)b0);
    }
    heavy_chunk[nh] = (int32_t)chunk_beg.size();
    const int32_t nchunks = (int32_t)chunk_beg.size();
    chunk_beg.push_back((int32_t)hl);
    GatherK &g = c->gk;
    g.n_targets = NT;
    g.nnz = nnz;
    g.n_chunks = nchunks;
    g.n_heavy = nh;
    TRY(upload(c, const_cast<int32_t **>(&g.off), off.data(), N + 1));
    TRY(dalloc(c, &g.buf, (size_t)ncontrib));
    TRY(upload(c, const_cast<int32_t **>(&g.tptr), tptr.data(), NT + 1));

    TRY(upload(c, const_cast<int32_t **>(&g.chunk_beg), chunk_beg.data(), chunk_beg.size()));

    TRY(dalloc(c, &g.chunk_part, (size_t)nchunks));
    TRY(upload(c, const_cast<int32_t **>(&g.heavy_target), heavy_target.data(), heavy_target.size()));
    TRY(upload(c, const_cast<int32_t **>(&g.heavy_chunk), heavy_chunk.data(), heavy_chunk.size()));
    g.heavy_base = heavy_base;
    // form 1 (target-ordered stores, streamed reduction) unless the targets are
    // scattered in netlist order (cfg3: its stores then cost 8x, form 0 keeps
    // the compact buffer and gathers by index); measured in profiles/r01_f_tile_ab.md
    g.form = scattered_topology(d, c, iptr) ? 0 : 1;
    if (d->flags & EES_SETUP_GATHER_FORM0) g.form = 0;      // layout override (ees.h)
    if (d->flags & EES_SETUP_GATHER_FORM1) g.form = 1;
    c->st.gather_form = g.form;
    if (g.form == 0) {
        TRY(upload(c, const_cast<int32_t **>(&g.tidx), tidx.data(), tidx.size()));
        TRY(upload(c, const_cast<int32_t **>(&g.hidx), hidx.data(), hidx.size()));
    } else {
        TRY(dalloc(c, &g.tbuf, (size_t)ncontrib));
        TRY(upload(c, const_cast<int32_t **>(&g.tpos), tpos.data(), tpos.size()));
    }
    c->st.n_heavy_targets = nh;
    return EES_OK;
}

ees_status build_tile(const ees_desc *d, ees_ctx *c, const std::vector<int32_t> &raw_slot,
                      const std::vector<int64_t> &iptr, const std::vector<int32_t> &idev)
{
    const int32_t *TT[4] = {d->d, d->g, d->s, d->b};
    const int64_t N = c->n_dev;
    std::vector<double> beta((size_t)std::max<int64_t>(1, N));
    for (int64_t i = 0; i < N; i++) {
        const ees_model &m = c->models[d->model[i]];
        beta[i] = (m.kp * d->w[i]) / d->l[i];
    }
    // TILE form (ees_internal.h): items in HBM arrays (form 1, 5 CTAs/SM)
    // unless FETs are copied into several tiles, where the extra per-copy
    // loads cost more than the occupancy gains (form 0; measured: cfg3 1.6x
    // slower in form 1, cfg4 10% faster).
    int form = scattered_topology(d, c, iptr) ? 0 : 1;
    if (d->flags & EES_SETUP_TILE_FORM0) form = 0;          // layout override (ees.h)
    if (d->flags & EES_SETUP_TILE_FORM1) form = 1;
    int sms = 148, dev = 0;
    int grid = sms * tile_ctas(form);
    if (!c->host_only) {
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        grid = sms * tile_blocks_per_sm(form);
    }
    TileHost th;
    if (!build_tile_host(form, N, c->n_nodes, c->n, c->nnz, TT, raw_slot.data(), iptr, idev, c->rails,
                         c->row_ptr, c->col_idx, beta.data(), d->vprev, d->model, grid, th))
        return EES_EINVAL;
    c->st.tile_form = form;
    c->st.n_tiles = th.n_tiles;
    c->st.n_heavy_nodes = th.n_heavy;
    c->st.n_side_targets = th.n_side;
    c->st.n_tile_items = th.n_items;
    c->st.tile_blob_max = th.blob_max;
    c->st.n_tile_programs = th.n_progs;
    c->st.tile_store_waves = th.st_waves;
    c->st.tile_store_waves_naive = th.st_waves0;
    if (c->host_only) return EES_OK;
    TileK &k = c->tk;
    k.form = form;
    k.n_tiles = th.n_tiles;
    k.nnz = c->nnz;
    auto up = [&](auto **dst, const auto &vec) {
        using T = typename std::remove_reference<decltype(vec)>::type::value_type;
        return upload(c, const_cast<T **>(dst), vec.data(), vec.size());
    };
    {
        const uint32_t *td = nullptr;
        TRY(up(&td, th.tdesc));
        k.tdesc = reinterpret_cast<const uint4 *>(td);
    }
    TRY(up(&k.blob, th.blob));
    TRY(up(&k.prog, th.prog));
    TRY(up(&k.item_beta, th.item_beta));
    TRY(up(&k.item_v0, th.item_v0));
    TRY(up(&k.item_model, th.item_model));
    TRY(up(&k.sd_gid, th.sd_gid));
    TRY(up(&k.sd_part, th.sd_part));
    TRY(up(&k.hot_gid, th.hot_gid));
    k.n_side = th.n_side;
    k.n_side_big = th.n_side_big;
    k.n_side_cold = th.n_side_cold;
    k.n_hot = th.n_hot;
    k.hot_base = th.hot_base;
    TRY(dalloc(c, &k.hot_pre, (size_t)std::max(1, th.n_hot)));
    TRY(dalloc(c, &k.part, (size_t)th.n_parts));
    TRY(dalloc(c, &k.gbar, 2));
    if (cudaMemset(k.gbar, 0, 2 * sizeof(unsigned int)) != cudaSuccess) return EES_ECUDA;
    // persistent CTAs: no more than tiles (the hot parts are laid out for
    // `grid` CTAs; k_tile sums the first gridDim.x of them)
    c->tile_grid = th.grid;
    return EES_OK;
}

// Scratch of the tuning calls only: freed when tuning ends (not kept for the
// context's lifetime like the layouts).
struct TuneScratch {
    double *x = nullptr, *A = nullptr, *b = nullptr;
    cudaStream_t st = nullptr;
    ~TuneScratch()
    {
        if (st) cudaStreamSynchronize(st);
        cudaFree(x);
        cudaFree(A);
        cudaFree(b);
        if (st) cudaStreamDestroy(st);
    }
};

ees_status autotune(ees_ctx *c, bool full)
{
    TuneScratch sc;
    if (cudaMalloc(&sc.x, sizeof(double) * std::max(1, c->n)) != cudaSuccess ||
        cudaMalloc(&sc.A, sizeof(double) * std::max<int64_t>(1, c->nnz)) != cudaSuccess ||
        cudaMalloc(&sc.b, sizeof(double) * std::max(1, c->n)) != cudaSuccess) {
        cudaGetLastError();
        return EES_ENOMEM;
    }
    if (cudaStreamCreateWithFlags(&sc.st, cudaStreamNonBlocking) != cudaSuccess) return EES_ECUDA;
    double *x = sc.x, *A = sc.A, *b = sc.b;
    cudaStream_t st = sc.st;
    cudaMemsetAsync(x, 0, sizeof(double) * std::max(1, c->n), st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 1e300;
    int32_t bestv = EES_ATOMIC;
    ees_status rc = EES_OK;
    // mean of 5 back-to-back calls, best of 3 rounds (a round disturbed by
    // the host or a clock step does not decide the variant)
    auto time_variant = [&](int32_t v) -> double {
        for (int it = 0; it < 2 && rc == EES_OK; it++) rc = enqueue(c, v, x, 1e-12, A, b, st, nullptr);
        double best_ms = 1e300;
        for (int round = 0; round < 3 && rc == EES_OK; round++) {
            cudaEventRecord(e0, st);
            const int reps = 5;
            for (int it = 0; it < reps && rc == EES_OK; it++) rc = enqueue(c, v, x, 1e-12, A, b, st, nullptr);
            cudaEventRecord(e1, st);
            if (cudaEventSynchronize(e1) != cudaSuccess) rc = EES_ECUDA;
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            best_ms = std::min(best_ms, (double)ms / reps);
        }
        return best_ms;
    };
    // layout override (ees.h): force the COLOR form instead of timing both
    const char *mode = (c->setup_flags & EES_SETUP_COLOR_LAUNCH) ? "launch"
                       : (c->setup_flags & EES_SETUP_COLOR_COOP) ? "coop" : nullptr;
    for (int32_t v = EES_COLOR; v <= EES_COLOR_BUF && rc == EES_OK; v++) {
        if (!full && v != c->variant) continue;          // an explicit variant: its forms only
        double ms;
        if (v == EES_COLOR_BUF) {
            if (c->n_colors > 512) { c->st.tune_ms[v] = -1; continue; }
            ms = time_variant(v);
        } else if (v == EES_COLOR && c->hybrid) {
            c->color_coop = 0;
            if (c->n_colors > 512) { c->st.tune_ms[v] = -1; continue; }
            ms = time_variant(v);
        } else if (v == EES_COLOR && mode && (!std::strcmp(mode, "launch") || !std::strcmp(mode, "coop"))) {
            c->color_coop = !std::strcmp(mode, "coop") && c->coop_grid > 0;
            ms = time_variant(v);
        } else if (v == EES_ATOMIC) {
            // both ATOMIC forms: plain REDs, and one RED per run of equal entries
            c->atomic_agg = 0;
            ms = time_variant(v);
            if (rc == EES_OK) {
                c->atomic_agg = 1;
                const double ms2 = time_variant(v);
                if (ms2 < ms) ms = ms2;
                else c->atomic_agg = 0;
            }
        } else if (v == EES_COLOR) {
            // colour phasing pays one barrier per colour: past 512 colours it is
            // launch/barrier-bound by construction, not worth timing
            if (c->n_colors > 512) { c->st.tune_ms[v] = -1; continue; }
            c->color_coop = 0;
            ms = time_variant(v);
            if (c->coop_grid > 0 && rc == EES_OK) {
                c->color_coop = 1;
                const double ms2 = time_variant(v);
                if (ms2 < ms) ms = ms2;
                else c->color_coop = 0;
            }
        } else {
            ms = time_variant(v);
        }
        c->st.tune_ms[v] = ms;
        if (ms < best) { best = ms; bestv = v; }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (full) c->variant = bestv;
    return rc;
}

ees_status setup_impl(const ees_desc *d, ees_ctx *c)
{
    const double t0 = now_s();
    TRY(validate(d));
    c->n_nodes = d->n_nodes;
    c->n_extra = d->n_extra;
    c->n = d->n_nodes + d->n_extra;
    c->n_dev = d->n_dev;
    c->models.assign(d->models, d->models + d->n_models);
    c->rails.assign(d->rails, d->rails + d->n_rails);
    c->gmin = d->gmin;
    c->rule = d->conflict_rule;
    c->setup_flags = d->flags;
    const int64_t N = d->n_dev;

    std::vector<int64_t> iptr;
    std::vector<int32_t> idev;
    build_incidence(d, iptr, idev);
    TRY(build_pattern(d, c, iptr, idev));
    // stamp slots (raw CSR indices) per device and live pair
    std::vector<int32_t> raw_slot((size_t)(NPAIR * N));
    {
        const int32_t *TT[4] = {d->d, d->g, d->s, d->b};
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < N; i++)
            for (int p = 0; p < NPAIR; p++) {
                const int32_t r = TT[kPairRow[p]][i], col = TT[kPairCol[p]][i];
                raw_slot[p * N + i] = (r >= 0 && col >= 0) ? find_slot(c, r, col) : -1;
            }
    }
    c->st.setup_pattern_s = now_s() - t0;
    // rails: ordinals, rail x rail A entries, rail b rows
    std::vector<int32_t> rail_ord((size_t)std::max(1, c->n_nodes), -1);
    for (size_t r = 0; r < c->rails.size(); r++) rail_ord[c->rails[r]] = (int32_t)r;
    int32_t ne = 0;
    for (size_t r = 0; r < c->rails.size(); r++)
        for (size_t r2 = 0; r2 < c->rails.size(); r2++) {
            const int32_t k = find_slot(c, c->rails[r], c->rails[r2]);
            if (k >= 0) c->rail_target[ne++] = k;
        }
    c->n_rail_a = ne;
    for (size_t r = 0; r < c->rails.size(); r++) c->rail_target[ne++] = c->rails[r];
    c->n_rail_entries = ne;
    // colouring
    const double tc = now_s();
    std::vector<uint8_t> excluded((size_t)std::max(1, c->n_nodes), 0);
    if (d->conflict_rule != EES_CONFLICT_PAPER)
        for (int32_t r : c->rails) excluded[r] = 1;
    if (d->conflict_rule == EES_CONFLICT_HYBRID) {
        // nodes with more than K incident FETs leave the relation
        const int64_t K = d->heavy_degree > 0 ? d->heavy_degree : 64;
        for (int32_t v = 0; v < c->n_nodes; v++)
            if (iptr[v + 1] - iptr[v] > K) excluded[v] = 1;
        c->hybrid = true;
    }
    for (int32_t v = 0; v < c->n_nodes; v++) c->st.n_excluded_nodes += excluded[v];
    int32_t maxdeg = 0;
    c->n_colors = greedy_color(d, excluded, c->color, maxdeg);
    c->color_ptr.assign((size_t)c->n_colors + 1, 0);
    for (int64_t i = 0; i < N; i++) c->color_ptr[c->color[i] + 1]++;
    int64_t gmax = 0, gmin = N;
    for (int32_t col = 0; col < c->n_colors; col++) {
        gmax = std::max(gmax, c->color_ptr[col + 1]);
        gmin = std::min(gmin, c->color_ptr[col + 1]);
    }
    for (int32_t col = 0; col < c->n_colors; col++) c->color_ptr[col + 1] += c->color_ptr[col];
    c->st.setup_color_s = now_s() - tc;
    c->st.max_group = (int32_t)gmax;
    c->st.min_group = c->n_colors ? (int32_t)gmin : 0;
    c->st.max_conflict_node_degree = maxdeg;

    c->host_only = (d->flags & EES_SETUP_HOST_ONLY) != 0;
    if (c->host_only) {
        int64_t nc = 0;
        for (int64_t k = 0; k < NPAIR * N; k++) nc += raw_slot[k] >= 0;
        for (int64_t i = 0; i < N; i++)
            nc += (d->d[i] >= 0) + (d->g[i] >= 0) + (d->s[i] >= 0) + (d->b[i] >= 0);
        c->st.n_contributions = nc;
        TRY(build_hybrid(d, c, raw_slot, excluded));
        TRY(build_tile(d, c, raw_slot, iptr, idev));
        c->variant = d->variant == EES_AUTO ? EES_ATOMIC : d->variant;
        c->st.setup_s = now_s() - t0;
        return EES_OK;
    }
    TRY(build_layouts(d, c, raw_slot, rail_ord));
    TRY(build_hybrid(d, c, raw_slot, excluded));      // COLOR (hybrid rule) and COLOR_BUF
    TRY(build_gather(d, c, raw_slot, iptr));
    TRY(build_tile(d, c, raw_slot, iptr, idev));
    int sms = 148;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (N + kBlock - 1) / kBlock;
    c->atomic_grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * atomic_blocks_per_sm()));
    if (cudaDeviceSynchronize() != cudaSuccess) return EES_ECUDA;
    if (d->variant == EES_AUTO) {
        TRY(autotune(c, true));
    } else {
        c->variant = d->variant;
        if (d->variant == EES_COLOR || d->variant == EES_ATOMIC) TRY(autotune(c, false));   // pick its form
    }
    c->st.setup_s = now_s() - t0;
    return EES_OK;
}

void free_ctx(ees_ctx *c)
{
    if (!c) return;
    for (auto &m : c->marks) {
        cudaEventDestroy(m.a);
        cudaEventDestroy(m.b);
    }
    for (cudaEvent_t e : c->ev_free) cudaEventDestroy(e);
    for (void *p : c->allocs) cudaFree(p);
    delete c;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

ees_status ees_setup(const ees_desc *desc, ees_ctx **out)
{
    if (!out) return EES_EINVAL;
    *out = nullptr;
    ees_ctx *c = new (std::nothrow) ees_ctx();
    if (!c) return EES_ENOMEM;
    ees_status s;
    try {
        s = setup_impl(desc, c);
    } catch (const std::bad_alloc &) {
        s = EES_ENOMEM;
    } catch (...) {
        s = EES_EINVAL;
    }
    if (s != EES_OK) {
        free_ctx(c);
        return s;
    }
    *out = c;
    return EES_OK;
}

ees_status ees_pattern(const ees_ctx *c, int32_t *n, int64_t *nnz, const int32_t **row_ptr,
                       const int32_t **col_idx)
{
    if (!c) return EES_EINVAL;
    if (n) *n = c->n;
    if (nnz) *nnz = c->nnz;
    if (row_ptr) *row_ptr = c->row_ptr.data();
    if (col_idx) *col_idx = c->col_idx.data();
    return EES_OK;
}

ees_status ees_find_slot(const ees_ctx *c, int32_t row, int32_t col, int64_t *slot)
{
    if (!c || !slot || row < 0 || row >= c->n || col < 0 || col >= c->n) return EES_EINVAL;
    *slot = find_slot(c, row, col);
    return EES_OK;
}

ees_status ees_colors(const ees_ctx *c, const int32_t **color, int32_t *n_colors)
{
    if (!c) return EES_EINVAL;
    if (color) *color = c->color.data();
    if (n_colors) *n_colors = c->n_colors;
    return EES_OK;
}

ees_status ees_eval_stamp(ees_ctx *c, const double *x, double h, double *A, double *b, ees_stream stream)
{
    if (!c) return EES_EINVAL;
    if (!(h > 0.0)) return EES_EINVAL;           // rejects h <= 0 and NaN; +inf = DC
    if (c->host_only) return EES_ESTATE;
    if (c->n_dev == 0) return EES_OK;
    if (!x || !A || !b) return EES_EINVAL;
    int32_t nl = 0;
    ees_status s = enqueue(c, c->variant, x, h, A, b, (cudaStream_t)stream, &nl, c->timing);
    if (c->timing) c->timed_calls++;
    c->launches = nl;
    return s;
}

ees_status ees_eval_stamp_host(ees_ctx *c, const double *x, double h, double *A, double *b,
                               ees_stream stream, int32_t flags)
{
    if (flags & ~EES_HOST_ASSIGN) return EES_EINVAL;
    if (!c) return EES_EINVAL;
    if (!(h > 0.0)) return EES_EINVAL;
    if (c->host_only) return EES_ESTATE;
    if (!x || !A || !b) return EES_EINVAL;
    if (!c->hx) {
        TRY(dalloc(c, &c->hx, (size_t)c->n));
        TRY(dalloc(c, &c->hA, (size_t)c->nnz));
        TRY(dalloc(c, &c->hb, (size_t)c->n));
    }
    cudaStream_t st = (cudaStream_t)stream;
    const size_t bn = sizeof(double) * (size_t)c->n, ba = sizeof(double) * (size_t)c->nnz;
    if (cudaMemcpyAsync(c->hx, x, bn, cudaMemcpyHostToDevice, st) != cudaSuccess) return EES_ECUDA;
    if (flags & EES_HOST_ASSIGN) {
        if (cudaMemsetAsync(c->hA, 0, ba, st) != cudaSuccess) return EES_ECUDA;
        if (cudaMemsetAsync(c->hb, 0, bn, st) != cudaSuccess) return EES_ECUDA;
    } else {
        if (cudaMemcpyAsync(c->hA, A, ba, cudaMemcpyHostToDevice, st) != cudaSuccess) return EES_ECUDA;
        if (cudaMemcpyAsync(c->hb, b, bn, cudaMemcpyHostToDevice, st) != cudaSuccess) return EES_ECUDA;
    }
    ees_status s = ees_eval_stamp(c, c->hx, h, c->hA, c->hb, stream);
    if (s != EES_OK) return s;
    if (cudaMemcpyAsync(A, c->hA, ba, cudaMemcpyDeviceToHost, st) != cudaSuccess) return EES_ECUDA;
    if (cudaMemcpyAsync(b, c->hb, bn, cudaMemcpyDeviceToHost, st) != cudaSuccess) return EES_ECUDA;
    return cudaStreamSynchronize(st) == cudaSuccess ? EES_OK : EES_ECUDA;
}

ees_status ees_set_variant(ees_ctx *c, int32_t variant)
{
    if (!c || variant < EES_AUTO || variant > EES_COLOR_BUF) return EES_EINVAL;
    if (variant == EES_AUTO) {
        double best = 1e300;
        int32_t bv = c->variant;
        for (int v = EES_COLOR; v <= EES_COLOR_BUF; v++)
            if (c->st.tune_ms[v] > 0 && c->st.tune_ms[v] < best) { best = c->st.tune_ms[v]; bv = v; }
        c->variant = bv;
    } else {
        c->variant = variant;
    }
    return EES_OK;
}

ees_status ees_accept(ees_ctx *c, const double *x, ees_stream stream)
{
    if (!c) return EES_EINVAL;
    if (c->host_only) return EES_ESTATE;
    if (c->n_dev == 0) return EES_OK;
    if (!x) return EES_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const CallK call = make_call(c, x, 1.0, nullptr, nullptr);
    cudaError_t e = launch_accept_soa(c->L_gather.term, c->n_dev, call, c->L_gather.v0, st);
    if (e == cudaSuccess) e = launch_accept_soa(c->L_atomic.term, c->n_dev, call, c->L_atomic.v0, st);
    if (e == cudaSuccess) e = launch_accept_soa(c->L_color.term, c->n_dev, call, c->L_color.v0, st);
    if (e == cudaSuccess && c->hybrid)
        e = launch_accept_soa(c->L_colorh.term, c->n_dev, call, c->L_colorh.v0, st);
    if (e == cudaSuccess)
        e = launch_accept_tile(c->tk, call, c->tk.form == 1 ? const_cast<double *>(c->tk.item_v0) : nullptr, st);
    return e == cudaSuccess ? EES_OK : EES_ECUDA;
}

ees_status ees_set_work(ees_ctx *c, int32_t work)
{
    if (!c || work < 1) return EES_EINVAL;
    c->work = work;
    return EES_OK;
}

ees_status ees_fp64_peak(double *tflops)
{
    if (!tflops) return EES_EINVAL;
    return measure_fp64_peak(tflops) == cudaSuccess ? EES_OK : EES_ECUDA;
}

ees_status ees_red_throughput(int32_t mode, double *gops)
{
    if (!gops || (mode != 0 && mode != 1)) return EES_EINVAL;
    return measure_red_throughput(mode, gops) == cudaSuccess ? EES_OK : EES_ECUDA;
}

ees_status ees_stream_probe(const void *src, int64_t read_bytes, void *dst, int64_t write_bytes,
                            double *sink, ees_stream stream)
{
    if (!src || !dst || !sink || read_bytes < 0 || write_bytes < 0) return EES_EINVAL;
    if (((uintptr_t)src | (uintptr_t)dst) & 15) return EES_EINVAL;
    return launch_stream_probe(src, read_bytes, dst, write_bytes, sink, (cudaStream_t)stream) == cudaSuccess
               ? EES_OK
               : EES_ECUDA;
}

int64_t ees_abi_sizeof(int32_t which)
{
    return which == 0 ? (int64_t)sizeof(ees_desc) : which == 1 ? (int64_t)sizeof(ees_stats_t) : 0;
}

ees_status ees_stats(const ees_ctx *c, ees_stats_t *out)
{
    if (!c || !out) return EES_EINVAL;
    *out = c->st;
    out->n_dev = c->n_dev;
    out->nnz = c->nnz;
    out->n = c->n;
    out->n_colors = c->n_colors;
    out->variant_chosen = c->variant;
    out->n_rail_entries = c->n_rail_entries;
    out->launches_per_call = c->launches;
    out->atomic_form = c->atomic_agg;
    return EES_OK;
}

ees_status ees_set_timing(ees_ctx *c, int32_t enable)
{
    if (!c) return EES_EINVAL;
    c->timing = enable != 0;
    return EES_OK;
}

ees_status ees_phase_times(ees_ctx *c, double ms[4], int32_t *n_calls)
{
    if (!c || !ms) return EES_EINVAL;
    for (int k = 0; k < 4; k++) ms[k] = 0.0;
    cudaError_t err = cudaSuccess;
    for (auto &m : c->marks) {
        if (err == cudaSuccess) err = cudaEventSynchronize(m.b);
        float t = 0.f;
        if (err == cudaSuccess && cudaEventElapsedTime(&t, m.a, m.b) == cudaSuccess) ms[m.phase] += t;
        c->ev_free.push_back(m.a);
        c->ev_free.push_back(m.b);
    }
    c->marks.clear();
    if (n_calls) *n_calls = c->timed_calls;
    c->timed_calls = 0;
    return err == cudaSuccess ? EES_OK : EES_ECUDA;
}

ees_status ees_tile_trace(ees_ctx *c, const double *x, double h, double *A, double *b, ees_stream stream,
                          uint64_t *trace, int64_t cap, int32_t *n_ctas)
{
    if (!c || !trace || !n_ctas || !x || !A || !b || !(h > 0.0)) return EES_EINVAL;
    if (c->host_only || c->tk.n_tiles == 0) return EES_ESTATE;
    const int64_t need = (int64_t)c->tile_grid * kTraceSlots;
    if (cap < need) return EES_EINVAL;
    unsigned long long *d = nullptr;
    if (cudaMalloc(&d, sizeof(uint64_t) * need) != cudaSuccess) return EES_ENOMEM;
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(d, 0, sizeof(uint64_t) * need, st);
    TileK k = c->tk;
    k.trace = d;
    const CallK call = make_call(c, x, h, A, b);
    int nl = 0;
    cudaError_t e = launch_tile(k, call, c->tile_grid, st, &nl);
    if (e == cudaSuccess) e = cudaMemcpyAsync(trace, d, sizeof(uint64_t) * need, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d);
    *n_ctas = c->tile_grid;
    return e == cudaSuccess ? EES_OK : EES_ECUDA;
}

ees_status ees_race_probe(ees_ctx *c, const int32_t *color, int64_t *n_conflicts)
{
    if (!c || !n_conflicts) return EES_EINVAL;
    if (c->host_only) return EES_ESTATE;
    const int64_t N = c->n_dev;
    const int32_t *col = color ? color : c->color.data();
    int32_t C = 0;
    for (int64_t i = 0; i < N; i++) {
        if (col[i] < 0) return EES_EINVAL;
        C = std::max(C, col[i] + 1);
    }
    std::vector<int64_t> ptr((size_t)C + 1, 0);
    for (int64_t i = 0; i < N; i++) ptr[col[i] + 1]++;
    for (int32_t k = 0; k < C; k++) ptr[k + 1] += ptr[k];
    std::vector<int32_t> perm((size_t)std::max<int64_t>(1, N));
    {
        std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
        for (int64_t i = 0; i < N; i++) perm[fill[col[i]]++] = (int32_t)i;
    }
    if (!c->hybrid)                 // the probe reads the ATOMIC layout: its positions
        for (int64_t q = 0; q < N; q++) perm[q] = c->atomic_pos[perm[q]];
    int32_t *dperm = nullptr, *cnt_a = nullptr, *cnt_b = nullptr;
    unsigned long long *dout = nullptr;
    cudaError_t e = cudaMalloc(&dperm, sizeof(int32_t) * perm.size());
    e = e == cudaSuccess ? cudaMalloc(&cnt_a, sizeof(int32_t) * std::max<int64_t>(1, c->nnz)) : e;
    e = e == cudaSuccess ? cudaMalloc(&cnt_b, sizeof(int32_t) * std::max(1, c->n)) : e;
    e = e == cudaSuccess ? cudaMalloc(&dout, sizeof(unsigned long long)) : e;
    if (e == cudaSuccess) e = cudaMemcpy(dperm, perm.data(), sizeof(int32_t) * perm.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(dout, 0, sizeof(unsigned long long));
    for (int32_t k = 0; k < C && e == cudaSuccess; k++) {
        cudaMemsetAsync(cnt_a, 0, sizeof(int32_t) * c->nnz, 0);
        cudaMemsetAsync(cnt_b, 0, sizeof(int32_t) * c->n, 0);
        e = launch_race_probe(c->hybrid ? c->L_probe.k() : c->L_atomic.k(), dperm, ptr[k], ptr[k + 1] - ptr[k],
                              cnt_a, cnt_b, 0);
        if (e == cudaSuccess) e = launch_count_conflicts(cnt_a, c->nnz, dout, 0);
        if (e == cudaSuccess) e = launch_count_conflicts(cnt_b, c->n, dout, 0);
    }
    unsigned long long hout = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&hout, dout, sizeof(hout), cudaMemcpyDeviceToHost);
    cudaFree(dperm);
    cudaFree(cnt_a);
    cudaFree(cnt_b);
    cudaFree(dout);
    if (e != cudaSuccess) return EES_ECUDA;
    *n_conflicts = (int64_t)hout;
    return EES_OK;
}

ees_status ees_destroy(ees_ctx *c)
{
    if (!c) return EES_EINVAL;
    free_ctx(c);
    return EES_OK;
}

const char *ees_strerror(ees_status s)
{
    switch (s) {
    case EES_OK: return "ok";
    case EES_EINVAL: return "invalid argument";
    case EES_ENOMEM: return "out of memory";
    case EES_ECUDA: return "CUDA error";
    case EES_ESTATE: return "invalid context state";
    default: return "unknown status";
    }
}

}  // extern "C"
