// ees_kernels.cu -- sm_100a kernels of the evaluate+stamp hot path.
//
// Evaluation ("Compute Phase") is SPEC.md's Level-1 MOSFET
// with gmin and backward-Euler capacitor companions, read
// as SURVEY.md §8(c) / DESIGN.md §2: FP64, one thread per device, all
// intermediates in registers, SoA loads in the variant's device order.  It is
// fused into each stamping variant ("Stamp Phase"):
//
//   k_color        colour-phased, no atomics (P:36, P:62, P:80 ColorFused)
//   k_atomic       one pass, FP64 RED into A_vals / b
//   k_gather_*     contributions to scratch, then a deterministic per-entry
//                  segmented reduction (north_star "gather")
//   k_rail_final   deterministic fixed-order sum of per-block rail partials
//
// The path is HBM-bound (~46 FP64 flops vs ~100-155 compulsory bytes per
// device); there is no dense contraction, so no tensor cores.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "ees_internal.h"

namespace cg = cooperative_groups;

namespace ees {

// ---------------------------------------------------------------------------
// Device evaluation: Y (12 live pairs) and J (4 rows) of one FET.
// S:196 Level-1 + D/S swap + PMOS reflection; SURVEY §8(c) steps 1-8.
// ---------------------------------------------------------------------------
struct Stamp {
    double y[NPAIR];
    double j[4];
};

__device__ __forceinline__ void eval_fet1(const CardK &cd, double beta, double gmin, double VD,
                                          double VG, double VS, double v0gs, double v0gd,
                                          double v0db, Stamp &st)
{
    const double p = cd.p;
    const double vgs = p * (VG - VS);               // reflected frame
    const double vds = p * (VD - VS);
    const bool fwd = vds >= 0.0;                    // mode (A8: vds = 0 -> forward)
    const double u = fwd ? vgs : vgs - vds;         // D/S swap in reverse mode
    const double v = fwd ? vds : -vds;
    const double uov = u - cd.vt;
    const double op = 1.0 + cd.lam * v;
    const bool on = !(uov <= 0.0);                  // uov = 0 -> cutoff; NaN propagates (as the oracle)
    const bool sat = v >= uov;                      // v = uov -> saturation
    // q = f / (beta*op): saturation uov^2/2, triode uov*v - v^2/2
    const double q = sat ? 0.5 * uov * uov : uov * v - 0.5 * v * v;
    const double bop = beta * op;
    double f = bop * q;
    double fu = bop * (sat ? uov : v);
    double fv = (sat ? 0.0 : bop * (uov - v)) + beta * q * cd.lam;
    if (!on) { f = 0.0; fu = 0.0; fv = 0.0; }
    const double F = fwd ? f : -f;
    const double gm = fwd ? fu : -fu;               // terminal frame (A9)
    const double gds = fwd ? fv : fu + fv;
    const double I = p * F;
    const double ieq = I - gm * (VG - VS) - gds * (VD - VS);   // Norton
    const double g1 = cd.gcgs, g2 = cd.gcgd, g3 = cd.gcdb;     // C/h
    const double gmgds = gm + gds;
    st.y[DD] = gds + gmin + g2 + g3;
    st.y[DG] = gm - g2;
    st.y[DS] = -gmgds - gmin;
    st.y[DB] = -g3;
    st.y[GD] = -g2;
    st.y[GG] = g1 + g2;
    st.y[GS] = -g1;
    st.y[SD] = -gds - gmin;
    st.y[SG] = -gm - g1;
    st.y[SS] = gmgds + gmin + g1;
    st.y[BD] = -g3;
    st.y[BB] = g3;
    const double qgs = g1 * v0gs, qgd = g2 * v0gd, qdb = g3 * v0db;   // BE companions
    st.j[0] = -ieq - qgd + qdb;
    st.j[1] = qgs + qgd;
    st.j[2] = ieq - qgs;
    st.j[3] = -qdb;
}

// SPEC S:229 work multiplier: the evaluation arithmetic is repeated `work`
// times (BSIM4 cost emulation).  Each repetition reads
// the biases through a dependency on the previous result (+0.0 * y: exact
// for finite y), so the compiler cannot drop it; the result is the same.
// Kernels are instantiated with kRep = false (work == 1, no loop) and true.
template <bool kRep>
__device__ __forceinline__ void eval_fet(const CardK &cd, double beta, double gmin, double VD,
                                         double VG, double VS, double v0gs, double v0gd,
                                         double v0db, Stamp &st, int work)
{
    eval_fet1(cd, beta, gmin, VD, VG, VS, v0gs, v0gd, v0db, st);
    if (kRep)
    for (int r = 1; r < work; r++) {
        const double z = 0.0 * st.y[DD];
        eval_fet1(cd, beta, gmin, VD + z, VG + z, VS + z, v0gs, v0gd, v0db, st);
    }
}

__device__ __forceinline__ double volt(int t, const double *__restrict__ x, const double *s_railx)
{
    return t >= 0 ? __ldg(x + t) : (t == -1 ? 0.0 : s_railx[-2 - t]);
}

// Load + evaluate device i of layout dv.  Returns terminal codes in T.
template <bool kRep>
__device__ __forceinline__ void load_eval(const DevK &dv, const CallK &P, const CardK *s_cards,
                                          const double *s_railx, int64_t i, int4 &T, Stamp &st)
{
    T = __ldg(dv.term + i);
    const double beta = __ldg(dv.beta + i);
    const double a0 = __ldg(dv.v0 + i);
    const double a1 = __ldg(dv.v0 + dv.N + i);
    const double a2 = __ldg(dv.v0 + 2 * dv.N + i);
    const int m = __ldg(dv.model + i);
    const double VD = volt(T.x, P.x, s_railx);
    const double VG = volt(T.y, P.x, s_railx);
    const double VS = volt(T.z, P.x, s_railx);
    eval_fet<kRep>(s_cards[m], beta, P.gmin, VD, VG, VS, a0, a1, a2, st, P.work);
}

__device__ __forceinline__ void load_call_smem(const CallK &P, CardK *s_cards, double *s_railx)
{
    for (int k = threadIdx.x; k < P.n_models; k += blockDim.x) s_cards[k] = P.cards[k];
    for (int k = threadIdx.x; k < P.n_rail_nodes; k += blockDim.x) s_railx[k] = P.x[P.rail_node[k]];
}

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Rail side reduction, per warp: for every rail entry e, the warp's sum of
// this iteration's contributions is added (fixed order) to s_acc[warp][e].
// tc = (d, g, s, b) codes of the b rows (after any merge).
__device__ __forceinline__ void rail_accumulate(const CallK &P, const int32_t *slot, const int *tc,
                                                const Stamp &st, bool valid, double *s_acc)
{
    bool mine = false;
    if (valid) {
#pragma unroll
        for (int p = 0; p < NPAIR; p++) mine |= slot[p] <= -2;
#pragma unroll
        for (int a = 0; a < 4; a++) mine |= tc[a] <= -2;
    }
    if (!__any_sync(0xffffffffu, mine)) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = 0; e < P.n_rail_entries; e++) {
        double v = 0.0;
        if (mine) {
            if (e < P.n_rail_a) {
                const int code = -2 - e;
#pragma unroll
                for (int p = 0; p < NPAIR; p++) v += slot[p] == code ? st.y[p] : 0.0;
            } else {
                const int code = -2 - (e - P.n_rail_a);
#pragma unroll
                for (int a = 0; a < 4; a++) v += tc[a] == code ? st.j[a] : 0.0;
            }
        }
        v = warp_sum(v);
        if (lane == 0) s_acc[warp * P.n_rail_entries + e] += v;
    }
}

// Source tied to bulk (every PMOS of the inverter configs): DS/DB, SD/BD and
// SS/BB address the same entry and J[S]/J[B] the same row -- fold them so one
// RMW carries both (the sum is exact up to one rounding, inside 1e-12 sum|c|).
__device__ __forceinline__ void merge_source_bulk(const int4 &T, Stamp &st, int32_t *slot, int *tc)
{
    if (T.z == T.w && T.z != -1) {
        st.y[DS] += st.y[DB];
        st.y[SD] += st.y[BD];
        st.y[SS] += st.y[BB];
        st.j[2] += st.j[3];
        slot[DB] = -1;
        slot[BD] = -1;
        slot[BB] = -1;
        tc[3] = -1;
    }
}

// ---------------------------------------------------------------------------
// ATOMIC: grid-stride over devices (class order), RED.F64 into A and b;
// rail entries reduced per block, one atomic per block and entry at the end.
// All per-device loads (data + 12 slots) are issued before the x gather.
// Hot entries: lanes of a warp are consecutive devices, and
// devices that share an entry are mostly consecutive in the netlist (a hub's
// fanout, an inverter's N and P), so for each pair / row a warp first checks
// (one shuffle + vote) whether a lane repeats its left neighbour's entry; if
// so, a segmented warp scan sums each run of equal entries and only the run's
// last lane issues the RED -- one same-address RED per run instead of one per
// lane (the L2 serialises same-address atomics, P:31's lock analogue).  The
// scan costs instructions where runs are short and the kernel is latency
// bound (cfg1), so setup times both forms (kAgg) and keeps the faster.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void red_run(double *base, int32_t k, double v, int lane)
{
    const int32_t kp = __shfl_up_sync(0xffffffffu, k, 1);
    const bool dup = lane > 0 && k >= 0 && k == kp;
    if (__any_sync(0xffffffffu, dup)) {
        const int32_t kn = __shfl_down_sync(0xffffffffu, k, 1);
        bool f = !dup;                                   // lane has reached its run's head
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, v, d);
            const bool ft = __shfl_up_sync(0xffffffffu, f, d);
            if (lane >= d && !f) {
                v += t;
                f = ft;
            }
        }
        if (k >= 0 && (lane == 31 || kn != k)) atomicAdd(base + k, v);
    } else if (k >= 0) {
        atomicAdd(base + k, v);
    }
}

#ifndef EES_ATOMIC_MINB
#define EES_ATOMIC_MINB 4          // resident 256-thread blocks per SM the register budget targets
#endif
template <bool kRep, bool kAgg>
__global__ void __launch_bounds__(kBlock, EES_ATOMIC_MINB) k_atomic(DevK dv, CallK P)
{
    __shared__ CardK s_cards[EES_MAX_MODELS];
    __shared__ double s_railx[EES_MAX_RAILS];
    extern __shared__ double s_acc[];   // [warps][n_rail_entries]
    load_call_smem(P, s_cards, s_railx);
    const int nw = blockDim.x >> 5;
    const int lane = threadIdx.x & 31;
    for (int k = threadIdx.x; k < nw * P.n_rail_entries; k += blockDim.x) s_acc[k] = 0.0;
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // warp-uniform trip count so the run scans' and rail_accumulate's shuffles are full-warp
    const int64_t base0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    for (int64_t base = base0; base < dv.N; base += stride) {
        const int64_t i = base + lane;
        const bool valid = i < dv.N;
        int4 T = make_int4(-1, -1, -1, -1);
        Stamp st;
        int32_t slot[NPAIR];
        int tc[4] = {-1, -1, -1, -1};
        if (valid) {
            T = __ldg(dv.term + i);
            const double beta = __ldg(dv.beta + i);
            const double a0 = __ldg(dv.v0 + i);
            const double a1 = __ldg(dv.v0 + dv.N + i);
            const double a2 = __ldg(dv.v0 + 2 * dv.N + i);
            const int m = __ldg(dv.model + i);
            // codes dead by the device's class are not loaded (DevK::cls_a / cls_b)
            const bool dead_s = i < dv.cls_a, dead_b = i < dv.cls_b;
#pragma unroll
            for (int p = 0; p < NPAIR; p++) {
                const bool sp = p == DS || p == GS || p == SD || p == SG || p == SS;
                const bool bp = p == DB || p == BD || p == BB;
                slot[p] = (dead_b && bp) || (dead_s && sp) ? -1 : __ldg(dv.slot + (int64_t)p * dv.N + i);
            }
            const double VD = volt(T.x, P.x, s_railx);
            const double VG = volt(T.y, P.x, s_railx);
            const double VS = volt(T.z, P.x, s_railx);
            eval_fet<kRep>(s_cards[m], beta, P.gmin, VD, VG, VS, a0, a1, a2, st, P.work);
            tc[0] = T.x; tc[1] = T.y; tc[2] = T.z; tc[3] = T.w;
            merge_source_bulk(T, st, slot, tc);
        } else {
#pragma unroll
            for (int p = 0; p < NPAIR; p++) {
                slot[p] = -1;
                st.y[p] = 0.0;
            }
#pragma unroll
            for (int a = 0; a < 4; a++) st.j[a] = 0.0;
        }
        if (kAgg) {
#pragma unroll
            for (int p = 0; p < NPAIR; p++) red_run(P.A, slot[p], st.y[p], lane);
#pragma unroll
            for (int a = 0; a < 4; a++) red_run(P.b, tc[a], st.j[a], lane);
        } else {
#pragma unroll
            for (int p = 0; p < NPAIR; p++)
                if (slot[p] >= 0) atomicAdd(P.A + slot[p], st.y[p]);
#pragma unroll
            for (int a = 0; a < 4; a++)
                if (tc[a] >= 0) atomicAdd(P.b + tc[a], st.j[a]);
        }
        if (P.n_rail_entries) rail_accumulate(P, slot, tc, st, valid, s_acc);
    }
    if (P.n_rail_entries) {
        __syncthreads();
        for (int e = threadIdx.x; e < P.n_rail_entries; e += blockDim.x) {
            double v = 0.0;
            for (int w = 0; w < nw; w++) v += s_acc[w * P.n_rail_entries + e];
            double *dst = e < P.n_rail_a ? P.A + P.rail_target[e] : P.b + P.rail_target[e];
            atomicAdd(dst, v);
        }
    }
}

// ---------------------------------------------------------------------------
// COLOR: one launch per colour; devices of a colour share no non-rail node,
// so plain read-modify-write is race-free.  Rail entries go to a
// per-block partial (deterministic), summed by k_rail_final.
// ---------------------------------------------------------------------------
template <bool kRep>
__global__ void __launch_bounds__(kBlock) k_color(DevK dv, CallK P, int64_t begin, int64_t count,
                                                  double *partials)
{
    __shared__ CardK s_cards[EES_MAX_MODELS];
    __shared__ double s_railx[EES_MAX_RAILS];
    extern __shared__ double s_acc[];
    load_call_smem(P, s_cards, s_railx);
    const int nw = blockDim.x >> 5;
    for (int k = threadIdx.x; k < nw * P.n_rail_entries; k += blockDim.x) s_acc[k] = 0.0;
    __syncthreads();
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = q < count;
    const int64_t i = begin + q;
    int4 T = make_int4(-1, -1, -1, -1);
    Stamp st;
    int32_t slot[NPAIR];
    int tc[4] = {-1, -1, -1, -1};
    if (valid) {
#pragma unroll
        for (int p = 0; p < NPAIR; p++) slot[p] = __ldg(dv.slot + (int64_t)p * dv.N + i);
        load_eval<kRep>(dv, P, s_cards, s_railx, i, T, st);
        tc[0] = T.x; tc[1] = T.y; tc[2] = T.z; tc[3] = T.w;
        merge_source_bulk(T, st, slot, tc);
#pragma unroll
        for (int p = 0; p < NPAIR; p++)
            if (slot[p] >= 0) P.A[slot[p]] += st.y[p];
#pragma unroll
        for (int a = 0; a < 4; a++)
            if (tc[a] >= 0) P.b[tc[a]] += st.j[a];
    } else {
#pragma unroll
        for (int p = 0; p < NPAIR; p++) slot[p] = -1;
    }
    if (P.n_rail_entries) {
        rail_accumulate(P, slot, tc, st, valid, s_acc);
        __syncthreads();
        for (int e = threadIdx.x; e < P.n_rail_entries; e += blockDim.x) {
            double v = 0.0;
            for (int w = 0; w < nw; w++) v += s_acc[w * P.n_rail_entries + e];
            partials[(int64_t)blockIdx.x * P.n_rail_entries + e] = v;
        }
    }
}

// Fixed-order reduction of the rail partials: one block per rail entry; each
// thread sums a fixed strided subset, then a fixed shuffle/smem tree.
__global__ void __launch_bounds__(kBlock) k_rail_final(CallK P, const double *partials,
                                                       int64_t n_blocks)
{
    __shared__ double s_w[kBlock / 32];
    const int e = blockIdx.x;
    double v = 0.0;
    for (int64_t k = threadIdx.x; k < n_blocks; k += blockDim.x)
        v += partials[k * P.n_rail_entries + e];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += s_w[w];
        double *dst = e < P.n_rail_a ? P.A + P.rail_target[e] : P.b + P.rail_target[e];
        *dst += t;
    }
}

// ---------------------------------------------------------------------------
// GATHER (deterministic): K3a evaluates and writes each device's live
// contributions contiguously (pairs in order, then b rows), staged through
// shared memory so the global store is coalesced; K3b reduces every target
// (A entry, then b row) over its contributor list in list order; heavy lists
// are split into fixed chunks reduced by whole blocks (K3b tail blocks) and
// summed in chunk order by K3c.
// ---------------------------------------------------------------------------
template <bool kRep>
__global__ void __launch_bounds__(kBlock) k_gather_eval(DevK dv, GatherK gk, CallK P)
{
    __shared__ CardK s_cards[EES_MAX_MODELS];
    __shared__ double s_railx[EES_MAX_RAILS];
    __shared__ double s_buf[kBlock * (NPAIR + 4)];
    load_call_smem(P, s_cards, s_railx);
    __syncthreads();
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x;
    const int64_t i = i0 + threadIdx.x;
    const int64_t iend = min((int64_t)dv.N, i0 + blockDim.x);
    const int32_t base = gk.off[i0];
    const int32_t total = gk.off[iend] - base;
    if (i < dv.N) {
        int4 T;
        Stamp st;
        load_eval<kRep>(dv, P, s_cards, s_railx, i, T, st);
        const int tc[4] = {T.x, T.y, T.z, T.w};
        int o = gk.off[i] - base;
#pragma unroll
        for (int p = 0; p < NPAIR; p++)
            if (tc[pair_row(p)] >= 0 && tc[pair_col(p)] >= 0) s_buf[o++] = st.y[p];
#pragma unroll
        for (int a = 0; a < 4; a++)
            if (tc[a] >= 0) s_buf[o++] = st.j[a];
    }
    __syncthreads();
    for (int k = threadIdx.x; k < total; k += blockDim.x) gk.buf[base + k] = s_buf[k];
}

__global__ void __launch_bounds__(kBlock) k_gather_reduce(GatherK gk, CallK P, int64_t n_light_blocks)
{
    if (blockIdx.x < n_light_blocks) {
        const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (t >= gk.n_targets) return;
        const int32_t b0 = gk.tptr[t], b1 = gk.tptr[t + 1];
        if (b0 == b1) return;
        double s = 0.0;
        for (int32_t k = b0; k < b1; k++) s += gk.buf[__ldg(gk.tidx + k)];
        if (t < gk.nnz) P.A[t] += s;
        else P.b[t - gk.nnz] += s;
        return;
    }
    // heavy chunk: fixed-shape block reduction
    __shared__ double s_w[kBlock / 32];
    const int64_t c = blockIdx.x - n_light_blocks;
    const int32_t b0 = gk.chunk_beg[c], b1 = gk.chunk_beg[c + 1];
    double v = 0.0;
    for (int32_t k = b0 + threadIdx.x; k < b1; k += blockDim.x) v += gk.buf[__ldg(gk.hidx + k)];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += s_w[w];
        gk.chunk_part[c] = t;
    }
}

// ---------------------------------------------------------------------------
// GATHER, target-ordered (form 1): the evaluation stores each contribution
// straight at its place in its target's list (scattered stores, fire-and-
// forget), so the reduction streams the buffer: a thread per target sums its
// contiguous list in list order (neighbouring threads read neighbouring lists,
// so a warp's loads share cache lines; deterministic).  Heavy lists
// (> kHeavyLen) are chunk-reduced from their contiguous ranges.  (A warp-
// shuffle segmented scan over 32 targets measured 1.4x slower: the lists are
// short, profiles/r01_f_tile_ab.md.)
// ---------------------------------------------------------------------------
template <bool kRep>
__global__ void __launch_bounds__(kBlock) k_gather_eval_t(DevK dv, GatherK gk, CallK P)
{
    __shared__ CardK s_cards[EES_MAX_MODELS];
    __shared__ double s_railx[EES_MAX_RAILS];
    load_call_smem(P, s_cards, s_railx);
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= dv.N) return;
    int32_t pos[16];
#pragma unroll
    for (int p = 0; p < 16; p++) pos[p] = __ldg(gk.tpos + (int64_t)p * dv.N + i);
    int4 T;
    Stamp st;
    load_eval<kRep>(dv, P, s_cards, s_railx, i, T, st);
#pragma unroll
    for (int p = 0; p < NPAIR; p++)
        if (pos[p] >= 0) gk.tbuf[pos[p]] = st.y[p];
#pragma unroll
    for (int a = 0; a < 4; a++)
        if (pos[NPAIR + a] >= 0) gk.tbuf[pos[NPAIR + a]] = st.j[a];
}

__global__ void __launch_bounds__(kBlock) k_gather_reduce_t(GatherK gk, CallK P, int64_t n_light_blocks)
{
    if (blockIdx.x < n_light_blocks) {
        // thread per target over its contiguous list (neighbouring threads
        // read neighbouring lists: the warp's loads share cache lines)
        const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (t >= gk.n_targets) return;
        const int32_t b0 = gk.tptr[t], b1 = gk.tptr[t + 1];
        if (b0 == b1) return;
        double s = 0.0;
        int32_t k = b0;
        for (; k + 4 <= b1; k += 4) {
            const double a = gk.tbuf[k], b = gk.tbuf[k + 1], c = gk.tbuf[k + 2], d = gk.tbuf[k + 3];
            s += a;
            s += b;
            s += c;
            s += d;
        }
        for (; k < b1; k++) s += gk.tbuf[k];
        if (t < gk.nnz) P.A[t] += s;
        else P.b[t - gk.nnz] += s;
        return;
    }
    // heavy chunk: fixed-shape block reduction over a contiguous range
    __shared__ double s_w[kBlock / 32];
    const int64_t c = blockIdx.x - n_light_blocks;
    const int64_t b0 = gk.heavy_base + gk.chunk_beg[c], b1 = gk.heavy_base + gk.chunk_beg[c + 1];
    double v = 0.0;
    for (int64_t k = b0 + threadIdx.x; k < b1; k += blockDim.x) v += gk.tbuf[k];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += s_w[w];
        gk.chunk_part[c] = t;
    }
}

__global__ void k_gather_heavy(GatherK gk, CallK P)
{
    const int h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= gk.n_heavy) return;
    double s = 0.0;
    for (int32_t c = gk.heavy_chunk[h]; c < gk.heavy_chunk[h + 1]; c++) s += gk.chunk_part[c];
    const int64_t t = gk.heavy_target[h];
    if (t < gk.nnz) P.A[t] += s;
    else P.b[t - gk.nnz] += s;
}

// ---------------------------------------------------------------------------
// COLOR under the degree-threshold hybrid rule: one
// launch per colour; targets no two FETs of a colour share get a plain RMW,
// side targets (heavy x heavy entries, heavy b rows with several writers) get
// their contribution stored in its own scratch slot.  After the last colour,
// k_side_chunks sums each chunk of a side target's slots (fixed tree) and
// k_side_apply adds the chunk sums of each target in chunk order.
// ---------------------------------------------------------------------------
template <bool kRep>
__global__ void __launch_bounds__(kBlock) k_color_h(DevK dv, CallK P, int64_t begin, int64_t count,
                                                    double *side)
{
    __shared__ CardK s_cards[EES_MAX_MODELS];
    for (int k = threadIdx.x; k < P.n_models; k += blockDim.x) s_cards[k] = P.cards[k];
    __syncthreads();
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= count) return;
    const int64_t i = begin + q;
    int32_t slot[NPAIR + 4];
#pragma unroll
    for (int p = 0; p < NPAIR + 4; p++) slot[p] = __ldg(dv.slot + (int64_t)p * dv.N + i);
    const int4 T = __ldg(dv.term + i);
    const double beta = __ldg(dv.beta + i);
    const double a0 = __ldg(dv.v0 + i), a1 = __ldg(dv.v0 + dv.N + i), a2 = __ldg(dv.v0 + 2 * dv.N + i);
    const int m = __ldg(dv.model + i);
    const double VD = T.x >= 0 ? __ldg(P.x + T.x) : 0.0;
    const double VG = T.y >= 0 ? __ldg(P.x + T.y) : 0.0;
    const double VS = T.z >= 0 ? __ldg(P.x + T.z) : 0.0;
    Stamp st;
    eval_fet<kRep>(s_cards[m], beta, P.gmin, VD, VG, VS, a0, a1, a2, st, P.work);
#pragma unroll
    for (int p = 0; p < NPAIR; p++) {
        if (slot[p] >= 0) P.A[slot[p]] += st.y[p];
        else if (slot[p] <= -2) side[-2 - slot[p]] = st.y[p];
    }
#pragma unroll
    for (int a = 0; a < 4; a++) {
        const int32_t k = slot[NPAIR + a];
        if (k >= 0) P.b[k] += st.j[a];
        else if (k <= -2) side[-2 - k] = st.j[a];
    }
}

// The paper's non-fused "Color" (Table I; NEXT-2): after k_gather_eval
// has written every FET's live contributions to the buffer (netlist order,
// off[i]), one launch per colour stamps them: thread q of colour c reads FET
// perm[q]'s contributions and applies the same codes as k_color_h.
__global__ void __launch_bounds__(kBlock) k_color_stamp(DevK dv16, GatherK gk, CallK P, const int32_t *perm,
                                                        int64_t begin, int64_t count, double *side)
{
    const int64_t q0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q0 >= count) return;
    const int64_t q = begin + q0;
    const int64_t i = __ldg(perm + q);
    const int4 T = __ldg(dv16.term + q);
    const int tc[4] = {T.x, T.y, T.z, T.w};
    int32_t o = __ldg(gk.off + i);
#pragma unroll
    for (int p = 0; p < NPAIR; p++)
        if (tc[pair_row(p)] >= 0 && tc[pair_col(p)] >= 0) {
            const double y = gk.buf[o++];
            const int32_t k = __ldg(dv16.slot + (int64_t)p * dv16.N + q);
            if (k >= 0) P.A[k] += y;
            else if (k <= -2) side[-2 - k] = y;
        }
#pragma unroll
    for (int a = 0; a < 4; a++)
        if (tc[a] >= 0) {
            const double j = gk.buf[o++];
            const int32_t k = __ldg(dv16.slot + (int64_t)(NPAIR + a) * dv16.N + q);
            if (k >= 0) P.b[k] += j;
            else if (k <= -2) side[-2 - k] = j;
        }
}

cudaError_t launch_color_stamp(const DevK &dv16, const GatherK &gk, const CallK &call, const int32_t *perm,
                               int64_t begin, int64_t count, double *side_buf, cudaStream_t st)
{
    if (count == 0) return cudaSuccess;
    k_color_stamp<<<(unsigned)((count + kBlock - 1) / kBlock), kBlock, 0, st>>>(dv16, gk, call, perm, begin,
                                                                                count, side_buf);
    return cudaPeekAtLastError();
}

__global__ void __launch_bounds__(kBlock) k_side_chunks(SideK sk)
{
    __shared__ double s_w[kBlock / 32];
    const int64_t lo = sk.chunk_lo[blockIdx.x], hi = sk.chunk_lo[blockIdx.x + 1];
    double v = 0.0;
    for (int64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) v += sk.buf[k];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += s_w[w];
        sk.chunk_part[blockIdx.x] = t;
    }
}

__global__ void k_side_apply(SideK sk, CallK P)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= sk.n_side) return;
    double t = 0.0;
    for (int32_t c = sk.side_chunk[s]; c < sk.side_chunk[s + 1]; c++) t += sk.chunk_part[c];
    const int64_t g = sk.side_gid[s];
    if (g < sk.nnz) P.A[g] += t;
    else P.b[g - sk.nnz] += t;
}

cudaError_t launch_color_h(const DevK &dv16, const CallK &call, int64_t begin, int64_t count,
                           double *side_buf, cudaStream_t st)
{
    if (count == 0) return cudaSuccess;
    const unsigned grid = (unsigned)((count + kBlock - 1) / kBlock);
    if (call.work > 1) k_color_h<true><<<grid, kBlock, 0, st>>>(dv16, call, begin, count, side_buf);
    else k_color_h<false><<<grid, kBlock, 0, st>>>(dv16, call, begin, count, side_buf);
    return cudaPeekAtLastError();
}

cudaError_t launch_side_sum(const SideK &sk, const CallK &call, cudaStream_t st, int *n_launches)
{
    *n_launches = 0;
    if (sk.n_side == 0) return cudaSuccess;
    k_side_chunks<<<sk.n_chunks, kBlock, 0, st>>>(sk);
    k_side_apply<<<(sk.n_side + 127) / 128, 128, 0, st>>>(sk, call);
    *n_launches = 2;
    return cudaPeekAtLastError();
}

// ---------------------------------------------------------------------------
// NEXT-4 state update (S:212 update_state, Fig. 1 accept branch): after a
// converged step at x, every FET's companion state becomes the converged
// branch voltages v_prev = (VG - VS, VG - VD, VD - VB) (physical frame), in
// every layout's copy of it.  k_accept_soa: one SoA layout (terms plain or
// rail-coded); k_accept_tile: the TILE item state (tile order, terms in the blobs).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock) k_accept_soa(const int4 *term, int64_t N, CallK P, double *v0)
{
    __shared__ double s_railx[EES_MAX_RAILS];
    for (int k = threadIdx.x; k < P.n_rail_nodes; k += blockDim.x) s_railx[k] = P.x[P.rail_node[k]];
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const int4 T = term[i];
        const double VD = volt(T.x, P.x, s_railx), VG = volt(T.y, P.x, s_railx);
        const double VS = volt(T.z, P.x, s_railx), VB = volt(T.w, P.x, s_railx);
        v0[i] = VG - VS;
        v0[N + i] = VG - VD;
        v0[2 * N + i] = VD - VB;
    }
}

__global__ void __launch_bounds__(kTileThreads) k_accept_tile(TileK tk, CallK P, double *item_v0)
{
    unsigned char *b = const_cast<unsigned char *>(tk.blob) + 16 * (size_t)tk.tdesc[blockIdx.x].x;
    const TileHdr *h = reinterpret_cast<const TileHdr *>(b);
    const int ni = h->n_items;
    const int4 *term = reinterpret_cast<const int4 *>(b + h->off_items);
    // form 1: v0[3] per item in the tile-order array; form 0: v0[3][ni] in the blob
    double *v0 = item_v0 ? item_v0 + (int64_t)blockIdx.x * kTileItems * 3
                         : reinterpret_cast<double *>(b + h->off_items + 16 * (size_t)ni) + ni;
    const int s1 = item_v0 ? 3 : 1, s2 = item_v0 ? 1 : ni;     // item stride, component stride
    for (int i = threadIdx.x; i < ni; i += blockDim.x) {
        const int4 T = term[i];
        const double VD = T.x >= 0 ? P.x[T.x] : 0.0, VG = T.y >= 0 ? P.x[T.y] : 0.0;
        const double VS = T.z >= 0 ? P.x[T.z] : 0.0, VB = T.w >= 0 ? P.x[T.w] : 0.0;
        v0[s1 * i] = VG - VS;
        v0[s1 * i + s2] = VG - VD;
        v0[s1 * i + 2 * s2] = VD - VB;
    }
}

cudaError_t launch_accept_soa(const int4 *term, int64_t N, const CallK &call, double *v0, cudaStream_t st)
{
    if (N == 0) return cudaSuccess;
    const int64_t grid = std::min<int64_t>((N + kBlock - 1) / kBlock, 148 * 16);
    k_accept_soa<<<(unsigned)grid, kBlock, 0, st>>>(term, N, call, v0);
    return cudaPeekAtLastError();
}

cudaError_t launch_accept_tile(const TileK &tk, const CallK &call, double *item_v0, cudaStream_t st)
{
    if (tk.n_tiles == 0) return cudaSuccess;
    k_accept_tile<<<tk.n_tiles, kTileThreads, 0, st>>>(tk, call, item_v0);
    return cudaPeekAtLastError();
}

// ---------------------------------------------------------------------------
// FP64 pipe peak: 8 independent FMA chains per thread, one
// resident wave; flops = 2 * 8 * iters per thread.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_fp64_peak(double *out, int iters, double a, double c)
{
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; k++) r[k] = threadIdx.x * 1e-9 + k;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) r[k] = fma(r[k], a, c);
    }
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 8; k++) t += r[k];
    if (t == 12345.678) out[0] = t;      // practically never: keeps the chains live
}

cudaError_t measure_fp64_peak(double *tflops)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double *out = nullptr;
    cudaError_t e = cudaMalloc(&out, sizeof(double));
    if (e != cudaSuccess) return e;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * 8, iters = 1 << 14;
    k_fp64_peak<<<grid, 256>>>(out, 64, 0.999999, 1e-7);       // warm-up
    cudaEventRecord(e0);
    k_fp64_peak<<<grid, 256>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    e = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    *tflops = 2.0 * 8.0 * iters * (double)grid * 256 / (ms * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return e == cudaSuccess ? cudaPeekAtLastError() : e;
}

// ---------------------------------------------------------------------------
// FP64 RED throughput: every thread issues `iters` REDs of
// 1.0 to a 64 MiB buffer -- its own address per iteration (mode 0, spread
// over L2 slices) or its warp's one address (mode 1, same-address).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_red_peak(double *buf, int64_t n, int iters, int mode)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    for (int it = 0; it < iters; it++) {
        const int64_t k = mode == 0 ? (t + (int64_t)it * T) % n : ((t >> 5) * 37 + it) % n;
        atomicAdd(buf + k, 1.0);
    }
}

cudaError_t measure_red_throughput(int mode, double *gops)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t n = (64ll << 20) / 8;
    double *buf = nullptr;
    cudaError_t e = cudaMalloc(&buf, n * sizeof(double));
    if (e != cudaSuccess) return e;
    cudaMemset(buf, 0, n * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * 8, iters = 64;
    k_red_peak<<<grid, 256>>>(buf, n, 4, mode);
    cudaEventRecord(e0);
    k_red_peak<<<grid, 256>>>(buf, n, iters, mode);
    cudaEventRecord(e1);
    e = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    *gops = (double)iters * grid * 256 / (ms * 1e-3) / 1e9;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    return e == cudaSuccess ? cudaPeekAtLastError() : e;
}

// ---------------------------------------------------------------------------
// Streaming probe (the size calibration of the HBM roofline):
// one launch reads `nr` 16-byte vectors of src and writes `nw` vectors of dst
// -- the read/write mix of one eval+stamp call's algorithmic bytes -- with
// 16-byte non-allocating loads, four in flight per thread, grid-stride over a
// grid of a whole number of waves.  The written values depend on the loads,
// so neither side can be dropped.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double2 ld_stream(const double2 *p)
{
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

__global__ void __launch_bounds__(256) k_stream_probe(const double2 *__restrict__ src, int64_t nr,
                                                      double2 *__restrict__ dst, int64_t nw, double *sink)
{
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = nr > nw ? nr : nw;
    double acc = 0.0;
    int64_t i = t0;
    for (; i + 3 * T < n; i += 4 * T) {
        double2 v[4];
#pragma unroll
        for (int k = 0; k < 4; k++) v[k] = i + k * T < nr ? ld_stream(src + i + k * T) : make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            acc += v[k].x + v[k].y;
            if (i + k * T < nw) dst[i + k * T] = make_double2(v[k].x + 1.0, v[k].y);
        }
    }
    for (; i < n; i += T) {
        const double2 v = i < nr ? ld_stream(src + i) : make_double2(0.0, 0.0);
        acc += v.x + v.y;
        if (i < nw) dst[i] = make_double2(v.x + 1.0, v.y);
    }
    if (acc == 12345.678) sink[0] = acc;      // practically never: keeps the loads live
}

cudaError_t launch_stream_probe(const void *src, int64_t read_bytes, void *dst, int64_t write_bytes,
                                double *sink, cudaStream_t st)
{
    int dev = 0, sms = 148, bps = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_stream_probe, 256, 0);
    const int64_t nr = read_bytes / 16, nw = write_bytes / 16;
    const int64_t want = ((nr > nw ? nr : nw) + 255) / 256;
    const int64_t grid = want < (int64_t)sms * (bps > 0 ? bps : 1) ? (want > 0 ? want : 1) : (int64_t)sms * (bps > 0 ? bps : 1);
    k_stream_probe<<<(unsigned)grid, 256, 0, st>>>(static_cast<const double2 *>(src), nr, static_cast<double2 *>(dst),
                                                   nw, sink);
    return cudaPeekAtLastError();
}

// ---------------------------------------------------------------------------
// Race instrument: per colour, count distinct-device writers
// of every non-rail A entry and b row.
// ---------------------------------------------------------------------------
__global__ void k_race_probe(DevK dv, const int32_t *perm, int64_t begin, int64_t count,
                             int32_t *cnt_a, int32_t *cnt_b)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= count) return;
    const int64_t i = perm[begin + q];
    int32_t slot[NPAIR];
#pragma unroll
    for (int p = 0; p < NPAIR; p++) slot[p] = dv.slot[(int64_t)p * dv.N + i];
#pragma unroll
    for (int p = 0; p < NPAIR; p++) {
        bool dup = false;
#pragma unroll
        for (int r = 0; r < p; r++) dup |= slot[r] == slot[p];
        if (slot[p] >= 0 && !dup) atomicAdd(cnt_a + slot[p], 1);
    }
    const int4 T = dv.term[i];
    const int tc[4] = {T.x, T.y, T.z, T.w};
#pragma unroll
    for (int a = 0; a < 4; a++) {
        bool dup = false;
#pragma unroll
        for (int r = 0; r < a; r++) dup |= tc[r] == tc[a];
        if (tc[a] >= 0 && !dup) atomicAdd(cnt_b + tc[a], 1);
    }
}

__global__ void k_count_conflicts(const int32_t *cnt, int64_t n, unsigned long long *out)
{
    unsigned long long local = 0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x)
        local += cnt[k] > 1;
    if (local) atomicAdd(out, local);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static size_t rail_smem(const CallK &P) { return sizeof(double) * (kBlock / 32) * P.n_rail_entries; }

int atomic_blocks_per_sm()
{
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_atomic<false, true>, kBlock,
                                                  sizeof(double) * (kBlock / 32) * kMaxRailEntries);
    return nb > 0 ? nb : 1;
}

cudaError_t launch_atomic(const DevK &dv, const CallK &call, int grid, bool agg, cudaStream_t st)
{
    if (dv.N == 0) return cudaSuccess;
    const size_t sm = rail_smem(call);
    if (call.work > 1) {
        if (agg) k_atomic<true, true><<<grid, kBlock, sm, st>>>(dv, call);
        else k_atomic<true, false><<<grid, kBlock, sm, st>>>(dv, call);
    } else {
        if (agg) k_atomic<false, true><<<grid, kBlock, sm, st>>>(dv, call);
        else k_atomic<false, false><<<grid, kBlock, sm, st>>>(dv, call);
    }
    return cudaPeekAtLastError();
}

// ---------------------------------------------------------------------------
// COLOR, persistent form (Table I "Color": one parallel region with a barrier
// between colours): one cooperative launch, grid.sync()
// between colours.  A FET's data, slots and x gather do not depend on earlier
// colours, so the first FET of colour c+1 is fetched before the barrier and
// only the A/b read-modify-write stays behind it.  Rail entries accumulate
// per warp across colours; block 0 sums the block parts in block order.
// ---------------------------------------------------------------------------
struct Fetched {
    int4 T;
    double beta, a0, a1, a2, VD, VG, VS;
    int m;
    int32_t slot[NPAIR];
};

__device__ __forceinline__ void fetch_dev(const DevK &dv, const CallK &P, const double *s_railx,
                                          int64_t i, bool valid, Fetched &f)
{
    if (!valid) {
        f.T = make_int4(-1, -1, -1, -1);
        return;
    }
    f.T = __ldg(dv.term + i);
    f.beta = __ldg(dv.beta + i);
    f.a0 = __ldg(dv.v0 + i);
    f.a1 = __ldg(dv.v0 + dv.N + i);
    f.a2 = __ldg(dv.v0 + 2 * dv.N + i);
    f.m = __ldg(dv.model + i);
#pragma unroll
    for (int p = 0; p < NPAIR; p++) f.slot[p] = __ldg(dv.slot + (int64_t)p * dv.N + i);
    f.VD = volt(f.T.x, P.x, s_railx);
    f.VG = volt(f.T.y, P.x, s_railx);
    f.VS = volt(f.T.z, P.x, s_railx);
}

template <bool kRep>
__global__ void __launch_bounds__(kBlock, 2) k_color_coop(DevK dv, CallK P, const int64_t *cptr,
                                                          int32_t C, double *partials)
{
    cg::grid_group grid = cg::this_grid();
    __shared__ CardK s_cards[EES_MAX_MODELS];
    __shared__ double s_railx[EES_MAX_RAILS];
    extern __shared__ double s_acc[];
    load_call_smem(P, s_cards, s_railx);
    const int nw = blockDim.x >> 5;
    for (int k = threadIdx.x; k < nw * P.n_rail_entries; k += blockDim.x) s_acc[k] = 0.0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t G = (int64_t)gridDim.x * blockDim.x;
    const int64_t wbase = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    Fetched cur;
    {
        const int64_t i = cptr[0] + wbase + lane;
        fetch_dev(dv, P, s_railx, i, C > 0 && i < cptr[1], cur);
    }
    for (int32_t c = 0; c < C; c++) {
        const int64_t end = cptr[c + 1];
        bool first = true;
        for (int64_t base = cptr[c] + wbase; base < end; base += G) {
            const int64_t i = base + lane;
            const bool valid = i < end;
            Fetched f;
            if (first) f = cur;
            else fetch_dev(dv, P, s_railx, i, valid, f);
            first = false;
            Stamp st;
            int tc[4] = {-1, -1, -1, -1};
            if (valid) {
                eval_fet<kRep>(s_cards[f.m], f.beta, P.gmin, f.VD, f.VG, f.VS, f.a0, f.a1, f.a2, st, P.work);
                tc[0] = f.T.x; tc[1] = f.T.y; tc[2] = f.T.z; tc[3] = f.T.w;
                merge_source_bulk(f.T, st, f.slot, tc);
#pragma unroll
                for (int p = 0; p < NPAIR; p++)
                    if (f.slot[p] >= 0) P.A[f.slot[p]] += st.y[p];
#pragma unroll
                for (int a = 0; a < 4; a++)
                    if (tc[a] >= 0) P.b[tc[a]] += st.j[a];
            } else {
#pragma unroll
                for (int p = 0; p < NPAIR; p++) f.slot[p] = -1;
            }
            if (P.n_rail_entries) rail_accumulate(P, f.slot, tc, st, valid, s_acc);
        }
        if (c + 1 < C) {
            const int64_t i = cptr[c + 1] + wbase + lane;
            fetch_dev(dv, P, s_railx, i, i < cptr[c + 2], cur);
        }
        grid.sync();
    }
    if (P.n_rail_entries) {
        __syncthreads();
        for (int e = threadIdx.x; e < P.n_rail_entries; e += blockDim.x) {
            double v = 0.0;
            for (int w = 0; w < nw; w++) v += s_acc[w * P.n_rail_entries + e];
            partials[(int64_t)blockIdx.x * P.n_rail_entries + e] = v;
        }
        __threadfence();
        grid.sync();
        if (blockIdx.x == 0) {
            const int warp = threadIdx.x >> 5;
            for (int e = warp; e < P.n_rail_entries; e += nw) {
                double v = 0.0;
                for (int64_t k = lane; k < gridDim.x; k += 32) v += __ldcg(partials + k * P.n_rail_entries + e);
                v = warp_sum(v);
                if (lane == 0) {
                    double *dst = e < P.n_rail_a ? P.A + P.rail_target[e] : P.b + P.rail_target[e];
                    *dst += v;
                }
            }
        }
    }
}

int color_coop_blocks_per_sm()
{
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_color_coop<true>, kBlock,
                                                  sizeof(double) * (kBlock / 32) * kMaxRailEntries);
    return nb;
}

cudaError_t launch_color_coop(const DevK &dv, const CallK &call, const int64_t *cptr_dev, int32_t C,
                              double *partials, int grid, cudaStream_t st)
{
    if (dv.N == 0 || C == 0) return cudaSuccess;
    DevK a0 = dv;
    CallK a1 = call;
    const int64_t *a2 = cptr_dev;
    int32_t a3 = C;
    double *a4 = partials;
    void *args[] = {&a0, &a1, &a2, &a3, &a4};
    const void *fn = call.work > 1 ? (const void *)k_color_coop<true> : (const void *)k_color_coop<false>;
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kBlock), args,
                                       rail_smem(call), st);
}

cudaError_t launch_color(const DevK &dv, const CallK &call, int64_t begin, int64_t count,
                         double *partials, cudaStream_t st)
{
    if (count == 0) return cudaSuccess;
    const int64_t grid = (count + kBlock - 1) / kBlock;
    if (call.work > 1) k_color<true><<<(unsigned)grid, kBlock, rail_smem(call), st>>>(dv, call, begin, count, partials);
    else k_color<false><<<(unsigned)grid, kBlock, rail_smem(call), st>>>(dv, call, begin, count, partials);
    return cudaPeekAtLastError();
}

cudaError_t launch_rail_finalize(const CallK &call, const double *partials, int64_t n_blocks,
                                 cudaStream_t st)
{
    if (call.n_rail_entries == 0 || n_blocks == 0) return cudaSuccess;
    k_rail_final<<<call.n_rail_entries, kBlock, 0, st>>>(call, partials, n_blocks);
    return cudaPeekAtLastError();
}

cudaError_t launch_gather_phase(const DevK &dv, const GatherK &gk, const CallK &call, cudaStream_t st,
                                int phase, int *n_launches)
{
    *n_launches = 0;
    if (dv.N == 0) return cudaSuccess;
    if (phase == 0) {
        const int64_t grid = (dv.N + kBlock - 1) / kBlock;
        if (gk.form == 1) {
            if (call.work > 1) k_gather_eval_t<true><<<(unsigned)grid, kBlock, 0, st>>>(dv, gk, call);
            else k_gather_eval_t<false><<<(unsigned)grid, kBlock, 0, st>>>(dv, gk, call);
        } else {
            if (call.work > 1) k_gather_eval<true><<<(unsigned)grid, kBlock, 0, st>>>(dv, gk, call);
            else k_gather_eval<false><<<(unsigned)grid, kBlock, 0, st>>>(dv, gk, call);
        }
        *n_launches = 1;
    } else if (phase == 1) {
        const int64_t light = (gk.n_targets + kBlock - 1) / kBlock;
        if (gk.form == 1) k_gather_reduce_t<<<(unsigned)(light + gk.n_chunks), kBlock, 0, st>>>(gk, call, light);
        else k_gather_reduce<<<(unsigned)(light + gk.n_chunks), kBlock, 0, st>>>(gk, call, light);
        *n_launches = 1;
    } else if (gk.n_heavy) {
        k_gather_heavy<<<(gk.n_heavy + 127) / 128, 128, 0, st>>>(gk, call);
        *n_launches = 1;
    }
    return cudaPeekAtLastError();
}

// COLOR_BUF's compute phase: the compact per-device ContributionBuffer
cudaError_t launch_eval_compact(const DevK &dv, const GatherK &gk, const CallK &call, cudaStream_t st)
{
    if (dv.N == 0) return cudaSuccess;
    const int64_t grid = (dv.N + kBlock - 1) / kBlock;
    if (call.work > 1) k_gather_eval<true><<<(unsigned)grid, kBlock, 0, st>>>(dv, gk, call);
    else k_gather_eval<false><<<(unsigned)grid, kBlock, 0, st>>>(dv, gk, call);
    return cudaPeekAtLastError();
}

cudaError_t launch_gather(const DevK &dv, const GatherK &gk, const CallK &call, cudaStream_t st,
                          int *n_launches)
{
    int total = 0;
    for (int ph = 0; ph < 3; ph++) {
        int k = 0;
        cudaError_t e = launch_gather_phase(dv, gk, call, st, ph, &k);
        total += k;
        if (e != cudaSuccess) return e;
    }
    if (n_launches) *n_launches = total;
    return cudaSuccess;
}

cudaError_t launch_race_probe(const DevK &dv, const int32_t *perm, int64_t begin, int64_t count,
                              int32_t *cnt_a, int32_t *cnt_b, cudaStream_t st)
{
    if (count == 0) return cudaSuccess;
    k_race_probe<<<(unsigned)((count + kBlock - 1) / kBlock), kBlock, 0, st>>>(dv, perm, begin,
                                                                               count, cnt_a, cnt_b);
    return cudaPeekAtLastError();
}

cudaError_t launch_count_conflicts(const int32_t *cnt, int64_t n, unsigned long long *out,
                                   cudaStream_t st)
{
    if (n == 0) return cudaSuccess;
    k_count_conflicts<<<296, kBlock, 0, st>>>(cnt, n, out);
    return cudaPeekAtLastError();
}

// ---------------------------------------------------------------------------
// TILE (deterministic, one launch; +1 when side targets are many): persistent
// CTAs walk the row tiles blockIdx.x, +gridDim.x, ... (layout and the
// ownership rule in ees_internal.h).  Per tile t:
//   eval    each thread evaluates one item (FET copy) and stores its 16
//           contributions in shared memory (one of tile_bufs(form) slot
//           buffers); then it gathers the item data and x values of tile t+G,
//           whose blob the TMA brought in a tile earlier, so their latency
//           hides behind the reduction;
//   B1      contributions complete, and every thread is done with tile t-G ->
//           thread 0 refills tile t-G's stage with tile t+(kStages-1)G;
//   reduce  per length class, each thread sums whole targets (fixed-length
//           unrolled loops, list order) and adds each sum to its destination
//           with one RED: A and b entries owned by this tile receive exactly
//           one addition each, so the result equals a plain read-modify-write
//           and no old value is loaded by the SM.  Long targets: one warp
//           each (lane-strided, fixed shuffle tree).  Side targets: the part
//           goes to its slot (plain store) or, for the hot ones (rails), into
//           the CTA's running sum in shared memory (tile order);
//   (B0)    with one slot buffer, a barrier before the next evaluation.
// After the last tile, hot partials are stored per CTA, and side targets are
// summed in part order by the warps of the whole grid after a grid barrier.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// bulk L2 prefetch of a tile's CSR block of A (its REDs then find the sectors in L2)
__device__ __forceinline__ void l2_prefetch_block(const double *A, int32_t lo, int32_t n)
{
#if EES_A_PREFETCH
    if (n <= 0) return;
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(A + lo) & ~(uintptr_t)15;
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(A + lo + n) + 15) & ~(uintptr_t)15;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
#endif
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "EES_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra EES_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

template <int kForm>
constexpr size_t tile_smem()
{
    return sizeof(double) * sc_slots(kForm) * tile_bufs(kForm) + tile_stages(kForm) * (size_t)stage_max(kForm);
}

// What a thread gathers from global memory one tile ahead: its item's node
// voltages and (form 1) the item data from the tile-order arrays.
struct TileRegs {
    double VD, VG, VS;
    double beta, v0a, v0b, v0c;
    int model;
    int tied;                  // source tied to bulk (terms z == w, not ground)
};

template <int kForm>
__device__ __forceinline__ void tile_gather(const unsigned char *blob, int32_t tile, const TileK &tk,
                                            const CallK &P, TileRegs &R)
{
    const int tid = threadIdx.x;
    const TileHdr *h = reinterpret_cast<const TileHdr *>(blob);
    R.VD = R.VG = R.VS = 0.0;
    R.tied = 0;
    if (tid < h->n_items) {
        const bool full = tid < h->n_full;            // gate-row items: caps only (no x, no beta)
        if (kForm == 1) {
            const int64_t q = (int64_t)tile * kTileItems + tid;
            R.v0a = __ldg(tk.item_v0 + 3 * q);
            R.v0b = __ldg(tk.item_v0 + 3 * q + 1);
            R.model = __ldg(tk.item_model + q);
            if (full) {
                R.beta = __ldg(tk.item_beta + q);
                R.v0c = __ldg(tk.item_v0 + 3 * q + 2);
            }
        }
        if (full) {
            const int4 T = reinterpret_cast<const int4 *>(blob + h->off_items)[tid];
            R.VD = T.x >= 0 ? __ldg(P.x + T.x) : 0.0;
            R.VG = T.y >= 0 ? __ldg(P.x + T.y) : 0.0;
            R.VS = T.z >= 0 ? __ldg(P.x + T.z) : 0.0;
            R.tied = T.z == T.w && T.z != -1;
        }
    }
}

// FP64 reduction without a result (RED.E.ADD.F64): fire and forget
__device__ __forceinline__ void red_add(double *p, double v)
{
#ifdef EES_DIAG_STORE            // diagnostic A/B only (wrong sums): a plain store instead
    *p = v;
#else
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
#endif
}

// Output of the reduction: the tile's destination pointers (one per base,
// ees_internal.h: A + g or b + g - nnz, set per tile from the staged head).
struct TileOut {
    double *A, *Bm;            // A, and b - nnz (so that b row r is Bm + nnz + r)
    int32_t nnz;
    uint32_t bptr;             // shared-memory address of the tile's [kTileBases] pointers
};

// destination d: pointer base[d >> 28] plus d's low 28 bits
__device__ __forceinline__ double *tile_dst(const TileOut &o, uint32_t d)
{
    uint64_t p, a;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(p) : "r"(o.bptr + ((d >> 25) & 0x78u)));
    asm("mad.wide.u32 %0, %1, 8, %2;" : "=l"(a) : "r"(d & 0x0FFFFFFFu), "l"(p));   // one IMAD.WIDE.U32
    return reinterpret_cast<double *>(a);
}

// RED under a predicate (no branch around it)
__device__ __forceinline__ void red_add_if(uint32_t pred, double *p, double v)
{
#ifdef EES_DIAG_STORE
    if (pred) *p = v;
#else
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q red.global.add.f64 [%0], %1;\n}" ::"l"(p), "d"(v),
                 "r"(pred)
                 : "memory");
#endif
}

__device__ __forceinline__ double sc_ld(const unsigned char *sc, uint32_t byte)
{
    return *reinterpret_cast<const double *>(sc + byte);
}

__device__ __forceinline__ double lds_f64(uint32_t a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ uint32_t lds_u16(uint32_t a)
{
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}

// A side target's part for this tile: its part slot (plain store) or the
// CTA's running sum of a hot target (one writer per tile, tiles in order).
__device__ __forceinline__ void side_put(const SideEnt *sents, uint32_t e, const TileK &tk, double *s_hot, double v)
{
    const SideEnt se = sents[e];
    if (se.slot >= 0) tk.part[se.slot] = v;
    else s_hot[-1 - se.slot] += v;
}

// A group class (owned targets longer than kOpMax, group size gs =
// cls_group(L)): a group of gs lanes per target, lane j summing the target's
// entries j, j+gs, ... in four fixed partial sums, then a fixed xor shuffle
// tree within the group; the group's first lane adds the sum (one RED).  All
// lanes of a warp run the same number of iterations (shuffles need them).
__device__ __forceinline__ void tile_cls_group(const TileCls c, int r, const uint32_t *dst, const uint32_t *meta,
                                               const uint16_t *ent, const unsigned char *sc, const TileOut &o,
                                               const SideEnt *sents, const TileK &tk, double *s_hot)
{
    const int n = c.n, lg = c.lg, gs = 1 << lg;
    const int lgn = kLogTileThreads - lg;                 // log2(kTileThreads / gs)
    const int gi = r >> lg, lj = r & (gs - 1);
    const int k0 = (gi - (int)c.rot) & ((1 << lgn) - 1);
    const int mine = k0 < n ? ((n - 1 - k0) >> lgn) + 1 : 0;
    const int iters = __reduce_max_sync(0xffffffffu, mine);
    for (int it = 0; it < iters; it++) {
        const int k = k0 + (it << lgn);
        const bool act = k < n;
        double s = 0.0;
        if (act) {
            // the lane's entries lj, lj+gs, ...: four partial sums (fixed
            // order, four loads in flight), combined as (s0 + s1) + (s2 + s3)
            const uint32_t m = meta[k];
            const uint16_t *e = ent + (m & 0xFFFFu);
            const int L = (int)(m >> 16);
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int p = lj;
            for (; p + 3 * gs < L; p += 4 * gs) {
                s0 += sc_ld(sc, e[p]);
                s1 += sc_ld(sc, e[p + gs]);
                s2 += sc_ld(sc, e[p + 2 * gs]);
                s3 += sc_ld(sc, e[p + 3 * gs]);
            }
            for (; p < L; p += gs) s0 += sc_ld(sc, e[p]);
            s = (s0 + s1) + (s2 + s3);
        }
        for (int off = gs >> 1; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (act && lj == 0) {
            if (c.side) side_put(sents, dst[k], tk, s_hot, s);    // (warp-uniform)
            else red_add(tile_dst(o, dst[k]), s);
        }
    }
}

// Fixed-order sum of one side target's parts by a whole warp (fixed lane
// stride, eight loads in flight per lane, shuffle tree).
__device__ __forceinline__ void side_finish(const TileK &tk, const CallK &P, int32_t sid, int lane)
{
    const int32_t q0 = __ldg(tk.sd_part + 2 * sid), q1 = __ldg(tk.sd_part + 2 * sid + 1);
    const int32_t g = __ldg(tk.sd_gid + sid);
    double *dst = g < tk.nnz ? P.A + g : P.b + (g - tk.nnz);
    const double pre = lane == 0 ? *dst : 0.0;
    double u = 0.0;
    for (int32_t qb = q0; qb < q1; qb += 256) {
        double a[8];
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const int32_t q = qb + r * 32 + lane;
            a[r] = q < q1 ? __ldcg(tk.part + q) : 0.0;
        }
#pragma unroll
        for (int r = 0; r < 8; r++) u += a[r];
    }
    u = warp_sum(u);
    if (lane == 0) *dst = pre + u;
}

__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// slots: 0 start, 1 first blob staged, 2+2*it evaluated (next tile's gathers
// issued), 3+2*it reduced and written (while below kTraceSlots-2),
// kTraceSlots-2 side ticket, kTraceSlots-1 end
#define TILE_TRACE_AT(slot, limit)                                                  \
    do {                                                                            \
        if (kTrace && tid == 0 && (slot) < (limit))                                 \
            tk.trace[(size_t)blockIdx.x * kTraceSlots + (slot)] = globaltimer();    \
    } while (0)
#define TILE_TRACE(slot) TILE_TRACE_AT(slot, kTraceSlots - 2)
#define TILE_TRACE_TAIL(slot) TILE_TRACE_AT(slot, kTraceSlots)

// Evaluate item `it` of a staged tile and store its 16 contributions at
// slots p*kTileItems + it of the slot buffer (ees_internal.h).
__device__ __forceinline__ void sts_f64(uint32_t a, double v)
{
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

// form 1: item it's 16 contribution positions in the staged program
// (ees_internal.h: [2][ni] uint4, two conflict-free LDS.128)
__device__ __forceinline__ void tile_pos(const unsigned char *blob, int it, uint4 &pa, uint4 &pb)
{
    const TileHdr *h = reinterpret_cast<const TileHdr *>(blob);
    const unsigned char *prog = blob + h->head_bytes;
    const uint4 *pp = reinterpret_cast<const uint4 *>(prog + reinterpret_cast<const ProgHdr5 *>(prog)->off_pos);
    pa = pp[it];
    pb = pp[h->n_items + it];
}

template <bool kRep, int kForm>
__device__ __forceinline__ void tile_eval_item(const unsigned char *blob, const TileRegs &cur, int it, double *scd,
                                               const CardK *s_cards, const CallK &P)
{
    const TileHdr *h = reinterpret_cast<const TileHdr *>(blob);
    const int ni = h->n_items;
    if (it >= h->n_full) {
        // gate-row item: only GD, GG, GS and J[G] are listed -- the BE
        // companions of cgs (G,S) and cgd (G,D), eval_fet1's gate row
        const CardK &cd = s_cards[kForm == 1 ? cur.model : blob[h->off_items + 48 * ni + it]];
        const double v0gs = kForm == 1 ? cur.v0a : reinterpret_cast<const double *>(blob + h->off_items + 24 * ni)[it];
        const double v0gd = kForm == 1 ? cur.v0b : reinterpret_cast<const double *>(blob + h->off_items + 32 * ni)[it];
        const double g1 = cd.gcgs, g2 = cd.gcgd;
        if (kForm == 1) {
            const uint32_t sc32 = smem_u32(scd);
            uint4 pa, pb;
            tile_pos(blob, it, pa, pb);
            const uint32_t w[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
            auto at = [&](int q) { return sc32 + (q & 1 ? w[q >> 1] >> 16 : w[q >> 1] & 0xFFFFu); };
            sts_f64(at(GD), -g2);
            sts_f64(at(GG), g1 + g2);
            sts_f64(at(GS), -g1);
            sts_f64(at(NPAIR + 1), g1 * v0gs + g2 * v0gd);
            return;
        }
        scd[GD * kTileItems + it] = -g2;
        scd[GG * kTileItems + it] = g1 + g2;
        scd[GS * kTileItems + it] = -g1;
        scd[(NPAIR + 1) * kTileItems + it] = g1 * v0gs + g2 * v0gd;
        return;
    }
    Stamp st;
    if (kForm == 1) {
        eval_fet<kRep>(s_cards[cur.model], cur.beta, P.gmin, cur.VD, cur.VG, cur.VS, cur.v0a, cur.v0b, cur.v0c, st,
                       P.work);
    } else {
        const double *bt = reinterpret_cast<const double *>(blob + h->off_items + 16 * ni);
        const uint8_t *md = blob + h->off_items + 48 * ni;
        eval_fet<kRep>(s_cards[md[it]], bt[it], P.gmin, cur.VD, cur.VG, cur.VS, bt[ni + it], bt[2 * ni + it],
                       bt[3 * ni + it], st, P.work);
    }
    if (cur.tied) {                       // source tied to bulk: one entry each (ees_internal.h)
        st.y[DS] += st.y[DB];
        st.y[SD] += st.y[BD];
        st.y[SS] += st.y[BB];
        st.j[2] += st.j[3];
    }
    if constexpr (kForm == 1) {           // v5: each contribution straight to its pair slot
        const uint32_t sc32 = smem_u32(scd);
        uint4 pa, pb;
        tile_pos(blob, it, pa, pb);
        const uint32_t w[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
#pragma unroll
        for (int p = 0; p < 16; p++) {
            const uint32_t off = p & 1 ? w[p >> 1] >> 16 : w[p >> 1] & 0xFFFFu;
            sts_f64(sc32 + off, p < NPAIR ? st.y[p] : st.j[p - NPAIR]);
        }
    } else {
#pragma unroll
        for (int p = 0; p < NPAIR; p++) scd[p * kTileItems + it] = st.y[p];
#pragma unroll
        for (int a = 0; a < 4; a++) scd[(NPAIR + a) * kTileItems + it] = st.j[a];
    }
}

// TILE v5 (form 1, ees_internal.h ProgHdr5): thread r's pair of row s is
// the 16 bytes at (s * kTileItems + r) * 16 of the slot buffer; it reads
// them (one LDS.128), adds both halves to its running sum (one where the pad
// bit marks an odd target's last pair) and, where the row's emit bit is set,
// adds the sum to its next destination (one RED; a side piece's sum is its part).
__device__ __forceinline__ void tile_grp5(const TileCls c, int r, const uint32_t *dst, const uint32_t *meta,
                                          uint32_t g32, const TileOut &o)
{
    const int n = c.n, lg = c.lg, gs = 1 << lg;
    const int lgn = kLogTileThreads - lg;
    const int gi = r >> lg, lj = r & (gs - 1);
    const int k0 = (gi - (int)c.rot) & ((1 << lgn) - 1);
    const int mine = k0 < n ? ((n - 1 - k0) >> lgn) + 1 : 0;
    const int iters = __reduce_max_sync(0xffffffffu, mine);
    for (int it = 0; it < iters; it++) {
        const int k = k0 + (it << lgn);
        const bool act = k < n;
        double s = 0.0;
        if (act) {
            const uint32_t m = meta[k];
            const uint32_t e = g32 + 8 * (m & 0xFFFFu);       // the target's first entry
            const int L = (int)(m >> 16);
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int p = lj;
            auto take = [&](int q) { return lds_f64(e + 8 * q); };
            for (; p + 3 * gs < L; p += 4 * gs) {
                s0 += take(p);
                s1 += take(p + gs);
                s2 += take(p + 2 * gs);
                s3 += take(p + 3 * gs);
            }
            for (; p < L; p += gs) s0 += take(p);
            s = (s0 + s1) + (s2 + s3);
        }
        for (int off = gs >> 1; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (act && lj == 0) red_add(tile_dst(o, dst[k]), s);
    }
}

__device__ __forceinline__ void tile_reduce5(const unsigned char *blob, const unsigned char *sc, int r,
                                             const TileOut &out, const TileK &tk, double *s_hot)
{
#ifdef EES_DIAG_NOREDUCE
    return;
#endif
    const TileHdr *h = reinterpret_cast<const TileHdr *>(blob);
    const unsigned char *prog = blob + h->head_bytes;
    const ProgHdr5 *ph = reinterpret_cast<const ProgHdr5 *>(prog);
    const uint32_t p32 = smem_u32(prog), sc32 = smem_u32(sc);
    {
        const uint32_t w = lds_u32(p32 + ph->off_oseq + 4 * r);
        const uint32_t em = (w >> kSeqEmit) & 0x7Fu;
        const int ns = em ? 32 - __clz(em) : 0;                // rows end with the last emit
        uint32_t dst = p32 + ph->off_odst + 4 * (w & ((1u << kSeqStartBits) - 1));
        const SideEnt *sents = reinterpret_cast<const SideEnt *>(blob + h->off_side);
        const uint32_t a = sc32 + 16 * r;
        double acc = 0.0;
#pragma unroll
        for (int st = 0; st < kScRows; st++) {
            if (st < ns) {
                double v0, v1;
                const uint32_t q = a + st * 16 * kTileItems;
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v0), "=d"(v1) : "r"(q));
                acc += v0;
                if (!((w >> (kSeqPad + st)) & 1u)) acc += v1;   // an odd target's last pair: one half
                if ((em >> st) & 1u) {                           // the target is complete
                    const uint32_t d = lds_u32(dst);
                    dst += 4;
                    if ((w >> (kSeqSide + st)) & 1u) side_put(sents, d, tk, s_hot, acc);
                    else red_add(tile_dst(out, d), acc);
                    acc = 0.0;
                }
            }
        }
    }
    const int ncl = ph->n_cls;
    if (ncl) {
        const TileCls *cls = reinterpret_cast<const TileCls *>(prog + ph->off_cls);
        const uint32_t *dst = reinterpret_cast<const uint32_t *>(prog + ph->off_dst);
        const uint32_t *meta = reinterpret_cast<const uint32_t *>(prog + ph->off_meta);
        for (int ci = 0; ci < ncl; ci++) {
            const TileCls c = cls[ci];
            tile_grp5(c, r, dst + c.dst, meta + c.meta, sc32 + 8 * ph->gbase, out);
        }
    }
}

// The reduction program of one staged tile, run by kTileThreads threads with
// thread index r (0 .. kTileThreads-1; whole warps): the owned op stream,
// the group classes, then the side op stream (ees_internal.h).
__device__ __forceinline__ void tile_reduce(const unsigned char *blob, const unsigned char *sc, int r,
                                            const TileOut &out, const TileK &tk, double *s_hot)
{
#ifdef EES_DIAG_NOREDUCE         // diagnostic A/B only (no stamps): evaluation alone
    return;
#endif
    const TileHdr *h = reinterpret_cast<const TileHdr *>(blob);
    const unsigned char *prog = blob + h->head_bytes;
    const ProgHdr *ph = reinterpret_cast<const ProgHdr *>(prog);
    {
        // owned op stream: pair-ops of this thread's sequence, one RED per target
        // (the last pair of a sequence always emits, so the destination read
        // ahead of an emit is always the sequence's own)
        if (r < ph->n_oseq) {
            const uint32_t p32 = smem_u32(prog), sc32 = smem_u32(sc);
            const uint32_t sw = lds_u16(p32 + ph->off_ostart + 2 * r);
            const int ns = (int)(sw >> kSeqStartBits);
            uint32_t row = p32 + ph->off_orow;                               // u16 row offsets
            const uint32_t ops = p32 + ph->off_ops + 4 * r;
            uint32_t dst = p32 + ph->off_odst + 4 * (sw & ((1u << kSeqStartBits) - 1));
            double acc = 0.0;
#pragma unroll 2
            for (int st = 0; st < ns; st++, row += 2) {
                const uint32_t w = lds_u32(ops + 4 * lds_u16(row));
                acc += lds_f64(sc32 + (w & 0xFFF8u));
                acc += lds_f64(sc32 + (w >> 16));
                const uint32_t em = w & kEmitBit;              // the target is complete
                const uint32_t d = lds_u32(dst);
                dst += em;                                     // kEmitBit = 4: one destination
                red_add_if(em, tile_dst(out, d), acc);
                acc = em ? 0.0 : acc;
            }
        }
    }
    {
        // group classes (targets longer than kOpMax)
        const int ncl = ph->n_cls;
        const TileCls *cls = reinterpret_cast<const TileCls *>(prog + ph->off_cls);
        const uint32_t *dst = reinterpret_cast<const uint32_t *>(prog + ph->off_dst);
        const uint32_t *meta = reinterpret_cast<const uint32_t *>(prog + ph->off_meta);
        const uint16_t *ent = reinterpret_cast<const uint16_t *>(prog + ph->off_ent);
        const SideEnt *sents = reinterpret_cast<const SideEnt *>(blob + h->off_side);
        for (int ci = 0; ci < ncl; ci++) {
            const TileCls c = cls[ci];
            tile_cls_group(c, r, dst + c.dst, meta + c.meta, ent, sc, out, sents, tk, s_hot);
        }
    }
    {
        // side op stream (sequences in reversed thread order): each piece's sum
        // is its part (plain store) or adds to the CTA's running sum of a hot
        // target's piece (one writer per tile)
        const int j = kTileThreads - 1 - r;
        if (j < ph->n_sseq) {
            const SideEnt *sents = reinterpret_cast<const SideEnt *>(blob + h->off_side);
            const uint32_t p32 = smem_u32(prog), sc32 = smem_u32(sc);
            const uint32_t sw = lds_u16(p32 + ph->off_sstart + 2 * j);
            const int ns = (int)(sw >> kSeqStartBits);
            uint32_t row = p32 + ph->off_srow;
            const uint32_t ops = p32 + ph->off_sops + 4 * j;
            uint32_t dst = p32 + ph->off_sdst + 2 * (sw & ((1u << kSeqStartBits) - 1));
            double acc = 0.0;
            for (int st = 0; st < ns; st++, row += 2) {
                const uint32_t w = lds_u32(ops + 4 * lds_u16(row));
                acc += lds_f64(sc32 + (w & 0xFFF8u));
                acc += lds_f64(sc32 + (w >> 16));
                if (w & kEmitBit) {
                    side_put(sents, lds_u16(dst), tk, s_hot, acc);
                    dst += 2;
                    acc = 0.0;
                }
            }
        }
    }
}

// Grid-wide barrier of the co-resident (cooperatively launched) grid: one
// thread per CTA arrives on a counter and, unless last, polls the generation
// word with a back-off sleep (the cooperative-groups barrier spins, and its
// polling warps take issue slots from the CTAs still working on the same SM);
// the last arrival resets the counter and advances the generation.
__device__ __forceinline__ void grid_barrier(unsigned int *bar, unsigned int nblocks)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int *gen = bar + 1;
        const unsigned int g0 = *gen;
        __threadfence();                                   // this CTA's writes before its arrival
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);                         // release
        } else {
            while (*gen == g0) __nanosleep(256);
        }
        __threadfence();                                   // acquire: the others' writes after
    }
    __syncthreads();
}

// After the last tile (all threads of the CTA): hot partials per CTA; then,
// after a grid-wide barrier (the kernel is launched cooperatively: its grid
// is the co-resident persistent grid), every warp of the grid sums a fixed
// share of the side targets, each in part order (fixed lane stride, fixed
// shuffle tree): deterministic, and no second launch or single finishing CTA.
template <bool kTrace>
__device__ __forceinline__ void tile_finish(const TileK &tk, const CallK &P, const double *s_hot)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x;
    const int32_t G = gridDim.x;
    if (!tk.n_side) return;
    __syncthreads();
    for (int h = tid; h < tk.n_hot; h += nt) {
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < kHotPieces; q++) v += s_hot[h * kHotPieces + q];   // piece order
        tk.part[tk.hot_base + (int64_t)h * G + blockIdx.x] = v;
    }
    grid_barrier(tk.gbar, G);
    TILE_TRACE_TAIL(kTraceSlots - 2);
    const int nw = nt >> 5;
    const int64_t gw = (int64_t)blockIdx.x * nw + warp, n_gw = (int64_t)G * nw;
    // hot targets (one part per CTA) first: warps 0 .. n_hot-1 of the grid
    for (int64_t h = gw; h < tk.n_hot; h += n_gw) {
        const double *pp = tk.part + tk.hot_base + h * G;
        double u = 0.0;
        for (int q0 = 0; q0 < G; q0 += 256) {
            double a[8];
#pragma unroll
            for (int r = 0; r < 8; r++) {
                const int q = q0 + r * 32 + lane;
                a[r] = q < G ? __ldcg(pp + q) : 0.0;
            }
#pragma unroll
            for (int r = 0; r < 8; r++) u += a[r];
        }
        u = warp_sum(u);
        if (lane == 0) {
            const int32_t g = tk.hot_gid[h];
            double *d = g < tk.nnz ? P.A + g : P.b + (g - tk.nnz);
            *d = __ldcg(tk.hot_pre + h) + u;
        }
    }
    // cold side targets: those of at most 8 parts one per thread (parts in
    // order), the rest one per warp (side_finish) -- one round of latency for
    // the many small ones (cfg2's bit lines, cfg4's hub loads)
    const int64_t gt = (int64_t)blockIdx.x * nt + tid, n_gt = (int64_t)G * nt;
    for (int64_t sid = tk.n_side_big + gt; sid < tk.n_side_cold; sid += n_gt) {
        const int32_t q0 = __ldg(tk.sd_part + 2 * sid), q1 = __ldg(tk.sd_part + 2 * sid + 1);
        double a[8];
#pragma unroll
        for (int r = 0; r < 8; r++) a[r] = q0 + r < q1 ? __ldcg(tk.part + q0 + r) : 0.0;
        double u = a[0];
#pragma unroll
        for (int r = 1; r < 8; r++) u += a[r];
        const int32_t g = __ldg(tk.sd_gid + sid);
        double *dst = g < tk.nnz ? P.A + g : P.b + (g - tk.nnz);
        *dst = *dst + u;
    }
    for (int64_t sid = gw; sid < tk.n_side_big; sid += n_gw) side_finish(tk, P, (int32_t)sid, lane);
}

// TILE kernel prologue: hot targets, card copy, mbarriers and the first
// NSTAGES blobs in flight.
#define TILE_PROLOGUE(NT, NSTAGES)                                                               \
    extern __shared__ __align__(16) unsigned char smem[];                                        \
    __shared__ CardK s_cards[EES_MAX_MODELS];                                                    \
    __shared__ __align__(8) uint64_t s_bar[NSTAGES];                                             \
    __shared__ double s_hot[kMaxHot * kHotPieces];                                               \
    const int tid = threadIdx.x;                                                                 \
    const int32_t G = gridDim.x;                                                                 \
    for (int k = tid; k < kMaxHot * kHotPieces; k += (NT)) s_hot[k] = 0.0;                       \
    if (tid < tk.n_hot && blockIdx.x == 0) {  /* hot targets' old values (written after the  */  \
        const int32_t g = tk.hot_gid[tid];       /* grid barrier only)                         */  \
        tk.hot_pre[tid] = g < tk.nnz ? P.A[g] : P.b[g - tk.nnz];                                 \
    }                                                                                            \
    auto issue_at = [&](uint4 d, int stage) {   /* head, then the program right after it */     \
        unsigned char *sd = s_stage + (size_t)stage * kStage;                                    \
        mbar_expect_tx(&s_bar[stage], d.y + d.w);                                                \
        tma_bulk_g2s(sd, tk.blob + 16 * (size_t)d.x, d.y, &s_bar[stage]);                       \
        tma_bulk_g2s(sd + d.y, tk.prog + 16 * (size_t)d.z, d.w, &s_bar[stage]);                 \
    };                                                                                           \
    auto issue = [&](int32_t tile, int stage) { issue_at(__ldg(tk.tdesc + tile), stage); };     \
    __shared__ double *s_bptr[2 * kTileBases];    /* two tiles (a second slot buffer has no B0) */ \
    __shared__ __align__(16) uint4 s_rf;          /* the refill's tdesc entry (bulk copy) */        \
    __shared__ __align__(8) uint64_t s_rf_bar;                                                   \
    uint32_t rf_phase = 0;                                                                       \
    TileOut out;                                                                                 \
    out.A = P.A;                                                                                 \
    out.Bm = P.b - tk.nnz;                                                                       \
    out.nnz = (int32_t)tk.nnz;                    /* < 2^31 (setup) */                           \
    out.bptr = 0;                                 /* per tile: s_bptr + (it & 1) * kTileBases */ \
    const int32_t t0 = blockIdx.x;                                                               \
    if (tid == 0) {                                                                              \
        for (int k = 0; k < (NSTAGES); k++) mbar_init(&s_bar[k], 1);                             \
        mbar_init(&s_rf_bar, 1);                                                                 \
        for (int k = 0; k < (NSTAGES); k++)                                                      \
            if (t0 + k * G < tk.n_tiles) issue(t0 + k * G, k);                                   \
    }                                                                                            \
    for (int k = tid; k < P.n_models; k += (NT)) s_cards[k] = P.cards[k];                        \
    __syncthreads();                                                                             \
    TILE_TRACE(0)

// One CTA of kTileThreads threads does both phases of a tile (barriers B1,
// and B0 with a single slot buffer).
template <bool kTrace, bool kRep, int kForm>
__global__ void __launch_bounds__(kTileThreads, tile_ctas(kForm)) k_tile(TileK tk, CallK P)
{
    constexpr int kBuf = tile_bufs(kForm);
    constexpr int kStage = stage_max(kForm);
#define s_stage (smem + sizeof(double) * sc_slots(kForm) * kBuf)
    constexpr int kStg = tile_stages(kForm);
    TILE_PROLOGUE(kTileThreads, kStg);
    unsigned char *s_c = smem;                                           // [kBuf][kScSlots] doubles
    if (kForm == 0 && tid < kBuf) {
        reinterpret_cast<double *>(s_c + (size_t)tid * 8 * kScSlots)[16 * kTileItems] = 0.0;   // zero slot
    }
    uint32_t parity = 0;                 // bit k: phase of s_bar[k]
    int it = 0;
    int stage = 0;
#if EES_LATE_GATHER
    TileRegs R;
    if (t0 < tk.n_tiles) {
        mbar_wait(&s_bar[0], 0);
        parity ^= 1u;
        tile_gather<kForm>(s_stage, t0, tk, P, R);
    }
    TILE_TRACE(1);
    for (int32_t t = t0; t < tk.n_tiles; t += G) {
        const unsigned char *blob = s_stage + (size_t)stage * kStage;
        unsigned char *sc = s_c + (kBuf == 2 ? (size_t)(it & 1) * 8 * sc_slots(kForm) : 0);
        const int32_t tr = t + kStg * G;              // the refill of this tile's stage (after B0)
        uint4 rf = make_uint4(0, 0, 0, 0);
        if (tid == 0 && tr < tk.n_tiles) rf = __ldg(tk.tdesc + tr);
        TileOut o = out;
        o.bptr = smem_u32(s_bptr + (it & 1) * kTileBases);
        if (tid < kTileBases) {
            const int32_t g = reinterpret_cast<const TileHdr *>(blob)->base[tid];
            s_bptr[(it & 1) * kTileBases + tid] = g < out.nnz ? out.A + g : out.Bm + g;
        }
        if (tid < reinterpret_cast<const TileHdr *>(blob)->n_items)
            tile_eval_item<kRep, kForm>(blob, R, tid, reinterpret_cast<double *>(sc), s_cards, P);
        TILE_TRACE(2 + 2 * it);
        __syncthreads();                                        // B1
        const int32_t tn = t + G;
        const int sn = stage + 1 == kStg ? 0 : stage + 1;
        if (tn < tk.n_tiles) {                                  // next tile's gathers hide behind the reduction
            mbar_wait(&s_bar[sn], (parity >> sn) & 1u);
            parity ^= 1u << sn;
            tile_gather<kForm>(s_stage + (size_t)sn * kStage, tn, tk, P, R);
        }
        if (kForm == 1) tile_reduce5(blob, sc, tid, o, tk, s_hot);
        else tile_reduce(blob, sc, tid, o, tk, s_hot);
        TILE_TRACE(3 + 2 * it);
        __syncthreads();                                        // B0
        if (tid == 0 && tr < tk.n_tiles) issue_at(rf, stage);  // this tile's stage is free
        stage = sn;
        it++;
    }
#else
    TileRegs ra, rb;
    if (t0 < tk.n_tiles) {
        mbar_wait(&s_bar[0], 0);
        parity ^= 1u;
        tile_gather<kForm>(s_stage, t0, tk, P, ra);
    }
    TILE_TRACE(1);
    // one tile; the two register sets alternate (no copies between tiles)
    auto step = [&](int32_t t, const TileRegs &cur, TileRegs &nxt) {
        const unsigned char *blob = s_stage + (size_t)stage * kStage;
        unsigned char *sc = s_c + (kBuf == 2 ? (size_t)(it & 1) * 8 * sc_slots(kForm) : 0);
        // the blob this iteration's refill (at B1) will fetch: its offsets are
        // loaded now, so warp 0 does not wait on global memory after B1
        const int32_t tr = t - G + kStg * G;
#if EES_TDESC_ASYNC
        // ... through a bulk copy into shared memory with its own mbarrier:
        // with a register load the compiler put the first use right behind
        // it, and warp 0 (hence the CTA, at B1) waited a global-memory latency
        // per tile (cp.async + wait_all waited for the gathers as well)
        if (tid == 0 && it > 0 && tr < tk.n_tiles) {
            mbar_expect_tx(&s_rf_bar, 16);
            tma_bulk_g2s(&s_rf, tk.tdesc + tr, 16, &s_rf_bar);
        }
#else
        uint4 rf = make_uint4(0, 0, 0, 0);
        if (tid == 0 && it > 0 && tr < tk.n_tiles) rf = __ldg(tk.tdesc + tr);
#endif
        TileOut o = out;
        o.bptr = smem_u32(s_bptr + (it & 1) * kTileBases);
        if (tid < kTileBases) {                 // this tile's destination pointers (read after B1)
            const int32_t g = reinterpret_cast<const TileHdr *>(blob)->base[tid];
            s_bptr[(it & 1) * kTileBases + tid] = g < out.nnz ? out.A + g : out.Bm + g;
        }
        if (tid < reinterpret_cast<const TileHdr *>(blob)->n_items)
            tile_eval_item<kRep, kForm>(blob, cur, tid, reinterpret_cast<double *>(sc), s_cards, P);
        // next tile: its blob was issued >= one tile ago; start its gathers now
        const int32_t tn = t + G;
        const int sn = stage + 1 == kStg ? 0 : stage + 1;
        if (tn < tk.n_tiles) {
            mbar_wait(&s_bar[sn], (parity >> sn) & 1u);
            parity ^= 1u << sn;
            tile_gather<kForm>(s_stage + (size_t)sn * kStage, tn, tk, P, nxt);
            if (tid == 32) {                                    // warp 1: the next tile's A block into L2
                const TileHdr *hn = reinterpret_cast<const TileHdr *>(s_stage + (size_t)sn * kStage);
                l2_prefetch_block(P.A, hn->a_lo, hn->a_n);
            }
        }
        TILE_TRACE(2 + 2 * it);
        __syncthreads();                                        // B1
        if (tid == 0 && it > 0 && tr < tk.n_tiles) {            // refill the stage of tile t-G
#if EES_TDESC_ASYNC
            mbar_wait(&s_rf_bar, rf_phase);
            rf_phase ^= 1u;
            const uint4 rf = s_rf;
#endif
            issue_at(rf, stage == 0 ? kStg - 1 : stage - 1);
        }
        if (kForm == 1) tile_reduce5(blob, sc, tid, o, tk, s_hot);
        else tile_reduce(blob, sc, tid, o, tk, s_hot);
        TILE_TRACE(3 + 2 * it);
        if (kBuf == 1) __syncthreads();                         // B0: slots free for the next tile
        stage = sn;
        it++;
    };
#ifndef EES_TILE_UNROLL2
#define EES_TILE_UNROLL2 1
#endif
    if (EES_TILE_UNROLL2) {
        for (int32_t t = t0; t < tk.n_tiles;) {
            step(t, ra, rb);
            t += G;
            if (t >= tk.n_tiles) break;
            step(t, rb, ra);
            t += G;
        }
    } else {                            // one copy of the loop body (half the code), one register copy
        for (int32_t t = t0; t < tk.n_tiles; t += G) {
            step(t, ra, rb);
            ra = rb;
        }
    }
#endif
    tile_finish<kTrace>(tk, P, s_hot);
    TILE_TRACE_TAIL(kTraceSlots - 1);
#undef s_stage
}


template <int kForm>
static int tile_bps()
{
    constexpr int smem = (int)tile_smem<kForm>();
    cudaFuncSetAttribute(k_tile<false, false, kForm>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_tile<true, false, kForm>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_tile<false, true, kForm>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    // one grid serves every instantiation (the hot-part layout, and the
    // cooperative launch needs it co-resident): the smallest occupancy
    int nb = 0, nb2 = 0, nb3 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tile<false, false, kForm>, kTileThreads, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb2, k_tile<false, true, kForm>, kTileThreads, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb3, k_tile<true, false, kForm>, kTileThreads, smem);
    nb = std::min(nb, std::min(nb2 > 0 ? nb2 : nb, nb3 > 0 ? nb3 : nb));
    return nb > 0 ? nb : 1;
}

int tile_blocks_per_sm(int form) { return form == 1 ? tile_bps<1>() : tile_bps<0>(); }

// Cooperative launch when side targets need the grid barrier (the grid is
// the co-resident persistent grid: SMs x tile_blocks_per_sm, capped by tiles).
template <int kForm>
static cudaError_t launch_tile_form(const TileK &tk, const CallK &call, int grid, cudaStream_t st)
{
    constexpr size_t smem = tile_smem<kForm>();
    const void *fn = tk.trace ? (const void *)k_tile<true, false, kForm>
                     : call.work > 1 ? (const void *)k_tile<false, true, kForm>
                                     : (const void *)k_tile<false, false, kForm>;
    TileK a0 = tk;
    CallK a1 = call;
    void *args[] = {&a0, &a1};
    if (tk.n_side) return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kTileThreads), args, smem, st);
    return cudaLaunchKernel(fn, dim3(grid), dim3(kTileThreads), args, smem, st);
}

cudaError_t launch_tile(const TileK &tk, const CallK &call, int grid, cudaStream_t st, int *n_launches)
{
    *n_launches = 0;
    if (tk.n_tiles == 0) return cudaSuccess;
    const cudaError_t e = tk.form == 1 ? launch_tile_form<1>(tk, call, grid, st) : launch_tile_form<0>(tk, call, grid, st);
    *n_launches = 1;
    return e == cudaSuccess ? cudaPeekAtLastError() : e;
}

}  // namespace ees
