/*
 * ees_oracle.c -- TEST INFRASTRUCTURE ONLY (not product code).
 *
 * A plain, slow, obviously-correct CPU implementation of what the hot path
 * computes: one Newton-Raphson evaluate+stamp of every MOSFET into the MNA
 * matrix A (CSR values) and right-hand side b,
 * the conflict-graph greedy colouring and, for timing only,
 * the paper's Table I CPU kernels loadsingle / loadomp / ColorFused.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
 * --impl reference legs may load this library.  It shares no code, header,
 * table or helper with paper_2604_03079_b200/ (the CUDA path); the only
 * shared thing is the seeded input generator module netgen/.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math -shared -fPIC
 * (no FMA contraction, IEEE division: SURVEY §8(c) "Floating-point flags").
 *
 * Notation follows SURVEY.md §8(c) (the reading of SPEC S:196, S:229-232 that
 * DESIGN.md §2 records): terminals D=0 G=1 S=2 B=3, p = polarity, vt = p*vt0,
 * beta = (kp*W)/L, Gc = C/h, gmin across D-S.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { TD = 0, TG = 1, TS = 2, TB = 3 };

typedef struct {
    int32_t polarity;          /* +1 NMOS, -1 PMOS */
    double vt0, kp, lam;       /* SPICE sign convention: PMOS vt0 < 0 */
    double cgs, cgd, cdb;      /* farads */
} orc_model;

/* ------------------------------------------------------------------------
 * Level-1 channel, SPEC S:196 as read in SURVEY §8(c) steps 1-5.
 * out = {I_ch (D->S through the channel), gm = dI/dV_G, gds = dI/dV_D}
 * info = {region (0 cutoff, 1 triode, 2 saturation), mode (+1 fwd, -1 rev)}
 * --------------------------------------------------------------------- */
void orc_channel(int32_t p, double vt0, double lam, double beta,
                 double VD, double VG, double VS, double out[3], int32_t info[2])
{
    double vt = p * vt0;                          /* step 0: vt = p*vt0 (A4) */
    double vgs = p * (VG - VS);                   /* step 1: reflected frame */
    double vds = p * (VD - VS);
    double u, v;
    int32_t s;
    if (vds >= 0) { u = vgs; v = vds; s = +1; }   /* step 2: mode (A8 tie -> fwd) */
    else          { u = vgs - vds; v = -vds; s = -1; }   /* D/S swap */
    double uov = u - vt;                          /* step 3 */
    double op = 1.0 + lam * v;
    double f, fu, fv;
    int32_t region;
    if (uov <= 0) {                               /* cutoff: Id = 0 */
        f = 0; fu = 0; fv = 0; region = 0;
    } else if (v >= uov) {                        /* saturation: (kp/2)(W/L)(Vgs-Vt)^2(1+lam Vds) */
        f  = beta / 2 * uov * uov * op;
        fu = beta * uov * op;
        fv = beta / 2 * uov * uov * lam;
        region = 2;
    } else {                                      /* triode: kp(W/L)((Vgs-Vt)Vds - Vds^2/2)(1+lam Vds) */
        double q = uov * v - v * v / 2;
        f  = beta * q * op;
        fu = beta * v * op;
        fv = beta * (uov - v) * op + beta * q * lam;
        region = 1;
    }
    double F, Fgs, Fds;                           /* step 4 */
    if (s > 0) { F = f;  Fgs = fu;  Fds = fv; }
    else       { F = -f; Fgs = -fu; Fds = fu + fv; }
    out[0] = p * F;                               /* step 5: I_ch = p F */
    out[1] = Fgs;                                 /* gm  (terminal frame, A9) */
    out[2] = Fds;                                 /* gds */
    info[0] = region;
    info[1] = s;
}

/* ------------------------------------------------------------------------
 * One device's elementary MNA contributions (Ho et al. MNA element stamps,
 * P:29, with the Norton current written as its three
 * terms).  Y entries are (row terminal, col terminal, value); J entries are
 * (row terminal, value) with the KCL row convention sum_j Y V = J.
 * Returns counts via ny/nj (24 and 12).
 * --------------------------------------------------------------------- */
#define ORC_NY 24
#define ORC_NJ 12

static void add_y(int32_t *ya, int32_t *yc, double *yv, int *k, int a, int c, double v)
{ ya[*k] = a; yc[*k] = c; yv[*k] = v; (*k)++; }
static void add_j(int32_t *ja, double *jv, int *k, int a, double v)
{ ja[*k] = a; jv[*k] = v; (*k)++; }

void orc_device_stamps(const orc_model *m, double beta, double gmin, double h,
                       const double V[4], const double v0[3],
                       int32_t *ya, int32_t *yc, double *yv, int32_t *ny,
                       int32_t *ja, double *jv, int32_t *nj)
{
    double o[3];
    int32_t info[2];
    orc_channel(m->polarity, m->vt0, m->lam, beta, V[TD], V[TG], V[TS], o, info);
    double I = o[0], gm = o[1], gds = o[2];
    int k = 0, q = 0;
    /* channel transconductance: VCCS gm*(V_G - V_S) from D to S */
    add_y(ya, yc, yv, &k, TD, TG, +gm);
    add_y(ya, yc, yv, &k, TD, TS, -gm);
    add_y(ya, yc, yv, &k, TS, TG, -gm);
    add_y(ya, yc, yv, &k, TS, TS, +gm);
    /* channel output conductance gds between D and S */
    add_y(ya, yc, yv, &k, TD, TD, +gds);
    add_y(ya, yc, yv, &k, TD, TS, -gds);
    add_y(ya, yc, yv, &k, TS, TD, -gds);
    add_y(ya, yc, yv, &k, TS, TS, +gds);
    /* gmin across D-S, linear: no J term */
    add_y(ya, yc, yv, &k, TD, TD, +gmin);
    add_y(ya, yc, yv, &k, TD, TS, -gmin);
    add_y(ya, yc, yv, &k, TS, TD, -gmin);
    add_y(ya, yc, yv, &k, TS, TS, +gmin);
    /* backward-Euler capacitor companions ("Geq = C/dt, Ieq = -(C/dt) v_prev") */
    const int cap_a[3] = { TG, TG, TD };
    const int cap_c[3] = { TS, TD, TB };
    const double cap_C[3] = { m->cgs, m->cgd, m->cdb };
    for (int t = 0; t < 3; t++) {
        double Gc = cap_C[t] / h;
        int a = cap_a[t], c = cap_c[t];
        add_y(ya, yc, yv, &k, a, a, +Gc);
        add_y(ya, yc, yv, &k, c, c, +Gc);
        add_y(ya, yc, yv, &k, a, c, -Gc);
        add_y(ya, yc, yv, &k, c, a, -Gc);
        double Jc = Gc * v0[t];
        add_j(ja, jv, &q, a, +Jc);
        add_j(ja, jv, &q, c, -Jc);
    }
    /* Norton current Ieq = I - gm*(V_G-V_S) - gds*(V_D-V_S) leaving D, entering S:
     * J[D] -= Ieq, J[S] += Ieq, written term by term. */
    double tgm = gm * (V[TG] - V[TS]);
    double tgd = gds * (V[TD] - V[TS]);
    add_j(ja, jv, &q, TD, -I);
    add_j(ja, jv, &q, TD, +tgm);
    add_j(ja, jv, &q, TD, +tgd);
    add_j(ja, jv, &q, TS, +I);
    add_j(ja, jv, &q, TS, -tgm);
    add_j(ja, jv, &q, TS, -tgd);
    *ny = k;
    *nj = q;
}

/* ------------------------------------------------------------------------
 * Sparsity pattern, SPEC S:114-131 reserve/finalize: every ordered pair of
 * non-ground terminals of every device, plus the caller's extra entries;
 * sorted, de-duplicated.  Keys are row*n + col.  `keys` must hold
 * 16*n_dev + n_extra entries; returns nnz (keys[0..nnz) sorted unique).
 * --------------------------------------------------------------------- */
static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

int64_t orc_pattern(int64_t n, int64_t n_dev, const int32_t *d, const int32_t *g,
                    const int32_t *s, const int32_t *b, int64_t n_extra,
                    const int32_t *er, const int32_t *ec, int64_t *keys)
{
    int64_t m = 0;
    for (int64_t i = 0; i < n_dev; i++) {
        int32_t T[4] = { d[i], g[i], s[i], b[i] };
        for (int a = 0; a < 4; a++)
            for (int c = 0; c < 4; c++)
                if (T[a] >= 0 && T[c] >= 0)
                    keys[m++] = (int64_t)T[a] * n + T[c];
    }
    for (int64_t e = 0; e < n_extra; e++)
        keys[m++] = (int64_t)er[e] * n + ec[e];
    qsort(keys, (size_t)m, sizeof(int64_t), cmp_i64);
    int64_t u = 0;
    for (int64_t i = 0; i < m; i++)
        if (u == 0 || keys[i] != keys[u - 1]) keys[u++] = keys[i];
    return u;
}

static int64_t find_key(const int64_t *keys, int64_t nnz, int64_t key)
{
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (keys[mid] < key) lo = mid + 1; else hi = mid;
    }
    return (lo < nnz && keys[lo] == key) ? lo : -1;
}

/* Neumaier compensated summation (sum + comp) with an |c| shadow. */
static void neumaier(double *sum, double *comp, double *abssum, double x)
{
    double s = *sum, t = s + x;
    if (fabs(s) >= fabs(x)) *comp += (s - t) + x;
    else                    *comp += (x - t) + s;
    *sum = t;
    *abssum += fabs(x);
}

/* ------------------------------------------------------------------------
 * The reference result: SPEC S:339 loadsingle "defines the REFERENCE
 * result" -- devices in netlist order, compute then stamp, each elementary
 * contribution accumulated into its (row, col) entry.  Accumulation is
 * Neumaier-compensated (SURVEY §8(c) comparison rule), with the sum of
 * absolute elementary contributions kept beside each entry for the
 * 1e-12 * sum|c| tolerance (BASELINE.json north_star).
 * A_sum/A_abs [nnz] and b_sum/b_abs [n] are IN/OUT: they start from the
 * caller's initial values (accumulate semantics).
 * Returns 0, or -1 if a contribution has no pattern entry.
 * --------------------------------------------------------------------- */
int32_t orc_reference(int64_t n, int64_t nnz, const int64_t *keys, int64_t n_dev,
                      const int32_t *d, const int32_t *g, const int32_t *s, const int32_t *b,
                      const double *w, const double *l, const int32_t *model,
                      const double *vprev /* [3][n_dev] */, const orc_model *models,
                      double gmin, double h, const double *x,
                      double *A_sum, double *A_abs, double *b_sum, double *b_abs)
{
    double *A_comp = calloc((size_t)(nnz ? nnz : 1), sizeof(double));
    double *b_comp = calloc((size_t)(n ? n : 1), sizeof(double));
    int32_t ya[ORC_NY], yc[ORC_NY], ja[ORC_NJ], ny, nj;
    double yv[ORC_NY], jv[ORC_NJ];
    int32_t rc = 0;
    for (int64_t i = 0; i < n_dev && rc == 0; i++) {
        const orc_model *m = &models[model[i]];
        double beta = (m->kp * w[i]) / l[i];
        int32_t T[4] = { d[i], g[i], s[i], b[i] };
        double V[4], v0[3];
        for (int a = 0; a < 4; a++) V[a] = T[a] >= 0 ? x[T[a]] : 0.0;
        for (int t = 0; t < 3; t++) v0[t] = vprev[t * n_dev + i];
        orc_device_stamps(m, beta, gmin, h, V, v0, ya, yc, yv, &ny, ja, jv, &nj);
        for (int e = 0; e < ny; e++) {
            int32_t r = T[ya[e]], c = T[yc[e]];
            if (r < 0 || c < 0) continue;           /* ground elimination */
            int64_t k = find_key(keys, nnz, (int64_t)r * n + c);
            if (k < 0) { rc = -1; break; }
            neumaier(&A_sum[k], &A_comp[k], &A_abs[k], yv[e]);
        }
        for (int e = 0; e < nj; e++) {
            int32_t r = T[ja[e]];
            if (r < 0) continue;
            neumaier(&b_sum[r], &b_comp[r], &b_abs[r], jv[e]);
        }
    }
    for (int64_t k = 0; k < nnz; k++) A_sum[k] += A_comp[k];
    for (int64_t r = 0; r < n; r++) b_sum[r] += b_comp[r];
    free(A_comp);
    free(b_comp);
    return rc;
}

/* ------------------------------------------------------------------------
 * Greedy first-fit colouring of the conflict graph ("visiting vertices
 * in an order and assigning each vertex the smallest color not used by its
 * already-colored neighbors"; P:60 edge iff two FETs share a non-ground
 * node).  `excluded[node]` != 0 removes a node from the conflict relation
 * (SURVEY A1 reading: supply rails; all zero = paper-literal rule).
 * Visit order = netlist order.  Written the plain way:
 * for device i, every earlier device j incident on a shared conflict node
 * forbids its colour.  Returns C.
 * --------------------------------------------------------------------- */
static int64_t *incidence(int64_t n_nodes, int64_t n_dev, const int32_t *d, const int32_t *g,
                          const int32_t *s, const int32_t *b, const uint8_t *excluded,
                          int64_t **ptr_out)
{
    int64_t *ptr = calloc((size_t)n_nodes + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n_dev; i++) {
        int32_t T[4] = { d[i], g[i], s[i], b[i] };
        for (int a = 0; a < 4; a++) {
            int dup = 0;
            for (int c = 0; c < a; c++) dup |= (T[c] == T[a]);
            if (T[a] >= 0 && !dup && !excluded[T[a]]) ptr[T[a] + 1]++;
        }
    }
    for (int64_t v = 0; v < n_nodes; v++) ptr[v + 1] += ptr[v];
    int64_t *fill = malloc(sizeof(int64_t) * (size_t)(n_nodes + 1));
    memcpy(fill, ptr, sizeof(int64_t) * (size_t)(n_nodes + 1));
    int64_t *dev = malloc(sizeof(int64_t) * (size_t)(ptr[n_nodes] ? ptr[n_nodes] : 1));
    for (int64_t i = 0; i < n_dev; i++) {           /* ascending device order per node */
        int32_t T[4] = { d[i], g[i], s[i], b[i] };
        for (int a = 0; a < 4; a++) {
            int dup = 0;
            for (int c = 0; c < a; c++) dup |= (T[c] == T[a]);
            if (T[a] >= 0 && !dup && !excluded[T[a]]) dev[fill[T[a]]++] = i;
        }
    }
    free(fill);
    *ptr_out = ptr;
    return dev;
}

int32_t orc_greedy_color(int64_t n_nodes, int64_t n_dev, const int32_t *d, const int32_t *g,
                         const int32_t *s, const int32_t *b, const uint8_t *excluded,
                         int32_t *color)
{
    int64_t *ptr;
    int64_t *dev = incidence(n_nodes, n_dev, d, g, s, b, excluded, &ptr);
    int64_t *forbid = malloc(sizeof(int64_t) * (size_t)(n_dev + 1));
    for (int64_t c = 0; c <= n_dev; c++) forbid[c] = -1;
    int32_t C = 0;
    for (int64_t i = 0; i < n_dev; i++) {
        int32_t T[4] = { d[i], g[i], s[i], b[i] };
        for (int a = 0; a < 4; a++) {
            if (T[a] < 0 || excluded[T[a]]) continue;
            for (int64_t e = ptr[T[a]]; e < ptr[T[a] + 1]; e++) {
                int64_t j = dev[e];
                if (j >= i) break;                   /* only already-coloured neighbours */
                forbid[color[j]] = i;
            }
        }
        int32_t c = 0;
        while (forbid[c] == i) c++;
        color[i] = c;
        if (c + 1 > C) C = c + 1;
    }
    free(forbid);
    free(dev);
    free(ptr);
    return n_dev ? C : 0;
}

/* Exhaustive validity scan: for every conflict node, the colours of
 * its incident devices are pairwise distinct.  Returns the number of
 * violating (node, device) incidences (0 = valid). */
int64_t orc_color_violations(int64_t n_nodes, int64_t n_dev, const int32_t *d, const int32_t *g,
                             const int32_t *s, const int32_t *b, const uint8_t *excluded,
                             const int32_t *color, int32_t n_colors)
{
    int64_t *ptr;
    int64_t *dev = incidence(n_nodes, n_dev, d, g, s, b, excluded, &ptr);
    int64_t *seen = malloc(sizeof(int64_t) * (size_t)(n_colors + 1));
    for (int32_t c = 0; c <= n_colors; c++) seen[c] = -1;
    int64_t bad = 0;
    for (int64_t v = 0; v < n_nodes; v++)
        for (int64_t e = ptr[v]; e < ptr[v + 1]; e++) {
            int32_t c = color[dev[e]];
            if (c < 0 || c >= n_colors) { bad++; continue; }
            if (seen[c] == v) bad++;
            seen[c] = v;
        }
    free(seen);
    free(dev);
    free(ptr);
    return bad;
}

/* ------------------------------------------------------------------------
 * CPU baselines (timed, never used for parity): the paper's Table I kernels
 * in plain FP64 over a precomputed stamp plan
 * (S:108 StampPlan = handles per device), built once at setup.
 * plan_y[i*ORC_NY + e] = A index of device i's e-th Y contribution (-1 if a
 * terminal is ground); plan_j likewise for J (row, or -1).
 * --------------------------------------------------------------------- */
typedef struct {
    int64_t n, nnz, n_dev;
    int64_t *plan_y;      /* [n_dev*ORC_NY] */
    int32_t *plan_j;      /* [n_dev*ORC_NJ] */
    double *beta;         /* [n_dev] */
    const int32_t *T[4];
    const int32_t *model;
    const double *vprev;
    orc_model *models;
    int32_t n_models;
    /* ColorFused schedule */
    int32_t n_colors;
    int64_t *color_ptr;   /* [C+1] */
    int64_t *perm;        /* devices grouped by colour, netlist order inside */
    int32_t *rail_y;      /* [nnz] rail-entry index of A slot (-1 if not rail x rail) */
    int32_t *rail_j;      /* [n] rail-entry index of b row (-1 if not rail) */
    int32_t n_rail;
    double *buf;          /* loadomp ContributionBuffer [n_dev*(NY+NJ)] */
} orc_plan;

static void dev_contrib(const orc_plan *P, int64_t i, double gmin, double h, const double *x,
                        double *yv, double *jv)
{
    const orc_model *m = &P->models[P->model[i]];
    double V[4], v0[3];
    int32_t ya[ORC_NY], yc[ORC_NY], ja[ORC_NJ], ny, nj;
    for (int a = 0; a < 4; a++) { int32_t t = P->T[a][i]; V[a] = t >= 0 ? x[t] : 0.0; }
    for (int t = 0; t < 3; t++) v0[t] = P->vprev[t * P->n_dev + i];
    orc_device_stamps(m, P->beta[i], gmin, h, V, v0, ya, yc, yv, &ny, ja, jv, &nj);
}

void *orc_plan_create(int64_t n, int64_t nnz, const int64_t *keys, int64_t n_dev,
                      const int32_t *d, const int32_t *g, const int32_t *s, const int32_t *b,
                      const double *w, const double *l, const int32_t *model,
                      const double *vprev, const orc_model *models, int32_t n_models,
                      const int32_t *color, int32_t n_colors, const uint8_t *is_rail)
{
    orc_plan *P = calloc(1, sizeof(orc_plan));
    P->n = n; P->nnz = nnz; P->n_dev = n_dev;
    P->T[0] = d; P->T[1] = g; P->T[2] = s; P->T[3] = b;
    P->model = model; P->vprev = vprev;
    P->models = malloc(sizeof(orc_model) * (size_t)(n_models ? n_models : 1));
    memcpy(P->models, models, sizeof(orc_model) * (size_t)n_models);
    P->n_models = n_models;
    P->plan_y = malloc(sizeof(int64_t) * (size_t)(n_dev * ORC_NY + 1));
    P->plan_j = malloc(sizeof(int32_t) * (size_t)(n_dev * ORC_NJ + 1));
    P->beta = malloc(sizeof(double) * (size_t)(n_dev + 1));
    P->buf = malloc(sizeof(double) * (size_t)(n_dev * (ORC_NY + ORC_NJ) + 1));
    int32_t ya[ORC_NY], yc[ORC_NY], ja[ORC_NJ], ny, nj;
    double yv[ORC_NY], jv[ORC_NJ];
    double V[4] = { 0, 0, 0, 0 }, v0[3] = { 0, 0, 0 };
    orc_model dummy = { 1, 0, 1, 0, 0, 0, 0 };
    orc_device_stamps(&dummy, 1.0, 0.0, 1.0, V, v0, ya, yc, yv, &ny, ja, jv, &nj);  /* fixed layout */
    for (int64_t i = 0; i < n_dev; i++) {
        const orc_model *m = &models[model[i]];
        P->beta[i] = (m->kp * w[i]) / l[i];
        int32_t T[4] = { d[i], g[i], s[i], b[i] };
        for (int e = 0; e < ny; e++) {
            int32_t r = T[ya[e]], c = T[yc[e]];
            P->plan_y[i * ORC_NY + e] = (r < 0 || c < 0) ? -1 : find_key(keys, nnz, (int64_t)r * n + c);
        }
        for (int e = 0; e < nj; e++) P->plan_j[i * ORC_NJ + e] = T[ja[e]];
    }
    /* colour groups */
    P->n_colors = n_colors;
    P->color_ptr = calloc((size_t)n_colors + 2, sizeof(int64_t));
    P->perm = malloc(sizeof(int64_t) * (size_t)(n_dev + 1));
    if (color) {
        for (int64_t i = 0; i < n_dev; i++) P->color_ptr[color[i] + 1]++;
        for (int32_t c = 0; c < n_colors; c++) P->color_ptr[c + 1] += P->color_ptr[c];
        int64_t *fill = malloc(sizeof(int64_t) * ((size_t)n_colors + 1));
        memcpy(fill, P->color_ptr, sizeof(int64_t) * ((size_t)n_colors + 1));
        for (int64_t i = 0; i < n_dev; i++) P->perm[fill[color[i]]++] = i;
        free(fill);
    }
    /* rail x rail A entries and rail b rows take a per-thread side sum in ColorFused */
    P->rail_y = malloc(sizeof(int32_t) * (size_t)(nnz + 1));
    P->rail_j = malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t nr = 0;
    for (int64_t k = 0; k < nnz; k++) {
        int64_t r = keys[k] / n, c = keys[k] % n;
        P->rail_y[k] = (is_rail && is_rail[r] && is_rail[c]) ? nr++ : -1;
    }
    for (int64_t r = 0; r < n; r++) P->rail_j[r] = (is_rail && is_rail[r]) ? nr++ : -1;
    P->n_rail = nr;
    return P;
}

void orc_plan_destroy(void *p)
{
    orc_plan *P = p;
    if (!P) return;
    free(P->models); free(P->plan_y); free(P->plan_j); free(P->beta); free(P->buf);
    free(P->color_ptr); free(P->perm); free(P->rail_y); free(P->rail_j);
    free(P);
}

/* loadsingle: sequential compute + stamp, plain FP64 += */
void orc_loadsingle(void *p, double gmin, double h, const double *x, double *A, double *bv)
{
    orc_plan *P = p;
    double yv[ORC_NY], jv[ORC_NJ];
    for (int64_t i = 0; i < P->n_dev; i++) {
        dev_contrib(P, i, gmin, h, x, yv, jv);
        const int64_t *py = &P->plan_y[i * ORC_NY];
        const int32_t *pj = &P->plan_j[i * ORC_NJ];
        for (int e = 0; e < ORC_NY; e++) if (py[e] >= 0) A[py[e]] += yv[e];
        for (int e = 0; e < ORC_NJ; e++) if (pj[e] >= 0) bv[pj[e]] += jv[e];
    }
}

/* loadomp: parallel compute into the ContributionBuffer,
 * then a sequential stamp in netlist order (bitwise equal to loadsingle). */
void orc_loadomp(void *p, int32_t threads, double gmin, double h, const double *x,
                 double *A, double *bv)
{
    orc_plan *P = p;
    const int W = ORC_NY + ORC_NJ;
    #pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t i = 0; i < P->n_dev; i++)
        dev_contrib(P, i, gmin, h, x, &P->buf[i * W], &P->buf[i * W + ORC_NY]);
    for (int64_t i = 0; i < P->n_dev; i++) {
        const double *yv = &P->buf[i * W], *jv = yv + ORC_NY;
        const int64_t *py = &P->plan_y[i * ORC_NY];
        const int32_t *pj = &P->plan_j[i * ORC_NJ];
        for (int e = 0; e < ORC_NY; e++) if (py[e] >= 0) A[py[e]] += yv[e];
        for (int e = 0; e < ORC_NJ; e++) if (pj[e] >= 0) bv[pj[e]] += jv[e];
    }
}

/* ColorFused: per colour, a parallel for in which each
 * device computes and immediately stamps; rail x rail entries and rail b rows
 * (shared by same-colour devices under the SURVEY A1 reading) go to
 * per-thread partials summed in thread order at the end. */
void orc_colorfused(void *p, int32_t threads, double gmin, double h, const double *x,
                    double *A, double *bv)
{
    orc_plan *P = p;
    int32_t NR = P->n_rail;
    double *part = calloc((size_t)threads * (size_t)(NR ? NR : 1), sizeof(double));
    #pragma omp parallel num_threads(threads)
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        double *my = &part[(size_t)tid * (size_t)(NR ? NR : 1)];
        double yv[ORC_NY], jv[ORC_NJ];
        for (int32_t c = 0; c < P->n_colors; c++) {
            #pragma omp for schedule(static)
            for (int64_t q = P->color_ptr[c]; q < P->color_ptr[c + 1]; q++) {
                int64_t i = P->perm[q];
                dev_contrib(P, i, gmin, h, x, yv, jv);
                const int64_t *py = &P->plan_y[i * ORC_NY];
                const int32_t *pj = &P->plan_j[i * ORC_NJ];
                for (int e = 0; e < ORC_NY; e++) {
                    int64_t k = py[e];
                    if (k < 0) continue;
                    int32_t r = P->rail_y[k];
                    if (r >= 0) my[r] += yv[e]; else A[k] += yv[e];
                }
                for (int e = 0; e < ORC_NJ; e++) {
                    int32_t row = pj[e];
                    if (row < 0) continue;
                    int32_t r = P->rail_j[row];
                    if (r >= 0) my[r] += jv[e]; else bv[row] += jv[e];
                }
            }   /* implicit barrier between colours */
        }
    }
    for (int t = 0; t < threads; t++)
        for (int64_t k = 0; k < P->nnz; k++)
            if (NR && P->rail_y[k] >= 0) A[k] += part[(size_t)t * NR + P->rail_y[k]];
    for (int t = 0; t < threads; t++)
        for (int64_t r = 0; r < P->n; r++)
            if (NR && P->rail_j[r] >= 0) bv[r] += part[(size_t)t * NR + P->rail_j[r]];
    free(part);
}

int32_t orc_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
