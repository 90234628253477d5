/*
 * gcp_oracle.c -- plain, slow, fp64 CPU oracle for stochastic GCP-Adam.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2605_20353_b200/) never imports, links or calls it,
 * and this file shares no code, header or table with the CUDA library.
 *
 * Every function follows the paper (arXiv 2605.20353, /root/reference/PAPER.md,
 * cited as P:line) step by step, in its order and notation, with the readings
 * listed in DESIGN.md §3 where the paper is silent (cited as "reading Rn").
 * Nothing is blocked, fused or reordered beyond what the cited passage states.
 * Single-threaded, double precision throughout.
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): Philox known-answer vectors,
 * closed forms of f and df/dm, brute-force dense Khatri-Rao MTTKRP, central
 * finite differences of the enumerated objective, the Gaussian CP
 * least-squares gradient identity, the Poisson closed-form gradient,
 * unbiasedness of the sampled estimators, Adam worked examples.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

enum { ORC_OK = 0, ORC_E_ARG = 1, ORC_E_RANGE = 2, ORC_E_DUP = 3,
       ORC_E_NO_NONZEROS = 4, ORC_E_NO_ZEROS = 5, ORC_E_REJECT_CAP = 6,
       ORC_E_OOM = 9 };
enum { ORC_GAUSSIAN = 0, ORC_POISSON = 1, ORC_BERNOULLI = 2 };
enum { ORC_STRATIFIED = 0, ORC_SEMI_STRATIFIED = 1 };
/* Philox "kind" field of the counter (reading R11 / DESIGN.md §3.3). */
enum { KIND_GRAD_NZ = 0, KIND_GRAD_Z = 1, KIND_F_NZ = 2, KIND_F_Z = 3, KIND_INIT = 4 };

#define REJECTION_CAP 1000          /* reading R5 */
#define POISSON_EPS 1e-10           /* reading R3  */

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11 "Random123"): 10 rounds of            */
/*   (c0,c1,c2,c3) -> (hi(M1*c2)^c1^k0, lo(M1*c2), hi(M0*c0)^c3^k1, lo(M0*c0)) */
/* with the key bumped by the Weyl constants between rounds.                  */
/* ------------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* The two 64-bit words of one Philox call (reading R11). */
static void philox_words(uint64_t seed, uint32_t slot, uint32_t rank, uint32_t kind,
                         uint32_t attempt, uint32_t group, uint32_t it, uint64_t W[2])
{
    uint32_t ctr[4] = { slot, rank, (kind << 28) | (attempt << 4) | group, it };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint32_t o[4];
    orc_philox4x32_10(ctr, key, o);
    W[0] = (uint64_t)o[0] | ((uint64_t)o[1] << 32);
    W[1] = (uint64_t)o[2] | ((uint64_t)o[3] << 32);
}

/* Map a uniform 64-bit word to {0..n-1}: floor(W*n / 2^64) (reading R11). */
static uint64_t range_map(uint64_t W, uint64_t n)
{
    return (uint64_t)(((u128)W * (u128)n) >> 64);
}

uint64_t orc_range_map(uint64_t W, uint64_t n) { return range_map(W, n); }

/* ------------------------------------------------------------------------ */
/* Sparse tensor X in coordinate format, one rank's block.        */
/* ------------------------------------------------------------------------ */
typedef struct {
    int d;
    int64_t dims[32];      /* global I_k */
    int64_t lo[32], hi[32];/* block bounds [lo_k, hi_k) of this rank */
    int64_t N;             /* nonzeros stored in this block */
    int64_t *subs;         /* N*d global coordinates, lexicographically sorted */
    double *vals;          /* N values */
} orc_tensor;

static int g_sort_d;
static const int64_t *g_sort_subs;
/* lexicographic comparison, i_1 most significant (reading R15) */
static int lex_cmp(const int64_t *a, const int64_t *b, int d)
{
    for (int k = 0; k < d; ++k) {
        if (a[k] < b[k]) return -1;
        if (a[k] > b[k]) return 1;
    }
    return 0;
}
static int perm_cmp(const void *pa, const void *pb)
{
    int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
    int c = lex_cmp(g_sort_subs + a * g_sort_d, g_sort_subs + b * g_sort_d, g_sort_d);
    if (c) return c;
    return (a > b) - (a < b);
}

void orc_tensor_free(orc_tensor *t)
{
    if (!t) return;
    free(t->subs); free(t->vals); free(t);
}

/* Build the block tensor: validate, sort lexicographically, reject duplicates.
 * lo/hi may be NULL (whole tensor). */
int orc_tensor_new(int d, const int64_t *dims, const int64_t *lo, const int64_t *hi,
                   int64_t nnz, const int64_t *subs, const double *vals, orc_tensor **out)
{
    *out = NULL;
    if (d < 2 || d > 32 || nnz < 0) return ORC_E_ARG;
    for (int k = 0; k < d; ++k) if (dims[k] < 1 || dims[k] > 0xFFFFFFFFLL) return ORC_E_ARG;
    orc_tensor *t = (orc_tensor *)calloc(1, sizeof(orc_tensor));
    if (!t) return ORC_E_OOM;
    t->d = d;
    for (int k = 0; k < d; ++k) {
        t->dims[k] = dims[k];
        t->lo[k] = lo ? lo[k] : 0;
        t->hi[k] = hi ? hi[k] : dims[k];
        if (t->lo[k] < 0 || t->hi[k] > dims[k] || t->lo[k] > t->hi[k]) { free(t); return ORC_E_ARG; }
    }
    for (int64_t n = 0; n < nnz; ++n) {
        for (int k = 0; k < d; ++k) {
            int64_t i = subs[n * d + k];
            if (i < t->lo[k] || i >= t->hi[k]) { free(t); return ORC_E_RANGE; }
        }
        if (!isfinite(vals[n])) { free(t); return ORC_E_ARG; }
    }
    int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
    t->subs = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz * d : 1));
    t->vals = (double *)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
    if (!perm || !t->subs || !t->vals) { free(perm); orc_tensor_free(t); return ORC_E_OOM; }
    for (int64_t n = 0; n < nnz; ++n) perm[n] = n;
    g_sort_d = d; g_sort_subs = subs;
    qsort(perm, (size_t)nnz, sizeof(int64_t), perm_cmp);
    for (int64_t n = 0; n < nnz; ++n) {
        memcpy(t->subs + n * d, subs + perm[n] * d, sizeof(int64_t) * d);
        t->vals[n] = vals[perm[n]];
    }
    free(perm);
    for (int64_t n = 1; n < nnz; ++n)
        if (lex_cmp(t->subs + (n - 1) * d, t->subs + n * d, d) == 0) { orc_tensor_free(t); return ORC_E_DUP; }
    t->N = nnz;
    *out = t;
    return ORC_OK;
}

int64_t orc_tensor_nnz(const orc_tensor *t) { return t->N; }

void orc_tensor_sorted(const orc_tensor *t, int64_t *subs_out, double *vals_out)
{
    memcpy(subs_out, t->subs, sizeof(int64_t) * (size_t)(t->N * t->d));
    memcpy(vals_out, t->vals, sizeof(double) * (size_t)t->N);
}

/* M_w = prod_k (hi_k - lo_k), exact (reading R22: u128). */
static u128 block_M(const orc_tensor *t)
{
    u128 M = 1;
    for (int k = 0; k < t->d; ++k) M *= (u128)(t->hi[k] - t->lo[k]);
    return M;
}

double orc_tensor_M(const orc_tensor *t) { return (double)block_M(t); }

/* Membership by binary search of the sorted nonzero list, O(log N). */
int orc_tensor_contains(const orc_tensor *t, const int64_t *coords)
{
    int64_t a = 0, b = t->N;      /* search [a, b) */
    while (a < b) {
        int64_t mid = a + (b - a) / 2;
        int c = lex_cmp(t->subs + mid * t->d, coords, t->d);
        if (c == 0) return 1;
        if (c < 0) a = mid + 1; else b = mid;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Stratified sampling with the counter discipline of reading R11 */
/* ------------------------------------------------------------------------ */

/* Nonzero slot: j uniform over [0, N) with replacement (reading R4). */
static int64_t draw_nonzero(const orc_tensor *t, uint64_t seed, uint32_t rank, uint32_t kind,
                            uint32_t it, uint32_t slot)
{
    uint64_t W[2];
    philox_words(seed, slot, rank, kind, 0, 0, it, W);
    return (int64_t)range_map(W[0], (uint64_t)t->N);
}

/* Zero candidate, attempt a: "d integers i_1..i_d each randomly chosen out of
 * the ranges [1..I_1],...,[1..I_d]", within this rank's block.
 * Mode k uses word W_{k mod 2} of Philox group floor(k/2). */
static void draw_candidate(const orc_tensor *t, uint64_t seed, uint32_t rank, uint32_t kind,
                           uint32_t it, uint32_t slot, uint32_t attempt, int64_t *coords)
{
    uint64_t W[2];
    for (int k = 0; k < t->d; ++k) {
        if (k % 2 == 0) philox_words(seed, slot, rank, kind, attempt, (uint32_t)(k / 2), it, W);
        coords[k] = t->lo[k] + (int64_t)range_map(W[k % 2], (uint64_t)(t->hi[k] - t->lo[k]));
    }
}

/* Zero slot: "If it is not found, the sample corresponds to a zero, otherwise
 * the process repeats until the sampled entry is not found".
 * Returns attempts used (>=1) or -1 when the cap is hit (reading R5). */
static int draw_zero(const orc_tensor *t, uint64_t seed, uint32_t rank, uint32_t kind,
                     uint32_t it, uint32_t slot, int stratified, int64_t *coords)
{
    for (uint32_t a = 0; a < REJECTION_CAP; ++a) {
        draw_candidate(t, seed, rank, kind, it, slot, a, coords);
        if (!stratified) return 1;              /* semi-stratified: no search */
        if (!orc_tensor_contains(t, coords)) return (int)a + 1;
    }
    return -1;
}

/* ------------------------------------------------------------------------ */
/* Kruskal model (P:23-29 with lambda).  Factor rows of this block:  */
/* A[k] holds (hi_k - lo_k) x R values, row-major; row i_k - lo_k.               */
/* ------------------------------------------------------------------------ */
typedef struct {
    int d, R;
    const double *lambda;       /* R */
    const double *A[32];        /* per mode, block rows x R */
} orc_model;

static void make_model(orc_model *m, const orc_tensor *t, int R, const double *lambda,
                       const double *A_flat)
{
    m->d = t->d; m->R = R; m->lambda = lambda;
    size_t off = 0;
    for (int k = 0; k < t->d; ++k) {
        m->A[k] = A_flat + off;
        off += (size_t)(t->hi[k] - t->lo[k]) * (size_t)R;
    }
}

/* m_i = sum_r lambda_r prod_k a^(k)_{i_k r} */
static double model_value(const orc_model *m, const orc_tensor *t, const int64_t *coords)
{
    double s = 0.0;
    for (int r = 0; r < m->R; ++r) {
        double p = m->lambda[r];
        for (int k = 0; k < m->d; ++k) p *= m->A[k][(coords[k] - t->lo[k]) * m->R + r];
        s += p;
    }
    return s;
}

/* sum_r |lambda_r prod_k a| : rounding-error scale of m (tolerance only). */
static double model_abs(const orc_model *m, const orc_tensor *t, const int64_t *coords)
{
    double s = 0.0;
    for (int r = 0; r < m->R; ++r) {
        double p = fabs(m->lambda[r]);
        for (int k = 0; k < m->d; ++k) p *= fabs(m->A[k][(coords[k] - t->lo[k]) * m->R + r]);
        s += p;
    }
    return s;
}

double orc_model_value(const orc_tensor *t, int R, const double *lambda, const double *A_flat,
                       const int64_t *coords)
{
    orc_model m; make_model(&m, t, R, lambda, A_flat);
    return model_value(&m, t, coords);
}

/* ------------------------------------------------------------------------ */
/* Losses (reading R3: the standard GCP forms of Hong-Kolda-Duersch)  */
/* ------------------------------------------------------------------------ */
static double softplus(double m) { return (m > 0 ? m : 0.0) + log1p(exp(-fabs(m))); }
static double sigmoid(double m)
{
    if (m >= 0) return 1.0 / (1.0 + exp(-m));
    double e = exp(m);
    return e / (1.0 + e);
}

double orc_loss_f(int loss, double x, double m)
{
    switch (loss) {
    case ORC_GAUSSIAN:  return (x - m) * (x - m);
    case ORC_POISSON:   return m - x * log(m + POISSON_EPS);
    case ORC_BERNOULLI: return softplus(m) - x * m;
    }
    return NAN;
}

double orc_loss_df(int loss, double x, double m)
{
    switch (loss) {
    case ORC_GAUSSIAN:  return 2.0 * (m - x);
    case ORC_POISSON:   return 1.0 - x / (m + POISSON_EPS);
    case ORC_BERNOULLI: return sigmoid(m) - x;
    }
    return NAN;
}

double orc_loss_lower(int loss) { return loss == ORC_POISSON ? 0.0 : -INFINITY; }

/* Rounding-error scale of df/dm at (x, m) given mabs = sum_r |terms| (tolerance
 * only; DESIGN.md §5.2 derives it).  Not part of the method. */
static double df_scale(int loss, double x, double m, double mabs)
{
    switch (loss) {
    case ORC_GAUSSIAN:  return 2.0 * (mabs + fabs(x));
    case ORC_POISSON: {
        double den = m + POISSON_EPS;
        return 1.0 + fabs(x) / fabs(den) + fabs(x) * mabs / (den * den);
    }
    case ORC_BERNOULLI: {
        double s = sigmoid(m);
        return s + fabs(x) + s * (1.0 - s) * mabs;
    }
    }
    return NAN;
}
static double f_scale(int loss, double x, double m, double mabs)
{
    switch (loss) {
    case ORC_GAUSSIAN:  return (fabs(x) + mabs) * (fabs(x) + mabs);
    case ORC_POISSON:   return mabs + fabs(x * log(m + POISSON_EPS)) + fabs(x) * mabs / fabs(m + POISSON_EPS);
    case ORC_BERNOULLI: return softplus(m) + fabs(x * m) + (1.0 + fabs(x)) * mabs;
    }
    return NAN;
}

/* ------------------------------------------------------------------------ */
/* Per-rank sample counts and weights (reading R13)                 */
/* ------------------------------------------------------------------------ */
int64_t orc_alloc_count(int64_t total, int P, int w)
{
    return total / P + (w < total % P ? 1 : 0);
}

/* w_nz = N_w / p_w; w_z = (M_w - N_w) / q_w */
static double weight_nz(const orc_tensor *t, int64_t p_w) { return (double)t->N / (double)p_w; }
static double weight_z(const orc_tensor *t, int64_t q_w)
{
    return (double)(block_M(t) - (u128)t->N) / (double)q_w;
}

/* ------------------------------------------------------------------------ */
/* Sample export: the entries of Y~.  For slots [first, first+count) */
/* of one stratum writes global coords, the nonzero index j (-1 for zeros), the   */
/* weight and the attempts used.  Returns ORC_E_REJECT_CAP with *err_slot set.    */
/* ------------------------------------------------------------------------ */
int orc_sample_export(const orc_tensor *t, int strategy, int stratum, uint64_t seed,
                      uint32_t rank, uint32_t it, int f_samples, int64_t n_stratum,
                      int64_t first, int64_t count,
                      int64_t *subs_out, int64_t *j_out, double *w_out, int32_t *att_out,
                      int64_t *err_slot)
{
    int d = t->d;
    int stratified = (strategy == ORC_STRATIFIED) || f_samples;
    if (stratum == 0) {
        if (n_stratum > 0 && t->N == 0) return ORC_E_NO_NONZEROS;
        uint32_t kind = f_samples ? KIND_F_NZ : KIND_GRAD_NZ;
        double w = weight_nz(t, n_stratum);
        for (int64_t s = first; s < first + count; ++s) {
            int64_t j = draw_nonzero(t, seed, rank, kind, it, (uint32_t)s);
            memcpy(subs_out + (s - first) * d, t->subs + j * d, sizeof(int64_t) * d);
            if (j_out) j_out[s - first] = j;
            if (w_out) w_out[s - first] = w;
            if (att_out) att_out[s - first] = 1;
        }
    } else {
        if (n_stratum > 0 && stratified && block_M(t) == (u128)t->N) return ORC_E_NO_ZEROS;
        uint32_t kind = f_samples ? KIND_F_Z : KIND_GRAD_Z;
        double w = weight_z(t, n_stratum);
        for (int64_t s = first; s < first + count; ++s) {
            int a = draw_zero(t, seed, rank, kind, it, (uint32_t)s, stratified, subs_out + (s - first) * d);
            if (a < 0) { if (err_slot) *err_slot = s; return ORC_E_REJECT_CAP; }
            if (j_out) j_out[s - first] = -1;
            if (w_out) w_out[s - first] = w;
            if (att_out) att_out[s - first] = a;
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Sparse MTTKRP of a list of entries (coords, y) (Eq. gcp-gradient, */
/* reading R2): G^(k)[i_k, r] += y * lambda_r * prod_{j != k} A^(j)[i_j, r],     */
/* in entry-list order.  G has the layout of A (block rows).                    */
/* ------------------------------------------------------------------------ */
static void mttkrp_entry(const orc_model *m, const orc_tensor *t, const int64_t *coords,
                         double y, double *G_flat, double yabs, double *S_flat)
{
    size_t off = 0;
    for (int k = 0; k < m->d; ++k) {
        int64_t row = coords[k] - t->lo[k];
        for (int r = 0; r < m->R; ++r) {
            double z = m->lambda[r];                     /* product over j != k, no division */
            for (int j = 0; j < m->d; ++j)
                if (j != k) z *= m->A[j][(coords[j] - t->lo[j]) * m->R + r];
            G_flat[off + row * m->R + r] += y * z;
            if (S_flat) S_flat[off + row * m->R + r] += yabs * fabs(z);
        }
        off += (size_t)(t->hi[k] - t->lo[k]) * (size_t)m->R;
    }
}

void orc_mttkrp(const orc_tensor *t, int R, const double *lambda, const double *A_flat,
                int64_t n, const int64_t *coords, const double *y, double *G_flat)
{
    orc_model m; make_model(&m, t, R, lambda, A_flat);
    for (int64_t e = 0; e < n; ++e) mttkrp_entry(&m, t, coords + e * t->d, y[e], G_flat, 0.0, NULL);
}

/* Y~ entry value for one sample (semi-stratified P:569-573). */
static double sample_y(int loss, int strategy, int is_nz, double w, double x, double m)
{
    if (is_nz) {
        if (strategy == ORC_SEMI_STRATIFIED)
            return w * (orc_loss_df(loss, x, m) - orc_loss_df(loss, 0.0, m));
        return w * orc_loss_df(loss, x, m);
    }
    return w * orc_loss_df(loss, 0.0, m);
}

/* Non-fused step 1: build Y~ (coords + values) for all p_w + q_w slots. */
int orc_build_Y(const orc_tensor *t, int R, const double *lambda, const double *A_flat,
                int loss, int strategy, uint64_t seed, uint32_t rank, uint32_t it,
                int64_t p_w, int64_t q_w, int64_t *coords_out, double *y_out, int64_t *err_slot)
{
    orc_model m; make_model(&m, t, R, lambda, A_flat);
    int d = t->d;
    int st;
    for (int64_t s = 0; s < p_w; ++s) {
        int64_t *c = coords_out + s * d;
        double w;
        int64_t j;
        st = orc_sample_export(t, strategy, 0, seed, rank, it, 0, p_w, s, 1, c, &j, &w, NULL, err_slot);
        if (st) return st;
        y_out[s] = sample_y(loss, strategy, 1, w, t->vals[j], model_value(&m, t, c));
    }
    for (int64_t s = 0; s < q_w; ++s) {
        int64_t *c = coords_out + (p_w + s) * d;
        double w;
        st = orc_sample_export(t, strategy, 1, seed, rank, it, 0, q_w, s, 1, c, NULL, &w, NULL, err_slot);
        if (st) return st;
        y_out[p_w + s] = sample_y(loss, strategy, 0, w, 0.0, model_value(&m, t, c));
    }
    return ORC_OK;
}

/* Fused Sampling-MTTKRP: for each sampled entry in slot order
 * (nonzero slots, then zero slots), its contribution goes straight into every
 * G^(k); Y~ is never built.  Adds into G_flat (and the tolerance scale S_flat,
 * nullable) and returns the sampled loss sum_s w f(x, m) in *loss_out. */
int orc_sampled_grad(const orc_tensor *t, int R, const double *lambda, const double *A_flat,
                     int loss, int strategy, uint64_t seed, uint32_t rank, uint32_t it,
                     int64_t p_w, int64_t q_w, double *G_flat, double *S_flat,
                     double *loss_out, double *loss_scale_out, int64_t *err_slot)
{
    orc_model m; make_model(&m, t, R, lambda, A_flat);
    int d = t->d;
    int64_t coords[32];
    double lsum = 0.0, lscale = 0.0;
    if (p_w > 0 && t->N == 0) return ORC_E_NO_NONZEROS;
    if (q_w > 0 && strategy == ORC_STRATIFIED && block_M(t) == (u128)t->N) return ORC_E_NO_ZEROS;
    double w_nz = p_w > 0 ? weight_nz(t, p_w) : 0.0;
    double w_z = q_w > 0 ? weight_z(t, q_w) : 0.0;
    for (int64_t s = 0; s < p_w; ++s) {
        int64_t j = draw_nonzero(t, seed, rank, KIND_GRAD_NZ, it, (uint32_t)s);
        memcpy(coords, t->subs + j * d, sizeof(int64_t) * d);
        double x = t->vals[j];
        double mv = model_value(&m, t, coords);
        double y = sample_y(loss, strategy, 1, w_nz, x, mv);
        double ys = 0.0;
        if (S_flat) {
            double ma = model_abs(&m, t, coords);
            ys = fabs(w_nz) * (df_scale(loss, x, mv, ma) +
                               (strategy == ORC_SEMI_STRATIFIED ? df_scale(loss, 0.0, mv, ma) : 0.0));
        }
        mttkrp_entry(&m, t, coords, y, G_flat, ys, S_flat);
        lsum += w_nz * orc_loss_f(loss, x, mv);
        if (loss_scale_out) lscale += fabs(w_nz) * f_scale(loss, x, mv, model_abs(&m, t, coords));
    }
    for (int64_t s = 0; s < q_w; ++s) {
        int a = draw_zero(t, seed, rank, KIND_GRAD_Z, it, (uint32_t)s, strategy == ORC_STRATIFIED, coords);
        if (a < 0) { if (err_slot) *err_slot = s; return ORC_E_REJECT_CAP; }
        double mv = model_value(&m, t, coords);
        double y = sample_y(loss, strategy, 0, w_z, 0.0, mv);
        double ys = S_flat ? fabs(w_z) * df_scale(loss, 0.0, mv, model_abs(&m, t, coords)) : 0.0;
        mttkrp_entry(&m, t, coords, y, G_flat, ys, S_flat);
        lsum += w_z * orc_loss_f(loss, 0.0, mv);
        if (loss_scale_out) lscale += fabs(w_z) * f_scale(loss, 0.0, mv, model_abs(&m, t, coords));
    }
    if (loss_out) *loss_out = lsum;
    if (loss_scale_out) *loss_scale_out = lscale;   /* tolerance scale of lsum (C18), as in orc_loss_estimate */
    return ORC_OK;
}

/* Loss estimate over a fixed stratified f-sample set (reading R19):
 * F^ = (N_w/f_nz) sum_nz f(x, m) + ((M_w-N_w)/f_z) sum_z f(0, m), exact rejection,
 * kinds 2/3 and iteration word 0xFFFFFFFF.  *scale_out = the same sum of |terms|
 * rounding scales (tolerance only). */
int orc_loss_estimate(const orc_tensor *t, int R, const double *lambda, const double *A_flat,
                      int loss, uint64_t seed, uint32_t rank, int64_t f_nz, int64_t f_z,
                      double *est_out, double *scale_out, int64_t *err_slot)
{
    orc_model m; make_model(&m, t, R, lambda, A_flat);
    int d = t->d;
    int64_t coords[32];
    const uint32_t it = 0xFFFFFFFFu;
    if (f_nz > 0 && t->N == 0) return ORC_E_NO_NONZEROS;
    if (f_z > 0 && block_M(t) == (u128)t->N) return ORC_E_NO_ZEROS;
    double snz = 0.0, sz = 0.0, scale = 0.0;
    double w_nz = f_nz > 0 ? weight_nz(t, f_nz) : 0.0;
    double w_z = f_z > 0 ? weight_z(t, f_z) : 0.0;
    for (int64_t s = 0; s < f_nz; ++s) {
        int64_t j = draw_nonzero(t, seed, rank, KIND_F_NZ, it, (uint32_t)s);
        memcpy(coords, t->subs + j * d, sizeof(int64_t) * d);
        double mv = model_value(&m, t, coords);
        snz += orc_loss_f(loss, t->vals[j], mv);
        scale += fabs(w_nz) * f_scale(loss, t->vals[j], mv, model_abs(&m, t, coords));
    }
    for (int64_t s = 0; s < f_z; ++s) {
        int a = draw_zero(t, seed, rank, KIND_F_Z, it, (uint32_t)s, 1, coords);
        if (a < 0) { if (err_slot) *err_slot = s; return ORC_E_REJECT_CAP; }
        double mv = model_value(&m, t, coords);
        sz += orc_loss_f(loss, 0.0, mv);
        scale += fabs(w_z) * f_scale(loss, 0.0, mv, model_abs(&m, t, coords));
    }
    *est_out = w_nz * snz + w_z * sz;
    if (scale_out) *scale_out = scale;
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Dense definitions by enumerating all M entries of the block.    */
/* Guarded: M <= 2e7.                                                          */
/* ------------------------------------------------------------------------ */
static int next_index(int64_t *c, const orc_tensor *t)
{
    for (int k = t->d - 1; k >= 0; --k) {
        if (++c[k] < t->hi[k]) return 1;
        c[k] = t->lo[k];
    }
    return 0;
}

static double lookup_value(const orc_tensor *t, const int64_t *coords)
{
    int64_t a = 0, b = t->N;
    while (a < b) {
        int64_t mid = a + (b - a) / 2;
        int c = lex_cmp(t->subs + mid * t->d, coords, t->d);
        if (c == 0) return t->vals[mid];
        if (c < 0) a = mid + 1; else b = mid;
    }
    return 0.0;
}

/* F(X, M) = sum over all i of f(x_i, m_i)  (Eq. gcp-model) */
int orc_full_loss(const orc_tensor *t, int R, const double *lambda, const double *A_flat,
                  int loss, double *out)
{
    if (block_M(t) > (u128)20000000) return ORC_E_ARG;
    orc_model m; make_model(&m, t, R, lambda, A_flat);
    int64_t c[32];
    for (int k = 0; k < t->d; ++k) c[k] = t->lo[k];
    double F = 0.0;
    if (block_M(t) > 0) do {
        F += orc_loss_f(loss, lookup_value(t, c), model_value(&m, t, c));
    } while (next_index(c, t));
    *out = F;
    return ORC_OK;
}

/* G^(k) = Y_(k) Z_k with y_i = df/dm(x_i, m_i) over ALL entries. */
int orc_full_grad(const orc_tensor *t, int R, const double *lambda, const double *A_flat,
                  int loss, double *G_flat)
{
    if (block_M(t) > (u128)20000000) return ORC_E_ARG;
    orc_model m; make_model(&m, t, R, lambda, A_flat);
    int64_t c[32];
    for (int k = 0; k < t->d; ++k) c[k] = t->lo[k];
    if (block_M(t) > 0) do {
        double y = orc_loss_df(loss, lookup_value(t, c), model_value(&m, t, c));
        mttkrp_entry(&m, t, c, y, G_flat, 0.0, NULL);
    } while (next_index(c, t));
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Adam update, Alg. 1, one pass over the contiguous array         */
/* (P:634-640).  t is the step number after increment (reading R7).           */
/* ------------------------------------------------------------------------ */
void orc_adam(int64_t n, double *A, const double *G, double *B, double *C, int64_t t,
              double alpha, double beta1, double beta2, double eps, double lower)
{
    double bc1 = 1.0 - pow(beta1, (double)t);
    double bc2 = 1.0 - pow(beta2, (double)t);
    for (int64_t i = 0; i < n; ++i) {
        B[i] = beta1 * B[i] + (1.0 - beta1) * G[i];                 /* line 5 */
        C[i] = beta2 * C[i] + (1.0 - beta2) * G[i] * G[i];          /* line 6 */
        double Bh = B[i] / bc1;                                     /* line 7 */
        double Ch = C[i] / bc2;                                     /* line 8 */
        A[i] = A[i] - alpha * (Bh / sqrt(Ch + eps));                /* line 9, eps inside sqrt */
        if (A[i] < lower) A[i] = lower;                             /* line 10, max{A, l} */
    }
}

/* ------------------------------------------------------------------------ */
/* Factor initialisation (reading R12): element e of the unpadded mode-major    */
/* concatenation of the GLOBAL factors = (W0 >> 11) * 2^-53 of Philox counter   */
/* (lo32 e, hi32 e, 4<<28, 0) under the init seed.                              */
/* ------------------------------------------------------------------------ */
void orc_factor_init(uint64_t seed, int d, const int64_t *dims, int R, double *out)
{
    int64_t total = 0;
    for (int k = 0; k < d; ++k) total += dims[k] * R;
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    for (int64_t e = 0; e < total; ++e) {
        uint32_t ctr[4] = { (uint32_t)e, (uint32_t)((uint64_t)e >> 32), (uint32_t)KIND_INIT << 28, 0 };
        uint32_t o[4];
        orc_philox4x32_10(ctr, key, o);
        uint64_t W0 = (uint64_t)o[0] | ((uint64_t)o[1] << 32);
        out[e] = (double)(W0 >> 11) * 0x1.0p-53;
    }
}

/* ------------------------------------------------------------------------ */
/* Medium-grained grid: over all ordered d-tuples (N_1..N_d) with  */
/* prod N_k = P, minimise sum_k I_k * P/N_k; ties -> lexicographically smallest */
/* (reading R14).  Returns the objective.                                       */
/* ------------------------------------------------------------------------ */
static void grid_rec(int P, int d, const int64_t *dims, int k, int rem, int *cur,
                     int *best, double *best_obj)
{
    if (k == d - 1) {
        cur[k] = rem;
        double obj = 0.0;
        for (int j = 0; j < d; ++j) obj += (double)dims[j] * (double)(P / cur[j]);
        /* enumeration is in lexicographic order, so strict < keeps the smallest tuple */
        if (obj < *best_obj) { *best_obj = obj; memcpy(best, cur, sizeof(int) * d); }
        return;
    }
    for (int n = 1; n <= rem; ++n)
        if (rem % n == 0) { cur[k] = n; grid_rec(P, d, dims, k + 1, rem / n, cur, best, best_obj); }
}

double orc_grid_plan(int P, int d, const int64_t *dims, int *grid_out)
{
    int cur[32];
    double best = INFINITY;
    grid_rec(P, d, dims, 0, P, cur, grid_out, &best);
    return best;
}

/* ------------------------------------------------------------------------ */
/* OpenMP timing variants (built with -fopenmp).  Same    */
/* estimator and the same draws as orc_sampled_grad / orc_loss_estimate /      */
/* orc_adam: the slots of each stratum split into nthreads contiguous ranges,   */
/* thread-private G and sums, reduced in thread order.  Used only to time the   */
/* CPU baseline on all host cores; pinned to the serial functions (fixed        */
/* summation order aside) in tests/test_oracle_estimators.py.                  */
/* ------------------------------------------------------------------------ */
static int grad_range(const orc_tensor *t, const orc_model *m, int loss, int strategy, uint64_t seed,
                      uint32_t rank, uint32_t it, double w_nz, double w_z, int64_t nz0, int64_t nz1,
                      int64_t z0, int64_t z1, double *G_flat, double *lsum)
{
    int d = t->d;
    int64_t coords[32];
    for (int64_t s = nz0; s < nz1; ++s) {
        int64_t j = draw_nonzero(t, seed, rank, KIND_GRAD_NZ, it, (uint32_t)s);
        memcpy(coords, t->subs + j * d, sizeof(int64_t) * d);
        double x = t->vals[j];
        double mv = model_value(m, t, coords);
        mttkrp_entry(m, t, coords, sample_y(loss, strategy, 1, w_nz, x, mv), G_flat, 0.0, NULL);
        *lsum += w_nz * orc_loss_f(loss, x, mv);
    }
    for (int64_t s = z0; s < z1; ++s) {
        if (draw_zero(t, seed, rank, KIND_GRAD_Z, it, (uint32_t)s, strategy == ORC_STRATIFIED, coords) < 0)
            return ORC_E_REJECT_CAP;
        double mv = model_value(m, t, coords);
        mttkrp_entry(m, t, coords, sample_y(loss, strategy, 0, w_z, 0.0, mv), G_flat, 0.0, NULL);
        *lsum += w_z * orc_loss_f(loss, 0.0, mv);
    }
    return ORC_OK;
}

static int64_t coef_count(const orc_tensor *t, int R)
{
    int64_t n = 0;
    for (int k = 0; k < t->d; ++k) n += (t->hi[k] - t->lo[k]) * (int64_t)R;
    return n;
}

int orc_sampled_grad_par(const orc_tensor *t, int R, const double *lambda, const double *A_flat,
                         int loss, int strategy, uint64_t seed, uint32_t rank, uint32_t it,
                         int64_t p_w, int64_t q_w, double *G_flat, double *loss_out, int nthreads)
{
    orc_model m; make_model(&m, t, R, lambda, A_flat);
    if (p_w > 0 && t->N == 0) return ORC_E_NO_NONZEROS;
    if (q_w > 0 && strategy == ORC_STRATIFIED && block_M(t) == (u128)t->N) return ORC_E_NO_ZEROS;
    if (nthreads < 1) nthreads = 1;
    double w_nz = p_w > 0 ? weight_nz(t, p_w) : 0.0;
    double w_z = q_w > 0 ? weight_z(t, q_w) : 0.0;
    int64_t nc = coef_count(t, R);
    double *priv = calloc((size_t)nthreads * (size_t)nc, sizeof(double));
    double *ls = calloc((size_t)nthreads, sizeof(double));
    int *st = calloc((size_t)nthreads, sizeof(int));
    if (!priv || !ls || !st) { free(priv); free(ls); free(st); return ORC_E_OOM; }
#pragma omp parallel for num_threads(nthreads) schedule(static, 1)
    for (int w = 0; w < nthreads; ++w)
        st[w] = grad_range(t, &m, loss, strategy, seed, rank, it, w_nz, w_z,
                           p_w * w / nthreads, p_w * (w + 1) / nthreads,
                           q_w * w / nthreads, q_w * (w + 1) / nthreads, priv + (size_t)w * nc, &ls[w]);
    int rc = ORC_OK;
    double lsum = 0.0;
    for (int w = 0; w < nthreads; ++w) {
        if (st[w]) rc = st[w];
        lsum += ls[w];
    }
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (int64_t e = 0; e < nc; ++e) {
        double a = G_flat[e];
        for (int w = 0; w < nthreads; ++w) a += priv[(size_t)w * nc + e];   /* fixed thread order */
        G_flat[e] = a;
    }
    if (loss_out) *loss_out = lsum;
    free(priv); free(ls); free(st);
    return rc;
}

int orc_loss_estimate_par(const orc_tensor *t, int R, const double *lambda, const double *A_flat,
                          int loss, uint64_t seed, uint32_t rank, int64_t f_nz, int64_t f_z,
                          double *est_out, int nthreads)
{
    orc_model m; make_model(&m, t, R, lambda, A_flat);
    const uint32_t it = 0xFFFFFFFFu;
    if (f_nz > 0 && t->N == 0) return ORC_E_NO_NONZEROS;
    if (f_z > 0 && block_M(t) == (u128)t->N) return ORC_E_NO_ZEROS;
    if (nthreads < 1) nthreads = 1;
    double w_nz = f_nz > 0 ? weight_nz(t, f_nz) : 0.0;
    double w_z = f_z > 0 ? weight_z(t, f_z) : 0.0;
    double *snz = calloc((size_t)nthreads, sizeof(double)), *sz = calloc((size_t)nthreads, sizeof(double));
    int *st = calloc((size_t)nthreads, sizeof(int));
    if (!snz || !sz || !st) { free(snz); free(sz); free(st); return ORC_E_OOM; }
#pragma omp parallel for num_threads(nthreads) schedule(static, 1)
    for (int w = 0; w < nthreads; ++w) {
        int64_t coords[32];
        for (int64_t s = f_nz * w / nthreads; s < f_nz * (w + 1) / nthreads; ++s) {
            int64_t j = draw_nonzero(t, seed, rank, KIND_F_NZ, it, (uint32_t)s);
            memcpy(coords, t->subs + j * t->d, sizeof(int64_t) * t->d);
            snz[w] += orc_loss_f(loss, t->vals[j], model_value(&m, t, coords));
        }
        for (int64_t s = f_z * w / nthreads; s < f_z * (w + 1) / nthreads; ++s) {
            if (draw_zero(t, seed, rank, KIND_F_Z, it, (uint32_t)s, 1, coords) < 0) { st[w] = ORC_E_REJECT_CAP; break; }
            sz[w] += orc_loss_f(loss, 0.0, model_value(&m, t, coords));
        }
    }
    double a = 0.0, b = 0.0;
    int rc = ORC_OK;
    for (int w = 0; w < nthreads; ++w) { a += snz[w]; b += sz[w]; if (st[w]) rc = st[w]; }
    *est_out = w_nz * a + w_z * b;
    free(snz); free(sz); free(st);
    return rc;
}

void orc_adam_par(int64_t n, double *A, const double *G, double *B, double *C, int64_t t,
                  double alpha, double beta1, double beta2, double eps, double lower, int nthreads)
{
    double bc1 = 1.0 - pow(beta1, (double)t);
    double bc2 = 1.0 - pow(beta2, (double)t);
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        B[i] = beta1 * B[i] + (1.0 - beta1) * G[i];
        C[i] = beta2 * C[i] + (1.0 - beta2) * G[i] * G[i];
        double a = A[i] - alpha * ((B[i] / bc1) / sqrt(C[i] / bc2 + eps));
        A[i] = a < lower ? lower : a;
    }
}
