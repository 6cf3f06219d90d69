/*
 * oracle/hc_oracle.c -- plain, slow, obviously-correct CPU reference of the
 * HCAttention decode hot path (arXiv 2507.19823, §3.2 "Heterogeneous
 * Attention Computation", Eqs. 1-5).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2507_19823_b200/csrc).  Citations: "P:n" = line n of
 * /root/reference/PAPER.md; "R<k>" = the numbered reading in DESIGN.md §2.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (no fast-math), so
 * every float operation below is one IEEE-754 binary32 operation, in the
 * order written.  fmaf() is the correctly-rounded fused multiply-add.
 *
 * Parity status: every function is pinned by tests/test_oracle_pins.py
 * except or_decode_unit's absolute accuracy at tau<1 ("parity unpinned",
 * DESIGN.md C-P10 -- the paper prints no numbers for it).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_EXPORT __attribute__((visibility("default")))

/* IEEE binary16 -> binary32, exact (bit-level). */
static float or_h2f(uint16_t h)
{
    uint32_t sign = (uint32_t)(h >> 15) << 31;
    uint32_t exp = (h >> 10) & 0x1f;
    uint32_t man = h & 0x3ff;
    uint32_t bits;
    if (exp == 0) {
        if (man == 0) {
            bits = sign;
        } else { /* subnormal: value = man * 2^-24 */
            float v = (float)man * 0x1p-24f;
            memcpy(&bits, &v, 4);
            bits |= sign;
        }
    } else if (exp == 31) {
        bits = sign | 0x7f800000u | (man << 13);
    } else {
        bits = sign | ((exp + 112u) << 23) | (man << 13);
    }
    float f;
    memcpy(&f, &bits, 4);
    return f;
}

OR_EXPORT float or_half_to_float(uint16_t h) { return or_h2f(h); }

/* ------------------------------------------------------------------------
 * R1 -- key encoding.  P:227 (§3.2): "Each sub-group is represented as nearest
 * neighbor of the centroids in the codebook ... an index matrix P".  Metric
 * unstated -> squared Euclidean; ties -> lowest centroid index (DESIGN R1).
 *   dist = 0; for e: diff = k[e] - C[m][e]; dist = fmaf(diff, diff, dist)
 *   code = argmin_m dist, strict '<' in ascending m.
 * keys [rows][d] fp16; C [cbg][c][dbar] fp32; codes out row-major [rows][g].
 * ---------------------------------------------------------------------- */
OR_EXPORT void or_encode(const uint16_t *keys, int64_t rows, int d, int g, int c, int cbg,
                         const float *C, uint16_t *codes)
{
    const int dbar = d / g;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; ++r) {
        for (int i = 0; i < g; ++i) {
            const float *Ci = C + (size_t)(cbg == 1 ? 0 : i) * c * dbar;
            float kbar[64];
            for (int e = 0; e < dbar; ++e) kbar[e] = or_h2f(keys[r * d + i * dbar + e]);
            int best = 0;
            float best_dist = 0.0f;
            for (int m = 0; m < c; ++m) {
                float dist = 0.0f;
                for (int e = 0; e < dbar; ++e) {
                    float diff = kbar[e] - Ci[(size_t)m * dbar + e];
                    dist = fmaf(diff, diff, dist);
                }
                if (m == 0 || dist < best_dist) {
                    best_dist = dist;
                    best = m;
                }
            }
            codes[r * g + i] = (uint16_t)best;
        }
    }
}

/* ------------------------------------------------------------------------
 * f4 -- one MiniBatchKMeans step ("MiniBatchKMeans [Sculley 2010] implemented in
 * Scikit-learn ... batch size of 10,000"; codebooks per group, §3.1).  Sculley's
 * Alg. 1 with the per-centre learning rate 1/v, in its batched (scikit-learn) form:
 *   1. labels: every sampled key's sub-vectors are assigned with the centres as they are
 *      at the start of the step -- R1's nearest-centroid rule (or_encode);
 *   2. per centre m of codebook slice ci: n_m = #assigned, s_m = Σ assigned sub-vectors;
 *      if n_m > 0:  C_m <- (C_m·v_m + s_m) / (v_m + n_m),  v_m <- v_m + n_m
 *      (= Alg. 1's sequential updates c <- (1-1/v)c + x/v over the batch).
 * Arithmetic (DESIGN F4): s_m exact in int64 units of 2^-24 (every fp16 value is an
 * integer multiple of 2^-24 below 2^16); the update in double, written as
 *   q = ((double)C·(double)v + (double)s·2^-24) / (double)(v + n),  C = (float)q (RN).
 * sample [b] = key row indices (the caller draws them); labels [b][g] (optional).
 * ---------------------------------------------------------------------- */
OR_EXPORT int or_kmeans_step(const uint16_t *keys, int64_t n_keys, int d, int g, int c, int cbg,
                             const int64_t *sample, int64_t b, float *C, int64_t *counts,
                             uint16_t *labels)
{
    const int dbar = d / g;
    if (b <= 0) return 0;
    uint16_t *batch = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)b * d);
    uint16_t *lab = labels ? labels : (uint16_t *)malloc(sizeof(uint16_t) * (size_t)b * g);
    for (int64_t s = 0; s < b; ++s) {
        if (sample[s] < 0 || sample[s] >= n_keys) return 3;
        memcpy(batch + s * d, keys + sample[s] * d, sizeof(uint16_t) * (size_t)d);
    }
    or_encode(batch, b, d, g, c, cbg, C, lab);
    int64_t *S = (int64_t *)calloc((size_t)cbg * c * dbar, sizeof(int64_t));
    int64_t *n = (int64_t *)calloc((size_t)cbg * c, sizeof(int64_t));
    for (int64_t s = 0; s < b; ++s)
        for (int i = 0; i < g; ++i) {
            const int ci = cbg == 1 ? 0 : i;
            const int m = lab[s * g + i];
            n[(size_t)ci * c + m] += 1;
            for (int e = 0; e < dbar; ++e)
                S[((size_t)ci * c + m) * dbar + e] +=
                    (int64_t)ldexp((double)or_h2f(batch[s * d + i * dbar + e]), 24);
        }
    for (int64_t cm = 0; cm < (int64_t)cbg * c; ++cm) {
        if (!n[cm]) continue;
        const int64_t v = counts[cm];
        for (int e = 0; e < dbar; ++e) {
            const double num = (double)C[cm * dbar + e] * (double)v + (double)S[cm * dbar + e] * 0x1p-24;
            C[cm * dbar + e] = (float)(num / (double)(v + n[cm]));
        }
        counts[cm] = v + n[cm];
    }
    free(S);
    free(n);
    free(batch);
    if (!labels) free(lab);
    return 0;
}

/* Eq. 2 Q(K): row j = concat_i C[i][P[j][i]]. codes [n][g] row-major. */
OR_EXPORT void or_reconstruct(const uint16_t *codes, int64_t n, int d, int g, int c, int cbg,
                              const float *C, float *out)
{
    const int dbar = d / g;
    for (int64_t j = 0; j < n; ++j)
        for (int i = 0; i < g; ++i) {
            const float *Ci = C + (size_t)(cbg == 1 ? 0 : i) * c * dbar;
            for (int e = 0; e < dbar; ++e)
                out[j * d + i * dbar + e] = Ci[(size_t)codes[j * g + i] * dbar + e];
        }
}

/* ------------------------------------------------------------------------
 * R2 -- query/codebook table.  P:229: "T = q̄·C where T ∈ R^{g×c}".
 *   t = q[i*dbar]*C[i][m][0]; t = fmaf(q[i*dbar+e], C[i][m][e], t), e=1..dbar-1
 * Fixed-point storage (DESIGN R2): one power-of-two scale per query head from the
 * Cauchy-Schwarz-style bound (computable before any table entry exists):
 *   Cabs[ci][e] = max_m |C[ci][m][e]|
 *   A_i = |q_0|*Cabs[ci][0]; A_i = fmaf(|q_e|, Cabs[ci][e], A_i)   (same chain as t)
 *   A   = max_i A_i    (>= |t| for every entry, exactly, by monotone rounding)
 *   e_h = 100 if A < 2^-100 else clamp(top - floor(log2 A), -100, 100);
 *   T_fx = clamp(rint(t * 2^e_h), -Tmax, Tmax)   (rint = ties-to-even)
 * with (top, Tmax) = (14, 32767) for the default 16-bit table and (6, 127) for the 8-bit
 * table variant (DESIGN R2b).
 * q [G][d] fp16 -> T32 [G][g][c] fp32 (may be NULL), Tfx [G][g][c] int16, e [G].
 * ---------------------------------------------------------------------- */
static float or_pow2f(int e) /* exact 2^e for -126 <= e <= 127 */
{
    uint32_t bits = (uint32_t)(e + 127) << 23;
    float f;
    memcpy(&f, &bits, 4);
    return f;
}

/* Cabs[ci][e] = max over centroids m of |C[ci][m][e]|  -> out [cbg][dbar] */
OR_EXPORT void or_codebook_absmax(const float *C, int cbg, int c, int dbar, float *out)
{
    for (int ci = 0; ci < cbg; ++ci)
        for (int e = 0; e < dbar; ++e) {
            float mx = 0.0f;
            for (int m = 0; m < c; ++m) {
                float a = fabsf(C[((size_t)ci * c + m) * dbar + e]);
                if (a > mx) mx = a;
            }
            out[ci * dbar + e] = mx;
        }
}

/* A_h of R2 for one query head q [d] */
OR_EXPORT float or_table_bound(const uint16_t *q, int d, int g, int cbg, const float *Cabs)
{
    const int dbar = d / g;
    float A = 0.0f;
    for (int i = 0; i < g; ++i) {
        const float *ca = Cabs + (size_t)(cbg == 1 ? 0 : i) * dbar;
        float b = fabsf(or_h2f(q[i * dbar])) * ca[0];
        for (int e = 1; e < dbar; ++e) b = fmaf(fabsf(or_h2f(q[i * dbar + e])), ca[e], b);
        if (b > A) A = b;
    }
    return A;
}

static int or_scale_exponent_top(float A, int top)
{
    if (!(A >= 0x1p-100f)) return 100;
    int ex;
    (void)frexpf(A, &ex); /* A = f * 2^ex, f in [0.5, 1) -> floor(log2 A) = ex - 1 */
    int e = top - (ex - 1);
    if (e < -100) e = -100;
    if (e > 100) e = 100;
    return e;
}

OR_EXPORT int or_scale_exponent(float A) { return or_scale_exponent_top(A, 14); }

OR_EXPORT void or_table_bits(const uint16_t *q, int G, int d, int g, int c, int cbg, const float *C,
                             float *T32, int16_t *Tfx, int32_t *e_out, int lut_bits)
{
    const int dbar = d / g;
    const int top = lut_bits == 8 ? 6 : 14;
    const float tmax = lut_bits == 8 ? 127.0f : 32767.0f;
    float *t = (float *)malloc(sizeof(float) * (size_t)g * c);
    float *Cabs = (float *)malloc(sizeof(float) * (size_t)cbg * dbar);
    or_codebook_absmax(C, cbg, c, dbar, Cabs);
    for (int h = 0; h < G; ++h) {
        for (int i = 0; i < g; ++i) {
            const float *Ci = C + (size_t)(cbg == 1 ? 0 : i) * c * dbar;
            for (int m = 0; m < c; ++m) {
                float acc = or_h2f(q[h * d + i * dbar]) * Ci[(size_t)m * dbar];
                for (int e = 1; e < dbar; ++e)
                    acc = fmaf(or_h2f(q[h * d + i * dbar + e]), Ci[(size_t)m * dbar + e], acc);
                t[(size_t)i * c + m] = acc;
            }
        }
        int e_h = or_scale_exponent_top(or_table_bound(q + (size_t)h * d, d, g, cbg, Cabs), top);
        float s = or_pow2f(e_h);
        for (size_t k = 0; k < (size_t)g * c; ++k) {
            float v = rintf(t[k] * s);
            if (v > tmax) v = tmax;
            if (v < -tmax) v = -tmax;
            Tfx[(size_t)h * g * c + k] = (int16_t)v;
            if (T32) T32[(size_t)h * g * c + k] = t[k];
        }
        e_out[h] = e_h;
    }
    free(Cabs);
    free(t);
}

OR_EXPORT void or_table(const uint16_t *q, int G, int d, int g, int c, int cbg, const float *C,
                        float *T32, int16_t *Tfx, int32_t *e_out)
{
    or_table_bits(q, G, d, g, c, cbg, C, T32, Tfx, e_out, 16);
}

/* ------------------------------------------------------------------------
 * R3 -- approximate scores, Eq. 3: z̃_j = Σ_{i=1..g} T_{i,P_{j,i}}.
 * Integer (exact) sum of the fixed-point table entries.  P is group-major:
 * P[i*stride + j].  Tfx for ONE head [g][c].
 * ---------------------------------------------------------------------- */
OR_EXPORT void or_scores(const int16_t *Tfx, const uint16_t *P, int64_t n, int64_t stride, int g,
                         int c, int32_t *z)
{
    for (int64_t j = 0; j < n; ++j) {
        int32_t acc = 0;
        for (int i = 0; i < g; ++i) acc += Tfx[(size_t)i * c + P[(size_t)i * stride + j]];
        z[j] = acc;
    }
}

/* Resident (unquantized recent-window) tokens score exactly (SPEC S:449,
 * DESIGN R3b): acc = fmaf chain over e = 0..d-1; then onto the same grid:
 *   z_fx = rint(clamp(acc * 2^e_h, -2^22, 2^22)). */
OR_EXPORT void or_resident_scores(const uint16_t *q, const uint16_t *rk, int64_t nres, int d,
                                  int e_h, int32_t *z)
{
    float s = or_pow2f(e_h);
    for (int64_t r = 0; r < nres; ++r) {
        float acc = 0.0f;
        for (int e = 0; e < d; ++e) acc = fmaf(or_h2f(q[e]), or_h2f(rk[r * d + e]), acc);
        float v = acc * s;
        if (v > 4194304.0f) v = 4194304.0f;
        if (v < -4194304.0f) v = -4194304.0f;
        z[r] = (int32_t)rintf(v);
    }
}

/* ------------------------------------------------------------------------
 * R4 -- normalisation ã = softmax(z̃/√d) as exact fixed-point mass.
 *   kappa_h = fp32(log2(e)/sqrt(d)) * 2^-e_h
 *   x = -(float)Δ * kappa_h, Δ = M - z_j
 *   exp2_det(x): x < -40 -> W = 0; n = floor(x); f = x - n;
 *                p = Horner(c6..c0, f) with fmaf;  W = trunc(p * 2^(40+n))
 *   ã_j = W_j / S,  S = Σ_j W_j  (uint64, exact).
 * Coefficients: degree-6 fit of 2^f on [0,1), DESIGN R4 (max rel err 6.2e-8).
 * ---------------------------------------------------------------------- */
OR_EXPORT float or_kappa(int d, int e_h)
{
    float k0 = (float)(1.4426950408889634 / sqrt((double)d));
    return k0 * or_pow2f(-e_h);
}

OR_EXPORT float or_exp2_poly(float f)
{
    const float c0 = 0x1.000000p+0f, c1 = 0x1.62e42ap-1f, c2 = 0x1.ebfd9ap-3f,
                c3 = 0x1.c68562p-5f, c4 = 0x1.3d24eap-7f, c5 = 0x1.46301cp-10f,
                c6 = 0x1.c6e292p-13f;
    float p = c6;
    p = fmaf(p, f, c5);
    p = fmaf(p, f, c4);
    p = fmaf(p, f, c3);
    p = fmaf(p, f, c2);
    p = fmaf(p, f, c1);
    p = fmaf(p, f, c0);
    return p;
}

OR_EXPORT uint64_t or_mass(uint32_t delta, float kappa)
{
    float x = -((float)delta * kappa);
    if (x < -40.0f) return 0;
    float nf = floorf(x);
    float f = x - nf;
    float p = or_exp2_poly(f);
    float v = p * or_pow2f(40 + (int)nf);
    return (uint64_t)v; /* truncation toward zero */
}

/* ------------------------------------------------------------------------
 * R5 -- cumulative-magnitude eviction, Eq. 4:
 *   sort ã descending (ties: lower index first, DESIGN R5);
 *   k* = min{k : Σ_{r<=k} a_(r) >= τ}  evaluated exactly as
 *        Σ_{r<=k} W_(r) >= Θ,  Θ = ceil(τ_q·S / 2^24), τ_q = rint(τ·2^24);
 *   τ_q >= 2^24 (τ = 1) -> k* = n;   k_sel = min(k*, k_max).
 * Outputs idx ascending, weights W_j/S (renorm: W_j / Σ_sel W).
 * ---------------------------------------------------------------------- */
typedef struct {
    uint32_t delta;
    int64_t j;
} or_item;

static int or_cmp(const void *a, const void *b)
{
    const or_item *x = (const or_item *)a, *y = (const or_item *)b;
    if (x->delta != y->delta) return x->delta < y->delta ? -1 : 1;
    return x->j < y->j ? -1 : (x->j > y->j ? 1 : 0);
}

static int or_cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

OR_EXPORT uint64_t or_threshold(uint32_t tau_q, uint64_t S)
{
    unsigned __int128 p = (unsigned __int128)tau_q * (unsigned __int128)S;
    p += ((unsigned __int128)1 << 24) - 1;
    return (uint64_t)(p >> 24);
}

OR_EXPORT uint32_t or_tau_q(float tau) { return (uint32_t)rint((double)tau * 16777216.0); }

/* z [n] int32 fixed-point scores of one head (quantized then resident). */
OR_EXPORT int or_select(const int32_t *z, int64_t n, int e_h, int d, float tau, int64_t k_max,
                        int renorm, int32_t *idx_out, double *w_out, int64_t *k_sel_out,
                        uint64_t *S_out, int32_t *M_out, int64_t *kstar_out)
{
    if (n <= 0) return 5;
    int32_t M = z[0];
    for (int64_t j = 1; j < n; ++j)
        if (z[j] > M) M = z[j];
    float kappa = or_kappa(d, e_h);
    or_item *it = (or_item *)malloc(sizeof(or_item) * (size_t)n);
    uint64_t S = 0;
    for (int64_t j = 0; j < n; ++j) {
        it[j].delta = (uint32_t)((int64_t)M - (int64_t)z[j]);
        it[j].j = j;
        S += or_mass(it[j].delta, kappa);
    }
    qsort(it, (size_t)n, sizeof(or_item), or_cmp);
    uint32_t tq = or_tau_q(tau);
    int64_t kstar;
    if (tq >= 16777216u) {
        kstar = n;
    } else {
        uint64_t theta = or_threshold(tq, S);
        uint64_t cum = 0;
        kstar = n;
        for (int64_t k = 1; k <= n; ++k) {
            cum += or_mass(it[k - 1].delta, kappa);
            if (cum >= theta) {
                kstar = k;
                break;
            }
        }
    }
    int64_t ksel = kstar < k_max ? kstar : k_max;
    int64_t *sel = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ksel > 0 ? ksel : 1));
    uint64_t selmass = 0;
    for (int64_t k = 0; k < ksel; ++k) {
        sel[k] = it[k].j;
        selmass += or_mass(it[k].delta, kappa);
    }
    qsort(sel, (size_t)ksel, sizeof(int64_t), or_cmp_i64);
    double denom = renorm ? (double)selmass : (double)S;
    for (int64_t k = 0; k < ksel; ++k) {
        idx_out[k] = (int32_t)sel[k];
        uint64_t W = or_mass((uint32_t)((int64_t)M - (int64_t)z[sel[k]]), kappa);
        w_out[k] = (double)W / denom;
    }
    *k_sel_out = ksel;
    if (S_out) *S_out = S;
    if (M_out) *M_out = M;
    if (kstar_out) *kstar_out = kstar;
    free(sel);
    free(it);
    return 0;
}

/* Standalone selection on real-valued scores (hc_select_topk's input), DESIGN
 * R5b: A = max|z|; e = 100 if A < 2^-100 else clamp(22 - floor(log2 A) - 1, -100,
 * 100) so |z·2^e| < 2^22; z_fx = rint(clamp(z·2^e, ±2^22)); then or_select. */
/* The R5b grid alone: returns e and writes z_fx [n] (step 1 of or_select_float). */
OR_EXPORT int or_float_grid(const float *zf, int64_t n, int32_t *z)
{
    float A = 0.0f;
    for (int64_t j = 0; j < n; ++j)
        if (fabsf(zf[j]) > A) A = fabsf(zf[j]);
    int e = 100;
    if (A >= 0x1p-100f) {
        int ex;
        (void)frexpf(A, &ex);
        e = 21 - (ex - 1);
        if (e < -100) e = -100;
        if (e > 100) e = 100;
    }
    float s = or_pow2f(e);
    for (int64_t j = 0; j < n; ++j) {
        float v = zf[j] * s;
        if (v > 4194304.0f) v = 4194304.0f;
        if (v < -4194304.0f) v = -4194304.0f;
        z[j] = (int32_t)rintf(v);
    }
    return e;
}

OR_EXPORT int or_select_float(const float *zf, int64_t n, int d, float tau, int64_t k_max,
                              int renorm, int32_t *idx_out, double *w_out, int64_t *k_sel_out)
{
    if (n <= 0) return 5;
    int32_t *z = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int e = or_float_grid(zf, n, z);
    int rc = or_select(z, n, e, d, tau, k_max, renorm, idx_out, w_out, k_sel_out, 0, 0, 0);
    free(z);
    return rc;
}

/* ------------------------------------------------------------------------
 * R8 (NEXT f3(iii); SURVEY F8 "per query head or per KV head") -- shared selection
 * per KV head.  Reading (DESIGN.md §2 R8): the G query heads of one KV head keep ONE
 * index set, chosen by Eq. 4 applied to their head-averaged attention
 * distribution ā_j = (1/G) Σ_h ã_{h,j} (ã from Eq. 2's softmax).  Exactly:
 *   W_{h,j} = R4 mass of head h (own M_h, κ_h);      S_h = Σ_j W_{h,j};
 *   ρ_h = floor((2^104 - 1) / S_h);                   Â_{h,j} = floor(W_{h,j}·ρ_h / 2^64)
 *   (≈ 2^40·ã_{h,j});  A_j = Σ_h Â_{h,j} (≈ G·2^40·ā_j);  S_A = Σ_j A_j;
 *   Θ = ceil(τ_q·S_A / 2^24); order (A desc, j asc); k* = min{k : Σ_{r<k} A_(r) >= Θ};
 *   τ_q >= 2^24 -> all; k_sel = min(k*, k_max).
 * Each head h then applies Eq. 5 with its OWN weights W_{h,j} / S_h over the shared set
 * (w_out[h][k], idx ascending).  z [G][n] int32 fixed-point scores, e [G] their exponents.
 * ---------------------------------------------------------------------- */
typedef struct {
    uint64_t A;
    int64_t j;
} or_gitem;

static int or_cmp_g(const void *a, const void *b)
{
    const or_gitem *x = (const or_gitem *)a, *y = (const or_gitem *)b;
    if (x->A != y->A) return x->A > y->A ? -1 : 1; /* A descending */
    return x->j < y->j ? -1 : (x->j > y->j ? 1 : 0);
}

OR_EXPORT int or_select_shared(const int32_t *z, int G, int64_t n, const int32_t *e, int d,
                               float tau, int64_t k_max, int32_t *idx_out, double *w_out,
                               int64_t *k_sel_out, uint64_t *SA_out, int64_t *kstar_out,
                               uint64_t *A_out)
{
    if (n <= 0) return 5;
    if (G < 1 || G > 8) return 1;
    int32_t M[8];
    float kap[8];
    uint64_t S[8], rho[8];
    for (int h = 0; h < G; ++h) {
        const int32_t *zh = z + (size_t)h * n;
        M[h] = zh[0];
        for (int64_t j = 1; j < n; ++j)
            if (zh[j] > M[h]) M[h] = zh[j];
        kap[h] = or_kappa(d, e[h]);
        S[h] = 0;
        for (int64_t j = 0; j < n; ++j)
            S[h] += or_mass((uint32_t)((int64_t)M[h] - (int64_t)zh[j]), kap[h]);
        unsigned __int128 num = ((unsigned __int128)1 << 104) - 1;
        rho[h] = (uint64_t)(num / S[h]);
    }
    or_gitem *it = (or_gitem *)malloc(sizeof(or_gitem) * (size_t)n);
    uint64_t SA = 0;
    for (int64_t j = 0; j < n; ++j) {
        uint64_t A = 0;
        for (int h = 0; h < G; ++h) {
            uint64_t W = or_mass((uint32_t)((int64_t)M[h] - (int64_t)z[(size_t)h * n + j]), kap[h]);
            A += (uint64_t)(((unsigned __int128)W * rho[h]) >> 64);
        }
        it[j].A = A;
        it[j].j = j;
        if (A_out) A_out[j] = A;
        SA += A;
    }
    qsort(it, (size_t)n, sizeof(or_gitem), or_cmp_g);
    uint32_t tq = or_tau_q(tau);
    int64_t kstar = n;
    if (tq < 16777216u) {
        uint64_t theta = or_threshold(tq, SA), cum = 0;
        for (int64_t k = 1; k <= n; ++k) {
            cum += it[k - 1].A;
            if (cum >= theta) {
                kstar = k;
                break;
            }
        }
    }
    int64_t ksel = kstar < k_max ? kstar : k_max;
    int64_t *sel = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ksel > 0 ? ksel : 1));
    for (int64_t k = 0; k < ksel; ++k) sel[k] = it[k].j;
    qsort(sel, (size_t)ksel, sizeof(int64_t), or_cmp_i64);
    for (int64_t k = 0; k < ksel; ++k) {
        idx_out[k] = (int32_t)sel[k];
        for (int h = 0; h < G; ++h) {
            uint64_t W = or_mass((uint32_t)((int64_t)M[h] - (int64_t)z[(size_t)h * n + sel[k]]), kap[h]);
            w_out[(size_t)h * k_max + k] = (double)W / (double)S[h];
        }
    }
    *k_sel_out = ksel;
    if (SA_out) *SA_out = SA;
    if (kstar_out) *kstar_out = kstar;
    free(sel);
    free(it);
    return 0;
}

/* ------------------------------------------------------------------------
 * R6 -- sparse weighted sum, Eq. 5: ỹ = Σ_{i∈Π_k*} ã*_i V_i,
 * accumulated in double, in ascending-index order.  V rows fp16 [*][d].
 * ---------------------------------------------------------------------- */
OR_EXPORT void or_gather(const int32_t *idx, const double *w, int64_t k, const uint16_t *V, int d,
                         double *out)
{
    for (int e = 0; e < d; ++e) out[e] = 0.0;
    for (int64_t r = 0; r < k; ++r)
        for (int e = 0; e < d; ++e) out[e] += w[r] * (double)or_h2f(V[(size_t)idx[r] * d + e]);
}

/* Eq. 1: exact attention y = softmax(q·Kᵀ/√d)·V in double. */
OR_EXPORT void or_exact_attention(const uint16_t *q, const uint16_t *K, const uint16_t *V, int64_t n,
                                  int d, double *out)
{
    double *z = (double *)malloc(sizeof(double) * (size_t)n);
    double M = -INFINITY;
    for (int64_t j = 0; j < n; ++j) {
        double acc = 0.0;
        for (int e = 0; e < d; ++e) acc += (double)or_h2f(q[e]) * (double)or_h2f(K[j * d + e]);
        z[j] = acc / sqrt((double)d);
        if (z[j] > M) M = z[j];
    }
    double S = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        z[j] = exp(z[j] - M);
        S += z[j];
    }
    for (int e = 0; e < d; ++e) out[e] = 0.0;
    for (int64_t j = 0; j < n; ++j)
        for (int e = 0; e < d; ++e) out[e] += (z[j] / S) * (double)or_h2f(V[j * d + e]);
    free(z);
}

/* ------------------------------------------------------------------------
 * f4 (iii) -- App. B "Enhanced prefilling with block-wise attention": the
 * prompt is cut into blocks of bs tokens; "attention is computed exclusively between a
 * designated anchor block and the current processing block".  Reading (DESIGN F5): the
 * anchor is block 0; query i of block kb = i / bs attends to the keys j with
 *   j <= i                      if kb == 0 (causal inside the anchor block),
 *   j < bs  or  kb*bs <= j <= i otherwise (the whole anchor + causal inside its block),
 * with softmax(q·k/√d) in double (Eq. 1 restricted to that key set).  q [n][Hq][d],
 * k, v [n][Hkv][d] fp16, query head h uses KV head h / (Hq/Hkv); out [n][Hq][d] double.
 * ---------------------------------------------------------------------- */
OR_EXPORT void or_blockwise_attention(const uint16_t *q, const uint16_t *k, const uint16_t *v,
                                      int64_t n, int Hq, int Hkv, int d, int64_t bs, double *out)
{
    const int G = Hq / Hkv;
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
    for (int64_t i = 0; i < n; ++i)
        for (int h = 0; h < Hq; ++h) {
            const int kv = h / G;
            const int64_t kb = i / bs;
            double *z = (double *)malloc(sizeof(double) * (size_t)(i + 1));
            char *ok = (char *)malloc((size_t)(i + 1));
            double M = -INFINITY;
            for (int64_t j = 0; j <= i; ++j) {
                ok[j] = (char)(kb == 0 || j < bs || j >= kb * bs);
                if (!ok[j]) continue;
                double acc = 0.0;
                for (int e = 0; e < d; ++e)
                    acc += (double)or_h2f(q[(i * Hq + h) * d + e]) * (double)or_h2f(k[(j * Hkv + kv) * d + e]);
                z[j] = acc / sqrt((double)d);
                if (z[j] > M) M = z[j];
            }
            double S = 0.0;
            for (int64_t j = 0; j <= i; ++j)
                if (ok[j]) {
                    z[j] = exp(z[j] - M);
                    S += z[j];
                }
            double *o = out + (i * Hq + h) * d;
            for (int e = 0; e < d; ++e) o[e] = 0.0;
            for (int64_t j = 0; j <= i; ++j)
                if (ok[j])
                    for (int e = 0; e < d; ++e) o[e] += (z[j] / S) * (double)or_h2f(v[(j * Hkv + kv) * d + e]);
            free(z);
            free(ok);
        }
}

/* ------------------------------------------------------------------------
 * One decode unit (batch b, layer l, KV head kv) for its G GQA query heads
 * (head h of the unit uses KV head kv, DESIGN R7), steps R2 -> R6 in the
 * paper's order.  Candidates j in [0, nq) are quantized (codes P, group-major,
 * stride), j in [nq, nq+nres) are resident exact tokens (rk, rv).
 * V [nq][d] fp16 holds the offloaded values of the quantized tokens.
 * Outputs per head h: z [G][nq+nres], e [G], idx [G][k_max], w [G][k_max],
 * k_sel [G], S [G], M [G], kstar [G], out [G][d] (double).
 * ---------------------------------------------------------------------- */
OR_EXPORT int or_decode_unit_bits(const uint16_t *q, int G, int d, int g, int c, int cbg,
                                  const float *C, const uint16_t *P, int64_t nq, int64_t stride,
                                  const uint16_t *V, const uint16_t *rk, const uint16_t *rv,
                                  int64_t nres, float tau, int64_t k_max, int renorm, int32_t *z,
                                  int32_t *e_out, int32_t *idx, double *w, int64_t *k_sel,
                                  uint64_t *S, int32_t *M, int64_t *kstar, double *out,
                                  int lut_bits)
{
    int64_t n = nq + nres;
    if (n <= 0) return 5;
    int16_t *Tfx = (int16_t *)malloc(sizeof(int16_t) * (size_t)G * g * c);
    or_table_bits(q, G, d, g, c, cbg, C, NULL, Tfx, e_out, lut_bits);
    for (int h = 0; h < G; ++h) {
        int32_t *zh = z + (size_t)h * n;
        or_scores(Tfx + (size_t)h * g * c, P, nq, stride, g, c, zh);
        if (nres > 0) or_resident_scores(q + (size_t)h * d, rk, nres, d, e_out[h], zh + nq);
        int rc = or_select(zh, n, e_out[h], d, tau, k_max, renorm, idx + (size_t)h * k_max,
                           w + (size_t)h * k_max, k_sel + h, S + h, M + h, kstar + h);
        if (rc) {
            free(Tfx);
            return rc;
        }
        double *oh = out + (size_t)h * d;
        for (int e = 0; e < d; ++e) oh[e] = 0.0;
        for (int64_t r = 0; r < k_sel[h]; ++r) {
            int64_t j = idx[(size_t)h * k_max + r];
            const uint16_t *row = j < nq ? V + (size_t)j * d : rv + (size_t)(j - nq) * d;
            double wr = w[(size_t)h * k_max + r];
            for (int e = 0; e < d; ++e) oh[e] += wr * (double)or_h2f(row[e]);
        }
    }
    free(Tfx);
    return 0;
}

OR_EXPORT int or_decode_unit(const uint16_t *q, int G, int d, int g, int c, int cbg, const float *C,
                             const uint16_t *P, int64_t nq, int64_t stride, const uint16_t *V,
                             const uint16_t *rk, const uint16_t *rv, int64_t nres, float tau,
                             int64_t k_max, int renorm, int32_t *z, int32_t *e_out,
                             int32_t *idx, double *w, int64_t *k_sel, uint64_t *S, int32_t *M,
                             int64_t *kstar, double *out)
{
    return or_decode_unit_bits(q, G, d, g, c, cbg, C, P, nq, stride, V, rk, rv, nres, tau, k_max,
                               renorm, z, e_out, idx, w, k_sel, S, M, kstar, out, 16);
}
