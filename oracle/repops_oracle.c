/*
 * oracle/repops_oracle.c -- the CPU ORACLE for the RepOps hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2502_19405_b200/) never imports, links or calls it,
 * and shares no source, header, table or constant generator with it.
 *
 * Plain, slow, single-threaded C.  Every function executes the canonical
 * operation order of the paper's method step by step in IEEE-754 binary32
 * with round-to-nearest-even:
 *   - compile with  -O2 -ffp-contract=off -fno-fast-math  (SSE2 math on
 *     x86-64; FLT_EVAL_METHOD == 0), so that  a*b+c  is TWO roundings and the
 *     only single-rounding multiply-add is an explicit fmaf();
 *   - FTZ/DAZ must be clear: orc_fpenv_ok() checks MXCSR.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section named beside it).
 * Readings of points the paper leaves open are listed in DESIGN.md §3
 * ("Readings") and numbered R1..; each function names the reading it uses.
 *
 * Parity pins (what ties this file to something other than itself) live in
 * tests/test_oracle_*.py.  Every function here is pinned; none is "parity
 * unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#if defined(__x86_64__)
#include <xmmintrin.h>
#endif

typedef int64_t i64;

/* ---------------------------------------------------------------- helpers */
static float bits2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t f2bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* Reading R10: every op output NaN is written as the canonical 0x7FC00000. */
static float canon(float x) { return (x != x) ? bits2f(0x7FC00000u) : x; }

int orc_fpenv_ok(void) {
#if defined(__x86_64__)
    unsigned csr = _mm_getcsr();
    /* bit 15 = FTZ, bit 6 = DAZ, bits 13-14 = rounding control (00 = RN) */
    return ((csr & 0x8040u) == 0u) && ((csr & 0x6000u) == 0u);
#else
    return 1;
#endif
}

/* ======================================================================
 * R-GEMM  -- P:598-609 (Sec 3.2 listing "repops matrix multiplication"):
 *   for i (any order), for j (any order):
 *       sum = 0;  for k = 0 .. K-1 (fixed order): sum = sum + a*b;  C = sum
 * Readings: R1 "sum + a*b" is one fused fma; R2 acc starts at +0.0 and k is
 * ascending (fixed by the listing); R3 bias / scale are applied once after
 * the full K fold.  op(A)(i,k) = transA ? A[k*lda+i] : A[i*lda+k];
 * op(B)(k,j) = transB ? B[j*ldb+k] : B[k*ldb+j]  (addressing only).
 * epi: 0 = none, 1 = bias  C = acc + bias[j],  2 = scale  C = acc * scale.
 * ==================================================================== */
void orc_gemm(i64 M, i64 N, i64 K,
              const float *A, i64 lda, int transA,
              const float *B, i64 ldb, int transB,
              int epi, const float *bias, float scale,
              float *C, i64 ldc)
{
    for (i64 i = 0; i < M; ++i) {
        for (i64 j = 0; j < N; ++j) {
            float sum = 0.0f;
            for (i64 k = 0; k < K; ++k) {
                float a = transA ? A[k * lda + i] : A[i * lda + k];
                float b = transB ? B[j * ldb + k] : B[k * ldb + j];
                sum = fmaf(a, b, sum);
            }
            if (epi == 1) sum = sum + bias[j];
            else if (epi == 2) sum = sum * scale;
            C[i * ldc + j] = canon(sum);
        }
    }
}

/* ======================================================================
 * R-CSUM / R-CDOT -- P:588-590 (Sec 3.2: "in the dimensions where order is
 * critical, we either perform the operations serially or synchronize
 * threads to enforce a deterministic execution order").  Reading R4: the
 * fixed order is
 *   n <= 4096: p[s] = +0 (s < 128); for i ascending: p[i%128] += x[i];
 *              TREE128: for h = 64,32,...,1: for s < h: p[s] = p[s] + p[s+h]
 *   n >  4096: CSUM over the list of CSUMs of the 4096-element tiles.
 * CDOT is identical with the slot update p = fma(u_i, v_i, p); its tile
 * results are combined with CSUM.
 * ==================================================================== */
#define ORC_SLOTS 128
#define ORC_TILE 4096

static float tree128(float *p) {
    for (int h = ORC_SLOTS / 2; h >= 1; h /= 2)
        for (int s = 0; s < h; ++s) p[s] = p[s] + p[s + h];
    return p[0];
}

static float csum_tile(const float *x, i64 n, i64 stride) {
    float p[ORC_SLOTS];
    for (int s = 0; s < ORC_SLOTS; ++s) p[s] = 0.0f;
    for (i64 i = 0; i < n; ++i) p[i % ORC_SLOTS] = p[i % ORC_SLOTS] + x[i * stride];
    return tree128(p);
}

float orc_csum(const float *x, i64 n, i64 stride) {
    if (n <= ORC_TILE) return csum_tile(x, n, stride);
    i64 nt = (n + ORC_TILE - 1) / ORC_TILE;
    float *t = (float *)malloc((size_t)nt * sizeof(float));
    for (i64 q = 0; q < nt; ++q) {
        i64 len = (n - q * ORC_TILE < ORC_TILE) ? n - q * ORC_TILE : ORC_TILE;
        t[q] = csum_tile(x + q * ORC_TILE * stride, len, stride);
    }
    float r = orc_csum(t, nt, 1);
    free(t);
    return r;
}

static float cdot_tile(const float *u, const float *v, i64 n) {
    float p[ORC_SLOTS];
    for (int s = 0; s < ORC_SLOTS; ++s) p[s] = 0.0f;
    for (i64 i = 0; i < n; ++i) p[i % ORC_SLOTS] = fmaf(u[i], v[i], p[i % ORC_SLOTS]);
    return tree128(p);
}

float orc_cdot(const float *u, const float *v, i64 n) {
    if (n <= ORC_TILE) return cdot_tile(u, v, n);
    i64 nt = (n + ORC_TILE - 1) / ORC_TILE;
    float *t = (float *)malloc((size_t)nt * sizeof(float));
    for (i64 q = 0; q < nt; ++q) {
        i64 len = (n - q * ORC_TILE < ORC_TILE) ? n - q * ORC_TILE : ORC_TILE;
        t[q] = cdot_tile(u + q * ORC_TILE, v + q * ORC_TILE, len);
    }
    float r = orc_csum(t, nt, 1);
    free(t);
    return r;
}

/* row-wise CSUM of a rows x cols matrix (leading dimension ld) */
void orc_sum_rows(const float *x, i64 rows, i64 cols, i64 ld, float *out) {
    for (i64 r = 0; r < rows; ++r) out[r] = canon(orc_csum(x + r * ld, cols, 1));
}

/* R-SEQ (reading R4, token axis; same principle as the listing's k loop,
 * P:603-606): out[j] = fold over rows r0..r1-1 ascending of acc + x[r][j],
 * acc starting at +0.  Rows are split into nseg equal contiguous segments
 * (one per data-parallel shard); out is nseg x cols. */
void orc_sum_cols_seq(const float *x, i64 rows, i64 cols, i64 ld, i64 nseg, float *out) {
    i64 per = rows / nseg;
    for (i64 s = 0; s < nseg; ++s)
        for (i64 j = 0; j < cols; ++j) {
            float acc = 0.0f;
            for (i64 r = s * per; r < (s + 1) * per; ++r) acc = acc + x[r * ld + j];
            out[s * cols + j] = canon(acc);
        }
}

/* ======================================================================
 * Software math -- P:571-574 (Sec 3.1: RepOps "re-implements common ML
 * operators and mathematical functions (like exp, sin, cos, tanh) in a way
 * that controls the order of floating point operators").  Reading R5: the
 * algorithms are the Cephes single-precision ones written as a fixed chain
 * of IEEE RN operations (fmaf where written, else separate mul/add).
 * ==================================================================== */
static float pow2i(int k) { return bits2f((uint32_t)(k + 127) << 23); } /* -126 <= k <= 127 */

float orc_exp(float x) {
    if (x != x) return bits2f(0x7FC00000u);
    if (x > 89.0f) return bits2f(0x7F800000u);
    if (x < -104.0f) return 0.0f;
    float t = x * 1.44269504088896341f;              /* log2(e) = 0x3FB8AA3B */
    float kf = (t + 12582912.0f) - 12582912.0f;      /* round to nearest even integer */
    float r = fmaf(kf, -0.693359375f, x);            /* Cephes C1 */
    r = fmaf(kf, 2.12194440e-4f, r);                 /* minus Cephes C2 = -2.12194440e-4 */
    float p = 1.9875691500E-4f;
    p = fmaf(p, r, 1.3981999507E-3f);
    p = fmaf(p, r, 8.3334519073E-3f);
    p = fmaf(p, r, 4.1665795894E-2f);
    p = fmaf(p, r, 1.6666665459E-1f);
    p = fmaf(p, r, 5.0000001201E-1f);
    float y = fmaf(p, r * r, r) + 1.0f;
    int k = (int)kf;
    int k1 = k >> 1;            /* arithmetic shift: floor(k/2) */
    int k2 = k - k1;
    return (y * pow2i(k1)) * pow2i(k2);
}

float orc_log(float x) {
    if (x != x) return bits2f(0x7FC00000u);
    if (x < 0.0f) return bits2f(0x7FC00000u);
    if (x == 0.0f) return bits2f(0xFF800000u);
    if (x == bits2f(0x7F800000u)) return x;
    int e = 0;
    if (x < 1.17549435e-38f) { x = x * 8388608.0f; e = -23; }  /* subnormal: exact x 2^23 */
    uint32_t u = f2bits(x);
    e += (int)((u >> 23) & 0xFFu) - 126;
    float m = bits2f((u & 0x007FFFFFu) | 0x3F000000u);        /* m in [0.5, 1) */
    if (m < 0.70710678f) { e -= 1; m = m + m; }
    float f = m - 1.0f;
    float z = f * f;
    float p = 7.0376836292E-2f;
    p = fmaf(p, f, -1.1514610310E-1f);
    p = fmaf(p, f, 1.1676998740E-1f);
    p = fmaf(p, f, -1.2420140846E-1f);
    p = fmaf(p, f, 1.4249322787E-1f);
    p = fmaf(p, f, -1.6668057665E-1f);
    p = fmaf(p, f, 2.0000714765E-1f);
    p = fmaf(p, f, -2.4999993993E-1f);
    p = fmaf(p, f, 3.3333331174E-1f);
    float ef = (float)e;
    float y = (p * f) * z;
    y = fmaf(ef, -2.12194440e-4f, y);
    y = fmaf(z, -0.5f, y);
    y = f + y;
    y = fmaf(ef, 0.693359375f, y);
    return y;
}

float orc_tanh(float u) {
    if (u != u) return bits2f(0x7FC00000u);
    float a = fabsf(u);
    float t;
    if (a < 0.625f) {
        float z = u * u;
        float p = -5.70498872745E-3f;
        p = fmaf(p, z, 2.06390887954E-2f);
        p = fmaf(p, z, -5.37397155531E-2f);
        p = fmaf(p, z, 1.33314422036E-1f);
        p = fmaf(p, z, -3.33332819422E-1f);
        t = fmaf(p * z, a, a);
    } else {
        float aa = (a < 44.0f) ? a : 44.0f;
        float e = orc_exp(aa + aa);
        t = 1.0f - 2.0f / (e + 1.0f);
    }
    return copysignf(t, u);
}

/* sin / cos ("exp, sin, cos, tanh"; reading R26): Cephes sinf/cosf --
 * octant j = trunc(|x| * 4/pi) rounded up to even, Cody-Waite reduction
 * r = ((|x| - y DP1) - y DP2) - y DP3 (separate mul / sub; |x| > 8192: |x| - y pi/4),
 * then on [-pi/4, pi/4] the sine polynomial r + r z P(z) (one fmaf) or the cosine
 * polynomial 1 - z/2 + z^2 Q(z), selected and signed by the octant.
 * |x| > 16777215 returns +0 (Cephes TLOSS); +-inf and NaN return NaN. */
static const float SC_FOPI = 1.27323954473516f, SC_PIO4 = 0.7853981633974483096f;
static const float SC_DP1 = 0.78515625f, SC_DP2 = 2.4187564849853515625e-4f, SC_DP3 = 3.77489497744594108e-8f;

static float sc_reduce(float a, int *oct) {
    float t = a * SC_FOPI;
    uint32_t j = (uint32_t)t;                 /* truncation; 0 <= t < 2^24 */
    float y = (float)j;
    if (j & 1u) { j += 1u; y = y + 1.0f; }
    *oct = (int)(j & 7u);
    if (a > 8192.0f) return a - y * SC_PIO4;
    return ((a - y * SC_DP1) - y * SC_DP2) - y * SC_DP3;
}

static float sc_sinpoly(float r, float z) {
    float p = fmaf(-1.9515295891E-4f, z, 8.3321608736E-3f);
    p = fmaf(p, z, -1.6666654611E-1f);
    return fmaf(p * z, r, r);
}

static float sc_cospoly(float z) {
    float p = fmaf(2.443315711809948E-5f, z, -1.388731625493765E-3f);
    p = fmaf(p, z, 4.166664568298827E-2f);
    float v = p * (z * z);
    v = v - 0.5f * z;
    return v + 1.0f;
}

float orc_sin(float x) {
    if (x != x || x == bits2f(0x7F800000u) || x == bits2f(0xFF800000u)) return bits2f(0x7FC00000u);
    int neg = x < 0.0f;
    float a = neg ? -x : x;
    if (a > 16777215.0f) return 0.0f;
    int j;
    float r = sc_reduce(a, &j);
    if (j > 3) { neg = !neg; j -= 4; }
    float z = r * r;
    float v = (j == 1 || j == 2) ? sc_cospoly(z) : sc_sinpoly(r, z);
    return neg ? -v : v;
}

float orc_cos(float x) {
    if (x != x || x == bits2f(0x7F800000u) || x == bits2f(0xFF800000u)) return bits2f(0x7FC00000u);
    float a = x < 0.0f ? -x : x;
    if (a > 16777215.0f) return 0.0f;
    int j, neg = 0;
    float r = sc_reduce(a, &j);
    if (j > 3) { neg = !neg; j -= 4; }
    if (j > 1) neg = !neg;
    float z = r * r;
    float v = (j == 1 || j == 2) ? sc_sinpoly(r, z) : sc_cospoly(z);
    return neg ? -v : v;
}

void orc_sin_vec(const float *x, i64 n, float *y) { for (i64 i = 0; i < n; ++i) y[i] = orc_sin(x[i]); }
void orc_cos_vec(const float *x, i64 n, float *y) { for (i64 i = 0; i < n; ++i) y[i] = orc_cos(x[i]); }

/* RoPE tables from the inverse frequencies (reading R26): angle = fmul(float(t), inv_freq[i]),
 * cos[t][i] = R-COS(angle), sin[t][i] = R-SIN(angle), t < T, i < h. */
void orc_rope_tables(const float *inv_freq, i64 T, i64 h, float *cosv, float *sinv) {
    for (i64 t = 0; t < T; ++t)
        for (i64 i = 0; i < h; ++i) {
            float ang = (float)t * inv_freq[i];
            cosv[t * h + i] = orc_cos(ang);
            sinv[t * h + i] = orc_sin(ang);
        }
}

/* erf (exact GELU of BERT-family models, "GeLU, and ERF"; reading R27):
 * Cephes erff / erfcf.  |x| <= 1: x T(x^2) (Horner, fmaf); |x| > 1: 1 - erfc(|x|) with
 * erfc(a) = exp(-a^2) (1/a) P(1/a^2) (P for a < 2, R for a >= 2), exp = R-EXP; the sign
 * of x is applied last (erf is odd).  a^2 is one rounded product. */
static float horner(const float *c, int n, float x) {
    float p = c[0];
    for (int i = 1; i <= n; ++i) p = fmaf(p, x, c[i]);
    return p;
}
static const float ERF_T[7] = {7.853861353153693E-5f, -8.010193625184903E-4f, 5.188327685732524E-3f,
                               -2.685381193529856E-2f, 1.128358514861418E-1f, -3.761262582423300E-1f,
                               1.128379165726710E+0f};
static const float ERFC_P[9] = {2.326819970068386E-2f, -1.387039388740657E-1f, 3.687424674597105E-1f,
                                -5.824733027278666E-1f, 6.210004621745983E-1f, -4.944515323274145E-1f,
                                3.404879937665872E-1f, -2.741127028184656E-1f, 5.638259427386472E-1f};
static const float ERFC_R[8] = {-1.047766399936249E+1f, 1.297719955372516E+1f, -7.495518717768503E+0f,
                                2.921019019210786E+0f, -1.015265279202700E+0f, 4.218463358204948E-1f,
                                -2.820767439740514E-1f, 5.641895067754075E-1f};

float orc_erf(float x) {
    if (x != x) return bits2f(0x7FC00000u);
    float a = fabsf(x);
    float y;
    if (a <= 1.0f) {
        y = a * horner(ERF_T, 6, a * a);
    } else if (a >= 10.0f) {
        y = 1.0f;
    } else {
        float z = orc_exp(-(a * a));
        float q = 1.0f / a;
        float p = (a < 2.0f) ? horner(ERFC_P, 8, q * q) : horner(ERFC_R, 7, q * q);
        y = 1.0f - (z * q) * p;
    }
    return x < 0.0f ? -y : y;
}

void orc_erf_vec(const float *x, i64 n, float *y) { for (i64 i = 0; i < n; ++i) y[i] = orc_erf(x[i]); }

/* exact GELU (R27): y = (0.5 x) (1 + erf(x * 0.70710678118654752)) */
void orc_gelu_erf(const float *x, i64 n, float *y) {
    for (i64 i = 0; i < n; ++i) {
        float v = x[i];
        y[i] = canon((0.5f * v) * (1.0f + orc_erf(v * 0.70710678118654752f)));
    }
}

/* exact GELU backward (R27): cdf = 0.5 (1 + erf(x / sqrt 2)), pdf = R-EXP(-(0.5 (x x))) / sqrt(2 pi),
 * dx = dy (cdf + x pdf) */
void orc_gelu_erf_backward(const float *x, const float *dy, i64 n, float *dx) {
    for (i64 i = 0; i < n; ++i) {
        float v = x[i];
        float cdf = 0.5f * (1.0f + orc_erf(v * 0.70710678118654752f));
        float pdf = orc_exp(-(0.5f * (v * v))) * 0.39894228040143268f;
        dx[i] = canon(dy[i] * (cdf + v * pdf));
    }
}

/* Deterministic pseudorandomness ("built-in support for deterministic
 * pseudorandomness generation in PyTorch and CUDA"; reading R28): Philox4x32-10, the
 * counter-based generator behind curand's Philox4_32_10 and PyTorch's CUDA generator
 * (Salmon et al., SC'11).  One round: (hi0, lo0) = M0 * c0, (hi1, lo1) = M1 * c2 (64-bit
 * products), c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); the key is bumped by
 * (W0, W1) between rounds; 10 rounds. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* R28 draw of element i: block b = i / 4 with counter (b lo, b hi, stream lo, stream hi) and
 * key (seed lo, seed hi); word i % 4 of the block; u = (word >> 8) * 2^-24 in [0, 1)
 * (exact in binary32). */
static float rand_u(uint64_t seed, uint64_t stream, i64 i) {
    uint64_t b = (uint64_t)i >> 2;
    uint32_t ctr[4] = {(uint32_t)b, (uint32_t)(b >> 32), (uint32_t)stream, (uint32_t)(stream >> 32)};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t w[4];
    orc_philox4x32_10(ctr, key, w);
    return (float)(w[i & 3] >> 8) * 5.9604644775390625e-8f;
}

void orc_rand_uniform(uint64_t seed, uint64_t stream, i64 n, float *y) {
    for (i64 i = 0; i < n; ++i) y[i] = rand_u(seed, stream, i);
}

/* R28 dropout: keep_i = (u_i >= p); scale = 1 / (1 - p) (binary32 ops);
 * y_i = keep_i ? x_i * scale : +0; mask_i = keep_i (optional).  Backward regenerates the
 * mask from (seed, stream, i): dx_i = keep_i ? dy_i * scale : +0. */
void orc_dropout(const float *x, i64 n, float p, uint64_t seed, uint64_t stream, float *y, uint8_t *mask) {
    float scale = 1.0f / (1.0f - p);
    for (i64 i = 0; i < n; ++i) {
        int keep = rand_u(seed, stream, i) >= p;
        y[i] = keep ? canon(x[i] * scale) : 0.0f;
        if (mask) mask[i] = (uint8_t)keep;
    }
}

void orc_dropout_backward(const float *dy, i64 n, float p, uint64_t seed, uint64_t stream, float *dx) {
    float scale = 1.0f / (1.0f - p);
    for (i64 i = 0; i < n; ++i) dx[i] = (rand_u(seed, stream, i) >= p) ? canon(dy[i] * scale) : 0.0f;
}

/* Lower-precision storage ("RepOps works with any lower precision ...
 * (particularly FP16)"; reading R30): tensors may be STORED as bfloat16 / binary16 while
 * every operation computes in binary32.  Widening is exact; narrowing rounds to nearest
 * even (IEEE 754 convertFormat), with gradual underflow, overflow to +-inf and the
 * canonical NaNs 0x7FC0 (bf16) / 0x7E00 (f16). */
uint16_t orc_f32_to_bf16(float x) {
    uint32_t u = f2bits(x);
    if (x != x) return 0x7FC0u;
    u += 0x7FFFu + ((u >> 16) & 1u);      /* RN-even on the 16 dropped bits */
    return (uint16_t)(u >> 16);
}
float orc_bf16_to_f32(uint16_t h) { return bits2f((uint32_t)h << 16); }

/* binary16 by its definition: the representable value nearest |x| (ties to the even
 * significand), computed exactly in double (power-of-two scalings and rint). */
uint16_t orc_f32_to_f16(float x) {
    if (x != x) return 0x7E00u;
    uint16_t sign = (f2bits(x) >> 16) & 0x8000u;
    double a = fabs((double)x);
    if (a >= 65520.0) return sign | 0x7C00u;               /* halfway to 2^16 or above -> inf */
    if (a < ldexp(1.0, -14)) {                             /* subnormal: multiples of 2^-24 */
        double m = rint(a * ldexp(1.0, 24));               /* m <= 1024 (1024 = min normal) */
        return sign | (uint16_t)m;
    }
    int e;
    frexp(a, &e);                                          /* a in [2^(e-1), 2^e) */
    e -= 1;                                                /* a in [2^e, 2^(e+1)), e in [-14, 15] */
    double m = rint(a * ldexp(1.0, 10 - e));               /* significand in [1024, 2048] */
    return sign | (uint16_t)((((uint32_t)(e + 15)) << 10) + (uint32_t)m - 1024u);
}
float orc_f16_to_f32(uint16_t h) {
    int sign = h >> 15, e = (h >> 10) & 0x1F, m = h & 0x3FF;
    double v;
    if (e == 31) return m ? bits2f(0x7FC00000u) : (sign ? -INFINITY : INFINITY);
    v = (e == 0) ? ldexp((double)m, -24) : ldexp((double)(m + 1024), e - 25);
    return (float)(sign ? -v : v);                         /* exact */
}

/* dtype codes (repops.h verde_dtype): 1 = f32, 4 = bf16, 5 = f16 */
static float ld_elem(const void *p, int dt, i64 i) {
    if (dt == 4) return orc_bf16_to_f32(((const uint16_t *)p)[i]);
    if (dt == 5) return orc_f16_to_f32(((const uint16_t *)p)[i]);
    return ((const float *)p)[i];
}
static void st_elem(void *p, int dt, i64 i, float v) {
    if (dt == 4) ((uint16_t *)p)[i] = orc_f32_to_bf16(v);
    else if (dt == 5) ((uint16_t *)p)[i] = orc_f32_to_f16(v);
    else ((float *)p)[i] = canon(v);
}

/* 2-D convert (rows x cols, leading dimensions in elements). */
void orc_convert(const void *src, int sdt, i64 rows, i64 cols, i64 lds, void *dst, int ddt, i64 ldd) {
    for (i64 r = 0; r < rows; ++r)
        for (i64 c = 0; c < cols; ++c) st_elem(dst, ddt, r * ldd + c, ld_elem(src, sdt, r * lds + c));
}

/* R30 GEMM on stored operands: C = narrow_cdt(R-GEMM(widen(A), widen(B)) with epi);
 * the K fold is R-GEMM's (binary32 fma, k ascending). */
void orc_gemm(i64 M, i64 N, i64 K, const float *A, i64 lda, int transA, const float *B, i64 ldb, int transB,
              int epi, const float *bias, float scale, float *Cm, i64 ldc);
void orc_gemm_ex(i64 M, i64 N, i64 K, const void *A, int adt, i64 lda, int transA, const void *B, int bdt, i64 ldb,
                 int transB, int epi, const float *bias, float scale, void *Cm, int cdt, i64 ldc) {
    i64 ar = transA ? K : M, ac = transA ? M : K, br = transB ? N : K, bc = transB ? K : N;
    float *a = (float *)malloc(sizeof(float) * (size_t)(ar * ac + 1));
    float *b = (float *)malloc(sizeof(float) * (size_t)(br * bc + 1));
    float *c = (float *)malloc(sizeof(float) * (size_t)(M * N + 1));
    orc_convert(A, adt, ar, ac, lda, a, 1, ac);
    orc_convert(B, bdt, br, bc, ldb, b, 1, bc);
    orc_gemm(M, N, K, a, ac, transA, b, bc, transB, epi, bias, scale, c, N);
    orc_convert(c, 1, M, N, N, Cm, cdt, ldc);
    free(a); free(b); free(c);
}

/* Reading R6: rsqrt = IEEE fdiv(1, IEEE fsqrt(x)), both correctly rounded. */
float orc_rsqrt(float x) { return canon(1.0f / sqrtf(x)); }

void orc_exp_vec(const float *x, i64 n, float *y) { for (i64 i = 0; i < n; ++i) y[i] = canon(orc_exp(x[i])); }
void orc_log_vec(const float *x, i64 n, float *y) { for (i64 i = 0; i < n; ++i) y[i] = canon(orc_log(x[i])); }
void orc_tanh_vec(const float *x, i64 n, float *y) { for (i64 i = 0; i < n; ++i) y[i] = canon(orc_tanh(x[i])); }
void orc_rsqrt_vec(const float *x, i64 n, float *y) { for (i64 i = 0; i < n; ++i) y[i] = orc_rsqrt(x[i]); }

/* elementwise residual add: y = a + b */
void orc_add(const float *a, const float *b, i64 n, float *y) { for (i64 i = 0; i < n; ++i) y[i] = canon(a[i] + b[i]); }

/* ReLU (config 1 MLP, reading R24 in DESIGN.md):
 *   relu(x) = x if x > 0, else +0 (so -0 and negatives give +0); NaN -> canonical NaN.
 *   relu_backward(x, g) = g if x > 0, else +0 (subgradient at 0 is 0); NaN x -> NaN. */
void orc_relu(const float *x, i64 n, float *y) {
    for (i64 i = 0; i < n; ++i) y[i] = (x[i] != x[i]) ? canon(x[i]) : (x[i] > 0.0f ? x[i] : 0.0f);
}

void orc_relu_backward(const float *x, const float *g, i64 n, float *dx) {
    for (i64 i = 0; i < n; ++i) dx[i] = (x[i] != x[i]) ? canon(x[i]) : (x[i] > 0.0f ? canon(g[i]) : 0.0f);
}

/* GELU, tanh form (GPT-2), reading R5/R13 in DESIGN.md:
 *   u = sqrt(2/pi) * (x + 0.044715 x^3),  y = 0.5 x (1 + tanh u) */
void orc_gelu(const float *x, i64 n, float *y) {
    for (i64 i = 0; i < n; ++i) {
        float v = x[i];
        float x2 = v * v;
        float x3 = x2 * v;
        float inner = fmaf(0.044715f, x3, v);
        float u = 0.7978845608028654f * inner;
        float t = orc_tanh(u);
        y[i] = canon((0.5f * v) * (1.0f + t));
    }
}

/* dGELU/dx, recomputing x2 and t exactly as the forward does. */
void orc_gelu_backward(const float *x, const float *dy, i64 n, float *dx) {
    for (i64 i = 0; i < n; ++i) {
        float v = x[i];
        float x2 = v * v;
        float x3 = x2 * v;
        float inner = fmaf(0.044715f, x3, v);
        float u = 0.7978845608028654f * inner;
        float t = orc_tanh(u);
        float di = fmaf(0.134145f, x2, 1.0f);
        float s2 = 1.0f - t * t;
        float g = (0.5f * (1.0f + t)) + (((0.5f * v) * s2) * (0.7978845608028654f * di));
        dx[i] = canon(dy[i] * g);
    }
}

/* ======================================================================
 * Row max used by softmax / cross-entropy (reading R7): maximum over the
 * non-NaN valid entries (order-free), -inf if none; a zero maximum is
 * written as +0 so the value is unique.
 * ==================================================================== */
static float row_max(const float *x, i64 n) {
    float m = bits2f(0xFF800000u);
    for (i64 i = 0; i < n; ++i) {
        float v = x[i];
        if (v == v && v > m) m = v;
    }
    if (m == 0.0f) m = 0.0f;
    return m;
}

/* R-SOFTMAX (reading R7): e_i = exp(x_i - m); s = CSUM(e); r = 1/s;
 * y_i = e_i * r.  causal: rows % cols == 0; row r keeps (r mod cols)+1
 * entries, the rest are written +0. */
void orc_softmax(const float *x, i64 rows, i64 cols, i64 ldx, int causal, float *y, i64 ldy) {
    float *e = (float *)malloc((size_t)(cols > 0 ? cols : 1) * sizeof(float));
    for (i64 r = 0; r < rows; ++r) {
        const float *xr = x + r * ldx;
        float *yr = y + r * ldy;
        i64 L = causal ? (r % cols) + 1 : cols;
        float m = row_max(xr, L);
        for (i64 i = 0; i < L; ++i) e[i] = orc_exp(xr[i] - m);
        float s = orc_csum(e, L, 1);
        float rinv = 1.0f / s;
        for (i64 i = 0; i < L; ++i) yr[i] = canon(e[i] * rinv);
        for (i64 i = L; i < cols; ++i) yr[i] = 0.0f;
    }
    free(e);
}

/* R-SOFTMAX-BWD: c = CDOT(y, dy) over the full row; dx_i = (y_i (dy_i - c)) * scale */
void orc_softmax_backward(const float *y, i64 ldy, const float *dy, i64 lddy, i64 rows, i64 cols,
                          float scale, float *dx, i64 lddx) {
    for (i64 r = 0; r < rows; ++r) {
        const float *yr = y + r * ldy, *gr = dy + r * lddy;
        float c = orc_cdot(yr, gr, cols);
        for (i64 i = 0; i < cols; ++i) dx[r * lddx + i] = canon((yr[i] * (gr[i] - c)) * scale);
    }
}

/* ======================================================================
 * R-LN (LayerNorm; the paper lists it among RepOps operators).
 * Reading R8: two-pass biased variance, eps inside the square root.
 *   mu = CSUM(x)/n;  d_i = x_i - mu;  var = CDOT(d,d)/n;
 *   rstd = 1/sqrt(var + eps);  y_i = fma(d_i * rstd, gamma_i, beta_i)
 * ==================================================================== */
void orc_layernorm(const float *x, const float *gamma, const float *beta, i64 rows, i64 cols,
                   float eps, float *y, float *mean, float *rstd) {
    float *d = (float *)malloc((size_t)cols * sizeof(float));
    float n = (float)cols;
    for (i64 r = 0; r < rows; ++r) {
        const float *xr = x + r * cols;
        float mu = orc_csum(xr, cols, 1) / n;
        for (i64 i = 0; i < cols; ++i) d[i] = xr[i] - mu;
        float var = orc_cdot(d, d, cols) / n;
        float rs = 1.0f / sqrtf(var + eps);
        for (i64 i = 0; i < cols; ++i) y[r * cols + i] = canon(fmaf(d[i] * rs, gamma[i], beta[i]));
        if (mean) mean[r] = canon(mu);
        if (rstd) rstd[r] = canon(rs);
    }
    free(d);
}

/* LN backward, row part:  xh_i = (x_i - mu) * rstd;  g_i = dy_i * gamma_i;
 *   a = CSUM(g)/n;  b = CDOT(g, xh)/n;  dx_i = ((g_i - a) - xh_i * b) * rstd
 * If dres != NULL the result is dres_i + dx_i (residual-stream gradient). */
void orc_layernorm_backward(const float *dy, const float *x, const float *gamma,
                            const float *mean, const float *rstd, const float *dres,
                            i64 rows, i64 cols, float *dx) {
    float *g = (float *)malloc((size_t)cols * sizeof(float));
    float *xh = (float *)malloc((size_t)cols * sizeof(float));
    float n = (float)cols;
    for (i64 r = 0; r < rows; ++r) {
        for (i64 i = 0; i < cols; ++i) {
            xh[i] = (x[r * cols + i] - mean[r]) * rstd[r];
            g[i] = dy[r * cols + i] * gamma[i];
        }
        float a = orc_csum(g, cols, 1) / n;
        float b = orc_cdot(g, xh, cols) / n;
        for (i64 i = 0; i < cols; ++i) {
            float v = ((g[i] - a) - xh[i] * b) * rstd[r];
            if (dres) v = dres[r * cols + i] + v;
            dx[r * cols + i] = canon(v);
        }
    }
    free(g);
    free(xh);
}

/* LN parameter gradients per shard (R-SEQ over the shard's rows):
 *   dgamma_s[j] = fold_t fma(dy[t][j], xh[t][j], acc);  dbeta_s[j] = fold_t acc + dy[t][j] */
void orc_layernorm_backward_params(const float *dy, const float *x, const float *mean, const float *rstd,
                                   i64 rows, i64 cols, i64 nseg, float *dgamma, float *dbeta) {
    i64 per = rows / nseg;
    for (i64 s = 0; s < nseg; ++s)
        for (i64 j = 0; j < cols; ++j) {
            float ag = 0.0f, ab = 0.0f;
            for (i64 t = s * per; t < (s + 1) * per; ++t) {
                float xh = (x[t * cols + j] - mean[t]) * rstd[t];
                ag = fmaf(dy[t * cols + j], xh, ag);
                ab = ab + dy[t * cols + j];
            }
            dgamma[s * cols + j] = canon(ag);
            dbeta[s * cols + j] = canon(ab);
        }
}

/* ======================================================================
 * Llama operators (BASELINE config 4; readings R20-R22 in DESIGN.md).
 * R-RMSNORM: ms = CDOT(x,x)/n;  rstd = 1/sqrt(ms + eps);  y_i = (x_i * rstd) * w_i
 * R-SWIGLU:  h_i = silu(g_i) * u_i,  silu(g) = g / (1 + exp(-g))   (-g: sign flip, exact)
 * R-ROPE:    rotate-half form with cos/sin tables given as inputs [T, hd/2]:
 *            y_i     = x_i * c_i - x_{i+h} * s_i,   y_{i+h} = x_{i+h} * c_i + x_i * s_i
 *            for each token t, head, i < h = hd/2 (t indexes the table rows)
 * ==================================================================== */
void orc_rmsnorm(const float *x, const float *w, i64 rows, i64 cols, float eps, float *y, float *rstd) {
    float n = (float)cols;
    for (i64 r = 0; r < rows; ++r) {
        const float *xr = x + r * cols;
        float ms = orc_cdot(xr, xr, cols) / n;
        float rs = 1.0f / sqrtf(ms + eps);
        for (i64 i = 0; i < cols; ++i) y[r * cols + i] = canon((xr[i] * rs) * w[i]);
        if (rstd) rstd[r] = canon(rs);
    }
}

static float silu(float g) { return g / (1.0f + orc_exp(-g)); }

void orc_swiglu(const float *g, const float *u, i64 n, float *h) {
    for (i64 i = 0; i < n; ++i) h[i] = canon(silu(g[i]) * u[i]);
}

void orc_rope(const float *x, i64 ntok, i64 nhead, i64 hd, i64 ld, const float *cosv, const float *sinv,
              float *y, i64 ldy) {
    i64 h = hd / 2;
    for (i64 t = 0; t < ntok; ++t)
        for (i64 q = 0; q < nhead; ++q) {
            const float *xi = x + t * ld + q * hd;
            float *yo = y + t * ldy + q * hd;
            for (i64 i = 0; i < h; ++i) {
                float c = cosv[t * h + i], s = sinv[t * h + i];
                float a = xi[i], b = xi[i + h];
                yo[i] = canon((a * c) - (b * s));
                yo[i + h] = canon((b * c) + (a * s));
            }
        }
}

/* ======================================================================
 * R-CE: cross entropy over a row of V logits (leading dimension ld).
 *   m = max;  s = CSUM(exp(x_i - m));  loss = (m + log s) - x_label
 *   dlogit_i = ((exp(x_i - m) * (1/s)) - [i == label]) * scale
 * dlogits may alias logits (the row is fully read before it is written).
 * ==================================================================== */
void orc_cross_entropy(const float *logits, i64 rows, i64 V, i64 ld, const int32_t *labels,
                       float scale, float *loss, float *dlogits, i64 ldd) {
    float *e = (float *)malloc((size_t)V * sizeof(float));
    for (i64 r = 0; r < rows; ++r) {
        const float *xr = logits + r * ld;
        float m = row_max(xr, V);
        for (i64 i = 0; i < V; ++i) e[i] = orc_exp(xr[i] - m);
        float s = orc_csum(e, V, 1);
        float xl = xr[labels[r]];
        if (loss) loss[r] = canon((m + orc_log(s)) - xl);
        if (dlogits) {
            float rinv = 1.0f / s;
            for (i64 i = 0; i < V; ++i) {
                float p = e[i] * rinv;
                float d = (i == labels[r]) ? p - 1.0f : p - 0.0f;
                dlogits[r * ldd + i] = canon(d * scale);
            }
        }
    }
    free(e);
}

/* ======================================================================
 * R-EMB: token + position embedding.
 *   fwd: x0[t][c] = wte[tok_t][c] + wpe[t mod T][c]
 *   bwd (one shard): dwte is accumulated INTO (it holds the shard's tied
 *   lm-head gradient), dwpe is written:
 *     for each vocab row v used by the shard:
 *        dwte[v][c] = dwte[v][c] + fold_{t ascending, tok_t == v} (acc + dx0[t][c])
 *     for each position p < min(ntok, T):  dwpe[p][c] = fold_{t ascending, t mod T == p} ...
 * (the fold is the one-hot GEMM's ascending-token order, reading R4)
 * ==================================================================== */
void orc_embedding(const int32_t *tok, i64 ntok, i64 T, const float *wte, const float *wpe, i64 C, float *x0) {
    for (i64 t = 0; t < ntok; ++t)
        for (i64 c = 0; c < C; ++c)
            x0[t * C + c] = canon(wte[(i64)tok[t] * C + c] + wpe[(t % T) * C + c]);
}

void orc_embedding_backward(const int32_t *tok, i64 ntok, i64 T, const float *dx0, i64 C,
                            float *dwte, float *dwpe) {
    /* dwte: rows touched, in order of first occurrence (the order does not
     * matter: each row's fold is independent) */
    for (i64 t = 0; t < ntok; ++t) {
        int first = 1;
        for (i64 u = 0; u < t; ++u) if (tok[u] == tok[t]) { first = 0; break; }
        if (!first) continue;
        for (i64 c = 0; c < C; ++c) {
            float acc = 0.0f;
            for (i64 u = t; u < ntok; ++u) if (tok[u] == tok[t]) acc = acc + dx0[u * C + c];
            i64 o = (i64)tok[t] * C + c;
            dwte[o] = canon(dwte[o] + acc);
        }
    }
    if (dwpe) {
        i64 np = ntok < T ? ntok : T;
        for (i64 p = 0; p < np; ++p)
            for (i64 c = 0; c < C; ++c) {
                float acc = 0.0f;
                for (i64 u = p; u < ntok; u += T) acc = acc + dx0[u * C + c];
                dwpe[p * C + c] = canon(acc);
            }
    }
}

/* ======================================================================
 * R-TREE_S: canonical data-parallel gradient combine (reading R14; the paper
 * leaves the collective order to future work).  nparts is a power
 * of two; T(lo,1) = g_lo;  T(lo,n) = T(lo,n/2) + T(lo+n/2,n/2), elementwise.
 * ==================================================================== */
static float tree_elem(const float *const *parts, int lo, int n, i64 i) {
    if (n == 1) return parts[lo][i];
    return tree_elem(parts, lo, n / 2, i) + tree_elem(parts, lo + n / 2, n / 2, i);
}

void orc_tree_sum(const float *const *parts, int nparts, i64 n, float *out) {
    for (i64 i = 0; i < n; ++i) out[i] = canon(tree_elem(parts, 0, nparts, i));
}

/* ======================================================================
 * R-ADAMW (reading R15): Adam ("parameter updates and an optimizer
 * state update"; Adam state P:262) with decoupled weight decay, one fixed
 * elementwise chain.  bc1 = 1 - b1^t, bc2 = 1 - b2^t with b^t formed by t-1
 * float multiplications of b.
 *   m' = b1*m + (1-b1)*g;   v' = b2*v + (1-b2)*(g*g)
 *   upd = (m'/bc1) / (sqrt(v'/bc2) + eps);  if decay: upd = upd + wd*p
 *   p' = p - lr*upd
 * ==================================================================== */
static float powf_iter(float b, i64 t) {
    float r = b;
    for (i64 i = 1; i < t; ++i) r = r * b;
    return r;
}

void orc_adamw(float *p, const float *g, float *m, float *v, i64 n, i64 step,
               float lr, float b1, float b2, float eps, float wd, int decay) {
    float bc1 = 1.0f - powf_iter(b1, step);
    float bc2 = 1.0f - powf_iter(b2, step);
    float omb1 = 1.0f - b1, omb2 = 1.0f - b2;
    for (i64 i = 0; i < n; ++i) {
        float gi = g[i];
        float mi = (b1 * m[i]) + (omb1 * gi);
        float vi = (b2 * v[i]) + (omb2 * (gi * gi));
        float upd = (mi / bc1) / (sqrtf(vi / bc2) + eps);
        if (decay) upd = upd + wd * p[i];
        p[i] = canon(p[i] - lr * upd);
        m[i] = canon(mi);
        v[i] = canon(vi);
    }
}

/* ======================================================================
 * SHA-256, FIPS 180-4 -- the hash the paper names for commitments
 * ("a standard collision-resistant hash function like SHA-256").
 * Straight from the standard: message schedule, 64 rounds, big-endian.
 * ==================================================================== */
static const uint32_t K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

typedef struct { uint32_t h[8]; uint8_t buf[64]; uint64_t len; size_t fill; } orc_sha;

static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

static void sha_block(uint32_t *h, const uint8_t *blk) {
    uint32_t w[64];
    for (int t = 0; t < 16; ++t)
        w[t] = ((uint32_t)blk[4 * t] << 24) | ((uint32_t)blk[4 * t + 1] << 16) |
               ((uint32_t)blk[4 * t + 2] << 8) | (uint32_t)blk[4 * t + 3];
    for (int t = 16; t < 64; ++t) {
        uint32_t s0 = rotr(w[t - 15], 7) ^ rotr(w[t - 15], 18) ^ (w[t - 15] >> 3);
        uint32_t s1 = rotr(w[t - 2], 17) ^ rotr(w[t - 2], 19) ^ (w[t - 2] >> 10);
        w[t] = w[t - 16] + s0 + w[t - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int t = 0; t < 64; ++t) {
        uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        uint32_t ch = (e & f) ^ (~e & g);
        uint32_t t1 = hh + S1 + ch + K256[t] + w[t];
        uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        uint32_t maj = (a & b) ^ (a & c) ^ (b & c);
        uint32_t t2 = S0 + maj;
        hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

static void sha_init(orc_sha *s) {
    static const uint32_t H0[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                                   0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    memcpy(s->h, H0, sizeof H0);
    s->len = 0;
    s->fill = 0;
}

static void sha_update(orc_sha *s, const void *data, size_t n) {
    const uint8_t *p = (const uint8_t *)data;
    s->len += n;
    while (n > 0) {
        size_t take = 64 - s->fill;
        if (take > n) take = n;
        memcpy(s->buf + s->fill, p, take);
        s->fill += take; p += take; n -= take;
        if (s->fill == 64) { sha_block(s->h, s->buf); s->fill = 0; }
    }
}

static void sha_final(orc_sha *s, uint8_t out[32]) {
    uint64_t bits = s->len * 8u;
    uint8_t pad = 0x80;
    sha_update(s, &pad, 1);
    uint8_t z = 0;
    while (s->fill != 56) sha_update(s, &z, 1);
    uint8_t lenbe[8];
    for (int i = 0; i < 8; ++i) lenbe[i] = (uint8_t)(bits >> (56 - 8 * i));
    sha_update(s, lenbe, 8);
    for (int i = 0; i < 8; ++i) {
        out[4 * i] = (uint8_t)(s->h[i] >> 24); out[4 * i + 1] = (uint8_t)(s->h[i] >> 16);
        out[4 * i + 2] = (uint8_t)(s->h[i] >> 8); out[4 * i + 3] = (uint8_t)s->h[i];
    }
}

void orc_sha256(const uint8_t *data, i64 n, uint8_t out[32]) {
    orc_sha s;
    sha_init(&s);
    sha_update(&s, data, (size_t)n);
    sha_final(&s, out);
}

/* ======================================================================
 * R-MERKLE -- "a Merkle (binary hash) tree" over the node hashes (Fig. 2,
 * P:446-464).  Reading R12: RFC 6962 Merkle Tree Hash, written out as its
 * recursive definition:
 *   MTH({})   = SHA-256()
 *   MTH({d})  = SHA-256(0x00 || d)
 *   MTH(D[n]) = SHA-256(0x01 || MTH(D[0:k]) || MTH(D[k:n])),  k = largest power of two < n
 * Entry i is data[off[i] .. off[i+1]).
 * ==================================================================== */
static void mth_off(const uint8_t *data, const i64 *off, i64 lo, i64 n, uint8_t out[32]) {
    orc_sha s;
    sha_init(&s);
    if (n == 1) {
        uint8_t pre = 0x00;
        sha_update(&s, &pre, 1);
        sha_update(&s, data + off[lo], (size_t)(off[lo + 1] - off[lo]));
        sha_final(&s, out);
        return;
    }
    i64 k = 1;
    while (k * 2 < n) k *= 2;
    uint8_t l[32], r[32];
    mth_off(data, off, lo, k, l);
    mth_off(data, off, lo + k, n - k, r);
    uint8_t pre = 0x01;
    sha_update(&s, &pre, 1);
    sha_update(&s, l, 32);
    sha_update(&s, r, 32);
    sha_final(&s, out);
}

/* MTH over n variable-length entries (offsets has n+1 entries); n == 0 gives SHA-256(). */
void orc_mth(const uint8_t *data, const i64 *off, i64 n, uint8_t out[32]) {
    if (n == 0) { orc_sha256(NULL, 0, out); return; }
    mth_off(data, off, 0, n, out);
}

/* MTH over entries of `stride` bytes (the last one may be shorter: total nbytes) */
static void mth_strided(const uint8_t *data, i64 nbytes, i64 stride, uint8_t out[32]) {
    i64 n = (nbytes + stride - 1) / stride;
    i64 *off = (i64 *)malloc((size_t)(n + 1) * sizeof(i64));
    for (i64 i = 0; i < n; ++i) off[i] = i * stride;
    off[n] = nbytes;
    mth_off(data, off, 0, n, out);
    free(off);
}

/* Step root over n node digests (32 bytes each).  n == 0 is an error (-1). */
int orc_merkle_root(const uint8_t *leaves, i64 n, uint8_t out[32]) {
    if (n <= 0) return -1;
    mth_strided(leaves, 32 * n, 32, out);
    return 0;
}

/* R-TCOMMIT (reading R11): commitment to one tensor (an operator output,
 * "hashes of all tensors sent into and emitted out of the node").
 *   data bytes = little-endian binary32 image;  chunks of 4096 bytes (last short)
 *   data_root  = MTH(chunks)   (SHA-256() when nbytes == 0)
 *   digest     = SHA-256(0x54 || u8 dtype || u64le rank || u64le dims[rank] ||
 *                        u64le nbytes || u32le 4096 || data_root)            */
void orc_commit_tensor(const uint8_t *data, i64 nbytes, int dtype, int rank, const i64 *dims, uint8_t out[32]) {
    uint8_t root[32];
    if (nbytes == 0) orc_sha256(NULL, 0, root);
    else mth_strided(data, nbytes, 4096, root);
    orc_sha s;
    sha_init(&s);
    uint8_t b = 0x54;
    sha_update(&s, &b, 1);
    b = (uint8_t)dtype;
    sha_update(&s, &b, 1);
    uint8_t le[8];
    uint64_t vals[2 + 16];
    int nv = 0;
    if (rank > 16) rank = 16;
    vals[nv++] = (uint64_t)rank;
    for (int i = 0; i < rank; ++i) vals[nv++] = (uint64_t)dims[i];
    vals[nv++] = (uint64_t)nbytes;
    for (int q = 0; q < nv; ++q) {
        for (int i = 0; i < 8; ++i) le[i] = (uint8_t)(vals[q] >> (8 * i));
        sha_update(&s, le, 8);
    }
    uint8_t ch[4] = {0x00, 0x10, 0x00, 0x00}; /* 4096 little-endian */
    sha_update(&s, ch, 4);
    sha_update(&s, root, 32);
    sha_final(&s, out);
}

/* tensor data root alone (the MTH over 4096-byte chunks), for tests */
void orc_data_root(const uint8_t *data, i64 nbytes, uint8_t out[32]) {
    if (nbytes == 0) { orc_sha256(NULL, 0, out); return; }
    mth_strided(data, nbytes, 4096, out);
}
