/*
 * repops.h -- C ABI of the B200-native RepOps / Verde hot path (librepops.so).
 *
 * Paper: "Verde: Verification via Refereed Delegation for Machine Learning
 * Programs" (arXiv 2502.19405).  Citations "P:n" are lines of the paper text
 * (PAPER.md); "Rk" are the readings listed in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *   - Return an int status: REPOPS_OK (0) or a REPOPS_E* code.  The message of
 *     the last failure on the calling thread is repops_last_error().  No C++
 *     exception crosses this boundary.
 *   - Tensor pointers are DEVICE pointers owned by the caller; the library
 *     allocates nothing persistent and never frees caller memory.  Host
 *     pointers are marked (host) and are only borrowed for the call.
 *   - Layout is row-major with an explicit leading dimension (elements).
 *     Alignment is never required for correctness; aligned rows take 128-bit
 *     paths with identical bits.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Device entry
 *     points only enqueue work and return without synchronising.
 *   - Determinism contract: output bits are a pure function of the input
 *     bits, the shapes and the fixed constants of DESIGN.md §3 -- never of the
 *     stream, the tile configuration, the SM count or the number of GPUs.
 *   - All floating point is IEEE-754 binary32, round to nearest even, no
 *     flush-to-zero, no contraction (explicit fma only where written).  A NaN
 *     result is always written as the canonical 0x7FC00000 (R10).
 *   - NaN / Inf inputs are data, not errors.
 */
#ifndef REPOPS_H
#define REPOPS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define REPOPS_ABI_VERSION 1

enum repops_status {
    REPOPS_OK = 0,
    REPOPS_EINVAL = 1,   /* null pointer, negative size, ld < row length, bad enum */
    REPOPS_ESHAPE = 2,   /* shapes inconsistent (e.g. causal with rows % cols != 0) */
    REPOPS_ECUDA = 3,    /* a CUDA runtime call or kernel launch failed */
    REPOPS_ENOSPACE = 4  /* caller workspace too small */
};

enum repops_epilogue {
    REPOPS_EPI_NONE = 0,  /* C = acc                      */
    REPOPS_EPI_BIAS = 1,  /* C = fadd(acc, bias[j])       */
    REPOPS_EPI_SCALE = 2  /* C = fmul(acc, scale)         */
};

enum verde_dtype { VERDE_F32 = 1, VERDE_I32 = 2, VERDE_U8 = 3, VERDE_BF16 = 4, VERDE_F16 = 5 };

int repops_abi_version(void);
const char *repops_last_error(void);
/* Number of kernels this library has enqueued in this process (all threads).
 * bench.py reports the difference across its timed region as gpu_launches. */
int64_t repops_launch_count(void);

/* ------------------------------------------------------------------ GEMM
 * R-GEMM, PAPER.md P:598-609 (Sec. 3.2 listing): for every (i, j)
 *     acc = +0;  for k = 0 .. K-1 ascending: acc = fma(opA(i,k), opB(k,j), acc)
 *     C[i*ldc + j] = epi(acc)
 * opA(i,k) = transA ? A[k*lda + i] : A[i*lda + k]   (A is M x K, or K x M if transA)
 * opB(k,j) = transB ? B[j*ldb + k] : B[k*ldb + j]   (B is K x N, or N x K if transB)
 * K is never split; only M/N are tiled.  K == 0 gives C = epi(+0).
 * bias: device, N floats (epi == BIAS); scale: host float (epi == SCALE).
 * Errors: EINVAL for M,N,K < 0, null pointers with nonzero extent, lda/ldb/ldc
 * smaller than the stored row length, unknown epi. */
int repops_gemm(int64_t M, int64_t N, int64_t K,
                const float *A, int64_t lda, int transA,
                const float *B, int64_t ldb, int transB,
                int epi, const float *bias, float scale,
                float *C, int64_t ldc, void *stream);

/* Batched R-GEMM over a two-level batch (b0 < batch0, b1 < batch1), e.g.
 * (sequence, head) for attention.  Problem (b0, b1) uses
 *   A + b0*sA0 + b1*sA1,  B + b0*sB0 + b1*sB1,  C + b0*sC0 + b1*sC1   (elements).
 * Every problem is an independent R-GEMM with the same M, N, K, ld*, trans*. */
int repops_gemm_strided_batched(int64_t M, int64_t N, int64_t K,
                                const float *A, int64_t lda, int transA, int64_t sA0, int64_t sA1,
                                const float *B, int64_t ldb, int transB, int64_t sB0, int64_t sB1,
                                int epi, const float *bias, float scale,
                                float *C, int64_t ldc, int64_t sC0, int64_t sC1,
                                int64_t batch0, int64_t batch1, void *stream);

/* R-GEMM with its elementwise consumer fused into the epilogue: C as
 * repops_gemm, and C2[i][j] = R-GELU(C[i][j]) (post = REPOPS_POST_GELU) or
 * R-GELU-backward at X[i][j] with dy = C[i][j] (REPOPS_POST_GELU_BACKWARD).  C2's bits
 * equal repops_gelu / repops_gelu_backward applied to C (same device functions).
 * Shapes the fused A^T kernel does not take run the GEMM and the separate launch (then
 * C, C2, X must be contiguous: ld = N).  X, C2: device, caller-owned.  Errors: REPOPS_EINVAL. */
#define REPOPS_POST_GELU 1
#define REPOPS_POST_GELU_BACKWARD 2
int repops_gemm_post(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, int transA, const float *B,
                     int64_t ldb, int transB, int epi, const float *bias, float scale, float *C, int64_t ldc, int post,
                     const float *X, int64_t ldx, float *C2, int64_t ldc2, void *stream);

/* Causal structure of attention (R-ATTN, DESIGN R29 / R31), exact.
 * repops_gemm_strided_batched_causal: repops_gemm_strided_batched plus `causal`:
 *   0  none (identical to repops_gemm_strided_batched);
 *   1  outputs with column > row are NOT computed or written (the caller guarantees they
 *      are never read, e.g. operator-internal scores under R29 -- the causal softmax reads
 *      columns <= row only); all other outputs are bit-identical to the full GEMM;
 *   2  the caller guarantees op(A)[i][k] == +0 for k > i (causal softmax output).  Each
 *      output tile folds k only up to its last row; the skipped terms fma(+0, B[k][j], acc)
 *      are applied in closed form from kflags (below), so every output is bit-identical
 *      to the full K fold for every input, including non-finite B and -0 accumulators.
 *   kflags (causal 2, device, uint8): per problem [K + 1][ldf] from repops_causal_suffix_flags
 *   of the same B (problem strides sF0, sF1; ldf >= N).  op(A) = A and op(B) = B only
 *   (transA = transB = 0) for causal 2.  Errors: REPOPS_EINVAL.
 * repops_causal_suffix_flags: F[b][k][n] for k = 0..K (rows of stride ldf): bit 0 = some
 *   B[k'][n], k' >= k, is +-inf or NaN; bit 1 = every B[k'][n], k' >= k, has its sign bit
 *   set; row K = 2 (empty suffix).  B: K x N, row stride ldb, problem strides sB0, sB1;
 *   batch0 x batch1 problems.  Integer logic only. */
int repops_gemm_strided_batched_causal(int64_t M, int64_t N, int64_t K,
                                       const float *A, int64_t lda, int transA, int64_t sA0, int64_t sA1,
                                       const float *B, int64_t ldb, int transB, int64_t sB0, int64_t sB1,
                                       int epi, const float *bias, float scale,
                                       float *C, int64_t ldc, int64_t sC0, int64_t sC1,
                                       int64_t batch0, int64_t batch1, int causal, const uint8_t *kflags,
                                       int64_t ldf, int64_t sF0, int64_t sF1, void *stream);
int repops_causal_suffix_flags(const float *B, int64_t K, int64_t N, int64_t ldb, int64_t sB0, int64_t sB1,
                               int64_t batch0, int64_t batch1, uint8_t *flags, int64_t ldf, int64_t sF0,
                               int64_t sF1, void *stream);

/* Lower-precision STORAGE, binary32 compute ("RepOps works with any lower
 * precision ... (particularly FP16)"; reading R30).  dtypes: VERDE_F32, VERDE_BF16,
 * VERDE_F16 (2-byte elements).  Widening is exact; narrowing is IEEE round to nearest
 * even with gradual underflow and overflow to +-inf; NaN is written canonically
 * (0x7FC00000 / 0x7FC0 / 0x7E00).
 * repops_convert: dst[r][c] = convert(src[r][c]), rows x cols, leading dims lds / ldd in
 *   elements of their own type.  Errors: REPOPS_EINVAL (dtype, ld < cols, null).
 * repops_gemm_ex: C = narrow_c(R-GEMM(widen(op(A)), widen(op(B))) with epilogue `epi`);
 *   A, B, C device buffers of their dtypes; bias is float (binary32).  Operands that are
 *   not f32 are widened into the caller's workspace `ws` (device, >=
 *   repops_gemm_ex_workspace_bytes(...) bytes; REPOPS_ENOSPACE if smaller); the K fold
 *   is exactly R-GEMM's, so an all-f32 call equals repops_gemm bit for bit. */
int repops_convert(const void *src, int src_dtype, int64_t rows, int64_t cols, int64_t lds, void *dst, int dst_dtype,
                   int64_t ldd, void *stream);
int64_t repops_gemm_ex_workspace_bytes(int64_t M, int64_t N, int64_t K, int a_dtype, int b_dtype, int c_dtype);
int repops_gemm_ex(int64_t M, int64_t N, int64_t K, const void *A, int a_dtype, int64_t lda, int transA, const void *B,
                   int b_dtype, int64_t ldb, int transB, int epi, const float *bias, float scale, void *C, int c_dtype,
                   int64_t ldc, void *ws, int64_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ reductions
 * R-CSUM (R4): n <= 4096: 128 slots from +0, x[i] into slot i%128
 * ascending, then TREE128 (h = 64..1: p[s] = p[s] + p[s+h]); longer rows are
 * the CSUM of their 4096-element tile CSUMs.  Rows up to 4096*4096 elements.
 * out: device, rows floats. */
int repops_sum_rows(const float *x, int64_t rows, int64_t cols, int64_t ld, float *out, void *stream);

/* R-SEQ (R4): rows split into nseg equal contiguous segments (rows % nseg == 0);
 * out[s*ldo + j] = fold over the segment's rows ascending of (acc + x[r*ld+j]), acc = +0
 * (ldo >= cols: e.g. the flat per-shard gradient length, to write each shard's row in place). */
int repops_sum_cols_seq(const float *x, int64_t rows, int64_t cols, int64_t ld, int64_t nseg,
                        float *out, int64_t ldo, void *stream);

/* R-TREE_S (R14): out = T(parts[0..nparts)), T(lo,1) = parts[lo],
 * T(lo,n) = fadd(T(lo,n/2), T(lo+n/2,n/2)), elementwise over n floats.
 * parts: HOST array of nparts DEVICE pointers; nparts in {1,2,4,8,16}. */
int repops_tree_sum(const float *const *parts, int nparts, int64_t n, float *out, void *stream);

/* ------------------------------------------------------------------ row operators
 * R-SOFTMAX (R7): per row, m = max of the valid non-NaN entries (+0 if zero);
 * e_i = exp(x_i - m); s = CSUM(e); y_i = e_i * (1/s).  causal != 0 requires
 * rows % cols == 0; row r keeps (r mod cols)+1 entries and writes +0 elsewhere.
 * y may alias x when ldy == ldx. */
int repops_softmax(const float *x, int64_t rows, int64_t cols, int64_t ldx, int causal,
                   float *y, int64_t ldy, void *stream);

/* R-SOFTMAX-BWD: c = CDOT(y, dy) over the full row; dx_i = fmul(fmul(y_i, dy_i - c), scale).
 * dx may alias dy. */
int repops_softmax_backward(const float *y, int64_t ldy, const float *dy, int64_t lddy,
                            int64_t rows, int64_t cols, float scale, float *dx, int64_t lddx,
                            void *stream);

/* R-LN (P:834-835 lists LayerNorm among RepOps operators; R8): contiguous rows.
 * mu = CSUM(x)/n; d = x - mu; var = CDOT(d,d)/n; rstd = 1/sqrt(var + eps);
 * y = fma(d*rstd, gamma, beta).  mean / rstd (rows floats) are optional (NULL). */
int repops_layernorm(const float *x, const float *gamma, const float *beta, int64_t rows,
                     int64_t cols, float eps, float *y, float *mean, float *rstd, void *stream);

/* LN backward, row part: xh = (x - mean)*rstd; g = dy*gamma; a = CSUM(g)/n;
 * b = CDOT(g, xh)/n; dx = ((g - a) - xh*b)*rstd; if dres != NULL: dx = dres + dx. */
int repops_layernorm_backward(const float *dy, const float *x, const float *gamma,
                              const float *mean, const float *rstd, const float *dres,
                              int64_t rows, int64_t cols, float *dx, void *stream);

/* LN parameter gradients per segment (R-SEQ): dgamma[s*ldo + j] = fold fma(dy, xh, acc),
 * dbeta[s*ldo + j] = fold (acc + dy), xh = (x - mean)*rstd recomputed as in the forward. */
int repops_layernorm_backward_params(const float *dy, const float *x, const float *mean,
                                     const float *rstd, int64_t rows, int64_t cols, int64_t nseg,
                                     float *dgamma, float *dbeta, int64_t ldo, void *stream);

/* R-CE: per row of V logits: m = max; s = CSUM(exp(x - m));
 * loss[r] = (m + log s) - x[label];  dlogits_i = ((exp(x_i - m)*(1/s)) - [i == label]) * scale.
 * labels: device int32[rows], each in [0, V).  loss / dlogits optional (NULL);
 * dlogits may alias logits (ldd == ld). */
int repops_cross_entropy(const float *logits, int64_t rows, int64_t V, int64_t ld,
                         const int32_t *labels, float scale, float *loss, float *dlogits,
                         int64_t ldd, void *stream);

/* Fused causal attention forward (P:571-574 operators, R-ATTN):
 * per (b0 < batch0, b1 < batch1) with Q = Q + b0 s0 + b1 s1 (same for K, V), rows of
 * stride ld, head dim hd:
 *   S[i][j] = R-GEMM(Q, K^T) with the SCALE epilogue (every j < T),
 *   P       = R-SOFTMAX(S) (causal: row i keeps keys j <= i, masked P = +0),
 *   O[i][n] = R-GEMM(P, V) over all T keys.
 * Bit-identical to repops_gemm_strided_batched(SCALE) -> repops_softmax -> repops_gemm:
 * the same operation sequence per element, without the HBM round trips of S and P.
 * S, P: [T][T] blocks at S + b0 sp0 + b1 sp1 (row stride T), optional (NULL = not
 * stored).  O: rows of stride ldo at O + b0 so0 + b1 so1.  All rows 16-byte aligned.
 * Supported: hd = 64, T % 128 == 0, T <= 512 (repops_attention_fwd_supported);
 * otherwise REPOPS_ESHAPE (use the unfused composition).  REPOPS_EINVAL: null,
 * misaligned, ld < hd. */
int repops_attention_fwd_supported(int64_t T, int64_t hd);
int repops_attention_fwd(int64_t T, int64_t hd, const float *Q, const float *K, const float *V, int64_t ld,
                         int64_t s0, int64_t s1, float scale, int causal, float *S, float *P, int64_t sp0,
                         int64_t sp1, float *O, int64_t ldo, int64_t so0, int64_t so1, int64_t batch0,
                         int64_t batch1, void *stream);

/* Attention scores + softmax fused, the probabilities only (f4, R7, R29, R31):
 * per (b0 < batch0, b1 < batch1), with Q rows of stride ldq at Q + b0 sq0 + b1 sq1 and K
 * rows of stride ldk at K + b0 sk0 + b1 sk1 (head dim hd; sk1 = 0 shares one K among the
 * inner batch, e.g. grouped-query attention), P = R-SOFTMAX(R-GEMM(Q, K^T) with the SCALE
 * epilogue) (causal: row i keeps keys j <= i, masked P = +0, every element of the [T][T]
 * block written).  The scores stay in shared memory (operator scratch, R29); with causal set
 * only the key blocks a CTA's rows read are computed (R31).  Bit-identical to
 * repops_gemm_strided_batched(SCALE) -> repops_softmax.  P: [T][T] blocks at
 * P + b0 sp0 + b1 sp1 (row stride T); device, caller-owned, 16-byte aligned rows.
 * Supported (repops_attention_probs_supported): hd = 64 with T % 32 == 0, T <= 1024 (GPT-2),
 * hd = 128 with T % 16 == 0, T <= 2048 (Llama), else REPOPS_ESHAPE; REPOPS_EINVAL: null,
 * misaligned, ldq / ldk < hd. */
int repops_attention_probs_supported(int64_t T, int64_t hd);
int repops_attention_probs(int64_t T, int64_t hd, const float *Q, int64_t ldq, int64_t sq0, int64_t sq1,
                           const float *K, int64_t ldk, int64_t sk0, int64_t sk1, float scale, int causal,
                           float *P, int64_t sp0, int64_t sp1, int64_t batch0, int64_t batch1, void *stream);

/* The backward twin (f4; R7's backward, R29): per (b0, b1), dP = R-GEMM(dO, V^T) (no
 * epilogue) over every key, kept in shared memory, then the softmax backward of each row:
 * c = CDOT(P row, dP row), dS = canon(fmul(fmul(P, fsub(dP, c)), scale)).  Bit-identical to
 * repops_gemm_strided_batched(dO, V^T) -> repops_softmax_backward(P, dP, scale).  dO rows:
 * stride ldo at dO + b0 so0 + b1 so1; V rows: stride ldv at V + b0 sv0 + b1 sv1 (head dim
 * hd); P, dS: [T][T] blocks (row stride T) at P + b0 sp0 + b1 sp1, dS + b0 sd0 + b1 sd1;
 * device, caller-owned, 16-byte aligned rows.  Supported: hd = 64, T % 32 == 0, T <= 1024
 * (REPOPS_ESHAPE otherwise); REPOPS_EINVAL: null, misaligned, ldo / ldv < hd. */
int repops_attention_dscores(int64_t T, int64_t hd, const float *dO, int64_t ldo, int64_t so0, int64_t so1,
                             const float *V, int64_t ldv, int64_t sv0, int64_t sv1, const float *P, int64_t sp0,
                             int64_t sp1, float scale, float *dS, int64_t sd0, int64_t sd1, int64_t batch0,
                             int64_t batch1, void *stream);

/* ------------------------------------------------------------------ elementwise
 * Software math (R5/R6): fixed IEEE-RN op chains. */
int repops_exp(const float *x, int64_t n, float *y, void *stream);
int repops_log(const float *x, int64_t n, float *y, void *stream);
int repops_tanh(const float *x, int64_t n, float *y, void *stream);
int repops_rsqrt(const float *x, int64_t n, float *y, void *stream);   /* fdiv(1, fsqrt(x)) */
int repops_gelu(const float *x, int64_t n, float *y, void *stream);    /* tanh form, R13 */
int repops_gelu_backward(const float *x, const float *dy, int64_t n, float *dx, void *stream);
int repops_add(const float *a, const float *b, int64_t n, float *y, void *stream);
/* ReLU (config-1 MLP; reading R24): y = x > 0 ? x : +0 (-0 and negatives
 * give +0); dx = x > 0 ? g : +0 (subgradient 0 at x = 0); a NaN x gives the canonical NaN.
 * x, g, y, dx: device float[n], contiguous; y / dx may alias x / g. */
int repops_relu(const float *x, int64_t n, float *y, void *stream);
/* sin / cos (P:572 lists them among the re-implemented functions; reading R26): the
 * Cephes sinf / cosf chains; |x| > 16777215 -> +0, +-inf / NaN -> NaN. */
int repops_sin(const float *x, int64_t n, float *y, void *stream);
int repops_cos(const float *x, int64_t n, float *y, void *stream);
/* erf and exact GELU (BERT-family models; "LayerNorm, GeLU, and ERF"; reading R27):
 * erf = the Cephes erff / erfcf chain (DESIGN.md §3 R27, exp = R-EXP); NaN -> canonical NaN.
 * gelu_erf: y = fmul(fmul(0.5, x), fadd(1, erf(fmul(x, 1/sqrt 2)))).
 * gelu_erf_backward: dx = dy * (cdf + x * pdf), cdf = 0.5 (1 + erf(x / sqrt 2)),
 * pdf = R-EXP(-(0.5 x^2)) * 1/sqrt(2 pi), each product / sum one rounded op in that order.
 * x, dy, y, dx: device float[n], contiguous (any alignment); y / dx may alias x / dy.
 * Errors: REPOPS_EINVAL for n < 0 or a null pointer with n > 0. */
int repops_erf(const float *x, int64_t n, float *y, void *stream);
int repops_gelu_erf(const float *x, int64_t n, float *y, void *stream);
int repops_gelu_erf_backward(const float *x, const float *dy, int64_t n, float *dx, void *stream);
/* Deterministic pseudorandomness (reading R28): Philox4x32-10 (curand's /
 * PyTorch's CUDA counter-based generator).  Element i = word (i mod 4) of the Philox
 * block with counter (floor(i/4) lo, hi, stream_id lo, hi) and key (seed lo, hi);
 * u_i = (word >> 8) * 2^-24 in [0, 1).  Pure function of (seed, stream_id, i): any
 * launch configuration, any device, any slicing of i gives the same draws.
 * repops_rand_uniform: y[i] = u_i (device float[n]).
 * repops_dropout: keep_i = u_i >= p, scale = fdiv(1, fsub(1, p)),
 *   y[i] = keep_i ? fmul(x[i], scale) : +0; mask (device uint8[n], nullable) = keep_i.
 * repops_dropout_backward: dx[i] = keep_i ? fmul(dy[i], scale) : +0 (mask regenerated).
 * y / dx may alias x / dy.  Errors: REPOPS_EINVAL (n < 0, p outside [0, 1], null). */
int repops_rand_uniform(uint64_t seed, uint64_t stream_id, int64_t n, float *y, void *stream);
int repops_dropout(const float *x, int64_t n, float p, uint64_t seed, uint64_t stream_id, float *y, uint8_t *mask,
                   void *stream);
int repops_dropout_backward(const float *dy, int64_t n, float p, uint64_t seed, uint64_t stream_id, float *dx,
                            void *stream);
/* RoPE tables (R26): cos[t][i] = R-COS(a), sin[t][i] = R-SIN(a), a = fmul(float(t), inv_freq[i]),
 * t < T (< 2^24), i < h.  inv_freq: device float[h]; cos, sin: device float[T * h] (row-major). */
int repops_rope_tables(const float *inv_freq, int64_t T, int64_t h, float *cosv, float *sinv, void *stream);
int repops_relu_backward(const float *x, const float *g, int64_t n, float *dx, void *stream);

/* R-EMB forward: x0[t][c] = fadd(wte[tok[t]][c], wpe[t mod T][c]); tok device int32. */
int repops_embedding(const int32_t *tok, int64_t ntok, int64_t T, const float *wte,
                     const float *wpe, int64_t C, float *x0, void *stream);
/* R-EMB backward for one data-parallel shard.  dwte is accumulated INTO (it holds
 * the tied lm-head gradient of the shard), dwpe is overwritten:
 * dwte[v][c] = fadd(dwte[v][c], fold over t ascending with tok[t]==v of (acc + dx0[t][c]));
 * dwpe[p][c] = fold over t ascending with t mod T == p (p < min(ntok, T)).  Untouched
 * rows keep their bits.  dwpe may be NULL. */
int repops_embedding_backward(const int32_t *tok, int64_t ntok, int64_t T, const float *dx0,
                              int64_t C, float *dwte, float *dwpe, void *stream);

/* R-ADAMW (R15): in place on p, m, v (n floats), g read-only.  bc1 = 1 - b1^step,
 * bc2 = 1 - b2^step with b^step by iterated binary32 multiplication (host side). */
int repops_adamw(float *p, const float *g, float *m, float *v, int64_t n, int64_t step,
                 float lr, float b1, float b2, float eps, float wd, int decay, void *stream);
/* R-ADAMW over nseg (<= 256) parameter tensors stored back to back in p, g, m, v
 * (one launch per optimizer step): tensor k = elements [seg_start[k], seg_start[k+1]),
 * seg_start[0] == 0, with weight decay iff decay[k] != 0.  Bit-identical to nseg
 * repops_adamw calls.  seg_start (nseg + 1) and decay (nseg) are host arrays. */
int repops_adamw_segments(float *p, const float *g, float *m, float *v, int nseg, const int64_t *seg_start,
                          const uint8_t *decay, int64_t step, float lr, float b1, float b2, float eps, float wd,
                          void *stream);

/* ------------------------------------------------------------------ Llama operators (config 4)
 * R-RMSNORM (R20): ms = CDOT(x,x)/n; rstd = fdiv(1, fsqrt(ms + eps)); y = fmul(fmul(x, rstd), w).
 * Contiguous rows, cols <= 4096; rstd (rows floats) optional. */
int repops_rmsnorm(const float *x, const float *w, int64_t rows, int64_t cols, float eps, float *y, float *rstd,
                   void *stream);
/* R-SWIGLU (R21): h = fmul(fdiv(g, fadd(1, exp(-g))), u), exp = R-EXP, -g an exact sign flip. */
int repops_swiglu(const float *g, const float *u, int64_t n, float *h, void *stream);
/* R-ROPE (R22), rotate-half form with cos/sin tables [ntok, hd/2] given as inputs:
 * y_i = x_i c_i - x_{i+h} s_i,  y_{i+h} = x_{i+h} c_i + x_i s_i  per (token, head), h = hd/2.
 * x, y: [ntok, ld/ldy] rows holding nhead*hd values; y may alias x. */
int repops_rope(const float *x, int64_t ntok, int64_t nhead, int64_t hd, int64_t ld, const float *cos_t,
                const float *sin_t, float *y, int64_t ldy, void *stream);
/* out[t][c] = table[idx[t]][c] (exact gather; token embedding without positions). */
int repops_gather_rows(const float *table, const int32_t *idx, int64_t n, int64_t C, float *out, void *stream);
/* Synthetic-input generator (not part of the method): out[i] = the SplitMix64
 * uniform of synth.uniform(seed) (24-bit grid in [-1,1), times `scale` rounded
 * once); lets multi-GB weights be generated on the device bit-identically. */
int repops_fill_uniform(float *out, int64_t n, uint64_t seed, double scale, void *stream);

/* Strided 2-D copy (data movement only): dst[r*ldd + c] = src[r*lds + c], r < rows, c < cols.
 * Used to place all-gathered tensor-parallel column blocks into one activation. */
int repops_copy2d(const float *src, int64_t rows, int64_t cols, int64_t lds, float *dst, int64_t ldd, void *stream);
/* Batched form: for b < nb, dst + b*sd <- src + b*ss (rows x cols, row strides lds / ldd;
 * element offsets).  One launch places all nb tensor-parallel blocks of an activation. */
int repops_copy2d_batched(const float *src, int64_t rows, int64_t cols, int64_t lds, int64_t ss, float *dst,
                          int64_t ldd, int64_t sd, int64_t nb, void *stream);

/* Transpose (data movement only, bit-exact): y[j*ldy + i] = x[i*ldx + j] for a
 * rows x cols x.  Used to give backward GEMMs an n-contiguous weight operand. */
int repops_transpose(const float *x, int64_t rows, int64_t cols, int64_t ldx, float *y, int64_t ldy, void *stream);

/* Fault injection (Verde config 5): flips bit `bit` (0..31) of 32-bit element
 * `elem` of the device buffer `data`. */
int repops_flip_bit(void *data, int64_t elem, int bit, void *stream);

/* ------------------------------------------------------------------ Verde commitments
 * R-TCOMMIT (P:240-244 SHA-256 commitment; P:393-406 tensor hashes in the node;
 * R11): data bytes (little-endian image) are cut into 4096-byte chunks (last
 * one short); leaf_i = SHA-256(0x00 || chunk_i); data_root = RFC 6962 MTH
 * (SHA-256() for 0 bytes); digest = SHA-256(0x54 || u8 dtype || u64le rank ||
 * u64le dims[rank] || u64le nbytes || u32le 4096 || data_root).            */
typedef struct {
    const void *data;   /* device */
    int64_t nbytes;
    int32_t dtype;      /* verde_dtype */
    int32_t rank;       /* 0..8 */
    int64_t dims[8];
    uint8_t *digest;    /* device, 32 bytes */
    int32_t mode;       /* 0 = tensor digest; 1 = data_root only (MTH over chunks, no header) */
    int32_t reserved;
    /* Incremental commitment of a tensor rewritten in place in a few chunks (all optional,
     * NULL = unused; the digest is the same R-TCOMMIT digest either way):
     * leaves_out  device [nchunks x 32 B]: the chunk leaf hashes are also stored here (an
     *             opaque per-chunk leaf record, only meant to be passed as base_leaves);
     * base_leaves device [nchunks x 32 B] from an earlier leaves_out of a tensor of the same
     *             nbytes, with dirty: device uint8 [nchunks]: chunk c is hashed iff dirty[c]
     *             != 0, otherwise its leaf is taken from base_leaves[c].  The CALLER
     *             guarantees that every clean chunk holds exactly the bytes base_leaves[c]
     *             was hashed from (e.g. EMBED_BWD, which adds into the rows of the shard's
     *             tokens only); chunks are then not re-read, so a violated guarantee gives a
     *             digest of the wrong bytes. */
    uint8_t *leaves_out;
    const uint8_t *base_leaves;
    const uint8_t *dirty;
} verde_tensor_desc;

/* Digest of a tensor whose byte image was committed as k equal, contiguous
 * slabs (one per GPU, mode = 1): each slab must hold 2^j whole 4096-byte
 * chunks, so every slab root is an aligned RFC 6962 subtree and the tensor's
 * data_root is the plain binary tree SHA-256(0x01 || L || R) over the k slab
 * roots (k a power of two).  Identical to committing the whole tensor.
 * subroots, dims, out32: host.  EINVAL if the slab geometry is not aligned. */
int verde_digest_from_subroots(const uint8_t *subroots, int64_t k, int dtype, int rank, const int64_t *dims,
                               int64_t nbytes, uint8_t *out32);

/* Dirty-chunk flags for an incremental commitment (verde_tensor_desc.dirty) of a row-major
 * tensor whose rows `rows[0..n)` (int32, device; duplicates allowed) were rewritten:
 * flags[c] = 1 iff bytes [4096 c, 4096 c + 4096) of the tensor meet one of those rows
 * (row r = bytes [r row_bytes, (r + 1) row_bytes)), else 0; all = 1 sets every flag (full
 * re-hash).  flags: device uint8 [nchunks], nchunks = ceil(nbytes / 4096).  One launch. */
int verde_dirty_chunks(const int32_t *rows, int64_t n, int64_t row_bytes, int64_t nbytes, int all,
                       uint8_t *flags, void *stream);

/* Diagnostic (measurement aid, not part of the method): the R-GEMM's practical FP32 ceiling.
 * ctas x 128 threads each run `iters` rounds of 32 independent FFMA2 (64 FMA = 128 flops)
 * on register-resident operands -- no loads, no shared memory.  out: device float
 * [ctas * 128] (a fold of each thread's accumulators).  Time it with events on `stream`. */
int repops_ffma2_probe(int64_t ctas, int64_t iters, float *out, void *stream);

/* Diagnostic (measurement aid, not part of the method): the commitment's practical ALU
 * ceiling.  ctas x 128 threads each run `iters` SHA-256 compressions (the leaf kernel's
 * instruction sequence) on a register-resident block -- no memory traffic; 64 bytes per
 * compression.  out: device uint32 [ctas * 128] (a fold of each thread's final state, so
 * nothing is optimised away).  Time it with events on `stream`. */
int verde_sha256_probe(int64_t ctas, int64_t iters, uint32_t *out, void *stream);

/* Workspace (device bytes) needed to commit the given tensors in one call. */
int64_t verde_commit_workspace_bytes(const verde_tensor_desc *descs /* host */, int n);
/* Commit n tensors in one batched launch sequence; digests are written to
 * device memory asynchronously.  ws: device workspace >= the size above. */
int verde_commit_tensors(const verde_tensor_desc *descs /* host */, int n, void *ws,
                         int64_t ws_bytes, void *stream);
/* Reusable commit of a fixed set of tensors (static shapes and addresses, as
 * in a training step that re-uses its buffers).  create() builds the plan and
 * uploads its tables into `ws` with one synchronous copy; every run() then
 * only enqueues the leaf / reduce / header kernels on `stream` (no host
 * traffic, capturable in a CUDA graph).  `ws` (>= verde_commit_workspace_bytes)
 * is owned by the caller and must outlive the plan; runs of one plan must not
 * overlap.  destroy() frees the host-side plan object. */
typedef struct verde_commit_plan verde_commit_plan;
int verde_commit_plan_create(const verde_tensor_desc *descs /* host */, int n, void *ws, int64_t ws_bytes,
                             verde_commit_plan **plan);
int verde_commit_plan_run(const verde_commit_plan *plan, void *stream);
void verde_commit_plan_destroy(verde_commit_plan *plan);

/* Single-tensor convenience form (dims: host int64[rank]). */
int verde_commit_tensor(const void *data, int64_t nbytes, int dtype, int rank, const int64_t *dims,
                        uint8_t *digest32, void *ws, int64_t ws_bytes, void *stream);

/* R-MERKLE (Fig. 2; R12): RFC 6962 MTH over n 32-byte entries (host),
 * root32 (host).  n == 0 -> REPOPS_EINVAL. */
int verde_merkle_root(const uint8_t *leaves, int64_t n, uint8_t *root32);

/* RFC 6962 MTH over n leaf HASHES (MTH of one leaf = the leaf hash itself), e.g.
 * the chunk leaves of verde_chunk_leaves: equals the data_root of R11.  Host. */
int verde_merkle_root_hashed(const uint8_t *leaf_hashes, int64_t n, uint8_t *root32);

/* Merkle membership proofs (Fig. 2 caption; Case 2(a)):
 * RFC 6962 §2.1.1 audit path PATH(m, D[n]) of item m, sibling roots leaf level first.
 * items: n x 32 host bytes, entries (hashed = 0: leaf = SHA-256(0x00 || entry)) or
 * leaf hashes (hashed = 1).  path: host, room for 64 x 32 bytes; *len = path length. */
int verde_merkle_audit_path(const uint8_t *items, int64_t n, int64_t m, int hashed, uint8_t *path, int32_t *len);
/* RFC 9162 §2.1.3.2 check that leaf_hash is item m of an n-leaf tree with root32;
 * *ok = 1 if it is, 0 otherwise (a failed proof is not an error).  All host. */
int verde_merkle_verify_path(const uint8_t *leaf_hash, int64_t m, int64_t n, const uint8_t *path, int32_t len,
                             const uint8_t *root32, int *ok);

/* R-TCOMMIT header over a given data root: SHA-256(0x54 || dtype || rank || dims ||
 * nbytes || 4096 || data_root) (data_root ignored, SHA-256 of nothing used, when
 * nbytes == 0).  Lets the referee check claimed chunk leaves against a tensor
 * digest.  Host. */
int verde_tensor_digest_from_root(const uint8_t *data_root, int dtype, int rank, const int64_t *dims,
                                  int64_t nbytes, uint8_t *out32);

/* R11 leaf hashes SHA-256(0x00 || chunk) of every 4096-byte chunk of a device
 * buffer (last chunk ragged) into leaves (device, ceil(nbytes/4096) x 32 bytes):
 * what a trainer serves for intra-tensor bisection. */
int verde_chunk_leaves(const void *data, int64_t nbytes, uint8_t *leaves, void *stream);

/* As verde_first_divergence, over leaf HASHES (the trees of verde_merkle_root_hashed). */
int verde_first_divergence_hashed(const uint8_t *seq0, const uint8_t *seq1, int64_t n, int64_t *d_out,
                                  int64_t *rounds_out);

/* SHA-256 of a host buffer (host). */
int verde_sha256(const uint8_t *data, int64_t n, uint8_t *out32);

/* R-NODE (the AugmentedCGNode box; R13 in DESIGN.md): the node digest
 * SHA-256( 0x4E || u32 index || u16 op || u32 shard || u32 n_attr ||
 *          (u32 key, u64 value)*n_attr || u32 n_in || (u32 src_node, u32 src_slot)*n_in ||
 *          u32 n_out_nodes || (u32 dst_node)*n_out_nodes || u32 n_out ||
 *          in_digests (32*n_in) || out_digests (32*n_out) ), little-endian. All host. */
typedef struct {
    uint32_t index;
    uint16_t op;
    uint32_t shard;
    int32_t n_attr;
    const uint32_t *attr_keys;   /* ascending */
    const uint64_t *attr_vals;
    int32_t n_in;
    const uint32_t *in_src_node;
    const uint32_t *in_src_slot;
    const uint8_t *in_digests;   /* 32 * n_in */
    int32_t n_dst;
    const uint32_t *dst_nodes;
    int32_t n_out;
    const uint8_t *out_digests;  /* 32 * n_out */
} verde_node;

int verde_node_digest(const verde_node *node, uint8_t *out32);

/* Batched R-NODE + R-MERKLE for a whole step (all host).  Node i's digest is
 * SHA-256( blob[offs[i] .. offs[i+1]) || table[slots[j]] for j in [soffs[i], soffs[i+1]) )
 * where blob holds the static part of each node's serialisation above (0x4E ..
 * u32 n_out) and the slots name its input then output tensor digests in
 * `table` (n_slots x 32 bytes).  out: n x 32 node digests; root32 (nullable):
 * RFC 6962 MTH over them -- the step checkpoint (Fig. 2). */
int verde_node_digests(int64_t n, const uint8_t *blob, const int64_t *offs, const int64_t *slots,
                       const int64_t *soffs, const uint8_t *table, int64_t n_slots, uint8_t *out,
                       uint8_t *root32);

/* The same step root computed on the DEVICE from device-resident inputs, as a
 * reusable plan: blob/offs/slots/soffs are the static node serialisations and
 * slot lists above (device copies), table the device digest table that the
 * commit plans fill.  run() enqueues: one thread per node hashing its
 * serialisation + gathered digests; RFC 6962 leaves; aligned 256-group reduce
 * passes; writes node_out (n x 32, nullable) and root_out (32 bytes, device).
 * ws >= verde_root_plan_workspace_bytes(n) is caller-owned and outlives the plan. */
typedef struct verde_root_plan verde_root_plan;
int64_t verde_root_plan_workspace_bytes(int64_t n);
int verde_root_plan_create(int64_t n, const uint8_t *blob, const int64_t *offs, const int64_t *slots,
                           const int64_t *soffs, const uint8_t *table, uint8_t *node_out, uint8_t *root_out,
                           void *ws, int64_t ws_bytes, verde_root_plan **plan);
int verde_root_plan_run(const verde_root_plan *plan, void *stream);
void verde_root_plan_destroy(verde_root_plan *plan);

/* First index d with seq0[d] != seq1[d] over n 32-byte digests (Alg. 2 line 8,
 * P:429-430), found by descending the two RFC 6962 trees from the roots
 * (O(log n) subtree comparisons).  *d_out = -1 if the sequences are equal. */
int verde_first_divergence(const uint8_t *seq0, const uint8_t *seq1, int64_t n, int64_t *d_out,
                           int64_t *rounds_out);

/* ------------------------------------------------------------------ peer memory (multi-GPU DP combine)
 * R-TREE_S over G ranks as one kernel per rank over NVLink peer memory (reading R14;
 * the combine order of the collective is future work in the paper, P:642-650;
 * SURVEY §8(f) f1).  Memory exchanged between processes is allocated here and shared
 * with CUDA IPC handles (64 opaque bytes, passed between ranks by the caller, e.g.
 * over torch.distributed).  These are the only entry points that allocate.
 *
 * repops_ipc_alloc: cudaMalloc(nbytes) zero-filled; *ptr = device pointer owned by the
 *   caller (release with repops_ipc_free), handle64 (host, 64 bytes) = its IPC handle.
 * repops_ipc_open: map a peer's handle into this process (*ptr; unmap with
 *   repops_ipc_close).  A handle cannot be opened in the process that created it.
 * repops_p2p_tree_combine: for i in [lo, hi):
 *     v = balanced tree over q of parts[q][i] (((p0+p1)+(p2+p3))+..., fadd, R-TREE_S top
 *     levels), outs[q][i] = v for every q.
 *   parts / outs: host arrays of G device pointers (local or peer-mapped), each a
 *   float[>= hi] buffer; G in {1, 2, 4, 8}.  Bits equal repops_tree_sum(parts, G) on
 *   [lo, hi) for any slicing.  status: nullable device int32 written by a preceding
 *   repops_p2p_wait on the same stream; when *status != 0 (a peer did not signal in
 *   time) the kernel stores nothing, so no stale partial reaches any rank's gradient
 *   buffer and no peer buffer is written while a late peer may still read it; the
 *   caller must check the status before trusting the step (P2PTreeCombine.check).
 *   Errors: REPOPS_EINVAL (bad G, slice, null pointer).
 * repops_p2p_signal: after all prior work on `stream`, release-store (system scope)
 *   `epoch` into peer_flags[q][slot] for every q < G (peer_flags: host array of G device
 *   uint32 arrays of >= G entries, local or peer-mapped).
 * repops_p2p_wait: stall `stream` until every flags[j], j < G, has reached `epoch`
 *   (wrap-around compare), acquire (system scope).  Bounded: after timeout_ms the wait
 *   gives up and, if status (device int32) is non-null, sets *status = 1. */
int repops_ipc_alloc(int64_t nbytes, void **ptr, uint8_t *handle64);
int repops_ipc_open(const uint8_t *handle64, void **ptr);
int repops_ipc_close(void *ptr);
int repops_ipc_free(void *ptr);
int repops_p2p_tree_combine(const float *const *parts, int G, int64_t lo, int64_t hi, float *const *outs,
                            const int32_t *status, void *stream);
int repops_p2p_signal(uint32_t *const *peer_flags, int G, int slot, uint32_t epoch, void *stream);
int repops_p2p_wait(const uint32_t *flags, int G, uint32_t epoch, int64_t timeout_ms, int32_t *status,
                    void *stream);

#ifdef __cplusplus
}
#endif
#endif /* REPOPS_H */
