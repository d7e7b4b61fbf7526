// attention.cu -- fused non-online causal attention forward.
//
// One CTA owns BM = 64 query rows of one (batch, head) and keeps their FULL score
// rows in shared memory (no online softmax, so no rescaling and no reordering):
//   phase 1  S[i][j] = canon(fmul(fold_{k ascending} fma(Q[i,k], K[j,k], +0), scale))
//            for every key j (R-GEMM with the SCALE epilogue), K streamed
//            through shared memory in 128-key chunks (cp.async double buffer);
//   phase 2  P = R-SOFTMAX causal of each row (reading R7): warp per row, max over
//            the valid keys, exp_rn, the 128-slot CSUM + TREE128, y = e * fdiv(1, s);
//   phase 3  O[i][n] = canon(fold_{j ascending over ALL T keys} fma(P[i][j], V[j][n], +0))
//            (R-GEMM, masked P = +0 terms included exactly as the unfused GEMM does).
// Every output element is produced by the same operation sequence as the unfused
// composition repops_gemm(SCALE) -> repops_softmax(causal) -> repops_gemm, so S, P and O
// are bit-identical to it (and to the oracle); what the fusion removes is the HBM
// round trip of S and P between three launches.  S / P are written only if requested
// (they are committed tensors of the GPT-2 step).
//
// Shapes: head dim 64, T a multiple of 128 and <= 512 (GPT-2); other shapes are
// rejected by the ABI (the unfused path covers them).
#include <cstdlib>

#include "attention.cuh"
#include "common.cuh"

#ifndef RO_ATTN_VARIANT_DEFAULT
#define RO_ATTN_VARIANT_DEFAULT 3
#endif

namespace {

using namespace ro;

constexpr int HD = 64;
constexpr int KLD = HD + 4;  // K chunk row stride (words): rows of one warp fall in distinct banks
// variants: <BM query rows, KC keys per chunk, THREADS>.  (64, 128, 256): 213 KB, 1 CTA / SM;
// (32, 64, 128): 109 KB, 2 CTAs / SM so one CTA's softmax overlaps the other's FFMA2 phases

RO_DEV void cp16(float *dst, const float *src) {
    unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
RO_DEV void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
RO_DEV void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

struct AttnArgs {
    const float *Q, *K, *V;
    int64_t ld, s0, s1;      // row stride of Q/K/V, batch strides (outer, inner)
    float *S, *P;            // [T][T] per (batch, head), may be null
    int64_t sp0, sp1;
    float *O;
    int64_t ldo, so0, so1;
    int64_t batch1, nbatch;
    int T;
    int causal, skip;
    float scale;
};

// rows [r0, r0 + KC) of a [.][HD] operand (row stride ld) -> dst rows of stride DLD
template <int DLD, int KC, int THREADS>
RO_DEV void load_chunk(float *dst, const float *src, int64_t ld, int tid) {
#pragma unroll
    for (int q = 0; q < KC * HD / 4 / THREADS; ++q) {
        const int c = tid + q * THREADS;
        const int r = c / (HD / 4), k4 = (c % (HD / 4)) * 4;
        cp16(dst + r * DLD + k4, src + (int64_t)r * ld + k4);
    }
}

template <int BM, int KC, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) attn_fwd_kernel(AttnArgs a) {
    // phase-1 thread tile: TM1 keys x TN1 queries; phase-3: TM3 rows x 4 columns
    constexpr int TX = 16, TY = THREADS / TX, WX = TX / 8;
    constexpr int TN1 = BM / TX, TM1 = KC / TY, TM3 = BM / TY;
    static_assert(TN1 == 2 || TN1 == 4, "phase-1 query pairs");
    extern __shared__ __align__(16) float sm[];
    const int T = a.T, SLD = T + 4;
    float *Qt = sm;                    // [HD][BM]  Q^T of this row block
    float *Ss = Qt + HD * BM;          // [BM][T + 4] score rows, then probability rows
    float *Kc = Ss + BM * SLD;         // [2][KC][KLD] K chunks, later [2][KC][HD] V chunks

    __shared__ unsigned long long vflags[2];  // V suffix (keys >= kend): [0] any non-finite, [1] all sign bits
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // heaviest row blocks first (causal: block qb folds qb + 1 chunks), (batch, head) fastest
    const int nqb = T / BM;
    const int64_t bh = blockIdx.x % a.nbatch, b0 = bh / a.batch1, b1 = bh % a.batch1;
    const int q0 = (nqb - 1 - (int)(blockIdx.x / a.nbatch)) * BM;
    const float *Q = a.Q + b0 * a.s0 + b1 * a.s1;
    const float *K = a.K + b0 * a.s0 + b1 * a.s1;
    const float *V = a.V + b0 * a.s0 + b1 * a.s1;
    const int nchunks = T / KC;
    // R31: with the scores scratch (S not stored) and a causal mask, the rows of this block
    // read keys < q0 + BM only: phase 1 computes the chunks that hold them, phase 3 folds
    // them and applies the remaining fma(+0, V[j][n], acc) terms in closed form
    const int nch = a.skip ? min(nchunks, (q0 + BM + KC - 1) / KC) : nchunks;
    const int kend = nch * KC;
    if (tid == 0) {
        vflags[0] = 0ull;
        vflags[1] = ~0ull;
    }
    __syncthreads();
    if (kend < T) {
        // per column n: bit n of [0] = some V[j][n], j >= kend, non-finite; of [1] = every
        // such V[j][n] has its sign bit set (integer logic, loads independent of the rest)
        const int cq = tid % (HD / 4);
        unsigned nf = 0u, neg = 0xFu;
        for (int j = kend + tid / (HD / 4); j < T; j += THREADS / (HD / 4)) {
            const uint4 u = __ldg(reinterpret_cast<const uint4 *>(V + (int64_t)j * a.ld + cq * 4));
            const unsigned w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                nf |= (((w[c] & 0x7F800000u) == 0x7F800000u) ? 1u : 0u) << c;
                neg &= ((w[c] >> 31) << c) | ~(1u << c);
            }
        }
        atomicOr(&vflags[0], (unsigned long long)nf << (4 * cq));
        atomicAnd(&vflags[1], ~(((unsigned long long)(~neg & 0xFu)) << (4 * cq)));
    }

    // K chunk 0 in flight while Q^T is staged
    load_chunk<KLD, KC, THREADS>(Kc, K, a.ld, tid);
    cp_commit();
#pragma unroll
    for (int q = 0; q < BM * HD / 4 / THREADS; ++q) {
        const int c = tid + q * THREADS;
        const int r = c % BM, kq = (c / BM) * 4;  // a warp: 32 consecutive rows, one k quad
        const float4 v = __ldg(reinterpret_cast<const float4 *>(Q + (int64_t)(q0 + r) * a.ld + kq));
        Qt[(kq + 0) * BM + r] = v.x;
        Qt[(kq + 1) * BM + r] = v.y;
        Qt[(kq + 2) * BM + r] = v.z;
        Qt[(kq + 3) * BM + r] = v.w;
    }

    // ---------------- phase 1: S^T chunk [KC keys x BM queries] per iteration
    // thread: TM1 keys (ty + TY r) x TN1 queries (tx * TN1 + c); warps 8 (n) x 4 (m) lanes
    {
        const int tx = (warp % WX) * 8 + (lane & 7);
        const int ty = (warp / WX) * 4 + (lane >> 3);
        for (int ch = 0; ch < nch; ++ch) {
            if (ch + 1 < nch)
                load_chunk<KLD, KC, THREADS>(Kc + ((ch + 1) & 1) * KC * KLD, K + (int64_t)(ch + 1) * KC * a.ld, a.ld,
                                             tid);
            cp_commit();
            cp_wait<1>();
            __syncthreads();
            const float *Kb = Kc + (ch & 1) * KC * KLD;
            float2 acc[TM1][TN1 / 2];
#pragma unroll
            for (int r = 0; r < TM1; ++r)
#pragma unroll
                for (int h = 0; h < TN1 / 2; ++h) acc[r][h] = make_float2(0.f, 0.f);  // +0 (R2)
#pragma unroll
            for (int kg = 0; kg < HD; kg += 4) {
                float ak[TM1][4];
#pragma unroll
                for (int r = 0; r < TM1; ++r) {
                    const float4 v = *reinterpret_cast<const float4 *>(Kb + (ty + TY * r) * KLD + kg);
                    ak[r][0] = v.x; ak[r][1] = v.y; ak[r][2] = v.z; ak[r][3] = v.w;
                }
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    float2 bq[TN1 / 2];
                    if constexpr (TN1 == 4) {
                        const float4 q4 = *reinterpret_cast<const float4 *>(Qt + (kg + kk) * BM + tx * 4);
                        bq[0] = make_float2(q4.x, q4.y);
                        bq[1] = make_float2(q4.z, q4.w);
                    } else {
                        bq[0] = *reinterpret_cast<const float2 *>(Qt + (kg + kk) * BM + tx * 2);
                    }
#pragma unroll
                    for (int r = 0; r < TM1; ++r) {
                        const float2 av = make_float2(ak[r][kk], ak[r][kk]);
#pragma unroll
                        for (int h = 0; h < TN1 / 2; ++h)  // fma(K[j,k], Q[i,k], acc): commutative
                            acc[r][h] = __ffma2_rn(av, bq[h], acc[r][h]);
                    }
                }
            }
            // epilogue (R3, R10): S = canon(fmul(acc, scale)) into the query-major rows
#pragma unroll
            for (int r = 0; r < TM1; ++r) {
                const int j = ch * KC + ty + TY * r;
#pragma unroll
                for (int h = 0; h < TN1 / 2; ++h) {
                    Ss[(tx * TN1 + 2 * h) * SLD + j] = canon(__fmul_rn(acc[r][h].x, a.scale));
                    Ss[(tx * TN1 + 2 * h + 1) * SLD + j] = canon(__fmul_rn(acc[r][h].y, a.scale));
                }
            }
            __syncthreads();  // chunk buffer free for the prefetch two iterations on
        }
    }

    // V chunk 0 in flight during the softmax (the K buffers are free)
    load_chunk<HD, KC, THREADS>(Kc, V, a.ld, tid);
    cp_commit();

    // write the score rows (coalesced float4)
    if (a.S) {
        float *Sg = a.S + b0 * a.sp0 + b1 * a.sp1 + (int64_t)q0 * T;
        for (int c = tid; c < BM * T / 4; c += THREADS) {
            const int r = c / (T / 4), j4 = (c % (T / 4)) * 4;
            *reinterpret_cast<float4 *>(Sg + (int64_t)r * T + j4) = *reinterpret_cast<const float4 *>(Ss + r * SLD + j4);
        }
    }

    __syncthreads();  // the score rows are read by the copy above before phase 2 overwrites them

    // ---------------- phase 2: causal softmax, warp per row (softmax_warp's order)
    for (int r = warp; r < BM; r += THREADS / 32) {
        float *row = Ss + r * SLD;
        const int L = a.causal ? q0 + r + 1 : T;
        float m = __uint_as_float(0xFF800000u);
        for (int b = 0; b < L; b += 128) {
            const int i = b + 4 * lane;
            const float4 v = *reinterpret_cast<const float4 *>(row + i);  // i + 3 < T always
            if (i < L) m = fmaxf(m, v.x);
            if (i + 1 < L) m = fmaxf(m, v.y);
            if (i + 2 < L) m = fmaxf(m, v.z);
            if (i + 3 < L) m = fmaxf(m, v.w);
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL, m, off));
        m = (m == 0.0f) ? 0.0f : m;
        float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
        for (int b = 0; b < L; b += 128) {
            const int i = b + 4 * lane;
            const float4 v = *reinterpret_cast<const float4 *>(row + i);
            if (i < L) p0 = __fadd_rn(p0, exp_rn(__fsub_rn(v.x, m)));
            if (i + 1 < L) p1 = __fadd_rn(p1, exp_rn(__fsub_rn(v.y, m)));
            if (i + 2 < L) p2 = __fadd_rn(p2, exp_rn(__fsub_rn(v.z, m)));
            if (i + 3 < L) p3 = __fadd_rn(p3, exp_rn(__fsub_rn(v.w, m)));
        }
        const float rinv = __fdiv_rn(1.0f, tree128(p0, p1, p2, p3));
        float *Pg = a.P ? a.P + b0 * a.sp0 + b1 * a.sp1 + (int64_t)(q0 + r) * T : nullptr;
        if (Pg)
            for (int i = kend + 4 * lane; i < T; i += 128) *reinterpret_cast<float4 *>(Pg + i) = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int b = 0; b < kend; b += 128) {
            const int i = b + 4 * lane;
            const float4 v = *reinterpret_cast<const float4 *>(row + i);
            float o[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) o[c] = (i + c < L) ? canon(__fmul_rn(exp_rn(__fsub_rn(o[c], m)), rinv)) : 0.0f;
            const float4 y = make_float4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<float4 *>(row + i) = y;
            if (Pg) *reinterpret_cast<float4 *>(Pg + i) = y;
        }
    }

    // ---------------- phase 3: O = P V, keys ascending over all T (thread: TM3 rows x 4 cols)
    {
        const int tx = (warp % WX) * 8 + (lane & 7);   // cols tx * 4 .. + 3
        const int ty = (warp / WX) * 4 + (lane >> 3);  // rows ty + TY r
        float2 acc[TM3][2];
#pragma unroll
        for (int r = 0; r < TM3; ++r) acc[r][0] = acc[r][1] = make_float2(0.f, 0.f);
        for (int ch = 0; ch < nch; ++ch) {
            if (ch + 1 < nch)
                load_chunk<HD, KC, THREADS>(Kc + ((ch + 1) & 1) * KC * KLD, V + (int64_t)(ch + 1) * KC * a.ld, a.ld,
                                            tid);
            cp_commit();
            cp_wait<1>();
            __syncthreads();  // V chunk landed; (first iteration) every probability row written
            const float *Vb = Kc + (ch & 1) * KC * KLD;
            const float *Pr = Ss + ch * KC;
#pragma unroll 4
            for (int kg = 0; kg < KC; kg += 4) {
                float ap[TM3][4];
#pragma unroll
                for (int r = 0; r < TM3; ++r) {
                    const float4 v = *reinterpret_cast<const float4 *>(Pr + (ty + TY * r) * SLD + kg);
                    ap[r][0] = v.x; ap[r][1] = v.y; ap[r][2] = v.z; ap[r][3] = v.w;
                }
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const float4 bv = *reinterpret_cast<const float4 *>(Vb + (kg + kk) * HD + tx * 4);
                    const float2 b01 = make_float2(bv.x, bv.y), b23 = make_float2(bv.z, bv.w);
#pragma unroll
                    for (int r = 0; r < TM3; ++r) {
                        const float2 av = make_float2(ap[r][kk], ap[r][kk]);
                        acc[r][0] = __ffma2_rn(av, b01, acc[r][0]);
                        acc[r][1] = __ffma2_rn(av, b23, acc[r][1]);
                    }
                }
            }
            __syncthreads();
        }
        if (kend < T) {
            // the skipped terms fma(+0, V[j][n], acc), j >= kend (R31): a non-finite V gives
            // NaN; otherwise only acc = -0 can change, to +0 unless every V[j][n] is negative
            const unsigned long long nfm = vflags[0], negm = vflags[1];
#pragma unroll
            for (int r = 0; r < TM3; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int n = tx * 4 + c;
                    float &x = (c & 1) ? acc[r][c >> 1].y : acc[r][c >> 1].x;
                    if ((nfm >> n) & 1ull) x = __uint_as_float(0x7FC00000u);
                    else if (__float_as_uint(x) == 0x80000000u && !((negm >> n) & 1ull)) x = 0.0f;
                }
        }
        float *Og = a.O + b0 * a.so0 + b1 * a.so1;
#pragma unroll
        for (int r = 0; r < TM3; ++r) {
            const int i = q0 + ty + TY * r;
            *reinterpret_cast<float4 *>(Og + (int64_t)i * a.ldo + tx * 4) =
                make_float4(canon(acc[r][0].x), canon(acc[r][0].y), canon(acc[r][1].x), canon(acc[r][1].y));
        }
    }
}

// ---------------------------------------------------------------- scores + softmax (P only)
// The attention operator's first half for the GPT-2 training step (R29: S is operator
// scratch, P is kept for the PV R-GEMM and the backward): one CTA of PS_THREADS threads owns
// PS_BM query rows of one (batch, head); S is computed straight into shared memory with a
// GEMM-sized register tile (4 queries x 8 keys per thread, d ascending from +0, then
// canon(fmul(acc, scale))), then each warp runs softmax_warp's sequence on its rows and
// writes P.  S never reaches HBM; bits equal repops_gemm(SCALE) -> repops_softmax.
//
// MODE 1 (the backward twin, repops_attention_dscores): the same phase 1 computes
// dP = canon(fold_d fma(dO[i,d], V[j,d], +0)) for every key j (no epilogue; the softmax
// backward's row fold reads every column), and phase 2 is softmax_bwd_warp's sequence:
// c = CDOT(P row, dP row) (128 slots of fma from +0, then TREE128), dS = canon(fmul(fmul(P,
// fsub(dP, c)), scale)).  dP never reaches HBM; bits equal repops_gemm -> repops_softmax_backward.
constexpr int PS_THREADS = 256, PS_DS = 8, PS_KLD = PS_DS + 4, PS_NST = 3;
// Row block per head dim: 64 -> 32 query rows (8 q-groups x 4 key groups of lanes per warp,
// 256-key blocks); 128 (Llama) -> 16 rows (4 x 8 lanes per warp, 512-key blocks) so the score
// rows of T = 2048 fit beside the K ring (16 x 2052 x 4 B + 3 x 512 x 12 x 4 B + Q^T = 211 KB).
template <int PHD> struct ProbGeom {
    static constexpr int BM = PHD == 64 ? 32 : 16;
    static constexpr int NQG = BM / 4;                 // query groups (lanes along q)
    static constexpr int NKG = 32 / NQG;               // key groups (lanes along keys)
    static constexpr int KW = NKG * 8;                 // keys per warp
    static constexpr int KB = KW * (PS_THREADS / 32);  // keys per block
};

struct ProbArgs {
    const float *A, *B;          // rows of A (Q or dO) and B (K or V), head dim PHD
    int64_t lda, sa0, sa1, ldb, sb0, sb1;
    const float *Pin;            // MODE 1: P blocks (row stride T)
    int64_t spi0, spi1;
    float *out;                  // MODE 0: P, MODE 1: dS (row stride T)
    int64_t so0, so1;
    int64_t batch1, nbatch;
    int T, causal;
    float scale;
};

template <int MODE, int PHD>
__global__ void __launch_bounds__(PS_THREADS, PHD == 64 ? 2 : 1) attn_probs_kernel(ProbArgs a) {
    using G = ProbGeom<PHD>;
    constexpr int PS_BM = G::BM, PS_KB = G::KB, NQG = G::NQG, NKG = G::NKG, KW = G::KW;
    extern __shared__ __align__(16) float sm[];
    const int T = a.T, SLD = T + 4;
    float *Qt = sm;                       // [PHD][PS_BM]
    float *Ss = Qt + PHD * PS_BM;         // [PS_BM][T + 4]
    float *Ks = Ss + PS_BM * SLD;         // [PS_NST][PS_KB][PS_KLD] ring of d-slices of a key block
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nqb = T / PS_BM;
    const int64_t bh = blockIdx.x % a.nbatch, b0 = bh / a.batch1, b1 = bh % a.batch1;
    const int q0 = (nqb - 1 - (int)(blockIdx.x / a.nbatch)) * PS_BM;
    const float *Q = a.A + b0 * a.sa0 + b1 * a.sa1;
    const float *K = a.B + b0 * a.sb0 + b1 * a.sb1;
    // causal: the rows read keys < q0 + PS_BM only (R31: the other scores are never read)
    const int kneed = (MODE == 0 && a.causal) ? min(T, q0 + PS_BM) : T;

#pragma unroll
    for (int q = 0; q < PS_BM * PHD / 4 / PS_THREADS; ++q) {
        const int c = tid + q * PS_THREADS;
        const int r = c % PS_BM, kq = (c / PS_BM) * 4;
        const float4 v = __ldg(reinterpret_cast<const float4 *>(Q + (int64_t)(q0 + r) * a.lda + kq));
        Qt[(kq + 0) * PS_BM + r] = v.x;
        Qt[(kq + 1) * PS_BM + r] = v.y;
        Qt[(kq + 2) * PS_BM + r] = v.z;
        Qt[(kq + 3) * PS_BM + r] = v.w;
    }

    // thread tile: queries 4 qg .. 4 qg + 3, keys kb + KW warp + kg + NKG j (j < 8)
    const int qg = lane % NQG, kg = lane / NQG;
    for (int kb = 0; kb < kneed; kb += PS_KB) {
        const int nk = min(PS_KB, kneed - kb);           // keys of this block that are read
        // staged rows: whole warps' key ranges, never past the T keys of the head (a warp's
        // keys >= T compute on stale shared memory and are not stored)
        const int nrows = min((nk + KW - 1) / KW * KW, T - kb);
        const bool active = KW * warp < nk;              // warp-uniform
        auto stage = [&](int buf, int ds) {              // K[kb .. kb + nrows)[ds .. ds + 8)
            float *dst = Ks + buf * PS_KB * PS_KLD;
            for (int c = tid; c < nrows * (PS_DS / 4); c += PS_THREADS) {
                const int r = c / (PS_DS / 4), k4 = (c % (PS_DS / 4)) * 4;
                cp16(dst + r * PS_KLD + k4, K + (int64_t)(kb + r) * a.ldb + ds + k4);
            }
        };
        float2 acc[8][2];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = make_float2(0.f, 0.f);  // +0 (R2)
#pragma unroll
        for (int s = 0; s < PS_NST - 1; ++s) {
            stage(s, s * PS_DS);
            cp_commit();
        }
        for (int s = 0; s < PHD / PS_DS; ++s) {
            if (s + PS_NST - 1 < PHD / PS_DS) stage((s + PS_NST - 1) % PS_NST, (s + PS_NST - 1) * PS_DS);
            cp_commit();
            cp_wait<PS_NST - 1>();
            __syncthreads();
            if (active) {
                const float *Kb = Ks + (s % PS_NST) * PS_KB * PS_KLD + (KW * warp + kg) * PS_KLD;
#pragma unroll
                for (int d4 = 0; d4 < PS_DS; d4 += 4) {
                    float kv[8][4];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float4 v = *reinterpret_cast<const float4 *>(Kb + NKG * j * PS_KLD + d4);
                        kv[j][0] = v.x; kv[j][1] = v.y; kv[j][2] = v.z; kv[j][3] = v.w;
                    }
#pragma unroll
                    for (int dd = 0; dd < 4; ++dd) {
                        const float4 q4 = *reinterpret_cast<const float4 *>(Qt + (s * PS_DS + d4 + dd) * PS_BM + 4 * qg);
                        const float2 qa = make_float2(q4.x, q4.y), qb = make_float2(q4.z, q4.w);
#pragma unroll
                        for (int j = 0; j < 8; ++j) {  // fma(K[j,d], Q[i,d], acc): commutative
                            const float2 kk = make_float2(kv[j][dd], kv[j][dd]);
                            acc[j][0] = __ffma2_rn(kk, qa, acc[j][0]);
                            acc[j][1] = __ffma2_rn(kk, qb, acc[j][1]);
                        }
                    }
                }
            }
            __syncthreads();  // slice buffer free for the stage PS_NST slices on
        }
        if (active) {  // epilogue (R3, R10): MODE 0 S = canon(fmul(acc, scale)), MODE 1 dP = canon(acc)
            auto epi = [&](float x) { return MODE == 0 ? canon(__fmul_rn(x, a.scale)) : canon(x); };
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int key = kb + KW * warp + kg + NKG * j;
                if (key >= T) continue;   // (T % KW != 0 with hd 128) -- a row holds T + 4 columns
                float *srow = Ss + 4 * qg * SLD + key;
                srow[0] = epi(acc[j][0].x);
                srow[SLD] = epi(acc[j][0].y);
                srow[2 * SLD] = epi(acc[j][1].x);
                srow[3 * SLD] = epi(acc[j][1].y);
            }
        }
    }
    __syncthreads();

    if constexpr (MODE == 1) {
        // softmax backward, warp per row (softmax_bwd_warp's order): c = CDOT(P, dP) over all T
        // columns, dS = canon(fmul(fmul(P, fsub(dP, c)), scale)); T <= 1024 is one CSUM tile
        for (int r = warp; r < PS_BM; r += PS_THREADS / 32) {
            const float *dp = Ss + r * SLD;
            const float *pr = a.Pin + b0 * a.spi0 + b1 * a.spi1 + (int64_t)(q0 + r) * T;
            float *dr = a.out + b0 * a.so0 + b1 * a.so1 + (int64_t)(q0 + r) * T;
            float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
            for (int b = 0; b < T; b += 128) {
                const int i = b + 4 * lane;
                if (i >= T) break;  // T % 4 == 0
                const float4 y = __ldg(reinterpret_cast<const float4 *>(pr + i));
                const float4 g = *reinterpret_cast<const float4 *>(dp + i);
                p0 = __fmaf_rn(y.x, g.x, p0);
                p1 = __fmaf_rn(y.y, g.y, p1);
                p2 = __fmaf_rn(y.z, g.z, p2);
                p3 = __fmaf_rn(y.w, g.w, p3);
            }
            const float c = tree128(p0, p1, p2, p3);
            for (int b = 0; b < T; b += 128) {
                const int i = b + 4 * lane;
                if (i >= T) break;
                const float4 y = __ldg(reinterpret_cast<const float4 *>(pr + i));
                const float4 g = *reinterpret_cast<const float4 *>(dp + i);
                float4 o;
                o.x = canon(__fmul_rn(__fmul_rn(y.x, __fsub_rn(g.x, c)), a.scale));
                o.y = canon(__fmul_rn(__fmul_rn(y.y, __fsub_rn(g.y, c)), a.scale));
                o.z = canon(__fmul_rn(__fmul_rn(y.z, __fsub_rn(g.z, c)), a.scale));
                o.w = canon(__fmul_rn(__fmul_rn(y.w, __fsub_rn(g.w, c)), a.scale));
                *reinterpret_cast<float4 *>(dr + i) = o;
            }
        }
        return;
    }

    // softmax, warp per row (softmax_warp's order: R7), P rows written in full (+0 masked)
    for (int r = warp; r < PS_BM; r += PS_THREADS / 32) {
        float *row = Ss + r * SLD;
        const int L = a.causal ? q0 + r + 1 : T;
        float m = __uint_as_float(0xFF800000u);
        for (int b = 0; b < L; b += 128) {
            const int i = b + 4 * lane;
            const float4 v = *reinterpret_cast<const float4 *>(row + i);
            if (i < L) m = fmaxf(m, v.x);
            if (i + 1 < L) m = fmaxf(m, v.y);
            if (i + 2 < L) m = fmaxf(m, v.z);
            if (i + 3 < L) m = fmaxf(m, v.w);
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL, m, off));
        m = (m == 0.0f) ? 0.0f : m;
        float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
        for (int b = 0; b < L; b += 128) {  // e = exp(x - m) replaces x in place (computed once)
            const int i = b + 4 * lane;
            float4 v = *reinterpret_cast<const float4 *>(row + i);
            if (i < L) p0 = __fadd_rn(p0, v.x = exp_rn(__fsub_rn(v.x, m)));
            if (i + 1 < L) p1 = __fadd_rn(p1, v.y = exp_rn(__fsub_rn(v.y, m)));
            if (i + 2 < L) p2 = __fadd_rn(p2, v.z = exp_rn(__fsub_rn(v.z, m)));
            if (i + 3 < L) p3 = __fadd_rn(p3, v.w = exp_rn(__fsub_rn(v.w, m)));
            if (i < L) *reinterpret_cast<float4 *>(row + i) = v;
        }
        const float rinv = __fdiv_rn(1.0f, tree128(p0, p1, p2, p3));
        float *Pg = a.out + b0 * a.so0 + b1 * a.so1 + (int64_t)(q0 + r) * T;
        for (int b = 0; b < T; b += 128) {
            const int i = b + 4 * lane;
            if (i >= T) break;  // T % 4 == 0: i < T covers the whole float4
            float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
            if (i < L) {
                const float4 v = *reinterpret_cast<const float4 *>(row + i);
                float o[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int c = 0; c < 4; ++c) o[c] = (i + c < L) ? canon(__fmul_rn(o[c], rinv)) : 0.0f;
                y = make_float4(o[0], o[1], o[2], o[3]);
            }
            *reinterpret_cast<float4 *>(Pg + i) = y;  // kept in L2 for the PV R-GEMM
        }
    }
}

}  // namespace

// (BM, KC, THREADS): 0 = (64, 128, 256), 1 = (32, 64, 128), 2 = (64, 64, 256), 3 = (32, 64, 256);
// REPOPS_ATTN_VARIANT overrides
static int attn_variant() {
    const char *e = getenv("REPOPS_ATTN_VARIANT");  // read per launch: tests switch it in-process
    return e ? atoi(e) : RO_ATTN_VARIANT_DEFAULT;
}

template <int BM, int KC>
static size_t smem_bytes(int64_t T) {
    return (size_t)(HD * BM + BM * (T + 4) + 2 * KC * KLD) * sizeof(float);
}

size_t attention_fwd_smem_bytes(int64_t T) {
    switch (attn_variant()) {
        case 0: return smem_bytes<64, 128>(T);
        case 2: return smem_bytes<64, 64>(T);
        default: return smem_bytes<32, 64>(T);
    }
}

bool attention_fwd_supported(int64_t T, int64_t hd) {
    return hd == HD && T > 0 && T % 128 == 0 && smem_bytes<64, 128>(T) <= 227 * 1024;
}

template <int BM, int KC, int THREADS>
static cudaError_t launch_variant(const AttnArgs &a, int64_t batch, cudaStream_t s) {
    const size_t smem = smem_bytes<BM, KC>(a.T);
    static size_t attr = 0;
    if (smem > attr) {
        cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<BM, KC, THREADS>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = smem;
    }
    AttnArgs b = a;
    b.nbatch = batch;
    attn_fwd_kernel<BM, KC, THREADS><<<(unsigned)(a.T / BM * batch), THREADS, smem, s>>>(b);
    return cudaGetLastError();
}

cudaError_t launch_attention_fwd(int64_t T, const float *Q, const float *K, const float *V, int64_t ld, int64_t s0,
                                 int64_t s1, float scale, int causal, float *S, float *P, int64_t sp0, int64_t sp1,
                                 float *O, int64_t ldo, int64_t so0, int64_t so1, int64_t batch0, int64_t batch1,
                                 cudaStream_t s) {
    if (batch0 * batch1 == 0 || T == 0) return cudaSuccess;
    // the skip needs the scores to be scratch: a caller that stores S gets every column
    AttnArgs a{Q, K, V, ld, s0, s1, S, P, sp0, sp1, O, ldo, so0, so1, batch1, 0, (int)T, causal, (causal && !S) ? 1 : 0,
               scale};
    switch (attn_variant()) {
        case 0: return launch_variant<64, 128, 256>(a, batch0 * batch1, s);
        case 2: return launch_variant<64, 64, 256>(a, batch0 * batch1, s);
        case 3: return launch_variant<32, 64, 256>(a, batch0 * batch1, s);
        default: return launch_variant<32, 64, 128>(a, batch0 * batch1, s);
    }
}


template <int PHD>
static size_t probs_smem_bytes_t(int64_t T) {
    using G = ProbGeom<PHD>;
    return (size_t)(PHD * G::BM + G::BM * (T + 4) + PS_NST * G::KB * PS_KLD) * sizeof(float);
}

static size_t probs_smem_bytes(int64_t T, int64_t hd) {
    return hd == 64 ? probs_smem_bytes_t<64>(T) : probs_smem_bytes_t<128>(T);
}

bool attention_probs_supported(int64_t T, int64_t hd) {
    if (hd != 64 && hd != 128) return false;
    const int bm = hd == 64 ? ProbGeom<64>::BM : ProbGeom<128>::BM;
    return T > 0 && T % bm == 0 && T % 4 == 0 && probs_smem_bytes(T, hd) <= 227 * 1024;
}

bool attention_dscores_supported(int64_t T, int64_t hd) { return hd == 64 && attention_probs_supported(T, hd); }

template <int MODE, int PHD>
static cudaError_t launch_probs_mode(const ProbArgs &a, int64_t nb, cudaStream_t s) {
    const size_t smem = probs_smem_bytes_t<PHD>(a.T);
    static size_t attr = 0;
    if (smem > attr) {
        cudaError_t e = cudaFuncSetAttribute(attn_probs_kernel<MODE, PHD>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = smem;
    }
    attn_probs_kernel<MODE, PHD><<<(unsigned)(a.T / ProbGeom<PHD>::BM * nb), PS_THREADS, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_attention_probs(int64_t T, int64_t hd, const float *Q, const float *K, int64_t ld, int64_t s0,
                                   int64_t s1, int64_t ldk, int64_t sk0, int64_t sk1, float scale, int causal,
                                   float *P, int64_t sp0, int64_t sp1, int64_t batch0, int64_t batch1,
                                   cudaStream_t s) {
    if (batch0 * batch1 == 0 || T == 0) return cudaSuccess;
    ProbArgs a{Q, K, ld, s0, s1, ldk, sk0, sk1, nullptr, 0, 0, P, sp0, sp1, batch1, batch0 * batch1, (int)T, causal,
               scale};
    return hd == 64 ? launch_probs_mode<0, 64>(a, batch0 * batch1, s) : launch_probs_mode<0, 128>(a, batch0 * batch1, s);
}

cudaError_t launch_attention_dscores(int64_t T, const float *dO, int64_t ldo, int64_t so0, int64_t so1,
                                     const float *V, int64_t ldv, int64_t sv0, int64_t sv1, const float *P,
                                     int64_t sp0, int64_t sp1, float scale, float *dS, int64_t sd0, int64_t sd1,
                                     int64_t batch0, int64_t batch1, cudaStream_t s) {
    if (batch0 * batch1 == 0 || T == 0) return cudaSuccess;
    ProbArgs a{dO, V, ldo, so0, so1, ldv, sv0, sv1, P, sp0, sp1, dS, sd0, sd1, batch1, batch0 * batch1, (int)T, 0,
               scale};
    return launch_probs_mode<1, 64>(a, batch0 * batch1, s);
}
