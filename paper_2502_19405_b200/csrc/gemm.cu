// gemm.cu -- R-GEMM on the FP32 CUDA cores of sm_100a.
//
// Canonical order: every output element is ONE thread-private accumulator that
// starts at +0 and takes fma(opA(i,k), opB(k,j), acc) for k = 0, 1, ..., K-1.
// Parallelism is only over (i, j) -- CTA tiles, warp tiles, thread micro-tiles
// ("parallelise the order-insensitive dimensions").  K is never
// split and never padded (zero padding is NOT bit-neutral: fma(0,0,-0) = +0
// and an fma can underflow to -0), so a ragged last K tile runs a short loop.
// Tensor cores are deliberately not used: their internal accumulation order is
// not IEEE-sequential (north_star).
//
// Kernel (v2).  CTA tile BM x BN (128 x 128, 256 threads, 8 x 8 outputs per
// thread; or 64 x 64, 128 threads, 8 x 4), BK = 16, STAGES-deep cp.async ring
// (global -> shared without registers; src-size zero-fill at the M/N/K edges).
// Operand tiles keep their global orientation in shared memory:
//   "mn-contiguous" (A^T stored K x M, or B stored K x N): [BK][BM] rows, the
//      thread reads its 4 consecutive rows/cols at one k with one LDS.128;
//   "k-contiguous"  (A stored M x K, or B^T stored N x K): [BM][BK+4] rows, the
//      thread owns rows ty + TY*i and reads KG consecutive k of each row with
//      one LDS.64/.128 (row stride 20 words -> the 4 / 8 rows a warp touches
//      fall in disjoint bank groups).
// Warps are 8 (n) x 4 (m) lanes so one LDS instruction touches <= 128 bytes.
// CTAs are rasterised in groups of GROUP_M row tiles so the A and B panels of
// concurrently running CTAs are shared through L2.
#include "common.cuh"
#include "gemm.cuh"

namespace {

using ro::canon;

constexpr int GROUP_M = 16;  // row tiles per rasterisation group

RO_DEV void cp_async16(float *dst, const float *src, int bytes) {
    unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
}
RO_DEV void cp_async4(float *dst, const float *src, int bytes) {
    unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
}
RO_DEV void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
RO_DEV void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Copy an R x L tile (contiguous along L in global memory, leading dimension
// ld) into shared memory with row stride SLD.  Only rows < rvalid and columns
// < lvalid are read; the rest of each 16-byte chunk is zero filled.
template <int R, int L, int SLD, int THREADS, bool VEC>
RO_DEV void tile_async(float *dst, const float *__restrict__ src, int64_t ld, int64_t rvalid, int64_t lvalid,
                       int tid) {
    constexpr int CPR = L / 4;
    constexpr int TOTAL = R * CPR;
    static_assert(TOTAL % THREADS == 0, "tile/threads mismatch");
#pragma unroll
    for (int q = 0; q < TOTAL / THREADS; ++q) {
        const int c = tid + q * THREADS;
        const int r = c / CPR;
        const int l = (c % CPR) * 4;
        float *d = dst + r * SLD + l;
        const float *s = src + (int64_t)r * ld + l;
        if (VEC) {
            int64_t rem = lvalid - l;
            int bytes = (r < rvalid && rem > 0) ? (rem >= 4 ? 16 : (int)rem * 4) : 0;
            cp_async16(d, bytes ? s : src, bytes);
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                int bytes = (r < rvalid && l + e < lvalid) ? 4 : 0;
                cp_async4(d + e, bytes ? s + e : src, bytes);
            }
        }
    }
}

template <int BM, int BN, int BK, int TM, int TN, bool TA, bool TB, int KGO = 0>
struct Cfg {
    static constexpr int TX = BN / TN;          // threads along n
    static constexpr int TY = BM / TM;          // threads along m
    static constexpr int THREADS = TX * TY;
    static constexpr int WX = TX / 8;           // warps along n (8 lanes each)
    static constexpr int SKP = BK + 4;          // k-contiguous row stride (words)
    // shared-memory stage layout
    static constexpr int A_WORDS = TA ? BK * BM : BM * SKP;
    static constexpr int B_WORDS = TB ? BN * SKP : BK * BN;
    static constexpr int STAGE_WORDS = A_WORDS + B_WORDS;
    // k-group width for k-contiguous operands (LDS.64 when both are k-contiguous)
    static constexpr int KG = KGO ? KGO : ((!TA && TB) ? 2 : 4);
};

template <int BM, int BN, int BK, int TM, int TN, int STAGES, int MINB, int KGO, bool TA, bool TB, bool VEC>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), MINB) gemm_kernel(GemmParams p) {
    using CF = Cfg<BM, BN, BK, TM, TN, TA, TB, KGO>;
    constexpr int THREADS = CF::THREADS;
    constexpr int TX = CF::TX, TY = CF::TY, SKP = CF::SKP, KG = CF::KG;
    extern __shared__ __align__(16) float smem[];

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int tx = (warp % CF::WX) * 8 + (lane & 7);
    const int ty = (warp / CF::WX) * 4 + (lane >> 3);

    // grouped rasterisation of the (m, n) tile grid
    const int64_t tiles_m = (p.M + BM - 1) / BM, tiles_n = (p.N + BN - 1) / BN;
    const int64_t t = blockIdx.x;
    const int64_t per_group = (int64_t)GROUP_M * tiles_n;
    const int64_t g = t / per_group;
    const int64_t first_m = g * GROUP_M;
    const int64_t gsz = min((int64_t)GROUP_M, tiles_m - first_m);
    const int64_t tm_ = first_m + (t % per_group) % gsz;
    const int64_t tn_ = (t % per_group) / gsz;
    const int64_t m0 = tm_ * BM, n0 = tn_ * BN;

    const int64_t b0 = blockIdx.y / p.batch1, b1 = blockIdx.y % p.batch1;
    const float *__restrict__ A = p.A + b0 * p.sA0 + b1 * p.sA1;
    const float *__restrict__ B = p.B + b0 * p.sB0 + b1 * p.sB1;
    float *__restrict__ Cp = p.C + b0 * p.sC0 + b1 * p.sC1;
    const int64_t M = p.M, N = p.N, K = p.K;

    auto load_stage = [&](int slot, int64_t kt) {
        float *As = smem + slot * CF::STAGE_WORDS;
        float *Bs = As + CF::A_WORDS;
        const int64_t k0 = kt * BK;
        if (TA)  // A stored K x M: tile rows = k, contiguous m
            tile_async<BK, BM, BM, THREADS, VEC>(As, A + k0 * p.lda + m0, p.lda, K - k0, M - m0, tid);
        else     // A stored M x K: tile rows = m, contiguous k
            tile_async<BM, BK, SKP, THREADS, VEC>(As, A + m0 * p.lda + k0, p.lda, M - m0, K - k0, tid);
        if (TB)  // B stored N x K
            tile_async<BN, BK, SKP, THREADS, VEC>(Bs, B + n0 * p.ldb + k0, p.ldb, N - n0, K - k0, tid);
        else     // B stored K x N
            tile_async<BK, BN, BN, THREADS, VEC>(Bs, B + k0 * p.ldb + n0, p.ldb, K - k0, N - n0, tid);
    };

    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;  // +0 (R2)

    const int64_t ktiles = (K + BK - 1) / BK;
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ktiles) load_stage(s, s);
        cp_commit();
    }

    // fragment address helpers
    // mn-contiguous A: rows (i/4)*(BM/(TM/4)) + ty*4 + i%4 ; k-contiguous A: rows ty + TY*i
    // mn-contiguous B: cols (j/4)*(BN/(TN/4)) + tx*4 + j%4 ; k-contiguous B: cols tx + TX*j
    for (int64_t kt = 0; kt < ktiles; ++kt) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        {
            const int64_t nk = kt + STAGES - 1;
            if (nk < ktiles) load_stage((int)(nk % STAGES), nk);
            cp_commit();
        }
        const float *As = smem + (int)(kt % STAGES) * CF::STAGE_WORDS;
        const float *Bs = As + CF::A_WORDS;
        const int kmax = (int)min((int64_t)BK, K - kt * BK);
        if (kmax == BK) {
#pragma unroll
            for (int kg = 0; kg < BK; kg += KG) {
                float ak[TA ? 1 : TM][KG], bk[TB ? TN : 1][KG];
                if (!TA) {
#pragma unroll
                    for (int i = 0; i < TM; ++i) {
                        const float *src = As + (ty + TY * i) * SKP + kg;
                        if (KG == 4) {
                            float4 v = *reinterpret_cast<const float4 *>(src);
                            ak[i][0] = v.x; ak[i][KG > 1 ? 1 : 0] = v.y;
                            ak[i][KG > 2 ? 2 : 0] = v.z; ak[i][KG > 3 ? 3 : 0] = v.w;
                        } else {
                            float2 v = *reinterpret_cast<const float2 *>(src);
                            ak[i][0] = v.x; ak[i][KG > 1 ? 1 : 0] = v.y;
                        }
                    }
                }
                if (TB) {
#pragma unroll
                    for (int j = 0; j < TN; ++j) {
                        const float *src = Bs + (tx + TX * j) * SKP + kg;
                        if (KG == 4) {
                            float4 v = *reinterpret_cast<const float4 *>(src);
                            bk[j][0] = v.x; bk[j][KG > 1 ? 1 : 0] = v.y;
                            bk[j][KG > 2 ? 2 : 0] = v.z; bk[j][KG > 3 ? 3 : 0] = v.w;
                        } else {
                            float2 v = *reinterpret_cast<const float2 *>(src);
                            bk[j][0] = v.x; bk[j][KG > 1 ? 1 : 0] = v.y;
                        }
                    }
                }
#pragma unroll
                for (int kk = 0; kk < KG; ++kk) {
                    float a[TM], b[TN];
                    if (TA) {
#pragma unroll
                        for (int h = 0; h < TM / 4; ++h) {
                            float4 v = *reinterpret_cast<const float4 *>(As + (kg + kk) * BM + h * (BM / (TM / 4)) + ty * 4);
                            a[h * 4] = v.x; a[h * 4 + 1] = v.y; a[h * 4 + 2] = v.z; a[h * 4 + 3] = v.w;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < TM; ++i) a[i] = ak[i][kk];
                    }
                    if (!TB) {
#pragma unroll
                        for (int h = 0; h < TN / 4; ++h) {
                            float4 v = *reinterpret_cast<const float4 *>(Bs + (kg + kk) * BN + h * (BN / (TN / 4)) + tx * 4);
                            b[h * 4] = v.x; b[h * 4 + 1] = v.y; b[h * 4 + 2] = v.z; b[h * 4 + 3] = v.w;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < TN; ++j) b[j] = bk[j][kk];
                    }
#pragma unroll
                    for (int i = 0; i < TM; ++i)
#pragma unroll
                        for (int j = 0; j < TN; ++j) acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
                }
            }
        } else {
            // ragged last K tile: the real k only, ascending (no zero padding)
            for (int k = 0; k < kmax; ++k) {
                float a[TM], b[TN];
#pragma unroll
                for (int i = 0; i < TM; ++i)
                    a[i] = TA ? As[k * BM + (i / 4) * (BM / (TM / 4)) + ty * 4 + (i % 4)] : As[(ty + TY * i) * SKP + k];
#pragma unroll
                for (int j = 0; j < TN; ++j)
                    b[j] = TB ? Bs[(tx + TX * j) * SKP + k] : Bs[k * BN + (j / 4) * (BN / (TN / 4)) + tx * 4 + (j % 4)];
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN; ++j) acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
            }
        }
    }
    cp_wait<0>();

    // epilogue (R3): epi(acc) once, NaN canonicalised (R10)
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int64_t m = m0 + (TA ? (i / 4) * (BM / (TM / 4)) + ty * 4 + (i % 4) : ty + TY * i);
        if (m >= M) continue;
        float *crow = Cp + m * p.ldc;
        if (!TB) {
#pragma unroll
            for (int h = 0; h < TN / 4; ++h) {
                const int64_t n = n0 + h * (BN / (TN / 4)) + tx * 4;
                float v[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float x = acc[i][h * 4 + c];
                    if (p.epi == 1) x = (n + c < N) ? __fadd_rn(x, __ldg(p.bias + n + c)) : x;
                    else if (p.epi == 2) x = __fmul_rn(x, p.scale);
                    v[c] = canon(x);
                }
                if (p.vecC && n + 4 <= N) {
                    *reinterpret_cast<float4 *>(crow + n) = make_float4(v[0], v[1], v[2], v[3]);
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (n + c < N) crow[n + c] = v[c];
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int64_t n = n0 + tx + TX * j;
                if (n >= N) continue;
                float x = acc[i][j];
                if (p.epi == 1) x = __fadd_rn(x, __ldg(p.bias + n));
                else if (p.epi == 2) x = __fmul_rn(x, p.scale);
                crow[n] = canon(x);
            }
        }
    }
}

template <int BM, int BN, int BK, int TM, int TN, int STAGES, int MINB, int KGO, bool TA, bool TB, bool VEC>
cudaError_t launch_one(const GemmParams &p, cudaStream_t s) {
    using CF = Cfg<BM, BN, BK, TM, TN, TA, TB, KGO>;
    const size_t smem = (size_t)STAGES * CF::STAGE_WORDS * sizeof(float);
    auto kern = gemm_kernel<BM, BN, BK, TM, TN, STAGES, MINB, KGO, TA, TB, VEC>;
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int64_t tiles = ((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN);
    dim3 grid((unsigned)tiles, (unsigned)(p.batch0 * p.batch1));
    kern<<<grid, CF::THREADS, smem, s>>>(p);
    return cudaGetLastError();
}

template <int BM, int BN, int BK, int TM, int TN, int STAGES, int MINB, int KGO = 0>
cudaError_t launch_cfg(const GemmParams &p, cudaStream_t s) {
    const bool vec = p.vecA && p.vecB;
#define RO_GEMM_CASE(TA_, TB_)                                                                        \
    if ((bool)p.transA == TA_ && (bool)p.transB == TB_)                                               \
        return vec ? launch_one<BM, BN, BK, TM, TN, STAGES, MINB, KGO, TA_, TB_, true>(p, s)          \
                   : launch_one<BM, BN, BK, TM, TN, STAGES, MINB, KGO, TA_, TB_, false>(p, s);
    RO_GEMM_CASE(false, false)
    RO_GEMM_CASE(false, true)
    RO_GEMM_CASE(true, false)
    RO_GEMM_CASE(true, true)
#undef RO_GEMM_CASE
    return cudaErrorInvalidValue;
}

}  // namespace

// Tile configurations (all bits-neutral: only the M/N tiling differs).
//   0: 128 x 128, 8 x 8 per thread, 3 stages, 2 CTAs/SM   (large problems)
//   1:  64 x  64, 8 x 4 per thread, 3 stages              (small M*N)
//   2..5: tuning variants (selected by the benchmarks / tools/gemm_tune.py)
int gemm_num_cfgs() { return 6; }

cudaError_t gemm_launch(const GemmParams &p, cudaStream_t s, int force_cfg) {
    if (p.M == 0 || p.N == 0 || p.batch0 * p.batch1 == 0) return cudaSuccess;
    if (p.batch0 * p.batch1 > 65535) return cudaErrorInvalidValue;
    int cfg = force_cfg;
    if (cfg < 0) {
        int64_t tiles128 = ((p.M + 127) / 128) * ((p.N + 127) / 128) * p.batch0 * p.batch1;
        cfg = (tiles128 >= 2 * 148) ? 0 : 1;
    }
    switch (cfg) {
        case 0: return launch_cfg<128, 128, 16, 8, 8, 3, 2>(p, s);
        case 1: return launch_cfg<64, 64, 16, 8, 4, 3, 2>(p, s);
        case 2: return launch_cfg<128, 128, 16, 8, 8, 4, 1>(p, s);
        case 3: return launch_cfg<128, 256, 16, 8, 16, 3, 1>(p, s);
        case 4: return launch_cfg<256, 128, 16, 16, 8, 3, 1>(p, s);
        case 5: return launch_cfg<128, 128, 16, 8, 8, 3, 2, 2>(p, s);
        default: return cudaErrorInvalidValue;
    }
}
