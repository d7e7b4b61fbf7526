// gemm.cu -- R-GEMM on the FP32 CUDA cores of sm_100a.
//
// Canonical order: every output element is ONE thread-private accumulator that
// starts at +0 and takes fma(opA(i,k), opB(k,j), acc) for k = 0, 1, ..., K-1.
// Parallelism is only over (i, j) -- CTA tiles, warp tiles, thread micro-tiles
// ("parallelise the order-insensitive dimensions").  K is never
// split, never padded (zero padding is NOT bit-neutral: fma(0,0,-0) = +0 and
// an fma can underflow to -0), so the last K tile runs a short tail loop.
//
// Tensor cores are deliberately not used: their internal accumulation order
// is not IEEE-sequential (north_star).
//
// Kernel shape (v2): CTA tile BM x BN = 128 x 128, BK = 16, 256 threads, each
// thread an 8 x 8 register micro-tile (64 independent FMA chains).  Tiles of
// A and B are staged in shared memory k-major ([BK][BM] / [BK][BN]) through a
// register prefetch of the next k-tile, double buffered, one __syncthreads per
// k-tile.  A (row-major, not transposed) and B^T are transposed on the way
// into shared memory so the inner loop reads 4 consecutive rows/cols with one
// LDS.128.  A 64 x 64 configuration (128 threads, 4 x 8 per thread) serves
// small M*N; the choice is bits-neutral (only M/N tiling changes).
#include "common.cuh"
#include "gemm.cuh"

namespace {

using ro::canon;

template <int BM, int BN, int BK, int TM, int TN, bool TA, bool TB>
struct GemmCfg {
    static constexpr int THREADS = (BM / TM) * (BN / TN);
    static constexpr int TX = BN / TN;  // threads along N
    static constexpr int TY = BM / TM;  // threads along M
    static constexpr int APAD = TA ? 0 : 4;  // padding for transposed stores (bank spread)
    static constexpr int BPAD = TB ? 4 : 0;
    static constexpr int A_ELEMS = BM * BK / THREADS;  // per-thread loads of the A tile
    static constexpr int B_ELEMS = BN * BK / THREADS;
};

// Loads of one BK-tile of A into registers (ra) -- element mapping chosen so
// that global reads are coalesced along the contiguous dimension.
template <class Cfg, int BM, int BK, bool TA>
RO_DEV void load_a(float (&ra)[Cfg::A_ELEMS], const float *__restrict__ A, int64_t lda, int64_t M, int64_t K,
                   int64_t m0, int64_t k0, int tid, bool vec) {
    constexpr int E = Cfg::A_ELEMS;
    if (!TA) {
        // A[m][k], contiguous along k: consecutive threads take consecutive rows so
        // that the transposing shared-memory stores below are bank-conflict free
        int r = tid % BM;
        int kq = (tid / BM) * E;
        int64_t m = m0 + r;
        int64_t k = k0 + kq;
        const float *src = A + m * lda + k;
        if (vec && m < M && k + E <= K) {
#pragma unroll
            for (int q = 0; q < E; q += 4) {
                float4 v = __ldg(reinterpret_cast<const float4 *>(src + q));
                ra[q] = v.x; ra[q + 1] = v.y; ra[q + 2] = v.z; ra[q + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int q = 0; q < E; ++q) ra[q] = (m < M && k + q < K) ? __ldg(src + q) : 0.f;
        }
    } else {
        // A stored K x M: A[k][m], contiguous along m
        constexpr int PER_ROW = BM / E;
        int kr = tid / PER_ROW;
        int mq = (tid % PER_ROW) * E;
        int64_t k = k0 + kr;
        int64_t m = m0 + mq;
        const float *src = A + k * lda + m;
        if (vec && k < K && m + E <= M) {
#pragma unroll
            for (int q = 0; q < E; q += 4) {
                float4 v = __ldg(reinterpret_cast<const float4 *>(src + q));
                ra[q] = v.x; ra[q + 1] = v.y; ra[q + 2] = v.z; ra[q + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int q = 0; q < E; ++q) ra[q] = (k < K && m + q < M) ? __ldg(src + q) : 0.f;
        }
    }
}

template <class Cfg, int BM, int BK, bool TA>
RO_DEV void store_a(float *As, const float (&ra)[Cfg::A_ELEMS], int tid) {
    constexpr int E = Cfg::A_ELEMS;
    constexpr int LDA_S = BM + Cfg::APAD;
    if (!TA) {
        int r = tid % BM;
        int kq = (tid / BM) * E;
#pragma unroll
        for (int q = 0; q < E; ++q) As[(kq + q) * LDA_S + r] = ra[q];
    } else {
        constexpr int PER_ROW = BM / E;
        int kr = tid / PER_ROW;
        int mq = (tid % PER_ROW) * E;
#pragma unroll
        for (int q = 0; q < E; q += 4)
            *reinterpret_cast<float4 *>(&As[kr * LDA_S + mq + q]) = make_float4(ra[q], ra[q + 1], ra[q + 2], ra[q + 3]);
    }
}

template <class Cfg, int BN, int BK, bool TB>
RO_DEV void load_b(float (&rb)[Cfg::B_ELEMS], const float *__restrict__ B, int64_t ldb, int64_t N, int64_t K,
                   int64_t n0, int64_t k0, int tid, bool vec) {
    constexpr int E = Cfg::B_ELEMS;
    if (!TB) {
        // B[k][n], contiguous along n
        constexpr int PER_ROW = BN / E;
        int kr = tid / PER_ROW;
        int nq = (tid % PER_ROW) * E;
        int64_t k = k0 + kr;
        int64_t n = n0 + nq;
        const float *src = B + k * ldb + n;
        if (vec && k < K && n + E <= N) {
#pragma unroll
            for (int q = 0; q < E; q += 4) {
                float4 v = __ldg(reinterpret_cast<const float4 *>(src + q));
                rb[q] = v.x; rb[q + 1] = v.y; rb[q + 2] = v.z; rb[q + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int q = 0; q < E; ++q) rb[q] = (k < K && n + q < N) ? __ldg(src + q) : 0.f;
        }
    } else {
        // B stored N x K: B[n][k], contiguous along k
        int r = tid % BN;
        int kq = (tid / BN) * E;
        int64_t n = n0 + r;
        int64_t k = k0 + kq;
        const float *src = B + n * ldb + k;
        if (vec && n < N && k + E <= K) {
#pragma unroll
            for (int q = 0; q < E; q += 4) {
                float4 v = __ldg(reinterpret_cast<const float4 *>(src + q));
                rb[q] = v.x; rb[q + 1] = v.y; rb[q + 2] = v.z; rb[q + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int q = 0; q < E; ++q) rb[q] = (n < N && k + q < K) ? __ldg(src + q) : 0.f;
        }
    }
}

template <class Cfg, int BN, int BK, bool TB>
RO_DEV void store_b(float *Bs, const float (&rb)[Cfg::B_ELEMS], int tid) {
    constexpr int E = Cfg::B_ELEMS;
    constexpr int LDB_S = BN + Cfg::BPAD;
    if (!TB) {
        constexpr int PER_ROW = BN / E;
        int kr = tid / PER_ROW;
        int nq = (tid % PER_ROW) * E;
#pragma unroll
        for (int q = 0; q < E; q += 4)
            *reinterpret_cast<float4 *>(&Bs[kr * LDB_S + nq + q]) = make_float4(rb[q], rb[q + 1], rb[q + 2], rb[q + 3]);
    } else {
        int r = tid % BN;
        int kq = (tid / BN) * E;
#pragma unroll
        for (int q = 0; q < E; ++q) Bs[(kq + q) * LDB_S + r] = rb[q];
    }
}

// One k step of the micro-tile: rows ty*4.. and ty*4+BM/2.., cols tx*4.. and tx*4+BN/2..
template <int BM, int BN, int TM, int TN, int LDA_S, int LDB_S>
RO_DEV void mma_step(float (&acc)[TM][TN], const float *As, const float *Bs, int kk, int tx, int ty) {
    float a[TM], b[TN];
#pragma unroll
    for (int h = 0; h < TM / 4; ++h) {
        float4 v = *reinterpret_cast<const float4 *>(&As[kk * LDA_S + h * (BM / (TM / 4)) + ty * 4]);
        a[h * 4] = v.x; a[h * 4 + 1] = v.y; a[h * 4 + 2] = v.z; a[h * 4 + 3] = v.w;
    }
#pragma unroll
    for (int h = 0; h < TN / 4; ++h) {
        float4 v = *reinterpret_cast<const float4 *>(&Bs[kk * LDB_S + h * (BN / (TN / 4)) + tx * 4]);
        b[h * 4] = v.x; b[h * 4 + 1] = v.y; b[h * 4 + 2] = v.z; b[h * 4 + 3] = v.w;
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
}

template <int BM, int BN, int BK, int TM, int TN, bool TA, bool TB>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), 2)
gemm_kernel(GemmParams p) {
    using Cfg = GemmCfg<BM, BN, BK, TM, TN, TA, TB>;
    constexpr int LDA_S = BM + Cfg::APAD;
    constexpr int LDB_S = BN + Cfg::BPAD;
    __shared__ __align__(16) float As[2][BK * LDA_S];
    __shared__ __align__(16) float Bs[2][BK * LDB_S];

    const int tid = threadIdx.x;
    const int tx = tid % Cfg::TX;
    const int ty = tid / Cfg::TX;
    const int64_t bz = blockIdx.z;
    const int64_t b0 = bz / p.batch1, b1 = bz % p.batch1;
    const float *__restrict__ A = p.A + b0 * p.sA0 + b1 * p.sA1;
    const float *__restrict__ B = p.B + b0 * p.sB0 + b1 * p.sB1;
    float *__restrict__ Cp = p.C + b0 * p.sC0 + b1 * p.sC1;
    const int64_t m0 = (int64_t)blockIdx.y * BM;
    const int64_t n0 = (int64_t)blockIdx.x * BN;
    const int64_t M = p.M, N = p.N, K = p.K;

    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;  // +0 (R2)

    float ra[Cfg::A_ELEMS], rb[Cfg::B_ELEMS];
    const int64_t ktiles = (K + BK - 1) / BK;
    if (ktiles > 0) {
        load_a<Cfg, BM, BK, TA>(ra, A, p.lda, M, K, m0, 0, tid, p.vecA);
        load_b<Cfg, BN, BK, TB>(rb, B, p.ldb, N, K, n0, 0, tid, p.vecB);
        store_a<Cfg, BM, BK, TA>(As[0], ra, tid);
        store_b<Cfg, BN, BK, TB>(Bs[0], rb, tid);
        __syncthreads();
    }
    for (int64_t kt = 0; kt < ktiles; ++kt) {
        const int cur = (int)(kt & 1);
        const bool has_next = kt + 1 < ktiles;
        if (has_next) {
            load_a<Cfg, BM, BK, TA>(ra, A, p.lda, M, K, m0, (kt + 1) * BK, tid, p.vecA);
            load_b<Cfg, BN, BK, TB>(rb, B, p.ldb, N, K, n0, (kt + 1) * BK, tid, p.vecB);
        }
        const int64_t krem = K - kt * BK;
        if (krem >= BK) {
#pragma unroll
            for (int kk = 0; kk < BK; ++kk)
                mma_step<BM, BN, TM, TN, LDA_S, LDB_S>(acc, As[cur], Bs[cur], kk, tx, ty);
        } else {
            // K tail: only the real k values, still ascending (no zero padding)
            for (int kk = 0; kk < (int)krem; ++kk)
                mma_step<BM, BN, TM, TN, LDA_S, LDB_S>(acc, As[cur], Bs[cur], kk, tx, ty);
        }
        if (has_next) {
            store_a<Cfg, BM, BK, TA>(As[cur ^ 1], ra, tid);
            store_b<Cfg, BN, BK, TB>(Bs[cur ^ 1], rb, tid);
        }
        __syncthreads();
    }

    // epilogue (R3): epi(acc) once, NaN canonicalised (R10)
#pragma unroll
    for (int hi = 0; hi < TM / 4; ++hi)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = hi * 4 + r;
            const int64_t m = m0 + hi * (BM / (TM / 4)) + ty * 4 + r;
            if (m >= M) continue;
#pragma unroll
            for (int hj = 0; hj < TN / 4; ++hj) {
                const int64_t n = n0 + hj * (BN / (TN / 4)) + tx * 4;
                float v[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float x = acc[i][hj * 4 + c];
                    if (p.epi == 1) x = (n + c < N) ? __fadd_rn(x, __ldg(p.bias + n + c)) : x;
                    else if (p.epi == 2) x = __fmul_rn(x, p.scale);
                    v[c] = canon(x);
                }
                float *dst = Cp + m * p.ldc + n;
                if (p.vecC && n + 4 <= N) {
                    *reinterpret_cast<float4 *>(dst) = make_float4(v[0], v[1], v[2], v[3]);
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (n + c < N) dst[c] = v[c];
                }
            }
        }
}

template <int BM, int BN, int BK, int TM, int TN>
cudaError_t launch_cfg(const GemmParams &p, cudaStream_t s) {
    dim3 grid((unsigned)((p.N + BN - 1) / BN), (unsigned)((p.M + BM - 1) / BM), (unsigned)(p.batch0 * p.batch1));
    dim3 block((BM / TM) * (BN / TN));
    if (!p.transA && !p.transB) gemm_kernel<BM, BN, BK, TM, TN, false, false><<<grid, block, 0, s>>>(p);
    else if (!p.transA && p.transB) gemm_kernel<BM, BN, BK, TM, TN, false, true><<<grid, block, 0, s>>>(p);
    else if (p.transA && !p.transB) gemm_kernel<BM, BN, BK, TM, TN, true, false><<<grid, block, 0, s>>>(p);
    else gemm_kernel<BM, BN, BK, TM, TN, true, true><<<grid, block, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

// Tile-config choice (bits-neutral): big tiles when there are enough of them
// to fill the 148 SMs, else 64 x 64.
cudaError_t gemm_launch(const GemmParams &p, cudaStream_t s, int force_cfg) {
    if (p.M == 0 || p.N == 0 || p.batch0 * p.batch1 == 0) return cudaSuccess;
    int cfg = force_cfg;
    if (cfg < 0) {
        int64_t tiles128 = ((p.M + 127) / 128) * ((p.N + 127) / 128) * p.batch0 * p.batch1;
        cfg = (tiles128 >= 120) ? 0 : 1;
    }
    if (cfg == 0) return launch_cfg<128, 128, 16, 8, 8>(p, s);
    return launch_cfg<64, 64, 16, 4, 8>(p, s);
}
