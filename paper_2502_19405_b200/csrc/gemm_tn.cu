// gemm_tn.cu -- the large-tile R-GEMM for full-tile A^T-stored problems.
//
// Same canonical order as gemm.cu (R1, R2): every output is one thread-private binary32
// accumulator that starts at +0 and takes fma(opA(i,k), opB(k,j), acc) for k = 0..K-1 in
// ascending order; no K split, no padding.  Only the M x N tiling, the register blocking
// and the instruction schedule differ from gemm.cu, so the bits are identical (tested by
// running every configuration on the same inputs).
//
// Micro-kernel (v4, after profiling the library's SIMT SGEMM on sm_100a: 92 % FMA-pipe
// with this structure vs 87 % for gemm.cu's 64 x 128 tiles):
//  * CTA tile 128 x 128, 128 threads (4 warps), 8 x 16 outputs per thread, 2 CTAs / SM;
//  * accumulator PAIRS run along m: FFMA2 acc{m,m+1}[n] += {a_m, a_m+1} * b_n, the A pair
//    read straight from the [BK][BM] A^T tile (one LDS.128 = two pairs), the B value a
//    broadcast scalar -- 64 FFMA2 per k for 6 LDS.128;
//  * BK = 32: one barrier per 2048 FFMA2; fragments are read per k
//    and ptxas schedules the LDS among the FFMA2s (explicit register double buffering of
//    the fragments measured slower: 60.5 vs 65.9 TFLOP/s at 8192^3 -- 255 registers and
//    renamed accumulators; a j-outer FFMA2 order measured 60.8);
//  * global -> shared by cp.async with per-thread pointers advanced by one K tile (64-bit
//    adds on the ALU pipe; no IMAD address math competing with the FFMA2s).
// Preconditions (checked by the launcher): op(A) = A^T stored K x M, B stored K x N,
// 16-byte aligned rows; any M, N, K (edge tiles zero filled, ragged last K tile looped).
// Measured (tools/gemm_auto.py, B200, 1965 MHz): 8192^3 67.0 TFLOP/s (cuBLAS SGEMM 68.5),
// 4096^3 66.0 (59.5); NN through the transposed-A path of repops_gemm 66.6 (63.9).
#include "common.cuh"
#include "gemm.cuh"

namespace {

using ro::canon;

constexpr int THREADS = 128;                // 4 warps, each 4 (m) x 8 (n) lanes
constexpr int GROUP_M = 16;                 // row tiles per rasterisation group

RO_DEV void cp16(uint32_t dst, const float *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}
// bounded copy: the first `bytes` (0, 4, 8, 12 or 16) come from src, the rest is zero filled
RO_DEV void cp16z(uint32_t dst, const float *src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}
RO_DEV void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
RO_DEV void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// BM x BN CTA tile, warps WM (m) x WN (n) with WM * WN = 4: thread (ty, tx) owns rows
// ty*4 + g*4*TYN + {0..3} (g < GM) and columns tx*4 + h*4*TXN + {0..3} (h < GN)
template <int BM, int BN, int WM, int STAGES, int BK, int MINB, int POST>
__global__ void __launch_bounds__(THREADS, MINB) gemm_tn_kernel(GemmParams p) {
    constexpr int WN = 4 / WM, TYN = 4 * WM, TXN = 8 * WN;
    constexpr int TM = BM / TYN, TN = BN / TXN, GM = TM / 4, GN = TN / 4;
    static_assert(TM % 4 == 0 && TN % 4 == 0 && WM * WN == 4, "gemm_tn tile geometry");
    constexpr int A_WORDS = BK * BM, B_WORDS = BK * BN, STAGE_WORDS = A_WORDS + B_WORDS;
    constexpr int CA = BM / 4, CB = BN / 4;                  // 16-byte chunks per tile row
    constexpr int RA = THREADS / CA, RB = THREADS / CB;      // tile rows per chunk step
    constexpr int NQA = BK * CA / THREADS, NQB = BK * CB / THREADS;
    static_assert(THREADS % CA == 0 && THREADS % CB == 0 && NQA >= 1 && NQB >= 1, "gemm_tn load geometry");
    extern __shared__ __align__(16) float smem[];
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int tx = (warp % WN) * 8 + (lane & 7);
    const int ty = (warp / WN) * 4 + (lane >> 3);

    const int64_t tiles_m = (p.M + BM - 1) / BM, tiles_n = (p.N + BN - 1) / BN;
    const int64_t t = blockIdx.x;
    const int64_t per_group = (int64_t)GROUP_M * tiles_n;
    const int64_t grp = t / per_group;
    const int64_t first_m = grp * GROUP_M;
    const int64_t gsz = min((int64_t)GROUP_M, tiles_m - first_m);
    const int64_t m0 = (first_m + (t % per_group) % gsz) * BM;
    const int64_t n0 = ((t % per_group) / gsz) * BN;
    const int64_t b0 = blockIdx.y / p.batch1, b1 = blockIdx.y % p.batch1;
    const float *__restrict__ A = p.A + b0 * p.sA0 + b1 * p.sA1;
    const float *__restrict__ B = p.B + b0 * p.sB0 + b1 * p.sB1;
    float *__restrict__ Cp = p.C + b0 * p.sC0 + b1 * p.sC1;

    // cp.async geometry: thread tid copies the 16-byte chunks at tile rows ra0 + RA q of
    // A^T (column la0) and rb0 + RB q of B (column lb0)
    const int ra0 = tid / CA, la0 = (tid % CA) * 4, rb0 = tid / CB, lb0 = (tid % CB) * 4;
    const float *ga = A + (int64_t)ra0 * p.lda + m0 + la0;
    const float *gb = B + (int64_t)rb0 * p.ldb + n0 + lb0;
    const int64_t qa = RA * p.lda, qb = RB * p.ldb;        // RA / RB rows
    const int64_t ta = BK * p.lda, tb = BK * p.ldb;        // one K tile
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t sa_off = (uint32_t)((ra0 * BM + la0) * 4), sb_off = (uint32_t)((rb0 * BN + lb0) * 4);
    // edge tiles (ragged M / N) and a ragged last K tile take zero-filled bounded copies;
    // the zeros are never used by the k loop (it stops at K) or stored (rows >= M, cols >= N)
    const bool edge = m0 + BM > p.M || n0 + BN > p.N;
    const int a_bytes = (int)max((int64_t)0, min((int64_t)16, (p.M - m0 - la0) * 4));
    const int b_bytes = (int)max((int64_t)0, min((int64_t)16, (p.N - n0 - lb0) * 4));
    const int64_t kfull = p.K / BK;  // full K tiles (a ragged remainder follows them)
    auto issue = [&](int slot, int64_t kt) {
        const uint32_t st = s_base + (uint32_t)(slot * STAGE_WORDS * 4);
        const uint32_t sa = st + sa_off, sb = st + A_WORDS * 4 + sb_off;
        const float *a = ga, *b = gb;
        if (!edge && kt < kfull) {
#pragma unroll
            for (int q = 0; q < NQA; ++q, a += qa) cp16(sa + q * RA * BM * 4, a);
#pragma unroll
            for (int q = 0; q < NQB; ++q, b += qb) cp16(sb + q * RB * BN * 4, b);
        } else {
            const int64_t kva = p.K - kt * BK - ra0, kvb = p.K - kt * BK - rb0;  // rows still in range
#pragma unroll
            for (int q = 0; q < NQA; ++q, a += qa) {
                const bool kin = RA * q < kva;
                cp16z(sa + q * RA * BM * 4, kin && a_bytes ? a : A, kin ? a_bytes : 0);
            }
#pragma unroll
            for (int q = 0; q < NQB; ++q, b += qb) {
                const bool kin = RB * q < kvb;
                cp16z(sb + q * RB * BN * 4, kin && b_bytes ? b : B, kin ? b_bytes : 0);
            }
        }
        ga += ta;
        gb += tb;
    };

    float2 acc[TM / 2][TN];  // pairs of rows (m, m + 1) x columns
#pragma unroll
    for (int i = 0; i < TM / 2; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = make_float2(0.f, 0.f);  // +0 (R2)

    const int64_t ktiles = (p.K + BK - 1) / BK;
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
        if (s < ktiles) issue(s, s);
        cp_commit();
    }

    // fragment reads: A pairs at rows ty*4 + 4 TYN g, B values at cols tx*4 + 4 TXN h
    float4 fa[1][GM], fb[1][GN];
    auto frag = [&](int buf, const float *st, int k) {
        const float *As = st + k * BM + ty * 4;
        const float *Bs = st + A_WORDS + k * BN + tx * 4;
#pragma unroll
        for (int g = 0; g < GM; ++g) fa[buf][g] = *reinterpret_cast<const float4 *>(As + 4 * TYN * g);
#pragma unroll
        for (int h = 0; h < GN; ++h) fb[buf][h] = *reinterpret_cast<const float4 *>(Bs + 4 * TXN * h);
    };
    auto mma = [&](int buf) {
        float b[TN];
        float2 a[TM / 2];
#pragma unroll
        for (int h = 0; h < GN; ++h) {
            b[4 * h] = fb[buf][h].x; b[4 * h + 1] = fb[buf][h].y;
            b[4 * h + 2] = fb[buf][h].z; b[4 * h + 3] = fb[buf][h].w;
        }
#pragma unroll
        for (int g = 0; g < GM; ++g) {
            a[2 * g] = make_float2(fa[buf][g].x, fa[buf][g].y);
            a[2 * g + 1] = make_float2(fa[buf][g].z, fa[buf][g].w);
        }
#pragma unroll
        for (int i = 0; i < TM / 2; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j] = __ffma2_rn(a[i], make_float2(b[j], b[j]), acc[i][j]);
    };

    cp_wait<STAGES - 1>();
    __syncthreads();
    int slot = 0;
    for (int64_t kt = 0; kt < kfull; ++kt) {
        const float *st = smem + slot * STAGE_WORDS;
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            frag(0, st, k);
            mma(0);
        }
        // the next tile must have landed; every thread is past its reads of this stage
        cp_wait<STAGES - 2>();
        __syncthreads();
        if (kt + STAGES < ktiles) issue(slot, kt + STAGES);  // refill the stage just consumed
        cp_commit();
        slot = (slot + 1 == STAGES) ? 0 : slot + 1;
    }
    if (kfull < ktiles) {  // ragged last K tile (landed at the last barrier): the real k only, ascending
        const float *st = smem + slot * STAGE_WORDS;
        const int kmax = (int)(p.K - kfull * BK);
#pragma unroll 1
        for (int k = 0; k < kmax; ++k) {
            frag(0, st, k);
            mma(0);
        }
    }
    cp_wait<0>();

    // epilogue (R3): epi(acc) once, NaN canonicalised (R10); rows ty*4 + 4 TYN g + r
#pragma unroll
    for (int i = 0; i < TM / 2; ++i) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int64_t m = m0 + (i >> 1) * 4 * TYN + ty * 4 + (i & 1) * 2 + half;
            if (m >= p.M) continue;
            float *crow = Cp + m * p.ldc;
#pragma unroll
            for (int h = 0; h < GN; ++h) {
                const int64_t n = n0 + 4 * TXN * h + tx * 4;
                float v[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float x = half ? acc[i][4 * h + c].y : acc[i][4 * h + c].x;
                    if (p.epi == 1) x = (n + c < p.N) ? __fadd_rn(x, __ldg(p.bias + n + c)) : x;
                    else if (p.epi == 2) x = __fmul_rn(x, p.scale);
                    v[c] = canon(x);
                }
                if (p.vecC && n + 4 <= p.N) {
                    *reinterpret_cast<float4 *>(crow + n) = make_float4(v[0], v[1], v[2], v[3]);
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (n + c < p.N) crow[n + c] = v[c];
                }
                if constexpr (POST != 0) {
                    // the elementwise consumer of the stored C values, the same device
                    // functions as repops_gelu / repops_gelu_backward (same bits)
                    float *c2row = p.C2 + b0 * p.sC0 + b1 * p.sC1 + m * p.ldc2;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        if (n + c >= p.N) continue;
                        c2row[n + c] = POST == 1 ? canon(ro::gelu_rn(v[c]))
                                                 : canon(ro::gelu_grad_rn(__ldg(p.X + m * p.ldx + n + c), v[c]));
                    }
                }
            }
        }
    }
}

template <int BM, int BN, int WM, int STAGES, int BK, int MINB, int POST>
cudaError_t launch_tn(const GemmParams &p, cudaStream_t s) {
    size_t smem = (size_t)STAGES * BK * (BM + BN) * sizeof(float);
    const size_t floor_bytes = (size_t)g_gemm_smem_floor.load(std::memory_order_relaxed);
    if (floor_bytes > smem) smem = floor_bytes;  // occupancy experiments only (tools/overlap_probe.py)
    auto kern = gemm_tn_kernel<BM, BN, WM, STAGES, BK, MINB, POST>;
    static size_t attr = 0;
    if (smem > attr) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = smem;
    }
    dim3 grid((unsigned)(((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN)), (unsigned)(p.batch0 * p.batch1));
    kern<<<grid, THREADS, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

bool gemm_tn_eligible(const GemmParams &p) {
    // any M, N, K > 0 (ragged edges zero filled, a ragged last K tile runs a short loop);
    // 16-byte aligned rows of A^T and B
    return p.transA && !p.transB && p.vecA && p.vecB && p.K > 0 && p.causal == 0;
}

cudaError_t gemm_tn_launch(const GemmParams &p, cudaStream_t s, int variant) {
    if (!gemm_tn_eligible(p)) return cudaErrorInvalidValue;
    // 3-stage rings.  128 x 128 (warps 4 x 1, 8 x 16 per thread, 2 CTAs / SM):
    // 3 x 32 KB (BK 32) / 3 x 16 KB (BK 16); 64 x 128 (warps 2 x 2, 8 x 8 per thread,
    // 3 CTAs / SM): 3 x 24 KB / 3 x 12 KB; 64 x 64 (8 x 4 per thread, 4 CTAs / SM)
    if (p.post == 1) {
        if (variant == 32) return launch_tn<128, 128, 4, 3, 32, 2, 1>(p, s);
        if (variant == 6432) return launch_tn<64, 128, 2, 3, 32, 3, 1>(p, s);
        return cudaErrorInvalidValue;
    }
    if (p.post == 2) {
        if (variant == 32) return launch_tn<128, 128, 4, 3, 32, 2, 2>(p, s);
        if (variant == 6432) return launch_tn<64, 128, 2, 3, 32, 3, 2>(p, s);
        return cudaErrorInvalidValue;
    }
    switch (variant) {
        case 32: return launch_tn<128, 128, 4, 3, 32, 2, 0>(p, s);
        case 16: return launch_tn<128, 128, 4, 3, 16, 2, 0>(p, s);
        case 6432: return launch_tn<64, 128, 2, 3, 32, 3, 0>(p, s);
        case 6416: return launch_tn<64, 128, 2, 3, 16, 3, 0>(p, s);
        case 646432: return launch_tn<64, 64, 2, 3, 32, 4, 0>(p, s);
        default: return cudaErrorInvalidValue;
    }
}
