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

constexpr int BM = 128, BN = 128, THREADS = 128;
constexpr int TM = 8, TN = 16;              // outputs per thread
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

template <int STAGES, int BK>
__global__ void __launch_bounds__(THREADS, 2) gemm_tn_kernel(GemmParams p) {
    constexpr int A_WORDS = BK * BM, B_WORDS = BK * BN, STAGE_WORDS = A_WORDS + B_WORDS;
    constexpr int NQ = BK / 4;  // 16-byte chunks per thread per operand and K tile
    extern __shared__ __align__(16) float smem[];
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int tx = lane & 7;                 // n: columns tx*4 + 32 h + {0..3}, h < 4
    const int ty = warp * 4 + (lane >> 3);   // m: rows ty*4 + 64 g + {0..3}, g < 2

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

    // cp.async geometry: a K tile of A^T is 16 rows x 128 floats = 512 16-byte chunks,
    // of B also 512: 4 chunks per thread each, rows r0 + 4q, column l0 (both operands)
    const int r0 = tid >> 5, l0 = (tid & 31) * 4;
    const float *ga = A + (int64_t)r0 * p.lda + m0 + l0;
    const float *gb = B + (int64_t)r0 * p.ldb + n0 + l0;
    const int64_t qa = 4 * p.lda, qb = 4 * p.ldb;          // 4 rows
    const int64_t ta = BK * p.lda, tb = BK * p.ldb;        // one K tile
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t s_off = (uint32_t)((r0 * BM + l0) * 4);
    // edge tiles (ragged M / N) and a ragged last K tile take zero-filled bounded copies;
    // the zeros are never used by the k loop (it stops at K) or stored (rows >= M, cols >= N)
    const bool edge = m0 + BM > p.M || n0 + BN > p.N;
    const int a_bytes = (int)max((int64_t)0, min((int64_t)16, (p.M - m0 - l0) * 4));
    const int b_bytes = (int)max((int64_t)0, min((int64_t)16, (p.N - n0 - l0) * 4));
    const int64_t kfull = p.K / BK;  // full K tiles (a ragged remainder follows them)
    auto issue = [&](int slot, int64_t kt) {
        const uint32_t sa = s_base + (uint32_t)(slot * STAGE_WORDS * 4) + s_off;
        const uint32_t sb = sa + A_WORDS * 4;
        const float *a = ga, *b = gb;
        if (!edge && kt < kfull) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                cp16(sa + q * 4 * BM * 4, a);
                cp16(sb + q * 4 * BN * 4, b);
                a += qa;
                b += qb;
            }
        } else {
            const int64_t kvalid = p.K - kt * BK - r0;  // rows r0 + 4q < kvalid are in range
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const bool kin = 4 * q < kvalid;
                cp16z(sa + q * 4 * BM * 4, kin && a_bytes ? a : A, kin ? a_bytes : 0);
                cp16z(sb + q * 4 * BN * 4, kin && b_bytes ? b : B, kin ? b_bytes : 0);
                a += qa;
                b += qb;
            }
        }
        ga += ta;
        gb += tb;
    };

    float2 acc[TM / 2][TN];
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

    // fragment reads: A pairs at rows ty*4 + 64 g, B values at cols tx*4 + 32 h
    float4 fa[1][2], fb[1][4];
    auto frag = [&](int buf, const float *st, int k) {
        const float *As = st + k * BM + ty * 4;
        const float *Bs = st + A_WORDS + k * BN + tx * 4;
#pragma unroll
        for (int g = 0; g < 2; ++g) fa[buf][g] = *reinterpret_cast<const float4 *>(As + 64 * g);
#pragma unroll
        for (int h = 0; h < 4; ++h) fb[buf][h] = *reinterpret_cast<const float4 *>(Bs + 32 * h);
    };
    auto mma = [&](int buf) {
        const float b[16] = {fb[buf][0].x, fb[buf][0].y, fb[buf][0].z, fb[buf][0].w,
                             fb[buf][1].x, fb[buf][1].y, fb[buf][1].z, fb[buf][1].w,
                             fb[buf][2].x, fb[buf][2].y, fb[buf][2].z, fb[buf][2].w,
                             fb[buf][3].x, fb[buf][3].y, fb[buf][3].z, fb[buf][3].w};
        const float2 a[4] = {make_float2(fa[buf][0].x, fa[buf][0].y), make_float2(fa[buf][0].z, fa[buf][0].w),
                             make_float2(fa[buf][1].x, fa[buf][1].y), make_float2(fa[buf][1].z, fa[buf][1].w)};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[i][j] = __ffma2_rn(a[i], make_float2(b[j], b[j]), acc[i][j]);
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

    // epilogue (R3): epi(acc) once, NaN canonicalised (R10); rows ty*4 + 64 g + r
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int64_t m = m0 + (i >> 1) * 64 + ty * 4 + (i & 1) * 2 + half;
            if (m >= p.M) continue;
            float *crow = Cp + m * p.ldc;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const int64_t n = n0 + 32 * h + tx * 4;
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
            }
        }
    }
}

template <int STAGES, int BK>
cudaError_t launch_tn(const GemmParams &p, cudaStream_t s) {
    size_t smem = (size_t)STAGES * BK * (BM + BN) * sizeof(float);
    const size_t floor_bytes = (size_t)g_gemm_smem_floor.load(std::memory_order_relaxed);
    if (floor_bytes > smem) smem = floor_bytes;  // occupancy experiments only (tools/overlap_probe.py)
    auto kern = gemm_tn_kernel<STAGES, BK>;
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

cudaError_t gemm_tn_launch(const GemmParams &p, cudaStream_t s, int bk) {
    if (!gemm_tn_eligible(p)) return cudaErrorInvalidValue;
    // 3-stage ring: 3 x 32 KB (BK 32) or 3 x 16 KB (BK 16) of shared memory, 2 CTAs / SM
    if (bk == 32) return launch_tn<3, 32>(p, s);
    return launch_tn<3, 16>(p, s);
}
