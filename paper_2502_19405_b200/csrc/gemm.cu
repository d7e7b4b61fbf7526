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
// Kernel (v3).
//  * FFMA2: the micro-kernel issues __ffma2_rn (SASS FFMA2: two binary32 FMAs
//    per lane, each exactly __fmaf_rn, with the A value broadcast from a
//    scalar register).  Accumulators are float2 pairs along n.  Half the FMA
//    instructions of a scalar-FFMA kernel, which is what the v2 profile was
//    limited by (issue / register-bank dispatch stalls).
//  * CTA tile BM x BN (128 x 128, 256 threads, 8 x 8 outputs per thread;
//    or 64 x 64, 128 threads, 8 x 4), BK = 16, STAGES-deep ring in shared
//    memory.  A tiles arrive by cp.async in their global orientation:
//      A^T stored K x M  -> [BK][BM]: 4 consecutive rows at one k = one LDS.128
//      A   stored M x K  -> [BM][BK+4]: rows ty + TY*i, 4 consecutive k of a
//                           row = one LDS.128 (row stride 20 words: the rows a
//                           warp touches fall in disjoint bank groups); with
//                           XP this tile is then transposed shared->shared
//                           into [BK][BM] (double buffered, one extra barrier
//                           per K tile) and read like A^T
//    B tiles are always [BK][BN] (n contiguous) so B pairs are natural float2:
//      B stored K x N    -> cp.async;
//      B^T stored N x K  -> register-staged 4-k loads, transposed on the
//                           store into shared memory (conflict-free: a warp
//                           writes 32 consecutive n of one k row).
//  * Warps are 8 (n) x 4 (m) lanes so one LDS touches <= 128 bytes.
//  * CTAs are rasterised in groups of GROUP_M row tiles (L2 reuse of panels).
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

RO_DEV void cp_async16_s(uint32_t dst, const float *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}

// Interior fast path of tile_async (every chunk in range, 16-byte aligned rows, no
// predicates) as a stateful per-thread loader: the thread's chunk c = tid + q*THREADS
// sits at row r0 + q*RPQ, column l0 of the tile, so one global pointer (advanced by one
// K tile per issue) plus a constant row step addresses all of its chunks -- 64-bit adds
// on the ALU pipe instead of per-chunk IMAD address math on the FMA pipe the FFMA2s use.
// Tiles must be issued in K order (the ring prefetches kt = 0, 1, 2, ... in sequence).
template <int R, int L, int SLD, int THREADS>
struct FullLoader {
    static constexpr int CPR = L / 4;
    static_assert(THREADS % CPR == 0 && (R * CPR) % THREADS == 0, "full-tile loader geometry");
    static constexpr int RPQ = THREADS / CPR;  // tile rows between a thread's chunks
    static constexpr int NQ = R * CPR / THREADS;
    const float *src;
    int64_t qstep, tstep;  // elements: RPQ rows; one K tile
    uint32_t soff;         // bytes: the thread's first chunk within the tile
    RO_DEV void init(const float *base, int64_t ld, int64_t tile_step, int tid) {
        const int r = tid / CPR, l = (tid % CPR) * 4;
        src = base + (int64_t)r * ld + l;
        qstep = (int64_t)RPQ * ld;
        tstep = tile_step;
        soff = (uint32_t)((r * SLD + l) * 4);
    }
    RO_DEV void issue(uint32_t stile) {
        const float *g = src;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            cp_async16_s(stile + soff + q * RPQ * SLD * 4, g);
            g += qstep;
        }
        src += tstep;
    }
};

// B^T stored N x K (k contiguous): each thread loads 4 consecutive k of rows
// n = (tid % BN) (+ BN*... for more chunks) into registers ...
template <int BN, int BK, int THREADS>
struct BtStage {
    static constexpr int CHUNKS = BN * BK / 4 / THREADS;  // float4 chunks per thread
    float v[CHUNKS][4];
};

template <int BN, int BK, int THREADS, bool VEC>
RO_DEV void bt_load(BtStage<BN, BK, THREADS> &st, const float *__restrict__ src, int64_t ld, int64_t nvalid,
                    int64_t kvalid, int tid) {
#pragma unroll
    for (int q = 0; q < BtStage<BN, BK, THREADS>::CHUNKS; ++q) {
        const int c = tid + q * THREADS;
        const int n = c % BN;           // consecutive threads -> consecutive n
        const int kq = (c / BN) * 4;
        const float *s = src + (int64_t)n * ld + kq;
        if (VEC && n < nvalid && kq + 4 <= kvalid) {
            float4 x = __ldg(reinterpret_cast<const float4 *>(s));
            st.v[q][0] = x.x; st.v[q][1] = x.y; st.v[q][2] = x.z; st.v[q][3] = x.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) st.v[q][e] = (n < nvalid && kq + e < kvalid) ? __ldg(s + e) : 0.f;
        }
    }
}

template <int BN, int BK, int THREADS>
RO_DEV void bt_store(float *Bs, const BtStage<BN, BK, THREADS> &st, int tid) {
#pragma unroll
    for (int q = 0; q < BtStage<BN, BK, THREADS>::CHUNKS; ++q) {
        const int c = tid + q * THREADS;
        const int n = c % BN;
        const int kq = (c / BN) * 4;
#pragma unroll
        for (int e = 0; e < 4; ++e) Bs[(kq + e) * BN + n] = st.v[q][e];
    }
}

template <int BM, int BN, int BK, int TM, int TN, bool TA>
struct Cfg {
    static constexpr int TX = BN / TN;          // threads along n
    static constexpr int TY = BM / TM;          // threads along m
    static constexpr int THREADS = TX * TY;
    static constexpr int WX = TX / 8;           // warps along n (8 lanes each)
    static constexpr int SKP = BK + 4;          // k-contiguous A row stride (words)
    static constexpr int A_WORDS = TA ? BK * BM : BM * SKP;
    static constexpr int B_WORDS = BK * BN;
    static constexpr int STAGE_WORDS = A_WORDS + B_WORDS;
    static constexpr int NP = TN / 2;           // accumulator pairs per row
};

template <int BM, int BN, int BK, int TM, int TN, int STAGES, int MINB, int KG, bool TA, bool TB, int LD, bool XP>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), MINB) gemm_kernel(GemmParams p) {
    // XP: an A stored M x K is transposed shared->shared into [BK][BM] once per
    // K tile, so the micro-kernel reads it exactly like A^T (2 LDS.128 per k)
    constexpr bool XA = XP && !TA;
    constexpr bool AT = TA || XA;
    using CF = Cfg<BM, BN, BK, TM, TN, TA>;
    constexpr int THREADS = CF::THREADS;
    constexpr int TX = CF::TX, TY = CF::TY, SKP = CF::SKP, NP = CF::NP;
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
    const int64_t m0 = (first_m + (t % per_group) % gsz) * BM;
    const int64_t n0 = ((t % per_group) / gsz) * BN;

    const int64_t b0 = blockIdx.y / p.batch1, b1 = blockIdx.y % p.batch1;
    const float *__restrict__ A = p.A + b0 * p.sA0 + b1 * p.sA1;
    const float *__restrict__ B = p.B + b0 * p.sB0 + b1 * p.sB1;
    float *__restrict__ Cp = p.C + b0 * p.sC0 + b1 * p.sC1;
    const int64_t M = p.M, N = p.N;
    if (p.causal == 1 && n0 > m0 + BM - 1) return;  // every output of the tile is masked
    // causal A: the tile's rows end at m0 + BM - 1, so op(A)[i][k] = +0 for k >= m0 + BM
    const int64_t K = (p.causal == 2) ? min(p.K, m0 + BM) : p.K;

    // LD == 2: the launcher proved every tile full and aligned -> predicate-free loads
    constexpr bool VEC = LD >= 1;
    const uint32_t smem_s = (uint32_t)__cvta_generic_to_shared(smem);
    FullLoader<TA ? BK : BM, TA ? BM : BK, TA ? BM : SKP, THREADS> lda_;
    FullLoader<BK, BN, BN, THREADS> ldb_;
    if constexpr (LD == 2) {
        if (TA) lda_.init(A + m0, p.lda, (int64_t)BK * p.lda, tid);
        else lda_.init(A + m0 * p.lda, p.lda, BK, tid);
        if (!TB) ldb_.init(B + n0, p.ldb, (int64_t)BK * p.ldb, tid);
    }
    auto load_a = [&](int slot, int64_t kt) {
        float *As = smem + slot * CF::STAGE_WORDS;
        const int64_t k0 = kt * BK;
        if constexpr (LD == 2) {
            if (k0 + BK <= K) {  // every K tile but a ragged last one (always issued in K order)
                const uint32_t st = smem_s + (uint32_t)(slot * CF::STAGE_WORDS * 4);
                lda_.issue(st);
                if (!TB) ldb_.issue(st + CF::A_WORDS * 4);
                return;
            }
        }
        if (TA)  // A stored K x M: tile rows = k, contiguous m
            tile_async<BK, BM, BM, THREADS, VEC>(As, A + k0 * p.lda + m0, p.lda, K - k0, M - m0, tid);
        else     // A stored M x K: tile rows = m, contiguous k
            tile_async<BM, BK, SKP, THREADS, VEC>(As, A + m0 * p.lda + k0, p.lda, M - m0, K - k0, tid);
        if (!TB) {  // B stored K x N -> [BK][BN] directly
            float *Bs = As + CF::A_WORDS;
            tile_async<BK, BN, BN, THREADS, VEC>(Bs, B + k0 * p.ldb + n0, p.ldb, K - k0, N - n0, tid);
        }
    };
    BtStage<BN, BK, THREADS> bst;  // register stage for B^T (TB only)
    auto load_bt = [&](int64_t kt) {
        const int64_t k0 = kt * BK;
        bt_load<BN, BK, THREADS, VEC>(bst, B + n0 * p.ldb + k0, p.ldb, N - n0, K - k0, tid);
    };
    auto store_bt = [&](int slot) { bt_store<BN, BK, THREADS>(smem + slot * CF::STAGE_WORDS + CF::A_WORDS, bst, tid); };

    float2 acc[TM][NP];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < NP; ++j) acc[i][j] = make_float2(0.f, 0.f);  // +0 (R2)

    const int64_t ktiles = (K + BK - 1) / BK;
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ktiles) {
            load_a(s, s);
            if (TB) { load_bt(s); store_bt(s); }
        }
        cp_commit();
    }

    int cur_slot = 0, nxt_slot = STAGES - 1;  // ring positions of tile kt and kt + STAGES - 1
    for (int64_t kt = 0; kt < ktiles; ++kt) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        const int64_t nk = kt + STAGES - 1;
        const bool pref = nk < ktiles;
        if (pref) {
            load_a(nxt_slot, nk);
            if (TB) load_bt(nk);
        }
        cp_commit();
        const int slot_now = cur_slot, slot_pref = nxt_slot;
        cur_slot = (cur_slot + 1 == STAGES) ? 0 : cur_slot + 1;
        nxt_slot = (nxt_slot + 1 == STAGES) ? 0 : nxt_slot + 1;
        const float *As = smem + slot_now * CF::STAGE_WORDS;
        const float *Bs = As + CF::A_WORDS;
        const int kmax = (int)min((int64_t)BK, K - kt * BK);
        if (kmax == BK) {
            const float *Ac = As;  // A in [BK][BM] layout (AT only)
            if constexpr (XA) {
                float *At = smem + STAGES * CF::STAGE_WORDS + (int)(kt & 1) * (BK * BM);
#pragma unroll
                for (int q = 0; q < BM * BK / 4 / THREADS; ++q) {
                    const int c = tid + q * THREADS;
                    const int r = c % BM, kq = (c / BM) * 4;  // a warp: 32 consecutive rows, one k quad
                    const float4 v = *reinterpret_cast<const float4 *>(As + r * SKP + kq);
                    At[(kq + 0) * BM + r] = v.x;
                    At[(kq + 1) * BM + r] = v.y;
                    At[(kq + 2) * BM + r] = v.z;
                    At[(kq + 3) * BM + r] = v.w;
                }
                __syncthreads();  // At[kt & 1] complete (the other buffer may still be read)
                Ac = At;
            }
#pragma unroll
            for (int kg = 0; kg < BK; kg += KG) {
                float ak[AT ? 1 : TM][KG];
                if (!AT) {
#pragma unroll
                    for (int i = 0; i < TM; ++i) {
                        if constexpr (KG == 4) {
                            float4 v = *reinterpret_cast<const float4 *>(As + (ty + TY * i) * SKP + kg);
                            ak[i][0] = v.x; ak[i][1] = v.y; ak[i][2] = v.z; ak[i][3] = v.w;
                        } else {
                            float2 v = *reinterpret_cast<const float2 *>(As + (ty + TY * i) * SKP + kg);
                            ak[i][0] = v.x; ak[i][1] = v.y;
                        }
                    }
                }
#pragma unroll
                for (int kk = 0; kk < KG; ++kk) {
                    float a[TM];
                    float2 b[NP];
                    if (AT) {
#pragma unroll
                        for (int h = 0; h < TM / 4; ++h) {
                            float4 v = *reinterpret_cast<const float4 *>(Ac + (kg + kk) * BM + h * (BM / (TM / 4)) + ty * 4);
                            a[h * 4] = v.x; a[h * 4 + 1] = v.y; a[h * 4 + 2] = v.z; a[h * 4 + 3] = v.w;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < TM; ++i) a[i] = ak[i][kk];
                    }
#pragma unroll
                    for (int h = 0; h < TN / 4; ++h) {
                        float4 v = *reinterpret_cast<const float4 *>(Bs + (kg + kk) * BN + h * (BN / (TN / 4)) + tx * 4);
                        b[2 * h] = make_float2(v.x, v.y);
                        b[2 * h + 1] = make_float2(v.z, v.w);
                    }
#pragma unroll
                    for (int i = 0; i < TM; ++i)
#pragma unroll
                        for (int j = 0; j < NP; ++j) acc[i][j] = __ffma2_rn(make_float2(a[i], a[i]), b[j], acc[i][j]);
                }
            }
        } else {
            // ragged last K tile: the real k only, ascending (no zero padding)
            for (int k = 0; k < kmax; ++k) {
                float a[TM];
                float2 b[NP];
#pragma unroll
                for (int i = 0; i < TM; ++i) {
                    const int rat = (i / 4) * (BM / (TM / 4)) + ty * 4 + (i % 4);  // row in the AT mapping
                    a[i] = TA ? As[k * BM + rat] : XA ? As[rat * SKP + k] : As[(ty + TY * i) * SKP + k];
                }
#pragma unroll
                for (int h = 0; h < TN / 4; ++h) {
                    const float *src = Bs + k * BN + h * (BN / (TN / 4)) + tx * 4;
                    b[2 * h] = make_float2(src[0], src[1]);
                    b[2 * h + 1] = make_float2(src[2], src[3]);
                }
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < NP; ++j) acc[i][j] = __ffma2_rn(make_float2(a[i], a[i]), b[j], acc[i][j]);
            }
        }
        if (TB && pref) store_bt(slot_pref);  // slot of tile kt-1: free since this iteration's barrier
    }
    cp_wait<0>();

    if (p.causal == 2 && K < p.K) {
        // the skipped terms fma(+0, B[k][j], acc), k = K .. p.K - 1, in closed form: a
        // non-finite B gives NaN (0 * inf, NaN); otherwise only acc = -0 can change, to +0
        // unless every skipped B[k][j] is negative (-0 + -0 = -0, -0 + +0 = +0 under RN)
        const uint8_t *fl = p.kflags + b0 * p.sF0 + b1 * p.sF1 + K * p.ldf;
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < NP; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int h = j / 2, c = (j % 2) * 2 + e;
                    const int64_t n = n0 + h * (BN / (TN / 4)) + tx * 4 + c;
                    if (n >= N) continue;
                    const uint8_t f = fl[n];
                    float &x = e ? acc[i][j].y : acc[i][j].x;
                    if (f & 1) x = __uint_as_float(0x7FC00000u);
                    else if (__float_as_uint(x) == 0x80000000u && !(f & 2)) x = 0.0f;
                }
    }

    // epilogue (R3): epi(acc) once, NaN canonicalised (R10)
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int64_t m = m0 + (AT ? (i / 4) * (BM / (TM / 4)) + ty * 4 + (i % 4) : ty + TY * i);
        if (m >= M) continue;
        float *crow = Cp + m * p.ldc;
#pragma unroll
        for (int h = 0; h < TN / 4; ++h) {
            const int64_t n = n0 + h * (BN / (TN / 4)) + tx * 4;
            float v[4] = {acc[i][2 * h].x, acc[i][2 * h].y, acc[i][2 * h + 1].x, acc[i][2 * h + 1].y};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                float x = v[c];
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
    }
}

template <int BM, int BN, int BK, int TM, int TN, int STAGES, int MINB, int KG, bool TA, bool TB, int LD, bool XP>
cudaError_t launch_one(const GemmParams &p, cudaStream_t s) {
    using CF = Cfg<BM, BN, BK, TM, TN, TA>;
    size_t smem = (size_t)(STAGES * CF::STAGE_WORDS + (XP && !TA ? 2 * BK * BM : 0)) * sizeof(float);
    const size_t floor_bytes = (size_t)g_gemm_smem_floor.load(std::memory_order_relaxed);
    if (floor_bytes > smem) smem = floor_bytes;  // occupancy experiments only (tools/overlap_probe.py)
    auto kern = gemm_kernel<BM, BN, BK, TM, TN, STAGES, MINB, KG, TA, TB, LD, XP>;
    static size_t attr_bytes = 0;  // per instantiation
    if (smem > attr_bytes) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_bytes = smem;
    }
    const int64_t tiles = ((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN);
    dim3 grid((unsigned)tiles, (unsigned)(p.batch0 * p.batch1));
    kern<<<grid, CF::THREADS, smem, s>>>(p);
    return cudaGetLastError();
}

template <int BM, int BN, int BK, int TM, int TN, int STAGES, int MINB, int KG = 4, bool XP = false>
cudaError_t launch_cfg(const GemmParams &p, cudaStream_t s) {
    const bool vec = p.vecA && p.vecB;
    // full: every M/N tile complete (a ragged last K tile takes the bounded load)
    const bool full = vec && p.M % BM == 0 && p.N % BN == 0;
#define RO_GEMM_CASE(TA_, TB_)                                                                   \
    if ((bool)p.transA == TA_ && (bool)p.transB == TB_)                                          \
        return full ? launch_one<BM, BN, BK, TM, TN, STAGES, MINB, KG, TA_, TB_, 2, XP>(p, s)        \
                    : vec ? launch_one<BM, BN, BK, TM, TN, STAGES, MINB, KG, TA_, TB_, 1, XP>(p, s)  \
                          : launch_one<BM, BN, BK, TM, TN, STAGES, MINB, KG, TA_, TB_, 0, XP>(p, s);
    RO_GEMM_CASE(false, false)
    RO_GEMM_CASE(false, true)
    RO_GEMM_CASE(true, false)
    RO_GEMM_CASE(true, true)
#undef RO_GEMM_CASE
    return cudaErrorInvalidValue;
}

}  // namespace

// Tile configurations (all bits-neutral: only the M/N tiling differs).
//   0: 128 x 128, 8 x 8 per thread, 3 stages, 2 CTAs/SM
//   1:  64 x  64, 8 x 4 per thread, 3 stages
//   3: 128 x 256 (8 x 16), 4: 256 x 128 (16 x 8), 1 CTA/SM
//   5: 128 x 64, 6: 64 x 128 (8 x 8), 3 CTAs/SM  -- the usual winners
//   2, 7, 8, 9: stage / fragment / occupancy variants kept for tools/gemm_tune.py
//   10..14: 6, 5, 3, 1, 4 with XP (A stored M x K transposed in shared memory)
//   15..18: stage / BK variants of 10; 19: 16 x 32 latency tiles
//   20, 21: gemm_tn.cu 128 x 128 full-tile A^T kernel (BK 32 / 16)
int gemm_num_cfgs() { return 25; }

int gemm_tn_choice(const GemmParams &p) {
    if (!gemm_tn_eligible(p)) return p.post != 0 ? 22 : -1;
    if (p.post == 0 && p.M * p.N * p.batch0 * p.batch1 <= (int64_t)ro_host::num_sms() * 16 * 32 * 4) return -1;
    // A^T-stored problems: gemm_tn.cu's 128 x 128 (cfg 20) and 64 x 128 (cfg 22) tiles and
    // the 128 x 64 tiles of gemm.cu.  Cost = tiles on the busiest SM x tile work / rate
    // (measured on B200: one or two CTAs of either kernel nearly saturate an SM, so the
    // SM-count quantisation of the tile count is what decides; tools/gemm_tune.py)
    struct C { int id, bm, bn; double rate; };
    static const C cand[] = {{20, 128, 128, 66.9}, {22, 64, 128, 66.0}, {5, 128, 64, 60.0}};
    const int64_t nb = p.batch0 * p.batch1;
    const int64_t sms = ro_host::num_sms();
    double best = 1e300;
    int cfg = -1;
    for (const C &c : cand) {
        if (p.post != 0 && c.id == 5) continue;
        const int64_t tiles = ((p.M + c.bm - 1) / c.bm) * ((p.N + c.bn - 1) / c.bn) * nb;
        const double t = (double)((tiles + sms - 1) / sms) * c.bm * c.bn / c.rate;
        if (t < best) { best = t; cfg = c.id; }
    }
    return cfg;
}
std::atomic<int> g_gemm_smem_floor{0};

cudaError_t gemm_launch(const GemmParams &p, cudaStream_t s, int force_cfg) {
    if (p.M == 0 || p.N == 0 || p.batch0 * p.batch1 == 0) return cudaSuccess;
    if (p.batch0 * p.batch1 > 65535) return cudaErrorInvalidValue;
    int cfg = force_cfg;
    if (cfg < 0) cfg = gemm_tn_choice(p);
    if (p.post != 0) {  // fused elementwise epilogue: gemm_tn's 128 x 128 / 64 x 128 tiles only
        if (!gemm_tn_eligible(p)) return cudaErrorInvalidValue;
        return gemm_tn_launch(p, s, cfg == 20 ? 32 : 6432);
    }
    if (cfg < 0) {
        // Wave-quantisation cost model (bits-neutral choice): time ~ waves x tile
        // area / sustained rate, rates measured on B200 with tools/gemm_tune.py and
        // tools/gpt2_gemm_tune.py (TFLOP/s on large, full-wave problems).
        struct C { int id, bm, bn, occ; double rate; };
        static const C cand[] = {{6, 64, 128, 3, 55.0}, {3, 128, 256, 1, 55.0}, {5, 128, 64, 3, 53.0},
                                 {4, 256, 128, 1, 49.0}, {1, 64, 64, 2, 48.0}};
        const int64_t nb = p.batch0 * p.batch1;
        const int sms = ro_host::num_sms();
        double best = 1e300;
        for (const C &c : cand) {
            if (c.id == 4 && !(!p.transA && p.transB)) continue;  // 256x128 only wins for NT
            const int64_t tiles = ((p.M + c.bm - 1) / c.bm) * ((p.N + c.bn - 1) / c.bn) * nb;
            const int64_t slots = (int64_t)sms * c.occ;
            const int64_t waves = (tiles + slots - 1) / slots;
            const double t = (double)waves * c.bm * c.bn * c.occ / c.rate;
            if (t < best * 0.97) { best = t; cfg = c.id; }
        }
        // NN: same tiles with the A operand transposed in shared memory (+1..3%, tools/gemm_tune.py)
        if (!p.transA && !p.transB && cfg == 6) cfg = 10;
        // far below one wave of the large tiles: the per-thread K chain (TM x TN FFMA per k)
        // is the latency, so take the small-tile configuration
        if (p.M * p.N * nb <= (int64_t)sms * 16 * 32 * 4) cfg = 19;
    }
    switch (cfg) {
        case 0: return launch_cfg<128, 128, 16, 8, 8, 3, 2, 4>(p, s);
        case 1: return launch_cfg<64, 64, 16, 8, 4, 3, 2>(p, s);
        case 2: return launch_cfg<128, 128, 16, 8, 8, 4, 1>(p, s);
        case 3: return launch_cfg<128, 256, 16, 8, 16, 3, 1, 4>(p, s);
        case 4: return launch_cfg<256, 128, 16, 16, 8, 3, 1, 4>(p, s);
        case 5: return launch_cfg<128, 64, 16, 8, 8, 3, 3>(p, s);
        case 6: return launch_cfg<64, 128, 16, 8, 8, 3, 3>(p, s);
        case 7: return launch_cfg<64, 128, 16, 8, 8, 3, 3, 2>(p, s);
        case 8: return launch_cfg<128, 64, 16, 8, 8, 3, 3, 2>(p, s);
        case 9: return launch_cfg<64, 128, 16, 8, 8, 3, 2>(p, s);
        case 10: return launch_cfg<64, 128, 16, 8, 8, 3, 3, 4, true>(p, s);
        case 11: return launch_cfg<128, 64, 16, 8, 8, 3, 3, 4, true>(p, s);
        case 12: return launch_cfg<128, 256, 16, 8, 16, 3, 1, 4, true>(p, s);
        case 13: return launch_cfg<64, 64, 16, 8, 4, 3, 2, 4, true>(p, s);
        case 14: return launch_cfg<256, 128, 16, 16, 8, 3, 1, 4, true>(p, s);
        case 15: return launch_cfg<64, 128, 16, 8, 8, 4, 3, 4, true>(p, s);
        case 16: return launch_cfg<64, 128, 16, 8, 8, 5, 3, 4, true>(p, s);
        case 17: return launch_cfg<64, 128, 32, 8, 8, 3, 2, 4, true>(p, s);
        case 18: return launch_cfg<64, 128, 32, 8, 8, 2, 3, 4, true>(p, s);
        // 16 x 32 tiles, one warp, 4 x 4 per thread: latency configuration for problems
        // far below one wave (config 1's MLP, 128^3): 8 FFMA2 per k per thread instead of 32
        case 19: return launch_cfg<16, 32, 16, 4, 4, 3, 16, 4, true>(p, s);
        // gemm_tn.cu: 128 x 128 tiles, pair-along-m FFMA2 (BK = 32 when K allows, else 16);
        // shapes it does not take run the same 128 x 128 x 16 tiling in this kernel
        case 20:
        case 21:
            if (gemm_tn_eligible(p)) return gemm_tn_launch(p, s, cfg == 20 ? 32 : 16);
            return launch_cfg<128, 128, 16, 8, 16, 3, 2>(p, s);
        // gemm_tn.cu 64 x 128 tiles (8 x 8 per thread, pairs along m, 3 CTAs / SM), BK 32 / 16
        case 22:
        case 23:
            if (gemm_tn_eligible(p)) return gemm_tn_launch(p, s, cfg == 22 ? 6432 : 6416);
            return launch_cfg<64, 128, 16, 8, 8, 3, 3>(p, s);
        // gemm_tn.cu 64 x 64 tiles (8 x 4 per thread, 4 CTAs / SM): N = 64 problems (attention)
        case 24:
            if (gemm_tn_eligible(p)) return gemm_tn_launch(p, s, 646432);
            return launch_cfg<64, 64, 16, 8, 4, 3, 2>(p, s);
        default: return cudaErrorInvalidValue;
    }
}

// ------------------------------------------------------------------ diagnostic: FFMA2 ceiling
// The R-GEMM's practical FP32 ceiling: every thread runs `iters` rounds of 32 independent
// FFMA2 chains (64 FMA per round) on register-resident operands -- the FMA pipe with no
// loads, no shared memory, no barriers.  2 flops per FMA.
namespace {
__global__ void __launch_bounds__(128) ffma2_probe_kernel(int64_t iters, float *out) {
    const float g = (float)(blockIdx.x * blockDim.x + threadIdx.x);
    float2 acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = make_float2(g + i, g - i);
    const float2 a = make_float2(1.0000001f, 0.9999999f), b = make_float2(1e-7f, -1e-7f);
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = __ffma2_rn(acc[i], a, b);
    }
    float x = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) x = __fadd_rn(x, __fadd_rn(acc[i].x, acc[i].y));
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}
}  // namespace

cudaError_t launch_ffma2_probe(int64_t ctas, int64_t iters, float *out, cudaStream_t s) {
    if (ctas <= 0 || iters <= 0) return cudaSuccess;
    ffma2_probe_kernel<<<(unsigned)ctas, 128, 0, s>>>(iters, out);
    return cudaGetLastError();
}
