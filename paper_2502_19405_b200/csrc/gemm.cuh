// gemm.cuh -- parameters of the R-GEMM launch (internal to librepops.so).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

struct GemmParams {
    int64_t M, N, K;
    const float *A;
    int64_t lda, sA0, sA1;
    const float *B;
    int64_t ldb, sB0, sB1;
    float *C;
    int64_t ldc, sC0, sC1;
    int64_t batch0, batch1;
    int transA, transB;
    int epi;
    const float *bias;
    float scale;
    bool vecA, vecB, vecC;  // 16-byte alignment of every row start (speed only)
    // causal structure (f4, exact): 0 none; 1 = outputs with column > row are never read
    // (scratch scores): CTA tiles entirely above the diagonal are skipped; 2 = op(A)[i][k]
    // is +0 for k > i (causal probabilities): a CTA tile's K fold stops after its last
    // row, and the skipped fma(+0, B[k][j], acc) terms are applied in closed form from
    // kflags[k][j] (bit 0: some B[k'][j], k' >= k, is non-finite; bit 1: every such B
    // has its sign bit set) -- bit-identical to the full fold for every input
    int causal;
    const uint8_t *kflags;
    int64_t ldf, sF0, sF1;
    // fused elementwise consumer of C (gemm_tn only; bits of C2 = the separate kernel's):
    // 0 none; 1 = C2 = R-GELU(C); 2 = C2 = R-GELU backward at X with dy = C
    int post;
    const float *X;
    int64_t ldx;
    float *C2;
    int64_t ldc2;
};

// force_cfg: -1 = automatic, else one of gemm_num_cfgs() tile configurations (bits-neutral)
cudaError_t gemm_launch(const GemmParams &p, cudaStream_t s, int force_cfg);
int gemm_num_cfgs();
// gemm_tn.cu: 128 x 128 x 16 full-tile kernel for op(A) = A^T, op(B) = B (bits-neutral)
bool gemm_tn_eligible(const GemmParams &p);
cudaError_t gemm_tn_launch(const GemmParams &p, cudaStream_t s, int bk);
// cost-model choice between gemm_tn's tiles for an eligible problem (20 / 22) or -1
int gemm_tn_choice(const GemmParams &p);
// tuning hook: minimum dynamic shared memory per GEMM CTA (limits occupancy; bits-neutral)
extern std::atomic<int> g_gemm_smem_floor;
// diagnostic: register-resident FFMA2 rate (the R-GEMM's practical ceiling)
cudaError_t launch_ffma2_probe(int64_t ctas, int64_t iters, float *out, cudaStream_t s);
