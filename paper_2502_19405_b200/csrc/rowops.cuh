// rowops.cuh -- launchers of the row reductions / row operators (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

constexpr int64_t TILE_ELEMS = 4096;  // R4 tile

cudaError_t launch_sum_rows(const float *x, int64_t rows, int64_t cols, int64_t ld, float *out, cudaStream_t s);
cudaError_t launch_sum_cols_seq(const float *x, int64_t rows, int64_t cols, int64_t ld, int64_t nseg, float *out,
                                int64_t ldo, cudaStream_t s);
cudaError_t launch_softmax(const float *x, int64_t rows, int64_t cols, int64_t ldx, int causal, float *y,
                           int64_t ldy, cudaStream_t s);
cudaError_t launch_softmax_backward(const float *y, int64_t ldy, const float *dy, int64_t lddy, int64_t rows,
                                    int64_t cols, float scale, float *dx, int64_t lddx, cudaStream_t s);
cudaError_t launch_layernorm(const float *x, const float *g, const float *b, int64_t rows, int64_t cols, float eps,
                             float *y, float *mean, float *rstd, cudaStream_t s);
cudaError_t launch_layernorm_backward(const float *dy, const float *x, const float *g, const float *mean,
                                      const float *rstd, const float *dres, int64_t rows, int64_t cols, float *dx,
                                      cudaStream_t s);
cudaError_t launch_layernorm_params(const float *dy, const float *x, const float *mean, const float *rstd,
                                    int64_t rows, int64_t cols, int64_t nseg, float *dg, float *db, int64_t ldo,
                                    cudaStream_t s);
cudaError_t launch_rmsnorm(const float *x, const float *w, int64_t rows, int64_t cols, float eps, float *y,
                           float *rstd, cudaStream_t s);
cudaError_t launch_cross_entropy(const float *logits, int64_t rows, int64_t V, int64_t ld, const int32_t *labels,
                                 float scale, float *loss, float *dlogits, int64_t ldd, cudaStream_t s);
