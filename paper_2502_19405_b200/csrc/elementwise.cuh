// elementwise.cuh -- launchers of the per-element operators (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

cudaError_t launch_exp(const float *x, int64_t n, float *y, cudaStream_t s);
cudaError_t launch_log(const float *x, int64_t n, float *y, cudaStream_t s);
cudaError_t launch_tanh(const float *x, int64_t n, float *y, cudaStream_t s);
cudaError_t launch_rsqrt(const float *x, int64_t n, float *y, cudaStream_t s);
cudaError_t launch_gelu(const float *x, int64_t n, float *y, cudaStream_t s);
constexpr int ADAM_MAX_SEGS = 256;
cudaError_t launch_adamw_segments(float *p, const float *g, float *m, float *v, int nseg, const int64_t *start,
                                  const uint8_t *decay, float lr, float b1, float b2, float eps, float wd, float bc1,
                                  float bc2, float omb1, float omb2, cudaStream_t s);
cudaError_t launch_sin(const float *x, int64_t n, float *y, cudaStream_t s);
cudaError_t launch_cos(const float *x, int64_t n, float *y, cudaStream_t s);
cudaError_t launch_erf(const float *x, int64_t n, float *y, cudaStream_t s);
cudaError_t launch_gelu_erf(const float *x, int64_t n, float *y, cudaStream_t s);
cudaError_t launch_gelu_erf_backward(const float *x, const float *dy, int64_t n, float *dx, cudaStream_t s);
cudaError_t launch_rope_tables(const float *inv_freq, int64_t T, int64_t h, float *cosv, float *sinv, cudaStream_t s);
cudaError_t launch_relu(const float *x, int64_t n, float *y, cudaStream_t s);
cudaError_t launch_relu_backward(const float *x, const float *g, int64_t n, float *dx, cudaStream_t s);
cudaError_t launch_gelu_backward(const float *x, const float *dy, int64_t n, float *dx, cudaStream_t s);
cudaError_t launch_add(const float *a, const float *b, int64_t n, float *y, cudaStream_t s);
cudaError_t launch_tree_sum(const float *const *parts, int nparts, int64_t n, float *out, cudaStream_t s);
cudaError_t launch_adamw(float *p, const float *g, float *m, float *v, int64_t n, float lr, float b1, float b2,
                         float eps, float wd, float bc1, float bc2, float omb1, float omb2, int decay,
                         cudaStream_t s);
cudaError_t launch_embedding(const int32_t *tok, int64_t ntok, int64_t T, const float *wte, const float *wpe,
                             int64_t C, float *x0, cudaStream_t s);
cudaError_t launch_embedding_backward(const int32_t *tok, int64_t ntok, int64_t T, const float *dx0, int64_t C,
                                      float *dwte, float *dwpe, cudaStream_t s);
cudaError_t launch_flip_bit(void *data, int64_t elem, int bit, cudaStream_t s);
cudaError_t launch_copy2d_batched(const float *src, int64_t rows, int64_t cols, int64_t lds, int64_t ss, float *dst,
                                  int64_t ldd, int64_t sd, int64_t nb, cudaStream_t s);
cudaError_t launch_copy2d(const float *src, int64_t rows, int64_t cols, int64_t lds, float *dst, int64_t ldd,
                          cudaStream_t s);
cudaError_t launch_swiglu(const float *g, const float *u, int64_t n, float *h, cudaStream_t s);
cudaError_t launch_rope(const float *x, int64_t ntok, int64_t nhead, int64_t hd, int64_t ld, const float *c,
                        const float *sn, float *y, int64_t ldy, cudaStream_t s);
cudaError_t launch_gather_rows(const float *table, const int32_t *idx, int64_t n, int64_t C, float *out,
                               cudaStream_t s);
cudaError_t launch_fill_uniform(float *out, int64_t n, uint64_t seed, double scale, cudaStream_t s);
cudaError_t launch_causal_flags(const float *B, int64_t K, int64_t N, int64_t ldb, int64_t sB0, int64_t sB1,
                                int64_t b0, int64_t b1, uint8_t *F, int64_t ldf, int64_t sF0, int64_t sF1,
                                cudaStream_t s);
cudaError_t launch_transpose(const float *x, int64_t rows, int64_t cols, int64_t ldx, float *y, int64_t ldy,
                             cudaStream_t s);
cudaError_t launch_rand_uniform(uint64_t seed, uint64_t stream, int64_t n, float *y, cudaStream_t s);
cudaError_t launch_dropout(const float *x, int64_t n, float p, uint64_t seed, uint64_t stream, float *y,
                           uint8_t *mask, cudaStream_t s);
cudaError_t launch_dropout_backward(const float *dy, int64_t n, float p, uint64_t seed, uint64_t stream, float *dx,
                                    cudaStream_t s);
cudaError_t launch_convert(const void *src, int sdt, int64_t rows, int64_t cols, int64_t lds, void *dst, int ddt,
                           int64_t ldd, cudaStream_t s);
