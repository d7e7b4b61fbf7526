// attention.cuh -- fused causal attention forward (internal).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

bool attention_fwd_supported(int64_t T, int64_t hd);
size_t attention_fwd_smem_bytes(int64_t T);
cudaError_t launch_attention_fwd(int64_t T, const float *Q, const float *K, const float *V, int64_t ld, int64_t s0,
                                 int64_t s1, float scale, int causal, float *S, float *P, int64_t sp0, int64_t sp1,
                                 float *O, int64_t ldo, int64_t so0, int64_t so1, int64_t batch0, int64_t batch1,
                                 cudaStream_t s);
bool attention_probs_supported(int64_t T, int64_t hd);
bool attention_dscores_supported(int64_t T, int64_t hd);
cudaError_t launch_attention_probs(int64_t T, int64_t hd, const float *Q, const float *K, int64_t ld, int64_t s0,
                                   int64_t s1, int64_t ldk, int64_t sk0, int64_t sk1, float scale, int causal,
                                   float *P, int64_t sp0, int64_t sp1, int64_t batch0, int64_t batch1,
                                   cudaStream_t s);
cudaError_t launch_attention_dscores(int64_t T, const float *dO, int64_t ldo, int64_t so0, int64_t so1,
                                     const float *V, int64_t ldv, int64_t sv0, int64_t sv1, const float *P,
                                     int64_t sp0, int64_t sp1, float scale, float *dS, int64_t sd0, int64_t sd1,
                                     int64_t batch0, int64_t batch1, cudaStream_t s);
