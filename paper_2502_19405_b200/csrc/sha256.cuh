// sha256.cuh -- batched tensor commitment launcher (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/repops.h"

int64_t commit_workspace_bytes(const verde_tensor_desc *d, int n);
// returns cudaErrorMemoryAllocation (and *need) if ws_bytes is too small
cudaError_t commit_launch(const verde_tensor_desc *d, int n, void *ws, int64_t ws_bytes, cudaStream_t s,
                          int64_t *need, int *nkernels);
cudaError_t commit_plan_create(const verde_tensor_desc *d, int n, void *ws, int64_t ws_bytes, void **out,
                               int64_t *need);
cudaError_t commit_plan_run(const void *plan, cudaStream_t s, int *nkernels);
int64_t root_plan_workspace(int64_t n);
cudaError_t root_plan_create(int64_t n, const uint8_t *blob, const int64_t *offs, const int64_t *slots,
                             const int64_t *soffs, const uint8_t *table, uint8_t *node_out, uint8_t *root_out,
                             void *ws, int64_t ws_bytes, void **out);
cudaError_t root_plan_run(const void *plan, cudaStream_t s, int *nkernels);
void root_plan_destroy(void *plan);
void commit_plan_destroy(void *plan);
// R11 leaf hashes of every 4096-byte chunk of one buffer (device -> device)
cudaError_t chunk_leaves_launch(const uint8_t *data, int64_t nbytes, uint8_t *leaves, cudaStream_t s);
// tuning hook: resident leaf-kernel CTAs per SM (co-residency with GEMMs; bits-neutral)
extern std::atomic<int> g_leaf_ctas_per_sm;
cudaError_t launch_dirty_chunks(const int32_t *rows, int64_t n, int64_t row_bytes, int64_t nbytes, int all,
                                uint8_t *flags, cudaStream_t s);
cudaError_t launch_sha_probe(int64_t ctas, int64_t iters, uint32_t *out, cudaStream_t s);
