// p2p.cuh -- launchers of the peer-memory gradient combine (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

constexpr int P2P_MAX_PEERS = 8;

cudaError_t launch_p2p_tree_combine(const float *const *parts, int G, int64_t lo, int64_t hi, float *const *outs,
                                    const int32_t *status, cudaStream_t s);
cudaError_t launch_p2p_signal(uint32_t *const *peer_flags, int G, int slot, uint32_t epoch, cudaStream_t s);
cudaError_t launch_p2p_wait(const uint32_t *flags, int G, uint32_t epoch, int64_t timeout_ns, int32_t *status,
                            cudaStream_t s);
