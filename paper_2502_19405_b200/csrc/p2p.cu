// p2p.cu -- canonical data-parallel gradient combine over peer memory.
//
// R-TREE_S (reading R14; the paper leaves the collective's combine order to future
// work) evaluated as ONE kernel per rank over NVLink peer memory instead of
// an NCCL all-to-all + all-gather: every rank owns a slice [lo, hi) of the gradient,
// loads that slice of the G subtree partials straight from the peers' buffers (P2P
// loads), applies the top log2(G) levels of the balanced tree in registers, and stores
// the sum into every rank's gradient buffer (P2P stores).  Per rank that moves
// 2 (G-1)/G x P x 4 bytes over NVLink -- the bandwidth-optimal volume -- with no
// staging buffer and no separate copy kernels; the arithmetic is elementwise, so the
// slicing cannot change a bit.
//
// Ordering between ranks uses epoch flags in IPC-shared device memory: a signal kernel
// release-stores `epoch` into slot `me` of every peer's flag array (system scope, after
// the producing kernels of the same stream have completed), and a wait kernel spins
// with acquire loads until every slot has reached `epoch`.  The spin is bounded: after
// `timeout_ms` it records a failure in a device status word instead of hanging.
#include "common.cuh"
#include "p2p.cuh"

namespace {

using namespace ro;

RO_DEV uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct PeerIn { const float *p[P2P_MAX_PEERS]; };
struct PeerOut { float *p[P2P_MAX_PEERS]; };
struct PeerFlags { uint32_t *p[P2P_MAX_PEERS]; };

template <int G>
__global__ void __launch_bounds__(256) p2p_tree_kernel(PeerIn in, int64_t lo, int64_t hi, PeerOut out, bool vec,
                                                            const int32_t *status) {
    // a timed-out wait before this launch: store nothing (no stale partial is combined,
    // no peer buffer is written while a late peer may still be reading it)
    if (status && *reinterpret_cast<const volatile int32_t *>(status) != 0) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = hi - lo;
    const int64_t n4 = vec ? n / 4 : 0;
    for (int64_t i = t0; i < n4; i += stride) {
        float4 v[G];
#pragma unroll
        for (int q = 0; q < G; ++q) v[q] = __ldcg(reinterpret_cast<const float4 *>(in.p[q] + lo) + i);
#pragma unroll
        for (int w = 1; w < G; w <<= 1)
#pragma unroll
            for (int q = 0; q < G; q += 2 * w) {
                v[q].x = __fadd_rn(v[q].x, v[q + w].x);
                v[q].y = __fadd_rn(v[q].y, v[q + w].y);
                v[q].z = __fadd_rn(v[q].z, v[q + w].z);
                v[q].w = __fadd_rn(v[q].w, v[q + w].w);
            }
        const float4 r = make_float4(canon(v[0].x), canon(v[0].y), canon(v[0].z), canon(v[0].w));
#pragma unroll
        for (int q = 0; q < G; ++q) __stcg(reinterpret_cast<float4 *>(out.p[q] + lo) + i, r);
    }
    for (int64_t i = n4 * 4 + t0; i < n; i += stride) {
        float v[G];
#pragma unroll
        for (int q = 0; q < G; ++q) v[q] = __ldcg(in.p[q] + lo + i);
#pragma unroll
        for (int w = 1; w < G; w <<= 1)
#pragma unroll
            for (int q = 0; q < G; q += 2 * w) v[q] = __fadd_rn(v[q], v[q + w]);
        const float r = canon(v[0]);
#pragma unroll
        for (int q = 0; q < G; ++q) __stcg(out.p[q] + lo + i, r);
    }
}

__global__ void p2p_signal_kernel(PeerFlags flags, int G, int slot, uint32_t epoch) {
    if (threadIdx.x != 0) return;
    __threadfence_system();
    for (int q = 0; q < G; ++q) {
        uint32_t *f = flags.p[q] + slot;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
    }
}

__global__ void p2p_wait_kernel(const uint32_t *flags, int G, uint32_t epoch, int64_t timeout_ns, int32_t *status) {
    const int q = threadIdx.x;
    if (q < G) {
        const uint64_t t0 = globaltimer();
        for (;;) {
            uint32_t v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + q) : "memory");
            if ((int32_t)(v - epoch) >= 0) break;
            if ((int64_t)(globaltimer() - t0) > timeout_ns) {
                if (status) atomicExch(status, 1);
                break;
            }
            __nanosleep(200);
        }
    }
    __syncthreads();
}

}  // namespace

cudaError_t launch_p2p_tree_combine(const float *const *parts, int G, int64_t lo, int64_t hi, float *const *outs,
                                    const int32_t *status, cudaStream_t s) {
    if (hi <= lo) return cudaSuccess;
    PeerIn in{};
    PeerOut out{};
    bool vec = ((lo & 3) == 0);
    for (int q = 0; q < G; ++q) {
        in.p[q] = parts[q];
        out.p[q] = outs[q];
        vec = vec && ((reinterpret_cast<uintptr_t>(parts[q]) | reinterpret_cast<uintptr_t>(outs[q])) & 15u) == 0;
    }
    const int64_t n = hi - lo;
    int64_t want = (n / 4 + 255) / 256;
    int64_t cap = (int64_t)ro_host::num_sms() * 8;
    const int grid = (int)(want < 1 ? 1 : (want > cap ? cap : want));
    switch (G) {
        case 1: p2p_tree_kernel<1><<<grid, 256, 0, s>>>(in, lo, hi, out, vec, status); break;
        case 2: p2p_tree_kernel<2><<<grid, 256, 0, s>>>(in, lo, hi, out, vec, status); break;
        case 4: p2p_tree_kernel<4><<<grid, 256, 0, s>>>(in, lo, hi, out, vec, status); break;
        case 8: p2p_tree_kernel<8><<<grid, 256, 0, s>>>(in, lo, hi, out, vec, status); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_p2p_signal(uint32_t *const *peer_flags, int G, int slot, uint32_t epoch, cudaStream_t s) {
    PeerFlags f{};
    for (int q = 0; q < G; ++q) f.p[q] = peer_flags[q];
    p2p_signal_kernel<<<1, 32, 0, s>>>(f, G, slot, epoch);
    return cudaGetLastError();
}

cudaError_t launch_p2p_wait(const uint32_t *flags, int G, uint32_t epoch, int64_t timeout_ns, int32_t *status,
                            cudaStream_t s) {
    p2p_wait_kernel<<<1, 32, 0, s>>>(flags, G, epoch, timeout_ns, status);
    return cudaGetLastError();
}
