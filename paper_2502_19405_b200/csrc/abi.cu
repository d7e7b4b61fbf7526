// abi.cu -- the extern "C" boundary of librepops.so (include/repops.h).
//
// Host side only: argument validation, thread-local error messages, tile /
// launch selection (always bits-neutral), the host-side Verde pieces (SHA-256
// of small host buffers, the step Merkle root, node digests, divergence
// search).  Every compute step on a tensor runs in the kernels of gemm.cu,
// rowops.cu, elementwise.cu and sha256.cu.
#include <atomic>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/repops.h"
#include "attention.cuh"
#include "common.cuh"
#include "elementwise.cuh"
#include "gemm.cuh"
#include "p2p.cuh"
#include "rowops.cuh"
#include "sha256.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

std::atomic<int64_t> g_launches{0};
std::atomic<int> g_force_cfg{-1};  // tuning override of the GEMM tile choice (bits-neutral)

// every launcher behind cuda_status() enqueues exactly one kernel on success
// (verde_commit_tensors adds its extra kernels itself)
int cuda_status(cudaError_t e, const char *what) {
    if (e == cudaSuccess) {
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return REPOPS_OK;
    }
    return fail(REPOPS_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }
inline bool a16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

#define REQ(cond, ...) \
    do {               \
        if (!(cond)) return fail(REPOPS_EINVAL, __VA_ARGS__); \
    } while (0)

// ------------------------------------------------------------------ host SHA-256 (FIPS 180-4)
class Sha256 {
  public:
    Sha256() { reset(); }
    void reset() {
        static const uint32_t iv[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                                       0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
        memcpy(h_, iv, sizeof iv);
        total_ = 0;
        used_ = 0;
    }
    Sha256 &put(const void *p, size_t n) {
        const uint8_t *b = static_cast<const uint8_t *>(p);
        total_ += n;
        if (used_) {
            size_t k = std::min(n, (size_t)64 - used_);
            memcpy(blk_ + used_, b, k);
            used_ += k; b += k; n -= k;
            if (used_ == 64) { block(blk_); used_ = 0; }
        }
        while (n >= 64) { block(b); b += 64; n -= 64; }
        if (n) { memcpy(blk_, b, n); used_ = n; }
        return *this;
    }
    Sha256 &u8(uint8_t v) { return put(&v, 1); }
    Sha256 &u16(uint16_t v) { uint8_t b[2] = {(uint8_t)v, (uint8_t)(v >> 8)}; return put(b, 2); }
    Sha256 &u32(uint32_t v) {
        uint8_t b[4];
        for (int i = 0; i < 4; ++i) b[i] = (uint8_t)(v >> (8 * i));
        return put(b, 4);
    }
    Sha256 &u64(uint64_t v) {
        uint8_t b[8];
        for (int i = 0; i < 8; ++i) b[i] = (uint8_t)(v >> (8 * i));
        return put(b, 8);
    }
    void done(uint8_t out[32]) {
        uint64_t bits = total_ * 8;
        uint8_t pad[72] = {0x80};
        size_t padlen = (used_ < 56) ? 56 - used_ : 120 - used_;
        uint8_t lenbe[8];
        for (int i = 0; i < 8; ++i) lenbe[i] = (uint8_t)(bits >> (56 - 8 * i));
        put(pad, padlen);
        put(lenbe, 8);
        for (int i = 0; i < 8; ++i)
            for (int q = 0; q < 4; ++q) out[4 * i + q] = (uint8_t)(h_[i] >> (24 - 8 * q));
    }

  private:
    static uint32_t ror(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }
    void block(const uint8_t *p) {
        static const uint32_t k[64] = {
            0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
            0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
            0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
            0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
            0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
            0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
            0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
            0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};
        uint32_t w[64];
        for (int i = 0; i < 16; ++i)
            w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
        for (int i = 16; i < 64; ++i)
            w[i] = w[i - 16] + (ror(w[i - 15], 7) ^ ror(w[i - 15], 18) ^ (w[i - 15] >> 3)) + w[i - 7] +
                   (ror(w[i - 2], 17) ^ ror(w[i - 2], 19) ^ (w[i - 2] >> 10));
        uint32_t v[8];
        memcpy(v, h_, sizeof v);
        for (int i = 0; i < 64; ++i) {
            uint32_t t1 = v[7] + (ror(v[4], 6) ^ ror(v[4], 11) ^ ror(v[4], 25)) + ((v[4] & v[5]) ^ (~v[4] & v[6])) +
                          k[i] + w[i];
            uint32_t t2 = (ror(v[0], 2) ^ ror(v[0], 13) ^ ror(v[0], 22)) + ((v[0] & v[1]) ^ (v[0] & v[2]) ^ (v[1] & v[2]));
            memmove(v + 1, v, 7 * sizeof(uint32_t));
            v[4] += t1;
            v[0] = t1 + t2;
        }
        for (int i = 0; i < 8; ++i) h_[i] += v[i];
    }
    uint32_t h_[8];
    uint8_t blk_[64];
    uint64_t total_;
    size_t used_;
};

struct Node32 { uint8_t b[32]; };

// RFC 6962 MTH of entries[lo, lo+n)  (entries are 32-byte digests).  hashed:
// the items already are leaf hashes (e.g. SHA-256(0x00 || chunk) from the GPU),
// so MTH of a single item is the item itself.
Node32 mth(const uint8_t *e, int64_t lo, int64_t n, bool hashed = false) {
    Node32 out;
    Sha256 h;
    if (n == 1) {
        if (hashed) memcpy(out.b, e + 32 * lo, 32);
        else h.u8(0x00).put(e + 32 * lo, 32).done(out.b);
        return out;
    }
    int64_t k = 1;
    while (2 * k < n) k *= 2;
    Node32 l = mth(e, lo, k, hashed), r = mth(e, lo + k, n - k, hashed);
    h.u8(0x01).put(l.b, 32).put(r.b, 32).done(out.b);
    return out;
}

// RFC 6962 §2.1.1 PATH(m, D[lo, lo+n)): sibling subtree roots, leaf level first
void audit_path(const uint8_t *e, int64_t lo, int64_t n, int64_t m, bool hashed, std::vector<Node32> &out) {
    if (n <= 1) return;
    int64_t k = 1;
    while (2 * k < n) k *= 2;
    if (m < k) {
        audit_path(e, lo, k, m, hashed, out);
        out.push_back(mth(e, lo + k, n - k, hashed));
    } else {
        audit_path(e, lo + k, n - k, m - k, hashed, out);
        out.push_back(mth(e, lo, k, hashed));
    }
}

}  // namespace

namespace ro_host {
int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    }
    return sms;
}
}  // namespace ro_host

extern "C" {

int repops_abi_version(void) { return REPOPS_ABI_VERSION; }
int64_t repops_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
const char *repops_last_error(void) { return g_err.c_str(); }

// ------------------------------------------------------------------ GEMM
static int gemm_common(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, int transA, int64_t sA0,
                       int64_t sA1, const float *B, int64_t ldb, int transB, int64_t sB0, int64_t sB1, int epi,
                       const float *bias, float scale, float *C, int64_t ldc, int64_t sC0, int64_t sC1, int64_t b0,
                       int64_t b1, void *stream, int force_cfg, int causal = 0, const uint8_t *kflags = nullptr,
                       int64_t ldf = 0, int64_t sF0 = 0, int64_t sF1 = 0, int post = 0, const float *X = nullptr,
                       int64_t ldx = 0, float *C2 = nullptr, int64_t ldc2 = 0) {
    REQ(M >= 0 && N >= 0 && K >= 0 && b0 >= 0 && b1 >= 0, "gemm: negative extent");
    REQ(causal >= 0 && causal <= 2, "gemm: causal mode %d not in {0, 1, 2}", causal);
    REQ(causal != 2 || (kflags && ldf >= N && !transA && !transB), "gemm: causal 2 needs kflags, ldf >= N, NN");
    REQ(epi >= REPOPS_EPI_NONE && epi <= REPOPS_EPI_SCALE, "gemm: unknown epilogue %d", epi);
    if (M == 0 || N == 0 || b0 == 0 || b1 == 0) return REPOPS_OK;
    REQ(C != nullptr, "gemm: C is null");
    REQ(ldc >= N, "gemm: ldc %lld < N %lld", (long long)ldc, (long long)N);
    if (K > 0) {
        REQ(A != nullptr && B != nullptr, "gemm: A or B is null");
        REQ(lda >= (transA ? M : K), "gemm: lda too small");
        REQ(ldb >= (transB ? K : N), "gemm: ldb too small");
    }
    REQ(epi != REPOPS_EPI_BIAS || bias != nullptr, "gemm: bias epilogue without bias");
    GemmParams p{};
    p.M = M; p.N = N; p.K = K;
    p.A = A; p.lda = lda; p.sA0 = sA0; p.sA1 = sA1;
    p.B = B; p.ldb = ldb; p.sB0 = sB0; p.sB1 = sB1;
    p.C = C; p.ldc = ldc; p.sC0 = sC0; p.sC1 = sC1;
    p.batch0 = b0; p.batch1 = b1;
    p.transA = transA ? 1 : 0; p.transB = transB ? 1 : 0;
    p.epi = epi; p.bias = bias; p.scale = scale;
    p.vecA = a16(A) && lda % 4 == 0 && sA0 % 4 == 0 && sA1 % 4 == 0;
    p.vecB = a16(B) && ldb % 4 == 0 && sB0 % 4 == 0 && sB1 % 4 == 0;
    p.vecC = a16(C) && ldc % 4 == 0 && sC0 % 4 == 0 && sC1 % 4 == 0;
    p.causal = causal;
    p.kflags = kflags;
    p.ldf = ldf; p.sF0 = sF0; p.sF1 = sF1;
    p.post = post; p.X = X; p.ldx = ldx; p.C2 = C2; p.ldc2 = ldc2;
    if (force_cfg < 0) force_cfg = g_force_cfg.load(std::memory_order_relaxed);
    // Large single NN products run as (A^T)^T B: A is transposed (a bit-exact copy) into a
    // stream-ordered temporary and the A^T-tile kernel runs -- the row-major A tile costs
    // the shared->shared transpose of every K tile (~8 % at 8192^3), one transpose pass
    // costs < 1 %.  The K order of every output is unchanged, so are its bits (R2).
    if (!transA && causal == 0 && post == 0 && force_cfg < 0 && b0 * b1 == 1 && K > 0 && p.vecA && (double)M * N * K >= 1073741824.0 &&
        M % 4 == 0) {
        void *tmp = nullptr;
        cudaStream_t st = S(stream);
        static std::once_flag pool_once;  // keep freed temporaries cached in the stream-ordered pool
        std::call_once(pool_once, [] {
            int dev = 0;
            cudaMemPool_t pool;
            if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t keep = 1ull << 30;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
            cudaGetLastError();
        });
        if (cudaMallocAsync(&tmp, (size_t)(M * K) * sizeof(float), st) == cudaSuccess) {
            cudaError_t e = launch_transpose(A, M, K, lda, reinterpret_cast<float *>(tmp), M, st);
            if (e == cudaSuccess) {
                GemmParams q = p;
                q.A = reinterpret_cast<const float *>(tmp);
                q.lda = M;
                q.transA = 1;
                q.vecA = true;
                e = gemm_launch(q, st, force_cfg);
            }
            cudaError_t f = cudaFreeAsync(tmp, st);
            if (e == cudaSuccess && f == cudaSuccess) g_launches.fetch_add(1, std::memory_order_relaxed);  // transpose
            return cuda_status(e != cudaSuccess ? e : f, "gemm launch (transposed A)");
        }
        cudaGetLastError();  // no temporary: fall back to the direct kernel below
    }
    return cuda_status(gemm_launch(p, S(stream), force_cfg), "gemm launch");
}

int repops_gemm(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, int transA, const float *B, int64_t ldb,
                int transB, int epi, const float *bias, float scale, float *C, int64_t ldc, void *stream) {
    return gemm_common(M, N, K, A, lda, transA, 0, 0, B, ldb, transB, 0, 0, epi, bias, scale, C, ldc, 0, 0, 1, 1,
                       stream, -1);
}

int repops_gemm_post(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, int transA, const float *B,
                     int64_t ldb, int transB, int epi, const float *bias, float scale, float *C, int64_t ldc, int post,
                     const float *X, int64_t ldx, float *C2, int64_t ldc2, void *stream) {
    REQ(post == REPOPS_POST_GELU || post == REPOPS_POST_GELU_BACKWARD, "gemm_post: unknown post %d", post);
    REQ(C2 && ldc2 >= N && (post != REPOPS_POST_GELU_BACKWARD || (X && ldx >= N)), "gemm_post: bad C2 / X");
    if (M == 0 || N == 0) return REPOPS_OK;
    GemmParams q{};
    q.M = M; q.N = N; q.K = K; q.transA = transA ? 1 : 0; q.transB = transB ? 1 : 0;
    q.vecA = a16(A) && lda % 4 == 0;
    q.vecB = a16(B) && ldb % 4 == 0;
    q.post = post;
    if (gemm_tn_eligible(q) && g_force_cfg.load(std::memory_order_relaxed) < 0) {
        int st = gemm_common(M, N, K, A, lda, transA, 0, 0, B, ldb, transB, 0, 0, epi, bias, scale, C, ldc, 0, 0, 1,
                             1, stream, -1, 0, nullptr, 0, 0, 0, post, X, ldx, C2, ldc2);
        return st;
    }
    // not the A^T kernel's shape: the GEMM, then the separate elementwise launch (same bits)
    REQ(ldc == N && ldc2 == N && (post != REPOPS_POST_GELU_BACKWARD || ldx == N),
        "gemm_post: the unfused fallback needs contiguous C, C2 and X");
    int st = repops_gemm(M, N, K, A, lda, transA, B, ldb, transB, epi, bias, scale, C, ldc, stream);
    if (st != REPOPS_OK) return st;
    return post == REPOPS_POST_GELU ? repops_gelu(C, M * N, C2, stream)
                                    : repops_gelu_backward(X, C, M * N, C2, stream);
}

int repops_gemm_strided_batched(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, int transA, int64_t sA0,
                                int64_t sA1, const float *B, int64_t ldb, int transB, int64_t sB0, int64_t sB1, int epi,
                                const float *bias, float scale, float *C, int64_t ldc, int64_t sC0, int64_t sC1,
                                int64_t batch0, int64_t batch1, void *stream) {
    return gemm_common(M, N, K, A, lda, transA, sA0, sA1, B, ldb, transB, sB0, sB1, epi, bias, scale, C, ldc, sC0,
                       sC1, batch0, batch1, stream, -1);
}

int repops_gemm_strided_batched_causal(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, int transA,
                                       int64_t sA0, int64_t sA1, const float *B, int64_t ldb, int transB, int64_t sB0,
                                       int64_t sB1, int epi, const float *bias, float scale, float *C, int64_t ldc,
                                       int64_t sC0, int64_t sC1, int64_t batch0, int64_t batch1, int causal,
                                       const uint8_t *kflags, int64_t ldf, int64_t sF0, int64_t sF1, void *stream) {
    return gemm_common(M, N, K, A, lda, transA, sA0, sA1, B, ldb, transB, sB0, sB1, epi, bias, scale, C, ldc, sC0,
                       sC1, batch0, batch1, stream, -1, causal, kflags, ldf, sF0, sF1);
}

int repops_causal_suffix_flags(const float *B, int64_t K, int64_t N, int64_t ldb, int64_t sB0, int64_t sB1,
                               int64_t batch0, int64_t batch1, uint8_t *flags, int64_t ldf, int64_t sF0, int64_t sF1,
                               void *stream) {
    REQ(K >= 0 && N >= 0 && batch0 >= 0 && batch1 >= 0, "causal_suffix_flags: negative extent");
    REQ(flags && ldf >= N && (K == 0 || (B && ldb >= N)), "causal_suffix_flags: bad pointer / leading dimension");
    REQ(batch0 * batch1 <= 65535, "causal_suffix_flags: too many problems");
    return cuda_status(launch_causal_flags(B, K, N, ldb, sB0, sB1, batch0, batch1, flags, ldf, sF0, sF1, S(stream)),
                       "causal_suffix_flags");
}

// ------------------------------------------------------------------ fused attention (f4)
int repops_attention_fwd_supported(int64_t T, int64_t hd) { return attention_fwd_supported(T, hd) ? 1 : 0; }

int repops_attention_probs_supported(int64_t T, int64_t hd) { return attention_probs_supported(T, hd) ? 1 : 0; }

int repops_attention_probs(int64_t T, int64_t hd, const float *Q, int64_t ldq, int64_t sq0, int64_t sq1,
                           const float *K, int64_t ldk, int64_t sk0, int64_t sk1, float scale, int causal,
                           float *P, int64_t sp0, int64_t sp1, int64_t batch0, int64_t batch1, void *stream) {
    REQ(T >= 0 && hd >= 0 && batch0 >= 0 && batch1 >= 0, "attention_probs: negative extent");
    if (T == 0 || batch0 * batch1 == 0) return REPOPS_OK;
    if (!attention_probs_supported(T, hd))
        return fail(REPOPS_ESHAPE,
                    "attention_probs: T = %lld, hd = %lld unsupported (hd 64: T %% 32 == 0, T <= 1024; "
                    "hd 128: T %% 16 == 0, T <= 2048)", (long long)T, (long long)hd);
    REQ(Q && K && P, "attention_probs: null pointer");
    REQ(ldq >= hd && ldk >= hd, "attention_probs: leading dimension < hd");
    const bool al = a16(Q) && a16(K) && a16(P) && ldq % 4 == 0 && ldk % 4 == 0 && sq0 % 4 == 0 && sq1 % 4 == 0 &&
                    sk0 % 4 == 0 && sk1 % 4 == 0 && sp0 % 4 == 0 && sp1 % 4 == 0;
    REQ(al, "attention_probs: rows must be 16-byte aligned");
    return cuda_status(launch_attention_probs(T, hd, Q, K, ldq, sq0, sq1, ldk, sk0, sk1, scale, causal, P, sp0, sp1,
                                              batch0, batch1, S(stream)),
                       "attention_probs");
}

int repops_attention_dscores(int64_t T, int64_t hd, const float *dO, int64_t ldo, int64_t so0, int64_t so1,
                             const float *V, int64_t ldv, int64_t sv0, int64_t sv1, const float *P, int64_t sp0,
                             int64_t sp1, float scale, float *dS, int64_t sd0, int64_t sd1, int64_t batch0,
                             int64_t batch1, void *stream) {
    REQ(T >= 0 && hd >= 0 && batch0 >= 0 && batch1 >= 0, "attention_dscores: negative extent");
    if (T == 0 || batch0 * batch1 == 0) return REPOPS_OK;
    if (!attention_dscores_supported(T, hd))
        return fail(REPOPS_ESHAPE, "attention_dscores: T = %lld, hd = %lld unsupported (hd 64, T %% 32 == 0, T <= 1024)",
                    (long long)T, (long long)hd);
    REQ(dO && V && P && dS, "attention_dscores: null pointer");
    REQ(ldo >= hd && ldv >= hd, "attention_dscores: leading dimension < hd");
    const bool al = a16(dO) && a16(V) && a16(P) && a16(dS) && ldo % 4 == 0 && ldv % 4 == 0 && so0 % 4 == 0 &&
                    so1 % 4 == 0 && sv0 % 4 == 0 && sv1 % 4 == 0 && sp0 % 4 == 0 && sp1 % 4 == 0 && sd0 % 4 == 0 &&
                    sd1 % 4 == 0;
    REQ(al, "attention_dscores: rows must be 16-byte aligned");
    return cuda_status(launch_attention_dscores(T, dO, ldo, so0, so1, V, ldv, sv0, sv1, P, sp0, sp1, scale, dS, sd0,
                                                sd1, batch0, batch1, S(stream)),
                       "attention_dscores");
}

int repops_attention_fwd(int64_t T, int64_t hd, const float *Q, const float *K, const float *V, int64_t ld,
                         int64_t s0, int64_t s1, float scale, int causal, float *Sout, float *Pout, int64_t sp0,
                         int64_t sp1, float *O, int64_t ldo, int64_t so0, int64_t so1, int64_t batch0,
                         int64_t batch1, void *stream) {
    REQ(T >= 0 && hd >= 0 && batch0 >= 0 && batch1 >= 0, "attention_fwd: negative extent");
    if (T == 0 || batch0 * batch1 == 0) return REPOPS_OK;
    if (!attention_fwd_supported(T, hd))
        return fail(REPOPS_ESHAPE, "attention_fwd: T = %lld, hd = %lld unsupported (hd 64, T %% 128 == 0, T <= 512)",
                    (long long)T, (long long)hd);
    REQ(Q && K && V && O, "attention_fwd: null pointer");
    REQ(ld >= hd && ldo >= hd, "attention_fwd: leading dimension < hd");
    REQ(batch0 * batch1 <= 65535, "attention_fwd: too many (batch, head) pairs");
    const bool al = a16(Q) && a16(K) && a16(V) && a16(O) && (!Sout || a16(Sout)) && (!Pout || a16(Pout)) && ld % 4 == 0 &&
                    ldo % 4 == 0 && s0 % 4 == 0 && s1 % 4 == 0 && so0 % 4 == 0 && so1 % 4 == 0 && sp0 % 4 == 0 &&
                    sp1 % 4 == 0;
    REQ(al, "attention_fwd: rows must be 16-byte aligned");
    return cuda_status(launch_attention_fwd(T, Q, K, V, ld, s0, s1, scale, causal, Sout, Pout, sp0, sp1, O, ldo, so0, so1,
                                            batch0, batch1, S(stream)),
                       "attention_fwd");
}

// ------------------------------------------------------------------ R30 stored precision
static bool lp_dtype(int dt) { return dt == VERDE_F32 || dt == VERDE_BF16 || dt == VERDE_F16; }
static int64_t lp_size(int dt) { return dt == VERDE_F32 ? 4 : 2; }
static int64_t align256(int64_t b) { return (b + 255) & ~int64_t(255); }

int repops_convert(const void *src, int src_dtype, int64_t rows, int64_t cols, int64_t lds, void *dst, int dst_dtype,
                   int64_t ldd, void *stream) {
    REQ(lp_dtype(src_dtype) && lp_dtype(dst_dtype), "convert: dtypes %d -> %d not in {f32, bf16, f16}", src_dtype,
        dst_dtype);
    REQ(rows >= 0 && cols >= 0 && lds >= cols && ldd >= cols, "convert: bad extent / leading dimension");
    if (rows * cols == 0) return REPOPS_OK;
    REQ(src && dst, "convert: null pointer");
    return cuda_status(launch_convert(src, src_dtype, rows, cols, lds, dst, dst_dtype, ldd, S(stream)), "convert");
}

int64_t repops_gemm_ex_workspace_bytes(int64_t M, int64_t N, int64_t K, int a_dtype, int b_dtype, int c_dtype) {
    int64_t b = 0;
    if (a_dtype != VERDE_F32) b += align256(M * K * 4);
    if (b_dtype != VERDE_F32) b += align256(K * N * 4);
    if (c_dtype != VERDE_F32) b += align256(M * N * 4);
    return b;
}

int repops_gemm_ex(int64_t M, int64_t N, int64_t K, const void *A, int a_dtype, int64_t lda, int transA, const void *B,
                   int b_dtype, int64_t ldb, int transB, int epi, const float *bias, float scale, void *C, int c_dtype,
                   int64_t ldc, void *ws, int64_t ws_bytes, void *stream) {
    REQ(lp_dtype(a_dtype) && lp_dtype(b_dtype) && lp_dtype(c_dtype), "gemm_ex: dtype not in {f32, bf16, f16}");
    REQ(M >= 0 && N >= 0 && K >= 0, "gemm_ex: negative extent");
    const int64_t need = repops_gemm_ex_workspace_bytes(M, N, K, a_dtype, b_dtype, c_dtype);
    if (need > 0) REQ(ws != nullptr, "gemm_ex: workspace required");
    if (ws_bytes < need) return fail(REPOPS_ENOSPACE, "gemm_ex: workspace %lld < %lld bytes", (long long)ws_bytes,
                                     (long long)need);
    char *w = static_cast<char *>(ws);
    const float *a = static_cast<const float *>(A), *b = static_cast<const float *>(B);
    int64_t la = lda, lb = ldb;
    int st;
    if (a_dtype != VERDE_F32 && M * K > 0) {   // widen A in its stored orientation, packed
        const int64_t r = transA ? K : M, c = transA ? M : K;
        REQ(A && lda >= c, "gemm_ex: A null or lda too small");
        if ((st = repops_convert(A, a_dtype, r, c, lda, w, VERDE_F32, c, stream)) != REPOPS_OK) return st;
        a = reinterpret_cast<const float *>(w);
        la = c;
        w += align256(M * K * 4);
    }
    if (b_dtype != VERDE_F32 && K * N > 0) {
        const int64_t r = transB ? N : K, c = transB ? K : N;
        REQ(B && ldb >= c, "gemm_ex: B null or ldb too small");
        if ((st = repops_convert(B, b_dtype, r, c, ldb, w, VERDE_F32, c, stream)) != REPOPS_OK) return st;
        b = reinterpret_cast<const float *>(w);
        lb = c;
        w += align256(K * N * 4);
    }
    if (c_dtype == VERDE_F32)
        return repops_gemm(M, N, K, a, la, transA, b, lb, transB, epi, bias, scale, static_cast<float *>(C), ldc,
                           stream);
    REQ(C && ldc >= N, "gemm_ex: C null or ldc too small");
    float *c32 = reinterpret_cast<float *>(w);
    if ((st = repops_gemm(M, N, K, a, la, transA, b, lb, transB, epi, bias, scale, c32, N, stream)) != REPOPS_OK)
        return st;
    return repops_convert(c32, VERDE_F32, M, N, N, C, c_dtype, ldc, stream);
}

// Tuning hook (not in repops.h): process-wide override of the automatic tile
// choice (-1 = automatic).  Bits never depend on it.
int repops_gemm_force_cfg(int cfg) {
    REQ(cfg >= -1 && cfg < gemm_num_cfgs(), "gemm_force_cfg: unknown configuration %d", cfg);
    g_force_cfg.store(cfg);
    return REPOPS_OK;
}

// Tuning hook (not in repops.h): minimum dynamic shared memory per GEMM CTA, used
// to cap GEMM occupancy in co-residency experiments.  Bits never depend on it.
int repops_gemm_smem_floor(int bytes) {
    REQ(bytes >= 0 && bytes <= 227 * 1024, "gemm_smem_floor: %d bytes out of range", bytes);
    g_gemm_smem_floor.store(bytes);
    return REPOPS_OK;
}

// Tuning hook (not in repops.h): cap on resident SHA-256 leaf CTAs per SM.
int repops_commit_ctas_per_sm(int n) {
    REQ(n >= 1 && n <= 64, "commit_ctas_per_sm: %d out of range", n);
    g_leaf_ctas_per_sm.store(n);
    return REPOPS_OK;
}

// Test hook (not in repops.h): number of tile configurations repops_gemm_cfg accepts.
int repops_gemm_num_cfgs() { return gemm_num_cfgs(); }

// Test hook (not in repops.h): force a tile configuration to prove bits-neutrality.
int repops_gemm_cfg(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, int transA, const float *B,
                    int64_t ldb, int transB, int epi, const float *bias, float scale, float *C, int64_t ldc,
                    void *stream, int cfg) {
    REQ(cfg >= 0 && cfg < gemm_num_cfgs(), "gemm_cfg: unknown tile configuration %d", cfg);
    return gemm_common(M, N, K, A, lda, transA, 0, 0, B, ldb, transB, 0, 0, epi, bias, scale, C, ldc, 0, 0, 1, 1,
                       stream, cfg);
}

// ------------------------------------------------------------------ reductions
int repops_sum_rows(const float *x, int64_t rows, int64_t cols, int64_t ld, float *out, void *stream) {
    REQ(rows >= 0 && cols >= 0, "sum_rows: negative extent");
    if (rows == 0) return REPOPS_OK;
    REQ(out && (cols == 0 || x), "sum_rows: null pointer");
    REQ(ld >= cols, "sum_rows: ld < cols");
    REQ(cols <= TILE_ELEMS * TILE_ELEMS, "sum_rows: row longer than 4096 tiles");
    return cuda_status(launch_sum_rows(x, rows, cols, ld, out, S(stream)), "sum_rows");
}

int repops_sum_cols_seq(const float *x, int64_t rows, int64_t cols, int64_t ld, int64_t nseg, float *out,
                        int64_t ldo, void *stream) {
    REQ(rows >= 0 && cols >= 0 && nseg >= 1, "sum_cols_seq: bad extent");
    REQ(rows % nseg == 0, "sum_cols_seq: rows %% nseg != 0");
    if (cols == 0) return REPOPS_OK;
    REQ(out && (rows == 0 || x), "sum_cols_seq: null pointer");
    REQ(ld >= cols && ldo >= cols, "sum_cols_seq: ld/ldo < cols");
    return cuda_status(launch_sum_cols_seq(x, rows, cols, ld, nseg, out, ldo, S(stream)), "sum_cols_seq");
}

int repops_tree_sum(const float *const *parts, int nparts, int64_t n, float *out, void *stream) {
    REQ(nparts == 1 || nparts == 2 || nparts == 4 || nparts == 8 || nparts == 16, "tree_sum: nparts %d", nparts);
    REQ(n >= 0, "tree_sum: negative n");
    if (n == 0) return REPOPS_OK;
    REQ(parts && out, "tree_sum: null pointer");
    for (int q = 0; q < nparts; ++q) REQ(parts[q], "tree_sum: null part");
    return cuda_status(launch_tree_sum(parts, nparts, n, out, S(stream)), "tree_sum");
}

// ------------------------------------------------------------------ row operators
int repops_softmax(const float *x, int64_t rows, int64_t cols, int64_t ldx, int causal, float *y, int64_t ldy,
                   void *stream) {
    REQ(rows >= 0 && cols >= 0, "softmax: negative extent");
    if (rows == 0 || cols == 0) return REPOPS_OK;
    REQ(x && y, "softmax: null pointer");
    REQ(ldx >= cols && ldy >= cols, "softmax: ld < cols");
    REQ(cols <= TILE_ELEMS * TILE_ELEMS, "softmax: row too long");
    if (causal && rows % cols != 0) return fail(REPOPS_ESHAPE, "softmax: causal needs rows %% cols == 0");
    return cuda_status(launch_softmax(x, rows, cols, ldx, causal ? 1 : 0, y, ldy, S(stream)), "softmax");
}

int repops_softmax_backward(const float *y, int64_t ldy, const float *dy, int64_t lddy, int64_t rows, int64_t cols,
                            float scale, float *dx, int64_t lddx, void *stream) {
    REQ(rows >= 0 && cols >= 0, "softmax_backward: negative extent");
    if (rows == 0 || cols == 0) return REPOPS_OK;
    REQ(y && dy && dx, "softmax_backward: null pointer");
    REQ(ldy >= cols && lddy >= cols && lddx >= cols, "softmax_backward: ld < cols");
    REQ(cols <= TILE_ELEMS * TILE_ELEMS, "softmax_backward: row too long");
    return cuda_status(launch_softmax_backward(y, ldy, dy, lddy, rows, cols, scale, dx, lddx, S(stream)),
                       "softmax_backward");
}

int repops_layernorm(const float *x, const float *gamma, const float *beta, int64_t rows, int64_t cols, float eps,
                     float *y, float *mean, float *rstd, void *stream) {
    REQ(rows >= 0 && cols >= 1, "layernorm: bad extent");
    REQ(cols <= TILE_ELEMS, "layernorm: cols > 4096 not supported");
    if (rows == 0) return REPOPS_OK;
    REQ(x && gamma && beta && y, "layernorm: null pointer");
    return cuda_status(launch_layernorm(x, gamma, beta, rows, cols, eps, y, mean, rstd, S(stream)), "layernorm");
}

int repops_layernorm_backward(const float *dy, const float *x, const float *gamma, const float *mean,
                              const float *rstd, const float *dres, int64_t rows, int64_t cols, float *dx,
                              void *stream) {
    REQ(rows >= 0 && cols >= 1, "layernorm_backward: bad extent");
    REQ(cols <= TILE_ELEMS, "layernorm_backward: cols > 4096 not supported");
    if (rows == 0) return REPOPS_OK;
    REQ(dy && x && gamma && mean && rstd && dx, "layernorm_backward: null pointer");
    return cuda_status(launch_layernorm_backward(dy, x, gamma, mean, rstd, dres, rows, cols, dx, S(stream)),
                       "layernorm_backward");
}

int repops_layernorm_backward_params(const float *dy, const float *x, const float *mean, const float *rstd,
                                     int64_t rows, int64_t cols, int64_t nseg, float *dgamma, float *dbeta,
                                     int64_t ldo, void *stream) {
    REQ(rows >= 0 && cols >= 0 && nseg >= 1 && rows % nseg == 0, "layernorm_backward_params: bad extent");
    if (cols == 0) return REPOPS_OK;
    REQ(dgamma && dbeta && (rows == 0 || (dy && x && mean && rstd)), "layernorm_backward_params: null pointer");
    REQ(ldo >= cols, "layernorm_backward_params: ldo < cols");
    return cuda_status(launch_layernorm_params(dy, x, mean, rstd, rows, cols, nseg, dgamma, dbeta, ldo, S(stream)),
                       "layernorm_backward_params");
}

int repops_cross_entropy(const float *logits, int64_t rows, int64_t V, int64_t ld, const int32_t *labels, float scale,
                         float *loss, float *dlogits, int64_t ldd, void *stream) {
    REQ(rows >= 0 && V >= 1, "cross_entropy: bad extent");
    if (rows == 0) return REPOPS_OK;
    REQ(logits && labels, "cross_entropy: null pointer");
    REQ(ld >= V && (!dlogits || ldd >= V), "cross_entropy: ld < V");
    REQ(V <= TILE_ELEMS * TILE_ELEMS, "cross_entropy: V too large");
    return cuda_status(launch_cross_entropy(logits, rows, V, ld, labels, scale, loss, dlogits, ldd, S(stream)),
                       "cross_entropy");
}

// ------------------------------------------------------------------ elementwise
#define UNARY(name, fn)                                                           \
    int name(const float *x, int64_t n, float *y, void *stream) {                 \
        REQ(n >= 0, #name ": negative n");                                         \
        if (n == 0) return REPOPS_OK;                                              \
        REQ(x && y, #name ": null pointer");                                       \
        return cuda_status(fn(x, n, y, S(stream)), #name);                         \
    }
UNARY(repops_exp, launch_exp)
UNARY(repops_log, launch_log)
UNARY(repops_tanh, launch_tanh)
UNARY(repops_rsqrt, launch_rsqrt)
UNARY(repops_gelu, launch_gelu)
UNARY(repops_relu, launch_relu)
UNARY(repops_sin, launch_sin)
UNARY(repops_cos, launch_cos)
UNARY(repops_erf, launch_erf)
UNARY(repops_gelu_erf, launch_gelu_erf)

int repops_rand_uniform(uint64_t seed, uint64_t stream_id, int64_t n, float *y, void *stream) {
    REQ(n >= 0, "rand_uniform: negative n");
    if (n == 0) return REPOPS_OK;
    REQ(y, "rand_uniform: null pointer");
    return cuda_status(launch_rand_uniform(seed, stream_id, n, y, S(stream)), "rand_uniform");
}

int repops_dropout(const float *x, int64_t n, float p, uint64_t seed, uint64_t stream_id, float *y, uint8_t *mask,
                   void *stream) {
    REQ(n >= 0, "dropout: negative n");
    REQ(p >= 0.0f && p <= 1.0f, "dropout: p = %g outside [0, 1]", (double)p);
    if (n == 0) return REPOPS_OK;
    REQ(x && y, "dropout: null pointer");
    return cuda_status(launch_dropout(x, n, p, seed, stream_id, y, mask, S(stream)), "dropout");
}

int repops_dropout_backward(const float *dy, int64_t n, float p, uint64_t seed, uint64_t stream_id, float *dx,
                            void *stream) {
    REQ(n >= 0, "dropout_backward: negative n");
    REQ(p >= 0.0f && p <= 1.0f, "dropout_backward: p = %g outside [0, 1]", (double)p);
    if (n == 0) return REPOPS_OK;
    REQ(dy && dx, "dropout_backward: null pointer");
    return cuda_status(launch_dropout_backward(dy, n, p, seed, stream_id, dx, S(stream)), "dropout_backward");
}

int repops_gelu_erf_backward(const float *x, const float *dy, int64_t n, float *dx, void *stream) {
    REQ(n >= 0, "gelu_erf_backward: negative n");
    if (n == 0) return REPOPS_OK;
    REQ(x && dy && dx, "gelu_erf_backward: null pointer");
    return cuda_status(launch_gelu_erf_backward(x, dy, n, dx, S(stream)), "gelu_erf_backward");
}

int repops_rope_tables(const float *inv_freq, int64_t T, int64_t h, float *cosv, float *sinv, void *stream) {
    REQ(T >= 0 && h >= 0 && T < (1 << 24), "rope_tables: bad T / h");
    if (T * h == 0) return REPOPS_OK;
    REQ(inv_freq && cosv && sinv, "rope_tables: null pointer");
    return cuda_status(launch_rope_tables(inv_freq, T, h, cosv, sinv, S(stream)), "rope_tables");
}

int repops_relu_backward(const float *x, const float *g, int64_t n, float *dx, void *stream) {
    REQ(n >= 0, "relu_backward: negative n");
    if (n == 0) return REPOPS_OK;
    REQ(x && g && dx, "relu_backward: null pointer");
    return cuda_status(launch_relu_backward(x, g, n, dx, S(stream)), "relu_backward");
}

int repops_gelu_backward(const float *x, const float *dy, int64_t n, float *dx, void *stream) {
    REQ(n >= 0, "gelu_backward: negative n");
    if (n == 0) return REPOPS_OK;
    REQ(x && dy && dx, "gelu_backward: null pointer");
    return cuda_status(launch_gelu_backward(x, dy, n, dx, S(stream)), "gelu_backward");
}

int repops_add(const float *a, const float *b, int64_t n, float *y, void *stream) {
    REQ(n >= 0, "add: negative n");
    if (n == 0) return REPOPS_OK;
    REQ(a && b && y, "add: null pointer");
    return cuda_status(launch_add(a, b, n, y, S(stream)), "add");
}

int repops_embedding(const int32_t *tok, int64_t ntok, int64_t T, const float *wte, const float *wpe, int64_t C,
                     float *x0, void *stream) {
    REQ(ntok >= 0 && T >= 1 && C >= 0, "embedding: bad extent");
    if (ntok == 0 || C == 0) return REPOPS_OK;
    REQ(tok && wte && wpe && x0, "embedding: null pointer");
    return cuda_status(launch_embedding(tok, ntok, T, wte, wpe, C, x0, S(stream)), "embedding");
}

int repops_embedding_backward(const int32_t *tok, int64_t ntok, int64_t T, const float *dx0, int64_t C, float *dwte,
                              float *dwpe, void *stream) {
    REQ(ntok >= 0 && T >= 1 && C >= 0, "embedding_backward: bad extent");
    REQ(ntok <= 16384, "embedding_backward: at most 16384 tokens per shard");
    if (ntok == 0 || C == 0) return REPOPS_OK;
    REQ(tok && dx0 && dwte, "embedding_backward: null pointer");
    return cuda_status(launch_embedding_backward(tok, ntok, T, dx0, C, dwte, dwpe, S(stream)), "embedding_backward");
}

int repops_adamw_segments(float *p, const float *g, float *m, float *v, int nseg, const int64_t *seg_start,
                          const uint8_t *decay, int64_t step, float lr, float b1, float b2, float eps, float wd,
                          void *stream) {
    REQ(nseg >= 1 && nseg <= ADAM_MAX_SEGS && seg_start && decay && step >= 1, "adamw_segments: bad segments");
    REQ(seg_start[0] == 0, "adamw_segments: seg_start[0] must be 0");
    for (int k = 0; k < nseg; ++k) REQ(seg_start[k + 1] >= seg_start[k], "adamw_segments: starts must not decrease");
    if (seg_start[nseg] == 0) return REPOPS_OK;
    REQ(p && g && m && v, "adamw_segments: null pointer");
    volatile float pw1 = b1, pw2 = b2;  // R15, as repops_adamw
    for (int64_t i = 1; i < step; ++i) {
        pw1 = pw1 * b1;
        pw2 = pw2 * b2;
    }
    volatile float bc1 = 1.0f - pw1, bc2 = 1.0f - pw2, omb1 = 1.0f - b1, omb2 = 1.0f - b2;
    return cuda_status(launch_adamw_segments(p, g, m, v, nseg, seg_start, decay, lr, b1, b2, eps, wd, bc1, bc2, omb1,
                                             omb2, S(stream)),
                       "adamw_segments");
}

int repops_adamw(float *p, const float *g, float *m, float *v, int64_t n, int64_t step, float lr, float b1, float b2,
                 float eps, float wd, int decay, void *stream) {
    REQ(n >= 0 && step >= 1, "adamw: bad n/step");
    if (n == 0) return REPOPS_OK;
    REQ(p && g && m && v, "adamw: null pointer");
    // bc = 1 - b^step, b^step by iterated binary32 multiplication (R15); no contraction here
    volatile float pw1 = b1, pw2 = b2;
    for (int64_t i = 1; i < step; ++i) {
        pw1 = pw1 * b1;
        pw2 = pw2 * b2;
    }
    volatile float bc1 = 1.0f - pw1, bc2 = 1.0f - pw2, omb1 = 1.0f - b1, omb2 = 1.0f - b2;
    return cuda_status(launch_adamw(p, g, m, v, n, lr, b1, b2, eps, wd, bc1, bc2, omb1, omb2, decay ? 1 : 0,
                                    S(stream)),
                       "adamw");
}

int repops_rmsnorm(const float *x, const float *w, int64_t rows, int64_t cols, float eps, float *y, float *rstd,
                   void *stream) {
    REQ(rows >= 0 && cols >= 1 && cols <= TILE_ELEMS, "rmsnorm: need 1 <= cols <= 4096");
    if (rows == 0) return REPOPS_OK;
    REQ(x && w && y, "rmsnorm: null pointer");
    return cuda_status(launch_rmsnorm(x, w, rows, cols, eps, y, rstd, S(stream)), "rmsnorm");
}

int repops_swiglu(const float *g, const float *u, int64_t n, float *h, void *stream) {
    REQ(n >= 0, "swiglu: negative n");
    if (n == 0) return REPOPS_OK;
    REQ(g && u && h, "swiglu: null pointer");
    return cuda_status(launch_swiglu(g, u, n, h, S(stream)), "swiglu");
}

int repops_rope(const float *x, int64_t ntok, int64_t nhead, int64_t hd, int64_t ld, const float *cos_t,
                const float *sin_t, float *y, int64_t ldy, void *stream) {
    REQ(ntok >= 0 && nhead >= 0 && hd >= 2 && hd % 2 == 0, "rope: bad shape");
    if (ntok == 0 || nhead == 0) return REPOPS_OK;
    REQ(x && cos_t && sin_t && y && ld >= nhead * hd && ldy >= nhead * hd, "rope: bad pointer / ld");
    return cuda_status(launch_rope(x, ntok, nhead, hd, ld, cos_t, sin_t, y, ldy, S(stream)), "rope");
}

int repops_gather_rows(const float *table, const int32_t *idx, int64_t n, int64_t C, float *out, void *stream) {
    REQ(n >= 0 && C >= 0, "gather_rows: negative extent");
    if (n == 0 || C == 0) return REPOPS_OK;
    REQ(table && idx && out, "gather_rows: null pointer");
    return cuda_status(launch_gather_rows(table, idx, n, C, out, S(stream)), "gather_rows");
}

int repops_fill_uniform(float *out, int64_t n, uint64_t seed, double scale, void *stream) {
    REQ(n >= 0 && (n == 0 || out), "fill_uniform: bad argument");
    if (n == 0) return REPOPS_OK;
    return cuda_status(launch_fill_uniform(out, n, seed, scale, S(stream)), "fill_uniform");
}

int repops_copy2d_batched(const float *src, int64_t rows, int64_t cols, int64_t lds, int64_t ss, float *dst,
                          int64_t ldd, int64_t sd, int64_t nb, void *stream) {
    REQ(rows >= 0 && cols >= 0 && nb >= 0, "copy2d_batched: negative extent");
    if (rows == 0 || cols == 0 || nb == 0) return REPOPS_OK;
    REQ(src && dst && lds >= cols && ldd >= cols && nb <= 65535, "copy2d_batched: bad pointer / ld / batch");
    return cuda_status(launch_copy2d_batched(src, rows, cols, lds, ss, dst, ldd, sd, nb, S(stream)), "copy2d_batched");
}

int repops_copy2d(const float *src, int64_t rows, int64_t cols, int64_t lds, float *dst, int64_t ldd, void *stream) {
    REQ(rows >= 0 && cols >= 0, "copy2d: negative extent");
    if (rows == 0 || cols == 0) return REPOPS_OK;
    REQ(src && dst && lds >= cols && ldd >= cols, "copy2d: bad pointer / ld");
    return cuda_status(launch_copy2d(src, rows, cols, lds, dst, ldd, S(stream)), "copy2d");
}

int repops_transpose(const float *x, int64_t rows, int64_t cols, int64_t ldx, float *y, int64_t ldy, void *stream) {
    REQ(rows >= 0 && cols >= 0, "transpose: negative extent");
    if (rows == 0 || cols == 0) return REPOPS_OK;
    REQ(x && y && ldx >= cols && ldy >= rows, "transpose: bad pointer or leading dimension");
    return cuda_status(launch_transpose(x, rows, cols, ldx, y, ldy, S(stream)), "transpose");
}

int repops_flip_bit(void *data, int64_t elem, int bit, void *stream) {
    REQ(data && elem >= 0 && bit >= 0 && bit < 32, "flip_bit: bad argument");
    return cuda_status(launch_flip_bit(data, elem, bit, S(stream)), "flip_bit");
}

// ------------------------------------------------------------------ Verde
int repops_ffma2_probe(int64_t ctas, int64_t iters, float *out, void *stream) {
    REQ(ctas >= 0 && ctas <= 65535 * 64 && iters >= 0, "ffma2_probe: bad extent");
    REQ(out || ctas == 0, "ffma2_probe: null output");
    return cuda_status(launch_ffma2_probe(ctas, iters, out, S(stream)), "ffma2_probe");
}

int verde_sha256_probe(int64_t ctas, int64_t iters, uint32_t *out, void *stream) {
    REQ(ctas >= 0 && ctas <= 65535 * 64 && iters >= 0, "sha256_probe: bad extent");
    REQ(out || ctas == 0, "sha256_probe: null output");
    return cuda_status(launch_sha_probe(ctas, iters, out, S(stream)), "sha256_probe");
}

int verde_dirty_chunks(const int32_t *rows, int64_t n, int64_t row_bytes, int64_t nbytes, int all, uint8_t *flags,
                       void *stream) {
    REQ(n >= 0 && row_bytes > 0 && nbytes >= 0, "dirty_chunks: negative extent");
    REQ(flags && (all || n == 0 || rows), "dirty_chunks: null pointer");
    REQ(n <= 12288, "dirty_chunks: at most 12288 rows per call");
    return cuda_status(launch_dirty_chunks(rows, n, row_bytes, nbytes, all, flags, S(stream)), "dirty_chunks");
}

int64_t verde_commit_workspace_bytes(const verde_tensor_desc *descs, int n) {
    if (!descs || n <= 0) return 0;
    return commit_workspace_bytes(descs, n);
}

int verde_commit_tensors(const verde_tensor_desc *descs, int n, void *ws, int64_t ws_bytes, void *stream) {
    REQ(n >= 0, "commit: negative n");
    if (n == 0) return REPOPS_OK;
    REQ(descs != nullptr, "commit: null descriptors");
    for (int t = 0; t < n; ++t) {
        REQ(descs[t].nbytes >= 0 && (descs[t].nbytes == 0 || descs[t].data), "commit: tensor %d has no data", t);
        REQ(descs[t].rank >= 0 && descs[t].rank <= 8, "commit: tensor %d rank %d", t, descs[t].rank);
        REQ(descs[t].digest != nullptr, "commit: tensor %d has no digest buffer", t);
        REQ(!descs[t].base_leaves || descs[t].dirty, "commit: tensor %d has base_leaves without dirty flags", t);
    }
    REQ(ws != nullptr, "commit: null workspace");
    int64_t need = 0;
    int nk = 0;
    cudaError_t e = commit_launch(descs, n, ws, ws_bytes, S(stream), &need, &nk);
    if (e == cudaErrorMemoryAllocation && ws_bytes < need)
        return fail(REPOPS_ENOSPACE, "commit: workspace %lld < %lld bytes", (long long)ws_bytes, (long long)need);
    if (e == cudaSuccess) g_launches.fetch_add(nk - 1, std::memory_order_relaxed);
    return cuda_status(e, "commit");
}

int verde_commit_plan_create(const verde_tensor_desc *descs, int n, void *ws, int64_t ws_bytes,
                             verde_commit_plan **plan) {
    REQ(n >= 1 && descs && ws && plan, "commit_plan_create: bad argument");
    for (int t = 0; t < n; ++t) {
        REQ(descs[t].nbytes >= 0 && (descs[t].nbytes == 0 || descs[t].data), "commit_plan: tensor %d has no data", t);
        REQ(descs[t].rank >= 0 && descs[t].rank <= 8, "commit_plan: tensor %d rank %d", t, descs[t].rank);
        REQ(descs[t].digest != nullptr, "commit_plan: tensor %d has no digest buffer", t);
        REQ(!descs[t].base_leaves || descs[t].dirty, "commit_plan: tensor %d has base_leaves without dirty flags", t);
    }
    int64_t need = 0;
    void *out = nullptr;
    cudaError_t e = commit_plan_create(descs, n, ws, ws_bytes, &out, &need);
    if (e == cudaErrorMemoryAllocation && ws_bytes < need)
        return fail(REPOPS_ENOSPACE, "commit_plan: workspace %lld < %lld bytes", (long long)ws_bytes, (long long)need);
    if (e != cudaSuccess) return fail(REPOPS_ECUDA, "commit_plan_create: %s", cudaGetErrorString(e));
    *plan = reinterpret_cast<verde_commit_plan *>(out);
    return REPOPS_OK;
}

int verde_commit_plan_run(const verde_commit_plan *plan, void *stream) {
    REQ(plan, "commit_plan_run: null plan");
    int nk = 0;
    cudaError_t e = commit_plan_run(plan, S(stream), &nk);
    if (e == cudaSuccess) g_launches.fetch_add(nk - 1, std::memory_order_relaxed);
    return cuda_status(e, "commit_plan_run");
}

void verde_commit_plan_destroy(verde_commit_plan *plan) {
    if (plan) commit_plan_destroy(plan);
}

int verde_commit_tensor(const void *data, int64_t nbytes, int dtype, int rank, const int64_t *dims, uint8_t *digest32,
                        void *ws, int64_t ws_bytes, void *stream) {
    REQ(rank >= 0 && rank <= 8 && (rank == 0 || dims), "commit_tensor: bad rank/dims");
    verde_tensor_desc d{};
    d.data = data;
    d.nbytes = nbytes;
    d.dtype = dtype;
    d.rank = rank;
    for (int i = 0; i < rank; ++i) d.dims[i] = dims[i];
    d.digest = digest32;
    return verde_commit_tensors(&d, 1, ws, ws_bytes, stream);
}

int verde_digest_from_subroots(const uint8_t *subroots, int64_t k, int dtype, int rank, const int64_t *dims,
                               int64_t nbytes, uint8_t *out32) {
    REQ(subroots && out32 && k >= 1 && (k & (k - 1)) == 0, "digest_from_subroots: k must be a power of two");
    REQ(rank >= 0 && rank <= 8 && (rank == 0 || dims), "digest_from_subroots: bad rank");
    REQ(nbytes > 0 && nbytes % (k * 4096) == 0, "digest_from_subroots: slabs must be whole 4096-byte chunks");
    int64_t chunks = nbytes / k / 4096;
    REQ((chunks & (chunks - 1)) == 0, "digest_from_subroots: slab chunk count must be a power of two");
    std::vector<Node32> level((size_t)k);
    for (int64_t i = 0; i < k; ++i) memcpy(level[i].b, subroots + 32 * i, 32);
    while (level.size() > 1) {
        std::vector<Node32> nxt(level.size() / 2);
        for (size_t i = 0; i < nxt.size(); ++i) {
            Sha256 h;
            h.u8(0x01).put(level[2 * i].b, 32).put(level[2 * i + 1].b, 32).done(nxt[i].b);
        }
        level.swap(nxt);
    }
    Sha256 h;
    h.u8(0x54).u8((uint8_t)dtype).u64((uint64_t)rank);
    for (int i = 0; i < rank; ++i) h.u64((uint64_t)dims[i]);
    h.u64((uint64_t)nbytes).u32(4096).put(level[0].b, 32).done(out32);
    return REPOPS_OK;
}

int verde_merkle_root(const uint8_t *leaves, int64_t n, uint8_t *root32) {
    if (n <= 0) return fail(REPOPS_EINVAL, "merkle_root: empty leaf list");
    REQ(leaves && root32, "merkle_root: null pointer");
    Node32 r = mth(leaves, 0, n);
    memcpy(root32, r.b, 32);
    return REPOPS_OK;
}

int verde_merkle_root_hashed(const uint8_t *leaf_hashes, int64_t n, uint8_t *root32) {
    if (n <= 0) return fail(REPOPS_EINVAL, "merkle_root_hashed: empty leaf list");
    REQ(leaf_hashes && root32, "merkle_root_hashed: null pointer");
    Node32 r = mth(leaf_hashes, 0, n, true);
    memcpy(root32, r.b, 32);
    return REPOPS_OK;
}

int verde_merkle_audit_path(const uint8_t *items, int64_t n, int64_t m, int hashed, uint8_t *path, int32_t *len) {
    REQ(items && path && len && n >= 1 && m >= 0 && m < n, "merkle_audit_path: bad argument");
    std::vector<Node32> p;
    audit_path(items, 0, n, m, hashed != 0, p);
    for (size_t i = 0; i < p.size(); ++i) memcpy(path + 32 * i, p[i].b, 32);
    *len = (int32_t)p.size();
    return REPOPS_OK;
}

int verde_merkle_verify_path(const uint8_t *leaf_hash, int64_t m, int64_t n, const uint8_t *path, int32_t len,
                             const uint8_t *root32, int *ok) {
    REQ(leaf_hash && root32 && ok && (len == 0 || path) && n >= 1 && m >= 0 && m < n && len >= 0,
        "merkle_verify_path: bad argument");
    // RFC 9162 §2.1.3.2 inclusion-proof verification
    int64_t fn = m, sn = n - 1;
    Node32 r;
    memcpy(r.b, leaf_hash, 32);
    *ok = 0;
    for (int32_t i = 0; i < len; ++i) {
        if (sn == 0) return REPOPS_OK;
        const uint8_t *p = path + 32 * i;
        Sha256 h;
        if ((fn & 1) || fn == sn) {
            h.u8(0x01).put(p, 32).put(r.b, 32).done(r.b);
            if (!(fn & 1))
                while (!(fn & 1) && fn != 0) { fn >>= 1; sn >>= 1; }
        } else {
            h.u8(0x01).put(r.b, 32).put(p, 32).done(r.b);
        }
        fn >>= 1;
        sn >>= 1;
    }
    *ok = (sn == 0 && memcmp(r.b, root32, 32) == 0) ? 1 : 0;
    return REPOPS_OK;
}

int verde_tensor_digest_from_root(const uint8_t *data_root, int dtype, int rank, const int64_t *dims,
                                  int64_t nbytes, uint8_t *out32) {
    REQ(out32 && rank >= 0 && rank <= 8 && (rank == 0 || dims) && nbytes >= 0, "tensor_digest_from_root: bad argument");
    uint8_t empty[32];
    if (nbytes == 0) {
        Sha256 e;
        e.done(empty);
        data_root = empty;
    }
    REQ(data_root, "tensor_digest_from_root: null root");
    Sha256 h;
    h.u8(0x54).u8((uint8_t)dtype).u64((uint64_t)rank);
    for (int i = 0; i < rank; ++i) h.u64((uint64_t)dims[i]);
    h.u64((uint64_t)nbytes).u32(4096).put(data_root, 32).done(out32);
    return REPOPS_OK;
}

int verde_chunk_leaves(const void *data, int64_t nbytes, uint8_t *leaves, void *stream) {
    REQ(nbytes >= 0, "chunk_leaves: negative size");
    if (nbytes == 0) return REPOPS_OK;
    REQ(data && leaves, "chunk_leaves: null pointer");
    return cuda_status(chunk_leaves_launch(static_cast<const uint8_t *>(data), nbytes, leaves, S(stream)),
                       "chunk_leaves");
}

int verde_first_divergence_hashed(const uint8_t *seq0, const uint8_t *seq1, int64_t n, int64_t *d_out,
                                  int64_t *rounds_out) {
    REQ(n >= 1 && seq0 && seq1 && d_out, "first_divergence_hashed: bad argument");
    int64_t lo = 0, len = n, rounds = 1;
    Node32 a = mth(seq0, 0, n, true), b = mth(seq1, 0, n, true);
    if (memcmp(a.b, b.b, 32) == 0) {
        *d_out = -1;
        if (rounds_out) *rounds_out = rounds;
        return REPOPS_OK;
    }
    while (len > 1) {
        int64_t k = 1;
        while (2 * k < len) k *= 2;
        Node32 l0 = mth(seq0, lo, k, true), l1 = mth(seq1, lo, k, true);
        ++rounds;
        if (memcmp(l0.b, l1.b, 32) != 0) len = k;
        else { lo += k; len -= k; }
    }
    *d_out = lo;
    if (rounds_out) *rounds_out = rounds;
    return REPOPS_OK;
}

int verde_sha256(const uint8_t *data, int64_t n, uint8_t *out32) {
    REQ(n >= 0 && out32 && (n == 0 || data), "sha256: bad argument");
    Sha256 h;
    if (n) h.put(data, (size_t)n);
    h.done(out32);
    return REPOPS_OK;
}

int verde_node_digest(const verde_node *node, uint8_t *out32) {
    REQ(node && out32, "node_digest: null pointer");
    const verde_node &nd = *node;
    REQ(nd.n_attr >= 0 && nd.n_in >= 0 && nd.n_out >= 0 && nd.n_dst >= 0, "node_digest: negative count");
    for (int i = 1; i < nd.n_attr; ++i) REQ(nd.attr_keys[i - 1] < nd.attr_keys[i], "node_digest: attr keys not ascending");
    Sha256 h;
    h.u8(0x4E).u32(nd.index).u16(nd.op).u32(nd.shard);
    h.u32((uint32_t)nd.n_attr);
    for (int i = 0; i < nd.n_attr; ++i) h.u32(nd.attr_keys[i]).u64(nd.attr_vals[i]);
    h.u32((uint32_t)nd.n_in);
    for (int i = 0; i < nd.n_in; ++i) h.u32(nd.in_src_node[i]).u32(nd.in_src_slot[i]);
    h.u32((uint32_t)nd.n_dst);
    for (int i = 0; i < nd.n_dst; ++i) h.u32(nd.dst_nodes[i]);
    h.u32((uint32_t)nd.n_out);
    if (nd.n_in) h.put(nd.in_digests, 32 * (size_t)nd.n_in);
    if (nd.n_out) h.put(nd.out_digests, 32 * (size_t)nd.n_out);
    h.done(out32);
    return REPOPS_OK;
}

int verde_node_digests(int64_t n, const uint8_t *blob, const int64_t *offs, const int64_t *slots, const int64_t *soffs,
                       const uint8_t *table, int64_t n_slots, uint8_t *out, uint8_t *root32) {
    REQ(n >= 1 && blob && offs && slots && soffs && table && out, "node_digests: bad argument");
    for (int64_t i = 0; i < n; ++i) {
        REQ(offs[i] <= offs[i + 1] && soffs[i] <= soffs[i + 1], "node_digests: offsets not monotone at %lld",
            (long long)i);
        Sha256 h;
        h.put(blob + offs[i], (size_t)(offs[i + 1] - offs[i]));
        for (int64_t j = soffs[i]; j < soffs[i + 1]; ++j) {
            REQ(slots[j] >= 0 && slots[j] < n_slots, "node_digests: slot out of range");
            h.put(table + 32 * slots[j], 32);
        }
        h.done(out + 32 * i);
    }
    if (root32) {
        Node32 r = mth(out, 0, n);
        memcpy(root32, r.b, 32);
    }
    return REPOPS_OK;
}

int64_t verde_root_plan_workspace_bytes(int64_t n) { return n >= 1 ? root_plan_workspace(n) : 0; }

int verde_root_plan_create(int64_t n, const uint8_t *blob, const int64_t *offs, const int64_t *slots,
                           const int64_t *soffs, const uint8_t *table, uint8_t *node_out, uint8_t *root_out,
                           void *ws, int64_t ws_bytes, verde_root_plan **plan) {
    REQ(n >= 1 && blob && offs && slots && soffs && table && root_out && ws && plan, "root_plan_create: bad argument");
    void *out = nullptr;
    cudaError_t e = root_plan_create(n, blob, offs, slots, soffs, table, node_out, root_out, ws, ws_bytes, &out);
    if (e == cudaErrorMemoryAllocation)
        return fail(REPOPS_ENOSPACE, "root_plan: workspace %lld < %lld", (long long)ws_bytes,
                    (long long)root_plan_workspace(n));
    if (e != cudaSuccess) return fail(REPOPS_ECUDA, "root_plan_create: %s", cudaGetErrorString(e));
    *plan = reinterpret_cast<verde_root_plan *>(out);
    return REPOPS_OK;
}

int verde_root_plan_run(const verde_root_plan *plan, void *stream) {
    REQ(plan, "root_plan_run: null plan");
    int nk = 0;
    cudaError_t e = root_plan_run(plan, S(stream), &nk);
    if (e == cudaSuccess) g_launches.fetch_add(nk - 1, std::memory_order_relaxed);
    return cuda_status(e, "root_plan_run");
}

void verde_root_plan_destroy(verde_root_plan *plan) {
    if (plan) root_plan_destroy(plan);
}

int verde_first_divergence(const uint8_t *seq0, const uint8_t *seq1, int64_t n, int64_t *d_out, int64_t *rounds_out) {
    REQ(n >= 1 && seq0 && seq1 && d_out, "first_divergence: bad argument");
    // Descend the two RFC 6962 trees: at each node compare the LEFT subtree roots;
    // equal -> the first difference is in the right subtree.
    int64_t lo = 0, len = n, rounds = 0;
    Node32 a = mth(seq0, 0, n), b = mth(seq1, 0, n);
    ++rounds;
    if (memcmp(a.b, b.b, 32) == 0) {
        *d_out = -1;
        if (rounds_out) *rounds_out = rounds;
        return REPOPS_OK;
    }
    while (len > 1) {
        int64_t k = 1;
        while (2 * k < len) k *= 2;
        Node32 l0 = mth(seq0, lo, k), l1 = mth(seq1, lo, k);
        ++rounds;
        if (memcmp(l0.b, l1.b, 32) != 0) {
            len = k;
        } else {
            lo += k;
            len -= k;
        }
    }
    *d_out = lo;
    if (rounds_out) *rounds_out = rounds;
    return REPOPS_OK;
}

// ------------------------------------------------------------------ peer memory
int repops_ipc_alloc(int64_t nbytes, void **ptr, uint8_t *handle64) {
    REQ(nbytes > 0 && ptr && handle64, "ipc_alloc: bad argument");
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, (size_t)nbytes);
    if (e != cudaSuccess) return fail(REPOPS_ECUDA, "ipc_alloc: cudaMalloc(%lld): %s", (long long)nbytes,
                                      cudaGetErrorString(e));
    e = cudaMemset(p, 0, (size_t)nbytes);
    cudaIpcMemHandle_t h;
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
        cudaFree(p);
        return fail(REPOPS_ECUDA, "ipc_alloc: %s", cudaGetErrorString(e));
    }
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(handle64, &h, 64);
    *ptr = p;
    return REPOPS_OK;
}

int repops_ipc_open(const uint8_t *handle64, void **ptr) {
    REQ(handle64 && ptr, "ipc_open: bad argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    void *p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(REPOPS_ECUDA, "ipc_open: %s", cudaGetErrorString(e));
    *ptr = p;
    return REPOPS_OK;
}

int repops_ipc_close(void *ptr) {
    REQ(ptr, "ipc_close: null pointer");
    cudaError_t e = cudaIpcCloseMemHandle(ptr);
    return e == cudaSuccess ? REPOPS_OK : fail(REPOPS_ECUDA, "ipc_close: %s", cudaGetErrorString(e));
}

int repops_ipc_free(void *ptr) {
    REQ(ptr, "ipc_free: null pointer");
    cudaError_t e = cudaFree(ptr);
    return e == cudaSuccess ? REPOPS_OK : fail(REPOPS_ECUDA, "ipc_free: %s", cudaGetErrorString(e));
}

int repops_p2p_tree_combine(const float *const *parts, int G, int64_t lo, int64_t hi, float *const *outs,
                            const int32_t *status, void *stream) {
    REQ(G == 1 || G == 2 || G == 4 || G == 8, "p2p_tree_combine: G = %d is not 1, 2, 4 or 8", G);
    REQ(lo >= 0 && hi >= lo, "p2p_tree_combine: bad slice [%lld, %lld)", (long long)lo, (long long)hi);
    if (hi == lo) return REPOPS_OK;
    REQ(parts && outs, "p2p_tree_combine: null pointer array");
    for (int q = 0; q < G; ++q) REQ(parts[q] && outs[q], "p2p_tree_combine: null peer pointer %d", q);
    return cuda_status(launch_p2p_tree_combine(parts, G, lo, hi, outs, status, S(stream)), "p2p_tree_combine");
}

int repops_p2p_signal(uint32_t *const *peer_flags, int G, int slot, uint32_t epoch, void *stream) {
    REQ(G >= 1 && G <= P2P_MAX_PEERS && slot >= 0 && slot < G && peer_flags, "p2p_signal: bad argument");
    for (int q = 0; q < G; ++q) REQ(peer_flags[q], "p2p_signal: null peer flag array %d", q);
    return cuda_status(launch_p2p_signal(peer_flags, G, slot, epoch, S(stream)), "p2p_signal");
}

int repops_p2p_wait(const uint32_t *flags, int G, uint32_t epoch, int64_t timeout_ms, int32_t *status,
                    void *stream) {
    REQ(G >= 1 && G <= P2P_MAX_PEERS && flags && timeout_ms > 0, "p2p_wait: bad argument");
    return cuda_status(launch_p2p_wait(flags, G, epoch, timeout_ms * 1000000, status, S(stream)), "p2p_wait");
}

}  // extern "C"
