// elementwise.cu -- order-free (per element) operators: software math
// (R5/R6), GELU, residual add, R-TREE_S (R14), AdamW (R15),
// embedding forward/backward (R-EMB), fault injection.
//
// HBM-bound: grid-stride loops over float4 with a grid of a few waves of the
// 148 SMs; each element's arithmetic is the fixed chain in common.cuh.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "elementwise.cuh"

namespace {

using namespace ro;

template <class F>
__global__ void unary_kernel(const float *__restrict__ x, int64_t n, float *__restrict__ y, F f) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n4 = (aligned16(x) && aligned16(y)) ? n / 4 : 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 v = reinterpret_cast<const float4 *>(x)[i];
        reinterpret_cast<float4 *>(y)[i] = make_float4(f(v.x), f(v.y), f(v.z), f(v.w));
    }
    for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) y[i] = f(x[i]);
}

template <class F>
__global__ void binary_kernel(const float *__restrict__ a, const float *__restrict__ b, int64_t n,
                              float *__restrict__ y, F f) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n4 = (aligned16(a) && aligned16(b) && aligned16(y)) ? n / 4 : 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 u = reinterpret_cast<const float4 *>(a)[i];
        float4 v = reinterpret_cast<const float4 *>(b)[i];
        reinterpret_cast<float4 *>(y)[i] = make_float4(f(u.x, v.x), f(u.y, v.y), f(u.z, v.z), f(u.w, v.w));
    }
    for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) y[i] = f(a[i], b[i]);
}

struct ExpF { RO_DEV float operator()(float x) const { return canon(exp_rn(x)); } };
struct LogF { RO_DEV float operator()(float x) const { return canon(log_rn(x)); } };
struct TanhF { RO_DEV float operator()(float x) const { return canon(tanh_rn(x)); } };
struct RsqrtF { RO_DEV float operator()(float x) const { return canon(rsqrt_rn(x)); } };
struct GeluF { RO_DEV float operator()(float x) const { return canon(gelu_rn(x)); } };
struct GeluBwdF { RO_DEV float operator()(float x, float dy) const { return canon(gelu_grad_rn(x, dy)); } };
struct ErfF { RO_DEV float operator()(float x) const { return ro::erf_rn(x); } };
struct GeluErfF { RO_DEV float operator()(float x) const { return canon(ro::gelu_erf_rn(x)); } };
struct GeluErfBwdF { RO_DEV float operator()(float x, float dy) const { return canon(ro::gelu_erf_grad_rn(x, dy)); } };
struct SinF { RO_DEV float operator()(float x) const { return ro::sincos_rn(x, false); } };
struct CosF { RO_DEV float operator()(float x) const { return ro::sincos_rn(x, true); } };
// R26 RoPE tables: angle = fmul(float(t), inv_freq[i]); one thread per (t, i)
__global__ void rope_tables_kernel(const float *__restrict__ inv_freq, int64_t T, int64_t h, float *__restrict__ cosv,
                                   float *__restrict__ sinv) {
    const int64_t n = T * h;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = q / h, i = q % h;
        const float ang = __fmul_rn((float)t, __ldg(inv_freq + i));  // t < 2^24: exact conversion
        cosv[q] = ro::sincos_rn(ang, true);
        sinv[q] = ro::sincos_rn(ang, false);
    }
}
// R28 deterministic pseudorandomness: Philox4x32-10 (curand / PyTorch CUDA generator).
// One thread per 4-element block b: counter (b lo, b hi, stream lo, stream hi), key =
// seed; element 4b + j takes word j, u = (word >> 8) * 2^-24.
RO_DEV uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}
RO_DEV float u24(uint32_t w) { return __uint2float_rn(w >> 8) * 5.9604644775390625e-8f; }  // exact

// mode 0: uniform draws y = u; mode 1: dropout y = keep ? x * scale : +0 (+ mask);
// mode 2: dropout backward (x = dy)
template <int MODE>
__global__ void philox_kernel(const float *__restrict__ x, int64_t n, float p, uint2 key, uint64_t stream,
                              float *__restrict__ y, uint8_t *__restrict__ mask) {
    const int64_t nb = (n + 3) / 4;
    const float scale = __fdiv_rn(1.0f, __fsub_rn(1.0f, p));
    const bool vec = aligned16(y) && (MODE == 0 || aligned16(x)) &&
                     ((reinterpret_cast<uintptr_t>(mask) & 3u) == 0);
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        const uint4 w = philox4x32_10(make_uint4((uint32_t)b, (uint32_t)((uint64_t)b >> 32), (uint32_t)stream,
                                                 (uint32_t)(stream >> 32)), key);
        const float u[4] = {u24(w.x), u24(w.y), u24(w.z), u24(w.w)};
        const int64_t i0 = 4 * b;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        const bool full = i0 + 4 <= n;
        if (MODE != 0) {
            if (full && vec) {
                const float4 t = __ldg(reinterpret_cast<const float4 *>(x) + b);
                v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (i0 + j < n) v[j] = x[i0 + j];
            }
        }
        float r[4];
        uint8_t keep[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            keep[j] = u[j] >= p;
            r[j] = MODE == 0 ? u[j] : (keep[j] ? canon(__fmul_rn(v[j], scale)) : 0.0f);
        }
        if (full && vec) {
            reinterpret_cast<float4 *>(y)[b] = make_float4(r[0], r[1], r[2], r[3]);
            if (MODE == 1 && mask)
                reinterpret_cast<uchar4 *>(mask)[b] = make_uchar4(keep[0], keep[1], keep[2], keep[3]);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (i0 + j < n) {
                    y[i0 + j] = r[j];
                    if (MODE == 1 && mask) mask[i0 + j] = keep[j];
                }
        }
    }
}

// R30 lower-precision storage: widen exactly, narrow RN-even (cvt.rn), canonical NaNs.
// dtype codes: 1 = f32, 4 = bf16, 5 = f16.
RO_DEV float ld_lp(const void *p, int dt, int64_t i) {
    if (dt == 4) return __uint_as_float((uint32_t)reinterpret_cast<const uint16_t *>(p)[i] << 16);
    if (dt == 5) return __half2float(reinterpret_cast<const __half *>(p)[i]);
    return reinterpret_cast<const float *>(p)[i];
}
RO_DEV void st_lp(void *p, int dt, int64_t i, float v) {
    if (dt == 4) {
        const __nv_bfloat16 h = __float2bfloat16_rn(v);
        reinterpret_cast<uint16_t *>(p)[i] = (v != v) ? (uint16_t)0x7FC0u : *reinterpret_cast<const uint16_t *>(&h);
    } else if (dt == 5) {
        const __half h = __float2half_rn(v);
        reinterpret_cast<uint16_t *>(p)[i] = (v != v) ? (uint16_t)0x7E00u : __half_as_ushort(h);
    } else {
        reinterpret_cast<float *>(p)[i] = canon(v);
    }
}
template <int SDT, int DDT>
__global__ void convert_kernel(const void *__restrict__ src, int64_t rows, int64_t cols, int64_t lds,
                               void *__restrict__ dst, int64_t ldd) {
    const int64_t n = rows * cols;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = q / cols, c = q - r * cols;
        st_lp(dst, DDT, r * ldd + c, ld_lp(src, SDT, r * lds + c));
    }
}

// R24 (config-1 MLP): relu(x) = x > 0 ? x : +0; relu'(x) g = x > 0 ? g : +0; NaN x -> NaN
struct ReluF {
    RO_DEV float operator()(float x) const { return x != x ? canon(x) : (x > 0.f ? x : 0.f); }
};
struct ReluBwdF {
    RO_DEV float operator()(float x, float g) const { return x != x ? canon(x) : (x > 0.f ? canon(g) : 0.f); }
};
struct AddF { RO_DEV float operator()(float a, float b) const { return canon(__fadd_rn(a, b)); } };

// R-TREE_S: balanced pairwise tree over up to 16 parts, leaves are the parts themselves
struct Parts { const float *p[16]; };

template <int NP>
RO_DEV float tree_at(const Parts &ps, int64_t i) {
    float v[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) v[q] = __ldg(ps.p[q] + i);
#pragma unroll
    for (int w = 1; w < NP; w <<= 1)
#pragma unroll
        for (int q = 0; q < NP; q += 2 * w) v[q] = __fadd_rn(v[q], v[q + w]);
    return v[0];
}

template <int NP>
__global__ void tree_kernel(Parts ps, int64_t n, float *__restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    bool al = aligned16(out);
#pragma unroll
    for (int q = 0; q < NP; ++q) al = al && aligned16(ps.p[q]);
    const int64_t n4 = al ? n / 4 : 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 v[NP];
#pragma unroll
        for (int q = 0; q < NP; ++q) v[q] = __ldg(reinterpret_cast<const float4 *>(ps.p[q]) + i);
#pragma unroll
        for (int w = 1; w < NP; w <<= 1)
#pragma unroll
            for (int q = 0; q < NP; q += 2 * w) {
                v[q].x = __fadd_rn(v[q].x, v[q + w].x);
                v[q].y = __fadd_rn(v[q].y, v[q + w].y);
                v[q].z = __fadd_rn(v[q].z, v[q + w].z);
                v[q].w = __fadd_rn(v[q].w, v[q + w].w);
            }
        reinterpret_cast<float4 *>(out)[i] = make_float4(canon(v[0].x), canon(v[0].y), canon(v[0].z), canon(v[0].w));
    }
    for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = canon(tree_at<NP>(ps, i));
}

// R-ADAMW element chain (oracle: orc_adamw)
struct AdamHyper { float lr, b1, b2, eps, wd, bc1, bc2, omb1, omb2; int decay; };

RO_DEV void adam_elem(float &p, float g, float &m, float &v, const AdamHyper &h) {
    float mi = __fadd_rn(__fmul_rn(h.b1, m), __fmul_rn(h.omb1, g));
    float vi = __fadd_rn(__fmul_rn(h.b2, v), __fmul_rn(h.omb2, __fmul_rn(g, g)));
    float upd = __fdiv_rn(__fdiv_rn(mi, h.bc1), __fadd_rn(__fsqrt_rn(__fdiv_rn(vi, h.bc2)), h.eps));
    if (h.decay) upd = __fadd_rn(upd, __fmul_rn(h.wd, p));
    p = canon(__fsub_rn(p, __fmul_rn(h.lr, upd)));
    m = canon(mi);
    v = canon(vi);
}

__global__ void adamw_kernel(float *__restrict__ p, const float *__restrict__ g, float *__restrict__ m,
                             float *__restrict__ v, int64_t n, AdamHyper h) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const bool al = aligned16(p) && aligned16(g) && aligned16(m) && aligned16(v);
    const int64_t n4 = al ? n / 4 : 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 pp = reinterpret_cast<float4 *>(p)[i];
        float4 gg = __ldg(reinterpret_cast<const float4 *>(g) + i);
        float4 mm = reinterpret_cast<float4 *>(m)[i];
        float4 vv = reinterpret_cast<float4 *>(v)[i];
        adam_elem(pp.x, gg.x, mm.x, vv.x, h);
        adam_elem(pp.y, gg.y, mm.y, vv.y, h);
        adam_elem(pp.z, gg.z, mm.z, vv.z, h);
        adam_elem(pp.w, gg.w, mm.w, vv.w, h);
        reinterpret_cast<float4 *>(p)[i] = pp;
        reinterpret_cast<float4 *>(m)[i] = mm;
        reinterpret_cast<float4 *>(v)[i] = vv;
    }
    for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        float pp = p[i], mm = m[i], vv = v[i];
        adam_elem(pp, g[i], mm, vv, h);
        p[i] = pp;
        m[i] = mm;
        v[i] = vv;
    }
}

// AdamW over many parameter tensors stored back to back (one launch per step):
// element i belongs to segment k with start[k] <= i < start[k+1], whose decay flag
// selects the weight-decay term; the element chain is adam_elem (same bits as the
// per-tensor launch).
struct AdamSegs {
    int64_t start[ADAM_MAX_SEGS + 1];
    uint8_t decay[ADAM_MAX_SEGS];
    int n;
};

RO_DEV int adam_seg_of(const AdamSegs &s, int64_t i) {
    int lo = 0, hi = s.n;  // start[lo] <= i < start[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s.start[mid] <= i) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void adamw_seg_kernel(float *__restrict__ p, const float *__restrict__ g, float *__restrict__ m,
                                 float *__restrict__ v, int64_t n, AdamHyper h, AdamSegs segs) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const bool al = aligned16(p) && aligned16(g) && aligned16(m) && aligned16(v);
    const int64_t n4 = al ? n / 4 : 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 pp = reinterpret_cast<float4 *>(p)[i];
        float4 gg = __ldg(reinterpret_cast<const float4 *>(g) + i);
        float4 mm = reinterpret_cast<float4 *>(m)[i];
        float4 vv = reinterpret_cast<float4 *>(v)[i];
        const int k = adam_seg_of(segs, 4 * i);
        AdamHyper hk = h;
        hk.decay = segs.decay[k];
        if (4 * i + 3 < segs.start[k + 1]) {  // the usual case: all four in one tensor
            adam_elem(pp.x, gg.x, mm.x, vv.x, hk);
            adam_elem(pp.y, gg.y, mm.y, vv.y, hk);
            adam_elem(pp.z, gg.z, mm.z, vv.z, hk);
            adam_elem(pp.w, gg.w, mm.w, vv.w, hk);
        } else {
            float *pe = &pp.x, *me = &mm.x, *ve = &vv.x;
            const float *ge = &gg.x;
            for (int e = 0; e < 4; ++e) {
                hk.decay = segs.decay[adam_seg_of(segs, 4 * i + e)];
                adam_elem(pe[e], ge[e], me[e], ve[e], hk);
            }
        }
        reinterpret_cast<float4 *>(p)[i] = pp;
        reinterpret_cast<float4 *>(m)[i] = mm;
        reinterpret_cast<float4 *>(v)[i] = vv;
    }
    for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        float pp = p[i], mm = m[i], vv = v[i];
        AdamHyper hk = h;
        hk.decay = segs.decay[adam_seg_of(segs, i)];
        adam_elem(pp, g[i], mm, vv, hk);
        p[i] = pp;
        m[i] = mm;
        v[i] = vv;
    }
}

// R-EMB forward: x0[t][c] = wte[tok[t]][c] + wpe[t mod T][c]; one CTA-row per token
__global__ void embedding_kernel(const int32_t *__restrict__ tok, int64_t ntok, int64_t T,
                                 const float *__restrict__ wte, const float *__restrict__ wpe, int64_t C,
                                 float *__restrict__ x0) {
    int64_t t = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
    if (t >= ntok) return;
    const float *a = wte + (int64_t)__ldg(tok + t) * C;
    const float *b = wpe + (t % T) * C;
    float *o = x0 + t * C;
    for (int64_t c = threadIdx.x; c < C; c += blockDim.x) o[c] = canon(__fadd_rn(__ldg(a + c), __ldg(b + c)));
}

// R-EMB backward for one shard.  One CTA per token position u: if u is the
// first occurrence of its token, it folds dx0 over all positions t >= u with
// the same token, in ascending t, and adds the fold into dwte[token].
// Position rows of dwpe likewise (CTAs with u < T handle position u).
__global__ void embedding_bwd_kernel(const int32_t *__restrict__ tok, int64_t ntok, int64_t T,
                                     const float *__restrict__ dx0, int64_t C, float *__restrict__ dwte,
                                     float *__restrict__ dwpe) {
    // stok[0..ntok): the shard's tokens; occ[0..nocc): the positions holding token v, ascending
    extern __shared__ int32_t stok[];
    int32_t *occ = stok + ntok;
    __shared__ int nocc;
    const int64_t u = blockIdx.x;
    for (int64_t i = threadIdx.x; i < ntok; i += blockDim.x) stok[i] = __ldg(tok + i);
    __syncthreads();
    const int32_t v = stok[u];
    // position u owns vocabulary row v iff v does not occur before u (checked in parallel)
    int earlier = 0;
    for (int64_t i = threadIdx.x; i < u; i += blockDim.x) earlier |= (stok[i] == v);
    const bool first = !__syncthreads_or(earlier);
    if (first) {
        if (threadIdx.x < 32) {  // warp 0 lists the occurrences of v in ascending order
            int n = 0;
            for (int64_t b = u; b < ntok; b += 32) {
                const int64_t t = b + threadIdx.x;
                const unsigned m = __ballot_sync(0xffffffffu, t < ntok && stok[t] == v);
                if (t < ntok && stok[t] == v) occ[n + __popc(m & ((1u << threadIdx.x) - 1u))] = (int32_t)t;
                n += __popc(m);
            }
            if (threadIdx.x == 0) nocc = n;
        }
        __syncthreads();
        const int n = nocc;
        for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
            float acc = 0.f;  // R-SEQ over the shard's tokens equal to v, ascending
            for (int q = 0; q < n; ++q) acc = __fadd_rn(acc, __ldg(dx0 + (int64_t)occ[q] * C + c));
            float *o = dwte + (int64_t)v * C + c;
            *o = canon(__fadd_rn(*o, acc));
        }
    }
    if (dwpe && u < T) {
        for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
            float acc = 0.f;
            for (int64_t t = u; t < ntok; t += T) acc = __fadd_rn(acc, __ldg(dx0 + t * C + c));
            dwpe[u * C + c] = canon(acc);  // overwritten (position rows have no other producer)
        }
    }
}

__global__ void flip_bit_kernel(uint32_t *data, int64_t elem, int bit) { data[elem] ^= (1u << bit); }

int ew_grid(int64_t n) {
    int64_t blocks = (n / 4 + 255) / 256;
    int64_t cap = (int64_t)ro_host::num_sms() * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (int)blocks;
}

}  // namespace

template <class F>
static cudaError_t run_unary(const float *x, int64_t n, float *y, cudaStream_t s, F f) {
    if (n == 0) return cudaSuccess;
    unary_kernel<<<ew_grid(n), 256, 0, s>>>(x, n, y, f);
    return cudaGetLastError();
}

cudaError_t launch_exp(const float *x, int64_t n, float *y, cudaStream_t s) { return run_unary(x, n, y, s, ExpF{}); }
cudaError_t launch_log(const float *x, int64_t n, float *y, cudaStream_t s) { return run_unary(x, n, y, s, LogF{}); }
cudaError_t launch_tanh(const float *x, int64_t n, float *y, cudaStream_t s) { return run_unary(x, n, y, s, TanhF{}); }
cudaError_t launch_rsqrt(const float *x, int64_t n, float *y, cudaStream_t s) { return run_unary(x, n, y, s, RsqrtF{}); }
cudaError_t launch_gelu(const float *x, int64_t n, float *y, cudaStream_t s) { return run_unary(x, n, y, s, GeluF{}); }

cudaError_t launch_relu(const float *x, int64_t n, float *y, cudaStream_t s) { return run_unary(x, n, y, s, ReluF{}); }
cudaError_t launch_sin(const float *x, int64_t n, float *y, cudaStream_t s) { return run_unary(x, n, y, s, SinF{}); }
cudaError_t launch_cos(const float *x, int64_t n, float *y, cudaStream_t s) { return run_unary(x, n, y, s, CosF{}); }
cudaError_t launch_convert(const void *src, int sdt, int64_t rows, int64_t cols, int64_t lds, void *dst, int ddt,
                           int64_t ldd, cudaStream_t s) {
    const int64_t n = rows * cols;
    if (n == 0) return cudaSuccess;
    const int grid = ew_grid(n);
#define RO_CONV(a, b) \
    if (sdt == a && ddt == b) { convert_kernel<a, b><<<grid, 256, 0, s>>>(src, rows, cols, lds, dst, ldd); return cudaGetLastError(); }
    RO_CONV(1, 1) RO_CONV(1, 4) RO_CONV(1, 5) RO_CONV(4, 1) RO_CONV(4, 4) RO_CONV(4, 5) RO_CONV(5, 1) RO_CONV(5, 4)
    RO_CONV(5, 5)
#undef RO_CONV
    return cudaErrorInvalidValue;
}

static cudaError_t run_philox(int mode, const float *x, int64_t n, float p, uint64_t seed, uint64_t stream,
                              float *y, uint8_t *mask, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    const int grid = ew_grid((n + 3) / 4 * 4);
    if (mode == 0) philox_kernel<0><<<grid, 256, 0, s>>>(x, n, p, key, stream, y, mask);
    else if (mode == 1) philox_kernel<1><<<grid, 256, 0, s>>>(x, n, p, key, stream, y, mask);
    else philox_kernel<2><<<grid, 256, 0, s>>>(x, n, p, key, stream, y, mask);
    return cudaGetLastError();
}
cudaError_t launch_rand_uniform(uint64_t seed, uint64_t stream, int64_t n, float *y, cudaStream_t s) {
    return run_philox(0, nullptr, n, 0.0f, seed, stream, y, nullptr, s);
}
cudaError_t launch_dropout(const float *x, int64_t n, float p, uint64_t seed, uint64_t stream, float *y,
                           uint8_t *mask, cudaStream_t s) {
    return run_philox(1, x, n, p, seed, stream, y, mask, s);
}
cudaError_t launch_dropout_backward(const float *dy, int64_t n, float p, uint64_t seed, uint64_t stream, float *dx,
                                    cudaStream_t s) {
    return run_philox(2, dy, n, p, seed, stream, dx, nullptr, s);
}
cudaError_t launch_erf(const float *x, int64_t n, float *y, cudaStream_t s) { return run_unary(x, n, y, s, ErfF{}); }
cudaError_t launch_gelu_erf(const float *x, int64_t n, float *y, cudaStream_t s) {
    return run_unary(x, n, y, s, GeluErfF{});
}
cudaError_t launch_gelu_erf_backward(const float *x, const float *dy, int64_t n, float *dx, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    binary_kernel<<<ew_grid(n), 256, 0, s>>>(x, dy, n, dx, GeluErfBwdF{});
    return cudaGetLastError();
}
cudaError_t launch_rope_tables(const float *inv_freq, int64_t T, int64_t h, float *cosv, float *sinv, cudaStream_t s) {
    if (T * h == 0) return cudaSuccess;
    rope_tables_kernel<<<ew_grid(T * h), 256, 0, s>>>(inv_freq, T, h, cosv, sinv);
    return cudaGetLastError();
}

cudaError_t launch_relu_backward(const float *x, const float *g, int64_t n, float *dx, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    binary_kernel<<<ew_grid(n), 256, 0, s>>>(x, g, n, dx, ReluBwdF{});
    return cudaGetLastError();
}

cudaError_t launch_gelu_backward(const float *x, const float *dy, int64_t n, float *dx, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    binary_kernel<<<ew_grid(n), 256, 0, s>>>(x, dy, n, dx, GeluBwdF{});
    return cudaGetLastError();
}

cudaError_t launch_add(const float *a, const float *b, int64_t n, float *y, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    binary_kernel<<<ew_grid(n), 256, 0, s>>>(a, b, n, y, AddF{});
    return cudaGetLastError();
}

cudaError_t launch_tree_sum(const float *const *parts, int nparts, int64_t n, float *out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    Parts ps{};
    for (int q = 0; q < nparts; ++q) ps.p[q] = parts[q];
    int g = ew_grid(n * (nparts > 2 ? 1 : 1));
    switch (nparts) {
        case 1: tree_kernel<1><<<g, 256, 0, s>>>(ps, n, out); break;
        case 2: tree_kernel<2><<<g, 256, 0, s>>>(ps, n, out); break;
        case 4: tree_kernel<4><<<g, 256, 0, s>>>(ps, n, out); break;
        case 8: tree_kernel<8><<<g, 256, 0, s>>>(ps, n, out); break;
        case 16: tree_kernel<16><<<g, 256, 0, s>>>(ps, n, out); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_adamw(float *p, const float *g, float *m, float *v, int64_t n, float lr, float b1, float b2,
                         float eps, float wd, float bc1, float bc2, float omb1, float omb2, int decay,
                         cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    AdamHyper h{lr, b1, b2, eps, wd, bc1, bc2, omb1, omb2, decay};
    adamw_kernel<<<ew_grid(n), 256, 0, s>>>(p, g, m, v, n, h);
    return cudaGetLastError();
}

cudaError_t launch_adamw_segments(float *p, const float *g, float *m, float *v, int nseg, const int64_t *start,
                                  const uint8_t *decay, float lr, float b1, float b2, float eps, float wd, float bc1,
                                  float bc2, float omb1, float omb2, cudaStream_t s) {
    const int64_t n = start[nseg];
    if (n == 0) return cudaSuccess;
    AdamHyper h{lr, b1, b2, eps, wd, bc1, bc2, omb1, omb2, 0};
    AdamSegs segs{};
    for (int k = 0; k <= nseg; ++k) segs.start[k] = start[k];
    for (int k = 0; k < nseg; ++k) segs.decay[k] = decay[k] ? 1 : 0;
    segs.n = nseg;
    adamw_seg_kernel<<<ew_grid(n), 256, 0, s>>>(p, g, m, v, n, h, segs);
    return cudaGetLastError();
}

cudaError_t launch_embedding(const int32_t *tok, int64_t ntok, int64_t T, const float *wte, const float *wpe,
                             int64_t C, float *x0, cudaStream_t s) {
    if (ntok == 0) return cudaSuccess;
    dim3 block(128, 4);
    embedding_kernel<<<(unsigned)((ntok + 3) / 4), block, 0, s>>>(tok, ntok, T, wte, wpe, C, x0);
    return cudaGetLastError();
}

cudaError_t launch_embedding_backward(const int32_t *tok, int64_t ntok, int64_t T, const float *dx0, int64_t C,
                                      float *dwte, float *dwpe, cudaStream_t s) {
    if (ntok == 0) return cudaSuccess;
    size_t smem = (size_t)2 * ntok * sizeof(int32_t);  // tokens + the occurrence list
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(embedding_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    embedding_bwd_kernel<<<(unsigned)ntok, 256, smem, s>>>(tok, ntok, T, dx0, C, dwte, dwpe);
    return cudaGetLastError();
}

cudaError_t launch_flip_bit(void *data, int64_t elem, int bit, cudaStream_t s) {
    flip_bit_kernel<<<1, 1, 0, s>>>(reinterpret_cast<uint32_t *>(data), elem, bit);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ transpose (data movement only)
namespace {
__global__ void transpose_kernel(const float *__restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                                 float *__restrict__ y, int64_t ldy) {
    __shared__ float t[32][33];
    const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) t[i][threadIdx.x] = __ldg(x + r * ldx + c);
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) y[c * ldy + r] = t[threadIdx.x][i];
    }
}

// 64 x 64 tiles, 256 threads, 16-byte loads and stores (rows of x and y 16-byte
// aligned); ragged edges fall back to scalar accesses inside the same tile.
__global__ void __launch_bounds__(256) transpose64_kernel(const float *__restrict__ x, int64_t rows, int64_t cols,
                                                          int64_t ldx, float *__restrict__ y, int64_t ldy) {
    __shared__ float t[64][65];
    const int64_t c0 = (int64_t)blockIdx.x * 64, r0 = (int64_t)blockIdx.y * 64;
    const int tid = threadIdx.x;
    const bool full = r0 + 64 <= rows && c0 + 64 <= cols;
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // 64 rows x 16 float4
        const int i = (tid >> 4) + 16 * q, j = (tid & 15) * 4;
        const int64_t r = r0 + i, c = c0 + j;
        if (full) {
            const float4 v = __ldg(reinterpret_cast<const float4 *>(x + r * ldx + c));
            t[i][j] = v.x; t[i][j + 1] = v.y; t[i][j + 2] = v.z; t[i][j + 3] = v.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (r < rows && c + e < cols) t[i][j + e] = __ldg(x + r * ldx + c + e);
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // 64 output rows (= x columns) x 16 float4
        const int i = (tid >> 4) + 16 * q, j = (tid & 15) * 4;
        const int64_t c = c0 + i, r = r0 + j;
        if (full) {
            *reinterpret_cast<float4 *>(y + c * ldy + r) = make_float4(t[j][i], t[j + 1][i], t[j + 2][i], t[j + 3][i]);
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (c < cols && r + e < rows) y[c * ldy + r + e] = t[j + e][i];
        }
    }
}
}  // namespace

// ------------------------------------------------------------------ Llama operators (config 4)
namespace {
struct SwiGluF {
    // R-SWIGLU: silu(g) * u, silu(g) = g / (1 + exp(-g)); -g is an exact sign flip
    RO_DEV float operator()(float g, float u) const {
        float e = ro::exp_rn(__uint_as_float(__float_as_uint(g) ^ 0x80000000u));
        return ro::canon(__fmul_rn(__fdiv_rn(g, __fadd_rn(1.0f, e)), u));
    }
};

// R-ROPE, rotate-half form, one thread per (token, head, i < hd/2)
__global__ void rope_kernel(const float *__restrict__ x, int64_t ntok, int64_t nhead, int64_t hd, int64_t ld,
                            const float *__restrict__ cosv, const float *__restrict__ sinv, float *__restrict__ y,
                            int64_t ldy) {
    const int64_t h = hd / 2;
    const int64_t total = ntok * nhead * h;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx % h, q = (idx / h) % nhead, t = idx / (h * nhead);
        const float c = __ldg(cosv + t * h + i), s = __ldg(sinv + t * h + i);
        const float a = __ldg(x + t * ld + q * hd + i), b = __ldg(x + t * ld + q * hd + i + h);
        y[t * ldy + q * hd + i] = ro::canon(__fsub_rn(__fmul_rn(a, c), __fmul_rn(b, s)));
        y[t * ldy + q * hd + i + h] = ro::canon(__fadd_rn(__fmul_rn(b, c), __fmul_rn(a, s)));
    }
}

__global__ void gather_rows_kernel(const float *__restrict__ table, const int32_t *__restrict__ idx, int64_t n,
                                   int64_t C, float *__restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
    if (t >= n) return;
    const float *src = table + (int64_t)__ldg(idx + t) * C;
    for (int64_t c = threadIdx.x; c < C; c += blockDim.x) out[t * C + c] = __ldg(src + c);
}

// synthetic-input generator, bit-identical to synth.uniform: element i of stream
// `seed` = ((splitmix64(seed + (i+1)*golden) >> 40) * 2^-23 - 1) [* scale, rounded once]
__global__ void fill_uniform_kernel(float *__restrict__ out, int64_t n, uint64_t seed, double scale, int use_scale) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z = z ^ (z >> 31);
        const double u = (double)(z >> 40) * (1.0 / 8388608.0) - 1.0;  // exact
        const float f = (float)u;                                       // exact (24-bit grid)
        out[i] = use_scale ? (float)((double)f * scale) : f;
    }
}
}  // namespace

namespace {
// batch b of rows x cols: dst + b*sd <- src + b*ss (row strides lds / ldd); float4 when
// every row start is 16-byte aligned, else scalar.  Data movement only.
template <bool V4>
__global__ void copy2d_kernel(const float *__restrict__ src, int64_t rows, int64_t cols, int64_t lds, int64_t ss,
                              float *__restrict__ dst, int64_t ldd, int64_t sd) {
    const int64_t b = blockIdx.z;
    src += b * ss;
    dst += b * sd;
    const int64_t w = V4 ? cols / 4 : cols;
    const int64_t n = rows * w;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / w, c = i % w;
        if (V4)
            reinterpret_cast<float4 *>(dst + r * ldd)[c] = __ldg(reinterpret_cast<const float4 *>(src + r * lds) + c);
        else
            dst[r * ldd + c] = src[r * lds + c];
    }
}
}  // namespace

cudaError_t launch_copy2d_batched(const float *src, int64_t rows, int64_t cols, int64_t lds, int64_t ss, float *dst,
                                  int64_t ldd, int64_t sd, int64_t nb, cudaStream_t s) {
    if (rows == 0 || cols == 0 || nb == 0) return cudaSuccess;
    const bool v4 = ((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 16 == 0) && cols % 4 == 0 && lds % 4 == 0 &&
                    ldd % 4 == 0 && ss % 4 == 0 && sd % 4 == 0;
    const int64_t work = rows * (v4 ? cols / 4 : cols);
    const int64_t per = max((int64_t)1, (int64_t)ro_host::num_sms() * 8 / nb);
    dim3 grid((unsigned)max((int64_t)1, min((work + 255) / 256, per)), 1, (unsigned)nb);
    if (v4) copy2d_kernel<true><<<grid, 256, 0, s>>>(src, rows, cols, lds, ss, dst, ldd, sd);
    else copy2d_kernel<false><<<grid, 256, 0, s>>>(src, rows, cols, lds, ss, dst, ldd, sd);
    return cudaGetLastError();
}

cudaError_t launch_copy2d(const float *src, int64_t rows, int64_t cols, int64_t lds, float *dst, int64_t ldd,
                          cudaStream_t s) {
    return launch_copy2d_batched(src, rows, cols, lds, 0, dst, ldd, 0, 1, s);
}

cudaError_t launch_swiglu(const float *g, const float *u, int64_t n, float *h, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    binary_kernel<<<ew_grid(n), 256, 0, s>>>(g, u, n, h, SwiGluF{});
    return cudaGetLastError();
}

cudaError_t launch_rope(const float *x, int64_t ntok, int64_t nhead, int64_t hd, int64_t ld, const float *c,
                        const float *sn, float *y, int64_t ldy, cudaStream_t s) {
    const int64_t total = ntok * nhead * (hd / 2);
    if (total == 0) return cudaSuccess;
    rope_kernel<<<ew_grid(4 * total), 256, 0, s>>>(x, ntok, nhead, hd, ld, c, sn, y, ldy);
    return cudaGetLastError();
}

cudaError_t launch_gather_rows(const float *table, const int32_t *idx, int64_t n, int64_t C, float *out,
                               cudaStream_t s) {
    if (n == 0 || C == 0) return cudaSuccess;
    gather_rows_kernel<<<(unsigned)((n + 3) / 4), dim3(128, 4), 0, s>>>(table, idx, n, C, out);
    return cudaGetLastError();
}

cudaError_t launch_fill_uniform(float *out, int64_t n, uint64_t seed, double scale, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    fill_uniform_kernel<<<ew_grid(4 * n), 256, 0, s>>>(out, n, seed, scale, scale != 1.0);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ causal suffix flags (f4)
// flags[b][k][n], k = 0..K: bit 0 = some B[k'][n], k' >= k, is non-finite; bit 1 = every
// B[k'][n], k' >= k, has its sign bit set (row K: the empty suffix, bits = 2).  One CTA of
// 32 columns x 8 row segments: each thread folds its segment, the segment carries are
// combined from the bottom, then each thread writes its rows.  Integer logic only.
namespace {
__global__ void __launch_bounds__(256) causal_flags_kernel(const float *__restrict__ B, int64_t K, int64_t N,
                                                           int64_t ldb, int64_t sB0, int64_t sB1, int64_t b1n,
                                                           uint8_t *__restrict__ F, int64_t ldf, int64_t sF0,
                                                           int64_t sF1) {
    __shared__ uint8_t carry[8][32];
    const int cx = threadIdx.x & 31, sg = threadIdx.x >> 5;
    const int64_t n = (int64_t)blockIdx.x * 32 + cx;
    const int64_t bb0 = blockIdx.y / b1n, bb1 = blockIdx.y % b1n;
    const float *Bb = B + bb0 * sB0 + bb1 * sB1;
    uint8_t *Fb = F + bb0 * sF0 + bb1 * sF1;
    const int64_t seg = (K + 7) / 8;
    const int64_t k0 = min(K, sg * seg), k1 = min(K, k0 + seg);
    auto bits = [&](int64_t k) -> uint32_t {  // flag bits of the single element B[k][n]
        const uint32_t u = __float_as_uint(Bb[k * ldb + n]);
        return (((u & 0x7F800000u) == 0x7F800000u) ? 1u : 0u) | ((u >> 31) << 1);
    };
    uint32_t f = 2u;  // empty segment: nothing non-finite, all negative (vacuously)
    if (n < N)
        for (int64_t k = k1 - 1; k >= k0; --k) {
            const uint32_t e = bits(k);
            f = (f & 1u) | (e & 1u) | (f & e & 2u);
        }
    carry[sg][cx] = (uint8_t)f;
    __syncthreads();
    uint32_t c = 2u;  // suffix of the segments below this one
    for (int q = 7; q > sg; --q) c = (c & 1u) | (carry[q][cx] & 1u) | (c & carry[q][cx] & 2u);
    if (n >= N) return;
    if (sg == 7 || k1 == K) Fb[K * ldf + n] = 2u;
    f = c;
    for (int64_t k = k1 - 1; k >= k0; --k) {
        const uint32_t e = bits(k);
        f = (f & 1u) | (e & 1u) | (f & e & 2u);
        Fb[k * ldf + n] = (uint8_t)f;
    }
}
}  // namespace

cudaError_t launch_causal_flags(const float *B, int64_t K, int64_t N, int64_t ldb, int64_t sB0, int64_t sB1,
                                int64_t b0, int64_t b1, uint8_t *F, int64_t ldf, int64_t sF0, int64_t sF1,
                                cudaStream_t s) {
    if (N == 0 || b0 * b1 == 0) return cudaSuccess;
    dim3 grid((unsigned)((N + 31) / 32), (unsigned)(b0 * b1));
    causal_flags_kernel<<<grid, 256, 0, s>>>(B, K, N, ldb, sB0, sB1, b1, F, ldf, sF0, sF1);
    return cudaGetLastError();
}

cudaError_t launch_transpose(const float *x, int64_t rows, int64_t cols, int64_t ldx, float *y, int64_t ldy,
                             cudaStream_t s) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    const bool vec = ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0) && ldx % 4 == 0 && ldy % 4 == 0;
    if (vec && (rows + 63) / 64 <= 65535) {
        dim3 grid((unsigned)((cols + 63) / 64), (unsigned)((rows + 63) / 64));
        transpose64_kernel<<<grid, 256, 0, s>>>(x, rows, cols, ldx, y, ldy);
        return cudaGetLastError();
    }
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(x, rows, cols, ldx, y, ldy);
    return cudaGetLastError();
}
