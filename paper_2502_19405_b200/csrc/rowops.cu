// rowops.cu -- canonical row reductions and the row operators built on them:
// R-CSUM / R-CDOT (reading R4), softmax fwd/bwd (R7),
// LayerNorm fwd/bwd (R8), cross-entropy, token-axis R-SEQ folds.
//
// GPU mapping of R-CSUM: one warp owns a 4096-element tile; lane l owns slots
// 4l..4l+3 and reads elements b + 4l .. b + 4l + 3 (one float4) for b = 0,
// 128, 256, ... in ascending order, so every slot is folded in the canonical
// ascending order; TREE128 is a shuffle butterfly (common.cuh).  Rows longer
// than one tile give one warp per tile and a final warp CSUM over the tile
// results.  Everything that is order-free (max, elementwise math) is done in
// whatever order is fastest.
#include "common.cuh"
#include "rowops.cuh"

namespace {

using namespace ro;

// float4 read of elements i..i+3 of `row` (entries >= n are 0)
RO_DEV float4 ld4(const float *__restrict__ row, int64_t i, int64_t n, bool al) {
    // plain (coherent) loads: cross_entropy may write the row it reads (aliasing)
    if (al && i + 3 < n) return *reinterpret_cast<const float4 *>(row + i);
    float4 v;
    v.x = (i < n) ? row[i] : 0.f;
    v.y = (i + 1 < n) ? row[i + 1] : 0.f;
    v.z = (i + 2 < n) ? row[i + 2] : 0.f;
    v.w = (i + 3 < n) ? row[i + 3] : 0.f;
    return v;
}

RO_DEV float warp_max(float m) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL, m, off));
    return m;
}

// max over x[0..n) skipping NaN (fmaxf ignores a NaN operand); zero -> +0
RO_DEV float warp_row_max(const float *__restrict__ row, int64_t n, int lane, bool al) {
    float m = __uint_as_float(0xFF800000u);
    for (int64_t b = 0; b < n; b += 128) {
        int64_t i = b + 4 * lane;
        float4 v = ld4(row, i, n, al);
        if (i < n) m = fmaxf(m, v.x);
        if (i + 1 < n) m = fmaxf(m, v.y);
        if (i + 2 < n) m = fmaxf(m, v.z);
        if (i + 3 < n) m = fmaxf(m, v.w);
    }
    m = warp_max(m);
    return (m == 0.0f) ? 0.0f : m;
}

// Tile CSUM of exp(x_i - m) over row[t0 .. t0+n), n <= 4096.
RO_DEV float warp_expsum_tile(const float *__restrict__ row, int64_t t0, int64_t n, float m, int lane, bool al) {
    float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
    const float *x = row + t0;
    for (int64_t b = 0; b < n; b += 128) {
        int64_t i = b + 4 * lane;
        float4 v = ld4(x, i, n, al);
        if (i < n) p0 = __fadd_rn(p0, exp_rn(__fsub_rn(v.x, m)));
        if (i + 1 < n) p1 = __fadd_rn(p1, exp_rn(__fsub_rn(v.y, m)));
        if (i + 2 < n) p2 = __fadd_rn(p2, exp_rn(__fsub_rn(v.z, m)));
        if (i + 3 < n) p3 = __fadd_rn(p3, exp_rn(__fsub_rn(v.w, m)));
    }
    return tree128(p0, p1, p2, p3);
}

// Tile CDOT of u, v over [t0, t0+n), n <= 4096.
RO_DEV float warp_cdot_tile(const float *__restrict__ u, const float *__restrict__ v, int64_t n, int lane, bool al) {
    float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
    for (int64_t b = 0; b < n; b += 128) {
        int64_t i = b + 4 * lane;
        float4 a = ld4(u, i, n, al);
        float4 c = ld4(v, i, n, al);
        if (i < n) p0 = __fmaf_rn(a.x, c.x, p0);
        if (i + 1 < n) p1 = __fmaf_rn(a.y, c.y, p1);
        if (i + 2 < n) p2 = __fmaf_rn(a.z, c.z, p2);
        if (i + 3 < n) p3 = __fmaf_rn(a.w, c.w, p3);
    }
    return tree128(p0, p1, p2, p3);
}

RO_DEV bool al16(const float *p) { return aligned16(p); }

// ------------------------------------------------------------------ CSUM rows
__global__ void sum_rows_warp(const float *__restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                              float *__restrict__ out) {
    int lane = threadIdx.x & 31;
    int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= rows) return;
    const float *row = x + r * ld;
    float s = warp_csum_tile(row, (int)cols, lane);
    if (lane == 0) out[r] = canon(s);
}

// one CTA (8 warps) per row with cols > 4096
__global__ void sum_rows_cta(const float *__restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                             float *__restrict__ out) {
    extern __shared__ float tsum[];
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int64_t r = blockIdx.x;
    const float *row = x + r * ld;
    int64_t nt = (cols + TILE - 1) / TILE;
    for (int64_t t = w; t < nt; t += nw) {
        int64_t n = min((int64_t)TILE, cols - t * TILE);
        float s = warp_csum_tile(row + t * TILE, (int)n, lane);
        if (lane == 0) tsum[t] = s;
    }
    __syncthreads();
    if (w == 0) {
        float s = warp_csum_tile(tsum, (int)nt, lane);
        if (lane == 0) out[r] = canon(s);
    }
}

// ------------------------------------------------------------------ R-SEQ column folds
// A column fold is one sequential chain per (segment, column) -- the canonical
// order leaves no parallelism inside it -- so the kernel hides the load latency
// instead: a CTA owns FC = 32 columns of one segment; all 8 warps stream
// FR-row chunks of the [rows x 32] panel into shared memory with coalesced
// 128-byte row reads (double buffered), and warp 0's 32 lanes run the 32 folds
// out of shared memory (lane = column: conflict-free).
constexpr int FC = 32, FR = 64;  // panel columns, rows per double-buffered chunk

__global__ void __launch_bounds__(256) sum_cols_seq_kernel(const float *__restrict__ x, int64_t rows, int64_t cols,
                                                           int64_t ld, int64_t nseg, float *__restrict__ out,
                                                           int64_t ldo) {
    __shared__ float tile[2][FR][FC];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t j0 = (int64_t)blockIdx.x * FC;
    const int64_t s = blockIdx.y;
    const int64_t per = rows / nseg;
    const float *base = x + s * per * ld;
    const int64_t jl = j0 + lane;
    const int64_t nch = (per + FR - 1) / FR;
    auto load = [&](int buf, int64_t c) {
        float v[FR / 8];  // all loads of this warp in flight before the shared stores
#pragma unroll
        for (int q = 0; q < FR / 8; ++q) {
            const int64_t t = c * FR + w + 8 * q;
            v[q] = (t < per && jl < cols) ? __ldg(base + t * ld + jl) : 0.f;
        }
#pragma unroll
        for (int q = 0; q < FR / 8; ++q) tile[buf][w + 8 * q][lane] = v[q];
    };
    float acc = 0.f;
    if (nch > 0) load(0, 0);
    __syncthreads();
    for (int64_t c = 0; c < nch; ++c) {
        if (c + 1 < nch) load((int)((c + 1) & 1), c + 1);
        if (w == 0) {
            const int n = (int)min((int64_t)FR, per - c * FR);
            const float(*tb)[FC] = tile[c & 1];
#pragma unroll 8
            for (int r = 0; r < n; ++r) acc = __fadd_rn(acc, tb[r][lane]);  // ascending rows
        }
        __syncthreads();
    }
    if (w == 0 && jl < cols) out[s * ldo + jl] = canon(acc);
}

// ------------------------------------------------------------------ softmax
// warp per row, row length <= 4096 (one CSUM tile)
__global__ void softmax_warp(const float *__restrict__ x, int64_t rows, int64_t cols, int64_t ldx, int causal,
                             float *__restrict__ y, int64_t ldy) {
    int lane = threadIdx.x & 31;
    int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= rows) return;
    const float *xr = x + r * ldx;
    float *yr = y + r * ldy;
    const int64_t L = causal ? (r % cols) + 1 : cols;
    const bool al = al16(xr);
    float m = warp_row_max(xr, L, lane, al);
    float s = warp_expsum_tile(xr, 0, L, m, lane, al);
    float rinv = __fdiv_rn(1.0f, s);
    const bool aly = al16(yr);
    for (int64_t b = 0; b < cols; b += 128) {
        int64_t i = b + 4 * lane;
        float4 v = ld4(xr, i, L, al);
        float o[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) o[c] = (i + c < L) ? canon(__fmul_rn(exp_rn(__fsub_rn(o[c], m)), rinv)) : 0.0f;
        if (aly && i + 3 < cols) {
            *reinterpret_cast<float4 *>(yr + i) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (i + c < cols) yr[i + c] = o[c];
        }
    }
}

// warp per row, row length <= 128 * NQ, row held in registers: one global read, exp
// computed once (the same e_i feed the slot sums and the outputs), one global write.
// Lane l owns elements b + 4l .. b + 4l + 3 for b = 0, 128, ... exactly as
// softmax_warp, so the max, the 128-slot CSUM order and every output bit are identical.
template <int NQ>
__global__ void softmax_warp_reg(const float *__restrict__ x, int64_t rows, int64_t cols, int64_t ldx, int causal,
                                 float *__restrict__ y, int64_t ldy) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= rows) return;
    const float *xr = x + r * ldx;
    float *yr = y + r * ldy;
    const int64_t L = causal ? (r % cols) + 1 : cols;
    const bool al = al16(xr);
    float v[NQ][4];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int64_t i = 128 * q + 4 * lane;
        if (128 * q < L) {  // warp-uniform: chunks past the valid length are never read
            const float4 t = ld4(xr, i, L, al);
            v[q][0] = t.x; v[q][1] = t.y; v[q][2] = t.z; v[q][3] = t.w;
        } else {
            v[q][0] = v[q][1] = v[q][2] = v[q][3] = 0.f;
        }
    }
    float m = __uint_as_float(0xFF800000u);
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (128 * q + 4 * lane + c < L) m = fmaxf(m, v[q][c]);
    m = warp_max(m);
    m = (m == 0.0f) ? 0.0f : m;
    float p[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (128 * q + 4 * lane + c < L) {
                v[q][c] = exp_rn(__fsub_rn(v[q][c], m));
                p[c] = __fadd_rn(p[c], v[q][c]);
            }
    const float rinv = __fdiv_rn(1.0f, tree128(p[0], p[1], p[2], p[3]));
    const bool aly = al16(yr);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int64_t i = 128 * q + 4 * lane;
        if (128 * q >= cols) break;
        float o[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) o[c] = (i + c < L) ? canon(__fmul_rn(v[q][c], rinv)) : 0.0f;
        if (aly && i + 3 < cols) {
            *reinterpret_cast<float4 *>(yr + i) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (i + c < cols) yr[i + c] = o[c];
        }
    }
}

// CTA per row (cols > 4096): tiles of 4096 per warp, CSUM over tile sums
__global__ void softmax_cta(const float *__restrict__ x, int64_t rows, int64_t cols, int64_t ldx, int causal,
                            float *__restrict__ y, int64_t ldy) {
    extern __shared__ float sm[];  // [nt] tile sums, then [32] scratch
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int64_t r = blockIdx.x;
    const float *xr = x + r * ldx;
    float *yr = y + r * ldy;
    const int64_t L = causal ? (r % cols) + 1 : cols;
    const int64_t nt = (L + TILE - 1) / TILE;
    float *scratch = sm + ((nt + 3) & ~3);
    const bool al = al16(xr);
    // max: each warp over its tiles, then across warps
    float m = __uint_as_float(0xFF800000u);
    for (int64_t t = w; t < nt; t += nw) {
        int64_t n = min((int64_t)TILE, L - t * TILE);
        m = fmaxf(m, warp_row_max(xr + t * TILE, n, lane, al));
    }
    if (lane == 0) scratch[w] = m;
    __syncthreads();
    m = (lane < nw) ? scratch[lane] : __uint_as_float(0xFF800000u);
    m = warp_max(m);
    m = (m == 0.0f) ? 0.0f : m;
    for (int64_t t = w; t < nt; t += nw) {
        int64_t n = min((int64_t)TILE, L - t * TILE);
        float s = warp_expsum_tile(xr, t * TILE, n, m, lane, al);
        if (lane == 0) sm[t] = s;
    }
    __syncthreads();
    float s;
    if (nt == 1) s = sm[0];
    else s = warp_csum_tile(sm, (int)nt, lane);  // every warp computes the same value
    float rinv = __fdiv_rn(1.0f, s);
    for (int64_t i = threadIdx.x; i < cols; i += blockDim.x)
        yr[i] = (i < L) ? canon(__fmul_rn(exp_rn(__fsub_rn(__ldg(xr + i), m)), rinv)) : 0.0f;
}

// backward: c = CDOT(y, dy) over cols; dx = (y*(dy - c))*scale
__global__ void softmax_bwd_warp(const float *__restrict__ y, int64_t ldy, const float *__restrict__ dy,
                                 int64_t lddy, int64_t rows, int64_t cols, float scale, float *dx, int64_t lddx) {
    int lane = threadIdx.x & 31;
    int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= rows) return;
    const float *yr = y + r * ldy;
    const float *gr = dy + r * lddy;
    float *dr = dx + r * lddx;
    const bool al = al16(yr) && al16(gr);
    float c = warp_cdot_tile(yr, gr, cols, lane, al);
    const bool ald = al16(dr);
    for (int64_t b = 0; b < cols; b += 128) {
        int64_t i = b + 4 * lane;
        float4 a = ld4(yr, i, cols, al);
        float4 g = ld4(gr, i, cols, al);
        float o[4];
        o[0] = canon(__fmul_rn(__fmul_rn(a.x, __fsub_rn(g.x, c)), scale));
        o[1] = canon(__fmul_rn(__fmul_rn(a.y, __fsub_rn(g.y, c)), scale));
        o[2] = canon(__fmul_rn(__fmul_rn(a.z, __fsub_rn(g.z, c)), scale));
        o[3] = canon(__fmul_rn(__fmul_rn(a.w, __fsub_rn(g.w, c)), scale));
        if (ald && i + 3 < cols) {
            *reinterpret_cast<float4 *>(dr + i) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (i + q < cols) dr[i + q] = o[q];
        }
    }
}

__global__ void softmax_bwd_cta(const float *__restrict__ y, int64_t ldy, const float *__restrict__ dy,
                                int64_t lddy, int64_t rows, int64_t cols, float scale, float *dx, int64_t lddx) {
    extern __shared__ float sm[];
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int64_t r = blockIdx.x;
    const float *yr = y + r * ldy;
    const float *gr = dy + r * lddy;
    float *dr = dx + r * lddx;
    const bool al = al16(yr) && al16(gr);
    const int64_t nt = (cols + TILE - 1) / TILE;
    for (int64_t t = w; t < nt; t += nw) {
        int64_t n = min((int64_t)TILE, cols - t * TILE);
        float s = warp_cdot_tile(yr + t * TILE, gr + t * TILE, n, lane, al);
        if (lane == 0) sm[t] = s;
    }
    __syncthreads();
    float c = (nt == 1) ? sm[0] : warp_csum_tile(sm, (int)nt, lane);
    __syncthreads();
    for (int64_t i = threadIdx.x; i < cols; i += blockDim.x)
        dr[i] = canon(__fmul_rn(__fmul_rn(__ldg(yr + i), __fsub_rn(__ldg(gr + i), c)), scale));
}

// ------------------------------------------------------------------ LayerNorm (cols <= 4096)
__global__ void layernorm_warp(const float *__restrict__ x, const float *__restrict__ gamma,
                               const float *__restrict__ beta, int64_t rows, int64_t cols, float eps,
                               float *__restrict__ y, float *__restrict__ mean, float *__restrict__ rstd) {
    int lane = threadIdx.x & 31;
    int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= rows) return;
    const float *xr = x + r * cols;
    float *yr = y + r * cols;
    const bool al = al16(xr) && al16(gamma) && al16(beta) && al16(yr);
    const float n = (float)cols;
    float mu = __fdiv_rn(warp_csum_tile(xr, (int)cols, lane), n);
    // var = CDOT(d, d) / n with d_i = x_i - mu
    float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
    for (int64_t b = 0; b < cols; b += 128) {
        int64_t i = b + 4 * lane;
        float4 v = ld4(xr, i, cols, al);
        float d0 = __fsub_rn(v.x, mu), d1 = __fsub_rn(v.y, mu), d2 = __fsub_rn(v.z, mu), d3 = __fsub_rn(v.w, mu);
        if (i < cols) p0 = __fmaf_rn(d0, d0, p0);
        if (i + 1 < cols) p1 = __fmaf_rn(d1, d1, p1);
        if (i + 2 < cols) p2 = __fmaf_rn(d2, d2, p2);
        if (i + 3 < cols) p3 = __fmaf_rn(d3, d3, p3);
    }
    float var = __fdiv_rn(tree128(p0, p1, p2, p3), n);
    float rs = rsqrt_rn(__fadd_rn(var, eps));
    for (int64_t b = 0; b < cols; b += 128) {
        int64_t i = b + 4 * lane;
        float4 v = ld4(xr, i, cols, al);
        float4 g = ld4(gamma, i, cols, al);
        float4 be = ld4(beta, i, cols, al);
        float o[4];
        o[0] = canon(__fmaf_rn(__fmul_rn(__fsub_rn(v.x, mu), rs), g.x, be.x));
        o[1] = canon(__fmaf_rn(__fmul_rn(__fsub_rn(v.y, mu), rs), g.y, be.y));
        o[2] = canon(__fmaf_rn(__fmul_rn(__fsub_rn(v.z, mu), rs), g.z, be.z));
        o[3] = canon(__fmaf_rn(__fmul_rn(__fsub_rn(v.w, mu), rs), g.w, be.w));
        if (al && i + 3 < cols) {
            *reinterpret_cast<float4 *>(yr + i) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (i + q < cols) yr[i + q] = o[q];
        }
    }
    if (lane == 0) {
        if (mean) mean[r] = canon(mu);
        if (rstd) rstd[r] = canon(rs);
    }
}

// R-RMSNORM (cols <= 4096): ms = CDOT(x,x)/n; rstd = 1/sqrt(ms+eps); y = (x*rstd)*w
__global__ void rmsnorm_warp(const float *__restrict__ x, const float *__restrict__ w, int64_t rows, int64_t cols,
                             float eps, float *__restrict__ y, float *__restrict__ rstd) {
    int lane = threadIdx.x & 31;
    int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= rows) return;
    const float *xr = x + r * cols;
    float *yr = y + r * cols;
    const bool al = al16(xr) && al16(w) && al16(yr);
    const float ms = __fdiv_rn(warp_cdot_tile(xr, xr, cols, lane, al), (float)cols);
    const float rs = rsqrt_rn(__fadd_rn(ms, eps));
    for (int64_t b = 0; b < cols; b += 128) {
        int64_t i = b + 4 * lane;
        float4 v = ld4(xr, i, cols, al);
        float4 g = ld4(w, i, cols, al);
        float o[4] = {canon(__fmul_rn(__fmul_rn(v.x, rs), g.x)), canon(__fmul_rn(__fmul_rn(v.y, rs), g.y)),
                      canon(__fmul_rn(__fmul_rn(v.z, rs), g.z)), canon(__fmul_rn(__fmul_rn(v.w, rs), g.w))};
        if (al && i + 3 < cols) {
            *reinterpret_cast<float4 *>(yr + i) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (i + q < cols) yr[i + q] = o[q];
        }
    }
    if (lane == 0 && rstd) rstd[r] = canon(rs);
}

__global__ void layernorm_bwd_warp(const float *__restrict__ dy, const float *__restrict__ x,
                                   const float *__restrict__ gamma, const float *__restrict__ mean,
                                   const float *__restrict__ rstd, const float *__restrict__ dres, int64_t rows,
                                   int64_t cols, float *__restrict__ dx) {
    int lane = threadIdx.x & 31;
    int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= rows) return;
    const float *xr = x + r * cols;
    const float *gr = dy + r * cols;
    float *dr = dx + r * cols;
    const float *rr = dres ? dres + r * cols : nullptr;
    const bool al = al16(xr) && al16(gr) && al16(gamma) && al16(dr) && (!rr || al16(rr));
    const float n = (float)cols;
    const float mu = __ldg(mean + r), rs = __ldg(rstd + r);
    // a = CSUM(g)/n, b = CDOT(g, xh)/n, g = dy*gamma, xh = (x - mu)*rstd
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f, q0 = 0.f, q1 = 0.f, q2 = 0.f, q3 = 0.f;
    for (int64_t b = 0; b < cols; b += 128) {
        int64_t i = b + 4 * lane;
        float4 v = ld4(xr, i, cols, al);
        float4 d = ld4(gr, i, cols, al);
        float4 gm = ld4(gamma, i, cols, al);
        float g0 = __fmul_rn(d.x, gm.x), g1 = __fmul_rn(d.y, gm.y), g2 = __fmul_rn(d.z, gm.z), g3 = __fmul_rn(d.w, gm.w);
        float h0 = __fmul_rn(__fsub_rn(v.x, mu), rs), h1 = __fmul_rn(__fsub_rn(v.y, mu), rs);
        float h2 = __fmul_rn(__fsub_rn(v.z, mu), rs), h3 = __fmul_rn(__fsub_rn(v.w, mu), rs);
        if (i < cols) { s0 = __fadd_rn(s0, g0); q0 = __fmaf_rn(g0, h0, q0); }
        if (i + 1 < cols) { s1 = __fadd_rn(s1, g1); q1 = __fmaf_rn(g1, h1, q1); }
        if (i + 2 < cols) { s2 = __fadd_rn(s2, g2); q2 = __fmaf_rn(g2, h2, q2); }
        if (i + 3 < cols) { s3 = __fadd_rn(s3, g3); q3 = __fmaf_rn(g3, h3, q3); }
    }
    const float a = __fdiv_rn(tree128(s0, s1, s2, s3), n);
    const float bb = __fdiv_rn(tree128(q0, q1, q2, q3), n);
    for (int64_t b = 0; b < cols; b += 128) {
        int64_t i = b + 4 * lane;
        float4 v = ld4(xr, i, cols, al);
        float4 d = ld4(gr, i, cols, al);
        float4 gm = ld4(gamma, i, cols, al);
        float4 re = rr ? ld4(rr, i, cols, al) : make_float4(0.f, 0.f, 0.f, 0.f);
        float xv[4] = {v.x, v.y, v.z, v.w}, dv[4] = {d.x, d.y, d.z, d.w}, gv[4] = {gm.x, gm.y, gm.z, gm.w};
        float rv[4] = {re.x, re.y, re.z, re.w}, o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float g = __fmul_rn(dv[q], gv[q]);
            float xh = __fmul_rn(__fsub_rn(xv[q], mu), rs);
            float val = __fmul_rn(__fsub_rn(__fsub_rn(g, a), __fmul_rn(xh, bb)), rs);
            if (rr) val = __fadd_rn(rv[q], val);
            o[q] = canon(val);
        }
        if (al && i + 3 < cols) {
            *reinterpret_cast<float4 *>(dr + i) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (i + q < cols) dr[i + q] = o[q];
        }
    }
}

__global__ void layernorm_params_kernel(const float *__restrict__ dy, const float *__restrict__ x,
                                        const float *__restrict__ mean, const float *__restrict__ rstd,
                                        int64_t rows, int64_t cols, int64_t nseg, float *__restrict__ dgamma,
                                        float *__restrict__ dbeta, int64_t ldo) {
    // same panel-streaming structure as sum_cols_seq_kernel; the folded value
    // xh = (x - mean[t]) * rstd[t] is recomputed exactly as in the forward
    __shared__ float tdy[2][FR][FC], txh[2][FR][FC];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t j0 = (int64_t)blockIdx.x * FC;
    const int64_t s = blockIdx.y;
    const int64_t per = rows / nseg;
    const int64_t jl = j0 + lane;
    const int64_t nch = (per + FR - 1) / FR;
    auto load = [&](int buf, int64_t c) {
        float vd[FR / 8], vx[FR / 8], vm[FR / 8], vr[FR / 8];  // every load in flight first
#pragma unroll
        for (int q = 0; q < FR / 8; ++q) {
            const int r = w + 8 * q;
            const int64_t t = s * per + c * FR + r;
            const bool ok = (c * FR + r < per) && jl < cols;
            vd[q] = ok ? __ldg(dy + t * cols + jl) : 0.f;
            vx[q] = ok ? __ldg(x + t * cols + jl) : 0.f;
            vm[q] = ok ? __ldg(mean + t) : 0.f;
            vr[q] = ok ? __ldg(rstd + t) : 0.f;
        }
#pragma unroll
        for (int q = 0; q < FR / 8; ++q) {
            const int r = w + 8 * q;
            const bool ok = (c * FR + r < per) && jl < cols;
            tdy[buf][r][lane] = vd[q];
            txh[buf][r][lane] = ok ? __fmul_rn(__fsub_rn(vx[q], vm[q]), vr[q]) : 0.f;
        }
    };
    float ag = 0.f, ab = 0.f;
    if (nch > 0) load(0, 0);
    __syncthreads();
    for (int64_t c = 0; c < nch; ++c) {
        if (c + 1 < nch) load((int)((c + 1) & 1), c + 1);
        if (w == 0) {
            const int n = (int)min((int64_t)FR, per - c * FR);
            const int b = (int)(c & 1);
#pragma unroll 8
            for (int r = 0; r < n; ++r) {  // ascending rows of the segment
                const float d = tdy[b][r][lane];
                ag = __fmaf_rn(d, txh[b][r][lane], ag);
                ab = __fadd_rn(ab, d);
            }
        }
        __syncthreads();
    }
    if (w == 0 && jl < cols) {
        dgamma[s * ldo + jl] = canon(ag);
        dbeta[s * ldo + jl] = canon(ab);
    }
}

// ------------------------------------------------------------------ cross entropy (CTA per row)
__global__ void cross_entropy_cta(const float *logits, int64_t rows, int64_t V, int64_t ld,
                                  const int32_t *__restrict__ labels, float scale, float *__restrict__ loss,
                                  float *dlogits, int64_t ldd) {
    extern __shared__ float sm[];
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int64_t r = blockIdx.x;
    const float *xr = logits + r * ld;
    const int64_t nt = (V + TILE - 1) / TILE;
    float *scratch = sm + ((nt + 3) & ~3);
    const bool al = al16(xr);
    float m = __uint_as_float(0xFF800000u);
    for (int64_t t = w; t < nt; t += nw) {
        int64_t n = min((int64_t)TILE, V - t * TILE);
        m = fmaxf(m, warp_row_max(xr + t * TILE, n, lane, al));
    }
    if (lane == 0) scratch[w] = m;
    __syncthreads();
    m = (lane < nw) ? scratch[lane] : __uint_as_float(0xFF800000u);
    m = warp_max(m);
    m = (m == 0.0f) ? 0.0f : m;
    for (int64_t t = w; t < nt; t += nw) {
        int64_t n = min((int64_t)TILE, V - t * TILE);
        float s = warp_expsum_tile(xr, t * TILE, n, m, lane, al);
        if (lane == 0) sm[t] = s;
    }
    __syncthreads();
    const float s = (nt == 1) ? sm[0] : warp_csum_tile(sm, (int)nt, lane);
    const int32_t lab = __ldg(labels + r);
    const float xl = xr[lab];
    if (loss && threadIdx.x == 0) loss[r] = canon(__fsub_rn(__fadd_rn(m, log_rn(s)), xl));
    if (dlogits) {
        __syncthreads();  // all reads of the row above happen before any aliased write
        const float rinv = __fdiv_rn(1.0f, s);
        float *dr = dlogits + r * ldd;
        for (int64_t i = threadIdx.x; i < V; i += blockDim.x) {
            float p = __fmul_rn(exp_rn(__fsub_rn(xr[i], m)), rinv);
            float d = __fsub_rn(p, (i == lab) ? 1.0f : 0.0f);
            dr[i] = canon(__fmul_rn(d, scale));
        }
    }
}

// Cross entropy with the whole row staged in shared memory (V <= CE_SMEM_MAX): one HBM
// read of the logits (cp.async), exp computed once and kept in shared memory for the
// gradient; the max, the per-tile 128-slot CSUMs, the CSUM over tile sums and every
// output operation are those of cross_entropy_cta, so the bits are identical.
constexpr int CE_THREADS = 1024;

__global__ void __launch_bounds__(CE_THREADS, 1) cross_entropy_smem(
    const float *logits, int64_t rows, int64_t V, int64_t ld, const int32_t *__restrict__ labels, float scale,
    float *__restrict__ loss, float *dlogits, int64_t ldd) {
    extern __shared__ __align__(16) float sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = CE_THREADS / 32;
    const int64_t r = blockIdx.x;
    const float *xr = logits + r * ld;
    const int Vi = (int)V, V4 = Vi & ~3, Vp = (Vi + 3) & ~3;
    const int nt = (Vi + TILE - 1) / TILE;
    float *row = sm;
    float *tsum = sm + Vp;
    float *scratch = tsum + ((nt + 3) & ~3);
    for (int i = 4 * threadIdx.x; i < V4; i += 4 * CE_THREADS) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(row + i);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(xr + i));
    }
    asm volatile("cp.async.commit_group;\n" ::);
    for (int i = V4 + threadIdx.x; i < Vp; i += CE_THREADS) row[i] = (i < Vi) ? xr[i] : 0.f;
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    // max over the row (order-free; NaN ignored, zero -> +0 as in cross_entropy_cta)
    float m = __uint_as_float(0xFF800000u);
    for (int i = threadIdx.x; i < Vi; i += CE_THREADS) m = fmaxf(m, row[i]);
    m = warp_max(m);
    if (lane == 0) scratch[w] = m;
    __syncthreads();
    m = (lane < nw) ? scratch[lane] : __uint_as_float(0xFF800000u);
    m = warp_max(m);
    m = (m == 0.0f) ? 0.0f : m;
    // per-tile CSUM of e = exp(x - m) (warp_expsum_tile's slot order); e kept in place
    for (int t = w; t < nt; t += nw) {
        const int t0 = t * TILE, n = min(TILE, Vi - t0);
        float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
        for (int b = 0; b < n; b += 128) {
            const int i = b + 4 * lane;
            if (i >= n) continue;  // (i < n implies i + 3 < Vp: the float4 stays in the row)
            float4 v = *reinterpret_cast<const float4 *>(row + t0 + i);
            { v.x = exp_rn(__fsub_rn(v.x, m)); p0 = __fadd_rn(p0, v.x); }
            if (i + 1 < n) { v.y = exp_rn(__fsub_rn(v.y, m)); p1 = __fadd_rn(p1, v.y); }
            if (i + 2 < n) { v.z = exp_rn(__fsub_rn(v.z, m)); p2 = __fadd_rn(p2, v.z); }
            if (i + 3 < n) { v.w = exp_rn(__fsub_rn(v.w, m)); p3 = __fadd_rn(p3, v.w); }
            *reinterpret_cast<float4 *>(row + t0 + i) = v;
        }
        const float ts = tree128(p0, p1, p2, p3);
        if (lane == 0) tsum[t] = ts;
    }
    __syncthreads();
    const float s = (nt == 1) ? tsum[0] : warp_csum_tile(tsum, nt, lane);
    const int32_t lab = __ldg(labels + r);
    const float xl = xr[lab];
    if (loss && threadIdx.x == 0) loss[r] = canon(__fsub_rn(__fadd_rn(m, log_rn(s)), xl));
    if (dlogits) {
        __syncthreads();  // every read of the global row (xl) before an aliased write
        const float rinv = __fdiv_rn(1.0f, s);
        float *dr = dlogits + r * ldd;
        for (int i = threadIdx.x; i < Vi; i += CE_THREADS) {
            const float p = __fmul_rn(row[i], rinv);
            const float d = __fsub_rn(p, (i == lab) ? 1.0f : 0.0f);
            dr[i] = canon(__fmul_rn(d, scale));
        }
    }
}

}  // namespace

// ------------------------------------------------------------------ launchers
static int rows_grid(int64_t rows, int warps_per_block) {
    return (int)((rows + warps_per_block - 1) / warps_per_block);
}

cudaError_t launch_sum_rows(const float *x, int64_t rows, int64_t cols, int64_t ld, float *out, cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    if (cols <= TILE_ELEMS) sum_rows_warp<<<rows_grid(rows, 8), 256, 0, s>>>(x, rows, cols, ld, out);
    else {
        size_t nt = (size_t)((cols + TILE_ELEMS - 1) / TILE_ELEMS);
        sum_rows_cta<<<(unsigned)rows, 256, nt * sizeof(float), s>>>(x, rows, cols, ld, out);
    }
    return cudaGetLastError();
}

cudaError_t launch_sum_cols_seq(const float *x, int64_t rows, int64_t cols, int64_t ld, int64_t nseg, float *out,
                                int64_t ldo, cudaStream_t s) {
    if (cols == 0 || nseg == 0) return cudaSuccess;
    dim3 grid((unsigned)((cols + FC - 1) / FC), (unsigned)nseg);
    sum_cols_seq_kernel<<<grid, 256, 0, s>>>(x, rows, cols, ld, nseg, out, ldo);
    return cudaGetLastError();
}

cudaError_t launch_softmax(const float *x, int64_t rows, int64_t cols, int64_t ldx, int causal, float *y,
                           int64_t ldy, cudaStream_t s) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    if (cols <= 512)
        softmax_warp_reg<4><<<rows_grid(rows, 8), 256, 0, s>>>(x, rows, cols, ldx, causal, y, ldy);
    else if (cols <= 1024)
        softmax_warp_reg<8><<<rows_grid(rows, 8), 256, 0, s>>>(x, rows, cols, ldx, causal, y, ldy);
    else if (cols <= TILE_ELEMS) softmax_warp<<<rows_grid(rows, 8), 256, 0, s>>>(x, rows, cols, ldx, causal, y, ldy);
    else {
        size_t nt = (size_t)((cols + TILE_ELEMS - 1) / TILE_ELEMS);
        softmax_cta<<<(unsigned)rows, 512, (((nt + 3) & ~3ull) + 32) * sizeof(float), s>>>(x, rows, cols, ldx,
                                                                                          causal, y, ldy);
    }
    return cudaGetLastError();
}

cudaError_t launch_softmax_backward(const float *y, int64_t ldy, const float *dy, int64_t lddy, int64_t rows,
                                    int64_t cols, float scale, float *dx, int64_t lddx, cudaStream_t s) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    if (cols <= TILE_ELEMS)
        softmax_bwd_warp<<<rows_grid(rows, 8), 256, 0, s>>>(y, ldy, dy, lddy, rows, cols, scale, dx, lddx);
    else {
        size_t nt = (size_t)((cols + TILE_ELEMS - 1) / TILE_ELEMS);
        softmax_bwd_cta<<<(unsigned)rows, 512, nt * sizeof(float), s>>>(y, ldy, dy, lddy, rows, cols, scale, dx,
                                                                       lddx);
    }
    return cudaGetLastError();
}

cudaError_t launch_layernorm(const float *x, const float *g, const float *b, int64_t rows, int64_t cols, float eps,
                             float *y, float *mean, float *rstd, cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    layernorm_warp<<<rows_grid(rows, 8), 256, 0, s>>>(x, g, b, rows, cols, eps, y, mean, rstd);
    return cudaGetLastError();
}

cudaError_t launch_layernorm_backward(const float *dy, const float *x, const float *g, const float *mean,
                                      const float *rstd, const float *dres, int64_t rows, int64_t cols, float *dx,
                                      cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    layernorm_bwd_warp<<<rows_grid(rows, 8), 256, 0, s>>>(dy, x, g, mean, rstd, dres, rows, cols, dx);
    return cudaGetLastError();
}

cudaError_t launch_layernorm_params(const float *dy, const float *x, const float *mean, const float *rstd,
                                    int64_t rows, int64_t cols, int64_t nseg, float *dg, float *db, int64_t ldo,
                                    cudaStream_t s) {
    if (cols == 0 || nseg == 0) return cudaSuccess;
    dim3 grid((unsigned)((cols + FC - 1) / FC), (unsigned)nseg);
    layernorm_params_kernel<<<grid, 256, 0, s>>>(dy, x, mean, rstd, rows, cols, nseg, dg, db, ldo);
    return cudaGetLastError();
}

cudaError_t launch_rmsnorm(const float *x, const float *w, int64_t rows, int64_t cols, float eps, float *y,
                           float *rstd, cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    rmsnorm_warp<<<rows_grid(rows, 8), 256, 0, s>>>(x, w, rows, cols, eps, y, rstd);
    return cudaGetLastError();
}

cudaError_t launch_cross_entropy(const float *logits, int64_t rows, int64_t V, int64_t ld, const int32_t *labels,
                                 float scale, float *loss, float *dlogits, int64_t ldd, cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    size_t nt = (size_t)((V + TILE_ELEMS - 1) / TILE_ELEMS);
    const size_t smem = (size_t)(((V + 3) & ~3ll) + ((nt + 3) & ~3ull) + 32) * sizeof(float);
    const bool al = ((reinterpret_cast<uintptr_t>(logits) & 15u) == 0) && (ld % 4 == 0);
    if (al && smem <= 227 * 1024) {
        static size_t attr = 0;
        if (smem > attr) {
            cudaError_t e = cudaFuncSetAttribute(cross_entropy_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (e != cudaSuccess) return e;
            attr = smem;
        }
        cross_entropy_smem<<<(unsigned)rows, CE_THREADS, smem, s>>>(logits, rows, V, ld, labels, scale, loss, dlogits,
                                                                     ldd);
        return cudaGetLastError();
    }
    cross_entropy_cta<<<(unsigned)rows, 512, (((nt + 3) & ~3ull) + 32) * sizeof(float), s>>>(
        logits, rows, V, ld, labels, scale, loss, dlogits, ldd);
    return cudaGetLastError();
}
