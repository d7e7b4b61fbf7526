// sha256.cu -- Verde tensor commitments on the GPU (R-TCOMMIT, reading R11).
//
// The paper commits every tensor entering / leaving a graph node with
// "a standard collision-resistant hash function like SHA-256" (PAPER.md
// P:240-244, box P:400-406).  A flat SHA-256 is a strictly sequential chain
// of compressions; this build cuts each tensor into 4096-byte chunks and
// commits to their RFC 6962 Merkle tree (R11), which is embarrassingly
// parallel and lets the referee later descend to one chunk.
//
// Launch sequence for a batch of tensors (verde_commit_tensors):
//   1. leaf kernel   : one thread per 4 KiB chunk -> SHA-256(0x00 || chunk)
//                      (65 compressions; the 1-byte prefix is absorbed with a
//                      byte permute per message word: PRMT)
//   2. reduce passes : one CTA per aligned group of <= 256 nodes of one tensor
//                      reduces them level by level in shared memory with
//                      RFC 6962 odd-node promotion (== the recursive MTH,
//                      because groups are aligned powers of two)
//   3. header kernel : one thread per tensor -> SHA-256(0x54 || dtype || rank
//                      || dims || nbytes || 4096 || data_root)
// SHA-256 is integer-ALU bound on sm_100a (rotates = SHF, Ch/Maj/xor = LOP3,
// adds = IADD3/IMAD), not HBM bound; see DESIGN.md §5.
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

#include "common.cuh"
#include "sha256.cuh"

#ifndef RO_SHA_MODE_DEFAULT
#define RO_SHA_MODE_DEFAULT 3
#endif

namespace {

__constant__ uint32_t kK[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

struct Digest { uint32_t h[8]; };

RO_DEV uint32_t rotr(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

RO_DEV void init_state(uint32_t s[8]) {
    s[0] = 0x6a09e667; s[1] = 0xbb67ae85; s[2] = 0x3c6ef372; s[3] = 0xa54ff53a;
    s[4] = 0x510e527f; s[5] = 0x9b05688c; s[6] = 0x1f83d9ab; s[7] = 0x5be0cd19;
}

// runtime 1 (constant bank, unknown to ptxas): a * kOne + b is an IMAD on the FMA pipe,
// so adds can be moved off the saturated ALU pipe (SHF / LOP3 / IADD3); bits unchanged
__constant__ uint32_t kOne = 1u;

RO_DEV uint32_t madd(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(kOne), "r"(b));
    return r;
}

// powers of two in the constant bank (unknown to ptxas): x >> n = mul.hi(x, 2^(32-n)) and
// rotr(x, n) = lo + hi of mul.wide(x, 2^(32-n)) (disjoint halves) run on the FMA pipe
__constant__ uint32_t kP2[32] = {1u, 2u, 4u, 8u, 16u, 32u, 64u, 128u, 256u, 512u, 1024u, 2048u, 4096u, 8192u,
                                 16384u, 32768u, 65536u, 131072u, 262144u, 524288u, 1048576u, 2097152u, 4194304u,
                                 8388608u, 16777216u, 33554432u, 67108864u, 134217728u, 268435456u, 536870912u,
                                 1073741824u, 2147483648u};
RO_DEV uint32_t shr_fma(uint32_t x, int n) {
    uint32_t r;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(kP2[32 - n]));
    return r;
}
RO_DEV uint32_t rotr_fma(uint32_t x, int n) {
    uint64_t p;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(x), "r"(kP2[32 - n]));
    return madd((uint32_t)p, (uint32_t)(p >> 32));
}

// FIPS 180-4 compression of one 512-bit block (w = big-endian message words).
// MODE (bits-neutral pipe balance): 0 = all adds on the ALU pipe (IADD3); 1 = the round
// adds (t1, e, a) as IMAD on the FMA pipe; 2 = also the message-schedule adds; 3 = also
// the schedule's shifts (IMAD.HI); 4 = 3 + one rotate of Sigma0 / Sigma1 (IMAD.WIDE);
// 5 = 3 + every remaining add.  Measured on B200 (tools/commit_one.py --time, 1 GiB):
// 743 / 818 / 846 / 853 / 757 / 854 GB/s for modes 0..5 -> default 3 (ALU ops per 64-byte
// block 1287 -> 949, the rest on the FMA pipe).  Occupancy is register-bound (56 regs,
// 9 CTAs of 128 / SM; more CTAs spill).
template <int MODE>
RO_DEV void compress_m(uint32_t s[8], uint32_t w[16]) {
    uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#pragma unroll
    for (int t = 0; t < 64; ++t) {
        uint32_t wt;
        if (t < 16) {
            wt = w[t];
        } else {
            uint32_t w15 = w[(t - 15) & 15], w2 = w[(t - 2) & 15];
            uint32_t s0 = rotr(w15, 7) ^ rotr(w15, 18) ^ (MODE >= 3 ? shr_fma(w15, 3) : (w15 >> 3));
            uint32_t s1 = rotr(w2, 17) ^ rotr(w2, 19) ^ (MODE >= 3 ? shr_fma(w2, 10) : (w2 >> 10));
            if (MODE >= 5)
                wt = w[t & 15] = madd(madd(w[t & 15], s0), madd(w[(t - 7) & 15], s1));
            else if (MODE >= 2)
                wt = w[t & 15] = madd(w[t & 15], s0) + madd(w[(t - 7) & 15], s1);
            else
                wt = w[t & 15] = w[t & 15] + s0 + w[(t - 7) & 15] + s1;
        }
        uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ (MODE == 4 ? rotr_fma(e, 25) : rotr(e, 25));
        uint32_t ch = (e & f) ^ (~e & g);
        uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ (MODE == 4 ? rotr_fma(a, 22) : rotr(a, 22));
        uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        uint32_t t1;
        if (MODE >= 5) {
            t1 = madd(madd(h, kK[t]), madd(S1, madd(ch, wt)));
            h = g; g = f; f = e; e = madd(d, t1); d = c; c = b; b = a; a = madd(t1, madd(S0, mj));
        } else if (MODE >= 1) {
            t1 = madd(madd(h, kK[t]), madd(S1, ch + wt));
            h = g; g = f; f = e; e = madd(d, t1); d = c; c = b; b = a; a = madd(t1, S0 + mj);
        } else {
            t1 = h + S1 + ch + kK[t] + wt;
            h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + S0 + mj;
        }
    }
    s[0] += a; s[1] += b; s[2] += c; s[3] += d; s[4] += e; s[5] += f; s[6] += g; s[7] += h;
}

RO_DEV void compress(uint32_t s[8], uint32_t w[16]) { compress_m<0>(s, w); }

// SHA-256 of a short local byte message (<= 119 bytes -> at most 2 blocks)
RO_DEV void sha_small(const uint8_t *msg, int len, uint32_t out[8]) {
    init_state(out);
    const int nblk = (len + 9 + 63) / 64;
    for (int blk = 0; blk < nblk; ++blk) {
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            uint32_t word = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                int m = blk * 64 + i * 4 + q;
                uint32_t byte;
                if (m < len) byte = msg[m];
                else if (m == len) byte = 0x80;
                else if (m >= nblk * 64 - 8) {
                    uint64_t bits = (uint64_t)len * 8;
                    byte = (uint32_t)(bits >> (8 * (nblk * 64 - 1 - m))) & 0xFF;
                } else byte = 0;
                word = (word << 8) | byte;
            }
            w[i] = word;
        }
        compress(out, w);
    }
}

// message byte m of (0x00 || data[0..len)) with SHA padding, total blocks nblk
RO_DEV uint32_t leaf_msg_byte(const uint8_t *data, int64_t len, int64_t m, int64_t nblk) {
    if (m == 0) return 0x00;
    if (m <= len) return data[m - 1];
    if (m == len + 1) return 0x80;
    if (m >= nblk * 64 - 8) {
        uint64_t bits = (uint64_t)(len + 1) * 8;
        return (uint32_t)(bits >> (8 * (nblk * 64 - 1 - m))) & 0xFF;
    }
    return 0;
}

// SHA-256(0x00 || chunk), chunk = data[0..len), len <= 4096
template <int MODE = 0>
RO_DEV void hash_leaf(const uint8_t *__restrict__ data, int64_t len, uint32_t st[8]) {
    init_state(st);
    const int64_t nblk = (len + 1 + 9 + 63) / 64;
    const bool al = ro::aligned16(data);
    int64_t blk = 0;
    if (al) {
        // fast path: blocks whose 16 data words D[16j .. 16j+15] are all in range
        const uint4 *d4 = reinterpret_cast<const uint4 *>(data);
        uint32_t prev = 0;  // word holding the 0x00 prefix byte in its top byte
        for (; blk * 64 + 64 <= len; ++blk) {
            uint32_t D[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint4 v = __ldg(d4 + blk * 4 + q);
                D[4 * q] = v.x; D[4 * q + 1] = v.y; D[4 * q + 2] = v.z; D[4 * q + 3] = v.w;
            }
            uint32_t w[16];
            w[0] = __byte_perm(prev, D[0], 0x3456);
#pragma unroll
            for (int i = 1; i < 16; ++i) w[i] = __byte_perm(D[i - 1], D[i], 0x3456);
            prev = D[15];
            compress_m<MODE>(st, w);
        }
        if (len == 4096) {
            // a full chunk's final block: its last data byte, 0x80, zeros, and the message
            // length 4097 * 8 bits -- the next "memory word" is the bytes 80 00 00 00
            uint32_t w[16];
            w[0] = __byte_perm(prev, 0x00000080u, 0x3456);
#pragma unroll
            for (int i = 1; i < 15; ++i) w[i] = 0;
            w[15] = 4097u * 8u;
            compress_m<MODE>(st, w);
            return;
        }
    }
    for (; blk < nblk; ++blk) {
        uint32_t w[16];
#pragma unroll 4
        for (int i = 0; i < 16; ++i) {
            uint32_t word = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) word = (word << 8) | leaf_msg_byte(data, len, blk * 64 + i * 4 + q, nblk);
            w[i] = word;
        }
        compress(st, w);
    }
}

// SHA-256(0x01 || L || R) with L, R given as state words (big-endian digest)
RO_DEV void hash_node(const uint32_t L[8], const uint32_t R[8], uint32_t st[8]) {
    init_state(st);
    uint32_t w[16];
    w[0] = 0x01000000u | (L[0] >> 8);
#pragma unroll
    for (int i = 1; i < 8; ++i) w[i] = __funnelshift_r(L[i], L[i - 1], 8);
    w[8] = __funnelshift_r(R[0], L[7], 8);
#pragma unroll
    for (int i = 1; i < 8; ++i) w[8 + i] = __funnelshift_r(R[i], R[i - 1], 8);
    compress(st, w);
    w[0] = (R[7] << 24) | 0x00800000u;
#pragma unroll
    for (int i = 1; i < 15; ++i) w[i] = 0;
    w[15] = 65 * 8;
    compress(st, w);
}

struct DevTensor {
    const uint8_t *data;
    int64_t nbytes;
    int64_t dims[8];
    uint8_t *digest;
    int32_t dtype, rank, mode;
    Digest *leaves_out;          // optional copy of the leaf hashes
    const Digest *base_leaves;   // optional: clean chunks take their leaf from here
    const uint8_t *dirty;        //           (chunk c hashed iff dirty[c])
};

RO_DEV int64_t find_seg(const int64_t *prefix, int n, int64_t g) {
    // largest t with prefix[t] <= g (prefix nondecreasing, prefix[0] = 0)
    int lo = 0, hi = n;
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (prefix[mid] <= g) lo = mid; else hi = mid;
    }
    return lo;
}

template <int MODE>
__global__ void leaf_kernel(const DevTensor *__restrict__ ts, int n, const int64_t *__restrict__ chunk_prefix,
                            int64_t total, Digest *__restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += stride) {
        int t = (int)find_seg(chunk_prefix, n, g);
        int64_t c = g - chunk_prefix[t];
        const DevTensor &T = ts[t];
        Digest d;
        if (T.base_leaves && !T.dirty[c]) {
            d = T.base_leaves[c];  // incremental commit: the chunk's bytes are unchanged
        } else {
            int64_t off = c * 4096;
            int64_t len = T.nbytes - off < 4096 ? T.nbytes - off : 4096;
            uint32_t st[8];
            hash_leaf<MODE>(T.data + off, len, st);
#pragma unroll
            for (int i = 0; i < 8; ++i) d.h[i] = st[i];
        }
        if (T.leaves_out) T.leaves_out[c] = d;
        out[g] = d;
    }
}

// leaf hashes of one buffer: thread g hashes chunk g (verde_chunk_leaves)
__global__ void chunk_leaf_kernel(const uint8_t *__restrict__ data, int64_t nbytes, int64_t nchunks,
                                  uint8_t *__restrict__ out) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= nchunks) return;
    const int64_t off = g * 4096;
    uint32_t st[8];
    hash_leaf(data + off, nbytes - off < 4096 ? nbytes - off : 4096, st);
    uint8_t *o = out + 32 * g;  // big-endian digest bytes
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        o[4 * i] = (uint8_t)(st[i] >> 24); o[4 * i + 1] = (uint8_t)(st[i] >> 16);
        o[4 * i + 2] = (uint8_t)(st[i] >> 8); o[4 * i + 3] = (uint8_t)st[i];
    }
}

// one CTA (128 threads) per group of <= 256 nodes of one tensor
__global__ void reduce_kernel(const int64_t *__restrict__ block_prefix, const int64_t *__restrict__ cur_off,
                              const int64_t *__restrict__ cur_cnt, const int64_t *__restrict__ nxt_off, int n,
                              const Digest *__restrict__ cur, Digest *__restrict__ nxt) {
    __shared__ Digest sm[256];
    const int64_t b = blockIdx.x;
    const int t = (int)find_seg(block_prefix, n, b);
    const int64_t j = b - block_prefix[t];
    const int64_t base = cur_off[t] + j * 256;
    int cnt = (int)min((int64_t)256, cur_cnt[t] - j * 256);
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) sm[i] = cur[base + i];
    __syncthreads();
    while (cnt > 1) {
        const int pairs = cnt >> 1;
        Digest r;
        int i = threadIdx.x;
        if (i < pairs) hash_node(sm[2 * i].h, sm[2 * i + 1].h, r.h);
        const bool promote = (cnt & 1) && threadIdx.x == 0;
        Digest last;
        if (promote) last = sm[cnt - 1];
        __syncthreads();
        if (i < pairs) sm[i] = r;
        if (promote) sm[pairs] = last;
        cnt = pairs + (cnt & 1);
        __syncthreads();
    }
    if (threadIdx.x == 0) nxt[nxt_off[t] + j] = sm[0];
}

__global__ void header_kernel(const DevTensor *__restrict__ ts, int n, const int64_t *__restrict__ root_off,
                              const Digest *__restrict__ roots) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const DevTensor &T = ts[t];
    uint32_t root[8];
    if (T.nbytes == 0) {
        sha_small(nullptr, 0, root);
    } else {
        const Digest &d = roots[root_off[t]];
#pragma unroll
        for (int i = 0; i < 8; ++i) root[i] = d.h[i];
    }
    uint8_t msg[128];
    int len = 0;
    msg[len++] = 0x54;
    msg[len++] = (uint8_t)T.dtype;
    auto put64 = [&](uint64_t v) {
        for (int i = 0; i < 8; ++i) msg[len++] = (uint8_t)(v >> (8 * i));
    };
    put64((uint64_t)T.rank);
    for (int i = 0; i < T.rank; ++i) put64((uint64_t)T.dims[i]);
    put64((uint64_t)T.nbytes);
    msg[len++] = 0x00; msg[len++] = 0x10; msg[len++] = 0x00; msg[len++] = 0x00;  // u32le 4096
    for (int i = 0; i < 8; ++i) {
        msg[len++] = (uint8_t)(root[i] >> 24); msg[len++] = (uint8_t)(root[i] >> 16);
        msg[len++] = (uint8_t)(root[i] >> 8); msg[len++] = (uint8_t)root[i];
    }
    uint32_t out[8];
    if (T.mode == 1) {
        for (int i = 0; i < 8; ++i) out[i] = root[i];  // data_root only (slab of a sharded tensor)
    } else {
        sha_small(msg, len, out);
    }
    for (int i = 0; i < 8; ++i) {
        T.digest[4 * i] = (uint8_t)(out[i] >> 24); T.digest[4 * i + 1] = (uint8_t)(out[i] >> 16);
        T.digest[4 * i + 2] = (uint8_t)(out[i] >> 8); T.digest[4 * i + 3] = (uint8_t)out[i];
    }
}

inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Host-side plan of one batched commit: tables + workspace layout.
struct Plan {
    int n = 0;
    int64_t total_chunks = 0;
    std::vector<int64_t> chunk_prefix;                   // n+1
    struct Pass { std::vector<int64_t> block_prefix, cur_off, cur_cnt, nxt_off; int64_t blocks; bool to_b; };
    std::vector<Pass> passes;
    std::vector<int64_t> root_off;                       // n, offsets into the final buffer
    bool final_in_b = false;
    int64_t bufA = 0, bufB = 0;                          // digests
};

Plan make_plan(const verde_tensor_desc *d, int n) {
    Plan p;
    p.n = n;
    p.chunk_prefix.assign(n + 1, 0);
    std::vector<int64_t> cnt(n);
    for (int t = 0; t < n; ++t) {
        cnt[t] = (d[t].nbytes + 4095) / 4096;
        p.chunk_prefix[t + 1] = p.chunk_prefix[t] + cnt[t];
    }
    p.total_chunks = p.chunk_prefix[n];
    p.bufA = p.total_chunks > 0 ? p.total_chunks : 1;
    std::vector<int64_t> off(n);
    for (int t = 0; t < n; ++t) off[t] = p.chunk_prefix[t];
    bool in_b = false;
    int64_t maxB = 1;
    for (;;) {
        int64_t mx = 0;
        for (int t = 0; t < n; ++t) mx = cnt[t] > mx ? cnt[t] : mx;
        if (mx <= 1) break;
        Plan::Pass ps;
        ps.block_prefix.assign(n + 1, 0);
        ps.cur_off = off;
        ps.cur_cnt = cnt;
        ps.nxt_off.assign(n, 0);
        std::vector<int64_t> ncnt(n);
        int64_t acc = 0;
        for (int t = 0; t < n; ++t) {
            int64_t blocks = (cnt[t] + 255) / 256;
            ps.block_prefix[t + 1] = ps.block_prefix[t] + blocks;
            ps.nxt_off[t] = acc;
            ncnt[t] = blocks;
            acc += blocks;
        }
        ps.blocks = ps.block_prefix[n];
        ps.to_b = !in_b;
        if (!in_b && acc > maxB) maxB = acc;
        p.passes.push_back(ps);
        off = ps.nxt_off;
        cnt = ncnt;
        in_b = !in_b;
    }
    p.root_off = off;
    p.final_in_b = in_b;
    p.bufB = maxB;
    return p;
}

struct Layout {
    int64_t tensors, tables, bufA, bufB, total;
    std::vector<int64_t> blob;  // int64 tables, concatenated
    // offsets (in int64 units) of each table inside blob
    int64_t chunk_prefix_at, root_off_at;
    std::vector<int64_t> pass_at;  // 4 tables per pass, consecutive
};

Layout make_layout(const Plan &p) {
    Layout L;
    L.chunk_prefix_at = 0;
    L.blob.insert(L.blob.end(), p.chunk_prefix.begin(), p.chunk_prefix.end());
    L.root_off_at = (int64_t)L.blob.size();
    L.blob.insert(L.blob.end(), p.root_off.begin(), p.root_off.end());
    for (const auto &ps : p.passes) {
        L.pass_at.push_back((int64_t)L.blob.size());
        L.blob.insert(L.blob.end(), ps.block_prefix.begin(), ps.block_prefix.end());
        L.blob.insert(L.blob.end(), ps.cur_off.begin(), ps.cur_off.end());
        L.blob.insert(L.blob.end(), ps.cur_cnt.begin(), ps.cur_cnt.end());
        L.blob.insert(L.blob.end(), ps.nxt_off.begin(), ps.nxt_off.end());
    }
    L.tensors = 0;
    L.tables = align_up((int64_t)sizeof(DevTensor) * p.n, 256);
    L.bufA = L.tables + align_up((int64_t)L.blob.size() * 8, 256);
    L.bufB = L.bufA + align_up(p.bufA * (int64_t)sizeof(Digest), 256);
    L.total = L.bufB + align_up(p.bufB * (int64_t)sizeof(Digest), 256);
    return L;
}

}  // namespace

int64_t commit_workspace_bytes(const verde_tensor_desc *d, int n) {
    if (n <= 0) return 0;
    Plan p = make_plan(d, n);
    return make_layout(p).total;
}

// A prepared commit: host plan + workspace layout; the tables already live in
// the device workspace, so running it only launches kernels.
struct CommitPlanImpl {
    Plan p;
    Layout L;
    uint8_t *base;
    int n;
};

static std::vector<uint8_t> stage_tables(const verde_tensor_desc *d, int n, const Layout &L) {
    std::vector<uint8_t> host((size_t)L.bufA);
    std::vector<DevTensor> dt(n);
    for (int t = 0; t < n; ++t) {
        dt[t].data = reinterpret_cast<const uint8_t *>(d[t].data);
        dt[t].nbytes = d[t].nbytes;
        for (int i = 0; i < 8; ++i) dt[t].dims[i] = (i < d[t].rank) ? d[t].dims[i] : 0;
        dt[t].digest = d[t].digest;
        dt[t].dtype = d[t].dtype;
        dt[t].rank = d[t].rank;
        dt[t].mode = d[t].mode;
        dt[t].leaves_out = reinterpret_cast<Digest *>(d[t].leaves_out);
        dt[t].base_leaves = reinterpret_cast<const Digest *>(d[t].base_leaves);
        dt[t].dirty = d[t].base_leaves ? d[t].dirty : nullptr;
    }
    memcpy(host.data(), dt.data(), sizeof(DevTensor) * n);
    memcpy(host.data() + L.tables, L.blob.data(), L.blob.size() * 8);
    return host;
}

std::atomic<int> g_leaf_ctas_per_sm{16};  // leaf-kernel residency cap (tuning hook; bits-neutral)

static cudaError_t run_kernels(const Plan &p, const Layout &L, uint8_t *base, int n, cudaStream_t s, int *nkernels) {
    cudaError_t e;
    const DevTensor *dts = reinterpret_cast<const DevTensor *>(base);
    const int64_t *tab = reinterpret_cast<const int64_t *>(base + L.tables);
    Digest *A = reinterpret_cast<Digest *>(base + L.bufA);
    Digest *B = reinterpret_cast<Digest *>(base + L.bufB);
    if (p.total_chunks > 0) {
        int64_t blocks = (p.total_chunks + 127) / 128;
        int64_t cap = (int64_t)ro_host::num_sms() * g_leaf_ctas_per_sm.load(std::memory_order_relaxed);
        if (blocks > cap) blocks = cap;
        static const int sha_mode = [] {  // tuning hook (bits-neutral): REPOPS_SHA_MODE=0/1/2
            const char *e = getenv("REPOPS_SHA_MODE");
            return e ? atoi(e) : RO_SHA_MODE_DEFAULT;
        }();
        if (sha_mode == 5)
            leaf_kernel<5><<<(unsigned)blocks, 128, 0, s>>>(dts, n, tab + L.chunk_prefix_at, p.total_chunks, A);
        else if (sha_mode == 4)
            leaf_kernel<4><<<(unsigned)blocks, 128, 0, s>>>(dts, n, tab + L.chunk_prefix_at, p.total_chunks, A);
        else if (sha_mode == 3)
            leaf_kernel<3><<<(unsigned)blocks, 128, 0, s>>>(dts, n, tab + L.chunk_prefix_at, p.total_chunks, A);
        else if (sha_mode == 2)
            leaf_kernel<2><<<(unsigned)blocks, 128, 0, s>>>(dts, n, tab + L.chunk_prefix_at, p.total_chunks, A);
        else if (sha_mode == 1)
            leaf_kernel<1><<<(unsigned)blocks, 128, 0, s>>>(dts, n, tab + L.chunk_prefix_at, p.total_chunks, A);
        else
            leaf_kernel<0><<<(unsigned)blocks, 128, 0, s>>>(dts, n, tab + L.chunk_prefix_at, p.total_chunks, A);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    for (size_t q = 0; q < p.passes.size(); ++q) {
        const auto &ps = p.passes[q];
        const int64_t *pt = tab + L.pass_at[q];
        const Digest *cur = ps.to_b ? A : B;
        Digest *nxt = ps.to_b ? B : A;
        reduce_kernel<<<(unsigned)ps.blocks, 128, 0, s>>>(pt, pt + (n + 1), pt + (n + 1) + n, pt + (n + 1) + 2 * n, n,
                                                          cur, nxt);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    *nkernels = (p.total_chunks > 0 ? 1 : 0) + (int)p.passes.size() + 1;
    header_kernel<<<(n + 63) / 64, 64, 0, s>>>(dts, n, tab + L.root_off_at, p.final_in_b ? B : A);
    return cudaGetLastError();
}

cudaError_t commit_launch(const verde_tensor_desc *d, int n, void *ws, int64_t ws_bytes, cudaStream_t s,
                          int64_t *need, int *nkernels) {
    *nkernels = 0;
    if (n <= 0) return cudaSuccess;
    Plan p = make_plan(d, n);
    Layout L = make_layout(p);
    *need = L.total;
    if (ws_bytes < L.total) return cudaErrorMemoryAllocation;
    uint8_t *base = reinterpret_cast<uint8_t *>(ws);
    std::vector<uint8_t> host = stage_tables(d, n, L);
    // pageable source: returns once the bytes are staged, so `host` may be freed after
    cudaError_t e = cudaMemcpyAsync(base, host.data(), (size_t)L.bufA, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    return run_kernels(p, L, base, n, s, nkernels);
}

cudaError_t commit_plan_create(const verde_tensor_desc *d, int n, void *ws, int64_t ws_bytes, void **out,
                               int64_t *need) {
    Plan p = make_plan(d, n);
    Layout L = make_layout(p);
    *need = L.total;
    if (ws_bytes < L.total) return cudaErrorMemoryAllocation;
    std::vector<uint8_t> host = stage_tables(d, n, L);
    cudaError_t e = cudaMemcpy(ws, host.data(), (size_t)L.bufA, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return e;
    *out = new CommitPlanImpl{std::move(p), std::move(L), reinterpret_cast<uint8_t *>(ws), n};
    return cudaSuccess;
}

cudaError_t commit_plan_run(const void *plan, cudaStream_t s, int *nkernels) {
    const CommitPlanImpl *c = reinterpret_cast<const CommitPlanImpl *>(plan);
    return run_kernels(c->p, c->L, c->base, c->n, s, nkernels);
}

void commit_plan_destroy(void *plan) { delete reinterpret_cast<CommitPlanImpl *>(plan); }

// ---------------------------------------------------------------------------------
// Step root on the device (R-NODE + R-MERKLE): node digests from the static node
// serialisations and the device digest table, then the RFC 6962 root over them.
namespace {

// SHA-256 of blob[a, b) || table[32*slots[j]] for j in [sa, sb) -- streamed in 64-byte blocks
__global__ void node_digest_kernel(const uint8_t *__restrict__ blob, const int64_t *__restrict__ offs,
                                   const int64_t *__restrict__ slots, const int64_t *__restrict__ soffs,
                                   const uint8_t *__restrict__ table, int64_t n, Digest *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t pa = offs[i], pb = offs[i + 1], sa = soffs[i], sb = soffs[i + 1];
    const int64_t len = (pb - pa) + 32 * (sb - sa);
    auto byte_at = [&](int64_t m) -> uint32_t {
        if (m < pb - pa) return blob[pa + m];
        const int64_t q = m - (pb - pa);
        return table[32 * slots[sa + q / 32] + (q % 32)];
    };
    uint32_t st[8];
    init_state(st);
    const int64_t nblk = (len + 9 + 63) / 64;
    for (int64_t blk = 0; blk < nblk; ++blk) {
        uint32_t w[16];
        for (int j = 0; j < 16; ++j) {
            uint32_t word = 0;
            for (int q = 0; q < 4; ++q) {
                const int64_t m = blk * 64 + j * 4 + q;
                uint32_t b;
                if (m < len) b = byte_at(m);
                else if (m == len) b = 0x80;
                else if (m >= nblk * 64 - 8) b = (uint32_t)(((uint64_t)len * 8) >> (8 * (nblk * 64 - 1 - m))) & 0xFF;
                else b = 0;
                word = (word << 8) | b;
            }
            w[j] = word;
        }
        compress(st, w);
    }
    Digest d;
    for (int j = 0; j < 8; ++j) d.h[j] = st[j];
    out[i] = d;
}

// RFC 6962 leaf hash of 32-byte entries: SHA-256(0x00 || entry), entry as state words
__global__ void entry_leaf_kernel(const Digest *__restrict__ e, int64_t n, Digest *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t *h = e[i].h;
    uint32_t w[16];
    w[0] = h[0] >> 8;
    for (int j = 1; j < 8; ++j) w[j] = __funnelshift_r(h[j], h[j - 1], 8);
    w[8] = (h[7] << 24) | 0x00800000u;
    for (int j = 9; j < 15; ++j) w[j] = 0;
    w[15] = 33 * 8;
    uint32_t st[8];
    init_state(st);
    compress(st, w);
    Digest d;
    for (int j = 0; j < 8; ++j) d.h[j] = st[j];
    out[i] = d;
}

__global__ void digest_bytes_kernel(const Digest *__restrict__ in, int64_t n, uint8_t *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * 8) return;
    const uint32_t v = in[i / 8].h[i % 8];
    uint8_t *o = out + 4 * i;
    o[0] = (uint8_t)(v >> 24); o[1] = (uint8_t)(v >> 16); o[2] = (uint8_t)(v >> 8); o[3] = (uint8_t)v;
}

}  // namespace

struct RootPlanImpl {
    int64_t n;
    const uint8_t *blob;
    const int64_t *offs, *slots, *soffs;
    const uint8_t *table;
    uint8_t *node_out, *root_out;
    // workspace: node digests (as words) | leaf digests A | level buffer B | pass tables
    Digest *nodes, *A, *B;
    std::vector<int64_t> pass_blocks;  // reduce passes: number of CTAs each
    std::vector<int64_t *> pass_tab;   // per pass: 4 int64 tables of length 2,1,1,1 (one "tensor")
    std::vector<bool> pass_to_b;
    bool final_in_b;
};

int64_t root_plan_workspace(int64_t n) {
    int64_t passes = 0, c = n;
    while (c > 1) { c = (c + 255) / 256; ++passes; }
    return align_up(n * 32, 256) * 2 + align_up(((n + 255) / 256 + 1) * 32, 256) + 256 * (passes + 1);
}

cudaError_t root_plan_create(int64_t n, const uint8_t *blob, const int64_t *offs, const int64_t *slots,
                             const int64_t *soffs, const uint8_t *table, uint8_t *node_out, uint8_t *root_out,
                             void *ws, int64_t ws_bytes, void **out) {
    if (ws_bytes < root_plan_workspace(n)) return cudaErrorMemoryAllocation;
    RootPlanImpl *p = new RootPlanImpl{};
    p->n = n; p->blob = blob; p->offs = offs; p->slots = slots; p->soffs = soffs; p->table = table;
    p->node_out = node_out; p->root_out = root_out;
    uint8_t *base = reinterpret_cast<uint8_t *>(ws);
    p->nodes = reinterpret_cast<Digest *>(base);
    p->A = reinterpret_cast<Digest *>(base + align_up(n * 32, 256));
    p->B = reinterpret_cast<Digest *>(base + 2 * align_up(n * 32, 256));
    uint8_t *tabs = base + 2 * align_up(n * 32, 256) + align_up(((n + 255) / 256 + 1) * 32, 256);
    // passes over a single "tensor" of n leaves: ping-pong A -> B -> A ...
    int64_t cnt = n;
    bool in_b = false;
    std::vector<int64_t> host;
    while (cnt > 1) {
        const int64_t blocks = (cnt + 255) / 256;
        int64_t t[5] = {0, blocks, 0, cnt, 0};  // block_prefix[2], cur_off, cur_cnt, nxt_off
        int64_t *dst = reinterpret_cast<int64_t *>(tabs + 256 * p->pass_tab.size());
        cudaError_t e = cudaMemcpy(dst, t, sizeof t, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) { delete p; return e; }
        p->pass_tab.push_back(dst);
        p->pass_blocks.push_back(blocks);
        p->pass_to_b.push_back(!in_b);
        in_b = !in_b;
        cnt = blocks;
    }
    p->final_in_b = in_b;
    *out = p;
    return cudaSuccess;
}

cudaError_t root_plan_run(const void *plan, cudaStream_t s, int *nkernels) {
    const RootPlanImpl *p = reinterpret_cast<const RootPlanImpl *>(plan);
    const int64_t n = p->n;
    const unsigned g = (unsigned)((n + 127) / 128);
    node_digest_kernel<<<g, 128, 0, s>>>(p->blob, p->offs, p->slots, p->soffs, p->table, n, p->nodes);
    entry_leaf_kernel<<<g, 128, 0, s>>>(p->nodes, n, p->A);
    int nk = 2;
    for (size_t q = 0; q < p->pass_tab.size(); ++q) {
        const int64_t *t = p->pass_tab[q];
        const Digest *cur = p->pass_to_b[q] ? p->A : p->B;
        Digest *nxt = p->pass_to_b[q] ? p->B : p->A;
        reduce_kernel<<<(unsigned)p->pass_blocks[q], 128, 0, s>>>(t, t + 2, t + 3, t + 4, 1, cur, nxt);
        ++nk;
    }
    const Digest *root = (n == 1) ? p->A : (p->final_in_b ? p->B : p->A);
    if (p->node_out) {
        digest_bytes_kernel<<<(unsigned)((n * 8 + 255) / 256), 256, 0, s>>>(p->nodes, n, p->node_out);
        ++nk;
    }
    digest_bytes_kernel<<<1, 32, 0, s>>>(root, 1, p->root_out);
    *nkernels = nk + 1;
    return cudaGetLastError();
}

void root_plan_destroy(void *plan) { delete reinterpret_cast<RootPlanImpl *>(plan); }

cudaError_t chunk_leaves_launch(const uint8_t *data, int64_t nbytes, uint8_t *leaves, cudaStream_t s) {
    const int64_t n = (nbytes + 4095) / 4096;
    chunk_leaf_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(data, nbytes, n, leaves);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ incremental commit flags
namespace {
__global__ void dirty_chunks_kernel(const int32_t *__restrict__ rows, int64_t n, int64_t row_bytes, int64_t nchunks,
                                    int all, uint8_t *__restrict__ flags) {
    extern __shared__ int32_t srow[];
    if (!all)
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) srow[i] = rows[i];
    __syncthreads();
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    uint8_t f = all ? 1 : 0;
    if (!all) {
        const int64_t r0 = c * 4096 / row_bytes, r1 = (c * 4096 + 4095) / row_bytes;  // rows the chunk meets
        for (int64_t i = 0; i < n && !f; ++i) f = (srow[i] >= r0 && srow[i] <= r1) ? 1 : 0;
    }
    flags[c] = f;
}
}  // namespace

cudaError_t launch_dirty_chunks(const int32_t *rows, int64_t n, int64_t row_bytes, int64_t nbytes, int all,
                                uint8_t *flags, cudaStream_t s) {
    const int64_t nchunks = (nbytes + 4095) / 4096;
    if (nchunks == 0) return cudaSuccess;
    const size_t smem = all ? 0 : (size_t)n * sizeof(int32_t);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(dirty_chunks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    dirty_chunks_kernel<<<(unsigned)((nchunks + 255) / 256), 256, smem, s>>>(rows, n, row_bytes, nchunks, all, flags);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ diagnostic: compression ceiling
// The commit kernels' practical ALU ceiling: every thread runs `iters` SHA-256 compressions
// (the leaf kernel's compress_m<RO_SHA_MODE_DEFAULT>) on a register-resident message block,
// each block's words perturbed by the previous state so nothing folds away -- no loads, no
// byte shifting, no tree.  Bytes "hashed" = 64 per compression.
namespace {
__global__ void __launch_bounds__(128) sha_probe_kernel(int64_t iters, uint32_t *out) {
    uint32_t st[8], w[16];
    init_state(st);
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = g * 0x9E3779B9u + (uint32_t)i;
    for (int64_t it = 0; it < iters; ++it) {
        compress_m<RO_SHA_MODE_DEFAULT>(st, w);
        w[it & 15] ^= st[0];
    }
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) x ^= st[i];
    out[g] = x;
}
}  // namespace

cudaError_t launch_sha_probe(int64_t ctas, int64_t iters, uint32_t *out, cudaStream_t s) {
    if (ctas <= 0 || iters <= 0) return cudaSuccess;
    sha_probe_kernel<<<(unsigned)ctas, 128, 0, s>>>(iters, out);
    return cudaGetLastError();
}
