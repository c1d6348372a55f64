// pack.cu -- A1 ternarise-and-pack, unpack, standalone A4 requant, A8 prediction.
//
// Packed layout (include/tn.h, reading R3): uint32 [n][d][h][w][2][cw]; per voxel
// cw sign words (bit = +1) then cw mask words (bit = nonzero); channel c is bit
// c%32 of word c/32.  Encoding: PAPER.md:118 ("2 bits per entry that encode the
// sign and value") and Fig. 3, mask = nonzero (reading R2).
//
// All kernels here are HBM-bound streaming kernels: one thread per voxel (or per
// 4 voxels for the vectorised packers), coalesced along the innermost axis.
#include "tn_internal.cuh"

#include <algorithm>

#include <climits>
#include <cstdlib>

namespace tn {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void report_bad(int64_t* d_bad, int64_t idx) {
    if (d_bad != nullptr && idx != LLONG_MAX)
        atomicMin(reinterpret_cast<long long*>(d_bad), static_cast<long long>(idx));
}

// ----------------------------------------------------------------------------
// Integer / float codes NCDHW -> packed.  VPT consecutive voxels per thread
// (vector loads along the contiguous DHW axis), CW words per plane held in
// registers and written as one 8/16/32-byte store per voxel.
// ----------------------------------------------------------------------------
template <typename T> struct Vec4;
template <> struct Vec4<int8_t>  { using type = char4; };
template <> struct Vec4<int32_t> { using type = int4; };
template <> struct Vec4<float>   { using type = float4; };

template <typename T>
struct Classify;
template <> struct Classify<int8_t> {
    float t_lo, t_hi;
    __device__ __forceinline__ int operator()(int8_t v, bool& ok) const {
        ok = (v >= -1 && v <= 1);
        return v;
    }
};
template <> struct Classify<int32_t> {
    float t_lo, t_hi;
    __device__ __forceinline__ int operator()(int32_t v, bool& ok) const {
        ok = (v >= -1 && v <= 1);
        return v;
    }
};
template <> struct Classify<float> {
    float t_lo, t_hi;
    // Eq. 6 with folded normalisation thresholds (reading R7).
    __device__ __forceinline__ int operator()(float v, bool& ok) const {
        ok = isfinite(v);
        return v > t_hi ? 1 : (v < t_lo ? -1 : 0);
    }
};

template <int CW>
__device__ __forceinline__ void store_voxel(uint32_t* dst, const uint32_t (&s)[CW], const uint32_t (&m)[CW]) {
    if constexpr (CW == 1) {
        *reinterpret_cast<uint2*>(dst) = make_uint2(s[0], m[0]);
    } else if constexpr (CW == 2) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(s[0], s[1], m[0], m[1]);
    } else if constexpr (CW == 4) {
        reinterpret_cast<uint4*>(dst)[0] = make_uint4(s[0], s[1], s[2], s[3]);
        reinterpret_cast<uint4*>(dst)[1] = make_uint4(m[0], m[1], m[2], m[3]);
    } else {
#pragma unroll
        for (int j = 0; j < CW; ++j) { dst[j] = s[j]; dst[CW + j] = m[j]; }
    }
}

template <typename T, int CW, int VPT>
__global__ void __launch_bounds__(kThreads)
pack_kernel(const T* __restrict__ x, int C, int64_t DHW, int64_t total, Classify<T> cls,
            uint32_t* __restrict__ xp, int64_t* d_bad) {
    const int64_t g0 = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) * VPT;
    if (g0 >= total) return;
    const int64_t n = g0 / DHW;
    const int64_t v0 = g0 - n * DHW;
    const T* xb = x + n * C * DHW + v0;
    uint32_t s[VPT][CW], m[VPT][CW];
#pragma unroll
    for (int i = 0; i < VPT; ++i)
#pragma unroll
        for (int j = 0; j < CW; ++j) { s[i][j] = 0u; m[i][j] = 0u; }
    int64_t bad = LLONG_MAX;
#pragma unroll
    for (int j = 0; j < CW; ++j) {
        const int cend = min(C, 32 * (j + 1));
        for (int c = 32 * j; c < cend; ++c) {
            T vals[VPT];
            if constexpr (VPT == 4) {
                auto q = *reinterpret_cast<const typename Vec4<T>::type*>(xb + c * DHW);
                vals[0] = q.x; vals[1] = q.y; vals[2] = q.z; vals[3] = q.w;
            } else {
                vals[0] = xb[c * DHW];
            }
            const uint32_t bit = 1u << (c & 31);
#pragma unroll
            for (int i = 0; i < VPT; ++i) {
                bool ok;
                const int t = cls(vals[i], ok);
                if (!ok) {
                    const int64_t idx = (n * C + c) * DHW + v0 + i;
                    bad = min(bad, idx);
                    continue;
                }
                m[i][j] |= (t != 0) ? bit : 0u;
                s[i][j] |= (t == 1) ? bit : 0u;
            }
        }
    }
    report_bad(d_bad, bad);
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
        if (g0 + i < total) store_voxel<CW>(xp + (g0 + i) * 2 * CW, s[i], m[i]);
    }
}

// Generic fallback: one thread per (voxel, word); any C.
template <typename T>
__global__ void __launch_bounds__(kThreads)
pack_generic_kernel(const T* __restrict__ x, int C, int cw, int64_t DHW, int64_t total,
                    Classify<T> cls, uint32_t* __restrict__ xp, int64_t* d_bad) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    if (t >= total * cw) return;
    const int64_t g = t / cw;
    const int j = static_cast<int>(t - g * cw);
    const int64_t n = g / DHW;
    const int64_t v = g - n * DHW;
    uint32_t s = 0, m = 0;
    int64_t bad = LLONG_MAX;
    const int cend = min(C, 32 * (j + 1));
    for (int c = 32 * j; c < cend; ++c) {
        bool ok;
        const int64_t idx = (n * C + c) * DHW + v;
        const int q = cls(x[idx], ok);
        if (!ok) { bad = min(bad, idx); continue; }
        const uint32_t bit = 1u << (c & 31);
        m |= (q != 0) ? bit : 0u;
        s |= (q == 1) ? bit : 0u;
    }
    report_bad(d_bad, bad);
    xp[g * 2 * cw + j] = s;
    xp[g * 2 * cw + cw + j] = m;
}

// ----------------------------------------------------------------------------
// int8 fast path: 4 voxels per thread (one 32-bit load per channel), SWAR
// classification of the 4 voxels in one 32-bit word.  For a word q of 4 int8 codes:
//   lsb  = q & 0x01010101              (nonzero bit of each byte: 0x01, 0xFF -> 1)
//   t7   = (q >> 7) & 0x01010101       (bit 7 of each byte)
//   pos  = lsb & ~t7                   (+1 <=> byte == 0x01)
// and the byte is a valid code iff bits 1..7 all equal bit 7 and (bit 7 => lsb).
// Bits of 8 consecutive channels accumulate per byte lane (acc += bit << j),
// so byte i of acc holds voxel i's 8 channel bits; a 4x4 byte transpose (PRMT)
// of the four 8-channel groups then forms each voxel's 32-channel word.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void transpose4x4(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                             uint32_t& w0, uint32_t& w1, uint32_t& w2, uint32_t& w3) {
    const uint32_t t0 = __byte_perm(a0, a1, 0x5140), t1 = __byte_perm(a0, a1, 0x7362);
    const uint32_t t2 = __byte_perm(a2, a3, 0x5140), t3 = __byte_perm(a2, a3, 0x7362);
    w0 = __byte_perm(t0, t2, 0x5410);
    w1 = __byte_perm(t0, t2, 0x7632);
    w2 = __byte_perm(t1, t3, 0x5410);
    w3 = __byte_perm(t1, t3, 0x7632);
}

template <int CW>
__global__ void __launch_bounds__(kThreads, 3)
pack_i8_swar_kernel(const int8_t* __restrict__ x, int C, int64_t DHW, int64_t total,
                    uint32_t* __restrict__ xp, int64_t* d_bad) {
    // 4 voxels per thread: one 32-bit load per channel (a warp reads 128
    // contiguous bytes per channel), 16 channel loads in flight per thread.
    constexpr int VPT = 4;
    const int64_t g0 = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) * VPT;
    if (g0 >= total) return;
    const int64_t n = g0 / DHW;
    const int64_t v0 = g0 - n * DHW;
    const int8_t* xb = x + n * C * DHW + v0;
    uint32_t os[VPT][CW], om[VPT][CW];
    uint32_t bad = 0;
#pragma unroll
    for (int j = 0; j < CW; ++j) {
        // all 32 channel loads of this word first (32 x 128 B per warp in flight)
        uint32_t q[32];
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
            const int c = 32 * j + jj;
            q[jj] = c < C ? __ldg(reinterpret_cast<const uint32_t*>(xb + c * DHW)) : 0u;
        }
        uint32_t accS[4], accM[4];   // [group of 8 channels]
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            uint32_t as = 0u, am = 0u;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                const uint32_t w = q[8 * g + jj];
                const uint32_t lsb = w & 0x01010101u;
                const uint32_t t7 = (w >> 7) & 0x01010101u;
                const uint32_t pos = lsb & ~t7;
                bad |= ((w & 0xFEFEFEFEu) ^ (t7 * 0xFEu)) | (t7 & ~lsb);
                am += lsb << jj;
                as += pos << jj;
            }
            accS[g] = as;
            accM[g] = am;
        }
        transpose4x4(accS[0], accS[1], accS[2], accS[3], os[0][j], os[1][j], os[2][j], os[3][j]);
        transpose4x4(accM[0], accM[1], accM[2], accM[3], om[0][j], om[1][j], om[2][j], om[3][j]);
    }
    if (bad != 0u) {
        // rare slow path: find this thread's first offending NCDHW index exactly
        int64_t first = LLONG_MAX;
        for (int c = 0; c < C; ++c)
            for (int i = 0; i < VPT; ++i) {
                const int8_t v = xb[c * DHW + i];
                if (v < -1 || v > 1) first = min(first, (n * C + c) * DHW + v0 + i);
            }
        report_bad(d_bad, first);
    }
#pragma unroll
    for (int i = 0; i < VPT; ++i) store_voxel<CW>(xp + (g0 + i) * 2 * CW, os[i], om[i]);
}

// Shared-memory-staged variant: one tile of kPackTile (256) consecutive voxels per CTA
// (16 KB of shared memory for C = 64, 13 CTAs co-resident per SM).  The threads copy the
// tile's C channel rows (contiguous 256-byte runs in DRAM) with 16-byte cp.async in eight
// commit groups of 8 channels, then byte-lane SWAR over 4 voxels per thread from shared
// memory (consecutive threads read consecutive words of a channel row: conflict-free),
// accumulating each byte's nonzero bit and negative bit (sign = mask & ~negative at the
// end); the bit work on a group overlaps the arrival of the later groups.  Validation
// work only when d_bad is given.  Triggers the dependent conv's programmatic launch at
// its start.  Needs DHW % 256 == 0, C <= 64, 16-byte input.
// C1: 18.0 us for 64 MiB in + 16 MiB out (4.7 TB/s; 1-D bulk copies per channel row:
// 18.7 us; 512-voxel tiles with per-channel validation: 24 us; register-only variant
// below: 31 us).
#ifndef TN_PACK_TILE
#define TN_PACK_TILE 256
#endif
constexpr int kPackTile = TN_PACK_TILE;
template <int CW, bool CHECK>
__global__ void __launch_bounds__(kPackTile / 4)
pack_i8_bulk_kernel(const int8_t* __restrict__ x, int C, int64_t DHW, int64_t ntiles,
                    uint32_t* __restrict__ xp, int64_t* d_bad) {
    extern __shared__ __align__(128) uint8_t sx[];          // [C][kPackTile]
    // let a PDL-launched consumer (the conv) start its prologue as SMs free up; it still
    // waits (griddepcontrol.wait) for this whole grid before reading the packed tensor
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int64_t tile = blockIdx.x;
    if (tile >= ntiles) return;
    const int64_t t0 = tile * kPackTile;
    {
        // every thread copies 16-byte pieces of the channel rows with cp.async, one commit
        // group per 8 channels, so the bit work on a group overlaps the later groups' arrival
        const int64_t n = t0 / DHW;
        const int8_t* xb = x + n * C * DHW + (t0 - n * DHW);
        constexpr int kPieces = kPackTile / 16;      // per channel row
#pragma unroll
        for (int gq = 0; gq < 4 * CW; ++gq) {
            const int c0 = 8 * gq, c1 = min(C, c0 + 8);
            for (int e = threadIdx.x; e < (c1 - c0) * kPieces; e += kPackTile / 4) {
                const int c = c0 + e / kPieces, pc = e % kPieces;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(
                                 __cvta_generic_to_shared(sx + c * kPackTile + 16 * pc))),
                             "l"(xb + c * DHW + 16 * pc) : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
    }
    const int i4 = threadIdx.x;                 // this thread's 4 voxels of the tile
    uint32_t os[4][CW], om[4][CW];
    uint32_t bad = 0;
#pragma unroll
    for (int j = 0; j < CW; ++j) {
        uint32_t accS[4], accM[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            // wait for this thread's copies of group 4j+g, then for everyone's
            const int left = 4 * CW - 1 - (4 * j + g);
            if (left >= 7) asm volatile("cp.async.wait_group 7;" ::: "memory");
            else if (left == 6) asm volatile("cp.async.wait_group 6;" ::: "memory");
            else if (left == 5) asm volatile("cp.async.wait_group 5;" ::: "memory");
            else if (left == 4) asm volatile("cp.async.wait_group 4;" ::: "memory");
            else if (left == 3) asm volatile("cp.async.wait_group 3;" ::: "memory");
            else if (left == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
            else if (left == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
            else asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
            // bit jj of each byte: lsb (nonzero) and bit 7 (negative) of channel 8g + jj;
            // the fields are disjoint, so sign = mask & ~negative at the end
            uint32_t an = 0u, am = 0u;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                const int c = 32 * j + 8 * g + jj;
                const uint32_t w = c < C ? reinterpret_cast<const uint32_t*>(sx + c * kPackTile)[i4] : 0u;
                if (CHECK) {
                    const uint32_t lsb = w & 0x01010101u, t7 = (w >> 7) & 0x01010101u;
                    bad |= ((w & 0xFEFEFEFEu) ^ (t7 * 0xFEu)) | (t7 & ~lsb);
                }
                am |= (w << jj) & (0x01010101u << jj);
                an |= (w >> (7 - jj)) & (0x01010101u << jj);
            }
            accS[g] = am & ~an;
            accM[g] = am;
        }
        transpose4x4(accS[0], accS[1], accS[2], accS[3], os[0][j], os[1][j], os[2][j], os[3][j]);
        transpose4x4(accM[0], accM[1], accM[2], accM[3], om[0][j], om[1][j], om[2][j], om[3][j]);
    }
    if (CHECK && bad != 0u) {
        const int64_t n = t0 / DHW, v0 = t0 - n * DHW;
        int64_t first = LLONG_MAX;
        for (int c = 0; c < C; ++c)
            for (int i = 0; i < 4; ++i) {
                const int8_t v = static_cast<int8_t>(sx[c * kPackTile + 4 * i4 + i]);
                if (v < -1 || v > 1) first = min(first, (n * C + c) * DHW + v0 + 4 * i4 + i);
            }
        report_bad(d_bad, first);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) store_voxel<CW>(xp + (t0 + 4 * i4 + i) * 2 * CW, os[i], om[i]);
}

template <typename T>
cudaError_t pack_dispatch(const T* x, tn_dims xd, Classify<T> cls, uint32_t* xp, int64_t* d_bad,
                          cudaStream_t st) {
    const int64_t DHW = static_cast<int64_t>(xd.d) * xd.h * xd.w;
    const int64_t total = DHW * xd.n;
    if (total == 0) return cudaSuccess;
    const int cw = (xd.c + 31) / 32;
    const bool vec4 = (DHW % 4 == 0) && (reinterpret_cast<uintptr_t>(x) % (4 * sizeof(T)) == 0);
#define TN_PACK_CASE(CWV)                                                                    \
    if (cw == CWV) {                                                                         \
        if (vec4) {                                                                          \
            const int64_t nt = (total + 3) / 4;                                              \
            pack_kernel<T, CWV, 4><<<static_cast<unsigned>((nt + kThreads - 1) / kThreads), \
                                      kThreads, 0, st>>>(x, xd.c, DHW, total, cls, xp, d_bad); \
        } else {                                                                             \
            pack_kernel<T, CWV, 1><<<static_cast<unsigned>((total + kThreads - 1) / kThreads), \
                                      kThreads, 0, st>>>(x, xd.c, DHW, total, cls, xp, d_bad); \
        }                                                                                    \
        return cudaGetLastError();                                                           \
    }
    TN_PACK_CASE(1)
    TN_PACK_CASE(2)
    TN_PACK_CASE(4)
#undef TN_PACK_CASE
    const int64_t nt = total * cw;
    pack_generic_kernel<T><<<static_cast<unsigned>((nt + kThreads - 1) / kThreads), kThreads, 0, st>>>(
        x, xd.c, cw, DHW, total, cls, xp, d_bad);
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------
// Weights int8 [K][C][27] -> [K][27][2][CW]; one thread per (k, tap, word).
// ----------------------------------------------------------------------------
__global__ void pack_weights_kernel(const int8_t* __restrict__ w, int K, int C, int cw,
                                    uint32_t* __restrict__ wp, int64_t* d_bad) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= K * 27 * cw) return;
    const int j = t % cw;
    const int tap = (t / cw) % 27;
    const int k = t / (cw * 27);
    uint32_t s = 0, m = 0;
    int64_t bad = LLONG_MAX;
    const int cend = min(C, 32 * (j + 1));
    for (int c = 32 * j; c < cend; ++c) {
        const int64_t idx = (static_cast<int64_t>(k) * C + c) * 27 + tap;
        const int8_t v = w[idx];
        if (v < -1 || v > 1) { bad = min(bad, idx); continue; }
        const uint32_t bit = 1u << (c & 31);
        m |= (v != 0) ? bit : 0u;
        s |= (v == 1) ? bit : 0u;
    }
    report_bad(d_bad, bad);
    uint32_t* dst = wp + (static_cast<int64_t>(k) * 27 + tap) * 2 * cw;
    dst[j] = s;
    dst[cw + j] = m;
}

// ----------------------------------------------------------------------------
// Unpack: packed -> int8 NCDHW, with canonical-form validation.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
unpack_kernel(const uint32_t* __restrict__ xp, int C, int cw, int64_t DHW, int64_t total,
              int8_t* __restrict__ x, int64_t* d_bad) {
    const int64_t g = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    if (g >= total) return;
    const int64_t n = g / DHW;
    const int64_t v = g - n * DHW;
    const uint32_t* src = xp + g * 2 * cw;
    int64_t bad = LLONG_MAX;
    for (int j = 0; j < cw; ++j) {
        const uint32_t s = src[j], m = src[cw + j];
        const int cend = min(C, 32 * (j + 1));
        for (int c = 32 * j; c < cend; ++c) {
            const int b = c & 31;
            const uint32_t sb = (s >> b) & 1u, mb = (m >> b) & 1u;
            const int64_t idx = (n * C + c) * DHW + v;
            if (sb && !mb) bad = min(bad, idx);
            x[idx] = static_cast<int8_t>(mb ? (sb ? 1 : -1) : 0);
        }
        if (cend < 32 * (j + 1)) {
            const uint32_t padmask = 0xFFFFFFFFu << (cend & 31);
            if ((s | m) & padmask) bad = min(bad, (n * C + (C - 1)) * DHW + v);
        }
    }
    report_bad(d_bad, bad);
}

// ----------------------------------------------------------------------------
// Standalone requant (A4): int32 channel-last [V][K] -> packed [V][2][cwo].
// One warp per (voxel, word): lane l owns channel 32*word + l; the sign and
// mask words are warp ballots.  Reads are coalesced along K.
// Rule (reading R5): +1 if acc >= hi[k]; else -1 if acc <= lo[k]; else 0.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
requant_kernel(const int32_t* __restrict__ y, int64_t V, int K, int cwo,
               const int32_t* __restrict__ lo, const int32_t* __restrict__ hi,
               uint32_t* __restrict__ yp) {
    const int64_t warp = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= V * cwo) return;
    const int64_t v = warp / cwo;
    const int j = static_cast<int>(warp - v * cwo);
    const int k = 32 * j + lane;
    bool pos = false, neg = false;
    if (k < K) {
        const int32_t a = y[v * K + k];
        pos = a >= __ldg(hi + k);
        neg = !pos && a <= __ldg(lo + k);
    }
    const uint32_t s = __ballot_sync(0xFFFFFFFFu, pos);
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, pos || neg);
    if (lane == 0) {
        yp[v * 2 * cwo + j] = s;
        yp[v * 2 * cwo + cwo + j] = m;
    }
}

// ----------------------------------------------------------------------------
// Prediction (A8): logits[n][j][v] = b[j] + sum_c w[j][c] * t_c in fp32, c
// ascending within quads of 4 channels, quads ascending (reading R12).  One thread per voxel; C <= 32.
// ----------------------------------------------------------------------------
constexpr int kMaxClass = 8;
__global__ void __launch_bounds__(kThreads)
predict_kernel(const uint32_t* __restrict__ tp, int C, int64_t DHW, int64_t total,
               const float* __restrict__ w, const float* __restrict__ b, int nclass,
               float* __restrict__ logits, int64_t cstride) {
    __shared__ float sw[kMaxClass * 64];
    __shared__ float sb[kMaxClass];
    for (int i = threadIdx.x; i < nclass * C; i += kThreads) sw[i] = w[i];
    if (threadIdx.x < nclass) sb[threadIdx.x] = b[threadIdx.x];
    __syncthreads();
    const int64_t g = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    if (g >= total) return;
    const int cw = (C + 31) / 32;                 // C <= 64: one or two words per plane
    uint32_t ws[2] = {0u, 0u}, wm[2] = {0u, 0u};
    for (int q = 0; q < cw; ++q) { ws[q] = tp[g * 2 * cw + q]; wm[q] = tp[g * 2 * cw + cw + q]; }
    const int64_t n = g / DHW;
    const int64_t v = g - n * DHW;
    for (int j = 0; j < nclass; ++j) {
        // b + sum over channel quads of ((((t0 w0) + t1 w1) + t2 w2) + t3 w3): the
        // summation order the tensor-core epilogue's quad tables reproduce exactly
        float acc = sb[j];
        for (int c0 = 0; c0 < C; c0 += 4) {
            float part = 0.0f;
            for (int c = c0; c < c0 + 4 && c < C; ++c) {
                const float wv = sw[j * C + c];
                const bool nz = (wm[c >> 5] >> (c & 31)) & 1u;
                const bool p = (ws[c >> 5] >> (c & 31)) & 1u;
                part += nz ? (p ? wv : -wv) : 0.0f;
            }
            acc += part;
        }
        logits[(n * nclass + j) * cstride + v] = acc;
    }
}

// The same sums through per-block quad tables (as the fused tensor-core epilogue): entry
// (mask nibble | sign nibble << 4) of quad qd and class j is (((t0 w0) + t1 w1) + t2 w2) + t3 w3
// for the quad's four channels, so b + the quads' entries in ascending order is bit-identical to
// predict_kernel.  Table layout [qd][entry][class]; persistent grid, one table build per block.
template <int CW>
__global__ void __launch_bounds__(256)
predict_quad_kernel(const uint32_t* __restrict__ tp, int C, int64_t DHW, int64_t total,
                    const float* __restrict__ w, const float* __restrict__ b, int nclass,
                    float* __restrict__ logits, int64_t cstride) {
    extern __shared__ float tab[];                // [8 * CW][256][nclass]
    __shared__ float sb[kMaxClass];
    constexpr int NQ = 8 * CW;
    for (int e = threadIdx.x; e < NQ * 256 * nclass; e += blockDim.x) {
        const int j = e % nclass, idx = (e / nclass) & 255, qd = e / (256 * nclass);
        float part = 0.0f;
        for (int i = 0; i < 4; ++i) {
            const int c = 4 * qd + i;
            const float wv = c < C ? __ldg(w + j * C + c) : 0.0f;
            const bool nz = (idx >> i) & 1, ps = (idx >> (4 + i)) & 1;
            part += nz ? (ps ? wv : -wv) : 0.0f;
        }
        tab[e] = part;
    }
    if (threadIdx.x < nclass) sb[threadIdx.x] = b[threadIdx.x];
    __syncthreads();
    const int nq = (C + 3) / 4;
    for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < total;
         g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint32_t ws[CW], wm[CW];
        if constexpr (CW == 1) {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(tp) + g);
            ws[0] = v.x; wm[0] = v.y;
        } else {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(tp) + g);
            ws[0] = v.x; ws[1] = v.y; wm[0] = v.z; wm[1] = v.w;
        }
        const int64_t n = g / DHW, v = g - n * DHW;
        if (nclass == 2) {
            float a0 = sb[0], a1 = sb[1];
#pragma unroll
            for (int qd = 0; qd < NQ; ++qd) {
                if (qd < nq) {
                    const uint32_t sh = 4 * (qd & 7);
                    const uint32_t ix = ((wm[qd >> 3] >> sh) & 0xFu) | (((ws[qd >> 3] >> sh) & 0xFu) << 4);
                    const float2 e2 = *reinterpret_cast<const float2*>(tab + (qd * 256 + ix) * 2);
                    a0 += e2.x;
                    a1 += e2.y;
                }
            }
            logits[(n * 2) * cstride + v] = a0;
            logits[(n * 2 + 1) * cstride + v] = a1;
        } else {
            for (int j = 0; j < nclass; ++j) {
                float a = sb[j];
#pragma unroll
                for (int qd = 0; qd < NQ; ++qd) {
                    if (qd < nq) {
                        const uint32_t sh = 4 * (qd & 7);
                        const uint32_t ix = ((wm[qd >> 3] >> sh) & 0xFu) | (((ws[qd >> 3] >> sh) & 0xFu) << 4);
                        a += tab[(qd * 256 + ix) * nclass + j];
                    }
                }
                logits[(n * nclass + j) * cstride + v] = a;
            }
        }
    }
}

__global__ void bad_init_kernel(int64_t* d_bad) { *d_bad = LLONG_MAX; }

}  // namespace

cudaError_t launch_pack_i8(const int8_t* x, tn_dims xd, uint32_t* xp, int64_t* d_bad, cudaStream_t s) {
    const int64_t DHW = static_cast<int64_t>(xd.d) * xd.h * xd.w;
    const int64_t total = DHW * xd.n;
    const int cw = (xd.c + 31) / 32;
    if (total > 0 && DHW % kPackTile == 0 && (reinterpret_cast<uintptr_t>(x) & 15u) == 0 && (cw == 1 || cw == 2)) {
        // one 256-voxel tile per CTA (measured on C1: 256 > 512 > 1024 > 128 voxels; a
        // persistent double-buffered grid is slower at every CTAs-per-SM count, 26.3-121 us)
        const int64_t ntiles = total / kPackTile;
        const size_t smem = static_cast<size_t>(xd.c) * kPackTile;
        const unsigned blocks = static_cast<unsigned>(ntiles);
        if (d_bad != nullptr) {
            if (cw == 1) pack_i8_bulk_kernel<1, true><<<blocks, kPackTile / 4, smem, s>>>(x, xd.c, DHW, ntiles, xp, d_bad);
            else pack_i8_bulk_kernel<2, true><<<blocks, kPackTile / 4, smem, s>>>(x, xd.c, DHW, ntiles, xp, d_bad);
        } else {
            if (cw == 1) pack_i8_bulk_kernel<1, false><<<blocks, kPackTile / 4, smem, s>>>(x, xd.c, DHW, ntiles, xp, d_bad);
            else pack_i8_bulk_kernel<2, false><<<blocks, kPackTile / 4, smem, s>>>(x, xd.c, DHW, ntiles, xp, d_bad);
        }
        return cudaGetLastError();
    }
    if (total > 0 && DHW % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15u) == 0 &&
        (cw == 1 || cw == 2 || cw == 4)) {
        const int64_t nt = total / 4;
        const unsigned blocks = static_cast<unsigned>((nt + kThreads - 1) / kThreads);
        if (cw == 1) pack_i8_swar_kernel<1><<<blocks, kThreads, 0, s>>>(x, xd.c, DHW, total, xp, d_bad);
        else if (cw == 2) pack_i8_swar_kernel<2><<<blocks, kThreads, 0, s>>>(x, xd.c, DHW, total, xp, d_bad);
        else pack_i8_swar_kernel<4><<<blocks, kThreads, 0, s>>>(x, xd.c, DHW, total, xp, d_bad);
        return cudaGetLastError();
    }
    return pack_dispatch<int8_t>(x, xd, Classify<int8_t>{0.f, 0.f}, xp, d_bad, s);
}
cudaError_t launch_pack_i32(const int32_t* x, tn_dims xd, uint32_t* xp, int64_t* d_bad, cudaStream_t s) {
    return pack_dispatch<int32_t>(x, xd, Classify<int32_t>{0.f, 0.f}, xp, d_bad, s);
}
cudaError_t launch_pack_f32(const float* x, tn_dims xd, float t_lo, float t_hi, uint32_t* xp,
                            int64_t* d_bad, cudaStream_t s) {
    return pack_dispatch<float>(x, xd, Classify<float>{t_lo, t_hi}, xp, d_bad, s);
}

__global__ void stream_fence_kernel() {}

cudaError_t launch_pack_weights(const int8_t* w, int k, int c, uint32_t* wp, int64_t* d_bad,
                                cudaStream_t s) {
    const int cw = (c + 31) / 32;
    const int nt = k * 27 * cw;
    pack_weights_kernel<<<(nt + 127) / 128, 128, 0, s>>>(w, k, c, cw, wp, d_bad);
    // The conv kernels stage their filter bank before griddepcontrol.wait (programmatic
    // dependent launch), so the packed weights must not come from the kernel launched
    // immediately before a conv: an empty kernel after the packing keeps that true even
    // when the caller convolves right away.
    stream_fence_kernel<<<1, 32, 0, s>>>();
    return cudaGetLastError();
}

cudaError_t launch_unpack(const uint32_t* xp, tn_dims xd, int8_t* x, int64_t* d_bad, cudaStream_t s) {
    const int64_t DHW = static_cast<int64_t>(xd.d) * xd.h * xd.w;
    const int64_t total = DHW * xd.n;
    if (total == 0) return cudaSuccess;
    unpack_kernel<<<static_cast<unsigned>((total + kThreads - 1) / kThreads), kThreads, 0, s>>>(
        xp, xd.c, (xd.c + 31) / 32, DHW, total, x, d_bad);
    return cudaGetLastError();
}

cudaError_t launch_requant(const int32_t* y, tn_dims yd, const int32_t* lo, const int32_t* hi,
                           uint32_t* yp, cudaStream_t s) {
    const int64_t V = static_cast<int64_t>(yd.n) * yd.d * yd.h * yd.w;
    if (V == 0) return cudaSuccess;
    const int cwo = (yd.c + 31) / 32;
    const int64_t threads = V * cwo * 32;
    requant_kernel<<<static_cast<unsigned>((threads + kThreads - 1) / kThreads), kThreads, 0, s>>>(
        y, V, yd.c, cwo, lo, hi, yp);
    return cudaGetLastError();
}

cudaError_t launch_predict(const uint32_t* tp, tn_dims td, const float* w, const float* b,
                           int nclass, float* logits, cudaStream_t s, int64_t cstride) {
    const int64_t DHW = static_cast<int64_t>(td.d) * td.h * td.w;
    const int64_t total = DHW * td.n;
    if (total == 0) return cudaSuccess;
    const int cw = (td.c + 31) / 32;
    if (total >= (1 << 16) && (reinterpret_cast<uintptr_t>(tp) & 15u) == 0 && cw <= 2) {
        // large tensors: quad tables (bit-identical sums), a persistent grid of 4 blocks per SM
        static int nsm = 0;
        if (nsm == 0) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            if (nsm <= 0) nsm = 148;
        }
        const size_t smem = static_cast<size_t>(8 * cw) * 256 * nclass * sizeof(float);   // <= 128 KB
        const unsigned grid = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 4 * nsm));
        if (cw == 1) {
            cudaFuncSetAttribute(predict_quad_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
            predict_quad_kernel<1><<<grid, 256, smem, s>>>(tp, td.c, DHW, total, w, b, nclass, logits,
                                                           cstride < 0 ? DHW : cstride);
        } else {
            cudaFuncSetAttribute(predict_quad_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
            predict_quad_kernel<2><<<grid, 256, smem, s>>>(tp, td.c, DHW, total, w, b, nclass, logits,
                                                           cstride < 0 ? DHW : cstride);
        }
        return cudaGetLastError();
    }
    predict_kernel<<<static_cast<unsigned>((total + kThreads - 1) / kThreads), kThreads, 0, s>>>(
        tp, td.c, DHW, total, w, b, nclass, logits, cstride < 0 ? DHW : cstride);
    return cudaGetLastError();
}

cudaError_t launch_bad_init(int64_t* d_bad, cudaStream_t s) {
    bad_init_kernel<<<1, 1, 0, s>>>(d_bad);
    return cudaGetLastError();
}

}  // namespace tn
