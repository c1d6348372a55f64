// conv_wide.cu -- the wide one-plane ("2D") layers of Table 1 (reading R18) on
// the tcgen05 tensor cores: C up to 512 input channels (one or two segments, each a multiple of
// 64, the first optionally nearest-x2 upsampled in y and x) and K up to 256 output channels, at
// stride 1 or 2 with pad 1 -- the layers whose filter banks do not fit shared memory next to the
// operands of the tap-offset z-merged kernel (conv_tz.cu), which ran them on the CUDA-core
// popc kernel.
//
// The arithmetic is Eq. 9 on {-1,0,+1} operands held as exact FP4 E2M1 values
// (kind::mxf4 with unit UE8M0 scales; f32 accumulation of integers < 2^24 is exact), over the
// 3x3 window of the middle kernel plane (a one-plane input meets only dz = 1; the other planes
// multiply the zero padding), followed by the fused integer thresholds (reading R5) and the
// 2-bit repack, or the int32 accumulators.
//
// Structure.  Output positions of a plane form a raster of pitch Po = Wo + 1 (one zero separator
// column per row), cut into strips of T tiles of 128 positions; a unit is (plane n, strip,
// output-channel group of N <= 128).  The contraction runs over 64-channel chunks: per chunk the
// expanders write the strip's FP4 rows (two 16-byte halves per row, stride-2 layers one image
// per input phase) and every active tap (dy, dx) of every tile is ONE 128 x N x 64 MMA whose A
// descriptor starts at the tap's row offset (the taps are descriptor offsets, as in conv_tz).
// The B operand of a chunk -- the taps' N x 64 FP4 weights -- comes from a prepared image in
// global memory ([group][chunk][active tap][half][N][16 B], built once by tz_prepare, taps whose
// weights are all zero left out: the 1x1 layers #7/#8 run one MMA per chunk), copied by one
// thread with a 1-D bulk copy into a two-slot ring.  Accumulators: one TMEM buffer of T tiles
// (or two of fewer tiles, whose epilogue then overlaps the next unit's MMAs).  One-plane layers of
// 64 channels in and out at stride 1 run here too (no z-merge: more tiles per strip than conv_tz).
//
// Warp roles: 0-7 epilogue (TMEM lane quadrant = warp % 4, column half = warp / 4), 8-15
// expanders, 16 MMA issuer (and TMEM allocation), 17 B loader.
#include "tn_internal.cuh"

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tc_ptx.cuh"

namespace tn {

struct TzPrep;   // conv_tz.cu

namespace {

constexpr int kWEpiWarps = 8;                         // two per TMEM lane quadrant (column halves)
constexpr int kWExpWarps = 8;
constexpr int kWExpThreads = kWExpWarps * 32;
constexpr int kWMmaWarp = kWEpiWarps + kWExpWarps;   // 16
constexpr int kWLoadWarp = kWMmaWarp + 1;              // 17
constexpr int kWThreads = (kWLoadWarp + 1) * 32;       // 576
constexpr int kWMaxA = 4;                              // A ring slots
constexpr int kWB = 2;                                 // B ring slots
constexpr int kWMaxN = 128;

struct WPlan {
    int s;                 // stride 1 / 2
    int N;                 // MMA N (output channels per group, 64 or 128)
    int ngroup;            // output-channel groups (ceil(K / N))
    int T;                 // tiles per strip
    int nbuf;              // TMEM accumulator buffers of T * N columns (2: a unit's epilogue overlaps
                           // the next unit's MMAs; 1: more tiles per strip, fewer halo rows and B bytes)
    int NT, nstrip, Po, RS, REG, nph;
    int nchunk;            // 64-channel chunks over both segments
    int chunk0[kMaxSeg];   // first chunk of each segment
    int ntap;              // active taps
    int8_t tap[9];         // active tap (dy * 3 + dx), ascending
    int a_row[9], a_ph[9]; // per active tap: A row offset and phase image
    int slot_bytes, nslot, b_bytes;
    int64_t units;         // N * nstrip * ngroup
    uint32_t po_magic;
    int step_q, step_r;
};

__device__ __forceinline__ int div_po_w(uint32_t q, uint32_t magic) { return static_cast<int>(__umulhi(q, magic)); }

__device__ __forceinline__ void mma_mxf4_acc(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t sfa,
                                             uint32_t sfb, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(sfa), "r"(sfb), "r"(acc)
        : "memory");
}
__host__ __device__ constexpr uint32_t idesc_w(int n) {   // E2M1 x E2M1, UE8M0 scales, K-major, M = 128
    return (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
}

// unit u of the CTA's contiguous range -> (plane n, strip, group)
struct WUnit { int n, strip, grp; };
__device__ __forceinline__ WUnit w_unit(int64_t u, const WPlan& pl) {
    WUnit r;
    r.grp = static_cast<int>(u % pl.ngroup);
    const int64_t v = u / pl.ngroup;
    r.strip = static_cast<int>(v % pl.nstrip);
    r.n = static_cast<int>(v / pl.nstrip);
    return r;
}

template <int STR, int NSEG, int N>
__global__ void __launch_bounds__(kWThreads, 1) conv_wide_kernel(const ConvDesc cd, const WPlan pl) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr int NPH = STR == 1 ? 1 : 4;
    constexpr int NW = N / 32;                                 // output words per position (sign or mask)
    uint8_t* s_b = smem;                                       // [kWB][b_bytes]
    uint8_t* s_a = s_b + kWB * pl.b_bytes;                     // [nslot][phase][2][REG]
    // per channel, as f32 bits: nh = 0.5 - hi and lmh = lo - hi + 1 (exact: |hi|, |lo| <= 2^20);
    // with d = acc + nh (never zero for integer acc): acc >= hi <=> d > 0, acc > lo <=> lmh - d < 0
    int* s_hi = reinterpret_cast<int*>(s_a + pl.nslot * pl.slot_bytes);   // [ngroup * N] nh
    int* s_lo = s_hi + pl.ngroup * N;                                      // [ngroup * N] lmh
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_lo + pl.ngroup * N);
    uint64_t* a_full = bars;                                   // [kWMaxA]
    uint64_t* a_free = a_full + kWMaxA;
    uint64_t* b_full = a_free + kWMaxA;                        // [kWB]
    uint64_t* b_free = b_full + kWB;
    uint64_t* acc_full = b_free + kWB;                         // [2]
    uint64_t* acc_empty = acc_full + 2;
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(acc_empty + 2);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const bool fused = cd.yp != nullptr;
    const int Kp = pl.ngroup * N;

    for (int k = threadIdx.x; k < Kp; k += kWThreads) {
        int h = 1 << 20, l = -(1 << 20);                      // padded channels: always 0
        if (fused && k < cd.K) { h = clamp_threshold(__ldg(cd.hi + k)); l = clamp_threshold(__ldg(cd.lo + k)); }
        s_hi[k] = __float_as_int(0.5f - static_cast<float>(h));
        s_lo[k] = __float_as_int(static_cast<float>(l - h + 1));
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < kWMaxA; ++i) { mbar_init(a_full + i, kWExpThreads); mbar_init(a_free + i, 1); }
        for (int i = 0; i < kWB; ++i) { mbar_init(b_full + i, 1); mbar_init(b_free + i, 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(acc_full + i, 1); mbar_init(acc_empty + i, kWEpiWarps * 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kWMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;
    if (warp < 4) {   // unit block scales (UE8M0 2^0) for the MMAs, columns 480..511
        int sf[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) sf[i] = 0x7F7F7F7F;
        tmem_st16(tmem + (static_cast<uint32_t>(32 * warp) << 16) + 480, sf);
        tmem_st16(tmem + (static_cast<uint32_t>(32 * warp) << 16) + 496, sf);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_launch_dependents();
    pdl_wait();   // the previous layer's activations are complete and visible from here on

    const int64_t u_beg = pl.units * blockIdx.x / gridDim.x, u_end = pl.units * (blockIdx.x + 1) / gridDim.x;
    const int T = pl.T;

    if (warp >= kWEpiWarps && warp < kWMmaWarp) {
        // ================= expanders: packed words of one 64-channel chunk -> FP4 strip rows
        const int et = threadIdx.x - kWEpiWarps * 32;
        int64_t g = 0;   // (unit, chunk) items so far
        for (int64_t u = u_beg; u < u_end; ++u) {
            const WUnit wu = w_unit(u, pl);
            const int qa = wu.strip * 128 * T - (pl.Po + 1);   // raster position of A row 0
            for (int q = 0; q < pl.nchunk; ++q, ++g) {
                const int slot = static_cast<int>(g % pl.nslot);
                if (g >= pl.nslot) mbar_wait(a_free + slot, static_cast<uint32_t>((g / pl.nslot - 1) & 1));
                const int sg = (NSEG == 2 && q >= pl.chunk0[1]) ? 1 : 0;
                const SegDesc& sd = cd.seg[sg];
                const int ql = q - pl.chunk0[sg];
                const uint32_t* base = sd.xp + static_cast<int64_t>(wu.n) * sd.H * sd.W * 2 * sd.cw;
                const uint32_t a0 = smem_u32(s_a + slot * pl.slot_bytes);
                // row r <-> output raster position qa + r = (y, x); (y, x) advance incrementally
                int r = et;
                int y, x;
                {
                    const uint32_t tq = static_cast<uint32_t>(qa + r + 2 * pl.Po);
                    y = div_po_w(tq, pl.po_magic) - 2;
                    x = static_cast<int>(tq) - (y + 2) * pl.Po;
                }
                for (; r < pl.RS; r += kWExpThreads) {
                    const bool vo = x < cd.Wo && y >= 0;
#pragma unroll
                    for (int ph = 0; ph < NPH; ++ph) {
                        const int yi = STR == 2 ? 2 * y + (ph >> 1) : y, xi = STR == 2 ? 2 * x + (ph & 1) : x;
                        const bool v = vo && yi < cd.Hci && xi < cd.Wci;
                        uint2 sw = make_uint2(0u, 0u), mw = make_uint2(0u, 0u);
                        if (v) {
                            const int ys = sd.up ? (yi >> 1) : yi, xs = sd.up ? (xi >> 1) : xi;
                            const uint32_t* p = base + (static_cast<int64_t>(ys) * sd.W + xs) * 2 * sd.cw + 2 * ql;
                            sw = __ldg(reinterpret_cast<const uint2*>(p));
                            mw = __ldg(reinterpret_cast<const uint2*>(p + sd.cw));
                        }
                        const uint32_t dst = a0 + (ph * 2) * pl.REG + r * 16;
                        sts128(dst, expand32_f4(sw.x, mw.x));
                        sts128(dst + pl.REG, expand32_f4(sw.y, mw.y));
                    }
                    x += pl.step_r;
                    y += pl.step_q;
                    if (x >= pl.Po) { x -= pl.Po; ++y; }
                }
                fence_proxy_async();
                mbar_arrive(a_full + slot);
            }
        }
    } else if (warp == kWLoadWarp) {
        // ================= B loader: the chunk's prepared taps -> B ring
        if (lane == 0) {
            int64_t g = 0;
            for (int64_t u = u_beg; u < u_end; ++u) {
                const WUnit wu = w_unit(u, pl);
                for (int q = 0; q < pl.nchunk; ++q, ++g) {
                    const int bs = static_cast<int>(g % kWB);
                    if (g >= kWB) mbar_wait(b_free + bs, static_cast<uint32_t>((g / kWB - 1) & 1));
                    mbar_arrive_expect_tx(b_full + bs, pl.b_bytes);
                    const uint8_t* src = reinterpret_cast<const uint8_t*>(cd.bimg) +
                                         (static_cast<int64_t>(wu.grp) * pl.nchunk + q) * pl.b_bytes;
                    bulk_g2s(s_b + bs * pl.b_bytes, src, pl.b_bytes, b_full + bs);
                }
            }
        }
    } else if (warp == kWMmaWarp) {
        // ================= MMA issuer
        if (elect_one()) {
            const uint32_t idesc = idesc_w(N);
            const uint32_t sfa = tmem + 480, sfb = tmem + 496;
            const uint32_t a_base = smem_u32(s_a), b_base = smem_u32(s_b);
            auto desc = [](uint32_t addr, uint32_t lbo) {
                return (static_cast<uint64_t>(0x4008u) << 32) | (((addr >> 4) & 0x3FFFu) | ((lbo >> 4) << 16));
            };
            int64_t g = 0, ui = 0;
            for (int64_t u = u_beg; u < u_end; ++u, ++ui) {
                const int buf = static_cast<int>(ui % pl.nbuf);
                if (ui >= pl.nbuf) mbar_wait(acc_empty + buf, static_cast<uint32_t>((ui / pl.nbuf - 1) & 1));
                tc_fence_after();
                const uint32_t d0 = tmem + buf * (T * N);
                for (int q = 0; q < pl.nchunk; ++q, ++g) {
                    const int slot = static_cast<int>(g % pl.nslot), bs = static_cast<int>(g % kWB);
                    mbar_wait(a_full + slot, static_cast<uint32_t>((g / pl.nslot) & 1));
                    mbar_wait(b_full + bs, static_cast<uint32_t>((g / kWB) & 1));
                    tc_fence_after();
                    const uint32_t sa = a_base + slot * pl.slot_bytes, sb = b_base + bs * pl.b_bytes;
                    for (int t = 0; t < T; ++t)
                        for (int i = 0; i < pl.ntap; ++i) {
                            const uint64_t ad = desc(sa + pl.a_ph[i] * 2 * pl.REG + (128 * t + pl.a_row[i]) * 16,
                                                     pl.REG);
                            const uint64_t bd = desc(sb + i * 2 * N * 16, N * 16);
                            mma_mxf4_acc(d0 + t * N, ad, bd, idesc, sfa, sfb, (q > 0 || i > 0) ? 1u : 0u);
                        }
                    tc_commit(a_free + slot);
                    tc_commit(b_free + bs);
                }
                tc_commit(acc_full + buf);
            }
        }
        __syncwarp();
    } else {
        // ================= epilogue (TMEM lane quadrant warp % 4, output-channel half warp / 4)
        constexpr int NH = N / 2, NWH = NW / 2;                  // channels / words per half
        const int qd = warp & 3, hf = warp >> 2;
        const uint32_t lane_base = static_cast<uint32_t>(32 * qd) << 16;
        int64_t ui = 0;
        for (int64_t u = u_beg; u < u_end; ++u, ++ui) {
            const WUnit wu = w_unit(u, pl);
            const int buf = static_cast<int>(ui % pl.nbuf);
            mbar_wait(acc_full + buf, static_cast<uint32_t>((ui / pl.nbuf) & 1));
            tc_fence_after();
            const int Tv = min(T, pl.NT - wu.strip * T);
            for (int t = 0; t < Tv; ++t) {
                const int qpos = wu.strip * 128 * T + 128 * t + 32 * qd + lane;
                const int y = div_po_w(static_cast<uint32_t>(qpos), pl.po_magic);
                const int x = qpos - y * pl.Po;
                const bool vpos = x < cd.Wo && y < cd.Ho;
                const int64_t v = (static_cast<int64_t>(wu.n) * cd.Ho + y) * cd.Wo + x;
                uint32_t sb[NWH > 0 ? NWH : 1], mb[NWH > 0 ? NWH : 1];
#pragma unroll
                for (int c = 0; c < NH; c += 16) {
                    int acc[16];
                    const int cc = hf * NH + c;                  // column / channel within the group
                    tmem_ld16(tmem + lane_base + buf * (T * N) + t * N + cc, acc);
                    tmem_wait_ld();
                    const int k0 = wu.grp * N + cc;
                    if (fused) {
                        uint32_t nhi = 0u, nlo = 0u;
#pragma unroll
                        for (int i4 = 3; i4 >= 0; --i4) {
                            const int4 h4 = *reinterpret_cast<const int4*>(s_hi + k0 + 4 * i4);
                            const int4 l4 = *reinterpret_cast<const int4*>(s_lo + k0 + 4 * i4);
                            const int hv[4] = {h4.x, h4.y, h4.z, h4.w}, lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
                            for (int j = 3; j >= 0; --j) {
                                const float d = __int_as_float(acc[4 * i4 + j]) + __int_as_float(hv[j]);
                                nhi = __funnelshift_l(static_cast<uint32_t>(__float_as_int(d)), nhi, 1);
                                nlo = __funnelshift_l(static_cast<uint32_t>(__float_as_int(__int_as_float(lv[j]) - d)),
                                                      nlo, 1);
                            }
                        }
                        const uint32_t s16 = ~nhi & 0xFFFFu, m16 = ~(nhi & nlo) & 0xFFFFu;
                        const int w = c >> 5, sh = c & 31;
                        if (sh == 0) { sb[w] = s16; mb[w] = m16; }
                        else { sb[w] |= s16 << sh; mb[w] |= m16 << sh; }
                    } else if (vpos) {
                        int32_t* dst = cd.y + v * cd.K;
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (k0 + i < cd.K) dst[k0 + i] = __float2int_rn(__int_as_float(acc[i]));
                    }
                }
                if (fused && vpos) {
                    const int w0 = wu.grp * NW + hf * NWH;        // first output word of this half
                    uint32_t* dst = cd.yp + v * 2 * cd.cwo + w0;
                    if constexpr (NH >= 32) {
#pragma unroll
                        for (int w = 0; w < NWH; ++w) {
                            if (w0 + w < cd.cwo) {
                                dst[w] = sb[w];
                                dst[cd.cwo + w] = mb[w];
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(acc_empty + buf);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kWMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// Prepared image: for active tap i of chunk q (segment sg, local chunk ql) of group g,
// half h (channels 32h..32h+31 of the chunk), row n: the FP4 weights of output channel
// g*N + n (zero rows past K), the middle kernel plane's tap (dy, dx).
__global__ void wide_image_kernel(const ConvDesc cd, const WPlan pl, uint4* out) {
    const int per_chunk = pl.ntap * 2 * pl.N;
    const int64_t total = static_cast<int64_t>(pl.ngroup) * pl.nchunk * per_chunk;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int n = static_cast<int>(e % pl.N);
        const int h = static_cast<int>((e / pl.N) % 2);
        const int i = static_cast<int>((e / (2 * pl.N)) % pl.ntap);
        const int q = static_cast<int>((e / per_chunk) % pl.nchunk);
        const int g = static_cast<int>(e / (static_cast<int64_t>(per_chunk) * pl.nchunk));
        const int k = g * pl.N + n;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (k < cd.K) {
            const int sg = (cd.nseg == 2 && q >= pl.chunk0[1]) ? 1 : 0;
            const int ql = q - pl.chunk0[sg];
            const int cw = cd.seg[sg].cw;
            const uint32_t* src = cd.seg[sg].wp + (static_cast<int64_t>(k) * 27 + 9 + pl.tap[i]) * 2 * cw;
            v = expand32_f4(src[2 * ql + h], src[cw + 2 * ql + h]);
        }
        out[e] = v;
    }
}

// taps (dy, dx) of the middle plane with any nonzero weight, as a bit mask
__global__ void wide_tapmask_kernel(const ConvDesc cd, unsigned* mask) {
    unsigned m = 0u;
    for (int sg = 0; sg < cd.nseg; ++sg) {
        const int cw = cd.seg[sg].cw;
        const int64_t total = static_cast<int64_t>(cd.K) * 9 * cw;
        for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
             e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const int w = static_cast<int>(e % cw);
            const int t = static_cast<int>((e / cw) % 9);
            const int64_t k = e / (9 * cw);
            if (cd.seg[sg].wp[(k * 27 + 9 + t) * 2 * cw + cw + w] != 0u) m |= 1u << t;   // mask word
        }
    }
    m = __reduce_or_sync(0xFFFFFFFFu, m);
    if ((threadIdx.x & 31) == 0 && m) atomicOr(mask, m);
}

size_t w_smem(const WPlan& pl) {
    return kWB * static_cast<size_t>(pl.b_bytes) + static_cast<size_t>(pl.nslot) * pl.slot_bytes +
           2 * static_cast<size_t>(pl.ngroup) * pl.N * sizeof(int) + (2 * kWMaxA + 2 * kWB + 4) * 8 + 16;
}

int w_num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0, v = 0;
        n = (cudaGetDevice(&dev) == cudaSuccess &&
             cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) ? v : 148;
        cudaGetLastError();
    }
    return n;
}

// tapmask: active taps (bit dy*3+dx); the plan's B bytes and MMA schedule follow it.
bool plan_wide(const ConvDesc& cd, unsigned tapmask, WPlan& pl) {
    constexpr size_t kSmemMax = 227 * 1024;
    if (cd.nseg < 1 || cd.nseg > 2 || cd.Dci != 1 || cd.Do != 1 || cd.zo_beg != 0) return false;
    if (cd.zstep > 1 || cd.halo_lo != nullptr || cd.halo_hi != nullptr || cd.logits != nullptr) return false;
    for (int a = 0; a < 3; ++a)
        if (cd.s[a] != cd.s[0] || cd.p[a] != 1 || cd.dl[a] != 1) return false;
    if (cd.s[0] != 1 && cd.s[0] != 2) return false;
    if (cd.K < 1 || cd.K > 256) return false;
    pl.s = cd.s[0];
    int c_tot = 0;
    pl.nchunk = 0;
    for (int i = 0; i < cd.nseg; ++i) {
        const SegDesc& sd = cd.seg[i];
        if (sd.c % 64 != 0 || sd.up == 1 || sd.D != 1 || sd.zbeg != 0) return false;
        if (i == 0 && cd.nseg == 2 && sd.up != 2) return false;
        if (i == 1 && sd.up) return false;
        if (cd.nseg == 1 && sd.up) return false;
        pl.chunk0[i] = pl.nchunk;
        pl.nchunk += sd.c / 64;
        c_tot += sd.c;
    }
    // 64 channels in and out: stride 1 only (at stride 2 the tap-offset kernel is faster, Table 1 #3)
    if (c_tot <= 64 && cd.K <= 64 && pl.s != 1) return false;
    if (cd.Ho != out_extent(cd.Hci, pl.s, 1, 1) || cd.Wo != out_extent(cd.Wci, pl.s, 1, 1)) return false;
    if (pl.s == 2 && (cd.Hci % 2 || cd.Wci % 2)) return false;
    pl.N = cd.K <= 64 ? 64 : 128;
    pl.ngroup = (cd.K + pl.N - 1) / pl.N;
    pl.nph = pl.s == 1 ? 1 : 4;
    pl.Po = cd.Wo + 1;
    const int64_t npo = static_cast<int64_t>(cd.Ho) * pl.Po;
    if (npo + 4 * pl.Po > (1 << 22) || pl.Po > 4096) return false;
    pl.NT = static_cast<int>((npo + 127) / 128);
    pl.po_magic = static_cast<uint32_t>((0x100000000ull + pl.Po - 1) / pl.Po);
    pl.step_q = kWExpThreads / pl.Po;
    pl.step_r = kWExpThreads % pl.Po;
    pl.ntap = 0;
    for (int t = 0; t < 9; ++t) {
        if (!((tapmask >> t) & 1u)) continue;
        const int dy = t / 3, dx = t % 3;
        int ph = 0, oy = dy, ox = dx;
        if (pl.s == 2) {
            const int py = dy == 1 ? 0 : 1, px = dx == 1 ? 0 : 1;
            oy = dy == 0 ? 0 : 1;
            ox = dx == 0 ? 0 : 1;
            ph = py * 2 + px;
        }
        pl.tap[pl.ntap] = static_cast<int8_t>(t);
        pl.a_ph[pl.ntap] = ph;
        pl.a_row[pl.ntap] = oy * pl.Po + ox;
        ++pl.ntap;
    }
    if (pl.ntap == 0) {   // an all-zero filter bank: one (zero) tap keeps the schedule uniform
        pl.tap[0] = 4;
        pl.a_ph[0] = 0;
        pl.a_row[0] = pl.s == 1 ? pl.Po + 1 : 0;
        pl.ntap = 1;
    }
    pl.b_bytes = pl.ntap * 2 * pl.N * 16;
    // TMEM: nbuf accumulator buffers of T * N columns below the scale columns (480..511).  One
    // buffer of more tiles measured faster on every Table-1 layer than two (the expanders and
    // the B stream bound the layers, and more tiles per strip cut both); TN_WIDE_NBUF overrides.
    static const char* env_nbuf = ab_env("TN_WIDE_NBUF");
    pl.nbuf = env_nbuf ? std::max(1, std::min(2, atoi(env_nbuf))) : 1;
    const int tmax = (pl.nbuf == 2 ? 240 : 480) / pl.N;
    int tstart = std::min(tmax, pl.NT);
    while (tstart > 1 && static_cast<int64_t>(cd.N) * ((pl.NT + tstart - 1) / tstart) * pl.ngroup < w_num_sms())
        --tstart;
    for (int T = tstart; T >= 1; --T) {
        pl.T = T;
        pl.nstrip = (pl.NT + T - 1) / T;
        pl.RS = 128 * T + (pl.s == 1 ? 2 * (pl.Po + 1) : pl.Po + 1);
        pl.REG = (pl.RS * 16 + 127) / 128 * 128;
        pl.slot_bytes = pl.nph * 2 * pl.REG;
        for (int ns = kWMaxA; ns >= 2; --ns) {
            pl.nslot = ns;
            if (w_smem(pl) <= kSmemMax) {
                pl.units = static_cast<int64_t>(cd.N) * pl.nstrip * pl.ngroup;
                return pl.units > 0;
            }
        }
    }
    return false;
}

}  // namespace

bool conv_wide_supported(const ConvDesc& cd) {
    WPlan pl{};
    return plan_wide(cd, 0x1FFu, pl);
}

// a prepared wide image (TzPrep with kind 1 in conv_tz.cu holds it)
cudaError_t wide_prepare(const ConvDesc& cd, uint4** img, int* bytes, unsigned* tapmask_out, cudaStream_t st) {
    *img = nullptr;
    *bytes = 0;
    unsigned* d_mask = nullptr;
    cudaError_t e = cudaMallocAsync(&d_mask, sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(d_mask, 0, sizeof(unsigned), st);
    wide_tapmask_kernel<<<64, 256, 0, st>>>(cd, d_mask);
    unsigned mask = 0;
    cudaMemcpyAsync(&mask, d_mask, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    cudaFreeAsync(d_mask, st);
    if (e != cudaSuccess) return e;
    WPlan pl{};
    if (!plan_wide(cd, mask, pl)) return cudaErrorNotSupported;
    const int64_t nb = static_cast<int64_t>(pl.ngroup) * pl.nchunk * pl.b_bytes;
    e = cudaMalloc(img, nb);
    if (e != cudaSuccess) return e;
    wide_image_kernel<<<256, 256, 0, st>>>(cd, pl, *img);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { cudaFree(*img); *img = nullptr; return e; }
    *bytes = static_cast<int>(nb);
    *tapmask_out = mask;
    return cudaSuccess;
}

// img: a prepared image for tapmask, or nullptr (then an image with all nine taps is built
// into stream-ordered scratch memory for this call)
cudaError_t launch_conv_wide(const ConvDesc& cd0, const uint4* img, unsigned tapmask, cudaStream_t st) {
    WPlan pl{};
    if (img == nullptr) tapmask = 0x1FFu;
    if (!plan_wide(cd0, tapmask, pl)) return cudaErrorNotSupported;
    ConvDesc cd = cd0;
    uint4* tmp = nullptr;
    if (img == nullptr) {
        const int64_t nb = static_cast<int64_t>(pl.ngroup) * pl.nchunk * pl.b_bytes;
        cudaError_t e = cudaMallocAsync(&tmp, nb, st);
        if (e != cudaSuccess) return e;
        wide_image_kernel<<<256, 256, 0, st>>>(cd, pl, tmp);
        img = tmp;
    }
    cd.bimg = img;
    void (*kern)(ConvDesc, WPlan) = nullptr;
    const int ns = cd.nseg;
    if (pl.s == 1 && ns == 1) kern = pl.N == 64 ? conv_wide_kernel<1, 1, 64> : conv_wide_kernel<1, 1, 128>;
    if (pl.s == 1 && ns == 2) kern = pl.N == 64 ? conv_wide_kernel<1, 2, 64> : conv_wide_kernel<1, 2, 128>;
    if (pl.s == 2 && ns == 1) kern = pl.N == 64 ? conv_wide_kernel<2, 1, 64> : conv_wide_kernel<2, 1, 128>;
    cudaError_t e = cudaErrorNotSupported;
    if (kern != nullptr) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e == cudaSuccess) {
            const int cap = persistent_grid_cap() > 0 ? std::min(persistent_grid_cap(), w_num_sms()) : w_num_sms();
            const int grid = static_cast<int>(std::min<int64_t>(pl.units, cap));
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(static_cast<unsigned>(grid));
            cfg.blockDim = dim3(kWThreads);
            cfg.dynamicSmemBytes = w_smem(pl);
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            e = cudaLaunchKernelEx(&cfg, kern, cd, pl);
            if (e == cudaSuccess) e = cudaGetLastError();
        }
    }
    if (tmp != nullptr) cudaFreeAsync(tmp, st);
    return e;
}

}  // namespace tn
