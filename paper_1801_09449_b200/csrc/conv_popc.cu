// conv_popc.cu -- ternary 3x3x3 convolution as Eq. 9's masked Hamming distance
// on the CUDA cores, with the fused A4 requant epilogue.
//
// Per (output voxel, output channel k, tap, word):
//     m   = mA & mW                 (joint nonzero support; reading R1: AND mask)
//     d   = m & (sA ^ sW)           (opposite signs)
//     acc += popc(m) - 2*popc(d)    (= popc(m & ~(sA^sW)) - popc(m & (sA^sW)), Eq. 9)
// accumulated in int32 (|acc| <= 27*C).
//
// Structure: one CTA = 128 threads = an output tile of 512 voxels (TX x TY x TZ)
// of one batch item, all K output channels.  The packed input brick (tile +
// halo, every segment, with the nearest-x2 upsample gather and zero padding
// applied while staging) and the packed filter banks live in shared memory;
// each thread owns 4 voxels and loops K in chunks of 8 channels, so one
// 128-bit LDS of activation words feeds 8 channels and one broadcast LDS of
// weight words feeds 4 voxels.  The requant epilogue sets output bits in a
// shared staging tile that is written back with 8/16-byte stores.
#include "tn_internal.cuh"

#include <climits>

namespace tn {
namespace {

constexpr int kThreads = 128;
constexpr int kVPT = 4;             // voxels per thread
constexpr int kTile = kThreads * kVPT;
constexpr int kKC = 8;              // output channels per register chunk

struct Tiling {
    int TX, TY, TZ;                 // output tile
    int BX, BY, BZ;                 // input brick (conv-input coordinates)
    int tiles_x, tiles_y, tiles_z;
    int a0, a1;                     // kernel planes dz in [a0, a1] that can meet data (2D: only dz = 1)
};

template <int CW>
struct Words { uint32_t s[CW]; uint32_t m[CW]; };

template <int CW>
__device__ __forceinline__ Words<CW> lds_words(const uint32_t* p) {
    Words<CW> r;
    if constexpr (CW == 1) {
        const uint2 q = *reinterpret_cast<const uint2*>(p);
        r.s[0] = q.x; r.m[0] = q.y;
    } else if constexpr (CW == 2) {
        const uint4 q = *reinterpret_cast<const uint4*>(p);
        r.s[0] = q.x; r.s[1] = q.y; r.m[0] = q.z; r.m[1] = q.w;
    } else {
#pragma unroll
        for (int j = 0; j < CW; j += 4) {
            const uint4 a = *reinterpret_cast<const uint4*>(p + j);
            const uint4 b = *reinterpret_cast<const uint4*>(p + CW + j);
            r.s[j] = a.x; r.s[j + 1] = a.y; r.s[j + 2] = a.z; r.s[j + 3] = a.w;
            r.m[j] = b.x; r.m[j + 1] = b.y; r.m[j + 2] = b.z; r.m[j + 3] = b.w;
        }
    }
    return r;
}

// Stage one segment's brick: brick voxel (bz,by,bx) <-> conv-input coordinate
// (zi0+bz, yi0+by, xi0+bx); out-of-range coordinates are zero padding (all bits
// clear = ternary 0); upsampled segments read source voxel (z>>1, y>>1, x>>1).
template <int CW>
__device__ void stage_brick(uint32_t* __restrict__ dst, const SegDesc& sg, const ConvDesc& cd,
                            int n, int zi0, int yi0, int xi0, int BX, int BY, int BZ) {
    const int nb = BX * BY * BZ;
    for (int i = threadIdx.x; i < nb; i += kThreads) {
        const int bx = i % BX;
        const int by = (i / BX) % BY;
        const int bz = i / (BX * BY);
        const int zi = zi0 + bz, yi = yi0 + by, xi = xi0 + bx;
        uint32_t* d = dst + static_cast<int64_t>(i) * 2 * CW;
        bool inb = zi >= 0 && zi < cd.Dci && yi >= 0 && yi < cd.Hci && xi >= 0 && xi < cd.Wci;
        int zs = zi, ys = yi, xs = xi;
        if (sg.up == 1) zs >>= 1;              // up 2: nearest x2 in y and x only
        if (sg.up) { ys >>= 1; xs >>= 1; }
        zs -= sg.zbeg;
        inb = inb && zs >= 0 && zs < sg.D && ys < sg.H && xs < sg.W;
        if (inb) {
            const uint32_t* src = sg.xp +
                ((((static_cast<int64_t>(n) * sg.D + zs) * sg.H + ys) * sg.W + xs) * 2 * CW);
            if constexpr (CW == 1) {
                *reinterpret_cast<uint2*>(d) = __ldg(reinterpret_cast<const uint2*>(src));
            } else {
#pragma unroll
                for (int j = 0; j < 2 * CW; j += 4)
                    *reinterpret_cast<uint4*>(d + j) = __ldg(reinterpret_cast<const uint4*>(src + j));
            }
        } else {
            if constexpr (CW == 1) {
                *reinterpret_cast<uint2*>(d) = make_uint2(0u, 0u);
            } else {
#pragma unroll
                for (int j = 0; j < 2 * CW; j += 4)
                    *reinterpret_cast<uint4*>(d + j) = make_uint4(0u, 0u, 0u, 0u);
            }
        }
    }
}

template <int CW>
__global__ void __launch_bounds__(kThreads)
conv_popc_kernel(const ConvDesc cd, const Tiling tl, int Kpad) {
    extern __shared__ __align__(16) uint32_t smem[];
    const int brick_words = (tl.BX * tl.BY * tl.BZ * 2 * CW + 3) & ~3;   // 16-byte aligned
    const int wt_words = kKC * 27 * 2 * CW;                     // one chunk of kKC output channels
    uint32_t* s_brick = smem;                                   // [nseg][brick]
    uint32_t* s_w = s_brick + cd.nseg * brick_words;            // [nseg][kKC][27][2CW]
    const bool fused = cd.yp != nullptr;
    uint32_t* s_out = s_w + cd.nseg * wt_words;                 // [kTile][2][cwo] (fused only)

    int t = blockIdx.x;
    const int tx = t % tl.tiles_x; t /= tl.tiles_x;
    const int ty = t % tl.tiles_y; t /= tl.tiles_y;
    const int tz = t % tl.tiles_z; t /= tl.tiles_z;
    const int n = t;
    const int zo0 = tz * tl.TZ, yo0 = ty * tl.TY, xo0 = tx * tl.TX;
    // (2D tiles stage only the one input plane the middle kernel plane reads)
    const int zi0 = (cd.zo_beg + zo0) * cd.s[0] - cd.p[0] + tl.a0 * cd.dl[0];
    const int yi0 = yo0 * cd.s[1] - cd.p[1];
    const int xi0 = xo0 * cd.s[2] - cd.p[2];

    for (int sgi = 0; sgi < cd.nseg; ++sgi)
        stage_brick<CW>(s_brick + sgi * brick_words, cd.seg[sgi], cd, n, zi0, yi0, xi0,
                        tl.BX, tl.BY, tl.BZ);
    // filter banks chunk by chunk of kKC output channels (K real rows, zero rows up to Kpad),
    // so wide banks (Table 1's 256 x 512 x 27) need only one chunk of shared memory
    auto stage_weights = [&](int k0) {
        for (int sgi = 0; sgi < cd.nseg; ++sgi) {
            const int real_words = min(cd.K - k0, kKC) * 27 * 2 * CW;
            const uint32_t* wsrc = cd.seg[sgi].wp + static_cast<int64_t>(k0) * 27 * 2 * CW;
            uint32_t* wdst = s_w + sgi * wt_words;
            if ((real_words & 3) == 0) {
                for (int i = threadIdx.x; i < wt_words / 4; i += kThreads)
                    reinterpret_cast<uint4*>(wdst)[i] = 4 * i < real_words
                        ? __ldg(reinterpret_cast<const uint4*>(wsrc) + i) : make_uint4(0u, 0u, 0u, 0u);
            } else {
                for (int i = threadIdx.x; i < wt_words; i += kThreads) wdst[i] = i < real_words ? __ldg(wsrc + i) : 0u;
            }
        }
    };
    (void)Kpad;
    if (fused) {
        for (int i = threadIdx.x; i < kTile * 2 * cd.cwo; i += kThreads) s_out[i] = 0u;
    }

    // this thread's voxels
    int boff[kVPT];
    bool valid[kVPT];
    int64_t vox[kVPT];
#pragma unroll
    for (int i = 0; i < kVPT; ++i) {
        const int lin = threadIdx.x + kThreads * i;
        const bool in_tile = lin < tl.TX * tl.TY * tl.TZ;        // 2D tiles can hold fewer than kTile voxels
        const int ox = lin % tl.TX;
        const int oy = (lin / tl.TX) % tl.TY;
        const int oz = in_tile ? lin / (tl.TX * tl.TY) : 0;
        boff[i] = in_tile ? ((oz * cd.s[0]) * tl.BY + oy * cd.s[1]) * tl.BX + ox * cd.s[2] : 0;
        const int zo = zo0 + oz, yo = yo0 + oy, xo = xo0 + ox;
        valid[i] = in_tile && zo < cd.Do && yo < cd.Ho && xo < cd.Wo;
        vox[i] = (((static_cast<int64_t>(n) * cd.Do + zo) * cd.Ho + yo) * cd.Wo + xo);
    }
    const int step_z = cd.dl[0] * tl.BY * tl.BX, step_y = cd.dl[1] * tl.BX, step_x = cd.dl[2];

    for (int k0 = 0; k0 < cd.K; k0 += kKC) {
        if (k0 > 0) __syncthreads();          // everyone is done with the previous chunk
        stage_weights(k0);
        __syncthreads();
        int acc[kVPT][kKC];
#pragma unroll
        for (int i = 0; i < kVPT; ++i)
#pragma unroll
            for (int kk = 0; kk < kKC; ++kk) acc[i][kk] = 0;

        for (int sgi = 0; sgi < cd.nseg; ++sgi) {
            const uint32_t* bb = s_brick + sgi * brick_words;
            const uint32_t* wb = s_w + sgi * wt_words;
#pragma unroll 1
            for (int tap = 9 * tl.a0; tap < 9 * (tl.a1 + 1); ++tap) {
                const int a = tap / 9, b = (tap / 3) % 3, e = tap % 3;
                const int toff = (a - tl.a0) * step_z + b * step_y + e * step_x;
                Words<CW> av[kVPT];
#pragma unroll
                for (int i = 0; i < kVPT; ++i) av[i] = lds_words<CW>(bb + (boff[i] + toff) * 2 * CW);
#pragma unroll
                for (int kk = 0; kk < kKC; ++kk) {
                    const Words<CW> wv = lds_words<CW>(wb + (kk * 27 + tap) * 2 * CW);
#pragma unroll
                    for (int i = 0; i < kVPT; ++i) {
#pragma unroll
                        for (int j = 0; j < CW; ++j) {
                            const uint32_t m = av[i].m[j] & wv.m[j];
                            const uint32_t d = (av[i].s[j] ^ wv.s[j]) & m;
                            acc[i][kk] += __popc(m) - 2 * __popc(d);
                        }
                    }
                }
            }
        }

        if (!fused) {
#pragma unroll
            for (int i = 0; i < kVPT; ++i) {
                if (!valid[i]) continue;
                int32_t* dst = cd.y + vox[i] * cd.K + k0;
                if (k0 + kKC <= cd.K && (cd.K % 4) == 0) {
                    reinterpret_cast<int4*>(dst)[0] = make_int4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
                    reinterpret_cast<int4*>(dst)[1] = make_int4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
                } else {
#pragma unroll
                    for (int kk = 0; kk < kKC; ++kk)
                        if (k0 + kk < cd.K) dst[kk] = acc[i][kk];
                }
            }
        } else {
            // A4 epilogue (reading R5): +1 if acc >= hi; else -1 if acc <= lo; else 0.
            const int j = k0 >> 5;
            uint32_t sbits[kVPT], mbits[kVPT];
#pragma unroll
            for (int i = 0; i < kVPT; ++i) { sbits[i] = 0u; mbits[i] = 0u; }
#pragma unroll
            for (int kk = 0; kk < kKC; ++kk) {
                const int k = k0 + kk;
                if (k >= cd.K) break;
                const int32_t hi = __ldg(cd.hi + k), lo = __ldg(cd.lo + k);
                const uint32_t bit = 1u << (k & 31);
#pragma unroll
                for (int i = 0; i < kVPT; ++i) {
                    const bool pos = acc[i][kk] >= hi;
                    const bool neg = !pos && acc[i][kk] <= lo;
                    sbits[i] |= pos ? bit : 0u;
                    mbits[i] |= (pos || neg) ? bit : 0u;
                }
            }
#pragma unroll
            for (int i = 0; i < kVPT; ++i) {
                const int lin = threadIdx.x + kThreads * i;
                s_out[(lin * 2) * cd.cwo + j] |= sbits[i];
                s_out[(lin * 2 + 1) * cd.cwo + j] |= mbits[i];
            }
        }
    }

    if (fused) {
        // each thread owns its voxels' staging words: no barrier needed
#pragma unroll
        for (int i = 0; i < kVPT; ++i) {
            if (!valid[i]) continue;
            const int lin = threadIdx.x + kThreads * i;
            const uint32_t* src = s_out + lin * 2 * cd.cwo;
            uint32_t* dst = cd.yp + vox[i] * 2 * cd.cwo;
            if (cd.cwo == 1) {
                *reinterpret_cast<uint2*>(dst) = make_uint2(src[0], src[1]);
            } else if (cd.cwo == 2) {
                *reinterpret_cast<uint4*>(dst) = make_uint4(src[0], src[1], src[2], src[3]);
            } else {
                for (int q = 0; q < 2 * cd.cwo; ++q) dst[q] = src[q];
            }
            if (cd.halo_lo != nullptr || cd.halo_hi != nullptr) {   // NEXT-1 slab boundary planes (N = 1)
                const int64_t hw = static_cast<int64_t>(cd.Ho) * cd.Wo;
                const int zo = static_cast<int>((vox[i] / hw) % cd.Do);
                halo_store_words(cd.halo_lo, cd.halo_hi, zo, cd.Do, vox[i] % hw, src, 2 * cd.cwo);
            }
        }
    }
}

// ----------------------------------------------------------------------------
// First layer (A7): Eq. 6 on the float input (reading R7) fused with the conv
// from one channel and the A4 epilogue.  With C = 1 the 27 taps are packed into
// one word per voxel (tap t -> bit t), so each output channel costs
// 2 LOP3 + 2 POPC.  Tile 512 voxels; brick of int8 codes in shared memory.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
conv_first_kernel(const FirstDesc fd, const Tiling tl) {
    extern __shared__ __align__(16) uint32_t smem[];
    int8_t* s_code = reinterpret_cast<int8_t*>(smem);                      // [BZ][BY][BX]
    const int nb = tl.BX * tl.BY * tl.BZ;
    uint32_t* s_wt = smem + (nb + 3) / 4;                                   // [K][2] tap-packed
    __shared__ int64_t s_bad;

    int t = blockIdx.x;
    const int tx = t % tl.tiles_x; t /= tl.tiles_x;
    const int ty = t % tl.tiles_y; t /= tl.tiles_y;
    const int tz = t % tl.tiles_z; t /= tl.tiles_z;
    const int n = t;
    const int zo0 = tz * tl.TZ, yo0 = ty * tl.TY, xo0 = tx * tl.TX;
    const int zi0 = (fd.zo_beg + zo0) * fd.s[0] - fd.p[0];
    const int yi0 = yo0 * fd.s[1] - fd.p[1];
    const int xi0 = xo0 * fd.s[2] - fd.p[2];
    if (threadIdx.x == 0) s_bad = LLONG_MAX;
    __syncthreads();

    int64_t bad = LLONG_MAX;
    for (int i = threadIdx.x; i < nb; i += kThreads) {
        const int bx = i % tl.BX;
        const int by = (i / tl.BX) % tl.BY;
        const int bz = i / (tl.BX * tl.BY);
        const int zg = zi0 + bz, yi = yi0 + by, xi = xi0 + bx;
        const int zb = zg - fd.zbeg;
        int8_t code = 0;
        if (zg >= 0 && zg < fd.Dg && yi >= 0 && yi < fd.H && xi >= 0 && xi < fd.W && zb >= 0 && zb < fd.D) {
            const int64_t off = ((static_cast<int64_t>(n) * fd.D + zb) * fd.H + yi) * fd.W + xi;
            const float v = __ldg(fd.x + off);
            if (!isfinite(v)) {
                bad = min(bad, static_cast<int64_t>(n) * fd.bad_nstride + fd.bad_base +
                                   (static_cast<int64_t>(zb) * fd.H + yi) * fd.W + xi);
            }
            code = v > fd.t_hi ? 1 : (v < fd.t_lo ? -1 : 0);
        }
        s_code[i] = code;
    }
    // tap-packed weights: one thread per (k, tap) loads its word pair in parallel
    for (int i = threadIdx.x; i < 2 * fd.K; i += kThreads) s_wt[i] = 0u;
    __syncthreads();
    for (int i = threadIdx.x; i < 27 * fd.K; i += kThreads) {
        const int k = i / 27, tap = i - 27 * k;
        const uint2 q = __ldg(reinterpret_cast<const uint2*>(fd.wp + i * 2));
        if (q.x & 1u) atomicOr(s_wt + 2 * k, 1u << tap);
        if (q.y & 1u) atomicOr(s_wt + 2 * k + 1, 1u << tap);
    }
    if (bad != LLONG_MAX) atomicMin(reinterpret_cast<long long*>(&s_bad), static_cast<long long>(bad));
    __syncthreads();
    if (threadIdx.x == 0 && s_bad != LLONG_MAX && fd.d_bad != nullptr)
        atomicMin(reinterpret_cast<long long*>(fd.d_bad), static_cast<long long>(s_bad));

    for (int i = 0; i < kVPT; ++i) {
        const int lin = threadIdx.x + kThreads * i;
        const int ox = lin % tl.TX;
        const int oy = (lin / tl.TX) % tl.TY;
        const int oz = lin / (tl.TX * tl.TY);
        const int zo = zo0 + oz, yo = yo0 + oy, xo = xo0 + ox;
        if (zo >= fd.Do || yo >= fd.Ho || xo >= fd.Wo) continue;
        const int base = ((oz * fd.s[0]) * tl.BY + oy * fd.s[1]) * tl.BX + ox * fd.s[2];
        uint32_t as = 0, am = 0;
#pragma unroll
        for (int tap = 0; tap < 27; ++tap) {
            const int a = tap / 9, b = (tap / 3) % 3, e = tap % 3;
            const int8_t c = s_code[base + (a * fd.dl[0] * tl.BY + b * fd.dl[1]) * tl.BX + e * fd.dl[2]];
            as |= (c == 1 ? 1u : 0u) << tap;
            am |= (c != 0 ? 1u : 0u) << tap;
        }
        uint32_t os = 0, om = 0;
        for (int k = 0; k < fd.K; ++k) {
            const uint32_t m = am & s_wt[2 * k + 1];
            const uint32_t d = (as ^ s_wt[2 * k]) & m;
            const int acc = __popc(m) - 2 * __popc(d);
            const bool pos = acc >= __ldg(fd.hi + k);
            const bool neg = !pos && acc <= __ldg(fd.lo + k);
            os |= (pos ? 1u : 0u) << k;
            om |= ((pos || neg) ? 1u : 0u) << k;
        }
        const int64_t v = ((static_cast<int64_t>(n) * fd.Do + zo) * fd.Ho + yo) * fd.Wo + xo;
        *reinterpret_cast<uint2*>(fd.yp + v * 2) = make_uint2(os, om);
        if (fd.halo_lo != nullptr || fd.halo_hi != nullptr) {   // NEXT-1 slab boundary planes (N = 1)
            const uint32_t wds[2] = {os, om};
            halo_store_words(fd.halo_lo, fd.halo_hi, zo, fd.Do, static_cast<int64_t>(yo) * fd.Wo + xo, wds, 2);
        }
    }
}

// two_d: one output plane whose only input plane is met by the middle kernel plane (one-plane
// volumes with pad = dilation in z: Table 1's 2D layers) -> one-plane tiles, 9 taps.
Tiling make_tiling(int Do, int Ho, int Wo, int N, const int* s, const int* dl, int tx_pref, bool two_d = false) {
    Tiling tl;
    tl.TX = tx_pref;
    while (tl.TX > 4 && tl.TX / 2 >= Wo) tl.TX /= 2;
    int rest = kTile / tl.TX;
    tl.TY = two_d ? rest : 8;
    while (tl.TY > 1 && tl.TY / 2 >= Ho) tl.TY /= 2;
    if (tl.TY > rest) tl.TY = rest;
    tl.TZ = rest / tl.TY;
    if (two_d) tl.TZ = 1;
    tl.a0 = two_d ? 1 : 0;
    tl.a1 = two_d ? 1 : 2;
    tl.BX = (tl.TX - 1) * s[2] + 2 * dl[2] + 1;
    tl.BY = (tl.TY - 1) * s[1] + 2 * dl[1] + 1;
    tl.BZ = two_d ? 1 : (tl.TZ - 1) * s[0] + 2 * dl[0] + 1;
    tl.tiles_x = (Wo + tl.TX - 1) / tl.TX;
    tl.tiles_y = (Ho + tl.TY - 1) / tl.TY;
    tl.tiles_z = (Do + tl.TZ - 1) / tl.TZ;
    (void)N;
    return tl;
}

template <int CW>
cudaError_t launch_popc_cw(const ConvDesc& cd, cudaStream_t st) {
    const bool two_d = cd.Do == 1 && cd.Dci == 1 && cd.zo_beg == 0 && cd.p[0] == cd.dl[0];
    const Tiling tl = make_tiling(cd.Do, cd.Ho, cd.Wo, cd.N, cd.s, cd.dl, 16, two_d);
    const int Kpad = (cd.K + kKC - 1) / kKC * kKC;
    const int brick_words = (tl.BX * tl.BY * tl.BZ * 2 * CW + 3) & ~3;
    size_t smem = sizeof(uint32_t) * (static_cast<size_t>(cd.nseg) * (brick_words + kKC * 27 * 2 * CW));
    if (cd.yp) smem += sizeof(uint32_t) * kTile * 2 * cd.cwo;
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(conv_popc_kernel<CW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int64_t blocks = static_cast<int64_t>(tl.tiles_x) * tl.tiles_y * tl.tiles_z * cd.N;
    if (blocks == 0) return cudaSuccess;
    if (blocks > INT_MAX) return cudaErrorInvalidConfiguration;
    conv_popc_kernel<CW><<<static_cast<unsigned>(blocks), kThreads, smem, st>>>(cd, tl, Kpad);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_conv_popc(const ConvDesc& cd, cudaStream_t st) {
    switch (cd.seg[0].cw) {
        case 1: return launch_popc_cw<1>(cd, st);
        case 2: return launch_popc_cw<2>(cd, st);
        case 4: return launch_popc_cw<4>(cd, st);
        case 8: return launch_popc_cw<8>(cd, st);     // up to 256 channels per segment (Table 1's widest)
        default: return cudaErrorNotSupported;
    }
}

cudaError_t launch_conv_first(const FirstDesc& fd, cudaStream_t st) {
    // tensor-core path (conv_tz.cu) where it covers the shape, else the popc kernel below
    if (first_kernel_tz_allowed() && conv_tz_first_supported(fd)) return launch_conv_tz_first(fd, st);
    const Tiling tl = make_tiling(fd.Do, fd.Ho, fd.Wo, fd.N, fd.s, fd.dl, 32);
    const int nb = tl.BX * tl.BY * tl.BZ;
    const size_t smem = sizeof(uint32_t) * ((nb + 3) / 4 + 2 * fd.K);
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(conv_first_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int64_t blocks = static_cast<int64_t>(tl.tiles_x) * tl.tiles_y * tl.tiles_z * fd.N;
    if (blocks == 0) return cudaSuccess;
    conv_first_kernel<<<static_cast<unsigned>(blocks), kThreads, smem, st>>>(fd, tl);
    return cudaGetLastError();
}

}  // namespace tn
