// conv_tc.cu -- ternary conv3d on the 5th-generation tensor cores (sm_100a):
// tcgen05.mma kind::i8 implicit GEMM with int32 accumulators in TMEM and the
// fused A4 requant epilogue.
//
// The HBM format stays the paper's 2-bit sign/mask bitplanes (PAPER.md:118,
// Fig. 3 :130); {-1,0,+1} is expanded to int8 in shared memory only.  The
// product sum is the same integer as Eq. 9's popcount form:
// int8 products of ternary values accumulated exactly in int32.
//
// Implicit GEMM with tap merging along N.  For a fixed (dz, dy) the 3 dx taps
// differ only by a one-voxel shift along x, so instead of shifting the A operand
// three times they become three column blocks of B:
//     D[m][(dx,k)] += sum_c A_(dz,dy)[m][c] * W[k][c][dz][dy][dx]
// with M = 128 consecutive positions of a "row-padded" plane (each row of W
// voxels followed by one zero separator, pitch P = W + 1, so x-1 / x+1 at the row
// ends read zeros), N = 3K, and K-dim = the channels of the three dy windows of
// one plane.  The epilogue combines out[m] = D[m-1][0,:] + D[m][1,:] + D[m+1][2,:]
// with warp shuffles (rows are TMEM lanes), so each 128-row tile yields 126
// outputs.  Per tile: 3 planes x (3*C/32) MMAs of 128 x 3K x 32.
//
// CTA = 9 warps, persistent (one CTA per SM, grid = #SMs), tiles split evenly:
//   warps 0-3  epilogue: tcgen05.ld of the accumulator (one TMEM lane quadrant
//              each), dx combine, integer-threshold requant, packed stores
//   warps 4-7  producers: load packed words (coalesced 8/16 B per position),
//              expand bits -> int8 into the canonical K-major no-swizzle UMMA
//              layout, one plane (3 dy windows) per ring slot (4 slots)
//   warp 8     TMEM allocation + single-thread tcgen05.mma issue + commits
// A tile walk goes along z for fixed (n, position tile), so each input plane is
// expanded once and used by three consecutive tiles.  The filter bank (int8,
// 3 x 3C x 3K bytes) is expanded once per CTA and stays resident in smem.
#include "tn_internal.cuh"

#include <climits>

namespace tn {
namespace {

constexpr int kEpiWarps = 4;
constexpr int kProdWarps = 4;
constexpr int kThreadsTC = (kEpiWarps + kProdWarps + 1) * 32;
constexpr int kRows = 128;               // UMMA M
constexpr int kOutPerTile = kRows - 2;   // rows 1..126 are outputs
constexpr int kSlots = 4;                // plane ring
constexpr int kChunkBytes = kRows * 16;  // one 16-channel K-chunk of one window

struct TcPlan {
    int P;          // positions per padded row = Wci + 1
    int NP;         // positions per plane = Hci * P
    int NQ;         // position tiles per plane
    int64_t T;      // tiles = N * NQ * Do
    int cch[2];     // 16-channel chunks per segment
    int cch_tot;    // chunks per window (all segments)
    int nchp;       // chunks per plane slot: 3 * cch_tot rounded up to even
    int ring_bytes, w_bytes;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TN_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TN_WAIT_%=;\n\t}" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, no swizzle (canonical "interleave"
// layout: 8-row x 16-byte core matrices; rows 16 B apart, 8-row groups SBO
// apart, the two 16-byte K halves of a K=32 instruction LBO apart).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) |
           (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// Instruction descriptor: s32 accumulate, s8 x s8, both K-major, M=128, N.
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | ((128u >> 4) << 24);
}

// 16 ternary lanes (bits sh..sh+15 of a sign / mask word pair) -> 16 int8.
__device__ __forceinline__ uint4 expand16(uint32_t s, uint32_t m, int sh) {
    const uint32_t mm = m >> sh, nn = (m & ~s) >> sh;
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t mb = (((mm >> (4 * i)) & 0xFu) * 0x00204081u) & 0x01010101u;
        const uint32_t nb = (((nn >> (4 * i)) & 0xFu) * 0x00204081u) & 0x01010101u;
        o[i] = mb + nb * 0xFEu;          // +1 -> 0x01, -1 -> 0xFF, 0 -> 0x00
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

// ---------------------------------------------------------------- tile walk
struct Walk {
    int64_t t, t_end;
    int Do, NQ;
    __device__ Walk(int64_t T, int Do_, int NQ_) : Do(Do_), NQ(NQ_) {
        t = T * blockIdx.x / gridDim.x;
        t_end = T * (blockIdx.x + 1) / gridDim.x;
    }
    // next run of consecutive z for one (n, position tile); false when done
    __device__ bool next(int& n, int& tq, int& zf, int& zl) {
        if (t >= t_end) return false;
        const int64_t col = t / Do;
        zf = static_cast<int>(t - col * Do);
        const int64_t len = min(static_cast<int64_t>(Do - zf), t_end - t);
        zl = zf + static_cast<int>(len) - 1;
        n = static_cast<int>(col / NQ);
        tq = static_cast<int>(col - static_cast<int64_t>(n) * NQ);
        t += len;
        return true;
    }
};

template <int K>
__global__ void __launch_bounds__(kThreadsTC, 1)
conv_tc_kernel(const ConvDesc cd, const TcPlan pl) {
    constexpr int N = 3 * K;
    constexpr int KC = K / 16;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* s_ring = smem;                                   // [slot][chunk][128][16]
    uint8_t* s_w = smem + pl.ring_bytes;                      // [dz][chunk][N][16]
    int* s_x = reinterpret_cast<int*>(s_w + pl.w_bytes);      // [2][4][2][16] boundary rows
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_x + 2 * 4 * 2 * 16);
    uint64_t* plane_full = bars;           // [4]
    uint64_t* slot_free = bars + 4;        // [4]
    uint64_t* acc_full = bars + 8;         // [2]
    uint64_t* acc_empty = bars + 10;       // [2]
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + 12);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int slot_bytes = pl.nchp * kChunkBytes;
    const int wdz_bytes = pl.nchp * N * 16;

    // ---- one-time setup: zero the ring (padding chunks stay zero), expand the
    // packed filter bank into the B-operand image, init barriers, alloc TMEM.
    for (int i = threadIdx.x; i < pl.ring_bytes / 16; i += kThreadsTC)
        reinterpret_cast<uint4*>(s_ring)[i] = make_uint4(0u, 0u, 0u, 0u);
    {
        const int units = 3 * pl.nchp * N;  // 16-byte units (dz, chunk, n)
        for (int u = threadIdx.x; u < units; u += kThreadsTC) {
            const int nrow = u % N;
            const int ch = (u / N) % pl.nchp;
            const int dz = u / (N * pl.nchp);
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (ch < 3 * pl.cch_tot) {
                const int dy = ch / pl.cch_tot;
                int j = ch - dy * pl.cch_tot;
                const int sg = (j >= pl.cch[0]) ? 1 : 0;
                if (sg) j -= pl.cch[0];
                const int dx = nrow / K, k = nrow - dx * K;
                const int tap = (dz * 3 + dy) * 3 + dx;
                const int cw = cd.seg[sg].cw;
                const uint32_t* src = cd.seg[sg].wp + (static_cast<int64_t>(k) * 27 + tap) * 2 * cw;
                const int word = (16 * j) >> 5, sh = (16 * j) & 31;
                v = expand16(__ldg(src + word), __ldg(src + cw + word), sh);
            }
            *reinterpret_cast<uint4*>(s_w + dz * wdz_bytes + ch * (N * 16) + nrow * 16) = v;
        }
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) { mbar_init(plane_full + i, kProdWarps * 32); mbar_init(slot_free + i, 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(acc_full + i, 1); mbar_init(acc_empty + i, kEpiWarps * 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    constexpr uint32_t kTmemCols = (2 * N <= 128) ? 128 : (2 * N <= 256 ? 256 : 512);
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_proxy_async();   // ring zeros + weight image visible to the tensor core
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *s_tmem;

    if (warp >= kEpiWarps && warp < kEpiWarps + kProdWarps) {
        // ================= producers: expand one plane (3 dy windows) per slot
        const int m = threadIdx.x - kEpiWarps * 32;    // row 0..127
        Walk wk(pl.T, cd.Do, pl.NQ);
        int n, tq, zf, zl;
        uint32_t g = 0;
        while (wk.next(n, tq, zf, zl)) {
            const int q0 = tq * kOutPerTile - 1;
            for (int zp = zf - 1; zp <= zl + 1; ++zp, ++g) {
                const int s = g & 3;
                if (g >= 4) mbar_wait(slot_free + s, ((g >> 2) - 1) & 1);
                uint8_t* slot = s_ring + s * slot_bytes;
                const int zg = cd.zo_beg + zp;    // global conv-input plane
                const bool zin = zg >= 0 && zg < cd.Dci;
#pragma unroll
                for (int dy = 0; dy < 3; ++dy) {
                    const int p = q0 + (dy - 1) * pl.P + m;
                    const int y = p >= 0 ? p / pl.P : -1;
                    const int x = p - y * pl.P;
                    const bool in = zin && p >= 0 && y < cd.Hci && x < cd.Wci;
                    int choff = dy * pl.cch_tot;
                    for (int sg = 0; sg < cd.nseg; ++sg) {
                        const SegDesc& sd = cd.seg[sg];
                        uint32_t sw[2] = {0u, 0u}, mw[2] = {0u, 0u};
                        if (in) {
                            int zs = zg, ys = y, xs = x;
                            if (sd.up) { zs >>= 1; ys >>= 1; xs >>= 1; }
                            zs -= sd.zbeg;
                            if (zs >= 0 && zs < sd.D) {
                                const uint32_t* src =
                                    sd.xp + (((static_cast<int64_t>(n) * sd.D + zs) * sd.H + ys) * sd.W + xs) * 2 * sd.cw;
                                if (sd.cw == 1) {
                                    const uint2 q = __ldg(reinterpret_cast<const uint2*>(src));
                                    sw[0] = q.x; mw[0] = q.y;
                                } else {
                                    const uint4 q = __ldg(reinterpret_cast<const uint4*>(src));
                                    sw[0] = q.x; sw[1] = q.y; mw[0] = q.z; mw[1] = q.w;
                                }
                            }
                        }
                        for (int j = 0; j < pl.cch[sg]; ++j) {
                            const int word = j >> 1, sh = (j & 1) * 16;
                            const uint4 v = expand16(word ? sw[1] : sw[0], word ? mw[1] : mw[0], sh);
                            *reinterpret_cast<uint4*>(slot + (choff + j) * kChunkBytes + m * 16) = v;
                        }
                        choff += pl.cch[sg];
                    }
                }
                fence_proxy_async();
                mbar_arrive(plane_full + s);
            }
        }
    } else if (warp == 8) {
        // ================= MMA issuer (one thread)
        if (lane == 0) {
            const uint32_t idesc = idesc_i8(N);
            const uint32_t ring_a = smem_u32(s_ring), w_a = smem_u32(s_w);
            Walk wk(pl.T, cd.Do, pl.NQ);
            int n, tq, zf, zl;
            uint32_t gbase = 0, tc = 0;
            while (wk.next(n, tq, zf, zl)) {
                for (int z = zf; z <= zl; ++z, ++tc) {
                    const uint32_t a = gbase + (z - zf);
                    for (int dz = 0; dz < 3; ++dz) mbar_wait(plane_full + ((a + dz) & 3), ((a + dz) >> 2) & 1);
                    const uint32_t buf = tc & 1;
                    if (tc >= 2) mbar_wait(acc_empty + buf, ((tc >> 1) - 1) & 1);
                    tc_fence_after();
                    const uint32_t d = tmem_base + buf * N;
                    uint32_t acc = 0;
                    for (int dz = 0; dz < 3; ++dz) {
                        const uint32_t sa = ring_a + ((a + dz) & 3) * slot_bytes;
                        const uint32_t sb = w_a + dz * wdz_bytes;
                        for (int j = 0; j < pl.nchp / 2; ++j) {
                            const uint64_t ad = umma_desc(sa + 2 * j * kChunkBytes, kChunkBytes, 128);
                            const uint64_t bd = umma_desc(sb + 2 * j * N * 16, N * 16, 128);
                            tc_mma_i8(d, ad, bd, idesc, acc);
                            acc = 1;
                        }
                    }
                    tc_commit(acc_full + buf);
                    tc_commit(slot_free + (a & 3));
                    if (z == zl) {
                        tc_commit(slot_free + ((a + 1) & 3));
                        tc_commit(slot_free + ((a + 2) & 3));
                    }
                }
                gbase += (zl - zf) + 3;
            }
        }
        __syncwarp();
    } else {
        // ================= epilogue: warps 0-3, row m = 32*warp + lane
        const int q = warp;
        const int m = 32 * q + lane;
        const bool fused = cd.yp != nullptr;
        Walk wk(pl.T, cd.Do, pl.NQ);
        int n, tq, zf, zl;
        uint32_t tc = 0;
        int par = 0;
        while (wk.next(n, tq, zf, zl)) {
            const int q0 = tq * kOutPerTile - 1;
            const int p = q0 + m;
            const int y = p >= 0 ? p / pl.P : 0;
            const int x = p - y * pl.P;
            const bool vrow = m >= 1 && m <= kOutPerTile && p < pl.NP && x < cd.Wo && y < cd.Ho;
            for (int z = zf; z <= zl; ++z, ++tc) {
                const uint32_t buf = tc & 1;
                mbar_wait(acc_full + buf, (tc >> 1) & 1);
                tc_fence_after();
                const uint32_t taddr = tmem_base + (static_cast<uint32_t>(32 * q) << 16) + buf * N;
                uint32_t osw[(K + 31) / 32], omw[(K + 31) / 32];
#pragma unroll
                for (int i = 0; i < (K + 31) / 32; ++i) { osw[i] = 0u; omw[i] = 0u; }
                const int64_t vox = ((static_cast<int64_t>(n) * cd.Do + z) * cd.Ho + y) * cd.Wo + x;
#pragma unroll
                for (int kc = 0; kc < KC; ++kc) {
                    int d0[16], d1[16], d2[16];
                    tmem_ld16(taddr + 0 * K + 16 * kc, d0);
                    tmem_ld16(taddr + 1 * K + 16 * kc, d1);
                    tmem_ld16(taddr + 2 * K + 16 * kc, d2);
                    tmem_wait_ld();
                    int* xb = s_x + par * (4 * 2 * 16);
                    if (lane == 31) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) xb[(q * 2 + 0) * 16 + i] = d0[i];
                    }
                    if (lane == 0) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) xb[(q * 2 + 1) * 16 + i] = d2[i];
                    }
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    int accv[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        int up = __shfl_up_sync(0xFFFFFFFFu, d0[i], 1);
                        int dn = __shfl_down_sync(0xFFFFFFFFu, d2[i], 1);
                        if (lane == 0) up = q > 0 ? xb[((q - 1) * 2 + 0) * 16 + i] : 0;
                        if (lane == 31) dn = q < 3 ? xb[((q + 1) * 2 + 1) * 16 + i] : 0;
                        accv[i] = up + d1[i] + dn;
                    }
                    par ^= 1;
                    if (fused) {
                        // A4 (reading R5): +1 if acc >= hi; else -1 if acc <= lo; else 0
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const int k = 16 * kc + i;
                            const bool pos = accv[i] >= __ldg(cd.hi + k);
                            const bool neg = !pos && accv[i] <= __ldg(cd.lo + k);
                            osw[k >> 5] |= (pos ? 1u : 0u) << (k & 31);
                            omw[k >> 5] |= ((pos || neg) ? 1u : 0u) << (k & 31);
                        }
                    } else if (vrow && z < cd.Do) {
                        int4* dst = reinterpret_cast<int4*>(cd.y + vox * K + 16 * kc);
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            dst[i] = make_int4(accv[4 * i], accv[4 * i + 1], accv[4 * i + 2], accv[4 * i + 3]);
                    }
                }
                tc_fence_before();
                mbar_arrive(acc_empty + buf);
                if (fused && vrow) {
                    uint32_t* dst = cd.yp + vox * 2 * ((K + 31) / 32);
                    if constexpr (K <= 32) {
                        *reinterpret_cast<uint2*>(dst) = make_uint2(osw[0], omw[0]);
                    } else {
                        *reinterpret_cast<uint4*>(dst) = make_uint4(osw[0], osw[1], omw[0], omw[1]);
                    }
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
    }
}

int g_num_sms = 0;

}  // namespace

static bool plan_full(const ConvDesc& cd, TcPlan& pl) {
    if (cd.nseg < 1 || cd.nseg > 2) return false;
    for (int a = 0; a < 3; ++a)
        if (cd.s[a] != 1 || cd.p[a] != 1 || cd.dl[a] != 1) return false;
    if (cd.K != 16 && cd.K != 32 && cd.K != 48 && cd.K != 64) return false;
    pl.cch_tot = 0;
    pl.cch[1] = 0;
    for (int i = 0; i < cd.nseg; ++i) {
        const int c = cd.seg[i].c;
        if (c <= 0 || c % 16 != 0) return false;
        if ((c + 31) / 32 != cd.seg[i].cw) return false;
        pl.cch[i] = c / 16;
        pl.cch_tot += pl.cch[i];
    }
    if (pl.cch_tot > 4) return false;     // C <= 64 (resident filter bank)
    pl.nchp = (3 * pl.cch_tot + 1) & ~1;
    pl.P = cd.Wci + 1;
    const int64_t np = static_cast<int64_t>(cd.Hci) * pl.P;
    if (np > INT_MAX / 2) return false;
    pl.NP = static_cast<int>(np);
    pl.NQ = (pl.NP + kOutPerTile - 1) / kOutPerTile;
    pl.T = static_cast<int64_t>(cd.N) * pl.NQ * cd.Do;
    pl.ring_bytes = kSlots * pl.nchp * kChunkBytes;
    pl.w_bytes = 3 * pl.nchp * 3 * cd.K * 16;
    if (cd.Do != cd.Dci || cd.Ho != cd.Hci || cd.Wo != cd.Wci) return false;
    return true;
}

static size_t smem_bytes(const TcPlan& pl) {
    return static_cast<size_t>(pl.ring_bytes) + pl.w_bytes + 2 * 4 * 2 * 16 * sizeof(int) + 12 * 8 + 16;
}

bool conv_tc_supported(const ConvDesc& cd) {
    TcPlan pl{};
    if (!plan_full(cd, pl)) return false;
    return smem_bytes(pl) <= 227 * 1024 && pl.T > 0;
}

cudaError_t launch_conv_tc(const ConvDesc& cd, cudaStream_t st) {
    TcPlan pl{};
    if (!plan_full(cd, pl)) return cudaErrorNotSupported;
    const size_t smem = smem_bytes(pl);
    if (smem > 227 * 1024) return cudaErrorNotSupported;
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t grid = pl.T < g_num_sms ? pl.T : g_num_sms;
    if (grid <= 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
#define TN_TC_CASE(KV)                                                                                  \
    case KV:                                                                                            \
        e = cudaFuncSetAttribute(conv_tc_kernel<KV>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                 static_cast<int>(smem));                                               \
        if (e != cudaSuccess) return e;                                                                 \
        conv_tc_kernel<KV><<<static_cast<unsigned>(grid), kThreadsTC, smem, st>>>(cd, pl);               \
        break;
    switch (cd.K) {
        TN_TC_CASE(16)
        TN_TC_CASE(32)
        TN_TC_CASE(48)
        TN_TC_CASE(64)
        default: return cudaErrorNotSupported;
    }
#undef TN_TC_CASE
    return cudaGetLastError();
}

}  // namespace tn
