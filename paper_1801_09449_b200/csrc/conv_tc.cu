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
// CTA = 13 warps, persistent (one CTA per SM, grid = #SMs), tiles split evenly:
//   warps 0-7  epilogue: tcgen05.ld of the accumulator (two warps per TMEM lane
//              quadrant, each owning half of the output channels), dx combine
//              with warp shuffles, integer-threshold requant, packed stores
//   warps 8-11 producers: load packed words one plane ahead into registers
//              (coalesced 8/16 B per position), expand bits -> int8 into the
//              canonical K-major no-swizzle UMMA layout, one plane (the 3 dy
//              windows) per ring slot (4-8 slots, as shared memory allows)
//   warp 12    TMEM allocation + single-thread tcgen05.mma issue + commits
// A tile walk goes along z for fixed (n, position tile), so each input plane is
// expanded once and used by three consecutive tiles.  The filter bank (int8,
// 3 x 3C x 3K bytes) is expanded once per CTA and stays resident in smem.
// Tiles are 4 runs of 32 rows (one per lane quadrant) overlapping by 2, so each
// output's x-neighbours live in its own warp: 120 outputs per 128-row tile.
#include "tn_internal.cuh"
#include "tc_ptx.cuh"

#include <algorithm>
#include <climits>

#ifndef TN_EXP_NOPROD
#define TN_EXP_NOPROD 0
#endif
#ifndef TN_EXP_NOFENCE
#define TN_EXP_NOFENCE 0
#endif
#ifndef TN_EXP_NOEPI
#define TN_EXP_NOEPI 0
#endif
#ifndef TN_EXP_TRACE
#define TN_EXP_TRACE 0
#endif
#ifndef TN_EXP_NOLOAD
#define TN_EXP_NOLOAD 0
#endif
#ifndef TN_EXP_PROF
#define TN_EXP_PROF 0
#endif
#if TN_EXP_TRACE || TN_EXP_PROF
__device__ long long g_trace[4096];
#define SSTAMP(i) do { if (threadIdx.x == 0) g_trace[2560 + 8 * blockIdx.x + (i)] = clock64() - k_begin; } while (0)
#endif
#if TN_EXP_PROF
#define PSTAMP(v) long long v = clock64()
#define PACC(acc, t0) acc += clock64() - (t0)
#else
#define PSTAMP(v) do { } while (0)
#define PACC(acc, t0) do { } while (0)
#endif
#if TN_EXP_TRACE
#define TRACE(i, cond) do { if ((cond) && blockIdx.x == 0 && (i) < 2048) g_trace[(i)] = clock64(); } while (0)
#else
#define TRACE(i, cond) do { } while (0)
#endif

namespace tn {
namespace {

constexpr int kEpiWarps = 8;             // 2 per TMEM lane quadrant (K split in halves)
constexpr int kLoadWarps = 4;            // cp.async packed rows -> staging (one row per thread)
constexpr int kExpWarps = 8;             // staging -> int8 UMMA layout: two groups of 4 (one row per
                                         // thread) expanding alternate planes
constexpr int kLoadWarp0 = kEpiWarps;
constexpr int kExpWarp0 = kEpiWarps + kLoadWarps;
constexpr int kMmaWarp = kEpiWarps + kLoadWarps + kExpWarps;
constexpr int kThreadsTC = (kMmaWarp + 1) * 32;
constexpr int kMaxStage = 16;
constexpr int kMaxClass = 8;
constexpr int kRows = 128;               // UMMA M
constexpr int kOutPerWarp = 30;          // lanes 1..30 of each 32-row run are outputs
constexpr int kOutPerTile = 4 * kOutPerWarp;
constexpr int kChunkBytes = kRows * 16;  // one 16-channel K-chunk of one window

// Row m of a tile <-> position q0 + row_pos(m): four runs of 32 consecutive
// positions, one per TMEM lane quadrant, overlapping by two so that every
// output row (lanes 1..30) has both x-neighbours inside its own warp.
__host__ __device__ __forceinline__ int row_pos(int m) { return kOutPerWarp * (m >> 5) + (m & 31) - 1; }

struct TcPlan {
    int P;          // positions per padded row = Wci + 1
    int NP;         // positions per plane = Hci * P
    int NQ;         // position tiles per plane
    int s;          // stride (1 or 2, all axes)
    int ntx;        // stride 2: position tiles per (even) conv-input row
    int64_t T;      // tiles = N * NQ * Do
    int cch[2];     // 16-channel chunks per segment
    int cch_tot;    // chunks per window (all segments)
    int nchp;       // chunks per plane slot: 3 * cch_tot rounded up to even
    int nslot;      // plane ring depth (4..8)
    int nstage;     // packed staging depth (2..4)
    int stage_bytes;
    int ring_bytes, w_bytes;
    int ptab_floats;    // fused-prediction quad tables (0 if not fused)
    int wstage;         // packed weights staged through the ring during setup
};
constexpr int kMaxSlots = 16;
constexpr int kMaxAcc = 4;

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

// First position (row-padded conv-input plane) of position tile tq.  Stride 1:
// tiles are contiguous runs of the plane; stride 2: tiles cover the even rows
// only (the output rows), ntx tiles per row.
__device__ __forceinline__ int tile_q0(const TcPlan& pl, int tq) {
    if (pl.s == 1) return tq * kOutPerTile;
    const int yr = tq / pl.ntx;
    return 2 * yr * pl.P + (tq - yr * pl.ntx) * kOutPerTile;
}

// Producer-side walk over the planes a CTA expands, in order: for each run of
// tiles (z in [zf, zl]) the planes zf-1 .. zl+1.  Per run it caches each row's
// (y, x) offsets in the three dy windows (per segment).
struct PlaneCursor {
    Walk wk;
    int n, tq, zf, zl, zp;
    bool valid;
    int yx[3][kMaxSeg];
    bool ok[3];
    __device__ PlaneCursor(const TcPlan& pl, const ConvDesc& cd, int m) : wk(pl.T, cd.Do, pl.NQ) {
        valid = wk.next(n, tq, zf, zl);
        if (valid) start_run(pl, cd, m);
    }
    __device__ void start_run(const TcPlan& pl, const ConvDesc& cd, int m) {
        zp = pl.s * zf - 1;          // conv-input planes s*zf-1 .. s*zl+1 of this run
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) {
            const int p = tile_q0(pl, tq) + row_pos(m) + (dy - 1) * pl.P;
            const int y = p >= 0 ? p / pl.P : -1;
            const int x = p - y * pl.P;
            ok[dy] = p >= 0 && y < cd.Hci && x < cd.Wci;
#pragma unroll
            for (int sg = 0; sg < kMaxSeg; ++sg) {
                const SegDesc& sd = cd.seg[sg];
                const int ys = sd.up ? (y >> 1) : y, xs = sd.up ? (x >> 1) : x;
                yx[dy][sg] = ys * sd.W + xs;
            }
        }
    }
    __device__ void advance(const TcPlan& pl, const ConvDesc& cd, int m) {
        if (++zp > pl.s * zl + 1) {
            valid = wk.next(n, tq, zf, zl);
            if (valid) start_run(pl, cd, m);
        }
    }
};

template <int K, int NSEG, int CT, int STR>
__global__ void __launch_bounds__(kThreadsTC, 1)
conv_tc_kernel(const ConvDesc cd, const TcPlan pl) {
    constexpr int N = 3 * K;
    constexpr int NCHP = (3 * CT + 1) & ~1;   // chunks per plane slot (== NCHP)
    constexpr int HALF = NCHP / 2;            // K=32 MMAs per plane
    // macro tile: ZT consecutive output planes share one MMA round / barrier set;
    // two macro buffers of ZT accumulators of N columns fit in TMEM (<= 384 of 512)
    constexpr int ZT = K == 16 ? 4 : (K == 32 ? 2 : 1);
    constexpr int PB = 1;                     // planes per producer batch
    constexpr int PMAX = STR * (ZT - 1) + 3;  // conv-input planes read by a full macro tile
    constexpr int CWO = (K + 31) / 32;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* s_ring = smem;                                   // [slot][chunk][128][16]
    uint8_t* s_w = smem + pl.ring_bytes;                      // [dz][chunk][N][16]
    uint8_t* s_stage = s_w + pl.w_bytes;                      // [stage][seg][dy][128][16] packed rows
    int* s_lo = reinterpret_cast<int*>(s_stage + pl.nstage * pl.stage_bytes);  // [K]
    int* s_hi = s_lo + K;                                     // [K]
    float* s_pred = reinterpret_cast<float*>(s_hi + K);       // [kMaxClass] bias, then quad tables
    float* s_ptab = s_pred + kMaxClass;                       // [nclass][K/4][256] (fused A8 only)
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_ptab + pl.ptab_floats);
    uint64_t* plane_full = bars;                           // [kMaxSlots]
    uint64_t* slot_free = bars + kMaxSlots;                // [kMaxSlots]
    uint64_t* acc_full = bars + 2 * kMaxSlots;             // [kMaxAcc]
    uint64_t* acc_empty = bars + 2 * kMaxSlots + kMaxAcc;  // [kMaxAcc]
    uint64_t* staged_full = bars + 2 * kMaxSlots + 2 * kMaxAcc;           // [kMaxStage]
    uint64_t* staged_empty = staged_full + kMaxStage;                      // [kMaxStage]
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(staged_empty + kMaxStage);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    constexpr int slot_bytes = NCHP * kChunkBytes;
    constexpr int wdz_bytes = NCHP * N * 16;
    const bool fused = cd.yp != nullptr;
#if TN_EXP_PROF
    const long long k_begin = clock64();
#endif

    // ---- one-time setup: expand the packed filter bank into the B-operand image.
    // The packed words are first staged (cp.async, all in flight at once) in the
    // ring, which is unused until the roles start; each (k, tap) word pair is then
    // expanded once into its CT 16-channel units.  The ring needs no zeroing: the
    // B rows of a padding chunk are zero, so whatever A holds there adds 0.
    {
        int lo_r = 0, hi_r = 0;
        if (fused && threadIdx.x < K) {
            lo_r = clamp_threshold(__ldg(cd.lo + threadIdx.x));
            hi_r = clamp_threshold(__ldg(cd.hi + threadIdx.x));
        }
        const uint32_t* wsrc[kMaxSeg];
        {
            uint32_t* s_wp = reinterpret_cast<uint32_t*>(s_ring);
            int ofs = 0;
#pragma unroll
            for (int sg = 0; sg < NSEG; ++sg) {
                wsrc[sg] = cd.seg[sg].wp;
                if (pl.wstage) {
                    const int n4 = K * 27 * 2 * cd.seg[sg].cw / 4;     // uint4 units (K % 16 == 0)
                    const uint4* g = reinterpret_cast<const uint4*>(cd.seg[sg].wp);
                    for (int i = threadIdx.x; i < n4; i += kThreadsTC)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s_wp + ofs + 4 * i)),
                                     "l"(g + i) : "memory");
                    wsrc[sg] = s_wp + ofs;
                    ofs += 4 * n4;
                }
            }
            asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
        }
        if (fused && threadIdx.x < K) { s_lo[threadIdx.x] = lo_r; s_hi[threadIdx.x] = hi_r; }
        __syncthreads();
#if TN_EXP_PROF
        SSTAMP(0);
#endif
#pragma unroll
        for (int sg = 0; sg < NSEG; ++sg) {
            const int cw = cd.seg[sg].cw, cch = pl.cch[sg], choff = sg ? pl.cch[0] : 0;
            for (int pr = threadIdx.x; pr < K * 27; pr += kThreadsTC) {
                // consecutive threads take consecutive k of one tap: conflict-free 16-byte stores
                const int tap = pr / K, k = pr - K * tap;
                const int dz = tap / 9, dy = (tap / 3) % 3, dx = tap % 3;
                const uint32_t* src = wsrc[sg] + (k * 27 + tap) * 2 * cw;
                uint32_t sw[2], mw[2];
                if (cw == 1) {
                    const uint2 t = *reinterpret_cast<const uint2*>(src);
                    sw[0] = t.x; mw[0] = t.y; sw[1] = mw[1] = 0u;
                } else {
                    const uint4 t = *reinterpret_cast<const uint4*>(src);
                    sw[0] = t.x; sw[1] = t.y; mw[0] = t.z; mw[1] = t.w;
                }
                uint8_t* dst = s_w + dz * wdz_bytes + (dy * CT + choff) * (N * 16) + (dx * K + k) * 16;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (j < cch)
                        *reinterpret_cast<uint4*>(dst + j * (N * 16)) = expand16(sw[j >> 1], mw[j >> 1], 16 * (j & 1));
            }
        }
        if (NCHP > 3 * CT)
            for (int u = threadIdx.x; u < 3 * N; u += kThreadsTC)
                *reinterpret_cast<uint4*>(s_w + (u / N) * wdz_bytes + (3 * CT) * (N * 16) + (u % N) * 16) =
                    make_uint4(0u, 0u, 0u, 0u);
        __syncthreads();   // the staged words in the ring are dead from here on
    }
#if TN_EXP_PROF
    SSTAMP(1);
    SSTAMP(2);
#endif
    if (fused && cd.logits != nullptr) {
        for (int i = threadIdx.x; i < cd.nclass; i += kThreadsTC) s_pred[i] = __ldg(cd.pb + i);
        // quad tables: entry (mask nibble | sign nibble << 4) = (((t0 w0) + t1 w1) + t2 w2) + t3 w3
        for (int e = threadIdx.x; e < cd.nclass * (K / 4) * 256; e += kThreadsTC) {
            const int idx = e & 255, qd = (e >> 8) % (K / 4), j = e / (256 * (K / 4));
            float part = 0.0f;
            for (int i = 0; i < 4; ++i) {
                const float wv = __ldg(cd.pw + j * K + 4 * qd + i);
                const bool nz = (idx >> i) & 1, ps = (idx >> (4 + i)) & 1;
                part += nz ? (ps ? wv : -wv) : 0.0f;
            }
            s_ptab[e] = part;
        }
    }
    {   // one barrier per thread (a serial init loop costs ~1 us)
        const int t = threadIdx.x;
        if (t < kMaxSlots) { mbar_init(plane_full + t, kRows); mbar_init(slot_free + t, 1); }
        else if (t < kMaxSlots + kMaxStage) {
            mbar_init(staged_full + t - kMaxSlots, kLoadWarps * 32);
            mbar_init(staged_empty + t - kMaxSlots, kRows);
        } else if (t < kMaxSlots + kMaxStage + kMaxAcc) {
            mbar_init(acc_full + t - kMaxSlots - kMaxStage, 1);
            mbar_init(acc_empty + t - kMaxSlots - kMaxStage, kEpiWarps * 32);
        }
        if (t < kMaxSlots + kMaxStage + kMaxAcc) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
#if TN_EXP_PROF
    SSTAMP(3);
#endif
    constexpr uint32_t kTmemCols = (2 * ZT * N <= 128) ? 128 : (2 * ZT * N <= 256 ? 256 : 512);
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
#if TN_EXP_PROF
    SSTAMP(4);
#endif
    fence_proxy_async();   // ring zeros + weight image visible to the tensor core
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *s_tmem;
    pdl_launch_dependents();
    pdl_wait();   // activations of the previous layer are complete and visible from here on
#if TN_EXP_PROF
    if (threadIdx.x == 0) g_trace[16 * blockIdx.x + 14] = clock64() - k_begin;
#endif

    uint32_t total_planes = 0;
    if (warp >= kLoadWarp0 && warp < kMmaWarp) {
        Walk wk(pl.T, cd.Do, pl.NQ);
        int n, tq, zf, zl;
        while (wk.next(n, tq, zf, zl)) total_planes += pl.s * (zl - zf) + 3;
    }
    if (warp >= kLoadWarp0 && warp < kExpWarp0) {
        // ================= loaders: cp.async each row's packed words of one plane
        // (3 dy windows x segments) into a staging slot; zero-fill outside the
        // volume.  Completion is signalled on staged_full by the async unit, so
        // these threads never stall on the loads and run up to nstage planes ahead.
        const int m = threadIdx.x - kLoadWarp0 * 32;
        PlaneCursor cur(pl, cd, m);
        const uint32_t NS = pl.nstage;
#if TN_EXP_PROF
        long long l_wait = 0;
        const long long l_begin = clock64();
#endif
        // incremental ring bookkeeping (no integer divisions in the loop)
        uint32_t st = 0, st_round = 0;
        for (uint32_t g = 0; g < total_planes; ++g) {
            {
                PSTAMP(l0);
                if (st_round > 0) mbar_wait(staged_empty + st, (st_round - 1) & 1);
                PACC(l_wait, l0);
                const int zg = pl.s * cd.zo_beg + cur.zp;   // global conv-input plane
                const bool zin = zg >= 0 && zg < cd.Dci;
#pragma unroll
                for (int sg = 0; sg < NSEG; ++sg) {
                    const SegDesc& sd = cd.seg[sg];
                    const int zs = (sd.up ? (zg >> 1) : zg) - sd.zbeg;
                    const bool zok = zin && zs >= 0 && zs < sd.D;
                    const int64_t pbase = (static_cast<int64_t>(cur.n) * sd.D + zs) * sd.H * sd.W;
#pragma unroll
                    for (int dy = 0; dy < 3; ++dy) {
                        const bool ok = zok && cur.ok[dy];
                        const uint32_t* src = ok ? sd.xp + (pbase + cur.yx[dy][sg]) * 2 * sd.cw : sd.xp;
                        const uint32_t dst =
                            smem_u32(s_stage + st * pl.stage_bytes + ((sg * 3 + dy) * kRows + m) * 16);
#if TN_EXP_NOLOAD
                        if (ok && reinterpret_cast<uintptr_t>(src) == 1) asm volatile("trap;");
                        continue;
#endif
                        if (sd.cw == 1)
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
                                         "r"(ok ? 8 : 0) : "memory");
                        else
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                                         "r"(ok ? 16 : 0) : "memory");
                    }
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(staged_full + st))
                             : "memory");
                TRACE(1200 + g, g < 64 && m == 0);
                cur.advance(pl, cd, m);
                if (++st == NS) { st = 0; ++st_round; }
            }
        }
#if TN_EXP_PROF
        if (m == 0) {
            long long* o = g_trace + 16 * blockIdx.x;
            o[12] = clock64() - l_begin; o[13] = l_wait;
        }
#endif
    } else if (warp >= kExpWarp0 && warp < kMmaWarp) {
        // ================= expanders: staging (packed) -> ring slot (int8, UMMA
        // K-major no-swizzle layout), then the generic->async proxy fence.  These
        // threads have no global loads in flight, so the fence is cheap.
        const int m = (threadIdx.x - kExpWarp0 * 32) & (kRows - 1);
        const uint32_t eg = (warp - kExpWarp0) >> 2;     // this group expands planes g % 2 == eg
        const uint32_t S = pl.nslot, NS = pl.nstage;
#if TN_EXP_PROF
        long long e_staged = 0, e_slot = 0, e_work = 0, e_fence = 0;
        const long long e_begin = clock64();
#endif
        // Planes in batches of PB: one wait per barrier kind and one proxy fence per
        // batch (barriers of both rings complete in plane order, so waiting for
        // the batch's last plane covers the earlier ones).
        // incremental ring bookkeeping (no integer divisions in the loop): plane g
        // uses stage st (round st_r) and ring slot sl (round sl_r); this group
        // steps g by 2
        uint32_t st = eg, st_r = 0, sl = eg, sl_r = 0;
        for (uint32_t g0 = eg; g0 < total_planes; g0 += 2) {
            const uint32_t nb = 1;
            TRACE(1000 + 2 * g0, g0 < 64 && m == 0);
            PSTAMP(p0);
            mbar_wait(staged_full + st, st_r & 1);
            PACC(e_staged, p0);
            TRACE(1001 + 2 * g0, g0 < 64 && m == 0);
            PSTAMP(p1);
            if (sl_r > 0) mbar_wait(slot_free + sl, (sl_r - 1) & 1);
            PACC(e_slot, p1);
            TRACE(601 + 2 * g0, g0 < 64 && m == 0);
            PSTAMP(p2);
            for (uint32_t g = g0; g < g0 + nb; ++g) {
                uint4 v[NSEG][3];
#pragma unroll
                for (int sg = 0; sg < NSEG; ++sg)
#pragma unroll
                    for (int dy = 0; dy < 3; ++dy)
                        v[sg][dy] = *reinterpret_cast<const uint4*>(s_stage + st * pl.stage_bytes +
                                                                    ((sg * 3 + dy) * kRows + m) * 16);
                mbar_arrive(staged_empty + st);
                uint8_t* slot = s_ring + sl * slot_bytes + m * 16;
#if TN_EXP_NOPROD
                if (v[0][0].x == 0x12345u)
#endif
#pragma unroll
                for (int sg = 0; sg < NSEG; ++sg) {
                    const int choff = sg ? pl.cch[0] : 0;
                    const int cch = pl.cch[sg];
                    const bool two = cd.seg[sg].cw == 2;
#pragma unroll
                    for (int dy = 0; dy < 3; ++dy) {
                        const uint4 q = v[sg][dy];
                        const uint32_t s0 = q.x, m0 = two ? q.z : q.y, s1 = q.y, m1 = q.w;
                        uint8_t* dst = slot + (dy * CT + choff) * kChunkBytes;
                        *reinterpret_cast<uint4*>(dst) = expand16(s0, m0, 0);
                        if (cch > 1) *reinterpret_cast<uint4*>(dst + kChunkBytes) = expand16(s0, m0, 16);
                        if (cch > 2) *reinterpret_cast<uint4*>(dst + 2 * kChunkBytes) = expand16(s1, m1, 0);
                        if (cch > 3) *reinterpret_cast<uint4*>(dst + 3 * kChunkBytes) = expand16(s1, m1, 16);
                    }
                }
            }
            PACC(e_work, p2);
            PSTAMP(p3);
            fence_proxy_async();
            PACC(e_fence, p3);
            mbar_arrive(plane_full + sl);
            TRACE(800 + g0, g0 < 64 && m == 0);
            st += 2;
            if (st >= NS) { st -= NS; ++st_r; }
            sl += 2;
            if (sl >= S) { sl -= S; ++sl_r; }
        }
#if TN_EXP_PROF
        if (m == 0) {
            long long* o = g_trace + 16 * blockIdx.x;
            o[0] = clock64() - e_begin; o[1] = e_staged; o[2] = e_slot; o[3] = e_work; o[4] = e_fence;
            o[5] = total_planes;
        }
#endif
    } else if (warp == kMmaWarp) {
        // ================= MMA issuer: the whole warp walks the schedule (so
        // descriptors stay warp-uniform, in uniform registers) and one elected
        // lane issues each tcgen05.mma / tcgen05.commit.
        const uint32_t idesc = idesc_i8(N);
        const uint64_t adesc0 = umma_desc(smem_u32(s_ring), kChunkBytes, 128);
        const uint64_t bdesc0 = umma_desc(smem_u32(s_w), N * 16, 128);
        const bool leader = elect_one();
        Walk wk(pl.T, cd.Do, pl.NQ);
        int n, tq, zf, zl;
        const uint32_t S = pl.nslot;
        const uint64_t aslot = static_cast<uint64_t>(slot_bytes >> 4);   // descriptor step per ring slot
        // Incremental ring / accumulator bookkeeping (no divisions in the loop):
        // plane a (first plane of the current macro tile) lives in slot sa, phase pa.
        uint32_t sa = 0, pa = 0, buf = 0, round = 0, mt = 0;
#if TN_EXP_PROF
        long long m_accw = 0, m_planew = 0;
        const long long m_begin = clock64();
#endif
        auto next_slot = [S](uint32_t sl, uint32_t ph, uint32_t& sl2, uint32_t& ph2) {
            sl2 = sl + 1;
            ph2 = ph;
            if (sl2 == S) { sl2 = 0; ph2 ^= 1u; }
        };
        while (wk.next(n, tq, zf, zl)) {
            for (int z = zf; z <= zl; z += ZT, ++mt) {
                const int zt = min(ZT, zl - z + 1);          // output planes in this macro tile
                const int np = STR * (zt - 1) + 3;           // conv-input planes it reads: a .. a+np-1
                uint32_t sl[PMAX], ph[PMAX];
                sl[0] = sa;
                ph[0] = pa;
#pragma unroll
                for (int i = 1; i < PMAX; ++i) next_slot(sl[i - 1], ph[i - 1], sl[i], ph[i]);
                TRACE(5 * mt + 0, mt < 64 && leader);
                PSTAMP(q0);
                if (round > 0) mbar_wait(acc_empty + buf, (round - 1) & 1);
                PACC(m_accw, q0);
                TRACE(5 * mt + 1, mt < 64 && leader);
                // each expander group completes its planes in order, so waiting for
                // the newest plane of each group (a+np-1 and a+np-2) covers all of them
                uint32_t s_new = sl[PMAX - 1], p_new = ph[PMAX - 1], s_prv = sl[PMAX - 2], p_prv = ph[PMAX - 2];
#pragma unroll
                for (int i = 2; i < PMAX; ++i)
                    if (i == np - 1) { s_new = sl[i]; p_new = ph[i]; s_prv = sl[i - 1]; p_prv = ph[i - 1]; }
                PSTAMP(q1);
                mbar_wait(plane_full + s_prv, p_prv);
                mbar_wait(plane_full + s_new, p_new);
                PACC(m_planew, q1);
                TRACE(5 * mt + 2, mt < 64 && leader);
                tc_fence_after();
                if (leader) {
#pragma unroll
                    for (int zz = 0; zz < ZT; ++zz) {
                        if (zz < zt) {
                            const uint32_t d = tmem_base + (buf * ZT + zz) * N;
#pragma unroll
                            for (int dz = 0; dz < 3; ++dz) {
                                const uint64_t ad = adesc0 + sl[STR * zz + dz] * aslot;
                                const uint64_t bd = bdesc0 + static_cast<uint64_t>((dz * wdz_bytes) >> 4);
#pragma unroll
                                for (int j = 0; j < HALF; ++j)
                                    tc_mma_i8(d, ad + static_cast<uint64_t>((2 * j * kChunkBytes) >> 4),
                                              bd + static_cast<uint64_t>((2 * j * N * 16) >> 4), idesc,
                                              (dz | j) != 0);
                            }
                        }
                    }
                    tc_commit(acc_full + buf);
                    const bool last = (z + zt - 1 == zl);
#pragma unroll
                    for (int i = 0; i < PMAX; ++i) {
                        // planes a .. a+STR*zt-1 are not needed by the next macro tile; at
                        // the end of the run none of this tile's planes is
                        if (i < STR * zt || (last && i < np)) tc_commit(slot_free + sl[i]);
                    }
                }
                __syncwarp();
                TRACE(320 + mt, mt < 64 && leader);
                // advance to plane a + STR*zt
#pragma unroll
                for (int i = 1; i < PMAX; ++i)
                    if (i == STR * zt) { sa = sl[i]; pa = ph[i]; }
                buf ^= 1u;
                if (buf == 0) ++round;
            }
            // the run's remaining planes (a+STR*zt .. a+np-1 of its last macro tile)
#pragma unroll
            for (int i = 0; i < 3 - STR; ++i) {
                uint32_t t1, qq1;
                next_slot(sa, pa, t1, qq1);
                sa = t1;
                pa = qq1;
            }
        }
#if TN_EXP_PROF
        if (leader) {
            long long* o = g_trace + 16 * blockIdx.x;
            o[6] = clock64() - m_begin; o[7] = m_accw; o[8] = m_planew; o[9] = mt;
        }
#endif
    } else {
        // ================= epilogue: warps 0-7 = two groups of four (one warp per
        // TMEM lane quadrant q).  K <= 32: group h takes the macro tile's planes
        // zz with zz % 2 == h (all channels); K = 64 (one plane per macro tile):
        // group h takes channels [32h, 32h + 32).
        const int q = warp & 3;
        const int h = warp >> 2;
        const int kc0 = (K > 32) ? 2 * h : 0;
        const int word = (K > 32) ? h : 0;
        Walk wk(pl.T, cd.Do, pl.NQ);
        int n, tq, zf, zl;
        uint32_t buf = 0, round = 0, mt = 0;
#if TN_EXP_PROF
        long long ep_wait = 0;
        const long long ep_begin = clock64();
#endif
        while (wk.next(n, tq, zf, zl)) {
            const int p = tile_q0(pl, tq) + row_pos(32 * q + lane);
            const int yi = p >= 0 ? p / pl.P : 0;      // conv-input coordinates of this row
            const int xi = p - yi * pl.P;
            const bool ctr = STR == 1 || ((yi | xi) & 1) == 0;    // stride 2: even-even centres only
            const int y = yi / STR, x = xi / STR;                    // output coordinates
            const bool vpos = lane >= 1 && lane <= kOutPerWarp && p < pl.NP && ctr && xi < cd.Wci &&
                              yi < cd.Hci && x < cd.Wo && y < cd.Ho;
            for (int z = zf; z <= zl; z += ZT, ++mt) {
                const int zt = min(ZT, zl - z + 1);
                PSTAMP(r0);
                mbar_wait(acc_full + buf, round & 1);
                PACC(ep_wait, r0);
                TRACE(400 + mt, mt < 64 && threadIdx.x == 1);
                tc_fence_after();
#pragma unroll
                for (int zz = 0; zz < ZT; ++zz) {
                    const bool mine = zz < zt && (K > 32 || (zz & 1) == h);
                    if (!mine) continue;
                    const uint32_t taddr =
                        tmem_base + (static_cast<uint32_t>(32 * q) << 16) + (buf * ZT + zz) * N;
                    const int zo = z + zz;
                    const int64_t vox = ((static_cast<int64_t>(n) * cd.Do + zo) * cd.Ho + y) * cd.Wo + x;
                    uint32_t nhi = 0u, nlo = 0u;   // collected high channel first (see below)
#pragma unroll
                    for (int cc = 1; cc >= 0; --cc) {
                        const int kc = kc0 + cc;
                        if (16 * kc >= K) continue;
#if TN_EXP_NOEPI
                        if (mt != 0xFFFFFFFFu) break;
#endif
                        // out[m] = D[m-1][dx=0] + D[m][dx=1] + D[m+1][dx=2] (rows = lanes)
                        int accv[16], dd[16];
                        tmem_ld16(taddr + 1 * K + 16 * kc, accv);
                        tmem_ld16(taddr + 0 * K + 16 * kc, dd);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i) accv[i] += __shfl_up_sync(0xFFFFFFFFu, dd[i], 1);
                        tmem_ld16(taddr + 2 * K + 16 * kc, dd);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i) accv[i] += __shfl_down_sync(0xFFFFFFFFu, dd[i], 1);
                        if (cd.y_in != nullptr && vpos) {   // partial sums of an earlier channel split
                            const int4* src = reinterpret_cast<const int4*>(cd.y_in + vox * K + 16 * kc);
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const int4 t = __ldg(src + i);
                                accv[4 * i] += t.x; accv[4 * i + 1] += t.y;
                                accv[4 * i + 2] += t.z; accv[4 * i + 3] += t.w;
                            }
                        }
                        if (fused) {
                            // A4 (reading R5): +1 if acc >= hi; else -1 if acc <= lo; else 0.
                            // Sign bits of (acc - hi) and (lo - acc) are shifted in with funnel
                            // shifts, channels high to low: bit i of nhi = (acc_i < hi_i),
                            // bit i of nlo = (acc_i > lo_i); then sign = ~nhi, mask = ~(nhi & nlo).
#pragma unroll
                            for (int i4 = 3; i4 >= 0; --i4) {
                                const int4 h4 = *reinterpret_cast<const int4*>(s_hi + 16 * kc + 4 * i4);
                                const int4 l4 = *reinterpret_cast<const int4*>(s_lo + 16 * kc + 4 * i4);
                                const int hh[4] = {h4.x, h4.y, h4.z, h4.w}, ll[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
                                for (int i = 3; i >= 0; --i) {
                                    const int a = accv[4 * i4 + i];
                                    nhi = __funnelshift_l(static_cast<uint32_t>(a - hh[i]), nhi, 1);
                                    nlo = __funnelshift_l(static_cast<uint32_t>(ll[i] - a), nlo, 1);
                                }
                            }
                        } else if (vpos) {
                            int4* dst = reinterpret_cast<int4*>(cd.y + vox * K + 16 * kc);
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                dst[i] = make_int4(accv[4 * i], accv[4 * i + 1], accv[4 * i + 2], accv[4 * i + 3]);
                        }
                    }
                    // channels were shifted in from the highest present one down to the
                    // word's channel 0; the word holds min(K - 32*word, 32) channels
                    const uint32_t sbits = fused ? ~nhi & (K - 32 * word >= 32 ? 0xFFFFFFFFu : ((1u << (K - 32 * word)) - 1u)) : 0u;
                    const uint32_t mbits = fused ? ~(nhi & nlo) & (K - 32 * word >= 32 ? 0xFFFFFFFFu : ((1u << (K - 32 * word)) - 1u)) : 0u;
                    if (fused && vpos && cd.logits != nullptr) {
                        // A8 (reading R12): b + sum_k w_k t_k in fp32, k ascending -- the
                        // same operations as predict_kernel; K <= 32 so this warp holds all k
                        const int64_t v = (static_cast<int64_t>(zo) * cd.Ho + y) * cd.Wo + x;
                        for (int j = 0; j < cd.nclass; ++j) {
                            float acc = s_pred[j];
                            const float* tab = s_ptab + j * (K / 4) * 256;
#pragma unroll
                            for (int qd = 0; qd < (K < 32 ? K : 32) / 4; ++qd) {
                                const uint32_t idx = ((mbits >> (4 * qd)) & 0xFu) | (((sbits >> (4 * qd)) & 0xFu) << 4);
                                acc += tab[qd * 256 + idx];
                            }
                            cd.logits[(static_cast<int64_t>(n) * cd.nclass + j) * cd.lstride + v] = acc;
                        }
                    }
                    if (fused && vpos && !(cd.logits != nullptr && cd.no_yp)) {
                        uint32_t* dst = cd.yp + vox * 2 * CWO;
                        if constexpr (CWO == 1) {
                            *reinterpret_cast<uint2*>(dst) = make_uint2(sbits, mbits);
                        } else {
                            dst[word] = sbits;
                            dst[CWO + word] = mbits;
                        }
                        if (cd.halo_lo != nullptr || cd.halo_hi != nullptr) {   // NEXT-1 slab boundary planes
                            const int64_t voff = static_cast<int64_t>(y) * cd.Wo + x;
                            uint32_t* hl = cd.halo_lo ? cd.halo_lo + voff * 2 * CWO + (CWO == 1 ? 0 : word) : nullptr;
                            uint32_t* hh = cd.halo_hi ? cd.halo_hi + voff * 2 * CWO + (CWO == 1 ? 0 : word) : nullptr;
                            const uint32_t wds[2] = {sbits, mbits};
                            if (CWO == 1) {
                                halo_store_words(hl, hh, zo, cd.Do, 0, wds, 2);
                            } else {   // this warp's word of each bitplane
                                halo_store_words(hl, hh, zo, cd.Do, 0, wds, 1);
                                halo_store_words(hl ? hl + CWO : nullptr, hh ? hh + CWO : nullptr, zo, cd.Do, 0, wds + 1, 1);
                            }
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(acc_empty + buf);
                TRACE(500 + mt, mt < 64 && threadIdx.x == 1);
                buf ^= 1u;
                if (buf == 0) ++round;
            }
        }
#if TN_EXP_PROF
        if (threadIdx.x == 0) {
            long long* o = g_trace + 16 * blockIdx.x;
            o[10] = clock64() - ep_begin; o[11] = ep_wait;
        }
#endif
    }

    tc_fence_before();
    __syncthreads();
#if TN_EXP_PROF
    if (threadIdx.x == 0) g_trace[16 * blockIdx.x + 15] = clock64() - k_begin;
#endif
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
    }
}

int g_num_sms = 0;

}  // namespace

static bool plan_full(const ConvDesc& cd, TcPlan& pl) {
    if (cd.nseg < 1 || cd.nseg > 2) return false;
    for (int a = 0; a < 3; ++a)
        if (cd.s[a] != cd.s[0] || cd.p[a] != 1 || cd.dl[a] != 1) return false;
    if (cd.s[0] != 1 && !(cd.s[0] == 2 && cd.nseg == 1)) return false;
    if (cd.K != 16 && cd.K != 32 && cd.K != 64) return false;
    pl.s = cd.s[0];
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
    pl.ntx = (cd.Wci + kOutPerTile - 1) / kOutPerTile;
    pl.NQ = pl.s == 1 ? (pl.NP + kOutPerTile - 1) / kOutPerTile : ((cd.Hci + 1) / 2) * pl.ntx;
    pl.T = static_cast<int64_t>(cd.N) * pl.NQ * cd.Do;
    pl.w_bytes = 3 * pl.nchp * 3 * cd.K * 16;
    const int slot_bytes = pl.nchp * kChunkBytes;
    pl.ptab_floats = cd.logits != nullptr ? cd.nclass * (cd.K / 4) * 256 : 0;
    const int fixed = pl.w_bytes + 2 * cd.K * 4 + (kMaxClass + pl.ptab_floats) * 4 +
                      (2 * kMaxSlots + 2 * kMaxAcc + 2 * kMaxStage) * 8 + 64;
    pl.stage_bytes = cd.nseg * 3 * kRows * 16;
    // ring depth: at least the macro tile's ZT + 2 planes + 1 being filled; packed
    // staging depth: deep enough to cover HBM/L2 latency (the loaders run ahead)
    const int zt = cd.K == 16 ? 4 : (cd.K == 32 ? 2 : 1);
    const int pmax = pl.s * (zt - 1) + 3;
    pl.nslot = std::min(kMaxSlots, pmax + pl.s * zt + 2);
    pl.nstage = kMaxStage;
    while (fixed + pl.nslot * slot_bytes + pl.nstage * pl.stage_bytes > 225 * 1024) {
        if (pl.nstage > 8) --pl.nstage;
        else if (pl.nslot > pmax + 1) --pl.nslot;
        else if (pl.nstage > 2) --pl.nstage;
        else return false;
    }
    pl.ring_bytes = pl.nslot * slot_bytes;
    {
        int64_t wbytes = 0;
        bool al = true;
        for (int i = 0; i < cd.nseg; ++i) {
            wbytes += static_cast<int64_t>(cd.K) * 27 * 2 * cd.seg[i].cw * 4;
            al = al && (reinterpret_cast<uintptr_t>(cd.seg[i].wp) & 15) == 0;
        }
        pl.wstage = al && wbytes <= pl.ring_bytes;
        if (!pl.wstage) return false;   // the setup stages the packed filter bank in the ring
    }
    if (cd.Do != out_extent(cd.Dci, pl.s, 1, 1) || cd.Ho != out_extent(cd.Hci, pl.s, 1, 1) ||
        cd.Wo != out_extent(cd.Wci, pl.s, 1, 1))
        return false;
    return true;
}

// Launched with programmatic stream serialisation (PDL): the setup overlaps the previous kernel's tail.
static cudaError_t launch_one(void (*kern)(ConvDesc, TcPlan), const ConvDesc& cd, const TcPlan& pl, int64_t grid,
                              size_t smem, cudaStream_t st) {
    // cudaFuncSetAttribute is a slow host call: raise the kernel's smem limit once
    // to the maximum instead of per launch.
    static void* configured[48] = {nullptr};
    bool done = false;
    for (void* f : configured) done = done || f == reinterpret_cast<void*>(kern);
    if (!done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        for (void*& f : configured)
            if (f == nullptr) { f = reinterpret_cast<void*>(kern); break; }
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kThreadsTC);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // see pdl_wait in the kernel
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, cd, pl);
}

template <int K>
static cudaError_t dispatch_ct(const ConvDesc& cd, const TcPlan& pl, int64_t grid, size_t smem, cudaStream_t st) {
    if (cd.nseg == 1 && pl.s == 1) {
        switch (pl.cch_tot) {
            case 1: return launch_one(conv_tc_kernel<K, 1, 1, 1>, cd, pl, grid, smem, st);
            case 2: return launch_one(conv_tc_kernel<K, 1, 2, 1>, cd, pl, grid, smem, st);
            case 3: return launch_one(conv_tc_kernel<K, 1, 3, 1>, cd, pl, grid, smem, st);
            case 4: return launch_one(conv_tc_kernel<K, 1, 4, 1>, cd, pl, grid, smem, st);
        }
    } else if (cd.nseg == 1) {
        switch (pl.cch_tot) {
            case 1: return launch_one(conv_tc_kernel<K, 1, 1, 2>, cd, pl, grid, smem, st);
            case 2: return launch_one(conv_tc_kernel<K, 1, 2, 2>, cd, pl, grid, smem, st);
            case 3: return launch_one(conv_tc_kernel<K, 1, 3, 2>, cd, pl, grid, smem, st);
            case 4: return launch_one(conv_tc_kernel<K, 1, 4, 2>, cd, pl, grid, smem, st);
        }
    } else {
        switch (pl.cch_tot) {
            case 2: return launch_one(conv_tc_kernel<K, 2, 2, 1>, cd, pl, grid, smem, st);
            case 3: return launch_one(conv_tc_kernel<K, 2, 3, 1>, cd, pl, grid, smem, st);
            case 4: return launch_one(conv_tc_kernel<K, 2, 4, 1>, cd, pl, grid, smem, st);
        }
    }
    return cudaErrorNotSupported;
}

static size_t smem_bytes(const TcPlan& pl, int K) {
    return static_cast<size_t>(pl.ring_bytes) + pl.w_bytes + static_cast<size_t>(pl.nstage) * pl.stage_bytes +
           2 * K * sizeof(int) + (kMaxClass + pl.ptab_floats) * sizeof(float) +
           (2 * kMaxSlots + 2 * kMaxAcc + 2 * kMaxStage) * 8 + 16;
}

bool conv_tc_supported(const ConvDesc& cd) {
    if (cd.logits != nullptr &&
        (cd.K > 32 || cd.nclass < 1 || cd.nclass > kMaxClass || cd.yp == nullptr || cd.nclass * cd.K > 64))
        return false;   // quad tables: nclass * K/4 * 1 KB <= 16 KB
    TcPlan pl{};
    if (!plan_full(cd, pl)) return false;
    return smem_bytes(pl, cd.K) <= 227 * 1024 && pl.T > 0;
}

cudaError_t launch_conv_tc(const ConvDesc& cd, cudaStream_t st) {
    TcPlan pl{};
    if (!plan_full(cd, pl)) return cudaErrorNotSupported;
    const size_t smem = smem_bytes(pl, cd.K);
    if (smem > 227 * 1024) return cudaErrorNotSupported;
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int cap = persistent_grid_cap() > 0 ? std::min(persistent_grid_cap(), g_num_sms) : g_num_sms;
    const int64_t grid = pl.T < cap ? pl.T : cap;
    if (grid <= 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    switch (cd.K) {
        case 16: e = dispatch_ct<16>(cd, pl, grid, smem, st); break;
        case 32: e = dispatch_ct<32>(cd, pl, grid, smem, st); break;
        case 64: e = dispatch_ct<64>(cd, pl, grid, smem, st); break;
        default: return cudaErrorNotSupported;
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace tn

#if TN_EXP_TRACE || TN_EXP_PROF
extern "C" int tn_exp_trace(long long* host, int n) {
    return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace, sizeof(long long) * (n < 4096 ? n : 4096)));
}
#endif
