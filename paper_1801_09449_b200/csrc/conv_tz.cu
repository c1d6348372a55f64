// conv_tz.cu -- ternary conv3d on the tcgen05 tensor cores with the taps folded
// into the UMMA descriptors ("tap-offset") and the three kernel planes dz merged
// along N ("z-merged").  Written for the layers with few channels (C, K <= 64,
// 27*C*K small enough for the filter bank to sit in shared memory three times
// over) -- every tensor-core shape of the library.
//
// The arithmetic is the same integer as Eq. 9: int8 products
// of ternary values {-1,0,+1} accumulated exactly in int32, over the 3x3x3
// window of Sec. 2 with zero padding; the fused epilogue applies
// the integer thresholds of reading R5/R6 and repacks into the
// paper's 2-bit sign/mask format (Fig. 3 :130).
//
// Layout.  Output positions of a plane are a raster with pitch Po = Wo + 1 (one
// separator column per row).  A CTA expands, per input plane, a strip of
// RS = 128*T + halo consecutive raster rows into int8 (16 channels = 16 bytes per
// row and chunk) in the canonical K-major no-swizzle UMMA layout, where row r
// sits at byte 16*r (8-row core matrices, SBO = 128).  Tap (dy, dx) of an
// output tile is then the same buffer at a row offset: the descriptor start moves
// by 16*(dy*Po + dx) bytes, and the second 16-channel half of a K = 32 MMA is any
// other (tap, chunk) slice at LBO = the byte distance between them (both checked
// on B200 by tools/desc_test.cu: arbitrary 16-byte starts and LBOs, overlapping
// or not, run at full rate).  So each input voxel is expanded once per plane and
// per strip, and no shifted copies exist.  Stride 2 uses four phase images
// (even/odd rows x even/odd columns), each in the output raster, so every tap is
// again a plain offset.
//
// z-merge.  An input plane i feeds up to three output planes (z = i+1-dz).  The B
// operand holds the filter blocks of the three dz side by side (N = 3K), and the
// accumulators of the three outputs of a tile sit in three adjacent TMEM column
// blocks, so one MMA per K-slice pair updates all three.  Output z lives in TMEM
// block sigma = u mod 3 (u = the CTA's running output index); the three blocks a
// plane touches are always {0,1,2} in a rotation, handled by three rotations of
// the B blocks stored as the cyclic sequence [dz2 dz1 dz0 dz2 dz1].  Stride 2:
// odd planes feed two outputs (rotations [dz2 dz0] / [dz0 dz2]), even planes one.
// The epilogue re-initialises a block after reading it (to -hi, so the
// accumulator holds acc - hi and the A4 compare is a sign bit), so the MMAs always
// accumulate.
//
// CTA = 19 warps, persistent, one per SM:
//   warps 0-7   epilogue, two groups of four (one warp per TMEM lane quadrant);
//               group g takes the tiles t % 2 == g of every output plane
//   warps 8-15  expanders: packed rows (staging) -> int8 A strip of one plane
//   warps 16-17 MMA issuers: one elected lane of warp 16 + w runs the schedule of
//               the tiles t % 2 == w (waits, tcgen05.mma, commits)
//   warp 18     loader: one elected lane issues 1-D bulk copies (cp.async.bulk)
//               of the contiguous packed rows a strip needs, per plane and segment
#include "tn_internal.cuh"

#include <cstdio>
#include <cstdlib>
#include "tc_ptx.cuh"

#include <algorithm>
#include <cstring>
#include <climits>
#include <vector>

// TN_TRACE builds (profiling only; python paper_1801_09449_b200/build.py --trace writes
// libtn_trace.so): per-CTA cycle counters of each warp role's barrier waits, read back with
// tn_trace_read().  Slots: 0 kernel, 1 loader waits, 2 expander staged waits, 3 expander
// slot waits, 4 MMA plane waits, 5 MMA accumulator waits, 6 epilogue waits, 7 epilogue busy.
#ifdef TN_TRACE
__device__ unsigned long long g_tn_trace[1024 * 8];
#define TN_TW(slot, rec, stmt)                                                           \
    do {                                                                                 \
        const long long _t0 = clock64();                                                 \
        stmt;                                                                            \
        if (rec) atomicAdd(&g_tn_trace[blockIdx.x * 8 + (slot)], clock64() - _t0);      \
    } while (0)
extern "C" int tn_trace_read(unsigned long long* host, int n, int reset) {
    const int m = n < 1024 * 8 ? n : 1024 * 8;
    cudaError_t e = cudaMemcpyFromSymbol(host, g_tn_trace, sizeof(unsigned long long) * m);
    if (reset) {
        static unsigned long long zero[1024 * 8];
        cudaMemcpyToSymbol(g_tn_trace, zero, sizeof(zero));
    }
    return static_cast<int>(e);
}
#else
#define TN_TW(slot, rec, stmt) stmt
#endif

// TN_CHECK builds (python paper_1801_09449_b200/build.py --check writes libtn_check.so): device
// bounds checks on every bulk copy, staged read, A-operand write and output store of the TZ
// kernel; a violation traps (a loud CUDA error).  The stand-in for compute-sanitizer, which is
// closed on this GPU pool.
#ifdef TN_CHECK
#define TN_ASSERT(c)                                                                                 \
    do {                                                                                             \
        if (!(c)) {                                                                                  \
            printf("TN_CHECK failed: %s (conv_tz.cu:%d) block %d thread %d\n", #c, __LINE__, blockIdx.x, \
                   threadIdx.x);                                                                     \
            __trap();                                                                                \
        }                                                                                            \
    } while (0)
#else
#define TN_ASSERT(c) do { } while (0)
#endif

namespace tn {
namespace {

// MMA issuers (tiles t % kZMmaWarps): one thread's per-tile wait / commit
// overhead exceeds the 5 x 44 cycles a K = 16 tile keeps the tensor pipe busy.
constexpr int kZMmaWarps = 2;
// Expander warps: the expansion is latency-bound per warp, so as many as the
// register budget allows (the fused-prediction variants need more registers).
// Measured (configs[3] layers): 12 expander warps win for one-chunk and four-chunk
// strips, 8 for two-chunk strips (#12, #13) and the fused-prediction variant.
#ifndef TN_EXP64
#define TN_EXP64 9   // expander warps at K = 64 (20 warps in all: 96 registers per thread)
#endif
// Plain K = 16 layers (stride 1, not FIRST, no prediction; configs[3] #2, #12): the epilogue is the
// critical role, so three groups of four epilogue warps and eight expander warps (measured on
// #2, one 128x256x256 volume: (groups, expanders) = (2, 12) 91.9 us, (2, 8) 90.1, (3, 12) 91.9,
// (3, 8) 82.1, (3, 6) 85.4, (4, 8) 88.4; the two-segment #13 stays at two groups)
#ifndef TN_E16
#define TN_E16 3
#endif
#ifndef TN_X16
#define TN_X16 8
#endif
// (groups, expander warps) of the K = 16 layers with the fused prediction (#14: (2, 8) 893 us,
// (2, 6) 873, (3, 6) 804, (3, 4) 786 per configs[3] batch), of the first layer (#1: (2, 12) 702,
// (2, 8) 725, (3, 8) 736, (3, 12) 723) and of the two-channel-chunk layers (#13: (2, 8) 820,
// (2, 12) 801, (3, 12) 782, (2, 16) 869, (1, 16) 1096, (1, 12) 1045, (3, 6) 906, (2, 6) 923)
#ifndef TN_EP16
#define TN_EP16 3
#endif
#ifndef TN_XP16
#define TN_XP16 4
#endif
#ifndef TN_EF16
#define TN_EF16 2
#endif
#ifndef TN_XF16
#define TN_XF16 12
#endif
#ifndef TN_E2S
#define TN_E2S 3
#endif
#ifndef TN_X2S
#define TN_X2S 12
#endif
#ifndef TN_EFF4
#define TN_EFF4 3    // the FP4 first layer (FF4; #1: (3, 8) 537 us, (2, 8) 613, (3, 12) 605, (3, 4) 657, (4, 4) 658)
#endif
#ifndef TN_XFF4
#define TN_XFF4 8
#endif
// plain: stride 1 and not the int8 first layer; first: the int8 first layer; ff4: the FP4 first layer
__host__ __device__ constexpr int tz_exp_warps(int k, bool pred, int ct, bool plain, bool first = false, bool ff4 = false) {
    return k == 16 && ff4 ? TN_XFF4
         : k == 16 && first ? TN_XF16
         : k == 16 && pred && plain && ct == 1 ? TN_XP16
         : k == 16 && !pred && plain && ct == 2 ? TN_X2S
         : (k == 16 && !pred && plain) ? TN_X16 : ((pred || ct == 2) ? 8 : (k == 64 ? TN_EXP64 : 12));
}
// epilogue groups of four warps (one per TMEM lane quadrant); group g takes tiles t % groups == g
// (three groups for K = 16 measured 2 % slower on configs[3]: the SMSPs' issue slots are shared)
__host__ __device__ constexpr int tz_epi_groups(int k, bool pred, int ct, bool plain, bool first = false, bool ff4 = false) {
    return k == 16 && ff4 ? TN_EFF4
         : k == 16 && first ? TN_EF16
         : k == 16 && pred && plain && ct == 1 ? TN_EP16
         : k == 16 && !pred && plain && ct == 2 ? TN_E2S
         : (k == 16 && !pred && plain && ct == 1) ? TN_E16 : 2;
}
__host__ __device__ constexpr int tz_threads(int k, bool pred, int ct, bool plain, bool first = false, bool ff4 = false) {
    return (4 * tz_epi_groups(k, pred, ct, plain, first, ff4) + tz_exp_warps(k, pred, ct, plain, first, ff4) + kZMmaWarps + 1) *
           32;
}
constexpr int kZMaxMma = 18;          // ceil(9 taps x 4 chunks / 2)
constexpr int kZMaxAcc = 32;          // TMEM blocks (RO x T)
constexpr int kZMaxSlot = 4;          // A ring
constexpr int kZMaxStage = 4;         // packed staging ring
constexpr int kZMaxClass = 8;
constexpr int kZBiasA = 4096;         // K = 16 accumulator-start MMA: A constants [half][128 rows][16 B]
// B start rows [mma][half][K rows][16 B]: K = 64 FP4 takes two start MMAs (|start| <= 1729.5 > 1344)
__host__ __device__ constexpr int tz_bias_mmas(int k, bool f4) { return f4 && k == 64 ? 2 : 1; }
__host__ __device__ constexpr int tz_bias_bytes(int k, bool f4) { return kZBiasA + tz_bias_mmas(k, f4) * k * 32; }

struct TzPlan {
    int s;                  // stride (1 or 2, all axes)
    int RO;                 // output blocks per tile in TMEM (3 for s = 1, 2 for s = 2)
    int Po, NPo, NT;        // output raster pitch (Wo + 1), positions per plane, 128-row tiles per plane
    int T, nstrip;          // tiles per strip, strips per plane
    int RS, REG;            // strip rows per (phase, chunk) region, region bytes
    int nph;                // phase images (1 or 4)
    int slot_bytes, nslot;  // A ring
    int stage_bytes, nstage;
    int seg_off[kMaxSeg];   // byte offset of each segment's rows within a stage
    int cch[kMaxSeg];       // 16-channel chunks per segment
    int nmma;
    int a_off[kZMaxMma];    // per MMA: A start (bytes from the slot base) and LBO (bytes)
    int a_lbo[kZMaxMma];
    int8_t sl_tap[2 * kZMaxMma];    // per K-slice (sorted order): tap (dy*3+dx) and chunk, -1 = zero slice
    int8_t sl_chunk[2 * kZMaxMma];
    int8_t sl_tapb[2 * kZMaxMma];   // F4 two-position slices (C = 16): second tap, -1 = none
    int8_t sl_seg[2 * kZMaxMma];    // F4: segment of the slice
    int f4;                 // FP4 (kind::mxf4) operands
    int nreg;               // F4: 16-byte A regions per phase (per position); reg0[seg] = first region of seg
    int reg0[kMaxSeg];
    int NB;                 // B blocks (5 for s = 1, 4 for s = 2)
    int b_bytes;
    int64_t units;          // N * nstrip * Do
    uint32_t po_magic;      // ceil(2^32 / Po)
    int step_q, step_r;     // 256 rows (one expander sweep) = step_q raster rows + step_r positions
    int code_off, code_pitch, code_bytes;   // FIRST: ternary code planes (2 buffers) after the stages
    int wpad;               // bytes after the code planes so that the packed filter bank fits from s_a on
    int ptab_floats;
    int kp;                 // output channels padded to the kernel's K (16 / 32 / 64)
    int dil;                // in-plane dilation (taps dy*dil*Po + dx*dil); z dilation = residue classes
    int qoff, yoff;         // strip start offset dil*Po + dil; raster rows added to keep dividends >= 0
    int bias_bytes;         // accumulator-start MMA operands (A constants 4 KB + B rows), K = 16 or FP4
    int bpv;                // staged bytes per voxel (raster staging)
    int onep;               // one-plane volume (Dci = Do = 1): one TMEM block per tile, no z-merge
    int rstg;               // raster staging (F4, one plain segment, stride 1): the loader copies each packed
                            // row to pitch Po, so staged voxel = strip row and separators stay zero
};

// q / Po for 0 <= q with q * Po < 2^32
__device__ __forceinline__ int div_po(uint32_t q, uint32_t magic) { return static_cast<int>(__umulhi(q, magic)); }

// Walk over a CTA's contiguous range of units (n, strip, output plane), in runs
// of consecutive output planes of one (n, strip).
struct ZWalk {
    int64_t t, t_end;
    int Do, nstrip;
    __device__ ZWalk(int64_t U, int Do_, int nstrip_) : Do(Do_), nstrip(nstrip_) {
        t = U * blockIdx.x / gridDim.x;
        t_end = U * (blockIdx.x + 1) / gridDim.x;
    }
    __device__ bool next(int& n, int& strip, int& zf, int& zl) {
        if (t >= t_end) return false;
        const int64_t col = t / Do;
        zf = static_cast<int>(t - col * Do);
        const int64_t len = min(static_cast<int64_t>(Do - zf), t_end - t);
        zl = zf + static_cast<int>(len) - 1;
        n = static_cast<int>(col / nstrip);
        strip = static_cast<int>(col - static_cast<int64_t>(n) * nstrip);
        t += len;
        return true;
    }
};

// Global conv-input planes of a run of (local) output planes [zf, zl].
__device__ __forceinline__ void run_planes(const TzPlan& pl, const ConvDesc& cd, int zf, int zl, int& i0, int& i1) {
    i0 = max(pl.s * (cd.zo_beg + zf) - 1, 0);
    i1 = min(pl.s * (cd.zo_beg + zl) + 1, cd.Dci - 1);
}

// Source rows of segment sg that the strip's A rows read: [ya, ya + nrows).
__device__ __forceinline__ void strip_rows(const TzPlan& pl, const ConvDesc& cd, int strip, int sg, int& ya,
                                           int& nrows) {
    const int qa = strip * 128 * pl.T - pl.qoff;
    const int qb = qa + pl.RS - 1;
    const uint32_t two = static_cast<uint32_t>(pl.yoff * pl.Po);
    int ylo = div_po(static_cast<uint32_t>(qa) + two, pl.po_magic) - pl.yoff;
    int yhi = div_po(static_cast<uint32_t>(qb) + two, pl.po_magic) - pl.yoff;
    if (pl.s == 2) { ylo = 2 * ylo; yhi = 2 * yhi + 1; }
    ylo = max(ylo, 0);
    yhi = min(yhi, cd.Hci - 1);
    const SegDesc& sd = cd.seg[sg];
    if (sd.up) { ylo >>= 1; yhi >>= 1; }
    yhi = min(yhi, sd.H - 1);
    ya = ylo;
    nrows = max(yhi - ylo + 1, 0);
}

// B image entry u of a plan (the filter bank as the UMMA B operand): MMA m, half h = K-slice
// j = 2m + h, block b (dz of the block sequence), row k: 16 channels of W[k][chunk][dz][dy][dx]
// as int8, or 32 FP4 nibbles.  wsrc[sg]: segment sg's packed filter bank [K][27][2][cw] (staged
// in shared memory by the conv, read from global memory by the prepare kernel).
template <int K, int NSEG, int STR, bool FIRST, bool F4, int NB, bool ONEP = false>
__device__ __forceinline__ uint4 bimage_entry(const ConvDesc& cd, const TzPlan& pl, const uint32_t* const* wsrc,
                                              int u) {
    constexpr int rows = NB * K;
    const int row = u % rows;
    const int j = u / rows;                    // slice index (2m + h)
    const int b = row / K, k = row - b * K;
    // (ONEP: one-plane layers, only the middle kernel plane meets data)
    const int dz = ONEP ? 1 : STR == 1 ? (2 - (b % 3)) : (b == 0 || b == 2 ? 0 : (b == 1 ? 2 : 1));
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    const int tap = k < cd.K ? pl.sl_tap[j] : -1;    // padded output channels: zero filters
    if (FIRST && !F4) {
        if (j == 0) {   // byte (dy*3 + dx) = w[k][0][dz][dy][dx]
            uint32_t wv[4] = {0u, 0u, 0u, 0u};
            for (int t9 = 0; t9 < 9; ++t9) {
                const uint32_t* src = wsrc[0] + (k * 27 + dz * 9 + t9) * 2;
                const uint32_t sb = src[0] & 1u, mb = src[1] & 1u;
                const uint32_t byte = mb ? (sb ? 0x01u : 0xFFu) : 0u;
                wv[t9 >> 2] |= byte << (8 * (t9 & 3));
            }
            v = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
    } else if (F4) {
        if (tap >= 0) {
            const int sg = pl.sl_seg[j];
            const int cw = cd.seg[sg].cw;
            const uint32_t* src = wsrc[sg] + (k * 27 + dz * 9 + tap) * 2 * cw;
            if (cd.seg[sg].c <= 16) {       // [tap a ch 0-15 | tap b ch 0-15]
                const uint2 a2 = expand16_f4(src[0], src[cw], 0);
                uint2 b2 = make_uint2(0u, 0u);
                const int tb = pl.sl_tapb[j];
                if (tb >= 0) {
                    const uint32_t* s2 = wsrc[sg] + (k * 27 + dz * 9 + tb) * 2 * cw;
                    b2 = expand16_f4(s2[0], s2[cw], 0);
                }
                v = make_uint4(a2.x, a2.y, b2.x, b2.y);
            } else {                        // 32 channels 32c .. 32c+31
                const int c = pl.sl_chunk[j];
                const uint2 a2 = expand16_f4(src[c], src[cw + c], 0);
                const uint2 b2 = expand16_f4(src[c], src[cw + c], 16);
                v = make_uint4(a2.x, a2.y, b2.x, b2.y);
            }
        }
    } else if (tap >= 0) {
        int c = pl.sl_chunk[j];
        const int sg = (NSEG > 1 && c >= pl.cch[0]) ? 1 : 0;
        if (sg) c -= pl.cch[0];
        const int cw = cd.seg[sg].cw;
        const uint32_t* src = wsrc[sg] + (k * 27 + dz * 9 + tap) * 2 * cw;
        const int word = c >> 1, sh = 16 * (c & 1);
        v = expand16(src[word], src[cw + word], sh);
    }
    return v;
}
// K = 64 at stride 1 splits wrapping MMAs over four TMEM blocks (the five-block rotated B image
// would not fit shared memory next to the int8 operands), except with FP4 operands of one
// C <= 64 segment, whose rotated image (92 KB) fits: three blocks, no split, two tiles per strip.
__host__ __device__ constexpr bool tz_split(int K, int STR, bool F4, int CT) {
    return STR == 1 && K == 64 && !(F4 && CT <= 4);
}
template <int K, int STR, bool F4, int CT>
__host__ __device__ constexpr int tz_nb() { return STR == 1 ? (tz_split(K, STR, F4, CT) ? 3 : 5) : 4; }

// Prepared filter bank (tn_weights_prepare / the FCN at create): the B image built once in global
// memory, same layout as in shared memory ([j][NB*K][16 B]); the conv then copies it instead of
// staging and expanding the packed bank in every CTA.
template <int K, int CT, int NSEG, int STR, bool FIRST, bool F4, bool ONEP = false>
__global__ void bimage_build_kernel(const ConvDesc cd, const TzPlan pl, uint4* out) {
    const uint32_t* wsrc[kMaxSeg] = {cd.seg[0].wp, cd.seg[kMaxSeg - 1].wp};
    constexpr int NB = ONEP ? 1 : tz_nb<K, STR, F4, CT>();
    const int total = pl.nmma * 2 * NB * K;
    for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < total; u += gridDim.x * blockDim.x)
        out[u] = bimage_entry<K, NSEG, STR, FIRST, F4, NB, ONEP>(cd, pl, wsrc, u);
}

template <int K, int CT, int NSEG, int STR, bool PRED, bool FIRST, bool F4, bool ONEP = false>
__global__ void __launch_bounds__(tz_threads(K, PRED, CT, STR == 1 && (!FIRST || F4), FIRST && !F4, FIRST && F4), 1)
conv_tz_kernel(const ConvDesc cd, const TzPlan pl) {
    // FIRST with F4 (FF4): the float input staged in raster rows, Eq. 6 applied per position and
    // the code fed as a one-channel FP4 segment (the C = 16 F4 path); FIRST alone (FI8): int8 rows
    // of the position's 9 in-plane taps
    constexpr bool FF4 = FIRST && F4, FI8 = FIRST && !F4;
    constexpr bool PLAIN = STR == 1 && !FI8;
    constexpr int kZExpThreads = tz_exp_warps(K, PRED, CT, PLAIN, FI8, FF4) * 32;
    constexpr int kZEpiGroups = tz_epi_groups(K, PRED, CT, PLAIN, FI8, FF4);
    constexpr int kZEpiWarps = 4 * kZEpiGroups;
    constexpr int kZExpWarp0 = kZEpiWarps;
    constexpr int kZMmaWarp = kZEpiWarps + tz_exp_warps(K, PRED, CT, PLAIN, FI8, FF4);
    constexpr int kZLoadWarp = kZMmaWarp + kZMmaWarps;
    constexpr int kZThreads = tz_threads(K, PRED, CT, PLAIN, FI8, FF4);
    // FIRST (A7, reading R7): seg[0] is the float input; the expanders apply Eq. 6
    // and pack each position's 9 in-plane taps (dy, dx) into one 16-byte A row, so
    // a plane is one K-slice (one MMA with a zero-weight second half) and the dz
    // taps are the z-merged B blocks as usual.
    // K = 64 (stride 1): four blocks per tile, the B blocks in plain order and a
    // plane's MMAs split in two where its outputs wrap around the block ring
    // (the rotated-B sequence would not fit shared memory next to C = 64 strips).
    // F4: ternary operands as FP4 E2M1 (kind::mxf4, unit UE8M0 block scales in TMEM
    // columns 480..511): exact (f32 accumulation of integers < 2^24), half the
    // shared-memory bytes per MAC and twice the int8 MMA rate.  C = 16 segments
    // hold two consecutive positions per 16-byte row (taps dx, dx+1 in one K-half).
    // ONEP (one-plane volumes, Table 1's 2D layers): no z-merge -- one TMEM block per tile, the
    // B image holds the middle kernel plane only, and TMEM fits up to 480 / K tiles per strip
    constexpr bool SPLIT = !ONEP && tz_split(K, STR, F4, CT);
    constexpr int RO = ONEP ? 1 : STR == 1 ? (SPLIT ? 4 : 3) : 2;
    constexpr int NPH = STR == 1 ? 1 : 4;
    constexpr int NB = ONEP ? 1 : tz_nb<K, STR, F4, CT>();
    constexpr int CWO = (K + 31) / 32;
    // K = 16: a new output's accumulator block is started by an MMA (accumulate = 0) of constant A
    // rows with B rows summing to its start value (-hi; F4: 1/2 - hi), issued just before the
    // output's first data MMA; the epilogue only loads the block and hands it back
    // (K = 32 FP4: #4 194 -> 182 us, #11 225 -> 217; K = 64 FP4 measured slower -- C1's conv 59.4 ->
    // 61.4 us: its MMA issuer is the busiest role and the two start MMAs add 2 to its 9 per tile)
    constexpr bool BIAS = K == 16 || (F4 && K == 32);
    constexpr int NBM = tz_bias_mmas(K, F4);
    extern __shared__ __align__(128) uint8_t smem[];
    // [B image][A ring][staging ring][FIRST code planes][wpad]: during setup the packed filter
    // bank is staged in the contiguous span from the A ring to the end of wpad
    uint8_t* s_b = smem;                                         // [mma][half][NB*K][16]
    uint8_t* s_a = s_b + pl.b_bytes;                             // [slot][phase][chunk][RS][16]
    uint8_t* s_stage = s_a + pl.nslot * pl.slot_bytes;           // [stage] packed rows per segment
    // K = 16: [A constants][B start rows] of the accumulator-start MMA (BIAS, below)
    uint8_t* s_bias = s_stage + pl.nstage * pl.stage_bytes + 2 * pl.code_bytes + pl.wpad;
    int* s_nhi = reinterpret_cast<int*>(s_bias + pl.bias_bytes);   // [K] -hi
    int* s_lmh = s_nhi + K;                                      // [K] lo - hi
    float* s_pred = reinterpret_cast<float*>(s_lmh + K);         // [kZMaxClass] bias, then quad tables
    float* s_ptab = s_pred + kZMaxClass;
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_ptab + pl.ptab_floats);
    uint64_t* plane_full = bars;                                 // [kZMaxSlot]
    uint64_t* plane_free = plane_full + kZMaxSlot;               // [kZMaxSlot]
    uint64_t* staged_full = plane_free + kZMaxSlot;              // [kZMaxStage]
    uint64_t* staged_empty = staged_full + kZMaxStage;           // [kZMaxStage]
    uint64_t* acc_full = staged_empty + kZMaxStage;              // [kZMaxAcc]
    uint64_t* acc_empty = acc_full + kZMaxAcc;                   // [kZMaxAcc]
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(acc_empty + kZMaxAcc);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const bool fused = cd.yp != nullptr;
    const int T = pl.T;
    const int NU = T;      // synchronisation units per strip: one per tile
    const int zst = cd.zstep > 0 ? cd.zstep : 1;           // dilation: plane step of the residue class
    const int64_t dbuf = cd.Dbuf > 0 ? cd.Dbuf : cd.Do;    // output buffer depth

    // ---- setup: stage the packed filter bank (cp.async) in the A ring, expand it
    // into the B image, thresholds, barriers, TMEM.
    {
        // channels k >= cd.K (K padded to 16 / 32 / 64) have zero filters and "always 0" thresholds
        int hi_r = 1 << 20, lo_r = -(1 << 20);
        if (fused && threadIdx.x < cd.K) {
            lo_r = clamp_threshold(__ldg(cd.lo + threadIdx.x));
            hi_r = clamp_threshold(__ldg(cd.hi + threadIdx.x));
        }
        if (BIAS) {   // |acc| <= 27 * 16 * CT: thresholds beyond act as "never" / "always"
            constexpr int M = 27 * 16 * CT + 1;
            hi_r = max(-M, min(hi_r, M));
            lo_r = max(-M, min(lo_r, M));
        }
        const uint32_t* wsrc[kMaxSeg];
        uint32_t* s_wp = reinterpret_cast<uint32_t*>(s_a);
        int ofs = 0;
        const bool prepared = cd.bimg != nullptr;   // (the host matched its plan to this launch's)
        if (prepared) {
            for (int i = threadIdx.x; i < pl.b_bytes / 16; i += kZThreads)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s_b + 16 * i)), "l"(cd.bimg + i)
                             : "memory");
        }
#pragma unroll
        for (int sg = 0; sg < NSEG && !prepared; ++sg) {
            const int nw = cd.K * 27 * 2 * (FIRST ? 1 : cd.seg[sg].cw);   // words (odd K: not a multiple of 4)
            const int n4 = nw / 4;
            const uint4* g = reinterpret_cast<const uint4*>(cd.seg[sg].wp);
            for (int i = threadIdx.x; i < n4; i += kZThreads)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s_wp + ofs + 4 * i)), "l"(g + i)
                             : "memory");
            for (int i = 4 * n4 + threadIdx.x; i < nw; i += kZThreads)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(s_wp + ofs + i)),
                             "l"(cd.seg[sg].wp + i)
                             : "memory");
            wsrc[sg] = s_wp + ofs;
            ofs += (nw + 3) & ~3;
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
        if (BIAS) {   // accumulator-start MMA operands: A constants, B rows summing to the start value
            for (int i = threadIdx.x; i < kZBiasA / 16; i += kZThreads) {
                const uint32_t c = F4 ? (i < kZBiasA / 32 ? 0x22222222u : 0x77777777u) : 0x01010101u;   // 1.0 | 6.0; int8 1
                reinterpret_cast<uint4*>(s_bias)[i] = make_uint4(c, c, c, c);
            }
            // B start rows, one byte per thread: start MMA j, channel k, K half h, byte b (FP4 with two
            // start MMAs: the first carries up to +-1300 of the start value, the second the rest)
            for (int i = threadIdx.x; i < NBM * K * 32; i += kZThreads) {
                const int j = i / (K * 32), k = (i >> 5) % K, h = (i >> 4) & 1, b = i & 15;
                int hk = 1 << 20;
                if (fused && k < cd.K) hk = clamp_threshold(__ldg(cd.hi + k));
                constexpr int M = 27 * 16 * CT + 1;
                hk = max(-M, min(hk, M));
                const float v = fused ? 0.5f - static_cast<float>(hk) : 0.0f;
                const float va = NBM == 1 ? v : fmaxf(-1300.0f, fminf(v, 1300.0f));
                s_bias[kZBiasA + j * K * 32 + h * K * 16 + k * 16 + b] =
                    F4 ? e2m1_start_byte(j == 0 ? va : v - va, h, b) : i8_start_byte(fused ? -hk : 0, 16 * h + b);
            }
        }
        if (threadIdx.x < K) {
            if (F4) {   // f32 accumulators: acc - hi + 1/2 (exact: |hi|, |lo| <= 2^20, |acc| < 2^12)
                s_nhi[threadIdx.x] = __float_as_int(fused ? 0.5f - static_cast<float>(hi_r) : 0.0f);
                s_lmh[threadIdx.x] = __float_as_int(static_cast<float>(lo_r - hi_r + 1));
            } else {
                s_nhi[threadIdx.x] = fused ? -hi_r : 0;
                s_lmh[threadIdx.x] = lo_r - hi_r;
            }
        }
        {   // barriers, one per thread
            const int t = threadIdx.x;
            if (t < kZMaxSlot) { mbar_init(plane_full + t, kZExpThreads); mbar_init(plane_free + t, kZMmaWarps); }
            else if (t < kZMaxSlot + kZMaxStage) {
                mbar_init(staged_full + t - kZMaxSlot, 1);
                mbar_init(staged_empty + t - kZMaxSlot, kZExpThreads);
            } else if (t >= 64 && t < 64 + kZMaxAcc) {
                mbar_init(acc_full + t - 64, 1);
                mbar_init(acc_empty + t - 64, 128);
            }
            if (t < kZMaxSlot + kZMaxStage || (t >= 64 && t < 64 + kZMaxAcc))
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        // B image (unless a prepared one was copied)
        if (!prepared) {
            const int total = pl.nmma * 2 * NB * K;
            for (int u = threadIdx.x; u < total; u += kZThreads)
                *reinterpret_cast<uint4*>(s_b + static_cast<size_t>(u) * 16) =
                    bimage_entry<K, NSEG, STR, FIRST, F4, NB, ONEP>(cd, pl, wsrc, u);
        }
        if (pl.rstg) {   // raster staging: separator slots and rows outside the volume stay zero
            __syncthreads();   // (the unprepared B image was read from the packed bank staged here)
            // (FF4: a float Eq. 6 maps to 0, the midpoint of t_lo <= t_hi)
            // Only the separator slots [W, Po) of each row slot: data slots are always copied before
            // they are read, and rows outside the volume are never read.
            const uint32_t f = FF4 ? __float_as_uint(0.5f * cd.t_lo + 0.5f * cd.t_hi) : 0u;
            const int pitch = pl.Po * pl.bpv, sep = (pl.Po - cd.seg[0].W) * pl.bpv / 4;
            const int rows = pl.stage_bytes / pitch;
            for (int i = threadIdx.x; i < pl.nstage * rows * sep; i += kZThreads) {
                const int stg = i / (rows * sep), rw = (i / sep) % rows, w = i % sep;
                reinterpret_cast<uint32_t*>(s_stage + stg * pl.stage_bytes + rw * pitch + cd.seg[0].W * pl.bpv)[w] = f;
            }
        }
        if (PRED) {
            for (int i = threadIdx.x; i < cd.nclass; i += kZThreads) s_pred[i] = __ldg(cd.pb + i);
            // quad tables: entry (mask nibble | sign nibble << 4) = (((t0 w0) + t1 w1) + t2 w2) + t3 w3
            for (int e = threadIdx.x; e < cd.nclass * (K / 4) * 256; e += kZThreads) {
                const int idx = e & 255, qd = (e >> 8) % (K / 4), j = e / (256 * (K / 4));
                float part = 0.0f;
                for (int i = 0; i < 4; ++i) {
                    const float wv = __ldg(cd.pw + j * K + 4 * qd + i);
                    const bool nz = (idx >> i) & 1, ps = (idx >> (4 + i)) & 1;
                    part += nz ? (ps ? wv : -wv) : 0.0f;
                }
                // two classes: both classes' entries side by side (one 8-byte lookup per quad)
                s_ptab[(cd.nclass == 2 && K == 16) ? ((qd * 256 + idx) * 2 + j) : e] = part;
            }
        }
        if (warp == kZMmaWarp) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                         "r"(512));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        fence_proxy_async();   // B image visible to the tensor core
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }
    const uint32_t tmem_base = *s_tmem;
#ifdef TN_TRACE
    const long long k_t0 = clock64();
#endif
    pdl_launch_dependents();

    if (warp < kZEpiWarps) {
        // ---- initialise this warp's TMEM blocks (its quadrant, its tiles, all RO blocks)
        // (K = 16: -hi, see the epilogue's REGT; K >= 32: zero, -hi is added in the requant)
        const int q = warp & 3, g = warp >> 2;
        int iv[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) iv[k] = K == 16 ? s_nhi[k] : 0;
        for (int t = 0; t < T; ++t)
            if (t % kZEpiGroups == g)
            for (int b = 0; b < RO; ++b)
#pragma unroll
                for (int c = 0; c < K; c += 16)
                    tmem_st16(tmem_base + (static_cast<uint32_t>(32 * q) << 16) + (t * RO + b) * K + c, iv);
        if (F4 && g == 0) {   // unit block scales (UE8M0 0x7F = 2^0) in columns 480..511
            int sf[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) sf[i] = 0x7F7F7F7F;
            tmem_st16(tmem_base + (static_cast<uint32_t>(32 * q) << 16) + 480, sf);
            tmem_st16(tmem_base + (static_cast<uint32_t>(32 * q) << 16) + 496, sf);
        }
        tmem_wait_st();
        tc_fence_before();
    }
    pdl_wait();   // activations of the previous layer are complete and visible from here on
    __syncthreads();
    tc_fence_after();

    const uint32_t two_po = static_cast<uint32_t>(pl.yoff * pl.Po);   // keeps raster dividends >= 0
    if (warp == kZLoadWarp) {
        // ================= loader: per plane and segment one bulk copy of the
        // contiguous packed rows the strip reads (zero-size outside the buffer)
        if (lane == 0) {
            ZWalk wk(pl.units, cd.Do, pl.nstrip);
            int n, strip, zf, zl;
            uint32_t st = 0, st_r = 0;
            while (wk.next(n, strip, zf, zl)) {
                int i0, i1;
                run_planes(pl, cd, zf, zl, i0, i1);
                int ya[kMaxSeg], nr[kMaxSeg];
#pragma unroll
                for (int sg = 0; sg < NSEG; ++sg) strip_rows(pl, cd, strip, sg, ya[sg], nr[sg]);
                for (int i = i0; i <= i1; ++i) {
                    if (st_r > 0) mbar_wait(staged_empty + st, (st_r - 1) & 1);
                    if constexpr (F4 && NSEG == 1 && STR == 1) {
                        if (pl.rstg) {   // one bulk copy per packed (FF4: float) row, to its slot of pitch Po
                            const SegDesc& sd = cd.seg[0];
                            const int zs = cd.zres + i * zst - sd.zbeg;
                            const int nrow = (zs >= 0 && zs < sd.D) ? nr[0] : 0;
                            constexpr int kVb = FF4 ? 4 : 8;     // staged bytes per voxel and 32-lane word
                            const uint32_t rb = static_cast<uint32_t>(sd.W) * kVb * sd.cw;
                            const char* sp0 = FF4 ? reinterpret_cast<const char*>(cd.xf + ((static_cast<int64_t>(n) * sd.D + zs) * sd.H + ya[0]) * sd.W)
                                                  : reinterpret_cast<const char*>(sd.xp + ((static_cast<int64_t>(n) * sd.D + zs) * sd.H + ya[0]) * sd.W * 2 * sd.cw);
                            mbar_arrive_expect_tx(staged_full + st, nrow * rb);
                            uint8_t* dst = s_stage + st * pl.stage_bytes;
                            for (int y = 0; y < nrow; ++y) {
                                TN_ASSERT((y + 1) * pl.Po * kVb * sd.cw <= pl.stage_bytes);
                                bulk_g2s(dst + y * pl.Po * kVb * sd.cw, sp0 + static_cast<int64_t>(y) * rb, rb, staged_full + st);
                            }
                            if (++st == static_cast<uint32_t>(pl.nstage)) { st = 0; ++st_r; }
                            continue;
                        }
                    }
                    uint32_t bytes[kMaxSeg];
                    const uint32_t* src[kMaxSeg];
                    uint32_t total = 0;
#pragma unroll
                    for (int sg = 0; sg < NSEG; ++sg) {
                        const SegDesc& sd = cd.seg[sg];
                        const int zs = (sd.up == 1 ? (i >> 1) : cd.zres + i * zst) - sd.zbeg;
                        const bool ok = zs >= 0 && zs < sd.D && nr[sg] > 0;
                        if (FIRST) {
                            bytes[sg] = ok ? static_cast<uint32_t>(nr[sg]) * sd.W * 4u : 0u;
                            src[sg] = reinterpret_cast<const uint32_t*>(
                                cd.xf + ((static_cast<int64_t>(n) * sd.D + zs) * sd.H + ya[sg]) * sd.W);
                        } else {
                            // rows of 8*cw bytes: with cw = 1 and an odd W the range may start or end
                            // 8 bytes off a 16-byte boundary.  Copy the aligned superset (the
                            // expanders skip the 8-byte head); if its last 16 bytes would cross the
                            // end of the buffer, those 8 valid bytes take a plain load instead.
                            const uint32_t* sp0 =
                                sd.xp + ((static_cast<int64_t>(n) * sd.D + zs) * sd.H + ya[sg]) * sd.W * 2 * sd.cw;
                            const uint32_t head = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(sp0)) & 15u;
                            src[sg] = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(sp0) - head);
                            bytes[sg] = 0u;
                            if (ok) {
                                const uint32_t nb = static_cast<uint32_t>(nr[sg]) * sd.W * 8u * sd.cw;
                                uint32_t al = (head + nb + 15u) & ~15u;
                                const char* buf_end = reinterpret_cast<const char*>(sd.xp) +
                                                      static_cast<int64_t>(cd.N) * sd.D * sd.H * sd.W * 8 * sd.cw;
                                if (reinterpret_cast<const char*>(src[sg]) + al > buf_end) {
                                    al -= 16u;
                                    *reinterpret_cast<uint2*>(s_stage + st * pl.stage_bytes + pl.seg_off[sg] + al) =
                                        *reinterpret_cast<const uint2*>(buf_end - 8);
                                }
                                bytes[sg] = al;
                            }
                        }
                        total += bytes[sg];
                    }
                    mbar_arrive_expect_tx(staged_full + st, total);
#pragma unroll
                    for (int sg = 0; sg < NSEG; ++sg) {
#ifdef TN_CHECK
                        const char* b0 = FIRST ? reinterpret_cast<const char*>(cd.xf) : reinterpret_cast<const char*>(cd.seg[sg].xp);
                        const char* s0 = reinterpret_cast<const char*>(src[sg]);
                        TN_ASSERT(bytes[sg] == 0 ||
                                  (s0 >= b0 - 15 && s0 + bytes[sg] <= b0 + static_cast<int64_t>(cd.N) * cd.seg[sg].D *
                                                                             cd.seg[sg].H * cd.seg[sg].W *
                                                                             (FIRST ? 4 : 8 * cd.seg[sg].cw)));
                        TN_ASSERT(pl.seg_off[sg] + static_cast<int>(bytes[sg]) <=
                                  (sg + 1 < NSEG ? pl.seg_off[sg + 1] : pl.stage_bytes));
#endif
                        if (bytes[sg]) bulk_g2s(s_stage + st * pl.stage_bytes + pl.seg_off[sg], src[sg], bytes[sg],
                                                staged_full + st);
                    }
                    if (++st == static_cast<uint32_t>(pl.nstage)) { st = 0; ++st_r; }
                }
            }
        }
    } else if (warp >= kZExpWarp0 && warp < kZMmaWarp) {
        // ================= expanders: staged packed rows -> int8 strip of one plane
        const int et = threadIdx.x - kZExpWarp0 * 32;
        ZWalk wk(pl.units, cd.Do, pl.nstrip);
        int n, strip, zf, zl;
        uint32_t st = 0, st_r = 0, as = 0, as_r = 0;
        uint32_t e_par = 0;    // FIRST: code-plane double buffer parity (planes processed)
        (void)e_par;
        while (wk.next(n, strip, zf, zl)) {
            int i0, i1;
            run_planes(pl, cd, zf, zl, i0, i1);
            int ya[kMaxSeg], nr[kMaxSeg];
#pragma unroll
            for (int sg = 0; sg < NSEG; ++sg) strip_rows(pl, cd, strip, sg, ya[sg], nr[sg]);
            const int qa = strip * 128 * T - pl.qoff;
            for (int i = i0; i <= i1; ++i) {
                // one warp polls the barriers, the others park on a named barrier (polling
                // expander warps took ~15 % of the SM's issue slots from the epilogue)
                if (et < 32) {
                    TN_TW(2, et == 0, mbar_wait(staged_full + st, st_r & 1));
                    if (as_r > 0) TN_TW(3, et == 0, mbar_wait(plane_free + as, (as_r - 1) & 1));
                }
                asm volatile("bar.sync 2, %0;" ::"r"(kZExpThreads) : "memory");
                bool zok[kMaxSeg];
                uint32_t head[kMaxSeg];    // the loader's 16-byte alignment head of each segment's rows
#pragma unroll
                for (int sg = 0; sg < NSEG; ++sg) {
                    const SegDesc& sd = cd.seg[sg];
                    const int zs = (sd.up == 1 ? (i >> 1) : cd.zres + i * zst) - sd.zbeg;
                    zok[sg] = zs >= 0 && zs < sd.D;
                    head[sg] = FIRST ? 0u : static_cast<uint32_t>(reinterpret_cast<uintptr_t>(
                        sd.xp + ((static_cast<int64_t>(n) * sd.D + zs) * sd.H + ya[sg]) * sd.W * 2 * sd.cw)) & 15u;
                }
                const uint8_t* stg = s_stage + st * pl.stage_bytes;
                uint8_t* slot = s_a + as * pl.slot_bytes;
                if constexpr (FI8) {
                    // step 1: Eq. 6 on the staged float rows -> int8 codes (zero border of
                    // 4 columns and one row each side); non-finite -> d_bad
                    const SegDesc& sd = cd.seg[0];
                    uint8_t* code = s_stage + pl.code_off + (e_par & 1) * pl.code_bytes;
                    ++e_par;
                    const int W = sd.W, CP = pl.code_pitch, nrr = nr[0] + 2;
                    const int zb = i - sd.zbeg;
#pragma unroll 4
                    for (int e = et; e < nrr * (CP / 4); e += kZExpThreads) {
                        const int row = e / (CP / 4), c4 = e - row * (CP / 4);
                        const int x0 = 4 * c4 - 4;               // first of 4 voxels in this word
                        uint32_t wv = 0u;
                        if (zok[0] && row >= 1 && row <= nr[0] && x0 >= 0 && x0 < W) {
                            const float4 f = *reinterpret_cast<const float4*>(stg + ((row - 1) * W + x0) * 4);
                            const float fv[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
                            for (int b = 0; b < 4; ++b) {
                                const float v = fv[b];
                                if (!isfinite(v) && cd.d_bad != nullptr)
                                    atomicMin(reinterpret_cast<long long*>(cd.d_bad),
                                              static_cast<long long>(static_cast<int64_t>(n) * cd.bad_nstride + cd.bad_base +
                                                                     (static_cast<int64_t>(zb) * sd.H + ya[0] + row - 1) * W + x0 + b));
                                const uint32_t c = v > cd.t_hi ? 0x01u : (v < cd.t_lo ? 0xFFu : 0u);
                                wv |= c << (8 * b);
                            }
                        }
                        *reinterpret_cast<uint32_t*>(code + row * CP + 4 * c4) = wv;
                    }
                    asm volatile("bar.sync 1, %0;" ::"r"(kZExpThreads) : "memory");
                    // step 2: one 16-byte A row per output position of the strip: the 3x3
                    // in-plane window (bytes dy*3+dx), zero for separator / outside rows
                    const int q0 = strip * 128 * T;
#pragma unroll 4
                    for (int r = et; r < 128 * T; r += kZExpThreads) {
                        const int q = q0 + r;
                        const int y = div_po(static_cast<uint32_t>(q), pl.po_magic);
                        const int x = q - y * pl.Po;
                        uint4 a = make_uint4(0u, 0u, 0u, 0u);
                        if (x < W && y < sd.H) {
                            const int c0 = x + 3;                // code column of x - 1
                            const uint32_t sel = 0x3210u + (c0 & 3) * 0x1111u;
                            const uint8_t* rp = code + (y - ya[0]) * CP + (c0 & ~3);   // code row of y - 1
                            uint32_t rw[3];
#pragma unroll
                            for (int dy = 0; dy < 3; ++dy) {
                                const uint32_t* wp4 = reinterpret_cast<const uint32_t*>(rp + dy * CP);
                                rw[dy] = __byte_perm(wp4[0], wp4[1], sel);
                            }
                            a.x = __byte_perm(rw[0], rw[1], 0x4210u);
                            a.y = __byte_perm(rw[1], rw[2], 0x5421u);
                            a.z = rw[2] >> 16 & 0xFFu;
                        }
                        *reinterpret_cast<uint4*>(slot + r * 16) = a;
                    }
                } else {
                if constexpr (F4) {
                // FP4 rows: C = 16 segments write the position into the low half of
                // row r and the high half of row r-1 (a 16-byte guard row precedes each
                // region); C = 32 / 64 segments write one / two 16-byte rows.
                // A nearest-x2 upsampled C = 16 segment feeds 4 positions per source
                // voxel and plane: its staged words are converted to FP4 in place first
                // (packed 16 channels and FP4 16 channels are both 8 bytes).
                constexpr int CS = 16 * CT / NSEG;            // channels per segment (FP4 plans: 16, 32, 64)
                constexpr int BPV = FF4 ? 4 : (CS > 32 ? 16 : 8);   // staged bytes per voxel (FF4: a float)
                constexpr bool UPC = NSEG == 2 && CS == 16;
                if constexpr (UPC) {
                    uint2* p0 = reinterpret_cast<uint2*>(const_cast<uint8_t*>(stg) + pl.seg_off[0] + head[0]);
                    const int nv = nr[0] * cd.seg[0].W;
                    for (int e = et; e < nv; e += kZExpThreads) {
                        const uint2 w = p0[e];
                        p0[e] = expand16_f4_c16(w.x, w.y);
                    }
                    asm volatile("bar.sync 1, %0;" ::"r"(kZExpThreads) : "memory");
                }
                bool done_rows = false;
                if constexpr (NSEG == 1 && STR == 1) {
                    if (pl.rstg) {
                        // raster staging: strip row r is staged voxel r - rlo (rows [rlo, rhi) hold the
                        // copied packed rows, separators zero), so a row is one load, the expansion
                        // and its stores
                        int rlo = ya[0] * pl.Po - qa;
                        const int rhi = zok[0] ? rlo + nr[0] * pl.Po : rlo;
                        const uint32_t nval = static_cast<uint32_t>(rhi - rlo);
                        const uint32_t sbase = smem_u32(stg) - static_cast<uint32_t>(rlo * BPV);
                        const uint32_t a0 = smem_u32(slot) + 16;
#pragma unroll 2
                        for (int r = et; r < pl.RS; r += kZExpThreads) {
                            const bool ok = static_cast<uint32_t>(r - rlo) < nval;
                            const uint32_t dst = a0 + r * 16;
                            TN_ASSERT(!ok || (sbase + r * BPV >= smem_u32(stg) && sbase + (r + 1) * BPV <= smem_u32(stg) + pl.stage_bytes));
                            if constexpr (FF4) {
                                // A7 (reading R7): Eq. 6 with the float32 constants; the code is
                                // channel 0 of a 16-channel FP4 position (+1 -> 0x2, -1 -> 0xA)
                                float v = 0.5f * cd.t_lo + 0.5f * cd.t_hi;
                                if (ok) v = __uint_as_float(lds32(sbase + r * BPV));
                                const uint32_t c = v > cd.t_hi ? 0x2u : (v < cd.t_lo ? 0xAu : 0u);
                                if (!isfinite(v) && cd.d_bad != nullptr) {   // (separators hold a finite value)
                                    const int q = qa + r, y = q / pl.Po, x = q - y * pl.Po;
                                    atomicMin(reinterpret_cast<long long*>(cd.d_bad),
                                              static_cast<long long>(static_cast<int64_t>(n) * cd.bad_nstride + cd.bad_base +
                                                                     ((static_cast<int64_t>(i) - cd.seg[0].zbeg) * cd.seg[0].H + y) * cd.seg[0].W + x));
                                }
                                sts64(dst, make_uint2(c, 0u));
                                sts64(dst - 8, make_uint2(c, 0u));
                            } else if constexpr (CS == 16) {
                                uint2 w = make_uint2(0u, 0u);
                                if (ok) w = lds64(sbase + r * BPV);
                                const uint2 e = expand16_f4_c16(w.x, w.y);
                                sts64(dst, e);
                                sts64(dst - 8, e);
                            } else if constexpr (CS == 32) {
                                uint2 w = make_uint2(0u, 0u);
                                if (ok) w = lds64(sbase + r * BPV);
                                sts128(dst, expand32_f4(w.x, w.y));
                            } else {
                                uint4 w = make_uint4(0u, 0u, 0u, 0u);
                                if (ok) w = lds128(sbase + r * BPV);
                                sts128(dst, expand32_f4(w.x, w.z));
                                sts128(dst + pl.REG, expand32_f4(w.y, w.w));
                            }
                        }
                        done_rows = true;
                    }
                }
                // Row r of the strip = output raster position (y, x) (pitch Po); the plain
                // segment's staged voxel index L = y * Wp + x (stride 2: phase (py, px) reads
                // 2L + py * Wp + px) and the row's A address advance incrementally.
                int r = done_rows ? pl.RS : et;
                int y, x;
                {
                    const uint32_t tq = static_cast<uint32_t>(qa + r) + two_po;
                    y = div_po(tq, pl.po_magic) - pl.yoff;
                    x = static_cast<int>(tq) - (y + pl.yoff) * pl.Po;
                }
                const int Wp = cd.seg[NSEG - 1].W;
                int L = y * Wp + x;
                const int dL = pl.step_q * Wp + pl.step_r, dLw = Wp - pl.Po;
                uint32_t pbase[NSEG];
#pragma unroll
                for (int sg = 0; sg < NSEG; ++sg)
                    pbase[sg] = smem_u32(stg + pl.seg_off[sg] + head[sg]) - static_cast<uint32_t>(ya[sg] * cd.seg[sg].W * BPV);
                const uint32_t a0 = smem_u32(slot) + 16;
                const int Wo = cd.Wo;
                const unsigned Ho = static_cast<unsigned>(cd.Ho);
                for (; r < pl.RS; r += kZExpThreads) {
                    const bool v = x < Wo && static_cast<unsigned>(y) < Ho;
                    const uint32_t arow = a0 + r * 16;
#pragma unroll
                    for (int ph = 0; ph < NPH; ++ph) {
#pragma unroll
                        for (int sg = 0; sg < NSEG; ++sg) {
                            uint32_t src;
                            if (NSEG == 2 && sg == 0)     // nearest x2 (stride 1 only)
                                src = pbase[0] + static_cast<uint32_t>(((y >> 1) * cd.seg[0].W + (x >> 1)) * BPV);
                            else if (STR == 2)
                                src = pbase[sg] + static_cast<uint32_t>((2 * L + (ph >> 1) * Wp + (ph & 1)) * BPV);
                            else
                                src = pbase[sg] + static_cast<uint32_t>(L * BPV);
                            const bool ok = v && zok[sg];
                            const uint32_t dst = arow + (ph * pl.nreg + pl.reg0[sg]) * pl.REG;
                            TN_ASSERT(dst + (CS > 32 ? pl.REG + 16 : 16) <= smem_u32(slot) + pl.slot_bytes && dst >= smem_u32(slot) + 8);
                            TN_ASSERT(!(v && zok[sg]) || (src >= smem_u32(stg) + pl.seg_off[sg] &&
                                                          src + BPV <= smem_u32(stg) + pl.stage_bytes));
                            if constexpr (CS == 16) {
                                uint2 w = make_uint2(0u, 0u);
                                if (ok) w = lds64(src);
                                const uint2 e = (NSEG == 2 && sg == 0) ? w : expand16_f4_c16(w.x, w.y);
                                sts64(dst, e);
                                sts64(dst - 8, e);
                            } else if constexpr (CS == 32) {
                                uint2 w = make_uint2(0u, 0u);
                                if (ok) w = lds64(src);
                                sts128(dst, expand32_f4(w.x, w.y));
                            } else {
                                uint4 w = make_uint4(0u, 0u, 0u, 0u);
                                if (ok) w = lds128(src);
                                sts128(dst, expand32_f4(w.x, w.z));
                                sts128(dst + pl.REG, expand32_f4(w.y, w.w));
                            }
                        }
                    }
                    x += pl.step_r;
                    y += pl.step_q;
                    L += dL;
                    if (x >= pl.Po) { x -= pl.Po; ++y; L += dLw; }
                }
                } else {
                // Rows r = et + 256 j: (y, x) of the output raster tracked incrementally
                // (256 = qd * Po + rd), all phases of a row from the same (y, x).
                int r = et;
                int y, x;
                {
                    const uint32_t tq = static_cast<uint32_t>(qa + r) + two_po;
                    y = div_po(tq, pl.po_magic) - pl.yoff;
                    x = static_cast<int>(tq) - (y + pl.yoff) * pl.Po;
                }
                for (; r < pl.RS; r += kZExpThreads) {
                    const bool vx = x < cd.Wo && y >= 0;
#pragma unroll
                    for (int ph = 0; ph < NPH; ++ph) {
                        const int py = ph >> 1, px = ph & 1;
                        const int yi = STR == 2 ? 2 * y + py : y, xi = STR == 2 ? 2 * x + px : x;
                        const bool v = vx && yi < cd.Hci && xi < cd.Wci;
                        uint8_t* dst = slot + (ph * CT) * pl.REG + r * 16;
#pragma unroll
                        for (int sg = 0; sg < NSEG; ++sg) {
                            const SegDesc& sd = cd.seg[sg];
                            constexpr bool kUp0 = NSEG == 2;      // plan: two segments = [up, skip]
                            const bool up = sg == 0 && kUp0;
                            const int ys = up ? (yi >> 1) : yi, xs = up ? (xi >> 1) : xi;
                            const bool ok = v && zok[sg];
                            const uint8_t* sp = stg + pl.seg_off[sg] + head[sg] + ((ys - ya[sg]) * sd.W + xs) * 8 * sd.cw;
                            const int choff = sg ? pl.cch[0] : 0;
                            if (sd.cw == 1) {
                                uint2 w = make_uint2(0u, 0u);
                                if (ok) w = *reinterpret_cast<const uint2*>(sp);
                                *reinterpret_cast<uint4*>(dst + choff * pl.REG) = expand16(w.x, w.y, 0);
                                if (pl.cch[sg] > 1) *reinterpret_cast<uint4*>(dst + (choff + 1) * pl.REG) = expand16(w.x, w.y, 16);
                            } else {
                                uint4 w = make_uint4(0u, 0u, 0u, 0u);
                                if (ok) w = *reinterpret_cast<const uint4*>(sp);
                                const int cch = pl.cch[sg];
                                *reinterpret_cast<uint4*>(dst + choff * pl.REG) = expand16(w.x, w.z, 0);
                                if (cch > 1) *reinterpret_cast<uint4*>(dst + (choff + 1) * pl.REG) = expand16(w.x, w.z, 16);
                                if (cch > 2) *reinterpret_cast<uint4*>(dst + (choff + 2) * pl.REG) = expand16(w.y, w.w, 0);
                                if (cch > 3) *reinterpret_cast<uint4*>(dst + (choff + 3) * pl.REG) = expand16(w.y, w.w, 16);
                            }
                        }
                    }
                    x += pl.step_r;
                    y += pl.step_q;
                    if (x >= pl.Po) { x -= pl.Po; ++y; }
                }
                }   // !F4
                }   // !FIRST
                mbar_arrive(staged_empty + st);
                fence_proxy_async();
                mbar_arrive(plane_full + as);
                if (++st == static_cast<uint32_t>(pl.nstage)) { st = 0; ++st_r; }
                if (++as == static_cast<uint32_t>(pl.nslot)) { as = 0; ++as_r; }
            }
        }
    } else if (warp >= kZMmaWarp && warp < kZMmaWarp + kZMmaWarps) {
        // ================= MMA issuers (warp mw takes the tiles t % 2 == mw).  Descriptor low words are precomputed per
        // K-slice pair (start address and LBO); per (slot, tile) only an add remains,
        // so the issue loop stays well under the 40+ cycles one N = 3K MMA takes.
        // F4 slices: 6 per C = 16 segment (two-position rows), 9 per 32 channels
        constexpr int NMMA = F4 ? (NSEG == 1 ? (CT == 1 ? 3 : (CT == 2 ? 5 : 9))
                                             : (CT == 2 ? 6 : (CT == 3 ? 8 : (CT == 4 ? 9 : 18))))
                                : (FIRST ? 1 : (9 * CT + 1) / 2);
        const uint32_t sfa = tmem_base + 480, sfb = tmem_base + 496;
        auto idesc_n = [](uint32_t n) { return F4 ? idesc_mxf4(static_cast<int>(n)) : idesc_i8(static_cast<int>(n)); };
        auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
            if constexpr (F4) tc_mma_mxf4(d, a, b, id, sfa, sfb);
            else tc_mma_i8(d, a, b, id, 1u);
        };
        const bool leader = elect_one();
        const uint32_t a_base = smem_u32(s_a), b_base = smem_u32(s_b);
        const uint32_t b_half = NB * K * 16;          // LBO of B (bytes between the two K halves)
        const uint32_t b_mma16 = (2 * b_half) >> 4;   // descriptor step per MMA's B operand
        uint32_t a_lo[NMMA];
#pragma unroll
        for (int m = 0; m < NMMA; ++m)
            a_lo[m] = (((a_base + pl.a_off[m]) >> 4) & 0x3FFFu) | ((static_cast<uint32_t>(pl.a_lbo[m]) >> 4) << 16);
        const uint32_t b_lo0 = ((b_base >> 4) & 0x3FFFu) | ((b_half >> 4) << 16);
        auto desc64 = [](uint32_t lo) { return (static_cast<uint64_t>(0x4008u) << 32) | lo; };   // SBO 128, v1
        // accumulator-start MMA(s) (BIAS): A constants (LBO 2048), B start rows (LBO 16 K), N = K; the
        // first overwrites the block
        const uint64_t bias_a = desc64(((smem_u32(s_bias) >> 4) & 0x3FFFu) | ((2048u >> 4) << 16));
        const uint64_t bias_b = desc64(((smem_u32(s_bias + kZBiasA) >> 4) & 0x3FFFu) | (static_cast<uint32_t>(K) << 16));
        auto start_mma = [&](uint32_t d) {
#pragma unroll
            for (int j = 0; j < NBM; ++j) {
                if constexpr (F4) tc_mma_mxf4_acc(d, bias_a, bias_b + j * 2 * K, idesc_n(K), sfa, sfb, j > 0 ? 1u : 0u);
                else tc_mma_i8(d, bias_a, bias_b, idesc_n(K), 0u);
            }
        };
        // One lane runs the whole schedule (waits, MMAs, commits are per-thread
        // operations), so no warp-level bookkeeping sits in the per-tile loop.
        if (leader) {
#ifdef TN_TRACE
            const long long m_t0 = clock64();
#endif
            ZWalk wk(pl.units, cd.Do, pl.nstrip);
            int n, strip, zf, zl;
            uint32_t as = 0, as_r = 0;
            uint32_t u_run = 0;                        // running output index of the run's first plane
            while (wk.next(n, strip, zf, zl)) {
                int i0, i1;
                run_planes(pl, cd, zf, zl, i0, i1);
                const int Tv = min(T, pl.NT - strip * T);
                const int zg0 = cd.zo_beg + zf, zg1 = cd.zo_beg + zl;
                for (int i = i0; i <= i1; ++i) {
                    if constexpr (STR == 1 && !SPLIT && !ONEP) {
                        // steady state, decided without the per-output bookkeeping below (the
                        // issuing thread is latency-bound): plane i starts output i+1 (its block
                        // was used before: wait for the epilogue), completes output i-1 (commit)
                        // and continues output i; all three outputs in the run
                        const uint32_t u_lo = u_run + static_cast<uint32_t>(i - 1 - zg0);
                        if (i >= 1 && i + 2 <= cd.Dci && i - 1 >= zg0 && i + 1 <= zg1 && u_lo + 2 >= RO) {
                            const uint32_t r = u_lo % RO;                // sigma of output i-1
                            const uint32_t b0 = r == 0 ? 0 : (r == 1 ? 2 : 1);
                            const uint32_t bl_full = b_lo0 + b0 * K;
                            const uint32_t un = u_lo + 2;
                            const int v0 = warp - kZMmaWarp;
                            const uint32_t wbar = smem_u32(acc_empty + (un % RO) * NU + v0), wpar = ((un / RO) - 1) & 1;
                            const uint32_t cbar = smem_u32(acc_full + r * NU + v0);
                            constexpr uint32_t kBarStep = 8 * kZMmaWarps;
                            const uint32_t idesc = idesc_n(RO * K);
                            TN_TW(4, warp == kZMmaWarp, mbar_wait(plane_full + as, as_r & 1));
                            const uint32_t a_slot16 = (as * pl.slot_bytes) >> 4;
                            int k = 0;
                            for (int v = v0; v < NU; v += kZMmaWarps, ++k) {   // (units past Tv: empty commit)
                                TN_TW(5, warp == kZMmaWarp, mbar_wait_addr(wbar + k * kBarStep, wpar));
                                tc_fence_after();
                                if (v < Tv) {
                                    const uint32_t a_t = a_slot16 + v * 128;
                                    const uint32_t d_tile = tmem_base + v * RO * K;
                                    if constexpr (BIAS) start_mma(d_tile + (un % RO) * K);
                                    TN_TW(1, warp == kZMmaWarp, {
#pragma unroll
                                    for (int m = 0; m < NMMA; ++m)
                                        mma(d_tile, desc64(a_lo[m] + a_t), desc64(bl_full + m * b_mma16), idesc);
                                    });
                                }
                                tc_commit_addr(cbar + k * kBarStep);
                            }
                            tc_commit(plane_free + as);
                            if (++as == static_cast<uint32_t>(pl.nslot)) { as = 0; ++as_r; }
                            continue;
                        }
                    }
                    // outputs touched by plane i: STR 1: z = i-1, i, i+1 (dz = 2, 1, 0);
                    // STR 2: z with 2z-1 <= i <= 2z+1
                    int zlo, zhi;
                    if (STR == 1) { zlo = max(i - 1, zg0); zhi = min(i + 1, zg1); }
                    else { zlo = max(i >> 1, zg0); zhi = min((i + 1) >> 1, zg1); }
                    const int nz = zhi - zlo + 1;
                    const bool full = nz == RO;
                    // per plane: blocks newly started (wait for the epilogue), completed
                    // (commit), and for partial planes each output's block and B block
                    uint32_t new_bar[3] = {0, 0, 0}, new_par[3] = {0, 0, 0}, done_bar[3] = {0, 0, 0};
                    uint32_t sgl_d[3] = {0, 0, 0}, sgl_b[3] = {0, 0, 0};
                    bool is_new[3] = {false, false, false}, is_done[3] = {false, false, false};
                    bool is_first[3] = {false, false, false};    // plane i starts output zlo + j
                    const uint32_t u_lo = u_run + (zlo - zg0);
#pragma unroll
                    for (int j = 0; j < 3; ++j) {
                        const int z = zlo + j;
                        if (j < nz) {
                            const uint32_t u = u_lo + j;
                            const uint32_t sg = u % RO;
                            const int first = max(STR * z - 1, 0), last = min(STR * z + 1, cd.Dci - 1);
                            is_new[j] = first == i && u >= static_cast<uint32_t>(RO);
                            is_first[j] = first == i;
                            new_bar[j] = sg * NU;
                            new_par[j] = ((u / RO) - 1) & 1;
                            is_done[j] = last == i;
                            done_bar[j] = sg * NU;
                            const int dz = i - STR * z + 1;
                            // block holding dz: s1 [2 1 0 ..] -> 2 - dz; s2 [0 2 0 1] -> dz0:0 dz2:1 dz1:3
                            sgl_b[j] = ONEP ? 0 : STR == 1 ? 2 - dz : (dz == 0 ? 0 : (dz == 2 ? 1 : 3));
                            sgl_d[j] = sg * K;
                        }
                    }
                    uint32_t bl_full = b_lo0;
                    // SPLIT: blocks sigma(u_lo) .. in up to two contiguous groups
                    uint32_t g_n1 = 0, g_n2 = 0, g_d1 = 0, g_b1 = 0, g_b2 = 0;
                    if constexpr (SPLIT) {
                        const uint32_t s0 = u_lo % RO;
                        const uint32_t blk0 = static_cast<uint32_t>(zlo - (i - 1));
                        g_n1 = min(static_cast<uint32_t>(nz), RO - s0);
                        g_n2 = nz - g_n1;
                        g_d1 = s0 * K;
                        g_b1 = b_lo0 + blk0 * K;
                        g_b2 = b_lo0 + (blk0 + g_n1) * K;
                    }
                    if (!SPLIT && full) {
                        // rotation: block position p holds the output with sigma = p
                        const uint32_t r = u_lo % RO;                 // sigma of the lowest output
                        const uint32_t b0 = ONEP ? 0 : STR == 1 ? (r == 0 ? 0 : (r == 1 ? 2 : 1)) : (r ? 0 : 1);
                        bl_full = b_lo0 + b0 * K;
                    }
                    TN_TW(4, warp == kZMmaWarp, mbar_wait(plane_full + as, as_r & 1));
                    const uint32_t a_slot16 = (as * pl.slot_bytes) >> 4;
                    // steady-state fast path (stride 1, rotated B): the plane starts output
                    // i+1 (one wait per tile) and completes output i-1 (one commit per tile);
                    // descriptors precomputed per plane, so a tile is ~2 + 2*NMMA instructions
                    const bool fast = !SPLIT && STR == 1 && full && is_new[2] && !is_new[0] && !is_new[1] &&
                                      is_done[0] && !is_done[1] && !is_done[2];
                    if (fast) {
                        uint32_t a_pl[NMMA], b_pl[NMMA];
#pragma unroll
                        for (int m = 0; m < NMMA; ++m) { a_pl[m] = a_lo[m] + a_slot16; b_pl[m] = bl_full + m * b_mma16; }
                        const uint32_t idesc = idesc_n(RO * K);
                        const int v0 = warp - kZMmaWarp;
                        const uint32_t wbar = smem_u32(acc_empty + new_bar[2] + v0), wpar = new_par[2];
                        const uint32_t cbar = smem_u32(acc_full + done_bar[0] + v0);
                        constexpr uint32_t kBarStep = 8 * kZMmaWarps;
                        int k = 0;
                        for (int v = v0; v < NU; v += kZMmaWarps, ++k) {   // (units past Tv: empty commit)
                            TN_TW(5, warp == kZMmaWarp, mbar_wait_addr(wbar + k * kBarStep, wpar));
                            tc_fence_after();
                            const int t1 = min(v + 1, Tv);
                            TN_TW(1, warp == kZMmaWarp, {
                            for (int t = v; t < t1; ++t) {
                                const uint32_t a_add = t * 128;
                                const uint32_t d_tile = tmem_base + t * RO * K;
                                if constexpr (BIAS) start_mma(d_tile + sgl_d[2]);
#pragma unroll
                                for (int m = 0; m < NMMA; ++m)
                                    mma(d_tile, desc64(a_pl[m] + a_add), desc64(b_pl[m]), idesc);
                            }
                            });
                            tc_commit_addr(cbar + k * kBarStep);
                        }
                    } else
                    // every synchronisation unit of the strip takes part, also those past the
                    // last tile of a ragged strip (no MMAs, an empty commit): the per-unit
                    // barriers then advance one phase per output plane in every strip, which the
                    // parities assume when a CTA's range continues into a full strip (n > 1)
                    for (int v = warp - kZMmaWarp; v < NU; v += kZMmaWarps) {
#pragma unroll
                        for (int j = 0; j < 3; ++j)
                            if (is_new[j]) TN_TW(5, warp == kZMmaWarp, mbar_wait(acc_empty + new_bar[j] + v, new_par[j]));
                        tc_fence_after();
                        const int t1 = min(v + 1, Tv);
                        for (int t = v; t < t1; ++t) {
                        const uint32_t a_add = a_slot16 + t * 128;    // (t * 128 rows * 16 B) >> 4
                        const uint32_t d_tile = tmem_base + t * RO * K;
                        if constexpr (BIAS) {
#pragma unroll
                            for (int j = 0; j < 3; ++j)
                                if (is_first[j]) start_mma(d_tile + sgl_d[j]);
                        }
                        if constexpr (SPLIT) {
                            const uint32_t idesc1 = idesc_n(g_n1 * K);
#pragma unroll
                            for (int m = 0; m < NMMA; ++m)
                                mma(d_tile + g_d1, desc64(a_lo[m] + a_add), desc64(g_b1 + m * b_mma16), idesc1);
                            if (g_n2) {
                                const uint32_t idesc2 = idesc_n(g_n2 * K);
#pragma unroll
                                for (int m = 0; m < NMMA; ++m)
                                    mma(d_tile, desc64(a_lo[m] + a_add), desc64(g_b2 + m * b_mma16), idesc2);
                            }
                        } else if (full) {
                            const uint32_t idesc = idesc_n(RO * K);
#pragma unroll
                            for (int m = 0; m < NMMA; ++m)
                                mma(d_tile, desc64(a_lo[m] + a_add), desc64(bl_full + m * b_mma16), idesc);
                        } else {
                            const uint32_t idesc = idesc_n(K);
#pragma unroll
                            for (int j = 0; j < 3; ++j) {
                                if (j < nz) {
                                    const uint32_t bl = b_lo0 + sgl_b[j] * K;
#pragma unroll
                                    for (int m = 0; m < NMMA; ++m)
                                        mma(d_tile + sgl_d[j], desc64(a_lo[m] + a_add), desc64(bl + m * b_mma16),
                                                  idesc);
                                }
                            }
                        }
                        }   // tiles of the unit
#pragma unroll
                        for (int j = 0; j < 3; ++j)
                            if (is_done[j]) tc_commit(acc_full + done_bar[j] + v);
                    }
                    tc_commit(plane_free + as);
                    if (++as == static_cast<uint32_t>(pl.nslot)) { as = 0; ++as_r; }
                }
                u_run += zl - zf + 1;
            }
#ifdef TN_TRACE
            if (warp == kZMmaWarp) atomicAdd(&g_tn_trace[blockIdx.x * 8 + 7], clock64() - m_t0);   // MMA role span
#endif
        }
        __syncwarp();
    } else {
        // ================= epilogue
        const int q = warp & 3, g = warp >> 2;
        ZWalk wk(pl.units, cd.Do, pl.nstrip);
        int n, strip, zf, zl;
        uint32_t u = 0;
        const uint32_t lane_base = static_cast<uint32_t>(32 * q) << 16;
        // K = 16: thresholds and the re-init values live in registers
        constexpr bool REGT = K == 16;
        constexpr bool LMHR = REGT;   // (thresholds re-read from shared memory per tile: #2 +3 %)
        int r_lmh[16];
        if constexpr (LMHR) {
#pragma unroll
            for (int k = 0; k < 16; ++k) r_lmh[k] = s_lmh[k];
        }
        while (wk.next(n, strip, zf, zl)) {
            const int Tv = min(T, pl.NT - strip * T);
            const int q_lane = strip * 128 * T + 32 * q + lane;
            for (int z = zf; z <= zl; ++z, ++u) {
                const uint32_t sgm = u % RO, par = (u / RO) & 1;
                const int zg = cd.zres + z * zst;                   // output plane in the buffer
                const int64_t vplane = (static_cast<int64_t>(n) * dbuf + zg) * cd.Ho * cd.Wo;
                // raster position of this lane in tile t -> (offset within the plane, valid)
                auto position = [&](int t, int& voff) {
                    const int qpos = q_lane + t * 128;
                    const int y = div_po(static_cast<uint32_t>(qpos), pl.po_magic);
                    const int x = qpos - y * pl.Po;
                    voff = y * cd.Wo + x;
                    return x < cd.Wo && y < cd.Ho;
                };
                // the requantised codes of one position: A8 prediction (last layer), packed store,
                // NEXT-1 halo stores
                auto finish = [&](int voff, const uint32_t (&sbits)[CWO], const uint32_t (&mbits)[CWO]) {
                    if (PRED) {
                        // A8 (reading R12): b + sum_k w_k t_k in fp32, k ascending (quad tables)
                        const int64_t v = static_cast<int64_t>(zg) * cd.Ho * cd.Wo + voff;
                        if (cd.nclass == 2 && K == 16) {
                            // quad indices (mask nibble | sign nibble << 4): bytes of q02 = quads 0, 2;
                            // bytes of q13 = quads 1, 3
                            const uint32_t q02 = (mbits[0] & 0x0F0Fu) | ((sbits[0] & 0x0F0Fu) << 4);
                            const uint32_t q13 = ((mbits[0] >> 4) & 0x0F0Fu) | (sbits[0] & 0xF0F0u);
                            const uint32_t idx[4] = {q02 & 0xFFu, q13 & 0xFFu, (q02 >> 8) & 0xFFu, (q13 >> 8) & 0xFFu};
                            float a0 = s_pred[0], a1 = s_pred[1];
#pragma unroll
                            for (int qd = 0; qd < 4; ++qd) {
                                const float2 e2 = *reinterpret_cast<const float2*>(s_ptab + (qd * 256 + idx[qd]) * 2);
                                a0 += e2.x;
                                a1 += e2.y;
                            }
                            float* lg = cd.logits + static_cast<int64_t>(n) * 2 * cd.lstride + v;
                            lg[0] = a0;
                            lg[cd.lstride] = a1;
                        } else {
                            for (int j = 0; j < cd.nclass; ++j) {
                                float a = s_pred[j];
                                const float* tab = s_ptab + j * (K / 4) * 256;
#pragma unroll
                                for (int qd = 0; qd < K / 4; ++qd) {
                                    const uint32_t w = qd >> 3, sh = 4 * (qd & 7);
                                    const uint32_t ix = ((mbits[w] >> sh) & 0xFu) | (((sbits[w] >> sh) & 0xFu) << 4);
                                    a += tab[qd * 256 + ix];
                                }
                                cd.logits[(static_cast<int64_t>(n) * cd.nclass + j) * cd.lstride + v] = a;
                            }
                        }
                        if (cd.no_yp) return;   // last FCN layer: only the logits are consumed
                    }
                    TN_ASSERT(voff >= 0 && voff < cd.Ho * cd.Wo && vplane + voff < static_cast<int64_t>(cd.N) * dbuf * cd.Ho * cd.Wo);
                    uint32_t* dst = cd.yp + (vplane + voff) * 2 * CWO;
                    if constexpr (CWO == 1) {
                        *reinterpret_cast<uint2*>(dst) = make_uint2(sbits[0], mbits[0]);
                    } else {
                        *reinterpret_cast<uint4*>(dst) = make_uint4(sbits[0], sbits[1], mbits[0], mbits[1]);
                    }
                    if (cd.halo_lo != nullptr || cd.halo_hi != nullptr) {   // NEXT-1 slab boundary planes
                        const uint32_t wds[4] = {sbits[0], CWO == 1 ? mbits[0] : sbits[CWO - 1], mbits[0], mbits[CWO - 1]};
                        halo_store_words(cd.halo_lo, cd.halo_hi, z, cd.Do, voff, wds, 2 * CWO);
                    }
                };
                // A4 (reading R5) on one 16-channel chunk: acc holds acc - hi (initialised to -hi).
                // +1 if acc >= hi; else -1 if acc <= lo; else 0.  Bit k of nhi = (acc_k < hi_k); bit k
                // of nlo = (acc_k > lo_k) = ((lo-hi) - d < 0).  F4: f32 accumulators start at 0.5 - hi
                // and lmh = lo - hi + 1, so d and lmh - d are never zero (acc integer): no
                // sign-of-zero ambiguity.  Returns sign bits (low 16) and mask bits (high 16).
                auto requant16 = [&](const int* acc, const int* lmh, const int* nh) {
                    uint32_t nhi = 0u, nlo = 0u;
#pragma unroll
                    for (int i = 15; i >= 0; --i) {
                        // int8 K >= 32: the block started at zero, so d = acc + (-hi) here; the
                        // accumulator-start MMA (BIAS) already started it at -hi (F4: 0.5 - hi)
                        const int d = (REGT || BIAS) ? acc[i]
                                           : (F4 ? __float_as_int(__int_as_float(acc[i]) + __int_as_float(nh[i]))
                                                 : acc[i] + nh[i]);
                        nhi = __funnelshift_l(static_cast<uint32_t>(d), nhi, 1);
                        const int e = F4 ? __float_as_int(__int_as_float(lmh[i]) - __int_as_float(d)) : lmh[i] - d;
                        nlo = __funnelshift_l(static_cast<uint32_t>(e), nlo, 1);
                    }
                    return (~nhi & 0xFFFFu) | ((~(nhi & nlo) & 0xFFFFu) << 16);
                };
                for (int v = g; v < NU; v += kZEpiGroups) {   // all units (see the MMA issuer)
                    TN_TW(6, threadIdx.x == 0, mbar_wait(acc_full + sgm * NU + v, par));
                    tc_fence_after();
                    const int t = v;                      // one tile per unit
                    if (t >= Tv) {                        // past a ragged strip's last tile: no MMAs ran,
                        mbar_arrive(acc_empty + sgm * NU + v);   // the block still holds its initial values
                        continue;
                    }
                    const uint32_t taddr = tmem_base + lane_base + (t * RO + sgm) * K;
                    int voff;
                    const bool vpos = position(t, voff);
                    uint32_t sbits[CWO], mbits[CWO];
                    // K <= 32: the whole tile's accumulators go to registers first and the block is
                    // re-initialised and handed back to the MMA issuer at once, so the next MMAs into
                    // it overlap this tile's requant / stores.  K = 64: chunk by chunk (registers).
                    constexpr bool EARLY = K <= 32 || (!SPLIT && STR == 1);
                    constexpr int NCH = EARLY ? K / 16 : 1;
                    int accs[NCH][16];
                    // the output that reuses the block starts at -hi (K = 16, thresholds in registers)
                    // or at zero (K >= 32: no threshold loads and no value registers before the
                    // hand-back; the requant adds -hi)
                    // (K = 16: the accumulator-start MMA re-initialises the block, nothing to store)
                    auto reinit = [&](int c) {
                        if constexpr (!BIAS) tmem_st16_fill(taddr + c, 0);
                    };
                    if constexpr (EARLY) {
#pragma unroll
                        for (int ch = 0; ch < NCH; ++ch) tmem_ld16(taddr + 16 * ch, accs[ch]);
                        tmem_wait_ld();
                        if constexpr (!BIAS) {
#pragma unroll
                            for (int ch = 0; ch < NCH; ++ch) reinit(16 * ch);
                            tmem_wait_st();
                        }
                        tc_fence_before();
                        mbar_arrive(acc_empty + sgm * NU + v);
                    }
#pragma unroll
                    for (int c = 0; c < K; c += 16) {
                        int* acc = accs[EARLY ? c / 16 : 0];
                        if constexpr (!EARLY) {
                            tmem_ld16(taddr + c, accs[0]);
                            tmem_wait_ld();
                        }
                        int lmh[16], nh[16];
                        if constexpr (LMHR) {
#pragma unroll
                            for (int i = 0; i < 16; ++i) lmh[i] = r_lmh[i];
                        } else {
#pragma unroll
                            for (int i4 = 0; i4 < 4; ++i4) {
                                const int4 l4 = *reinterpret_cast<const int4*>(s_lmh + c + 4 * i4);
                                lmh[4 * i4] = l4.x; lmh[4 * i4 + 1] = l4.y; lmh[4 * i4 + 2] = l4.z; lmh[4 * i4 + 3] = l4.w;
                                const int4 h4 = *reinterpret_cast<const int4*>(s_nhi + c + 4 * i4);
                                nh[4 * i4] = h4.x; nh[4 * i4 + 1] = h4.y; nh[4 * i4 + 2] = h4.z; nh[4 * i4 + 3] = h4.w;
                            }
                        }
                        if (fused) {
                            const uint32_t bits = requant16(acc, lmh, nh);
                            const int w = c >> 5, sh = c & 31;
                            const uint32_t sb = (bits & 0xFFFFu) << sh, mb = (bits >> 16) << sh;
                            if (sh == 0) { sbits[w] = sb; mbits[w] = mb; }
                            else { sbits[w] |= sb; mbits[w] |= mb; }
                        } else if (vpos) {
                            if (F4) {
#pragma unroll
                                for (int i = 0; i < 16; ++i) acc[i] = __float2int_rn(__int_as_float(acc[i]));
                            }
                            TN_ASSERT(vplane + voff < static_cast<int64_t>(cd.N) * dbuf * cd.Ho * cd.Wo);
                            if (cd.K == K) {
                                int4* dst = reinterpret_cast<int4*>(cd.y + (vplane + voff) * K + c);
#pragma unroll
                                for (int i = 0; i < 4; ++i)
                                    dst[i] = make_int4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
                            } else {   // padded K: the logical channels only (row pitch cd.K)
                                int32_t* dst = cd.y + (vplane + voff) * cd.K;
#pragma unroll
                                for (int i = 0; i < 16; ++i)
                                    if (c + i < cd.K) dst[c + i] = acc[i];
                            }
                        }
                        if constexpr (!EARLY) reinit(c);
                    }
                    if constexpr (!EARLY) {
                        tmem_wait_st();
                        tc_fence_before();
                        mbar_arrive(acc_empty + sgm * NU + v);
                    }
                    if (fused && vpos) finish(voff, sbits, mbits);
                }
            }
        }
    }


    tc_fence_before();
    __syncthreads();
#ifdef TN_TRACE
    if (threadIdx.x == 0) atomicAdd(&g_tn_trace[blockIdx.x * 8 + 0], clock64() - k_t0);
#endif
    if (warp == kZMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
    }
}

int g_num_sms_z = 0;

// Persistent grid for `units` units over at most `cap` CTAs.  When a CTA gets only a few units the
// launch is bound by the longest CTA (ceil(units / cap) units), so the same critical path is kept
// with every CTA at that count (fewer CTAs contend for the prologue's B-image copies, TMEM
// allocation and the shared input planes).  Measured: configs[0] 160 units -> 80 CTAs of two,
// 7.61 -> 6.92 us per launch; configs[1] / configs[2] unchanged at any limit from 2 to 64 units.
int tz_grid(int64_t units, int cap) {
    static const bool no_bal = ab_env("TN_TZ_NO_BALANCE") != nullptr;   // A/B switch (measurement)
    const int64_t per = (units + cap - 1) / cap;
    if (no_bal || per > 4) return static_cast<int>(std::min<int64_t>(units, cap));
    return static_cast<int>((units + per - 1) / per);
}

}  // namespace

// ---------------------------------------------------------------- host plan
static int round_up(int v, int a) { return (v + a - 1) / a * a; }

// Launch with programmatic stream serialisation (see pdl_wait in the kernel).
static cudaError_t launch_pdl(void (*kern)(ConvDesc, TzPlan), int grid, int threads, size_t smem, cudaStream_t st,
                              const ConvDesc& cd, const TzPlan& pl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(static_cast<unsigned>(threads));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, cd, pl);
    return e != cudaSuccess ? e : cudaGetLastError();
}

static size_t tz_smem(const TzPlan& pl, int K) {
    return static_cast<size_t>(pl.nslot) * pl.slot_bytes + pl.b_bytes + static_cast<size_t>(pl.nstage) * pl.stage_bytes +
           2 * static_cast<size_t>(pl.code_bytes) + pl.wpad + pl.bias_bytes +
           2 * K * sizeof(int) + (kZMaxClass + pl.ptab_floats) * sizeof(float) +
           (2 * kZMaxSlot + 2 * kZMaxStage + 2 * kZMaxAcc) * 8 + 16;
}

static int tz_num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0, v = 0;
        n = (cudaGetDevice(&dev) == cudaSuccess &&
             cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) ? v : 148;
        cudaGetLastError();   // no device (CPU-side planning): clear the error, assume B200
    }
    return n;
}

static bool plan_tz(const ConvDesc& cd, TzPlan& pl, bool first = false, bool f4 = false) {
    constexpr size_t kSmemMax = 227 * 1024;
    if (cd.nseg < 1 || cd.nseg > 2) return false;
    // isotropic: stride 1 or 2 with pad 1, or stride 1 with pad = dilation > 1 (int8 operands,
    // one plain segment; the caller launches each z residue class mod the dilation separately)
    for (int a = 0; a < 3; ++a)
        if (cd.s[a] != cd.s[0] || cd.p[a] != cd.dl[0] || cd.dl[a] != cd.dl[0]) return false;
    pl.s = cd.s[0];
    pl.dil = cd.dl[0];
    if (pl.dil < 1 || (pl.dil > 1 && (pl.s != 1 || f4 || first || cd.nseg != 1))) return false;
    if (pl.s != 1 && !(pl.s == 2 && cd.nseg == 1 && cd.seg[0].up == 0)) return false;
    // the kernel fixes the segment pattern: one plain segment, or [nearest-x2 upsampled, plain]
    // (up 1 = nearest x2 in z, y, x; up 2 = in y and x only, the 2D decoders of Table 1)
    if (cd.nseg == 1 ? cd.seg[0].up != 0 : (cd.seg[0].up == 0 || cd.seg[1].up != 0)) return false;
    // K padded to the next of 16 / 32 / 64 (zero filters, "always 0" thresholds for the pad)
    if (cd.K < 1 || cd.K > 64) return false;
    pl.kp = cd.K <= 16 ? 16 : (cd.K <= 32 ? 32 : 64);
    if (cd.logits != nullptr && (cd.K != pl.kp || cd.K > 32 || cd.nclass < 1 || cd.nclass > kZMaxClass ||
                                 cd.yp == nullptr || cd.nclass * cd.K > 64))
        return false;
    int ct = 0;
    pl.cch[1] = 0;
    for (int i = 0; i < cd.nseg && !first; ++i) {
        const SegDesc& sd = cd.seg[i];
        // 16-channel chunks; padding lanes are zero in the packed format (reading R4)
        if (sd.c <= 0 || sd.c > 64 || (sd.c + 31) / 32 != sd.cw) return false;
        if ((reinterpret_cast<uintptr_t>(sd.xp) & 15) || (reinterpret_cast<uintptr_t>(sd.wp) & 15)) return false;
        pl.cch[i] = (sd.c + 15) / 16;
        ct += pl.cch[i];
    }
    if (first) {   // one float input channel; 9 in-plane taps per 16-byte A row
        const SegDesc& sd = cd.seg[0];
        if (cd.nseg != 1 || pl.s != 1 || sd.up || sd.c != 1 || sd.W % 4 != 0 || cd.K > 32 || cd.logits != nullptr) return false;
        if (f4 && !(cd.t_lo <= cd.t_hi)) return false;   // FF4 separators: a value Eq. 6 maps to 0
        if ((reinterpret_cast<uintptr_t>(cd.xf) & 15) || (reinterpret_cast<uintptr_t>(sd.wp) & 15)) return false;
        pl.cch[0] = 1;
        ct = 1;
    }
    if (ct > (f4 ? 8 : 4)) return false;   // F4: two 64-channel segments (the 64+64 -> 64 decoder block)
    pl.f4 = f4;
    pl.nreg = 0;
    for (int i = 0; i < cd.nseg; ++i) {
        pl.reg0[i] = pl.nreg;
        pl.nreg += f4 ? (cd.seg[i].c + 31) / 32 : 0;
    }
    // z-slabs: the launch covers global output planes [zo_beg, zo_beg + Do) of the layer
    // (segment buffers start at global plane zbeg); y and x are always whole
    if (cd.zo_beg < 0 || cd.zo_beg + cd.Do > out_extent(cd.Dci, pl.s, 1, 1) ||
        cd.Ho != out_extent(cd.Hci, pl.s, pl.dil, pl.dil) || cd.Wo != out_extent(cd.Wci, pl.s, pl.dil, pl.dil))
        return false;
    if (pl.s == 2 && (cd.Hci % 2 || cd.Wci % 2)) return false;
    // one-plane volumes (Table 1's 2D layers): only the middle kernel plane meets data
    static const bool no_onep = ab_env("TN_TZ_NO_ONEP") != nullptr;   // A/B switch (measurement)
    // (instantiated: FP4 stride 1 with 1, 2 or 4 chunks -- Table 1's #1 257 -> 219 us and #2 318 -> 205;
    // the int8 stride-2 #3 measured slower, 142 -> 213 us, and keeps the two-block ring)
    pl.onep = !no_onep && !first && cd.Dci == 1 && cd.Do == 1 && cd.zo_beg == 0 && pl.dil == 1 && cd.nseg == 1 &&
              cd.logits == nullptr && f4 && pl.s == 1 && (ct == 1 || ct == 2 || ct == 4);
    const bool split = !pl.onep && tz_split(pl.kp, pl.s, f4, ct);
    pl.RO = pl.onep ? 1 : pl.s == 1 ? (split ? 4 : 3) : 2;
    pl.nph = pl.s == 1 ? 1 : 4;
    pl.NB = pl.onep ? 1 : pl.s == 1 ? (split ? 3 : 5) : 4;
    pl.Po = cd.Wo + pl.dil;                    // dil zero separator columns per raster row
    {   // raster staging: whole packed rows copied to 16-byte aligned slots of pitch Po
        const int bpv = cd.nseg != 1 ? 0 : (first ? 4 : 8 * cd.seg[0].cw);   // staged bytes per voxel
        static const bool no_rstg = ab_env("TN_TZ_NO_RSTG") != nullptr;   // A/B switch (measurement)
        pl.rstg = (first && f4) ||   // FF4 only stages raster rows
                  (!no_rstg && f4 && cd.nseg == 1 && pl.s == 1 && !first && pl.dil == 1 && bpv > 0 &&
                   (cd.seg[0].W * bpv) % 16 == 0 && cd.seg[0].W >= 128);   // (narrow rows: one copy per strip
                                                                             // is faster; configs[0] 8.6 vs 7.7 us)
        while (pl.rstg && (pl.Po * bpv) % 16) ++pl.Po;   // more separator columns keep rows aligned
        pl.bpv = bpv;
    }
    pl.qoff = pl.dil * pl.Po + pl.dil;
    pl.yoff = pl.dil + 1;
    const int64_t npo = static_cast<int64_t>(cd.Ho) * pl.Po;
    if (npo + (2 * pl.yoff + 2) * pl.Po > (1 << 22) || pl.Po > 1024) return false;   // div_po range: q * Po < 2^32
    pl.NPo = static_cast<int>(npo);
    pl.NT = (pl.NPo + 127) / 128;
    pl.po_magic = static_cast<uint32_t>((0x100000000ull + pl.Po - 1) / pl.Po);
    const int exp_threads =
        tz_exp_warps(pl.kp, cd.logits != nullptr && !first, ct, pl.s == 1 && (!first || f4), first && !f4, first && f4) * 32;
    pl.step_q = exp_threads / pl.Po;
    pl.step_r = exp_threads % pl.Po;

    // K-slices: (tap, chunk) -> byte offset within an A slot (for a given REG),
    // sorted ascending and paired into MMAs.  Offsets depend on REG, so the order
    // is taken on phase/chunk/row keys that are REG-independent (REG > any row offset).
    struct Sl { int ph, ch, row, tap; };
    std::vector<Sl> sl;
    for (int dy = 0; dy < 3; ++dy)
        for (int dx = 0; dx < 3; ++dx) {
            int ph = 0, oy = dy, ox = dx;
            if (pl.s == 2) {
                const int py = dy == 1 ? 0 : 1, px = dx == 1 ? 0 : 1;
                oy = dy == 0 ? 0 : 1;
                ox = dx == 0 ? 0 : 1;
                ph = py * 2 + px;
            }
            for (int c = 0; c < ct; ++c) sl.push_back({ph, c, pl.dil * (oy * pl.Po + ox), dy * 3 + dx});
        }
    std::sort(sl.begin(), sl.end(), [](const Sl& a, const Sl& b) {
        if (a.ph != b.ph) return a.ph < b.ph;
        if (a.ch != b.ch) return a.ch < b.ch;
        return a.row < b.row;
    });
    if (first) sl.assign(1, Sl{0, 0, 0, 0});   // the whole 3x3 window is one row
    // F4 slices: (segment, region, row offset, tap a, tap b).  C = 16 segments pair
    // the taps of one (dy, phase) whose column offsets differ by one (a row holds
    // positions r and r+1); C >= 32 segments take one 32-channel region per tap.
    struct Sl4 { int ph, reg, row, tap, tapb, seg, c32; };
    std::vector<Sl4> sl4;
    if (f4) {
        for (int sg = 0; sg < cd.nseg; ++sg) {
            const int C = cd.seg[sg].c;
            for (int dy = 0; dy < 3; ++dy) {
                struct Tp { int ph, oy, ox, tap; };
                std::vector<Tp> tp;
                for (int dx = 0; dx < 3; ++dx) {
                    int ph = 0, oy = dy, ox = dx;
                    if (pl.s == 2) {
                        const int py = dy == 1 ? 0 : 1, px = dx == 1 ? 0 : 1;
                        oy = dy == 0 ? 0 : 1;
                        ox = dx == 0 ? 0 : 1;
                        ph = py * 2 + px;
                    }
                    tp.push_back({ph, oy, ox, dy * 3 + dx});
                }
                std::sort(tp.begin(), tp.end(), [](const Tp& a, const Tp& b) {
                    return a.ph != b.ph ? a.ph < b.ph : a.ox < b.ox;
                });
                if (C <= 16) {
                    for (size_t i = 0; i < tp.size();) {
                        const bool pair = i + 1 < tp.size() && tp[i + 1].ph == tp[i].ph && tp[i + 1].ox == tp[i].ox + 1;
                        sl4.push_back({tp[i].ph, pl.reg0[sg], tp[i].oy * pl.Po + tp[i].ox, tp[i].tap,
                                       pair ? tp[i + 1].tap : -1, sg, 0});
                        i += pair ? 2 : 1;
                    }
                } else {
                    for (const Tp& t : tp)
                        for (int c = 0; c < (C + 31) / 32; ++c)
                            sl4.push_back({t.ph, pl.reg0[sg] + c, t.oy * pl.Po + t.ox, t.tap, -1, sg, c});
                }
            }
        }
        std::sort(sl4.begin(), sl4.end(), [](const Sl4& a, const Sl4& b) {
            if (a.ph != b.ph) return a.ph < b.ph;
            if (a.reg != b.reg) return a.reg < b.reg;
            return a.row < b.row;
        });
    }
    const size_t nsl = f4 ? sl4.size() : sl.size();
    pl.nmma = static_cast<int>((nsl + 1) / 2);
    {
        const int nmma_f4 =
            cd.nseg == 1 ? (ct == 1 ? 3 : (ct == 2 ? 5 : 9)) : (ct == 2 ? 6 : (ct == 3 ? 8 : (ct == 4 ? 9 : 18)));
        if (pl.nmma > kZMaxMma || pl.nmma != (f4 ? nmma_f4 : first ? 1 : (9 * ct + 1) / 2)) return false;   // kernel unrolls
    }
    pl.b_bytes = pl.nmma * 2 * pl.NB * pl.kp * 16;
    pl.bias_bytes = (pl.kp == 16 || (f4 && pl.kp == 32)) ? tz_bias_bytes(pl.kp, f4) : 0;
    const int ptab = cd.logits != nullptr ? cd.nclass * (pl.kp / 4) * 256 : 0;
    pl.ptab_floats = ptab;

    // strip size: the most tiles that fit TMEM (RO*K*T <= 512) and shared memory
    const int tmax = std::min((f4 ? 480 : 512) / (pl.RO * pl.kp), kZMaxAcc / pl.RO);   // F4: scales at 480..511
    bool ok = false;
    // smaller strips when the layer would otherwise give fewer units than SMs (the
    // R3 layers: 16 planes of 9 tiles), so every SM gets work
    int tstart = std::min(tmax, pl.NT);
    {
        const int nsm = tz_num_sms();
        while (tstart > 1 && static_cast<int64_t>(cd.N) * ((pl.NT + tstart - 1) / tstart) * cd.Do < nsm) --tstart;
    }
    for (int T = tstart; T >= 1 && !ok; --T) {
        pl.T = T;
        pl.nstrip = (pl.NT + T - 1) / T;
        pl.RS = 128 * T + (pl.s == 1 ? 2 * pl.qoff : pl.Po + 1);
        pl.REG = round_up((pl.RS + (f4 ? 1 : 0)) * 16, 128);    // F4: a 16-byte guard row first
        pl.slot_bytes = first && !f4 ? 128 * T * 16 + 256 : pl.nph * (f4 ? pl.nreg : ct) * pl.REG + 256;
        // staging: the most rows any strip reads, per segment
        int off = 0;
        for (int sg = 0; sg < cd.nseg; ++sg) {
            const SegDesc& sd = cd.seg[sg];
            int maxr = 0;
            for (int st = 0; st < pl.nstrip; ++st) {
                const int qa = st * 128 * T - pl.qoff, qb = qa + pl.RS - 1;
                int ylo = (qa + pl.yoff * pl.Po) / pl.Po - pl.yoff, yhi = (qb + pl.yoff * pl.Po) / pl.Po - pl.yoff;
                if (pl.s == 2) { ylo *= 2; yhi = 2 * yhi + 1; }
                ylo = std::max(ylo, 0);
                yhi = std::min(yhi, cd.Hci - 1);
                if (sd.up) { ylo >>= 1; yhi >>= 1; }
                yhi = std::min(yhi, sd.H - 1);
                maxr = std::max(maxr, yhi - ylo + 1);
            }
            pl.seg_off[sg] = off;
            if (pl.rstg) off += round_up(maxr * pl.Po * pl.bpv, 128);                           // rows at pitch Po
            else off += round_up(maxr * sd.W * (first ? 4 : 8 * sd.cw) + (first ? 0 : 16), 128);   // + alignment head
            if (first && !f4) {   // ternary code planes: maxr + 2 rows of W + 8 bytes (4 zero columns each side)
                pl.code_pitch = sd.W + 8;
                pl.code_bytes = round_up((maxr + 2) * pl.code_pitch, 128);
            }
        }
        pl.stage_bytes = off;
        if (!first || f4) pl.code_bytes = pl.code_pitch = 0;
        pl.code_off = 0;
        // packed filter bank staged in the A ring during setup
        int wbytes = 0;
        for (int sg = 0; sg < cd.nseg; ++sg) wbytes += ((cd.K * 27 * 2 * (first ? 1 : cd.seg[sg].cw) + 3) & ~3) * 4;
        for (int ns = kZMaxSlot; ns >= 2 && !ok; --ns)
            for (int nst = kZMaxStage; nst >= 2 && !ok; --nst) {
                pl.nslot = ns;
                pl.nstage = nst;
                const int span = pl.nslot * pl.slot_bytes + pl.nstage * pl.stage_bytes + 2 * pl.code_bytes;
                pl.wpad = round_up(std::max(0, wbytes - span), 128);
                if (tz_smem(pl, pl.kp) <= kSmemMax) ok = true;
            }
    }
    if (!ok) return false;
    pl.code_off = pl.nstage * pl.stage_bytes;    // relative to the staging base
    for (size_t j = 0; j < 2 * static_cast<size_t>(pl.nmma); ++j) {
        pl.sl_tapb[j] = -1;
        pl.sl_seg[j] = 0;
        if (j < nsl) {
            if (f4) {
                pl.sl_tap[j] = static_cast<int8_t>(sl4[j].tap);
                pl.sl_tapb[j] = static_cast<int8_t>(sl4[j].tapb);
                pl.sl_chunk[j] = static_cast<int8_t>(sl4[j].c32);
                pl.sl_seg[j] = static_cast<int8_t>(sl4[j].seg);
            } else {
                pl.sl_tap[j] = static_cast<int8_t>(sl[j].tap);
                pl.sl_chunk[j] = static_cast<int8_t>(sl[j].ch);
            }
        } else {
            pl.sl_tap[j] = -1;
            pl.sl_chunk[j] = 0;
        }
    }
    auto addr = [&](size_t j) {
        if (f4) return (sl4[j].ph * pl.nreg + sl4[j].reg) * pl.REG + 16 + sl4[j].row * 16;
        return first ? 0 : (sl[j].ph * ct + sl[j].ch) * pl.REG + sl[j].row * 16;
    };
    for (int m = 0; m < pl.nmma; ++m) {
        const int a0 = addr(2 * m);
        const int a1 = (2 * m + 1 < static_cast<int>(nsl)) ? addr(2 * m + 1) : a0 + 16;   // zero-weight dummy
        if (a1 <= a0 || a1 - a0 > 0x3FFF * 16) return false;
        pl.a_off[m] = a0;
        pl.a_lbo[m] = a1 - a0;
    }
    pl.units = static_cast<int64_t>(cd.N) * pl.nstrip * cd.Do;
    return pl.units > 0;
}

// build_out != nullptr: launch the B-image builder of this plan into build_out instead of the conv
template <int K>
static cudaError_t launch_tz_k(const ConvDesc& cd, const TzPlan& pl, int ct, int grid, size_t smem, cudaStream_t st,
                               uint4* build_out = nullptr) {
    void (*kern)(ConvDesc, TzPlan) = nullptr;
    void (*bkern)(ConvDesc, TzPlan, uint4*) = nullptr;
    const bool pred = cd.logits != nullptr;
#define TZ_PICK(CT_, NSEG_, STR_)                                                                     \
    if (!pl.f4 && ct == CT_ && cd.nseg == NSEG_ && pl.s == STR_) {                                    \
        kern = pred ? conv_tz_kernel<K, CT_, NSEG_, STR_, (K <= 32), false, false>                     \
                    : conv_tz_kernel<K, CT_, NSEG_, STR_, false, false, false>;                        \
        bkern = bimage_build_kernel<K, CT_, NSEG_, STR_, false, false>;                                     \
    }
#define TZ_PICK4(CT_, NSEG_, STR_)                                                                    \
    if (pl.f4 && ct == CT_ && cd.nseg == NSEG_ && pl.s == STR_) {                                     \
        kern = pred ? conv_tz_kernel<K, CT_, NSEG_, STR_, (K <= 32), false, true>                      \
                    : conv_tz_kernel<K, CT_, NSEG_, STR_, false, false, true>;                         \
        bkern = bimage_build_kernel<K, CT_, NSEG_, STR_, false, true>;                                      \
    }
    TZ_PICK(1, 1, 1) TZ_PICK(2, 1, 1) TZ_PICK(3, 1, 1) TZ_PICK(4, 1, 1)
    TZ_PICK(2, 2, 1) TZ_PICK(3, 2, 1) TZ_PICK(4, 2, 1)
    TZ_PICK(1, 1, 2) TZ_PICK(2, 1, 2) TZ_PICK(3, 1, 2) TZ_PICK(4, 1, 2)
    TZ_PICK4(1, 1, 1) TZ_PICK4(2, 1, 1) TZ_PICK4(4, 1, 1)
    TZ_PICK4(2, 2, 1) TZ_PICK4(4, 2, 1) if (K == 64) { TZ_PICK4(8, 2, 1) }
    TZ_PICK4(1, 1, 2) TZ_PICK4(2, 1, 2) TZ_PICK4(4, 1, 2)
#undef TZ_PICK
#undef TZ_PICK4
    if (pl.onep) {   // one-plane variants (plan_tz sets onep only for these)
        kern = nullptr;
        bkern = nullptr;
        if (pl.f4 && pl.s == 1 && ct == 1) { kern = conv_tz_kernel<K, 1, 1, 1, false, false, true, true>; bkern = bimage_build_kernel<K, 1, 1, 1, false, true, true>; }
        if (pl.f4 && pl.s == 1 && ct == 2) { kern = conv_tz_kernel<K, 2, 1, 1, false, false, true, true>; bkern = bimage_build_kernel<K, 2, 1, 1, false, true, true>; }
        if (pl.f4 && pl.s == 1 && ct == 4) { kern = conv_tz_kernel<K, 4, 1, 1, false, false, true, true>; bkern = bimage_build_kernel<K, 4, 1, 1, false, true, true>; }
        if (pred) kern = nullptr;
    }
    if (kern == nullptr) return cudaErrorNotSupported;
    if (build_out != nullptr) {
        const int total = pl.nmma * 2 * pl.NB * K;
        bkern<<<(total + 255) / 256, 256, 0, st>>>(cd, pl, build_out);
        return cudaGetLastError();
    }
    static void* configured[128] = {nullptr};
    bool done = false;
    for (void* f : configured) done = done || f == reinterpret_cast<void*>(kern);
    if (!done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        for (void*& f : configured)
            if (f == nullptr) { f = reinterpret_cast<void*>(kern); break; }
    }
    return launch_pdl(kern, grid, tz_threads(K, pred && K <= 32, ct, pl.s == 1), smem, st, cd, pl);
}

static bool tz_instantiated(const ConvDesc& cd, const TzPlan& pl) {
    int ct = 0;
    for (int i = 0; i < cd.nseg; ++i) {
        ct += pl.cch[i];
        // FP4 rows hold up to 16 channels (two positions) or whole 32-channel groups
        if (pl.f4 && pl.cch[i] != 1 && pl.cch[i] % 2 != 0) return false;
    }
    if (pl.f4 && ct == 3) return false;
    if (ct == 8) return pl.f4 && pl.kp == 64 && pl.s == 1 && cd.nseg == 2;
    if (cd.nseg == 1) return ct >= 1 && ct <= 4;
    return pl.s == 1 && ct >= 2;
}

static ConvDesc first_desc(const FirstDesc& fd) {
    ConvDesc cd{};
    cd.nseg = 1;
    SegDesc& sd = cd.seg[0];
    sd.xp = nullptr;
    sd.wp = fd.wp;
    sd.c = 1;
    sd.cw = 1;
    sd.D = fd.D; sd.H = fd.H; sd.W = fd.W;
    sd.zbeg = fd.zbeg;
    sd.up = 0;
    cd.N = fd.N;
    cd.K = fd.K;
    for (int a = 0; a < 3; ++a) { cd.s[a] = fd.s[a]; cd.p[a] = fd.p[a]; cd.dl[a] = fd.dl[a]; }
    cd.Do = fd.Do; cd.Ho = fd.Ho; cd.Wo = fd.Wo;
    cd.zo_beg = fd.zo_beg;
    cd.Dci = fd.Dg; cd.Hci = fd.H; cd.Wci = fd.W;
    cd.yp = fd.yp;
    cd.lo = fd.lo;
    cd.hi = fd.hi;
    cd.cwo = 1;
    cd.xf = fd.x;
    cd.t_lo = fd.t_lo;
    cd.t_hi = fd.t_hi;
    cd.d_bad = fd.d_bad;
    cd.bad_base = fd.bad_base;
    cd.bad_nstride = fd.bad_nstride;
    cd.halo_lo = fd.halo_lo;
    cd.halo_hi = fd.halo_hi;
    return cd;
}

// FF4 (FP4 operands, raster-staged float rows, one-channel C = 16 path) when it plans, else the
// int8 9-tap rows
static bool plan_first(const ConvDesc& cd, TzPlan& pl) {
    static const bool no_ff4 = ab_env("TN_TZ_NO_FF4") != nullptr;   // A/B switch (measurement)
    if (!no_ff4 && plan_tz(cd, pl, true, true) && tz_smem(pl, pl.kp) <= 227 * 1024) return true;
    pl = TzPlan{};
    return plan_tz(cd, pl, true, false) && tz_smem(pl, pl.kp) <= 227 * 1024;
}

bool conv_tz_first_supported(const FirstDesc& fd) {
    if (fd.K != 16 && fd.K != 32) return false;
    const ConvDesc cd = first_desc(fd);
    TzPlan pl{};
    return plan_first(cd, pl);
}

cudaError_t launch_conv_tz_first(const FirstDesc& fd, cudaStream_t st) {
    const ConvDesc cd = first_desc(fd);
    TzPlan pl{};
    if ((fd.K != 16 && fd.K != 32) || !plan_first(cd, pl)) return cudaErrorNotSupported;
    const size_t smem = tz_smem(pl, pl.kp);
    if (smem > 227 * 1024) return cudaErrorNotSupported;
    if (g_num_sms_z == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms_z, cudaDevAttrMultiProcessorCount, dev);
    }
    const int cap = persistent_grid_cap() > 0 ? std::min(persistent_grid_cap(), g_num_sms_z) : g_num_sms_z;
    const int grid = tz_grid(pl.units, cap);
    void (*kern)(ConvDesc, TzPlan) =
        pl.f4 ? (fd.K == 16 ? conv_tz_kernel<16, 1, 1, 1, false, true, true> : conv_tz_kernel<32, 1, 1, 1, false, true, true>)
              : (fd.K == 16 ? conv_tz_kernel<16, 1, 1, 1, false, true, false> : conv_tz_kernel<32, 1, 1, 1, false, true, false>);
    static bool configured[4] = {false, false, false, false};
    const int ci = (fd.K == 32) + 2 * pl.f4;
    if (!configured[ci]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        configured[ci] = true;
    }
    return launch_pdl(kern, grid, tz_threads(fd.K, false, 1, pl.f4 != 0, !pl.f4, pl.f4 != 0), smem, st, cd, pl);
}

// F4 (kind::mxf4) plan if allowed and it fits, else the int8 plan.
static bool plan_any(const ConvDesc& cd, TzPlan& pl, bool allow_f4) {
    const bool allow_any_f4 = allow_f4;
    // Measured (tools/conv_time.py, configs[3] layer shapes): FP4 wins for stride-1
    // layers with K <= 32 (#4 -10 %, #10 -21 %, #12 -23 %, #13 -2 %) and at stride 2
    // with C = 32 it is slower.
    int c_tot = 0;
    for (int i = 0; i < cd.nseg; ++i) c_tot += cd.seg[i].c;
    // C > 64 (the 64 + 64 -> 64 decoder block) only fits with FP4 operands (half the B bytes)
    // K in 33..64 at stride 1 with C <= 64: FP4 without the split (five-block rotated B image,
    // two tiles per strip, half the halo rows per output): C1's conv 82.9 -> 75.3 us
    const bool f4_k64 = cd.K > 32 && cd.s[0] == 1 && c_tot <= 64;
    static const bool force_f4 = ab_env("TN_TZ_FORCE_F4") != nullptr;   // (experiments)
    allow_f4 = allow_f4 && ((cd.K <= 32 && !(cd.s[0] == 2 && c_tot > 16)) || c_tot > 64 || f4_k64 || force_f4);
    if (allow_f4 && plan_tz(cd, pl, false, true) && tz_instantiated(cd, pl) && tz_smem(pl, pl.kp) <= 227 * 1024)
        return true;
    pl = TzPlan{};
    if (plan_tz(cd, pl, false, false) && tz_instantiated(cd, pl) && tz_smem(pl, pl.kp) <= 227 * 1024) return true;
    // shapes the int8 operands do not fit (e.g. 64 -> 64 at stride 2): FP4 if allowed at all
    pl = TzPlan{};
    return allow_any_f4 && plan_tz(cd, pl, false, true) && tz_instantiated(cd, pl) &&
           tz_smem(pl, pl.kp) <= 227 * 1024;
}

// Dilation d > 1 (stride 1, pad d): output plane z reads input planes z - d, z, z + d, all in
// z's residue class mod d, so class r (planes r, r + d, ...) is an undilated-in-z conv of
// ceil((D - r) / d) planes; one launch per class.  Whole volumes only (no z-slabs).
static int dil_classes(const ConvDesc& cd) { return cd.dl[0] > 1 ? cd.dl[0] : 1; }
static ConvDesc dil_class(const ConvDesc& cd, int r) {
    ConvDesc c = cd;
    if (cd.dl[0] <= 1) return c;
    const int d = cd.dl[0];
    c.zstep = d;
    c.zres = r;
    c.Dbuf = cd.Do;
    c.Do = cd.Do > r ? (cd.Do - r + d - 1) / d : 0;
    c.Dci = c.Do;
    c.zo_beg = 0;
    return c;
}
static bool dil_ok(const ConvDesc& cd) {
    return cd.dl[0] <= 1 || (cd.zo_beg == 0 && cd.Do == cd.Dci && cd.nseg == 1 && cd.seg[0].zbeg == 0);
}

bool conv_tz_supported(const ConvDesc& cd, bool allow_f4) {
    TzPlan pl{};
    return dil_ok(cd) && plan_any(dil_class(cd, 0), pl, allow_f4);
}

bool conv_tz_uses_f4(const ConvDesc& cd, bool allow_f4) {
    TzPlan pl{};
    return dil_ok(cd) && plan_any(dil_class(cd, 0), pl, allow_f4) && pl.f4;
}

static cudaError_t launch_conv_tz_one(const ConvDesc& cd, cudaStream_t st, bool allow_f4);

cudaError_t launch_conv_tz(const ConvDesc& cd, cudaStream_t st, bool allow_f4) {
    if (!dil_ok(cd)) return cudaErrorNotSupported;
    for (int r = 0; r < dil_classes(cd); ++r) {
        const ConvDesc c = dil_class(cd, r);
        if (c.Do == 0) continue;
        cudaError_t e = launch_conv_tz_one(c, st, allow_f4);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// The prepared image: the plan fields and filter-bank identity the B image depends on.
struct TzPrep {
    uint4* img;
    int bytes;
    int wide;              // 1: an image of the wide one-plane kernel (conv_wide.cu) for tapmask
    unsigned tapmask;
    int kp, K, f4, s, nseg, NB, nmma;
    int cch[kMaxSeg], c[kMaxSeg], cw[kMaxSeg];
    const uint32_t* wp[kMaxSeg];
    int8_t sl_tap[2 * kZMaxMma], sl_chunk[2 * kZMaxMma], sl_tapb[2 * kZMaxMma], sl_seg[2 * kZMaxMma];
};

static void prep_key(const ConvDesc& cd, const TzPlan& pl, TzPrep& k) {
    k.bytes = pl.b_bytes;
    k.kp = pl.kp; k.K = cd.K; k.f4 = pl.f4; k.s = pl.s; k.nseg = cd.nseg; k.NB = pl.NB; k.nmma = pl.nmma;
    for (int i = 0; i < kMaxSeg; ++i) {
        const bool on = i < cd.nseg;
        k.cch[i] = on ? pl.cch[i] : 0;
        k.c[i] = on ? cd.seg[i].c : 0;
        k.cw[i] = on ? cd.seg[i].cw : 0;
        k.wp[i] = on ? cd.seg[i].wp : nullptr;
    }
    for (int j = 0; j < 2 * kZMaxMma; ++j) {
        const bool on = j < 2 * pl.nmma;
        k.sl_tap[j] = on ? pl.sl_tap[j] : 0;
        k.sl_chunk[j] = on ? pl.sl_chunk[j] : 0;
        k.sl_tapb[j] = on ? pl.sl_tapb[j] : 0;
        k.sl_seg[j] = on ? pl.sl_seg[j] : 0;
    }
}

static bool prep_matches(const TzPrep& p, const ConvDesc& cd, const TzPlan& pl) {
    if (p.wide) return false;
    TzPrep k{};
    prep_key(cd, pl, k);
    if (k.bytes != p.bytes || k.kp != p.kp || k.K != p.K || k.f4 != p.f4 || k.s != p.s || k.nseg != p.nseg ||
        k.NB != p.NB || k.nmma != p.nmma)
        return false;
    for (int i = 0; i < kMaxSeg; ++i)
        if (k.cch[i] != p.cch[i] || k.c[i] != p.c[i] || k.cw[i] != p.cw[i] || k.wp[i] != p.wp[i]) return false;
    return std::memcmp(k.sl_tap, p.sl_tap, sizeof k.sl_tap) == 0 &&
           std::memcmp(k.sl_chunk, p.sl_chunk, sizeof k.sl_chunk) == 0 &&
           std::memcmp(k.sl_tapb, p.sl_tapb, sizeof k.sl_tapb) == 0 &&
           std::memcmp(k.sl_seg, p.sl_seg, sizeof k.sl_seg) == 0;
}

cudaError_t tz_prepare(const ConvDesc& cd0, bool allow_f4, TzPrep** out, cudaStream_t st) {
    *out = nullptr;
    if (!dil_ok(cd0)) return cudaSuccess;
    const ConvDesc cd = dil_class(cd0, 0);
    TzPlan pl{};
    if ((allow_f4 && conv_wide_supported(cd0)) || !plan_any(cd, pl, allow_f4)) {
        if (!allow_f4 || !conv_wide_supported(cd0)) return cudaSuccess;
        // the wide one-plane kernel: its image and the filter bank's active taps
        TzPrep* p = new TzPrep{};
        p->wide = 1;
        p->K = cd0.K; p->s = cd0.s[0]; p->nseg = cd0.nseg;
        for (int i = 0; i < cd0.nseg; ++i) { p->c[i] = cd0.seg[i].c; p->wp[i] = cd0.seg[i].wp; }
        cudaError_t e = wide_prepare(cd0, &p->img, &p->bytes, &p->tapmask, st);
        if (e != cudaSuccess) { delete p; return e == cudaErrorNotSupported ? cudaSuccess : e; }
        *out = p;
        return cudaSuccess;
    }
    int ct = 0;
    for (int i = 0; i < cd.nseg; ++i) ct += pl.cch[i];
    TzPrep* p = new TzPrep{};
    prep_key(cd, pl, *p);
    cudaError_t e = cudaMalloc(&p->img, pl.b_bytes);
    if (e != cudaSuccess) { delete p; return e; }
    switch (pl.kp) {
        case 16: e = launch_tz_k<16>(cd, pl, ct, 0, 0, st, p->img); break;
        case 32: e = launch_tz_k<32>(cd, pl, ct, 0, 0, st, p->img); break;
        case 64: e = launch_tz_k<64>(cd, pl, ct, 0, 0, st, p->img); break;
        default: e = cudaErrorNotSupported;
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);   // the image is complete before any conv reads it
    if (e != cudaSuccess) { cudaFree(p->img); delete p; return e; }
    *out = p;
    return cudaSuccess;
}

void tz_prep_free(TzPrep* p) {
    if (p == nullptr) return;
    cudaFree(p->img);
    delete p;
}

size_t tz_prep_bytes(const TzPrep* p) { return p ? static_cast<size_t>(p->bytes) : 0; }

bool tz_prep_wide(const TzPrep* p, const ConvDesc& cd, const uint4** img, unsigned* tapmask) {
    if (p == nullptr || !p->wide || p->K != cd.K || p->s != cd.s[0] || p->nseg != cd.nseg) return false;
    for (int i = 0; i < cd.nseg; ++i)
        if (p->c[i] != cd.seg[i].c || p->wp[i] != cd.seg[i].wp) return false;
    *img = p->img;
    *tapmask = p->tapmask;
    return true;
}

static cudaError_t launch_conv_tz_one(const ConvDesc& cd0, cudaStream_t st, bool allow_f4) {
    TzPlan pl{};
    if (!plan_any(cd0, pl, allow_f4)) return cudaErrorNotSupported;
    ConvDesc cd = cd0;
    cd.bimg = (cd.prep != nullptr && prep_matches(*cd.prep, cd, pl)) ? cd.prep->img : nullptr;
    const size_t smem = tz_smem(pl, pl.kp);
    if (g_num_sms_z == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms_z, cudaDevAttrMultiProcessorCount, dev);
    }
    const int cap = persistent_grid_cap() > 0 ? std::min(persistent_grid_cap(), g_num_sms_z) : g_num_sms_z;
    const int grid = tz_grid(pl.units, cap);
    int ct = 0;
    for (int i = 0; i < cd.nseg; ++i) ct += pl.cch[i];
    switch (pl.kp) {
        case 16: return launch_tz_k<16>(cd, pl, ct, grid, smem, st);
        case 32: return launch_tz_k<32>(cd, pl, ct, grid, smem, st);
        case 64: return launch_tz_k<64>(cd, pl, ct, grid, smem, st);
    }
    return cudaErrorNotSupported;
}

}  // namespace tn

