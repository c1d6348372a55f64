// tn_internal.cuh -- internal kernel parameter blocks and helpers for libtn.so.
// Not part of the ABI (include/tn.h is).  sm_100a only.
#pragma once

#include <cstdint>
#include <cstddef>
#include <cuda_runtime.h>
#include <cstdio>
#include <nvtx3/nvToolsExt.h>

#include "../../include/tn.h"

namespace tn {

constexpr int kMaxSeg = 2;

// One input segment of a (possibly concatenated) convolution, in the
// coordinates of the segment's own buffer.  "Source resolution" is the
// resolution the buffer is stored at (low resolution if up == 1).
struct SegDesc {
    const uint32_t* xp;   // packed [n][D][H][W][2][cw]
    const uint32_t* wp;   // packed weights [K][27][2][cw]
    int c;                // logical channels of this segment
    int cw;               // words per bitplane per voxel
    int D, H, W;          // buffer extents (source resolution)
    int zbeg;             // global source-resolution z of buffer plane 0 (slabs)
    int up;               // nearest x2 upsampling of this segment
};

// A ternary conv launch: output buffer [N][Do][Ho][Wo] covering global output
// planes [zo_beg, zo_beg + Do).  Conv-input ("ci") coordinates are at the
// resolution after upsampling; the global ci extents Dci/Hci/Wci define the
// zero padding.
struct TzPrep;   // conv_tz.cu: a prepared B image

struct ConvDesc {
    SegDesc seg[kMaxSeg];
    int nseg;
    int N, K;
    int s[3], p[3], dl[3];        // z, y, x
    int Do, Ho, Wo;
    int zo_beg;
    int Dci, Hci, Wci;            // global conv-input extents (z, y, x)
    // outputs: exactly one of y / yp
    int32_t* y;                   // int32 channel-last [N][Do][Ho][Wo][K]
    uint32_t* yp;                 // packed [N][Do][Ho][Wo][2][cwo]
    const int32_t* lo;
    const int32_t* hi;
    int cwo;
    // Optional A8 fused into the requant epilogue (tensor-core kernel, K <= 32):
    // logits[(n*nclass + j)*lstride + (z*Ho + y)*Wo + x] = pb[j] + sum_k pw[j][k]*t_k
    // (fp32, k ascending); the packed output yp is written as well.
    float* logits;
    int64_t lstride;
    const float* pw;
    const float* pb;
    int nclass;
    int no_yp;                    // with fused logits: skip the packed output (only the logits are used)
    // First layer (A7) on the tensor-core TZ kernel: seg[0] describes the float
    // input (c = 1, xp unused); Eq. 6 band (t_lo, t_hi); non-finite inputs are
    // reported through d_bad (flat index n * bad_nstride + bad_base + (zb*H+y)*W+x).
    const float* xf;
    float t_lo, t_hi;
    int64_t* d_bad;
    int64_t bad_base, bad_nstride;
    // NEXT-1 (z-slabs, N = 1): when set, the requant epilogue also stores output plane 0
    // into halo_lo and plane Do-1 into halo_hi ([Ho][Wo][2][cwo] each) -- the neighbouring
    // slabs' halo planes, in peer memory over NVLink (or another slab's buffer on one device).
    uint32_t* halo_lo;
    uint32_t* halo_hi;
    // Dilation (tensor-core kernel, stride 1, pad = dilation): a launch covers one residue class
    // of planes z = zres + j * zstep; Do / Dci / zo_beg then count class planes and Dbuf is the
    // output buffer's depth.  zstep == 0 means 1 (no classes), Dbuf == 0 means Do.
    int zstep, zres, Dbuf;
    // Prepared filter bank (tensor-core kernel): the B image built once by tz_prepare; used by a
    // launch whose plan matches the one it was built for (else the bank is staged as usual).
    // bimg is set by the launcher from prep, never by callers.
    const TzPrep* prep;
    const uint4* bimg;
};

struct FirstDesc {
    const float* x;               // [N][1][D][H][W] (buffer), global z of plane 0 = zbeg
    int D, H, W, zbeg, Dg;        // Dg: global extent in z for padding
    float t_lo, t_hi;
    const uint32_t* wp;           // [K][27][2][1]
    int N, K;
    int s[3], p[3], dl[3];
    int Do, Ho, Wo, zo_beg;
    const int32_t* lo;
    const int32_t* hi;
    uint32_t* yp;                 // packed [N][Do][Ho][Wo][2][1]
    int64_t* d_bad;
    int64_t bad_base;             // flat index of buffer element 0 in the global tensor
    int64_t bad_nstride;          // global per-n stride (D_g*H*W)
    uint32_t* halo_lo;            // NEXT-1 boundary-plane stores (see ConvDesc)
    uint32_t* halo_hi;
};

// NEXT-1: store one voxel's packed words ([2][cwo]) to the neighbours' halo planes
// when its output plane is a slab boundary.  voff = (y * Wo + x) within the plane.
__device__ __forceinline__ void halo_store_words(uint32_t* halo_lo, uint32_t* halo_hi, int zo, int Do,
                                                 int64_t voff, const uint32_t* words, int nw) {
    if (zo == 0 && halo_lo != nullptr)
        for (int q = 0; q < nw; ++q) halo_lo[voff * nw + q] = words[q];
    if (zo == Do - 1 && halo_hi != nullptr)
        for (int q = 0; q < nw; ++q) halo_hi[voff * nw + q] = words[q];
}

// Kernel launchers (return cudaGetLastError()).
cudaError_t launch_pack_i8(const int8_t* x, tn_dims xd, uint32_t* xp, int64_t* d_bad, cudaStream_t s);
cudaError_t launch_pack_i32(const int32_t* x, tn_dims xd, uint32_t* xp, int64_t* d_bad, cudaStream_t s);
cudaError_t launch_pack_f32(const float* x, tn_dims xd, float t_lo, float t_hi, uint32_t* xp,
                            int64_t* d_bad, cudaStream_t s);
cudaError_t launch_pack_weights(const int8_t* w, int k, int c, uint32_t* wp, int64_t* d_bad,
                                cudaStream_t s);
cudaError_t launch_unpack(const uint32_t* xp, tn_dims xd, int8_t* x, int64_t* d_bad, cudaStream_t s);
cudaError_t launch_requant(const int32_t* y, tn_dims yd, const int32_t* lo, const int32_t* hi,
                           uint32_t* yp, cudaStream_t s);
// logits[(n*nclass + j)*cstride + v]; cstride < 0 means d*h*w of td.
cudaError_t launch_predict(const uint32_t* tp, tn_dims td, const float* w, const float* b,
                           int nclass, float* logits, cudaStream_t s, int64_t cstride = -1);
cudaError_t launch_bad_init(int64_t* d_bad, cudaStream_t s);

cudaError_t launch_conv_popc(const ConvDesc& cd, cudaStream_t s);
cudaError_t launch_conv_first(const FirstDesc& fd, cudaStream_t s);

// tcgen05 tap-offset, z-merged implicit GEMM (conv_tz.cu): C, K <= 64 with a
// small filter bank; returns cudaErrorNotSupported if the shape is outside what
// the kernel handles (the caller then uses the popc kernel).
// allow_f4: may use FP4 E2M1 operands (kind::mxf4; exact, twice the int8 rate).
bool        conv_tz_supported(const ConvDesc& cd, bool allow_f4 = true);
bool        conv_tz_uses_f4(const ConvDesc& cd, bool allow_f4 = true);
// A7 on the TZ kernel (stride 1, pad 1, K in {16, 32}, W % 4 == 0); false if the
// shape is outside it (the caller then uses conv_first_kernel).
bool        conv_tz_first_supported(const FirstDesc& fd);
cudaError_t launch_conv_tz_first(const FirstDesc& fd, cudaStream_t s);
// tn_set_grid_cap: upper bound on the persistent tensor-core grids (0 = #SMs).
int         persistent_grid_cap();
// Measurement A/B switches (TN_TZ_NO_*, TN_WIDE_NBUF): the environment value only in the A/B
// build (`build.py --ab`, libtn_ab.so, -DTN_AB); the product library ignores the environment.
const char* ab_env(const char* name);
// The first layer may use the TZ kernel under the current selector (AUTO or TZ).
bool        first_kernel_tz_allowed();
cudaError_t launch_conv_tz(const ConvDesc& cd, cudaStream_t s, bool allow_f4 = true);
// Build the B image of cd's filter bank for the plan a launch of cd would use (one small kernel on
// s, then a synchronize of s).  *out = nullptr (and cudaSuccess) when cd is not a tensor-core
// shape.  The image is a copy: it belongs to the bank's contents at prepare time.
cudaError_t tz_prepare(const ConvDesc& cd, bool allow_f4, TzPrep** out, cudaStream_t s);
void        tz_prep_free(TzPrep* p);
// The wide one-plane layers (conv_wide.cu): C or K beyond 64 (C % 64 == 0 per segment, K <= 256),
// D = 1, stride 1 / 2 with pad 1, FP4 operands.  img / tapmask from a prepared image (tz_prepare
// makes one when the tap-offset kernel does not take the layer), or nullptr: built per call.
bool        conv_wide_supported(const ConvDesc& cd);
cudaError_t wide_prepare(const ConvDesc& cd, uint4** img, int* bytes, unsigned* tapmask, cudaStream_t s);
cudaError_t launch_conv_wide(const ConvDesc& cd, const uint4* img, unsigned tapmask, cudaStream_t s);
// a prepared wide image matching cd (same banks, widths, K, stride)
bool        tz_prep_wide(const TzPrep* p, const ConvDesc& cd, const uint4** img, unsigned* tapmask);
// bytes of device memory the image holds (0 for nullptr)
size_t      tz_prep_bytes(const TzPrep* p);

}  // namespace tn

// The FCN object behind the opaque tn_fcn handle (fcn.cu, slab.cu).
#include <vector>
struct tn_fcn {
    std::vector<tn_layer> layers;
    std::vector<int> cin[tn::kMaxSeg];
    float t_lo, t_hi;
    const float* pred_w;
    const float* pred_b;
    int nclass;
    std::vector<tn::TzPrep*> prep;   // tn_fcn_prepare: per-layer B images (nullptr: none)
    ~tn_fcn() {
        for (tn::TzPrep* p : prep) tn::tz_prep_free(p);
    }
};

namespace tn {

// Conv dispatch (api.cu): kernel selection and launch.
tn_status run_conv(ConvDesc& cd, cudaStream_t st, const char* where);

// Host-side error text.
void set_error(const char* fmt, ...);

// NVTX range over a host scope (SURVEY.md §5 tracing): "tn <what>" or "tn <what> <i>" for
// per-layer ranges; visible to nsys / ncu --nvtx, a no-op without a tool attached.
struct NvtxRange {
    explicit NvtxRange(const char* what, int i = -1) {
        char b[96];
        if (i >= 0) std::snprintf(b, sizeof b, "tn %s %d", what, i);
        else std::snprintf(b, sizeof b, "tn %s", what);
        nvtxRangePushA(b);
    }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

inline int out_extent(int len, int s, int p, int dl) {
    int span = len + 2 * p - 2 * dl - 1;
    return span < 0 ? 0 : span / s + 1;
}

}  // namespace tn
