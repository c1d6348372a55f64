// api.cu -- the C ABI of libtn.so (include/tn.h): host-side validation, error
// text, descriptor construction and kernel selection.  No compute happens here;
// every step of the path runs in the kernels of pack.cu / conv_popc.cu /
// conv_tz.cu.
#include "tn_internal.cuh"

#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>

namespace tn {

static thread_local char g_err[512] = "";
static int g_conv_kernel = TN_KERNEL_AUTO;
static int g_grid_cap = 0;

int persistent_grid_cap() { return g_grid_cap; }
const char* ab_env(const char* name) {
#ifdef TN_AB
    return getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}
bool first_kernel_tz_allowed() {
    return g_conv_kernel == TN_KERNEL_AUTO || g_conv_kernel == TN_KERNEL_TZ || g_conv_kernel == TN_KERNEL_TZ8;
}

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

}  // namespace tn

using namespace tn;

namespace {

tn_status fail(tn_status st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    char buf[512];
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    set_error("%s", buf);
    return st;
}

tn_status cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return TN_OK;
    if (e == cudaErrorNotSupported) return fail(TN_EUNSUPPORTED, "%s: unsupported shape", where);
    if (e == cudaErrorInvalidConfiguration)
        return fail(TN_EUNSUPPORTED, "%s: shape needs more shared memory than an SM has", where);
    return fail(TN_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

tn_status check_ptr(const void* p, const char* name) {
    if (p == nullptr) return fail(TN_EINVAL, "%s is NULL", name);
    if (!aligned16(p)) return fail(TN_EALIGN, "%s is not 16-byte aligned", name);
    return TN_OK;
}

tn_status check_dims(tn_dims d, const char* name) {
    if (d.n < 0 || d.d < 0 || d.h < 0 || d.w < 0)
        return fail(TN_ESHAPE, "%s has a negative extent", name);
    if (d.c < 1) return fail(TN_EINVAL, "%s.c must be >= 1 (got %d)", name, d.c);
    return TN_OK;
}

bool empty(tn_dims d) { return d.n == 0 || d.d == 0 || d.h == 0 || d.w == 0; }

tn_status check_geom(tn_geom g) {
    for (int i = 0; i < 3; ++i) {
        if (g.stride[i] < 1) return fail(TN_EINVAL, "stride[%d] must be >= 1", i);
        if (g.pad[i] < 0) return fail(TN_EINVAL, "pad[%d] must be >= 0", i);
        if (g.dil[i] < 1) return fail(TN_EINVAL, "dil[%d] must be >= 1", i);
    }
    return TN_OK;
}

cudaStream_t cs(tn_stream s) { return reinterpret_cast<cudaStream_t>(s); }

#define TN_TRY(expr)                        \
    do {                                    \
        tn_status _st = (expr);             \
        if (_st != TN_OK) return _st;       \
    } while (0)

}  // namespace

extern "C" {

size_t tn_packed_bytes(tn_dims x) {
    if (x.n <= 0 || x.d <= 0 || x.h <= 0 || x.w <= 0 || x.c <= 0) return 0;
    return static_cast<size_t>(x.n) * x.d * x.h * x.w * 2 * ((x.c + 31) / 32) * 4;
}

size_t tn_weight_bytes(int32_t k, int32_t c) {
    if (k <= 0 || c <= 0) return 0;
    return static_cast<size_t>(k) * 27 * 2 * ((c + 31) / 32) * 4;
}

tn_status tn_conv_out_dims(tn_dims x, int32_t k, tn_geom g, tn_dims* out) {
    TN_TRY(check_dims(x, "x"));
    TN_TRY(check_geom(g));
    if (out == nullptr) return fail(TN_EINVAL, "out is NULL");
    if (k < 1) return fail(TN_EINVAL, "k must be >= 1");
    tn_dims o{x.n, k, out_extent(x.d, g.stride[0], g.pad[0], g.dil[0]),
              out_extent(x.h, g.stride[1], g.pad[1], g.dil[1]),
              out_extent(x.w, g.stride[2], g.pad[2], g.dil[2])};
    *out = o;
    if (!empty(x) && (o.d < 1 || o.h < 1 || o.w < 1))
        return fail(TN_ESHAPE, "conv output would be empty (%d x %d x %d)", o.d, o.h, o.w);
    return TN_OK;
}

const char* tn_last_error(void) { return g_err; }
const char* tn_version(void) { return "tn 0.1 (sm_100a)"; }

tn_status tn_bad_init(int64_t* d_bad, tn_stream stream) {
    if (d_bad == nullptr) return fail(TN_EINVAL, "d_bad is NULL");
    return cuda_status(launch_bad_init(d_bad, cs(stream)), "tn_bad_init");
}

tn_status tn_pack_i8(const int8_t* x, tn_dims xd, uint32_t* xp, int64_t* d_bad, tn_stream stream) {
    TN_TRY(check_dims(xd, "xd"));
    if (empty(xd)) return TN_OK;
    TN_TRY(check_ptr(x, "x"));
    TN_TRY(check_ptr(xp, "xp"));
    return cuda_status(launch_pack_i8(x, xd, xp, d_bad, cs(stream)), "tn_pack_i8");
}

tn_status tn_pack_i32(const int32_t* x, tn_dims xd, uint32_t* xp, int64_t* d_bad, tn_stream stream) {
    TN_TRY(check_dims(xd, "xd"));
    if (empty(xd)) return TN_OK;
    TN_TRY(check_ptr(x, "x"));
    TN_TRY(check_ptr(xp, "xp"));
    return cuda_status(launch_pack_i32(x, xd, xp, d_bad, cs(stream)), "tn_pack_i32");
}

tn_status tn_pack_f32(const float* x, tn_dims xd, float t_lo, float t_hi, uint32_t* xp,
                      int64_t* d_bad, tn_stream stream) {
    TN_TRY(check_dims(xd, "xd"));
    if (!(t_lo <= t_hi)) return fail(TN_EINVAL, "need t_lo <= t_hi (got %g, %g)", t_lo, t_hi);
    if (empty(xd)) return TN_OK;
    TN_TRY(check_ptr(x, "x"));
    TN_TRY(check_ptr(xp, "xp"));
    return cuda_status(launch_pack_f32(x, xd, t_lo, t_hi, xp, d_bad, cs(stream)), "tn_pack_f32");
}

tn_status tn_pack_weights(const int8_t* w, int32_t k, int32_t c, uint32_t* wp, int64_t* d_bad,
                          tn_stream stream) {
    if (k < 1 || c < 1) return fail(TN_EINVAL, "k and c must be >= 1 (got %d, %d)", k, c);
    TN_TRY(check_ptr(w, "w"));
    TN_TRY(check_ptr(wp, "wp"));
    return cuda_status(launch_pack_weights(w, k, c, wp, d_bad, cs(stream)), "tn_pack_weights");
}

tn_status tn_unpack(const uint32_t* xp, tn_dims xd, int8_t* x, int64_t* d_bad, tn_stream stream) {
    TN_TRY(check_dims(xd, "xd"));
    if (empty(xd)) return TN_OK;
    TN_TRY(check_ptr(xp, "xp"));
    TN_TRY(check_ptr(x, "x"));
    return cuda_status(launch_unpack(xp, xd, x, d_bad, cs(stream)), "tn_unpack");
}

tn_status tn_requant(const int32_t* y, tn_dims yd, const int32_t* lo, const int32_t* hi,
                     uint32_t* yp, tn_stream stream) {
    TN_TRY(check_dims(yd, "yd"));
    if (empty(yd)) return TN_OK;
    TN_TRY(check_ptr(y, "y"));
    TN_TRY(check_ptr(yp, "yp"));
    if (lo == nullptr || hi == nullptr) return fail(TN_EINVAL, "lo/hi is NULL");
    return cuda_status(launch_requant(y, yd, lo, hi, yp, cs(stream)), "tn_requant");
}

}  // extern "C"

namespace tn {

// Kernel choice for one conv launch under the process-wide selector:
// TN_KERNEL_TZ (the tcgen05 tap-offset z-merged kernel) where it covers the
// shape, else the CUDA-core popc kernel (Eq. 9 as XOR/AND/POPC: any geometry);
// a forced selector only takes its own kernel.  -1 if nothing covers the shape.
static int pick_kernel(const ConvDesc& cd, int mode) {
    // one-plane layers with 64-channel-multiple segments: the wide kernel (no z-merge, 2D strips)
    if ((mode == TN_KERNEL_AUTO || mode == TN_KERNEL_TZ) && conv_wide_supported(cd)) return TN_KERNEL_WIDE;
    if ((mode == TN_KERNEL_AUTO || mode == TN_KERNEL_TZ || mode == TN_KERNEL_TZ8) &&
        conv_tz_supported(cd, mode != TN_KERNEL_TZ8))
        return TN_KERNEL_TZ;
    // the wide one-plane layers (FP4 operands only: not under TZ8)
    if ((mode == TN_KERNEL_AUTO || mode == TN_KERNEL_TZ) && conv_wide_supported(cd)) return TN_KERNEL_WIDE;
    // TZ8 = AUTO with int8 TZ operands (falls back like AUTO)
    if ((mode == TN_KERNEL_AUTO || mode == TN_KERNEL_POPC || mode == TN_KERNEL_TZ8) && cd.logits == nullptr)
        return TN_KERNEL_POPC;
    return -1;
}

static cudaError_t launch_kernel(int kernel, const ConvDesc& cd, cudaStream_t st) {
    switch (kernel) {
        case TN_KERNEL_TZ: return launch_conv_tz(cd, st, g_conv_kernel != TN_KERNEL_TZ8);
        case TN_KERNEL_WIDE: {
            const uint4* img = nullptr;
            unsigned mask = 0x1FFu;
            if (!tz_prep_wide(cd.prep, cd, &img, &mask)) img = nullptr;
            return launch_conv_wide(cd, img, mask, st);
        }
        case TN_KERNEL_POPC: return launch_conv_popc(cd, st);
    }
    return cudaErrorNotSupported;
}

tn_status run_conv(ConvDesc& cd, cudaStream_t st, const char* where) {
    NvtxRange nv(where);
    if (cd.N == 0 || cd.Do == 0 || cd.Ho == 0 || cd.Wo == 0) return TN_OK;
    const int mode = g_conv_kernel;
    if (cd.logits != nullptr) {
        // fused prediction in the tensor-core epilogue; otherwise conv + predict kernel
        const int kf = pick_kernel(cd, mode);
        if (kf == TN_KERNEL_TZ) return cuda_status(launch_kernel(kf, cd, st), where);
        ConvDesc c2 = cd;
        c2.logits = nullptr;
        c2.no_yp = 0;   // the predict kernel reads the packed output
        tn_status s2 = run_conv(c2, st, where);
        if (s2 != TN_OK) return s2;
        const tn_dims td{cd.N, cd.K, cd.Do, cd.Ho, cd.Wo};
        return cuda_status(launch_predict(cd.yp, td, cd.pw, cd.pb, cd.nclass, cd.logits, st, cd.lstride), where);
    }
    const int kern = pick_kernel(cd, mode);
    if (kern < 0) return fail(TN_EUNSUPPORTED, "%s: the selected conv kernel (%d) does not cover this shape", where, mode);
    return cuda_status(launch_kernel(kern, cd, st), where);
}

tn_status build_conv(const tn_segment* segs, int nseg, int k, tn_geom g, const int32_t* lo,
                     const int32_t* hi, int32_t* y, uint32_t* yp, ConvDesc* out, tn_dims* od) {
    if (nseg < 1 || nseg > kMaxSeg) return fail(TN_EINVAL, "nseg must be 1 or 2 (got %d)", nseg);
    if (k < 1) return fail(TN_EINVAL, "k must be >= 1");
    TN_TRY(check_geom(g));
    if ((y == nullptr) == (yp == nullptr)) return fail(TN_EINVAL, "exactly one of y / yp must be given");
    if (yp != nullptr && (lo == nullptr || hi == nullptr)) return fail(TN_EINVAL, "requant needs lo and hi");
    ConvDesc cd{};
    cd.nseg = nseg;
    cd.K = k;
    int Dci = -1, Hci = -1, Wci = -1, N = -1;
    for (int i = 0; i < nseg; ++i) {
        const tn_segment& s = segs[i];
        TN_TRY(check_dims(s.d, "segment dims"));
        if (s.upsample < 0 || s.upsample > 2) return fail(TN_EINVAL, "upsample must be 0, 1 or 2");
        const int f = s.upsample ? 2 : 1, fz = s.upsample == 1 ? 2 : 1;   // 2: in-plane only (2D)
        if (i == 0) { Dci = s.d.d * fz; Hci = s.d.h * f; Wci = s.d.w * f; N = s.d.n; }
        if (s.d.d * fz != Dci || s.d.h * f != Hci || s.d.w * f != Wci || s.d.n != N)
            return fail(TN_ESHAPE, "segment %d extents differ from segment 0 after upsampling", i);
        SegDesc& sd = cd.seg[i];
        sd.xp = s.xp; sd.wp = s.wp;
        sd.c = s.d.c;
        sd.cw = (s.d.c + 31) / 32;
        sd.D = s.d.d; sd.H = s.d.h; sd.W = s.d.w; sd.zbeg = 0; sd.up = s.upsample;
        if (sd.cw != cd.seg[0].cw)
            return fail(TN_EUNSUPPORTED, "segments with different ceil(c/32) are not supported");
    }
    cd.N = N;
    for (int a = 0; a < 3; ++a) { cd.s[a] = g.stride[a]; cd.p[a] = g.pad[a]; cd.dl[a] = g.dil[a]; }
    cd.Dci = Dci; cd.Hci = Hci; cd.Wci = Wci;
    cd.Do = out_extent(Dci, g.stride[0], g.pad[0], g.dil[0]);
    cd.Ho = out_extent(Hci, g.stride[1], g.pad[1], g.dil[1]);
    cd.Wo = out_extent(Wci, g.stride[2], g.pad[2], g.dil[2]);
    cd.zo_beg = 0;
    const bool in_empty = N == 0 || Dci == 0 || Hci == 0 || Wci == 0;
    if (!in_empty && (cd.Do < 1 || cd.Ho < 1 || cd.Wo < 1))
        return fail(TN_ESHAPE, "conv output would be empty");
    cd.y = y; cd.yp = yp; cd.lo = lo; cd.hi = hi;
    cd.cwo = (k + 31) / 32;
    if (!in_empty) {
        for (int i = 0; i < nseg; ++i) {
            TN_TRY(check_ptr(segs[i].xp, "segment xp"));
            TN_TRY(check_ptr(segs[i].wp, "segment wp"));
        }
        TN_TRY(check_ptr(y ? static_cast<const void*>(y) : static_cast<const void*>(yp), "output"));
    }
    *out = cd;
    if (od) *od = tn_dims{N, k, cd.Do, cd.Ho, cd.Wo};
    return TN_OK;
}

}  // namespace tn

extern "C" {

tn_status tn_conv3d(const uint32_t* xp, tn_dims xd, const uint32_t* wp, int32_t k, tn_geom g,
                    int32_t* y, tn_stream stream) {
    TN_TRY(check_dims(xd, "xd"));
    tn_segment seg{xp, xd, 0, wp};
    ConvDesc cd;
    TN_TRY(build_conv(&seg, 1, k, g, nullptr, nullptr, y, nullptr, &cd, nullptr));
    return run_conv(cd, cs(stream), "tn_conv3d");
}

tn_status tn_conv3d_requant(const uint32_t* xp, tn_dims xd, const uint32_t* wp, int32_t k,
                            tn_geom g, const int32_t* lo, const int32_t* hi, uint32_t* yp,
                            tn_stream stream) {
    TN_TRY(check_dims(xd, "xd"));
    tn_segment seg{xp, xd, 0, wp};
    ConvDesc cd;
    TN_TRY(build_conv(&seg, 1, k, g, lo, hi, nullptr, yp, &cd, nullptr));
    return run_conv(cd, cs(stream), "tn_conv3d_requant");
}

tn_status tn_conv3d_seg(const tn_segment* segs, int32_t nseg, int32_t k, tn_geom g,
                        const int32_t* lo, const int32_t* hi, int32_t* y, uint32_t* yp,
                        tn_stream stream) {
    if (segs == nullptr) return fail(TN_EINVAL, "segs is NULL");
    ConvDesc cd;
    TN_TRY(build_conv(segs, nseg, k, g, lo, hi, y, yp, &cd, nullptr));
    return run_conv(cd, cs(stream), "tn_conv3d_seg");
}

struct tn_conv_prep {
    tn::TzPrep* tz;
};

tn_status tn_conv_prepare(const tn_segment* segs, int32_t nseg, int32_t k, tn_geom g, int32_t requant,
                          tn_conv_prep** out, tn_stream stream) {
    if (out == nullptr) return fail(TN_EINVAL, "tn_conv_prepare: out is NULL");
    *out = nullptr;
    if (segs == nullptr) return fail(TN_EINVAL, "tn_conv_prepare: segs is NULL");
    if (nseg < 1 || nseg > kMaxSeg) return fail(TN_EINVAL, "nseg must be 1 or 2 (got %d)", nseg);
    // the activations and outputs are not touched: stand-in pointers for build_conv's checks
    alignas(16) static const uint32_t dummy[4] = {0u, 0u, 0u, 0u};
    tn_segment sg[kMaxSeg];
    for (int i = 0; i < nseg; ++i) {
        sg[i] = segs[i];
        if (sg[i].xp == nullptr) sg[i].xp = dummy;
    }
    const int32_t* t = reinterpret_cast<const int32_t*>(dummy);
    int32_t* yo = reinterpret_cast<int32_t*>(const_cast<uint32_t*>(dummy));
    ConvDesc cd;
    TN_TRY(build_conv(sg, nseg, k, g, requant ? t : nullptr, requant ? t : nullptr, requant ? nullptr : yo,
                      requant ? const_cast<uint32_t*>(dummy) : nullptr, &cd, nullptr));
    tn_conv_prep* p = new tn_conv_prep{nullptr};
    const int pk = cd.N > 0 && cd.Do > 0 && cd.Ho > 0 && cd.Wo > 0 ? pick_kernel(cd, g_conv_kernel) : -1;
    if (pk == TN_KERNEL_TZ || pk == TN_KERNEL_WIDE) {
        const tn_status st = cuda_status(tz_prepare(cd, g_conv_kernel != TN_KERNEL_TZ8, &p->tz, cs(stream)),
                                         "tn_conv_prepare");
        if (st != TN_OK) { delete p; return st; }
    }
    *out = p;
    return TN_OK;
}

int64_t tn_conv_prep_bytes(const tn_conv_prep* p) {
    return p ? static_cast<int64_t>(tz_prep_bytes(p->tz)) : 0;
}

void tn_conv_prep_destroy(tn_conv_prep* p) {
    if (p == nullptr) return;
    tz_prep_free(p->tz);
    delete p;
}

tn_status tn_conv3d_requant_prepared(const tn_conv_prep* p, const uint32_t* xp, tn_dims xd,
                                     const uint32_t* wp, int32_t k, tn_geom g, const int32_t* lo,
                                     const int32_t* hi, uint32_t* yp, tn_stream stream) {
    TN_TRY(check_dims(xd, "xd"));
    tn_segment seg{xp, xd, 0, wp};
    ConvDesc cd;
    TN_TRY(build_conv(&seg, 1, k, g, lo, hi, nullptr, yp, &cd, nullptr));
    cd.prep = p ? p->tz : nullptr;
    return run_conv(cd, cs(stream), "tn_conv3d_requant_prepared");
}

tn_status tn_conv3d_seg_prepared(const tn_conv_prep* p, const tn_segment* segs, int32_t nseg,
                                 int32_t k, tn_geom g, const int32_t* lo, const int32_t* hi,
                                 int32_t* y, uint32_t* yp, tn_stream stream) {
    if (segs == nullptr) return fail(TN_EINVAL, "segs is NULL");
    ConvDesc cd;
    TN_TRY(build_conv(segs, nseg, k, g, lo, hi, y, yp, &cd, nullptr));
    cd.prep = p ? p->tz : nullptr;
    return run_conv(cd, cs(stream), "tn_conv3d_seg_prepared");
}

tn_status tn_conv3d_first(const float* x, tn_dims xd, float t_lo, float t_hi, const uint32_t* wp,
                          int32_t k, tn_geom g, const int32_t* lo, const int32_t* hi,
                          uint32_t* yp, int64_t* d_bad, tn_stream stream) {
    TN_TRY(check_dims(xd, "xd"));
    TN_TRY(check_geom(g));
    if (xd.c != 1) return fail(TN_ESHAPE, "tn_conv3d_first needs c == 1 (got %d)", xd.c);
    if (k < 1 || k > 32) return fail(TN_EUNSUPPORTED, "tn_conv3d_first supports 1 <= k <= 32 (got %d)", k);
    if (!(t_lo <= t_hi)) return fail(TN_EINVAL, "need t_lo <= t_hi");
    if (lo == nullptr || hi == nullptr) return fail(TN_EINVAL, "lo/hi is NULL");
    FirstDesc fd{};
    fd.D = xd.d; fd.H = xd.h; fd.W = xd.w; fd.zbeg = 0; fd.Dg = xd.d;
    fd.t_lo = t_lo; fd.t_hi = t_hi; fd.wp = wp; fd.N = xd.n; fd.K = k;
    for (int a = 0; a < 3; ++a) { fd.s[a] = g.stride[a]; fd.p[a] = g.pad[a]; fd.dl[a] = g.dil[a]; }
    fd.Do = out_extent(xd.d, g.stride[0], g.pad[0], g.dil[0]);
    fd.Ho = out_extent(xd.h, g.stride[1], g.pad[1], g.dil[1]);
    fd.Wo = out_extent(xd.w, g.stride[2], g.pad[2], g.dil[2]);
    fd.zo_beg = 0;
    fd.lo = lo; fd.hi = hi; fd.yp = yp; fd.d_bad = d_bad;
    fd.bad_base = 0;
    fd.bad_nstride = static_cast<int64_t>(xd.d) * xd.h * xd.w;
    fd.x = x;
    if (empty(xd)) return TN_OK;
    if (fd.Do < 1 || fd.Ho < 1 || fd.Wo < 1) return fail(TN_ESHAPE, "conv output would be empty");
    TN_TRY(check_ptr(x, "x"));
    TN_TRY(check_ptr(wp, "wp"));
    TN_TRY(check_ptr(yp, "yp"));
    return cuda_status(launch_conv_first(fd, cs(stream)), "tn_conv3d_first");
}

tn_status tn_predict(const uint32_t* tp, tn_dims td, const float* w, const float* b,
                     int32_t nclass, float* logits, tn_stream stream) {
    TN_TRY(check_dims(td, "td"));
    if (td.c > 64) return fail(TN_EUNSUPPORTED, "tn_predict supports c <= 64 (got %d)", td.c);
    if (nclass < 1 || nclass > 8) return fail(TN_EUNSUPPORTED, "tn_predict supports 1..8 classes");
    if (w == nullptr || b == nullptr) return fail(TN_EINVAL, "w/b is NULL");
    if (empty(td)) return TN_OK;
    TN_TRY(check_ptr(tp, "tp"));
    TN_TRY(check_ptr(logits, "logits"));
    return cuda_status(launch_predict(tp, td, w, b, nclass, logits, cs(stream)), "tn_predict");
}

tn_status tn_set_conv_kernel(int32_t which) {
    if (which != TN_KERNEL_AUTO && which != TN_KERNEL_POPC && which != TN_KERNEL_TZ && which != TN_KERNEL_TZ8)
        return fail(TN_EINVAL, "unknown kernel selector %d", which);
    g_conv_kernel = which;
    return TN_OK;
}

int32_t tn_get_conv_kernel(void) { return g_conv_kernel; }

tn_status tn_set_grid_cap(int32_t max_ctas) {
    if (max_ctas < 0) return fail(TN_EINVAL, "grid cap must be >= 0 (got %d)", max_ctas);
    g_grid_cap = max_ctas;
    return TN_OK;
}

int32_t tn_conv_operands_for(const tn_segment* segs, int32_t nseg, int32_t k, tn_geom g) {
    const int32_t kern = tn_conv_kernel_for(segs, nseg, k, g);
    if (kern == TN_KERNEL_WIDE) return 4;
    if (kern != TN_KERNEL_TZ) return 0;
    ConvDesc cd;
    uint32_t* dummy = reinterpret_cast<uint32_t*>(static_cast<uintptr_t>(256));
    static const int32_t zero = 0;
    tn_segment tmp[kMaxSeg];
    for (int i = 0; i < nseg && i < kMaxSeg; ++i) {
        tmp[i] = segs[i];
        if (tmp[i].xp == nullptr) tmp[i].xp = dummy;
        if (tmp[i].wp == nullptr) tmp[i].wp = dummy;
    }
    if (build_conv(tmp, nseg, k, g, &zero, &zero, nullptr, dummy, &cd, nullptr) != TN_OK) return 0;
    return conv_tz_uses_f4(cd, g_conv_kernel != TN_KERNEL_TZ8) ? 4 : 8;
}

int32_t tn_conv_kernel_for(const tn_segment* segs, int32_t nseg, int32_t k, tn_geom g) {
    if (segs == nullptr) return -1;
    // a dummy output pointer: only the shape logic of build_conv is used here
    ConvDesc cd;
    uint32_t* dummy = reinterpret_cast<uint32_t*>(static_cast<uintptr_t>(256));
    static const int32_t zero = 0;
    tn_segment tmp[kMaxSeg];
    for (int i = 0; i < nseg && i < kMaxSeg; ++i) {
        tmp[i] = segs[i];
        if (tmp[i].xp == nullptr) tmp[i].xp = dummy;
        if (tmp[i].wp == nullptr) tmp[i].wp = dummy;
    }
    if (build_conv(tmp, nseg, k, g, &zero, &zero, nullptr, dummy, &cd, nullptr) != TN_OK) return -1;
    const int kern = pick_kernel(cd, g_conv_kernel);
    if (kern == TN_KERNEL_POPC || kern < 0) {
        // the popc kernel covers every valid shape of a plain tn_conv3d_seg call
        return g_conv_kernel == TN_KERNEL_AUTO || g_conv_kernel == TN_KERNEL_POPC || g_conv_kernel == TN_KERNEL_TZ8
                   ? TN_KERNEL_POPC : -1;
    }
    return kern;
}

}  // extern "C"
