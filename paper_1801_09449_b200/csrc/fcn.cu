// fcn.cu -- A9: the ternary FCN driver (tn_fcn_*).  A host-side layer table
// (copied at create) is planned against the input extents into a packed
// activation workspace; tn_fcn_forward then queues one kernel per layer on the
// caller's stream: A7 first layer, A2-A6 ternary conv blocks with the fused A4
// epilogue (stride-2 downsampling, nearest-x2 upsample gathers and skip
// concatenation happen inside the conv kernels' loads), and the A8 prediction.
// Table 1 is the template; the concrete 3D table is given
// by the caller (reading R9; the Python binding's fcn_table()).
#include "tn_internal.cuh"

#include <algorithm>
#include <new>
#include <vector>


using namespace tn;



namespace {

struct LayerPlan {
    tn_dims out;
    size_t off;
    size_t bytes;
};

constexpr size_t kAlign = 256;

size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

tn_status plan(const tn_fcn* net, tn_dims xd, std::vector<LayerPlan>& P, size_t* total,
               size_t* scratch_off) {
    const int L = static_cast<int>(net->layers.size());
    P.assign(L, LayerPlan{});
    size_t off = 0;
    for (int i = 0; i < L; ++i) {
        const tn_layer& ly = net->layers[i];
        int d, h, w;
        if (ly.kind == TN_LAYER_FIRST) {
            d = xd.d; h = xd.h; w = xd.w;
        } else {
            d = h = w = -1;
            for (int sgi = 0; sgi < ly.nseg; ++sgi) {
                const tn_dims& sd = P[ly.src[sgi]].out;
                const int f = ly.upsample[sgi] ? 2 : 1, fz = ly.upsample[sgi] == 1 ? 2 : 1;
                if (sgi == 0) { d = sd.d * fz; h = sd.h * f; w = sd.w * f; }
                else if (sd.d * fz != d || sd.h * f != h || sd.w * f != w) {
                    set_error("layer %d: segment extents differ (%dx%dx%d vs %dx%dx%d)", i, sd.d * fz,
                              sd.h * f, sd.w * f, d, h, w);
                    return TN_ESHAPE;
                }
            }
        }
        const int s = ly.stride, pdl = ly.dil;
        tn_dims o{xd.n, ly.c_out, out_extent(d, s, pdl, pdl), out_extent(h, s, pdl, pdl),
                  out_extent(w, s, pdl, pdl)};
        if (o.d < 1 || o.h < 1 || o.w < 1) {
            set_error("layer %d: output would be empty for input %dx%dx%d", i, d, h, w);
            return TN_ESHAPE;
        }
        P[i].out = o;
        P[i].off = off;
        P[i].bytes = tn_packed_bytes(o);
        off = align_up(off + P[i].bytes);
    }
    // a multi-channel float input (e.g. Table 1's 15-slice stacks) is ternarised and packed
    // into this buffer first; layer 0 is then a regular conv from it
    *scratch_off = off;
    if (xd.c > 1) off = align_up(off + tn_packed_bytes(xd));
    *total = align_up(off);
    return TN_OK;
}

// The conv descriptor of layer i (anything but a one-channel TN_LAYER_FIRST) over workspace base.
ConvDesc layer_desc(const tn_fcn* net, const std::vector<LayerPlan>& P, int i, char* base, size_t soff, tn_dims xd,
                    float* logits) {
    const tn_layer& ly = net->layers[i];
    const int L = static_cast<int>(net->layers.size());
    const tn_dims& o = P[i].out;
    uint32_t* outp = reinterpret_cast<uint32_t*>(base + P[i].off);
    ConvDesc cd{};
    cd.nseg = ly.nseg;
    cd.N = xd.n;
    cd.K = ly.c_out;
    if (ly.kind == TN_LAYER_FIRST) {   // multi-channel input, packed into the workspace at soff
        SegDesc& sd = cd.seg[0];
        sd.xp = reinterpret_cast<const uint32_t*>(base + soff); sd.wp = ly.wp[0]; sd.c = xd.c;
        sd.cw = (xd.c + 31) / 32;
        sd.D = xd.d; sd.H = xd.h; sd.W = xd.w; sd.zbeg = 0; sd.up = 0;
    }
    for (int sgi = 0; sgi < ly.nseg && ly.kind != TN_LAYER_FIRST; ++sgi) {
        const LayerPlan& sp = P[ly.src[sgi]];
        SegDesc& sd = cd.seg[sgi];
        sd.xp = reinterpret_cast<const uint32_t*>(base + sp.off);
        sd.wp = ly.wp[sgi];
        sd.c = sp.out.c;
        sd.cw = (sp.out.c + 31) / 32;
        sd.D = sp.out.d; sd.H = sp.out.h; sd.W = sp.out.w;
        sd.zbeg = 0;
        sd.up = ly.upsample[sgi];
    }
    const int f = ly.upsample[0] ? 2 : 1, fz = ly.upsample[0] == 1 ? 2 : 1;
    cd.Dci = cd.seg[0].D * fz; cd.Hci = cd.seg[0].H * f; cd.Wci = cd.seg[0].W * f;
    for (int a = 0; a < 3; ++a) { cd.s[a] = ly.stride; cd.p[a] = ly.dil; cd.dl[a] = ly.dil; }
    cd.Do = o.d; cd.Ho = o.h; cd.Wo = o.w; cd.zo_beg = 0;
    cd.yp = outp; cd.y = nullptr; cd.lo = ly.lo; cd.hi = ly.hi;
    cd.cwo = (ly.c_out + 31) / 32;
    if (i == L - 1) {   // A8 fused into the last block's epilogue
        cd.logits = logits;
        cd.lstride = static_cast<int64_t>(o.d) * o.h * o.w;
        cd.pw = net->pred_w; cd.pb = net->pred_b; cd.nclass = net->nclass;
        cd.no_yp = 1;   // fused prediction: the last layer's packed codes are not stored
    }
    cd.prep = i < static_cast<int>(net->prep.size()) ? net->prep[i] : nullptr;
    return cd;
}

}  // namespace

extern "C" {

tn_status tn_fcn_create(const tn_layer* layers, int32_t n_layers, float t_lo, float t_hi,
                        const float* pred_w, const float* pred_b, int32_t nclass, tn_fcn** out) {
    if (out == nullptr || layers == nullptr) { set_error("layers/out is NULL"); return TN_EINVAL; }
    *out = nullptr;
    if (n_layers < 1) { set_error("need at least one layer"); return TN_EINVAL; }
    if (!(t_lo <= t_hi)) { set_error("need t_lo <= t_hi"); return TN_EINVAL; }
    if (nclass < 1 || nclass > 8) { set_error("nclass must be 1..8"); return TN_EUNSUPPORTED; }
    if (pred_w == nullptr || pred_b == nullptr) { set_error("pred_w/pred_b is NULL"); return TN_EINVAL; }
    tn_fcn* net = new (std::nothrow) tn_fcn();
    if (net == nullptr) { set_error("out of host memory"); return TN_EINVAL; }
    net->layers.assign(layers, layers + n_layers);
    net->t_lo = t_lo; net->t_hi = t_hi;
    net->pred_w = pred_w; net->pred_b = pred_b; net->nclass = nclass;
    for (int s = 0; s < kMaxSeg; ++s) net->cin[s].assign(n_layers, 0);
    auto bad = [&](tn_status st) { delete net; return st; };
    for (int i = 0; i < n_layers; ++i) {
        const tn_layer& ly = layers[i];
        if (ly.c_out < 1) { set_error("layer %d: c_out < 1", i); return bad(TN_EINVAL); }
        if (ly.stride < 1 || ly.stride > 2 || ly.dil < 1) {
            set_error("layer %d: stride must be 1 or 2 and dil >= 1", i);
            return bad(TN_EINVAL);
        }
        if (ly.lo == nullptr || ly.hi == nullptr) { set_error("layer %d: lo/hi NULL", i); return bad(TN_EINVAL); }
        if (ly.kind == TN_LAYER_FIRST) {
            if (i != 0 || ly.nseg != 1 || ly.src[0] != -1 || ly.upsample[0] != 0) {
                set_error("layer %d: the first layer must be entry 0 with one segment from input -1", i);
                return bad(TN_EINVAL);
            }
            if (ly.wp[0] == nullptr) { set_error("layer 0: wp NULL"); return bad(TN_EINVAL); }
            net->cin[0][0] = 1;
        } else if (ly.kind == TN_LAYER_CONV) {
            if (i == 0) { set_error("layer 0 must be TN_LAYER_FIRST"); return bad(TN_EINVAL); }
            if (ly.nseg < 1 || ly.nseg > kMaxSeg) { set_error("layer %d: nseg must be 1 or 2", i); return bad(TN_EINVAL); }
            for (int s = 0; s < ly.nseg; ++s) {
                if (ly.src[s] < 0 || ly.src[s] >= i) {
                    set_error("layer %d: src[%d] = %d must name an earlier layer", i, s, ly.src[s]);
                    return bad(TN_EINVAL);
                }
                if (ly.upsample[s] < 0 || ly.upsample[s] > 2) { set_error("layer %d: bad upsample", i); return bad(TN_EINVAL); }
                if (ly.wp[s] == nullptr) { set_error("layer %d: wp[%d] NULL", i, s); return bad(TN_EINVAL); }
                net->cin[s][i] = layers[ly.src[s]].c_out;
            }
            if (ly.nseg == 2 && (net->cin[0][i] + 31) / 32 != (net->cin[1][i] + 31) / 32) {
                set_error("layer %d: segments with different ceil(c/32) are not supported", i);
                return bad(TN_EUNSUPPORTED);
            }
        } else {
            set_error("layer %d: unknown kind %d", i, ly.kind);
            return bad(TN_EINVAL);
        }
    }
    if (layers[n_layers - 1].c_out > 64) { set_error("prediction needs c_out <= 64 on the last layer"); return bad(TN_EUNSUPPORTED); }
    *out = net;
    return TN_OK;
}

size_t tn_fcn_workspace_bytes(const tn_fcn* net, tn_dims xd) {
    if (net == nullptr) return 0;
    std::vector<LayerPlan> P;
    size_t total = 0;
    size_t soff = 0;
    if (plan(net, xd, P, &total, &soff) != TN_OK) return 0;
    return total;
}

const uint32_t* tn_fcn_layer_output(const tn_fcn* net, tn_dims xd, const void* ws, int32_t i,
                                    tn_dims* out_dims) {
    if (net == nullptr || ws == nullptr || i < 0 || i >= static_cast<int>(net->layers.size())) return nullptr;
    std::vector<LayerPlan> P;
    size_t total = 0;
    size_t soff = 0;
    if (plan(net, xd, P, &total, &soff) != TN_OK) return nullptr;
    if (out_dims) *out_dims = P[i].out;
    return reinterpret_cast<const uint32_t*>(static_cast<const char*>(ws) + P[i].off);
}

tn_status tn_fcn_forward(const tn_fcn* net, const float* x, tn_dims xd, float* logits, void* ws,
                         size_t ws_bytes, int64_t* d_bad, tn_stream stream) {
    return tn_fcn_forward_range(net, x, xd, logits, ws, ws_bytes, d_bad, 0, -1, stream);
}

tn_status tn_fcn_forward_range(const tn_fcn* net, const float* x, tn_dims xd, float* logits, void* ws,
                               size_t ws_bytes, int64_t* d_bad, int32_t first, int32_t last, tn_stream stream) {
    if (net == nullptr) { set_error("net is NULL"); return TN_EINVAL; }
    const int nl = static_cast<int>(net->layers.size());
    if (last < 0) last = nl;
    if (first < 0 || first > last || last > nl) {
        set_error("layer range [%d, %d) outside [0, %d)", first, last, nl);
        return TN_EINVAL;
    }
    if (xd.c < 1 || xd.c > 64) { set_error("FCN input needs 1 <= c <= 64 (got %d)", xd.c); return TN_ESHAPE; }
    if (xd.n < 1 || xd.d < 1 || xd.h < 1 || xd.w < 1) { set_error("FCN input must be non-empty"); return TN_ESHAPE; }
    std::vector<LayerPlan> P;
    size_t total = 0;
    size_t soff = 0;
    tn_status st = plan(net, xd, P, &total, &soff);
    if (st != TN_OK) return st;
    if (ws == nullptr || ws_bytes < total) {
        set_error("workspace too small: need %zu bytes, got %zu", total, ws_bytes);
        return TN_EINVAL;
    }
    if (x == nullptr || logits == nullptr) { set_error("x/logits is NULL"); return TN_EINVAL; }
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(logits) |
         reinterpret_cast<uintptr_t>(ws)) & 15u) {
        set_error("x, logits and ws must be 16-byte aligned");
        return TN_EALIGN;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    char* base = static_cast<char*>(ws);
    const int L = static_cast<int>(net->layers.size());
    for (int i = first; i < last; ++i) {
        NvtxRange nv("fcn layer", i + 1);   // Table 1 numbering (#1 .. #L)
        const tn_layer& ly = net->layers[i];
        uint32_t* outp = reinterpret_cast<uint32_t*>(base + P[i].off);
        const tn_dims& o = P[i].out;
        if (ly.kind == TN_LAYER_FIRST && xd.c == 1) {
            if (ly.c_out > 32) { set_error("a one-channel first layer supports c_out <= 32"); return TN_EUNSUPPORTED; }
            FirstDesc fd{};
            fd.x = x; fd.D = xd.d; fd.H = xd.h; fd.W = xd.w; fd.zbeg = 0; fd.Dg = xd.d;
            fd.t_lo = net->t_lo; fd.t_hi = net->t_hi; fd.wp = ly.wp[0];
            fd.N = xd.n; fd.K = ly.c_out;
            for (int a = 0; a < 3; ++a) { fd.s[a] = ly.stride; fd.p[a] = ly.dil; fd.dl[a] = ly.dil; }
            fd.Do = o.d; fd.Ho = o.h; fd.Wo = o.w; fd.zo_beg = 0;
            fd.lo = ly.lo; fd.hi = ly.hi; fd.yp = outp; fd.d_bad = d_bad;
            fd.bad_base = 0; fd.bad_nstride = static_cast<int64_t>(xd.d) * xd.h * xd.w;
            cudaError_t e = launch_conv_first(fd, s);
            if (e != cudaSuccess) { set_error("layer %d: %s", i, cudaGetErrorString(e)); return TN_ECUDA; }
            continue;
        }
        if (ly.kind == TN_LAYER_FIRST) {
            // A7 on a multi-channel float input (PAPER.md:180, 15 neighbouring slices per stack):
            // Eq. 6 + pack (tn_pack_f32's kernel, NaN -> d_bad), then layer 0 as a regular conv
            cudaError_t e = launch_pack_f32(x, xd, net->t_lo, net->t_hi, reinterpret_cast<uint32_t*>(base + soff),
                                            d_bad, s);
            if (e != cudaSuccess) { set_error("input pack: %s", cudaGetErrorString(e)); return TN_ECUDA; }
        }
        ConvDesc cd = layer_desc(net, P, i, base, soff, xd, logits);
        st = run_conv(cd, s, "tn_fcn_forward");
        if (st != TN_OK) return st;
    }
    if (last == L && net->layers[L - 1].kind == TN_LAYER_FIRST && xd.c == 1) {
        const LayerPlan& last = P[L - 1];
        cudaError_t e = launch_predict(reinterpret_cast<const uint32_t*>(base + last.off), last.out,
                                       net->pred_w, net->pred_b, net->nclass, logits, s);
        if (e != cudaSuccess) { set_error("prediction: %s", cudaGetErrorString(e)); return TN_ECUDA; }
    }
    return TN_OK;
}

tn_status tn_fcn_prepare(tn_fcn* net, tn_dims xd, tn_stream stream) {
    if (net == nullptr) { set_error("net is NULL"); return TN_EINVAL; }
    if (xd.c < 1 || xd.c > 64) { set_error("FCN input needs 1 <= c <= 64 (got %d)", xd.c); return TN_ESHAPE; }
    if (xd.n < 1 || xd.d < 1 || xd.h < 1 || xd.w < 1) { set_error("FCN input must be non-empty"); return TN_ESHAPE; }
    std::vector<LayerPlan> P;
    size_t total = 0, soff = 0;
    tn_status st = plan(net, xd, P, &total, &soff);
    if (st != TN_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const bool allow_f4 = tn_get_conv_kernel() != TN_KERNEL_TZ8;
    const int L = static_cast<int>(net->layers.size());
    std::vector<TzPrep*> prep(L, nullptr);
    // an image depends on the channel widths, banks and geometry only: the descriptors' buffer
    // pointers are never read (stand-in base); the logits pointer only selects the epilogue form
    alignas(16) static float dummy_logits[4];
    for (int i = 0; i < L; ++i) {
        if (net->layers[i].kind == TN_LAYER_FIRST && xd.c == 1) continue;   // dedicated first-layer kernel
        const ConvDesc cd = layer_desc(net, P, i, reinterpret_cast<char*>(256), soff, xd, dummy_logits);
        cudaError_t e = tz_prepare(cd, allow_f4, &prep[i], s);
        if (e != cudaSuccess) {
            for (TzPrep* q : prep) tz_prep_free(q);
            set_error("tn_fcn_prepare: layer %d: %s", i, cudaGetErrorString(e));
            return TN_ECUDA;
        }
    }
    for (TzPrep* q : net->prep) tz_prep_free(q);
    net->prep.swap(prep);
    return TN_OK;
}

size_t tn_fcn_prep_bytes(const tn_fcn* net) {
    size_t b = 0;
    if (net != nullptr)
        for (const TzPrep* q : net->prep) b += tz_prep_bytes(q);
    return b;
}

void tn_fcn_destroy(tn_fcn* net) { delete net; }

}  // extern "C"
