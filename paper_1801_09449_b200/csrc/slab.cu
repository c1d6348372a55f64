// slab.cu -- z-slab decomposition of the ternary FCN (BASELINE configs[4]):
// each rank owns planes [z0, z1) of one large volume; every layer's packed
// output is kept with one halo plane on each side, filled after the layer by a
// point-to-point exchange with the ranks owning the neighbouring slabs (NCCL
// send/recv over NVLink on the caller's stream).  Stride-1 convs read both
// halos, stride-2 convs the lower one, upsampled segments the low-resolution
// neighbours; planes outside the volume are never read (the kernels bound
// against the global extent), which is exactly the convolutions' zero padding.
// The same kernels as tn_fcn_forward run on the slab through the global z
// offsets in their descriptors (zo_beg / zbeg), so slab results are
// bit-identical to the whole-volume forward.
//
// tn_fcn_forward_slabs_local runs all slabs of one volume on one device with
// the halos exchanged by device copies (same kernels, same offsets, same
// schedule) -- a single-GPU emulation of the decomposition used by the tests.
#include "tn_internal.cuh"

#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <vector>


using namespace tn;



struct tn_comm {
    ncclComm_t comm;
    int rank, nranks;
};

namespace {

constexpr size_t kAlign = 256;
size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

struct SlabPlan {
    tn_dims g;                               // global input dims
    int z0, z1;
    size_t x_off, x_bytes, x_plane;          // extended float input [z0-1, z1+1)
    std::vector<tn_slab_layer> L;
    size_t scratch_off;      // int32 partial sums for split two-segment blocks
    size_t total;
};

tn_status make_slab_plan(const tn_fcn* net, tn_dims g, int z0, int z1, SlabPlan& sp) {
    const int nl = static_cast<int>(net->layers.size());
    if (g.n != 1 || g.c != 1) { set_error("slab forward needs n == 1 and c == 1"); return TN_ESHAPE; }
    if (g.d < 1 || g.h < 1 || g.w < 1) { set_error("empty volume"); return TN_ESHAPE; }
    // global extents per layer (same rule as the whole-volume plan)
    std::vector<tn_dims> out(nl);
    for (int i = 0; i < nl; ++i) {
        const tn_layer& ly = net->layers[i];
        int d, h, w;
        if (ly.kind == TN_LAYER_FIRST) { d = g.d; h = g.h; w = g.w; }
        else {
            const tn_dims& s = out[ly.src[0]];
            const int f = ly.upsample[0] ? 2 : 1;
            d = s.d * f; h = s.h * f; w = s.w * f;
        }
        if (ly.dil != 1) { set_error("slab forward supports dilation 1"); return TN_EUNSUPPORTED; }
        out[i] = tn_dims{1, ly.c_out, out_extent(d, ly.stride, 1, 1), out_extent(h, ly.stride, 1, 1),
                         out_extent(w, ly.stride, 1, 1)};
    }
    int maxscale = 1;
    for (int i = 0; i < nl; ++i) {
        if (out[i].d < 1 || g.d % out[i].d != 0) { set_error("layer %d: extent does not divide the volume", i); return TN_ESHAPE; }
        maxscale = std::max(maxscale, g.d / out[i].d);
    }
    if (z0 < 0 || z1 > g.d || z0 >= z1 || z0 % maxscale || z1 % maxscale) {
        set_error("slab [%d, %d) must be non-empty, inside [0, %d) and a multiple of %d", z0, z1, g.d, maxscale);
        return TN_ESHAPE;
    }
    sp.g = g; sp.z0 = z0; sp.z1 = z1;
    sp.x_plane = static_cast<size_t>(g.h) * g.w * sizeof(float);
    sp.x_off = 0;
    sp.x_bytes = sp.x_plane * (z1 - z0 + 2);
    size_t off = align_up(sp.x_bytes), scratch = 0;
    sp.L.assign(nl, tn_slab_layer{});
    for (int i = 0; i < nl; ++i) {
        tn_slab_layer& s = sp.L[i];
        const int scale = g.d / out[i].d;
        s.level_scale = scale;
        s.c = out[i].c; s.h = out[i].h; s.w = out[i].w;
        s.gd = out[i].d;
        s.z0 = z0 / scale; s.z1 = z1 / scale;
        s.halo = (i + 1 < nl) ? 1 : 0;       // the last layer only feeds the 1x1x1 prediction
        s.plane_bytes = static_cast<int64_t>(s.h) * s.w * 2 * ((s.c + 31) / 32) * 4;
        s.offset = static_cast<int64_t>(off);
        off = align_up(off + static_cast<size_t>(s.plane_bytes) * (s.z1 - s.z0 + 2));
        if (net->layers[i].nseg == 2 && net->cin[0][i] + net->cin[1][i] > 64)
            scratch = std::max(scratch, static_cast<size_t>(s.z1 - s.z0) * s.h * s.w * s.c * 4);
    }
    sp.scratch_off = off;
    sp.total = align_up(off + scratch);
    return TN_OK;
}

// Queue layer i's kernel for one slab (n = 1); the caller then fills the
// layer's halo planes (if sp.L[i].halo) before any consumer runs.
// logits/lstride: when i is the last layer, the A8 prediction is fused into it.
tn_status run_slab_layer(const tn_fcn* net, const SlabPlan& sp, char* ws, int i, int64_t* d_bad, cudaStream_t s,
                         float* logits, int64_t lstride) {
    {
        const tn_layer& ly = net->layers[i];
        const tn_slab_layer& o = sp.L[i];
        uint32_t* outp = reinterpret_cast<uint32_t*>(ws + o.offset + o.plane_bytes);   // skip the lower halo
        if (ly.kind == TN_LAYER_FIRST) {
            FirstDesc fd{};
            fd.x = reinterpret_cast<const float*>(ws + sp.x_off);
            fd.D = sp.z1 - sp.z0 + 2; fd.H = sp.g.h; fd.W = sp.g.w;
            fd.zbeg = sp.z0 - 1; fd.Dg = sp.g.d;
            fd.t_lo = net->t_lo; fd.t_hi = net->t_hi; fd.wp = ly.wp[0];
            fd.N = 1; fd.K = ly.c_out;
            for (int a = 0; a < 3; ++a) { fd.s[a] = ly.stride; fd.p[a] = 1; fd.dl[a] = 1; }
            fd.Do = o.z1 - o.z0; fd.Ho = o.h; fd.Wo = o.w; fd.zo_beg = o.z0;
            fd.lo = ly.lo; fd.hi = ly.hi; fd.yp = outp; fd.d_bad = d_bad;
            fd.bad_base = static_cast<int64_t>(sp.z0 - 1) * sp.g.h * sp.g.w;
            fd.bad_nstride = static_cast<int64_t>(sp.g.d) * sp.g.h * sp.g.w;
            cudaError_t e = launch_conv_first(fd, s);
            if (e != cudaSuccess) { set_error("slab layer %d: %s", i, cudaGetErrorString(e)); return TN_ECUDA; }
        } else {
            ConvDesc cd{};
            cd.nseg = ly.nseg;
            cd.N = 1;
            cd.K = ly.c_out;
            for (int sgi = 0; sgi < ly.nseg; ++sgi) {
                const tn_slab_layer& src = sp.L[ly.src[sgi]];
                SegDesc& sd = cd.seg[sgi];
                sd.xp = reinterpret_cast<const uint32_t*>(ws + src.offset);
                sd.wp = ly.wp[sgi];
                sd.c = src.c;
                sd.cw = (src.c + 31) / 32;
                sd.D = src.z1 - src.z0 + 2; sd.H = src.h; sd.W = src.w;
                sd.zbeg = src.z0 - 1;
                sd.up = ly.upsample[sgi];
            }
            const tn_slab_layer& s0 = sp.L[ly.src[0]];
            const int f = ly.upsample[0] ? 2 : 1;
            cd.Dci = s0.gd * f; cd.Hci = s0.h * f; cd.Wci = s0.w * f;
            for (int a = 0; a < 3; ++a) { cd.s[a] = ly.stride; cd.p[a] = 1; cd.dl[a] = 1; }
            cd.Do = o.z1 - o.z0; cd.Ho = o.h; cd.Wo = o.w; cd.zo_beg = o.z0;
            cd.yp = outp; cd.y = nullptr; cd.lo = ly.lo; cd.hi = ly.hi;
            cd.cwo = (ly.c_out + 31) / 32;
            if (i + 1 == static_cast<int>(net->layers.size())) {
                cd.logits = logits; cd.lstride = lstride;
                cd.pw = net->pred_w; cd.pb = net->pred_b; cd.nclass = net->nclass;
            }
            tn_status st = run_conv_scratch(cd, s, "slab conv", reinterpret_cast<int32_t*>(ws + sp.scratch_off));
            if (st != TN_OK) return st;
        }
    }
    return TN_OK;
}

tn_status nccl_status(ncclResult_t r, const char* where) {
    if (r == ncclSuccess) return TN_OK;
    set_error("%s: %s", where, ncclGetErrorString(r));
    return TN_ENCCL;
}

// Fill the lower / upper halo plane of a buffer of (planes) planes from the
// neighbouring ranks: my first owned plane goes down, my last goes up.
tn_status exchange_halo(tn_comm* c, char* buf, int64_t plane_bytes, int planes, cudaStream_t s) {
    const size_t pb = static_cast<size_t>(plane_bytes);
    ncclResult_t r = ncclGroupStart();
    if (r != ncclSuccess) return nccl_status(r, "ncclGroupStart");
    if (c->rank > 0) {
        ncclSend(buf + pb, pb, ncclUint8, c->rank - 1, c->comm, s);
        ncclRecv(buf, pb, ncclUint8, c->rank - 1, c->comm, s);
    }
    if (c->rank + 1 < c->nranks) {
        ncclSend(buf + pb * (planes - 2), pb, ncclUint8, c->rank + 1, c->comm, s);
        ncclRecv(buf + pb * (planes - 1), pb, ncclUint8, c->rank + 1, c->comm, s);
    }
    return nccl_status(ncclGroupEnd(), "halo exchange");
}

}  // namespace

extern "C" {

tn_status tn_comm_unique_id(void* id_out) {
    if (id_out == nullptr) { set_error("id_out is NULL"); return TN_EINVAL; }
    ncclUniqueId id;
    tn_status st = nccl_status(ncclGetUniqueId(&id), "ncclGetUniqueId");
    if (st != TN_OK) return st;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    memcpy(id_out, &id, sizeof(id));
    return TN_OK;
}

tn_status tn_comm_init(const void* nccl_unique_id, int32_t rank, int32_t nranks, tn_comm** out) {
    if (out == nullptr || nccl_unique_id == nullptr) { set_error("id/out is NULL"); return TN_EINVAL; }
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) { set_error("bad rank %d of %d", rank, nranks); return TN_EINVAL; }
    tn_comm* c = new (std::nothrow) tn_comm();
    if (c == nullptr) { set_error("out of host memory"); return TN_EINVAL; }
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof(id));
    tn_status st = nccl_status(ncclCommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
    if (st != TN_OK) { delete c; return st; }
    c->rank = rank;
    c->nranks = nranks;
    *out = c;
    return TN_OK;
}

void tn_comm_destroy(tn_comm* c) {
    if (c == nullptr) return;
    ncclCommDestroy(c->comm);
    delete c;
}

tn_status tn_fcn_slab_plan(const tn_fcn* net, tn_dims global, int32_t z0, int32_t z1, tn_slab_layer* out,
                           int32_t max_layers, size_t* ws_bytes) {
    if (net == nullptr) { set_error("net is NULL"); return TN_EINVAL; }
    SlabPlan sp;
    tn_status st = make_slab_plan(net, global, z0, z1, sp);
    if (st != TN_OK) return st;
    if (out != nullptr) {
        if (max_layers < static_cast<int32_t>(sp.L.size())) { set_error("max_layers too small"); return TN_EINVAL; }
        for (size_t i = 0; i < sp.L.size(); ++i) out[i] = sp.L[i];
    }
    if (ws_bytes) *ws_bytes = sp.total;
    return TN_OK;
}

size_t tn_fcn_slab_workspace_bytes(const tn_fcn* net, tn_dims global, int32_t z0, int32_t z1) {
    size_t b = 0;
    if (tn_fcn_slab_plan(net, global, z0, z1, nullptr, 0, &b) != TN_OK) return 0;
    return b;
}

tn_status tn_fcn_forward_slab(const tn_fcn* net, tn_comm* comm, const float* x_slab, tn_dims global, int32_t z0,
                              int32_t z1, float* logits_slab, void* ws, size_t ws_bytes, int64_t* d_bad,
                              tn_stream stream) {
    if (net == nullptr || comm == nullptr) { set_error("net/comm is NULL"); return TN_EINVAL; }
    SlabPlan sp;
    tn_status st = make_slab_plan(net, global, z0, z1, sp);
    if (st != TN_OK) return st;
    if (ws == nullptr || ws_bytes < sp.total) { set_error("workspace too small: need %zu", sp.total); return TN_EINVAL; }
    if (x_slab == nullptr || logits_slab == nullptr) { set_error("x/logits NULL"); return TN_EINVAL; }
    if ((reinterpret_cast<uintptr_t>(x_slab) | reinterpret_cast<uintptr_t>(logits_slab) |
         reinterpret_cast<uintptr_t>(ws)) & 15u) { set_error("pointers must be 16-byte aligned"); return TN_EALIGN; }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    char* base = static_cast<char*>(ws);
    // own input planes into the extended buffer, then the float halo planes
    cudaError_t e = cudaMemcpyAsync(base + sp.x_off + sp.x_plane, x_slab, sp.x_plane * (z1 - z0),
                                    cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) { set_error("input copy: %s", cudaGetErrorString(e)); return TN_ECUDA; }
    st = exchange_halo(comm, base + sp.x_off, static_cast<int64_t>(sp.x_plane), z1 - z0 + 2, s);
    if (st != TN_OK) return st;
    const int64_t lstride = static_cast<int64_t>(z1 - z0) * global.h * global.w;
    for (int i = 0; i < static_cast<int>(net->layers.size()); ++i) {
        st = run_slab_layer(net, sp, base, i, d_bad, s, logits_slab, lstride);
        if (st != TN_OK) return st;
        const tn_slab_layer& o = sp.L[i];
        if (o.halo) {
            st = exchange_halo(comm, base + o.offset, o.plane_bytes, o.z1 - o.z0 + 2, s);
            if (st != TN_OK) return st;
        }
    }
    return TN_OK;
}

size_t tn_fcn_slabs_local_workspace_bytes(const tn_fcn* net, tn_dims global, int32_t nslabs) {
    if (net == nullptr || nslabs < 1 || global.d % nslabs) return 0;
    size_t tot = 0;
    const int dz = global.d / nslabs;
    for (int r = 0; r < nslabs; ++r) {
        const size_t b = tn_fcn_slab_workspace_bytes(net, global, r * dz, (r + 1) * dz);
        if (b == 0) return 0;
        tot += align_up(b);
    }
    return tot;
}

tn_status tn_fcn_forward_slabs_local(const tn_fcn* net, const float* x, tn_dims global, int32_t nslabs,
                                     float* logits, void* ws, size_t ws_bytes, int64_t* d_bad, tn_stream stream) {
    if (net == nullptr || x == nullptr || logits == nullptr || ws == nullptr) { set_error("NULL argument"); return TN_EINVAL; }
    if (nslabs < 1 || global.d % nslabs) { set_error("nslabs must divide the depth"); return TN_ESHAPE; }
    const size_t need = tn_fcn_slabs_local_workspace_bytes(net, global, nslabs);
    if (need == 0) return TN_ESHAPE;
    if (ws_bytes < need) { set_error("workspace too small: need %zu", need); return TN_EINVAL; }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int dz = global.d / nslabs;
    std::vector<SlabPlan> P(nslabs);
    std::vector<char*> B(nslabs);
    char* p = static_cast<char*>(ws);
    for (int r = 0; r < nslabs; ++r) {
        tn_status st = make_slab_plan(net, global, r * dz, (r + 1) * dz, P[r]);
        if (st != TN_OK) return st;
        B[r] = p;
        p += align_up(P[r].total);
    }
    auto copy = [&](char* dst, const char* src, size_t n) -> tn_status {
        cudaError_t e = cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) { set_error("halo copy: %s", cudaGetErrorString(e)); return TN_ECUDA; }
        return TN_OK;
    };
    // halo exchange of one buffer kind across all slabs (device copies)
    auto exchange_all = [&](auto offset_of, auto plane_of, auto planes_of) -> tn_status {
        for (int r = 0; r < nslabs; ++r) {
            const size_t pb = plane_of(r);
            char* mine = B[r] + offset_of(r);
            const int np = planes_of(r);
            if (r > 0) {
                char* lower = B[r - 1] + offset_of(r - 1);
                tn_status st = copy(mine, lower + pb * (planes_of(r - 1) - 2), pb);
                if (st != TN_OK) return st;
            }
            if (r + 1 < nslabs) {
                char* upper = B[r + 1] + offset_of(r + 1);
                tn_status st = copy(mine + pb * (np - 1), upper + pb, pb);
                if (st != TN_OK) return st;
            }
        }
        return TN_OK;
    };
    const size_t xplane = P[0].x_plane;
    for (int r = 0; r < nslabs; ++r) {
        tn_status st = copy(B[r] + P[r].x_off + xplane, reinterpret_cast<const char*>(x) + xplane * r * dz, xplane * dz);
        if (st != TN_OK) return st;
    }
    tn_status st = exchange_all([&](int r) { return P[r].x_off; }, [&](int) { return xplane; },
                                [&](int) { return dz + 2; });
    if (st != TN_OK) return st;
    // layer-major across slabs: all slabs' layer i, then exchange its halos
    const int nl = static_cast<int>(net->layers.size());
    for (int i = 0; i < nl; ++i) {
        for (int r = 0; r < nslabs; ++r) {
            const int64_t cstride = static_cast<int64_t>(global.d) * global.h * global.w;
            float* lg = logits + static_cast<int64_t>(P[r].L.back().z0) * global.h * global.w;
            st = run_slab_layer(net, P[r], B[r], i, d_bad, s, lg, cstride);
            if (st != TN_OK) return st;
        }
        if (P[0].L[i].halo) {
            st = exchange_all([&](int r) { return static_cast<size_t>(P[r].L[i].offset); },
                              [&](int r) { return static_cast<size_t>(P[r].L[i].plane_bytes); },
                              [&](int r) { return P[r].L[i].z1 - P[r].L[i].z0 + 2; });
            if (st != TN_OK) return st;
        }
    }
    return TN_OK;
}

}  // extern "C"
