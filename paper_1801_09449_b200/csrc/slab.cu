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



// The communicator owns a comm stream and a pool of events: halo exchanges run on the comm
// stream, overlapping the interior planes computed on the caller's stream (tn_fcn_forward_slab).
constexpr int kCommEvents = 96;
struct tn_comm {
    ncclComm_t comm;
    int rank, nranks;
    cudaStream_t cs = nullptr;
    cudaEvent_t ev[kCommEvents] = {};
};

namespace {

constexpr size_t kAlign = 256;
size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

struct SlabPlan {
    tn_dims g;                               // global input dims
    int z0, z1;
    size_t x_off, x_bytes, x_plane;          // extended float input [z0-1, z1+1)
    int x_halo;                              // halo sides of the input (bit 0 lower, bit 1 upper)
    std::vector<tn_slab_layer> L;
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
            const int f = ly.upsample[0] ? 2 : 1, fz = ly.upsample[0] == 1 ? 2 : 1;
            d = s.d * fz; h = s.h * f; w = s.w * f;
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
    size_t off = align_up(sp.x_bytes);
    sp.L.assign(nl, tn_slab_layer{});
    for (int i = 0; i < nl; ++i) {
        tn_slab_layer& s = sp.L[i];
        const int scale = g.d / out[i].d;
        s.level_scale = scale;
        s.c = out[i].c; s.h = out[i].h; s.w = out[i].w;
        s.gd = out[i].d;
        s.z0 = z0 / scale; s.z1 = z1 / scale;
        s.halo = 0;                          // sides its consumers read (below); the last layer feeds only A8
        s.plane_bytes = static_cast<int64_t>(s.h) * s.w * 2 * ((s.c + 31) / 32) * 4;
        s.offset = static_cast<int64_t>(off);
        off = align_up(off + static_cast<size_t>(s.plane_bytes) * (s.z1 - s.z0 + 2));
    }
    // Halo sides each tensor's consumers read: a stride-1 conv (or a nearest-x2 upsampled segment)
    // reads one plane below and one above its owned range, a stride-2 conv only the plane below
    // (slab starts are even).  Bit 0 = lower halo, bit 1 = upper halo.
    sp.x_halo = 0;
    for (int j = 0; j < nl; ++j) {
        const tn_layer& ly = net->layers[j];
        for (int sgi = 0; sgi < ly.nseg; ++sgi) {
            const int sides = (ly.stride == 1 || ly.upsample[sgi] == 1) ? 3 : 1;
            if (ly.kind == TN_LAYER_FIRST) sp.x_halo |= sides;
            else sp.L[ly.src[sgi]].halo |= sides;
        }
    }
    sp.total = align_up(off);
    return TN_OK;
}

// Queue layer i's kernel for one slab (n = 1); the caller then fills the
// layer's halo planes (if sp.L[i].halo) before any consumer runs.
// logits/lstride: when i is the last layer, the A8 prediction is fused into it.
// za, zb: owned output planes [za, zb) of the layer (relative to its slab start; zb < 0 = all).
tn_status run_slab_layer(const tn_fcn* net, const SlabPlan& sp, char* ws, int i, int64_t* d_bad, cudaStream_t s,
                         float* logits, int64_t lstride, uint32_t* halo_lo = nullptr, uint32_t* halo_hi = nullptr,
                         int za = 0, int zb = -1) {
    NvtxRange nv("slab layer", i + 1);
    {
        const tn_layer& ly = net->layers[i];
        const tn_slab_layer& o = sp.L[i];
        if (zb < 0) zb = o.z1 - o.z0;
        if (za >= zb) return TN_OK;
        uint32_t* outp = reinterpret_cast<uint32_t*>(ws + o.offset + o.plane_bytes * (1 + za));   // skip the lower halo
        if (logits != nullptr) logits += static_cast<int64_t>(za) * o.h * o.w;
        if (ly.kind == TN_LAYER_FIRST) {
            FirstDesc fd{};
            fd.x = reinterpret_cast<const float*>(ws + sp.x_off);
            fd.D = sp.z1 - sp.z0 + 2; fd.H = sp.g.h; fd.W = sp.g.w;
            fd.zbeg = sp.z0 - 1; fd.Dg = sp.g.d;
            fd.t_lo = net->t_lo; fd.t_hi = net->t_hi; fd.wp = ly.wp[0];
            fd.N = 1; fd.K = ly.c_out;
            for (int a = 0; a < 3; ++a) { fd.s[a] = ly.stride; fd.p[a] = 1; fd.dl[a] = 1; }
            fd.Do = zb - za; fd.Ho = o.h; fd.Wo = o.w; fd.zo_beg = o.z0 + za;
            fd.lo = ly.lo; fd.hi = ly.hi; fd.yp = outp; fd.d_bad = d_bad;
            fd.bad_base = static_cast<int64_t>(sp.z0 - 1) * sp.g.h * sp.g.w;
            fd.bad_nstride = static_cast<int64_t>(sp.g.d) * sp.g.h * sp.g.w;
            fd.halo_lo = halo_lo; fd.halo_hi = halo_hi;
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
            const int f = ly.upsample[0] ? 2 : 1, fz = ly.upsample[0] == 1 ? 2 : 1;
            cd.Dci = s0.gd * fz; cd.Hci = s0.h * f; cd.Wci = s0.w * f;
            for (int a = 0; a < 3; ++a) { cd.s[a] = ly.stride; cd.p[a] = 1; cd.dl[a] = 1; }
            cd.Do = zb - za; cd.Ho = o.h; cd.Wo = o.w; cd.zo_beg = o.z0 + za;
            cd.yp = outp; cd.y = nullptr; cd.lo = ly.lo; cd.hi = ly.hi;
            cd.cwo = (ly.c_out + 31) / 32;
            cd.halo_lo = halo_lo; cd.halo_hi = halo_hi;
            cd.prep = i < static_cast<int>(net->prep.size()) ? net->prep[i] : nullptr;
            if (i + 1 == static_cast<int>(net->layers.size())) {
                cd.logits = logits; cd.lstride = lstride;
                cd.pw = net->pred_w; cd.pb = net->pred_b; cd.nclass = net->nclass;
                cd.no_yp = 1;
            }
            tn_status st = run_conv(cd, s, "slab conv");
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
// sides: bit 0 = my lower halo is read (so it is received from below, and the rank below
// receives my first plane as its upper halo only if it reads that side: both ranks derive the
// same plan, so a send is posted exactly when the peer posts the matching receive).
tn_status exchange_halo(tn_comm* c, char* buf, int64_t plane_bytes, int planes, int sides, cudaStream_t s) {
    NvtxRange nv("halo exchange");
    const size_t pb = static_cast<size_t>(plane_bytes);
    ncclResult_t r = ncclGroupStart();
    if (r != ncclSuccess) return nccl_status(r, "ncclGroupStart");
    if (c->rank > 0) {
        if (sides & 2) ncclSend(buf + pb, pb, ncclUint8, c->rank - 1, c->comm, s);
        if (sides & 1) ncclRecv(buf, pb, ncclUint8, c->rank - 1, c->comm, s);
    }
    if (c->rank + 1 < c->nranks) {
        if (sides & 1) ncclSend(buf + pb * (planes - 2), pb, ncclUint8, c->rank + 1, c->comm, s);
        if (sides & 2) ncclRecv(buf + pb * (planes - 1), pb, ncclUint8, c->rank + 1, c->comm, s);
    }
    return nccl_status(ncclGroupEnd(), "halo exchange");
}

// ---------------------------------------------------------------------------
// NEXT-1: halos without NCCL.  Each layer's requant epilogue stores its first /
// last owned output plane straight into the lower / upper neighbour's halo
// plane (ConvDesc::halo_lo / halo_hi: peer memory mapped over NVLink with CUDA
// IPC, or another slab's buffer when all slabs share one device), and a device
// flag replaces the send/recv pair.  Every slab owns two 64-bit progress flags
// (after its workspace): flags[0] is written by the lower neighbour, flags[1] by
// the upper one.  A neighbour's progress in forward e is stamped e * 64 + j:
//   j = 0       "finished forward e-1": its halo planes may be overwritten;
//   j = 1       its boundary input planes are in my x halo;
//   j = i + 2   layer i's boundary planes are in my halo planes of layer i.
// Layer i reads layers < i and the input, so it runs after stamp e*64 + i + 1
// from both neighbours: one one-thread kernel per stage publishes my stamp and
// waits for the neighbours' (the single-device emulation splits the two).  A stamp is stored with st.release.sys after the
// producing kernel in stream order and read with ld.acquire.sys, so the
// producer's peer stores are visible before the consumer's next kernel runs.
// A wait that sees no progress for 60 s traps (a loud CUDA error, never a hang).
constexpr size_t kFlagBytes = 256;

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// One thread: publish stamp `sig` to the neighbours' flags (if sig != 0), then wait
// until my own flags from the present neighbours reach `need` (if need != 0).
__global__ void halo_sync_kernel(unsigned long long* to_lower, unsigned long long* to_upper, unsigned long long sig,
                                 const unsigned long long* flags, int wait_lo, int wait_hi, unsigned long long need) {
    if (threadIdx.x != 0) return;
    if (sig != 0) {
        __threadfence_system();
        if (to_lower != nullptr) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(to_lower), "l"(sig) : "memory");
        if (to_upper != nullptr) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(to_upper), "l"(sig) : "memory");
    }
    if (need == 0) return;
    const unsigned long long t0 = global_ns();
    for (int side = 0; side < 2; ++side) {
        if (!(side == 0 ? wait_lo : wait_hi)) continue;
        while (ld_acquire_sys(flags + side) < need) {
            __nanosleep(100);
            if (global_ns() - t0 > 60ull * 1000000000ull) __trap();
        }
    }
}

// One slab as seen by the P2P schedule: its plan, its workspace and flags.
struct SlabView {
    const SlabPlan* p = nullptr;
    char* base = nullptr;
};

unsigned long long* flags_of(const SlabView& v) {
    return v.base ? reinterpret_cast<unsigned long long*>(v.base + v.p->total) : nullptr;
}

// Signal `sig` to the present neighbours (0: none) and wait for `need` from them (0: none).
tn_status p2p_sync(const SlabView& me, const SlabView& lower, const SlabView& upper, unsigned long long sig,
                   unsigned long long need, cudaStream_t s) {
    const bool hl = lower.base != nullptr, hh = upper.base != nullptr;
    if ((!hl && !hh) || (sig == 0 && need == 0)) return TN_OK;
    halo_sync_kernel<<<1, 32, 0, s>>>(hl ? flags_of(lower) + 1 : nullptr, hh ? flags_of(upper) + 0 : nullptr, sig,
                                      flags_of(me), hl ? 1 : 0, hh ? 1 : 0, need);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_error("halo flags: %s", cudaGetErrorString(e)); return TN_ECUDA; }
    return TN_OK;
}

// Phase "input": own float planes into my extended x buffer; my first plane into
// the lower neighbour's upper x halo, my last into the upper neighbour's lower one.
tn_status p2p_input(const SlabView& me, const SlabView& lower, const SlabView& upper, const float* x_slab,
                    cudaStream_t s) {
    const SlabPlan& sp = *me.p;
    const size_t xp = sp.x_plane;
    const int dz = sp.z1 - sp.z0;
    const char* src = reinterpret_cast<const char*>(x_slab);
    cudaError_t e = cudaMemcpyAsync(me.base + sp.x_off + xp, src, xp * dz, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && lower.base)
        e = cudaMemcpyAsync(lower.base + lower.p->x_off + xp * (lower.p->z1 - lower.p->z0 + 1), src, xp,
                            cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && upper.base)
        e = cudaMemcpyAsync(upper.base + upper.p->x_off, src + xp * (dz - 1), xp, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) { set_error("input planes: %s", cudaGetErrorString(e)); return TN_ECUDA; }
    return TN_OK;
}

// Phase "layer i": the conv with its boundary planes stored into the neighbours.
tn_status p2p_layer(const tn_fcn* net, const SlabView& me, const SlabView& lower, const SlabView& upper, int i,
                    int64_t* d_bad, cudaStream_t s, float* logits, int64_t lstride) {
    const tn_slab_layer& o = me.p->L[i];
    uint32_t* hlo = nullptr;
    uint32_t* hhi = nullptr;
    if ((o.halo & 2) && lower.base) {       // my first plane = the lower neighbour's upper halo
        const tn_slab_layer& lo = lower.p->L[i];
        hlo = reinterpret_cast<uint32_t*>(lower.base + lo.offset + lo.plane_bytes * (lo.z1 - lo.z0 + 1));
    }
    if ((o.halo & 1) && upper.base) hhi = reinterpret_cast<uint32_t*>(upper.base + upper.p->L[i].offset);
    return run_slab_layer(net, *me.p, me.base, i, d_bad, s, logits, lstride, hlo, hhi);
}

}  // namespace

// A rank's slab for the P2P path: workspace and flags allocated here (setup, not the hot
// path) so that one IPC handle maps both; neighbours' workspaces opened from handles.
struct tn_halo {
    SlabPlan me;
    char* ws = nullptr;
    SlabPlan nb[2];
    char* nb_ws[2] = {nullptr, nullptr};
    unsigned long long epoch = 0;
};

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
    cudaError_t e = cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking);
    for (int i = 0; i < kCommEvents && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) {
        set_error("comm stream/events: %s", cudaGetErrorString(e));
        tn_comm_destroy(c);
        return TN_ECUDA;
    }
    *out = c;
    return TN_OK;
}

void tn_comm_destroy(tn_comm* c) {
    if (c == nullptr) return;
    if (c->cs) cudaStreamSynchronize(c->cs);
    for (int i = 0; i < kCommEvents; ++i)
        if (c->ev[i]) cudaEventDestroy(c->ev[i]);
    if (c->cs) cudaStreamDestroy(c->cs);
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
    const int nl = static_cast<int>(net->layers.size());
    if (2 * nl + 2 > kCommEvents) { set_error("too many layers for the comm event pool"); return TN_EUNSUPPORTED; }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    char* base = static_cast<char*>(ws);
    // Overlapped schedule.  Per layer: the interior output planes (which read no halo) are
    // computed on `s` while the comm stream exchanges the previous layers' halos; then `s`
    // waits for the halos of this layer's inputs and computes the two boundary planes; their
    // event starts this layer's exchange (only the sides its consumers read) on the comm
    // stream.  Event pool: ev[2i] = layer i's boundary planes done, ev[2i+1] = layer i's halos
    // in place; ev[2nl] / ev[2nl+1] the same for the float input.
    cudaEvent_t* ev = comm->ev;
    auto check = [](cudaError_t e, const char* what) -> tn_status {
        if (e == cudaSuccess) return TN_OK;
        set_error("%s: %s", what, cudaGetErrorString(e));
        return TN_ECUDA;
    };
    auto post_exchange = [&](cudaEvent_t ready, cudaEvent_t done, char* buf, int64_t pb, int planes,
                             int sides) -> tn_status {
        tn_status st2 = check(cudaEventRecord(ready, s), "event record");
        if (st2 == TN_OK) st2 = check(cudaStreamWaitEvent(comm->cs, ready, 0), "comm wait");
        if (st2 == TN_OK) st2 = exchange_halo(comm, buf, pb, planes, sides, comm->cs);
        if (st2 == TN_OK) st2 = check(cudaEventRecord(done, comm->cs), "event record");
        return st2;
    };
    // own input planes into the extended buffer, then the float halo planes
    cudaError_t e = cudaMemcpyAsync(base + sp.x_off + sp.x_plane, x_slab, sp.x_plane * (z1 - z0),
                                    cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) { set_error("input copy: %s", cudaGetErrorString(e)); return TN_ECUDA; }
    if (sp.x_halo) {
        st = post_exchange(ev[2 * nl], ev[2 * nl + 1], base + sp.x_off, static_cast<int64_t>(sp.x_plane), z1 - z0 + 2,
                           sp.x_halo);
        if (st != TN_OK) return st;
    }
    const int64_t lstride = static_cast<int64_t>(z1 - z0) * global.h * global.w;
    for (int i = 0; i < nl; ++i) {
        const tn_layer& ly = net->layers[i];
        const tn_slab_layer& o = sp.L[i];
        const int dz = o.z1 - o.z0;
        // interior planes [1, dz - 1): no halo reads
        if (dz > 2) {
            st = run_slab_layer(net, sp, base, i, d_bad, s, logits_slab, lstride, nullptr, nullptr, 1, dz - 1);
            if (st != TN_OK) return st;
        }
        // the halos this layer's boundary planes read
        if (ly.kind == TN_LAYER_FIRST) {
            if (sp.x_halo && (st = check(cudaStreamWaitEvent(s, ev[2 * nl + 1], 0), "halo wait")) != TN_OK) return st;
        } else {
            for (int sgi = 0; sgi < ly.nseg; ++sgi)
                if ((st = check(cudaStreamWaitEvent(s, ev[2 * ly.src[sgi] + 1], 0), "halo wait")) != TN_OK) return st;
        }
        st = run_slab_layer(net, sp, base, i, d_bad, s, logits_slab, lstride, nullptr, nullptr, 0, 1);
        if (st == TN_OK && dz > 1)
            st = run_slab_layer(net, sp, base, i, d_bad, s, logits_slab, lstride, nullptr, nullptr, dz - 1, dz);
        if (st != TN_OK) return st;
        if (o.halo) {
            st = post_exchange(ev[2 * i], ev[2 * i + 1], base + o.offset, o.plane_bytes, dz + 2, o.halo);
            if (st != TN_OK) return st;
        }
    }
    // the caller's stream ends after every exchange this forward posted (workspace reuse)
    for (int i = 0; i < nl; ++i)
        if (sp.L[i].halo && (st = check(cudaStreamWaitEvent(s, ev[2 * i + 1], 0), "halo wait")) != TN_OK) return st;
    return TN_OK;
}

size_t tn_fcn_slabs_local_workspace_bytes(const tn_fcn* net, tn_dims global, int32_t nslabs) {
    if (net == nullptr || nslabs < 1 || global.d % nslabs) return 0;
    size_t tot = 0;
    const int dz = global.d / nslabs;
    for (int r = 0; r < nslabs; ++r) {
        const size_t b = tn_fcn_slab_workspace_bytes(net, global, r * dz, (r + 1) * dz);
        if (b == 0) return 0;
        tot += align_up(b + kFlagBytes);
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
        p += align_up(P[r].total + kFlagBytes);
    }
    auto copy = [&](char* dst, const char* src, size_t n) -> tn_status {
        cudaError_t e = cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) { set_error("halo copy: %s", cudaGetErrorString(e)); return TN_ECUDA; }
        return TN_OK;
    };
    // halo exchange of one buffer kind across all slabs (device copies)
    // (only the halo sides the consumers read: bit 0 lower, bit 1 upper)
    auto exchange_all = [&](auto offset_of, auto plane_of, auto planes_of, int sides) -> tn_status {
        for (int r = 0; r < nslabs; ++r) {
            const size_t pb = plane_of(r);
            char* mine = B[r] + offset_of(r);
            const int np = planes_of(r);
            if (r > 0 && (sides & 1)) {
                char* lower = B[r - 1] + offset_of(r - 1);
                tn_status st = copy(mine, lower + pb * (planes_of(r - 1) - 2), pb);
                if (st != TN_OK) return st;
            }
            if (r + 1 < nslabs && (sides & 2)) {
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
    // The overlapped schedule of tn_fcn_forward_slab, layer-major across the slabs on one
    // stream: every slab's interior planes of layer i run BEFORE the halos of layer i - 1 are
    // copied in (the copies stand for the exchange in flight), then the boundary planes; so
    // an interior plane that read a halo would see stale data and break bit-identity.
    const int nl = static_cast<int>(net->layers.size());
    const int64_t cstride = static_cast<int64_t>(global.d) * global.h * global.w;
    int pending = -1;                                  // layer whose halo copies are outstanding (-1: input)
    tn_status st = TN_OK;
    auto flush = [&]() -> tn_status {
        tn_status s2 = TN_OK;
        if (pending < 0) {
            if (P[0].x_halo)
                s2 = exchange_all([&](int r) { return P[r].x_off; }, [&](int) { return xplane; },
                                  [&](int) { return dz + 2; }, P[0].x_halo);
        } else if (P[0].L[pending].halo) {
            const int i = pending;
            s2 = exchange_all([&](int r) { return static_cast<size_t>(P[r].L[i].offset); },
                              [&](int r) { return static_cast<size_t>(P[r].L[i].plane_bytes); },
                              [&](int r) { return P[r].L[i].z1 - P[r].L[i].z0 + 2; }, P[0].L[i].halo);
        }
        return s2;
    };
    for (int i = 0; i < nl && st == TN_OK; ++i) {
        const int ldz = P[0].L[i].z1 - P[0].L[i].z0;
        for (int r = 0; r < nslabs && st == TN_OK && ldz > 2; ++r) {
            float* lg = logits + static_cast<int64_t>(P[r].L.back().z0) * global.h * global.w;
            st = run_slab_layer(net, P[r], B[r], i, d_bad, s, lg, cstride, nullptr, nullptr, 1, ldz - 1);
        }
        if (st == TN_OK) st = flush();
        for (int r = 0; r < nslabs && st == TN_OK; ++r) {
            float* lg = logits + static_cast<int64_t>(P[r].L.back().z0) * global.h * global.w;
            st = run_slab_layer(net, P[r], B[r], i, d_bad, s, lg, cstride, nullptr, nullptr, 0, 1);
            if (st == TN_OK && ldz > 1)
                st = run_slab_layer(net, P[r], B[r], i, d_bad, s, lg, cstride, nullptr, nullptr, ldz - 1, ldz);
        }
        pending = i;
    }
    if (st == TN_OK) st = flush();
    return st;
}

tn_status tn_fcn_forward_slabs_local_p2p(const tn_fcn* net, const float* x, tn_dims global, int32_t nslabs,
                                         float* logits, void* ws, size_t ws_bytes, int64_t* d_bad, tn_stream stream) {
    if (net == nullptr || x == nullptr || logits == nullptr || ws == nullptr) { set_error("NULL argument"); return TN_EINVAL; }
    if (nslabs < 1 || global.d % nslabs) { set_error("nslabs must divide the depth"); return TN_ESHAPE; }
    const size_t need = tn_fcn_slabs_local_workspace_bytes(net, global, nslabs);
    if (need == 0) return TN_ESHAPE;
    if (ws_bytes < need) { set_error("workspace too small: need %zu", need); return TN_EINVAL; }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int dz = global.d / nslabs;
    std::vector<SlabPlan> P(nslabs);
    std::vector<SlabView> V(nslabs + 2);          // V[r + 1] = slab r; V[0], V[nslabs + 1] = none
    char* p = static_cast<char*>(ws);
    for (int r = 0; r < nslabs; ++r) {
        tn_status st = make_slab_plan(net, global, r * dz, (r + 1) * dz, P[r]);
        if (st != TN_OK) return st;
        V[r + 1].p = &P[r];
        V[r + 1].base = p;
        p += align_up(P[r].total + kFlagBytes);
    }
    // stateless: the flags restart at epoch 1 every call (all slabs share this stream)
    for (int r = 0; r < nslabs; ++r) {
        cudaError_t e = cudaMemsetAsync(flags_of(V[r + 1]), 0, 2 * sizeof(unsigned long long), s);
        if (e != cudaSuccess) { set_error("flag reset: %s", cudaGetErrorString(e)); return TN_ECUDA; }
    }
    const unsigned long long E = 64;
    const int nl = static_cast<int>(net->layers.size());
    tn_status st = TN_OK;
    // the same phases as tn_fcn_forward_slab_p2p, interleaved layer-major across the slabs
    // (one stream: every slab signals a stage before any slab waits for it)
    for (int r = 1; r <= nslabs && st == TN_OK; ++r) st = p2p_sync(V[r], V[r - 1], V[r + 1], E + 0, 0, s);
    for (int r = 1; r <= nslabs && st == TN_OK; ++r) {
        st = p2p_sync(V[r], V[r - 1], V[r + 1], 0, E + 0, s);
        if (st == TN_OK)
            st = p2p_input(V[r], V[r - 1], V[r + 1], x + static_cast<int64_t>(r - 1) * dz * global.h * global.w, s);
        if (st == TN_OK) st = p2p_sync(V[r], V[r - 1], V[r + 1], E + 1, 0, s);
    }
    const int64_t cstride = static_cast<int64_t>(global.d) * global.h * global.w;
    for (int i = 0; i < nl && st == TN_OK; ++i) {
        for (int r = 1; r <= nslabs && st == TN_OK; ++r) {
            st = p2p_sync(V[r], V[r - 1], V[r + 1], 0, E + i + 1, s);
            float* lg = logits + static_cast<int64_t>(P[r - 1].L.back().z0) * global.h * global.w;
            if (st == TN_OK) st = p2p_layer(net, V[r], V[r - 1], V[r + 1], i, d_bad, s, lg, cstride);
            if (st == TN_OK && P[r - 1].L[i].halo) st = p2p_sync(V[r], V[r - 1], V[r + 1], E + i + 2, 0, s);
        }
    }
    return st;
}

tn_status tn_halo_create(const tn_fcn* net, tn_dims global, int32_t z0, int32_t z1, tn_halo** out) {
    if (net == nullptr || out == nullptr) { set_error("net/out is NULL"); return TN_EINVAL; }
    *out = nullptr;
    tn_halo* h = new (std::nothrow) tn_halo();
    if (h == nullptr) { set_error("out of host memory"); return TN_EINVAL; }
    tn_status st = make_slab_plan(net, global, z0, z1, h->me);
    if (st != TN_OK) { delete h; return st; }
    cudaError_t e = cudaMalloc(&h->ws, h->me.total + kFlagBytes);
    if (e == cudaSuccess) e = cudaMemset(h->ws + h->me.total, 0, kFlagBytes);
    if (e != cudaSuccess) {
        set_error("halo workspace: %s", cudaGetErrorString(e));
        if (h->ws) cudaFree(h->ws);
        delete h;
        return TN_ECUDA;
    }
    *out = h;
    return TN_OK;
}

tn_status tn_halo_export(const tn_halo* h, void* handle_out) {
    if (h == nullptr || handle_out == nullptr) { set_error("halo/handle is NULL"); return TN_EINVAL; }
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
    cudaIpcMemHandle_t m;
    cudaError_t e = cudaIpcGetMemHandle(&m, h->ws);
    if (e != cudaSuccess) { set_error("cudaIpcGetMemHandle: %s", cudaGetErrorString(e)); return TN_ECUDA; }
    memcpy(handle_out, &m, sizeof(m));
    return TN_OK;
}

tn_status tn_halo_connect(tn_halo* h, const tn_fcn* net, tn_dims global, const void* lower_handle, int32_t lower_z0,
                          const void* upper_handle, int32_t upper_z1) {
    if (h == nullptr || net == nullptr) { set_error("halo/net is NULL"); return TN_EINVAL; }
    if (h->nb_ws[0] || h->nb_ws[1]) { set_error("already connected"); return TN_EINVAL; }
    const void* hd[2] = {lower_handle, upper_handle};
    const int zr[2][2] = {{lower_z0, h->me.z0}, {h->me.z1, upper_z1}};
    for (int side = 0; side < 2; ++side) {
        if (hd[side] == nullptr) continue;
        tn_status st = make_slab_plan(net, global, zr[side][0], zr[side][1], h->nb[side]);
        if (st != TN_OK) return st;
        cudaIpcMemHandle_t m;
        memcpy(&m, hd[side], sizeof(m));
        void* ptr = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&ptr, m, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) { set_error("cudaIpcOpenMemHandle: %s", cudaGetErrorString(e)); return TN_ECUDA; }
        h->nb_ws[side] = static_cast<char*>(ptr);
    }
    return TN_OK;
}

size_t tn_halo_workspace_bytes(const tn_halo* h) { return h ? h->me.total + kFlagBytes : 0; }

tn_status tn_fcn_forward_slab_p2p(const tn_fcn* net, tn_halo* h, const float* x_slab, float* logits_slab,
                                  int64_t* d_bad, tn_stream stream) {
    if (net == nullptr || h == nullptr) { set_error("net/halo is NULL"); return TN_EINVAL; }
    if (x_slab == nullptr || logits_slab == nullptr) { set_error("x/logits NULL"); return TN_EINVAL; }
    if ((reinterpret_cast<uintptr_t>(x_slab) | reinterpret_cast<uintptr_t>(logits_slab)) & 15u) {
        set_error("pointers must be 16-byte aligned");
        return TN_EALIGN;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    SlabView me, lo, up;
    me.p = &h->me; me.base = h->ws;
    if (h->nb_ws[0]) { lo.p = &h->nb[0]; lo.base = h->nb_ws[0]; }
    if (h->nb_ws[1]) { up.p = &h->nb[1]; up.base = h->nb_ws[1]; }
    const unsigned long long E = 64ull * ++h->epoch;
    // one flag kernel per stage: publish my progress, then wait for the neighbours' same stage
    tn_status st = p2p_sync(me, lo, up, E + 0, E + 0, s);
    if (st == TN_OK) st = p2p_input(me, lo, up, x_slab, s);
    if (st == TN_OK) st = p2p_sync(me, lo, up, E + 1, E + 1, s);
    const int64_t lstride = static_cast<int64_t>(h->me.z1 - h->me.z0) * h->me.g.h * h->me.g.w;
    const int nl = static_cast<int>(net->layers.size());
    for (int i = 0; i < nl && st == TN_OK; ++i) {
        st = p2p_layer(net, me, lo, up, i, d_bad, s, logits_slab, lstride);
        if (st == TN_OK && h->me.L[i].halo) st = p2p_sync(me, lo, up, E + i + 2, E + i + 2, s);
    }
    return st;
}

void tn_halo_destroy(tn_halo* h) {
    if (h == nullptr) return;
    for (int side = 0; side < 2; ++side)
        if (h->nb_ws[side]) cudaIpcCloseMemHandle(h->nb_ws[side]);
    if (h->ws) cudaFree(h->ws);
    delete h;
}

}  // extern "C"
