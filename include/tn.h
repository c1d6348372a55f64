/*
 * tn.h -- C ABI of libtn.so, the B200 (sm_100a) TernaryNet inference hot path.
 *
 * The calls follow the paper's statement of the problem (Heinrich, Blendowski,
 * Oktay, "TernaryNet", arXiv 1801.09449; cited PAPER.md:<line>):
 *   pack ternary tensors into sign / nonzero-mask bitplanes (PAPER.md:118 and
 *   Fig. 3, :130), convolve them with ternary 3x3x3 filter banks where every
 *   inner product is Eq. 9's masked Hamming distance,
 *   requantise the int32 result to ternary with per-channel integer thresholds
 *   that fold alpha, batch norm and Eq. 6 (PAPER.md:91-95, :130,
 *   :135), chain these blocks into a U-Net-style FCN with skip concatenation and
 *   x2 up/down-sampling (Table 1), and finish with a float
 *   prediction layer.
 *
 * Conventions (readings R1-R16):
 *  - Every pointer is a DEVICE pointer unless documented "host".  Every call is
 *    asynchronous and stream-ordered on `stream` (a cudaStream_t; NULL = the
 *    legacy default stream).  The caller allocates and owns all memory; the
 *    library never allocates on the hot path (tn_fcn_create / tn_comm_init are
 *    setup calls).
 *  - Ternary codes: int8 in {-1, 0, +1}, logical layout NCDHW (PyTorch order).
 *  - Packed ternary tensor (reading R3): uint32 [n][d][h][w][2][cw],
 *    cw = ceil(c/32).  Per voxel the cw SIGN words come first (bit = 1 <=> +1),
 *    then the cw MASK words (bit = 1 <=> nonzero; reading R2).  Channel ch is
 *    bit (ch % 32) of word (ch / 32), LSB first.  Zero = (sign 0, mask 0);
 *    padding lanes are 0.  Byte size: tn_packed_bytes().
 *  - Packed weights: uint32 [k][27][2][cw] from int8 [k][c][3][3][3]; tap
 *    t = (dz*3 + dy)*3 + dx.
 *  - Convolutions are 3x3x3 cross-correlations with zero padding (PyTorch
 *    semantics).  Output extent per axis: (len + 2*pad - 2*dil - 1)/stride + 1.
 *  - Requantisation (reading R5): t = +1 if acc >= hi[k]; else -1 if
 *    acc <= lo[k]; else 0.
 *  - 16-byte alignment is required for every tensor pointer (128-bit I/O).
 *  - Programmatic dependent launch: the tensor-core convs start their prologue
 *    (filter bank, thresholds, prediction weights) while the previous kernel on
 *    the stream is still finishing, and wait for it (griddepcontrol.wait) only
 *    before reading activations.  So filter banks, thresholds and prediction
 *    weights must not be written by the kernel launched IMMEDIATELY before a conv
 *    (a copy, or any earlier kernel, is fine).  tn_pack_weights ends with an
 *    empty kernel so that packing and then convolving right away is safe.
 *
 * Errors: host-detectable errors return before any work is queued, with text in
 * tn_last_error().  Device-detected domain errors (a code outside {-1,0,1}, a
 * NaN/Inf float, a non-canonical packed word) are reported through the caller's
 * int64 *d_bad: the caller initialises it to INT64_MAX (tn_bad_init() queues
 * that), the kernel atomicMin()s the first offending flat NCDHW index into it;
 * outputs are unspecified when *d_bad != INT64_MAX after the stream syncs
 * ("domain error naming the offending index").  d_bad may be NULL
 * (no reporting).  CUDA / NCCL failures return TN_ECUDA / TN_ENCCL.  The
 * library never aborts and never throws across this ABI.
 */
#ifndef TN_H_
#define TN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* tn_stream; /* == cudaStream_t */

typedef enum {
    TN_OK = 0,
    TN_EINVAL = 1,        /* null pointer, bad enum, k/c < 1, ... */
    TN_ESHAPE = 2,        /* inconsistent or unsupported extents */
    TN_EALIGN = 3,        /* pointer not 16-byte aligned */
    TN_EUNSUPPORTED = 4,  /* valid request this build does not implement */
    TN_EDOMAIN = 5,       /* reserved (domain errors are reported via d_bad) */
    TN_ECUDA = 6,
    TN_ENCCL = 7
} tn_status;

typedef struct { int32_t n, c, d, h, w; } tn_dims;              /* logical NCDHW            */
typedef struct { int32_t stride[3], pad[3], dil[3]; } tn_geom;  /* z, y, x; kernel 3x3x3    */

/* ---- sizes and helpers (host) ------------------------------------------- */
size_t      tn_packed_bytes(tn_dims x);                /* n*d*h*w * 2*ceil(c/32) * 4   */
size_t      tn_weight_bytes(int32_t k, int32_t c);     /* k * 27 * 2*ceil(c/32) * 4    */
/* Output dims of a conv of x with k filters; TN_ESHAPE if an extent is < 1.        */
tn_status   tn_conv_out_dims(tn_dims x, int32_t k, tn_geom g, tn_dims* out /*host*/);
const char* tn_last_error(void);                       /* thread-local text            */
const char* tn_version(void);
/* Queue *d_bad = INT64_MAX on stream. */
tn_status   tn_bad_init(int64_t* d_bad, tn_stream stream);

/* ---- A1: ternarise and pack (Eq. 6) --- */
/* x int8 NCDHW codes -> xp packed.  Domain: code not in {-1,0,1}.            */
tn_status tn_pack_i8(const int8_t* x, tn_dims xd, uint32_t* xp, int64_t* d_bad, tn_stream stream);
/* x int32 NCDHW codes -> xp packed.  Domain: code not in {-1,0,1}.           */
tn_status tn_pack_i32(const int32_t* x, tn_dims xd, uint32_t* xp, int64_t* d_bad, tn_stream stream);
/* x float NCDHW -> Eq. 6 with folded normalisation (reading R7):
 * +1 if x > t_hi, -1 if x < t_lo, else 0.  Domain: NaN / Inf.  Needs t_lo <= t_hi. */
tn_status tn_pack_f32(const float* x, tn_dims xd, float t_lo, float t_hi, uint32_t* xp,
                      int64_t* d_bad, tn_stream stream);
/* w int8 [k][c][3][3][3] -> wp [k][27][2][cw].  Domain: code not in {-1,0,1}. */
tn_status tn_pack_weights(const int8_t* w, int32_t k, int32_t c, uint32_t* wp, int64_t* d_bad,
                          tn_stream stream);
/* xp packed -> x int8 NCDHW.  Domain: sign bit on a zero, or a padding lane set
 * (reported at the voxel's channel c-1 index).                               */
tn_status tn_unpack(const uint32_t* xp, tn_dims xd, int8_t* x, int64_t* d_bad, tn_stream stream);

/* ---- A2/A3/A5: ternary conv3d, Eq. 9 (dilation :135) ---- */
/* y int32 channel-last [n][do][ho][wo][k] (reading R14).                     */
tn_status tn_conv3d(const uint32_t* xp, tn_dims xd, const uint32_t* wp, int32_t k, tn_geom g,
                    int32_t* y, tn_stream stream);
/* A4 fused: yp packed [n][do][ho][wo][2][ceil(k/32)]; lo, hi int32 [k].      */
tn_status tn_conv3d_requant(const uint32_t* xp, tn_dims xd, const uint32_t* wp, int32_t k,
                            tn_geom g, const int32_t* lo, const int32_t* hi, uint32_t* yp,
                            tn_stream stream);
/* A4 standalone: y int32 channel-last [n][d][h][w][k] (yd.c == k) -> yp packed. */
tn_status tn_requant(const int32_t* y, tn_dims yd, const int32_t* lo, const int32_t* hi,
                     uint32_t* yp, tn_stream stream);

/* ---- A6: conv over [upsample_x2(a) | b] concatenation */
/* A convolution whose input is the channel concatenation of nseg (1 or 2)
 * packed segments, each optionally nearest-x2 upsampled (reading R10).  The
 * conv-input extents are the segments' common extents after upsampling.  The
 * conv is the sum of per-segment convs with the segment's slice of the filter
 * bank (channel order = segment order).  Exactly one of y (int32 channel-last)
 * or yp (packed, needs lo/hi) must be non-NULL.  All segments must have the
 * same ceil(c/32) in this build (TN_EUNSUPPORTED otherwise).                 */
typedef struct {
    const uint32_t* xp;   /* packed segment; if upsample, at LOW resolution      */
    tn_dims d;            /* its dims (low-resolution dims if upsample)          */
    int32_t upsample;     /* 0 = none, 1 = nearest x2 in z, y and x, 2 = nearest x2
                             in y and x only (the 2D decoders of Table 1, reading R18) */
    const uint32_t* wp;   /* packed weights of this segment [k][27][2][ceil(d.c/32)] */
} tn_segment;
tn_status tn_conv3d_seg(const tn_segment* segs /*host array*/, int32_t nseg, int32_t k,
                        tn_geom g, const int32_t* lo, const int32_t* hi, int32_t* y,
                        uint32_t* yp, tn_stream stream);

/* ---- Prepared filter banks (tensor-core kernel) --------------------------- */
/* The tensor-core conv kernel expands the packed filter bank into its UMMA B
 * operand image (Eq. 9's w as int8 or FP4 codes) in every
 * CTA of every launch.  tn_conv_prepare builds that image once, in device
 * memory, for a conv of these segments / k / g (requant != 0: the packed-output
 * form; 0: int32 output); the *_prepared calls then copy it instead.
 *   segs[i].xp may be NULL here (only d, upsample and wp are read); the spatial
 *   extents only steer the plan, the image is the same for any extents.
 *   The image is a COPY of the bank at prepare time and is tied to the wp
 *   pointers: after changing a bank's contents in place, prepare again.  A
 *   prepared call whose kernel plan differs from the prepared one (other wp
 *   pointers, segment widths, k, stride, dilation, kernel selector) is still
 *   correct: it stages the bank as the unprepared call does.
 *   *out receives a handle (also when the shape has no tensor-core plan:
 *   tn_conv_prep_bytes is then 0); the call synchronises `stream`.
 *   Errors: TN_EINVAL (NULL out/segs, bad k/nseg), TN_ESHAPE, TN_ECUDA.     */
typedef struct tn_conv_prep tn_conv_prep;
tn_status tn_conv_prepare(const tn_segment* segs /*host array*/, int32_t nseg, int32_t k, tn_geom g,
                          int32_t requant, tn_conv_prep** out, tn_stream stream);
int64_t   tn_conv_prep_bytes(const tn_conv_prep* p);   /* device bytes held (0: no image) */
void      tn_conv_prep_destroy(tn_conv_prep* p);        /* NULL is a no-op; not stream-ordered:
                                                           no launch using p may be pending */
/* Same arguments and results as tn_conv3d_requant / tn_conv3d_seg, plus p
 * (NULL = the unprepared call).                                              */
tn_status tn_conv3d_requant_prepared(const tn_conv_prep* p, const uint32_t* xp, tn_dims xd,
                                     const uint32_t* wp, int32_t k, tn_geom g, const int32_t* lo,
                                     const int32_t* hi, uint32_t* yp, tn_stream stream);
tn_status tn_conv3d_seg_prepared(const tn_conv_prep* p, const tn_segment* segs, int32_t nseg,
                                 int32_t k, tn_geom g, const int32_t* lo, const int32_t* hi,
                                 int32_t* y, uint32_t* yp, tn_stream stream);

/* ---- A7: first layer -- Eq. 6 on the float input fused with a conv from 1
 * channel and the requant epilogue (reading R7).
 * x float [n][1][d][h][w]; wp packed [k][27][2][1]; yp packed.  Domain: NaN/Inf. */
tn_status tn_conv3d_first(const float* x, tn_dims xd, float t_lo, float t_hi, const uint32_t* wp,
                          int32_t k, tn_geom g, const int32_t* lo, const int32_t* hi,
                          uint32_t* yp, int64_t* d_bad, tn_stream stream);

/* ---- A8: prediction, 1x1x1 float conv (reading R12) --- */
/* tp packed [n][d][h][w][2][ceil(td.c/32)] (td.c <= 64); w float [nclass][td.c];
 * b float [nclass]; logits float NCDHW [n][nclass][d][h][w].  Sum order: b, then
 * channel quads ascending, fp32.                                              */
tn_status tn_predict(const uint32_t* tp, tn_dims td, const float* w, const float* b,
                     int32_t nclass, float* logits, tn_stream stream);

/* ---- A9: the ternary FCN (Table 1 analogue, reading R9) ------------------- */
/* A layer table entry.  Layers run in table order; src[] refers to earlier
 * entries (or -1 = the network input, which requires kind TN_LAYER_FIRST).    */
enum { TN_LAYER_FIRST = 1, TN_LAYER_CONV = 2 };
typedef struct {
    int32_t kind;            /* TN_LAYER_FIRST (float input, 1 channel) or TN_LAYER_CONV */
    int32_t c_out;
    int32_t stride;          /* 1 or 2 in all three axes; pad = dil               */
    int32_t dil;             /* >= 1                                              */
    int32_t nseg;            /* 1 or 2 input segments (concatenated in this order) */
    int32_t src[2];          /* producing layer index, or -1 for the input        */
    int32_t upsample[2];     /* nearest x2 of that segment (0 / 1 / 2 as in tn_segment) */
    const uint32_t* wp[2];   /* packed weights per segment (borrowed)             */
    const int32_t* lo;       /* [c_out] (borrowed)                                */
    const int32_t* hi;       /* [c_out] (borrowed)                                */
} tn_layer;
typedef struct tn_fcn tn_fcn;
/* layers: host array, copied.  pred_w [nclass][c_out of the last layer] and
 * pred_b [nclass] are device pointers (borrowed).  t_lo/t_hi: Eq. 6 input band.
 * The input may have c >= 1 float channels (e.g. Table 1's 15-slice stacks,
 * reading R18): layer 0's packed weights are then [c_out][27][2][ceil(c/32)]; with
 * c == 1 layer 0 is the fused A7 kernel (c_out <= 32), with c > 1 the input is
 * ternarised and packed first (tn_pack_f32's kernel) and layer 0 is a regular conv.
 * The last layer has c_out <= 64 (the prediction's input).                     */
tn_status tn_fcn_create(const tn_layer* layers, int32_t n_layers, float t_lo, float t_hi,
                        const float* pred_w, const float* pred_b, int32_t nclass, tn_fcn** out);
size_t    tn_fcn_workspace_bytes(const tn_fcn* net, tn_dims xd);
/* x float [n][c][d][h][w] -> logits float [n][nclass][d][h][w]. */
tn_status tn_fcn_forward(const tn_fcn* net, const float* x, tn_dims xd, float* logits, void* ws,
                         size_t ws_bytes, int64_t* d_bad, tn_stream stream);
void      tn_fcn_destroy(tn_fcn* net);   /* also frees the images of tn_fcn_prepare */
/* Optional: build every tensor-core layer's filter-bank image (tn_conv_prepare)
 * for inputs of dims xd under the current kernel selector, replacing earlier
 * ones; later forwards (tn_fcn_forward*, slab variants) copy them instead of
 * expanding the banks in every CTA.  Forwards of other extents or selectors stay
 * correct (a layer whose plan differs stages its bank).  Synchronises stream;
 * not stream-ordered against pending forwards of net.  The images are copies of
 * the banks at prepare time: prepare again after changing weights in place.
 * Errors: TN_EINVAL (NULL net), TN_ESHAPE (xd), TN_ECUDA.                     */
tn_status tn_fcn_prepare(tn_fcn* net, tn_dims xd, tn_stream stream);
size_t    tn_fcn_prep_bytes(const tn_fcn* net);   /* device bytes the images hold */
/* The layers [first, last) of tn_fcn_forward only (last = -1: to the end; the
 * prediction runs with the last layer), reading earlier layers' outputs from ws.
 * Calling it for consecutive ranges on one stream is tn_fcn_forward; used to time
 * layers individually.  TN_EINVAL if the range is outside the table.          */
tn_status tn_fcn_forward_range(const tn_fcn* net, const float* x, tn_dims xd, float* logits, void* ws,
                               size_t ws_bytes, int64_t* d_bad, int32_t first, int32_t last,
                               tn_stream stream);

/* Internal-activation access for debugging and per-layer parity: after a
 * tn_fcn_forward on the same ws, returns the device pointer and dims of layer
 * i's packed output inside ws (NULL if out of range).  The LAST layer's codes
 * are only written when the prediction is not fused into its epilogue (the
 * CUDA-core fallback); the tensor-core kernels produce its logits only.       */
const uint32_t* tn_fcn_layer_output(const tn_fcn* net, tn_dims xd, const void* ws, int32_t i,
                                    tn_dims* out_dims /*host*/);

/* ---- Multi-GPU: z-slab decomposition of one volume (BASELINE configs[4]) ----
 * Rank r of nranks owns input planes [z0, z1) (multiples of the FCN's total
 * downsampling, 8 for the Table-1 analogue; ranks in z order).  Every layer's
 * packed output is kept with one halo plane per side, exchanged after the
 * layer with ranks r-1 / r+1 by NCCL send/recv on `stream` (NVLink through
 * NVSwitch); planes outside the volume are never read (zero padding).  Results
 * are bit-identical to tn_fcn_forward on the whole volume.  n must be 1.     */
typedef struct tn_comm tn_comm;
tn_status tn_comm_unique_id(void* id_out /*host, 128 bytes (ncclUniqueId)*/);
tn_status tn_comm_init(const void* nccl_unique_id /*host, 128 B*/, int32_t rank, int32_t nranks,
                       tn_comm** out);
void      tn_comm_destroy(tn_comm* comm);
/* Per-layer slab geometry (host planner; also used by the CPU tests). */
typedef struct {
    int32_t level_scale;    /* global depth / layer depth (1, 2, 4, 8)            */
    int32_t c, h, w, gd;    /* channels, in-plane extents, global depth of layer   */
    int32_t z0, z1;         /* owned planes at this layer's resolution             */
    int32_t halo;           /* 1 if the layer's halo planes are exchanged          */
    int64_t plane_bytes;    /* packed bytes per plane                              */
    int64_t offset;         /* byte offset of the buffer [z0-1, z1+1) in ws        */
} tn_slab_layer;
tn_status tn_fcn_slab_plan(const tn_fcn* net, tn_dims global, int32_t z0, int32_t z1,
                           tn_slab_layer* out /*host, n_layers or NULL*/, int32_t max_layers,
                           size_t* ws_bytes /*host, may be NULL*/);
size_t    tn_fcn_slab_workspace_bytes(const tn_fcn* net, tn_dims global, int32_t z0, int32_t z1);
/* x_slab float [1][1][z1-z0][h][w] (own planes); logits_slab float
 * [1][nclass][z1-z0][h][w].                                                    */
tn_status tn_fcn_forward_slab(const tn_fcn* net, tn_comm* comm, const float* x_slab, tn_dims global,
                              int32_t z0, int32_t z1, float* logits_slab, void* ws, size_t ws_bytes,
                              int64_t* d_bad, tn_stream stream);
/* Single-device emulation: all nslabs slabs of one volume on this GPU, layer by
 * layer, halos exchanged by device copies (same kernels, offsets and schedule
 * as tn_fcn_forward_slab).  x / logits as in tn_fcn_forward.                  */
size_t    tn_fcn_slabs_local_workspace_bytes(const tn_fcn* net, tn_dims global, int32_t nslabs);
tn_status tn_fcn_forward_slabs_local(const tn_fcn* net, const float* x, tn_dims global, int32_t nslabs,
                                     float* logits, void* ws, size_t ws_bytes, int64_t* d_bad,
                                     tn_stream stream);

/* ---- NEXT-1: epilogue-fused halos over NVLink P2P, no NCCL -----
 * The same z-slab decomposition, but each layer's fused requant epilogue also
 * stores its first / last owned output plane straight into the lower / upper
 * neighbour's halo plane (peer memory opened with CUDA IPC, NVLink through
 * NVSwitch), and a device progress flag replaces each send/recv pair: after
 * layer i, one thread of a one-CTA kernel stores stamp 64*epoch + i + 2 with
 * st.release.sys into both neighbours' flags and then waits (ld.acquire.sys)
 * for the same stamp from both neighbours before layer i + 1 runs (stamp
 * 64*epoch + 0 = "done with the previous forward", so halos are never
 * overwritten while still read; + 1 = input planes delivered).  A wait that sees no progress for 60 s traps
 * (a CUDA error on the caller's stream, never a silent hang).  Results are
 * bit-identical to tn_fcn_forward.  Setup calls allocate; the forward does not.
 *   tn_halo_create   plans rank's slab [z0, z1) and cudaMallocs its workspace
 *                    + flags (tn_halo_workspace_bytes);
 *   tn_halo_export   writes the 64-byte cudaIpcMemHandle of that workspace;
 *   tn_halo_connect  opens the neighbours' handles (NULL at the volume ends);
 *                    the lower neighbour owns [lower_z0, z0), the upper one
 *                    [z1, upper_z1); all ranks must use the same net and global;
 *   tn_fcn_forward_slab_p2p  one forward of the slab (x_slab / logits_slab as
 *                    in tn_fcn_forward_slab), every rank once per forward;
 *   tn_fcn_forward_slabs_local_p2p  all slabs on this device, layer-major, with
 *                    the same epilogue stores and flags (single-GPU check of the
 *                    schedule; workspace = tn_fcn_slabs_local_workspace_bytes). */
typedef struct tn_halo tn_halo;
tn_status tn_halo_create(const tn_fcn* net, tn_dims global, int32_t z0, int32_t z1, tn_halo** out);
size_t    tn_halo_workspace_bytes(const tn_halo* h);
tn_status tn_halo_export(const tn_halo* h, void* handle_out /*host, 64 bytes*/);
tn_status tn_halo_connect(tn_halo* h, const tn_fcn* net, tn_dims global,
                          const void* lower_handle /*host 64 B or NULL*/, int32_t lower_z0,
                          const void* upper_handle /*host 64 B or NULL*/, int32_t upper_z1);
tn_status tn_fcn_forward_slab_p2p(const tn_fcn* net, tn_halo* h, const float* x_slab, float* logits_slab,
                                  int64_t* d_bad, tn_stream stream);
tn_status tn_fcn_forward_slabs_local_p2p(const tn_fcn* net, const float* x, tn_dims global, int32_t nslabs,
                                         float* logits, void* ws, size_t ws_bytes, int64_t* d_bad,
                                         tn_stream stream);
void      tn_halo_destroy(tn_halo* h);

/* ---- Model preparation (host, not on the hot path) ---------
 * tn_ternarize_weights: Eq. 4 per output filter f of a float
 * filter bank w[k][n] (host, row-major; n = C_in * 27): Delta = 0.7/n sum|W_i|,
 * code +1 if W_i > Delta, 0 if |W_i| <= Delta, -1 else; alpha[f] = mean |W_i|
 * over the nonzero codes (0 if none).  sparsity in [0, 1) instead fixes the
 * zeros per filter: exactly ceil(sparsity * n) zeros at the
 * smallest |W_i| (stable by index), the rest sign(W_i); sparsity < 0 selects
 * Eq. 4.  Double precision.  codes[k][n] int8 and alpha[k] are host buffers.
 * TN_EDOMAIN on a non-finite weight (*bad_index = its flat index) or
 * sparsity >= 1; TN_EINVAL on NULL / empty arguments.
 * tn_fold_thresholds: per channel the conv output alpha * acc goes through
 * batch norm y = gamma * (alpha*acc - mean) / sqrt(var + eps) + beta and Eq. 6
 * (+1 if y > 0.5, -1 if y < -0.5, 0 else).  With
 * a = gamma*alpha/sqrt(var+eps), b = beta - gamma*mean/sqrt(var+eps) (double,
 * y = a*acc + b evaluated without FMA), the integer rule the epilogues apply
 * (+1 if acc >= hi; else -1 if acc <= lo; else 0) reproduces tern(y) for every
 * acc in [-max_abs_acc, max_abs_acc] (27 * C_in bounds |acc|).  If a < 0,
 * negate[c] = 1 and the thresholds are for the negated filter (the caller
 * negates that filter's codes); a == 0 gives the constant sentinels (hi =
 * INT32_MIN: always +1; lo = hi = INT32_MAX: always -1; lo = INT32_MIN, hi =
 * INT32_MAX: always 0).  All pointers host, k entries each.  TN_EDOMAIN on
 * non-finite parameters or var + eps <= 0.                                    */
tn_status tn_ternarize_weights(const float* w, int32_t k, int32_t n, float sparsity, int8_t* codes, float* alpha,
                               int64_t* bad_index);
tn_status tn_fold_thresholds(const float* alpha, const float* gamma, const float* beta, const float* mean,
                             const float* var, float eps, int32_t k, int32_t max_abs_acc, int32_t* lo, int32_t* hi,
                             int8_t* negate);

/* Kernel selection for the ternary conv (all exact; parity tests run each).
 *   TN_KERNEL_POPC  CUDA-core XOR/AND/POPC form of Eq. 9 (any geometry): the
 *                   paper's own method, and the fallback for shapes outside TZ
 *   TN_KERNEL_TZ    the tcgen05 kernel: taps as descriptor offsets and the three
 *                   kernel planes merged along N (stride 1/2, pad 1, C <= 64 per
 *                   launch in 16-channel chunks, K in {16, 32, 64}, small 27*C*K
 *                   filter bank); ternary operands as FP4 E2M1 (kind::mxf4,
 *                   unit block scales: exact) where they fit, else int8 (kind::i8)
 *   TN_KERNEL_TZ8   like AUTO, with the TZ kernel restricted to int8 operands
 * TN_KERNEL_AUTO picks TZ, else POPC per shape.  Host, process-wide.  (Value 2,
 * a retired second tensor-core kernel, is rejected with TN_EINVAL.)           */
enum { TN_KERNEL_AUTO = 0, TN_KERNEL_POPC = 1, TN_KERNEL_TZ = 3, TN_KERNEL_TZ8 = 4, TN_KERNEL_WIDE = 5 };
/* TN_KERNEL_WIDE is not a selector: tn_conv_kernel_for reports it for the wide
 * one-plane layers of Table 1 (reading R18: D = 1, C a multiple of 64 per segment
 * with C or K beyond 64, K <= 256, stride 1 / 2, pad 1, optional [up2d | skip]
 * segments), which AUTO and TZ run on a tcgen05 kernel with FP4 operands whose
 * filter bank streams from a prepared image (tn_conv_prepare / tn_fcn_prepare;
 * an unprepared call builds one per call).                                    */
tn_status tn_set_conv_kernel(int32_t which);
int32_t   tn_get_conv_kernel(void);
/* Upper bound on the CTAs of the persistent tensor-core conv grids (0 = one per
 * SM, the default).  Results do not depend on it (integer math); tests use a
 * small cap to give each CTA long runs of output planes.  Host, process-wide;
 * TN_EINVAL if max_ctas < 0.                                                  */
tn_status tn_set_grid_cap(int32_t max_ctas);
/* Which kernel (TN_KERNEL_POPC, _TZ or _WIDE) a tn_conv3d_seg call with these
 * arguments would run under the current selection; -1 if the call is invalid
 * (or a forced tensor-core kernel does not cover the shape).  Host only.      */
int32_t   tn_conv_kernel_for(const tn_segment* segs, int32_t nseg, int32_t k, tn_geom g);
/* Operand format of that call on the tensor-core kernel: 8 = int8 (kind::i8),
 * 4 = FP4 E2M1 (kind::mxf4, NEXT-2); 0 if it would not run on TN_KERNEL_TZ.     */
int32_t   tn_conv_operands_for(const tn_segment* segs, int32_t nseg, int32_t k, tn_geom g);

#ifdef __cplusplus
}
#endif
#endif /* TN_H_ */
