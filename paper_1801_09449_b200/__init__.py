"""paper_1801_09449_b200 -- B200-native TernaryNet inference hot path.

Thin ctypes binding over ``libtn.so`` (include/tn.h).  Function names match the
C ABI; this module only marshals arguments (torch CUDA tensors -> device
pointers, the current torch stream -> cudaStream_t) and raises on a non-OK
status.  Every step of the path runs in the library's sm_100a kernels; there is
no CPU fallback: if libtn.so is missing or cannot load, importing this package
raises.

PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TN_LIBTN_PATH") or os.path.join(_HERE, "libtn.so")  # override: experiments only

INT64_MAX = (1 << 63) - 1

TN_OK, TN_EINVAL, TN_ESHAPE, TN_EALIGN, TN_EUNSUPPORTED, TN_EDOMAIN, TN_ECUDA, TN_ENCCL = range(8)
TN_LAYER_FIRST, TN_LAYER_CONV = 1, 2
TN_KERNEL_AUTO, TN_KERNEL_POPC, TN_KERNEL_TZ, TN_KERNEL_TZ8 = 0, 1, 3, 4
TN_KERNEL_WIDE = 5   # reported by tn_conv_kernel_for for the wide one-plane layers (not a selector)
_STATUS = {0: "TN_OK", 1: "TN_EINVAL", 2: "TN_ESHAPE", 3: "TN_EALIGN", 4: "TN_EUNSUPPORTED",
           5: "TN_EDOMAIN", 6: "TN_ECUDA", 7: "TN_ENCCL"}


class TNError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {_STATUS.get(status, status)}: {msg}")
        self.status = status


class tn_dims(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("c", ctypes.c_int32), ("d", ctypes.c_int32),
                ("h", ctypes.c_int32), ("w", ctypes.c_int32)]


class tn_geom(ctypes.Structure):
    _fields_ = [("stride", ctypes.c_int32 * 3), ("pad", ctypes.c_int32 * 3), ("dil", ctypes.c_int32 * 3)]


class tn_segment(ctypes.Structure):
    _fields_ = [("xp", ctypes.c_void_p), ("d", tn_dims), ("upsample", ctypes.c_int32),
                ("wp", ctypes.c_void_p)]


class tn_slab_layer(ctypes.Structure):
    _fields_ = [("level_scale", ctypes.c_int32), ("c", ctypes.c_int32), ("h", ctypes.c_int32),
                ("w", ctypes.c_int32), ("gd", ctypes.c_int32), ("z0", ctypes.c_int32), ("z1", ctypes.c_int32),
                ("halo", ctypes.c_int32), ("plane_bytes", ctypes.c_int64), ("offset", ctypes.c_int64)]


class tn_layer(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("c_out", ctypes.c_int32), ("stride", ctypes.c_int32),
                ("dil", ctypes.c_int32), ("nseg", ctypes.c_int32), ("src", ctypes.c_int32 * 2),
                ("upsample", ctypes.c_int32 * 2), ("wp", ctypes.c_void_p * 2),
                ("lo", ctypes.c_void_p), ("hi", ctypes.c_void_p)]


# Every symbol include/tn.h declares: name -> (restype, argtypes).
_P, _I32, _I64, _F, _SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_size_t
_D, _G = tn_dims, tn_geom
SIGNATURES = {
    "tn_packed_bytes": (_SZ, [_D]),
    "tn_weight_bytes": (_SZ, [_I32, _I32]),
    "tn_conv_out_dims": (ctypes.c_int, [_D, _I32, _G, ctypes.POINTER(_D)]),
    "tn_last_error": (ctypes.c_char_p, []),
    "tn_version": (ctypes.c_char_p, []),
    "tn_bad_init": (ctypes.c_int, [_P, _P]),
    "tn_pack_i8": (ctypes.c_int, [_P, _D, _P, _P, _P]),
    "tn_pack_i32": (ctypes.c_int, [_P, _D, _P, _P, _P]),
    "tn_pack_f32": (ctypes.c_int, [_P, _D, _F, _F, _P, _P, _P]),
    "tn_pack_weights": (ctypes.c_int, [_P, _I32, _I32, _P, _P, _P]),
    "tn_unpack": (ctypes.c_int, [_P, _D, _P, _P, _P]),
    "tn_conv3d": (ctypes.c_int, [_P, _D, _P, _I32, _G, _P, _P]),
    "tn_conv3d_requant": (ctypes.c_int, [_P, _D, _P, _I32, _G, _P, _P, _P, _P]),
    "tn_requant": (ctypes.c_int, [_P, _D, _P, _P, _P, _P]),
    "tn_conv_prepare": (ctypes.c_int, [ctypes.POINTER(tn_segment), _I32, _I32, _G, _I32, ctypes.POINTER(_P), _P]),
    "tn_conv_prep_bytes": (_I64, [_P]),
    "tn_conv_prep_destroy": (None, [_P]),
    "tn_conv3d_requant_prepared": (ctypes.c_int, [_P, _P, _D, _P, _I32, _G, _P, _P, _P, _P]),
    "tn_conv3d_seg_prepared": (ctypes.c_int, [_P, ctypes.POINTER(tn_segment), _I32, _I32, _G, _P, _P, _P, _P,
                                              _P]),
    "tn_conv3d_seg": (ctypes.c_int, [ctypes.POINTER(tn_segment), _I32, _I32, _G, _P, _P, _P, _P, _P]),
    "tn_conv3d_first": (ctypes.c_int, [_P, _D, _F, _F, _P, _I32, _G, _P, _P, _P, _P, _P]),
    "tn_predict": (ctypes.c_int, [_P, _D, _P, _P, _I32, _P, _P]),
    "tn_fcn_create": (ctypes.c_int, [ctypes.POINTER(tn_layer), _I32, _F, _F, _P, _P, _I32,
                                     ctypes.POINTER(_P)]),
    "tn_fcn_workspace_bytes": (_SZ, [_P, _D]),
    "tn_fcn_forward": (ctypes.c_int, [_P, _P, _D, _P, _P, _SZ, _P, _P]),
    "tn_fcn_destroy": (None, [_P]),
    "tn_fcn_prepare": (ctypes.c_int, [_P, _D, _P]),
    "tn_fcn_prep_bytes": (_SZ, [_P]),
    "tn_fcn_forward_range": (ctypes.c_int, [_P, _P, _D, _P, _P, _SZ, _P, _I32, _I32, _P]),
    "tn_fcn_layer_output": (_P, [_P, _D, _P, _I32, ctypes.POINTER(_D)]),
    "tn_set_conv_kernel": (ctypes.c_int, [_I32]),
    "tn_get_conv_kernel": (_I32, []),
    "tn_set_grid_cap": (ctypes.c_int, [_I32]),
    "tn_ternarize_weights": (ctypes.c_int, [_P, _I32, _I32, ctypes.c_float, _P, _P, _P]),
    "tn_fold_thresholds": (ctypes.c_int, [_P, _P, _P, _P, _P, ctypes.c_float, _I32, _I32, _P, _P, _P]),
    "tn_conv_kernel_for": (_I32, [ctypes.POINTER(tn_segment), _I32, _I32, _G]),
    "tn_conv_operands_for": (_I32, [ctypes.POINTER(tn_segment), _I32, _I32, _G]),
    "tn_comm_unique_id": (ctypes.c_int, [_P]),
    "tn_comm_init": (ctypes.c_int, [_P, _I32, _I32, ctypes.POINTER(_P)]),
    "tn_comm_destroy": (None, [_P]),
    "tn_fcn_slab_plan": (ctypes.c_int, [_P, _D, _I32, _I32, ctypes.POINTER(tn_slab_layer), _I32,
                                        ctypes.POINTER(_SZ)]),
    "tn_fcn_slab_workspace_bytes": (_SZ, [_P, _D, _I32, _I32]),
    "tn_fcn_forward_slab": (ctypes.c_int, [_P, _P, _P, _D, _I32, _I32, _P, _P, _SZ, _P, _P]),
    "tn_fcn_slabs_local_workspace_bytes": (_SZ, [_P, _D, _I32]),
    "tn_fcn_forward_slabs_local": (ctypes.c_int, [_P, _P, _D, _I32, _P, _P, _SZ, _P, _P]),
    "tn_halo_create": (ctypes.c_int, [_P, _D, _I32, _I32, ctypes.POINTER(_P)]),
    "tn_halo_workspace_bytes": (_SZ, [_P]),
    "tn_halo_export": (ctypes.c_int, [_P, _P]),
    "tn_halo_connect": (ctypes.c_int, [_P, _P, _D, _P, _I32, _P, _I32]),
    "tn_fcn_forward_slab_p2p": (ctypes.c_int, [_P, _P, _P, _P, _P, _P]),
    "tn_fcn_forward_slabs_local_p2p": (ctypes.c_int, [_P, _P, _D, _I32, _P, _P, _SZ, _P, _P]),
    "tn_halo_destroy": (None, [_P]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1801_09449_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


# ----------------------------------------------------------------------------- helpers
def _check(status: int, where: str):
    if status != TN_OK:
        raise TNError(status, where, lib.tn_last_error().decode())


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def dims(n, c, d, h, w) -> tn_dims:
    return tn_dims(int(n), int(c), int(d), int(h), int(w))


def dims_of(x: torch.Tensor) -> tn_dims:
    assert x.dim() == 5, "expected an NCDHW tensor"
    return dims(*x.shape)


def geom(stride=1, pad=1, dil=1) -> tn_geom:
    t3 = lambda v: (v,) * 3 if isinstance(v, int) else tuple(v)
    g = tn_geom()
    for i, (s, p, d) in enumerate(zip(t3(stride), t3(pad), t3(dil))):
        g.stride[i], g.pad[i], g.dil[i] = s, p, d
    return g


def cw(c: int) -> int:
    return (c + 31) // 32


def packed_empty(n, c, d, h, w, device="cuda"):
    """Allocate a packed tensor [n,d,h,w,2,cw] (int32 storage of the uint32 words)."""
    return torch.empty((n, d, h, w, 2, cw(c)), dtype=torch.int32, device=device)


def bad_flag(device="cuda"):
    """An int64 device flag initialised to INT64_MAX (tn_bad_init)."""
    f = torch.empty(1, dtype=torch.int64, device=device)
    tn_bad_init(f)
    return f


def conv_out_dims(xd: tn_dims, k: int, g: tn_geom) -> tn_dims:
    out = tn_dims()
    _check(lib.tn_conv_out_dims(xd, k, g, ctypes.byref(out)), "tn_conv_out_dims")
    return out


# ----------------------------------------------------------------------------- the ABI
def tn_bad_init(d_bad, stream=None):
    _check(lib.tn_bad_init(_ptr(d_bad), _stream(stream)), "tn_bad_init")


def tn_pack_i8(x, xp=None, d_bad=None, stream=None):
    n, c, d, h, w = x.shape
    xp = packed_empty(n, c, d, h, w, x.device) if xp is None else xp
    _check(lib.tn_pack_i8(_ptr(x), dims_of(x), _ptr(xp), _ptr(d_bad), _stream(stream)), "tn_pack_i8")
    return xp


def tn_pack_i32(x, xp=None, d_bad=None, stream=None):
    n, c, d, h, w = x.shape
    xp = packed_empty(n, c, d, h, w, x.device) if xp is None else xp
    _check(lib.tn_pack_i32(_ptr(x), dims_of(x), _ptr(xp), _ptr(d_bad), _stream(stream)), "tn_pack_i32")
    return xp


def tn_pack_f32(x, t_lo, t_hi, xp=None, d_bad=None, stream=None):
    n, c, d, h, w = x.shape
    xp = packed_empty(n, c, d, h, w, x.device) if xp is None else xp
    _check(lib.tn_pack_f32(_ptr(x), dims_of(x), float(t_lo), float(t_hi), _ptr(xp), _ptr(d_bad),
                           _stream(stream)), "tn_pack_f32")
    return xp


def tn_pack_weights(w, wp=None, d_bad=None, stream=None):
    k, c = w.shape[:2]
    wp = torch.empty((k, 27, 2, cw(c)), dtype=torch.int32, device=w.device) if wp is None else wp
    _check(lib.tn_pack_weights(_ptr(w), k, c, _ptr(wp), _ptr(d_bad), _stream(stream)), "tn_pack_weights")
    return wp


def tn_unpack(xp, c, x=None, d_bad=None, stream=None):
    n, d, h, w = xp.shape[:4]
    x = torch.empty((n, c, d, h, w), dtype=torch.int8, device=xp.device) if x is None else x
    _check(lib.tn_unpack(_ptr(xp), dims(n, c, d, h, w), _ptr(x), _ptr(d_bad), _stream(stream)), "tn_unpack")
    return x


def tn_conv3d(xp, xd: tn_dims, wp, k, g: tn_geom, y=None, stream=None):
    od = conv_out_dims(xd, k, g)
    y = torch.empty((od.n, od.d, od.h, od.w, k), dtype=torch.int32, device=xp.device) if y is None else y
    _check(lib.tn_conv3d(_ptr(xp), xd, _ptr(wp), k, g, _ptr(y), _stream(stream)), "tn_conv3d")
    return y


def tn_conv3d_requant(xp, xd: tn_dims, wp, k, g: tn_geom, lo, hi, yp=None, stream=None):
    od = conv_out_dims(xd, k, g)
    yp = packed_empty(od.n, k, od.d, od.h, od.w, xp.device) if yp is None else yp
    _check(lib.tn_conv3d_requant(_ptr(xp), xd, _ptr(wp), k, g, _ptr(lo), _ptr(hi), _ptr(yp),
                                 _stream(stream)), "tn_conv3d_requant")
    return yp


def tn_requant(y, lo, hi, yp=None, stream=None):
    n, d, h, w, k = y.shape
    yp = packed_empty(n, k, d, h, w, y.device) if yp is None else yp
    _check(lib.tn_requant(_ptr(y), dims(n, k, d, h, w), _ptr(lo), _ptr(hi), _ptr(yp), _stream(stream)),
           "tn_requant")
    return yp


class ConvPrep:
    """A prepared filter bank (tn_conv_prepare): the tensor-core kernel's B image, built once."""

    def __init__(self, handle):
        self.handle = handle

    @property
    def nbytes(self) -> int:
        return int(lib.tn_conv_prep_bytes(self.handle)) if self.handle else 0

    def close(self):
        if self.handle and lib is not None:   # lib is None during interpreter shutdown
            lib.tn_conv_prep_destroy(self.handle)
        self.handle = None

    def __del__(self):
        self.close()


def _seg_array(segs):
    arr = (tn_segment * len(segs))()
    for i, (xp, d, up, wp) in enumerate(segs):
        arr[i] = tn_segment(xp.data_ptr() if xp is not None else None, d, int(up), wp.data_ptr())
    return arr


def tn_conv_prepare(segs, k, g: tn_geom, requant=True, stream=None) -> ConvPrep:
    """segs: list of (xp or None, tn_dims, upsample, wp), as for tn_conv3d_seg."""
    h = ctypes.c_void_p()
    _check(lib.tn_conv_prepare(_seg_array(segs), len(segs), k, g, int(bool(requant)), ctypes.byref(h),
                               _stream(stream)), "tn_conv_prepare")
    return ConvPrep(h.value)


def tn_conv3d_requant_prepared(prep, xp, xd: tn_dims, wp, k, g: tn_geom, lo, hi, yp=None, stream=None):
    od = conv_out_dims(xd, k, g)
    yp = packed_empty(od.n, k, od.d, od.h, od.w, xp.device) if yp is None else yp
    _check(lib.tn_conv3d_requant_prepared(prep.handle if prep is not None else None, _ptr(xp), xd, _ptr(wp), k, g,
                                          _ptr(lo), _ptr(hi), _ptr(yp), _stream(stream)),
           "tn_conv3d_requant_prepared")
    return yp


def _seg_out(segs, k, g, y, yp, requant):
    d0, up0 = segs[0][1], segs[0][2]
    f, fz = (2 if up0 else 1), (2 if up0 == 1 else 1)   # upsample 2: in-plane only
    od = conv_out_dims(dims(d0.n, 1, d0.d * fz, d0.h * f, d0.w * f), k, g)
    dev = segs[0][0].device
    if requant and yp is None and y is None:
        yp = packed_empty(od.n, k, od.d, od.h, od.w, dev)
    elif not requant and y is None and yp is None:
        y = torch.empty((od.n, od.d, od.h, od.w, k), dtype=torch.int32, device=dev)
    return y, yp


def tn_conv3d_seg_prepared(prep, segs, k, g: tn_geom, lo=None, hi=None, y=None, yp=None, requant=True,
                           stream=None):
    y, yp = _seg_out(segs, k, g, y, yp, requant)
    _check(lib.tn_conv3d_seg_prepared(prep.handle if prep is not None else None, _seg_array(segs), len(segs), k,
                                      g, _ptr(lo), _ptr(hi), _ptr(y), _ptr(yp), _stream(stream)),
           "tn_conv3d_seg_prepared")
    return yp if yp is not None else y


def tn_conv3d_seg(segs, k, g: tn_geom, lo=None, hi=None, y=None, yp=None, requant=True, stream=None):
    """segs: list of (xp, tn_dims, upsample, wp)."""
    arr = _seg_array(segs)
    d0, up0 = segs[0][1], segs[0][2]
    f, fz = (2 if up0 else 1), (2 if up0 == 1 else 1)   # upsample 2: in-plane only
    od = conv_out_dims(dims(d0.n, 1, d0.d * fz, d0.h * f, d0.w * f), k, g)
    dev = segs[0][0].device
    if requant and yp is None and y is None:
        yp = packed_empty(od.n, k, od.d, od.h, od.w, dev)
    elif not requant and y is None and yp is None:
        y = torch.empty((od.n, od.d, od.h, od.w, k), dtype=torch.int32, device=dev)
    _check(lib.tn_conv3d_seg(arr, len(segs), k, g, _ptr(lo), _ptr(hi), _ptr(y), _ptr(yp), _stream(stream)),
           "tn_conv3d_seg")
    return yp if yp is not None else y


def tn_conv3d_first(x, t_lo, t_hi, wp, k, g: tn_geom, lo, hi, yp=None, d_bad=None, stream=None):
    xd = dims_of(x)
    od = conv_out_dims(xd, k, g)
    yp = packed_empty(od.n, k, od.d, od.h, od.w, x.device) if yp is None else yp
    _check(lib.tn_conv3d_first(_ptr(x), xd, float(t_lo), float(t_hi), _ptr(wp), k, g, _ptr(lo), _ptr(hi),
                               _ptr(yp), _ptr(d_bad), _stream(stream)), "tn_conv3d_first")
    return yp


def tn_predict(tp, c, w, b, logits=None, stream=None):
    n, d, h, wd = tp.shape[:4]
    nclass = w.shape[0]
    logits = torch.empty((n, nclass, d, h, wd), dtype=torch.float32, device=tp.device) if logits is None else logits
    _check(lib.tn_predict(_ptr(tp), dims(n, c, d, h, wd), _ptr(w), _ptr(b), nclass, _ptr(logits),
                          _stream(stream)), "tn_predict")
    return logits


def tn_set_conv_kernel(which: int):
    _check(lib.tn_set_conv_kernel(int(which)), "tn_set_conv_kernel")


def tn_get_conv_kernel() -> int:
    return int(lib.tn_get_conv_kernel())


def tn_ternarize_weights(w, sparsity: float = -1.0):
    """Eq. 4 per output filter of a float filter bank w [K, ...] (host numpy);
    sparsity in [0, 1) fixes the zeros per filter instead.  Returns (codes int8
    of w's shape, alpha float32 [K])."""
    import numpy as np
    w = np.ascontiguousarray(w, dtype=np.float32)
    k = w.shape[0]
    n = int(w.size // k)
    codes = np.empty(w.shape, np.int8)
    alpha = np.empty(k, np.float32)
    bad = ctypes.c_int64(-1)
    st = lib.tn_ternarize_weights(w.ctypes.data_as(_P), k, n, float(sparsity), codes.ctypes.data_as(_P),
                                  alpha.ctypes.data_as(_P), ctypes.byref(bad))
    _check(st, "tn_ternarize_weights")
    return codes, alpha


def tn_fold_thresholds(alpha, gamma, beta, mean, var, eps: float, max_abs_acc: int):
    """Fold alpha, batch norm and Eq. 6 into integer thresholds (host numpy, K each).
    Returns (lo int32, hi int32, negate int8)."""
    import numpy as np
    arrs = [np.ascontiguousarray(v, dtype=np.float32) for v in (alpha, gamma, beta, mean, var)]
    k = arrs[0].shape[0]
    lo, hi, neg = np.empty(k, np.int32), np.empty(k, np.int32), np.empty(k, np.int8)
    st = lib.tn_fold_thresholds(*[a.ctypes.data_as(_P) for a in arrs], float(eps), k, int(max_abs_acc),
                                lo.ctypes.data_as(_P), hi.ctypes.data_as(_P), neg.ctypes.data_as(_P))
    _check(st, "tn_fold_thresholds")
    return lo, hi, neg


def tn_set_grid_cap(max_ctas: int):
    _check(lib.tn_set_grid_cap(int(max_ctas)), "tn_set_grid_cap")


def tn_conv_kernel_for(seg_dims, k, g: tn_geom, upsample=None) -> int:
    """Kernel a conv over segments with these dims would use (shape logic only)."""
    upsample = upsample or [0] * len(seg_dims)
    arr = (tn_segment * len(seg_dims))()
    for i, (d, up) in enumerate(zip(seg_dims, upsample)):
        arr[i] = tn_segment(None, d, int(up), None)
    return int(lib.tn_conv_kernel_for(arr, len(seg_dims), int(k), g))


def tn_conv_operands_for(seg_dims, k, g: tn_geom, upsample=None) -> int:
    """Tensor-core operand format (8 = int8, 4 = FP4; 0 = not on the tensor-core kernel)."""
    upsample = upsample or [0] * len(seg_dims)
    arr = (tn_segment * len(seg_dims))()
    for i, (d, up) in enumerate(zip(seg_dims, upsample)):
        arr[i] = tn_segment(None, d, int(up), None)
    return int(lib.tn_conv_operands_for(arr, len(seg_dims), int(k), g))


# ----------------------------------------------------------------------------- the FCN
def fcn_table():
    """The 3D ternary FCN (reading R9): Table 1 in 3D with channels
    16-32-64-64, stride-2 convs for the three AvgPool rows, nearest x2 upsampling,
    concat order [upsampled, skip], 1x1x1 float prediction.  Entries:
    (kind, c_out, stride, [(src, upsample), ...]); src -1 = the float input."""
    F, C = TN_LAYER_FIRST, TN_LAYER_CONV
    return [
        (F, 16, 1, [(-1, 0)]),           # 1  R0
        (C, 16, 1, [(0, 0)]),            # 2  R0  -> skip to 13
        (C, 16, 2, [(1, 0)]),            # 3  R0 -> R1
        (C, 32, 1, [(2, 0)]),            # 4  R1  -> skip to 11
        (C, 32, 2, [(3, 0)]),            # 5  R1 -> R2
        (C, 64, 1, [(4, 0)]),            # 6  R2  -> skip to 9
        (C, 64, 2, [(5, 0)]),            # 7  R2 -> R3
        (C, 64, 1, [(6, 0)]),            # 8  R3
        (C, 64, 1, [(7, 1), (5, 0)]),    # 9  [up(8) | 6] R2
        (C, 32, 1, [(8, 0)]),            # 10 R2
        (C, 32, 1, [(9, 1), (3, 0)]),    # 11 [up(10) | 4] R1
        (C, 16, 1, [(10, 0)]),           # 12 R1
        (C, 16, 1, [(11, 1), (1, 0)]),   # 13 [up(12) | 2] R0
        (C, 16, 1, [(12, 0)]),           # 14 R0
    ]


def fcn25_table():
    """Table 1's 2.5D U-Net (reading R18) for one-plane inputs [n][15][1][h][w]
    (15-slice stacks, the slices as layer 1's channels): 2D layers as 3x3x3 convs on one-plane
    volumes (only the middle kernel plane meets data), channels 32-64-128-256, stride-2 convs for
    the three AvgPool2D rows, nearest x2 in y and x (upsample 2) for the Upsample2D rows, skips
    #2->#13, #4->#11, #6->#9 as [upsampled, skip], the 1x1 layers #7/#8 as centre-tap filters."""
    F, C = TN_LAYER_FIRST, TN_LAYER_CONV
    return [
        (F, 32, 1, [(-1, 0)]),           # 1  15 slices -> 32
        (C, 64, 1, [(0, 0)]),            # 2  -> skip to 13
        (C, 64, 2, [(1, 0)]),            # 3  (+ AvgPool2D) /2
        (C, 128, 1, [(2, 0)]),           # 4  -> skip to 11
        (C, 128, 2, [(3, 0)]),           # 5  /4
        (C, 256, 1, [(4, 0)]),           # 6  -> skip to 9
        (C, 256, 2, [(5, 0)]),           # 7  1x1, /8
        (C, 256, 1, [(6, 0)]),           # 8  1x1
        (C, 256, 1, [(7, 2), (5, 0)]),   # 9  [up2d(8) | 6]
        (C, 128, 1, [(8, 0)]),           # 10
        (C, 128, 1, [(9, 2), (3, 0)]),   # 11 [up2d(10) | 4]
        (C, 64, 1, [(10, 0)]),           # 12
        (C, 64, 1, [(11, 2), (1, 0)]),   # 13 [up2d(12) | 2]
        (C, 64, 1, [(12, 0)]),           # 14
    ]


def fcn_macs_per_voxel(table=None) -> int:
    """Ternary MACs of one forward per input voxel (27 * cin * cout per output voxel,
    output voxels at 1/8^level of the input)."""
    table = table or fcn_table()
    level = []
    macs = 0.0
    cout = []
    for i, (_, co, s, segs) in enumerate(table):
        if segs[0][0] < 0:
            lv, cin = 0, 1
        else:
            src, up = segs[0]
            lv = level[src] - (1 if up else 0)
            cin = sum(cout[sj] for sj, _ in segs)
        lv += 1 if s == 2 else 0
        level.append(lv)
        cout.append(co)
        macs += 27.0 * cin * co / (8 ** lv)
    return int(round(macs))


class TernaryFCN:
    """tn_fcn_create / tn_fcn_forward over device-resident packed parameters.

    weights: 14 int8 tensors [cout][cin][3][3][3] (cin = the concatenated width for
    skip layers, channel order [upsampled, skip]); lo/hi: int32 [cout]; pred_w
    float [nclass][16], pred_b float [nclass].  Tensors may be numpy or torch."""

    def __init__(self, weights, lo, hi, pred_w, pred_b, t_lo, t_hi, table=None, device="cuda", c_in=1):
        self.table = table or fcn_table()
        dev = torch.device(device)
        as_t = lambda a, dt: torch.as_tensor(a).to(device=dev, dtype=dt).contiguous()
        self._keep = []
        layers = (tn_layer * len(self.table))()
        couts = [row[1] for row in self.table]
        for i, (kind, co, s, segs) in enumerate(self.table):
            w = as_t(weights[i], torch.int8)
            cins = [c_in] if segs[0][0] < 0 else [couts[sj] for sj, _ in segs]
            assert w.shape == (co, sum(cins), 3, 3, 3), (i, tuple(w.shape), cins)
            L = layers[i]
            L.kind, L.c_out, L.stride, L.dil, L.nseg = kind, co, s, 1, len(segs)
            c0 = 0
            for j, ((src, up), ci) in enumerate(zip(segs, cins)):
                wp = tn_pack_weights(w[:, c0:c0 + ci].contiguous())
                self._keep.append(wp)
                L.src[j], L.upsample[j], L.wp[j] = src, up, wp.data_ptr()
                c0 += ci
            lo_t, hi_t = as_t(lo[i], torch.int32), as_t(hi[i], torch.int32)
            self._keep += [lo_t, hi_t]
            L.lo, L.hi = lo_t.data_ptr(), hi_t.data_ptr()
        self.pred_w = as_t(pred_w, torch.float32)
        self.pred_b = as_t(pred_b, torch.float32)
        self.nclass = int(self.pred_w.shape[0])
        self.t_lo, self.t_hi = float(t_lo), float(t_hi)
        handle = ctypes.c_void_p()
        _check(lib.tn_fcn_create(layers, len(self.table), self.t_lo, self.t_hi, _ptr(self.pred_w),
                                 _ptr(self.pred_b), self.nclass, ctypes.byref(handle)), "tn_fcn_create")
        self.handle = handle
        torch.cuda.synchronize(dev)  # weights packed before the caller frees its int8 copies

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and lib is not None:   # lib is None during interpreter shutdown
            lib.tn_fcn_destroy(h)
            self.handle = None

    def workspace_bytes(self, xd: tn_dims) -> int:
        return int(lib.tn_fcn_workspace_bytes(self.handle, xd))

    def prepare(self, x_shape, stream=None) -> int:
        """tn_fcn_prepare: prebuild every tensor-core layer's filter-bank image for inputs of x_shape;
        returns the device bytes they hold."""
        _check(lib.tn_fcn_prepare(self.handle, dims(*x_shape), _stream(stream)), "tn_fcn_prepare")
        return int(lib.tn_fcn_prep_bytes(self.handle))

    def workspace(self, x_shape, device="cuda"):
        nb = self.workspace_bytes(dims(*x_shape))
        return torch.empty(max(nb, 16), dtype=torch.uint8, device=device)

    def forward(self, x, logits=None, ws=None, d_bad=None, stream=None):
        xd = dims_of(x)
        if ws is None:
            ws = self.workspace(x.shape, x.device)
        if logits is None:
            logits = torch.empty((xd.n, self.nclass, xd.d, xd.h, xd.w), dtype=torch.float32, device=x.device)
        _check(lib.tn_fcn_forward(self.handle, _ptr(x), xd, _ptr(logits), _ptr(ws), ws.numel(), _ptr(d_bad),
                                  _stream(stream)), "tn_fcn_forward")
        return logits

    __call__ = forward

    def forward_range(self, x, first, last, logits=None, ws=None, d_bad=None, stream=None):
        """Layers [first, last) of forward() only (last = -1: to the end, with the prediction)."""
        xd = dims_of(x)
        if ws is None:
            ws = self.workspace(x.shape, x.device)
        if logits is None:
            logits = torch.empty((xd.n, self.nclass, xd.d, xd.h, xd.w), dtype=torch.float32, device=x.device)
        _check(lib.tn_fcn_forward_range(self.handle, _ptr(x), xd, _ptr(logits), _ptr(ws), ws.numel(), _ptr(d_bad),
                                        int(first), int(last), _stream(stream)), "tn_fcn_forward_range")
        return logits

    def slab_plan(self, global_shape, z0, z1):
        """Per-layer slab geometry from the library's planner (host only)."""
        n = len(self.table)
        arr = (tn_slab_layer * n)()
        nb = ctypes.c_size_t()
        _check(lib.tn_fcn_slab_plan(self.handle, dims(*global_shape), int(z0), int(z1), arr, n, ctypes.byref(nb)),
               "tn_fcn_slab_plan")
        return list(arr), int(nb.value)

    def forward_slabs_local(self, x, nslabs, logits=None, ws=None, d_bad=None, stream=None):
        """All z-slabs of one volume on this device, halos by device copies."""
        xd = dims_of(x)
        if ws is None:
            nb = int(lib.tn_fcn_slabs_local_workspace_bytes(self.handle, xd, int(nslabs)))
            if nb == 0:
                raise TNError(TN_ESHAPE, "tn_fcn_slabs_local_workspace_bytes", lib.tn_last_error().decode())
            ws = torch.empty(nb, dtype=torch.uint8, device=x.device)
        if logits is None:
            logits = torch.empty((xd.n, self.nclass, xd.d, xd.h, xd.w), dtype=torch.float32, device=x.device)
        _check(lib.tn_fcn_forward_slabs_local(self.handle, _ptr(x), xd, int(nslabs), _ptr(logits), _ptr(ws),
                                              ws.numel(), _ptr(d_bad), _stream(stream)), "tn_fcn_forward_slabs_local")
        return logits

    def forward_slabs_local_p2p(self, x, nslabs, logits=None, ws=None, d_bad=None, stream=None):
        """All z-slabs on this device with the NEXT-1 schedule: epilogue stores into the
        neighbouring slabs' halo planes and device progress flags (no copies, no NCCL)."""
        xd = dims_of(x)
        if ws is None:
            nb = int(lib.tn_fcn_slabs_local_workspace_bytes(self.handle, xd, int(nslabs)))
            if nb == 0:
                raise TNError(TN_ESHAPE, "tn_fcn_slabs_local_workspace_bytes", lib.tn_last_error().decode())
            ws = torch.empty(nb, dtype=torch.uint8, device=x.device)
        if logits is None:
            logits = torch.empty((xd.n, self.nclass, xd.d, xd.h, xd.w), dtype=torch.float32, device=x.device)
        _check(lib.tn_fcn_forward_slabs_local_p2p(self.handle, _ptr(x), xd, int(nslabs), _ptr(logits), _ptr(ws),
                                                  ws.numel(), _ptr(d_bad), _stream(stream)),
               "tn_fcn_forward_slabs_local_p2p")
        return logits

    def forward_slab(self, comm, x_slab, global_shape, z0, z1, logits=None, ws=None, d_bad=None, stream=None):
        """This rank's slab [z0, z1) of a volume decomposed over the ranks of comm (NCCL halos)."""
        gd = dims(*global_shape)
        if ws is None:
            nb = int(lib.tn_fcn_slab_workspace_bytes(self.handle, gd, int(z0), int(z1)))
            ws = torch.empty(max(nb, 16), dtype=torch.uint8, device=x_slab.device)
        if logits is None:
            logits = torch.empty((1, self.nclass, z1 - z0, gd.h, gd.w), dtype=torch.float32, device=x_slab.device)
        _check(lib.tn_fcn_forward_slab(self.handle, comm.handle, _ptr(x_slab), gd, int(z0), int(z1), _ptr(logits),
                                       _ptr(ws), ws.numel(), _ptr(d_bad), _stream(stream)), "tn_fcn_forward_slab")
        return logits

    def layer_output(self, x_shape, ws, i):
        """(packed tensor view, dims) of layer i's output inside ws."""
        od = tn_dims()
        p = lib.tn_fcn_layer_output(self.handle, dims(*x_shape), _ptr(ws), int(i), ctypes.byref(od))
        if not p:
            raise IndexError(i)
        off = p - ws.data_ptr()
        nwords = od.n * od.d * od.h * od.w * 2 * cw(od.c)
        view = ws[off:off + 4 * nwords].view(torch.int32).view(od.n, od.d, od.h, od.w, 2, cw(od.c))
        return view, od


class HaloP2P:
    """NEXT-1: this rank's slab [z0, z1) of a volume split in z over the ranks of a
    torch.distributed group (ranks in z order, equal slabs), with halos stored by the
    conv epilogues straight into the neighbours' memory (CUDA IPC over NVLink) and
    device progress flags instead of NCCL.  The IPC handles travel through the group."""

    def __init__(self, net, global_shape, rank: int, world: int, group=None):
        import torch.distributed as dist
        gd = dims(*global_shape)
        D = gd.d
        if D % world:
            raise TNError(TN_ESHAPE, "HaloP2P", "depth must divide over the ranks")
        dz = D // world
        self.net, self.gd = net, gd
        self.z0, self.z1 = rank * dz, (rank + 1) * dz
        h = ctypes.c_void_p()
        _check(lib.tn_halo_create(net.handle, gd, self.z0, self.z1, ctypes.byref(h)), "tn_halo_create")
        self.handle = h
        mine = (ctypes.c_uint8 * 64)()
        _check(lib.tn_halo_export(h, mine), "tn_halo_export")
        handles = [bytes(mine)]
        if world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, bytes(mine), group=group)
        lo = (ctypes.c_uint8 * 64)(*handles[rank - 1]) if rank > 0 else None
        up = (ctypes.c_uint8 * 64)(*handles[rank + 1]) if rank + 1 < world else None
        _check(lib.tn_halo_connect(h, net.handle, gd, lo, self.z0 - dz, up, self.z1 + dz), "tn_halo_connect")

    def forward(self, x_slab, logits=None, d_bad=None, stream=None):
        if logits is None:
            logits = torch.empty((1, self.net.nclass, self.z1 - self.z0, self.gd.h, self.gd.w),
                                 dtype=torch.float32, device=x_slab.device)
        _check(lib.tn_fcn_forward_slab_p2p(self.net.handle, self.handle, _ptr(x_slab), _ptr(logits), _ptr(d_bad),
                                           _stream(stream)), "tn_fcn_forward_slab_p2p")
        return logits

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and lib is not None:
            lib.tn_halo_destroy(h)
            self.handle = None


class Comm:
    """tn_comm_init over a 128-byte NCCL unique id broadcast through torch.distributed."""

    def __init__(self, rank: int, world: int, group=None):
        import torch.distributed as dist
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            buf = (ctypes.c_uint8 * 128)()
            _check(lib.tn_comm_unique_id(buf), "tn_comm_unique_id")
            uid = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
        if world > 1:
            backend = dist.get_backend(group)
            t = uid.cuda() if backend == "nccl" else uid
            dist.broadcast(t, src=0, group=group)
            uid = t.cpu()
        raw = (ctypes.c_uint8 * 128)(*uid.tolist())
        h = ctypes.c_void_p()
        _check(lib.tn_comm_init(raw, int(rank), int(world), ctypes.byref(h)), "tn_comm_init")
        self.handle = h
        self.rank, self.world = rank, world

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            lib.tn_comm_destroy(h)
            self.handle = None
