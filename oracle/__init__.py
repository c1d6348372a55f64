"""CPU oracle for the TernaryNet inference hot path -- TEST INFRASTRUCTURE ONLY.

Thin ctypes/numpy wrapper over ``oracle/tn_oracle.c`` (plain C, compiled with
gcc by :func:`build`).  Only ``tests/``, ``__graft_entry__.smoke()`` and the
CPU legs of ``bench.py`` (``cpu_baseline`` and ``--impl reference``) may import
this package.  It shares no code with ``paper_1801_09449_b200`` (the CUDA
path) and never imports it.

Every function below names the PAPER.md passage it follows; the C source holds
the arithmetic.  Layouts: ternary codes are int8 NCDHW (PyTorch order); packed
tensors are uint32 ``[n][d][h][w][2][cw]`` (reading R3 in DESIGN.md).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tn_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_i8p = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_c = ctypes
_I, _L, _F = _c.c_int, _c.c_int64, _c.c_float


def build(force: bool = False) -> str:
    """Compile tn_oracle.c with gcc (-O2 -fopenmp).  Building is not using it."""
    stale = (not os.path.exists(_LIB_PATH)
             or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC))
    if force or stale:
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c99",
                               "-Wall", "-o", tmp, _SRC])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    lib = ctypes.CDLL(build())
    lib.oracle_tern_f32.argtypes = [_f32p, _L, _F, _F, _i8p]
    lib.oracle_tern_f32.restype = _L
    lib.oracle_pack.argtypes = [_i8p, _I, _I, _I, _I, _I, _u32p]
    lib.oracle_pack.restype = _L
    lib.oracle_unpack.argtypes = [_u32p, _I, _I, _I, _I, _I, _i8p]
    lib.oracle_unpack.restype = _L
    lib.oracle_pack_weights.argtypes = [_i8p, _I, _I, _u32p]
    lib.oracle_pack_weights.restype = _L
    lib.oracle_conv3d.argtypes = [_i8p, _I, _I, _I, _I, _I, _i8p, _I, _i32p, _i32p]
    lib.oracle_conv3d.restype = None
    lib.oracle_conv3d_at.argtypes = [_i8p, _I, _I, _I, _I, _I, _i8p, _I, _i32p, _i32p, _L, _i32p]
    lib.oracle_conv3d_at.restype = None
    lib.oracle_requant.argtypes = [_i32p, _I, _I, _L, _i32p, _i32p, _i8p]
    lib.oracle_requant.restype = None
    lib.oracle_upsample2.argtypes = [_i8p, _I, _I, _I, _I, _I, _i8p]
    lib.oracle_upsample2.restype = None
    lib.oracle_upsample2_yx.argtypes = [_i8p, _I, _I, _I, _I, _I, _i8p]
    lib.oracle_upsample2_yx.restype = None
    lib.oracle_concat.argtypes = [_i8p, _I, _i8p, _I, _I, _L, _i8p]
    lib.oracle_concat.restype = None
    lib.oracle_predict.argtypes = [_i8p, _I, _I, _L, _I, _f32p, _f32p, _f32p]
    lib.oracle_predict.restype = None
    pp = ctypes.POINTER(ctypes.c_void_p)
    lib.oracle_fcn_forward.argtypes = [_f32p, _I, _I, _I, _I, _F, _F, pp, pp, pp,
                                       _f32p, _f32p, _f32p, pp]
    lib.oracle_fcn_forward.restype = _L
    lib.oracle_num_threads.argtypes = []
    lib.oracle_num_threads.restype = _I
    _lib = lib
    return lib


def _triple(v):
    if isinstance(v, (int, np.integer)):
        return (int(v),) * 3
    t = tuple(int(a) for a in v)
    assert len(t) == 3
    return t


def out_extent(length: int, stride: int, pad: int, dil: int) -> int:
    span = length + 2 * pad - 2 * dil - 1
    return 0 if span < 0 else span // stride + 1


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def tern_f32(x, t_lo: float, t_hi: float):
    """Eq. 6 on the float input with folded normalisation
    thresholds (reading R7).  Returns (int8 codes, bad index or -1)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    t = np.empty(x.shape, dtype=np.int8)
    bad = _load().oracle_tern_f32(x.reshape(-1), x.size, t_lo, t_hi, t.reshape(-1))
    return t, int(bad)


def pack(x):
    """2-bit sign/mask encoding (Fig. 3; readings R2, R3).
    x: int8 NCDHW -> (uint32 [n,d,h,w,2,cw], bad)."""
    x = np.ascontiguousarray(x, dtype=np.int8)
    n, c, d, h, w = x.shape
    cw = (c + 31) // 32
    xp = np.empty((n, d, h, w, 2, cw), dtype=np.uint32)
    bad = _load().oracle_pack(x, n, c, d, h, w, xp)
    return xp, int(bad)


def unpack(xp, c: int):
    xp = np.ascontiguousarray(xp, dtype=np.uint32)
    n, d, h, w = xp.shape[:4]
    x = np.zeros((n, c, d, h, w), dtype=np.int8)
    bad = _load().oracle_unpack(xp, n, c, d, h, w, x)
    return x, int(bad)


def pack_weights(wt):
    """int8 [k,c,3,3,3] -> uint32 [k,27,2,cw]; tap t = (dz*3+dy)*3+dx."""
    wt = np.ascontiguousarray(wt, dtype=np.int8)
    k, c = wt.shape[:2]
    assert wt.shape[2:] == (3, 3, 3)
    cw = (c + 31) // 32
    wp = np.empty((k, 27, 2, cw), dtype=np.uint32)
    bad = _load().oracle_pack_weights(wt, k, c, wp)
    return wp, int(bad)


def _geom(stride, pad, dil):
    s, p, dl = _triple(stride), _triple(pad), _triple(dil)
    return np.array(s + p + dl, dtype=np.int32)


def conv3d(x, wt, stride=1, pad=1, dil=1):
    """Ternary 3x3x3 convolution = the integer sum Eq. 9 computes
    (dilation PAPER.md:135).  int8 NCDHW -> int32 NCDHW."""
    x = np.ascontiguousarray(x, dtype=np.int8)
    wt = np.ascontiguousarray(wt, dtype=np.int8)
    n, c, d, h, w = x.shape
    k = wt.shape[0]
    assert wt.shape == (k, c, 3, 3, 3)
    g = _geom(stride, pad, dil)
    od = out_extent(d, g[0], g[3], g[6])
    oh = out_extent(h, g[1], g[4], g[7])
    ow = out_extent(w, g[2], g[5], g[8])
    y = np.zeros((n, k, od, oh, ow), dtype=np.int32)
    if y.size:
        _load().oracle_conv3d(x, n, c, d, h, w, wt, k, g, y)
    return y


def conv3d_at(x, wt, at, stride=1, pad=1, dil=1):
    """Sampled outputs of :func:`conv3d`; at: int array [m,5] of (n,k,zo,yo,xo)."""
    x = np.ascontiguousarray(x, dtype=np.int8)
    wt = np.ascontiguousarray(wt, dtype=np.int8)
    at = np.ascontiguousarray(at, dtype=np.int32)
    n, c, d, h, w = x.shape
    k = wt.shape[0]
    out = np.zeros(at.shape[0], dtype=np.int32)
    _load().oracle_conv3d_at(x, n, c, d, h, w, wt, k, _geom(stride, pad, dil), at, at.shape[0], out)
    return out


def requant(acc, lo, hi):
    """Integer-threshold requantisation (Eq. 6; R5/R6).
    acc int32 [n,k,...] -> int8 codes."""
    acc = np.ascontiguousarray(acc, dtype=np.int32)
    n, k = acc.shape[:2]
    dhw = int(np.prod(acc.shape[2:])) if acc.ndim > 2 else 1
    t = np.empty(acc.shape, dtype=np.int8)
    _load().oracle_requant(acc, n, k, dhw, np.ascontiguousarray(lo, dtype=np.int32),
                           np.ascontiguousarray(hi, dtype=np.int32), t)
    return t


def upsample2(x):
    """Nearest x2 upsampling (reading R10)."""
    x = np.ascontiguousarray(x, dtype=np.int8)
    n, c, d, h, w = x.shape
    y = np.empty((n, c, 2 * d, 2 * h, 2 * w), dtype=np.int8)
    _load().oracle_upsample2(x, n, c, d, h, w, y)
    return y


def upsample2_yx(x):
    """Upsample2D of Table 1 (reading R18): nearest x2 in y and x."""
    x = np.ascontiguousarray(x, dtype=np.int8)
    n, c, d, h, w = x.shape
    y = np.empty((n, c, d, 2 * h, 2 * w), dtype=np.int8)
    _load().oracle_upsample2_yx(x, n, c, d, h, w, y)
    return y


def concat(a, b):
    """Channel concatenation [a, b] (Table 1 skips)."""
    a = np.ascontiguousarray(a, dtype=np.int8)
    b = np.ascontiguousarray(b, dtype=np.int8)
    assert a.shape[0] == b.shape[0] and a.shape[2:] == b.shape[2:]
    n, ca = a.shape[:2]
    cb = b.shape[1]
    dhw = int(np.prod(a.shape[2:]))
    y = np.empty((n, ca + cb) + a.shape[2:], dtype=np.int8)
    _load().oracle_concat(a, ca, b, cb, n, dhw, y)
    return y


def predict(t, w, b):
    """1x1x1 float prediction layer (reading R12)."""
    t = np.ascontiguousarray(t, dtype=np.int8)
    w = np.ascontiguousarray(w, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    n, c = t.shape[:2]
    nclass = w.shape[0]
    assert w.shape == (nclass, c) and b.shape == (nclass,)
    dhw = int(np.prod(t.shape[2:]))
    out = np.empty((n, nclass) + t.shape[2:], dtype=np.float32)
    _load().oracle_predict(t, n, c, dhw, nclass, w, b, out)
    return out


# The oracle's own statement of the FCN (reading R9); (cin, cout, stride).
FCN_LAYERS = [(1, 16, 1), (16, 16, 1), (16, 16, 2), (16, 32, 1), (32, 32, 2), (32, 64, 1),
              (64, 64, 2), (64, 64, 1), (128, 64, 1), (64, 32, 1), (64, 32, 1), (32, 16, 1),
              (32, 16, 1), (16, 16, 1)]


def fcn_forward(x, t_lo, t_hi, weights, lo, hi, pred_w, pred_b, want_acts=False):
    """The ternary FCN (reading R9).
    x float32 [n,1,d,h,w] -> (logits float32 [n,2,d,h,w], acts list or None, bad)."""
    lib = _load()
    x = np.ascontiguousarray(x, dtype=np.float32)
    n, c, d, h, w = x.shape
    assert c == 1 and d % 8 == 0 and h % 8 == 0 and w % 8 == 0
    assert len(weights) == 14 and len(lo) == 14 and len(hi) == 14
    Ws = [np.ascontiguousarray(a, dtype=np.int8) for a in weights]
    Ls = [np.ascontiguousarray(a, dtype=np.int32) for a in lo]
    Hs = [np.ascontiguousarray(a, dtype=np.int32) for a in hi]
    for i, (ci, co, _) in enumerate(FCN_LAYERS):
        assert Ws[i].shape == (co, ci, 3, 3, 3), (i, Ws[i].shape)
        assert Ls[i].shape == (co,) and Hs[i].shape == (co,)
    vp = ctypes.c_void_p
    arr = lambda xs: (vp * len(xs))(*[a.ctypes.data for a in xs])
    logits = np.empty((n, 2, d, h, w), dtype=np.float32)
    acts = None
    acts_arg = None
    if want_acts:
        acts = []
        res ={1: (d, h, w), 2: (d // 2, h // 2, w // 2), 3: (d // 4, h // 4, w // 4),
               4: (d // 8, h // 8, w // 8)}
        level = [1, 1, 2, 2, 3, 3, 4, 4, 3, 3, 2, 2, 1, 1]
        for i, (ci, co, s) in enumerate(FCN_LAYERS):
            acts.append(np.empty((n, co) + res[level[i]], dtype=np.int8))
        acts_arg = ctypes.cast(arr(acts), ctypes.POINTER(vp))
    bad = lib.oracle_fcn_forward(
        x, n, d, h, w, float(t_lo), float(t_hi),
        ctypes.cast(arr(Ws), ctypes.POINTER(vp)), ctypes.cast(arr(Ls), ctypes.POINTER(vp)),
        ctypes.cast(arr(Hs), ctypes.POINTER(vp)),
        np.ascontiguousarray(pred_w, dtype=np.float32), np.ascontiguousarray(pred_b, dtype=np.float32),
        logits, acts_arg)
    return logits, acts, int(bad)


# --------------------------------------------------------------------------- model preparation (NEXT-3)
def ternarize_weights(w, sparsity=None):
    """Eq. 4: per output filter (axis 0), Delta = 0.7/n * sum|W_i|;
    code +1 if W_i > Delta, 0 if |W_i| <= Delta, -1 else; alpha = mean |W_i| over the
    nonzero codes (0 if none).  With sparsity in [0, 1):
    exactly ceil(sparsity*n) zeros at the smallest |W_i| (stable by index), the rest
    sign(W_i).  Plain float64 loops over filters."""
    w = np.asarray(w, dtype=np.float32)
    k = w.shape[0]
    flat = w.reshape(k, -1).astype(np.float64)
    n = flat.shape[1]
    codes = np.zeros(flat.shape, np.int8)
    alpha = np.zeros(k, np.float64)
    for f in range(k):
        row = flat[f]
        if sparsity is None:
            delta = 0.7 / n * float(np.sum(np.abs(row)))
            for i in range(n):
                v = row[i]
                codes[f, i] = 1 if v > delta else (0 if abs(v) <= delta else -1)
        else:
            nz = int(np.ceil(float(np.float32(sparsity)) * n))
            order = np.argsort(np.abs(row), kind="stable")
            codes[f] = np.where(row > 0, 1, -1)
            codes[f, order[:nz]] = 0
        sel = codes[f] != 0
        alpha[f] = float(np.sum(np.abs(row[sel]))) / int(sel.sum()) if sel.any() else 0.0
    return codes.reshape(w.shape), alpha.astype(np.float32)


def fold_table(alpha, gamma, beta, mean, var, eps, max_abs_acc):
    """The definition the folded thresholds must reproduce (readings R5/R6): for every
    channel c and every integer accumulator acc in [-A, A], the ternary output
    tern(y) of Eq. 6 with y = a*acc + b, a = gamma*alpha/sqrt(var+eps),
    b = beta - gamma*mean/sqrt(var+eps) in float64 (the conv output alpha*acc through
    batch norm).  Returns int8 [K, 2A+1] (column j <-> acc = j - A)."""
    k = len(alpha)
    acc = np.arange(-max_abs_acc, max_abs_acc + 1, dtype=np.float64)
    out = np.zeros((k, acc.size), np.int8)
    for c in range(k):
        sd = np.sqrt(np.float64(var[c]) + np.float64(np.float32(eps)))
        a = np.float64(gamma[c]) * np.float64(alpha[c]) / sd
        b = np.float64(beta[c]) - np.float64(gamma[c]) * np.float64(mean[c]) / sd
        y = a * acc + b
        out[c] = np.where(y > 0.5, 1, np.where(y < -0.5, -1, 0))
    return out


# --------------------------------------------------------------------------- NEXT-4: Table 1's 2.5D U-Net
# The paper's own network (Table 1) with ternary blocks, reading R18: each
# input is a stack of 15 neighbouring CT slices whose slices are the channels of
# layer #1 ("3x3x15"); every layer is a 2D conv (3x3, or 1x1 at the lowest level as the caption
# says); the three AvgPool2D rows are stride-2 convs (reading R8); Upsample2D is nearest x2 in y
# and x; skips #2->#13, #4->#11, #6->#9 concatenated [upsampled, skip]; same padding (R11);
# 2-class 1x1 float prediction (R12).  A 2D conv here is conv3d on one-plane volumes
# (d = 1, pad 1 in z: only the kernel's middle plane dz = 1 meets data), so the weights are
# [cout][cin][3][3][3] whose other planes do not contribute; 1x1 layers use the centre tap only.
# Entries: (cin, cout, kernel, stride, skip source or None).
FCN25_LAYERS = [(15, 32, 3, 1, None), (32, 64, 3, 1, None), (64, 64, 3, 2, None), (64, 128, 3, 1, None),
                (128, 128, 3, 2, None), (128, 256, 3, 1, None), (256, 256, 1, 2, None), (256, 256, 1, 1, None),
                (512, 256, 3, 1, 5), (256, 128, 3, 1, None), (256, 128, 3, 1, 3), (128, 64, 3, 1, None),
                (128, 64, 3, 1, 1), (64, 64, 3, 1, None)]


def fcn25_forward(x, t_lo, t_hi, weights, lo, hi, pred_w, pred_b, want_acts=False):
    """Table 1's ternary 2.5D U-Net (reading R18) on stacks x float32 [n][15][1][h][w]:
    Eq. 6 on the normalised slices, then the 14 blocks (conv -> integer-threshold requant)
    in table order, the decoder inputs being concat(upsample2_yx(previous), skip), then the
    1x1 prediction.  Plain composition of the pinned primitives above.
    Returns (logits [n][2][1][h][w], acts or None, bad index)."""
    t, bad = tern_f32(x, t_lo, t_hi)
    acts = []
    cur = t
    for i, (cin, cout, k, s, skip) in enumerate(FCN25_LAYERS):
        inp = concat(upsample2_yx(cur), acts[skip]) if skip is not None else cur
        assert inp.shape[1] == cin, (i, inp.shape, cin)
        acc = conv3d(inp, weights[i], stride=s, pad=1)
        cur = requant(acc, lo[i], hi[i])
        acts.append(cur)
    logits = predict(cur, pred_w, pred_b)
    return logits, (acts if want_acts else None), bad
