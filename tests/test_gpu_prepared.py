"""Prepared filter banks (tn_conv_prepare, include/tn.h): a conv that copies the prebuilt B image
gives the same words as the unprepared call and the oracle (Eq. 9), bit-exact;
a prepared call whose plan does not match the image (other bank, other selector) stays correct."""
import zlib

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

CASES = [
    # (x shape NCDHW, k, stride, pad, dil)
    ((1, 16, 9, 17, 34), 16, 1, 1, 1),
    ((2, 32, 7, 10, 22), 32, 1, 1, 1),
    ((1, 64, 6, 10, 12), 32, 1, 1, 1),
    ((1, 32, 5, 6, 8), 64, 1, 1, 1),
    ((1, 64, 11, 20, 30), 64, 1, 1, 1),
    ((1, 16, 12, 18, 20), 16, 2, 1, 1),
    ((1, 64, 10, 12, 14), 64, 2, 1, 1),
    ((1, 33, 6, 7, 8), 5, 1, 1, 1),
    ((1, 48, 5, 6, 11), 16, 1, 1, 1),
    ((1, 32, 10, 14, 16), 32, 1, 3, 3),
    ((1, 64, 9, 40, 36), 24, 1, 2, 2),
    ((1, 128, 4, 5, 6), 16, 1, 1, 1),            # popc shape: a handle without an image
]


@pytest.fixture(scope="module")
def tn():
    import paper_1801_09449_b200 as tn
    return tn


@pytest.fixture(params=[3, 4, 0], ids=["tz", "tz8", "auto"])
def selector(request, tn):
    tn.tn_set_conv_kernel(request.param)
    yield request.param
    tn.tn_set_conv_kernel(tn.TN_KERNEL_AUTO)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def _inputs(shape, k):
    seed = zlib.crc32(str((shape, k)).encode()) % 1000
    x = synth.ternary_codes(shape, 0.5, seed=seed)
    w = synth.ternary_codes((k, shape[1], 3, 3, 3), 0.6, seed=seed + 1)
    lo, hi = synth.jittered_thresholds(k, synth.threshold_base(shape[1], 0.5), seed=k)
    return x, w, lo, hi


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[0])) + f"_k{c[1]}_s{c[2]}_d{c[4]}")
def test_prepared_conv_matches_oracle(tn, selector, case):
    shape, k, s, p, dl = case
    x, w, lo, hi = _inputs(shape, k)
    g = tn.geom(s, p, dl)
    xd = tn.dims(*shape)
    acc = oracle.conv3d(x, w, s, p, dl)
    ref, _ = oracle.pack(oracle.requant(acc, lo, hi))
    xp, wp = tn.tn_pack_i8(dev(x)), tn.tn_pack_weights(dev(w))
    on_tz = tn.tn_conv_kernel_for([xd], k, g) == tn.TN_KERNEL_TZ
    if selector == 3 and not on_tz:
        pytest.skip("shape outside the tensor-core kernel")
    prep = tn.tn_conv_prepare([(None, xd, 0, wp)], k, g, requant=True)
    assert (prep.nbytes > 0) == on_tz
    yp = tn.tn_conv3d_requant_prepared(prep, xp, xd, wp, k, g, dev(lo), dev(hi))
    np.testing.assert_array_equal(u32(yp), ref)
    # twice in a row on one stream (the image is read-only), and the int32 form
    yp2 = tn.tn_conv3d_requant_prepared(prep, xp, xd, wp, k, g, dev(lo), dev(hi))
    np.testing.assert_array_equal(u32(yp2), ref)
    prep_i = tn.tn_conv_prepare([(xp, xd, 0, wp)], k, g, requant=False)
    y = tn.tn_conv3d_seg_prepared(prep_i, [(xp, xd, 0, wp)], k, g, requant=False)
    np.testing.assert_array_equal(y.cpu().numpy(), acc.transpose(0, 2, 3, 4, 1))
    prep.close()
    prep_i.close()


def test_prepared_image_of_another_bank_is_not_used(tn):
    """The image belongs to the bank pointer it was built from: a call with another bank (or after a
    selector change) stages that bank as the unprepared call does."""
    shape, k = (1, 64, 6, 10, 12), 64
    x, w, lo, hi = _inputs(shape, k)
    w2 = synth.ternary_codes(w.shape, 0.6, seed=999)
    xd, g = tn.dims(*shape), tn.geom()
    xp, wp, wp2 = tn.tn_pack_i8(dev(x)), tn.tn_pack_weights(dev(w)), tn.tn_pack_weights(dev(w2))
    prep = tn.tn_conv_prepare([(None, xd, 0, wp)], k, g)
    assert prep.nbytes > 0
    ref2, _ = oracle.pack(oracle.requant(oracle.conv3d(x, w2), lo, hi))
    np.testing.assert_array_equal(u32(tn.tn_conv3d_requant_prepared(prep, xp, xd, wp2, k, g, dev(lo), dev(hi))),
                                  ref2)
    ref, _ = oracle.pack(oracle.requant(oracle.conv3d(x, w), lo, hi))
    try:
        tn.tn_set_conv_kernel(4)   # int8 operands: the FP4 image does not match
        np.testing.assert_array_equal(u32(tn.tn_conv3d_requant_prepared(prep, xp, xd, wp, k, g, dev(lo),
                                                                         dev(hi))), ref)
    finally:
        tn.tn_set_conv_kernel(0)
    np.testing.assert_array_equal(u32(tn.tn_conv3d_requant_prepared(None, xp, xd, wp, k, g, dev(lo), dev(hi))),
                                  ref)
    prep.close()


@pytest.mark.parametrize("low,cl,cs,k,up", [((3, 4, 5), 16, 16, 16, 1), ((4, 5, 6), 64, 64, 64, 1),
                                            ((4, 3, 6), 16, 32, 16, 1), ((3, 5, 4), 32, 32, 32, 2)])
def test_prepared_upsample_concat(tn, low, cl, cs, k, up):
    n = 1
    a = synth.ternary_codes((n, cl) + low, 0.5, seed=cl)
    hi_shape = (low[0] * (2 if up == 1 else 1), 2 * low[1], 2 * low[2])
    b = synth.ternary_codes((n, cs) + hi_shape, 0.5, seed=cs + 1)
    w = synth.ternary_codes((k, cl + cs, 3, 3, 3), 0.6, seed=k + 2)
    lo, hi = synth.jittered_thresholds(k, synth.threshold_base(cl + cs, 0.5), seed=3)
    ua = oracle.upsample2(a) if up == 1 else oracle.upsample2_yx(a)
    ref, _ = oracle.pack(oracle.requant(oracle.conv3d(oracle.concat(ua, b), w), lo, hi))
    ap, bp = tn.tn_pack_i8(dev(a)), tn.tn_pack_i8(dev(b))
    wa = tn.tn_pack_weights(dev(np.ascontiguousarray(w[:, :cl])))
    wb = tn.tn_pack_weights(dev(np.ascontiguousarray(w[:, cl:])))
    segs = [(ap, tn.dims(n, cl, *low), up, wa), (bp, tn.dims(n, cs, *hi_shape), 0, wb)]
    prep = tn.tn_conv_prepare(segs, k, tn.geom())
    assert prep.nbytes > 0
    yp = tn.tn_conv3d_seg_prepared(prep, segs, k, tn.geom(), dev(lo), dev(hi))
    np.testing.assert_array_equal(u32(yp), ref)


def _logit_tol(w, b):   # reading R13 (as in test_gpu_parity.py)
    return 1e-5 * (np.abs(b)[None, :, None, None, None] + np.abs(w).sum(1)[None, :, None, None, None])


@pytest.mark.parametrize("shape,prep_shape", [((2, 1, 16, 24, 40), (2, 1, 16, 24, 40)),
                                              ((1, 1, 32, 48, 48), (1, 1, 8, 8, 8))])
def test_prepared_fcn_matches_oracle(tn, shape, prep_shape):
    """tn_fcn_prepare (for this input's dims, or other dims: the images do not depend on the
    extents) then forward: every stored layer bit-exact against the oracle, logits within R13."""
    p = synth.fcn_params()
    x = synth.ct_volume(shape, seed=shape[3])
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
    nbytes = net.prepare(prep_shape)
    assert nbytes > 0
    ws = net.workspace(x.shape)
    got = net(dev(x), ws=ws).cpu().numpy()
    ref_logits, acts, _ = oracle.fcn_forward(x, p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"],
                                             p["pred_w"], p["pred_b"], want_acts=True)
    for i in range(13):
        view, _ = net.layer_output(x.shape, ws, i)
        np.testing.assert_array_equal(u32(view), oracle.pack(acts[i])[0], err_msg=f"layer #{i + 1}")
    tol = np.maximum(np.abs(ref_logits), _logit_tol(p["pred_w"], p["pred_b"]) / 1e-5) * 1e-5
    assert np.all(np.abs(got - ref_logits) <= tol)
    # the z-slab schedule reads the same images
    if shape[0] == 1:
        np.testing.assert_array_equal(net.forward_slabs_local(dev(x), 2).cpu().numpy(), got)


def test_prepared_fcn25_matches_oracle(tn):
    p = synth.fcn25_params()
    x = synth.ct_stacks(5, 48, 64, seed=12)[1:4]
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"],
                        table=tn.fcn25_table(), c_in=15)
    assert net.prepare(x.shape) > 0
    ws = net.workspace(x.shape)
    got = net(dev(x), ws=ws).cpu().numpy()
    ref_logits, acts, _ = oracle.fcn25_forward(x, p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"],
                                               p["pred_w"], p["pred_b"], want_acts=True)
    for i in range(14):
        view, _ = net.layer_output(x.shape, ws, i)
        np.testing.assert_array_equal(u32(view), oracle.pack(acts[i])[0], err_msg=f"layer #{i + 1}")
    tol = np.maximum(np.abs(ref_logits), _logit_tol(p["pred_w"], p["pred_b"]) / 1e-5) * 1e-5
    assert np.all(np.abs(got - ref_logits) <= tol)
