"""The wide one-plane layers of Table 1 (reading R18; TN_KERNEL_WIDE in include/tn.h): C a multiple
of 64 per segment with C or K beyond 64, K <= 256, stride 1 / 2, [up2d | skip] segments, on the
tcgen05 kernel with FP4 operands (conv_wide.cu).  Every int32 accumulator and packed word equals
the oracle's Eq. 9 conv bit for bit, prepared (tap-skipping image) or not."""
import zlib

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tn():
    import paper_1801_09449_b200 as tn
    return tn


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def u32(t):
    return t.cpu().numpy().view(np.uint32)


CASES = [
    # (n, c, h, w, k, stride)
    ((2, 64, 17, 22), 128, 1),      # Table 1 #4 shape class, ragged tiles
    ((1, 128, 30, 22), 128, 2),     # #5: stride 2
    ((2, 128, 15, 11), 256, 1),     # #6: two output-channel groups
    ((1, 256, 8, 12), 256, 1),
    ((3, 128, 9, 40), 64, 1),       # #12: K = 64 (N = 64, three tiles per strip)
    ((1, 512, 6, 7), 192, 1),       # K not a multiple of 128, C = 512
    ((2, 64, 3, 300), 96, 1),       # wide rows, several strips per plane
    ((1, 256, 12, 16), 256, 2),
    ((2, 64, 13, 40), 64, 1),       # #14: 64 -> 64 at stride 1 (N = 64, seven tiles per strip)
]


def _data(shape, k, seed, centre_only=False):
    n, c, h, w = shape
    x = synth.ternary_codes((n, c, 1, h, w), 0.5, seed=seed)
    wt = synth.ternary_codes((k, c, 3, 3, 3), 0.6, seed=seed + 1)
    if centre_only:
        m = np.zeros_like(wt)
        m[:, :, 1, 1, 1] = wt[:, :, 1, 1, 1]
        wt = m
    lo, hi = synth.jittered_thresholds(k, synth.threshold_base(c, 0.5, taps=1 if centre_only else 9), seed=k)
    return x, wt, lo, hi


@pytest.mark.parametrize("prepared", [False, True], ids=["per_call", "prepared"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[0])) + f"_k{c[1]}_s{c[2]}")
def test_wide_conv_matches_oracle(tn, case, prepared):
    shape, k, s = case
    x, wt, lo, hi = _data(shape, k, zlib.crc32(str(case).encode()) % 1000)
    xd, g = tn.dims(*x.shape), tn.geom(s)
    assert tn.tn_conv_kernel_for([xd], k, g) == tn.TN_KERNEL_WIDE
    acc = oracle.conv3d(x, wt, s, 1, 1)
    ref, _ = oracle.pack(oracle.requant(acc, lo, hi))
    xp, wp = tn.tn_pack_i8(dev(x)), tn.tn_pack_weights(dev(wt))
    segs = [(xp, xd, 0, wp)]
    prep = tn.tn_conv_prepare(segs, k, g) if prepared else None
    if prepared:
        assert prep.nbytes > 0
    yp = tn.tn_conv3d_seg_prepared(prep, segs, k, g, dev(lo), dev(hi))
    np.testing.assert_array_equal(u32(yp), ref)
    prep_i = tn.tn_conv_prepare(segs, k, g, requant=False) if prepared else None
    y = tn.tn_conv3d_seg_prepared(prep_i, segs, k, g, requant=False)
    np.testing.assert_array_equal(y.cpu().numpy(), acc.transpose(0, 2, 3, 4, 1))


@pytest.mark.parametrize("s", [1, 2])
def test_wide_centre_tap_filters(tn, s):
    """Table 1's 1x1 layers #7 / #8 as centre-tap filters: the prepared image keeps one tap (one MMA
    per chunk), the per-call image all nine; both equal the oracle."""
    shape, k = (2, 256, 10, 14), 256
    x, wt, lo, hi = _data(shape, k, 40 + s, centre_only=True)
    xd, g = tn.dims(*x.shape), tn.geom(s)
    ref, _ = oracle.pack(oracle.requant(oracle.conv3d(x, wt, s, 1, 1), lo, hi))
    xp, wp = tn.tn_pack_i8(dev(x)), tn.tn_pack_weights(dev(wt))
    segs = [(xp, xd, 0, wp)]
    prep = tn.tn_conv_prepare(segs, k, g)
    full = tn.tn_conv_prepare([(xp, xd, 0, tn.tn_pack_weights(dev(_data(shape, k, 7)[1])))], k, g)
    assert 0 < prep.nbytes and 9 * prep.nbytes == full.nbytes   # one active tap of nine
    np.testing.assert_array_equal(u32(tn.tn_conv3d_seg_prepared(prep, segs, k, g, dev(lo), dev(hi))), ref)
    np.testing.assert_array_equal(u32(tn.tn_conv3d_seg_prepared(None, segs, k, g, dev(lo), dev(hi))), ref)


@pytest.mark.parametrize("low,cl,cs,k", [((6, 5), 256, 256, 256), ((7, 9), 128, 128, 128), ((5, 11), 64, 64, 128)])
def test_wide_upsample_concat(tn, low, cl, cs, k):
    """Table 1's decoder rows #9 / #11: [nearest x2 in y and x of the coarse map | skip]."""
    n = 2
    a = synth.ternary_codes((n, cl, 1) + low, 0.5, seed=cl)
    b = synth.ternary_codes((n, cs, 1, 2 * low[0], 2 * low[1]), 0.5, seed=cs + 1)
    wt = synth.ternary_codes((k, cl + cs, 3, 3, 3), 0.6, seed=k + 2)
    lo, hi = synth.jittered_thresholds(k, synth.threshold_base(cl + cs, 0.5, taps=9), seed=3)
    acc = oracle.conv3d(oracle.concat(oracle.upsample2_yx(a), b), wt)
    ref, _ = oracle.pack(oracle.requant(acc, lo, hi))
    ap, bp = tn.tn_pack_i8(dev(a)), tn.tn_pack_i8(dev(b))
    wa = tn.tn_pack_weights(dev(np.ascontiguousarray(wt[:, :cl])))
    wb = tn.tn_pack_weights(dev(np.ascontiguousarray(wt[:, cl:])))
    segs = [(ap, tn.dims(n, cl, 1, *low), 2, wa), (bp, tn.dims(n, cs, 1, 2 * low[0], 2 * low[1]), 0, wb)]
    assert tn.tn_conv_kernel_for([d for _, d, _, _ in segs], k, tn.geom(), [2, 0]) == tn.TN_KERNEL_WIDE
    for prep in (None, tn.tn_conv_prepare(segs, k, tn.geom())):
        np.testing.assert_array_equal(u32(tn.tn_conv3d_seg_prepared(prep, segs, k, tn.geom(), dev(lo), dev(hi))), ref)
    y = tn.tn_conv3d_seg(segs, k, tn.geom(), requant=False)
    np.testing.assert_array_equal(y.cpu().numpy(), acc.transpose(0, 2, 3, 4, 1))


def test_wide_grid_capped_and_zero_bank(tn):
    """Few CTAs walking many units (ring wrap-around, both TMEM buffers), and an all-zero filter
    bank (no active tap: every output is 0, or the sentinel thresholds' constant)."""
    shape, k = (3, 128, 20, 30), 128
    x, wt, lo, hi = _data(shape, k, 77)
    xd, g = tn.dims(*x.shape), tn.geom()
    ref, _ = oracle.pack(oracle.requant(oracle.conv3d(x, wt), lo, hi))
    xp, wp = tn.tn_pack_i8(dev(x)), tn.tn_pack_weights(dev(wt))
    try:
        tn.tn_set_grid_cap(3)
        np.testing.assert_array_equal(u32(tn.tn_conv3d_requant(xp, xd, wp, k, g, dev(lo), dev(hi))), ref)
    finally:
        tn.tn_set_grid_cap(0)
    wz = tn.tn_pack_weights(dev(np.zeros_like(wt)))
    prep = tn.tn_conv_prepare([(xp, xd, 0, wz)], k, g)
    y = tn.tn_conv3d_seg_prepared(prep, [(xp, xd, 0, wz)], k, g, requant=False)
    assert not y.cpu().numpy().any()
