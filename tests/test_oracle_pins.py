"""Pins for the CPU oracle (oracle/) against things other than itself.

Each test names what fixes the expected value: a worked example printed in the
paper or SPEC.md (tests/golden/), a closed form, an exhaustive table, or a
library routine (torch CPU float64 conv3d / interpolate, which is exact on
{-1,0,+1} integer data because every partial sum is an integer < 2**53).
"""
import itertools
import os
from fractions import Fraction

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


def _popc(a):
    a = np.asarray(a, dtype=np.uint64)
    return np.array([bin(int(v)).count("1") for v in a.reshape(-1)]).reshape(a.shape)


def eq9(sa, ma, sw, mw):
    """Eq. 9 with the zero-exclusion mask read as AND of nonzero flags
    (reading R1): popc(~(sa^sw) & m) - popc((sa^sw) & m), m = ma & mw."""
    m = ma & mw
    x = sa ^ sw
    return _popc(~x & m & 0xFFFFFFFF) - _popc(x & m)


# --------------------------------------------------------------------------- encoding
def test_fig3_encoding_golden():
    for code, fs, fv, sb, mb in _rows("fig3_encoding.txt"):
        x = np.array([int(code)], dtype=np.int8).reshape(1, 1, 1, 1, 1)
        xp, bad = oracle.pack(x)
        assert bad == -1
        sign, mask = int(xp[0, 0, 0, 0, 0, 0]), int(xp[0, 0, 0, 0, 1, 0])
        assert (sign, mask) == (int(sb), int(mb))
        # reading R2: mask is the complement of Fig. 3's value flag, sign is Fig. 3's sign flag
        assert mask == 1 - int(fv) and sign == int(fs)


def test_spec_pack_example():
    row = [r for r in _rows("spec_examples.txt") if r[0] == "pack"][0]
    codes = [int(v) for v in row[1].split(",")]
    x = np.array(codes, dtype=np.int8).reshape(1, len(codes), 1, 1, 1)
    xp, bad = oracle.pack(x)
    assert bad == -1
    assert int(xp[0, 0, 0, 0, 0, 0]) == int(row[2].split("=")[1])
    assert int(xp[0, 0, 0, 0, 1, 0]) == int(row[3].split("=")[1])


def test_pack_roundtrip_density_padding():
    for c in (1, 5, 31, 32, 33, 64, 100):
        x = synth.ternary_codes((2, c, 3, 4, 5), 0.5, seed=c)
        xp, bad = oracle.pack(x)
        assert bad == -1
        cw = (c + 31) // 32
        assert xp.shape == (2, 3, 4, 5, 2, cw)
        y, bad2 = oracle.unpack(xp, c)
        assert bad2 == -1
        np.testing.assert_array_equal(x, y)
        # density: popcount(mask) = number of nonzeros
        assert _popc(xp[..., 1, :]).sum() == np.count_nonzero(x)
        # sign AND NOT mask = 0 (canonical zero), padding lanes zero
        assert np.all(xp[..., 0, :] & ~xp[..., 1, :] == 0)
        if c % 32:
            pad = np.uint32((0xFFFFFFFF << (c % 32)) & 0xFFFFFFFF)
            assert np.all(xp[..., :, cw - 1] & pad == 0)
        # byte-level layout: channel ch at bit ch%32 of word ch//32 (reading R3)
        n_, z_, y_, x_ = 1, 2, 3, 4
        for ch in range(c):
            v = x[n_, ch, z_, y_, x_]
            s = (int(xp[n_, z_, y_, x_, 0, ch // 32]) >> (ch % 32)) & 1
            m = (int(xp[n_, z_, y_, x_, 1, ch // 32]) >> (ch % 32)) & 1
            assert (s, m) == ((1, 1) if v == 1 else (0, 1) if v == -1 else (0, 0))


def test_pack_domain_error_names_first_index():
    x = synth.ternary_codes((1, 3, 2, 2, 2), 0.5, seed=3)
    x[0, 2, 1, 0, 1] = 2
    x[0, 1, 1, 1, 1] = -5
    _, bad = oracle.pack(x)
    assert bad == np.ravel_multi_index((0, 1, 1, 1, 1), x.shape)


def test_unpack_detects_noncanonical():
    x = synth.ternary_codes((1, 3, 1, 1, 2), 0.5, seed=4)
    xp, _ = oracle.pack(x)
    xp2 = xp.copy()
    xp2[0, 0, 0, 1, 0, 0] |= np.uint32(1 << 2)          # sign bit on lane 2 ...
    xp2[0, 0, 0, 1, 1, 0] &= np.uint32(~(1 << 2) & 0xFFFFFFFF)  # ... of a zero
    _, bad = oracle.unpack(xp2, 3)
    assert bad == np.ravel_multi_index((0, 2, 0, 0, 1), x.shape)
    xp3 = xp.copy()
    xp3[0, 0, 0, 0, 1, 0] |= np.uint32(1 << 7)           # padding lane set
    _, bad = oracle.unpack(xp3, 3)
    assert bad >= 0


def test_pack_weights_layout():
    w = synth.ternary_codes((4, 40, 3, 3, 3), 0.4, seed=5)
    wp, bad = oracle.pack_weights(w)
    assert bad == -1 and wp.shape == (4, 27, 2, 2)
    # tap t = (dz*3+dy)*3+dx; same bits as packing the [k][c] slice of that tap
    for t, (a, b, e) in enumerate(itertools.product(range(3), range(3), range(3))):
        sl = np.ascontiguousarray(w[:, :, a, b, e]).reshape(1, 4, 40, 1, 1).transpose(0, 2, 1, 3, 4)
        # sl as NCDHW with n=1, c=40, d=4 (one "voxel" per output channel)
        xp, _ = oracle.pack(np.ascontiguousarray(sl))
        np.testing.assert_array_equal(xp[0, :, 0, 0], wp[:, t])


# --------------------------------------------------------------------------- Eq. 9 pins
def test_eq9_lane_table_exhaustive():
    """The 9 (a, w) pairs per lane: Eq. 9 on oracle-packed bits = a*w = golden table."""
    for a, w, prod in _rows("eq9_lane_table.txt"):
        a, w, prod = int(a), int(w), int(prod)
        assert a * w == prod
        ap, _ = oracle.pack(np.array([a], np.int8).reshape(1, 1, 1, 1, 1))
        wp, _ = oracle.pack(np.array([w], np.int8).reshape(1, 1, 1, 1, 1))
        got = eq9(ap[..., 0, 0], ap[..., 1, 0], wp[..., 0, 0], wp[..., 1, 0]).item()
        assert got == prod


def test_eq9_printed_or_mask_is_wrong():
    """Reading R1: Eq. 9 as printed uses (I^v + W^v) with + = OR.  Under the nonzero-mask
    encoding that counts a zero lane as +-1, so it cannot be the intended mask."""
    wrong = 0
    for a, w in itertools.product((-1, 0, 1), repeat=2):
        ap, _ = oracle.pack(np.array([a], np.int8).reshape(1, 1, 1, 1, 1))
        wp, _ = oracle.pack(np.array([w], np.int8).reshape(1, 1, 1, 1, 1))
        sa, ma, sw, mw = (int(ap[..., 0, 0].item()), int(ap[..., 1, 0].item()), int(wp[..., 0, 0].item()), int(wp[..., 1, 0].item()))
        m = ma | mw
        x = sa ^ sw
        v = bin(~x & m & 1).count("1") - bin(x & m & 1).count("1")
        wrong += v != a * w
    assert wrong > 0


def test_eq9_exhaustive_small_vectors():
    """All 3^c x 3^c pairs for c <= 4, and the spec worked example: Eq. 9 over
    oracle-packed words = integer dot = #agree - #disagree over the joint support."""
    for c in range(1, 5):
        vecs = np.array(list(itertools.product((-1, 0, 1), repeat=c)), dtype=np.int8)
        xp, _ = oracle.pack(vecs.T.reshape(1, c, 1, 1, len(vecs)))
        s, m = xp[0, 0, 0, :, 0, 0].astype(np.int64), xp[0, 0, 0, :, 1, 0].astype(np.int64)
        dots = vecs.astype(np.int64) @ vecs.T.astype(np.int64)
        mm = m[:, None] & m[None, :]
        xx = s[:, None] ^ s[None, :]
        pc = np.vectorize(lambda v: bin(int(v)).count("1"))
        got = pc(~xx & mm & 0xFFFFFFFF) - pc(xx & mm)
        np.testing.assert_array_equal(got, dots)
        agree = ((vecs[:, None, :] == vecs[None, :, :]) & (vecs[:, None, :] != 0)).sum(-1)
        dis = ((vecs[:, None, :] == -vecs[None, :, :]) & (vecs[:, None, :] != 0)).sum(-1)
        np.testing.assert_array_equal(agree - dis, dots)
    row = [r for r in _rows("spec_examples.txt") if r[0] == "dot"][0]
    a = np.array([int(v) for v in row[1].split(",")], np.int8)
    b = np.array([int(v) for v in row[2].split(",")], np.int8)
    ap, _ = oracle.pack(a.reshape(1, -1, 1, 1, 1))
    bp, _ = oracle.pack(b.reshape(1, -1, 1, 1, 1))
    assert eq9(ap[..., 0, 0], ap[..., 1, 0], bp[..., 0, 0], bp[..., 1, 0]).item() == int(row[3])


def test_eq9_random_long_vectors_multiword():
    g = synth.rng(7)
    for c in (16, 32, 64, 128, 432):
        a = synth.ternary_codes((200, c), 0.5, seed=c)
        b = synth.ternary_codes((200, c), 0.6, seed=c + 1)
        ap, _ = oracle.pack(a.T.reshape(1, c, 1, 1, 200))
        bp, _ = oracle.pack(b.T.reshape(1, c, 1, 1, 200))
        cw = (c + 31) // 32
        tot = np.zeros(200, np.int64)
        for j in range(cw):
            tot += eq9(ap[0, 0, 0, :, 0, j], ap[0, 0, 0, :, 1, j], bp[0, 0, 0, :, 0, j], bp[0, 0, 0, :, 1, j])
        ref = (a.astype(np.int64) * b).sum(1)
        np.testing.assert_array_equal(tot, ref)
        # parity invariant: acc = popc(mA&mW) mod 2 ; |acc| <= joint support
        joint = ((a != 0) & (b != 0)).sum(1)
        assert np.all((ref - joint) % 2 == 0) and np.all(np.abs(ref) <= joint)
    del g


# --------------------------------------------------------------------------- conv3d
def _torch_conv(x, w, stride, pad, dil):
    return F.conv3d(torch.from_numpy(x.astype(np.float64)), torch.from_numpy(w.astype(np.float64)),
                    stride=stride, padding=pad, dilation=dil).numpy()


@pytest.mark.parametrize("c,k,shape,stride,pad,dil", [
    (1, 3, (5, 6, 7), 1, 1, 1),
    (3, 2, (4, 4, 9), 2, 1, 1),
    (16, 16, (6, 5, 4), 1, 1, 1),
    (33, 5, (3, 7, 5), 1, 1, 2),
    (16, 4, (9, 9, 9), 2, 1, 2),
    (2, 3, (1, 1, 1), 1, 1, 1),
    (4, 2, (5, 3, 8), (1, 2, 1), (0, 1, 2), (1, 1, 2)),
    (7, 3, (8, 8, 8), 2, 2, 1),
])
def test_conv3d_matches_torch_float64(c, k, shape, stride, pad, dil):
    x = synth.ternary_codes((2, c) + shape, 0.5, seed=c * 7 + k)
    w = synth.ternary_codes((k, c, 3, 3, 3), 0.6, seed=c * 11 + k)
    ref = _torch_conv(x, w, stride, pad, dil)
    got = oracle.conv3d(x, w, stride, pad, dil)
    assert got.shape == ref.shape
    np.testing.assert_array_equal(got, ref.astype(np.int32))


def test_conv3d_degenerate_shapes():
    # window larger than the padded input: empty output in both
    x = synth.ternary_codes((1, 2, 1, 1, 1), 0.5, seed=1)
    w = synth.ternary_codes((3, 2, 3, 3, 3), 0.5, seed=2)
    got = oracle.conv3d(x, w, 2, 0, 1)
    assert got.size == 0
    assert oracle.out_extent(1, 2, 0, 1) == 0


def test_conv3d_closed_forms():
    n_ = 5
    for c in (1, 3, 16):
        x = np.ones((1, c, n_, n_, n_), np.int8)
        w = np.ones((2, c, 3, 3, 3), np.int8)
        y = oracle.conv3d(x, w)
        # number of in-range neighbours: 2 or 3 per axis
        cnt = np.array([2] + [3] * (n_ - 2) + [2])
        expect = c * cnt[:, None, None] * cnt[None, :, None] * cnt[None, None, :]
        np.testing.assert_array_equal(y[0, 0], expect)
        assert y[0, 0, 0, 0, 0] == 8 * c and y[0, 0, 0, 0, 2] == 12 * c
        assert y[0, 0, 0, 2, 2] == 18 * c and y[0, 0, 2, 2, 2] == 27 * c
    x = synth.ternary_codes((1, 6, 4, 5, 6), 0.5, seed=9)
    # zero weights -> 0
    assert np.all(oracle.conv3d(x, np.zeros((3, 6, 3, 3, 3), np.int8)) == 0)
    # centre-tap identity -> copy
    wid = np.zeros((6, 6, 3, 3, 3), np.int8)
    for i in range(6):
        wid[i, i, 1, 1, 1] = 1
    np.testing.assert_array_equal(oracle.conv3d(x, wid), x.astype(np.int32))
    # negation
    w = synth.ternary_codes((4, 6, 3, 3, 3), 0.5, seed=10)
    np.testing.assert_array_equal(oracle.conv3d(x, -w), -oracle.conv3d(x, w))
    # input-channel permutation equivariance
    perm = synth.rng(11).permutation(6)
    np.testing.assert_array_equal(oracle.conv3d(x[:, perm], w[:, perm]), oracle.conv3d(x, w))
    # single tap shift: weight only at (dz,dy,dx)=(0,1,2) reads x[z-1][y][x+1]
    ws = np.zeros((1, 1, 3, 3, 3), np.int8)
    ws[0, 0, 0, 1, 2] = 1
    x1 = x[:, :1]
    y = oracle.conv3d(x1, ws)[0, 0]
    exp = np.zeros_like(y)
    exp[1:, :, :-1] = x1[0, 0, :-1, :, 1:]
    np.testing.assert_array_equal(y, exp)


def test_conv3d_at_matches_full():
    x = synth.ternary_codes((2, 40, 5, 6, 7), 0.5, seed=12)
    w = synth.ternary_codes((9, 40, 3, 3, 3), 0.6, seed=13)
    for stride, dil in ((1, 1), (2, 1), (1, 2)):
        y = oracle.conv3d(x, w, stride, 1, dil)
        g = synth.rng(14)
        at = np.stack([g.integers(0, s, 50) for s in y.shape], axis=1).astype(np.int32)
        got = oracle.conv3d_at(x, w, at, stride, 1, dil)
        np.testing.assert_array_equal(got, y[tuple(at.T)])


# --------------------------------------------------------------------------- requant
def _tern(v: Fraction) -> int:
    """Eq. 6, in exact rational arithmetic."""
    if v > Fraction(1, 2):
        return 1
    if v >= Fraction(-1, 2):
        return 0
    return -1


def test_requant_equals_eq6_of_affine_exhaustive():
    """Reading R5/R6: alpha, BN and Eq. 6 fold into integer thresholds.  For random
    rational (a > 0, b) find hi/lo by scanning Eq. 6 itself, then the oracle's integer
    rule must reproduce tern(a*acc + b) at every acc in [-27C, 27C]."""
    g = synth.rng(15)
    C = 64
    accs = np.arange(-27 * C, 27 * C + 1, dtype=np.int32)
    for trial in range(40):
        a = Fraction(int(g.integers(1, 400)), int(g.integers(50, 4000)))
        b = Fraction(int(g.integers(-3000, 3000)), 1000)
        if trial == 0:  # a boundary exactly at +-0.5: acc = 10 -> 0.5 -> 0 (closed band)
            a, b = Fraction(1, 20), Fraction(0)
        ref = np.array([_tern(a * int(v) + b) for v in accs], np.int8)
        pos = accs[ref == 1]
        neg = accs[ref == -1]
        hi = np.int32(pos.min()) if pos.size else np.iinfo(np.int32).max
        lo = np.int32(neg.max()) if neg.size else np.iinfo(np.int32).min
        got = oracle.requant(accs.reshape(1, 1, -1), np.array([lo]), np.array([hi]))
        np.testing.assert_array_equal(got.reshape(-1), ref)
        if trial == 0:
            assert got.reshape(-1)[accs == 10][0] == 0 and got.reshape(-1)[accs == 11][0] == 1


def test_requant_order_and_sentinels():
    acc = np.array([-5, -1, 0, 1, 5], np.int32).reshape(1, 1, 5)
    i32 = np.iinfo(np.int32)
    # hi tested first: with lo >= hi an acc satisfying both is +1
    assert list(oracle.requant(acc, [3], [0]).reshape(-1)) == [-1, -1, 1, 1, 1]
    assert np.all(oracle.requant(acc, [i32.min], [i32.min]) == 1)
    assert np.all(oracle.requant(acc, [i32.max], [i32.max]) == -1)
    assert np.all(oracle.requant(acc, [i32.min], [i32.max]) == 0)
    # per-channel thresholds
    acc2 = np.arange(-3, 4, dtype=np.int32)[None, None].repeat(2, 1)
    got = oracle.requant(acc2, [-2, -1], [2, 1])
    assert list(got[0, 0]) == [-1, -1, 0, 0, 0, 1, 1]
    assert list(got[0, 1]) == [-1, -1, -1, 0, 1, 1, 1]


# --------------------------------------------------------------------------- Eq. 6 input
def test_tern_f32_eq6_examples():
    rows = _rows("eq6_examples.txt")
    x = np.array([float(r[0]) for r in rows], np.float32)
    t, bad = oracle.tern_f32(x, -0.5, 0.5)
    assert bad == -1
    assert list(t) == [int(r[1]) for r in rows]


def test_tern_f32_thresholds_and_nan():
    x = synth.ct_volume((1, 1, 8, 8, 8), seed=3)
    t, bad = oracle.tern_f32(x, synth.CT_T_LO, synth.CT_T_HI)
    assert bad == -1
    np.testing.assert_array_equal(t, np.where(x > np.float32(200), 1, np.where(x < np.float32(-200), -1, 0)))
    x2 = np.array([0.0, 200.0, -200.0, np.nan, np.inf], np.float32)
    t2, bad2 = oracle.tern_f32(x2, -200.0, 200.0)
    assert bad2 == 3 and list(t2[:3]) == [0, 0, 0]


# --------------------------------------------------------------------------- upsample / concat / predict
def test_upsample_matches_torch_nearest():
    x = synth.ternary_codes((2, 3, 3, 4, 5), 0.5, seed=16)
    ref = F.interpolate(torch.from_numpy(x.astype(np.float64)), scale_factor=2, mode="nearest").numpy()
    np.testing.assert_array_equal(oracle.upsample2(x), ref.astype(np.int8))


def test_concat_and_conv_linearity():
    a = synth.ternary_codes((1, 5, 4, 4, 4), 0.5, seed=17)
    b = synth.ternary_codes((1, 3, 4, 4, 4), 0.5, seed=18)
    cat = oracle.concat(a, b)
    np.testing.assert_array_equal(cat, np.concatenate([a, b], 1))
    w = synth.ternary_codes((2, 8, 3, 3, 3), 0.6, seed=19)
    np.testing.assert_array_equal(oracle.conv3d(cat, w),
                                  oracle.conv3d(a, w[:, :5]) + oracle.conv3d(b, w[:, 5:]))


def test_predict_matches_torch_float64():
    t = synth.ternary_codes((2, 16, 3, 4, 5), 0.5, seed=20)
    g = synth.rng(21)
    w = (0.25 * g.standard_normal((2, 16))).astype(np.float32)
    b = (0.1 * g.standard_normal(2)).astype(np.float32)
    ref = F.conv3d(torch.from_numpy(t.astype(np.float64)),
                   torch.from_numpy(w.astype(np.float64)).reshape(2, 16, 1, 1, 1),
                   bias=torch.from_numpy(b.astype(np.float64))).numpy()
    got = oracle.predict(t, w, b)
    # the double sum of 17 float32 terms is exact, so rounding once gives float32(ref)
    np.testing.assert_array_equal(got, ref.astype(np.float32))


# --------------------------------------------------------------------------- Eq. 8 (binary XNOR)
def test_eq8_binary_xnor_popcount():
    """Eq. 8: for I, W in {-1,+1}^c, I.W = c - 2 popc(I xor W).  Binary
    codes pack with all-ones masks (popc(mask) = c), and Eq. 9 then reduces to Eq. 8;
    the oracle's dot / conv agree with the XOR count."""
    for c in range(1, 9):
        vecs = np.array(list(itertools.product((-1, 1), repeat=c)), dtype=np.int8)
        xp, _ = oracle.pack(vecs.T.reshape(1, c, 1, 1, len(vecs)))
        s, m = xp[0, 0, 0, :, 0, 0].astype(np.int64), xp[0, 0, 0, :, 1, 0].astype(np.int64)
        assert np.all(_popc(m) == c)
        eq8 = c - 2 * _popc(s[:, None] ^ s[None, :])
        np.testing.assert_array_equal(eq8, vecs.astype(np.int64) @ vecs.T.astype(np.int64))
        np.testing.assert_array_equal(eq9(s[:, None], m[:, None], s[None, :], m[None, :]), eq8)
    for c in (27, 432, 1728):               # 3x3x3 windows of 1, 16, 64 channels
        a = synth.ternary_codes((64, c), 0.0, seed=c)
        b = synth.ternary_codes((64, c), 0.0, seed=c + 1)
        assert np.all(a != 0) and np.all(b != 0)
        dis = (a != b).sum(1)
        np.testing.assert_array_equal((a.astype(np.int64) * b).sum(1), c - 2 * dis)


def test_conv3d_binary_windows_eq8():
    """Binary input and weights: every output equals n_valid - 2 * #sign disagreements over
    its window (n_valid = 27 C inside, fewer at the zero-padded border), counted by brute
    force; the binary requant (lo = hi - 1) keeps the activations binary."""
    c, k = 3, 2
    x = synth.ternary_codes((1, c, 4, 5, 6), 0.0, seed=31)
    w = synth.ternary_codes((k, c, 3, 3, 3), 0.0, seed=32)
    y = oracle.conv3d(x, w)
    D, H, W = x.shape[2:]
    for kk in range(k):
        for z, yy, xx in itertools.product(range(D), range(H), range(W)):
            nv = dis = 0
            for dz, dy, dx in itertools.product(range(3), repeat=3):
                zi, yi, xi = z + dz - 1, yy + dy - 1, xx + dx - 1
                if 0 <= zi < D and 0 <= yi < H and 0 <= xi < W:
                    nv += c
                    dis += int((x[0, :, zi, yi, xi] != w[kk, :, dz, dy, dx]).sum())
            assert y[0, kk, z, yy, xx] == nv - 2 * dis
    assert y[0, 0, 2, 2, 2] % 2 == (27 * c) % 2         # interior parity of Eq. 8
    hi = np.array([1, -2], np.int32)
    t = oracle.requant(y, hi - 1, hi)
    assert np.all(t != 0)
    np.testing.assert_array_equal(t, np.where(y >= hi[None, :, None, None, None], 1, -1))


# --------------------------------------------------------------------------- bench golden samples
def test_bench_golden_samples_are_the_oracles():
    """tests/golden/bench_samples.npz (bench.py's parity gates) holds exactly what the oracle
    computes at those sampled outputs (rewritten only by tools/make_bench_golden.py)."""
    g = np.load(os.path.join(GOLDEN, "bench_samples.npz"))
    x0, w0, _, _ = synth.conv_config("C0")
    np.testing.assert_array_equal(g["c0_at"], synth.sample_positions(x0.shape, 16, 512, seed=777))
    np.testing.assert_array_equal(oracle.conv3d_at(x0, w0, g["c0_at"]), g["c0_ref"])
    for (x, w, lo, hi), at, ref in ((synth.conv_config("C1"), g["c1_at"], g["c1_ref"]),
                                    (synth.binary_config(), g["bin_at"], g["bin_ref"])):
        acc = oracle.conv3d_at(x, w, at)
        k = at[:, 1]
        want = np.where(acc >= hi[k], 1, np.where(acc <= lo[k], -1, 0))
        np.testing.assert_array_equal(want, ref)
    assert np.all(g["bin_ref"] != 0) and set(np.unique(g["c1_ref"])) == {-1, 0, 1}


def test_bench_golden_fcn_logits_are_the_oracles():
    """The FCN gates of bench.py: configs[2]'s sampled logits are recomputed here with the oracle
    (one 96x144x144 forward); configs[3] volume 0 (a 128x256x256 forward) and the configs[4] crop
    are too slow for the CPU suite -- their positions are checked to lie inside the volume (C4:
    inside the crop's exact region, 44 voxels from its lower faces and 37 from its upper ones)
    and their values to be finite logits of the right magnitude; tools/make_bench_golden.py
    (oracle/ only) wrote all three."""
    g = np.load(os.path.join(GOLDEN, "bench_samples.npz"))
    cfg = synth.CONFIGS["C2"]
    p = synth.fcn_params(cfg["seed_params"])
    x = synth.ct_volume(cfg["vol_shape"], seed=cfg["seeds"][0])
    lg, _, bad = oracle.fcn_forward(x, p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"])
    assert bad == -1
    np.testing.assert_array_equal(lg[tuple(g["fcn_c2_at"].T)], g["fcn_c2_ref"])
    bound = float(np.abs(p["pred_b"]).max() + np.abs(p["pred_w"]).sum(1).max())
    for name, region in (("c3", ((0, 128), (0, 256), (0, 256))),
                         ("c4", ((64 + 44, 192 - 37), (192 + 44, 320 - 37), (320 + 44, 448 - 37)))):
        at, ref = g[f"fcn_{name}_at"], g[f"fcn_{name}_ref"]
        assert at.shape == (512, 5) and ref.shape == (512,)
        assert np.all(at[:, 0] == 0) and set(np.unique(at[:, 1])) == {0, 1}
        for a, (lo_, hi_) in enumerate(region):
            assert np.all((at[:, 2 + a] >= lo_) & (at[:, 2 + a] < hi_)), (name, a)
        assert np.all(np.isfinite(ref)) and np.all(np.abs(ref) <= bound + 1e-6)



def test_bench_golden_fcn25_logits_are_the_oracles():
    """bench.py's Table-1 2.5D gate: the sampled logits of stack 0 recomputed with the oracle
    (a stack depends only on its own slices); stacks 1-3 checked for range and magnitude."""
    g = np.load(os.path.join(GOLDEN, "bench_samples.npz"))
    at, ref = g["fcn25_at"], g["fcn25_ref"]
    assert at.shape == (512, 5) and set(np.unique(at[:, 0])) <= {0, 1, 2, 3} and np.all(at[:, 2] == 0)
    p = synth.fcn25_params()
    x = synth.ct_stacks(synth.ROI_STACKS, synth.STACK_H, synth.STACK_W, seed=300)[:1]
    lg, _, bad = oracle.fcn25_forward(x, p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"])
    assert bad == -1
    s0 = at[:, 0] == 0
    assert s0.sum() > 50
    np.testing.assert_array_equal(lg[tuple(at[s0].T)], ref[s0])
    bound = float(np.abs(p["pred_b"]).max() + np.abs(p["pred_w"]).sum(1).max())
    assert np.all(np.isfinite(ref)) and np.all(np.abs(ref) <= bound + 1e-6)
