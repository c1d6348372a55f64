"""GPU parity: every C-ABI entry point against the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): bit-exact for packed words and int32 accumulators;
logits within 1e-5 relative in the sense of reading R13:
    |g - o| <= 1e-5 * max(|o|, |b_j| + sum_c |w_jc|).
Sizes span several CTA tiles with ragged tails; C0 runs whole; C1 runs at full size
in the bench's launch configuration and is checked on sampled outputs.
"""
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


SELECTORS = {"popc": 1, "tz": 3, "tz8": 4, "auto": 0, "tz_cap3": 3, "tz8_cap3": 4}


@pytest.fixture(params=["popc", "tz", "tz8", "auto", "tz_cap3", "tz8_cap3"])
def kernel(request, tn):
    """Run a conv test with the CUDA-core popc kernel, one of the tcgen05 kernels
    (tz = FP4 operands where they fit, tz8 = int8 operands; skipped for shapes a
    kernel does not cover), or the automatic choice.  The _cap3
    variants cap the persistent grid at 3 CTAs, so each CTA walks long runs of
    output planes (TMEM block rotation, ring wrap-around, run boundaries)."""
    tn.tn_set_conv_kernel(SELECTORS[request.param])
    tn.tn_set_grid_cap(3 if request.param.endswith("cap3") else 0)
    yield request.param
    tn.tn_set_conv_kernel(tn.TN_KERNEL_AUTO)
    tn.tn_set_grid_cap(0)


@pytest.fixture(params=["popc", "tz8", "auto", "auto_cap5"])
def fcn_kernel(request, tn):
    tn.tn_set_conv_kernel({"popc": 1, "tz8": 4, "auto": 0, "auto_cap5": 0}[request.param])
    tn.tn_set_grid_cap(5 if request.param.endswith("cap5") else 0)
    yield request.param
    tn.tn_set_conv_kernel(tn.TN_KERNEL_AUTO)
    tn.tn_set_grid_cap(0)


def run_or_skip(kernel, fn, *a, **kw):
    import paper_1801_09449_b200 as tn
    try:
        return fn(*a, **kw)
    except tn.TNError as e:
        if kernel.startswith("tz") and e.status == tn.TN_EUNSUPPORTED:
            pytest.skip("shape outside this tcgen05 kernel")
        raise


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def bad_value(flag):
    torch.cuda.synchronize()
    return int(flag.item())


# --------------------------------------------------------------------------- A1 pack
@pytest.mark.parametrize("shape", [(1, 16, 32, 32, 32), (2, 1, 3, 5, 7), (1, 33, 4, 5, 6), (1, 64, 6, 7, 9),
                                   (2, 100, 3, 3, 4), (1, 130, 2, 3, 5), (1, 32, 1, 1, 1)])
def test_pack_i8_i32_matches_oracle(tn, shape):
    x = synth.ternary_codes(shape, 0.5, seed=sum(shape))
    ref, bad = oracle.pack(x)
    assert bad == -1
    flag = tn.bad_flag()
    got = tn.tn_pack_i8(dev(x), d_bad=flag)
    assert bad_value(flag) == tn.INT64_MAX
    np.testing.assert_array_equal(u32(got), ref)
    got32 = tn.tn_pack_i32(dev(x.astype(np.int32)))
    np.testing.assert_array_equal(u32(got32), ref)
    # roundtrip through tn_unpack
    back = tn.tn_unpack(got, shape[1], d_bad=flag)
    assert bad_value(flag) == tn.INT64_MAX
    np.testing.assert_array_equal(back.cpu().numpy(), x)


def test_pack_domain_errors(tn):
    x = synth.ternary_codes((1, 20, 4, 4, 8), 0.5, seed=1)
    x[0, 7, 2, 1, 3] = 3
    x[0, 19, 3, 3, 7] = -2
    flag = tn.bad_flag()
    tn.tn_pack_i8(dev(x), d_bad=flag)
    _, obad = oracle.pack(x)
    assert bad_value(flag) == obad == np.ravel_multi_index((0, 7, 2, 1, 3), x.shape)
    flag = tn.bad_flag()
    tn.tn_pack_i32(dev(x.astype(np.int32)), d_bad=flag)
    assert bad_value(flag) == obad


def test_pack_f32_eq6(tn):
    x = synth.ct_volume((2, 3, 8, 9, 12), seed=2)
    x[0, 1, 2, 3, 4] = np.float32(synth.CT_T_HI)  # boundary -> 0
    x[1, 2, 7, 8, 11] = np.float32(synth.CT_T_LO)
    t, bad = oracle.tern_f32(x, synth.CT_T_LO, synth.CT_T_HI)
    ref, _ = oracle.pack(t)
    flag = tn.bad_flag()
    got = tn.tn_pack_f32(dev(x), synth.CT_T_LO, synth.CT_T_HI, d_bad=flag)
    assert bad_value(flag) == tn.INT64_MAX
    np.testing.assert_array_equal(u32(got), ref)
    x[1, 0, 5, 5, 5] = np.nan
    x[1, 1, 0, 0, 0] = np.inf
    _, obad = oracle.tern_f32(x, synth.CT_T_LO, synth.CT_T_HI)
    flag = tn.bad_flag()
    tn.tn_pack_f32(dev(x), synth.CT_T_LO, synth.CT_T_HI, d_bad=flag)
    assert bad_value(flag) == obad


def test_pack_weights_and_unpack_noncanonical(tn):
    for k, c in ((16, 16), (64, 64), (5, 33), (3, 1), (64, 128)):
        w = synth.ternary_codes((k, c, 3, 3, 3), 0.6, seed=k * c)
        ref, _ = oracle.pack_weights(w)
        np.testing.assert_array_equal(u32(tn.tn_pack_weights(dev(w))), ref)
    x = synth.ternary_codes((1, 3, 1, 2, 2), 0.5, seed=4)
    xp, _ = oracle.pack(x)
    xp[0, 0, 1, 0, 0, 0] |= np.uint32(1 << 1)
    xp[0, 0, 1, 0, 1, 0] &= np.uint32(0xFFFFFFFD)
    _, obad = oracle.unpack(xp, 3)
    flag = tn.bad_flag()
    tn.tn_unpack(dev(xp.view(np.int32)), 3, d_bad=flag)
    assert bad_value(flag) == obad >= 0


# --------------------------------------------------------------------------- A2/A3/A5 conv
CONV_CASES = [
    # (x shape NCDHW, k, stride, pad, dil)
    ((1, 16, 32, 32, 32), 16, 1, 1, 1),          # C0 whole
    ((1, 16, 9, 17, 35), 16, 1, 1, 1),           # ragged tails in every axis
    ((2, 64, 7, 10, 21), 64, 1, 1, 1),
    ((1, 32, 12, 18, 20), 32, 2, 1, 1),          # stride 2 (A5)
    ((1, 64, 10, 12, 14), 64, 2, 1, 1),
    ((1, 33, 6, 7, 8), 5, 1, 1, 1),              # 2 words, ragged channels, odd K
    ((1, 16, 11, 12, 13), 16, 1, 2, 2),          # dilation 2
    ((1, 1, 5, 6, 7), 3, 1, 1, 1),               # one channel
    ((1, 128, 4, 5, 6), 16, 1, 1, 1),            # 4 words
    ((1, 16, 5, 6, 7), 7, (1, 2, 1), (0, 1, 2), (1, 1, 2)),  # anisotropic geometry
    ((1, 16, 1, 1, 1), 16, 1, 1, 1),             # a single voxel
    # tap-offset z-merged kernel (TZ) shapes: even W, C <= 64, small filter banks
    ((1, 16, 9, 17, 34), 16, 1, 1, 1),           # ragged tiles and strips
    ((2, 32, 7, 10, 22), 32, 1, 1, 1),
    ((1, 64, 6, 10, 12), 32, 1, 1, 1),           # 4 chunks, K = 32
    ((1, 32, 5, 6, 8), 64, 1, 1, 1),             # K = 64
    ((1, 16, 12, 18, 20), 16, 2, 1, 1),          # stride 2, phase images
    ((2, 32, 9, 14, 10), 32, 2, 1, 1),           # stride 2, odd depth
    ((1, 16, 3, 130, 140), 16, 1, 1, 1),         # several strips per plane
    ((1, 64, 11, 20, 30), 64, 1, 1, 1),          # C = K = 64: four TMEM blocks, wrap-split MMAs
    ((2, 64, 6, 9, 128), 64, 1, 1, 1),
    # odd W on TZ: 16-byte-aligned supersets of the packed rows (8 bytes per voxel)
    ((1, 16, 3, 5, 7), 16, 1, 1, 1),             # odd voxel count: the last 8 bytes take a plain load
    ((2, 32, 4, 6, 9), 32, 1, 1, 1),
    ((1, 48, 5, 6, 11), 16, 1, 1, 1),            # three 16-channel chunks
    ((1, 16, 4, 70, 131), 16, 1, 1, 1),          # several strips, odd rows
    # dilation on TZ (stride 1, pad = dilation): in-plane taps at dilated offsets, z residue classes
    ((1, 32, 10, 14, 16), 32, 1, 3, 3),
    ((2, 16, 7, 9, 20), 64, 1, 2, 2),
    ((1, 64, 9, 40, 36), 24, 1, 2, 2),           # padded K, several strips
    ((1, 20, 2, 5, 6), 16, 1, 4, 4),             # fewer planes than the dilation, padded C
]


def _case(shape, k, seed):
    x = synth.ternary_codes(shape, 0.5, seed=seed)
    w = synth.ternary_codes((k, shape[1], 3, 3, 3), 0.6, seed=seed + 1)
    return x, w


@pytest.mark.parametrize("case", CONV_CASES, ids=lambda c: "x".join(map(str, c[0])) + f"_k{c[1]}")
def test_conv3d_int32_matches_oracle(tn, kernel, case):
    shape, k, s, p, dl = case
    x, w = _case(shape, k, seed=zlib.crc32(str(case).encode()) % 1000)
    ref = oracle.conv3d(x, w, s, p, dl)                       # [n,k,do,ho,wo]
    xp = tn.tn_pack_i8(dev(x))
    wp = tn.tn_pack_weights(dev(w))
    y = run_or_skip(kernel, tn.tn_conv3d, xp, tn.dims(*shape), wp, k, tn.geom(s, p, dl))
    np.testing.assert_array_equal(y.cpu().numpy(), ref.transpose(0, 2, 3, 4, 1))


@pytest.mark.parametrize("case", CONV_CASES[:7] + CONV_CASES[11:], ids=lambda c: "x".join(map(str, c[0])) + f"_k{c[1]}")
def test_conv3d_requant_matches_oracle(tn, kernel, case):
    shape, k, s, p, dl = case
    x, w = _case(shape, k, seed=7 + shape[2])
    base = synth.threshold_base(shape[1], 0.5)
    lo, hi = synth.jittered_thresholds(k, base, seed=k)
    acc = oracle.conv3d(x, w, s, p, dl)
    ref, _ = oracle.pack(oracle.requant(acc, lo, hi))
    xp = tn.tn_pack_i8(dev(x))
    wp = tn.tn_pack_weights(dev(w))
    yp = run_or_skip(kernel, tn.tn_conv3d_requant, xp, tn.dims(*shape), wp, k, tn.geom(s, p, dl), dev(lo), dev(hi))
    np.testing.assert_array_equal(u32(yp), ref)
    # standalone requant of the int32 result gives the same words
    y = tn.tn_conv3d(xp, tn.dims(*shape), wp, k, tn.geom(s, p, dl))
    np.testing.assert_array_equal(u32(tn.tn_requant(y, dev(lo), dev(hi))), ref)


# One-plane volumes (D = 1, Table 1's 2D layers, reading R18): the tensor-core kernel's one-plane
# mode (one TMEM block per tile, the middle kernel plane only, wide strips): FP4 stride 1 with 1, 2
# and 4 16-channel chunks, int8 stride 2 with 4 chunks; batches so strips and stacks interleave.
ONEP_CASES = [((3, 16, 1, 40, 36), 16, 1), ((2, 15, 1, 48, 44), 32, 1), ((2, 32, 1, 30, 64), 64, 1),
              ((2, 64, 1, 24, 40), 64, 1), ((3, 64, 1, 20, 36), 64, 2), ((1, 64, 1, 34, 34), 32, 2),
              ((4, 32, 1, 9, 13), 16, 1)]


@pytest.mark.parametrize("case", ONEP_CASES, ids=lambda c: "x".join(map(str, c[0])) + f"_k{c[1]}_s{c[2]}")
def test_conv3d_one_plane_matches_oracle(tn, kernel, case):
    shape, k, s = case
    x, w = _case(shape, k, seed=300 + k + s)
    lo, hi = synth.jittered_thresholds(k, synth.threshold_base(shape[1], 0.5), seed=k + 1)
    acc = oracle.conv3d(x, w, s, 1, 1)
    ref, _ = oracle.pack(oracle.requant(acc, lo, hi))
    xp, wp, xd = tn.tn_pack_i8(dev(x)), tn.tn_pack_weights(dev(w)), tn.dims(*shape)
    y = run_or_skip(kernel, tn.tn_conv3d, xp, xd, wp, k, tn.geom(s))
    np.testing.assert_array_equal(y.cpu().numpy(), np.moveaxis(acc, 1, -1))
    yp = run_or_skip(kernel, tn.tn_conv3d_requant, xp, xd, wp, k, tn.geom(s), dev(lo), dev(hi))
    np.testing.assert_array_equal(u32(yp), ref)


def test_conv3d_requant_sentinel_thresholds(tn, kernel):
    """INT32 sentinel thresholds (always +1 / always -1 / always 0) and lo >= hi through
    the fused epilogues of every conv kernel (no overflow in acc - hi or lo - hi)."""
    i32 = np.iinfo(np.int32)
    shape, k = (1, 16, 6, 10, 12), 16
    x, w = _case(shape, k, seed=91)
    lo = np.full(k, -3, np.int32)
    hi = np.full(k, 3, np.int32)
    lo[0], hi[0] = i32.min, i32.min
    lo[1], hi[1] = i32.max, i32.max
    lo[2], hi[2] = i32.min, i32.max
    lo[3], hi[3] = 5, 0
    lo[4], hi[4] = i32.max, 0
    lo[5], hi[5] = i32.min, 1
    ref, _ = oracle.pack(oracle.requant(oracle.conv3d(x, w), lo, hi))
    yp = run_or_skip(kernel, tn.tn_conv3d_requant, tn.tn_pack_i8(dev(x)), tn.dims(*shape),
                     tn.tn_pack_weights(dev(w)), k, tn.geom(), dev(lo), dev(hi))
    np.testing.assert_array_equal(u32(yp), ref)


@pytest.mark.parametrize("case", [((1, 16, 9, 17, 34), 16, 1), ((1, 64, 6, 10, 12), 64, 1),
                                  ((1, 32, 12, 18, 20), 32, 2), ((1, 33, 5, 6, 7), 5, 1)],
                         ids=lambda c: "x".join(map(str, c[0])) + f"_k{c[1]}_s{c[2]}")
def test_conv3d_binary_eq8(tn, kernel, case):
    """NEXT-4 binary network (Eq. 8): {-1,+1} activations and weights are
    ternary codes with all-ones masks, and a binary sign activation is the requant with
    lo = hi - 1.  Every kernel runs them unchanged; outputs stay binary and match the oracle."""
    shape, k, s = case
    x = synth.ternary_codes(shape, 0.0, seed=shape[1] + k)
    w = synth.ternary_codes((k, shape[1], 3, 3, 3), 0.0, seed=shape[1] + k + 1)
    hi = synth.rng(k).integers(-3, 4, size=k).astype(np.int32)
    lo = hi - 1
    acc = oracle.conv3d(x, w, s)
    t = oracle.requant(acc, lo, hi)
    assert np.all(t != 0)
    ref, _ = oracle.pack(t)
    xp, wp = tn.tn_pack_i8(dev(x)), tn.tn_pack_weights(dev(w))
    y = run_or_skip(kernel, tn.tn_conv3d, xp, tn.dims(*shape), wp, k, tn.geom(s))
    np.testing.assert_array_equal(y.cpu().numpy(), acc.transpose(0, 2, 3, 4, 1))
    yp = run_or_skip(kernel, tn.tn_conv3d_requant, xp, tn.dims(*shape), wp, k, tn.geom(s), dev(lo), dev(hi))
    np.testing.assert_array_equal(u32(yp), ref)


@pytest.mark.parametrize("case", [((5, 16, 64, 128, 128), 16), ((8, 64, 16, 32, 32), 64), ((5, 32, 16, 64, 64), 32),
                                  ((3, 16, 24, 40, 130), 16)],
                         ids=lambda c: "x".join(map(str, c[0])) + f"_k{c[1]}")
def test_conv3d_batched_ranges_cross_samples(tn, kernel, case):
    """n > 1 with 148 persistent CTAs whose unit ranges run from the ragged last strip of one
    sample into the first strip of the next (regression: the per-unit barriers of a ragged
    strip must still advance, or the kernel deadlocks): the batched result equals the
    per-sample launches bit for bit, and sampled outputs equal the oracle."""
    shape, k = case
    x, w = _case(shape, k, seed=shape[0] * 13 + k)
    base = synth.threshold_base(shape[1], 0.5)
    lo, hi = synth.jittered_thresholds(k, base, seed=k + 1)
    xp, wp = tn.tn_pack_i8(dev(x)), tn.tn_pack_weights(dev(w))
    yp = run_or_skip(kernel, tn.tn_conv3d_requant, xp, tn.dims(*shape), wp, k, tn.geom(), dev(lo), dev(hi))
    one = (1,) + shape[1:]
    for i in range(shape[0]):
        yi = tn.tn_conv3d_requant(tn.tn_pack_i8(dev(x[i:i + 1])), tn.dims(*one), wp, k, tn.geom(), dev(lo), dev(hi))
        np.testing.assert_array_equal(u32(yp)[i:i + 1], u32(yi), err_msg=f"sample {i}")
    g = synth.rng(5)
    m = 200
    at = np.stack([g.integers(0, shape[0], m), g.integers(0, k, m), g.integers(0, shape[2], m),
                   g.integers(0, shape[3], m), g.integers(0, shape[4], m)], 1).astype(np.int32)
    acc = oracle.conv3d_at(x, w, at)
    n_, k_, z_, y_, x_ = at.T
    ref = np.where(acc >= hi[k_], 1, np.where(acc <= lo[k_], -1, 0))
    ypn = u32(yp)
    sb = (ypn[n_, z_, y_, x_, 0, k_ // 32] >> (k_ % 32)) & 1
    mb = (ypn[n_, z_, y_, x_, 1, k_ // 32] >> (k_ % 32)) & 1
    np.testing.assert_array_equal(np.where(mb == 1, np.where(sb == 1, 1, -1), 0), ref)


def test_conv3d_empty_inputs(tn, kernel):
    """Empty tensors (n = 0, or an empty spatial extent) are a successful no-op under every
    kernel selector; nothing is launched and the output stays untouched."""
    for shape in [(0, 16, 4, 4, 4), (1, 16, 0, 8, 8), (2, 64, 3, 0, 6)]:
        k = 16
        w = synth.ternary_codes((k, shape[1], 3, 3, 3), 0.6, seed=3)
        wp = tn.tn_pack_weights(dev(w))
        xp = torch.zeros(16, dtype=torch.int32, device="cuda")          # any valid aligned pointer
        lo = dev(np.full(k, -3, np.int32))
        hi = dev(np.full(k, 3, np.int32))
        sentinel = torch.full((64,), 7, dtype=torch.int32, device="cuda")
        assert tn.lib.tn_conv3d_requant(tn._ptr(xp), tn.dims(*shape), tn._ptr(wp), k, tn.geom(), tn._ptr(lo),
                                        tn._ptr(hi), tn._ptr(sentinel), tn._stream()) == tn.TN_OK
        assert tn.lib.tn_conv3d(tn._ptr(xp), tn.dims(*shape), tn._ptr(wp), k, tn.geom(), tn._ptr(sentinel),
                                tn._stream()) == tn.TN_OK
        torch.cuda.synchronize()
        assert bool((sentinel == 7).all())


@pytest.mark.parametrize("case", [((1, 16, 3, 4, 1100), 16, 1), ((1, 32, 4, 3, 1030), 32, 2), ((1, 16, 5, 6, 7), 1, 1),
                                  ((1, 16, 4, 130, 2), 16, 1), ((1, 64, 3, 2, 1024), 64, 1)],
                         ids=lambda c: "x".join(map(str, c[0])) + f"_k{c[1]}_s{c[2]}")
def test_conv3d_extreme_widths_and_tiny_k(tn, kernel, case):
    """Rows wider than the tap-offset kernel's raster limit (Po <= 1024: W = 1030 / 1100 fall
    back to the dx-merged or popcount kernel under AUTO), a 1024-wide row at the limit, K = 1,
    and a 2-voxel-wide strip: bit-exact against the oracle."""
    shape, k, s = case
    x, w = _case(shape, k, seed=sum(shape) + k)
    base = synth.threshold_base(shape[1], 0.5)
    lo, hi = synth.jittered_thresholds(k, base, seed=k + 7)
    acc = oracle.conv3d(x, w, s)
    ref, _ = oracle.pack(oracle.requant(acc, lo, hi))
    xp, wp = tn.tn_pack_i8(dev(x)), tn.tn_pack_weights(dev(w))
    y = run_or_skip(kernel, tn.tn_conv3d, xp, tn.dims(*shape), wp, k, tn.geom(s))
    np.testing.assert_array_equal(y.cpu().numpy(), acc.transpose(0, 2, 3, 4, 1))
    yp = run_or_skip(kernel, tn.tn_conv3d_requant, xp, tn.dims(*shape), wp, k, tn.geom(s), dev(lo), dev(hi))
    np.testing.assert_array_equal(u32(yp), ref)


def test_requant_sentinels_and_order(tn):
    i32 = np.iinfo(np.int32)
    y = np.arange(-40, 40, dtype=np.int32).reshape(1, 1, 1, 80, 1).repeat(40, axis=4)
    lo = np.full(40, -3, np.int32)
    hi = np.full(40, 3, np.int32)
    lo[0], hi[0] = i32.min, i32.min          # always +1
    lo[1], hi[1] = i32.max, i32.max          # always -1
    lo[2], hi[2] = i32.min, i32.max          # always 0
    lo[3], hi[3] = 5, 0                      # hi tested first
    ref, _ = oracle.pack(oracle.requant(np.ascontiguousarray(y.transpose(0, 4, 1, 2, 3)), lo, hi))
    np.testing.assert_array_equal(u32(tn.tn_requant(dev(y), dev(lo), dev(hi))), ref)


# --------------------------------------------------------------------------- A6 upsample + concat
@pytest.mark.parametrize("low,cl,cs,k", [((3, 4, 5), 16, 16, 16), ((2, 3, 9), 64, 64, 64),
                                         ((4, 4, 4), 32, 32, 32), ((1, 1, 1), 16, 16, 8),
                                         ((5, 6, 7), 16, 16, 16), ((3, 5, 4), 32, 32, 32), ((4, 3, 6), 16, 32, 16),
                                         ((4, 5, 6), 64, 64, 64)])
def test_conv3d_upsample_concat_matches_oracle(tn, kernel, low, cl, cs, k):
    n = 1
    a = synth.ternary_codes((n, cl) + low, 0.5, seed=cl)
    b = synth.ternary_codes((n, cs) + tuple(2 * v for v in low), 0.5, seed=cs + 1)
    w = synth.ternary_codes((k, cl + cs, 3, 3, 3), 0.6, seed=k + 2)
    base = synth.threshold_base(cl + cs, 0.5)
    lo, hi = synth.jittered_thresholds(k, base, seed=3)
    acc = oracle.conv3d(oracle.concat(oracle.upsample2(a), b), w)
    ref_t = oracle.requant(acc, lo, hi)
    ref, _ = oracle.pack(ref_t)
    ap, bp = tn.tn_pack_i8(dev(a)), tn.tn_pack_i8(dev(b))
    wa = tn.tn_pack_weights(dev(np.ascontiguousarray(w[:, :cl])))
    wb = tn.tn_pack_weights(dev(np.ascontiguousarray(w[:, cl:])))
    segs = [(ap, tn.dims(n, cl, *low), 1, wa), (bp, tn.dims(n, cs, *b.shape[2:]), 0, wb)]
    yp = run_or_skip(kernel, tn.tn_conv3d_seg, segs, k, tn.geom(), dev(lo), dev(hi))
    np.testing.assert_array_equal(u32(yp), ref)
    y = tn.tn_conv3d_seg(segs, k, tn.geom(), requant=False)
    np.testing.assert_array_equal(y.cpu().numpy(), acc.transpose(0, 2, 3, 4, 1))


# --------------------------------------------------------------------------- A7 first layer
@pytest.mark.parametrize("shape,stride", [((1, 1, 16, 24, 40), 1), ((2, 1, 7, 9, 33), 1), ((1, 1, 12, 16, 16), 2),
                                          ((2, 1, 9, 13, 20), 1), ((1, 1, 21, 35, 132), 1)])
def test_conv3d_first_matches_oracle(tn, kernel, shape, stride):
    """A7 + A3 + A4 of the first layer; under AUTO / TZ the tensor-core first-layer
    mode runs where it covers the shape (stride 1, W % 4 == 0), else the popc kernel."""
    x = synth.ct_volume(shape, seed=shape[3])
    w = synth.ternary_codes((16, 1, 3, 3, 3), 0.6, seed=5)
    lo, hi = synth.jittered_thresholds(16, synth.threshold_base(1, 0.38), seed=6)
    t, _ = oracle.tern_f32(x, synth.CT_T_LO, synth.CT_T_HI)
    ref, _ = oracle.pack(oracle.requant(oracle.conv3d(t, w, stride), lo, hi))
    flag = tn.bad_flag()
    yp = tn.tn_conv3d_first(dev(x), synth.CT_T_LO, synth.CT_T_HI, tn.tn_pack_weights(dev(w)), 16,
                            tn.geom(stride), dev(lo), dev(hi), d_bad=flag)
    assert bad_value(flag) == tn.INT64_MAX
    np.testing.assert_array_equal(u32(yp), ref)
    x[0, 0, 3, 4, 5] = np.nan
    flag = tn.bad_flag()
    tn.tn_conv3d_first(dev(x), synth.CT_T_LO, synth.CT_T_HI, tn.tn_pack_weights(dev(w)), 16,
                       tn.geom(stride), dev(lo), dev(hi), d_bad=flag)
    _, obad = oracle.tern_f32(x, synth.CT_T_LO, synth.CT_T_HI)
    assert bad_value(flag) == obad


# --------------------------------------------------------------------------- A8 prediction
def _logit_tol(w, b):
    return 1e-5 * (np.abs(b)[None, :, None, None, None] + np.abs(w).sum(1)[None, :, None, None, None])


def test_predict_matches_oracle(tn):
    t = synth.ternary_codes((2, 16, 5, 9, 13), 0.5, seed=8)
    p = synth.fcn_params()
    ref = oracle.predict(t, p["pred_w"], p["pred_b"])
    tp = tn.tn_pack_i8(dev(t))
    got = tn.tn_predict(tp, 16, dev(p["pred_w"]), dev(p["pred_b"])).cpu().numpy()
    tol = np.maximum(np.abs(ref), _logit_tol(p["pred_w"], p["pred_b"]) / 1e-5) * 1e-5
    assert np.all(np.abs(got - ref) <= tol)


@pytest.mark.parametrize("c,nclass", [(64, 2), (16, 2), (33, 3), (64, 8), (7, 1)])
def test_predict_large_quad_tables(tn, c, nclass):
    """tn_predict on large tensors (>= 65536 voxels) runs the quad-table kernel: logits within R13
    of the oracle, and bit-identical to the per-voxel kernel small tensors run (same sum order)."""
    t = synth.ternary_codes((3, c, 4, 64, 100), 0.5, seed=c)
    g = synth.rng(c + nclass)
    w = (0.25 * g.standard_normal((nclass, c))).astype(np.float32)
    b = (0.1 * g.standard_normal(nclass)).astype(np.float32)
    ref = oracle.predict(t, w, b)
    got = tn.tn_predict(tn.tn_pack_i8(dev(t)), c, dev(w), dev(b)).cpu().numpy()
    tol = np.maximum(np.abs(ref), _logit_tol(w, b) / 1e-5) * 1e-5
    assert np.all(np.abs(got - ref) <= tol)
    small = tn.tn_predict(tn.tn_pack_i8(dev(t[:1, :, :1])), c, dev(w), dev(b)).cpu().numpy()   # 6400 voxels
    np.testing.assert_array_equal(small, got[:1, :, :1])


# --------------------------------------------------------------------------- A9 FCN
def _fcn_compare(tn, x, p, per_layer=True):
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
    xd = dev(x)
    ws = net.workspace(x.shape)
    flag = tn.bad_flag()
    logits = net(xd, ws=ws, d_bad=flag)
    assert bad_value(flag) == tn.INT64_MAX
    ref_logits, acts, bad = oracle.fcn_forward(x, p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"],
                                               p["pred_w"], p["pred_b"], want_acts=per_layer)
    assert bad == -1
    if per_layer:
        # (the last layer's codes feed only the fused prediction and are not stored; the
        # logits below check them)
        for i in range(13):
            view, od = net.layer_output(x.shape, ws, i)
            ref, _ = oracle.pack(acts[i])
            np.testing.assert_array_equal(u32(view), ref, err_msg=f"layer #{i + 1}")
    got = logits.cpu().numpy()
    tol = np.maximum(np.abs(ref_logits), _logit_tol(p["pred_w"], p["pred_b"]) / 1e-5) * 1e-5
    assert np.all(np.abs(got - ref_logits) <= tol)
    return got


@pytest.mark.parametrize("nclass", [1, 3, 8])
def test_fcn_prediction_class_counts(tn, fcn_kernel, nclass):
    """A8 with 1, 3 and 8 classes (the fused epilogue's generic table path; the 2-class case is
    in every other FCN test): logits equal the oracle's prediction of the oracle's layer-14 codes."""
    shape = (2, 1, 16, 24, 40)
    x = synth.ct_volume(shape, seed=nclass)
    p = synth.fcn_params()
    g = synth.rng(70 + nclass)
    pw = (0.25 * g.standard_normal((nclass, 16))).astype(np.float32)
    pb = (0.1 * g.standard_normal(nclass)).astype(np.float32)
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], pw, pb, p["t_lo"], p["t_hi"])
    got = net(dev(x)).cpu().numpy()
    _, acts, _ = oracle.fcn_forward(x, p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"], p["pred_w"],
                                    p["pred_b"], want_acts=True)
    ref = oracle.predict(acts[13], pw, pb)
    assert got.shape == ref.shape
    tol = np.maximum(np.abs(ref), _logit_tol(pw, pb) / 1e-5) * 1e-5
    assert np.all(np.abs(got - ref) <= tol)


@pytest.mark.parametrize("shape", [(1, 1, 16, 16, 16), (1, 1, 32, 48, 48), (2, 1, 8, 24, 40), (3, 1, 32, 64, 64)])
def test_fcn_matches_oracle_small(tn, fcn_kernel, shape):
    x = synth.ct_volume(shape, seed=shape[3])
    _fcn_compare(tn, x, synth.fcn_params())


def test_fcn_c2_full_size_matches_oracle(tn):
    """BASELINE.json configs[2] at full size (96 x 144 x 144), every layer bit-exact."""
    cfg = synth.CONFIGS["C2"]
    x = synth.ct_volume(cfg["vol_shape"], seed=cfg["seeds"][0])
    _fcn_compare(tn, x, synth.fcn_params(cfg["seed_params"]))


# Backward dependency interval of one output voxel of the R9 FCN (1-D, by axis): it reads
# inputs from 37..44 voxels below to 30..37 above, depending on its position mod 8.
_FCN_DEP_BELOW, _FCN_DEP_ABOVE = 44, 37


@pytest.mark.parametrize("cfg_name,origin", [("C4", (64, 192, 320)), ("C4", (0, 0, 384)), ("C3", (0, 64, 128))])
def test_fcn_full_size_cropped_oracle(tn, cfg_name, origin):
    """configs[4] (1x1x256x512x512) and configs[3] (128x256x256) at full size on the GPU against
    the oracle on a 128^3 crop aligned to the FCN's /8 grid.  Outputs at least 44 voxels above
    the crop's lower faces and 37 below its upper faces depend only on inputs inside the crop
    (the R9 dependency interval), so they must equal the whole-volume logits (R13 tolerance);
    faces on the volume boundary pad with zeros in both, so the corner crop checks padding at
    full size too.  For C4 the 8-slab NEXT-1 schedule must reproduce the whole volume exactly."""
    cfg = synth.CONFIGS[cfg_name]
    shape = cfg["vol_shape"]
    p = synth.fcn_params(cfg["seed_params"])
    x = synth.ct_volume(shape, seed=cfg["seeds"][0])
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
    xd = dev(x)
    got = net(xd)
    n = 128
    sl = tuple(slice(o, o + n) for o in origin)
    ref, _, _ = oracle.fcn_forward(np.ascontiguousarray(x[(slice(None), slice(None)) + sl]), p["t_lo"], p["t_hi"],
                                   p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"])
    # comparable region per axis: the margin is only needed on faces inside the volume
    lo_ = [0 if o == 0 else _FCN_DEP_BELOW for o in origin]
    hi_ = [n if o + n == ext else n - _FCN_DEP_ABOVE for o, ext in zip(origin, shape[2:])]
    r = ref[:, :, lo_[0]:hi_[0], lo_[1]:hi_[1], lo_[2]:hi_[2]]
    g = got[:, :, origin[0] + lo_[0]:origin[0] + hi_[0], origin[1] + lo_[1]:origin[1] + hi_[1],
            origin[2] + lo_[2]:origin[2] + hi_[2]].cpu().numpy()
    assert r.size >= 2 * 40 ** 3
    tol = np.maximum(np.abs(r), _logit_tol(p["pred_w"], p["pred_b"]) / 1e-5) * 1e-5
    assert np.all(np.abs(g - r) <= tol)
    if cfg_name == "C4":
        np.testing.assert_array_equal(net.forward_slabs_local_p2p(xd, 8).cpu().numpy(), got.cpu().numpy())


def test_fcn_c3_full_volume_every_layer(tn):
    """configs[3] at full size in the bench's launch configuration (one batched forward of all 8
    CT-like volumes 128x256x256): volume 0 is compared WHOLE against the oracle's forward of the
    same volume -- every stored layer's packed words bit for bit, and the logits within R13 (the
    last layer's codes feed only the fused prediction and are checked through the logits)."""
    cfg = synth.CONFIGS["C3"]
    shape = cfg["vol_shape"]
    p = synth.fcn_params(cfg["seed_params"])
    vols = [synth.ct_volume(shape, seed=s) for s in cfg["seeds"]]
    xb = np.concatenate(vols, 0)
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
    ws = net.workspace(xb.shape)
    flag = tn.bad_flag()
    logits = net(dev(xb), ws=ws, d_bad=flag)
    assert bad_value(flag) == tn.INT64_MAX
    got_layers = [u32(net.layer_output(xb.shape, ws, i)[0][:1]) for i in range(13)]
    got_logits = logits[:1].cpu().numpy()
    del ws, logits
    ref_logits, acts, bad = oracle.fcn_forward(vols[0], p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"],
                                               p["pred_w"], p["pred_b"], want_acts=True)
    assert bad == -1
    for i in range(13):
        ref, _ = oracle.pack(acts[i])
        np.testing.assert_array_equal(got_layers[i], ref, err_msg=f"layer #{i + 1}")
    tol = np.maximum(np.abs(ref_logits), _logit_tol(p["pred_w"], p["pred_b"]) / 1e-5) * 1e-5
    assert np.all(np.abs(got_logits - ref_logits) <= tol)


# --------------------------------------------------------------------------- C1 at full size
def test_c1_full_size(tn):
    """configs[1] (1x64x64x128x128, K=64, fused requant) in the bench's launch configuration,
    compared WHOLE against the oracle: all 67.1 M int32 accumulators (tn_conv3d) and every
    packed output word (tn_conv3d_requant) against oracle.conv3d / requant / pack."""
    x, w, lo, hi = synth.conv_config("C1")
    xp = tn.tn_pack_i8(dev(x))
    wp = tn.tn_pack_weights(dev(w))
    xd = tn.dims(*x.shape)
    yp = u32(tn.tn_conv3d_requant(xp, xd, wp, 64, tn.geom(), dev(lo), dev(hi)))
    y = tn.tn_conv3d(xp, xd, wp, 64, tn.geom()).cpu().numpy()
    torch.cuda.synchronize()
    ref_acc = oracle.conv3d(x, w)                                   # [1,64,64,128,128]
    np.testing.assert_array_equal(y, ref_acc.transpose(0, 2, 3, 4, 1))
    ref_p, bad = oracle.pack(oracle.requant(ref_acc, lo, hi))
    assert bad == -1
    np.testing.assert_array_equal(yp, ref_p)


# The FCN's full-resolution layers of configs[3] (1 x C x 128 x 256 x 256) through
# every tensor-core kernel that covers them, in the persistent launch the FCN uses:
# sampled outputs against the oracle's per-output sum + the packed/int32 agreement.
C3_LAYER_CASES = [
    # (C, K, stride, kernel)
    (16, 16, 1, "tz"), (16, 16, 1, "tz8"), (16, 16, 2, "tz"), (16, 16, 2, "tz8"),
    (16, 32, 1, "tz"), (32, 16, 1, "tz"), (64, 32, 1, "tz"), (64, 64, 2, "tz"),
]


@pytest.mark.parametrize("case", C3_LAYER_CASES, ids=lambda c: f"c{c[0]}_k{c[1]}_s{c[2]}_{c[3]}")
def test_c3_layer_full_size_sampled(tn, case):
    c, k, s, kern = case
    shape = (1, c, 128, 256, 256)
    x = synth.ternary_codes(shape, 0.5, seed=31 + c + k + s)
    w = synth.ternary_codes((k, c, 3, 3, 3), 0.6, seed=32 + c + k + s)
    lo, hi = synth.jittered_thresholds(k, synth.threshold_base(c, 0.5), seed=33)
    tn.tn_set_conv_kernel(SELECTORS[kern])
    try:
        xp = tn.tn_pack_i8(dev(x))
        wp = tn.tn_pack_weights(dev(w))
        xd = tn.dims(*shape)
        yp = u32(tn.tn_conv3d_requant(xp, xd, wp, k, tn.geom(s), dev(lo), dev(hi)))
        y = tn.tn_conv3d(xp, xd, wp, k, tn.geom(s)).cpu().numpy()
    finally:
        tn.tn_set_conv_kernel(tn.TN_KERNEL_AUTO)
    do, ho, wo = y.shape[1:4]
    g = synth.rng(98)
    m = 4096
    at = np.stack([np.zeros(m, int), g.integers(0, k, m), g.integers(0, do, m), g.integers(0, ho, m),
                   g.integers(0, wo, m)], 1).astype(np.int32)
    at[:8, 2:] = [[0, 0, 0], [do - 1, ho - 1, wo - 1], [0, ho - 1, 0], [do - 1, 0, wo - 1], [do // 2, 0, wo // 2],
                  [do // 2, ho - 1, wo // 2], [0, ho // 2, wo // 2], [do - 1, ho // 2, wo // 2]]
    ref_acc = oracle.conv3d_at(x, w, at, s)
    n_, k_, z_, y_, x_ = at.T
    np.testing.assert_array_equal(y[n_, z_, y_, x_, k_], ref_acc)
    ref_t = np.where(ref_acc >= hi[k_], 1, np.where(ref_acc <= lo[k_], -1, 0))
    s_bit = (yp[n_, z_, y_, x_, 0, k_ // 32] >> (k_ % 32)) & 1
    m_bit = (yp[n_, z_, y_, x_, 1, k_ // 32] >> (k_ % 32)) & 1
    np.testing.assert_array_equal(np.where(m_bit == 1, np.where(s_bit == 1, 1, -1), 0), ref_t)
    np.testing.assert_array_equal(u32(tn.tn_requant(torch.from_numpy(y).cuda(), dev(lo), dev(hi))), yp)


# --------------------------------------------------------------------------- configs[4]: z-slabs
@pytest.mark.parametrize("shape,nslabs", [((1, 1, 32, 48, 48), 2), ((1, 1, 32, 48, 48), 4),
                                          ((1, 1, 64, 24, 40), 8)])
def test_fcn_slabs_local_bit_identical(tn, shape, nslabs):
    """All z-slabs on one device with halos exchanged by device copies (the overlapped schedule
    tn_fcn_forward_slab runs over NCCL: every interior plane is computed before the previous
    layer's halos are copied in, the boundary planes after) == the whole-volume forward, bit for
    bit.  The workspace starts as garbage, so an interior plane that read a halo would differ."""
    x = synth.ct_volume(shape, seed=11)
    p = synth.fcn_params()
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
    xd = dev(x)
    whole = net(xd).cpu().numpy()
    flag = tn.bad_flag()
    nb = int(tn.lib.tn_fcn_slabs_local_workspace_bytes(net.handle, tn.dims(*shape), nslabs))
    ws = torch.full((nb,), 0x5A, dtype=torch.uint8, device="cuda")
    slabs = net.forward_slabs_local(xd, nslabs, ws=ws, d_bad=flag).cpu().numpy()
    assert bad_value(flag) == tn.INT64_MAX
    np.testing.assert_array_equal(slabs, whole)
    ref, _, _ = oracle.fcn_forward(x, p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"])
    tol = np.maximum(np.abs(ref), _logit_tol(p["pred_w"], p["pred_b"]) / 1e-5) * 1e-5
    assert np.all(np.abs(slabs - ref) <= tol)


def test_fcn_slab_nccl_single_rank(tn):
    """tn_fcn_forward_slab through a 1-rank NCCL communicator (the degenerate slab)."""
    shape = (1, 1, 16, 32, 32)
    x = synth.ct_volume(shape, seed=12)
    p = synth.fcn_params()
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
    comm = tn.Comm(0, 1)
    xd = dev(x)
    got = net.forward_slab(comm, xd, shape, 0, shape[2]).cpu().numpy()
    np.testing.assert_array_equal(got, net(xd).cpu().numpy())
    # a non-multiple-of-8 slab is rejected before any work is queued
    with pytest.raises(tn.TNError):
        net.forward_slab(comm, xd, shape, 0, 12)


def test_fcn_nonfinite_input_reported(tn):
    """A non-finite CT value reaches d_bad as its flat NCDHW index (SPEC.md:39 pattern) through the
    batched FCN forward and through both slab schedules (global z offsets in bad_base)."""
    p = synth.fcn_params()
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
    shape = (2, 1, 16, 24, 40)
    x = synth.ct_volume(shape, seed=4)
    x[1, 0, 7, 3, 5] = np.nan
    x[1, 0, 9, 0, 0] = np.inf
    flag = tn.bad_flag()
    net(dev(x), d_bad=flag)
    _, obad = oracle.tern_f32(x, synth.CT_T_LO, synth.CT_T_HI)
    assert bad_value(flag) == obad == ((1 * 16 + 7) * 24 + 3) * 40 + 5
    shape = (1, 1, 32, 24, 40)
    x = synth.ct_volume(shape, seed=5)
    x[0, 0, 21, 2, 9] = -np.inf
    _, obad = oracle.tern_f32(x, synth.CT_T_LO, synth.CT_T_HI)
    for fn in (net.forward_slabs_local, net.forward_slabs_local_p2p):
        flag = tn.bad_flag()
        fn(dev(x), 2, d_bad=flag)
        assert bad_value(flag) == obad == (21 * 24 + 2) * 40 + 9


# --------------------------------------------------------------------------- NEXT-1: epilogue-fused halos
@pytest.mark.parametrize("shape,nslabs", [((1, 1, 32, 48, 48), 2), ((1, 1, 64, 24, 40), 8),
                                          ((1, 1, 16, 40, 56), 2)])
def test_fcn_slabs_local_p2p_bit_identical(tn, fcn_kernel, shape, nslabs):
    """NEXT-1 schedule on one device: every conv epilogue (TZ, popc, first layer) stores
    its boundary planes straight into the neighbouring slabs' halo planes and progress
    flags replace the copies; == the whole-volume forward bit for bit, also when the same
    workspace is reused (flags restart per call)."""
    x = synth.ct_volume(shape, seed=13)
    p = synth.fcn_params()
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
    xd = dev(x)
    whole = net(xd).cpu().numpy()
    nb = int(tn.lib.tn_fcn_slabs_local_workspace_bytes(net.handle, tn.dims(*shape), nslabs))
    ws = torch.full((nb,), 0x5A, dtype=torch.uint8, device="cuda")   # garbage halos must be overwritten
    flag = tn.bad_flag()
    for _ in range(2):
        got = net.forward_slabs_local_p2p(xd, nslabs, ws=ws, d_bad=flag).cpu().numpy()
        np.testing.assert_array_equal(got, whole)
    assert bad_value(flag) == tn.INT64_MAX


def test_fcn_halo_p2p_single_rank(tn):
    """The rank-side NEXT-1 entry points (tn_halo_create / export / connect /
    tn_fcn_forward_slab_p2p) with no neighbours: repeated forwards advance the epoch."""
    shape = (1, 1, 16, 32, 32)
    x = synth.ct_volume(shape, seed=14)
    p = synth.fcn_params()
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
    xd = dev(x)
    whole = net(xd).cpu().numpy()
    h = tn.HaloP2P(net, shape, 0, 1)
    assert int(tn.lib.tn_halo_workspace_bytes(h.handle)) > 0
    for _ in range(3):
        np.testing.assert_array_equal(h.forward(xd).cpu().numpy(), whole)
    del h


# --------------------------------------------------------------------------- NEXT-3: a float model prepared
def test_fcn_from_float_model_prepared_on_host(tn):
    """A float U-Net (random float filters + batch-norm statistics) prepared with the
    library's model-preparation calls -- Eq. 4 ternary weights (tn_ternarize_weights),
    alpha/BN/Eq. 6 folded into integer thresholds (tn_fold_thresholds), negated filters
    where the BN scale is negative -- then run by the FCN on the GPU: every layer's packed
    activations equal the oracle's with the same prepared parameters."""
    g = synth.rng(77)
    base = synth.fcn_params()
    weights, lo, hi = [], [], []
    for i, wt in enumerate(base["weights"]):
        k, c = wt.shape[:2]
        wf = (g.standard_normal(wt.shape) * g.uniform(0.02, 0.3)).astype(np.float32)
        codes, alpha = tn.tn_ternarize_weights(wf)
        o_codes, o_alpha = oracle.ternarize_weights(wf)
        np.testing.assert_array_equal(codes, o_codes)
        A = 27 * c
        sd_acc = np.sqrt(27 * c * 0.5 * (np.abs(codes.reshape(k, -1)) != 0).mean(1) + 1e-3)
        gamma = (g.standard_normal(k) * 0.8 + 0.2).astype(np.float32)
        beta = (g.standard_normal(k) * 0.3).astype(np.float32)
        mean = (g.standard_normal(k) * 0.3 * alpha * sd_acc).astype(np.float32)
        var = ((alpha * sd_acc) ** 2 * g.uniform(0.5, 2.0, k)).astype(np.float32)
        l, h, neg = tn.tn_fold_thresholds(alpha, gamma, beta, mean, var, 1e-5, A)
        tab = oracle.fold_table(alpha, gamma, beta, mean, var, 1e-5, A)
        acc = np.arange(-A, A + 1)
        for ch in range(k):
            a_eff = -acc if neg[ch] else acc
            assert np.array_equal(np.where(a_eff >= h[ch], 1, np.where(a_eff <= l[ch], -1, 0)), tab[ch])
        codes = np.where(neg.reshape((k,) + (1,) * (codes.ndim - 1)) == 1, -codes, codes).astype(np.int8)
        weights.append(codes)
        lo.append(l)
        hi.append(h)
    p = dict(base, weights=weights, lo=lo, hi=hi)
    x = synth.ct_volume((1, 1, 16, 24, 32), seed=78)
    _fcn_compare(tn, x, p)


# --------------------------------------------------------------------------- NEXT-4: Table 1's 2.5D U-Net
@pytest.mark.parametrize("n,h,w", [(3, 48, 64), (2, 240, 176)])
def test_fcn25_table1_network_matches_oracle(tn, n, h, w):
    """Table 1's ternary 2.5D U-Net (reading R18) on 15-slice stacks: the multi-channel input
    ternarised and packed, 2D layers as one-plane 3x3x3 convs (TZ up to 64 channels, popc beyond),
    stride-2 rows, 2D nearest upsampling (upsample 2) with skip concatenation, the 64-channel last
    layer with the unfused prediction: every layer bit-exact and the logits within R13."""
    p = synth.fcn25_params()
    x = synth.ct_stacks(n + 2, h, w, seed=12)[1:n + 1]
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"],
                        table=tn.fcn25_table(), c_in=15)
    ws = net.workspace(x.shape)
    flag = tn.bad_flag()
    logits = net(dev(x), ws=ws, d_bad=flag)
    assert bad_value(flag) == tn.INT64_MAX
    ref_logits, acts, bad = oracle.fcn25_forward(x, p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"],
                                                 p["pred_w"], p["pred_b"], want_acts=True)
    assert bad == -1
    for i in range(14):
        view, _ = net.layer_output(x.shape, ws, i)
        ref, _ = oracle.pack(acts[i])
        np.testing.assert_array_equal(u32(view), ref, err_msg=f"layer #{i + 1}")
    got = logits.cpu().numpy()
    tol = np.maximum(np.abs(ref_logits), _logit_tol(p["pred_w"], p["pred_b"]) / 1e-5) * 1e-5
    assert np.all(np.abs(got - ref_logits) <= tol)
    # a non-finite slice value is reported at its flat index through the multi-channel input pack
    x[1, 4, 0, 3, 5] = np.nan
    flag = tn.bad_flag()
    net(dev(x), ws=ws, d_bad=flag)
    assert bad_value(flag) == np.ravel_multi_index((1, 4, 0, 3, 5), x.shape)


# Threshold ties (reading R5: +1 iff acc >= hi, -1 iff acc <= lo): sparse filters put most
# accumulators on 0, +-1, +-2, and the thresholds sit exactly there -- lo = hi, lo = hi - 1,
# lo > hi, hi = 0 -- so every epilogue's compare (int8 acc - hi, the FP4 f32 start value
# 1/2 - hi, the K = 16 / 32 accumulator-start MMA, K = 64's zero start) meets its boundary
# values in bulk.  A compare that takes the sign of an exact zero wrongly fails here.
TIE_PAIRS = [(-1, 0), (0, 1), (-1, 1), (0, 0), (-2, 0), (0, 2), (1, 0), (-1, -1), (1, 1), (-2, 2), (2, 2), (-2, -2)]
TIE_CASES = [   # shape, k, stride, pad
    ((1, 16, 6, 20, 24), 16, 1, 1),
    ((1, 32, 5, 12, 40), 32, 1, 1),
    ((1, 64, 4, 10, 16), 64, 1, 1),
    ((1, 16, 1, 24, 40), 16, 1, 1),    # one plane (one-plane mode on FP4)
    ((1, 16, 6, 20, 24), 16, 2, 1),
    ((1, 48, 3, 9, 20), 32, 1, 1),     # ragged channel chunk
]


@pytest.mark.parametrize("case", TIE_CASES, ids=lambda c: "x".join(map(str, c[0])) + f"_k{c[1]}_s{c[2]}")
def test_conv3d_requant_threshold_ties(tn, kernel, case):
    shape, k, s, p = case
    seed = zlib.crc32(str(case).encode()) % 1000
    x = synth.ternary_codes(shape, 0.5, seed=seed)
    w = synth.ternary_codes((k, shape[1], 3, 3, 3), 1 - 6 / (27 * shape[1]), seed=seed + 1)   # ~6 nonzero taps
    lo = np.array([TIE_PAIRS[i % len(TIE_PAIRS)][0] for i in range(k)], dtype=np.int32)
    hi = np.array([TIE_PAIRS[i % len(TIE_PAIRS)][1] for i in range(k)], dtype=np.int32)
    acc = oracle.conv3d(x, w, s, p)
    ties = np.mean((acc == hi[None, :, None, None, None]) | (acc == lo[None, :, None, None, None]))
    assert ties > 0.25, f"the case must put accumulators on the thresholds ({ties:.2f})"
    ref, _ = oracle.pack(oracle.requant(acc, lo, hi))
    xp = tn.tn_pack_i8(dev(x))
    wp = tn.tn_pack_weights(dev(w))
    yp = run_or_skip(kernel, tn.tn_conv3d_requant, xp, tn.dims(*shape), wp, k, tn.geom(s, p), dev(lo), dev(hi))
    np.testing.assert_array_equal(u32(yp), ref)
    # the prepared-bank entry (the bench's and the FCN's path) too
    segs = [(xp, tn.dims(*shape), 0, wp)]
    prep = tn.tn_conv_prepare(segs, k, tn.geom(s, p))
    yp2 = run_or_skip(kernel, tn.tn_conv3d_seg_prepared, prep, segs, k, tn.geom(s, p), lo=dev(lo), hi=dev(hi))
    np.testing.assert_array_equal(u32(yp2), ref)
