"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/tn.h
declares, and its host-side validation answers without touching a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "tn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(tn_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


@pytest.fixture(scope="module")
def tn():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1801_09449_b200 as tn
    return tn


def test_library_exports_every_declared_symbol(tn):
    names = _declared_functions()
    assert len(names) >= 20
    raw = ctypes.CDLL(tn.LIB_PATH)
    for n in names:
        assert hasattr(raw, n), f"libtn.so does not export {n}"
    # the binding wraps exactly the declared set
    assert set(tn.SIGNATURES) == set(names)


def test_sizes_and_out_dims(tn):
    assert tn.lib.tn_packed_bytes(tn.dims(1, 64, 64, 128, 128)) == 1048576 * 16
    assert tn.lib.tn_packed_bytes(tn.dims(1, 16, 32, 32, 32)) == 32768 * 8
    assert tn.lib.tn_packed_bytes(tn.dims(2, 33, 1, 1, 1)) == 2 * 16
    assert tn.lib.tn_packed_bytes(tn.dims(0, 16, 4, 4, 4)) == 0
    assert tn.lib.tn_weight_bytes(64, 64) == 64 * 27 * 16
    od = tn.conv_out_dims(tn.dims(1, 16, 96, 144, 144), 16, tn.geom(2, 1, 1))
    assert (od.d, od.h, od.w, od.c) == (48, 72, 72, 16)
    od = tn.conv_out_dims(tn.dims(1, 3, 9, 9, 9), 5, tn.geom(1, 2, 2))
    assert (od.d, od.h, od.w) == (9, 9, 9)
    with pytest.raises(tn.TNError) as e:
        tn.conv_out_dims(tn.dims(1, 3, 1, 1, 1), 5, tn.geom(1, 0, 1))
    assert e.value.status == tn.TN_ESHAPE


def test_host_validation_before_any_launch(tn):
    d = tn.dims(1, 16, 4, 4, 4)
    g = tn.geom()
    assert tn.lib.tn_pack_i8(None, d, None, None, None) == tn.TN_EINVAL
    assert "NULL" in tn.lib.tn_last_error().decode()
    assert tn.lib.tn_pack_i8(ctypes.c_void_p(0x1003), d, ctypes.c_void_p(0x1000), None, None) == tn.TN_EALIGN
    assert tn.lib.tn_conv3d(None, d, None, 0, g, None, None) == tn.TN_EINVAL
    bad_g = tn.geom(0, 1, 1)
    assert tn.lib.tn_conv3d(ctypes.c_void_p(0x1000), d, ctypes.c_void_p(0x1000), 4, bad_g,
                            ctypes.c_void_p(0x1000), None) == tn.TN_EINVAL
    assert tn.lib.tn_pack_f32(ctypes.c_void_p(0x1000), tn.dims(1, 1, 4, 4, 4), 1.0, -1.0,
                              ctypes.c_void_p(0x1000), None, None) == tn.TN_EINVAL
    assert tn.lib.tn_conv3d_first(ctypes.c_void_p(0x1000), tn.dims(1, 2, 4, 4, 4), 0.0, 1.0,
                                  ctypes.c_void_p(0x1000), 16, g, ctypes.c_void_p(0x1000),
                                  ctypes.c_void_p(0x1000), ctypes.c_void_p(0x1000), None, None) == tn.TN_ESHAPE
    assert tn.lib.tn_predict(ctypes.c_void_p(0x1000), tn.dims(1, 65, 4, 4, 4), ctypes.c_void_p(0x1000),
                             ctypes.c_void_p(0x1000), 2, ctypes.c_void_p(0x1000), None) == tn.TN_EUNSUPPORTED
    # empty tensors are a successful no-op
    assert tn.lib.tn_pack_i8(None, tn.dims(1, 16, 0, 4, 4), None, None, None) == tn.TN_OK
    assert tn.lib.tn_set_conv_kernel(7) == tn.TN_EINVAL
    assert tn.lib.tn_set_conv_kernel(tn.TN_KERNEL_AUTO) == tn.TN_OK


def test_conv_prepare_host_logic(tn):
    """tn_conv_prepare validation, and a shape only the popc kernel covers: a handle holding no image,
    made without touching the device (no GPU here)."""
    g = tn.geom()
    h = ctypes.c_void_p()
    seg = (tn.tn_segment * 1)(tn.tn_segment(None, tn.dims(1, 128, 4, 5, 6), 0, 0x1000))
    assert tn.lib.tn_conv_prepare(seg, 1, 16, g, 1, None, None) == tn.TN_EINVAL
    assert tn.lib.tn_conv_prepare(None, 1, 16, g, 1, ctypes.byref(h), None) == tn.TN_EINVAL
    assert tn.lib.tn_conv_prepare(seg, 3, 16, g, 1, ctypes.byref(h), None) == tn.TN_EINVAL
    assert tn.lib.tn_conv_prepare(seg, 1, 0, g, 1, ctypes.byref(h), None) == tn.TN_EINVAL
    assert h.value is None
    assert tn.lib.tn_conv_prepare(seg, 1, 16, g, 1, ctypes.byref(h), None) == tn.TN_OK   # C = 128: popc
    assert h.value is not None and tn.lib.tn_conv_prep_bytes(h) == 0
    tn.lib.tn_conv_prep_destroy(h)
    tn.lib.tn_conv_prep_destroy(None)
    assert tn.lib.tn_conv_prep_bytes(None) == 0


def test_fcn_create_validation_and_workspace(tn):
    P = ctypes.c_void_p(0x1000)
    table = tn.fcn_table()
    layers = (tn.tn_layer * len(table))()
    for i, (kind, co, s, segs) in enumerate(table):
        L = layers[i]
        L.kind, L.c_out, L.stride, L.dil, L.nseg = kind, co, s, 1, len(segs)
        for j, (src, up) in enumerate(segs):
            L.src[j], L.upsample[j], L.wp[j] = src, up, 0x1000
        L.lo = L.hi = 0x1000
    h = ctypes.c_void_p()
    assert tn.lib.tn_fcn_create(layers, len(table), -200.0, 200.0, P, P, 2, ctypes.byref(h)) == tn.TN_OK
    ws = tn.lib.tn_fcn_workspace_bytes(h, tn.dims(1, 1, 96, 144, 144))
    R0 = 96 * 144 * 144
    # packed bytes/voxel: 8 for c <= 32, 16 for c = 64.  R0: #1 #2 #13 #14; R1: #3 #4 #11 #12;
    # R2: #5 (32) #6 (64) #9 (64) #10 (32); R3: #7 #8 (64)
    expect = 8 * R0 * 4 + 8 * (R0 // 8) * 4 + 48 * (R0 // 64) + 32 * (R0 // 512)
    assert abs(ws - expect) < 256 * 16
    tn.lib.tn_fcn_destroy(h)
    # a forward reference is rejected
    layers[3].src[0] = 5
    assert tn.lib.tn_fcn_create(layers, len(table), -200.0, 200.0, P, P, 2, ctypes.byref(h)) == tn.TN_EINVAL


def test_fcn_macs_per_voxel_matches_survey(tn):
    # 45,360 ternary MACs per input voxel; C2 = 90.30 G MAC
    assert tn.fcn_macs_per_voxel() == 45360
    assert abs(45360 * 96 * 144 * 144 / 1e9 - 90.30) < 0.01


def test_kernel_selection_host_logic(tn):
    """The per-shape kernel choice is host logic (no GPU): every configs[3] FCN layer and C1 run
    on the tap-offset tensor-core kernel (TZ); shapes outside it fall back to popc.  There is one
    tensor-core kernel: the retired dx-merged selector (2) is rejected."""
    d = tn.dims
    R0, R1, R2, R3 = (128, 256, 256), (64, 128, 128), (32, 64, 64), (16, 32, 32)
    tz, popc = tn.TN_KERNEL_TZ, tn.TN_KERNEL_POPC
    cases = [  # (segment dims, upsample flags, k, geom, expected)
        ([d(1, 64, 64, 128, 128)], None, 64, tn.geom(), tz),              # C1
        ([d(1, 16, *R0)], None, 16, tn.geom(), tz),                        # #2 / #14
        ([d(1, 16, *R0)], None, 16, tn.geom(2), tz),                       # #3
        ([d(1, 16, *R1)], None, 32, tn.geom(), tz),                        # #4
        ([d(1, 32, *R1)], None, 32, tn.geom(2), tz),                       # #5
        ([d(1, 64, *R2)], None, 64, tn.geom(2), tz),                       # #7 (FP4 operands)
        ([d(1, 64, *R3), d(1, 64, *R2)], [1, 0], 64, tn.geom(), tz),       # #9 (FP4, one pass)
        ([d(1, 16, *R1), d(1, 16, *R0)], [1, 0], 16, tn.geom(), tz),       # #13
        ([d(1, 16, 9, 17, 35)], None, 16, tn.geom(), tz),                  # odd W: aligned bulk rows
        ([d(1, 48, 9, 17, 35)], None, 32, tn.geom(), tz),                  # three 16-channel chunks
        ([d(1, 64, *R2)], None, 64, tn.geom(2), tz),                       # #7
        ([d(1, 16, 11, 12, 13)], None, 16, tn.geom(1, 2, 2), tz),          # dilation 2: z residue classes
        ([d(1, 16, 11, 12, 13)], None, 16, tn.geom(1, 1, 2), popc),        # pad != dilation
        ([d(1, 33, 6, 7, 8)], None, 5, tn.geom(), tz),                     # ragged C, K = 5: padded chunks
        ([d(1, 1, 5, 6, 7)], None, 3, tn.geom(), tz),                      # one channel, K = 3
        ([d(1, 128, 4, 5, 6)], None, 16, tn.geom(), popc),                 # C > 64: beyond the filter bank
        ([d(1, 16, 5, 6, 7)], None, 7, tn.geom((1, 2, 1), (0, 1, 2), (1, 1, 2)), popc),   # anisotropic
    ]
    for segs, up, k, g, want in cases:
        assert tn.tn_conv_kernel_for(segs, k, g, up) == want, (segs[0].c, k, want)
    # forced selectors answer for their own kernel only
    tn.tn_set_conv_kernel(tn.TN_KERNEL_TZ)
    try:
        assert tn.tn_conv_kernel_for([d(1, 64, 64, 128, 128)], 64, tn.geom()) == tz
        assert tn.tn_conv_kernel_for([d(1, 128, 4, 5, 6)], 16, tn.geom()) == -1
    finally:
        tn.tn_set_conv_kernel(tn.TN_KERNEL_AUTO)
    assert tn.lib.tn_set_conv_kernel(2) == tn.TN_EINVAL
    assert tn.lib.tn_set_grid_cap(-1) == tn.TN_EINVAL
    assert tn.lib.tn_set_grid_cap(0) == tn.TN_OK


def test_halo_p2p_host_validation(tn):
    """NEXT-1 setup calls validate before any allocation (no GPU needed)."""
    net = _dummy_fcn(tn)
    h = ctypes.c_void_p()
    # a slab that is not a multiple of the FCN's total downsampling (8)
    assert tn.lib.tn_halo_create(net, tn.dims(1, 1, 32, 16, 16), 0, 12, ctypes.byref(h)) == tn.TN_ESHAPE
    assert tn.lib.tn_halo_create(None, tn.dims(1, 1, 32, 16, 16), 0, 8, ctypes.byref(h)) == tn.TN_EINVAL
    assert tn.lib.tn_halo_export(None, None) == tn.TN_EINVAL
    assert tn.lib.tn_fcn_forward_slab_p2p(net, None, None, None, None, None) == tn.TN_EINVAL
    assert tn.lib.tn_halo_workspace_bytes(None) == 0
    tn.lib.tn_halo_destroy(None)
    # the single-device NEXT-1 schedule shares the emulation's workspace (+ 256 B of flags per slab)
    gd = tn.dims(1, 1, 32, 16, 16)
    per = sum(tn.lib.tn_fcn_slab_workspace_bytes(net, gd, 8 * r, 8 * r + 8) for r in range(4))
    assert tn.lib.tn_fcn_slabs_local_workspace_bytes(net, gd, 4) >= per + 4 * 256
    tn.lib.tn_fcn_destroy(net)


def _dummy_fcn(tn):
    table = tn.fcn_table()
    layers = (tn.tn_layer * len(table))()
    for i, (kind, co, s, segs) in enumerate(table):
        L = layers[i]
        L.kind, L.c_out, L.stride, L.dil, L.nseg = kind, co, s, 1, len(segs)
        for j, (src, up) in enumerate(segs):
            L.src[j], L.upsample[j], L.wp[j] = src, up, 0x1000
        L.lo = L.hi = 0x1000
    h = ctypes.c_void_p()
    P = ctypes.c_void_p(0x1000)
    assert tn.lib.tn_fcn_create(layers, len(table), -200.0, 200.0, P, P, 2, ctypes.byref(h)) == tn.TN_OK
    return h


@pytest.mark.parametrize("vol", [(96, 144, 144), (128, 256, 256), (256, 512, 512), (32, 48, 48)],
                         ids=["C2", "C3", "C4", "small"])
def test_every_fcn_layer_runs_on_the_tensor_core_kernel(tn, vol):
    """Host planning for every conv layer of the R9 FCN at the configs[2..4] volumes (and a small
    one): each plans onto the tcgen05 kernel (TZ) -- none silently falls back to popc (round-2
    regression: the 64+64 -> 64 block at configs[2]'s 36-wide R2 did)."""
    table = tn.fcn_table()
    ext = {}
    couts = [row[1] for row in table]
    for i, (kind, co, s, segs) in enumerate(table):
        if segs[0][0] < 0:
            ext[i] = vol
            continue
        src, up = segs[0]
        e = tuple(v * (2 if up else 1) for v in ext[src])
        dims = [tn.dims(1, couts[sj], *ext[sj]) for sj, _ in segs]
        ups = [u for _, u in segs]
        assert tn.tn_conv_kernel_for(dims, co, tn.geom(s), ups) == tn.TN_KERNEL_TZ, (vol, i + 1)
        ext[i] = tuple((v - 1) // s + 1 for v in e)


def test_fcn25_kernel_selection(tn):
    """Table 1's 2.5D U-Net (reading R18) at 240 x 176: the layers up to 64 channels plan onto the
    tensor-core kernel (TZ; 15 slice channels padded to 16), the 128 / 256-channel layers (whose
    filter banks exceed the resident B image) and the stride-1 64-channel decoder rows #13 / #14 onto
    the wide one-plane tensor-core kernel, with FP4 operands; under TZ8 (int8 operands only) the
    wide layers and #13 (128 input channels) fall back to popc, #14 to TZ."""
    table = tn.fcn25_table()
    couts = [row[1] for row in table]
    ext, picks, args = {}, [], []
    for i, (kind, co, s, segs) in enumerate(table):
        if segs[0][0] < 0:
            e, dims, ups = (1, 240, 176), [tn.dims(1, 15, 1, 240, 176)], [0]
        else:
            src, up = segs[0]
            z, y, x = ext[src]
            e = (z, y * 2, x * 2) if up else (z, y, x)
            dims, ups = [tn.dims(1, couts[sj], *ext[sj]) for sj, _ in segs], [u for _, u in segs]
        picks.append(tn.tn_conv_kernel_for(dims, co, tn.geom(s), ups))
        args.append((dims, co, tn.geom(s), ups))
        ext[i] = (1,) + tuple((v - 1) // s + 1 for v in e[1:])
    TZ, W = tn.TN_KERNEL_TZ, tn.TN_KERNEL_WIDE
    assert picks == [TZ, TZ, TZ, W, W, W, W, W, W, W, W, W, W, W]
    assert [tn.tn_conv_operands_for(d, co, g, u) for d, co, g, u in args[3:]] == [4] * 11
    try:
        tn.tn_set_conv_kernel(tn.TN_KERNEL_TZ8)
        assert [tn.tn_conv_kernel_for(d, co, g, u) for d, co, g, u in args[3:12]] == [tn.TN_KERNEL_POPC] * 9
        assert [tn.tn_conv_kernel_for(d, co, g, u) for d, co, g, u in args[12:]] == [tn.TN_KERNEL_POPC, TZ]
    finally:
        tn.tn_set_conv_kernel(tn.TN_KERNEL_AUTO)
