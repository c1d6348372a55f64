"""Small end-to-end invocations of every kernel family for compute-sanitizer:
C0 conv (int32 and fused requant), a 64 -> 64 conv (C1's int8 class, split TMEM ring), a stride-2
conv, an odd-width conv (aligned-superset bulk rows), a two-segment upsample+concat conv, the
first layer, the popc kernel (dilation 2), pack/unpack, and a 16^3 FCN forward -- all with the
persistent grid capped at 3 CTAs (long runs of planes per CTA, ring wrap-around), each checked
against the oracle.  usage: compute-sanitizer --tool T python tools/sanitize_smoke.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_1801_09449_b200 as tn


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def u32(t):
    return t.cpu().numpy().view(np.uint32)


tn.tn_set_grid_cap(int(os.environ.get("TN_SAN_CAP", "3")))
checks = 0
for shape, k, s, dl, requant in [((1, 16, 8, 12, 16), 16, 1, 1, False), ((1, 16, 8, 12, 16), 16, 1, 1, True),
                                 ((1, 64, 5, 7, 12), 64, 1, 1, True), ((1, 32, 6, 8, 10), 32, 2, 1, True),
                                 ((1, 16, 3, 5, 7), 16, 1, 1, True), ((1, 16, 6, 7, 9), 16, 1, 2, True)]:
    x = synth.ternary_codes(shape, 0.5, seed=sum(shape))
    w = synth.ternary_codes((k, shape[1], 3, 3, 3), 0.6, seed=k + s)
    lo, hi = synth.jittered_thresholds(k, synth.threshold_base(shape[1], 0.5), seed=4)
    acc = oracle.conv3d(x, w, s, dl, dl)
    xp, wp = tn.tn_pack_i8(dev(x)), tn.tn_pack_weights(dev(w))
    if requant:
        got = u32(tn.tn_conv3d_requant(xp, tn.dims(*shape), wp, k, tn.geom(s, dl, dl), dev(lo), dev(hi)))
        ref, _ = oracle.pack(oracle.requant(acc, lo, hi))
    else:
        got = tn.tn_conv3d(xp, tn.dims(*shape), wp, k, tn.geom(s, dl, dl)).cpu().numpy()
        ref = acc.transpose(0, 2, 3, 4, 1)
    assert np.array_equal(got, ref), (shape, k, s, dl)
    assert np.array_equal(tn.tn_unpack(xp, shape[1]).cpu().numpy(), x)
    checks += 1
# two-segment nearest-x2 upsample + concat (A6)
a = synth.ternary_codes((1, 16, 3, 4, 5), 0.5, seed=1)
b = synth.ternary_codes((1, 16, 6, 8, 10), 0.5, seed=2)
w = synth.ternary_codes((16, 32, 3, 3, 3), 0.6, seed=3)
lo, hi = synth.jittered_thresholds(16, synth.threshold_base(32, 0.5), seed=5)
ref, _ = oracle.pack(oracle.requant(oracle.conv3d(oracle.concat(oracle.upsample2(a), b), w), lo, hi))
segs = [(tn.tn_pack_i8(dev(a)), tn.dims(1, 16, 3, 4, 5), 1, tn.tn_pack_weights(dev(w[:, :16]))),
        (tn.tn_pack_i8(dev(b)), tn.dims(1, 16, 6, 8, 10), 0, tn.tn_pack_weights(dev(w[:, 16:])))]
assert np.array_equal(u32(tn.tn_conv3d_seg(segs, 16, tn.geom(), dev(lo), dev(hi))), ref)
checks += 1
# first layer (A7) and the FCN (A1-A9)
p = synth.fcn_params()
v = synth.ct_volume((1, 1, 16, 16, 16), seed=5)
net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
got = net(dev(v)).cpu().numpy()
ref, _, _ = oracle.fcn_forward(v, p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"])
tol = 1e-5 * np.maximum(np.abs(ref), (np.abs(p["pred_b"]) + np.abs(p["pred_w"]).sum(1))[None, :, None, None, None])
assert np.all(np.abs(got - ref) <= tol)
checks += 1
torch.cuda.synchronize()
print(f"sanitize smoke ok ({checks} checks)")
