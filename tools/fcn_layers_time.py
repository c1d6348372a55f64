"""Graph-replayed times of the configs[3] full-resolution FCN layer shapes (A7 first layer,
#2 16->16, #13 up(16)++16 -> 16, #14 16->16 + fused 2-class prediction) under AUTO."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
D, H, W = 128, 256, 256
lo, hi = synth.jittered_thresholds(16, 10, 1)
lo_d, hi_d = dev(lo), dev(hi)
x = dev(synth.ct_volume((1, 1, D, H, W), seed=3))
w1 = tn.tn_pack_weights(dev(synth.ternary_codes((16, 1, 3, 3, 3), 0.6, seed=2)))
a16 = tn.tn_pack_i8(dev(synth.ternary_codes((1, 16, D, H, W), 0.5, seed=4)))
l16 = tn.tn_pack_i8(dev(synth.ternary_codes((1, 16, D // 2, H // 2, W // 2), 0.5, seed=5)))
w16 = tn.tn_pack_weights(dev(synth.ternary_codes((16, 16, 3, 3, 3), 0.6, seed=6)))
w16b = tn.tn_pack_weights(dev(synth.ternary_codes((16, 16, 3, 3, 3), 0.6, seed=7)))
p = synth.fcn_params()
pw, pb = dev(p["pred_w"]), dev(p["pred_b"])
yp = tn.tn_conv3d_requant(a16, tn.dims(1, 16, D, H, W), w16, 16, tn.geom(), lo_d, hi_d)
logits = torch.empty((1, 2, D, H, W), device="cuda", dtype=torch.float32)
segs = [(l16, tn.dims(1, 16, D // 2, H // 2, W // 2), 1, w16), (a16, tn.dims(1, 16, D, H, W), 0, w16b)]
cases = {
    "#1 first": lambda: tn.tn_conv3d_first(x, synth.CT_T_LO, synth.CT_T_HI, w1, 16, tn.geom(), lo_d, hi_d, yp=yp),
    "#2 16->16": lambda: tn.tn_conv3d_requant(a16, tn.dims(1, 16, D, H, W), w16, 16, tn.geom(), lo_d, hi_d, yp),
    "#13 up16++16": lambda: tn.tn_conv3d_seg(segs, 16, tn.geom(), lo_d, hi_d, yp=yp),
}
if hasattr(tn, "tn_conv3d_predict"):
    cases["#14 +pred"] = lambda: tn.tn_conv3d_predict(a16, tn.dims(1, 16, D, H, W), w16, 16, lo_d, hi_d, pw, pb, yp, logits)
for name, fn in cases.items():
    fn(); torch.cuda.synchronize()
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(10):
            fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    print(f"{name:14s} {e0.elapsed_time(e1) / 10 * 1e3:7.1f} us", flush=True)
