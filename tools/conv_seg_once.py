"""Two launches of one two-segment conv [up_x2(a) | b] -> K (the FCN's decoder blocks), for ncu.
usage: python tools/conv_seg_once.py N D H W C_LOW C_SKIP K   (D, H, W = the skip segment's extents)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


n, D, H, W, cl, cs, k = (int(v) for v in sys.argv[1:8])
low = (D // 2, H // 2, W // 2)
a = synth.ternary_codes((n, cl) + low, 0.5, 1)
b = synth.ternary_codes((n, cs, D, H, W), 0.5, 2)
w = synth.ternary_codes((k, cl + cs, 3, 3, 3), 0.6, 3)
lo, hi = (dev(t) for t in synth.jittered_thresholds(k, 10, 1))
wa, wb = (tn.tn_pack_weights(dev(w[:, s])) for s in (slice(0, cl), slice(cl, cl + cs)))
segs = [(tn.tn_pack_i8(dev(a)), tn.dims(n, cl, *low), 1, wa), (tn.tn_pack_i8(dev(b)), tn.dims(n, cs, D, H, W), 0, wb)]
for _ in range(2):
    yp = tn.tn_conv3d_seg(segs, k, tn.geom(), lo, hi)
torch.cuda.synchronize()
print("ok")
