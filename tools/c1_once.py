"""One C1 step (tn_pack_i8 + tn_conv3d_requant, BASELINE configs[1]) for ncu --set full captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
x, w, lo, hi = synth.conv_config("C1")
xd = tn.dims(*x.shape)
xp = tn.tn_pack_i8(dev(x)); wp = tn.tn_pack_weights(dev(w))
lo_d, hi_d = dev(lo), dev(hi)
for _ in range(2):
    yp = tn.tn_conv3d_requant(xp, xd, wp, 64, tn.geom(), lo_d, hi_d)
torch.cuda.synchronize()
print("ok")
