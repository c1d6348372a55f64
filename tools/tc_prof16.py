import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
tn.tn_set_conv_kernel(tn.TN_KERNEL_TC)
shape, k = (1, 16, 32, 256, 256), 16
x = synth.ternary_codes(shape, 0.5, seed=1); w = synth.ternary_codes((k, 16, 3, 3, 3), 0.6, seed=2)
xp = tn.tn_pack_i8(dev(x)); wp = tn.tn_pack_weights(dev(w)); xd = tn.dims(*shape)
lo, hi = synth.jittered_thresholds(k, 10, 1)
for _ in range(2):
    tn.tn_conv3d_requant(xp, xd, wp, k, tn.geom(), dev(lo), dev(hi))
torch.cuda.synchronize(); print("ok")
