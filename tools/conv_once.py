"""Two conv3d_requant launches of one shape with one kernel, for ncu captures.
usage: python tools/conv_once.py C D H W K STRIDE {tz|tz8|popc|auto}"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
c, d, h, w, k, s = map(int, sys.argv[1:7])
kern = {"tz": tn.TN_KERNEL_TZ, "tz8": tn.TN_KERNEL_TZ8, "popc": tn.TN_KERNEL_POPC, "auto": tn.TN_KERNEL_AUTO}[sys.argv[7]]
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
shape = (1, c, d, h, w)
x = synth.ternary_codes(shape, 0.5, seed=1); wt = synth.ternary_codes((k, c, 3, 3, 3), 0.6, seed=2)
xp = tn.tn_pack_i8(dev(x)); wp = tn.tn_pack_weights(dev(wt)); xd = tn.dims(*shape)
lo, hi = synth.jittered_thresholds(k, 10, 1)
tn.tn_set_conv_kernel(kern)
for _ in range(2):
    tn.tn_conv3d_requant(xp, xd, wp, k, tn.geom(s), dev(lo), dev(hi))
torch.cuda.synchronize()
print("ok")
