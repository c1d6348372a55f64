import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
shape, k = ((1, int(sys.argv[1]), 32, 256, 256), int(sys.argv[2]))
x = synth.ternary_codes(shape, 0.5, seed=1); w = synth.ternary_codes((k, shape[1], 3, 3, 3), 0.6, seed=2)
xp = tn.tn_pack_i8(dev(x)); wp = tn.tn_pack_weights(dev(w)); xd = tn.dims(*shape)
lo, hi = synth.jittered_thresholds(k, 10, 1)
tn.tn_set_conv_kernel(tn.TN_KERNEL_TC)
for _ in range(3):
    yp = tn.tn_conv3d_requant(xp, xd, wp, k, tn.geom(), dev(lo), dev(hi)); torch.cuda.synchronize()
buf = (ctypes.c_longlong * 2048)()
tn.lib.tn_exp_trace(buf, 2048)
t = np.array(buf[:]); t0 = t[0]
T = lambda i: int(t[i] - t0) if t[i] else None
print("macro: start acc_empty_ok planes_ok | committed | epi_full epi_done")
for m in range(24):
    print(m, [T(5*m+j) for j in range(3)], T(320+m), '|', T(400+m), T(500+m))
print("plane: loader_issued | batch: exp_pre_staged exp_post_staged exp_post_slot exp_arrived")
for g in range(40):
    print(g, T(1200+g), '|', T(1000+2*g), T(1001+2*g), T(601+2*g), T(800+g))
