"""Per-role cycle breakdown of the TZ kernel (TN_EXP_PROF build, TN_LIBTN_PATH=exp/libtn_prof.so).
usage: python tools/tz_rolprof.py C D H W K STRIDE"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
c, d, h, w, k, s = map(int, sys.argv[1:7])
shape = (1, c, d, h, w)
tn.tn_set_conv_kernel(tn.TN_KERNEL_TZ)
x = synth.ternary_codes(shape, 0.5, seed=1); wt = synth.ternary_codes((k, c, 3, 3, 3), 0.6, seed=2)
xp = tn.tn_pack_i8(dev(x)); wp = tn.tn_pack_weights(dev(wt)); xd = tn.dims(*shape)
lo, hi = synth.jittered_thresholds(k, 10, 1)
for _ in range(3):
    tn.tn_conv3d_requant(xp, xd, wp, k, tn.geom(s), dev(lo), dev(hi)); torch.cuda.synchronize()
buf = (ctypes.c_longlong * (148 * 16))()
tn.lib.tn_exp_tztrace(buf, 148 * 16)
m = np.array(buf[:]).reshape(148, 16).astype(float).mean(0)
print(f"{shape} k={k} s={s}: planes/CTA {m[5]:.1f}")
print(f"  loader   total {m[0]:9.0f}  staged_empty-wait {m[1]:9.0f}")
print(f"  expander total {m[2]:9.0f}  staged_full-wait {m[3]:9.0f}  plane_free-wait {m[4]:9.0f}")
print(f"  mma      total {m[6]:9.0f}  plane_full-wait {m[7]:9.0f}  acc_empty-wait {m[8]:9.0f}")
print(f"  epilogue total {m[9]:9.0f}  acc_full-wait {m[10]:9.0f}")
