"""Per-role cycle breakdown of the TZ kernel (TN_EXP_PROF build: TN_LIBTN_PATH=exp/libtn_prof.so).
usage: python tools/tz_rolprof.py conv C D H W K STRIDE
       python tools/tz_rolprof.py first D H W K
       python tools/tz_rolprof.py seg CUP CSKIP D H W K       (nearest-x2 CUP @ D/2 ++ CSKIP @ D)
       python tools/tz_rolprof.py pred D H W                  (16 -> 16 + fused 2-class prediction)"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
mode, args = sys.argv[1], list(map(int, sys.argv[2:]))
tn.tn_set_conv_kernel(tn.TN_KERNEL_TZ)
lo, hi = synth.jittered_thresholds(32, 10, 1)
if mode == "conv":
    c, d, h, w, k, s = args
    x = synth.ternary_codes((1, c, d, h, w), 0.5, seed=1); wt = synth.ternary_codes((k, c, 3, 3, 3), 0.6, seed=2)
    xp, wp, xd = tn.tn_pack_i8(dev(x)), tn.tn_pack_weights(dev(wt)), tn.dims(1, c, d, h, w)
    run = lambda: tn.tn_conv3d_requant(xp, xd, wp, k, tn.geom(s), dev(lo[:k]), dev(hi[:k]))
elif mode == "first":
    d, h, w, k = args
    x = dev(synth.ct_volume((1, 1, d, h, w), seed=3)); wt = synth.ternary_codes((k, 1, 3, 3, 3), 0.6, seed=2)
    wp = tn.tn_pack_weights(dev(wt))
    run = lambda: tn.tn_conv3d_first(x, synth.CT_T_LO, synth.CT_T_HI, wp, k, tn.geom(), dev(lo[:k]), dev(hi[:k]))
elif mode == "seg":
    cu, cs, d, h, w, k = args
    a = synth.ternary_codes((1, cu, d // 2, h // 2, w // 2), 0.5, seed=4)
    b = synth.ternary_codes((1, cs, d, h, w), 0.5, seed=5)
    wa = tn.tn_pack_weights(dev(synth.ternary_codes((k, cu, 3, 3, 3), 0.6, seed=6)))
    wb = tn.tn_pack_weights(dev(synth.ternary_codes((k, cs, 3, 3, 3), 0.6, seed=7)))
    segs = [(tn.tn_pack_i8(dev(a)), tn.dims(1, cu, d // 2, h // 2, w // 2), 1, wa),
            (tn.tn_pack_i8(dev(b)), tn.dims(1, cs, d, h, w), 0, wb)]
    run = lambda: tn.tn_conv3d_seg(segs, k, tn.geom(), dev(lo[:k]), dev(hi[:k]))
else:
    raise SystemExit(__doc__)
for _ in range(3):
    run(); torch.cuda.synchronize()
buf = (ctypes.c_longlong * (148 * 16))()
tn.lib.tn_exp_tztrace(buf, 148 * 16)
A = np.array(buf[:]).reshape(148, 16).astype(float)
os.makedirs("gpurun_out", exist_ok=True)
np.save(f"gpurun_out/tzprof_{mode}_{'_'.join(map(str, args))}.npy", A)
m = A.mean(0)
gs, ge = A[:, 13], A[:, 14]
print(f"  kernel cycles mean {m[12]:.0f} max {A[:,12].max():.0f}; setup mean {m[11]:.0f} (weights staged at {m[15]:.0f}); "
      f"globaltimer span {(ge.max() - gs.min()) / 1e3:.1f} us, CTA start spread {(gs.max() - gs.min()) / 1e3:.1f} us, "
      f"end spread {(ge.max() - ge.min()) / 1e3:.1f} us")
print(f"{mode} {args}: planes/CTA {m[5]:.1f}")
print(f"  loader   total {m[0]:9.0f}  staged_empty-wait {m[1]:9.0f}")
print(f"  expander total {m[2]:9.0f}  staged_full-wait {m[3]:9.0f}  plane_free-wait {m[4]:9.0f}")
print(f"  mma      total {m[6]:9.0f}  plane_full-wait {m[7]:9.0f}  acc_empty-wait {m[8]:9.0f}")
print(f"  epilogue total {m[9]:9.0f}  acc_full-wait {m[10]:9.0f}")
