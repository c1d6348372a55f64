"""Per-role cycle breakdown (EXP_PROF build), averaged over CTAs."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
tn.tn_set_conv_kernel(tn.TN_KERNEL_TC)
for (shape, k) in (((1, 64, 64, 128, 128), 64), ((1, 16, 32, 256, 256), 16), ((1, 64, 32, 256, 256), 32)):
    x = synth.ternary_codes(shape, 0.5, seed=1); w = synth.ternary_codes((k, shape[1], 3, 3, 3), 0.6, seed=2)
    xp = tn.tn_pack_i8(dev(x)); wp = tn.tn_pack_weights(dev(w)); xd = tn.dims(*shape)
    lo, hi = synth.jittered_thresholds(k, 10, 1)
    for _ in range(3):
        tn.tn_conv3d_requant(xp, xd, wp, k, tn.geom(), dev(lo), dev(hi)); torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 4096)()
    tn.lib.tn_exp_trace(buf, 4096)
    t = np.array(buf[:2048]).reshape(128, 16)[:120].astype(float)
    m = t.mean(0)
    print(f"{shape} k={k}: planes/CTA {m[5]:.0f}, macro tiles {m[9]:.0f}")
    print(f"  expander total {m[0]:.0f}: staged-wait {m[1]:.0f}  slot-wait {m[2]:.0f}  work {m[3]:.0f}  fence {m[4]:.0f}")
    print(f"  mma total {m[6]:.0f}: acc_empty-wait {m[7]:.0f}  plane-wait {m[8]:.0f}")
    print(f"  epilogue total {m[10]:.0f}: acc_full-wait {m[11]:.0f}")
    print(f"  kernel total {m[15]:.0f} (max {t[:,15].max():.0f}): setup {m[14]:.0f} (max {t[:,14].max():.0f})")
    ss = np.array(buf[2560:2560 + 8 * 148]).reshape(148, 8)[:, :5].mean(0)
    print("  setup stamps (wstage, wexpand, ringzero, pred/thr, pre-alloc):", ss.astype(int))
    print(f"  loader total {m[12]:.0f}: staged_empty-wait {m[13]:.0f}", flush=True)
