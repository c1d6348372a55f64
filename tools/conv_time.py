"""Time one conv3d_requant launch per TZ operand type (FP4 / int8) on the FCN's configs[3] layer shapes
(CUDA-graph replays of 10 back-to-back launches, CUDA events)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
R0 = (128, 256, 256)
R1 = tuple(v // 2 for v in R0)
R2 = tuple(v // 4 for v in R0)
CASES = [  # (name, shape, k, stride)
    ("C1 64->64", (1, 64, 64, 128, 128), 64, 1),
    ("#2 16->16 R0", (1, 16) + R0, 16, 1),
    ("#3 16->16 s2", (1, 16) + R0, 16, 2),
    ("#4 16->32 R1", (1, 16) + R1, 32, 1),
    ("#5 32->32 s2", (1, 32) + R1, 32, 2),
    ("#6 32->64 R2", (1, 32) + R2, 64, 1),
    ("#10 64->32 R2", (1, 64) + R2, 32, 1),
    ("#12 32->16 R1", (1, 32) + R1, 16, 1),
    ("#7 64->64 s2", (1, 64) + R2, 64, 2),
]
sel = {"tz": tn.TN_KERNEL_TZ, "tz8": tn.TN_KERNEL_TZ8}
for name, shape, k, s in CASES:
    x = synth.ternary_codes(shape, 0.5, seed=1); w = synth.ternary_codes((k, shape[1], 3, 3, 3), 0.6, seed=2)
    xp = tn.tn_pack_i8(dev(x)); wp = tn.tn_pack_weights(dev(w)); xd = tn.dims(*shape)
    lo, hi = synth.jittered_thresholds(k, 10, 1)
    lo_d, hi_d = dev(lo), dev(hi)
    out = {}
    for kname, kv in sel.items():
        tn.tn_set_conv_kernel(kv)
        try:
            yp = tn.tn_conv3d_requant(xp, xd, wp, k, tn.geom(s), lo_d, hi_d)
        except tn.TNError:
            continue
        torch.cuda.synchronize()
        st = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(10):
                tn.tn_conv3d_requant(xp, xd, wp, k, tn.geom(s), lo_d, hi_d, yp)
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        out[kname] = (e0.elapsed_time(e1) / 10 * 1e3, u32 := yp.cpu().numpy().tobytes())
    tn.tn_set_conv_kernel(tn.TN_KERNEL_AUTO)
    od = [d // s for d in shape[2:]]
    macs = np.prod(od) * shape[1] * k * 27
    same = "" if len(out) < 2 else ("  (outputs identical)" if out["tz"][1] == out["tz8"][1] else "  OUTPUTS DIFFER")
    line = "  ".join(f"{kn}: {t:7.1f} us {macs / t / 1e6:7.1f} TMAC/s {2 * macs / t / 1e6 / 3325 * 100:5.1f}%"
                     for kn, (t, _) in out.items())
    print(f"{name:16s} {line}{same}", flush=True)
