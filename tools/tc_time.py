"""Time TC conv launches back to back (CUDA-graph captured to remove host overhead)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
tn.tn_set_conv_kernel(tn.TN_KERNEL_TC)
for (shape, k) in (((1, 64, 64, 128, 128), 64), ((1, 16, 32, 256, 256), 16), ((1, 32, 32, 256, 256), 16),
                   ((1, 32, 32, 256, 256), 32), ((1, 64, 32, 256, 256), 32), ((1, 64, 32, 128, 128), 64)):
    x = synth.ternary_codes(shape, 0.5, seed=1); w = synth.ternary_codes((k, shape[1], 3, 3, 3), 0.6, seed=2)
    xp = tn.tn_pack_i8(dev(x)); wp = tn.tn_pack_weights(dev(w)); xd = tn.dims(*shape)
    lo, hi = synth.jittered_thresholds(k, 10, 1)
    lo_d, hi_d = dev(lo), dev(hi)
    yp = tn.tn_conv3d_requant(xp, xd, wp, k, tn.geom(), lo_d, hi_d)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10):
            tn.tn_conv3d_requant(xp, xd, wp, k, tn.geom(), lo_d, hi_d, yp)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 10 * 1e3
    macs = np.prod(shape[2:]) * shape[1] * k * 27
    print(f"{shape} k={k}: {us:.1f} us  {macs/us/1e6:.1f} TMAC/s  {2*macs/us/1e6/3349*100:.1f}% of i8 peak", flush=True)
