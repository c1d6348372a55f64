"""configs[0] launch time vs the persistent grid cap (tn_set_grid_cap), prepared and unprepared filter
bank: where the fixed per-launch cost of a small layer goes.  usage: python tools/c0_sweep.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
x, w, _, _ = synth.conv_config("C0")
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
xp, wp, xd = tn.tn_pack_i8(dev(x)), tn.tn_pack_weights(dev(w)), tn.dims(*x.shape)
lo, hi = (dev(t) for t in synth.jittered_thresholds(16, 10, 1))
y = tn.tn_conv3d(xp, xd, wp, 16, tn.geom())
yp = tn.tn_conv3d_requant(xp, xd, wp, 16, tn.geom(), lo, hi)


def timed(fn, n=100):
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(n):
            fn(st)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / n)
    return np.median(ts)


for cap in (0, 96, 64, 32, 16, 8):
    tn.tn_set_grid_cap(cap)
    a = timed(lambda st: tn.tn_conv3d(xp, xd, wp, 16, tn.geom(), y=y, stream=st))
    b = timed(lambda st: tn.tn_conv3d_requant(xp, xd, wp, 16, tn.geom(), lo, hi, yp, stream=st))
    print(f"cap {cap:3d}: int32 {a:6.2f} us   requant {b:6.2f} us", flush=True)
tn.tn_set_grid_cap(0)
# an empty-ish launch floor: 1x16x1x8x8
x1 = synth.ternary_codes((1, 16, 1, 8, 8), 0.5, seed=3)
xp1, xd1 = tn.tn_pack_i8(dev(x1)), tn.dims(1, 16, 1, 8, 8)
y1 = tn.tn_conv3d(xp1, xd1, wp, 16, tn.geom())
print(f"1x16x1x8x8: {timed(lambda st: tn.tn_conv3d(xp1, xd1, wp, 16, tn.geom(), y=y1, stream=st)):6.2f} us")
