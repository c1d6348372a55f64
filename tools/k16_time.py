"""Device time of one TZ conv3d_requant launch of the K = 16 FCN layer #2 shape (16 -> 16 at R0, one
volume) as CUDA-graph replays of 10 launches; for A/B builds via TN_LIBTN_PATH.
usage: python tools/k16_time.py [C D H W K STRIDE]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
c, d, h, w, k, s = map(int, sys.argv[1:7]) if len(sys.argv) > 6 else (16, 128, 256, 256, 16, 1)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
shape = (1, c, d, h, w)
xp = tn.tn_pack_i8(dev(synth.ternary_codes(shape, 0.5, seed=1)))
wp = tn.tn_pack_weights(dev(synth.ternary_codes((k, c, 3, 3, 3), 0.6, seed=2)))
lo, hi = (dev(t) for t in synth.jittered_thresholds(k, 10, 1))
xd = tn.dims(*shape)
y = tn.tn_conv3d_requant(xp, xd, wp, k, tn.geom(s), lo, hi)
st = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for _ in range(10):
        tn.tn_conv3d_requant(xp, xd, wp, k, tn.geom(s), lo, hi, y, stream=st)
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(5):
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 10 * 1e3)
print(f"{os.environ.get('TN_LIBTN_PATH', 'libtn.so')}: {shape} K={k} s={s}: median {np.median(ts):.1f} us  min {min(ts):.1f} us")
