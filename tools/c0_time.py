"""configs[0] launch time: CUDA-graph replays of 100 tn_conv3d launches (1x16x32^3, 16 -> 16, int32
output), as the bench's c0 block; unprepared (tn_conv3d) and prepared (tn_conv_prepare once +
tn_conv3d_seg_prepared, requant off).  usage: python tools/c0_time.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
x, w, _, _ = synth.conv_config("C0")
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
xp, wp, xd = tn.tn_pack_i8(dev(x)), tn.tn_pack_weights(dev(w)), tn.dims(*x.shape)
y = tn.tn_conv3d(xp, xd, wp, 16, tn.geom())
segs = [(xp, xd, 0, wp)]
prep = tn.tn_conv_prepare(segs, 16, tn.geom(), requant=False)
y2 = tn.tn_conv3d_seg_prepared(prep, segs, 16, tn.geom(), requant=False)
torch.cuda.synchronize()
print("prepared bytes", prep.nbytes, "equal", torch.equal(y, y2))


def run(fn, label):
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(100):
            fn(st)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 10)
    print(f"C0 {label}: {np.median(ts):.2f} us per launch (min {min(ts):.2f})")


run(lambda st: tn.tn_conv3d(xp, xd, wp, 16, tn.geom(), y=y, stream=st), "unprepared")
run(lambda st: tn.tn_conv3d_seg_prepared(prep, segs, 16, tn.geom(), y=y2, requant=False, stream=st), "prepared")
