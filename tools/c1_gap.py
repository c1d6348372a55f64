"""Where the C1 conv's bench time goes: per-conv CUDA-event time under different
predecessors (back-to-back convs, after pack, after an L2 flush, both)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
x, w, lo, hi = synth.conv_config("C1")
xd = tn.dims(*x.shape)
x_d = dev(x)
xp = tn.tn_pack_i8(x_d); wp = tn.tn_pack_weights(dev(w))
lo_d, hi_d = dev(lo), dev(hi)
yp = tn.tn_conv3d_requant(xp, xd, wp, 64, tn.geom(), lo_d, hi_d)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
conv = lambda: tn.tn_conv3d_requant(xp, xd, wp, 64, tn.geom(), lo_d, hi_d, yp)
pack = lambda: tn.tn_pack_i8(x_d, xp)
def timed(pre, n=20):
    ts = []
    for _ in range(3):
        pre(); conv()
    for _ in range(n):
        pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); conv(); b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return np.median(ts), np.min(ts)
print("conv after conv (events around one)", timed(conv))
print("conv after pack", timed(pack))
print("conv after flush", timed(lambda: flush.zero_()))
print("conv after flush+pack", timed(lambda: (flush.zero_(), pack())))
print("conv after sleep", timed(lambda: torch.cuda._sleep(100000)))
# back-to-back average
for _ in range(5): conv()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s)
for _ in range(50): conv()
b.record(s); torch.cuda.synchronize()
print("back-to-back avg", a.elapsed_time(b) * 1e3 / 50)
def step_time(mid, n=20):
    ts = []
    for _ in range(n):
        flush.zero_()
        a, m, b = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(s); pack()
        if mid: m.record(s)
        conv(); b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return np.median(ts)
print("step flush|pack conv, middle event", step_time(True))
print("step flush|pack conv, no middle event", step_time(False))
scratch = torch.empty(64, dtype=torch.float32, device="cuda")
def clean_flush():
    flush.zero_()
    flush.view(torch.int32).sum()   # read back: dirty lines written out here
def step_time2(pre, n=20):
    ts = []
    for _ in range(n):
        pre()
        a, b = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        a.record(s); pack(); conv(); b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return np.median(ts)
print("step after zero_ flush", step_time2(lambda: flush.zero_()))
print("step after zero_+read flush", step_time2(clean_flush))
def pack_only(pre, n=20):
    ts = []
    for _ in range(n):
        pre()
        a, b = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        a.record(s); pack(); b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return np.median(ts)
print("pack after zero_ flush", pack_only(lambda: flush.zero_()))
print("pack after zero_+read flush", pack_only(clean_flush))
