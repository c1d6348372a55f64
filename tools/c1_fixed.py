"""Fixed vs per-plane cost of the C1-shaped conv (64->64, 128x128 planes): isolated
launches (after a GPU sleep) for D = 1..64 planes; the intercept is launch + prologue
+ pipeline fill + tail."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
s = torch.cuda.current_stream()
w = synth.ternary_codes((64, 64, 3, 3, 3), 0.6, seed=11)
wp = tn.tn_pack_weights(torch.from_numpy(w).cuda())
lo = torch.full((64,), -13, dtype=torch.int32, device="cuda"); hi = -lo
res = []
for D in (1, 2, 4, 8, 16, 32, 64):
    x = torch.from_numpy(synth.ternary_codes((1, 64, D, 128, 128), 0.5, seed=D)).cuda()
    xd = tn.dims(1, 64, D, 128, 128)
    xp = tn.tn_pack_i8(x)
    yp = tn.tn_conv3d_requant(xp, xd, wp, 64, tn.geom(), lo, hi)
    ts = []
    for i in range(15):
        torch.cuda._sleep(50000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); tn.tn_conv3d_requant(xp, xd, wp, 64, tn.geom(), lo, hi, yp); b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for i in range(20): tn.tn_conv3d_requant(xp, xd, wp, 64, tn.geom(), lo, hi, yp)
    b.record(s); torch.cuda.synchronize()
    res.append((D, np.median(ts[3:]), a.elapsed_time(b) * 1e3 / 20))
    print(f"D={D:3d} isolated {res[-1][1]:7.2f} us  back-to-back {res[-1][2]:7.2f} us", flush=True)
D = np.array([r[0] for r in res], float); t = np.array([r[1] for r in res])
m, c = np.polyfit(D[2:], t[2:], 1)
print(f"isolated fit (D>=4): {m:.3f} us/plane + {c:.2f} us fixed")
