"""Per-role barrier-wait cycles of one TZ conv (needs the TN_TRACE build:
python paper_1801_09449_b200/build.py --trace; run with TN_LIBTN_PATH=paper_1801_09449_b200/libtn_trace.so).
usage: python tools/tz_trace.py C D H W K STRIDE [N]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn

c, d, h, w, k, s = (int(v) for v in sys.argv[1:7])
n = int(sys.argv[7]) if len(sys.argv) > 7 else 1
shape = (n, c, d, h, w)
x = synth.ternary_codes(shape, 0.5, 1)
wt = synth.ternary_codes((k, c, 3, 3, 3), 0.6, 2)
lo, hi = (torch.from_numpy(t).cuda() for t in synth.jittered_thresholds(k, 10, 1))
xp, wp = tn.tn_pack_i8(torch.from_numpy(x).cuda()), tn.tn_pack_weights(torch.from_numpy(wt).cuda())
yp = tn.tn_conv3d_requant(xp, tn.dims(*shape), wp, k, tn.geom(s), lo, hi)
rd = tn.lib.tn_trace_read
rd.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
buf = np.zeros(1024 * 8, np.uint64)
torch.cuda.synchronize()
rd(buf.ctypes.data, buf.size, 1)
yp = tn.tn_conv3d_requant(xp, tn.dims(*shape), wp, k, tn.geom(s), lo, hi, yp)
torch.cuda.synchronize()
rd(buf.ctypes.data, buf.size, 1)
t = buf.reshape(1024, 8)[:148].astype(np.float64)
names = ["kernel", "mma issue (fast path)", "exp staged wait", "exp slot wait", "mma plane wait", "mma acc wait",
         "epi acc wait", "mma role span"]
for i, nm in enumerate(names):
    print(f"{nm:16s} mean {t[:, i].mean():10.0f}  max {t[:, i].max():10.0f}  frac {t[:, i].mean() / t[:, 0].mean():.2f}")
