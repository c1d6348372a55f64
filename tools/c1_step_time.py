"""C1 step timing (tn_pack_i8 + tn_conv3d_requant, PDL) with the bench's L2 flush between steps;
optionally with an NVML clock-sampling thread running (argv[1] = sampling period in ms)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
x, w, lo, hi = synth.conv_config("C1")
xd_, wp = torch.from_numpy(x).cuda(), tn.tn_pack_weights(torch.from_numpy(w).cuda())
lo_d, hi_d = torch.from_numpy(lo).cuda(), torch.from_numpy(hi).cuda()
xd, g = tn.dims(*x.shape), tn.geom()
xp, yp = tn.packed_empty(*x.shape), tn.packed_empty(*x.shape)
fw = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
fr = torch.zeros(32 << 20, dtype=torch.int64, device="cuda")
def flush():
    fw.zero_(); fr.sum()
prep = tn.tn_conv_prepare([(None, xd, 0, wp)], 64, g)
def sep():
    tn.tn_pack_i8(xd_, xp); tn.tn_conv3d_requant(xp, xd, wp, 64, g, lo_d, hi_d, yp)
def sep_prep():
    tn.tn_pack_i8(xd_, xp); tn.tn_conv3d_requant_prepared(prep, xp, xd, wp, 64, g, lo_d, hi_d, yp)
def conv():
    tn.tn_conv3d_requant(xp, xd, wp, 64, g, lo_d, hi_d, yp)
def conv_prep():
    tn.tn_conv3d_requant_prepared(prep, xp, xd, wp, 64, g, lo_d, hi_d, yp)
import threading, time
stop = threading.Event()
period = float(sys.argv[1]) / 1e3 if len(sys.argv) > 1 else 0.0
if period > 0:
    import pynvml
    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
    def poll():
        while not stop.is_set():
            pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(hnd)
            time.sleep(period)
    threading.Thread(target=poll, daemon=True).start()
for name, fn in (("step", sep), ("step_prep", sep_prep), ("conv", conv), ("conv_prep", conv_prep),
                 ("step", sep), ("step_prep", sep_prep)):
    for _ in range(3): fn()
    ts = []
    for _ in range(20):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{name:9s} mean {np.mean(ts) * 1e3:6.1f} us  median {np.median(ts) * 1e3:6.1f} us  min {np.min(ts) * 1e3:6.1f} us",
          flush=True)
