import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
import paper_1801_09449_b200 as tn
x, w, lo, hi = synth.conv_config("C1")
xd_, wp = torch.from_numpy(x).cuda(), tn.tn_pack_weights(torch.from_numpy(w).cuda())
lo_d, hi_d = torch.from_numpy(lo).cuda(), torch.from_numpy(hi).cuda()
xd, g = tn.dims(*x.shape), tn.geom()
xp, yp = tn.packed_empty(*x.shape), tn.packed_empty(*x.shape)
fw = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
fr = torch.zeros(32 << 20, dtype=torch.int64, device="cuda")
def flush(): fw.zero_(); fr.sum()
def step():
    tn.tn_pack_i8(xd_, xp); tn.tn_conv3d_requant(xp, xd, wp, 64, g, lo_d, hi_d, yp)
for _ in range(5): step()
torch.cuda.synchronize()
for pre in ("none", "sleep", "flush", "step", "sleep+step"):
    torch.cuda.synchronize()
    if "sleep" in pre: torch.cuda._sleep(4_000_000)
    if pre == "flush": flush()
    if "step" in pre: step()
    ev = []
    for i in range(6):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); step(); b.record(); ev.append((a, b))
    torch.cuda.synchronize()
    print(pre, [round(a.elapsed_time(b) * 1e3, 1) for a, b in ev], flush=True)
