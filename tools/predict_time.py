"""A8 prediction (tn_predict) on Table 1's last-layer shape: 138 stacks x 64 channels x 240 x 176."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
t = synth.ternary_codes((138, 64, 1, 240, 176), 0.5, seed=1)
tp = tn.tn_pack_i8(torch.from_numpy(t).cuda())
w, b = torch.randn(2, 64).cuda(), torch.randn(2).cuda()
out = tn.tn_predict(tp, 64, w, b)
for _ in range(3):
    tn.tn_predict(tp, 64, w, b, out)
torch.cuda.synchronize()
a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    tn.tn_predict(tp, 64, w, b, out)
c.record()
torch.cuda.synchronize()
us = a.elapsed_time(c) / 10 * 1e3
nb = tp.numel() * 4 + out.numel() * 4
print(f"predict {us:.1f} us  {nb / (us * 1e-6) / 1e9:.0f} GB/s")
