"""One tn_pack_i8 on C1 codes (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
x, w, lo, hi = synth.conv_config("C1")
xd = torch.from_numpy(x).cuda()
for _ in range(2):
    xp = tn.tn_pack_i8(xd)
torch.cuda.synchronize()
print("ok")
