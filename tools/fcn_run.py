"""One FCN forward on a C3-sized CT volume (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 1   # batched volumes
shape = (nb, 1, 128, 256, 256)
p = synth.fcn_params()
net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
x = torch.from_numpy(synth.ct_volume((1,) + shape[1:], seed=100)).cuda().repeat(nb, 1, 1, 1, 1).contiguous()
ws = net.workspace(shape)
for _ in range(2):
    net(x, ws=ws)
torch.cuda.synchronize()
print("ok")
