"""One configs[4] FCN forward (1 x 256 x 512 x 512) for ncu launch lists."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
cfg = synth.CONFIGS["C4"]; shape = cfg["vol_shape"]
p = synth.fcn_params(cfg["seed_params"])
net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
x = torch.from_numpy(synth.ct_volume((1, 1, 64, 512, 512), seed=200)).cuda().repeat(1, 1, 4, 1, 1).contiguous()
ws = net.workspace(shape)
for _ in range(2):
    net(x, ws=ws)
torch.cuda.synchronize()
print("ok")
