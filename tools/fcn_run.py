"""One FCN forward of a configs[2..4] volume shape (for ncu launch lists).
usage: python tools/fcn_run.py [nb] [C2|C3]   (nb batched volumes; default 1 x C3 128x256x256)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 1   # batched volumes
name = sys.argv[2] if len(sys.argv) > 2 else "C3"
cfg = synth.CONFIGS[name]
shape = (nb,) + tuple(cfg["vol_shape"][1:])
p = synth.fcn_params(cfg["seed_params"])
net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
x = torch.from_numpy(synth.ct_volume((1,) + shape[1:], seed=cfg["seeds"][0])).cuda().repeat(nb, 1, 1, 1, 1).contiguous()
net.prepare(shape)
ws = net.workspace(shape)
for _ in range(2):
    net(x, ws=ws)
torch.cuda.synchronize()
print("ok")
