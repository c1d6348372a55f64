import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
import paper_1801_09449_b200 as tn
shape = tuple(map(int, sys.argv[1:6]))
p = synth.fcn_params()
net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
x = torch.from_numpy(synth.ct_volume((1,) + shape[1:], seed=3)).cuda().repeat(shape[0], 1, 1, 1, 1).contiguous()
t0 = time.time()
out = net(x); torch.cuda.synchronize()
print(shape, "ok %.2f s" % (time.time() - t0), float(out.abs().sum()), flush=True)
