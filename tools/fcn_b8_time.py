"""Device time of one batched (n = 8) configs[3] FCN forward (CUDA events, 5 reps)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
cfg = synth.CONFIGS["C3"]; shape = cfg["vol_shape"]
p = synth.fcn_params(cfg["seed_params"])
net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
x = torch.from_numpy(synth.ct_volume(shape, seed=100)).cuda().repeat(8, 1, 1, 1, 1).contiguous()
ws = net.workspace(x.shape); lg = torch.empty((8, 2) + shape[2:], device="cuda")
ref = net(x[:1].contiguous()).clone()
net(x, logits=lg, ws=ws); torch.cuda.synchronize()
assert torch.equal(lg[7:8], ref), "batched result differs"
s = torch.cuda.current_stream()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s)
for _ in range(5): net(x, logits=lg, ws=ws)
b.record(s); torch.cuda.synchronize()
print("batched n=8: %.3f ms" % (a.elapsed_time(b) / 5))
