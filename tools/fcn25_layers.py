"""Per-layer device times of Table 1's 2.5D network (reading R18) over one ROI's 138 stacks
(tn_fcn_prepare first).  usage: python tools/fcn25_layers.py [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
p = synth.fcn25_params()
x = torch.from_numpy(synth.ct_stacks(synth.ROI_STACKS, synth.STACK_H, synth.STACK_W, seed=300)).cuda()
net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"],
                    table=tn.fcn25_table(), c_in=15)
net.prepare(tuple(x.shape))
ws = net.workspace(tuple(x.shape))
logits = torch.empty((x.shape[0], 2, 1, synth.STACK_H, synth.STACK_W), dtype=torch.float32, device="cuda")
net(x, logits=logits, ws=ws)
torch.cuda.synchronize()
L = len(net.table)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(L + 1)]
ms = np.zeros(L)
for _ in range(reps):
    torch.cuda._sleep(20_000_000)   # queue every launch before the GPU reaches them
    ev[0].record()
    for i in range(L):
        net.forward_range(x, i, i + 1 if i < L - 1 else -1, logits=logits, ws=ws)
        ev[i + 1].record()
    torch.cuda.synchronize()
    ms += [ev[i].elapsed_time(ev[i + 1]) for i in range(L)]
ms /= reps
for i in range(L):
    print(f"  #{i + 1:2d} {ms[i] * 1e3:8.1f} us")
print(f"  sum {ms.sum():.3f} ms")
