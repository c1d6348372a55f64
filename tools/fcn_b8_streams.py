"""configs[3]: one n = 8 forward vs two n = 4 forwards on two streams (device time)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
cfg = synth.CONFIGS["C3"]; shape = cfg["vol_shape"]
p = synth.fcn_params(cfg["seed_params"])
net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
x = torch.from_numpy(synth.ct_volume(shape, seed=100)).cuda().repeat(8, 1, 1, 1, 1).contiguous()
s0 = torch.cuda.current_stream()
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s0)
    for _ in range(reps): fn()
    b.record(s0); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
ws8 = net.workspace(x.shape); lg8 = torch.empty((8, 2) + shape[2:], device="cuda")
print("n=8 one stream: %.3f ms" % timeit(lambda: net(x, logits=lg8, ws=ws8)))
for parts in (2, 4):
    nb = 8 // parts
    st = [torch.cuda.Stream() for _ in range(parts)]
    xs = [x[i * nb:(i + 1) * nb] for i in range(parts)]
    wss = [net.workspace(xs[0].shape) for _ in range(parts)]
    lgs = [lg8[i * nb:(i + 1) * nb] for i in range(parts)]
    def run():
        ev = torch.cuda.Event(); ev.record(s0)
        for i in range(parts):
            st[i].wait_event(ev)
            net(xs[i], logits=lgs[i], ws=wss[i], stream=st[i])
        for i in range(parts):
            e = torch.cuda.Event(); e.record(st[i]); s0.wait_event(e)
    print("%d streams x n=%d: %.3f ms" % (parts, nb, timeit(run)))
