"""Per-layer and whole-forward device times of one FCN config (BASELINE configs[2..4]).
usage: python tools/fcn_layers.py {C2|C3|C4} [reps] [prep]   (prep: tn_fcn_prepare first)
Whole forward: eager stream launches (tn_fcn_forward) and one CUDA graph of `reps` forwards.
Per layer: a CUDA graph of `reps` back-to-back tn_fcn_forward_range(i, i+1) launches, timed
with events around one replay (no host launch gaps in the number)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = synth.CONFIGS[name]
p = synth.fcn_params(cfg["seed_params"])
net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
x = torch.cat([torch.from_numpy(synth.ct_volume(cfg["vol_shape"], seed=s)) for s in cfg["seeds"]], 0).cuda()
if len(sys.argv) > 3 and sys.argv[3] == "prep":
    print("prepared images:", net.prepare(tuple(x.shape)), "bytes")
ws = net.workspace(tuple(x.shape))
logits = torch.empty((x.shape[0], 2) + tuple(x.shape[2:]), dtype=torch.float32, device="cuda")
net(x, logits=logits, ws=ws)
torch.cuda.synchronize()


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def graph(fn):
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(reps):
            fn(st)
    g.replay()
    torch.cuda.synchronize()
    return g


eager = timed(lambda: [net(x, logits=logits, ws=ws) for _ in range(reps)]) / reps
gw = graph(lambda st: net(x, logits=logits, ws=ws, stream=st))
whole = timed(gw.replay) / reps
print(f"{name}: n={x.shape[0]} eager {eager:.3f} ms  graph {whole:.3f} ms per forward", flush=True)
L = len(net.table)
tot = 0.0
for i in range(L):
    gi = graph(lambda st, i=i: net.forward_range(x, i, i + 1 if i < L - 1 else -1, logits=logits, ws=ws, stream=st))
    t = timed(gi.replay) / reps
    tot += t
    print(f"  #{i + 1:2d} {t * 1e3:8.1f} us", flush=True)
print(f"  sum {tot:.3f} ms")
