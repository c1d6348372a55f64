"""configs[3] batch (8 CT volumes 128x256x256) through tn_fcn_forward: eager stream launches vs one
CUDA graph of the whole batch (host launch overhead check)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
cfg = synth.CONFIGS["C3"]
p = synth.fcn_params(cfg["seed_params"])
net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
shape = cfg["vol_shape"]
vols = [torch.from_numpy(synth.ct_volume(shape, seed=s)).cuda() for s in cfg["seeds"]]
ws = net.workspace(shape)
logits = torch.empty((1, 2) + shape[2:], dtype=torch.float32, device="cuda")
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for v in vols: net(v, logits=logits, ws=ws)
torch.cuda.synchronize()
def timed(fn, reps=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        t0 = time.perf_counter()
        for _ in range(reps): fn()
        t1 = time.perf_counter()
        e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, (t1 - t0) * 1e3 / reps
def eager():
    for v in vols: net(v, logits=logits, ws=ws)
ms, host = timed(eager)
print(f"eager: {ms:.3f} ms per batch on the device, host enqueue {host:.3f} ms")
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    eager()
g.replay(); torch.cuda.synchronize()
ms2, host2 = timed(g.replay)
print(f"graph: {ms2:.3f} ms per batch on the device, host enqueue {host2:.3f} ms")
