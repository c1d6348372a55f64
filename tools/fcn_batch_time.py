"""configs[3] on one GPU: 8 volumes as 8 sequential forwards vs one batched forward (n = 8,
4, 2), and on 2 streams; device time per batch of 8 (CUDA events)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
cfg = synth.CONFIGS["C3"]; shape = cfg["vol_shape"]
p = synth.fcn_params(cfg["seed_params"])
net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"])
vols = [torch.from_numpy(synth.ct_volume(shape, seed=s)).cuda() for s in cfg["seeds"]]
s0 = torch.cuda.current_stream()
def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s0)
    for _ in range(reps): fn()
    b.record(s0); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
ws = net.workspace(shape); lg = torch.empty((1, 2) + shape[2:], device="cuda")
print("sequential n=1 x8: %.3f ms" % timeit(lambda: [net(v, logits=lg, ws=ws) for v in vols]))
ref = [net(v).clone() for v in vols]
for nb in (2, 4, 8):
    xb = torch.cat(vols[:nb], 0).contiguous()
    bshape = (nb,) + shape[1:]
    wsb = net.workspace(bshape); lgb = torch.empty((nb, 2) + shape[2:], device="cuda")
    out = net(xb, logits=lgb, ws=wsb)
    assert all(torch.equal(out[i:i+1], ref[i]) for i in range(nb))
    print("batched n=%d x%d: %.3f ms" % (nb, 8 // nb, timeit(lambda: [net(xb, logits=lgb, ws=wsb) for _ in range(8 // nb)])))
    del wsb
st = [torch.cuda.Stream() for _ in range(2)]
wss = [net.workspace(shape) for _ in range(2)]; lgs = [torch.empty((1, 2) + shape[2:], device="cuda") for _ in range(2)]
def two_streams():
    ev = torch.cuda.Event(); ev.record(s0)
    for s in st: s.wait_event(ev)
    for i, v in enumerate(vols):
        with torch.cuda.stream(st[i % 2]):
            net(v, logits=lgs[i % 2], ws=wss[i % 2], stream=st[i % 2])
    for s in st:
        e = torch.cuda.Event(); e.record(s); s0.wait_event(e)
print("2 streams: %.3f ms" % timeit(two_streams))
