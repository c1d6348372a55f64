"""Time tn_pack_i8 on C1 codes (1x64x64x128x128): CUDA graph of 10 x (L2 flush + pack) minus
10 x flush, so host launch latency is not in the number."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
x, w, lo, hi = synth.conv_config("C1")
if len(sys.argv) > 1:   # optional shape override: N C D H W
    x = synth.ternary_codes(tuple(map(int, sys.argv[1:6])), 0.5, seed=10)
xd = torch.from_numpy(x).cuda()
xp = tn.tn_pack_i8(xd)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.Stream()
def graph(with_pack):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(10):
            flush.zero_()
            if with_pack:
                tn.lib.tn_pack_i8(tn._ptr(xd), tn.dims(*x.shape), tn._ptr(xp), None, tn._stream(None))
    return g
def run(g):
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / 10
ga, gb = graph(True), graph(False)
us = run(ga) - run(gb)
nb = x.size + x.size // x.shape[1] * 8 * ((x.shape[1] + 31) // 32)
print(f"pack {x.shape}: {us:.1f} us  {nb / us / 1e3:.0f} GB/s (flush-subtracted)")
