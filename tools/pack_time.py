"""C1's A1 pack (tn_pack_i8, 1x64x64x128x128 int8 -> 2-bit planes) timed alone with a cold L2:
device time per launch (events), and the HBM rate on its algorithmic bytes (64 MiB + 16 MiB)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
x, _, _, _ = synth.conv_config("C1")
xd_ = torch.from_numpy(x).cuda()
xp = tn.packed_empty(*x.shape)
fw = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
fr = torch.zeros(32 << 20, dtype=torch.int64, device="cuda")
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for _ in range(3):
    tn.tn_pack_i8(xd_, xp)
ts = []
for _ in range(reps):
    fw.zero_(); fr.sum()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); tn.tn_pack_i8(xd_, xp); b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
nb = x.size + xp.numel() * 4
print(f"pack median {np.median(ts) * 1e3:.2f} us  min {np.min(ts) * 1e3:.2f} us  "
      f"{nb / (np.median(ts) * 1e-3) / 1e9:.0f} GB/s", flush=True)
