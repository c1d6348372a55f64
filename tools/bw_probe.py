import torch, numpy as np
fw = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); fr = torch.zeros(32 << 20, dtype=torch.int64, device="cuda")
def t(fn, reps=20):
    for _ in range(3): fn()
    ts=[]
    for _ in range(reps):
        fw.zero_(); fr.sum()
        a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return np.median(ts)*1e3
x = torch.ones(64<<20, dtype=torch.uint8, device="cuda"); y = torch.empty(16<<20, dtype=torch.uint8, device="cuda")
y64 = torch.empty(64<<20, dtype=torch.uint8, device="cuda")
x80 = torch.ones(80<<20, dtype=torch.uint8, device="cuda")
print("copy 64MiB->64MiB us", t(lambda: y64.copy_(x)), "GB/s", 128*2**20/t(lambda: y64.copy_(x))/1e3)
print("copy 16MiB us", t(lambda: y.copy_(x[:16<<20])))
xs = x.view(torch.int64)
print("sum 64MiB us", t(lambda: xs.sum()), "GB/s", 64*2**20/t(lambda: xs.sum())/1e3)
print("copy 40MiB->40MiB (80MB traffic) us", t(lambda: x80[40<<20:].copy_(x80[:40<<20])))
