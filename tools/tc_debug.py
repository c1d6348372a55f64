import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1801_09449_b200 as tn
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
shape, k = (1, 64, 16, 128, 128), 64
x = synth.ternary_codes(shape, 0.5, seed=1); w = synth.ternary_codes((k, 64, 3, 3, 3), 0.6, seed=2)
xp = tn.tn_pack_i8(dev(x)); wp = tn.tn_pack_weights(dev(w)); xd = tn.dims(*shape)
tn.tn_set_conv_kernel(tn.TN_KERNEL_POPC)
yr = tn.tn_conv3d(xp, xd, wp, k, tn.geom()).cpu().numpy()
tn.tn_set_conv_kernel(tn.TN_KERNEL_TC)
for rep in range(4):
    y = torch.full((1, 16, 128, 128, 64), -7, dtype=torch.int32, device='cuda')
    torch.cuda.synchronize()
    t = time.time()
    tn.tn_conv3d(xp, xd, wp, k, tn.geom(), y=y)
    torch.cuda.synchronize()
    dt = time.time() - t
    yn = y.cpu().numpy()
    print(f"rep {rep}: {dt*1e6:.0f} us, equal {np.array_equal(yn, yr)}, untouched {np.mean(yn == -7):.4f}, err '{tn.lib.tn_last_error().decode()}'", flush=True)
