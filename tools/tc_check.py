"""Quick GPU check of the tcgen05 conv against the popc conv and the oracle."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_1801_09449_b200 as tn

def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
cases = [((1, 16, 4, 5, 6), 16), ((1, 16, 32, 32, 32), 16), ((1, 64, 5, 7, 9), 64), ((1, 32, 6, 20, 130), 32),
         ((2, 48, 3, 4, 5), 48), ((1, 64, 8, 128, 128), 64)]
for shape, k in cases:
    x = synth.ternary_codes(shape, 0.5, seed=1); w = synth.ternary_codes((k, shape[1], 3, 3, 3), 0.6, seed=2)
    xp = tn.tn_pack_i8(dev(x)); wp = tn.tn_pack_weights(dev(w)); xd = tn.dims(*shape)
    tn.tn_set_conv_kernel(tn.TN_KERNEL_POPC)
    yr = tn.tn_conv3d(xp, xd, wp, k, tn.geom()).cpu().numpy()
    tn.tn_set_conv_kernel(tn.TN_KERNEL_TC)
    t = time.time()
    y = tn.tn_conv3d(xp, xd, wp, k, tn.geom()); torch.cuda.synchronize()
    y = y.cpu().numpy()
    ok = np.array_equal(y, yr)
    msg = f"{shape} k={k}: tc==popc {ok}"
    if not ok:
        bad = np.argwhere(y != yr)
        msg += f" mismatches={len(bad)} first={bad[:3].tolist()} got={y[tuple(bad[0])]} ref={yr[tuple(bad[0])]}"
    if np.prod(shape) < 70000:
        ro = oracle.conv3d(x, w).transpose(0, 2, 3, 4, 1)
        msg += f" popc==oracle {np.array_equal(yr, ro)}"
    print(msg, flush=True)
