"""Quick GPU check of the tcgen05 conv against the popc conv and the oracle."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_1801_09449_b200 as tn

def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
cases = [((1, 16, 4, 5, 6), 16), ((1, 16, 32, 32, 32), 16), ((1, 64, 5, 7, 9), 64), ((1, 32, 6, 20, 130), 32),
         ((2, 32, 3, 4, 5), 64), ((1, 64, 8, 128, 128), 64)]
cases2 = [((1, 16, 8, 20, 36), 16), ((1, 32, 12, 18, 20), 32), ((1, 64, 10, 12, 14), 64), ((1, 16, 32, 64, 256), 16),
          ((1, 64, 9, 7, 5), 64)]
for shape, k in cases2:
    x = synth.ternary_codes(shape, 0.5, seed=5); w = synth.ternary_codes((k, shape[1], 3, 3, 3), 0.6, seed=6)
    xp = tn.tn_pack_i8(dev(x)); wp = tn.tn_pack_weights(dev(w)); xd = tn.dims(*shape)
    tn.tn_set_conv_kernel(tn.TN_KERNEL_POPC)
    yr = tn.tn_conv3d(xp, xd, wp, k, tn.geom(2)).cpu().numpy()
    tn.tn_set_conv_kernel(tn.TN_KERNEL_TC)
    y = tn.tn_conv3d(xp, xd, wp, k, tn.geom(2)).cpu().numpy()
    ok = np.array_equal(y, yr)
    msg = f"stride2 {shape} k={k}: tc==popc {ok}"
    if not ok:
        bad = np.argwhere(y != yr)
        msg += f" mismatches={len(bad)} first={bad[:3].tolist()}"
    print(msg, flush=True)
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

# timing on C1 (fused requant), both kernels
x, w, lo, hi = synth.conv_config("C1")
xp = tn.tn_pack_i8(dev(x)); wp = tn.tn_pack_weights(dev(w)); xd = tn.dims(*x.shape)
lo_d, hi_d = dev(lo), dev(hi)
res = {}
for name, sel in (("tc", tn.TN_KERNEL_TC), ("popc", tn.TN_KERNEL_POPC)):
    tn.tn_set_conv_kernel(sel)
    yp = tn.tn_conv3d_requant(xp, xd, wp, 64, tn.geom(), lo_d, hi_d)
    torch.cuda.synchronize()
    res[name] = yp.cpu().numpy()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20 if name == "tc" else 3
    e0.record()
    for _ in range(reps):
        tn.tn_conv3d_requant(xp, xd, wp, 64, tn.geom(), lo_d, hi_d, yp)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"C1 {name}: {ms*1e3:.1f} us  {115.964e9/ms/1e9:.1f} TMAC/s", flush=True)
print("C1 tc == popc (packed):", np.array_equal(res["tc"], res["popc"]))
# FCN layer-shaped cases (R0 of C3: 128x256x256) for K=16/C=16 and concat 16+16
for (c, k) in ((16, 16), (32, 16), (32, 32), (64, 32)):
    xs = synth.ternary_codes((1, c, 32, 256, 256), 0.5, seed=3)
    ws = synth.ternary_codes((k, c, 3, 3, 3), 0.6, seed=4)
    xp2 = tn.tn_pack_i8(dev(xs)); wp2 = tn.tn_pack_weights(dev(ws)); xd2 = tn.dims(*xs.shape)
    l2, h2 = synth.jittered_thresholds(k, 5, 1)
    outs = {}
    for name, sel in (("tc", tn.TN_KERNEL_TC), ("popc", tn.TN_KERNEL_POPC)):
        tn.tn_set_conv_kernel(sel)
        o = tn.tn_conv3d_requant(xp2, xd2, wp2, k, tn.geom(), dev(l2), dev(h2)); torch.cuda.synchronize()
        outs[name] = o.cpu().numpy()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            tn.tn_conv3d_requant(xp2, xd2, wp2, k, tn.geom(), dev(l2), dev(h2), o)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        macs = 32 * 256 * 256 * c * k * 27
        print(f"  c={c} k={k} 32x256x256 {name}: {ms*1e3:.1f} us {macs/ms/1e9:.1f} TMAC/s", flush=True)
    print("  equal:", np.array_equal(outs["tc"], outs["popc"]), flush=True)
