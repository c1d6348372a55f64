"""Write tests/golden/bench_samples.npz: the expected values bench.py's parity gates compare
against (sampled C0 / C1 / binary outputs, and sampled FCN logits of configs[2], of configs[3]
volume 0 and of configs[4] inside an oracle-computable crop).  Calls only oracle/ and synth/
(the bench itself does not import the oracle outside its cpu_baseline leg and the --impl
reference arm).
usage: python tools/make_bench_golden.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import oracle
import synth


def ternary_at(x, w, lo, hi, at):
    acc = oracle.conv3d_at(x, w, at)
    out = np.empty(len(at), np.int8)
    for i, (a, k) in enumerate(zip(acc, at[:, 1])):
        out[i] = oracle.requant(np.array(a, np.int32).reshape(1, 1, 1, 1, 1), lo[k:k + 1], hi[k:k + 1])[0, 0, 0, 0, 0]
    return out


def logit_positions(region, m, seed):
    """m random (n=0, class, z, y, x) inside region = ((z0,z1),(y0,y1),(x0,x1)), plus its 8 corners."""
    g = synth.rng(seed)
    at = np.stack([np.zeros(m, int), g.integers(0, 2, m)] + [g.integers(a, b, m) for a, b in region], 1)
    corners = [[0, j % 2] + [region[a][(j >> (a + 1)) & 1] - ((j >> (a + 1)) & 1) for a in range(3)] for j in range(8)]
    at[:8] = corners
    return at.astype(np.int32)


def fcn_logits(cfg_name, crop=None):
    cfg = synth.CONFIGS[cfg_name]
    p = synth.fcn_params(cfg["seed_params"])
    x = synth.ct_volume(cfg["vol_shape"], seed=cfg["seeds"][0])
    if crop is not None:
        x = np.ascontiguousarray(x[(slice(None), slice(None)) + tuple(slice(o, o + n) for o, n in crop)])
    logits, _, bad = oracle.fcn_forward(x, p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"], p["pred_w"],
                                        p["pred_b"])
    assert bad == -1
    return logits


def fcn25_golden(out):
    """NEXT-4 (Table 1's 2.5D U-Net, reading R18): sampled logits of the first 4 of the bench's
    138 stacks (240 x 176); a stack depends only on its own 15 slices, so these need the oracle
    on 4 stacks only."""
    p = synth.fcn25_params()
    x = synth.ct_stacks(synth.ROI_STACKS, synth.STACK_H, synth.STACK_W, seed=300)[:4]
    lg, _, bad = oracle.fcn25_forward(x, p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"], p["pred_w"],
                                      p["pred_b"])
    assert bad == -1
    g = synth.rng(904)
    m = 512
    at = np.stack([g.integers(0, 4, m), g.integers(0, 2, m), np.zeros(m, int), g.integers(0, synth.STACK_H, m),
                   g.integers(0, synth.STACK_W, m)], 1).astype(np.int32)
    out["fcn25_at"] = at
    out["fcn25_ref"] = lg[tuple(at.T)]


path = os.path.join(ROOT, "tests", "golden", "bench_samples.npz")
if "--only-fcn25" in sys.argv:
    out = dict(np.load(path))
    fcn25_golden(out)
    np.savez_compressed(path, **out)
    print("updated", path)
    sys.exit(0)
out = {}
x0, w0, _, _ = synth.conv_config("C0")
out["c0_at"] = synth.sample_positions(x0.shape, 16, 512, seed=777)
out["c0_ref"] = oracle.conv3d_at(x0, w0, out["c0_at"]).astype(np.int32)
x1, w1, lo1, hi1 = synth.conv_config("C1")
out["c1_at"] = synth.sample_positions(x1.shape, 64, 256, seed=1234)
out["c1_ref"] = ternary_at(x1, w1, lo1, hi1, out["c1_at"])
xb, wb, lob, hib = synth.binary_config()
out["bin_at"] = synth.sample_positions(xb.shape, 64, 128, seed=4321)
out["bin_ref"] = ternary_at(xb, wb, lob, hib, out["bin_at"])
assert np.all(out["bin_ref"] != 0)

# FCN logits (oracle forward of whole volumes; configs[4] through a 128^3 crop at the volume's
# centre, sampled only where the crop's outputs equal the whole volume's: at least 44 voxels
# inside its lower faces and 37 inside its upper faces, the FCN's dependency interval)
for name, seed in (("C2", 901), ("C3", 902)):
    lg = fcn_logits(name)
    D, H, W = lg.shape[2:]
    at = logit_positions(((0, D), (0, H), (0, W)), 512, seed)
    out[f"fcn_{name.lower()}_at"] = at
    out[f"fcn_{name.lower()}_ref"] = lg[tuple(at.T)]
    print(name, "done", flush=True)
crop = ((64, 128), (192, 128), (320, 128))
lg = fcn_logits("C4", crop)
region = tuple((o + 44, o + n - 37) for o, n in crop)
at = logit_positions(region, 512, 903)
loc = at.copy()
for a in range(3):
    loc[:, 2 + a] -= crop[a][0]
out["fcn_c4_at"] = at
out["fcn_c4_ref"] = lg[tuple(loc.T)]
fcn25_golden(out)
np.savez_compressed(path, **out)
print("wrote", path)
