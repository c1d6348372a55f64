"""NEXT-4: the oracle's statement of Table 1's 2.5D U-Net (reading R18), pinned (CPU only).

* Accounting: Table 1's MFlops column = out_h * out_w * kernel * cin * cout of
  every layer of oracle.FCN25_LAYERS at the printed sizes (tests/golden/table1_mflops.txt), and at
  the AvgPool2D rows' sizes for the stride-2 readings of #3 / #5 / #7 (R8) -- this pins every
  layer's channels, kernel size and stride against the paper's own numbers.
* Upsample2D: oracle.upsample2_yx equals torch's nearest interpolation in y and x.
* The whole network: oracle.fcn25_forward equals a float64 torch re-expression written from
  Table 1 (conv2d with 3x3 / 1x1 kernels, stride 2, nearest x2, cat, Eq. 6 thresholds,
  integer requant, 1x1 prediction) on small stacks, every layer and the logits.
"""
import os

import numpy as np
import torch
import torch.nn.functional as F

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _table1():
    rows = {}
    for line in open(os.path.join(GOLDEN, "table1_mflops.txt")):
        if line.startswith("#") or not line.strip():
            continue
        f = line.split()
        rows[int(f[0])] = dict(h=int(f[1]), w=int(f[2]), kel=int(f[3]), cin=int(f[4]), cout=int(f[5]),
                               mflops=int(f[6]), use=f[7] == "y")
    return rows


def test_fcn25_layer_table_reproduces_table1_mflops():
    rows = _table1()
    # sizes the MFlops imply where the printed (out)-size column is garbled: the stride-2 convs
    # produce the AvgPool2D rows' sizes (R8), #13 / #14 are 2 pixels larger than printed
    implied = {3: (114, 82), 5: (54, 38), 7: (26, 18), 13: (182, 118), 14: (180, 116)}
    for i, (cin, cout, k, s, skip) in enumerate(oracle.FCN25_LAYERS):
        r = rows[i + 1]
        h, w = (r["h"], r["w"]) if r["use"] else implied[i + 1]
        assert cout == r["cout"], i + 1
        assert k * k * cin == r["kel"] * r["cin"], i + 1          # #1: 3x3 over 15 slices = 3x3x15 x 1
        assert round(h * w * k * k * cin * cout / 1e6) == r["mflops"], (i + 1, h * w * k * k * cin * cout / 1e6)
        assert s == (2 if i + 1 in (3, 5, 7) else 1)
    # skips #2 -> #13, #4 -> #11, #6 -> #9 (Table 1's skip column), concatenated after the upsample
    assert [(i + 1, sk + 1) for i, (_, _, _, _, sk) in enumerate(oracle.FCN25_LAYERS) if sk is not None] == \
        [(9, 6), (11, 4), (13, 2)]


def test_upsample2_yx_is_nearest_interpolation():
    x = synth.ternary_codes((2, 3, 2, 5, 7), 0.5, seed=3)
    got = oracle.upsample2_yx(x)
    ref = F.interpolate(torch.from_numpy(x).double(), scale_factor=(1, 2, 2), mode="nearest").numpy()
    np.testing.assert_array_equal(got, ref.astype(np.int8))


def _torch_fcn25(x, p):
    """Float64 re-expression of Table 1's ternary 2.5D U-Net from its rows (reading R18)."""
    t = torch.from_numpy(x[:, :, 0]).double()                      # [n][15][h][w]
    t = torch.where(t > p["t_hi"], 1.0, torch.where(t < p["t_lo"], -1.0, 0.0)).double()
    acts, cur = [], t
    spec = [(3, 1, None), (3, 1, None), (3, 2, None), (3, 1, None), (3, 2, None), (3, 1, None), (1, 2, None),
            (1, 1, None), (3, 1, 5), (3, 1, None), (3, 1, 3), (3, 1, None), (3, 1, 1), (3, 1, None)]
    for i, (k, s, skip) in enumerate(spec):
        if skip is not None:
            cur = torch.cat([F.interpolate(cur, scale_factor=2, mode="nearest"), acts[skip]], 1)
        w3 = torch.from_numpy(p["weights"][i]).double()
        w2 = w3[:, :, 1] if k == 3 else w3[:, :, 1, 1:2, 1:2]
        acc = F.conv2d(cur, w2, stride=s, padding=k // 2)
        lo = torch.from_numpy(p["lo"][i]).double()[None, :, None, None]
        hi = torch.from_numpy(p["hi"][i]).double()[None, :, None, None]
        cur = torch.where(acc >= hi, 1.0, torch.where(acc <= lo, -1.0, 0.0)).double()
        acts.append(cur)
    w = torch.from_numpy(p["pred_w"]).double()
    logits = torch.einsum("jc,nchw->njhw", w, cur) + torch.from_numpy(p["pred_b"]).double()[None, :, None, None]
    return logits.numpy(), [a.numpy() for a in acts]


def test_oracle_fcn25_matches_torch_reexpression():
    p = synth.fcn25_params()
    x = synth.ct_stacks(3, 24, 40, seed=9)[1:3]                  # two stacks
    logits, acts, bad = oracle.fcn25_forward(x, p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"],
                                             p["pred_w"], p["pred_b"], want_acts=True)
    assert bad == -1
    ref_logits, ref_acts = _torch_fcn25(x, p)
    for i, (a, r) in enumerate(zip(acts, ref_acts)):
        np.testing.assert_array_equal(a[:, :, 0], r.astype(np.int8), err_msg=f"layer #{i + 1}")
        assert set(np.unique(a)) == {-1, 0, 1}, i                 # every layer exercises all three values
    np.testing.assert_allclose(logits[:, :, 0], ref_logits, rtol=0, atol=1e-5 * (np.abs(p["pred_w"]).sum() + 1))


def test_ct_stacks_are_neighbouring_slices():
    """A stack holds slices s-7 .. s+7 of one CT-like volume, zero outside."""
    st = synth.ct_stacks(10, 8, 8, seed=4)
    vol = synth.ct_volume((1, 1, 10, 8, 8), 4)[0, 0]
    np.testing.assert_array_equal(st[3, 7, 0], vol[3])
    np.testing.assert_array_equal(st[3, 9, 0], vol[5])
    assert not st[3, 0, 0].any() and not st[9, 14, 0].any()      # slices -4 and 16: outside
