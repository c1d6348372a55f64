"""Pin the oracle's FCN (reading R9) against an independent float64 torch re-expression.

The torch version restates the network with library routines (conv3d,
interpolate, cat) and Eq. 6-style integer thresholds; it shares nothing with
oracle/tn_oracle.c except the inputs from synth/.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth

# (cin, cout, stride, source layers) restated for the torch pin; 0 = ternarised input.
TORCH_FCN = {
    1: (1, 16, 1, [0]), 2: (16, 16, 1, [1]), 3: (16, 16, 2, [2]), 4: (16, 32, 1, [3]),
    5: (32, 32, 2, [4]), 6: (32, 64, 1, [5]), 7: (64, 64, 2, [6]), 8: (64, 64, 1, [7]),
    9: (128, 64, 1, ["up8", 6]), 10: (64, 32, 1, [9]), 11: (64, 32, 1, ["up10", 4]),
    12: (32, 16, 1, [11]), 13: (32, 16, 1, ["up12", 2]), 14: (16, 16, 1, [13]),
}


def torch_fcn(x, p):
    f64 = lambda a: torch.from_numpy(np.asarray(a).astype(np.float64))
    xt = f64(x)
    # Eq. 6 on float32 values: +1 above t_hi, -1 below t_lo
    a = {0: (xt > float(np.float32(p["t_hi"]))).double() - (xt < float(np.float32(p["t_lo"]))).double()}
    for i in range(1, 15):
        cin, cout, s, src = TORCH_FCN[i]
        parts = []
        for sname in src:
            if isinstance(sname, str):
                parts.append(F.interpolate(a[int(sname[2:])], scale_factor=2, mode="nearest"))
            else:
                parts.append(a[sname])
        inp = torch.cat(parts, 1)
        acc = F.conv3d(inp, f64(p["weights"][i - 1]), stride=s, padding=1)
        lo = f64(p["lo"][i - 1]).reshape(1, -1, 1, 1, 1)
        hi = f64(p["hi"][i - 1]).reshape(1, -1, 1, 1, 1)
        pos = acc >= hi
        a[i] = pos.double() - ((acc <= lo) & ~pos).double()
    logits = F.conv3d(a[14], f64(p["pred_w"]).reshape(2, 16, 1, 1, 1), bias=f64(p["pred_b"]))
    return logits.numpy(), [a[i].numpy().astype(np.int8) for i in range(1, 15)]


@pytest.mark.parametrize("shape,seed", [((1, 1, 16, 16, 16), 5), ((1, 1, 32, 48, 48), 6),
                                        ((2, 1, 8, 16, 24), 7)])
def test_fcn_matches_torch_reexpression(shape, seed):
    x = synth.ct_volume(shape, seed=seed)
    p = synth.fcn_params()
    logits, acts, bad = oracle.fcn_forward(x, p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"],
                                           p["pred_w"], p["pred_b"], want_acts=True)
    assert bad == -1
    ref_logits, ref_acts = torch_fcn(x, p)
    for i in range(14):
        np.testing.assert_array_equal(acts[i], ref_acts[i], err_msg=f"layer #{i + 1}")
        # activations are not degenerate (the threshold recipe keeps all three values)
        assert set(np.unique(acts[i])) == {-1, 0, 1}, f"layer #{i + 1}"
    np.testing.assert_array_equal(logits, ref_logits.astype(np.float32))


def test_fcn_nan_input_reported():
    x = synth.ct_volume((1, 1, 8, 8, 8), seed=1)
    x[0, 0, 3, 2, 1] = np.nan
    p = synth.fcn_params()
    _, _, bad = oracle.fcn_forward(x, p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"],
                                   p["pred_w"], p["pred_b"])
    assert bad == np.ravel_multi_index((0, 0, 3, 2, 1), x.shape)
