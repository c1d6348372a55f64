"""Write tests/golden/bench_samples.npz: the expected values bench.py's parity gates compare
against (sampled C0 / C1 / binary outputs).  Calls only oracle/ and synth/ (the bench itself
does not import the oracle outside its cpu_baseline leg and the --impl reference arm).
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


x0, w0, _, _ = synth.conv_config("C0")
c0_at = synth.sample_positions(x0.shape, 16, 512, seed=777)
c0_ref = oracle.conv3d_at(x0, w0, c0_at).astype(np.int32)
x1, w1, lo1, hi1 = synth.conv_config("C1")
c1_at = synth.sample_positions(x1.shape, 64, 256, seed=1234)
c1_ref = ternary_at(x1, w1, lo1, hi1, c1_at)
xb, wb, lob, hib = synth.binary_config()
bin_at = synth.sample_positions(xb.shape, 64, 128, seed=4321)
bin_ref = ternary_at(xb, wb, lob, hib, bin_at)
assert np.all(bin_ref != 0)
out = os.path.join(ROOT, "tests", "golden", "bench_samples.npz")
np.savez_compressed(out, c0_at=c0_at, c0_ref=c0_ref, c1_at=c1_at, c1_ref=c1_ref, bin_at=bin_at, bin_ref=bin_ref)
print("wrote", out)
