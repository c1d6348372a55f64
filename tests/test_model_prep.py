"""Model preparation: Eq. 4 ternary weights and the fold of alpha, batch
norm and Eq. 6 into the integer thresholds.  The oracle is pinned to the paper's worked
examples and to exact rational arithmetic; the library's host implementation
(tn_ternarize_weights / tn_fold_thresholds) must then match the oracle exactly."""
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

ROOT = os.path.dirname(os.path.abspath(__file__))


def _examples():
    rows = []
    for line in open(os.path.join(ROOT, "golden", "eq4_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        sp, w, c, a = [f.strip() for f in line.split("|")]
        rows.append((None if sp == "-" else float(sp), np.array(w.split(), np.float32),
                     np.array(c.split(), np.int8), float(a)))
    return rows


@pytest.fixture(scope="module")
def tn():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1801_09449_b200 as tn
    return tn


def test_oracle_eq4_worked_examples():
    for sp, w, codes, alpha in _examples():
        c, a = oracle.ternarize_weights(w[None], sp)
        np.testing.assert_array_equal(c[0], codes)
        assert abs(float(a[0]) - alpha) < 1e-6


def test_oracle_eq4_invariants():
    g = synth.rng(41)
    w = g.normal(0, 1, (32, 16, 3, 3, 3)).astype(np.float32)
    c, a = oracle.ternarize_weights(w)
    flat, cf = w.reshape(32, -1).astype(np.float64), c.reshape(32, -1)
    delta = 0.7 * np.abs(flat).mean(1)
    assert np.all(np.abs(flat[cf == 0]) <= np.repeat(delta, (cf == 0).sum(1)))     # Eq. 4 zero band
    assert np.all(np.sign(flat[cf != 0]) == cf[cf != 0])
    assert np.all(a >= 0) and np.all((a == 0) == (np.abs(cf).sum(1) == 0))
    # alpha minimises ||W - alpha W~||^2 over alpha for the chosen codes (Li et al.'s closed form)
    for f in range(4):
        m = cf[f] != 0
        best = np.abs(flat[f][m]).mean()
        assert abs(best - a[f]) < 1e-6
    # fixed sparsity: exactly ceil(s n) zeros per filter
    c5, _ = oracle.ternarize_weights(w, 0.5)
    assert np.all((c5.reshape(32, -1) == 0).sum(1) == int(np.ceil(0.5 * 432)))


def _tern(v):
    return 1 if v > Fraction(1, 2) else (0 if v >= Fraction(-1, 2) else -1)


def test_oracle_fold_table_is_eq6_exactly_for_dyadic_parameters():
    """Parameters whose float64 evaluation is exact (dyadic a, b; var + eps = 1): the
    oracle's table equals Eq. 6 of the affine map in exact rational arithmetic."""
    g = synth.rng(42)
    A = 27 * 16
    k = 24
    alpha = (g.integers(1, 64, k) / 64.0).astype(np.float32)
    gamma = (g.integers(-64, 64, k) / 16.0).astype(np.float32)
    beta = (g.integers(-64, 64, k) / 32.0).astype(np.float32)
    mean = (g.integers(-64, 64, k) / 8.0).astype(np.float32)
    var = np.zeros(k, np.float32)
    tab = oracle.fold_table(alpha, gamma, beta, mean, var, 1.0, A)
    for c in range(k):
        a = Fraction(float(gamma[c])) * Fraction(float(alpha[c]))
        b = Fraction(float(beta[c])) - Fraction(float(gamma[c])) * Fraction(float(mean[c]))
        ref = [_tern(a * acc + b) for acc in range(-A, A + 1)]
        assert list(tab[c]) == ref


@pytest.mark.parametrize("var_eps", [(0.0625, 0.1875), (3.75, 0.25), (15.75, 0.25), (48.0, 16.0)],
                         ids=["1/4", "4", "16", "64"])
def test_oracle_fold_table_bn_denominator_sqrt_var_plus_eps(var_eps):
    """The batch-norm denominator of the fold (the conv output alpha*acc is
    batch normalised, then Eq. 6): y = gamma*(alpha*acc - mean)/sqrt(var + eps) + beta.
    var + eps is a dyadic perfect square other than 1 (1/4, 4, 16, 64), so sqrt(var + eps) and
    every float64 step of the oracle are exact; the table must equal Eq. 6 of y in exact
    rational arithmetic.  The same parameters are checked to separate the plausible mistakes
    (no sqrt; sqrt(var) + eps; sqrt(var) without eps): each gives a different table, so a
    dropped or misplaced sqrt in the oracle fails this pin."""
    var_v, eps = var_eps
    g = synth.rng(45)
    A = 27 * 16
    k = 24
    alpha = (g.integers(1, 64, k) / 64.0).astype(np.float32)
    gamma = (g.integers(-64, 64, k) / 16.0).astype(np.float32)
    gamma[gamma == 0] = 1.0
    beta = (g.integers(-64, 64, k) / 32.0).astype(np.float32)
    mean = (g.integers(-64, 64, k) / 8.0).astype(np.float32)
    var = np.full(k, var_v, np.float32)
    s = Fraction(float(np.float32(var_v))) + Fraction(float(np.float32(eps)))
    sd = Fraction(int(round(float(s) ** 0.5 * 4)), 4)
    assert sd * sd == s and s != 1                 # an exact dyadic square root
    tab = oracle.fold_table(alpha, gamma, beta, mean, var, eps, A)
    accs = range(-A, A + 1)

    def table(den):
        out = []
        for c in range(k):
            a = Fraction(float(gamma[c])) * Fraction(float(alpha[c])) / den
            b = Fraction(float(beta[c])) - Fraction(float(gamma[c])) * Fraction(float(mean[c])) / den
            out.append([_tern(a * acc + b) for acc in accs])
        return out

    ref = table(sd)
    for c in range(k):
        assert list(tab[c]) == ref[c], f"channel {c}"
    # the pin separates the plausible mistakes
    wrong = {"no sqrt": s, "sqrt(var) + eps": Fraction(float(np.float32(var_v)) ** 0.5) + Fraction(float(eps)),
             "sqrt(var)": Fraction(float(np.float32(var_v)) ** 0.5)}
    for name, den in wrong.items():
        assert table(den) != ref, name


def test_library_ternarize_matches_oracle(tn):
    for sp, w, codes, alpha in _examples():
        c, a = tn.tn_ternarize_weights(w[None], -1.0 if sp is None else sp)
        np.testing.assert_array_equal(c[0], codes)
        assert abs(float(a[0]) - alpha) < 1e-6
    g = synth.rng(43)
    for shape in [(16, 1, 3, 3, 3), (64, 64, 3, 3, 3), (5, 33, 3, 3, 3)]:
        w = (g.normal(0, 1, shape) * g.uniform(0.01, 3)).astype(np.float32)
        for sp in (None, 0.5, 0.25, 0.0):
            oc, oa = oracle.ternarize_weights(w, sp)
            lc, la = tn.tn_ternarize_weights(w, -1.0 if sp is None else sp)
            np.testing.assert_array_equal(lc, oc)
            np.testing.assert_allclose(la, oa, rtol=1e-6)
    bad = np.ones((2, 27), np.float32)
    bad[1, 5] = np.nan
    with pytest.raises(tn.TNError) as e:
        tn.tn_ternarize_weights(bad)
    assert e.value.status == tn.TN_EDOMAIN
    with pytest.raises(tn.TNError):
        tn.tn_ternarize_weights(np.ones((2, 27), np.float32), 1.0)


def _apply(acc, lo, hi):
    return np.where(acc >= hi, 1, np.where(acc <= lo, -1, 0))


def test_library_fold_reproduces_eq6_at_every_accumulator(tn):
    """For every channel and every acc in [-27C, 27C], the integer rule on the (possibly
    negated) accumulator equals the oracle's Eq. 6 table; negative BN scales, zero alpha
    (constant channels) and boundaries landing exactly on +-0.5 included."""
    g = synth.rng(44)
    for C in (1, 16, 64):
        A = 27 * C
        k = 64
        alpha = g.uniform(0.05, 2.0, k).astype(np.float32)
        alpha[:3] = 0.0                                   # constant channels
        gamma = g.normal(0, 1, k).astype(np.float32)      # both signs
        beta = g.normal(0, 1, k).astype(np.float32)
        beta[:3] = [0.9, -0.9, 0.1]
        mean = g.normal(0, 3 * np.sqrt(C), k).astype(np.float32)
        var = g.uniform(0.1, 4 * C, k).astype(np.float32)
        # exact ties: a = 1/2^j, b chosen so that y = +-0.5 at an integer acc
        alpha[3], gamma[3], var[3], mean[3], beta[3] = 0.25, 1.0, 0.0, 0.0, -2.0   # y = acc/4 - 2: 0.5 at acc=10
        eps = 1e-5 if C > 1 else 0.0
        if eps == 0.0:
            var[:] = np.maximum(var, 1e-3)
            var[3] = 1.0
        tab = oracle.fold_table(alpha, gamma, beta, mean, var, eps, A)
        lo, hi, neg = tn.tn_fold_thresholds(alpha, gamma, beta, mean, var, eps, A)
        acc = np.arange(-A, A + 1, dtype=np.int64)
        for c in range(k):
            a_eff = -acc if neg[c] else acc
            np.testing.assert_array_equal(_apply(a_eff, lo[c], hi[c]), tab[c], err_msg=f"C={C} channel {c}")
        assert neg[(gamma < 0) & (alpha > 0)].all() and not neg[(gamma > 0) & (alpha > 0)].any()
