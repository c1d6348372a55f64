// prep.cu -- model preparation, host only, not on the hot path:
// Eq. 4 ternary weights (after Li et al.) and the fold of alpha,
// batch norm and Eq. 6's +-0.5 band into the
// per-channel integer thresholds (lo, hi) the conv epilogues apply (readings
// R5 / R6 in DESIGN.md).  Double precision; see include/tn.h for the contract.
#include "tn_internal.cuh"

#include <algorithm>
#include <climits>
#include <cmath>
#include <numeric>
#include <vector>

using namespace tn;

namespace {

// y(acc) = a * acc + b, evaluated as two separate double operations (no FMA)
inline double affine(double a, double b, int64_t acc) {
    volatile double p = a * static_cast<double>(acc);
    return p + b;
}

}  // namespace

extern "C" {

tn_status tn_ternarize_weights(const float* w, int32_t k, int32_t n, float sparsity, int8_t* codes, float* alpha,
                               int64_t* bad_index) {
    if (bad_index) *bad_index = -1;
    if (w == nullptr || codes == nullptr || alpha == nullptr) { set_error("w/codes/alpha is NULL"); return TN_EINVAL; }
    if (k < 1 || n < 1) { set_error("need k >= 1 and n >= 1 (got %d, %d)", k, n); return TN_EINVAL; }
    if (!(sparsity < 1.0f)) { set_error("sparsity must be < 1 (got %g)", sparsity); return TN_EDOMAIN; }
    for (int64_t i = 0; i < static_cast<int64_t>(k) * n; ++i)
        if (!std::isfinite(w[i])) {
            if (bad_index) *bad_index = i;
            set_error("non-finite weight at flat index %lld", static_cast<long long>(i));
            return TN_EDOMAIN;
        }
    std::vector<int> order(n);
    for (int f = 0; f < k; ++f) {
        const float* wf = w + static_cast<int64_t>(f) * n;
        int8_t* cf = codes + static_cast<int64_t>(f) * n;
        if (sparsity < 0.0f) {
            // Eq. 4: Delta = 0.7/n * sum |W_i|; +1 if W_i > Delta, 0 if |W_i| <= Delta, -1 else
            double s = 0.0;
            for (int i = 0; i < n; ++i) s += std::fabs(static_cast<double>(wf[i]));
            const double delta = 0.7 / n * s;
            for (int i = 0; i < n; ++i) {
                const double v = wf[i];
                cf[i] = static_cast<int8_t>(v > delta ? 1 : (std::fabs(v) <= delta ? 0 : -1));
            }
        } else {
            // fixed sparsity: exactly ceil(s*n) zeros at the smallest |W_i|,
            // ties broken by index; the rest are sign(W_i)
            const int nz = static_cast<int>(std::ceil(static_cast<double>(sparsity) * n));
            std::iota(order.begin(), order.end(), 0);
            std::stable_sort(order.begin(), order.end(), [wf](int a, int b) {
                return std::fabs(static_cast<double>(wf[a])) < std::fabs(static_cast<double>(wf[b]));
            });
            for (int i = 0; i < n; ++i) cf[i] = static_cast<int8_t>(wf[i] > 0.0f ? 1 : -1);
            for (int i = 0; i < nz; ++i) cf[order[i]] = 0;
        }
        // alpha = (1/n_Delta) sum_i |W~_i| |W_i|, 0 when every code is 0
        double num = 0.0;
        int64_t cnt = 0;
        for (int i = 0; i < n; ++i)
            if (cf[i] != 0) { num += std::fabs(static_cast<double>(wf[i])); ++cnt; }
        alpha[f] = cnt ? static_cast<float>(num / cnt) : 0.0f;
    }
    return TN_OK;
}

tn_status tn_fold_thresholds(const float* alpha, const float* gamma, const float* beta, const float* mean,
                             const float* var, float eps, int32_t k, int32_t max_abs_acc, int32_t* lo, int32_t* hi,
                             int8_t* negate) {
    if (!alpha || !gamma || !beta || !mean || !var || !lo || !hi || !negate) {
        set_error("a parameter pointer is NULL");
        return TN_EINVAL;
    }
    if (k < 1 || max_abs_acc < 0) { set_error("need k >= 1 and max_abs_acc >= 0"); return TN_EINVAL; }
    const int64_t A = max_abs_acc;
    for (int c = 0; c < k; ++c) {
        const double vs = static_cast<double>(var[c]) + static_cast<double>(eps);
        if (!(vs > 0.0) || !std::isfinite(vs) || !std::isfinite(alpha[c]) || !std::isfinite(gamma[c]) ||
            !std::isfinite(beta[c]) || !std::isfinite(mean[c])) {
            set_error("channel %d: non-finite parameters or var + eps <= 0", c);
            return TN_EDOMAIN;
        }
        const double sd = std::sqrt(vs);
        // y = gamma * (alpha * acc - mean) / sd + beta = a * acc + b  (reading R6)
        double a = static_cast<double>(gamma[c]) * static_cast<double>(alpha[c]) / sd;
        const double b = static_cast<double>(beta[c]) - static_cast<double>(gamma[c]) * static_cast<double>(mean[c]) / sd;
        negate[c] = a < 0.0 ? 1 : 0;   // negated filter: acc' = -acc, a' = -a > 0
        if (a < 0.0) a = -a;
        if (a == 0.0) {   // constant output tern(b): sentinels
            if (b > 0.5) { lo[c] = INT32_MIN; hi[c] = INT32_MIN; }
            else if (b < -0.5) { lo[c] = INT32_MAX; hi[c] = INT32_MAX; }
            else { lo[c] = INT32_MIN; hi[c] = INT32_MAX; }
            continue;
        }
        // hi = smallest acc in [-A, A] with y > 0.5 (else never: INT32_MAX); closed form, then
        // corrected against the predicate itself at the boundary integers
        int64_t h = static_cast<int64_t>(std::floor((0.5 - b) / a)) + 1;
        h = std::max<int64_t>(std::min<int64_t>(h, A + 1), -A);
        while (h > -A && affine(a, b, h - 1) > 0.5) --h;
        while (h <= A && !(affine(a, b, h) > 0.5)) ++h;
        hi[c] = h > A ? INT32_MAX : (h <= -A && affine(a, b, -A) > 0.5 ? INT32_MIN : static_cast<int32_t>(h));
        // lo = largest acc with y < -0.5 (else never: INT32_MIN)
        int64_t l = static_cast<int64_t>(std::ceil((-0.5 - b) / a)) - 1;
        l = std::max<int64_t>(std::min<int64_t>(l, A), -A - 1);
        while (l < A && affine(a, b, l + 1) < -0.5) ++l;
        while (l >= -A && !(affine(a, b, l) < -0.5)) --l;
        lo[c] = l < -A ? INT32_MIN : (l >= A && affine(a, b, A) < -0.5 ? INT32_MAX : static_cast<int32_t>(l));
    }
    return TN_OK;
}

}  // extern "C"
