// stats.cpp — the two-sided exact Wilcoxon rank-sum test on midranks (P:410,
// P:615; reading R-W1): W = sum of the doubled midranks of sample a; the null
// distribution of W over all C(n, n1) placements is counted with a subset-sum
// DP; p = min(1, 2 * min(P(W' <= W), P(W' >= W))).  n <= 32 (<= 16 repeats per
// candidate), so the counts fit in 64 bits and the test is always exact.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "internal.hpp"

namespace db200 {

double wilcoxon_p(const float* a, int n1, const float* b, int n2) {
    if (n1 <= 0 || n2 <= 0) return 1.0;
    const int n = n1 + n2;
    std::vector<float> v(n);
    for (int i = 0; i < n1; ++i) v[i] = a[i];
    for (int i = 0; i < n2; ++i) v[n1 + i] = b[i];
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return v[x] < v[y]; });
    std::vector<int> r2(n);  // twice the midrank
    for (int i = 0; i < n;) {
        int j = i;
        while (j + 1 < n && v[order[j + 1]] == v[order[i]]) ++j;
        for (int k = i; k <= j; ++k) r2[order[k]] = (i + 1) + (j + 1);
        i = j + 1;
    }
    int w = 0, maxs = 0;
    for (int i = 0; i < n1; ++i) w += r2[i];
    for (int i = 0; i < n; ++i) maxs += r2[i];
    // dp[k][s] = number of k-subsets of the first items with doubled-rank sum s
    std::vector<std::vector<uint64_t>> dp(n1 + 1, std::vector<uint64_t>(maxs + 1, 0));
    dp[0][0] = 1;
    for (int i = 0; i < n; ++i)
        for (int k = std::min(i + 1, n1); k >= 1; --k)
            for (int s = maxs; s >= r2[i]; --s) dp[k][s] += dp[k - 1][s - r2[i]];
    uint64_t le = 0, ge = 0, total = 0;
    for (int s = 0; s <= maxs; ++s) {
        total += dp[n1][s];
        if (s <= w) le += dp[n1][s];
        if (s >= w) ge += dp[n1][s];
    }
    const double p = 2.0 * (double)std::min(le, ge) / (double)total;
    return p < 1.0 ? p : 1.0;
}

}  // namespace db200

extern "C" tuner_status tuner_rank_sum_p(const float* a, int32_t n1, const float* b, int32_t n2, double* p) {
    if (!p || n1 < 0 || n2 < 0 || (n1 > 0 && !a) || (n2 > 0 && !b)) return db200::fail(TUNER_EINVAL, "bad arguments");
    if (n1 > 16 || n2 > 16) return db200::fail(TUNER_EINVAL, "at most 16 samples per side (exact test)");
    *p = db200::wilcoxon_p(a, n1, b, n2);
    return TUNER_OK;
}
