// Host-side planning helper of grid mode: which CTA owns which tile.
//
// k_grid reads its tile table by position: position p is slot p / G of CTA
// p % G, so CTA k has (T - 1 - k) / G + 1 tiles -- `per` = ceil(T / G) for the
// first T % G CTAs, per - 1 for the rest.  The order of the table is therefore
// the assignment.  In frame order (round-robin) a CTA's load is whatever sizes
// its positions happen to hold (edge tiles are smaller) plus a whole tile more
// on the CTAs with the extra slot.  tile_balance() returns an order in which
// every CTA's summed cost is close to the mean: the CTAs with a slot fewer take
// the x largest and the n - x smallest tiles, x chosen so that their share of
// the total cost equals their share of the CTAs, the others take the middle;
// inside each group tiles go largest-first to the least loaded CTA with a free
// slot.  The assignment changes no result (units of one colour class are
// independent and integer delta sums commute).
//
// cost[i] is the cost of tile i of one frame; tile t of the batch (t in [0, T),
// T a multiple of cost.size()) is tile t % cost.size() of frame t / cost.size().
// Returns order[p] = t; the identity when balancing does not lower the busiest
// CTA's cost.  busiest[0] / busiest[1]: that cost in frame order / as returned.
#pragma once
#include <algorithm>
#include <cmath>
#include <functional>
#include <queue>
#include <utility>
#include <vector>

static inline std::vector<long long> tile_balance(const std::vector<double> &cost, long long T, int G,
                                                  double busiest[2])
{
    std::vector<long long> order((size_t)T);
    for (long long t = 0; t < T; t++) order[(size_t)t] = t;
    auto tcost = [&](long long t) { return cost[(size_t)(t % (long long)cost.size())]; };
    std::vector<double> rr(G, 0.0);
    for (long long t = 0; t < T; t++) rr[(size_t)(t % G)] += tcost(t);
    const double rr_max = G > 0 && T > 0 ? *std::max_element(rr.begin(), rr.end()) : 0.0;
    busiest[0] = busiest[1] = rr_max;
    if (T <= G || G <= 0 || cost.empty()) return order;
    std::vector<long long> by_cost(order);
    std::stable_sort(by_cost.begin(), by_cost.end(), [&](long long a, long long b) { return tcost(a) > tcost(b); });
    const int nbig = (int)(T % G);
    const long long per = (T + G - 1) / G;
    std::vector<double> load(G, 0.0);
    std::vector<std::vector<long long>> mine((size_t)G);
    using Ent = std::pair<double, int>;  // (load, CTA): least loaded first, then lowest index
    auto fill = [&](const std::vector<long long> &ts, int c0, int c1, long long slots) {
        std::priority_queue<Ent, std::vector<Ent>, std::greater<Ent>> pq;
        for (int k = c0; k < c1; k++) pq.push(Ent(load[k], k));
        for (long long t : ts) {
            if (pq.empty()) return false;
            const int k = pq.top().second;
            pq.pop();
            mine[(size_t)k].push_back(t);
            load[k] += tcost(t);
            if ((long long)mine[(size_t)k].size() < slots) pq.push(Ent(load[k], k));
        }
        return true;
    };
    bool ok;
    if (nbig) {
        const size_t n_small = (size_t)(G - nbig) * (size_t)(per - 1), n = (size_t)T;
        std::vector<double> pre(n + 1, 0.0);
        for (size_t i = 0; i < n; i++) pre[i + 1] = pre[i] + tcost(by_cost[i]);
        const double target = pre[n] * (double)(G - nbig) / (double)G;
        size_t bx = 0;
        double bd = 1e300;
        for (size_t x = 0; x <= n_small; x++) {
            const double d = std::fabs(pre[x] + (pre[n] - pre[n - (n_small - x)]) - target);
            if (d < bd) {
                bd = d;
                bx = x;
            }
        }
        const size_t lo = n - (n_small - bx);
        std::vector<long long> small_ts(by_cost.begin(), by_cost.begin() + (long)bx);
        small_ts.insert(small_ts.end(), by_cost.begin() + (long)lo, by_cost.end());
        const std::vector<long long> big_ts(by_cost.begin() + (long)bx, by_cost.begin() + (long)lo);
        ok = fill(small_ts, nbig, G, per - 1) && fill(big_ts, 0, nbig, per);
    } else {
        ok = fill(by_cost, 0, G, per);
    }
    const double bal_max = *std::max_element(load.begin(), load.end());
    if (!ok || !(bal_max < rr_max)) return order;
    for (int k = 0; k < G; k++) {
        if ((long long)mine[(size_t)k].size() != (T - 1 - k) / G + 1) return order;  // (cannot happen)
        std::sort(mine[(size_t)k].begin(), mine[(size_t)k].end());  // frame order inside a CTA
    }
    for (int k = 0; k < G; k++)
        for (size_t j = 0; j < mine[(size_t)k].size(); j++) order[(size_t)k + j * (size_t)G] = mine[(size_t)k][j];
    busiest[1] = bal_max;
    return order;
}
