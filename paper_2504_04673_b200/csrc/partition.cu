// partition.cu -- native host partitioners: the reference's
// greedy_tv_partition (partition.py:257-289, with _bfs_order 292-310 and
// _refine_edgecut 313-339) and volume_balanced_refine (partition.py:342-428),
// restated in C++ with the same visiting orders, tie-breaks and float64
// comparisons, so the assignments are identical to the reference's (pinned
// by tests/golden/partition_golden.npz).  Host preprocessing, not the hot
// path: it makes the "graph-partitioned" / "volume-balanced" benchmark
// configurations feasible at products scale (the Python loops take hours).
//
// Inputs are CSR patterns (int64 row_ptr / col).  `pat` is the symmetric
// pattern without diagonal (partition._sym_pattern); `a` / `at` are the
// matrix and its transpose (for out- / in-neighbours).

#include <deque>

#include "common.cuh"

extern "C" {

// greedy_tv_partition: BFS-grown parts (cap (1+eps) * sum(w) / k, relaxed
// to max(w) when a single vertex exceeds it), then edgecut-reducing moves.
// Returns 1 in *relaxed when the cap was relaxed (the reference logs a
// warning).
int dg_host_greedy_tv(int64_t n, const int64_t* prp, const int64_t* pci, int32_t k,
                      double epsilon, int32_t max_passes, int64_t* assignment, int32_t* relaxed) {
  if (n < 0 || k < 1 || k > n) return set_err(DG_ERR_ARG, "greedy_tv: bad n / k");
  std::vector<int64_t> weight(n);
  double wsum = 0.0;
  int64_t wmax = 0;
  for (int64_t v = 0; v < n; ++v) {
    weight[v] = std::max<int64_t>(prp[v + 1] - prp[v], 1);
    wsum += (double)weight[v];
    wmax = std::max(wmax, weight[v]);
  }
  double cap = (1.0 + epsilon) * wsum / (double)k;
  *relaxed = 0;
  if ((double)wmax > cap) {
    cap = (double)wmax;
    *relaxed = 1;
  }
  // _bfs_order: BFS from every unseen vertex in ascending id, neighbours in
  // row order
  std::vector<int64_t> order;
  order.reserve(n);
  std::vector<char> seen(n, 0);
  std::deque<int64_t> q;
  for (int64_t s = 0; s < n; ++s) {
    if (seen[s]) continue;
    seen[s] = 1;
    q.push_back(s);
    while (!q.empty()) {
      const int64_t v = q.front();
      q.pop_front();
      order.push_back(v);
      for (int64_t e = prp[v]; e < prp[v + 1]; ++e) {
        const int64_t u = pci[e];
        if (!seen[u]) {
          seen[u] = 1;
          q.push_back(u);
        }
      }
    }
  }
  int64_t cur = 0, cur_w = 0;
  for (int64_t idx = 0; idx < n; ++idx) {
    const int64_t v = order[idx];
    const bool must_leave = (n - idx) == (k - cur - 1);
    if (cur < k - 1 && cur_w > 0 && ((double)(cur_w + weight[v]) > cap || must_leave)) {
      ++cur;
      cur_w = 0;
    }
    assignment[v] = cur;
    cur_w += weight[v];
  }
  // _refine_edgecut
  std::vector<int64_t> nbr((size_t)n * k, 0);
  for (int64_t v = 0; v < n; ++v)
    for (int64_t e = prp[v]; e < prp[v + 1]; ++e) ++nbr[(size_t)v * k + assignment[pci[e]]];
  std::vector<double> part_w(k, 0.0);
  for (int64_t v = 0; v < n; ++v) part_w[assignment[v]] += (double)weight[v];
  for (int32_t pass = 0; pass < max_passes; ++pass) {
    int64_t moved = 0;
    for (int64_t v = 0; v < n; ++v) {
      const int64_t s = assignment[v];
      int64_t best_t = -1, best_delta = 0;
      for (int64_t t = 0; t < k; ++t) {
        if (t == s || part_w[t] + (double)weight[v] > cap) continue;
        const int64_t delta = nbr[(size_t)v * k + s] - nbr[(size_t)v * k + t];
        if (delta < best_delta) {
          best_t = t;
          best_delta = delta;
        }
      }
      if (best_t >= 0) {
        assignment[v] = best_t;
        part_w[s] -= (double)weight[v];
        part_w[best_t] += (double)weight[v];
        for (int64_t e = prp[v]; e < prp[v + 1]; ++e) {
          const int64_t u = pci[e];
          --nbr[(size_t)u * k + s];
          ++nbr[(size_t)u * k + best_t];
        }
        ++moved;
      }
    }
    if (moved == 0) break;
  }
  return DG_OK;
}

// volume_balanced_refine: boundary-vertex moves scored by total send rows
// + lambda * change of the bottleneck part's send rows; strictly improving,
// balance-respecting, ascending vertex ids, ties to the lowest target part.
int dg_host_gvb(int64_t n, const int64_t* arp, const int64_t* aci, const int64_t* atrp,
                const int64_t* atci, const int64_t* prp, int32_t k, double lambda_max,
                double epsilon, int32_t max_passes, int64_t* assignment) {
  if (n < 0 || k < 1) return set_err(DG_ERR_ARG, "gvb: bad n / k");
  std::vector<int64_t> weight(n);
  double wsum = 0.0;
  int64_t wmax = 0;
  for (int64_t v = 0; v < n; ++v) {
    weight[v] = std::max<int64_t>(prp[v + 1] - prp[v], 1);
    wsum += (double)weight[v];
    wmax = std::max(wmax, weight[v]);
  }
  const double cap = std::max((1.0 + epsilon) * wsum / (double)k, (double)wmax);
  std::vector<double> part_w(k, 0.0);
  for (int64_t v = 0; v < n; ++v) part_w[assignment[v]] += (double)weight[v];
  // out_cnt[v, t]: out-neighbours of v (self-loops ignored) in part t
  std::vector<int64_t> out((size_t)n * k, 0);
  for (int64_t v = 0; v < n; ++v)
    for (int64_t e = arp[v]; e < arp[v + 1]; ++e)
      if (aci[e] != v) ++out[(size_t)v * k + assignment[aci[e]]];
  auto contribution = [&](int64_t v, int64_t own) -> int64_t {
    int64_t c = 0;
    for (int64_t t = 0; t < k; ++t) c += out[(size_t)v * k + t] != 0;
    return out[(size_t)v * k + own] > 0 ? c - 1 : c;
  };
  std::vector<int64_t> contrib(n);
  std::vector<int64_t> part_send(k, 0);
  for (int64_t v = 0; v < n; ++v) {
    contrib[v] = contribution(v, assignment[v]);
    part_send[assignment[v]] += contrib[v];
  }
  std::vector<int64_t> in_nbrs;
  std::vector<char> is_target(k);
  std::vector<int64_t> delta(k), best_delta(k), new_send(k);
  std::vector<std::pair<int64_t, int64_t>> nc, best_nc;   // (vertex, new contribution)
  for (int32_t pass = 0; pass < max_passes; ++pass) {
    int64_t moved = 0;
    for (int64_t v = 0; v < n; ++v) {
      const int64_t s = assignment[v];
      in_nbrs.clear();
      for (int64_t e = atrp[v]; e < atrp[v + 1]; ++e)
        if (atci[e] != v) in_nbrs.push_back(atci[e]);
      std::fill(is_target.begin(), is_target.end(), 0);
      for (int64_t t = 0; t < k; ++t)
        if (out[(size_t)v * k + t]) is_target[t] = 1;
      for (int64_t u : in_nbrs) is_target[assignment[u]] = 1;
      is_target[s] = 0;
      bool have_best = false;
      double best_cost = 0.0;
      int64_t best_t = -1;
      int64_t cur_max = 0;
      for (int64_t t = 0; t < k; ++t) cur_max = std::max(cur_max, part_send[t]);
      for (int64_t t = 0; t < k; ++t) {
        if (!is_target[t]) continue;
        if (part_w[t] + (double)weight[v] > cap) continue;
        std::fill(delta.begin(), delta.end(), 0);
        nc.clear();
        const int64_t cv = contribution(v, t);
        nc.emplace_back(v, cv);
        delta[s] -= contrib[v];
        delta[t] += cv;
        for (int64_t u : in_nbrs) {
          int64_t du = 0;
          const int64_t own_u = assignment[u];
          if (s != own_u && out[(size_t)u * k + s] == 1) du -= 1;
          if (t != own_u && out[(size_t)u * k + t] == 0) du += 1;
          if (du) {
            nc.emplace_back(u, contrib[u] + du);
            delta[own_u] += du;
          }
        }
        int64_t d_total = 0;
        int64_t new_max = 0;
        for (int64_t p = 0; p < k; ++p) {
          d_total += delta[p];
          new_max = std::max(new_max, part_send[p] + delta[p]);
        }
        const double d_cost = (double)d_total + lambda_max * (double)(new_max - cur_max);
        if (d_cost < 0.0 && (!have_best || d_cost < best_cost)) {
          have_best = true;
          best_cost = d_cost;
          best_t = t;
          best_delta = delta;
          best_nc = nc;
        }
      }
      if (!have_best) continue;
      for (int64_t u : in_nbrs) {
        --out[(size_t)u * k + s];
        ++out[(size_t)u * k + best_t];
      }
      for (auto& pr : best_nc) contrib[pr.first] = pr.second;
      for (int64_t p = 0; p < k; ++p) part_send[p] += best_delta[p];
      part_w[s] -= (double)weight[v];
      part_w[best_t] += (double)weight[v];
      assignment[v] = best_t;
      ++moved;
    }
    if (moved == 0) break;
  }
  return DG_OK;
}

}  // extern "C"
