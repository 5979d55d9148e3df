// Proportional subtree-to-GPU mapping of the merged supernodal elimination tree (SURVEY §8(e),
// north_star "partitioned across the 8xB200 box by subtree-to-GPU mapping of the etree").
//
// Walk from the root(s) with all P ranks.  A node that receives a group of more than one rank is a
// "top" supernode (owner -1): its children are split among the group in proportion to their
// subtree work (largest remainder; if there are more children than ranks, children are packed
// onto single ranks longest-processing-time first).  A child that receives a single rank makes its
// whole subtree local to that rank.  Deterministic: every rank computes the same map.
#include <algorithm>
#include <numeric>
#include <vector>

#include "symbolic.h"

namespace spchol {

void proportional_map(const Symbolic& S, const std::vector<double>& work, int world, std::vector<int>& owner,
                      std::vector<int>* top_lo, std::vector<int>* top_hi) {
  const int ns = S.nsuper;
  owner.assign(ns, 0);
  if (top_lo) top_lo->assign(ns, 0);
  if (top_hi) top_hi->assign(ns, 0);
  if (world <= 1 || ns == 0) return;
  std::vector<double> sub(work);
  for (int J = 0; J < ns; ++J)
    if (S.sparent[J] >= 0) sub[S.sparent[J]] += sub[J];   // children precede parents (postorder)
  std::vector<std::vector<int>> kids(ns + 1);                 // index ns = virtual root of the forest
  for (int J = 0; J < ns; ++J) kids[S.sparent[J] >= 0 ? S.sparent[J] : ns].push_back(J);
  auto subtree_to = [&](int J, int rank) {                    // J's subtree = [J - size + 1, J] in postorder
    std::vector<int> stack{J};
    while (!stack.empty()) {
      int v = stack.back();
      stack.pop_back();
      owner[v] = rank;
      for (int c : kids[v]) stack.push_back(c);
    }
  };
  struct Item { int node, lo, hi; };
  std::vector<Item> work_list{{ns, 0, world}};
  while (!work_list.empty()) {
    Item it = work_list.back();
    work_list.pop_back();
    const int P = it.hi - it.lo;
    if (it.node < ns) {
      if (P == 1) { subtree_to(it.node, it.lo); continue; }
      owner[it.node] = -1;
      if (top_lo) (*top_lo)[it.node] = it.lo;
      if (top_hi) (*top_hi)[it.node] = it.hi;
    }
    std::vector<int> ch = kids[it.node];
    if (ch.empty()) continue;
    std::stable_sort(ch.begin(), ch.end(), [&](int a, int b) { return sub[a] > sub[b]; });
    if ((int)ch.size() >= P) {
      // more children than ranks: LPT packing, each child's subtree local to one rank
      std::vector<double> load(P, 0.0);
      for (int c : ch) {
        int r = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        load[r] += sub[c];
        work_list.push_back({c, it.lo + r, it.lo + r + 1});
      }
      continue;
    }
    // fewer children than ranks: contiguous rank ranges proportional to subtree work (>= 1 each)
    double W = 0.0;
    for (int c : ch) W += sub[c];
    const int nc = (int)ch.size();
    std::vector<int> cnt(nc, 1);
    int left = P - nc;
    std::vector<double> want(nc);
    for (int i = 0; i < nc; ++i) want[i] = W > 0 ? P * sub[ch[i]] / W : (double)P / nc;
    while (left > 0) {   // give the next rank to the child with the largest unmet share
      int best = 0;
      double bv = -1e300;
      for (int i = 0; i < nc; ++i) {
        double v = want[i] - cnt[i];
        if (v > bv) { bv = v; best = i; }
      }
      cnt[best]++;
      --left;
    }
    int lo = it.lo;
    for (int i = 0; i < nc; ++i) {
      work_list.push_back({ch[i], lo, lo + cnt[i]});
      lo += cnt[i];
    }
  }
}

// Owner rank of every top supernode (fan-in factorization of the top).  The top levels run one
// after the other (each starts with the reduction of its panels), so the balance that matters is
// per level: within a level, heaviest first, each top supernode goes to the member of its rank
// group with the least work in that level.
void assign_top_owners(const std::vector<double>& work, const std::vector<int>& owner, const std::vector<int>& lo,
                       const std::vector<int>& hi, const std::vector<int>& level, int world,
                       std::vector<int>& top_owner) {
  const int ns = (int)owner.size();
  top_owner.assign(ns, -1);
  int nl = 0;
  for (int J = 0; J < ns; ++J) nl = std::max(nl, level[J] + 1);
  std::vector<std::vector<int>> by_level(nl);
  for (int J = 0; J < ns; ++J) if (owner[J] < 0) by_level[level[J]].push_back(J);
  for (auto& tops : by_level) {
    std::stable_sort(tops.begin(), tops.end(), [&](int a, int b) { return work[a] > work[b]; });
    std::vector<double> load(world, 0.0);
    for (int J : tops) {
      int best = lo[J];
      for (int r = lo[J]; r < hi[J]; ++r) if (load[r] < load[best]) best = r;
      top_owner[J] = best;
      load[best] += work[J];
    }
  }
}

}  // namespace spchol
