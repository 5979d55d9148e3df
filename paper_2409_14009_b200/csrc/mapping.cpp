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

void proportional_map(const Symbolic& S, const std::vector<double>& work, int world, std::vector<int>& owner) {
  const int ns = S.nsuper;
  owner.assign(ns, 0);
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

}  // namespace spchol
