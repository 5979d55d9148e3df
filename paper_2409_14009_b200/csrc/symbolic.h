// Host-side symbolic analysis result (spchol_analyze).  Integer only.
// P:n = PAPER.md line n (arXiv 2409.14009); R# = DESIGN.md reading.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace spchol {

struct Symbolic {
  int64_t n = 0, nnzA = 0;
  // O3 postorder of the etree of P A P^T: post[k] = user-permuted index numbered k
  std::vector<int32_t> post, parent3, cc3;
  int64_t nnzL = 0;
  double flops_exact = 0.0;     // sum cc^2
  // fundamental partition (postorder numbering) and the merge result
  std::vector<int32_t> ffirst, fparent, fgroup;
  int64_t added = 0;
  int32_t nmerges = 0;
  // final numbering (R6): perm_final[orig] = final
  std::vector<int32_t> perm_final, iperm_final;
  int32_t nsuper = 0;
  std::vector<int32_t> sfirst, sparent, snode;  // snode[final col] = supernode
  std::vector<int64_t> rows_ptr;
  std::vector<int32_t> rows;
  // relind: per (J, ancestor P) pair
  std::vector<int64_t> rel_ptr, rel_off;
  std::vector<int32_t> rel_anc, rel_q0, relind;
  std::vector<int32_t> parent_final, cc_final;
  // RLB blocks: per J, maximal runs of consecutive global rows of R_J inside one
  // ancestor's column range; q = first row position in rows(J), relindB of the first row
  std::vector<int64_t> blk_ptr;
  std::vector<int32_t> blk_q, blk_len, blk_anc, blk_relind;
  std::vector<int32_t> level;  // height of each supernode in the merged tree (leaves = 0)
  int32_t nlevels = 0;
  // A -> final lower position: for every stored entry e of A, (final col, position in rows(J))
  std::vector<int32_t> a_col;  // final column of entry e
  std::vector<int32_t> a_pos;  // row position q in rows(snode(col))
};

// Returns 0 or an SPCHOL_ERR_* code; err receives a message.
// pr = 1: partition refinement of the columns inside the supernodes (reading R14)
int analyze_symbolic(int64_t n, const int64_t* colptr, const int32_t* rowidx, const int32_t* perm,
                     double cap, int pr, Symbolic& S, std::string& err);

}  // namespace spchol
