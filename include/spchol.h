/*
 * spchol.h — C ABI of the B200-native right-looking supernodal sparse Cholesky (RL) library.
 *
 * Method: Karsavuran, Ng, Peyton, "GPU Accelerated Sparse Cholesky Factorization"
 * (arXiv 2409.14009).  Citations "P:n" are lines of that paper's PAPER.md, "S:n" lines of
 * SPEC.md (interfaces only), "R#" the readings listed in DESIGN.md.
 *
 * The problem: solve A x = b for sparse symmetric positive definite A via the
 * Cholesky factorization A = L L^T "using a right-looking approach", the "resulting triangular
 * factors ... used to compute the solution".
 *
 * Conventions for every call:
 *   - extern "C"; no C++ exception crosses the ABI; every call returns an int status
 *     (SPCHOL_OK = 0, negative = error) and on error sets a thread-local message readable with
 *     spchol_last_error().
 *   - Pointers are HOST pointers unless the name or comment says "device" (d_ prefix).
 *   - Index widths: column pointers and every L / panel offset are int64 (nnz(L) exceeds 2^31 on
 *     the 3-dof config); row indices and permutations are int32 (n < 2^31).
 *   - One handle must not be used from two threads at once.  Different handles are independent.
 */
#ifndef SPCHOL_H_
#define SPCHOL_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct spchol_handle spchol_handle;

enum {
  SPCHOL_OK = 0,
  SPCHOL_ERR_DIMENSION = -1,   /* n < 0, or array lengths inconsistent with n             */
  SPCHOL_ERR_VALIDATION = -2,  /* input violates the CSC contract, perm not a bijection   */
  SPCHOL_ERR_NOT_SPD = -3,     /* a pivot was <= 0 or NaN                  */
  SPCHOL_ERR_DEVICE_OOM = -4,  /* device allocation failed (panels do not fit)     */
  SPCHOL_ERR_CUDA = -5,        /* any other CUDA runtime error                            */
  SPCHOL_ERR_NCCL = -6,        /* multi-GPU exchange failed                               */
  SPCHOL_ERR_STATE = -7        /* call out of order (solve before a successful factor)    */
};

typedef struct {
  double merge_cap;     /* supernode merging stops before the cumulative added storage exceeds
                           merge_cap * nnz(L) (reading R4).  Default 0.25.
                           A negative value disables merging (fundamental partition). */
  int32_t device;       /* CUDA device ordinal used by this handle. Default 0.  A negative value
                           makes a host-only handle: analyze runs the symbolic phase and the
                           launch plan but allocates nothing on a device; factor/solve return
                           SPCHOL_ERR_STATE (used to check the symbolic phase without a GPU). */
  int32_t block;        /* column block width of the blocked cdiv (POTRF/TRSM) for large supernodes;
                           0 = library default (64).  Must be a multiple of 8 in [8, 64]. */
  int32_t small_max_k;  /* supernodes with k <= small_max_k and a panel that fits shared memory
                           are factored by the fused one-CTA-per-supernode kernel; 0 = default,
                           -1 = never. */
  int32_t use_graph;    /* 1 = capture the factor's launch sequence in a CUDA graph (default 1). */
  int32_t dist_rank;    /* multi-GPU: this process's rank (default 0), one process per GPU */
  int32_t dist_world;   /* multi-GPU: number of ranks (default 1).  With dist_world > 1 the merged
                           supernodal tree is mapped to ranks by proportional subtree-to-GPU mapping
                           (SURVEY §8(e)): each rank factors its own subtrees (phase A), their
                           boundary update blocks go to the owners of the ancestor block columns
                           (NCCL send/recv, phase B), and the top supernodes are factored block
                           column by block column over their rank groups (phase C).  Each rank holds
                           only its own part of L in device memory.  Needs update_mode 0, not
                           deterministic, and spchol_dist_attach_nccl. */
  int32_t subtree_streams; /* single GPU: independent subtrees (proportional mapping onto this many
                           virtual ranks) are factored concurrently on their own stream pairs, the
                           top supernodes after they join.  0 = default (4), 1 = one level-set
                           schedule for the whole tree. */
  int32_t update_mode;  /* 0 = RL (default): U_J formed in 64x64 tiles and scattered through relind
                           (P:307).  1 = RLB: per block pair (B, B') of
                           J's rows, L_{B',B} of B's ancestor updated directly (one relindB per
                           block).  Same factor; RLB has more, smaller tiles on this hardware. */
  int32_t deterministic; /* 1 = bitwise run-to-run reproducible factor (reading C-7):
                           each level's supernodes are split into column-conflict-free colour
                           classes (greedy, ascending supernode order; R_J1 and R_J2 disjoint within
                           a class), one launch per class, plain read-modify-write scatter instead of
                           FP64 RED; subtree_streams is forced to 1.  Requires update_mode 0.
                           Default 0.  (The solve's RED into shared ancestors stays unordered.) */
  int32_t partition_refinement; /* 1 = reorder the columns inside each supernode after merging so that the
                           rows every descendant has in it form fewer consecutive runs (fewer RLB
                           blocks; reading R14 in DESIGN.md).  Changes the final
                           permutation (and so the exact factor's pattern inside the panels), not
                           the panel storage.  Default 0. */
  int64_t device_mem_cap; /* single GPU, memory-capped (out-of-core) mode (P:484-489,
                           P:568): 0 = unlimited (default).  Otherwise the device arena is planned to
                           stay under this many bytes: the supernodal tree is split into a resident
                           top and subtree batches that share one device window; each batch is
                           factored in the window, its contributions land in the resident top panels
                           through the usual relind scatter, and its finished panels are copied to
                           pinned host memory (the solve streams them back batch by batch).  The cap
                           bounds the factor's device storage (window + resident top panels + kept
                           diagonal-block inverses = SPCHOL_Q_ARENA_BYTES); the metadata (A's values
                           and maps, relind, task lists) comes on top (SPCHOL_Q_DEVICE_BYTES).
                           Analyze fails with SPCHOL_ERR_DEVICE_OOM when even the top does not fit. */
} spchol_options;

/* Fill *opt with the defaults above. */
void spchol_default_options(spchol_options* opt);

/*
 * spchol_analyze — symbolic analysis (integer only, host) + device setup.
 *
 * Input A: n x n, lower triangle in CSC, 0-based. colptr[n+1] (int64, colptr[0]=0,
 * non-decreasing), rowidx[colptr[n]] (int32): within each column rows strictly increasing, first
 * entry of column j is the diagonal j (always stored), all rows in [j, n).  values[colptr[n]]
 * (FP64) may be NULL (then spchol_set_values must be called before factor).  A is taken as
 * lower + lower^T - diag.
 * perm: old -> new fill-reducing ordering (e.g. nested dissection), a bijection of
 * [0,n); NULL = identity.
 *
 * Steps: permute -> elimination tree -> postorder ->
 * column counts -> fundamental supernodes [LNP93] -> greedy child-parent merging at
 * merge_cap -> final permutation P_f (postorder of the merged supernodal tree) ->
 * rows(J) -> relative indices relind(J,P) via indmap -> level sets of the
 * supernodal tree, panel layout in one device arena, launch plan.  A's values (if given) are
 * uploaded to the device.
 *
 * Ownership: analyze deep-copies everything it needs; the caller may free its arrays on return.
 * The handle owns all host and device memory; spchol_destroy frees it.
 * Errors: DIMENSION (n < 0), VALIDATION (contract violations above; perm not a bijection),
 * DEVICE_OOM, CUDA.  On error *out is set to NULL.
 */
int spchol_analyze(int64_t n, const int64_t* colptr, const int32_t* rowidx, const double* values,
                   const int32_t* perm, const spchol_options* opt, spchol_handle** out);

/*
 * Save the symbolic analysis of h to a binary file (path); spchol_load_analysis rebuilds a handle
 * from it — launch plan and device state for opt (its merge_cap is ignored: the file's is used) —
 * without re-running analyze.  Values must then be given with spchol_set_values.  Errors:
 * VALIDATION (I/O failure, not an analysis file), plus those of analyze's device setup.
 */
int spchol_save_analysis(const spchol_handle* h, const char* path);
int spchol_load_analysis(const char* path, const spchol_options* opt, spchol_handle** out);

/* Replace A's values (same pattern as analyze; host array of colptr[n] doubles, copied to the
 * device on the handle's stream, synchronously w.r.t. the host buffer).  Single GPU, resident
 * arena: the panel arena is zeroed on a side stream during the upload (after the handle's earlier
 * work), so the next factor skips its own zeroing (a1); the previous factor's panels are gone. */
int spchol_set_values(spchol_handle* h, const double* values);

/* Same, from a device array (d_values, colptr[n] doubles), enqueued on the handle's stream. */
int spchol_set_values_device(spchol_handle* h, const double* d_values);

/* CUDA stream (cudaStream_t; NULL = the handle's own non-blocking stream, the default) on which
 * factor/solve enqueue their work.  Events recorded by the caller on the same stream bracket exactly that work. */
int spchol_set_stream(spchol_handle* h, void* stream);

/*
 * spchol_factor_async — enqueue the numeric RL factorization of
 * C_f = P_f A P_f^T on the handle's stream and return without synchronizing:
 *   a1 panel init: panels := 0, A's entries scattered into their supernode panels;
 *   per level of the supernodal elimination tree (leaves first), for every supernode J in it:
 *   a3/a4 cdiv(J): POTRF of the k_J x k_J diagonal block, TRSM of the t_J x k_J rest;
 *   a5/a6 U_J = L_{R,J} L_{R,J}^T (DSYRK) assembled into the ancestor panels through
 *   relind, fused in one kernel (no U workspace).
 * A failing pivot is recorded on the device (a7); read it with spchol_factor_status.
 */
int spchol_factor_async(spchol_handle* h);

/*
 * spchol_factor_status — synchronize the handle's stream; *fail_col = first failing column in
 * the final numbering (-1 if none), *fail_col_orig = the same column in the caller's original
 * numbering (-1 if none).  Returns SPCHOL_OK or SPCHOL_ERR_NOT_SPD (reading R8).
 * Either pointer may be NULL.
 */
int spchol_factor_status(spchol_handle* h, int64_t* fail_col, int64_t* fail_col_orig);

/* spchol_factor = spchol_factor_async + spchol_factor_status. */
int spchol_factor(spchol_handle* h, int64_t* fail_col, int64_t* fail_col_orig);

/*
 * spchol_solve — x = A^{-1} b with the computed factor: y = P_f b; L y' = y (forward, supernodes
 * leaves first); L^T z = y' (backward, root first); x = P_f^T z.  b, x: host arrays,
 * column-major n x nrhs with leading dimension ld >= n; b and x may alias.
 * Errors: STATE before a successful factor, DIMENSION on nrhs < 1 or ld < n.
 * Multi-GPU (dist_world > 1): collective — every rank calls it with the same b (only the entries
 * of the rows a rank holds are read) and receives the whole x; only solution segments travel
 * (a reduce per top block column forward, a broadcast backward, one all-reduce of x).
 */
int spchol_solve(spchol_handle* h, const double* b, double* x, int32_t nrhs, int64_t ld);

/* Same with device arrays, enqueued on `stream` (a cudaStream_t; NULL = the handle's stream, see
 * spchol_set_stream); no host synchronization. */
int spchol_solve_device(spchol_handle* h, const double* d_b, double* d_x, int32_t nrhs, int64_t ld, void* stream);

/* ---------------- introspection / parity exports ---------------- */
enum {
  SPCHOL_Q_N = 0,            /* n                                                         */
  SPCHOL_Q_NNZ_A = 1,        /* stored entries of A's lower triangle                       */
  SPCHOL_Q_NNZ_L = 2,        /* nnz(L) of the exact factor, diagonal included              */
  SPCHOL_Q_NFUND = 3,        /* fundamental supernodes                                     */
  SPCHOL_Q_NSUPER = 4,       /* supernodes after merging                                   */
  SPCHOL_Q_ADDED = 5,        /* stored entries added by merging                            */
  SPCHOL_Q_NLEVELS = 6,      /* levels of the merged supernodal tree                       */
  SPCHOL_Q_ROWS_LEN = 7,     /* sum_J m_J (length of the rows array)                       */
  SPCHOL_Q_NPAIRS = 8,       /* (J, ancestor P) pairs with a relind vector                 */
  SPCHOL_Q_RELIND_LEN = 9,   /* total relind entries                                       */
  SPCHOL_Q_PANEL_DOUBLES = 10, /* doubles in the device panel arena (incl. ld padding)     */
  SPCHOL_Q_NMERGES = 11,     /* merges applied                                             */
  SPCHOL_Q_FLOPS_EXACT = 12, /* sum_j cc_j^2 (the metric's flop count)                     */
  SPCHOL_Q_FLOPS_EXEC = 13,  /* flops of the supernodal algorithm incl. padding             */
  SPCHOL_Q_LAUNCHES = 14,    /* kernels launched by one factor                              */
  SPCHOL_Q_UPDATE_ENTRIES = 15, /* sum_J t_J (t_J+1)/2 scattered update entries             */
  SPCHOL_Q_NBLOCKS = 16,      /* RLB blocks over all supernodes                   */
  SPCHOL_Q_NMARKERS = 17,     /* multi-GPU: exchange points (markers) of this rank's phase C     */
  SPCHOL_Q_NTOP_DIST = 18,    /* multi-GPU: top supernodes distributed over their rank group     */
  SPCHOL_Q_DEVICE_BYTES = 19, /* device memory the handle owns (panels, inverses, plan; 0 if host-only) */
  SPCHOL_Q_COMM_SEND_BYTES = 20, /* multi-GPU: logical bytes this rank sends per factor (update runs +
                                    its broadcast block columns, once per receiving member); host-only too */
  SPCHOL_Q_COMM_RECV_BYTES = 21, /* multi-GPU: bytes this rank receives per factor                      */
  SPCHOL_Q_ARENA_BYTES = 22,  /* physical device bytes of this rank's panels + inverses (+ broadcast
                                 ring, update and receive regions under multi-GPU); host-only too    */
  SPCHOL_Q_DIST_GRAPH = 23,   /* multi-GPU: 1 if the factor (with its NCCL calls) replays as a CUDA graph */
  SPCHOL_Q_COMM_B_SEND_BYTES = 24, /* multi-GPU: bytes this rank sends in the boundary-block exchange
                                      after phase A (SURVEY §8(e) phase B); host-only too               */
  SPCHOL_Q_COMM_B_RECV_BYTES = 25, /* ... receives in it                                                 */
  SPCHOL_Q_NBATCHES = 26,     /* memory-capped mode: subtree batches (0 when not capped)                */
  SPCHOL_Q_HOST_BYTES = 27    /* memory-capped mode: pinned host bytes holding the finished batches     */
};
int spchol_query(const spchol_handle* h, int key, int64_t* value);

/*
 * Integer symbolic arrays (the bit-exact parity contract).  Any pointer may be NULL (skipped).
 * Sizes: post[n] (O3 postorder: post[k] = the user-permuted index numbered k), parent3[n] and
 * cc3[n] (etree / column counts in postorder numbering), ffirst[NFUND+1] (fundamental
 * partition, postorder numbering), fgroup[NFUND] (fundamental -> merged group = fundamental
 * index of the group's top), perm_final[n] (P_f, old -> final), sfirst[NSUPER+1], sparent[NSUPER],
 * rows_ptr[NSUPER+1], rows[ROWS_LEN] (final numbering, ascending), rel_ptr[NSUPER+1] (pairs of J),
 * rel_anc[NPAIRS], rel_q0[NPAIRS] (first row index q in rows(J) with rows(J)[q] >= f_P),
 * rel_off[NPAIRS+1], relind[RELIND_LEN], parent_final[n], cc_final[n], level[NSUPER].
 */
int spchol_export_symbolic(const spchol_handle* h, int32_t* post, int32_t* parent3, int32_t* cc3,
                           int32_t* ffirst, int32_t* fgroup, int32_t* perm_final, int32_t* sfirst,
                           int32_t* sparent, int64_t* rows_ptr, int32_t* rows, int64_t* rel_ptr,
                           int32_t* rel_anc, int32_t* rel_q0, int64_t* rel_off, int32_t* relind,
                           int32_t* parent_final, int32_t* cc_final, int32_t* level);

/*
 * RLB block structure: blk_ptr[NSUPER+1]; for each block b of supernode J
 * (blk_ptr[J] <= b < blk_ptr[J+1]): blk_q[b] = position in rows(J) of its first row, blk_len[b]
 * rows (consecutive global rows), blk_anc[b] = the ancestor supernode whose columns contain them,
 * blk_relind[b] = relindB = m_P - 1 - position of the first row in rows(P).  NBLOCKS entries.
 */
int spchol_export_blocks(const spchol_handle* h, int64_t* blk_ptr, int32_t* blk_q, int32_t* blk_len,
                         int32_t* blk_anc, int32_t* blk_relind);

/*
 * Copy the device panels back.  panel_off[NSUPER+1] (doubles; panel J occupies
 * [panel_off[J], panel_off[J] + ld[J] k_J), column-major with leading dimension ld[J] >= m_J; under
 * multi-GPU the panels are grouped by owning rank, top panels last and page-aligned, so offsets need
 * not increase with J; panel_off[NSUPER] = PANEL_DOUBLES),
 * ld[NSUPER], panels[PANEL_DOUBLES].  After factor, panel J column c (0 <= c < k_J), row q
 * (c <= q < m_J) holds L(rows(J)[q], sfirst[J] + c); entries inside the panel but outside the
 * exact pattern of L ("padding") are exactly +-0.0.  Synchronizes the stream.
 * Multi-GPU: every value export (panels, panel, factor CSC, diagonal) holds the entries this rank
 * owns (its subtrees, its top supernodes / block columns; spchol_export_mapping) and zeros
 * elsewhere, so the sum of the ranks' exports is L.  Not collective.
 */
int spchol_export_panels(const spchol_handle* h, int64_t* panel_off, int32_t* ld, double* panels);

/* Copy panel J (ld[J] k_J doubles, layout as above) to out.  Synchronizes. */
int spchol_export_panel(const spchol_handle* h, int32_t J, double* out);

/*
 * The exact factor L of C_f = P_f A P_f^T in CSC, final numbering:
 * Lp[n+1] (int64, = prefix sums of cc_final), Li[NNZ_L] (rows ascending within each column, the
 * diagonal first), Lx[NNZ_L] (values from the panels).  padding_nonzeros (optional) receives the
 * number of panel entries outside the exact pattern that are not exactly +-0.0 (must be 0).
 * Li / Lx / padding_nonzeros may be NULL.  Lp and Li work on host-only handles; Lx and
 * padding_nonzeros need a successful factor (else STATE).  Host work O(nnz(L)); synchronizes.
 */
int spchol_export_factor_csc(const spchol_handle* h, int64_t* Lp, int32_t* Li, double* Lx, int64_t* padding_nonzeros);

/* diag[j] = L(j,j) for every final column j (n doubles; log det A = 2 sum log diag).
 * Synchronizes the stream. */
int spchol_export_diagonal(spchol_handle* h, double* diag);

/* Kernel timing (CUDA events bracketing every launch of each kernel class on the handle's
 * stream while enabled; disabled by default and incompatible with graph replay, which is
 * bypassed while enabled).  kind: 0 = fused small-supernode kernel, 1 = POTRF, 2 = TRSM,
 * 3 = in-panel update GEMM, 4 = SYRK/GEMM + relind scatter (U_J), 5 = panel init, 6 = RLB
 * block-pair updates, 7 = fused outer-block cdiv (POTRF + TRSM + in-block updates in one launch).
 * Returns launches, summed milliseconds, algorithmic flops and bytes of that class since the last
 * reset.  spchol_kernel_stats synchronizes the stream. */
int spchol_enable_kernel_timing(spchol_handle* h, int enable);
int spchol_kernel_stats(spchol_handle* h, int kind, int64_t* launches, double* ms, double* flops,
                        double* bytes);

/* Per-launch trace of the timed launches since the last spchol_kernel_stats/enable call (timing
 * must be enabled): for launch i < min(cap, *count): kinds[i] (as above), levels[i] (level of the
 * supernodal tree, -1 for the init), ntasks[i] (CTAs), ms[i].  Diagnostics only. */
int spchol_kernel_trace(spchol_handle* h, int64_t cap, int64_t* count, int32_t* kinds, int32_t* levels,
                        int32_t* ntasks, double* ms);

/* ---------------- multi-GPU (one process per GPU) ---------------- */
/* Process-wide multi-GPU setup: this process is rank `rank` of `world`, and
 * `nccl_unique_id` (128 bytes, from spchol_dist_nccl_unique_id on one rank, broadcast by the caller)
 * names the communicator.  Every later spchol_analyze / spchol_load_analysis whose options keep the
 * default dist_world == 1 then builds a rank of that world and attaches the communicator itself, so
 * those calls become collective.  world == 1 clears the setting.  VALIDATION on bad arguments. */
int spchol_dist_init(int32_t rank, int32_t world, const void* nccl_unique_id);
/* Create an NCCL unique id (128 bytes) on one rank; the caller broadcasts it to the others. */
int spchol_dist_nccl_unique_id(void* out128);
/* Attach an NCCL communicator (ncclCommInitRank over dist_world ranks, this handle's dist_rank;
 * collective: every rank must call it).  NCCL is loaded with dlopen (libnccl.so.2). */
int spchol_dist_attach_nccl(spchol_handle* h, const void* unique_id128);
/* owner[NSUPER]: rank owning each supernode's subtree, -1 for the top supernodes (all 0 when
 * dist_world == 1); top_owner[NSUPER]: the rank that factors an undistributed top supernode, and
 * the rank owning block column 0 of a distributed one (block column C of a distributed top
 * supernode with rank group [lo, hi) belongs to lo + (C + top_owner - lo) mod (hi - lo)), -1
 * otherwise;
 * *top_off: first double of the top-panel region; *top_slot: first diagonal-inverse slot of the top
 * supernodes.  Any pointer may be NULL. */
int spchol_export_mapping(const spchol_handle* h, int32_t* owner, int32_t* top_owner, int64_t* top_off,
                          int64_t* top_slot);
/*
 * Multi-GPU phase C.  Top supernodes whose work reaches a threshold are distributed
 * over their rank group: block columns of W = 256 columns are owned cyclically; the owner of a
 * block column runs its cdiv (POTRF, TRSM, in-block updates) and broadcasts it to the rest of the
 * group (ncclBroadcast on the group's communicator), every member applies the trailing updates of
 * the block columns it owns and forms its partial U_J = sum over its block columns C of
 * L_{R,C} L_{R,C}^T.  After each top level (and after phase A), every update block travels to the
 * owners of its destination block columns (grouped ncclSend / ncclRecv, one message per column
 * run) and is extend-added there.  Smaller top supernodes are factored whole by top_owner.
 */
/* Executed flops of this rank's plan: phase A (own subtrees; the whole factor when dist_world == 1)
 * and, per level l < NLEVELS, phase C's share of that level (top_level may be NULL).  Works on
 * host-only handles (device < 0): the work model of the multi-GPU schedule. */
int spchol_dist_plan_flops(const spchol_handle* h, double* phase_a, double* top_level);

void spchol_destroy(spchol_handle* h);
const char* spchol_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SPCHOL_H_ */
