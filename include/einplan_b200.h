/* einplan_b200 inner C ABI: the B200 (sm_100a) kernel layer under the
 * einplan host API.
 *
 * The reference executes every binary step of a term with the host loop nest
 * naive_evaluate (proj/src/evaluate.cpp:7-63) called per virtual rank by
 * local_contract (proj/src/executor.cpp:126-154), then sums partial outputs
 * with allreduce (executor.cpp:80-108) and moves intermediates with
 * apply_plan (proj/src/redistribute.cpp:185-206).  The entry points below
 * replace those three calls with device kernels; the host executor
 * (einplan.h's einplan_run_json and eb_rank_*) drives them.
 *
 * Conventions: plain pointers and sizes only; device pointers everywhere a
 * tensor is named; `stream` is a cudaStream_t (NULL = legacy default);
 * return value is an eb_status (0 = ok) and eb_last_error() holds the
 * message.  There is no CPU fallback: without a usable sm_100 device every
 * compute entry point returns EB_E_DEVICE.
 */
#ifndef EINPLAN_B200_H
#define EINPLAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum eb_status {
  EB_OK = 0,
  EB_E_INVALID = 1, /* descriptor or argument rejected */
  EB_E_DEVICE = 2,  /* no sm_100 device / CUDA error */
  EB_E_COMM = 3     /* collective failed */
} eb_status;

const char* eb_last_error(void);
const char* eb_build_info(void); /* arch, nvcc version, build flags */

/* One factor matrix of a Khatri-Rao row: row-major [extent][ld], columns
 * 0..R-1 used. */
typedef struct eb_factor {
  const double* ptr;
  int64_t extent;
  int64_t ld;
} eb_factor;

enum { EB_ROW = 0, EB_COL = 1 };       /* which X dimension is contracted innermost */
enum { EB_REDUCE = 0, EB_BATCHED = 1 }; /* sum over the outer index, or one output per outer index */

/* The fused MTTKRP term / TTM step ("contraction" of one dense block).
 *
 * EB_ROW   X is [P][M][Q][L] row-major, contraction over l (contiguous):
 *            out[m][r] = sum_{p,q,l} X[p,m,q,l] * KRP(pre)[p,r] * KRP(mid)[q,r] * U[l,r]
 * EB_COL   X is [P][Q][M] row-major, contraction over q (strided):
 *   REDUCE   out[m][r]    = sum_{p,q} X[p,q,m] * KRP(pre)[p,r] * U[q,r]
 *   BATCHED  out[p][m][r] = sum_q     X[p,q,m] * U[q,r]          (TTM)
 * KRP(list)[x,r] = prod_f list[f].ptr[x_f * ld_f + r], x decomposed row-major
 * over the list's extents (empty list = 1).  U is row-major [L or Q][R].
 * This covers order-N MTTKRP in every mode (pre = modes before the output
 * mode, mid = modes between it and the last, U = the last (ROW) or the
 * second-to-last (COL) mode's factor) and every TTM of the TTMc chains. */
typedef struct eb_contract_desc {
  int variant; /* EB_ROW / EB_COL */
  int mode;    /* EB_REDUCE / EB_BATCHED (BATCHED requires EB_COL) */
  int64_t P, M, Q, L; /* L ignored for EB_COL */
  int64_t R;
  const double* X;
  const double* U;
  int64_t ldu;
  int n_pre;
  eb_factor pre[8];
  int n_mid;
  eb_factor mid[8];
  double* out;
} eb_contract_desc;

/* Device scratch the call needs (split-K partials, staged factor copies). */
size_t eb_contract_workspace(const eb_contract_desc* d);
int eb_contract(const eb_contract_desc* d, void* workspace, size_t workspace_bytes,
                void* stream);

/* Output scatter: the redistribution of a term's output fused into the
 * producing kernel's epilogue (a "push": apply_plan's message boxes,
 * redistribute.cpp:51-148 / 185-206, realised element by element).  Instead
 * of its dense output block the kernel stores every element straight into
 * the destination block(s) of the next term's placement — on the same
 * device (virtual ranks) or in the peers' mapped exchange heaps (NVLink
 * stores).  The kernel's natural output block is row-major over nd dims:
 * [0, n_outer) form its outer index, [n_outer, n_outer + n_row) its row, the
 * rest its column.  Dim d has local extent ext[d] and global base gbase[d];
 * the element at global coordinates g goes to destination rank
 *   sum_d (g_d / block[d]) * rank_stride[d] + rep_offset[k]   (k < n_rep)
 * at element offset sum_d (g_d % block[d]) * local_stride[d] of dest[rank].
 * Every coordinate and extent must be below 2^31. */
typedef struct eb_scatter {
  int nd, n_outer, n_row, n_rep;
  int64_t ext[8], gbase[8], block[8], rank_stride[8], local_stride[8];
  int64_t rep_offset[8];
  double* dest[64];
} eb_scatter;

/* Dimension-tree pair (CP-ALS sweep, order 3): one pass over X computes the
 * mode-0 MTTKRP (d: EB_ROW, EB_REDUCE, P = 1, one `mid` factor B, U = C) and
 * the mode-1 MTTKRP  out1[j][r] = sum_{i,k} X[i,j,k] A[i,r] C[k,r]:
 * T[i][j] = X[i][j][:] C is contracted once on DMMA and folded into
 * out[i] (x B[j]) and out1[j] (x A[i]) — 2R flops per X element for two
 * modes instead of 4R.  Needs M >= 128, R <= 64, L even.  The reference
 * runs each mode as its own einsum (two run() calls); the outputs are the
 * same up to FP64 summation order. */
size_t eb_mttkrp2_workspace(const eb_contract_desc* d);
int eb_mttkrp2(const eb_contract_desc* d, const double* A, int64_t lda, double* out1,
               void* workspace, size_t workspace_bytes, void* stream);

/* One CP-ALS sweep of an order-3 tensor (not in the
 * reference, which runs each MTTKRP as its own einsum): updates the factors
 * A [I][R], B [J][R], C [K][R] (device, row-major) in place —
 *   A = MTTKRP_0 ((B'B) (.) (C'C))^-1, B = MTTKRP_1 ((A'A) (.) (C'C))^-1,
 *   C = MTTKRP_2 ((A'A) (.) (B'B))^-1, each with the factors already updated —
 * with the dimension tree: T = X x_3 C is contracted once and serves modes 0
 * and 1, so X is read twice per sweep, not three times.  R <= 64, K even. */
size_t eb_cp3_als_workspace(int64_t I, int64_t J, int64_t K, int64_t R);
int eb_cp3_als_sweep(const double* X, int64_t I, int64_t J, int64_t K, int64_t R, double* A,
                     double* B, double* C, void* workspace, size_t workspace_bytes, void* stream);

/* Fused TTM pair: the two TTM steps of one fused term with the intermediate
 * kept on chip (TTMc-O5 terms [t0,t1] and [t2,out]; replaces two
 * local_contract calls, proj/src/executor.cpp:220-235):
 *   out[p][m][b][c] = sum_{j,k} X[p][j][k][m] * U1[j][b] * U2[k][c]
 * i.e. t0[p][k][m][b] = sum_j X U1 followed by out = sum_k t0 U2.
 * X row-major [P][Q1][Q2][M], U1 [Q1][ldu1], U2 [Q2][ldu2], out
 * [P][M][N1][N2].  Needs Q1 <= 64, N1 <= 16, N2 <= 16, M even; no workspace. */
typedef struct eb_ttm2_desc {
  int64_t P, Q1, Q2, M, N1, N2;
  const double* X;
  const double* U1;
  int64_t ldu1;
  const double* U2;
  int64_t ldu2;
  double* out;
} eb_ttm2_desc;

int eb_ttm2(const eb_ttm2_desc* d, void* stream);

/* Both terms of the TTMc-O5 schedule ([t0,t1], [t2,out]) in ONE persistent
 * launch when the t1 hand-over between them is a whole-block self message
 * (the reference's apply_plan copy, redistribute.cpp:185-206; C5 at P = 1,
 * 2, 8): term A (a: X -> a->out = t1) and term B (b: b->X == a->out, viewed
 * as [P][Q1b][Q2b][Mb] with Q1b Q2b Mb = Ma N1a N2a -> b->out).  t1 passes
 * through L2 (evict-last stores, discarded once read) instead of HBM; term B
 * of slab p starts once every term-A tile of p is stored (in-kernel counters,
 * workspace = eb_ttm2_chain_workspace(a) bytes, zeroed by the call). */
size_t eb_ttm2_chain_workspace(const eb_ttm2_desc* a);
int eb_ttm2_chain(const eb_ttm2_desc* a, const eb_ttm2_desc* b, void* workspace,
                  size_t workspace_bytes, void* stream);

/* Both TTMc-O5 terms with term B's second contraction folded into term A
 * (same hand-over condition as eb_ttm2_chain): term B's last mode m (Q2b,
 * a multiple of 16, <= 64) is the innermost mode of term A's rows, so
 *   s[p][R'][e][b c]  = sum_m t1[p][R'][m][b c] U2b[m][e]   (term A's epilogue)
 *   b->out[q][b c][d][e] = sum_l U1b[l][d] s[q][l][e][b c]   (a second kernel)
 * and t1 is never stored.  Reference: the two terms of the schedule
 * (executor.cpp:220-235) with the self hand-over (redistribute.cpp:185-206);
 * equal to it up to the summation order of l and m.  a->out and b->X are
 * ignored; workspace = eb_ttmc_fold_workspace(a, b) bytes (s).  Needs the
 * eb_ttm2 limits on both terms and N1b, N2b <= 16. */
size_t eb_ttmc_fold_workspace(const eb_ttm2_desc* a, const eb_ttm2_desc* b);
int eb_ttmc_fold(const eb_ttm2_desc* a, const eb_ttm2_desc* b, void* workspace,
                 size_t workspace_bytes, void* stream);

/* eb_contract (EB_COL, EB_BATCHED only) / eb_ttm2 with the scatter epilogue;
 * d->out is ignored. */
int eb_contract_scatter(const eb_contract_desc* d, const eb_scatter* s, void* workspace,
                        size_t workspace_bytes, void* stream);
int eb_ttm2_scatter(const eb_ttm2_desc* d, const eb_scatter* s, void* stream);


/* Generic binary (or unary) einsum step on dense row-major device blocks:
 * out[...] = sum over contracted symbols of lhs[...] * rhs[...] — the GPU
 * replacement of naive_evaluate for step shapes the fused kernels do not
 * cover (GEMM chains, KRP, OUTER, ELEMENTWISE).  Index strings as in the
 * reference step ("ijk,jka->ia"); `ext` gives one extent per ASCII code. */
int eb_step_generic(const char* lhs_indices, const char* rhs_indices,
                    const char* out_indices, const int64_t* ext, const double* lhs,
                    const double* rhs, double* out, void* stream);

/* Deterministic group sum on one device (virtual ranks): acc = 0.0, then
 * members added in the given (ascending-rank) order; result written to
 * every member (executor.cpp:80-108). */
int eb_group_sum(double* const* members, int n_members, int64_t n, void* stream);

/* The same ascending-rank sum written to `dst` only (members are read, not
 * written): the peer-memory allreduce, where members are the group's blocks
 * in the peers' exchange heaps (executor.cpp:91-98). */
int eb_group_sum_into(const double* const* members, int n_members, int64_t n, double* dst,
                      void* stream);

/* Strided box copy of one redistribution message between dense row-major
 * device blocks (redistribute.cpp:152-183); src may be a peer-mapped pointer
 * (the peer transport's pull).  Adjacent dims the box spans contiguously in
 * both blocks are merged; rows move as 16-byte vectors when aligned. */
int eb_copy_box(int nd, const double* src, const int64_t* src_shape, double* dst,
                const int64_t* dst_shape, const int64_t* oy_lo, const int64_t* oy_hi,
                const int64_t* ox_lo, void* stream);

/* Row padding for the DMMA path of odd contiguous extents (TMA needs 16-byte
 * row pitches): dst [rows][dcols] = src [rows][cols] with zero columns
 * cols..dcols-1. */
int eb_pad_rows(const double* src, int64_t rows, int64_t cols, double* dst, int64_t dcols,
                void* stream);

/* dst = src with its dims reordered: dst dim d is src dim perm[d] (both
 * dense row-major; the TTM step whose result order differs from the
 * kernel's [pre, post, b]). */
int eb_permute(int nd, const double* src, const int64_t* src_shape, const int* perm, double* dst,
               void* stream);

/* Any dense einsum with up to 8 operands, evaluated on the device (used for
 * run(..., verify) on the GPU: the reference compares against naive_evaluate,
 * executor.cpp:255-261). */
int eb_einsum_generic(int n_ops, const char* const* in_indices, const char* out_indices,
                      const int64_t* ext, const double* const* ops, double* out, void* stream);

/* Seeded input generation identical to random_tensor (tensor.cpp:55-63):
 * fills host memory with n values of the mt19937_64(seed) stream starting at
 * element `skip` of that stream. */
void eb_random_fill_host(double* out, int64_t n, uint64_t seed, int64_t skip);
/* the box [base, base + shape) of the row-major tensor random_tensor(gshape,
 * seed) would produce, written densely to out (one pass over the stream up
 * to the box's last element; memory O(box)) */
int eb_random_fill_block(double* out, uint64_t seed, int nd, const int64_t* gshape,
                         const int64_t* base, const int64_t* shape);
/* a stateful stream: consecutive eb_rng_fill calls continue where the last
 * one stopped (e.g. the 64-row i-slabs of C5's global X one after another,
 * one pass over the stream instead of one per slab) */
typedef struct eb_rng eb_rng;
int eb_rng_create(uint64_t seed, int64_t skip, eb_rng** out);
void eb_rng_fill(eb_rng* g, double* out, int64_t n);
void eb_rng_destroy(eb_rng* g);

void eb_free(void* p);
/* bytes in use in the current device's stream-ordered pool (where executors
 * allocate their per-run blocks): flat across repeated runs */
int eb_mem_in_use(int64_t* bytes);

/* Host-only planning: plan_report(make_pipeline(...)) as einplan/v1 JSON
 * (schedule.cpp:72-80, report.cpp:194-199).  No device needed. */
int eb_plan_json(const char* einsum, const char* dims, int64_t procs, double fast_mem,
                 int include_messages, char** json_out);

/* Path options (read once from EB_* environment variables at load; this
 * call changes them between runs): "no_fused_tma" 0/1, "no_rf" 0/1,
 * "rf_cfg" "RTxOS"|"auto", "ttm2_variant" 0/1/2, "fuse_ttm2" 0/1,
 * "gemm" 0 auto / 1 forced / 2 off (wide GEMM steps: one launch over
 * (row tile, 64-column block) items instead of per-64-column split-K),
 * "fuse_redistribution" 0/1 (TTM outputs pushed by the producing kernel into
 * the next term's blocks, eb_scatter), "chain_terms" 0/1 (two TTM-pair
 * terms joined by a self hand-over in one eb_ttm2_chain launch), "fold_terms"
 * 0/1 (such terms as eb_ttmc_fold, t1 never stored; default 0). */
int eb_set_option(const char* name, const char* value);

/* ---- rank-local executor (the GPU run(), executor.cpp:156-263) ----------
 * rank < 0: all `procs` ranks are virtual and resident on the current device
 *           (reductions = eb_group_sum, redistribution = eb_copy_box);
 * rank >= 0: this process is rank `rank` of `procs`, one GPU per process,
 *           collectives over NCCL (nccl_id = 128 bytes from
 *           eb_nccl_unique_id on rank 0, broadcast by the caller). */
typedef struct eb_exec eb_exec;

int eb_nccl_unique_id(void* out128);
int eb_exec_create(const char* einsum, const char* dims, int64_t procs, double fast_mem,
                   int64_t rank, const void* nccl_id, void* stream, eb_exec** out);
/* rank `rank` of `procs` processes on one node exchanging over peer memory
 * (CUDA IPC: the group's exchange heaps mapped by every rank; host barrier
 * in the POSIX shared-memory segment `group`, e.g. "/eb_job42", the same
 * string on every rank).  Works with one GPU per process (NVLink loads) and
 * with several processes on one GPU (the multi-rank tests).  No kernel waits
 * on another rank: each collective synchronises its stream, then meets the
 * peers on the host.  Every rank must call eb_exec_run / eb_exec_gather. */
int eb_exec_create_peer(const char* einsum, const char* dims, int64_t procs, double fast_mem,
                        int64_t rank, const char* group, void* stream, eb_exec** out);
/* hybrid (one process per GPU): the peer transport's mapped heaps and fused
 * redistributions, with the MTTKRP allreduces on NCCL (ncclCommSplit groups,
 * asynchronous on the communication stream); both a group name and a
 * 128-byte ncclUniqueId */
int eb_exec_create_hybrid(const char* einsum, const char* dims, int64_t procs, double fast_mem,
                          int64_t rank, const char* group, const void* nccl_id, void* stream,
                          eb_exec** out);
/* a second executor over the same ranks and the same communicator as `peer`
 * (an ncclUniqueId initialises exactly one communicator): e.g. the three
 * MTTKRP modes of a sweep on one process group */
int eb_exec_create_like(const char* einsum, const char* dims, double fast_mem, eb_exec* peer,
                        void* stream, eb_exec** out);
void eb_exec_destroy(eb_exec* h);
/* scatter (executor.cpp:48-65): host global inputs -> this process's blocks */
int eb_exec_stage(eb_exec* h, const double* const* host_inputs);
/* a NULL entry in host_inputs keeps that operand's device blocks as they are */
/* one process = one rank: the box (global base / shape, nd dims) of operand k
 * this rank holds, and staging from a host buffer holding just that box
 * (row-major) — no process needs the global tensor */
int eb_exec_block(eb_exec* h, int k, int64_t* base, int64_t* shape, int* nd);
int eb_exec_stage_block(eb_exec* h, int k, const double* host_block);
/* virtual ranks without the global tensor: operand k from a host buffer
 * holding its global sub-box [base, base + shape) (row-major, nd dims); the
 * owned ranks' blocks inside it are staged, *staged = how many */
int eb_exec_stage_region(eb_exec* h, int k, const int64_t* base, const int64_t* shape, int nd,
                         const double* host_region, int* staged);
/* alias operand k_dst of `dst` to the staged device blocks of operand k_src of
 * `src` (same shape and placement on every owned rank, checked); `dst` then
 * stages NULL for it (e.g. one X shared by the three modes of a CP-ALS sweep) */
int eb_exec_share_input(eb_exec* dst, int k_dst, eb_exec* src, int k_src);
/* all terms: local contractions + reductions + redistributions, device only */
int eb_exec_run(eb_exec* h);
/* Reductions on a side stream: with on = 1 a run's allreduces are issued on
 * an executor-owned stream (after the local contractions), so they overlap
 * work the caller queues next on `stream` (e.g. the next mode of a sweep);
 * eb_exec_join(h) then makes `stream` wait for them.  Later terms of the same
 * schedule, eb_exec_gather and the next eb_exec_run join implicitly.  Off by
 * default: every operation is then ordered on `stream`. */
int eb_exec_set_async_reduce(eb_exec* h, int on);
int eb_exec_join(eb_exec* h);
/* CUDA graph of one run (virtual or NCCL transport): eb_exec_capture runs
 * once eagerly (every block of the run then keeps its address), captures a
 * second run on the executor's stream and instantiates it; eb_exec_replay
 * launches the graph — the same kernels, copies and collectives, one host
 * call.  Re-staging inputs keeps the graph valid; capture again after
 * changing options or shared inputs.  EB_E_INVALID for the peer / hybrid
 * transports or the legacy default stream. */
int eb_exec_capture(eb_exec* h);
int eb_exec_replay(eb_exec* h);
/* CP sweep dimension tree: run `mode0` (ijk,ja,ka->ia) and `mode1`
 * (ijk,ia,ka->ja, X and the k factor shared from mode0 with
 * eb_exec_share_input, same grid, same stream) in one pass over X with
 * eb_mttkrp2, each output reduced over its own reference group.  *fused = 1
 * when the pair ran fused, 0 when it did not qualify and both executors were
 * run separately (same results). */
int eb_exec_run_pair(eb_exec* mode0, eb_exec* mode1, int* fused);
/* gather canonical output blocks to host (virtual mode, or rank 0; other
 * ranks pass NULL — collective for the peer transport) */
int eb_exec_gather(eb_exec* h, double* host_out);
int64_t eb_exec_output_elems(eb_exec* h);
/* out8 = {allreduce_volume, redistribute_volume, max_rank_sent,
 *         fused MTTKRP launches, TTM/GEMM launches, generic launches,
 *         tree flops, terms} of the last run */
int eb_exec_stats(eb_exec* h, int64_t* out8);
/* how many redistributions of the last run were fused into their producer
 * (pushed by the TTM epilogue, eb_scatter) */
int eb_exec_fused_redistributions(eb_exec* h);
/* run_report JSON of the last run (output sum from host_out, may be NULL) */
int eb_exec_report_json(eb_exec* h, const double* host_out, char** json_out);

/* Instrumentation: total kernel launches issued by this library; optional
 * CUDA-event bracketing of the dominant contraction kernel on its launch
 * stream (enable, run, then collect the summed milliseconds). */
long long eb_launch_count(void);
void eb_timer_enable(int on);
int eb_timer_collect(double* total_ms, long long* launches);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* EINPLAN_B200_H */
