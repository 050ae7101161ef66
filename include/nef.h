/*
 * nef.h — C ABI of the B200-native NNEinFact multiplicative-update sweep.
 *
 * The calls follow the paper's statement of the problem (arxiv 2602.02759):
 *   Algorithm 1 REQUIREs data Y, model_str, initial Theta, the loss and eps and returns
 *   Theta; masking per P:321.
 *   Model family / einsum string: eq:contraction_structure, eq:einsum.
 *   Update: Theta <- max(eps, Theta * g^{-1}(A/B)) (eq:explicit-update) with
 *   A, B = einsum(einstr_l, ..., a(Y,Yhat) | b(Y,Yhat), ...) (Alg. 1 lines 7-8).
 *   (alpha,beta)-divergence P:500-525; a, b P:529; g P:531-539.
 *
 * Conventions:
 *   - (alpha, beta) are in the PAPER's convention: KL = (1,0), squared Euclidean = (1,1)
 *     (P:526).  alpha = 0 is accepted only with beta = 1.
 *   - Y is float32, dense, row-major in OUTPUT-subscript order (the last output index is
 *     contiguous).  mask is uint8 of the same shape; nonzero = observed, 0 = missing;
 *     NULL = every entry observed.  Values of Y at missing entries are never used.
 *   - Factor ell (0-based, string order) is float32, row-major in its operand-subscript
 *     order, e.g. "abc" -> [R_a][R_b][R_c].
 *   - Index sizes: observed indices take `shape` in output order; contracted indices take
 *     `ranks` in order of first appearance, left to right (reading R18).
 *   - The loss trace is the SUM over observed entries of L_{alpha,beta}(y, max(yhat,1e-30))
 *     accumulated in float64 (reading R7); trace[0] = loss at the initial factors,
 *     trace[t] = loss after full sweep t.
 *
 * Ownership: the caller owns Y, mask, the factors and the workspace (device memory, e.g.
 * allocated by PyTorch).  A plan owns host metadata only and, after nef_plan_shard, its
 * NCCL communicator.  Factors are updated in place.  All device work is enqueued on
 * `cuda_stream` (a cudaStream_t; NULL = legacy default stream); nef_fit and nef_loss
 * return after their host outputs (trace, loss) have been copied back.
 *
 * Errors: every entry point returns NEF_OK (0) or an nef_status code; nef_last_error()
 * returns a thread-local human-readable detail.  Validation errors (PARSE, SHAPE, DOMAIN,
 * ARG, UNSUPPORTED) are detected before any device work and leave every buffer untouched.
 * CUDA / NCCL errors may arrive mid-run; the factors are then unspecified.
 * No CPU fallback exists: without a CUDA device every compute call returns NEF_E_CUDA.
 */
#ifndef NEF_H_
#define NEF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nef_plan_s* nef_plan_t;

enum nef_status {
  NEF_OK = 0,
  NEF_E_PARSE = 1,        /* malformed einsum string (grammar: subs(,subs)*->subs, [a-zA-Z])   */
  NEF_E_SHAPE = 2,        /* wrong number of dims/ranks, non-positive size, int64 overflow     */
  NEF_E_DOMAIN = 3,       /* (alpha,beta) outside the paper's decomposable family      */
  NEF_E_DATA = 4,         /* reserved: invalid data at an observed entry (debug checks)        */
  NEF_E_ARG = 5,          /* null/misaligned pointer, too-small workspace, bad ell, eps <= 0   */
  NEF_E_CUDA = 6,         /* CUDA runtime error or no device                                    */
  NEF_E_NCCL = 7,         /* NCCL error or NCCL library not loadable                            */
  NEF_E_UNSUPPORTED = 8   /* model string with no lowering in this build                        */
};

/* Loss specification (the decomposable losses of the paper).
 *   NEF_LOSS_AB        (alpha, beta)-divergence, P:500-539 (alpha, beta in the paper's convention)
 *   NEF_LOSS_NEGBIN    negative binomial in its mean, dispersion phi: L = (phi+x) log(phi+y) - x log y,
 *                      a = x/y, b = (phi+x)/(phi+y), g(lambda) = lambda
 *   NEF_LOSS_BERNOULLI Bernoulli in the odds mu: L = log(1+mu) - x log mu, a = x/y, b = 1/(1+y),
 *                      g(lambda) = lambda
 *   NEF_LOSS_BINOMIAL  binomial with n trials in the odds: L = n log(1+mu) - x log mu, a = x/y,
 *                      b = n/(1+y)
 *   NEF_LOSS_JS        Jensen-Shannon: a = log((x+y)/(2y)), b = 1, g = log
 * param: phi (NEGBIN) or n (BINOMIAL) for every entry, used when aux == NULL (must be > 0).
 * aux: optional device float tensor with Y's (local) shape and layout holding a per-entry phi_i or
 * n_i (NEGBIN / BINOMIAL only; else must be NULL).  It is streamed with Y (+4 B per entry): by the
 * tcgen05 kernel as a second TMA ring (16-byte aligned base; Y streamed as nef_fit's sentinel copy
 * or unmasked), else by the CUDA-core kernel.  Valid for yhat * (phi + yhat) < 3e38 (one shared
 * reciprocal per entry).  Domain errors: NEF_E_DOMAIN (unknown kind, alpha = 0
 * with beta != 1, param <= 0 without aux); NEF_E_ARG (aux misaligned / not applicable). */
enum nef_loss_kind { NEF_LOSS_AB = 0, NEF_LOSS_NEGBIN = 1, NEF_LOSS_BERNOULLI = 2, NEF_LOSS_BINOMIAL = 3, NEF_LOSS_JS = 4 };
typedef struct nef_loss_spec {
  int kind;              /* nef_loss_kind */
  double alpha, beta;    /* NEF_LOSS_AB */
  double param;          /* NEF_LOSS_NEGBIN: phi; NEF_LOSS_BINOMIAL: n (when aux == NULL) */
  const float* aux;      /* device, per-entry phi / n, or NULL */
} nef_loss_spec;

/* Stopping rules of P:497 for nef_fit_split (readings R30, R31): stop after the sweep at which
 * the validation loss rose (strictly, vs the previous sweep) for val_patience consecutive sweeps
 * (0 disables), or the training loss fell by less than min_rel_decrease relative to its previous
 * value (a rise counts), or max_iters sweeps ran; priority in that order.  Paper: 5, 1e-6, 5000. */
typedef struct nef_stop_rule {
  int max_iters;
  double min_rel_decrease;
  int val_patience;
} nef_stop_rule;
enum nef_stop_reason { NEF_STOP_PATIENCE = 1, NEF_STOP_PLATEAU = 2, NEF_STOP_MAX_ITERS = 3 };

/* Build a plan for `einsum` over a GLOBAL tensor of `n_modes` dims `shape` (output order)
 * with `n_ranks` contracted-index sizes `ranks` (first-appearance order).  Host only:
 * parses, builds einstr_l = swap(model_str, l) for every l (Alg. 1
 * lines 1-3) and lowers each factor update to a streamed row/col/bond form (DESIGN.md
 * §Planner).  On success *out receives a new plan (free with nef_plan_destroy). */
int nef_plan(const char* einsum, int n_modes, const int64_t* shape, int n_ranks, const int64_t* ranks,
             nef_plan_t* out);

/* Plan metadata.  n_factors = L; shard_mode = mode split across ranks (-1 if unsharded);
 * [local_begin, local_begin + local_len) = this rank's index range of that mode (whole
 * range if unsharded); workspace_bytes = device scratch nef_fit / nef_loss / nef_update
 * need for a problem WITH a mask (a maskless problem needs no more).  Any out-pointer may
 * be NULL.
 * Memory: workspace_bytes includes a 4-byte-per-local-entry copy of Y (the mask folded in as a
 * NaN sentinel, R22) that masked fits stream instead of Y + mask - e.g. +17.2 GB for
 * the 2048x2048x1024 tensor, on top of Y (17.2 GB) and the mask (4.3 GB); plus small per-factor
 * scratch (side operands, split partials, < 1 % of Y). */
int nef_plan_info(nef_plan_t plan, int* n_factors, int* shard_mode, int64_t* local_begin, int64_t* local_len,
                  size_t* workspace_bytes);

/* Shape of factor `ell` as seen by THIS rank (sharded factors are local slices).
 * dims must hold >= 8 entries; *ndim receives the operand's number of indices. */
int nef_factor_shape(nef_plan_t plan, int ell, int64_t* dims, int* ndim);

/* Local shape of Y on this rank (dims must hold >= 8 entries). */
int nef_local_shape(nef_plan_t plan, int64_t* dims, int* ndim);

/* Human-readable JSON description of the lowering (for tests / debugging).  Writes at
 * most `cap` bytes including the NUL; returns the full length needed in *len. */
int nef_plan_describe(nef_plan_t plan, char* buf, size_t cap, size_t* len);

/* Fit: run `iters` full Gauss-Seidel sweeps of Algorithm 1 in place on
 * `factors` (host array of L device pointers).  Y/mask are this rank's LOCAL tensor
 * (device, contiguous, 16-byte aligned).  eps > 0 is the floor of eq:obj.
 * loss_trace: host array of iters+1 doubles, or NULL.  workspace: device scratch of at
 * least nef_plan_info's workspace_bytes.  On a sharded plan the numerator/denominator of
 * every factor that does not contain the shard mode and the loss are all-reduced over
 * NCCL; every rank ends with identical replicated factors.
 * Once per fit (R22, R25): with a mask, the mask is folded into a copy of Y in the
 * workspace (missing -> canonical NaN) that the streaming passes read instead of Y + mask, and for the
 * (alpha,beta) pairs (1,0), (1,-0.5), (0.5,0) the data-only part of the loss is summed there
 * (without a mask, by a read-only pass when iters >= 3); Y and the mask are never written. */
int nef_fit(nef_plan_t plan, const float* Y, const uint8_t* mask, double alpha, double beta, double eps,
            float* const* factors, int iters, double* loss_trace, void* workspace, size_t ws_bytes,
            void* cuda_stream);

/* nef_fit for any loss of an nef_loss_spec: the (alpha,beta) entry point above is this with
 * NEF_LOSS_AB.  Same arguments, ownership and errors; aux (if any) is this rank's local slice. */
int nef_fit_ex(nef_plan_t plan, const float* Y, const uint8_t* mask, const nef_loss_spec* loss, double eps,
               float* const* factors, int iters, double* loss_trace, void* workspace, size_t ws_bytes,
               void* cuda_stream);

/* Train / validation / heldout protocol with the stopping rules of P:497.
 * labels: device uint8, Y's local shape: 0 = excluded (missing data), 1 = train, 2 = validation,
 * 3 = heldout (reading R29).  Algorithm 1 runs on the train entries only; once per sweep the
 * same streamed pass that updates the first factor also sums the loss of each role.
 * traces: host, 3 x (rule->max_iters + 1) doubles, role-major ([train][t], [validation][t],
 * [heldout][t]); entries 0..*sweeps are written (trace[r][t] = loss sum of role r after sweep t;
 * the paper's heldout metric is trace[2][t] / counts[2]).  counts: host int64[3], entries per
 * role.  On return the factors are the iterate after sweep *sweeps, the sweep at which a rule
 * fired (reading R32); *reason is an nef_stop_reason.  The host reads the three sums once per
 * sweep (pinned memory + an event, while the sweep continues on the stream).  Sharded plans
 * all-reduce the sums over NCCL.  Errors as nef_fit; NEF_E_ARG for a null labels / rule. */
int nef_fit_split(nef_plan_t plan, const float* Y, const uint8_t* labels, const nef_loss_spec* loss, double eps,
                  float* const* factors, const nef_stop_rule* rule, double* traces, int64_t* counts, int* sweeps,
                  int* reason, void* workspace, size_t ws_bytes, void* cuda_stream);

/* Batched random restarts (N4; the paper notes restarts help).  `restarts` independent
 * fits of the same Y / mask / loss from different initial factors: factors holds restarts x L
 * device pointers, restart-major (restart r's factor ell at factors[r * L + ell]), each updated in
 * place.  Every factor update's streamed pass is ONE launch for all restarts (launch index z =
 * restart) on the tcgen05 kernel, so the restarts' CTAs stream the same Y tiles together - Y is
 * read from HBM about once per update for all restarts (the others hit L2) - and their side
 * operands, reductions and updates are separate.  (Lowerings on the CUDA-core kernel run one
 * launch per restart.)  loss_traces: host, restarts x (iters + 1) doubles, restart-major, or NULL.
 * workspace: nef_restarts_workspace_bytes(plan, restarts) bytes (one plan workspace per restart,
 * sharing one sentinel copy of Y).  iters < 2048.  Errors as nef_fit. */
size_t nef_restarts_workspace_bytes(nef_plan_t plan, int restarts);
int nef_fit_restarts(nef_plan_t plan, const float* Y, const uint8_t* mask, const nef_loss_spec* loss, double eps,
                     float* const* factors, int restarts, int iters, double* loss_traces, void* workspace,
                     size_t ws_bytes, void* cuda_stream);

/* One factor update (Algorithm 1 lines 6-9 for a single ell), the step-level API. */
int nef_update(nef_plan_t plan, int ell, const float* Y, const uint8_t* mask, double alpha, double beta,
               double eps, float* const* factors, void* workspace, size_t ws_bytes, void* cuda_stream);

int nef_update_ex(nef_plan_t plan, int ell, const float* Y, const uint8_t* mask, const nef_loss_spec* loss,
                  double eps, float* const* factors, void* workspace, size_t ws_bytes, void* cuda_stream);

/* Numerator A and denominator B of the update of factor `ell` (Alg. 1 lines 7-8, before
 * any all-reduce), written to num/den (device, size of factor ell).  For tests and for
 * torch-driven collectives (all-reduce them, then nef_apply_update). */
int nef_num_den(nef_plan_t plan, int ell, const float* Y, const uint8_t* mask, double alpha, double beta,
                float* const* factors, float* num, float* den, void* workspace, size_t ws_bytes,
                void* cuda_stream);

int nef_num_den_ex(nef_plan_t plan, int ell, const float* Y, const uint8_t* mask, const nef_loss_spec* loss,
                   float* const* factors, float* num, float* den, void* workspace, size_t ws_bytes,
                   void* cuda_stream);

/* Theta_ell <- max(eps, Theta_ell * g^{-1}(num/den)) with den == 0 -> multiplier 1
 * (eq:explicit-update P:121; g per P:531-539, identity for NB / odds losses, exp for JS). */
int nef_apply_update(nef_plan_t plan, int ell, double alpha, double beta, double eps, float* const* factors,
                     const float* num, const float* den, void* cuda_stream);
int nef_apply_update_ex(nef_plan_t plan, int ell, const nef_loss_spec* loss, double eps, float* const* factors,
                        const float* num, const float* den, void* cuda_stream);

/* Loss sum over observed entries (fp64; eq:obj P:102-106, divergence P:500-525) and the number
 * of observed entries, for the current factors (all-reduced over ranks on a sharded plan). */
int nef_loss(nef_plan_t plan, const float* Y, const uint8_t* mask, double alpha, double beta,
             float* const* factors, double* loss_sum, int64_t* n_observed, void* workspace, size_t ws_bytes,
             void* cuda_stream);
int nef_loss_ex(nef_plan_t plan, const float* Y, const uint8_t* mask, const nef_loss_spec* loss,
                float* const* factors, double* loss_sum, int64_t* n_observed, void* workspace, size_t ws_bytes,
                void* cuda_stream);

/* End-to-end variant taking HOST buffers: copies Y (and mask) host->device into
 * `device_scratch`, the factors host->device, runs nef_fit, copies the factors back
 * device->host.  device_scratch must hold nef_host_scratch_bytes(plan, has_mask). */
size_t nef_host_scratch_bytes(nef_plan_t plan, int has_mask);
int nef_fit_host(nef_plan_t plan, const float* Y_host, const uint8_t* mask_host, double alpha, double beta,
                 double eps, float* const* factors_host, int iters, double* loss_trace, void* device_scratch,
                 size_t scratch_bytes, void* cuda_stream);

/* Multi-GPU.  Rank 0 calls nef_nccl_unique_id (128 bytes), the caller broadcasts the
 * bytes (e.g. torch.distributed), then every rank calls nef_plan_shard, which splits the
 * largest mode (ties -> outermost) into contiguous near-equal ranges and creates the NCCL
 * communicator on the current CUDA device (world == 1 creates none, unless the environment
 * sets NEF_NCCL_FORCE=1: a 1-rank communicator, so that the sharded path and its all-reduces
 * run on one GPU for testing). */
int nef_nccl_unique_id(void* out128);
int nef_plan_shard(nef_plan_t plan, int rank, int world, const void* nccl_unique_id);

/* The same split without a communicator (host planning only): the plan describes this rank's
 * local tensor (nef_plan_info: local_begin / local_len; nef_plan_describe: "factor_has_shard",
 * false = the factor's A|B must be summed over ranks).  nef_num_den then returns this rank's
 * partial A|B, which the caller all-reduces (e.g. torch.distributed) before nef_apply_update, and
 * nef_loss returns this rank's partial loss sum and observed count; nef_fit / nef_update on such
 * a plan with world > 1 return NEF_E_NCCL.
 * Errors: NEF_E_ARG (bad rank / world, already sharded), NEF_E_SHAPE (largest mode < world). */
int nef_plan_shard_host(nef_plan_t plan, int rank, int world);

/* Number of kernel launches the last nef_fit / nef_loss / nef_update call enqueued. */
int64_t nef_last_launch_count(void);

/* Live per-launch timing of the streaming (fused) kernel with CUDA events recorded on the
 * launch stream around every launch (used by bench.py for the roofline).  enable != 0
 * resets the counters and turns recording on; nef_profile_read synchronizes on the last
 * recorded event and returns the summed kernel time (ms), the number of launches and the
 * algorithmic bytes those launches had to read (Y: 4 B + mask: 1 B per entry). */
int nef_profile_enable(int enable);
int nef_profile_read(double* kernel_ms, int64_t* launches, double* algorithmic_bytes);

/* Select the streaming kernel: bit 0 clear = automatic (tcgen05 where supported), set = CUDA-core
 * FFMA kernel only; bit 1 set = no sweep graphs (nef_fit then launches every kernel of every sweep
 * itself instead of replaying its cached one-sweep CUDA graph); bit 2 set = no side-operand reuse
 * inside a sweep (every update recomputes its U and column tables; by default an update reads
 * the identical table an earlier update of the same sweep left in the workspace).
 * Process-wide; for tests and A/B measurement. */
int nef_set_kernel_policy(int policy);

/* Test hook: when device_buffer != NULL the tcgen05 streaming kernel writes the P_a tile
 * (a(Y,Yhat) after masking, TF32-rounded) of its first column tile in CTA (0,0) as 128 x 64
 * floats (row-major) to it.  NULL disables. */
int nef_debug_dump(float* device_buffer);

/* Diagnostics hook: when device_buffer != NULL the tcgen05 streaming kernel records, for
 * CTA (0,0) and its first 1024 column tiles, clock64() stamps of its pipeline hand-offs
 * (TMA issue, V generation, MMA issues, elementwise waits) as int64 [tile][16]. */
int nef_debug_trace(int64_t* device_buffer);

void nef_plan_destroy(nef_plan_t plan);
const char* nef_last_error(void);
const char* nef_version(void);

#ifdef __cplusplus
}
#endif
#endif /* NEF_H_ */
