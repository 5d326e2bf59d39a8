/* fsmc.h -- C ABI of the B200 multi-chain FSM MCMC engine (libfsmc.so).
 *
 * This is the drop-in boundary for the reference's multi-chain sampling path
 * (/root/reference/pkg/src/fsm_mcmc).  The reference is pure Python, so its
 * "FFI" is the Python call surface; each entry point below replaces the
 * reference function named beside it, and paper_2503_17405_b200/ is the
 * Python host mirror that binds it with ctypes (INTEGRATION.md shows the
 * stub a maintainer would add to the reference).
 *
 * Conventions: plain pointers and sizes only.  Every buffer is device memory
 * allocated by the caller (torch tensors in the Python host) unless marked
 * "host".  `stream` is a cudaStream_t passed as void*.  Entry points never
 * throw; they return an fsmc_status and record a message retrievable with
 * fsmc_last_error().  Launches are stream-ordered and never synchronise the
 * device except where noted.  Arithmetic is IEEE fp64 (the reference's).
 */
#ifndef FSMC_H
#define FSMC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSMC_ABI_VERSION 7   /* 7: prior-transform rows owned by chains, windowed parts 0..16, fsmc_dmath_eval */
#define FSMC_WORK_WORDS 256 /* uint32 words of fsmc_state.work */
#define FSMC_NINT 32        /* int64 slots per chain in fsmc_state.ints */
#define FSMC_MAX_MODES 8    /* mixture components in FSMC_T_MOG */

typedef enum {
  FSMC_OK = 0,
  FSMC_ERR_ARG = 1,          /* invalid argument (mirrors ValueError / KernelError) */
  FSMC_ERR_CUDA = 2,         /* CUDA runtime failure */
  FSMC_ERR_UNSUPPORTED = 3   /* configuration not compiled (dimension / lanes) */
} fsmc_status;

/* kernel families: drmh_kernel (kernels/drmh.py:63), elliptical_kernel
 * (kernels/elliptical.py:65), nuts_kernel (kernels/nuts.py:103),
 * slice_kernel (kernels/slice_sampling.py:50) */
enum { FSMC_DRMH = 1, FSMC_ESS = 2, FSMC_NUTS = 3, FSMC_SLICE = 4 };

/* step variants, lockstep.py:44 STEP_VARIANTS */
enum { FSMC_PLAIN = 0, FSMC_BUNDLED = 1, FSMC_AMORTIZED = 2 };

/* device log-density plugins (TargetModel, targets.py:45-60) */
enum {
  FSMC_T_GAUSS_DIAG = 1,     /* gaussian_target with diagonal factor            targets.py:74 */
  FSMC_T_GAUSS_DENSE = 2,    /* gaussian_target, dense L^-1 and precision       targets.py:100-114 */
  FSMC_T_GAUSS_EQUICORR = 3, /* gaussian_target whose covariance is a*I + b*11^T (closed form) */
  FSMC_T_MOG = 4,            /* correlated_mog_target                           targets.py:137 */
  FSMC_T_FUNNEL = 5,         /* Neal's funnel (BASELINE config 2) */
  FSMC_T_NANBAND = 6,        /* fault injection: std normal, `b` once x[0] > `a` */
  FSMC_T_LOGISTIC = 7,       /* -sum log(1+exp(-y*x)): GP-classification latent (f-space) */
  FSMC_T_FLAT = 8,           /* log density 0 */
  FSMC_T_LOGREG = 9,         /* Bayesian logistic regression, N(0, I) prior (BASELINE config 5) */
  FSMC_T_BOX = 10,           /* uniform on the box [a, b]^dim: 0 inside, -inf outside */
  FSMC_T_GP_HYPER = 11,      /* squared-exponential GP hyperparameters (sigma, tau, lam)  targets.py:191-265 */
  FSMC_T_EXTERNAL = 12       /* no device plugin: every evaluation comes from the caller's batched
                                evaluator (fsmc_advance / fsmc_init_deferred rounds); the
                                per-chain entry points report FSMC_E_TARGET */
};

/* Gaussian-prior split for the elliptical kernel (targets.py:37-42) */
enum { FSMC_PRIOR_NONE = 0, FSMC_PRIOR_IDENTITY = 1, FSMC_PRIOR_DENSE = 2 };

typedef struct fsmc_kernel {
  int32_t family;
  int32_t max_tries;            /* drmh: M */
  double proposal_scale;        /* drmh: proposal N(y, scale^2 I) */
  double step_size;             /* nuts: epsilon */
  int32_t max_depth;            /* nuts */
  int32_t split_body;           /* drmh: 1 = 4-way split proposal (drmh.py:106-156), 6 states */
  double divergence_threshold;  /* nuts */
  double slice_width;           /* slice: initial bracket width w */
  int32_t max_expansions;       /* slice: stepping-out budget */
  int32_t precision;            /* 0: fp64 arithmetic, the parity path (default); 1: the fp32
                                   throughput mode -- chain state and arithmetic in fp32, the
                                   draws still the reference's fp64 values (each rounded once),
                                   distributional parity only.  Compiled for the benchmark
                                   targets (DRMH on the MoG / funnel, d <= 10; NUTS on the
                                   equicorrelated Gaussian, d <= 128) in fsmc_run and the
                                   windowed DRMH runs; FSMC_ERR_UNSUPPORTED elsewhere. */
} fsmc_kernel;

typedef struct fsmc_target {
  int32_t kind;                 /* FSMC_T_* */
  int32_t dim;
  int32_t n_modes;              /* FSMC_T_MOG */
  int32_t prior_kind;           /* FSMC_PRIOR_* (elliptical kernel only) */
  double log_norm;              /* Gaussian / MoG normaliser, computed as the reference does */
  double a, b;                  /* EQUICORR/MOG: 1/a_perp, 1/(a+d*b); FUNNEL: a = v scale;
                                   NANBAND: a = threshold, b = value returned; BOX: bounds;
                                   GP_HYPER: a = jitter */
  int32_t full;                 /* set by the library: 1 = the full log density, 0 = the
                                   Gaussian-prior residual (elliptical kernel) */
  int32_t scratch;              /* extra shared-memory doubles per chain the plugin needs */
  double offsets[FSMC_MAX_MODES];  /* MOG mode offsets (mode k = offsets[k] * 1) */
  const double* mean;           /* [dim] or NULL (zero mean) */
  const double* diag;           /* [dim] GAUSS_DIAG: diagonal of L^-1 (dim 1: unused) */
  const double* diag2;          /* [dim] GAUSS_DIAG: diagonal of the precision */
  const double* mat_t;          /* [dim*dim] GAUSS_DENSE: (L^-1)^T row-major */
  const double* mat2_t;         /* [dim*dim] GAUSS_DENSE: precision^T row-major */
  const double* yvec;           /* [dim] LOGISTIC labels (+-1) */
  const double* prior_t;        /* [dim*dim] PRIOR_DENSE: L^T row-major (L lower-triangular) */
  const double* data;           /* LOGREG: [n_rows*dim] design matrix, row-major (labels in yvec);
                                   GP_HYPER: [n_rows*n_rows] squared distances (outputs in yvec) */
  int64_t n_rows;
} fsmc_target;

/* Per-chain structure-of-arrays state, allocated by the caller with the
 * sizes fsmc_state_layout() reports.  Replaces ChainBatch + the *Locals
 * records (lockstep.py:158-172, drmh.py:35, elliptical.py:32, nuts.py:64). */
typedef struct fsmc_state {
  int64_t m;                    /* chains in this state block */
  int64_t dim;
  int32_t n_vec;                /* vectors per chain */
  int32_t n_scal;               /* fp64 scalars per chain */
  double* vec;                  /* [m][n_vec][dim] */
  double* scal;                 /* [m][n_scal] */
  int64_t* ints;                /* [m][FSMC_NINT] */
  uint64_t seed;
  unsigned long long* err_key;  /* [1]; (tick << 24) | chain of the first failure, ~0 = none */
  uint32_t* work;               /* [FSMC_WORK_WORDS] device words owned by this state block: the
                                   chain queues and barrier words of the launches that run it
                                   (contents need not be initialised).  Two state blocks never
                                   share launch bookkeeping, so runs of different blocks may
                                   proceed concurrently on different streams and devices. */
} fsmc_state;

/* Per-sample observables of the CostLedger (lockstep.py:209-228). */
typedef struct fsmc_outputs {
  double* samples;              /* [n][m][dim] or NULL */
  int32_t* loop_counts;         /* [L][n][m]: executions of each loop state per sample */
  int32_t* sample_ticks;        /* [n][m] tick that finished each sample, or NULL */
  int64_t* loop_counts64;       /* [L][n][m] int64 (the reference's ledger type), used instead of
                                   loop_counts when non-NULL, so the counts go to the host as is */
} fsmc_outputs;

/* Host destinations of a run's outputs (pinned host memory), filled while the
 * run proceeds (fsmc_run_egress, fsmc_run_windowed_egress). */
typedef struct fsmc_egress {
  double* samples;              /* [n][m][dim] or NULL */
  int64_t* loop_counts;         /* [L][n][m] or NULL (needs outputs.loop_counts64) */
  int64_t* iter_counts;         /* [n][m] or NULL: a second copy of loop row `iter_loop`
                                   (the ledger's iter_counts when one loop state counts) */
  int32_t iter_loop;
  int32_t n_loops;              /* L */
} fsmc_egress;

/* indices into fsmc_state.ints (per chain) */
enum {
  FSMC_I_COUNTER = 0, FSMC_I_STREAM = 1, FSMC_I_STATE = 2, FSMC_I_TICK = 3, FSMC_I_COUNT = 4,
  FSMC_I_ERR_KIND = 5, FSMC_I_ERR_LABEL = 6, FSMC_I_ERR_TICK = 7, FSMC_I_ERR_ITER = 8,
  FSMC_I_SHARED = 9, FSMC_I_BLOCKS = 10 /* 6 slots */, FSMC_I_PEND = 16 /* 4 slots */,
  FSMC_I_FAMILY = 20 /* family-private slots 20..29 */,
  FSMC_I_DRAW0 = 30 /* counter at the end of init (draw-pattern origin) */,
  FSMC_I_RESUME = 31 /* batched mode: suspended-at-evaluation record */
};
/* error kinds in FSMC_I_ERR_KIND */
enum { FSMC_E_NONE = 0, FSMC_E_BLOCK = 1, FSMC_E_ZERO_START = 2, FSMC_E_GRAD = 3, FSMC_E_INIT = 4,
       FSMC_E_TARGET = 5 /* the plugin itself failed (TargetError, e.g. a kernel matrix not PD) */ };

int32_t fsmc_abi_version(void);
/* Kernels this library has launched so far (all entry points, all streams). */
int64_t fsmc_launch_count(void);
const char* fsmc_last_error(void);

/* Slots a chain of this kernel needs (vectors of `dim` doubles, scalars). */
fsmc_status fsmc_state_layout(const fsmc_kernel* k, int64_t dim, int32_t* n_vec,
                              int32_t* n_scal, int32_t* n_loop_states, int32_t* n_states);

/* Replaces prng.py:58-153 for bulk draws: out[i] = draw(seed, stream, counter+i).
 * kind 0: raw 64-bit words (uint64 out), 1: uniform, 2: standard normal. */
fsmc_status fsmc_prng_fill(uint64_t seed, uint64_t stream, uint64_t counter, int64_t count,
                           int32_t kind, void* out, void* stream_);

/* Replaces init_batch (lockstep.py:175-206): streams split(key(seed, parent_stream), .)
 * for chains chain_offset .. chain_offset+m-1, start x0 (+ jitter draws), and the
 * kernel's initial evaluation.  Failures land in the per-chain error slots and
 * err_key (tick 0). */
fsmc_status fsmc_init(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st,
                      uint64_t parent_stream, int64_t chain_offset, const double* x0,
                      double init_jitter, void* stream_);

/* Replaces run_fsm_batched's tick loop (lockstep.py:308-406).  Each chain
 * advances its own machine with no barrier.  mode 0: run each chain until it
 * holds n samples (finishing the tick) or reaches tick_limit; mode 1: run
 * each chain until tick_limit (the reference's surplus ticks).  `order` (host,
 * K entries) is the bundled executor order.  lanes = lanes per chain (0: auto). */
fsmc_status fsmc_run(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                     int32_t variant, const int32_t* order, int64_t tick_limit, int32_t mode,
                     const fsmc_outputs* out, int32_t lanes, void* stream_);

/* fsmc_run with output egress: `eg` (or NULL) names pinned host
 * destinations for the samples and the ledger's count matrices.  With parts > 1 the chains run
 * in `parts` contiguous parts launched back to back on two streams (each
 * part's blocks backfill the SMs the previous part's tail frees) and every
 * finished part's sample columns are copied to the host (one pitched copy)
 * on a device-owned egress stream while later parts still run; parts <= 1
 * copies after the run.  Results are identical to fsmc_run (chains are
 * independent).  The copies are ordered before later work on `stream`. */
fsmc_status fsmc_run_egress(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                            int32_t variant, const int32_t* order, int64_t tick_limit, int32_t mode,
                            const fsmc_outputs* out, int32_t lanes, int32_t parts, const fsmc_egress* eg,
                            void* stream);

/* Device -> host copy of `rows` rows of `width` bytes, both sides with row
 * pitch `pitch` (a chain range's columns of samples [n][m][dim]), ordered on
 * `stream`: the sample egress of the batched prior-transform rounds. */
fsmc_status fsmc_copy_to_host_2d(void* dst, const void* src, int64_t pitch, int64_t width, int64_t rows,
                                 void* stream);

/* Replaces run_standard_batched (lockstep.py:238-305): the lock-step
 * (vmap-style) baseline built from the same device blocks.  Every inner-loop
 * iteration ends at a grid-wide barrier, so a sample costs max over chains of
 * its loop count.  Chains beyond one co-resident wave run in successive
 * waves, each with its own barriers. */
fsmc_status fsmc_lockstep_run(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st,
                              int64_t n, const fsmc_outputs* out, int32_t lanes, void* stream_);

/* The lock-step baseline's barrier alone: the cooperative grid
 * fsmc_lockstep_run launches for this configuration (its first wave) runs
 * `iters` grid-wide "any chain active" barriers and nothing else.  Time it
 * with events on `stream`: the per-barrier cost the lock-step pays at every
 * while-loop test.  Uses st->work; the chain state is not touched. */
fsmc_status fsmc_lockstep_barrier_probe(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st,
                                        int64_t iters, int32_t lanes, void* stream);

/* fsmc_run for the DRMH kernels (drmh_kernel, split or not) with the draws
 * generated ahead of use.  Every DRMH proposal consumes dim normals then one
 * uniform (drmh.py:85-88), so a chain's draws from its current counter on are
 * known before it runs.  Rounds alternate two kernels until every chain is
 * done: a generator fills each unfinished chain's next `window` draws into
 * draws [m][window] (full occupancy, every lane busy), then the step kernel
 * runs each chain from its window until a tick could need more draws than
 * remain.  Samples, ledgers, ticks and errors are identical to fsmc_run's.
 * window >= dim + 1; `draws` holds m*window doubles plus 32 of slack (the step
 * kernel prefetches one proposal ahead).  Synchronises the stream every few
 * rounds (it reads the unfinished-chain count). */
fsmc_status fsmc_run_windowed(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                              int32_t variant, const int32_t* order, int64_t tick_limit, int32_t mode,
                              const fsmc_outputs* out, int64_t window, double* draws, int32_t lanes,
                              void* stream_);

/* fsmc_run_windowed with the chains in `parts` (1..16) contiguous parts, each
 * alternating its draw-generation and window kernels on its own stream
 * (internal streams, joined back to stream_ before returning), so the parts'
 * kernels fill each other's kernel tails and launch gaps.  parts = 0:
 * pipelined windows instead, one chain range with `draws` holding two windows
 * per chain ([2][m][window]); window r + 1 is generated while window r runs
 * (every window runs each unfinished chain exactly window / (dim + 1)
 * proposals; split-body DRMH is rejected).  Results are identical for any
 * parts.  FSMC_DRAW_BLOCKS_PER_SM / FSMC_WIN_BLOCKS_PER_SM (environment) cap
 * the two kernels' grids per SM so that several parts' kernels co-reside. */
fsmc_status fsmc_run_windowed_overlap(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                                      int32_t variant, const int32_t* order, int64_t tick_limit,
                                      int32_t mode, const fsmc_outputs* out, int64_t window, double* draws,
                                      int32_t lanes, int32_t parts, void* stream_);

/* fsmc_run_windowed_overlap with output egress: `eg` (or NULL) names pinned
 * host destinations for the samples and the count matrices.  Rows every chain has
 * finished are copied on a device-owned egress stream while the later rows
 * are still being sampled (the windowed run reads each part's lowest sample
 * count at its periodic progress checks), so the device-to-host transfer
 * overlaps the sampling instead of following it.  The copies are ordered
 * before any later work on `stream`: synchronise `stream` before reading. */
fsmc_status fsmc_run_windowed_egress(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                                     int32_t variant, const int32_t* order, int64_t tick_limit,
                                     int32_t mode, const fsmc_outputs* out, int64_t window, double* draws,
                                     int32_t lanes, int32_t parts, const fsmc_egress* eg, void* stream);

/* Replaces measure_block_costs' timing loop (lockstep.py:454-498): runs every
 * chain with the plain executor up to tick_limit like fsmc_run (mode 1) and
 * adds per-state clock64() cycles to cycles[16] (device, zeroed by the
 * caller): cycles[s-1] = state s's blocks excluding log-density evaluations,
 * cycles[8+s-1] = the evaluations requested in state s.  Chains run one per
 * warp where that layout is compiled, so divergent neighbours do not
 * inflate a chain's clock deltas. */
fsmc_status fsmc_profile_blocks(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st,
                                int64_t tick_limit, unsigned long long* cycles, void* stream_);

/* Batched plugin evaluation: lp[j] = log p(X[j]), grad[j] (if non-NULL) for
 * rows X[m][dim] (TargetModel.log_density / log_density_and_grad).  family /
 * lanes select the lane-group layout (0 = defaults) so a batched evaluation
 * reduces in the same order as the sampling kernel. */
fsmc_status fsmc_target_eval(const fsmc_target* t, const double* X, int64_t m, double* lp,
                             double* grad, int32_t family, int32_t lanes, void* stream_);

/* Batched-evaluation mode (the paper's amortized step, fsm.py:252-273, made
 * literal for dense targets).  Every chain advances, with no barrier, until
 * its next log-density request (or until it holds n samples / reaches
 * tick_limit, as in fsmc_run modes 0 / 1).  Each requesting chain appends
 * itself to a compact list: req_chain[k] = j and theta[k][:] = the point to
 * evaluate, k = atomicAdd(req_count, 1).  The caller evaluates every listed
 * point in ONE batched call (e.g. GEMMs across chains), writes lp[k] (and
 * grad[k][:] for gradient kernels), and calls fsmc_advance again: each chain
 * first consumes its result (lp, grad; the point itself is kept in the
 * chain's state, theta is write-only for the engine), then runs on to its
 * next request.  Repeat until *req_count == 0.  Samples, ticks and ledger
 * rows are identical to fsmc_run.
 * Buffers: theta/grad [m][dim], lp [m], req_chain [m] int32, req_count [1]. */
fsmc_status fsmc_advance(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                         int32_t variant, const int32_t* order, int64_t tick_limit, int32_t mode,
                         const fsmc_outputs* out, const double* lp, const double* grad,
                         double* theta, int32_t* req_chain, int32_t* req_count, int32_t lanes,
                         void* stream_);

/* Deferred init (targets evaluated only by a batched evaluator, e.g. the GP
 * hyperparameter target above 56 observations): fsmc_init_deferred is
 * fsmc_init (init_batch, lockstep.py:175-206: streams, jitter draws, x0)
 * without the starting point's evaluation; the caller evaluates every
 * chain's starting point x = vec[j][0][:] in one batched call and passes
 * the log densities lp [m] to fsmc_init_finish, which runs the Locals
 * constructor's checks (BlockFailure / TargetError records) as fsmc_init. */
fsmc_status fsmc_init_deferred(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st,
                               uint64_t parent_stream, int64_t chain_offset, const double* x0,
                               double init_jitter, void* stream_);
fsmc_status fsmc_init_finish(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, const double* lp,
                             void* stream_);

/* Lock-step baseline in batched-evaluation mode (run_standard_batched with an
 * evaluator; vmap semantics of the monolithic samplers, lockstep.py:238-305):
 * as fsmc_advance (plain executor, mode 0), but no chain starts sample s + 1
 * until every chain has finished sample s, and a chain waiting at that
 * barrier appends an idle request (its current point; the result is
 * discarded), as a vmapped while loop evaluates the whole batch each
 * iteration.  level [3] int64: set level[1] = 0 before the first call; each
 * call moves level[1] to level[0], leaves the minimum sample count over the
 * (non-failed) chains in level[1] and the number of real (non-idle) requests
 * in level[2].  A round whose requests are all idle (the slowest chains
 * finished their sample without a new request) needs no evaluation: vmap
 * would start the next iteration at once.  Repeat until *req_count == 0.
 * Samples and per-sample counts equal the FSM run's. */
fsmc_status fsmc_advance_lockstep(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                                  const fsmc_outputs* out, const double* lp, const double* grad,
                                  double* theta, int32_t* req_chain, int32_t* req_count, int64_t* level,
                                  int32_t lanes, void* stream_);

/* Batched prior transform (elliptical kernel, dense Gaussian prior): the
 * INIT block's nu = L eps (elliptical.py:73, prng.py:114-136 normal_vec with
 * chol) made one GEMM across chains.  Log densities are evaluated in place by
 * the plugin (as fsmc_run); every chain runs until its next INIT, draws eps,
 * and parks in its own row: nu[j][:] = eps, req_chain[j] = j, and
 * *req_count counts the parked chains.  The caller overwrites the rows with
 * L eps (e.g. nu = nu @ L^T over all m rows in one DGEMM, or
 * fsmc_prior_apply below; rows of chains that did not park are never read)
 * and calls again; each chain resumes INIT from its transformed row.  (A
 * compact row list would let a chain of the next round overwrite a row
 * before its previous owner has read it.)  Repeat until *req_count == 0.  Samples,
 * ticks and ledger rows are those of fsmc_run (bit-identical with
 * fsmc_prior_apply; within the GEMM's rounding otherwise). */
fsmc_status fsmc_advance_prior(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                               int32_t variant, const int32_t* order, int64_t tick_limit, int32_t mode,
                               const fsmc_outputs* out, double* nu, int32_t* req_chain,
                               int32_t* req_count, int32_t lanes, void* stream_);

/* fsmc_advance_prior over the chains [j_lo, j_hi) only, with its own chain
 * queue (part 0..7): the chains split in parts whose rounds run on their own
 * streams, so one part's GEMM overlaps another part's advance kernel.  nu and
 * req_chain point at the part's first row: chain j parks in row j - j_lo. */
fsmc_status fsmc_advance_prior_part(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                                    int32_t variant, const int32_t* order, int64_t tick_limit, int32_t mode,
                                    const fsmc_outputs* out, double* nu, int32_t* req_chain,
                                    int32_t* req_count, int32_t lanes, int64_t j_lo, int64_t j_hi,
                                    int32_t part, void* stream_);

/* Device math for tests: out[i] = f(x[i]) on the device, f = 0 CUDA's exp,
 * 1 exp_c (its constant-bank restatement), 2 gl_exp (glibc's exp restated),
 * 3 gl_log (glibc's log restated), 4 CUDA's log, 5 / 6 CUDA's sin / cos,
 * 7 / 8 the sin / cos halves of CUDA's sincos. */
fsmc_status fsmc_dmath_eval(int32_t fn, const double* x, int64_t n, double* out, void* stream_);

/* nu[r][:] = L nu[r][:] in place for r < k (L = the target's dense prior
 * factor), each row summed in the sampling kernel's order: the bit-exact
 * prior transform for fsmc_advance_prior. */
fsmc_status fsmc_prior_apply(const fsmc_target* t, double* nu, int64_t k, void* stream_);

/* nu[r] = L nu[r] for the k parked rows of a round (the ESS prior transform,
 * elliptical.py:73) on the fp64 tensor cores: a hand-written DMMA
 * (mma.sync m8n8k4 f64) triangular product out = eps L^T over 128 x 128
 * tiles, k slabs only up to each tile's diagonal; tmp [k][dim] is scratch.
 * Not bit-identical to the per-chain summation (tensor-core accumulation
 * order); the sampler's step counts match the reference's (tested). dim
 * must be even. */
fsmc_status fsmc_prior_trmm(const fsmc_target* t, double* nu, double* tmp, int64_t k, void* stream);
const char* fsmc_prior_trmm_last_error(void);

/* Logistic-regression evaluation epilogue over a tile of chains: given
 * Z [rows][N] = Theta X^T (fp32, from the contraction), labels y [N]:
 *   lp[r]   += sum_i y_i z_ri - log(1 + e^{z_ri})     (fp64 accumulation)
 *   R[r][i]  = y_i - sigmoid(z_ri)                    (fp32, in place over Z allowed)
 * One pass over Z; the caller adds -theta.theta/2 and forms G = R X - Theta. */
fsmc_status fsmc_logreg_epilogue(const float* Z, const float* y, int64_t rows, int64_t N,
                                 float* R, double* lp, void* stream_);

/* Fused tcgen05 evaluation of the logistic-regression target over k chains
 * (BASELINE config 5; d must be 256):  per 128-chain tile, S = Theta X^T and
 * G += (y - sigmoid(S)) X accumulate in TMEM (bf16 operands via TMA, fp32
 * accumulation), the logits never reach HBM.  theta [k][256] fp64 in,
 * lp [k] = theta.c - sum_i log(1+e^z_i) - theta.theta/2 and grad [k][256] =
 * c - sigmoid(Z) X - theta, with c = X^T y [256] (fp64, precomputed: the
 * label terms are linear in theta).  Scratch theta_bf16 holds
 * ceil(k/128)*128 x 256 bf16; x_bf16 [n_obs][256] and xt_bf16 [256][n_obs]
 * are the design matrix and its transpose in bf16 (n_obs a multiple of 8). */
fsmc_status fsmc_logreg_tc_eval(const double* theta, int64_t k, void* theta_bf16, const void* x_bf16,
                                const void* xt_bf16, const double* xty, int64_t n_obs, int64_t dim,
                                double* lp, double* grad, void* stream_);
/* The same with the operand type chosen: operand 0 = bf16 (as above), 1 =
 * fp16 (11-bit mantissa: theta is rounded ~8x more finely, the same tensor
 * issue rate); theta_h16 / x_h16 / xt_h16 then hold fp16. */
fsmc_status fsmc_logreg_tc_eval2(const double* theta, int64_t k, void* theta_h16, const void* x_h16,
                                 const void* xt_h16, const double* xty, int64_t n_obs, int64_t dim,
                                 double* lp, double* grad, int32_t operand, void* stream_);
const char* fsmc_logreg_tc_last_error(void);

/* Batched GP-hyperparameter marginal likelihood (targets.py:191-265) for k
 * requesting chains, theta [k][3] = (sigma, tau, lam): one CTA per chain, a
 * left-looking blocked Cholesky of K = tau^2 exp(-lam^2 D2) + (sigma^2 +
 * jitter) I formed on the fly from d2 [n][n], plus the forward solve and the
 * log determinant.  lp[j] = the marginal likelihood (residual != 0, the
 * elliptical kernel's residual) or the log density (+ the N(0, I) prior);
 * a matrix that is not positive definite yields the plugin's TargetError
 * payload.  work: work_slots x n x n doubles (one slot per concurrent CTA);
 * n <= fsmc_gp_lml_max_rows().
 * Errors: fsmc_gp_last_error(). */
size_t fsmc_gp_lml_smem_bytes(int64_t n);
int64_t fsmc_gp_lml_max_rows(void);   /* n limit of fsmc_gp_lml (shared memory) */
fsmc_status fsmc_gp_lml(const double* theta, int64_t k, const double* d2, const double* y, int64_t n,
                        double jitter, int32_t residual, double* work, int64_t work_slots, double* lp,
                        void* stream_);
/* The same with the gradient: grad [k][3] (or NULL for values only) gets the
 * reference's trace form (targets.py:238-254) from the factor the value pass
 * left in the workspace slot -- alpha = K^-1 y, W = L^-1 in the slot's upper
 * half, tr(K^-1), tr(K^-1 E) and tr(K^-1 (E o D2)) as sums of quadratic forms
 * in the rows of W -- minus theta unless `residual`.  No library call. */
fsmc_status fsmc_gp_lml_grad(const double* theta, int64_t k, const double* d2, const double* y, int64_t n,
                             double jitter, int32_t residual, double* work, int64_t work_slots, double* lp,
                             double* grad, void* stream_);
const char* fsmc_gp_last_error(void);

/* Cross-chain diagnostic partials for effective_sample_size / R-hat
 * (analysis.py:336-418).  samples [n][m][dim]; uses rows burn..n-1.
 *   chain_mean [m][dim] (computed when lag0 == 0), acov [32][dim] = sum over chains of
 *   the lag-(lag0+t) autocovariance (one tile of 32 lags per call;
 *   divided by the row count, analysis.py:344-347), chain_var [m][dim]
 *   (optional, lag0 == 0): each chain's population variance.  One coalesced
 *   pass over the samples per tile. */
fsmc_status fsmc_diag_partials(const double* samples, int64_t n, int64_t m, int64_t dim,
                               int64_t burn, int64_t lag0, int64_t n_lags, double* chain_mean,
                               double* acov, double* chain_var, void* stream_);

#ifdef __cplusplus
}
#endif
#endif
