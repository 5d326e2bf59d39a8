/* fsm_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's multi-chain FSM sampling path
 * (arXiv 2503.17405 reference, /root/reference/pkg/src/fsm_mcmc).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it, and only as the checker or the CPU baseline.
 * The product path (paper_2503_17405_b200/) never calls into it.
 *
 * Parity pin: tests/golden/ fixtures frozen from the live reference by
 * tests/golden/make_golden.py; tests/test_oracle_golden.py checks this
 * restatement against every fixture.
 */
#ifndef FSM_ORACLE_H
#define FSM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_DRMH = 1, OR_ESS = 2, OR_NUTS = 3, OR_SLICE = 4 };
enum { OR_PLAIN = 0, OR_BUNDLED = 1, OR_AMORTIZED = 2 };

/* target kinds (log-density plugin restatements, targets.py) */
enum {
  OR_T_GAUSS = 1,     /* gaussian_target(mean, chol)      targets.py:74-122 */
  OR_T_MOG = 2,       /* correlated_mog_target             targets.py:137-188 */
  OR_T_FUNNEL = 3,    /* Neal's funnel (new; make_golden.py funnel_target) */
  OR_T_NANBAND = 4,   /* fault-injection standard normal (make_golden.py) */
  OR_T_LOGISTIC = 5,  /* -sum logaddexp(0, -y*x)  (GP-classification f-space) */
  OR_T_FLAT = 6,      /* log_density = 0 */
  OR_T_LOGREG = 7,    /* Bayesian logistic regression, N(0, I) prior (make_golden.py logreg_target) */
  OR_T_BOX = 8,       /* 0 on [p0, p1]^d, -inf outside (pkg/tests/test_kernels.py:205-212) */
  OR_T_GP = 9         /* GP hyperparameters (sigma, tau, lam), targets.py:191-265; p0 = jitter,
                         data = [n*n] squared distances, yvec = [n] outputs */
};

typedef struct or_target {
  int32_t kind;
  int32_t dim;
  int32_t n_modes;      /* MoG */
  int32_t residual;     /* GP: 1 = marginal likelihood only (the Gaussian-prior residual) */
  double log_norm;      /* gaussian / mog normaliser as the reference computes it */
  double p0, p1;        /* funnel: v_scale; nanband: threshold, value */
  const double* mean;   /* [d]           gaussian */
  const double* L_inv;  /* [d*d] row-major, gaussian */
  const double* prec;   /* [d*d] row-major, gaussian / mog */
  const double* modes;  /* [K*d] row-major, mog */
  const double* yvec;   /* [d] logistic labels */
  /* Gaussian-prior split (elliptical kernel): prior chol + residual target */
  const double* prior_chol;   /* [d*d] lower-triangular, or NULL */
  int32_t prior_identity;     /* np.array_equal(L, eye(d)) */
  int32_t pad1;
  const double* data;         /* [n_rows*d] row-major design matrix (logreg), labels in yvec */
  int64_t n_rows;
} or_target;

typedef struct or_kernel {
  int32_t family;
  int32_t max_tries;        /* drmh */
  double proposal_scale;    /* drmh */
  double step_size;         /* nuts */
  int32_t max_depth;        /* nuts */
  int32_t pad;
  double divergence_threshold;
  double slice_width;       /* slice: initial width w */
  int32_t max_expansions;   /* slice */
  int32_t pad2;
} or_kernel;

typedef struct or_error {
  int64_t chain;       /* -1 = no error */
  int64_t iteration;   /* sample index (driver's counts[j]) */
  int64_t tick;
  int32_t kind;        /* 1 BlockFailure(nan/+inf), 2 zero-density start, 3 non-finite grad, 4 init failure */
  int32_t label;       /* state label index (1..K), 0 = shared, -1 = init, 7 = "slice" */
} or_error;

typedef struct or_run_out {
  double* samples;        /* [n][m][d] */
  int64_t* loop_counts;   /* [L][n][m]  (loop states in ascending order) */
  int64_t* sample_ticks;  /* [n][m] */
  int64_t* block_counts;  /* [K] aggregate (reference semantics, incl. surplus) */
  int64_t tick_count;
  int64_t native_shared;
  int64_t budget_exceeded; /* 1 -> TickBudgetExceeded; min count in n_done */
  int64_t n_done;          /* rows valid in the ledger */
  int64_t* sample_counts;  /* [m] */
  or_error err;
} or_run_out;

uint64_t or_mix64(uint64_t x);
uint64_t or_bits(uint64_t seed, uint64_t stream, uint64_t counter);
double or_uniform(uint64_t seed, uint64_t stream, uint64_t counter);
double or_normal(uint64_t seed, uint64_t stream, uint64_t counter);
double or_ndtri(double y);
uint64_t or_split_stream(uint64_t parent_stream, uint64_t i);
void or_fill(uint64_t seed, uint64_t stream, uint64_t counter, int64_t count, int kind, double* out);

int or_loop_states(const or_kernel* k, int32_t* states);  /* returns L */
int or_n_states(const or_kernel* k);

/* target evaluation (for target-level parity tests) */
double or_log_density(const or_target* t, const double* x);
double or_log_density_grad(const or_target* t, const double* x, double* g);

int or_run_fsm(const or_kernel* k, const or_target* t, int64_t m, uint64_t seed,
               int64_t chain_offset, const double* x0, double init_jitter, int64_t n,
               int32_t variant, const int32_t* order, int64_t tick_chunk,
               int64_t tick_budget, int32_t surplus, int32_t nthreads, or_run_out* out);

int or_run_standard(const or_kernel* k, const or_target* t, int64_t m, uint64_t seed,
                    int64_t chain_offset, const double* x0, double init_jitter, int64_t n,
                    int32_t nthreads, or_run_out* out);

#ifdef __cplusplus
}
#endif
#endif
