/* fsm_oracle.c -- TEST INFRASTRUCTURE ONLY (see fsm_oracle.h).
 *
 * A scalar, chain-at-a-time CPU restatement of the reference's multi-chain
 * FSM sampling path.  Every function cites the reference file:line it
 * follows (paths relative to /root/reference/pkg/src/fsm_mcmc/).  Built with
 * -ffp-contract=off so that every elementwise fp64 operation rounds once,
 * as numpy does; transcendental functions are glibc's (the reference calls
 * Python's math module, i.e. the same libm), and ndtri is the Cephes
 * algorithm scipy 1.18 ships (polevl/p1evl with separate multiply and add).
 *
 * Chains are independent (prng.py:84-94, lockstep.py:187), so the driver runs
 * each chain to completion instead of interleaving ticks; the two-phase stop
 * rule below reproduces the reference's tick-major loop (lockstep.py:359-406)
 * exactly, including the chunked stop check and the surplus ticks that the
 * aggregate counters include.
 */
#include "fsm_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ PRNG */
/* prng.py:25-34 */
#define MIX_A 0xBF58476D1CE4E5B9ULL
#define MIX_B 0x94D049BB133111EBULL
#define GOLDEN 0x9E3779B97F4A7C15ULL
#define STREAM_SALT 0xC2B2AE3D27D4EB4FULL
#define COUNTER_SALT 0x165667B19E3779F9ULL
#define INV_2_53 (1.0 / 9007199254740992.0)

/* prng.py:50-55 */
uint64_t or_mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * MIX_A;
  x = (x ^ (x >> 27)) * MIX_B;
  return x ^ (x >> 31);
}

/* prng.py:58-81: mix(mix(mix(seed+G) ^ mix(stream+SS)) ^ mix(counter+CS)) */
uint64_t or_bits(uint64_t seed, uint64_t stream, uint64_t counter) {
  uint64_t h = or_mix64(seed + GOLDEN);
  h = or_mix64(h ^ or_mix64(stream + STREAM_SALT));
  return or_mix64(h ^ or_mix64(counter + COUNTER_SALT));
}

/* prng.py:84-94 */
uint64_t or_split_stream(uint64_t parent_stream, uint64_t i) {
  return or_mix64(parent_stream * GOLDEN + i + 1);
}

/* Cephes ndtri as scipy.special.ndtri (coefficients: Cephes ndtri.c) */
static double polevl(double x, const double* c, int n) {
  double a = c[0];
  for (int i = 1; i <= n; i++) a = a * x + c[i];
  return a;
}
static double p1evl(double x, const double* c, int n) {
  double a = x + c[0];
  for (int i = 1; i < n; i++) a = a * x + c[i];
  return a;
}
static const double P0[5] = {-5.99633501014107895267E1, 9.80010754185999661536E1,
                             -5.66762857469070293439E1, 1.39312609387279679503E1,
                             -1.23916583867381258016E0};
static const double Q0[8] = {1.95448858338141759834E0,  4.67627912898881538453E0,
                             8.63602421390890590575E1,  -2.25462687854119370527E2,
                             2.00260212380060660359E2,  -8.20372256168333339912E1,
                             1.59056225126211695515E1,  -1.18331621121330003142E0};
static const double P1[9] = {4.05544892305962419923E0,  3.15251094599893866154E1,
                             5.71628192246421288162E1,  4.40805073893200834700E1,
                             1.46849561928858024014E1,  2.18663306850790267539E0,
                             -1.40256079171354495875E-1, -3.50424626827848203418E-2,
                             -8.57456785154685413611E-4};
static const double Q1[8] = {1.57799883256466749731E1,  4.53907635128879210584E1,
                             4.13172038254672030440E1,  1.50425385692907503408E1,
                             2.50464946208309415979E0,  -1.42182922854787788574E-1,
                             -3.80806407691578277194E-2, -9.33259480895457427372E-4};
static const double P2[9] = {3.23774891776946035970E0,  6.91522889068984211695E0,
                             3.93881025292474443415E0,  1.33303460815807542389E0,
                             2.01485389549179081538E-1, 1.23716634817820021358E-2,
                             3.01581553508235416007E-4, 2.65806974686737550832E-6,
                             6.23974539184983293730E-9};
static const double Q2[8] = {6.02427039364742014255E0,  3.67983563856160859403E0,
                             1.37702099489081330271E0,  2.16236993594496635890E-1,
                             1.34204006088543189037E-2, 3.28014464682127739104E-4,
                             2.89247864745380683936E-6, 6.79019408009981274425E-9};

double or_ndtri(double y0) {
  const double s2pi = 2.50662827463100050242E0;
  const double expm2 = 0.13533528323661269189;
  if (y0 == 0.0) return -INFINITY;
  if (y0 == 1.0) return INFINITY;
  if (y0 < 0.0 || y0 > 1.0) return NAN;
  int code = 1;
  double y = y0;
  if (y > 1.0 - expm2) {
    y = 1.0 - y;
    code = 0;
  }
  if (y > expm2) {
    y = y - 0.5;
    double y2 = y * y;
    double x = y + y * (y2 * polevl(y2, P0, 4) / p1evl(y2, Q0, 8));
    return x * s2pi;
  }
  double x = sqrt(-2.0 * log(y));
  double x0 = x - log(x) / x;
  double z = 1.0 / x;
  double x1;
  if (x < 8.0)
    x1 = z * polevl(z, P1, 8) / p1evl(z, Q1, 8);
  else
    x1 = z * polevl(z, P2, 8) / p1evl(z, Q2, 8);
  x = x0 - x1;
  if (code) x = -x;
  return x;
}

/* prng.py:97-100 */
double or_uniform(uint64_t seed, uint64_t stream, uint64_t counter) {
  return (double)(or_bits(seed, stream, counter) >> 11) * INV_2_53;
}
/* prng.py:103-111: ndtri((b + 0.5) * 2^-53), the add rounds in fp64 */
double or_normal(uint64_t seed, uint64_t stream, uint64_t counter) {
  uint64_t b = or_bits(seed, stream, counter) >> 11;
  return or_ndtri(((double)b + 0.5) * INV_2_53);
}

void or_fill(uint64_t seed, uint64_t stream, uint64_t counter, int64_t count, int kind,
             double* out) {
  for (int64_t i = 0; i < count; i++) {
    uint64_t c = counter + (uint64_t)i;
    if (kind == 0)
      ((uint64_t*)out)[i] = or_bits(seed, stream, c);
    else if (kind == 1)
      out[i] = or_uniform(seed, stream, c);
    else
      out[i] = or_normal(seed, stream, c);
  }
}

typedef struct rng {
  uint64_t seed, stream, counter;
} rng;
static double rng_uniform(rng* r) { return or_uniform(r->seed, r->stream, r->counter++); }
/* prng.py:114-136 (identity factor; the chol product is done by the caller) */
static void rng_normal_vec(rng* r, int d, double* z) {
  for (int i = 0; i < d; i++) z[i] = or_normal(r->seed, r->stream, r->counter++);
}

/* --------------------------------------------------------------- targets */
#define LOG_2PI 1.8378770664093453
static double dot(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int i = 0; i < d; i++) s += a[i] * b[i];
  return s;
}

/* numpy logaddexp(x, y) (npymath npy_logaddexp) */
static double np_logaddexp(double x, double y) {
  if (x == y) return x + 0.693147180559945309417232121458176568;
  double tmp = x - y;
  if (tmp > 0) return x + log1p(exp(-tmp));
  if (tmp <= 0) return y + log1p(exp(tmp));
  return tmp;
}

/* targets.py:74-122 (gaussian), 137-188 (mog); funnel/nanband/logistic are
 * restatements of the closures in tests/golden/make_golden.py.  Returns lp;
 * writes the gradient when g != NULL. */
static double target_eval(const or_target* t, const double* x, double* g, double* scratch) {
  const int d = t->dim;
  switch (t->kind) {
    case OR_T_GP: { /* targets.py:191-265 with LAPACK's operation order (dpotf2, dpotrs) */
      const int n = (int)t->n_rows;
      const double sigma = x[0], tau = x[1], lam = x[2];
      double* K = (double*)malloc(sizeof(double) * (size_t)n * (3 * n + 2));
      double* Ex = K + (size_t)n * n;
      double* Ki = Ex + (size_t)n * n;
      double* al = Ki + (size_t)n * n;
      double* tmp = al + n;
      const double nl2 = -(lam * lam), t2 = tau * tau, dg = sigma * sigma + t->p0;
      for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) {
          Ex[i * n + j] = exp(nl2 * t->data[i * n + j]);
          K[i * n + j] = t2 * Ex[i * n + j] + (i == j ? dg : 0.0);
        }
      /* left-looking Cholesky (dpotf2, lower) */
      for (int j = 0; j < n; j++) {
        double ajj = K[j * n + j];
        for (int k = 0; k < j; k++) ajj -= K[j * n + k] * K[j * n + k];
        if (!(ajj > 0.0)) { free(K); return NAN; }
        ajj = sqrt(ajj);
        K[j * n + j] = ajj;
        const double r = 1.0 / ajj;
        for (int i = j + 1; i < n; i++) {
          double a = K[i * n + j];
          for (int k = 0; k < j; k++) a -= K[i * n + k] * K[j * n + k];
          K[i * n + j] = a * r;
        }
      }
      /* alpha = K^-1 y (dpotrs: L z = y column-oriented, L^T alpha = z dot-form) */
      for (int i = 0; i < n; i++) al[i] = t->yvec[i];
      for (int k = 0; k < n; k++) {
        al[k] /= K[k * n + k];
        for (int i = k + 1; i < n; i++) al[i] -= al[k] * K[i * n + k];
      }
      for (int i = n - 1; i >= 0; i--) {
        double tv = al[i];
        for (int k = i + 1; k < n; k++) tv -= K[k * n + i] * al[k];
        al[i] = tv / K[i * n + i];
      }
      double q = 0.0, ld = 0.0;
      for (int i = 0; i < n; i++) {
        q += t->yvec[i] * al[i];
        ld += log(K[i * n + i]);
      }
      const double logdet = 2.0 * ld;
      const double lml = -0.5 * q - 0.5 * logdet - 0.5 * n * LOG_2PI;
      if (g) {
        /* K^-1 = cho_solve(cf, eye) column by column, then A = alpha alpha^T - K^-1 */
        for (int c = 0; c < n; c++) {
          for (int i = 0; i < n; i++) tmp[i] = (i == c) ? 1.0 : 0.0;
          for (int k = 0; k < n; k++) {
            tmp[k] /= K[k * n + k];
            for (int i = k + 1; i < n; i++) tmp[i] -= tmp[k] * K[i * n + k];
          }
          for (int i = n - 1; i >= 0; i--) {
            double tv = tmp[i];
            for (int k = i + 1; k < n; k++) tv -= K[k * n + i] * tmp[k];
            tmp[i] = tv / K[i * n + i];
          }
          for (int i = 0; i < n; i++) Ki[i * n + c] = tmp[i];
        }
        double tr = 0.0, se = 0.0, sed = 0.0;
        for (int i = 0; i < n; i++)
          for (int j = 0; j < n; j++) {
            const double A = al[i] * al[j] - Ki[i * n + j];
            if (i == j) tr += A;
            se += A * Ex[i * n + j];
            sed += A * Ex[i * n + j] * t->data[i * n + j];
          }
        g[0] = sigma * tr - x[0];
        g[1] = tau * se - x[1];
        g[2] = -lam * tau * tau * sed - x[2];
      }
      free(K);
      if (t->residual) return lml;
      return lml - 0.5 * ((x[0] * x[0] + x[1] * x[1]) + x[2] * x[2]) - 1.5 * LOG_2PI;
    }
    case OR_T_BOX: { /* uniform on [p0, p1]^d */
      if (g)
        for (int k = 0; k < d; k++) g[k] = 0.0;
      for (int k = 0; k < d; k++)
        if (!(x[k] >= t->p0 && x[k] <= t->p1)) return -INFINITY;
      return 0.0;
    }
    case OR_T_FLAT:
      if (g) memset(g, 0, sizeof(double) * d);
      return 0.0;
    case OR_T_GAUSS: {
      if (d == 1) { /* targets.py:83-98 */
        double mu = t->mean[0];
        double inv_var = t->prec[0];
        double r = x[0] - mu;
        if (g) g[0] = -r * inv_var;
        return t->log_norm - 0.5 * r * r * inv_var;
      }
      double* r = scratch;
      double* w = scratch + d;
      for (int i = 0; i < d; i++) r[i] = x[i] - t->mean[i];
      for (int i = 0; i < d; i++) w[i] = dot(t->L_inv + (size_t)i * d, r, d);
      if (g)
        for (int i = 0; i < d; i++) g[i] = -dot(t->prec + (size_t)i * d, r, d);
      return t->log_norm - 0.5 * dot(w, w, d);
    }
    case OR_T_MOG: {
      const int K = t->n_modes;
      double* diffs = scratch;          /* K*d */
      double* logs = scratch + K * d;   /* K */
      double* tmp = logs + K;           /* d */
      for (int k = 0; k < K; k++) {
        double* df = diffs + (size_t)k * d;
        for (int i = 0; i < d; i++) df[i] = x[i] - t->modes[(size_t)k * d + i];
        double q = 0.0;
        for (int i = 0; i < d; i++) q += df[i] * dot(t->prec + (size_t)i * d, df, d);
        logs[k] = t->log_norm - 0.5 * q;
      }
      double mx = logs[0];
      for (int k = 1; k < K; k++)
        if (logs[k] > mx) mx = logs[k];
      double total = 0.0;
      double wk[64];
      for (int k = 0; k < K; k++) {
        wk[k] = exp(logs[k] - mx);
        total += wk[k];
      }
      double lp = mx + log(total);
      if (g) {
        for (int i = 0; i < d; i++) {
          double s = 0.0;
          for (int k = 0; k < K; k++) s += (wk[k] / total) * diffs[(size_t)k * d + i];
          tmp[i] = s;
        }
        for (int i = 0; i < d; i++) g[i] = -dot(t->prec + (size_t)i * d, tmp, d);
      }
      return lp;
    }
    case OR_T_FUNNEL: {
      const double s = t->p0;
      double v = x[0];
      double ev = exp(-v);
      double q = dot(x + 1, x + 1, d - 1);
      double lp = -0.5 * (v / s) * (v / s) - log(s) - 0.5 * LOG_2PI - 0.5 * q * ev -
                  0.5 * (d - 1) * v - 0.5 * (d - 1) * LOG_2PI;
      if (g) {
        g[0] = -v / (s * s) + 0.5 * q * ev - 0.5 * (d - 1);
        for (int i = 1; i < d; i++) g[i] = -x[i] * ev;
      }
      return lp;
    }
    case OR_T_NANBAND: {
      if (g) memset(g, 0, sizeof(double) * d);
      if (x[0] > t->p0) return t->p1;
      return -0.5 * dot(x, x, d) - 0.5 * d * LOG_2PI;
    }
    case OR_T_LOGREG: {
      /* sum(y z - logaddexp(0, z)) - theta.theta/2; grad X^T (y - sigmoid(z)) - theta */
      const int64_t N = t->n_rows;
      double s = 0.0;
      if (g)
        for (int k = 0; k < d; k++) g[k] = 0.0;
      for (int64_t i = 0; i < N; i++) {
        const double* xi = t->data + (size_t)i * d;
        double z = dot(xi, x, d);
        double yi = t->yvec[i];
        s += yi * z - np_logaddexp(0.0, z);
        if (g) {
          double r = yi - 1.0 / (1.0 + exp(-z));
          for (int k = 0; k < d; k++) g[k] += xi[k] * r;
        }
      }
      if (g)
        for (int k = 0; k < d; k++) g[k] = g[k] - x[k];
      return s - 0.5 * dot(x, x, d);
    }
    case OR_T_LOGISTIC: {
      double s = 0.0;
      for (int i = 0; i < d; i++) s += np_logaddexp(0.0, -t->yvec[i] * x[i]);
      if (g)
        for (int i = 0; i < d; i++) {
          double yi = t->yvec[i];
          g[i] = yi / (1.0 + exp(yi * x[i]));
        }
      return -s;
    }
  }
  return NAN;
}

double or_log_density(const or_target* t, const double* x) {
  double* scratch = (double*)malloc(sizeof(double) * (size_t)(t->dim * (t->n_modes + 3) + 64));
  double v = target_eval(t, x, NULL, scratch);
  free(scratch);
  return v;
}
double or_log_density_grad(const or_target* t, const double* x, double* g) {
  double* scratch = (double*)malloc(sizeof(double) * (size_t)(t->dim * (t->n_modes + 3) + 64));
  double v = target_eval(t, x, g, scratch);
  free(scratch);
  return v;
}

/* ----------------------------------------------------------- chain state */
enum { ERR_NONE = 0, ERR_BLOCK = 1, ERR_ZERO_START = 2, ERR_GRAD = 3, ERR_INIT = 4 };

typedef struct chain {
  const or_kernel* k;
  const or_target* t;
  int d;
  rng r;
  int state;          /* FSM state 1..K */
  int64_t tick;       /* executor calls so far */
  int64_t count;      /* samples completed */
  int64_t pend[3];    /* per-sample loop executions (loop states ascending) */
  int64_t blocks[6];
  int64_t shared;
  int err_kind, err_label;
  int64_t err_tick, err_iter;
  double* x;
  double* scratch;
  /* drmh  (drmh.py:35-52) */
  double* y;
  double* ytmp;
  double lp_x, lp_y, lp_best;
  int try_index, accepted, n_inner;
  /* ess   (elliptical.py:32-58) */
  double* nu;
  double* xprop;
  double lp_fx, logy, theta, tmin, tmax, lp_fprop;
  int needs_shared;
  /* nuts  (nuts.py:64-100) */
  double *xl, *pl, *gl, *xr, *pr, *gr, *cx, *cp, *cg, *nx, *np_, *ng, *sub_xprop, *ck_x, *ck_p;
  double h0, log_sum_w, sub_log_sum_w;
  int depth, stopped, diverged, direction, sub_stop, n_double, n_check;
  int64_t steps_todo, steps_done;
  /* slice (slice_sampling.py:29-47) */
  double s_logy, s_left, s_right, s_lp_left, s_lp_right, s_x1, s_lp_x1, s_lp_x;
  int s_n_expand, s_n_shrink, s_accepted, s_cap_hits;
} chain;

static int fail(chain* c, int kind, int label) {
  c->err_kind = kind;
  c->err_label = label;
  c->err_tick = c->tick;
  c->err_iter = c->count;
  return -1;
}

/* kernels/base.py:62-66: NaN / +inf are failures, -inf is legitimate */
static int bad_lp(double v) { return isnan(v) || v == INFINITY; }

/* ------------------------------------------------------------------ DRMH */
/* drmh.py:55-60 */
static int drmh_accept_stage(chain* c, double lp_cand, double u) {
  if (lp_cand >= c->lp_x) return 1;
  double m_rel = c->lp_best > -INFINITY ? exp(c->lp_best - c->lp_x) : 0.0;
  double num = exp(lp_cand - c->lp_x) - m_rel;
  return num > 0.0 && u * (1.0 - m_rel) < num;
}
static int drmh_block(chain* c, int s) {
  const int d = c->d;
  if (s == 1) { /* drmh.py:73-80 */
    c->n_inner = 0;
    c->try_index = 0;
    c->accepted = 0;
    c->lp_best = -INFINITY;
    memcpy(c->y, c->x, sizeof(double) * d);
    c->lp_y = c->lp_x;
  } else if (s == 2) { /* drmh.py:82-95 */
    c->n_inner++;
    c->try_index++;
    rng_normal_vec(&c->r, d, c->ytmp);
    for (int i = 0; i < d; i++) c->ytmp[i] = c->y[i] + c->k->proposal_scale * c->ytmp[i];
    double lp = target_eval(c->t, c->ytmp, NULL, c->scratch);
    if (bad_lp(lp)) return fail(c, ERR_BLOCK, 2);
    double u = rng_uniform(&c->r);
    if (drmh_accept_stage(c, lp, u))
      c->accepted = 1;
    else if (lp > c->lp_best)
      c->lp_best = lp;
    memcpy(c->y, c->ytmp, sizeof(double) * d);
    c->lp_y = lp;
  } else { /* drmh.py:97-101 */
    if (c->accepted) {
      memcpy(c->x, c->y, sizeof(double) * d);
      c->lp_x = c->lp_y;
    }
  }
  return 0;
}
/* drmh.py:103-104 + fsm.py:281-304 */
static int drmh_transition(chain* c, int s) {
  if (s == 3) return 1;
  return (!c->accepted && c->try_index < c->k->max_tries) ? 2 : 3;
}

/* ------------------------------------------------------------------- ESS */
#define TWO_PI (2.0 * 3.141592653589793)
/* elliptical.py:61-62 */
static int ess_shared(chain* c) {
  c->lp_fprop = target_eval(c->t, c->xprop, NULL, c->scratch);
  if (bad_lp(c->lp_fprop)) return fail(c, ERR_BLOCK, 0);
  return 0;
}
static void ess_propose(chain* c) {
  const int d = c->d;
  double cs = cos(c->theta), sn = sin(c->theta);
  for (int i = 0; i < d; i++) c->xprop[i] = c->x[i] * cs + c->nu[i] * sn;
}
static int ess_block(chain* c, int s) {
  const int d = c->d;
  if (s == 1) { /* elliptical.py:68-82 */
    c->n_inner = 0;
    rng_normal_vec(&c->r, d, c->ytmp);
    if (c->t->prior_identity) {
      memcpy(c->nu, c->ytmp, sizeof(double) * d);
    } else {
      for (int i = 0; i < d; i++) c->nu[i] = dot(c->t->prior_chol + (size_t)i * d, c->ytmp, d);
    }
    double u = rng_uniform(&c->r);
    c->logy = c->lp_fx + log(1.0 - u);
    u = rng_uniform(&c->r);
    c->theta = TWO_PI * u;
    c->tmin = c->theta - TWO_PI;
    c->tmax = c->theta;
    ess_propose(c);
    c->needs_shared = 1;
  } else if (s == 2) { /* elliptical.py:84-95 */
    c->n_inner++;
    if (c->theta < 0.0)
      c->tmin = c->theta;
    else
      c->tmax = c->theta;
    double u = rng_uniform(&c->r);
    c->theta = c->tmin + u * (c->tmax - c->tmin);
    ess_propose(c);
    c->needs_shared = 1;
  } else { /* elliptical.py:97-100 */
    memcpy(c->x, c->xprop, sizeof(double) * d);
    c->lp_fx = c->lp_fprop;
  }
  return 0;
}
static int ess_transition(chain* c, int s) {
  if (s == 3) return 1;
  return c->lp_fprop < c->logy ? 2 : 3; /* elliptical.py:102-103 */
}

/* ------------------------------------------------------------------ NUTS */
/* nuts.py:39-45 */
static double nuts_logaddexp(double a, double b) {
  if (a == -INFINITY) return b;
  if (b == -INFINITY) return a;
  double hi = a >= b ? a : b, lo = a >= b ? b : a;
  return hi + log1p(exp(lo - hi));
}
static int popcount64(uint64_t v) { return __builtin_popcountll(v); }
static int nuts_lp_grad(chain* c, const double* x, double* g, double* lp) {
  *lp = target_eval(c->t, x, g, c->scratch);
  return 0;
}
static int nuts_block(chain* c, int s) {
  const int d = c->d;
  const double eps = c->k->step_size;
  if (s == 1) { /* nuts.py:114-134 */
    c->n_inner = 0;
    c->n_double = 0;
    c->n_check = 0;
    rng_normal_vec(&c->r, d, c->pl);
    double lp;
    nuts_lp_grad(c, c->x, c->gl, &lp);
    if (bad_lp(lp)) return fail(c, ERR_BLOCK, 1);
    if (lp == -INFINITY) return fail(c, ERR_ZERO_START, 1);
    for (int i = 0; i < d; i++)
      if (!isfinite(c->gl[i])) return fail(c, ERR_GRAD, 1);
    c->h0 = -lp + 0.5 * dot(c->pl, c->pl, d);
    memcpy(c->xl, c->x, sizeof(double) * d);
    memcpy(c->xr, c->x, sizeof(double) * d);
    memcpy(c->pr, c->pl, sizeof(double) * d);
    memcpy(c->gr, c->gl, sizeof(double) * d);
    memcpy(c->xprop, c->x, sizeof(double) * d);
    c->log_sum_w = 0.0;
    c->depth = 0;
    c->stopped = 0;
    c->diverged = 0;
  } else if (s == 2) { /* nuts.py:139-151 */
    double u = rng_uniform(&c->r);
    c->direction = u < 0.5 ? 1 : -1;
    if (c->direction == 1) {
      memcpy(c->cx, c->xr, sizeof(double) * d);
      memcpy(c->cp, c->pr, sizeof(double) * d);
      memcpy(c->cg, c->gr, sizeof(double) * d);
    } else {
      memcpy(c->cx, c->xl, sizeof(double) * d);
      memcpy(c->cp, c->pl, sizeof(double) * d);
      memcpy(c->cg, c->gl, sizeof(double) * d);
    }
    c->steps_todo = (int64_t)1 << c->depth;
    c->steps_done = 0;
    c->sub_log_sum_w = -INFINITY;
    c->sub_stop = 0;
    c->n_double++;
  } else if (s == 3) { /* nuts.py:153-189 */
    c->n_inner++;
    double eff = eps * c->direction;
    double he = 0.5 * eff;
    for (int i = 0; i < d; i++) c->ytmp[i] = c->cp[i] + he * c->cg[i]; /* p_half */
    for (int i = 0; i < d; i++) c->nx[i] = c->cx[i] + eff * c->ytmp[i];
    double lp;
    nuts_lp_grad(c, c->nx, c->ng, &lp);
    if (bad_lp(lp)) return fail(c, ERR_BLOCK, 3);
    for (int i = 0; i < d; i++)
      if (!isfinite(c->ng[i])) return fail(c, ERR_GRAD, 3);
    for (int i = 0; i < d; i++) c->np_[i] = c->ytmp[i] + he * c->ng[i];
    memcpy(c->cx, c->nx, sizeof(double) * d);
    memcpy(c->cp, c->np_, sizeof(double) * d);
    memcpy(c->cg, c->ng, sizeof(double) * d);
    double delta = (-lp + 0.5 * dot(c->np_, c->np_, d)) - c->h0;
    int64_t leaf = c->steps_done;
    if (!isfinite(delta) || delta > c->k->divergence_threshold) {
      c->diverged = 1;
    } else {
      double log_w = -delta;
      double new_lsw = nuts_logaddexp(c->sub_log_sum_w, log_w);
      double u = rng_uniform(&c->r);
      if (u < exp(log_w - new_lsw)) memcpy(c->sub_xprop, c->nx, sizeof(double) * d);
      c->sub_log_sum_w = new_lsw;
      if (leaf % 2 == 0) { /* nuts.py:48-50 */
        int slot = popcount64((uint64_t)leaf >> 1);
        memcpy(c->ck_x + (size_t)slot * d, c->nx, sizeof(double) * d);
        memcpy(c->ck_p + (size_t)slot * d, c->np_, sizeof(double) * d);
      } else { /* nuts.py:53-61, 180-187 */
        uint64_t lf = (uint64_t)leaf;
        uint64_t v = lf ^ (lf + 1);
        int trailing_ones = 64 - __builtin_clzll(v) - 1;
        int hi = popcount64(lf >> 1);
        int lo = hi - trailing_ones + 1;
        for (int sl = lo; sl <= hi; sl++) {
          const double* ckx = c->ck_x + (size_t)sl * d;
          const double* ckp = c->ck_p + (size_t)sl * d;
          for (int i = 0; i < d; i++) c->ytmp[i] = c->nx[i] - ckx[i];
          if (c->direction * dot(c->ytmp, ckp, d) < 0.0 ||
              c->direction * dot(c->ytmp, c->np_, d) < 0.0) {
            c->sub_stop = 1;
            break;
          }
        }
      }
    }
    c->steps_done++;
  } else if (s == 4) { /* nuts.py:195-212 */
    c->n_check++;
    if (c->sub_stop || c->diverged) {
      c->stopped = 1;
      return 0;
    }
    double total = nuts_logaddexp(c->log_sum_w, c->sub_log_sum_w);
    double u = rng_uniform(&c->r);
    if (u < exp(c->sub_log_sum_w - total)) memcpy(c->xprop, c->sub_xprop, sizeof(double) * d);
    c->log_sum_w = total;
    if (c->direction == 1) {
      memcpy(c->xr, c->cx, sizeof(double) * d);
      memcpy(c->pr, c->cp, sizeof(double) * d);
      memcpy(c->gr, c->cg, sizeof(double) * d);
    } else {
      memcpy(c->xl, c->cx, sizeof(double) * d);
      memcpy(c->pl, c->cp, sizeof(double) * d);
      memcpy(c->gl, c->cg, sizeof(double) * d);
    }
    for (int i = 0; i < d; i++) c->ytmp[i] = c->xr[i] - c->xl[i];
    if (dot(c->ytmp, c->pl, d) < 0.0 || dot(c->ytmp, c->pr, d) < 0.0) c->stopped = 1;
    c->depth++;
  } else { /* nuts.py:214-216 */
    memcpy(c->x, c->xprop, sizeof(double) * d);
  }
  return 0;
}
/* fsm.py:348-388 composed with nuts.py:136-137, 191-193 */
static int nuts_outer(chain* c) {
  return !c->stopped && !c->diverged && c->depth < c->k->max_depth;
}
static int nuts_transition(chain* c, int s) {
  if (s == 1 || s == 4) return nuts_outer(c) ? 2 : 5;
  if (s == 2 || s == 3)
    return (c->steps_done < c->steps_todo && !c->sub_stop && !c->diverged) ? 3 : 4;
  return 1;
}


/* ----------------------------------------------------------------- slice */
/* kernels/slice_sampling.py:50-156; _logp failures carry the label "slice" (7) */
#define SLICE_LABEL 7
static int slice_logp(chain* c, double v, double* out) {
  double lp = target_eval(c->t, &v, NULL, c->scratch);
  if (bad_lp(lp)) return fail(c, ERR_BLOCK, SLICE_LABEL);
  *out = lp;
  return 0;
}
static int slice_expand_continue(chain* c) { /* slice_sampling.py:86-88 */
  return (c->s_lp_left > c->s_logy || c->s_lp_right > c->s_logy) &&
         c->s_n_expand < c->k->max_expansions;
}
static int slice_block(chain* c, int s) {
  const double w = c->k->slice_width;
  if (s == 1) { /* _init_expand, slice_sampling.py:62-74 */
    c->n_inner = 0;
    c->s_n_expand = 0;
    c->s_n_shrink = 0;
    c->s_accepted = 0;
    double u = rng_uniform(&c->r);
    c->s_logy = c->s_lp_x + log(1.0 - u);
    u = rng_uniform(&c->r);
    double x0 = c->x[0];
    c->s_left = x0 - w * u;
    c->s_right = c->s_left + w;
    if (slice_logp(c, c->s_left, &c->s_lp_left)) return -1;
    if (slice_logp(c, c->s_right, &c->s_lp_right)) return -1;
  } else if (s == 2) { /* _expand, slice_sampling.py:76-84 */
    c->n_inner++;
    c->s_n_expand++;
    if (c->s_lp_left > c->s_logy) {
      c->s_left -= w;
      if (slice_logp(c, c->s_left, &c->s_lp_left)) return -1;
    } else {
      c->s_right += w;
      if (slice_logp(c, c->s_right, &c->s_lp_right)) return -1;
    }
    if (c->s_n_expand == c->k->max_expansions &&
        (c->s_lp_left > c->s_logy || c->s_lp_right > c->s_logy))
      c->s_cap_hits++;
  } else if (s == 4) { /* _shrink, slice_sampling.py:93-104 */
    c->n_inner++;
    c->s_n_shrink++;
    double u = rng_uniform(&c->r);
    c->s_x1 = c->s_left + u * (c->s_right - c->s_left);
    if (slice_logp(c, c->s_x1, &c->s_lp_x1)) return -1;
    if (c->s_lp_x1 > c->s_logy)
      c->s_accepted = 1;
    else if (c->s_x1 < c->x[0])
      c->s_left = c->s_x1;
    else
      c->s_right = c->s_x1;
  } else if (s == 5) { /* _done, slice_sampling.py:109-112 */
    c->x[0] = c->s_x1;
    c->s_lp_x = c->s_lp_x1;
  } /* s == 3: INIT-S is empty_block */
  return 0;
}
/* fsm.py:323-331: compose_sequential of two single loops */
static int slice_transition(chain* c, int s) {
  if (s == 1 || s == 2) return slice_expand_continue(c) ? 2 : 3;
  if (s == 3 || s == 4) return c->s_accepted ? 5 : 4;
  return 1;
}

/* ---------------------------------------------------------- FSM glue */
int or_n_states(const or_kernel* k) { return (k->family == OR_NUTS || k->family == OR_SLICE) ? 5 : 3; }
int or_loop_states(const or_kernel* k, int32_t* st) {
  if (k->family == OR_NUTS) {
    st[0] = 2; st[1] = 3; st[2] = 4;
    return 3;
  }
  if (k->family == OR_SLICE) {
    st[0] = 2; st[1] = 4;
    return 2;
  }
  st[0] = 2;
  return 1;
}
static int run_block(chain* c, int s) {
  switch (c->k->family) {
    case OR_DRMH: return drmh_block(c, s);
    case OR_ESS: return ess_block(c, s);
    case OR_SLICE: return slice_block(c, s);
    default: return nuts_block(c, s);
  }
}
static int transition(chain* c, int s) {
  switch (c->k->family) {
    case OR_DRMH: return drmh_transition(c, s);
    case OR_ESS: return ess_transition(c, s);
    case OR_SLICE: return slice_transition(c, s);
    default: return nuts_transition(c, s);
  }
}
/* fsm.py:174-179 (_run_shared) */
static int run_shared(chain* c, int* did) {
  if (c->k->family == OR_ESS && c->needs_shared) {
    c->needs_shared = 0;
    *did = 1;
    return ess_shared(c);
  }
  return 0;
}

typedef struct run_ctx {
  const or_kernel* k;
  const or_target* t;
  or_target tcopy;   /* the caller's target with `residual` set for the kernel family */
  int64_t m, n, chain_offset;
  uint64_t seed;
  const double* x0;
  double init_jitter;
  int32_t variant;
  int32_t order[6];
  int K, L;
  int32_t loop_st[3];
  or_run_out* out;
  chain* chains;
} run_ctx;

static void chain_alloc(chain* c, const or_kernel* k, const or_target* t) {
  memset(c, 0, sizeof(*c));
  c->k = k;
  c->t = t;
  c->d = t->dim;
  const int d = t->dim;
  int nd = 32 + 2 * (k->family == OR_NUTS ? k->max_depth : 0);
  double* buf = (double*)calloc((size_t)nd * d + (size_t)d * (t->n_modes + 3) + 64, sizeof(double));
  double* p = buf;
  c->x = p; p += d;
  c->y = p; p += d;
  c->ytmp = p; p += d;
  c->nu = p; p += d;
  c->xprop = p; p += d;
  c->xl = p; p += d; c->pl = p; p += d; c->gl = p; p += d;
  c->xr = p; p += d; c->pr = p; p += d; c->gr = p; p += d;
  c->cx = p; p += d; c->cp = p; p += d; c->cg = p; p += d;
  c->nx = p; p += d; c->np_ = p; p += d; c->ng = p; p += d;
  c->sub_xprop = p; p += d;
  if (k->family == OR_NUTS) {
    c->ck_x = p; p += (size_t)k->max_depth * d;
    c->ck_p = p; p += (size_t)k->max_depth * d;
  }
  c->scratch = p;
}
static void chain_free(chain* c) { free(c->x); }

/* lockstep.py:175-206 + the *Locals constructors */
static int chain_init(run_ctx* ctx, chain* c, int64_t j) {
  const int d = ctx->t->dim;
  c->r.seed = ctx->seed;
  c->r.stream = or_split_stream(0, (uint64_t)(ctx->chain_offset + j));
  c->r.counter = 0;
  for (int i = 0; i < d; i++) c->x[i] = ctx->x0 ? ctx->x0[i] : 0.0;
  if (ctx->init_jitter > 0.0) { /* lockstep.py:195-198 */
    rng_normal_vec(&c->r, d, c->ytmp);
    for (int i = 0; i < d; i++) c->x[i] = c->x[i] + ctx->init_jitter * c->ytmp[i];
  }
  c->state = 1;
  c->err_kind = ERR_NONE;
  if (ctx->k->family == OR_DRMH) { /* drmh.py:38-52 */
    c->lp_x = target_eval(ctx->t, c->x, NULL, c->scratch);
    if (bad_lp(c->lp_x)) return fail(c, ERR_INIT, 1);
    if (c->lp_x == -INFINITY) return fail(c, ERR_ZERO_START, -1);
    memcpy(c->y, c->x, sizeof(double) * d);
    c->lp_y = c->lp_x;
    c->lp_best = -INFINITY;
  } else if (ctx->k->family == OR_ESS) { /* elliptical.py:41-58 */
    c->lp_fx = target_eval(ctx->t, c->x, NULL, c->scratch);
    if (bad_lp(c->lp_fx)) return fail(c, ERR_INIT, 1);
    c->logy = c->lp_fx;
    memcpy(c->xprop, c->x, sizeof(double) * d);
    c->lp_fprop = c->lp_fx;
  } else if (ctx->k->family == OR_SLICE) { /* SliceLocals.__init__, slice_sampling.py:33-47 */
    c->s_lp_x = target_eval(ctx->t, c->x, NULL, c->scratch);
    if (bad_lp(c->s_lp_x)) return fail(c, ERR_INIT, 1);
    if (c->s_lp_x == -INFINITY) return fail(c, ERR_ZERO_START, -1);
    c->s_logy = c->s_lp_x;
    c->s_left = c->s_right = c->x[0];
    c->s_lp_left = c->s_lp_right = c->s_lp_x;
    c->s_x1 = c->x[0];
    c->s_lp_x1 = c->s_lp_x;
  } else {
    memcpy(c->xprop, c->x, sizeof(double) * d);
    c->sub_log_sum_w = -INFINITY;
  }
  return 0;
}

static int is_loop_state(run_ctx* ctx, int s) {
  for (int i = 0; i < ctx->L; i++)
    if (ctx->loop_st[i] == s) return i;
  return -1;
}

/* one executor call (fsm.py:182-195 / 230-249, lockstep.py:366-406) */
static int chain_tick(run_ctx* ctx, chain* c, int64_t j) {
  const int K = ctx->K;
  const int64_t n = ctx->n, m = ctx->m;
  or_run_out* out = ctx->out;
  c->tick++;
  int executed[6], ne = 0;
  int did = 0;
  if (ctx->variant != OR_BUNDLED) {
    int s = c->state;
    if (run_block(c, s)) return -1;
    if (run_shared(c, &did)) return -1;
    c->state = transition(c, s);
    executed[ne++] = s;
  } else {
    for (int p = 0; p < K; p++) {
      int s = ctx->order[p];
      if (c->state == s) {
        if (run_block(c, s)) return -1;
        if (run_shared(c, &did)) return -1;
        c->state = transition(c, s);
        executed[ne++] = s;
      }
    }
  }
  if (did) c->shared++;
  for (int e = 0; e < ne; e++) {
    int s = executed[e];
    c->blocks[s - 1]++;
    int li = is_loop_state(ctx, s);
    if (li >= 0) c->pend[li]++;
    if (s == K) {
      if (c->count < n) {
        for (int l = 0; l < ctx->L; l++) out->loop_counts[((size_t)l * n + c->count) * m + j] = c->pend[l];
        out->sample_ticks[(size_t)c->count * m + j] = c->tick;
        /* only the final block writes x (fsm.py:25-27); the flagged value
         * read after the call is the finished sample (lockstep.py:405-406) */
        memcpy(out->samples + ((size_t)c->count * m + j) * c->d, c->x, sizeof(double) * c->d);
      }
      for (int l = 0; l < ctx->L; l++) c->pend[l] = 0;
      c->count++;
    }
  }
  return 0;
}

typedef struct job {
  run_ctx* ctx;
  int64_t lo, hi;
  int64_t limit; /* phase 1: tick limit; phase 2: run-to tick */
  int phase;
} job;

static void* fsm_worker(void* arg) {
  job* jb = (job*)arg;
  run_ctx* ctx = jb->ctx;
  for (int64_t j = jb->lo; j < jb->hi; j++) {
    chain* c = &ctx->chains[j];
    if (c->err_kind != ERR_NONE) continue;
    if (jb->phase == 1) {
      while (c->count < ctx->n && c->tick < jb->limit)
        if (chain_tick(ctx, c, j)) break;
    } else {
      while (c->tick < jb->limit)
        if (chain_tick(ctx, c, j)) break;
    }
  }
  return NULL;
}

static void run_jobs(run_ctx* ctx, int nthreads, int phase, int64_t limit,
                     void* (*fn)(void*)) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > ctx->m) nthreads = (int)ctx->m;
  pthread_t th[256];
  job jobs[256];
  if (nthreads > 256) nthreads = 256;
  for (int i = 0; i < nthreads; i++) {
    jobs[i].ctx = ctx;
    jobs[i].lo = ctx->m * i / nthreads;
    jobs[i].hi = ctx->m * (i + 1) / nthreads;
    jobs[i].limit = limit;
    jobs[i].phase = phase;
    if (nthreads == 1)
      fn(&jobs[i]);
    else
      pthread_create(&th[i], NULL, fn, &jobs[i]);
  }
  if (nthreads > 1)
    for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
}

static void ctx_setup(run_ctx* ctx, const or_kernel* k, const or_target* t, int64_t m,
                      uint64_t seed, int64_t off, const double* x0, double jit, int64_t n,
                      or_run_out* out) {
  memset(ctx, 0, sizeof(*ctx));
  ctx->k = k;
  ctx->tcopy = *t;
  ctx->tcopy.residual = k->family == OR_ESS; /* ESS evaluates the prior residual */
  ctx->t = &ctx->tcopy;
  t = ctx->t;
  ctx->m = m;
  ctx->n = n;
  ctx->seed = seed;
  ctx->chain_offset = off;
  ctx->x0 = x0;
  ctx->init_jitter = jit;
  ctx->K = or_n_states(k);
  ctx->L = or_loop_states(k, ctx->loop_st);
  ctx->out = out;
  ctx->chains = (chain*)calloc((size_t)m, sizeof(chain));
  for (int64_t j = 0; j < m; j++) chain_alloc(&ctx->chains[j], k, t);
  out->err.chain = -1;
  out->budget_exceeded = 0;
}
static void ctx_free(run_ctx* ctx) {
  for (int64_t j = 0; j < ctx->m; j++) chain_free(&ctx->chains[j]);
  free(ctx->chains);
}

/* init_batch failures raise before any run (lockstep.py:175-206) */
static int init_all(run_ctx* ctx) {
  for (int64_t j = 0; j < ctx->m; j++) {
    chain* c = &ctx->chains[j];
    if (chain_init(ctx, c, j)) {
      ctx->out->err.chain = j;
      ctx->out->err.iteration = -1;
      ctx->out->err.tick = 0;
      ctx->out->err.kind = c->err_kind;
      ctx->out->err.label = c->err_label;
      return -1;
    }
  }
  return 0;
}

/* lockstep.py:308-416 */
int or_run_fsm(const or_kernel* k, const or_target* t, int64_t m, uint64_t seed,
               int64_t chain_offset, const double* x0, double init_jitter, int64_t n,
               int32_t variant, const int32_t* order, int64_t tick_chunk,
               int64_t tick_budget, int32_t surplus, int32_t nthreads, or_run_out* out) {
  run_ctx ctx;
  ctx_setup(&ctx, k, t, m, seed, chain_offset, x0, init_jitter, n, out);
  ctx.variant = variant;
  for (int i = 0; i < ctx.K; i++) ctx.order[i] = order ? order[i] : (i == 0 ? ctx.K : i);
  if (init_all(&ctx)) {
    ctx_free(&ctx);
    return 1;
  }
  /* the loop runs chunks while ticks + chunk <= budget (lockstep.py:360) */
  int64_t limit = tick_budget > 0 ? (tick_budget / tick_chunk) * tick_chunk : INT64_MAX;
  run_jobs(&ctx, nthreads, 1, limit, fsm_worker);
  /* global stop: first chunk boundary at which every chain holds n samples */
  int64_t tmax = 0, min_count = INT64_MAX;
  int all_done = 1;
  for (int64_t j = 0; j < m; j++) {
    chain* c = &ctx.chains[j];
    if (c->count < n) all_done = 0;
    if (c->err_kind == ERR_NONE && c->count >= n && c->tick > tmax) tmax = c->tick;
  }
  int64_t first_err = INT64_MAX;
  for (int64_t j = 0; j < m; j++)
    if (ctx.chains[j].err_kind != ERR_NONE && ctx.chains[j].err_tick < first_err)
      first_err = ctx.chains[j].err_tick;
  int64_t tick_count;
  if (all_done)
    tick_count = ((tmax + tick_chunk - 1) / tick_chunk) * tick_chunk;
  else
    tick_count = limit; /* a budget overrun (or an error) ends the run earlier */
  /* surplus ticks: finished chains keep stepping until the global stop or
   * the first failure, whichever comes first (lockstep.py:617-664) */
  int64_t run_to = tick_count < first_err ? tick_count : first_err;
  /* surplus = 0 (the CPU baseline beside the device's surplus=False runs):
   * the surplus ticks are skipped; only the aggregate counters change, and
   * ticks up to a failure still run so it is reported as the reference does */
  if (!surplus && first_err == INT64_MAX) run_to = INT64_MAX;
  if (run_to != INT64_MAX) run_jobs(&ctx, nthreads, 2, run_to, fsm_worker);
  /* first failure in (tick, chain) order (lockstep.py:648-649) */
  int64_t best_tick = INT64_MAX, best_j = -1;
  for (int64_t j = 0; j < m; j++) {
    chain* c = &ctx.chains[j];
    if (c->err_kind != ERR_NONE && c->err_tick < best_tick) {
      best_tick = c->err_tick;
      best_j = j;
    }
  }
  if (best_j >= 0 && best_tick <= tick_count) {
    chain* c = &ctx.chains[best_j];
    out->err.chain = best_j;
    out->err.iteration = c->err_iter;
    out->err.tick = c->err_tick;
    out->err.kind = c->err_kind;
    out->err.label = c->err_label;
    ctx_free(&ctx);
    return 1;
  }
  for (int64_t j = 0; j < m; j++) {
    chain* c = &ctx.chains[j];
    if (c->count < min_count) min_count = c->count;
    for (int s = 0; s < ctx.K; s++) out->block_counts[s] += c->blocks[s];
    out->native_shared += c->shared;
    if (out->sample_counts) out->sample_counts[j] = c->count;
  }
  out->tick_count = tick_count;
  out->n_done = min_count < n ? min_count : n;
  out->budget_exceeded = min_count < n;
  ctx_free(&ctx);
  return out->budget_exceeded ? 2 : 0;
}

/* ------------------------------------------------------- standard driver */
/* lockstep.py:238-305 with each kernel's monolithic sampler
 * (drmh.py:163-169, elliptical.py:122-132, nuts.py:237-248). */
static int monolithic(run_ctx* ctx, chain* c, int64_t* execs) {
  const int fam = ctx->k->family;
  int did = 0;
  if (fam == OR_DRMH) {
    drmh_block(c, 1);
    while (!c->accepted && c->try_index < c->k->max_tries)
      if (drmh_block(c, 2)) return -1;
    drmh_block(c, 3);
    execs[0] = c->n_inner;
  } else if (fam == OR_ESS) {
    ess_block(c, 1);
    if (run_shared(c, &did)) return -1;
    int n_shrink = 0;
    while (c->lp_fprop < c->logy) {
      ess_block(c, 2);
      n_shrink++;
      if (run_shared(c, &did)) return -1;
    }
    ess_block(c, 3);
    execs[0] = n_shrink;
  } else if (fam == OR_SLICE) { /* slice_sampling.py:135-143 */
    if (slice_block(c, 1)) return -1;
    while (slice_expand_continue(c))
      if (slice_block(c, 2)) return -1;
    while (!c->s_accepted)
      if (slice_block(c, 4)) return -1;
    slice_block(c, 5);
    execs[0] = c->s_n_expand;
    execs[1] = c->s_n_shrink;
  } else {
    if (nuts_block(c, 1)) return -1;
    while (nuts_outer(c)) {
      nuts_block(c, 2);
      while (c->steps_done < c->steps_todo && !c->sub_stop && !c->diverged)
        if (nuts_block(c, 3)) return -1;
      nuts_block(c, 4);
    }
    nuts_block(c, 5);
    execs[0] = c->n_double;
    execs[1] = c->n_inner;
    execs[2] = c->n_check;
  }
  return 0;
}

static void* std_worker(void* arg) {
  job* jb = (job*)arg;
  run_ctx* ctx = jb->ctx;
  or_run_out* out = ctx->out;
  const int64_t n = ctx->n, m = ctx->m;
  for (int64_t j = jb->lo; j < jb->hi; j++) {
    chain* c = &ctx->chains[j];
    for (int64_t i = 0; i < n; i++) {
      int64_t execs[3] = {0, 0, 0};
      c->count = i;
      if (monolithic(ctx, c, execs)) break;
      memcpy(out->samples + ((size_t)i * m + j) * c->d, c->x, sizeof(double) * c->d);
      for (int l = 0; l < ctx->L; l++) {
        out->loop_counts[((size_t)l * n + i) * m + j] = execs[l];
        c->blocks[ctx->loop_st[l] - 1] += execs[l];
      }
    }
  }
  return NULL;
}

int or_run_standard(const or_kernel* k, const or_target* t, int64_t m, uint64_t seed,
                    int64_t chain_offset, const double* x0, double init_jitter, int64_t n,
                    int32_t nthreads, or_run_out* out) {
  run_ctx ctx;
  ctx_setup(&ctx, k, t, m, seed, chain_offset, x0, init_jitter, n, out);
  if (init_all(&ctx)) {
    ctx_free(&ctx);
    return 1;
  }
  run_jobs(&ctx, nthreads, 1, 0, std_worker);
  int64_t best_i = INT64_MAX, best_j = -1;
  for (int64_t j = 0; j < m; j++) {
    chain* c = &ctx.chains[j];
    if (c->err_kind != ERR_NONE && c->err_iter < best_i) {
      best_i = c->err_iter;
      best_j = j;
    }
  }
  if (best_j >= 0) {
    chain* c = &ctx.chains[best_j];
    out->err.chain = best_j;
    out->err.iteration = c->err_iter;
    out->err.tick = -1;
    out->err.kind = c->err_kind;
    out->err.label = c->err_label;
    ctx_free(&ctx);
    return 1;
  }
  for (int64_t j = 0; j < m; j++) {
    chain* c = &ctx.chains[j];
    for (int s = 0; s < ctx.K; s++) out->block_counts[s] += c->blocks[s];
  }
  /* non-loop blocks run once per sample (lockstep.py:299-301) */
  for (int s = 1; s <= ctx.K; s++)
    if (is_loop_state(&ctx, s) < 0) out->block_counts[s - 1] += n * m;
  out->tick_count = n;
  out->n_done = n;
  ctx_free(&ctx);
  return 0;
}
