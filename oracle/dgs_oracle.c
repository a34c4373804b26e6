/*
 * dgs_oracle.c -- CPU restatement of lsap::dgs_parallel (TEST INFRASTRUCTURE).
 * See dgs_oracle.h for the contract and the parity pinning.  Compiled with
 * -O2 -ffp-contract=off (no FMA contraction), matching the reference's
 * "no -mfma" rule (proj/src/CMakeLists.txt:13-17): every add/sub below rounds
 * exactly like the reference's scalar kernel.
 */
#include "dgs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <pthread.h>
#include <stdatomic.h>
#include <unistd.h>

#define GOLDEN 0x9E3779B97F4A7C15ull
#define TRACE_CAP 100000 /* parallel.cpp:15 */

/* rng.hpp:25-29 */
uint64_t orc_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* rng.hpp:11-22: next() adds the golden gamma to the state, then finalises;
 * draw k therefore depends only on (seed, k). */
uint64_t orc_draw(uint64_t seed, uint64_t k) { return orc_mix64(seed + (k + 1) * GOLDEN); }

/* rng.hpp:32-34 */
double orc_unit_double(uint64_t u) { return (double)u / 18446744073709551615.0; }

/* rng.hpp:37-46: Fisher-Yates, j = next() % (i+1) for i = n-1 .. 1 */
void orc_random_perm(int32_t n, uint64_t seed, int32_t* p) {
  for (int32_t i = 0; i < n; ++i) p[i] = i;
  uint64_t k = 0;
  for (int32_t i = n - 1; i > 0; --i) {
    int32_t j = (int32_t)(orc_draw(seed, k++) % (uint64_t)(i + 1));
    int32_t t = p[i];
    p[i] = p[j];
    p[j] = t;
  }
}

/* bench.cpp:200-208 */
uint64_t orc_derive_instance_seed(uint64_t base_seed, int32_t n, int32_t instance_index) {
  return orc_mix64(orc_mix64(base_seed ^ (uint64_t)n) ^ (uint64_t)instance_index);
}
uint64_t orc_derive_run_seed(uint64_t instance_seed, int32_t rep_index) {
  return orc_mix64(instance_seed ^ (uint64_t)(rep_index + 1));
}

void orc_gen_uniform_int(double* a, int32_t n, uint64_t seed, uint64_t modulus) {
  const uint64_t total = (uint64_t)n * (uint64_t)n;
  for (uint64_t k = 0; k < total; ++k) a[k] = (double)(orc_draw(seed, k) % modulus);
}

void orc_gen_unit_f32(double* a, int32_t n, uint64_t seed) {
  const uint64_t total = (uint64_t)n * (uint64_t)n;
  for (uint64_t k = 0; k < total; ++k) a[k] = (double)(float)orc_unit_double(orc_draw(seed, k));
}

void orc_gen_unit_scaled(double* a, int32_t n, uint64_t seed, double scale) {
  const uint64_t total = (uint64_t)n * (uint64_t)n;
  for (uint64_t k = 0; k < total; ++k) a[k] = orc_unit_double(orc_draw(seed, k)) * scale;
}

/* up[i] = 1 << (next() % 6) for each sender i, then per peer p
 * x = next() % 1024, y = next() % 1024; lat = 1 + (|dx| + |dy|) / 16;
 * a[i][j] = i == j ? 0 : up[i] * (256 - lat).  Integers in [128, 8160]. */
void orc_gen_p2p(double* a, int32_t n, uint64_t seed) {
  int64_t* up = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* x = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* y = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int32_t i = 0; i < n; ++i) up[i] = (int64_t)1 << (orc_draw(seed, (uint64_t)i) % 6);
  for (int32_t p = 0; p < n; ++p) {
    x[p] = (int64_t)(orc_draw(seed, (uint64_t)n + 2 * (uint64_t)p) % 1024);
    y[p] = (int64_t)(orc_draw(seed, (uint64_t)n + 2 * (uint64_t)p + 1) % 1024);
  }
  for (int32_t i = 0; i < n; ++i)
    for (int32_t j = 0; j < n; ++j) {
      int64_t dx = x[i] - x[j], dy = y[i] - y[j];
      if (dx < 0) dx = -dx;
      if (dy < 0) dy = -dy;
      const int64_t lat = 1 + (dx + dy) / 16;
      a[(size_t)i * n + j] = i == j ? 0.0 : (double)(up[i] * (256 - lat));
    }
  free(up);
  free(x);
  free(y);
}

/* geom.cpp:15-33: x then y per point, each unit_double * bound; benefit is
 * sqrt(dx*dx + dy*dy) with no contraction. */
void orc_gen_geom(double* a, int32_t n, uint64_t seed, double bound) {
  double* xs = (double*)malloc(sizeof(double) * (size_t)n);
  double* ys = (double*)malloc(sizeof(double) * (size_t)n);
  for (int32_t k = 0; k < n; ++k) {
    xs[k] = orc_unit_double(orc_draw(seed, 2 * (uint64_t)k)) * bound;
    ys[k] = orc_unit_double(orc_draw(seed, 2 * (uint64_t)k + 1)) * bound;
  }
  for (int32_t i = 0; i < n; ++i)
    for (int32_t j = 0; j < n; ++j) {
      const double dx = xs[i] - xs[j];
      const double dy = ys[i] - ys[j];
      const double sx = dx * dx;
      const double sy = dy * dy;
      a[(size_t)i * n + j] = sqrt(sx + sy);
    }
  free(xs);
  free(ys);
}

/* core.cpp:9-15 */
int orc_validate(const double* a, int32_t n) {
  if (n < 1) return 1;
  const size_t total = (size_t)n * (size_t)n;
  for (size_t k = 0; k < total; ++k)
    if (!isfinite(a[k])) return 3;
  return 0;
}

/* core.cpp:17-24: ordered sum over jobs */
double orc_objective(const double* a, int32_t n, const int32_t* sigma) {
  double sum = 0.0;
  for (int32_t j = 0; j < n; ++j) sum += a[(size_t)sigma[j] * n + j];
  return sum;
}

/* kernels_scalar.cpp:6-25 */
void orc_exchange_scan(const double* primary, const double* cross, const int32_t* map,
                       int64_t stride, const double* current, double self_benefit,
                       int32_t skip, int32_t n, double eps, double* delta_out,
                       int32_t* partner_out) {
  double best = 0.0;
  int32_t best_k = -1;
  for (int32_t k = 0; k < n; ++k) {
    if (k == skip) continue;
    const double d = (primary[k] - self_benefit) + (cross[(int64_t)map[k] * stride] - current[k]);
    if (best_k < 0 ? d > eps : d > best) {
      best = d;
      best_k = k;
    }
  }
  if (best_k < 0) {
    *delta_out = 0.0;
    *partner_out = -1;
  } else {
    *delta_out = best;
    *partner_out = best_k;
  }
}

/* ------------------------------------------------------------------------- */
/* Solver state: solver_state.hpp:33-149                                      */
/* ------------------------------------------------------------------------- */
typedef struct {
  int32_t n;
  const double* a;
  double* a_cols; /* build_columns, solver_state.hpp:67-76 */
  int32_t *sigma, *tau;
  double *agent_current, *job_current;
  double value;
  double *agent_delta, *job_delta;
  int32_t *agent_partner, *job_partner;
} state_t;

static double now_ns(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec * 1e9 + (double)ts.tv_nsec;
}

static int state_init(state_t* st, const double* a, int32_t n, const int32_t* sigma) {
  memset(st, 0, sizeof(*st));
  st->n = n;
  st->a = a;
  const size_t N = (size_t)n;
  st->a_cols = (double*)malloc(sizeof(double) * N * N);
  st->sigma = (int32_t*)malloc(sizeof(int32_t) * N);
  st->tau = (int32_t*)malloc(sizeof(int32_t) * N);
  st->agent_current = (double*)malloc(sizeof(double) * N);
  st->job_current = (double*)malloc(sizeof(double) * N);
  st->agent_delta = (double*)calloc(N, sizeof(double));
  st->job_delta = (double*)calloc(N, sizeof(double));
  st->agent_partner = (int32_t*)malloc(sizeof(int32_t) * N);
  st->job_partner = (int32_t*)malloc(sizeof(int32_t) * N);
  if (!st->a_cols || !st->sigma || !st->tau || !st->agent_current || !st->job_current ||
      !st->agent_delta || !st->job_delta || !st->agent_partner || !st->job_partner)
    return -1;
  for (int32_t j = 0; j < n; ++j) {
    st->sigma[j] = sigma[j];
    st->tau[sigma[j]] = j;
  }
  /* solver_state.hpp:46-63 */
  for (int32_t j = 0; j < n; ++j) {
    st->job_current[j] = a[(size_t)sigma[j] * N + j];
    st->agent_current[sigma[j]] = st->job_current[j];
  }
  for (int32_t k = 0; k < n; ++k) st->agent_partner[k] = st->job_partner[k] = -1;
  /* build_columns: a_cols[j*n+i] = a[i*n+j] */
  for (int32_t i = 0; i < n; ++i)
    for (int32_t j = 0; j < n; ++j) st->a_cols[(size_t)j * N + i] = a[(size_t)i * N + j];
  return 0;
}

static void state_free(state_t* st) {
  free(st->a_cols);
  free(st->sigma);
  free(st->tau);
  free(st->agent_current);
  free(st->job_current);
  free(st->agent_delta);
  free(st->job_delta);
  free(st->agent_partner);
  free(st->job_partner);
}

/* solver_state.hpp:78-84, 94-98 */
static void eval_agent(state_t* st, int32_t i, double eps) {
  const size_t N = (size_t)st->n;
  const int32_t j_old = st->tau[i];
  orc_exchange_scan(st->a + (size_t)i * N, st->a_cols + (size_t)j_old * N, st->sigma, 1,
                    st->job_current, st->agent_current[i], j_old, st->n, eps,
                    &st->agent_delta[i], &st->agent_partner[i]);
}

/* solver_state.hpp:86-92, 100-104 */
static void eval_job(state_t* st, int32_t j, double eps) {
  const size_t N = (size_t)st->n;
  const int32_t holder = st->sigma[j];
  orc_exchange_scan(st->a_cols + (size_t)j * N, st->a + (size_t)holder * N, st->tau, 1,
                    st->agent_current, st->job_current[j], holder, st->n, eps,
                    &st->job_delta[j], &st->job_partner[j]);
}

/* solver_state.hpp:106-113 */
static double agent_proposal_delta(const state_t* st, int32_t i, int32_t j_new) {
  const size_t N = (size_t)st->n;
  const int32_t j_old = st->tau[i];
  const int32_t d = st->sigma[j_new];
  const double* A = st->a;
  return (A[i * N + j_new] - A[i * N + j_old]) + (A[d * N + j_old] - A[d * N + j_new]);
}

/* solver_state.hpp:115-122 */
static double job_proposal_delta(const state_t* st, int32_t i_new, int32_t j) {
  const size_t N = (size_t)st->n;
  const int32_t h = st->sigma[j];
  const int32_t j_old = st->tau[i_new];
  const double* A = st->a;
  return (A[i_new * N + j] - A[h * N + j]) + (A[h * N + j_old] - A[i_new * N + j_old]);
}

/* solver_state.hpp:126-139 */
static void apply_exchange(state_t* st, int32_t i, int32_t j_new, double delta) {
  const size_t N = (size_t)st->n;
  const int32_t j_old = st->tau[i];
  const int32_t d = st->sigma[j_new];
  st->sigma[j_new] = i;
  st->sigma[j_old] = d;
  st->tau[i] = j_new;
  st->tau[d] = j_old;
  st->agent_current[i] = st->a[i * N + j_new];
  st->agent_current[d] = st->a[d * N + j_old];
  st->job_current[j_new] = st->agent_current[i];
  st->job_current[j_old] = st->agent_current[d];
  st->value += delta;
}

/* Minimal chunked parallel-for standing in for ThreadPool::for_each_chunk
 * (thread_pool.hpp:44-74): workers claim 64-record chunks; every record slot
 * is written by exactly one worker from a frozen state, so results never
 * depend on the worker count (parallel.hpp:79-80). */
static int g_threads = 1;

typedef struct {
  state_t* st;
  double eps, deadline_at;
  const int32_t* list; /* NULL: full sweep over 2n records */
  int32_t list_len, agent_side;
  atomic_long next;
  atomic_int stop;
} pf_t;

static void* pf_worker(void* arg) {
  pf_t* p = (pf_t*)arg;
  const int64_t n = p->st->n;
  const int64_t total = p->list ? p->list_len : 2 * n;
  for (;;) {
    const int64_t lo = atomic_fetch_add(&p->next, 64);
    if (lo >= total || atomic_load(&p->stop)) break;
    const int64_t hi = lo + 64 < total ? lo + 64 : total;
    for (int64_t t = lo; t < hi; ++t) {
      if (p->list) {
        if (p->agent_side)
          eval_agent(p->st, p->list[t], p->eps);
        else
          eval_job(p->st, p->list[t], p->eps);
      } else if (t < n) {
        eval_agent(p->st, (int32_t)t, p->eps);
      } else {
        eval_job(p->st, (int32_t)(t - n), p->eps);
      }
      if ((t & 15) == 0 && p->deadline_at > 0 && now_ns() >= p->deadline_at) {
        atomic_store(&p->stop, 1);
        return NULL;
      }
    }
  }
  return NULL;
}

static int run_pf(state_t* st, double eps, double deadline_at, const int32_t* list,
                  int32_t len, int agent_side) {
  pf_t p;
  p.st = st;
  p.eps = eps;
  p.deadline_at = deadline_at;
  p.list = list;
  p.list_len = len;
  p.agent_side = agent_side;
  atomic_init(&p.next, 0);
  atomic_init(&p.stop, 0);
  const int64_t total = list ? len : 2 * (int64_t)st->n;
  int nt = g_threads;
  if (total < 256) nt = 1;
  pthread_t th[256];
  if (nt > 256) nt = 256;
  for (int k = 1; k < nt; ++k) pthread_create(&th[k], NULL, pf_worker, &p);
  pf_worker(&p);
  for (int k = 1; k < nt; ++k) pthread_join(th[k], NULL);
  return !atomic_load(&p.stop);
}

/* parallel.cpp:80-98 (records t<n agents, t>=n jobs; all read a frozen state) */
static int eval_all(state_t* st, double eps, double deadline_at) {
  return run_pf(st, eps, deadline_at, NULL, 0, 1);
}

/* parallel.cpp:100-124 */
static int reeval_lists(state_t* st, double eps, double deadline_at, const int32_t* agents,
                        int32_t na, const int32_t* jobs, int32_t nj) {
  if (!run_pf(st, eps, deadline_at, agents, na, 1)) return 0;
  return run_pf(st, eps, deadline_at, jobs, nj, 0);
}

void orc_evaluate_all(const double* a, int32_t n, const int32_t* sigma, double eps,
                      double* agent_delta, int32_t* agent_partner, double* job_delta,
                      int32_t* job_partner) {
  state_t st;
  if (state_init(&st, a, n, sigma) != 0) {
    state_free(&st);
    return;
  }
  eval_all(&st, eps, -1.0);
  memcpy(agent_delta, st.agent_delta, sizeof(double) * (size_t)n);
  memcpy(agent_partner, st.agent_partner, sizeof(int32_t) * (size_t)n);
  memcpy(job_delta, st.job_delta, sizeof(double) * (size_t)n);
  memcpy(job_partner, st.job_partner, sizeof(int32_t) * (size_t)n);
  state_free(&st);
}

/* parallel.cpp:35-76 */
int32_t orc_check_conflicts(int32_t n, const double* agent_delta, const int32_t* agent_partner,
                            const double* job_delta, const int32_t* job_partner,
                            const int32_t* sigma, uint8_t* agent_accepted,
                            uint8_t* job_accepted, uint8_t* res, uint8_t* con,
                            int32_t* conflicted_jobs) {
  int32_t ncj = 0;
  memset(agent_accepted, 0, (size_t)n);
  memset(job_accepted, 0, (size_t)n);
  memset(res, 0, (size_t)n);
  memset(con, 0, (size_t)n);
  for (int32_t i = 0; i < n; ++i) {
    if (!(agent_delta[i] > 0.0) || agent_partner[i] < 0) continue;
    const int32_t displaced = sigma[agent_partner[i]];
    if (res[i] || res[displaced]) {
      con[i] = 1;
    } else {
      res[i] = 1;
      res[displaced] = 1;
      agent_accepted[i] = 1;
    }
  }
  for (int32_t j = 0; j < n; ++j) {
    if (!(job_delta[j] > 0.0) || job_partner[j] < 0) continue;
    const int32_t holder = sigma[j];
    const int32_t i_new = job_partner[j];
    if (res[holder] || res[i_new]) {
      con[holder] = 1;
      conflicted_jobs[ncj++] = j;
    } else {
      res[holder] = 1;
      res[i_new] = 1;
      job_accepted[j] = 1;
    }
  }
  return ncj;
}

/* parallel.cpp:182-229 */
int32_t orc_apply_parallel_switches(const double* a, int32_t n, int32_t* sigma, int32_t* tau,
                                    double* value, const double* agent_delta,
                                    const int32_t* agent_partner, const uint8_t* agent_active,
                                    const double* job_delta, const int32_t* job_partner,
                                    const uint8_t* job_active, const uint8_t* agent_accepted,
                                    const uint8_t* job_accepted, double eps,
                                    int32_t* out_agent, int32_t* out_new_job,
                                    int32_t* out_old_job, int32_t* out_displaced,
                                    double* out_delta) {
  const size_t N = (size_t)n;
  /* actual deltas are computed against the frozen input (core.hpp:25-39) */
  int32_t* s0 = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t* t0 = (int32_t*)malloc(sizeof(int32_t) * N);
  uint8_t* ta = (uint8_t*)calloc(N, 1);
  uint8_t* tj = (uint8_t*)calloc(N, 1);
  memcpy(s0, sigma, sizeof(int32_t) * N);
  memcpy(t0, tau, sizeof(int32_t) * N);
  int32_t count = 0;
  int bad = 0;
  for (int pass = 0; pass < 2 && !bad; ++pass) {
    for (int32_t k = 0; k < n && !bad; ++k) {
      const int agent_side = pass == 0;
      if (!(agent_side ? agent_accepted[k] : job_accepted[k])) continue;
      const double rd = agent_side ? agent_delta[k] : job_delta[k];
      const int32_t rp = agent_side ? agent_partner[k] : job_partner[k];
      const uint8_t act = agent_side ? agent_active[k] : job_active[k];
      if (!act || !(rd > 0.0) || rp < 0) continue;
      int32_t agent, j_new;
      double actual;
      if (agent_side) {
        agent = k;
        j_new = rp;
        const int32_t j_old = t0[agent], d = s0[j_new];
        actual = (a[agent * N + j_new] - a[agent * N + j_old]) + (a[d * N + j_old] - a[d * N + j_new]);
      } else {
        agent = rp;
        j_new = k;
        const int32_t h = s0[j_new], j_old = t0[agent];
        actual = (a[agent * N + j_new] - a[h * N + j_new]) + (a[h * N + j_old] - a[agent * N + j_old]);
      }
      if (!(actual > eps)) continue;
      /* commit lambda, parallel.cpp:195-209 (reads the evolving output) */
      const int32_t j_old = tau[agent];
      const int32_t displaced = sigma[j_new];
      if (ta[agent] || ta[displaced] || tj[j_new] || tj[j_old]) {
        bad = 1;
        break;
      }
      ta[agent] = ta[displaced] = 1;
      tj[j_new] = tj[j_old] = 1;
      sigma[j_new] = agent;
      sigma[j_old] = displaced;
      tau[agent] = j_new;
      tau[displaced] = j_old;
      *value += actual;
      out_agent[count] = agent;
      out_new_job[count] = j_new;
      out_old_job[count] = j_old;
      out_displaced[count] = displaced;
      out_delta[count] = actual;
      ++count;
    }
  }
  free(s0);
  free(t0);
  free(ta);
  free(tj);
  return bad ? -1 : count;
}

static void push_trace(int64_t* ts, double* tv, int64_t cap, int64_t* len, int64_t sw, double v,
                       int force) {
  if (!force && *len >= TRACE_CAP) return;
  if (ts && tv && *len < cap) {
    ts[*len] = sw;
    tv[*len] = v;
  }
  ++*len;
}

/* parallel.cpp:231-352 */
static int dgs_run(const double* a, int32_t n, uint64_t seed, const int32_t* init_sigma, double eps,
                   int policy, int64_t deadline_ns, int threads, int32_t* sigma_out, int32_t* tau_out,
                   orc_stats* stats, int64_t* trace_switch, double* trace_value, int64_t trace_cap,
                   int64_t* trace_len);

int orc_dgs_parallel(const double* a, int32_t n, uint64_t seed, double eps, int policy,
                     int64_t deadline_ns, int threads, int32_t* sigma_out, int32_t* tau_out,
                     orc_stats* stats, int64_t* trace_switch, double* trace_value,
                     int64_t trace_cap, int64_t* trace_len) {
  return dgs_run(a, n, seed, NULL, eps, policy, deadline_ns, threads, sigma_out, tau_out, stats, trace_switch,
                 trace_value, trace_cap, trace_len);
}

int orc_dgs_parallel_from(const double* a, int32_t n, const int32_t* init_sigma, double eps, int policy,
                          int64_t deadline_ns, int threads, int32_t* sigma_out, int32_t* tau_out,
                          orc_stats* stats, int64_t* trace_switch, double* trace_value,
                          int64_t trace_cap, int64_t* trace_len) {
  return dgs_run(a, n, 0, init_sigma, eps, policy, deadline_ns, threads, sigma_out, tau_out, stats, trace_switch,
                 trace_value, trace_cap, trace_len);
}

int64_t orc_greedy_assignment(const double* a, int32_t n, int32_t* sigma_out) {
  const size_t N = (size_t)n;
  uint8_t* taken = (uint8_t*)calloc(N, 1);
  int32_t* un = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t* claim = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t* winner = (int32_t*)malloc(sizeof(int32_t) * N);
  double* wval = (double*)malloc(sizeof(double) * N);
  int32_t cnt = n;
  int64_t rounds = 0;
  for (int32_t i = 0; i < n; ++i) un[i] = i;
  for (int32_t j = 0; j < n; ++j) winner[j] = -1;
  while (cnt > 0) {
    ++rounds;
    for (int32_t k = 0; k < cnt; ++k) {  /* ascending agents within the list order */
      const int32_t i = un[k];
      const double* row = a + (size_t)i * N;
      int32_t bj = -1;
      double bv = -INFINITY;
      for (int32_t j = 0; j < n; ++j)
        if (!taken[j] && (bj < 0 || row[j] > bv)) {
          bv = row[j];
          bj = j;
        }
      claim[i] = bj;
      if (winner[bj] < 0 || bv > wval[bj] || (bv == wval[bj] && i < winner[bj])) {
        winner[bj] = i;
        wval[bj] = bv;
      }
    }
    int32_t m = 0;
    for (int32_t k = 0; k < cnt; ++k) {
      const int32_t i = un[k], j = claim[i];
      if (winner[j] == i) {
        sigma_out[j] = i;
        taken[j] = 1;
      } else {
        un[m++] = i;
      }
    }
    for (int32_t j = 0; j < n; ++j) winner[j] = -1;
    cnt = m;
  }
  free(taken);
  free(un);
  free(claim);
  free(winner);
  free(wval);
  return rounds;
}

static int dgs_run(const double* a, int32_t n, uint64_t seed, const int32_t* init_sigma, double eps,
                   int policy, int64_t deadline_ns, int threads, int32_t* sigma_out, int32_t* tau_out,
                   orc_stats* stats, int64_t* trace_switch, double* trace_value, int64_t trace_cap,
                   int64_t* trace_len) {
  int rc = orc_validate(a, n);
  if (rc) return rc;
  if (!(eps >= 0.0)) return 2;
  g_threads = threads > 0 ? threads : (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (g_threads < 1) g_threads = 1;
  const double start = now_ns();
  const double deadline_at = deadline_ns >= 0 ? start + (double)deadline_ns : -1.0;
  const size_t N = (size_t)n;
  memset(stats, 0, sizeof(*stats));
  int64_t tlen = 0;

  /* initial_random: dgs.cpp:22-25 */
  int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * N);
  if (init_sigma)
    memcpy(perm, init_sigma, sizeof(int32_t) * N);
  else
    orc_random_perm(n, seed, perm);
  state_t st;
  if (state_init(&st, a, n, perm) != 0) {
    free(perm);
    state_free(&st);
    return 4;
  }
  free(perm);
  st.value = orc_objective(a, n, st.sigma);
  push_trace(trace_switch, trace_value, trace_cap, &tlen, 0, st.value, 0);

  uint8_t* acc_a = (uint8_t*)malloc(N);
  uint8_t* acc_j = (uint8_t*)malloc(N);
  uint8_t* res = (uint8_t*)malloc(N);
  uint8_t* con = (uint8_t*)malloc(N);
  uint8_t* touched_agent = (uint8_t*)calloc(N, 1);
  uint8_t* touched_job = (uint8_t*)calloc(N, 1);
  uint8_t* item_mark = (uint8_t*)calloc(N, 1);
  int32_t* cjobs = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t* conflicted = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t* b_agent = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t* b_new = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t* b_old = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t* b_disp = (int32_t*)malloc(sizeof(int32_t) * N);
  double* b_delta = (double*)malloc(sizeof(double) * N);
  int32_t* ra = (int32_t*)malloc(sizeof(int32_t) * 2 * N);
  int32_t* rj = (int32_t*)malloc(sizeof(int32_t) * 2 * N);

  int expired = deadline_at > 0 && now_ns() >= deadline_at;
  while (!expired) {
    ++stats->outer_iterations;
    const double f_start = st.value;
    if (!eval_all(&st, eps, deadline_at)) {
      expired = 1;
      break;
    }
    stats->agent_scans += n;
    stats->job_scans += n;
    stats->pair_items += n;

    for (;;) {
      /* argmax continue test, parallel.cpp:265-267 */
      int any = 0;
      for (int32_t k = 0; k < n && !any; ++k)
        any = st.agent_delta[k] > 0.0 || st.job_delta[k] > 0.0;
      if (!any) break;
      ++stats->inner_iterations;

      const int32_t ncj = orc_check_conflicts(n, st.agent_delta, st.agent_partner, st.job_delta,
                                              st.job_partner, st.sigma, acc_a, acc_j, res, con,
                                              cjobs);
      int32_t ncon = 0;
      for (int32_t i = 0; i < n; ++i)
        if (con[i]) conflicted[ncon++] = i;

      /* select, parallel.cpp:276-292 */
      int32_t nb = 0;
      for (int32_t i = 0; i < n; ++i) {
        if (!acc_a[i]) continue;
        const int32_t j_new = st.agent_partner[i];
        st.agent_delta[i] = 0.0;
        st.agent_partner[i] = -1;
        const double actual = agent_proposal_delta(&st, i, j_new);
        if (actual > eps) {
          b_agent[nb] = i;
          b_new[nb] = j_new;
          b_old[nb] = st.tau[i];
          b_disp[nb] = st.sigma[j_new];
          b_delta[nb] = actual;
          ++nb;
        }
      }
      for (int32_t j = 0; j < n; ++j) {
        if (!acc_j[j]) continue;
        const int32_t i_new = st.job_partner[j];
        st.job_delta[j] = 0.0;
        st.job_partner[j] = -1;
        const double actual = job_proposal_delta(&st, i_new, j);
        if (actual > eps) {
          b_agent[nb] = i_new;
          b_new[nb] = j;
          b_old[nb] = st.tau[i_new];
          b_disp[nb] = st.sigma[j];
          b_delta[nb] = actual;
          ++nb;
        }
      }
      /* disjointness, parallel.cpp:296-302 */
      for (int32_t b = 0; b < nb; ++b) {
        if (touched_agent[b_agent[b]] || touched_agent[b_disp[b]] || touched_job[b_new[b]] ||
            touched_job[b_old[b]]) {
          rc = 5;
          goto done;
        }
        touched_agent[b_agent[b]] = touched_agent[b_disp[b]] = 1;
        touched_job[b_new[b]] = touched_job[b_old[b]] = 1;
      }
      /* apply in batch order, parallel.cpp:306-310 */
      for (int32_t b = 0; b < nb; ++b) {
        apply_exchange(&st, b_agent[b], b_new[b], b_delta[b]);
        ++stats->switches_applied;
        push_trace(trace_switch, trace_value, trace_cap, &tlen, stats->switches_applied, st.value,
                   0);
      }
      /* re-eval lists, parallel.cpp:312-330 */
      int32_t na = 0, nj = 0;
      for (int32_t b = 0; b < nb; ++b) {
        ra[na++] = b_agent[b];
        ra[na++] = b_disp[b];
        rj[nj++] = b_new[b];
        rj[nj++] = b_old[b];
      }
      if (policy == 0) {
        for (int32_t c = 0; c < ncon; ++c)
          if (!touched_agent[conflicted[c]]) ra[na++] = conflicted[c];
        for (int32_t c = 0; c < ncj; ++c)
          if (!touched_job[cjobs[c]]) rj[nj++] = cjobs[c];
      }
      for (int32_t b = 0; b < nb; ++b) {
        touched_agent[b_agent[b]] = touched_agent[b_disp[b]] = 0;
        touched_job[b_new[b]] = touched_job[b_old[b]] = 0;
      }
      /* instrumentation: distinct (agent, tau[agent]) pairs covering both lists */
      int64_t items = 0;
      for (int32_t k = 0; k < na; ++k)
        if (!item_mark[ra[k]]) {
          item_mark[ra[k]] = 1;
          ++items;
        }
      for (int32_t k = 0; k < nj; ++k)
        if (!item_mark[st.sigma[rj[k]]]) {
          item_mark[st.sigma[rj[k]]] = 1;
          ++items;
        }
      for (int32_t k = 0; k < na; ++k) item_mark[ra[k]] = 0;
      for (int32_t k = 0; k < nj; ++k) item_mark[st.sigma[rj[k]]] = 0;
      stats->pair_items += items;
      stats->agent_scans += na;
      stats->job_scans += nj;

      if (!reeval_lists(&st, eps, deadline_at, ra, na, rj, nj)) {
        expired = 1;
        break;
      }
      if (deadline_at > 0 && now_ns() >= deadline_at) {
        expired = 1;
        break;
      }
    }
    if (expired) break;
    if (tlen >= TRACE_CAP)
      push_trace(trace_switch, trace_value, trace_cap, &tlen, stats->switches_applied, st.value, 1);
    if (st.value == f_start) break;
  }
  stats->terminated_by = expired ? 1 : 0;
  /* snapshot_assignment, solver_state.hpp:141-148 */
  stats->value = orc_objective(a, n, st.sigma);
  memcpy(sigma_out, st.sigma, sizeof(int32_t) * N);
  if (tau_out) memcpy(tau_out, st.tau, sizeof(int32_t) * N);
  if (trace_len) *trace_len = tlen;
  rc = 0;
done:
  stats->elapsed_ms = (now_ns() - start) / 1e6;
  free(acc_a);
  free(acc_j);
  free(res);
  free(con);
  free(touched_agent);
  free(touched_job);
  free(item_mark);
  free(cjobs);
  free(conflicted);
  free(b_agent);
  free(b_new);
  free(b_old);
  free(b_disp);
  free(b_delta);
  free(ra);
  free(rj);
  state_free(&st);
  return rc;
}

/* ==== auction.cpp: synchronous (Jacobi) auction ============================ */

/* net_scan contract (kernels_scalar.cpp:40-54): max over k != skip of
 * row[k] - prices[k], first k on ties. */
static double orc_net_scan(const double* row, const double* prices, int32_t n, int32_t skip,
                           int32_t* best_k_out) {
  int32_t best_k = -1;
  double best = 0.0;
  for (int32_t k = 0; k < n; ++k) {
    if (k == skip) continue;
    const double d = row[k] - prices[k];
    if (best_k < 0 || d > best) {
      best = d;
      best_k = k;
    }
  }
  if (best_k_out) *best_k_out = best_k;
  return best_k < 0 ? 0.0 : best;
}

/* run_phase (auction.cpp:33-80); returns 0 when the deadline fired */
static int orc_auction_phase(const double* a, int32_t n, double* prices, int32_t* owner,
                             int32_t* assigned, int32_t* unassigned, double eps,
                             int64_t expire_round, int64_t* checks, orc_auction_stats* S,
                             double* bid_value, int32_t* bid_winner) {
  while (*unassigned > 0) {
    if (expire_round >= 0 && (*checks)++ >= expire_round) return 0;
    S->rounds++;
    for (int32_t j = 0; j < n; ++j) {
      bid_value[j] = -INFINITY;
      bid_winner[j] = -1;
    }
    for (int32_t i = 0; i < n; ++i) {
      if (assigned[i] >= 0) continue;
      const double* row = a + (size_t)i * n;
      int32_t bk = -1;
      const double best = orc_net_scan(row, prices, n, -1, &bk);
      const double second = n > 1 ? orc_net_scan(row, prices, n, bk, NULL) : best;
      const double bid = prices[bk] + (best - second) + eps;
      S->bids++;
      if (bid > bid_value[bk]) {  /* ascending i: ties go to the smallest agent */
        bid_value[bk] = bid;
        bid_winner[bk] = i;
      }
    }
    for (int32_t j = 0; j < n; ++j) {
      const int32_t w = bid_winner[j];
      if (w < 0) continue;
      const int32_t prev = owner[j];
      if (prev >= 0) {
        assigned[prev] = -1;
        ++*unassigned;
      }
      owner[j] = w;
      assigned[w] = j;
      --*unassigned;
      prices[j] = bid_value[j];
      S->switches++;
    }
  }
  return 1;
}

int orc_auction_solve(const double* a, int32_t n, int has_eps, double eps, int scaling,
                      double scale_factor, int64_t expire_round, int32_t* sigma_out,
                      double* prices_out, orc_auction_stats* stats) {
  orc_auction_stats S;
  memset(&S, 0, sizeof(S));
  if (n < 1 || orc_validate(a, n) != 0) return 1;
  if (has_eps && !(eps > 0.0)) return 1;        /* "auction: epsilon must be > 0" */
  if (!(scale_factor > 1.0)) return 1;          /* "auction: scale_factor must be > 1" */
  const size_t N = (size_t)n;
  double lo = a[0], hi = a[0];
  for (size_t k = 1; k < N * N; ++k) {          /* std::minmax_element (auction.cpp:116) */
    if (a[k] < lo) lo = a[k];
    if (!(a[k] < hi)) hi = a[k];
  }
  const double range = hi - lo;
  const double eps_target = has_eps ? eps : (range > 0.0 ? range / (2.0 * n) : 1.0);
  S.epsilon = eps_target;
  double* prices = (double*)calloc(N, sizeof(double));
  int32_t* owner = (int32_t*)malloc(N * sizeof(int32_t));
  int32_t* assigned = (int32_t*)malloc(N * sizeof(int32_t));
  double* bid_value = (double*)malloc(N * sizeof(double));
  int32_t* bid_winner = (int32_t*)malloc(N * sizeof(int32_t));
  int32_t unassigned = n;
  int64_t checks = 0;
  int finished = 1;
  double e = scaling ? (range > 0.0 ? range / 2.0 : eps_target) : eps_target;
  if (e < eps_target) e = eps_target;
  for (;;) {
    for (int32_t x = 0; x < n; ++x) owner[x] = assigned[x] = -1;  /* clear_assignment */
    unassigned = n;
    finished = orc_auction_phase(a, n, prices, owner, assigned, &unassigned, e, expire_round, &checks,
                                 &S, bid_value, bid_winner);
    if (!scaling || !finished || e <= eps_target) break;
    e = e / scale_factor;
    if (e < eps_target) e = eps_target;
  }
  if (!finished) {  /* complete_greedily (auction.cpp:84-106) */
    for (int32_t i = 0; i < n; ++i) {
      if (assigned[i] >= 0) continue;
      int32_t bj = -1;
      double best = -INFINITY;
      for (int32_t j = 0; j < n; ++j) {  /* free jobs in ascending order */
        if (owner[j] >= 0) continue;
        const double v = a[(size_t)i * n + j];
        if (v > best) {
          best = v;
          bj = j;
        }
      }
      owner[bj] = i;
      assigned[i] = bj;
    }
    S.terminated_by = 1;
    S.completed_greedily = 1;
  }
  memcpy(sigma_out, owner, N * sizeof(int32_t));
  S.value = orc_objective(a, n, owner);
  if (prices_out) memcpy(prices_out, prices, N * sizeof(double));
  if (stats) *stats = S;
  free(prices);
  free(owner);
  free(assigned);
  free(bid_value);
  free(bid_winner);
  return 0;
}
