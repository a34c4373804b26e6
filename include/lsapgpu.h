/*
 * lsapgpu.h -- C-ABI of the B200-native conflict-aware parallel DGS solver.
 *
 * This is the drop-in boundary for the reference's solver entry point and its
 * step APIs (paths relative to /root/reference/proj):
 *
 *   lsapgpu_solve                   replaces lsap::dgs_parallel
 *                                   (include/lsap/parallel.hpp:80, src/parallel.cpp:231-352)
 *   lsapgpu_evaluate_all            replaces lsap::evaluate_all_parallel
 *                                   (parallel.hpp:60-61, parallel.cpp:134-156)
 *   lsapgpu_check_conflicts         replaces lsap::check_conflicts
 *                                   (parallel.hpp:65, parallel.cpp:158-180)
 *   lsapgpu_apply_parallel_switches replaces lsap::apply_parallel_switches
 *                                   (parallel.hpp:71-74, parallel.cpp:182-229)
 *   lsapgpu_set_matrix              replaces Instance::validate + SolverState::build_columns
 *                                   (src/core.cpp:9-15, src/solver_state.hpp:67-76)
 *   lsapgpu_auction_solve           replaces lsap::auction_solve, the paper's comparator
 *                                   (include/lsap/baselines.hpp:12-36, src/auction.cpp:110-153)
 *   lsapgpu_random_perm / lsapgpu_objective
 *                                   host helpers equal to lsap::random_perm (include/lsap/rng.hpp:37-46)
 *                                   and lsap::objective (src/core.cpp:17-24)
 *
 * Plain pointers and sizes only.  Host buffers stay owned by the caller; the
 * context owns all device memory, streams and the cached CUDA graph.  One
 * context per host thread; contexts on different devices may run
 * concurrently.  Every call returns LSAPGPU_OK or an error code, with the
 * message (worded like the reference's lsap::Error, types.hpp:17-20) available
 * from lsapgpu_last_error().  There is no CPU fallback: without a usable
 * sm_100 device lsapgpu_create fails.
 */
#ifndef LSAPGPU_H
#define LSAPGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSAPGPU_OK 0
#define LSAPGPU_ERR_INVALID 1  /* lsap::Error: invalid instance / config / arguments */
#define LSAPGPU_ERR_CUDA 2     /* CUDA runtime failure (no device, OOM, launch error) */
#define LSAPGPU_ERR_INTERNAL 3 /* "internal: conflict check admitted overlapping exchanges" */
#define LSAPGPU_ERR_STATE 4    /* call order (e.g. solve before set_matrix) */

/* element type of a caller's matrix buffer */
#define LSAPGPU_F64 0
#define LSAPGPU_F32 1
#define LSAPGPU_I32 2
#define LSAPGPU_I16 3

/* device storage chosen by set_matrix (narrowest lossless) */
#define LSAPGPU_STORE_I16 0
#define LSAPGPU_STORE_I32 1
#define LSAPGPU_STORE_F32 2
#define LSAPGPU_STORE_F64 3

/* on-device synthetic instances (geom.cpp:15-33) */
#define LSAPGPU_GEN_UNIFORM_INT 1 /* (double)(next() % param) */
#define LSAPGPU_GEN_UNIT_F32 2    /* (double)(float)unit_double(next()) */
#define LSAPGPU_GEN_UNIT_SCALED 3 /* unit_double(next()) * param */
#define LSAPGPU_GEN_P2P 4         /* P2P-streaming shaped integers */
#define LSAPGPU_GEN_GEOM 5        /* Euclidean distances, bound = param */

/* ParallelConfig::Reeval (parallel.hpp:21-22) */
#define LSAPGPU_REEVAL_TOUCHED_AND_CONFLICTED 0
#define LSAPGPU_REEVAL_TOUCHED_ONLY 1

typedef struct lsapgpu_ctx lsapgpu_ctx;

typedef struct {
  uint64_t seed;              /* DgsConfig::seed (dgs.hpp:11) */
  double eps;                 /* DgsConfig::improvement_epsilon (dgs.hpp:15) */
  int32_t reeval;             /* LSAPGPU_REEVAL_* */
  int32_t use_graph;          /* 1: inner loop as one CUDA-graph launch (default); 0: host-stepped */
  int64_t deadline_ns;        /* DgsConfig::deadline; < 0 = none */
  const int32_t* init_sigma;  /* optional initial sigma (job -> agent); NULL = init_mode below */
  int32_t init_mode;          /* without init_sigma: LSAPGPU_INIT_RANDOM = random_perm(seed), the
                                 reference's initial_random (dgs.cpp:22-25); LSAPGPU_INIT_GREEDY =
                                 the device greedy assignment (extension, lsapgpu_greedy_assignment) */
  int32_t pad_;
} lsapgpu_params;
#define LSAPGPU_INIT_RANDOM 0
#define LSAPGPU_INIT_GREEDY 1

typedef struct {
  int64_t outer_iterations;   /* SolveReport::outer_iterations */
  int64_t switches_applied;   /* SolveReport::switches_applied */
  int32_t terminated_by;      /* 0 converged, 1 deadline (SolveReport::terminated_by) */
  double value;               /* SolveReport::assignment.value (ordered objective) */
  double elapsed_ms;          /* SolveReport::elapsed */
  /* instrumentation (not in SolveReport) */
  int64_t inner_iterations;   /* conflict-check batches */
  int64_t pair_items;         /* (agent, tau[agent]) rows scanned: full sweeps + re-evaluation */
  int64_t agent_scans;
  int64_t job_scans;
  int64_t lfmm_rounds;
  int64_t scan_launches;
  int64_t bytes_scanned;      /* algorithmic HBM bytes of the pair scans: pair_items * 2 * n * elem */
  int32_t storage;            /* LSAPGPU_STORE_* */
  int32_t scan_filter;        /* 0, or 8 / 16: the long-row scan's quantized filter copies */
  int64_t filter_kept;        /* filter scan: candidates verified exactly (all items of the solve) */
  int64_t filter_overflows;   /* filter scan: items verified by a whole-row exact scan (queue overflow) */
  int64_t host_log_orders;    /* passes whose delta log the host had to put in batch order itself
                                 (0 normally: the device orders it, log_order.cu) */
} lsapgpu_stats;

const char* lsapgpu_version(void);
int lsapgpu_device_count(void);

int lsapgpu_create(lsapgpu_ctx** out, int device);
void lsapgpu_destroy(lsapgpu_ctx* ctx);
const char* lsapgpu_last_error(const lsapgpu_ctx* ctx);
/* the stream all work of this context is ordered on (a cudaStream_t) */
void* lsapgpu_stream(lsapgpu_ctx* ctx);

/* Row-block placement for a multi-GPU solve (SURVEY §8(e) placement (i)):
 * this context will hold rows [n*rank/world, n*(rank+1)/world) of A -- the
 * agents this rank scans -- and all of AT (every other A[i][j] is read as
 * AT[j][i]), instead of full replicas of both.  Call before setting the
 * matrix; the matrix must then be solved with lsapgpu_solve_dist as that
 * rank of that many (single-GPU entry points refuse it).  world = 1 (the
 * default) holds every row.  Replaces nothing in the reference (its solver is
 * one process); sized for n beyond one full A + AT replica per GPU. */
int lsapgpu_set_placement(lsapgpu_ctx* ctx, int32_t rank, int32_t world);

/* Instance upload.  `data` is a row-major n x n matrix of `dtype` in host
 * memory (pinned or pageable).  Validates n >= 1 and finiteness exactly like
 * Instance::validate, chooses the narrowest lossless device storage, and
 * builds A and AT in HBM. */
int lsapgpu_set_matrix(lsapgpu_ctx* ctx, const void* data, int32_t n, int32_t dtype);
/* Same, for a matrix already in device memory of this context's device. */
int lsapgpu_set_matrix_device(lsapgpu_ctx* ctx, const void* dev_data, int32_t n, int32_t dtype);
/* Synthetic instance generated on the device (LSAPGPU_GEN_*). */
int lsapgpu_generate(lsapgpu_ctx* ctx, int32_t kind, int32_t n, uint64_t seed, double param);
int32_t lsapgpu_n(const lsapgpu_ctx* ctx);
int32_t lsapgpu_storage(const lsapgpu_ctx* ctx);
/* Copy rows of the (device) instance back as fp64, row-major nrows x n. */
int lsapgpu_read_rows(lsapgpu_ctx* ctx, const int32_t* rows, int32_t nrows, double* out);

/* lsap::dgs_parallel.  sigma_out / tau_out: n entries each (tau_out may be
 * NULL).  trace_switch / trace_value may be NULL; otherwise they receive up to
 * trace_cap entries of SolveReport::objective_trace and *trace_len its full
 * length. */
int lsapgpu_solve(lsapgpu_ctx* ctx, const lsapgpu_params* params, int32_t* sigma_out,
                  int32_t* tau_out, lsapgpu_stats* stats, int64_t* trace_switch,
                  double* trace_value, int64_t trace_cap, int64_t* trace_len);

/* Multi-GPU solve, one process (and context) per GPU, every rank holding the
 * full instance (SURVEY 8(e) placement (ii)).  Work items are owned by agent
 * index (i % world == rank); after each scan the library calls `allgather`
 * (enqueue on `stream`, e.g. ncclAllGather / torch.distributed over NVLink)
 * to exchange `bytes_per_rank` bytes from send_dev into recv_dev
 * (world * bytes_per_rank); the conflict check and apply then run replicated
 * and deterministic, so every rank returns the same result, equal to
 * lsapgpu_solve's.  world == 1 is lsapgpu_solve. */
typedef int (*lsapgpu_allgather_fn)(void* user, const void* send_dev, void* recv_dev,
                                    size_t bytes_per_rank, void* stream);
typedef struct {
  int32_t rank, world;
  lsapgpu_allgather_fn allgather;
  void* user;
  void* send_dev; /* >= lsapgpu_dist_exchange_bytes(n, world) bytes, device memory */
  void* recv_dev; /* world times that (peer mode: this rank's lsapgpu_dist_p2p_bytes buffer) */
  /* Peer-memory transport, used instead of `allgather` when non-NULL (world
   * <= 8): the receive buffer (lsapgpu_dist_p2p_bytes each) and the flag
   * array (world x uint64, zeroed before the first solve) of every rank,
   * mapped in this process (lsapgpu_ipc_open for other processes' buffers,
   * plain pointers for ranks sharing a device).  Each rank's pack kernel
   * stores its records straight into every replica over NVLink and raises its
   * flag there; no collective call.  All ranks must run the same sequence of
   * solves on these buffers. */
  void* const* peer_recv;
  uint64_t* const* peer_flags;
} lsapgpu_dist;
size_t lsapgpu_dist_exchange_bytes(int32_t n, int32_t world);
size_t lsapgpu_dist_p2p_bytes(int32_t n, int32_t world);
/* Zeroed device allocation of its own (cudaMalloc: the IPC handle maps the
 * allocation base) on `device`, and its release */
int lsapgpu_dev_alloc(int device, size_t bytes, void** dev_ptr);
int lsapgpu_dev_free(int device, void* dev_ptr);
/* CUDA IPC of a device allocation, as plain bytes (64-byte handle) */
int lsapgpu_ipc_handle(const void* dev_ptr, void* handle64);
int lsapgpu_ipc_open(const void* handle64, void** dev_ptr);
int lsapgpu_ipc_close(void* dev_ptr);
int lsapgpu_solve_dist(lsapgpu_ctx* ctx, const lsapgpu_params* params, const lsapgpu_dist* dist,
                       int32_t* sigma_out, int32_t* tau_out, lsapgpu_stats* stats,
                       int64_t* trace_switch, double* trace_value, int64_t trace_cap,
                       int64_t* trace_len);

/* lsap::evaluate_all_parallel: SoA records; partner -1 = inactive (delta 0). */
int lsapgpu_evaluate_all(lsapgpu_ctx* ctx, const int32_t* sigma, double eps, double* agent_delta,
                         int32_t* agent_partner, double* job_delta, int32_t* job_partner);

/* lsap::check_conflicts.  Inputs: tables with inactive deltas already 0 (the
 * normalisation check_conflicts applies, parallel.cpp:166-173) and sigma.
 * Outputs u8[n] masks and the ascending conflicted_jobs list (returns its
 * length through *n_conflicted_jobs).  Needs no matrix; n is given. */
int lsapgpu_check_conflicts(lsapgpu_ctx* ctx, int32_t n, const double* agent_delta,
                            const int32_t* agent_partner, const double* job_delta,
                            const int32_t* job_partner, const int32_t* sigma,
                            uint8_t* agent_accepted, uint8_t* job_accepted,
                            uint8_t* reserved_mask, uint8_t* conflicted_mask,
                            int32_t* conflicted_jobs, int32_t* n_conflicted_jobs);

/* lsap::apply_parallel_switches on the context's matrix.  sigma/tau/value are
 * updated in place; applied_* (n entries each) receive the applied exchanges
 * in commit order; returns the count through *n_applied. */
int lsapgpu_apply_parallel_switches(lsapgpu_ctx* ctx, int32_t* sigma, int32_t* tau, double* value,
                                    const double* agent_delta, const int32_t* agent_partner,
                                    const uint8_t* agent_active, const double* job_delta,
                                    const int32_t* job_partner, const uint8_t* job_active,
                                    const uint8_t* agent_accepted, const uint8_t* job_accepted,
                                    double eps, int32_t* applied_agent, int32_t* applied_new_job,
                                    int32_t* applied_old_job, int32_t* applied_displaced,
                                    double* applied_delta, int32_t* n_applied);

/* lsap::auction_solve: synchronous bidding rounds on the
 * context's matrix, every round of every epsilon phase inside one launch.
 * AuctionConfig (baselines.hpp:12-26): epsilon is used when has_epsilon
 * (else (max - min) / (2n), or 1.0 for a constant matrix); scaling /
 * scale_factor select epsilon scaling; deadline_ns < 0 = none, on expiry the
 * partial assignment is completed greedily (terminated_by 1,
 * completed_greedily 1).  Errors: "auction: epsilon must be > 0",
 * "auction: scale_factor must be > 1".  prices_out (n, nullable) receives
 * the final prices; round_prices (round_cap x n, nullable) the price vector
 * after each of the first round_cap rounds (the on_round observer). */
typedef struct {
  double epsilon;
  int32_t has_epsilon;
  int32_t scaling;
  double scale_factor; /* 4.0 in AuctionConfig */
  int64_t deadline_ns;
} lsapgpu_auction_params;
typedef struct {
  int64_t outer_iterations;   /* SolveReport::outer_iterations (bidding rounds) */
  int64_t switches_applied;   /* awards, displacements included */
  int32_t terminated_by;      /* 0 converged, 1 deadline */
  int32_t completed_greedily; /* SolveReport::completed_greedily */
  double value;               /* ordered objective of the final assignment */
  double elapsed_ms;
  /* instrumentation */
  int64_t bids;               /* agent row scans */
  int64_t phases;             /* epsilon phases run */
  double epsilon;             /* the target epsilon */
  int64_t bytes_scanned;      /* bids * n * (storage element + fp64 price) */
  int32_t storage;
  int32_t pad_;
} lsapgpu_auction_stats;
int lsapgpu_auction_solve(lsapgpu_ctx* ctx, const lsapgpu_auction_params* params, int32_t* sigma_out,
                          int32_t* tau_out, lsapgpu_auction_stats* stats, double* prices_out,
                          double* round_prices, int64_t round_cap);

/* Greedy assignment of the context's matrix (EXTENSION, not in the
 * reference: north-star item 2).  Rounds of: every unassigned agent claims its
 * best free job (row argmax, smallest job on ties); each claimed job goes to
 * the highest claim (smallest agent on ties); losers retry.  sigma_out: job ->
 * agent (n); *rounds (nullable) the number of claim rounds. */
int lsapgpu_greedy_assignment(lsapgpu_ctx* ctx, int32_t* sigma_out, int64_t* rounds);

/* Host helpers (sequential by nature; identical to the reference's). */
void lsapgpu_random_perm(int32_t n, uint64_t seed, int32_t* out);
int lsapgpu_objective(lsapgpu_ctx* ctx, const int32_t* sigma, double* value);

/* Cumulative counters of this context: bytes copied host->device and
 * device->host by the library, and kernels launched (graph-body kernels
 * included).  bench.py differences them around its timed region. */
int lsapgpu_counters(const lsapgpu_ctx* ctx, int64_t* h2d_bytes, int64_t* d2h_bytes,
                     int64_t* kernel_launches);

/* Instrumented re-run support for bench.py: time every pair-scan launch of
 * the last host-stepped solve with CUDA events on the launching stream.
 * Returns the summed pair-scan time (ms) and launch count (and the full-sweep
 * and commit-kernel shares) of the last solve that ran with use_graph = 0 and
 * timing enabled. */
int lsapgpu_set_scan_timing(lsapgpu_ctx* ctx, int enabled);
int lsapgpu_scan_timing(const lsapgpu_ctx* ctx, double* total_ms, int64_t* launches,
                        double* full_sweep_ms, int64_t* full_sweeps, double* commit_ms,
                        int64_t* commit_launches);

/* The pair-scan plan chosen for the current matrix (instrumentation): up to
 * cap of {kernel (0 streaming, 1 resident, 2 quantized filter), items or row
 * buffers per CTA, stage buffers or chunk slots, filter bits (0, 8, 16), CTAs,
 * threads per CTA, dynamic smem bytes, chunk, filter queue capacity, filter
 * aux in tensor memory (0 / 1)}.
 * Returns the number of values written, < 0 on error. */
int lsapgpu_scan_plan(const lsapgpu_ctx* ctx, int32_t* info, int32_t cap);

/* Device timeline (instrumentation, off by default): with capacity > 0 the
 * first CTA of every pair-scan and commit launch appends one entry
 * (%globaltimer ns << 4 | kind: 1 full sweep, 2 re-evaluation scan, 3 commit
 * start, 4 commit end) so graph-mode solves can be broken down by phase.
 * lsapgpu_timeline copies out and clears the entries; returns the count. */
int lsapgpu_set_timeline(lsapgpu_ctx* ctx, int32_t capacity);
int32_t lsapgpu_timeline(lsapgpu_ctx* ctx, uint64_t* out, int32_t capacity);

#ifdef __cplusplus
}
#endif
#endif /* LSAPGPU_H */
