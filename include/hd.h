/*
 * hd.h — C-ABI of the B200-native Householder Dice (HD) hot path.
 *
 * Drop-in boundary for the reference's probe-operator interface
 * (/root/reference/proj/include/lazymat/operators.hpp:29-49) and its
 * callers. Plain pointers and sizes only; no C++, Eigen or torch types.
 * Every entry point names the reference interface it replaces.
 *
 * Error model (types.hpp:32-43, 67-69; dynamics.hpp:50-51,65-66): every
 * function returns an hd_status; on failure hd_last_error() returns the
 * reference's message text (thread-local). HD_ERR_INVALID_ARGUMENT maps
 * std::invalid_argument (Python ValueError), HD_ERR_BUDGET_EXHAUSTED maps
 * BudgetExhausted, HD_ERR_RESOURCE_CAP maps ResourceCapExceeded,
 * HD_ERR_RUNTIME maps std::runtime_error (non-finite iterate). A failed
 * probe leaves the operator state untouched, like the reference.
 *
 * Threading: one handle per thread, no internal locking (
 * parallel.hpp:13-16). Determinism: the same config (seed, stream, draw
 * mode) and inputs give bit-identical outputs on the same GPU model.
 */
#ifndef HD_B200_H_
#define HD_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum hd_status {
  HD_OK = 0,
  HD_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (types.hpp:67-69) */
  HD_ERR_BUDGET_EXHAUSTED = 2, /* BudgetExhausted (types.hpp:32-35)       */
  HD_ERR_RESOURCE_CAP = 3,     /* ResourceCapExceeded (types.hpp:39-43)   */
  HD_ERR_RUNTIME = 4,          /* std::runtime_error (dynamics.hpp:65-66) */
  HD_ERR_CUDA = 5,
  HD_ERR_NCCL = 6
} hd_status;

typedef enum hd_ensemble { HD_GINIBRE = 0, HD_HAAR = 1, HD_GOE = 2 } hd_ensemble;
typedef enum hd_side { HD_RIGHT = 0, HD_LEFT = 1 } hd_side; /* types.hpp:26 */
typedef enum hd_dtype { HD_F64 = 0, HD_F32 = 1, HD_C128 = 2 /* complex<double>, interleaved (re, im) */ } hd_dtype;
/* Gaussian draws:
 *  PHILOX    device Philox4x32-10 keyed by (seed, stream), counter (row, probe):
 *            production, generated inside the streaming kernels;
 *  INJECTED  the caller pushes them in probe order (hd_push_draws);
 *  REFERENCE the reference's own RandomSource(seed, stream) stream
 *            (xoshiro256++ + ziggurat, random.cpp:78-176), generated on the
 *            host and queued: the same seed gives the reference's matrix. */
typedef enum hd_draw_mode { HD_DRAWS_PHILOX = 0, HD_DRAWS_INJECTED = 1, HD_DRAWS_REFERENCE = 2 } hd_draw_mode;
/* Exchange of a row-sharded operator group: NCCL across ranks
 * (one GPU each) or in-process for virtual shards (one host thread each). */
typedef struct hd_exchange hd_exchange;

/* reflect.hpp:33 SignRule; FaultFlags operators.hpp:16-22 */
typedef enum hd_sign_rule {
  HD_SIGN_STABLE = 0,
  HD_SIGN_NEGATIVE_AT_ZERO = 1,
  HD_SIGN_ZERO_WHEN_NEGATIVE = 2
} hd_sign_rule;

typedef struct hd_config {
  int32_t ensemble;      /* hd_ensemble                                      */
  int32_t dtype;         /* hd_dtype (storage + streaming precision)        */
  int64_t m, n;          /* Ginibre: m x n; Haar/GOE: n x n (m ignored)      */
  double sigma;          /* Ginibre entry std (ginibre.hpp:31); GOE inner σ  */
  uint64_t seed;         /* RandomSource(seed, stream) (random.hpp:130)      */
  uint64_t stream;
  int64_t capacity;      /* max probes this handle will serve (panel width);
                            0 = the full budget min(m,n) / n / floor(n/2)    */
  int32_t draw_mode;     /* hd_draw_mode                                     */
  int32_t skip_reflector;/* FaultFlags::skip_reflector                       */
  int32_t sign_rule;     /* FaultFlags::sign_rule                            */
  int32_t device;        /* CUDA device ordinal                              */
  /* Row sharding (north star: n beyond one GPU's HBM): shard_count > 1 makes
   * this handle shard `shard_rank` of an operator whose panels and vectors
   * are split into tile-aligned row slabs (hd_shard_plan); every shard must
   * make the same calls with its own rows of x / y (hd_shard_range), and
   * `capacity` (max probes per chain) is required. 0 or 1 without an
   * exchange = unsharded; a 1-shard group with an exchange runs the
   * sharded protocol (exchange after every streaming kernel) on one GPU. */
  int32_t shard_count;
  int32_t shard_rank;
  hd_exchange* exchange; /* the group's exchange (hd_exchange_create_*)     */
} hd_config;

typedef struct hd_op hd_op;

/* Exchanges and the shard plan. After every streaming kernel
 * the shards of one operator allreduce one buffer: the partial dot
 * products, shard 0's head rows and the status flags (NCCL over NVLink for
 * one rank per GPU; in-process for virtual shards, one host thread each). */
int hd_exchange_create_local(int32_t nshards, hd_exchange** out);
int hd_exchange_nccl_id(void* id_out /* 128 bytes, ncclGetUniqueId */);
int hd_exchange_create_nccl(const void* id, int32_t nranks, int32_t rank, int32_t device, hd_exchange** out);
int hd_exchange_destroy(hd_exchange* ex);
/* rows [begin, end) of an N-row dimension owned by shard `rank` of `count`:
 * tile-aligned slabs, shard 0 holding the head rows [0, head_rows) */
int hd_shard_plan(int64_t N, int32_t count, int32_t rank, int64_t head_rows, int64_t* begin, int64_t* end);
/* the rows this handle owns: dim 0 = n (right-probe input), 1 = m (output) */
int hd_shard_range(const hd_op* op, int32_t dim, int64_t* begin, int64_t* end);

/* Replaces the constructors GinibreOperator(m, n, sigma, RandomSource, faults)
 * (ginibre.hpp:31-42), HaarOperator(n, RandomSource, faults) (haar.hpp:24-31),
 * GOEOperator(n, RandomSource, faults) / GOEOperator(unique_ptr<Ginibre>)
 * (ensembles.hpp:100-109) and the bindings (module.cpp:68-111). */
int hd_create(const hd_config* cfg, hd_op** out);
int hd_destroy(hd_op* op);

/* ProbeOperator::rows/cols/remaining_probes (operators.hpp:33-40). */
int hd_shape(const hd_op* op, int64_t* rows, int64_t* cols);
int hd_remaining(const hd_op* op, int64_t* remaining);
/* GinibreOperator::probe_counts (ginibre.hpp:53) / HaarOperator::probe_count
 * (haar.hpp:37; returned as right = t, left = 0) and chain sizes. */
int hd_counts(const hd_op* op, int64_t* right, int64_t* left);
int hd_chain_sizes(const hd_op* op, int64_t* right_chain, int64_t* left_chain);

/* ProbeOperator::probe(x, side) (operators.hpp:41): y = Q x (right) or
 * Q^T x (left). x/y are host pointers (on_device = 0) or device pointers of
 * the operator's dtype (on_device = 1); a shard passes its own rows only. Validation order follows
 * check_probe_input then the budget check (operators.hpp:44-48,
 * ginibre.hpp:59-62). Synchronous: returns after y is written. `stream` is
 * the caller's cudaStream_t (NULL = the legacy default stream): the probe
 * runs on the handle's own stream, ordered after all work already enqueued
 * on `stream`, so a device x produced there is complete before it is read. */
int hd_probe(hd_op* op, const void* x, int64_t x_len, void* y, int64_t y_len, int32_t side, int32_t on_device,
             void* stream);

/* Parity mode: append caller-supplied N(0,1) draws (fp64) to the handle's
 * draw queue; each probe consumes one vector of its draw length (Ginibre
 * right: m, left: n; Haar: n; GOE: n per inner probe). */
int hd_push_draws(hd_op* op, const double* g, int64_t len, int32_t on_device);

/* Reset to the freshly constructed state (counters, chains, queue). */
int hd_reset(hd_op* op);

/* ---------------------------------------------------------------------------
 * Device-resident dynamics (replaces run_dynamics, dynamics.hpp:42-76, for the
 * built-in update maps of the BASELINE configs). */
typedef enum hd_update {
  HD_UPDATE_IDENTITY = 0,  /* x_{t+1} = y_t                                   */
  HD_UPDATE_NORMALIZE = 1, /* x_{t+1} = y_t / ||y_t|| (bench.cpp:25-28)       */
  HD_UPDATE_TANH_MIX = 2   /* x_{t+1} = tanh(2 y_t) + 0.1 x_{t-1} (depth 1)   */
} hd_update;

typedef enum hd_side_rule {
  HD_SIDES_ALTERNATE = 0, /* right on odd t, left on even t (bench.cpp:22-24) */
  HD_SIDES_RIGHT = 1,
  HD_SIDES_LEFT = 2
} hd_side_rule;

typedef struct hd_run_args {
  int32_t update;      /* hd_update                                          */
  int32_t side_rule;   /* hd_side_rule                                       */
  int64_t iterations;  /* T                                                  */
  const void* x1;      /* newest initial iterate                             */
  const void* x0;      /* older iterate for depth-1 maps (NULL = zeros)      */
  int32_t on_device;   /* pointers are device pointers of the op's dtype     */
  int32_t use_graph;   /* capture the T-step launch sequence in a CUDA graph */
  void* traj;          /* optional (T+1) x dim iterates x_1..x_{T+1}         */
  void* final_out;     /* optional x_{T+1}                                   */
  void* stream;        /* caller's cudaStream_t (NULL = legacy default); the
                          run is ordered after work already enqueued on it  */
} hd_run_args;

/* run_dynamics(op, spec): validation messages and the non-finite abort
 * ("run_dynamics: non-finite iterate at step N") follow dynamics.hpp:44-67. */
int hd_run(hd_op* op, const hd_run_args* args);

/* Asynchronous run: enqueue the whole T-step run (CUDA-graph replay when
 * use_graph) on the handle's own stream, ordered after `args->stream`, and
 * return; hd_wait completes it (status words, error reporting as hd_run, host
 * copies). Device outputs are valid once hd_wait returns. Many handles run
 * concurrently on their own streams (batched independent trials, config 3).
 * x1 / x0 must stay valid until hd_wait: a two-pass Haar run whose precision
 * guard fires is re-run from them. */
int hd_run_async(hd_op* op, const hd_run_args* args);
int hd_wait(hd_op* op);

/* Fresh operator state with a new RandomSource seed (Philox key), without a
 * host synchronisation: one captured run graph serves every trial seed. */
int hd_reseed(hd_op* op, uint64_t seed);

/* Batched independent trials (BASELINE config 3; the reference runs trials
 * on threads, parallel.hpp): `count` operators of one ensemble, shape and
 * dtype (device Philox draws, unsharded, real) each run `args` (iterations,
 * update, side_rule; device vectors) from a fresh state with its own seed,
 * x_1 = items[i].x1, writing x_{T+1} to items[i].out. Every kernel launch of
 * the run is issued once for all operators (gridDim.y = count); the launch
 * sequence is recorded and captured in one CUDA graph on the first call for a
 * given operator set and replayed afterwards. Asynchronous on args->stream;
 * the operators must be idle. Each trial equals a separate hd_run call up to
 * the rounding of its re-associated GEMV-T partial sums (a batched launch
 * gives each trial its share of the SMs, so the warp -> tile split differs:
 * <= 1e-11 relative, tests/test_gpu_batch.py), and repeated batched calls are
 * bitwise identical. Non-finite steps are not reported (each operator's status
 * words hold them). */
typedef struct hd_batch_item {
  const void* x1;  /* device x_1 (op dtype) */
  void* out;       /* device x_{T+1}        */
  uint64_t seed;   /* RandomSource seed     */
} hd_batch_item;
int hd_batch_run(hd_op* const* ops, int32_t count, const hd_run_args* args, const hd_batch_item* items);

/* User update map on device memory: called once per step after the probe
 * with y_t and the history window newest first (device pointers of the op's
 * dtype, each dim elements); must write x_{t+1} into `next` on `stream`.
 * Return non-zero to abort. (DynamicsSpec::update, dynamics.hpp:21-32.) */
typedef int (*hd_update_fn)(void* user, int64_t t, const void* y, const void* const* history, int32_t depth,
                            void* next, int64_t dim, void* stream);
typedef int32_t (*hd_side_fn)(void* user, int64_t t);

int hd_run_callback(hd_op* op, int64_t iterations, int32_t depth, const void* const* initial_dev,
                    hd_side_fn side_of, hd_update_fn update, void* user, void* final_out_dev);

/* ---------------------------------------------------------------------------
 * Device-resident application runs of the BASELINE workloads: the whole run
 * is one CUDA graph (no host synchronisation per probe); the update maps run
 * in the epilogue of each probe's output pass. The reference has neither map
 * (SPEC.md:439 lists AMP as a non-goal); both are defined once in the test
 * oracle (oracle/hd_oracle.cpp or_amp / or_spiked_power, same operation order)
 * and the probes are GinibreOperator::probe (ginibre.hpp:58-106) and
 * GOEOperator::probe (ensembles.hpp:117-127). Vectors are host pointers
 * (on_device = 0) or device pointers of the operator's dtype; curves are
 * double. Synchronous; errors as hd_run.
 *
 * AMP on a Ginibre design A (m x n), delta = m / n (BASELINE config 4):
 *   y = A beta + w (one right probe, experiments.cpp:80-82), x^0 = 0, z^0 = y,
 *   x^{t+1} = soft(x^t + A^T z^t, alpha ||z^t|| / sqrt(m))  (experiments.cpp:31-39)
 *   z^{t+1} = y - A x^{t+1} + (nnz(x^{t+1}) / n / delta) z^t
 *   mse_out[t] = ||x^{t+1} - beta||^2 / n; x_out = x^T. 2T + 1 probes. */
typedef struct hd_amp_args {
  const void* beta;   /* n  */
  const void* w;      /* m  */
  int64_t iterations; /* T  */
  double alpha;       /* threshold multiplier (1.5 in config 4) */
  void* x_out;        /* n  */
  double* mse_out;    /* T, optional */
  int32_t on_device;
  int32_t use_graph;
  void* stream;       /* caller's cudaStream_t (NULL = legacy default) */
} hd_amp_args;
int hd_run_amp(hd_op* op, const hd_amp_args* args);

/* Power method on a spiked GOE (BASELINE config 5): G the GOE operator,
 *   x_{t+1} = (G x_t + theta <u, x_t> u) / ||.||,  overlap_out[t] = <u, x_{t+1}>,
 * x_out = x_{T+1}. u should be a unit vector. */
typedef struct hd_spiked_args {
  const void* u;      /* n  */
  const void* x1;     /* n  */
  int64_t iterations; /* T GOE steps (2T inner probes) */
  double theta;
  void* x_out;        /* n  */
  double* overlap_out;/* T, optional */
  int32_t on_device;
  int32_t use_graph;
  void* stream;
} hd_spiked_args;
int hd_run_spiked(hd_op* op, const hd_spiked_args* args);

/* ---------------------------------------------------------------------------
 * Standalone reflector: make_reflector(p, offset, zero_tol, sign_rule) built
 * on the device and applied to `count` vectors x (each n long, contiguous)
 * into y (reflect.hpp:70-83,120-176; bindings module.cpp:48-66). Real
 * reflectors are self-adjoint. info (host, optional) receives c, s and the
 * identity flag. Validation messages follow reflect.hpp:124-127. */
int hd_reflector_apply(const double* p, int64_t n, int64_t offset, double zero_tol, int32_t sign_rule,
                       const double* x, double* y, int64_t count, int32_t on_device, double* info);

/* ---------------------------------------------------------------------------
 * Instrumentation: per-kernel-kind launch counts, device time (CUDA events
 * on the handle's stream) and algorithmic bytes. Off by default. */
typedef struct hd_kernel_stats {
  char name[32];
  int64_t launches;
  double ms;
  double alg_bytes;
} hd_kernel_stats;

int hd_set_profiling(hd_op* op, int32_t enabled);
int hd_get_stats(hd_op* op, hd_kernel_stats* out, int32_t max, int32_t* count);
int hd_reset_stats(hd_op* op);
/* Number of kernels this library launched on behalf of the handle. */
int hd_launch_count(const hd_op* op, int64_t* count);

const char* hd_last_error(void);

/* ---------------------------------------------------------------------------
 * The reference's RandomSource (random.hpp:55-112) on the host, for callers
 * that draw their data the way the reference does (experiments.cpp:124-125:
 * matrix stream 0, data stream 1). normal_vector fills `out` (len >= 1). */
typedef struct hd_rs hd_rs;
int hd_rs_create(uint64_t seed, uint64_t stream, hd_rs** out);
void hd_rs_destroy(hd_rs* rs);
uint64_t hd_rs_next_u64(hd_rs* rs);
double hd_rs_uniform(hd_rs* rs);
double hd_rs_normal(hd_rs* rs);
int hd_rs_normal_vector(hd_rs* rs, int64_t len, double* out);
/* sample_bernoulli_gaussian (experiments.cpp:19-29): per entry one uniform,
 * 0 when it is < rho, else sigma_s * normal() (polar). */
int hd_rs_bernoulli_gaussian(hd_rs* rs, int64_t n, double rho, double sigma_s, double* out);
uint64_t hd_derive_seed(uint64_t base, uint64_t index); /* random.cpp:73-76 */
/* The PHILOX draw stream: out[0..n) (device memory) = the Gaussian draw of
 * probe index `probe` that an operator with (seed, stream) generates on the
 * device (Philox4x32-10, key = seed, counter = (row pair, probe, stream);
 * Box-Muller on two 53-bit uniforms). Asynchronous on `stream_ptr`
 * (cudaStream_t, NULL = legacy default). */
int hd_philox_normals(uint64_t seed, uint64_t stream, int64_t probe, int64_t n, double* out, void* stream_ptr);
const char* hd_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HD_B200_H_ */
