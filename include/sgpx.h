/*
 * sgpx.h -- C ABI of the B200-native psi-statistics engine (libsgpx.so).
 *
 * Drop-in boundary for the data-parallel hot path of the reference
 * (arXiv 1410.4984 restatement under /root/reference/proj/include/sgp):
 *
 *   sgpx_sweep_stats        replaces sgp::detail::sweep_stats            psi_stats.hpp:108-326
 *                           (and the wrappers stats_deterministic :332, psi2_expected :379,
 *                            stats_expected :389, stats_grads :402, stats_grads_deterministic :415)
 *   sgpx_psi1_expected      replaces sgp::psi1_expected                  psi_stats.hpp:351-376
 *   sgpx_psi0_expected      replaces sgp::psi0_expected                  psi_stats.hpp:343-347
 *   sgpx_engine_*           replaces sgp::Engine (ctor :326-346, broadcast :358-367,
 *                           evaluate :370-450, run_pass :455-479) and Worker::pass :132-176
 *   sgpx_coordinate_host    the coordinator algebra of Engine::evaluate: factor_gram
 *                           (kernels.hpp:177-197) + bound_core (bound.hpp:84-119) +
 *                           adjoints_from_core (bound.hpp:196-226)
 *   sgpx_finish_host        gradient assembly of Engine::evaluate (parallel.hpp:414-421):
 *                           kern_grads(Z,Z,dKmm) (kernels.hpp:124-164) + jitter term
 *   sgpx_multi_*            sgp::Engine(workers) over several GPUs of one process: shards per
 *                           make_partition (parallel.hpp:28-41), NCCL allreduce exchanges
 *   sgpx_fit_*              FitSession + LbfgsState (model.hpp:100-168, optimizer.hpp:20-458) with
 *                           the parameter vector and the L-BFGS history resident on the device
 *   sgpx_rng_*              sgp::Rng::normal_matrix (common.hpp:45-97) generated on the device,
 *                           the init_gplvm Z-row choice (model.hpp:420-429)
 *   sgpx_io_*               write_matrix_bin / read_matrix_bin (io.hpp:114-153) + a streamed
 *                           loader straight into device memory
 *
 * Conventions
 *   - All matrices at this boundary are fp64, column-major with a leading
 *     dimension (Eigen::MatrixXd / Eigen::Ref with outer stride).  ld == 0
 *     means ld == rows.
 *   - Outputs are caller-allocated and fully overwritten (the reference
 *     allocates and overwrites, psi_stats.hpp:123-134).
 *   - Return codes: SGPX_OK, SGPX_INVALID_ARGUMENT (the reference throws
 *     std::invalid_argument via require(), common.hpp:24-26), SGPX_NUMERIC
 *     (sgp::NumericError, common.hpp:20-22), SGPX_CUDA, SGPX_NCCL,
 *     SGPX_INTERNAL.  The message of the last failure on the calling thread is
 *     sgpx_last_error().  No C++ exception crosses this boundary.
 *   - Threading: a context (one device + one stream + scratch) is
 *     single-threaded; different contexts may be driven concurrently from
 *     different host threads (reference: pure, reentrant).
 *   - Arithmetic (the precision mode, SGPX_PREC_*, recorded in every result):
 *       fast     psi2 exponents as a bilinear form on tcgen05 (two fp16 pieces, ~2^-22
 *                relative on the feature products), G = 2^D on MUFU.EX2 / FMA (2^-22), the
 *                psi2 contraction as 16-bit split MMAs (bf16 hi/lo ~2^-17 forward, scaled fp16
 *                hi/lo ~2^-22 backward); psi1 weights in fp32 (direct differences), its
 *                Psi = G^T Y and Y dPsi^T contractions as three-pass split-tf32 tcgen05 MMAs;
 *       precise  as fast with three fp16 exponent pieces (~2^-33) and fp16 forward MMA3 pieces;
 *       direct   direct-difference exponents and exp in fp64 (the reference's own form, ~1 ulp),
 *                fp64 contractions;
 *       syrk     (deterministic inputs; the AUTO choice there) Knm tiles in fp64, Phi = K^T K,
 *                Psi = K^T Y and dL/dK = 2 K U + Y dPsi^T as split-TF32 tensor-core GEMMs (three
 *                passes, ~2^-21 per product, fp32 within 512-row sub-chunks, fp64 across them),
 *                the gradient contraction in fp64;
 *     every sum across datapoints and across CTAs is fp64, all M-sized algebra is fp64.  AUTO
 *     picks syrk for deterministic inputs and fast / precise / direct for latent inputs from the
 *     spread of the inducing points.
 *   - There is no CPU fallback: without a CUDA device every compute entry point
 *     returns SGPX_CUDA.
 */
#ifndef SGPX_H_
#define SGPX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGPX_OK 0
#define SGPX_INVALID_ARGUMENT 1
#define SGPX_NUMERIC 2
#define SGPX_CUDA 3
#define SGPX_NCCL 4
#define SGPX_INTERNAL 5
#define SGPX_IO 6 /* file input / output (the reference's std::runtime_error in io.hpp) */

#define SGPX_ABI_VERSION 2

/* Precision modes (sgpx_engine_config.precision, sgpx_ctx_set_precision). */
#define SGPX_PREC_AUTO 0
#define SGPX_PREC_FAST 2
#define SGPX_PREC_PRECISE 3
#define SGPX_PREC_DIRECT 4
#define SGPX_PREC_SYRK 5 /* deterministic inputs: fp64 Knm tiles + split-TF32 tensor-core GEMMs */

/* Column-major views (Eigen::Ref<const Matrix> / Eigen::Ref<Matrix>). */
typedef struct {
  const double* data;
  int64_t rows, cols, ld;
} sgpx_cmat;

typedef struct {
  double* data;
  int64_t rows, cols, ld;
} sgpx_mmat;

/* sgp::KernelSpec (kernels.hpp:13-33): RBF-ARD, variance * exp(-1/2 sum_q (x_q-z_q)^2 / l_q^2). */
typedef struct {
  double variance;
  const double* lengthscales; /* q entries */
  int64_t q;
} sgpx_kernel_spec;

/* sgp::TileConfig (common.hpp:30-37).  Validated (both >= 1) and otherwise
 * ignored: the sm_100a launch geometry is fixed by the kernels. */
typedef struct {
  int64_t block_span, thread_span;
} sgpx_tile_config;

/* sgp::StatsAdjoints (psi_stats.hpp:56-60). d_phi_big must be symmetric. */
typedef struct {
  double d_phi;
  sgpx_cmat d_psi_y;   /* M x D */
  sgpx_cmat d_phi_big; /* M x M */
} sgpx_stats_adjoints;

/* sgp::SufficientStats (psi_stats.hpp:31-53). */
typedef struct {
  double phi;
  sgpx_mmat psi_y;   /* M x D out */
  sgpx_mmat phi_big; /* M x M out (symmetric) */
  double yy;
  int64_t n_count;
} sgpx_sufficient_stats;

/* sgp::StatsGrads (psi_stats.hpp:65-71).  d_mu / d_s are used only on the
 * expected path (data may be NULL otherwise). */
typedef struct {
  sgpx_mmat d_mu; /* N x Q */
  sgpx_mmat d_s;  /* N x Q */
  sgpx_mmat d_z;  /* M x Q */
  double d_variance;
  double* d_lengthscales; /* Q out */
} sgpx_stats_grads;

/* sgp::BoundBreakdown (bound.hpp:22-35). */
typedef struct {
  double total, log_det_term, data_fit_term, quadratic_term, trace_phi_term, trace_kmm_term, kl_term;
} sgpx_bound_breakdown;

typedef struct sgpx_ctx sgpx_ctx;
typedef struct sgpx_engine sgpx_engine;

/* ---- library / context ---------------------------------------------------- */
const char* sgpx_last_error(void);
int sgpx_abi_version(void);
/* Number of CUDA devices visible (0 on a host without GPU; never fails). */
int sgpx_device_count(void);
int sgpx_ctx_create(int device, sgpx_ctx** out);
int sgpx_ctx_destroy(sgpx_ctx* ctx);
/* Run all work of this context on an external cudaStream_t (e.g. torch's current stream). */
int sgpx_ctx_set_stream(sgpx_ctx* ctx, void* cuda_stream);
int sgpx_ctx_synchronize(sgpx_ctx* ctx);
/* Kernel launches issued by this context since creation (profiling evidence). */
int64_t sgpx_ctx_launch_count(const sgpx_ctx* ctx);
/* Precision mode of the one-shot entry points (sgpx_sweep_stats); SGPX_PREC_AUTO by default. */
int sgpx_ctx_set_precision(sgpx_ctx* ctx, int precision);
/* Mode the last sgpx_sweep_stats of this context ran in (SGPX_PREC_FAST / PRECISE / DIRECT / SYRK; 0 if
 * none) and, optionally, the inducing-point spread Tz that decided it. */
int sgpx_ctx_last_precision(const sgpx_ctx* ctx, double* z_spread);

/* ---- the sweep (psi_stats.hpp:108-326) ------------------------------------- */
/* expected != 0: q(X) = N(mu, diag s) path (Bayesian GP-LVM); otherwise mu is X
 * and s is ignored (may be empty).  adj == NULL: statistics only; grads, if
 * given, are zeroed with d_variance = 0 (psi_stats.hpp:128-134).  Host pointers. */
int sgpx_sweep_stats(sgpx_ctx* ctx, int expected, sgpx_cmat mu, sgpx_cmat s, sgpx_cmat y, sgpx_cmat z,
                     const sgpx_kernel_spec* kernel, const sgpx_tile_config* tiles,
                     const sgpx_stats_adjoints* adj, sgpx_sufficient_stats* stats, sgpx_stats_grads* grads);

/* psi1_expected (psi_stats.hpp:351-376): the N x M matrix E[k(x_n, z_m)]. */
int sgpx_psi1_expected(sgpx_ctx* ctx, sgpx_cmat mu, sgpx_cmat s, sgpx_cmat z, const sgpx_kernel_spec* kernel,
                       sgpx_mmat out);

/* psi0_expected (psi_stats.hpp:343-347): N * variance (validates q). */
int sgpx_psi0_expected(sgpx_cmat mu, sgpx_cmat s, const sgpx_kernel_spec* kernel, double* out);

/* ---- coordinator algebra (host fp64, no device needed) --------------------- */
/* Packed statistics vector (the allreduce #1 payload), fp64:
 *   [0] phi  [1] yy  [2] n_count  [3] kl  [4 .. 4+P) Phi upper triangle, pairs
 *   (a<=b) in m1-major order (psi_stats.hpp:85-97)  [4+P .. 4+P+M*D) Psi, M x D col-major.
 * P = M(M+1)/2. */
int64_t sgpx_packed_stats_count(int64_t m, int64_t d);
/* Packed global-gradient vector (allreduce #2 payload): [0] d_variance
 * [1 .. 1+Q) d_lengthscales  [1+Q .. 1+Q+M*Q) d_z col-major. */
int64_t sgpx_packed_grads_count(int64_t m, int64_t q);

/* Coordinator step of Engine::evaluate (parallel.hpp:378-408): factor_gram,
 * bound_core, KL term (latent), adjoints_from_core.  Inputs: the REDUCED packed
 * stats.  Outputs: breakdown; optional adjoints d_psi_y (M x D), d_phi_big
 * (M x M), d_kmm (M x M), scalars adj_scalars[0]=d_phi [1]=d_beta
 * [2]=jitter_factor used.  n/d: global N and D. */
int sgpx_coordinate_host(int kind, int64_t n, int64_t d, int64_t m, const double* packed_stats, sgpx_cmat z,
                         const sgpx_kernel_spec* kernel, double beta, double jitter_factor,
                         sgpx_bound_breakdown* bd, double* adj_scalars, double* d_psi_y, double* d_phi_big,
                         double* d_kmm);

/* Gradient assembly (parallel.hpp:414-421): given the REDUCED packed grads,
 * adds kern_grads(Z, Z, dKmm).d_z + .d_x, kern_grads.d_variance + jitter_factor
 * * tr(dKmm), kern_grads.d_lengthscales.  Writes d_z (M x Q), *d_variance, d_ls (Q). */
int sgpx_finish_host(int64_t m, int64_t q, const double* packed_grads, sgpx_cmat z, const sgpx_kernel_spec* kernel,
                     const double* d_kmm, double jitter_factor, double* d_z, double* d_variance, double* d_ls);

/* ---- engine (parallel.hpp:326-479), one instance per rank / GPU ------------ */
typedef struct {
  int kind;          /* 0 = regression (X fixed), 1 = latent (Bayesian GP-LVM) */
  int64_t n_global;  /* N over all ranks */
  int64_t row_begin; /* first global row owned here (make_partition, parallel.hpp:28-41) */
  int64_t n_local;   /* rows owned here */
  int64_t q, d, m;
  double jitter_factor; /* factor_gram start (default 1e-6, parallel.hpp:327) */
  int precision;        /* SGPX_PREC_* (AUTO: chosen per broadcast from the inducing points) */
} sgpx_engine_config;

typedef struct {
  sgpx_bound_breakdown bound;
  double phi, yy;
  int64_t n_count;
  double* psi_y;   /* optional host out, M x D */
  double* phi_big; /* optional host out, M x M */
  int has_grads;
  double* d_z;            /* optional host out, M x Q */
  double* d_lengthscales; /* optional host out, Q */
  double d_variance, d_beta;
  double jitter_factor_used;
  /* EngineTimings (parallel.hpp:296-301), seconds: passes and kernels are
   * device-event timed on the context stream; coordinator_s is host wall time. */
  double stats_pass_s, coordinator_s, grad_pass_s, wall_s;
  double fwd_kernel_s, bwd_kernel_s; /* the psi forward / backward kernels alone */
  int fwd_grid, bwd_grid;            /* persistent CTAs launched */
  int precision_used;                /* SGPX_PREC_FAST / PRECISE / DIRECT / SYRK of this evaluation */
  double z_spread;                   /* Tz = max_a sum_q ((z_aq - c_q) / l_q)^2, c = mean of Z */
  double psi2_fwd_kernel_s, psi2_bwd_kernel_s; /* the main psi2 kernel of each pass alone (first sub-shard) */
} sgpx_eval_result;

int sgpx_engine_create(sgpx_ctx* ctx, const sgpx_engine_config* cfg, sgpx_engine** out);
int sgpx_engine_destroy(sgpx_engine* eng);
/* Shard rows (the Worker copies, parallel.hpp:339-343).  on_device != 0: the
 * pointers are device memory on the context's device.  y: n_local x D;
 * x_or_mu, s: n_local x Q (s ignored for regression). */
int sgpx_engine_set_data(sgpx_engine* eng, sgpx_cmat x_or_mu, sgpx_cmat s, sgpx_cmat y, int on_device);
/* Engine::broadcast: global params (kernel, beta, Z: host memory, M x Q); mu/s (latent) optional
 * local slice, n_local x Q (data == NULL keeps the current; on_device != 0: device pointers, adopted).
 * Host mu / s are copied asynchronously: broadcast starts their sub-shard uploads on the engine's copy
 * stream and the next stats pass waits for each before its kernels, so the caller keeps both host
 * buffers alive and unchanged until that pass (sgpx_engine_evaluate / sgpx_engine_stats_pass) has
 * returned.  A later set_data waits for and supersedes the pending upload. */
int sgpx_engine_broadcast(sgpx_engine* eng, const sgpx_kernel_spec* kernel, double beta, sgpx_cmat z, sgpx_cmat mu,
                          sgpx_cmat s, int on_device);
/* Single-rank Engine::evaluate(with_grads): the whole pipeline, no collective. */
int sgpx_engine_evaluate(sgpx_engine* eng, int with_grads, sgpx_eval_result* out);
/* Multi-rank phases: the caller all-reduces (sum, fp64) the packed device
 * buffers between phases -- NCCL over NVLink, e.g. torch.distributed.all_reduce
 * on the context's stream. */
int sgpx_engine_stats_pass(sgpx_engine* eng, double** packed_dev, int64_t* count);
int sgpx_engine_coordinate(sgpx_engine* eng, int with_grads);
int sgpx_engine_grad_pass(sgpx_engine* eng, double** packed_dev, int64_t* count);
int sgpx_engine_finish(sgpx_engine* eng, sgpx_eval_result* out);
/* Local per-datapoint gradients (KL included), device, n_local x Q col-major (ld = n_local). */
int sgpx_engine_local_grads_device(sgpx_engine* eng, double** d_mu, double** d_s);
/* Register host buffers (n_local x Q, column-major with ld; pinned for overlap) that every
 * subsequent evaluate(with_grads) fills with d_mu / d_S -- streamed per sub-shard on a copy
 * stream while the remaining sub-shards compute (the reference's Engine returns local grads
 * in its result, parallel.hpp:424-429).  Null data pointers unregister. */
int sgpx_engine_set_local_grads_out(sgpx_engine* eng, sgpx_mmat d_mu, sgpx_mmat d_s);
int sgpx_engine_copy_local_grads(sgpx_engine* eng, sgpx_mmat d_mu, sgpx_mmat d_s);
/* predict (SparseGPRegression::predict / BayesianGPLVM::predict, model.hpp:181-217, 291-296, 378-383)
 * from the factors of the engine's last evaluation at the current parameters (the reference's
 * finalize()): mean = beta K*m G, var = variance - |L_k^-1 k*|^2 + |L_a^-1 k*|^2 (floored at 1e-15
 * variance, + 1/beta when observation != 0), the same column for every output dimension.  x_star: T x Q
 * host; mean / var: T x D host; cached_bound (nullable): that evaluation's bound. */
int sgpx_engine_predict(sgpx_engine* eng, sgpx_cmat x_star, int observation, sgpx_mmat mean, sgpx_mmat var,
                        double* cached_bound);

/* ---- multi-GPU engine: Engine(workers) (parallel.hpp:326-479) in one process --------------------
 * N is split by make_partition (parallel.hpp:28-41) into `workers` shards, shard i on devices[i], each
 * with its own context.  The two exchanges of an evaluation sum the packed buffers: shards sharing a
 * device are folded on it, then one ncclAllReduce (sum, fp64) runs across the distinct devices
 * (NCCL communicators from ncclCommInitAll; libnccl is opened at run time, SGPX_NCCL if absent).
 * cfg: kind, n_global, q, d, m, jitter_factor, precision (row_begin / n_local are per shard).
 * Host views cover all N rows; d_mu / d_s (latent, nullable) receive every shard's rows. */
typedef struct sgpx_multi sgpx_multi;
int sgpx_multi_create(int workers, const int* devices, const sgpx_engine_config* cfg, sgpx_multi** out);
int sgpx_multi_destroy(sgpx_multi* mu);
int sgpx_multi_workers(const sgpx_multi* mu);
int sgpx_multi_set_data(sgpx_multi* mu, sgpx_cmat x_or_mu, sgpx_cmat s, sgpx_cmat y);
int sgpx_multi_broadcast(sgpx_multi* mu, const sgpx_kernel_spec* kernel, double beta, sgpx_cmat z, sgpx_cmat mu_,
                         sgpx_cmat s);
int sgpx_multi_evaluate(sgpx_multi* mu, int with_grads, sgpx_eval_result* out, sgpx_mmat d_mu, sgpx_mmat d_s);

/* ---- the optimisation loop, resident on the device ----------------------------------------------
 * FitSession (model.hpp:100-168) with LbfgsState (optimizer.hpp:205-458) and the packed, log-transformed
 * parameter vector (optimizer.hpp:20-144) kept in device memory: each evaluation broadcasts the
 * device-resident mu / S to the engine and reads its d mu / d S in place; only the M-sized segment and
 * the line search's scalars cross to the host.  The objective is -bound (DistributedObjective,
 * model.hpp:61-92). */
typedef struct {
  int memory;           /* history pairs (10) */
  double c1, c2;        /* Wolfe constants (1e-4, 0.9) */
  double g_tol, f_tol;  /* gradient 2-norm stop (1e-5), relative value-change stop (1e-9) */
  int max_iters;        /* 500 */
  int max_evals;        /* 0 = unlimited */
  int max_line_search;  /* 40 */
} sgpx_lbfgs_options;   /* LbfgsOptions, optimizer.hpp:154-163 */

#define SGPX_FIT_RUNNING (-1)
#define SGPX_FIT_GRADIENT_CONVERGED 0
#define SGPX_FIT_VALUE_CONVERGED 1
#define SGPX_FIT_MAX_ITERATIONS 2
#define SGPX_FIT_MAX_EVALUATIONS 3
#define SGPX_FIT_LINE_SEARCH_FAILED 4

typedef struct sgpx_fit sgpx_fit;
void sgpx_lbfgs_default_options(sgpx_lbfgs_options* opts);
/* Pack the starting parameters (mu / s: host n_local x Q, NULL data for regression) and evaluate once
 * (LbfgsState::initialize).  The engine must have its data set; it stays owned by the caller. */
int sgpx_fit_create(sgpx_engine* eng, int64_t n_local, const sgpx_kernel_spec* kernel, double beta, sgpx_cmat z,
                    sgpx_cmat mu, sgpx_cmat s, const sgpx_lbfgs_options* opts, sgpx_fit** out);
/* One outer L-BFGS iteration (LbfgsState::step); *advanced = 0 once converged / stopped. */
int sgpx_fit_step(sgpx_fit* fit, int* advanced);
/* value = -bound at the current iterate, |grad|, iterations, evaluations, status (SGPX_FIT_*). */
int sgpx_fit_state(const sgpx_fit* fit, double* value, double* grad_norm, int* iterations, int* total_evals,
                   int* last_step_evals, int* status);
const char* sgpx_fit_message(const sgpx_fit* fit);
const char* sgpx_fit_last_error(void);
/* current_params (unpack): host outputs, any may be NULL (z: M x Q, mu / s: n_local x Q). */
int sgpx_fit_params(const sgpx_fit* fit, double* variance, double* lengthscales, double* beta, sgpx_mmat z,
                    sgpx_mmat mu, sgpx_mmat s);
int sgpx_fit_destroy(sgpx_fit* fit);

/* ---- seeded inputs and binary matrices ------------------------------------ */
/* Rng(seed).normal_matrix(rows, cols) (common.hpp:86-91), bit-for-bit the reference's splitmix64 +
 * Box-Muller stream up to the last-ulp differences of the device's fp64 log / sin / cos; out is
 * column-major (ld), device memory if on_device != 0, else host. */
int sgpx_rng_normal_matrix(sgpx_ctx* ctx, uint64_t seed, int64_t rows, int64_t cols, sgpx_mmat out, int on_device);
/* The M distinct row indices init_gplvm picks for Z with Rng(seed) (partial Fisher-Yates,
 * model.hpp:420-429); idx has m entries. */
int sgpx_rng_choose_rows(uint64_t seed, int64_t n, int64_t m, int64_t* idx);
/* Raw binary matrices: <base>.shape = "rows cols\n", <base>.bin = row-major little-endian fp64
 * (io.hpp:114-153).  Host read / write use column-major views; the device loader streams the file
 * through pinned slabs and transposes on the device (dev_out: device memory, column-major). */
int sgpx_io_matrix_shape(const char* base, int64_t* rows, int64_t* cols);
int sgpx_io_read_matrix(const char* base, sgpx_mmat out);
int sgpx_io_write_matrix(const char* base, sgpx_cmat m);
int sgpx_io_load_matrix_device(sgpx_ctx* ctx, const char* base, sgpx_mmat dev_out);

#ifdef __cplusplus
}
#endif
#endif /* SGPX_H_ */
