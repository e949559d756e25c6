// psi_kernels.cuh -- device-side contract of the sm_100a psi-statistics kernels.
//
// Reference: proj/include/sgp/psi_stats.hpp:108-326 (detail::sweep_stats).  The
// kernels compute the same sums with an algebraically equivalent factorisation
// of the exponents:
//
//   psi2:  log2 v_nab = L_na + L_nb + sum_q K_nq z_aq z_bq
//          L_na = sum_q [al_nq z_aq + be_nq z_aq^2] + B_n / 2
//          al = log2e*d2*mu, be = -log2e*(1/l^2 + d2)/4, K = log2e*(1/l^2 - d2)/2,
//          B_n = log2 c2_n - log2e * sum_q d2 mu^2,  d2 = 1/(2S + l^2)
//   psi1:  log2 v1_nm = b1_n - (log2e/2) sum_q d1 (mu - z_m)^2,  d1 = 1/(S + l^2)
//
// with mu and z translated by the mean of Z (exact invariance of the stationary
// kernel) so the fp32 terms stay O(1).  One inner (n, a, b) step is Q FFMA + 1 FADD
// + 1 MUFU.EX2 forward; the reference's direct form is ~3Q+4 flops.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace sgpx {

// Record a timing event; inside a stream capture (the evaluation's CUDA graph) as an external event
// node, so that the replayed graph still times its kernels.
inline cudaError_t record_event(void* ev, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
    return cudaEventRecordWithFlags(static_cast<cudaEvent_t>(ev), st, cudaEventRecordExternal);
  return cudaEventRecord(static_cast<cudaEvent_t>(ev), st);
}

constexpr int kMaxQ = 64;

// Exponent / precision mode of one evaluation, decided on the host from the
// inducing points before any launch (psi_select_mode) and recorded in every result:
//   kModeFast     row-tile tcgen05 path, two fp16 pieces per exponent feature, bf16 forward MMA3
//   kModePrecise  row-tile tcgen05 path, three fp16 pieces, scaled fp16 forward MMA3
//   kModeDirect   direct-difference kernels with fp64 exponents (psi_direct.cu): accurate for any
//                 spread of the data and any Q <= kMaxQ
//   kModeSyrk     deterministic inputs only: fp64 Knm tiles, Phi = K^T K, Psi = K^T Y and
//                 dL/dK = 2 K U + Y dPsi^T as split-TF32 tensor-core GEMMs (syrk.cu)
constexpr int kModeAuto = 0, kModeFast = 2, kModePrecise = 3, kModeDirect = 4, kModeSyrk = 5;

// Per-launch constants (passed by value; ~0.7 KB of kernel parameter space).
struct PsiConst {
  int64_t n;                  // rows of this launch (the shard / call)
  int64_t ld_mu, ld_s, ld_y;  // leading dimensions (elements) of the fp64 inputs
  const double* mu;           // n x q, column-major, device (X on the deterministic path)
  const double* s;            // n x q (expected path only)
  const double* y;            // n x d
  const float* zc;            // [mv][qv] centered inducing inputs, zero padded
  const double* z64;          // m x q column-major inducing inputs (fp64, uncentered)
  int q, qv, m, mv, d, dv;    // true and padded (multiple of 4) sizes
  int expected;
  float variance, log2_var;
  double variance_d;          // fp64 sigma^2 (psi1_expected matrix, d_variance)
  double center[kMaxQ];       // translation applied to mu and z (mean of Z rows)
  float il2[kMaxQ], l2[kMaxQ];
  double ls[kMaxQ];
  unsigned long long* prof;   // optional per-phase cycle counters (SGPX_TC_PROFILE=1), else null
  int mode;                   // kModeFast / kModePrecise / kModeDirect (psi_select_mode)
  void* ev_psi2[2];           // optional cudaEvent_t pair recorded around the main psi2 kernel (roofline)
  const float* rt_pairs_shared;  // row-tile forward: another sub-shard's pair operand (N-independent), else null
};

// Backward-only inputs.
struct BwdConst {
  const float* u;     // [mv][mv] symmetric dL/dPhi (upper triangle mirrored), zero padded
  const float* dpsi;  // [d][mv]  dL/dPsi transposed, zero padded
  const double* u64;     // the same two in fp64 (the direct kernels and the per-pair gradient terms)
  const double* dpsi64;
  double d_phi;       // dL/dphi
  int add_kl;         // latent engine pass: subtract KL gradients (parallel.hpp:163-166)
  int write_local;    // write d_mu / d_s
  double* d_mu;       // n x q col-major (ld = ld_g), fp64
  double* d_s;
  int64_t ld_g;
  const double* fwd_rt;  // row-tile path: the forward's feature / pair-sum region (rt_fwd_region)
  int skip_pair_terms;   // sub-shard passes: the per-pair gradient terms are added by one call only
  // row-tile backward: the N-independent pair operand (U-weighted pair features) and Y scales of an
  // earlier sub-shard's call (inputs, null = compute them), and where this call's are (outputs, optional)
  const float *rt_pre_shared, *rt_ys_shared;
  const float **rt_pre_out, **rt_ys_out;
};

// Packed per-CTA partial layouts (fp64, CTA-private rows, single-writer per slot):
//   forward : [0] yy  [1] kl  [2 .. 2+P) Phi pairs (m1-major)  [2+P .. 2+P+M*D) Psi (m + d*M)
//   backward: [0] d_variance  [1 .. 1+Q) d_lengthscales  [1+Q .. 1+Q+M*Q) d_z (a + q*M)
inline int64_t fwd_part_count(int m, int d) { return 2 + int64_t(m) * (m + 1) / 2 + int64_t(m) * d; }
inline int64_t bwd_part_count(int m, int q) { return 1 + q + int64_t(m) * q; }

struct LaunchGeom {
  int grid, threads;
  size_t smem;
};

// Latent dimensions with an instantiated row-tile / psi1 kernel; other Q are zero-padded up.
int instantiated_q(int q);

// Spread of the inducing points in lengthscale units about the centre P.center:
// Tz = max_a sum_q ((z_aq - c_q) / l_q)^2 (z: m x q column-major, host).  The exponent-as-GEMM
// error of the row-tile path grows with it; datapoints far from every inducing point
// do not need a bound (their terms underflow; the feature kernel zeroes rows whose exponents cannot
// reach the fp16 range).
double psi_z_spread(const PsiConst& P, const double* z_host, int64_t m);
// Mode for these inputs: `requested` (kModeAuto or a forced mode; SGPX_PSI_MODE=fast|precise|direct
// overrides auto for experiments) resolved against the measured envelope and the row-tile
// instantiations.  Forced fast / precise fall back to direct where the row-tile path cannot run.
int psi_select_mode(const PsiConst& P, const double* z_host, int64_t m, int requested);

// Launch geometry the launchers will use, so callers can size the partial buffers:
// geom->grid rows of fwd_part_count / bwd_part_count doubles.
int plan_forward(const PsiConst& P, int num_sms, LaunchGeom* geom);
int plan_backward(const PsiConst& P, int num_sms, LaunchGeom* geom);

// Host launchers, asynchronous on `stream`, by P.mode.  Forward: packed statistics (sgpx.h
// layout) and, in `part`, the pair sums and feature arrays the backward reuses; err_flag receives
// bit 1 for non-finite mu / x / y, bit 4 for a non-positive or non-finite S.  Backward: d mu / d S
// (B.write_local) and the packed gradient vector.  ev_begin / ev_end (cudaEvent_t, nullable) are
// recorded around the psi kernels so callers can time them alone (roofline evidence).
int psi_forward(const PsiConst& P, double* part, double* packed, int* err_flag, int num_sms,
                void* stream, LaunchGeom* geom, void* ev_begin = nullptr, void* ev_end = nullptr);
// phase (row-tile path only): 0 the whole pass, 1 the psi1 kernel alone (it needs d Psi, not d Phi),
// 2 the rest (psi2 kernels, reduction) -- so a caller can overlap the coordinator's d Phi with phase 1.
// reduce_stream / reduce_event (sub-shard passes): the partial-row reduction runs on reduce_stream after
// reduce_event (recorded on `stream`); the caller joins it before using `packed`.  psi1_grid_cap > 0:
// the psi1 kernel runs on at most that many CTAs (an SM left to a concurrent coordinator kernel); the
// partial-row layout stays the one of num_sms (the rows of absent CTAs stay zero).
int psi_backward(const PsiConst& P, const BwdConst& B, double* part, double* packed, int num_sms, void* stream,
                 LaunchGeom* geom, void* ev_begin = nullptr, void* ev_end = nullptr, int phase = 0,
                 void* reduce_stream = nullptr, void* reduce_event = nullptr, int psi1_grid_cap = 0);
// true when psi_backward can run in two phases for P (the row-tile path)
bool psi_backward_phased(const PsiConst& P);
// Where the forward left the region the backward reads (BwdConst::fwd_rt), and the per-pair sums
// inside it: sub-shard forwards add theirs into the first sub-shard's before the gradient pass.
const double* fwd_region(const PsiConst& P, const double* fwd_part, int num_sms);
double* fwd_pair_sums(const PsiConst& P, double* region, int num_sms, int64_t* count);
// the row-tile forward's pair operand inside `region` (N-independent: later sub-shards reuse the
// first one's through PsiConst::rt_pairs_shared); null off the row-tile path
const float* fwd_pair_operand(const PsiConst& P, const double* region, int num_sms);

// psi1 kernels paired with the row-tile psi2 (psi1_kernels.cu: any M; psi1_tile.cu: M <= 128).
int psi1_fwd_rows(const PsiConst& P, int num_sms);
int psi1_bwd_ctas(const PsiConst& P, int num_sms);
int psi1_bwd_rows(const PsiConst& P, int num_sms);
bool psi1_tile_supported(const PsiConst& P, bool bwd);
// tcgen05 psi1 (psi1_tc.cu): M <= 128, D <= 128 forward / D <= 64 backward; SGPX_PSI1=simt disables
bool psi1_tc_supported(const PsiConst& P, bool bwd);
int psi1_tc_rows(const PsiConst& P, int num_sms, bool bwd);
int psi1_tc_forward(const PsiConst& P, double* part, int64_t pstride, int rows, int* err_flag, int with_kl,
                    void* stream);
int psi1_tc_backward(const PsiConst& P, const BwdConst& B, double* part, int64_t pstride, int rows, void* stream);
int psi1_tile_rows(const PsiConst& P, int num_sms);
int psi1_tile_forward(const PsiConst& P, double* part, int64_t pstride, int rows, int* err_flag, int with_kl,
                      void* stream);
int psi1_tile_backward(const PsiConst& P, const BwdConst& B, double* part, int64_t pstride, int rows, void* stream);
int psi1_forward(const PsiConst& P, double* part_rows, int64_t pstride, int rows, int* err_flag, void* stream,
                 int with_kl);
int psi1_backward(const PsiConst& P, const BwdConst& B, double* part_rows, int64_t pstride, int rows, void* stream);
// Row-tile tensor-core psi2 (psi_rowtile.cu).  rt_forward writes Phi into packed[4 + p] (run it
// after the psi1 reduce) and keeps the per-pair gradient sums + feature arrays in `base`
// (rt_fwd_doubles) for rt_backward, which accumulates the psi2 parts of d_mu / d_s and writes the
// pair part of [dvar, dl, dz] (+ the datapoint part of dl) into the partial row `prow`.
bool rt_supported(const PsiConst& P);
bool use_rt(const PsiConst& P);
int64_t rt_fwd_doubles(const PsiConst& P, int num_sms);
int64_t rt_bwd_doubles(const PsiConst& P, int num_sms);
int rt_forward(const PsiConst& P, double* base, double* packed, int num_sms, void* stream);
int rt_backward(const PsiConst& P, const BwdConst& B, double* bbase, double* prow, int num_sms, void* stream);
double* rt_fwd_pair_sums(const PsiConst& P, double* region, int num_sms, int64_t* count);
const float* rt_fwd_pair_operand(const PsiConst& P, const double* region, int num_sms);
int rt_bwd_prepare(const PsiConst& P, const float* u, double* bbase, int num_sms, void* stream, const float** pre,
                   const float** ys);
// the row-tile backward's region inside psi_backward's partial buffer `part` (after the psi1 rows)
double* bwd_rt_region(const PsiConst& P, double* part, int num_sms);
// Direct-difference kernels (psi_direct.cu): the complete forward (validation, yy, KL, Phi, Psi) and
// backward (d mu, d S, d Z, d l, d var) with fp64 exponents.
bool direct_supported(const PsiConst& P);
int64_t direct_fwd_doubles(const PsiConst& P, int num_sms);
int64_t direct_bwd_doubles(const PsiConst& P, int num_sms);
int direct_forward(const PsiConst& P, double* base, double* packed, int* err_flag, int with_kl, int num_sms,
                   void* stream);
int direct_backward(const PsiConst& P, const BwdConst& B, double* bbase, double* packed, int num_sms, void* stream);
double* direct_fwd_pair_sums(const PsiConst& P, double* base, int num_sms, int64_t* count);
// Knm-tile SYRK path for deterministic inputs (syrk.cu).
bool syrk_supported(const PsiConst& P);
int64_t syrk_fwd_doubles(const PsiConst& P, int num_sms);
int64_t syrk_bwd_doubles(const PsiConst& P, int num_sms);
int syrk_forward(const PsiConst& P, double* base, double* packed, int* err_flag, int num_sms, void* stream);
int syrk_backward(const PsiConst& P, const BwdConst& B, double* base, double* packed, int num_sms, void* stream);
// Fixed-order reduction of backward partial rows into packed grads.
// tmp: bwd_reduce_tmp_doubles(pstride) doubles of scratch.
int64_t bwd_reduce_tmp_doubles(int64_t pstride);
int bwd_reduce_rows(const double* part, int64_t pstride, int rows, double* packed, double dvar0, double* tmp,
                    void* stream);

// Seeded inputs and binary matrices (synth.cu): Rng(seed).normal_matrix on the device (column-major,
// ld), the init_gplvm partial Fisher-Yates row choice, the io.hpp binary format (host read / write and
// a streamed device loader).  IO failures throw IoError.
int rng_normal_device(uint64_t seed, int64_t rows, int64_t cols, double* out, int64_t ld, void* stream);
void rng_choose_rows(uint64_t seed, int64_t n, int64_t m, int64_t* idx_out);
void io_read_shape(const char* base, int64_t* rows, int64_t* cols);
void io_read_host(const char* base, double* out, int64_t ld);
void io_write_host(const char* base, const double* a, int64_t rows, int64_t cols, int64_t ld);
void io_load_device(const char* base, double* dev_out, int64_t ld, void* stream);

// psi1_expected: out n x m col-major fp64 (ld_out).
int psi1_matrix(const PsiConst& P, double* out, int64_t ld_out, void* stream);
// Number of __global__ launches issued so far by this process (evidence counter); graph replays add
// their kernel count through launches_add.
int64_t launches_issued();
void launches_add(int64_t n);

}  // namespace sgpx
