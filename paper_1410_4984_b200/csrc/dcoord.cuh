// dcoord.cuh -- the coordinator of Engine::evaluate on the device (dcoord.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace sgpx {

// Scalar slots of the coordinator workspace (fp64, device).
enum DcScalar {
  kScLogDetK = 0,        // log |Kmm + jitter|
  kScJitterFactor = 1,   // factor_gram's jitter factor used
  kScLogDetA = 2,        // log |A|
  kScShiftA = 3,         // factor_spd's shift factor used
  kScStatus = 4,         // DcStatus bits of this evaluation
  kScStatusK = 5,        // DcStatus bits of the per-broadcast prefactor
  kScPg = 6,             // <Psi, G>
  kScKp = 7,             // <Kmm^-1, Phi>
  kScAp = 8,             // <A^-1, Phi>
  kScDPhi = 9,           // d phi
  kScBound = 10,         // 7 entries: total, log_det, data_fit, quadratic, trace_phi, trace_kmm, kl
  kScCount = 17
};
enum DcStatus { kStGramFailed = 1, kStAFailed = 2, kStNonFinite = 4, kStBadCount = 8, kStBadStats = 16 };

struct DcArgs {
  int m, mv, q, d, latent;
  int64_t n;                       // global N
  double var, beta, jitter_factor;
  const double* z;                 // M x Q column-major (device)
  const double* ls;                // Q (device)
  const double* packed;            // reduced packed statistics (sgpx.h layout, device)
  double *kmm, *lk, *wk, *kinv;    // per broadcast
  double *a, *la, *wa, *ainv, *phi, *g, *ggt, *tmp, *kpk, *phig, *dkmm, *w, *rs, *wz;
  double* sc;                      // kScCount scalars
  int* info;                       // [0] Kmm Cholesky, [1] A Cholesky
  double* result;                  // [d var, d l (Q), d Z (M Q), d beta]
};

// Workspace doubles for (m, q, d): the matrices above, packed back to back.
int64_t dc_workspace_doubles(int m, int q, int d);
// Point every array of `A` into `ws` (dc_workspace_doubles long); the int slots follow the doubles.
void dc_bind(DcArgs& A, double* ws);

int dc_upload_ls(const DcArgs& A, const double* ls, cudaStream_t st);  // A.ls <- ls (by value, Q <= 64)
int dc_prefactor(const DcArgs& A, cudaStream_t st);                 // per broadcast
// after allreduce #1: the bound terms and the backward's adjoint operands (fp32 + fp64)
int dc_bound(const DcArgs& A, float* u, float* dpsi, double* u64, double* dpsi64, cudaStream_t st);
// dc_bound + dc_deferred with the backward's psi1 operand first: on `st` A's factorisation and
// G = A^-1 Psi (d Psi ready when ev[0] fires); on `side2` (from ev[2], recorded on `st` first)
// Kmm^-1 Phi Kmm^-1 (ev[3]); on `side` (after ev[0]) L^-1, A^-1, G G^T, the bound terms and d Phi,
// then (after ev[3]) d Kmm, Phi G and the kern_grads terms, done when ev[1] fires -- the caller runs
// the psi1 backward kernels in between and makes `st` wait for ev[1] before the psi2 backward and the
// finish.  M > 112 (or no side streams): everything on `st`, ev[0] and ev[1] recorded after it.
int dc_bound_split(const DcArgs& A, float* u, float* dpsi, double* u64, double* dpsi64, cudaStream_t st,
                   cudaStream_t side, cudaStream_t side2, cudaEvent_t* ev);
int dc_deferred(const DcArgs& A, cudaStream_t st);                  // d Kmm, Phi G (before finish)
int dc_finish(const DcArgs& A, const double* pgrads, cudaStream_t st);  // after allreduce #2

// Prediction from the factors of the last coordination (predict_from_cache, model.hpp:197-217):
// xs T x Q (device, column-major), mean / var T x D (device); work: dc_predict_doubles.
int64_t dc_predict_doubles(int64_t t, int m, int q, int d);
int dc_predict(const DcArgs& A, const double* xs, int64_t t, int obs, double* work, double* mean, double* var,
               cudaStream_t st);

}  // namespace sgpx
