// psi1_tc.cu -- psi1 statistics and gradients with the D-wide contractions on tcgen05 (M <= 128).
//
// Reference: psi_stats.hpp:144-219 (psi1 block of the sweep: Psi += v1^T Y, and its adjoint).
// With log2 v1_nm = b1_n - (log2e / 2) sum_q d1_nq (mu_nq - z_mq)^2, d1 = 1 / (S + l^2) and mu, z
// translated by the mean of Z (the weights come out of SIMT direct differences, fp32, MUFU.EX2):
//
//   forward  (psi1_fwd_tc_kernel): per chunk of kFwdK datapoints the CTA forms G^T = v1^T
//            (128 inducing rows x kFwdK) and the Y chunk (D rows x kFwdK) in shared memory as tf32
//            hi/lo pieces and accumulates  Psi (128 x D) += G^T Y  in TMEM with three kind::tf32 MMAs
//            per K-step (hi.hi + hi.lo + lo.hi, ~fp32 products).  The accumulator is drained into fp64
//            registers every kGroup chunks (fp32 sums over kGroup * kFwdK = 64 datapoints).
//   backward (psi1_bwd_tc_kernel): per chunk of 128 datapoints  C (128 x M) = Y dPsi^T  (K = D) by
//            the same three-pass tf32 MMA, then a thread per (datapoint, half of the inducing points)
//            reads its C row from TMEM and forms G_nm = v1_nm C_nm with the per-datapoint sums
//            T_n = sum_m G_nm [1, z_m, z_m^2] in registers; R_mk = sum_n G_nm [d1 mu, d1]_nk from a
//            shared G tile; both finish as in psi1_tile.cu (d mu, d S, d l, d var; d Z = R - z R').
//
// Both write the same CTA-private partial rows as the SIMT tile kernels (psi1_tile.cu), which stay
// the path for shapes these do not take (M > 128, D > 128 forward / D > 64 backward).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "psi_common.cuh"
#include "psi_kernels.cuh"
#include "tc_util.cuh"

namespace sgpx {
extern std::atomic<int64_t> g_tc_launches;

namespace {
using namespace dev;

constexpr int kFwdK = 32;   // datapoints per forward chunk (MMA K)
constexpr int kBwdN = 128;  // datapoints per backward chunk (MMA M, TMEM lanes)

__host__ __device__ inline int fwd_dp(int d) { return (d + 15) / 16 * 16; }  // MMA N (Psi columns)

// ---------------------------------------------------------------------------------------------
// cp.async (LDGSTS) staging of raw fp64 rows: 8-byte copies, zero-filled when out of range
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(tc::smem_u32(dst)), "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// 2D TMA tile load (box [outer][inner] of a column-major fp64 matrix, rows past N zero-filled)
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(tc::smem_u32(mbar))
      : "memory");
}

// ---------------------------------------------------------------------------------------------
// forward: warp-specialised.  Producer warps (kFwdProd) copy each chunk's raw fp64 rows kRaw - 1 chunks
// ahead (2D TMA boxes, else 8-byte cp.async), convert them into a stage (per-datapoint mu - c, d1, 1/2 log2(d1 l^2); the Y
// chunk as tf32 pieces), and arrive on stage_full; consumer warps (kFwdCons) build the G^T tile of
// the chunk from the stage, and one of them issues the MMAs, whose commit (mma_done) frees the stage
// and the G buffer.  Two stages, two G buffers, two TMEM accumulators.
constexpr int kFwdCons = 256, kFwdProd = 256, kFwdThreads = kFwdCons + kFwdProd;
constexpr int kRaw = 4;  // raw-row buffers: copies run kRaw - 1 chunks ahead of the conversion
struct FwdSmem {  // byte offsets
  int g, y, raw, pd, bar, total;
  int raw_stride;  // bytes per raw buffer: mu [q][kFwdK], S [q][kFwdK], Y [d][kFwdK] doubles
  int pd_stride;   // bytes per stage of per-datapoint floats: a, -b, 1/2 log2(d1 l^2) [3][q][kFwdK]
};
__host__ __device__ inline FwdSmem fwd_smem(int q, int d) {
  FwdSmem L{};
  const int dp = fwd_dp(d);
  L.g = 0;                                     // [stage][piece][128 x kFwdK] floats
  L.y = L.g + 2 * 2 * 128 * kFwdK * 4;         // [stage][piece][dp x kFwdK] floats
  L.raw_stride = (2 * q + d) * kFwdK * 8;
  L.raw = L.y + 2 * 2 * dp * kFwdK * 4;        // [kRaw] raw rows
  L.pd_stride = 3 * q * kFwdK * 4;
  L.pd = L.raw + kRaw * L.raw_stride;          // [stage]
  L.bar = (L.pd + 2 * L.pd_stride + 15) / 16 * 16;  // stage_full[2], mma_done[2], raw_full[kRaw], TMEM slot
  L.total = L.bar + 8 * (4 + kRaw) + 16;
  return L;
}

// NB8: 8-column TMEM blocks drained per consumer thread (the 2 consumer warps of a lane quarter
// split the Psi columns).  Two TMEM accumulators (columns 0 / 128) alternate per aligned group of
// kGroup consecutive chunks (fp32 sums over kGroup * kFwdK datapoints, the same datapoints whatever
// the grid or sub-shard split); the previous group is drained into fp64 while the next one fills.
constexpr int kGroup = 2;
template <int Q, int NB8>
__global__ void __launch_bounds__(kFwdThreads, 1)
    psi1_fwd_tc_kernel(PsiConst P, int64_t nchunks, double* __restrict__ part, int64_t pstride, int* err_flag,
                       int with_kl, int bulk, const __grid_constant__ CUtensorMap tm_mu,
                       const __grid_constant__ CUtensorMap tm_s, const __grid_constant__ CUtensorMap tm_y) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = P.d, m = P.m, dp = fwd_dp(d);
  const FwdSmem L = fwd_smem(Q, d);
  float* gsm = reinterpret_cast<float*>(smem + L.g);
  float* ysm = reinterpret_cast<float*>(smem + L.y);
  uint64_t* stage_full = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* mma_done = stage_full + 2;
  uint64_t* raw_full = stage_full + 4;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L.bar + 8 * (4 + kRaw));
  for (int i = tid; i < 2 * 2 * dp * kFwdK; i += kFwdThreads) ysm[i] = 0.f;  // rows d >= D stay zero
  if (tid == 0) {
    tc::mbar_init(&stage_full[0], kFwdProd);
    tc::mbar_init(&stage_full[1], kFwdProd);
    tc::mbar_init(&mma_done[0], 1);
    tc::mbar_init(&mma_done[1], 1);
    for (int i = 0; i < kRaw; ++i) tc::mbar_init(&raw_full[i], 1);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(tslot, 256);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  // aligned groups of kGroup consecutive chunks: CTA b takes groups b, b + grid, ...
  const int64_t ngroups = (nchunks + kGroup - 1) / kGroup;
  const int64_t nlocal = blockIdx.x < ngroups ? ((ngroups - 1 - blockIdx.x) / gridDim.x + 1) * kGroup : 0;
  auto chunk_of = [&](int64_t l) { return (blockIdx.x + (l / kGroup) * int64_t(gridDim.x)) * kGroup + l % kGroup; };
  double yy_acc = 0.0, kl_acc = 0.0;
  __shared__ double red[2][kFwdThreads / 32];

  if (tid >= kFwdCons) {
    // ---------------- producers ----------------
    const int pt = tid - kFwdCons;
    // raw rows of a chunk (mu [Q], S [Q], Y [D] rows of kFwdK doubles): one 1D bulk (TMA) copy per row
    // when every row start is 16-byte aligned (`bulk`), else 8-byte cp.async; rows past N are not
    // read (the conversion masks them)
    auto prefetch = [&](int64_t chunk, int rb) {
      double* raw = reinterpret_cast<double*>(smem + L.raw + rb * L.raw_stride);
      const int64_t n0 = chunk * kFwdK;
      const int cnt = chunk < nchunks ? int(min(int64_t(kFwdK), P.n - n0)) : 0;
      const int nrows = 2 * Q + d;
      if (bulk) {  // three 2D TMA boxes: mu [q][kFwdK], S [q][kFwdK], Y [d][kFwdK]
        (void)cnt;
        if (pt == 0) {
          const uint32_t bytes = uint32_t(kFwdK * 8) * uint32_t(P.q * (P.expected ? 2 : 1) + d);
          tc::mbar_arrive_expect_tx(&raw_full[rb], bytes);
          const int c0 = int(n0);
          tma_2d(raw, &tm_mu, c0, 0, &raw_full[rb]);
          if (P.expected) tma_2d(raw + Q * kFwdK, &tm_s, c0, 0, &raw_full[rb]);
          tma_2d(raw + 2 * Q * kFwdK, &tm_y, c0, 0, &raw_full[rb]);
        }
      } else {
        const int tot = nrows * kFwdK;
        for (int i = pt; i < tot; i += kFwdProd) {
          const int nl = i % kFwdK, r = i / kFwdK;
          const int64_t n = n0 + nl;
          const bool ok = nl < cnt;
          const double* src;
          bool v = ok;
          if (r < Q) {
            v = ok && r < P.q;
            src = P.mu + int64_t(v ? r : 0) * P.ld_mu + (ok ? n : 0);
          } else if (r < 2 * Q) {
            v = ok && r - Q < P.q && P.expected;
            src = v ? P.s + int64_t(r - Q) * P.ld_s + n : P.mu;
          } else {
            src = P.y + int64_t(r - 2 * Q) * P.ld_y + (ok ? n : 0);
          }
          cp_async8(raw + i, src, v);
        }
        cp_commit();
      }
    };
    for (int i = 0; i < kRaw - 1; ++i) prefetch(i < nlocal ? chunk_of(i) : nchunks, i);
    for (int64_t l = 0; l < nlocal; ++l) {
      const int st = int(l & 1), rb = int(l % kRaw);
      const int64_t n0 = chunk_of(l) * kFwdK;
      tc::named_sync(1, kFwdProd);  // every producer is done with the raw buffer the next copy fills
      const int64_t ahead = l + kRaw - 1;
      prefetch(ahead < nlocal ? chunk_of(ahead) : nchunks, int(ahead % kRaw));
      if (bulk) {
        tc::mbar_wait(&raw_full[rb], uint32_t((l / kRaw) & 1));
      } else {
        cp_wait<kRaw - 1>();
        tc::named_sync(1, kFwdProd);  // chunk l's rows landed (all producers' copies)
      }
      if (l >= 2) tc::mbar_wait(&mma_done[st], uint32_t(((l - 2) >> 1) & 1));  // stage st consumed
      const double* raw = reinterpret_cast<const double*>(smem + L.raw + rb * L.raw_stride);
      float* pd = reinterpret_cast<float*>(smem + L.pd + st * L.pd_stride);
      int bad = 0;
#pragma unroll 2
      for (int i = pt; i < kFwdK * Q; i += kFwdProd) {  // psi_stats.hpp:144-159, validation, KL partial
        const int nl = i % kFwdK, q = i / kFwdK;
        const int64_t n = n0 + nl;
        // log2 v1 = b1 - sum_q (a - b z)^2 with b = sqrt(log2e d1 / 2), a = b (mu - c): the direct
        // difference d1 (mu - z)^2 log2e / 2 as one FFMA per term (see psi1_bwd_pipe_kernel)
        float a = 0.f, nb = 0.f, cl = 0.f;
        if (q < P.q && n < P.n) {
          const double md = raw[q * kFwdK + nl];
          const double sd = P.expected ? raw[(Q + q) * kFwdK + nl] : 0.0;
          bad |= isfinite(md) ? 0 : 1;
          if (P.expected) {
            bad |= (sd > 0.0 && isfinite(sd)) ? 0 : 4;
            kl_acc += 0.5 * (sd + md * md - log(sd) - 1.0);  // parallel.hpp:148-149
          }
          const float mu = float(md - P.center[q]);
          const float d1 = 1.f / (float(sd) + P.l2[q]);
          const float bq = sqrtf(0.5f * kLog2e * d1);
          a = bq * mu;
          nb = -bq;
          cl = 0.5f * log2f(d1 * P.l2[q]);
        }
        pd[q * kFwdK + nl] = a;
        pd[(Q + q) * kFwdK + nl] = nb;
        pd[(2 * Q + q) * kFwdK + nl] = cl;
      }

      float* yb = ysm + st * 2 * dp * kFwdK;  // the Y chunk as tf32 pieces: rows = output dims, K = datapoints
      // rotated start: the producers that took a second (datapoint, q) item above get the fewest Y items
      const int pr = (pt + kFwdProd - (kFwdK * Q) % kFwdProd) % kFwdProd;
#pragma unroll 4
      for (int i = pr; i < kFwdK * d; i += kFwdProd) {
        const int nl = i % kFwdK, dd = i / kFwdK;
        const double y = n0 + nl < P.n ? raw[(2 * Q + dd) * kFwdK + nl] : 0.0;
        bad |= isfinite(y) ? 0 : 1;
        yy_acc += y * y;
        const float f = float(y), hi = tc::tf32_hi(f);
        const int o = tc::canon(dd, nl, kFwdK);
        yb[o] = hi;
        yb[dp * kFwdK + o] = f - hi;
      }
      if (with_kl && bad) atomicOr(err_flag, bad);  // validation (psi_stats.hpp:119-120)
      tc::fence_async_smem();
      tc::mbar_arrive(&stage_full[st]);
    }
  } else {
    // ---------------- consumers ----------------
    // G^T tile: thread = inducing points {gm, gm + 64} x datapoints 8 gj .. 8 gj + 7 (16-byte stores)
    const int gm = tid & 63, gj = tid >> 6;
    float z[2][Q];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int q = 0; q < Q; ++q) z[i][q] = (q < P.q && gm + 64 * i < m) ? P.zc[(gm + 64 * i) * P.qv + q] : 0.f;
    // drain ownership: lane quarter wq (TMEM lanes = Psi rows m), column half wh
    const int wq = warp & 3, wh = warp >> 2;
    const int cw = dp / 2, row = 32 * wq + lane, c0 = wh * cw;
    double acc[NB8][8];
#pragma unroll
    for (int b = 0; b < NB8; ++b)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[b][j] = 0.0;
    const uint32_t idesc = tc::idesc_tf32(128, dp);
    auto drain = [&](int64_t group) {  // the group's MMAs are complete; add its accumulator into fp64
      const uint32_t base = tmem + (uint32_t(32 * wq) << 16) + uint32_t((group & 1) * 128);
#pragma unroll
      for (int b = 0; b < NB8; ++b) {
        if (8 * b < cw) {
          uint32_t r[8];
          tc::ld8(base + uint32_t(c0 + 8 * b), r);
          tc::ld_wait();
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[b][j] += double(__uint_as_float(r[j]));
        }
      }
    };
    for (int64_t l = 0; l < nlocal; ++l) {
      const int st = int(l & 1);
      const int64_t group = l / kGroup;
      if (l >= 2) {  // G buffer st free (chunk l - 2's MMAs done); the previous group complete
        tc::mbar_wait(&mma_done[st], uint32_t(((l - 2) >> 1) & 1));
        tc::fence_after();
        if (l % kGroup == kGroup - 1 && group >= 1) drain(group - 1);
      }
      tc::mbar_wait(&stage_full[st], uint32_t((l >> 1) & 1));
      const float* pd = reinterpret_cast<const float*>(smem + L.pd + st * L.pd_stride);
      float* gb = gsm + st * 2 * 128 * kFwdK;
      {
        float b[8], e[2][8];
        {  // b1 = log2 var + sum_q 1/2 log2(d1 l^2) (rows past N: -inf), formed once per warp: every lane
           // of a warp shares the 8 datapoints of gj; lane = (datapoint lane & 7, latent dims q = lane >> 3
           // mod 4), two butterfly steps, then the 8 sums are broadcast
          const int64_t n0 = chunk_of(l) * kFwdK;
          float bs = 0.f;
#pragma unroll
          for (int q = lane >> 3; q < Q; q += 4) bs += pd[(2 * Q + q) * kFwdK + 8 * gj + (lane & 7)];
          bs += __shfl_xor_sync(0xffffffffu, bs, 8);
          bs += __shfl_xor_sync(0xffffffffu, bs, 16);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            b[u] = P.log2_var + __shfl_sync(0xffffffffu, bs, u);
            if (n0 + 8 * gj + u >= P.n) b[u] = -CUDART_INF_F;
          }
        }
        float2 e2[2][4];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int u = 0; u < 4; ++u) e2[i][u] = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          float2 av[4], nv[4];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float4 a4 = *reinterpret_cast<const float4*>(pd + q * kFwdK + 8 * gj + 4 * h);
            const float4 n4 = *reinterpret_cast<const float4*>(pd + (Q + q) * kFwdK + 8 * gj + 4 * h);
            av[2 * h] = make_float2(a4.x, a4.y), av[2 * h + 1] = make_float2(a4.z, a4.w);
            nv[2 * h] = make_float2(n4.x, n4.y), nv[2 * h + 1] = make_float2(n4.z, n4.w);
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const float2 zz = make_float2(z[i][q], z[i][q]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float2 t = __ffma2_rn(nv[u], zz, av[u]);
              e2[i][u] = __ffma2_rn(t, t, e2[i][u]);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            e[i][2 * u] = e2[i][u].x;
            e[i][2 * u + 1] = e2[i][u].y;
          }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int mm = gm + 64 * i;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float hv[4], lv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float g = mm < m ? ex2(b[4 * h + u] - e[i][4 * h + u]) : 0.f;
              hv[u] = tc::tf32_hi(g);
              lv[u] = g - hv[u];
            }
            const int o = tc::canon(mm, 8 * gj + 4 * h, kFwdK);
            *reinterpret_cast<float4*>(gb + o) = make_float4(hv[0], hv[1], hv[2], hv[3]);
            *reinterpret_cast<float4*>(gb + 128 * kFwdK + o) = make_float4(lv[0], lv[1], lv[2], lv[3]);
          }
        }
      }
      tc::fence_async_smem();
      tc::fence_before();
      tc::named_sync(2, kFwdCons);  // G tile complete; the drain's TMEM reads are done
      if (warp == 0) {
        tc::fence_after();
        const float* yb = ysm + st * 2 * dp * kFwdK;
        const uint32_t ga = tc::smem_u32(gb), ya = tc::smem_u32(yb);
        const uint32_t glo = ga + 128 * kFwdK * 4, ylo = ya + dp * kFwdK * 4;
        const uint32_t dt = tmem + uint32_t((group & 1) * 128);
        const bool first = l % kGroup == 0;
#pragma unroll
        for (int ks = 0; ks < kFwdK / 8; ++ks) {
          const uint32_t o = uint32_t(ks) * 256;
          tc::mma_ss_w(dt, tc::desc(ga + o, kFwdK), tc::desc(ya + o, kFwdK), idesc, first && ks == 0 ? 0u : 1u);
          tc::mma_ss_w(dt, tc::desc(ga + o, kFwdK), tc::desc(ylo + o, kFwdK), idesc, 1u);
          tc::mma_ss_w(dt, tc::desc(glo + o, kFwdK), tc::desc(ya + o, kFwdK), idesc, 1u);
        }
        tc::commit_w(&mma_done[st]);
      }
    }
    if (nlocal > 0) {
      const int64_t last = nlocal - 1, glast = last / kGroup;  // nlocal is a multiple of kGroup
      tc::mbar_wait(&mma_done[last & 1], uint32_t((last >> 1) & 1));
      tc::fence_after();
      drain(glast);  // (the previous group was drained at the top of chunk `last`)
    }
    // the CTA's partial row: Psi (m + d M)
    double* const psi_part = part + int64_t(blockIdx.x) * pstride + 2 + int64_t(m) * (m + 1) / 2;
#pragma unroll
    for (int b = 0; b < NB8; ++b)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int col = c0 + 8 * b + j;
        if (8 * b + j < cw && col < d && row < m) psi_part[row + int64_t(col) * m] = acc[b][j];
      }
  }
  yy_acc = warp_sum_d(yy_acc);
  kl_acc = warp_sum_d(kl_acc);
  if (lane == 0) {
    red[0][warp] = yy_acc;
    red[1][warp] = kl_acc;
  }
  tc::fence_before();
  __syncthreads();
  if (tid == 0) {
    double s = 0.0, k = 0.0;
    for (int i = 0; i < kFwdThreads / 32; ++i) {
      s += red[0][i];
      k += red[1][i];
    }
    double* const cta_part = part + int64_t(blockIdx.x) * pstride;
    cta_part[0] = s;
    if (with_kl) cta_part[1] = k;
  }
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 256);
  }
}

// ---------------------------------------------------------------------------------------------
// backward: 512 threads; consumers = 4 warps per TMEM lane quarter, each a quarter of the inducing
// points.  The G tile of the R phase reuses the Y-piece region (free once the C MMA completed).
constexpr int kBwdThreads = 512;
struct BwdSmem {  // byte offsets
  int ya, pb, zs, hs, ts, mus, d1s, bar, total;
  int dk, mp, gst;
};
__host__ __device__ inline BwdSmem bwd_smem(int q, int d, int m) {
  BwdSmem L{};
  L.dk = (d + 7) / 8 * 8;
  L.mp = (m + 31) / 32 * 32;
  L.gst = L.mp + 1;
  const int nh = 1 + 2 * q;
  const int ya_bytes = 2 * kBwdN * L.dk * 4, gs_bytes = kBwdN * L.gst * 4, rsh_bytes = 2 * q * 128 * 8;
  L.ya = 0;                                               // [piece][128 x dk]; later G [128][mp + 1]
  int big = ya_bytes > gs_bytes ? ya_bytes : gs_bytes;
  big = big > rsh_bytes ? big : rsh_bytes;
  L.pb = (big + 127) / 128 * 128;                         // [piece][mp x dk]
  L.zs = L.pb + 2 * L.mp * L.dk * 4;                      // z [q][mp] and z^2 [q][mp]
  L.hs = L.zs + 2 * q * L.mp * 4;                         // H [128][2 q4]: d1 mu at 0, d1 at q4 (q4 = q rounded to 4)
  L.ts = L.hs + kBwdN * 2 * ((q + 3) / 4 * 4) * 4;        // T quarters [4][128][nh]
  L.mus = L.ts + 4 * kBwdN * nh * 4;                      // [q][128]
  L.d1s = L.mus + q * kBwdN * 4;
  L.bar = (L.d1s + q * kBwdN * 4 + 15) / 16 * 16;
  L.total = L.bar + 32;
  return L;
}

template <int Q>
__global__ void __launch_bounds__(kBwdThreads, 1)
    psi1_bwd_tc_kernel(PsiConst P, BwdConst B, int64_t nchunks, double* __restrict__ part, int64_t pstride) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int NH = 1 + 2 * Q, Q4 = (Q + 3) / 4 * 4, NT = kBwdThreads;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = P.d, m = P.m;
  const BwdSmem L = bwd_smem(Q, d, m);
  const int dk = L.dk, mp = L.mp, gst = L.gst;
  float* ya = reinterpret_cast<float*>(smem + L.ya);
  float* gs = reinterpret_cast<float*>(smem + L.ya);  // after the C MMA
  float* pb = reinterpret_cast<float*>(smem + L.pb);
  float* zs = reinterpret_cast<float*>(smem + L.zs);
  float* hs = reinterpret_cast<float*>(smem + L.hs);
  float* ts = reinterpret_cast<float*>(smem + L.ts);
  float* mus = reinterpret_cast<float*>(smem + L.mus);
  float* d1s = reinterpret_cast<float*>(smem + L.d1s);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L.bar + 16);
  // static operands: dPsi (rows = inducing points, K = output dims) as tf32 pieces, z and z^2
  for (int i = tid; i < mp * dk; i += NT) {
    const int mm = i / dk, dd = i % dk;
    const float v = (mm < m && dd < d) ? B.dpsi[dd * P.mv + mm] : 0.f;
    const float hi = tc::tf32_hi(v);
    const int o = tc::canon(mm, dd, dk);
    pb[o] = hi;
    pb[mp * dk + o] = v - hi;
  }
  for (int i = tid; i < Q * mp; i += NT) {
    const int q = i / mp, mm = i % mp;
    const float z = (q < P.q && mm < m) ? P.zc[mm * P.qv + q] : 0.f;
    zs[i] = z;
    zs[Q * mp + i] = z * z;
  }
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(tslot, 128);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t idesc = tc::idesc_tf32(128, mp);
  // consumer role: datapoint row cn (TMEM lane), inducing-point quarter ch
  const int wq = warp & 3, ch = warp >> 2, cn = 32 * wq + lane;
  const int mqw = mp / 4, mb0 = ch * mqw;
  // R role: inducing point rm, half rh of H (d1 mu or d1), half rn of each chunk's datapoints
  const int rm = tid & 127, rh = (tid >> 7) & 1, rn = tid >> 8;
  double racc[Q];
#pragma unroll
  for (int k = 0; k < Q; ++k) racc[k] = 0.0;
  // epilogue role: a fixed latent dimension per thread (threads past Q * (NT / Q) idle)
  const int eq = tid % Q;
  const bool ework = tid < Q * (NT / Q);
  double dl_acc = 0.0, dv_acc = 0.0;
  const double inv_var = 1.0 / P.variance_d;
  int64_t local = 0;
  for (int64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, ++local) {
    const int64_t n0 = chunk * kBwdN;
    // Y chunk as tf32 pieces: rows = datapoints, K = output dims (columns past D zero)
    for (int i = tid; i < kBwdN * dk; i += NT) {
      const int nl = i % kBwdN, dd = i / kBwdN;
      const int64_t n = n0 + nl;
      const float f = (n < P.n && dd < d) ? float(__ldg(P.y + dd * P.ld_y + n)) : 0.f;
      const float hi = tc::tf32_hi(f);
      const int o = tc::canon(nl, dd, dk);
      ya[o] = hi;
      ya[kBwdN * dk + o] = f - hi;
    }
    // per-datapoint constants
    for (int i = tid; i < kBwdN * Q; i += NT) {
      const int nl = i % kBwdN, q = i / kBwdN;
      const int64_t n = n0 + nl;
      float mu = 0.f, d1 = 0.f;
      if (q < P.q && n < P.n) {
        const double sd = P.expected ? __ldg(P.s + q * P.ld_s + n) : 0.0;
        mu = float(__ldg(P.mu + q * P.ld_mu + n) - P.center[q]);
        d1 = 1.f / (float(sd) + P.l2[q]);
      }
      mus[q * kBwdN + nl] = mu;
      d1s[q * kBwdN + nl] = d1;
      hs[nl * 2 * Q4 + q] = d1 * mu;
      hs[nl * 2 * Q4 + Q4 + q] = d1;
    }
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    if (warp == 0) {
      tc::fence_after();
      const uint32_t a = tc::smem_u32(ya), b = tc::smem_u32(pb);
      const uint32_t alo = a + kBwdN * dk * 4, blo = b + mp * dk * 4;
      for (int ks = 0; ks < dk / 8; ++ks) {
        const uint32_t o = uint32_t(ks) * 256;
        tc::mma_ss_w(tmem, tc::desc(a + o, dk), tc::desc(b + o, dk), idesc, ks == 0 ? 0u : 1u);
        tc::mma_ss_w(tmem, tc::desc(a + o, dk), tc::desc(blo + o, dk), idesc, 1u);
        tc::mma_ss_w(tmem, tc::desc(alo + o, dk), tc::desc(b + o, dk), idesc, 1u);
      }
      tc::commit_w(&bar[0]);
    }
    // consumer constants while the MMAs run
    float mu[Q], d1[Q];
    float b1 = -CUDART_INF_F;
    {
      const int64_t n = n0 + cn;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        mu[q] = mus[q * kBwdN + cn];
        d1[q] = d1s[q * kBwdN + cn];
      }
      if (n < P.n) {
        b1 = P.log2_var;
#pragma unroll
        for (int q = 0; q < Q; ++q)
          if (q < P.q) b1 += 0.5f * log2f(d1[q] * P.l2[q]);
      }
    }
    tc::mbar_wait(&bar[0], uint32_t(local & 1));
    tc::fence_after();
    __syncthreads();  // every warp past the wait: the Y pieces are dead, G may overwrite them
    // G_nm = v1_nm C_nm over this thread's inducing points, 8 at a time with z / z^2 read as 16-byte
    // vectors (q outer); T_n quarter in registers
    float t0 = 0.f, t1[Q], t2[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) t1[q] = t2[q] = 0.f;
    for (int cb = 0; cb < mqw; cb += 8) {
      const int mb = mb0 + cb;
      uint32_t r[8];
      tc::ld8(tmem + (uint32_t(32 * wq) << 16) + uint32_t(mb), r);
      float e[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) e[j] = 0.f;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const float4 za = *reinterpret_cast<const float4*>(zs + q * mp + mb);
        const float4 zb = *reinterpret_cast<const float4*>(zs + q * mp + mb + 4);
        const float zv[8] = {za.x, za.y, za.z, za.w, zb.x, zb.y, zb.z, zb.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float df = mu[q] - zv[j];
          e[j] = fmaf(df * df, d1[q], e[j]);
        }
      }
      tc::ld_wait();
      float g[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        g[j] = mb + j < m ? __uint_as_float(r[j]) * ex2(fmaf(-0.5f * kLog2e, e[j], b1)) : 0.f;
        gs[cn * gst + mb + j] = g[j];
        t0 += g[j];
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const float4 za = *reinterpret_cast<const float4*>(zs + q * mp + mb);
        const float4 zb = *reinterpret_cast<const float4*>(zs + q * mp + mb + 4);
        const float4 wa = *reinterpret_cast<const float4*>(zs + (Q + q) * mp + mb);
        const float4 wb = *reinterpret_cast<const float4*>(zs + (Q + q) * mp + mb + 4);
        const float zv[8] = {za.x, za.y, za.z, za.w, zb.x, zb.y, zb.z, zb.w};
        const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          t1[q] = fmaf(g[j], zv[j], t1[q]);
          t2[q] = fmaf(g[j], wv[j], t2[q]);
        }
      }
    }
    {
      float* tr = ts + (ch * kBwdN + cn) * NH;
      tr[0] = t0;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        tr[1 + q] = t1[q];
        tr[1 + Q + q] = t2[q];
      }
    }
    tc::fence_before();
    __syncthreads();
    // R_mk += sum_n G_nm H_nk over this thread's half of the datapoints (fp32 over 64 datapoints,
    // fp64 across chunks; the two datapoint halves added in order at the end)
    {
      float rr[Q];
#pragma unroll
      for (int k = 0; k < Q; ++k) rr[k] = 0.f;
      if (rm < m) {
#pragma unroll 2
        for (int nl = rn * (kBwdN / 2); nl < (rn + 1) * (kBwdN / 2); ++nl) {
          const float g = gs[nl * gst + rm];
          const float* hr = hs + nl * 2 * Q4 + rh * Q4;
#pragma unroll
          for (int k4 = 0; k4 < Q4; k4 += 4) {
            const float4 h4 = *reinterpret_cast<const float4*>(hr + k4);
            const float hv[4] = {h4.x, h4.y, h4.z, h4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (k4 + u < Q) rr[k4 + u] = fmaf(g, hv[u], rr[k4 + u]);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < Q; ++k) racc[k] += double(rr[k]);
    }
    // per-datapoint epilogue (psi_stats.hpp:200-219): d mu, d S (+ KL), d l, d var
    if (ework && eq < P.q) {
      const int q = eq;
      for (int nl = tid / Q; nl < kBwdN; nl += NT / Q) {
        const int64_t n = n0 + nl;
        if (n >= P.n) break;
        double p0 = 0.0, p1 = 0.0, p2 = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // the four quarters in order
          const float* tc_ = ts + (c * kBwdN + nl) * NH;
          p0 += double(tc_[0]);
          p1 += double(tc_[1 + q]);
          p2 += double(tc_[1 + Q + q]);
        }
        const double mu_ = mus[q * kBwdN + nl], dd1 = d1s[q * kBwdN + nl];
        const double s = P.expected ? P.s[q * P.ld_s + n] : 0.0, l = P.ls[q];
        const double q1 = mu_ * mu_ * p0 - 2.0 * mu_ * p1 + p2;
        dl_acc += s * dd1 * p0 / l + l * dd1 * dd1 * q1;
        if (q == 0) dv_acc += p0 * inv_var;
        if (B.write_local) {
          double dmu = -dd1 * (mu_ * p0 - p1);
          double ds = -0.5 * dd1 * p0 + 0.5 * dd1 * dd1 * q1;
          if (B.add_kl) {  // KL(q || N(0, I)) enters the bound with a minus sign (parallel.hpp:163-166)
            dmu -= P.mu[q * P.ld_mu + n];
            ds -= 0.5 * (1.0 - 1.0 / s);
          }
          B.d_mu[q * B.ld_g + n] = dmu;
          if (P.expected) B.d_s[q * B.ld_g + n] = ds;
        }
      }
    }
    tc::fence_before();
    __syncthreads();
  }
  // d z_mq = R_mq - z_mq R_m(Q+q)   (psi_stats.hpp:214), exchanged through shared memory: the two
  // datapoint halves of each R_mk added in order
  double* rsh = reinterpret_cast<double*>(smem + L.ya);  // [2Q][128] doubles
  for (int h = 0; h < 2; ++h) {
    if (rn == h)
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        double* p = rsh + (rh * Q + k) * 128 + rm;
        *p = h == 0 ? racc[k] : *p + racc[k];
      }
    __syncthreads();
  }
  __syncthreads();
  double* const rowp = part + int64_t(blockIdx.x) * pstride;
  for (int i = tid; i < m * P.q; i += NT) {
    const int m_ = i % m, q = i / m;
    const double z = zs[q * mp + m_];
    rowp[1 + P.q + m_ + int64_t(q) * m] = rsh[q * 128 + m_] - z * rsh[(Q + q) * 128 + m_];
  }
  // d l, d var: fixed-order block reduction
  __syncthreads();
  double* red = rsh;
  for (int k = 0; k <= P.q; ++k) {
    red[tid] = k < P.q ? (ework && eq == k ? dl_acc : 0.0) : dv_acc;
    __syncthreads();
    for (int w = NT / 2; w > 0; w >>= 1) {
      if (tid < w) red[tid] += red[tid + w];
      __syncthreads();
    }
    if (tid == 0) rowp[k < P.q ? 1 + k : 0] = red[0];
    __syncthreads();
  }
  if (warp == 0) tc::tmem_dealloc(tmem, 128);
}

// ---------------------------------------------------------------------------------------------
// backward, pipelined (psi1_bwd_pipe_kernel; the default where its tiles fit, Q <= 12): the same
// sums as psi1_bwd_tc_kernel with
//   * the raw fp64 rows of the next chunk arriving by 2D TMA while the current one is processed
//     (Y right after its conversion, mu / S once the epilogue has read them) -- the kernel above
//     stalls on every chunk's global loads (ncu: long_scoreboard the top stall);
//   * T_n quarters handed to the epilogue through TMEM (no 43 KB shared-memory quarter table);
//   * the weights from FFMA2 pairs of inducing points,
//         log2 v1_nm = b1_n - sum_q (a_nq - b_nq z_mq)^2,   b = sqrt(log2e d1 / 2),  a = b mu,
//     the same direct difference as (log2e / 2) d1 (mu - z)^2 with one FFMA per term instead of
//     FADD + FMUL + FFMA, and the T / R contractions as FFMA2 as well.
// Per chunk: [wait rows c] convert -> S1 -> (TMA Y c+1, C MMA) -> G phase (weights, G tile, T to
// TMEM) -> S2 -> epilogue (d mu, d S, d l, d var) -> S3 -> (TMA mu / S c+1) -> R phase -> S4.
constexpr int kB2Threads = 512;
struct Bwd2Smem {  // byte offsets
  int ya, pb, zs, hs, cl, rawy, rawms, bar, total;
  int dk, mn, mz, gst, hst;
};
__host__ __device__ inline Bwd2Smem bwd2_smem(int q, int d, int m) {
  Bwd2Smem L{};
  const int q4 = (q + 3) / 4 * 4;
  L.dk = (d + 7) / 8 * 8;
  L.mn = (m + 15) / 16 * 16;                     // C MMA N (rows of the dPsi operand)
  L.mz = (m + 3) / 4 * 4;                        // inducing points in blocks of 4
  L.gst = L.mz + ((4 - L.mz % 32) + 32) % 32;    // G row stride >= mz, = 4 (mod 32): conflict-free 16-byte rows
  L.hst = 4 * q4 + 4;                            // per-datapoint row: d1 mu | d1 | a | b
  const int ya_bytes = 2 * 128 * L.dk * 4, gs_bytes = 128 * L.gst * 4, rsh_bytes = 2 * q * 128 * 8;
  int big = ya_bytes > gs_bytes ? ya_bytes : gs_bytes;
  big = big > rsh_bytes ? big : rsh_bytes;
  L.ya = 0;                                      // Y pieces [2][128 x dk]; then G [128][gst]; finally R exchange
  L.pb = (big + 127) / 128 * 128;                // dPsi pieces [2][mn x dk]
  L.zs = L.pb + 2 * L.mn * L.dk * 4;             // z [q][mz], z^2 [q][mz]
  L.hs = L.zs + 2 * q * L.mz * 4;                // [128][hst]
  L.cl = L.hs + 128 * L.hst * 4;                 // [4][128]: partial sums of 1/2 log2(d1 l^2) per datapoint
  L.rawy = (L.cl + 4 * 128 * 4 + 127) / 128 * 128;  // TMA box: Y [d][128] doubles
  L.rawms = L.rawy + d * 128 * 8;                // TMA boxes: mu [q][128], S [q][128] doubles
  L.bar = L.rawms + 2 * q * 128 * 8;
  L.total = L.bar + 64;
  return L;
}
// TMEM column of T component (t1_q, t2_q) within a quarter's block: t0 first, then the latent
// dimensions grouped by q mod 4 (the epilogue warp of subset s reads one contiguous run)
__host__ __device__ constexpr int bwd2_tcol(int Q, int q) {
  int off = 1;
  for (int s = 0; s < (q & 3); ++s) off += 2 * ((Q - s + 3) / 4);
  return off + 2 * (q >> 2);
}
template <int Q>
__host__ __device__ constexpr int bwd2_nhp() { return (1 + 2 * Q + 7) / 8 * 8; }
template <int Q>
__host__ __device__ constexpr int bwd2_tmem_cols() { return 128 + 4 * bwd2_nhp<Q>() + 8 <= 256 ? 256 : 512; }

template <int Q>
__global__ void __launch_bounds__(kB2Threads, 1)
    psi1_bwd_pipe_kernel(PsiConst P, BwdConst B, int64_t nchunks, double* __restrict__ part, int64_t pstride,
                         const __grid_constant__ CUtensorMap tm_mu, const __grid_constant__ CUtensorMap tm_s,
                         const __grid_constant__ CUtensorMap tm_y) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int Q4 = (Q + 3) / 4 * 4, NT = kB2Threads, NHP = bwd2_nhp<Q>(), NQS = (Q + 3) / 4;
  constexpr int TCOLS = bwd2_tmem_cols<Q>();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = P.d, m = P.m, pq = P.q;
  const Bwd2Smem L = bwd2_smem(Q, d, m);
  const int dk = L.dk, mn = L.mn, mz = L.mz, gst = L.gst, hst = L.hst;
  float* ya = reinterpret_cast<float*>(smem + L.ya);
  float* gs = ya;  // after the C MMA
  float* pb = reinterpret_cast<float*>(smem + L.pb);
  float* zs = reinterpret_cast<float*>(smem + L.zs);
  float* hs = reinterpret_cast<float*>(smem + L.hs);
  float* clp = reinterpret_cast<float*>(smem + L.cl);
  double* rawy = reinterpret_cast<double*>(smem + L.rawy);
  double* rawm = reinterpret_cast<double*>(smem + L.rawms);
  double* raws = rawm + Q * 128;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);  // 0 Y landed, 1 mu / S landed, 2 C MMA done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L.bar + 32);
  // static operands: dPsi (rows = inducing points, K = output dims) as tf32 pieces, z and z^2
  for (int i = tid; i < mn * dk; i += NT) {
    const int mm = i / dk, dd = i % dk;
    const float v = (mm < m && dd < d) ? B.dpsi[dd * P.mv + mm] : 0.f;
    const float hi = tc::tf32_hi(v);
    const int o = tc::canon(mm, dd, dk);
    pb[o] = hi;
    pb[mn * dk + o] = v - hi;
  }
  for (int i = tid; i < Q * mz; i += NT) {
    const int q = i / mz, mm = i % mz;
    const float z = (q < pq && mm < m) ? P.zc[mm * P.qv + q] : 0.f;
    zs[i] = z;
    zs[Q * mz + i] = z * z;
  }
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::mbar_init(&bar[2], 1);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(tslot, TCOLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  const int64_t nlocal = blockIdx.x < nchunks ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t ybytes = 128u * 8u * uint32_t(d), msbytes = 128u * 8u * uint32_t(pq * (P.expected ? 2 : 1));
  auto load_y = [&](int64_t l) {
    tc::mbar_arrive_expect_tx(&bar[0], ybytes);
    tma_2d(rawy, &tm_y, int((blockIdx.x + l * gridDim.x) * 128), 0, &bar[0]);
  };
  auto load_ms = [&](int64_t l) {
    const int c0 = int((blockIdx.x + l * gridDim.x) * 128);
    tc::mbar_arrive_expect_tx(&bar[1], msbytes);
    tma_2d(rawm, &tm_mu, c0, 0, &bar[1]);
    if (P.expected) tma_2d(raws, &tm_s, c0, 0, &bar[1]);
  };
  if (tid == 0 && nlocal > 0) {
    load_y(0);
    load_ms(0);
  }
  const uint32_t idesc = tc::idesc_tf32(128, mn);
  // G phase / epilogue role: datapoint cn (TMEM lane), quarter ch (inducing-point blocks ch, ch + 4, ...;
  // latent dimensions ch, ch + 4, ... in the epilogue)
  const int wq = warp & 3, ch = warp >> 2, cn = 32 * wq + lane;
  const uint32_t t_row = tmem + (uint32_t(32 * wq) << 16);
  // R role: inducing point rm, half rh of H (d1 mu or d1), half rn of each chunk's datapoints
  const int rm = tid & 127, rh = (tid >> 7) & 1, rn = tid >> 8;
  double racc[Q];
#pragma unroll
  for (int k = 0; k < Q; ++k) racc[k] = 0.0;
  double dl_acc[NQS];
#pragma unroll
  for (int j = 0; j < NQS; ++j) dl_acc[j] = 0.0;
  double dv_acc = 0.0;
  const double inv_var = 1.0 / P.variance_d;
  const int nb4 = mz / 4;
  int toff = 1;  // this warp's run of (t1, t2) columns in every quarter's block
  for (int s = 0; s < ch; ++s) toff += 2 * ((Q - s + 3) / 4);
  for (int64_t l = 0; l < nlocal; ++l) {
    const int64_t n0 = (blockIdx.x + l * gridDim.x) * 128;
    const uint32_t ph = uint32_t(l & 1);
    tc::mbar_wait(&bar[0], ph);
    tc::mbar_wait(&bar[1], ph);
    // Y -> tf32 pieces (32 consecutive threads fill one core matrix: 8 datapoints x 4 dims)
    for (int i = tid; i < 128 * dk; i += NT) {
      const int kk = i & 3, r8 = (i >> 2) & 7, rest = i >> 5;
      const int nl = (rest & 15) * 8 + r8, dd = (rest >> 4) * 4 + kk;
      const float f = dd < d ? float(rawy[dd * 128 + nl]) : 0.f;
      const float hi = tc::tf32_hi(f);
      const int o = tc::canon(nl, dd, dk);
      ya[o] = hi;
      ya[128 * dk + o] = f - hi;
    }
    // per-datapoint rows (rows past N arrive zero-filled: finite constants, Y = 0 so G = 0); thread tid
    // always takes datapoint tid & 127 (latent dims tid >> 7, + 4, ...) and leaves its part of
    // b1 - log2 var = sum_q 1/2 log2(d1 l^2) in clp[tid >> 7]
    float clsum = 0.f;
    for (int i = tid; i < 128 * Q4; i += NT) {
      const int nl = i & 127, q = i >> 7;
      float mu = 0.f, d1 = 0.f;
      if (q < pq) {
        const double sd = P.expected ? raws[q * 128 + nl] : 0.0;
        mu = float(rawm[q * 128 + nl] - P.center[q]);
        d1 = 1.f / (float(sd) + P.l2[q]);
        clsum += 0.5f * log2f(d1 * P.l2[q]);
      }
      const float bq = sqrtf(0.5f * kLog2e * d1);
      float* h = hs + nl * hst;
      h[q] = d1 * mu;
      h[Q4 + q] = d1;
      h[2 * Q4 + q] = bq * mu;
      h[3 * Q4 + q] = bq;
    }
    clp[tid] = clsum;  // [tid >> 7][tid & 127]  (NT = 512 = 4 x 128)
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();  // S1: Y pieces and rows ready; raw Y consumed
    if (tid == 0 && l + 1 < nlocal) load_y(l + 1);
    if (warp == 0) {
      tc::fence_after();
      const uint32_t a = tc::smem_u32(ya), b = tc::smem_u32(pb);
      const uint32_t alo = a + 128 * dk * 4, blo = b + mn * dk * 4;
      for (int ks = 0; ks < dk / 8; ++ks) {
        const uint32_t o = uint32_t(ks) * 256;
        tc::mma_ss_w(tmem, tc::desc(a + o, dk), tc::desc(b + o, dk), idesc, ks == 0 ? 0u : 1u);
        tc::mma_ss_w(tmem, tc::desc(a + o, dk), tc::desc(blo + o, dk), idesc, 1u);
        tc::mma_ss_w(tmem, tc::desc(alo + o, dk), tc::desc(b + o, dk), idesc, 1u);
      }
      tc::commit_w(&bar[2]);
    }
    // G phase constants while the MMAs run
    float av[Q4], bv[Q4];
    const float b1 = P.log2_var + ((clp[cn] + clp[128 + cn]) + (clp[256 + cn] + clp[384 + cn]));
    {
      const float* h = hs + cn * hst;
#pragma unroll
      for (int k4 = 0; k4 < Q4; k4 += 4) {
        const float4 x = *reinterpret_cast<const float4*>(h + 2 * Q4 + k4);
        const float4 y = *reinterpret_cast<const float4*>(h + 3 * Q4 + k4);
        av[k4] = x.x, av[k4 + 1] = x.y, av[k4 + 2] = x.z, av[k4 + 3] = x.w;
        bv[k4] = y.x, bv[k4 + 1] = y.y, bv[k4 + 2] = y.z, bv[k4 + 3] = y.w;
      }
    }
    tc::mbar_wait(&bar[2], ph);
    tc::fence_after();
    float2 t0 = make_float2(0.f, 0.f), t1[Q], t2[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) t1[q] = t2[q] = make_float2(0.f, 0.f);
    const float2 b12 = make_float2(b1, b1);
    for (int blk = ch; blk < nb4; blk += 4) {
      const int mb = 4 * blk;
      uint32_t r[4];
      tc::ld4(t_row + uint32_t(mb), r);
      float2 e01 = make_float2(0.f, 0.f), e23 = e01;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const float4 z = *reinterpret_cast<const float4*>(zs + q * mz + mb);
        const float2 nb = make_float2(-bv[q], -bv[q]), aa = make_float2(av[q], av[q]);
        const float2 u01 = __ffma2_rn(nb, make_float2(z.x, z.y), aa);
        const float2 u23 = __ffma2_rn(nb, make_float2(z.z, z.w), aa);
        e01 = __ffma2_rn(u01, u01, e01);
        e23 = __ffma2_rn(u23, u23, e23);
      }
      e01 = __fadd2_rn(b12, make_float2(-e01.x, -e01.y));
      e23 = __fadd2_rn(b12, make_float2(-e23.x, -e23.y));
      tc::ld_wait();
      const float2 g01 = __fmul2_rn(make_float2(__uint_as_float(r[0]), __uint_as_float(r[1])),
                                    make_float2(ex2(e01.x), ex2(e01.y)));
      const float2 g23 = __fmul2_rn(make_float2(__uint_as_float(r[2]), __uint_as_float(r[3])),
                                    make_float2(ex2(e23.x), ex2(e23.y)));
      *reinterpret_cast<float4*>(gs + cn * gst + mb) = make_float4(g01.x, g01.y, g23.x, g23.y);
      t0 = __fadd2_rn(t0, g01);
      t0 = __fadd2_rn(t0, g23);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const float4 z = *reinterpret_cast<const float4*>(zs + q * mz + mb);
        const float4 w = *reinterpret_cast<const float4*>(zs + (Q + q) * mz + mb);
        t1[q] = __ffma2_rn(g01, make_float2(z.x, z.y), t1[q]);
        t1[q] = __ffma2_rn(g23, make_float2(z.z, z.w), t1[q]);
        t2[q] = __ffma2_rn(g01, make_float2(w.x, w.y), t2[q]);
        t2[q] = __ffma2_rn(g23, make_float2(w.z, w.w), t2[q]);
      }
    }
    {  // this quarter's T_n -> TMEM columns 128 + ch * NHP (t0, then the latent dims grouped by q mod 4)
      uint32_t w[NHP];
#pragma unroll
      for (int j = 0; j < NHP; ++j) w[j] = 0u;
      w[0] = __float_as_uint(t0.x + t0.y);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        w[bwd2_tcol(Q, q)] = __float_as_uint(t1[q].x + t1[q].y);
        w[bwd2_tcol(Q, q) + 1] = __float_as_uint(t2[q].x + t2[q].y);
      }
#pragma unroll
      for (int c8 = 0; c8 < NHP / 8; ++c8)
        tc::st8(t_row + uint32_t(128 + ch * NHP + 8 * c8), *reinterpret_cast<const uint32_t(*)[8]>(w + 8 * c8));
      tc::st_wait();
    }
    tc::fence_before();
    __syncthreads();  // S2: G tile and every quarter of T complete
    tc::fence_after();
    // per-datapoint epilogue (psi_stats.hpp:200-219): d mu, d S (+ KL), d l, d var for datapoint cn,
    // latent dimensions ch, ch + 4, ...; the four T quarters summed in order in fp64
    {
      const int64_t n = n0 + cn;
      double p0 = 0.0, p1[NQS], p2[NQS];
#pragma unroll
      for (int j = 0; j < NQS; ++j) p1[j] = p2[j] = 0.0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t w0, w[8];
        tc::ld1(t_row + uint32_t(128 + c * NHP), w0);
        tc::ld8(t_row + uint32_t(128 + c * NHP + toff), w);
        tc::ld_wait();
        p0 += double(__uint_as_float(w0));
#pragma unroll
        for (int j = 0; j < NQS; ++j) {
          p1[j] += double(__uint_as_float(w[2 * j]));
          p2[j] += double(__uint_as_float(w[2 * j + 1]));
        }
      }
      if (n < P.n) {
        if (ch == 0) dv_acc += p0 * inv_var;
#pragma unroll
        for (int j = 0; j < NQS; ++j) {
          const int q = ch + 4 * j;
          if (q < pq) {
            const double mu64 = rawm[q * 128 + cn];
            const double s = P.expected ? raws[q * 128 + cn] : 0.0, l = P.ls[q];
            const double mu_ = mu64 - P.center[q];
            const double dd1 = double(hs[cn * hst + Q4 + q]);
            const double q1 = mu_ * mu_ * p0 - 2.0 * mu_ * p1[j] + p2[j];
            dl_acc[j] += s * dd1 * p0 / l + l * dd1 * dd1 * q1;
            if (B.write_local) {
              double dmu = -dd1 * (mu_ * p0 - p1[j]);
              double ds = -0.5 * dd1 * p0 + 0.5 * dd1 * dd1 * q1;
              if (B.add_kl) {  // KL(q || N(0, I)) enters the bound with a minus sign (parallel.hpp:163-166)
                dmu -= mu64;
                ds -= 0.5 * (1.0 - 1.0 / s);
              }
              B.d_mu[q * B.ld_g + n] = dmu;
              if (P.expected) B.d_s[q * B.ld_g + n] = ds;
            }
          }
        }
      }
    }
    __syncthreads();  // S3: raw mu / S consumed
    if (tid == 0 && l + 1 < nlocal) load_ms(l + 1);
    // R_mk += sum_n G_nm H_nk over this thread's half of the datapoints (fp32 over 64 datapoints,
    // fp64 across chunks; the two datapoint halves added in order at the end)
    {
      float2 rr[Q4 / 2];
#pragma unroll
      for (int k = 0; k < Q4 / 2; ++k) rr[k] = make_float2(0.f, 0.f);
      if (rm < m) {
#pragma unroll 2
        for (int nl = rn * 64; nl < rn * 64 + 64; ++nl) {
          const float g = gs[nl * gst + rm];
          const float2 gg = make_float2(g, g);
          const float* hr = hs + nl * hst + rh * Q4;
#pragma unroll
          for (int k4 = 0; k4 < Q4; k4 += 4) {
            const float4 h4 = *reinterpret_cast<const float4*>(hr + k4);
            rr[k4 / 2] = __ffma2_rn(gg, make_float2(h4.x, h4.y), rr[k4 / 2]);
            rr[k4 / 2 + 1] = __ffma2_rn(gg, make_float2(h4.z, h4.w), rr[k4 / 2 + 1]);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < Q; ++k) racc[k] += double((k & 1) ? rr[k / 2].y : rr[k / 2].x);
    }
    tc::fence_before();
    __syncthreads();  // S4: G tile and rows consumed
  }
  // d z_mq = R_mq - z_mq R_m(Q+q)   (psi_stats.hpp:214), exchanged through shared memory: the two
  // datapoint halves of each R_mk added in order
  double* rsh = reinterpret_cast<double*>(smem + L.ya);  // [2Q][128] doubles
  for (int h = 0; h < 2; ++h) {
    if (rn == h)
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        double* p = rsh + (rh * Q + k) * 128 + rm;
        *p = h == 0 ? racc[k] : *p + racc[k];
      }
    __syncthreads();
  }
  double* const rowp = part + int64_t(blockIdx.x) * pstride;
  for (int i = tid; i < m * pq; i += NT) {
    const int m_ = i % m, q = i / m;
    const double z = zs[q * mz + m_];
    rowp[1 + pq + m_ + int64_t(q) * m] = rsh[q * 128 + m_] - z * rsh[(Q + q) * 128 + m_];
  }
  // d l, d var: fixed-order block reduction
  __syncthreads();
  double* red = rsh;
#pragma unroll 1
  for (int k = 0; k <= Q; ++k) {
    if (k < Q && k >= pq) continue;
    double v = 0.0;
    if (k == Q) {
      v = dv_acc;
    } else {
#pragma unroll
      for (int j = 0; j < NQS; ++j)
        if (ch + 4 * j == k) v = dl_acc[j];
    }
    red[tid] = v;
    __syncthreads();
    for (int w = NT / 2; w > 0; w >>= 1) {
      if (tid < w) red[tid] += red[tid + w];
      __syncthreads();
    }
    if (tid == 0) rowp[k < Q ? 1 + k : 0] = red[0];
    __syncthreads();
  }
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, TCOLS);
  }
}

PFN_cuTensorMapEncodeTiled tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(p);
  }();
  return fn;
}

template <int Q>
int launch_fwd(const PsiConst& P, double* part, int64_t pstride, int rows, int* err_flag, int with_kl,
               cudaStream_t st) {
  const FwdSmem L = fwd_smem(Q, P.d);
  const int64_t nchunks = (P.n + kFwdK - 1) / kFwdK;
  if (rows <= 0) return 0;
  const bool wide = fwd_dp(P.d) / 2 > 32;
  auto kern = wide ? psi1_fwd_tc_kernel<Q, 8> : psi1_fwd_tc_kernel<Q, 4>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total) != cudaSuccess) return 3;
  // TMA boxes when every column start is 16-byte aligned and the driver entry point is there
  auto al16 = [](const void* p, int64_t ld) { return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && ld % 2 == 0; };
  CUtensorMap tm[3];
  std::memset(tm, 0, sizeof(tm));
  int bulk = al16(P.mu, P.ld_mu) && (!P.expected || al16(P.s, P.ld_s)) && al16(P.y, P.ld_y) ? 1 : 0;
  if (bulk) {
    auto encode = tensor_map_encoder();
    auto make = [&](CUtensorMap* map, const double* base, int64_t ld, int cols) {
      cuuint64_t dims[2] = {cuuint64_t(P.n), cuuint64_t(cols)};
      cuuint64_t strides[1] = {cuuint64_t(ld) * 8};
      cuuint32_t box[2] = {cuuint32_t(kFwdK), cuuint32_t(cols)};
      cuuint32_t estr[2] = {1, 1};
      return encode && encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    bulk = make(&tm[0], P.mu, P.ld_mu, P.q) && (!P.expected || make(&tm[1], P.s, P.ld_s, P.q)) &&
                   make(&tm[2], P.y, P.ld_y, P.d)
               ? 1
               : 0;
  }
  kern<<<rows, kFwdThreads, L.total, st>>>(P, nchunks, part, pstride, err_flag, with_kl, bulk, tm[0], tm[1], tm[2]);
  g_tc_launches.fetch_add(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// 2D tensor map of a column-major fp64 matrix [n rows x cols] with a box of `box_rows` rows
// (rows past n zero-filled); false when the base / leading dimension is not 16-byte aligned
bool encode_rows(CUtensorMap* map, const double* base, int64_t ld, int64_t n, int cols, int box_rows) {
  auto encode = tensor_map_encoder();
  if (!encode || reinterpret_cast<uintptr_t>(base) % 16 != 0 || ld % 2 != 0) return false;
  cuuint64_t dims[2] = {cuuint64_t(n), cuuint64_t(cols)};
  cuuint64_t strides[1] = {cuuint64_t(ld) * 8};
  cuuint32_t box[2] = {cuuint32_t(box_rows), cuuint32_t(cols)};
  cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool env_bwd_old() {
  const char* e = getenv("SGPX_PSI1_BWD");
  return e && !strcmp(e, "old");
}

// The pipelined backward where it applies (Q <= 12, tiles within 227 KB, TMA-able rows); 1 = not taken
template <int Q>
int launch_bwd_pipe(const PsiConst& P, const BwdConst& B, double* part, int64_t pstride, int rows, cudaStream_t st) {
  if constexpr (Q > 12) {
    return 1;
  } else {
    if (env_bwd_old() || P.d > 64 || P.m > 128) return 1;
    const Bwd2Smem L = bwd2_smem(Q, P.d, P.m);
    if (L.total > 227 * 1024) return 1;
    CUtensorMap tm[3];
    std::memset(tm, 0, sizeof(tm));
    if (!encode_rows(&tm[0], P.mu, P.ld_mu, P.n, P.q, 128) ||
        (P.expected && !encode_rows(&tm[1], P.s, P.ld_s, P.n, P.q, 128)) ||
        !encode_rows(&tm[2], P.y, P.ld_y, P.n, P.d, 128))
      return 1;
    auto kern = psi1_bwd_pipe_kernel<Q>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total) != cudaSuccess) return 3;
    const int64_t nchunks = (P.n + 127) / 128;
    kern<<<rows, kB2Threads, L.total, st>>>(P, B, nchunks, part, pstride, tm[0], tm[1], tm[2]);
    g_tc_launches.fetch_add(1);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
  }
}

template <int Q>
int launch_bwd(const PsiConst& P, const BwdConst& B, double* part, int64_t pstride, int rows, cudaStream_t st) {
  const BwdSmem L = bwd_smem(Q, P.d, P.m);
  const int64_t nchunks = (P.n + kBwdN - 1) / kBwdN;
  if (rows <= 0) return 0;
  const int rc = launch_bwd_pipe<Q>(P, B, part, pstride, rows, st);
  if (rc != 1) return rc;
  auto kern = psi1_bwd_tc_kernel<Q>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total) != cudaSuccess) return 3;
  kern<<<rows, kBwdThreads, L.total, st>>>(P, B, nchunks, part, pstride);
  g_tc_launches.fetch_add(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

#define SGPX_P1TC_DISPATCH(FN, ...)      \
  switch (instantiated_q(P.q)) {         \
    case 1: return FN<1>(__VA_ARGS__);   \
    case 2: return FN<2>(__VA_ARGS__);   \
    case 3: return FN<3>(__VA_ARGS__);   \
    case 4: return FN<4>(__VA_ARGS__);   \
    case 5: return FN<5>(__VA_ARGS__);   \
    case 6: return FN<6>(__VA_ARGS__);   \
    case 8: return FN<8>(__VA_ARGS__);   \
    case 10: return FN<10>(__VA_ARGS__); \
    case 12: return FN<12>(__VA_ARGS__); \
    case 16: return FN<16>(__VA_ARGS__); \
    case 20: return FN<20>(__VA_ARGS__); \
    case 24: return FN<24>(__VA_ARGS__); \
    case 32: return FN<32>(__VA_ARGS__); \
    default: return 1;                   \
  }

bool env_simt() {
  const char* e = getenv("SGPX_PSI1");
  return e && !strcmp(e, "simt");
}

}  // namespace

bool psi1_tc_supported(const PsiConst& P, bool bwd) {
  if (env_simt() || P.m < 1 || P.m > 128 || P.q < 1 || P.d < 1) return false;
  const int q = instantiated_q(P.q);
  if (q <= 0 || q > 32) return false;
  if (bwd) {
    if (P.d > 64) return false;
    return bwd_smem(q, P.d, P.m).total <= 227 * 1024;
  }
  if (fwd_dp(P.d) > 128) return false;
  return fwd_smem(q, P.d).total <= 227 * 1024;
}
int psi1_tc_rows(const PsiConst& P, int num_sms, bool bwd) {
  const int64_t nchunks = (P.n + (bwd ? kBwdN : kFwdK) - 1) / (bwd ? kBwdN : kFwdK);
  return int(std::max<int64_t>(1, std::min<int64_t>(nchunks, int64_t(num_sms))));
}
int psi1_tc_forward(const PsiConst& P, double* part, int64_t pstride, int rows, int* err_flag, int with_kl,
                    void* stream) {
  SGPX_P1TC_DISPATCH(launch_fwd, P, part, pstride, rows, err_flag, with_kl, static_cast<cudaStream_t>(stream))
}
int psi1_tc_backward(const PsiConst& P, const BwdConst& B, double* part, int64_t pstride, int rows, void* stream) {
  SGPX_P1TC_DISPATCH(launch_bwd, P, B, part, pstride, rows, static_cast<cudaStream_t>(stream))
}

}  // namespace sgpx
