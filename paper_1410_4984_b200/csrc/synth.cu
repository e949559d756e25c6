// synth.cu -- the reference's seeded inputs and binary matrices, at HBM scale.
//
// Reference: sgp::Rng (proj/include/sgp/common.hpp:45-97), the Z choice of init_gplvm
// (model.hpp:420-429) and the raw binary matrix format (io.hpp:114-153).
//
// Rng is splitmix64 with state_t = seed + t * 0x9e3779b97f4a7c15 (seed 0 -> the golden constant), so
// its t-th u64 draw is a pure function of t: normal_matrix(rows, cols) visits (i, j) in row-major
// order, element k = i * cols + j is member (k & 1) of the Box-Muller pair built from draws
// 2 (k >> 1) + 1 and + 2 (next_normal caches the second member).  One thread per pair reproduces the
// stream for any size without a sequential pass; sqrt / log / sin / cos are CUDA's fp64 functions
// (within 1-2 ulp of glibc's, tests/test_gpu_northstar.py pins the agreement).
//
// Binary matrices: <base>.shape holds "rows cols\n", <base>.bin rows x cols float64 row-major
// little-endian.  The device loader streams the row-major file through pinned staging and
// transposes each slab on the device into the column-major (Eigen) layout of the engine.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "coordinator.hpp"
#include "psi_kernels.cuh"

namespace sgpx {
extern std::atomic<int64_t> g_tc_launches;

namespace {
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;

__host__ __device__ __forceinline__ uint64_t splitmix_at(uint64_t seed0, uint64_t t) {
  uint64_t z = seed0 + t * kGolden;  // state after t calls (t >= 1)
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ double uniform_of(uint64_t u) {  // (0, 1], common.hpp:58-60
  return (double(u >> 11) + 1.0) * 0x1.0p-53;
}

__global__ void rng_normal_kernel(uint64_t seed0, int64_t rows, int64_t cols, double* __restrict__ out, int64_t ld) {
  const int64_t total = rows * cols, pairs = (total + 1) / 2;
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < pairs; j += int64_t(gridDim.x) * blockDim.x) {
    const double u1 = uniform_of(splitmix_at(seed0, uint64_t(2 * j + 1)));
    const double u2 = uniform_of(splitmix_at(seed0, uint64_t(2 * j + 2)));
    const double r = sqrt(-2.0 * log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    double sa, ca;
    sincos(a, &sa, &ca);
    const int64_t k = 2 * j;
    out[(k / cols) + (k % cols) * ld] = r * ca;
    if (k + 1 < total) out[((k + 1) / cols) + ((k + 1) % cols) * ld] = r * sa;
  }
}

// rows [r0, r0 + nr) of a row-major slab (nr x cols) -> column-major out (ld)
__global__ void transpose_slab_kernel(const double* __restrict__ slab, int64_t nr, int64_t cols, int64_t r0,
                                      double* __restrict__ out, int64_t ld) {
  __shared__ double t[32][33];
  for (int64_t cb = blockIdx.y * 32; cb < cols; cb += int64_t(gridDim.y) * 32)
    for (int64_t rb = blockIdx.x * 32; rb < nr; rb += int64_t(gridDim.x) * 32) {
      for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = rb + i, c = cb + threadIdx.x;
        t[i][threadIdx.x] = (r < nr && c < cols) ? slab[r * cols + c] : 0.0;
      }
      __syncthreads();
      for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = cb + i, r = rb + threadIdx.x;
        if (r < nr && c < cols) out[(r0 + r) + c * ld] = t[threadIdx.x][i];
      }
      __syncthreads();
    }
}

void read_shape(const std::string& base, int64_t* rows, int64_t* cols) {
  std::ifstream shape(base + ".shape", std::ios::binary);
  if (!shape) throw IoError("cannot open: " + base + ".shape");
  long long r = 0, c = 0;
  shape >> r >> c;
  if (!shape || r < 0 || c < 0) throw IoError(base + ".shape:1: expected 'rows cols'");
  *rows = r;
  *cols = c;
}

}  // namespace

uint64_t rng_seed0(uint64_t seed) { return seed ? seed : kGolden; }

int rng_normal_device(uint64_t seed, int64_t rows, int64_t cols, double* out, int64_t ld, void* stream) {
  if (rows * cols == 0) return 0;
  const int64_t pairs = (rows * cols + 1) / 2;
  const int blocks = int(std::min<int64_t>((pairs + 255) / 256, 148 * 16));
  rng_normal_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(rng_seed0(seed), rows, cols, out, ld);
  g_tc_launches.fetch_add(1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// next_index (common.hpp:79-84) on the host stream of Rng(seed), partial Fisher-Yates of init_gplvm.
void rng_choose_rows(uint64_t seed, int64_t n, int64_t m, int64_t* idx_out) {
  const uint64_t s0 = rng_seed0(seed);
  uint64_t t = 0;
  std::unordered_map<int64_t, int64_t> swapped;  // sparse image of idx[] (identity elsewhere)
  auto at = [&](int64_t i) {
    auto it = swapped.find(i);
    return it == swapped.end() ? i : it->second;
  };
  for (int64_t i = 0; i < m; ++i) {
    const uint64_t range = uint64_t(n - i);
    const uint64_t limit = ~uint64_t{0} - (~uint64_t{0} % range);
    uint64_t v = splitmix_at(s0, ++t);
    while (v >= limit) v = splitmix_at(s0, ++t);
    const int64_t j = i + int64_t(v % range);
    const int64_t a = at(i), b = at(j);
    swapped[i] = b;
    swapped[j] = a;
    idx_out[i] = b;
  }
}

void io_read_shape(const char* base, int64_t* rows, int64_t* cols) { read_shape(base, rows, cols); }

void io_read_host(const char* base, double* out, int64_t ld) {
  int64_t rows = 0, cols = 0;
  read_shape(base, &rows, &cols);
  std::ifstream bin(std::string(base) + ".bin", std::ios::binary);
  if (!bin) throw IoError(std::string("cannot open: ") + base + ".bin");
  std::vector<double> row(size_t(std::max<int64_t>(cols, 1)));
  for (int64_t i = 0; i < rows; ++i) {
    if (!bin.read(reinterpret_cast<char*>(row.data()), std::streamsize(sizeof(double) * cols)))
      throw IoError(std::string(base) + ".bin: truncated at row " + std::to_string(i));
    for (int64_t j = 0; j < cols; ++j) out[i + j * ld] = row[size_t(j)];
  }
}

void io_write_host(const char* base, const double* a, int64_t rows, int64_t cols, int64_t ld) {
  {
    std::ofstream shape(std::string(base) + ".shape", std::ios::binary);
    if (!shape) throw IoError(std::string("cannot open for writing: ") + base + ".shape");
    shape << rows << ' ' << cols << '\n';
  }
  std::ofstream bin(std::string(base) + ".bin", std::ios::binary);
  if (!bin) throw IoError(std::string("cannot open for writing: ") + base + ".bin");
  std::vector<double> row(size_t(std::max<int64_t>(cols, 1)));
  for (int64_t i = 0; i < rows; ++i) {
    for (int64_t j = 0; j < cols; ++j) row[size_t(j)] = a[i + j * ld];
    bin.write(reinterpret_cast<const char*>(row.data()), std::streamsize(sizeof(double) * cols));
  }
  if (!bin) throw IoError(std::string("write failed: ") + base + ".bin");
}

// Stream <base>.bin through two pinned slabs (file read of slab k+1 overlaps the upload and the
// transpose of slab k) into a column-major device matrix.
void io_load_device(const char* base, double* dev_out, int64_t ld, void* stream_v) {
  cudaStream_t st = static_cast<cudaStream_t>(stream_v);
  int64_t rows = 0, cols = 0;
  read_shape(base, &rows, &cols);
  if (rows * cols == 0) return;
  FILE* f = fopen((std::string(base) + ".bin").c_str(), "rb");
  if (!f) throw IoError(std::string("cannot open: ") + base + ".bin");
  const int64_t slab_rows = std::max<int64_t>(1, (int64_t(64) << 20) / (8 * cols));  // ~64 MB slabs
  double* host[2] = {nullptr, nullptr};
  double* dev[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  auto cleanup = [&] {
    for (int i = 0; i < 2; ++i) {
      if (done[i]) cudaEventDestroy(done[i]);
      if (host[i]) cudaFreeHost(host[i]);
      if (dev[i]) cudaFree(dev[i]);
    }
    fclose(f);
  };
  try {
    const size_t bytes = sizeof(double) * size_t(slab_rows * cols);
    for (int i = 0; i < 2; ++i) {
      if (cudaMallocHost(&host[i], bytes) != cudaSuccess || cudaMalloc(&dev[i], bytes) != cudaSuccess ||
          cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming) != cudaSuccess)
        throw IoError("io: staging allocation failed");
    }
    int k = 0;
    for (int64_t r0 = 0; r0 < rows; r0 += slab_rows, k ^= 1) {
      const int64_t nr = std::min(slab_rows, rows - r0);
      if (cudaEventSynchronize(done[k]) != cudaSuccess) throw IoError("io: device error");
      const size_t want = size_t(nr * cols);
      if (fread(host[k], sizeof(double), want, f) != want)
        throw IoError(std::string(base) + ".bin: truncated at row " + std::to_string(r0));
      cudaMemcpyAsync(dev[k], host[k], sizeof(double) * want, cudaMemcpyHostToDevice, st);
      dim3 grid(unsigned(std::min<int64_t>((nr + 31) / 32, 4096)), unsigned(std::min<int64_t>((cols + 31) / 32, 64)));
      transpose_slab_kernel<<<grid, dim3(32, 8), 0, st>>>(dev[k], nr, cols, r0, dev_out, ld);
      g_tc_launches.fetch_add(1);
      cudaEventRecord(done[k], st);
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) throw IoError("io: device error");
  } catch (...) {
    cudaStreamSynchronize(st);
    cleanup();
    throw;
  }
  cleanup();
}

}  // namespace sgpx
