// K1: float64-accurate random projections of every point onto every table's
// direction (transform.py:125, engine.py:180), emitted as order-preserving
// uint64 keys for the rank split.  HBM-streaming: X is read once per table
// block through shared memory; directions stay resident in shared memory.
#include "common.cuh"

namespace geek {

constexpr int kProjThreads = 128;
constexpr int kProjPts = 2;     // points per thread
constexpr int kProjTB = 8;      // tables per pass
constexpr int kProjTile = kProjThreads * kProjPts;

// Bounds of the binary exponent window of a value as the exact-sum kernel
// decomposes it (v = M * 2^L, |M| < 2^P; numeric.py:19-40): lo <= L, hi >= L + P.
// Subnormals take the most negative L their format allows.
__device__ __forceinline__ void exp_window(float v, int& lo, int& hi) {
  const uint32_t b = __float_as_uint(v);
  const int e = (b >> 23) & 0xFF;
  if (e == 0xFF || (b & 0x7FFFFFFFu) == 0) return;
  const int L = e ? e - 150 : -172;
  lo = min(lo, L);
  hi = max(hi, e ? e - 126 : -148);
}

__device__ __forceinline__ void exp_window(double v, int& lo, int& hi) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
  const int e = (int)((b >> 52) & 0x7FF);
  if (e == 0x7FF || (b & 0x7FFFFFFFFFFFFFFFull) == 0) return;
  lo = min(lo, e ? e - 1075 : -1127);
  hi = max(hi, e ? e - 1022 : -1074);
}

template <class T>
__global__ void __launch_bounds__(kProjThreads) project_kernel(const T* __restrict__ X, uint64_t n,
                                                               int d, const double* __restrict__ A,
                                                               int m, uint64_t* __restrict__ keys,
                                                               int* exprange) {
  constexpr int kProjKT = sizeof(T) == 4 ? 32 : 16;  // dims per shared-memory tile (<= 33 KB)
  __shared__ double sA[kProjTB][kProjKT];
  __shared__ T sX[kProjKT][kProjTile + 1];
  const uint64_t tile0 = blockIdx.x * (uint64_t)kProjTile;
  int elo = 1 << 30, ehi = -(1 << 30);
  for (int j0 = 0; j0 < m; j0 += kProjTB) {
    double acc[kProjPts][kProjTB];
#pragma unroll
    for (int p = 0; p < kProjPts; ++p)
#pragma unroll
      for (int j = 0; j < kProjTB; ++j) acc[p][j] = 0.0;
    for (int k0 = 0; k0 < d; k0 += kProjKT) {
      __syncthreads();
      for (int e = threadIdx.x; e < kProjTB * kProjKT; e += kProjThreads) {
        int j = e / kProjKT, k = e % kProjKT;
        sA[j][k] = (j0 + j < m && k0 + k < d) ? A[(uint64_t)(j0 + j) * d + k0 + k] : 0.0;
      }
      // coalesced: consecutive threads read consecutive dims of a row
      for (int e = threadIdx.x; e < kProjTile * kProjKT; e += kProjThreads) {
        int pt = e / kProjKT, k = e % kProjKT;
        uint64_t i = tile0 + pt;
        const T v = (i < n && k0 + k < d) ? X[i * d + k0 + k] : T(0);
        sX[k][pt] = v;
        if (j0 == 0) exp_window(v, elo, ehi);  // fused exponent window (first table pass)
      }
      __syncthreads();
#pragma unroll 8
      for (int k = 0; k < kProjKT; ++k) {
        double x[kProjPts];
#pragma unroll
        for (int p = 0; p < kProjPts; ++p) x[p] = (double)sX[k][threadIdx.x + p * kProjThreads];
#pragma unroll
        for (int j = 0; j < kProjTB; ++j) {
          const double a = sA[j][k];
#pragma unroll
          for (int p = 0; p < kProjPts; ++p) acc[p][j] = fma(x[p], a, acc[p][j]);
        }
      }
    }
#pragma unroll
    for (int p = 0; p < kProjPts; ++p) {
      uint64_t i = tile0 + threadIdx.x + p * kProjThreads;
      if (i < n) {
#pragma unroll
        for (int j = 0; j < kProjTB; ++j)
          if (j0 + j < m) keys[(uint64_t)(j0 + j) * n + i] = f64_key(acc[p][j]);
      }
    }
  }
  if (exprange) {
    for (int o = 16; o; o >>= 1) {
      elo = min(elo, __shfl_xor_sync(0xffffffffu, elo, o));
      ehi = max(ehi, __shfl_xor_sync(0xffffffffu, ehi, o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&exprange[0], elo);
      atomicMax(&exprange[1], ehi);
    }
  }
}

template <class T>
__global__ void column_keys_kernel(const T* __restrict__ v, uint64_t n, uint64_t stride, uint64_t col,
                                   uint64_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = f64_key((double)v[i * stride + col]);
}

}  // namespace geek

using namespace geek;

extern "C" {

int geek_project_keys(const void* X, int dtype, uint64_t n, int d, const double* A, int m,
                      uint64_t* keys, int* exprange, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(dtype == 0 || dtype == 1, "dtype must be 0 (f32) or 1 (f64)");
  GEEK_REQUIRE(d >= 1 && m >= 1, "empty projection");
  if (n == 0) return GEEK_OK;
  unsigned grid = (unsigned)((n + kProjTile - 1) / kProjTile);
  if (dtype == 0)
    project_kernel<float><<<grid, kProjThreads, 0, s>>>((const float*)X, n, d, A, m, keys, exprange);
  else
    project_kernel<double><<<grid, kProjThreads, 0, s>>>((const double*)X, n, d, A, m, keys, exprange);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

int geek_column_keys(const void* values, int dtype, uint64_t n, uint64_t stride, uint64_t col,
                     uint64_t* keys, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(dtype == 0 || dtype == 1, "dtype must be 0 (f32) or 1 (f64)");
  if (n == 0) return GEEK_OK;
  if (dtype == 0)
    column_keys_kernel<float><<<grid_for(n, 256), 256, 0, s>>>((const float*)values, n, stride, col, keys);
  else
    column_keys_kernel<double><<<grid_for(n, 256), 256, 0, s>>>((const double*)values, n, stride, col, keys);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

}  // extern "C"
