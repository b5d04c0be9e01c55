// Rank-split boundary exceptions (north_star: "E2LSH floor codes ... may
// differ only where the projection lies within 1e-6 of a bucket boundary ...
// every such case is counted and reported").
//
// The reference ranks OpenBLAS dgemv projections (engine.py:178-181,
// transform.py:103-109); K1 computes the same float64 dot products in another
// summation order.  Both are within gamma_d * sum_k |x_k a_k| of the exact
// value, so two ids can swap order only if their keys are within twice that
// bound -- and a swap changes a bucket code only across a boundary.  This pass
// finds every bucket boundary's midpoint (max key of bucket s, min key of
// bucket s+1) and counts the ids whose key lies within
//   * tol_abs[j]           -- the rigorous bound: these ids' codes MAY differ
//                             from the reference's (listed, up to `cap`);
//   * rel_a * |midpoint|   -- e.g. 1e-12 relative;
//   * rel_b * |midpoint|   -- e.g. 1e-6 relative (north_star's window).
// Two stream-ordered passes over keys [m][n] and codes [n][stride]; no sync.
#include "common.cuh"

namespace geek {

__device__ __forceinline__ double key_to_f64(uint64_t k) {
  const uint64_t b = (k & 0x8000000000000000ull) ? (k ^ 0x8000000000000000ull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

constexpr int kBsWarps = 8;

// bucket extremes: bmin[j*t + c] / bmax[j*t + c] over the ids of bucket c.
// Lanes of a warp holding the same code combine in shared memory first (the
// bench data is cluster-ordered: one group per warp and table is typical).
__global__ void __launch_bounds__(kBsWarps * 32) bucket_extremes_kernel(const uint64_t* __restrict__ keys,
                                                                      const uint32_t* __restrict__ codes,
                                                                      uint64_t n, int m, uint64_t stride,
                                                                      uint64_t t, unsigned long long* bmin,
                                                                      unsigned long long* bmax) {
  __shared__ uint64_t skey[kBsWarps][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n; base += step) {
    const uint64_t i = base + lane;
    const bool ok = i < n;
    for (int j = 0; j < m; ++j) {
      const uint64_t key = ok ? __ldg(keys + (uint64_t)j * n + i) : 0ull;
      const uint32_t code = ok ? __ldg(codes + i * stride + j) : GEEK_NONE;
      skey[w][lane] = key;
      const unsigned grp = __match_any_sync(0xFFFFFFFFu, code);
      __syncwarp();
      if (ok && lane == __ffs(grp) - 1) {
        uint64_t lo = key, hi = key;
        for (unsigned g = grp & (grp - 1); g; g &= g - 1) {
          const uint64_t k2 = skey[w][__ffs(g) - 1];
          lo = k2 < lo ? k2 : lo;
          hi = k2 > hi ? k2 : hi;
        }
        atomicMin(bmin + (uint64_t)j * t + code, (unsigned long long)lo);
        atomicMax(bmax + (uint64_t)j * t + code, (unsigned long long)hi);
      }
      __syncwarp();
    }
  }
}

// mid[j*(t-1) + s] = midpoint of the keys either side of boundary s
__global__ void boundary_mid_kernel(const unsigned long long* bmin, const unsigned long long* bmax, int m,
                                    uint64_t t, double* mid) {
  const uint64_t nb = t - 1, total = (uint64_t)m * nb;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < total;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = q / nb, s = q % nb;
    const double lo = key_to_f64(bmax[j * t + s]), hi = key_to_f64(bmin[j * t + s + 1]);
    mid[q] = lo + 0.5 * (hi - lo);
  }
}

__global__ void __launch_bounds__(256) boundary_count_kernel(const uint64_t* __restrict__ keys,
                                                             const uint32_t* __restrict__ codes, uint64_t n,
                                                             int m, uint64_t stride, uint64_t t,
                                                             const double* __restrict__ mid,
                                                             const unsigned long long* __restrict__ bmin,
                                                             const unsigned long long* __restrict__ bmax,
                                                             const double* __restrict__ tol_abs, double rel_a,
                                                             double rel_b, unsigned long long* counts,
                                                             uint32_t* list, uint64_t cap) {
  const int lane = threadIdx.x & 31;
  const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t nb = t - 1;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n; base += step) {
    const uint64_t i = base + lane;
    const bool ok = i < n;
    unsigned ca = 0, cr1 = 0, cr2 = 0;
    for (int j = 0; j < m; ++j) {
      bool amb = false, r1 = false, r2 = false;
      if (ok && nb > 0) {
        const uint64_t key = __ldg(keys + (uint64_t)j * n + i);
        const double v = key_to_f64(key);
        const uint32_t c = __ldg(codes + i * stride + j);
        const double* mj = mid + (uint64_t)j * nb;
        const unsigned long long* lo = bmax + (uint64_t)j * t;  // lo[s] / hi[s+1]: keys either side of s
        const unsigned long long* hi = bmin + (uint64_t)j * t;
        double dist = INFINITY, scale = 0.0, adist = INFINITY;
        if (c > 0) {
          const double b = __ldg(mj + c - 1);
          dist = fabs(v - b);
          scale = fabs(b);
          // a boundary whose two keys are EQUAL is decided by id in any
          // implementation that computes equal keys for them (identical rows):
          // ids holding that exact key are not ambiguous there
          if (!(__ldg(lo + c - 1) == __ldg(hi + c) && key == __ldg(hi + c))) adist = dist;
        }
        if ((uint64_t)c < nb) {
          const double b = __ldg(mj + c);
          const double dd = fabs(v - b);
          dist = fmin(dist, dd);
          scale = fmax(scale, fabs(b));
          if (!(__ldg(lo + c) == __ldg(hi + c + 1) && key == __ldg(lo + c))) adist = fmin(adist, dd);
        }
        amb = adist <= __ldg(tol_abs + j);
        r1 = dist <= rel_a * scale;
        r2 = dist <= rel_b * scale;
        if (amb) {
          const unsigned long long pos = atomicAdd(&counts[3], 1ull);
          if (pos < cap) {
            list[2 * pos] = (uint32_t)j;
            list[2 * pos + 1] = (uint32_t)i;
          }
        }
      }
      ca += __popc(__ballot_sync(0xFFFFFFFFu, amb));
      cr1 += __popc(__ballot_sync(0xFFFFFFFFu, r1));
      cr2 += __popc(__ballot_sync(0xFFFFFFFFu, r2));
    }
    if (lane == 0) {
      if (ca) atomicAdd(&counts[0], (unsigned long long)ca);
      if (cr1) atomicAdd(&counts[1], (unsigned long long)cr1);
      if (cr2) atomicAdd(&counts[2], (unsigned long long)cr2);
    }
  }
}

}  // namespace geek

using namespace geek;

extern "C" {

uint64_t geek_split_boundary_workspace(uint64_t m, uint64_t t) { return m * t * 24 + 256; }

int geek_split_boundary_stats(const uint64_t* keys, uint64_t n, int m, uint64_t t, const uint32_t* codes,
                              uint64_t code_stride, const double* tol_abs, double rel_a, double rel_b,
                              unsigned long long* counts, uint32_t* list, uint64_t cap, void* workspace,
                              uint64_t workspace_bytes, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(m >= 1 && t >= 1 && t <= n, "bad boundary-stats shape");
  GEEK_REQUIRE(code_stride >= (uint64_t)m, "code stride below table count");
  GEEK_REQUIRE(workspace && workspace_bytes >= geek_split_boundary_workspace(m, t),
               "boundary stats need %llu workspace bytes",
               (unsigned long long)geek_split_boundary_workspace(m, t));
  GEEK_CHECK_CUDA(cudaMemsetAsync(counts, 0, 4 * sizeof(unsigned long long), s));
  if (t < 2) return GEEK_OK;
  char* ws = static_cast<char*>(workspace);
  auto* bmin = reinterpret_cast<unsigned long long*>(ws);
  auto* bmax = bmin + (uint64_t)m * t;
  auto* mid = reinterpret_cast<double*>(bmax + (uint64_t)m * t);
  GEEK_CHECK_CUDA(cudaMemsetAsync(bmin, 0xFF, (uint64_t)m * t * 8, s));
  GEEK_CHECK_CUDA(cudaMemsetAsync(bmax, 0x00, (uint64_t)m * t * 8, s));
  bucket_extremes_kernel<<<grid_for(n, kBsWarps * 32, 148 * 8), kBsWarps * 32, 0, s>>>(keys, codes, n, m,
                                                                                      code_stride, t, bmin, bmax);
  GEEK_CHECK_LAUNCH();
  boundary_mid_kernel<<<grid_for((uint64_t)m * (t - 1), 256), 256, 0, s>>>(bmin, bmax, m, t, mid);
  GEEK_CHECK_LAUNCH();
  boundary_count_kernel<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(keys, codes, n, m, code_stride, t, mid, bmin,
                                                                   bmax, tol_abs, rel_a, rel_b, counts, list, cap);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

}  // extern "C"
