// Refinement statistics keyed by the current labels (assignment.py:110-137,
// engine.py:519-537).  A refinement pass recomputes every non-empty cluster's
// center from its members; the members of cluster j are simply the rows with
// label j, so instead of materialising groups (a sort of n labels and a row
// gather) these kernels stream the rows once, coalesced, and fold each row
// into the statistics of its label:
//   * label_sums: exact base-2^32 digit column sums (the K7 representation,
//     centers.cu), accumulated in registers while consecutive rows share a
//     label and flushed with integer atomics when it changes -- exact and
//     order-free, so any shard split / launch shape gives the same digits.
//     Rows are visited in storage order, or through a label-sorted row
//     permutation when the labels change too often for register runs;
//   * label_mode_counts: per (cluster, attribute, code) counts (categorical
//     modes, seeding.py:180-185);
//   * label_sparse_counts: per (cluster, element) membership counts (sparse
//     modes, seeding.py:186-190).
#include "common.cuh"

namespace geek {

// v = M * 2^L exactly (|M| < 2^P), from the bit pattern; false for zero and
// non-finite values.  Subnormals keep L at the minimum exponent, which is >=
// the frexp-normalised exponent geek_exponent_range reports, so L - emin >= 0.
__device__ __forceinline__ bool split_bits(float v, long long& M, int& L) {
  const uint32_t u = __float_as_uint(v);
  const uint32_t E = (u >> 23) & 0xFF, f = u & 0x7FFFFF;
  if (E == 0xFF || (E == 0 && f == 0)) return false;
  const long long mag = E ? (long long)(f | 0x800000u) : (long long)f;
  M = (u >> 31) ? -mag : mag;
  L = (E ? (int)E : 1) - 150;
  return true;
}
__device__ __forceinline__ bool split_bits(double v, long long& M, int& L) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  const int E = (int)((u >> 52) & 0x7FF);
  const unsigned long long f = u & 0xFFFFFFFFFFFFFull;
  if (E == 0x7FF || (E == 0 && f == 0)) return false;
  const long long mag = E ? (long long)(f | (1ull << 52)) : (long long)f;
  M = (u >> 63) ? -mag : mag;
  L = (E ? E : 1) - 1075;
  return true;
}

constexpr int kRunRows = 256;  // rows per block-chunk
constexpr int kPrefetch = 8;   // row values loaded ahead per thread

// Lanes acc[q] hold sums of (M << rb) placed at digit q (weight 2^(32q)); a
// float32 term is < 2^56 in magnitude, so a lane absorbs 64 terms before it
// is carried down into 32-bit digits (normalise) -- 1 select-add per lane
// per term instead of splitting every term into three digits.
template <int ND>
__device__ __forceinline__ void normalise(long long (&acc)[ND]) {
#pragma unroll
  for (int q = 0; q + 1 < ND; ++q) {
    const long long c = acc[q] >> 32;  // floor
    acc[q] -= c * 4294967296ll;        // now in [0, 2^32)
    acc[q + 1] += c;
  }
}

template <int ND>
__device__ __forceinline__ void flush_digits(long long (&acc)[ND], long long* dst) {
  normalise<ND>(acc);
#pragma unroll
  for (int q = 0; q < ND; ++q) {
    if (acc[q]) atomicAdd(reinterpret_cast<unsigned long long*>(dst + q), (unsigned long long)acc[q]);
    acc[q] = 0;
  }
}

template <class T, int ND>
__device__ __forceinline__ void add_term(long long (&acc)[ND], T v, int emin) {
  long long M;
  int L;
  if (!split_bits(v, M, L)) return;
  const int sh = L - emin;  // >= 0
  const int q0 = sh >> 5, rb = sh & 31;
  if (sizeof(T) == 4) {  // |M << rb| < 2^56: one lane
    const long long w = M * (1ll << rb);
#pragma unroll
    for (int q = 0; q < ND; ++q) acc[q] += (q == q0) ? w : 0ll;
  } else {  // |M| < 2^53: low 32 bits of M << rb at q0, the rest (< 2^53 in magnitude) at q0 + 1
    const long long lo = (long long)(((unsigned long long)M << rb) & 0xFFFFFFFFull);
    const long long hi = (long long)(((__int128)M << rb) >> 32);
#pragma unroll
    for (int q = 0; q < ND; ++q) acc[q] += (q == q0) ? lo : ((q == q0 + 1) ? hi : 0ll);
  }
}

// rows r0..r0+rows of the (optionally permuted) row order; labels are read
// through the same order so a sorted permutation gives long label runs
template <class T, int ND>
__global__ void __launch_bounds__(128) label_sums_kernel(const T* __restrict__ X, uint64_t nrows, int d,
                                                         const int64_t* __restrict__ labels,
                                                         const int64_t* __restrict__ order, uint64_t k,
                                                         int emin, long long* __restrict__ digits) {
  __shared__ int32_t lab[kRunRows];
  __shared__ uint64_t row[kRunRows];            // element offset of the row in X
  __shared__ int32_t run8[kRunRows / kPrefetch];  // label of a full 8-row group with one label, else -1
  const uint64_t nchunks = (nrows + kRunRows - 1) / kRunRows;
  for (uint64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const uint64_t r0 = ch * kRunRows;
    const int rows = (int)min((uint64_t)kRunRows, nrows - r0);
    __syncthreads();
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
      const int64_t i = order ? order[r0 + r] : (int64_t)(r0 + r);
      const int64_t l = labels[i];
      row[r] = (uint64_t)i * d;
      lab[r] = (l >= 0 && (uint64_t)l < k) ? (int32_t)l : -1;
    }
    __syncthreads();
    for (int gi = threadIdx.x; gi < kRunRows / kPrefetch; gi += blockDim.x) {
      int32_t l = -1;
      if ((gi + 1) * kPrefetch <= rows) {
        l = lab[gi * kPrefetch];
        for (int u = 1; u < kPrefetch; ++u)
          if (lab[gi * kPrefetch + u] != l) l = -1;
      }
      run8[gi] = l;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
      long long acc[ND];
#pragma unroll
      for (int q = 0; q < ND; ++q) acc[q] = 0;
      int32_t cur = -1;
      int since = 0;  // terms since the last normalisation
      for (int rb = 0; rb < rows; rb += kPrefetch) {
        T v[kPrefetch];
#pragma unroll
        for (int u = 0; u < kPrefetch; ++u)
          v[u] = (rb + u < rows) ? X[row[rb + u] + c] : T(0);
        const int32_t g8 = run8[rb / kPrefetch];
        if (g8 >= 0 && g8 == cur) {  // inside a run: no per-row label checks
#pragma unroll
          for (int u = 0; u < kPrefetch; ++u) add_term<T, ND>(acc, v[u], emin);
          since += kPrefetch;
          if (since >= 64) {  // lanes hold < 72 terms of < 2^56 each
            normalise<ND>(acc);
            since = 0;
          }
          continue;
        }
        for (int u = 0; u < kPrefetch; ++u) {
          if (rb + u >= rows) break;
          const int32_t l = lab[rb + u];
          if (l != cur) {
            if (cur >= 0) flush_digits<ND>(acc, digits + ((uint64_t)cur * d + c) * ND);
            cur = l;
            since = 0;
          }
          if (cur < 0) continue;
          add_term<T, ND>(acc, v[u], emin);
          if (++since >= 64) {
            normalise<ND>(acc);
            since = 0;
          }
        }
      }
      if (cur >= 0) flush_digits<ND>(acc, digits + ((uint64_t)cur * d + c) * ND);
    }
  }
}

__global__ void label_mode_counts_kernel(const int32_t* __restrict__ codes, uint64_t nrows, int d,
                                         const int64_t* __restrict__ labels, uint64_t k, uint64_t cs,
                                         unsigned long long* counts) {
  const uint64_t total = nrows * (uint64_t)d;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = e / d;
    const int c = (int)(e - i * d);
    const int64_t l = labels[i];
    const int32_t code = codes[e];
    if (l < 0 || (uint64_t)l >= k || code < 0 || (uint64_t)code >= cs) continue;
    atomicAdd(counts + ((uint64_t)l * d + c) * cs + code, 1ull);
  }
}

// one warp per set
__global__ void label_sparse_counts_kernel(const uint32_t* __restrict__ set_flat,
                                           const uint64_t* __restrict__ set_off, uint64_t nrows,
                                           const int64_t* __restrict__ labels, uint64_t k, uint64_t universe,
                                           unsigned long long* counts) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t i = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < nrows; i += warps) {
    const int64_t l = labels[i];
    if (l < 0 || (uint64_t)l >= k) continue;
    unsigned long long* row = counts + (uint64_t)l * universe;
    for (uint64_t p = set_off[i] + lane; p < set_off[i + 1]; p += 32) {
      const uint32_t e = set_flat[p];
      if (e < universe) atomicAdd(row + e, 1ull);
    }
  }
}

template <class T, int ND>
static void launch_label_sums(const void* X, uint64_t nrows, int d, const int64_t* labels, const int64_t* order,
                              uint64_t k, int emin, long long* digits, cudaStream_t s) {
  const int threads = d >= 128 ? 128 : 32 * ((d + 31) / 32);
  const uint64_t nchunks = (nrows + kRunRows - 1) / kRunRows;
  label_sums_kernel<T, ND><<<grid_for(nchunks, 1, 148 * 16), threads, 0, s>>>((const T*)X, nrows, d, labels,
                                                                              order, k, emin, digits);
}

}  // namespace geek

using namespace geek;

extern "C" {

int geek_label_sums(const void* X, int dtype, uint64_t nrows, int d, const int64_t* labels, const int64_t* order,
                    uint64_t k, int emin, int nd, int64_t* digits, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(dtype == 0 || dtype == 1, "dtype must be 0 or 1");
  GEEK_REQUIRE(d > 0, "d must be positive");
  GEEK_REQUIRE(k < (1ull << 31), "k = %llu clusters exceeds the 31-bit label range", (unsigned long long)k);
  GEEK_REQUIRE(nd >= 3 && nd <= 40, "digit count %d outside [3, 40]", nd);
  if (nrows == 0 || k == 0) return GEEK_OK;
  long long* dg = reinterpret_cast<long long*>(digits);
#define GEEK_LSUMS_CASE(NDV)                                                          \
  case NDV:                                                                           \
    if (dtype == 0)                                                                   \
      launch_label_sums<float, NDV>(X, nrows, d, labels, order, k, emin, dg, s);             \
    else                                                                              \
      launch_label_sums<double, NDV>(X, nrows, d, labels, order, k, emin, dg, s);            \
    break;
  switch (nd) {
    GEEK_LSUMS_CASE(3)
    GEEK_LSUMS_CASE(4)
    GEEK_LSUMS_CASE(5)
    GEEK_LSUMS_CASE(6)
    GEEK_LSUMS_CASE(8)
    GEEK_LSUMS_CASE(12)
    GEEK_LSUMS_CASE(20)
    GEEK_LSUMS_CASE(40)
    default:
      set_error("digit count %d must be one of 3,4,5,6,8,12,20,40", nd);
      return GEEK_EINVAL;
  }
#undef GEEK_LSUMS_CASE
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

int geek_label_mode_counts(const int32_t* codes, uint64_t nrows, int d, const int64_t* labels, uint64_t k,
                           uint64_t cs, int64_t* counts, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(d > 0, "d must be positive");
  if (nrows == 0 || k == 0) return GEEK_OK;
  label_mode_counts_kernel<<<grid_for(nrows * d, 256), 256, 0, s>>>(
      codes, nrows, d, labels, k, cs, reinterpret_cast<unsigned long long*>(counts));
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

int geek_label_sparse_counts(const uint32_t* set_flat, const uint64_t* set_off, uint64_t nrows,
                             const int64_t* labels, uint64_t k, uint64_t universe, int64_t* counts, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (nrows == 0 || k == 0) return GEEK_OK;
  label_sparse_counts_kernel<<<grid_for(nrows, 8), 256, 0, s>>>(set_flat, set_off, nrows, labels, k, universe,
                                                                reinterpret_cast<unsigned long long*>(counts));
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

}  // extern "C"
