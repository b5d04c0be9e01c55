// K7: exact centroids (numeric.py:19-51).  Every coordinate is an integer
// multiple of 2^emin (emin = lowest mantissa bit over the data), so group
// column sums are exact integers; they are accumulated as base-2^32 digits in
// int64 lanes (each lane only ever receives values below 2^32 in magnitude,
// so 2^31 additions cannot overflow), merged with integer atomics (exact,
// order-free -- the property engine.py:481-516 relies on), and divided by the
// count with a single correctly rounded (half-even) rounding, which is what
// float(Fraction(S, count << 1074)) computes.
#include "common.cuh"

#include <algorithm>

namespace geek {

int bitlen_u64(uint64_t v) { return v ? 64 - __builtin_clzll(v) : 0; }

template <class T>
struct FloatBits;
template <>
struct FloatBits<float> {
  static constexpr int P = 24;
};
template <>
struct FloatBits<double> {
  static constexpr int P = 53;
};

// v = M * 2^L with |M| < 2^P integer; returns false for zero / non-finite
template <class T>
__device__ __forceinline__ bool decompose(T v, long long& M, int& L) {
  double x = (double)v;
  if (x == 0.0 || !isfinite(x)) return false;
  int e;
  double f = frexp(x, &e);  // x = f * 2^e, 0.5 <= |f| < 1
  M = (long long)ldexp(f, FloatBits<T>::P);
  L = e - FloatBits<T>::P;
  return true;
}

template <class T>
__global__ void exponent_range_kernel(const T* X, uint64_t total, int* out) {
  int lo = 1 << 30, hi = -(1 << 30);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    long long M;
    int L;
    if (decompose<T>(X[i], M, L)) {
      lo = min(lo, L);
      hi = max(hi, L + FloatBits<T>::P);
    }
  }
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&out[0], lo);
    atomicMax(&out[1], hi);
  }
}

constexpr int kSumChunk = 256;  // members per block

// chunk c of the member list covers members [off[g] + 256 (c - coff[g]), ...)
// of group g, coff = exclusive scan of ceil(size_g / 256): built on the device
__global__ void chunk_count_kernel(const uint64_t* off, uint64_t ngroups, uint64_t* cnt) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g <= ngroups;
       g += (uint64_t)gridDim.x * blockDim.x)
    cnt[g] = g < ngroups ? (off[g + 1] - off[g] + kSumChunk - 1) / kSumChunk : 0;
}

template <class T, int ND>
__global__ void exact_sums_kernel(const T* __restrict__ X, uint64_t nrows, int d, uint64_t row_lo,
                                  const uint32_t* __restrict__ flat, const uint64_t* __restrict__ off,
                                  const uint64_t* __restrict__ coff, uint64_t ngroups, int emin,
                                  long long* digits, unsigned* nonfinite) {
  const uint64_t nchunks = coff[ngroups];
  for (uint64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    uint64_t lo = 0, hi = ngroups;  // last g with coff[g] <= ch
    while (hi - lo > 1) {
      const uint64_t mid = (lo + hi) >> 1;
      if (coff[mid] <= ch) lo = mid;
      else hi = mid;
    }
    const uint64_t g = lo;
    const uint64_t b = off[g] + (ch - coff[g]) * kSumChunk;
    const uint64_t e = min(b + (uint64_t)kSumChunk, off[g + 1]);
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
      long long acc[ND];
#pragma unroll
      for (int q = 0; q < ND; ++q) acc[q] = 0;
      bool bad = false;
      for (uint64_t k = b; k < e; ++k) {
        const uint64_t id = flat[k];
        if (id < row_lo || id >= row_lo + nrows) continue;
        long long M;
        int L;
        const T xv = X[(id - row_lo) * d + c];
        if (!decompose<T>(xv, M, L)) {
          bad |= !isfinite((double)xv);
          continue;
        }
        const int sh = L - emin;  // >= 0
        const int q0 = sh >> 5, r = sh & 31;
        const __int128 v = (__int128)M << r;  // < 2^(P+32)
        const long long d0 = (long long)(uint32_t)(v & 0xFFFFFFFF);
        const long long d1 = (long long)(uint32_t)((v >> 32) & 0xFFFFFFFF);
        const long long d2 = (long long)(v >> 64);  // signed, small
#pragma unroll
        for (int q = 0; q < ND; ++q) acc[q] += (q == q0) * d0 + (q == q0 + 1) * d1 + (q == q0 + 2) * d2;
      }
      if (bad && nonfinite) atomicOr(nonfinite, 1u);
      long long* dst = digits + ((uint64_t)g * d + c) * ND;
#pragma unroll
      for (int q = 0; q < ND; ++q)
        if (acc[q]) atomicAdd(reinterpret_cast<unsigned long long*>(dst + q), (unsigned long long)acc[q]);
    }
  }
}

constexpr int kMaxWords = 48;

// correctly rounded S * 2^emin / count, S = sum_q digits[q] * 2^(32q)
__global__ void round_means_kernel(const long long* digits, const uint64_t* counts, uint64_t ngroups, int d,
                                   int emin, int nd, double* out) {
  const uint64_t total = ngroups * (uint64_t)d;
  for (uint64_t gc = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; gc < total;
       gc += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t g = gc / d;
    const uint64_t cnt = counts[g];
    const long long* dg = digits + gc * nd;
    // normalise into 32-bit words of a two's complement integer
    uint32_t w[kMaxWords];
    const int nw = nd + 2;
    __int128 carry = 0;
    for (int q = 0; q < nw; ++q) {
      __int128 v = carry + (q < nd ? (__int128)dg[q] : (__int128)0);
      w[q] = (uint32_t)(v & 0xFFFFFFFF);
      carry = v >> 32;  // arithmetic shift: floor division
    }
    const bool neg = carry < 0 || (w[nw - 1] & 0x80000000u);
    if (neg) {  // magnitude = two's complement negate
      uint64_t c = 1;
      for (int q = 0; q < nw; ++q) {
        uint64_t v = (uint64_t)(~w[q]) + c;
        w[q] = (uint32_t)v;
        c = v >> 32;
      }
    }
    int top = nw - 1;
    while (top >= 0 && w[top] == 0) --top;
    if (top < 0 || cnt == 0) {
      out[gc] = 0.0;
      continue;
    }
    const int la = top * 32 + (32 - __clz(w[top]));      // bitlen |S|
    const int lc = 64 - __clzll((long long)cnt);         // bitlen count
    // scale A by 2^z so the quotient has >= 56 significant bits
    int z = 57 - (la - lc);
    if (z < 0) z = 0;
    // long division of (A << z) by cnt, most significant word first
    uint32_t a[kMaxWords + 4];
    const int zw = z >> 5, zb = z & 31;
    const int na = top + 1 + zw + 1;
    for (int q = 0; q < na; ++q) a[q] = 0;
    for (int q = 0; q <= top; ++q) {
      uint64_t v = (uint64_t)w[q] << zb;
      a[q + zw] |= (uint32_t)v;
      a[q + zw + 1] |= (uint32_t)(v >> 32);
    }
    uint64_t rem = 0;
    for (int q = na - 1; q >= 0; --q) {
      unsigned __int128 cur = ((unsigned __int128)rem << 32) | a[q];
      a[q] = (uint32_t)(cur / cnt);
      rem = (uint64_t)(cur % cnt);
    }
    int qt = na - 1;
    while (qt > 0 && a[qt] == 0) --qt;
    const int lq = qt * 32 + (32 - __clz(a[qt]));  // >= 57
    // top 55 bits of the quotient: 53 mantissa + round bit + one more
    const int drop = lq - 54;  // bits below the 54-bit window (mantissa + round)
    uint64_t top54 = 0;
    bool sticky = rem != 0;
    for (int bit = lq - 1; bit >= 0; --bit) {
      const uint32_t bv = (a[bit >> 5] >> (bit & 31)) & 1u;
      if (bit >= drop) top54 = (top54 << 1) | bv;
      else if (bv) {
        sticky = true;
        break;
      }
    }
    uint64_t mant = top54 >> 1;
    const bool round = top54 & 1;
    if (round && (sticky || (mant & 1))) ++mant;
    int exp2 = drop + 1 + emin - z;  // value = mant * 2^exp2
    if (mant == (1ull << 53)) {
      mant >>= 1;
      ++exp2;
    }
    double r = ldexp((double)mant, exp2);
    out[gc] = neg ? -r : r;
  }
}

template <class T, int ND>
static void launch_sums(const void* X, uint64_t nrows, int d, uint64_t row_lo, const uint32_t* flat,
                        const uint64_t* off, const uint64_t* coff, uint64_t ngroups, int emin, long long* digits,
                        unsigned* nonfinite, cudaStream_t s) {
  int threads = d >= 128 ? 128 : 32 * ((d + 31) / 32);
  exact_sums_kernel<T, ND><<<148 * 16, threads, 0, s>>>((const T*)X, nrows, d, row_lo, flat, off, coff, ngroups,
                                                        emin, digits, nonfinite);
}

// sum over (group, column) of the bytes numeric.pack_bigints spends on the
// exact sum T = S * 2^(emin + 1074): 8 (length) + (bitlen|T| + 8) / 8 + 1
__global__ void pack_bytes_kernel(const long long* digits, uint64_t total, int nd, int emin,
                                  unsigned long long* out) {
  unsigned long long acc = 0;
  for (uint64_t gc = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; gc < total;
       gc += (uint64_t)gridDim.x * blockDim.x) {
    const long long* dg = digits + gc * nd;
    uint32_t w[kMaxWords];
    const int nw = nd + 2;
    __int128 carry = 0;
    for (int q = 0; q < nw; ++q) {
      __int128 v = carry + (q < nd ? (__int128)dg[q] : (__int128)0);
      w[q] = (uint32_t)(v & 0xFFFFFFFF);
      carry = v >> 32;
    }
    if (carry < 0 || (w[nw - 1] & 0x80000000u)) {
      uint64_t c = 1;
      for (int q = 0; q < nw; ++q) {
        uint64_t v = (uint64_t)(~w[q]) + c;
        w[q] = (uint32_t)v;
        c = v >> 32;
      }
    }
    int top = nw - 1;
    while (top >= 0 && w[top] == 0) --top;
    const long long bl = top < 0 ? 0 : (long long)top * 32 + (32 - __clz(w[top])) + emin + 1074;
    acc += 8 + (unsigned long long)((bl + 8) / 8 + 1);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

}  // namespace geek

using namespace geek;

namespace geek {
// exact exponent window of float32 values into out[0..1] (atomically merged)
int exponent_range_f32_device(const float* X, uint64_t total, int* out, cudaStream_t s) {
  if (total) {
    exponent_range_kernel<float><<<grid_for(total, 256, 148 * 8), 256, 0, s>>>(X, total, out);
    GEEK_CHECK_LAUNCH();
  }
  return GEEK_OK;
}
}  // namespace geek

extern "C" {

int geek_exponent_range(const void* X, int dtype, uint64_t n, int d, int* out_host, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(dtype == 0 || dtype == 1, "dtype must be 0 or 1");
  Scratch o;
  GEEK_TRY(o.alloc(8, s));
  int init[2] = {1 << 30, -(1 << 30)};
  GEEK_CHECK_CUDA(cudaMemcpyAsync(o.ptr, init, 8, cudaMemcpyHostToDevice, s));
  const uint64_t total = n * (uint64_t)d;
  if (total) {
    if (dtype == 0)
      exponent_range_kernel<float><<<grid_for(total, 256, 148 * 8), 256, 0, s>>>((const float*)X, total, o.as<int>());
    else
      exponent_range_kernel<double><<<grid_for(total, 256, 148 * 8), 256, 0, s>>>((const double*)X, total, o.as<int>());
    GEEK_CHECK_LAUNCH();
  }
  GEEK_CHECK_CUDA(cudaMemcpyAsync(out_host, o.ptr, 8, cudaMemcpyDeviceToHost, s));
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
  return GEEK_OK;
}

int geek_exact_sums(const void* X, int dtype, uint64_t nrows, int d, uint64_t row_lo, const uint32_t* flat,
                    const uint64_t* offsets, uint64_t ngroups, int emin, int nd, int64_t* digits,
                    unsigned* nonfinite, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(dtype == 0 || dtype == 1, "dtype must be 0 or 1");
  GEEK_REQUIRE(nd >= 3 && nd <= 40, "digit count %d outside [3, 40]", nd);
  if (ngroups == 0) return GEEK_OK;
  // chunk offsets on the device: no host round trip, stream-ordered
  Scratch cnt, coff;
  GEEK_TRY(cnt.alloc((ngroups + 1) * 8, s));
  GEEK_TRY(coff.alloc((ngroups + 1) * 8, s));
  chunk_count_kernel<<<grid_for(ngroups + 1, 256), 256, 0, s>>>(offsets, ngroups, cnt.as<uint64_t>());
  GEEK_CHECK_LAUNCH();
  GEEK_TRY(exclusive_scan_u64(cnt.as<uint64_t>(), coff.as<uint64_t>(), ngroups + 1, s));
  const uint64_t* dco = coff.as<uint64_t>();
  long long* dg = reinterpret_cast<long long*>(digits);
#define GEEK_SUMS_CASE(NDV)                                                                           \
  case NDV:                                                                                           \
    if (dtype == 0)                                                                                   \
      launch_sums<float, NDV>(X, nrows, d, row_lo, flat, offsets, dco, ngroups, emin, dg, nonfinite, s);  \
    else                                                                                              \
      launch_sums<double, NDV>(X, nrows, d, row_lo, flat, offsets, dco, ngroups, emin, dg, nonfinite, s); \
    break;
  switch (nd) {
    GEEK_SUMS_CASE(3)
    GEEK_SUMS_CASE(4)
    GEEK_SUMS_CASE(5)
    GEEK_SUMS_CASE(6)
    GEEK_SUMS_CASE(8)
    GEEK_SUMS_CASE(12)
    GEEK_SUMS_CASE(20)
    GEEK_SUMS_CASE(40)
    default:
      set_error("digit count %d must be one of 3,4,5,6,8,12,20,40", nd);
      return GEEK_EINVAL;
  }
#undef GEEK_SUMS_CASE
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

int geek_sum_pack_bytes(const int64_t* digits, uint64_t ngroups, int d, int nd, int emin,
                        unsigned long long* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(nd >= 1 && nd + 2 <= kMaxWords, "digit count %d too large", nd);
  const uint64_t total = ngroups * (uint64_t)d;
  if (total == 0) return GEEK_OK;
  pack_bytes_kernel<<<grid_for(total, 128), 128, 0, s>>>(reinterpret_cast<const long long*>(digits), total, nd,
                                                         emin, out);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

int geek_round_means(const int64_t* digits, const uint64_t* counts, uint64_t ngroups, int d, int emin, int nd,
                     double* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(nd >= 1 && nd + 2 <= kMaxWords, "digit count %d too large", nd);
  const uint64_t total = ngroups * (uint64_t)d;
  if (total == 0) return GEEK_OK;
  round_means_kernel<<<grid_for(total, 128), 128, 0, s>>>(reinterpret_cast<const long long*>(digits), counts,
                                                          ngroups, d, emin, nd, out);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

}  // extern "C"
