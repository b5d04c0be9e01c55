// Device primitives: exclusive scans, stable LSD radix sort of u32 pairs,
// lexicographic row argsort.  These back every group-by of the hot path
// (np.unique(axis=0) / np.lexsort / stable argsort in the reference).
#include "common.cuh"

#include <cstring>
#include <mutex>

namespace geek {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

const char* last_error() { return g_last_error.c_str(); }

Workspace*& tls_workspace() {
  static thread_local Workspace* w = nullptr;
  return w;
}

void ensure_pool() {
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

int validate_perms(const geek_perm_t* perms, int nperm) {
  GEEK_REQUIRE(nperm >= 1 && nperm <= kMaxPerms, "nperm %d outside [1, %d]", nperm, kMaxPerms);
  for (int i = 0; i < nperm; ++i) {
    const geek_perm_t& p = perms[i];
    GEEK_REQUIRE(p.u >= 1 && p.u <= 0xFFFFFFFFull, "perm %d: universe %llu outside [1, 2^32)", i,
                 (unsigned long long)p.u);
    if (p.table == GEEK_NONE) {
      GEEK_REQUIRE(p.s1 >= 1 && p.s2 >= 1 && p.s1 < 32 && p.s2 < 32, "perm %d: bad shifts", i);
      GEEK_REQUIRE((p.c1 & 1u) && (p.c2 & 1u), "perm %d: even multiplier", i);
    }
  }
  return GEEK_OK;
}

__global__ void iota_u32(uint32_t* p, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = static_cast<uint32_t>(i);
}

__global__ void fill_u32(uint32_t* p, uint32_t v, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// ---------------------------------------------------------------------------
// exclusive scan: tiles of 4096 (1024 threads x 4 items), recursive on sums

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const unsigned lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (unsigned)o) v += u;
  }
  return v;
}

template <class T>
__global__ void __launch_bounds__(1024) scan_tiles(const T* in, T* out, T* sums, uint64_t n) {
  __shared__ T wsum[32];
  const uint64_t base = blockIdx.x * 4096ull + threadIdx.x * 4ull;
  T v[4];
  T acc = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[i] = (base + i < n) ? in[base + i] : T(0);
    acc += v[i];
  }
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = warp_incl_scan(acc);
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = wsum[lane];
    T wi = warp_incl_scan(w);
    wsum[lane] = wi - w;
    if (lane == 31 && sums) sums[blockIdx.x] = wi;
  }
  __syncthreads();
  T run = wsum[warp] + inc - acc;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
}

template <class T>
__global__ void scan_add(T* out, const T* offs, uint64_t n) {
  const uint64_t base = blockIdx.x * 4096ull + threadIdx.x * 4ull;
  const T o = offs[blockIdx.x];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (base + i < n) out[base + i] += o;
}

template <class T>
static int exclusive_scan_impl(const T* in, T* out, uint64_t n, cudaStream_t s, uint64_t* total_host) {
  if (n == 0) {
    if (total_host) *total_host = 0;
    return GEEK_OK;
  }
  const uint64_t nb = (n + 4095) / 4096;
  Scratch sums, sums_scan;
  GEEK_TRY(sums.alloc(nb * sizeof(T), s));
  scan_tiles<T><<<(unsigned)nb, 1024, 0, s>>>(in, out, sums.as<T>(), n);
  GEEK_CHECK_LAUNCH();
  if (nb > 1) {
    GEEK_TRY(sums_scan.alloc(nb * sizeof(T), s));
    GEEK_TRY(exclusive_scan_impl<T>(sums.as<T>(), sums_scan.as<T>(), nb, s, nullptr));
    scan_add<T><<<(unsigned)nb, 1024, 0, s>>>(out, sums_scan.as<T>(), n);
    GEEK_CHECK_LAUNCH();
  }
  if (total_host) {
    T last_in, last_out;
    GEEK_CHECK_CUDA(cudaMemcpyAsync(&last_in, in + n - 1, sizeof(T), cudaMemcpyDeviceToHost, s));
    GEEK_CHECK_CUDA(cudaMemcpyAsync(&last_out, out + n - 1, sizeof(T), cudaMemcpyDeviceToHost, s));
    GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
    *total_host = static_cast<uint64_t>(last_in) + static_cast<uint64_t>(last_out);
  }
  return GEEK_OK;
}

int exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t s, uint64_t* total_host) {
  return exclusive_scan_impl<uint32_t>(in, out, n, s, total_host);
}
int exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, cudaStream_t s, uint64_t* total_host) {
  return exclusive_scan_impl<uint64_t>(in, out, n, s, total_host);
}

// ---------------------------------------------------------------------------
// stable LSD radix sort, 8-bit digits, tiles of 2048 = 8 warps x 256 items
// (warp w owns items [w*256, w*256+256) of the tile, item-major by lane)

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;

__global__ void __launch_bounds__(kSortThreads) radix_upsweep(const uint32_t* keys, uint64_t n,
                                                              int shift, uint32_t* counts,
                                                              uint32_t nblocks) {
  __shared__ uint32_t hist[256];
  hist[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = blockIdx.x * (uint64_t)kSortTile;
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    uint64_t e = base + i * kSortThreads + threadIdx.x;
    if (e < n) atomicAdd(&hist[(keys[e] >> shift) & 0xFF], 1u);
  }
  __syncthreads();
  counts[threadIdx.x * (uint64_t)nblocks + blockIdx.x] = hist[threadIdx.x];
}

__global__ void __launch_bounds__(kSortThreads) radix_downsweep(const uint32_t* kin, const uint32_t* vin,
                                                                uint32_t* kout, uint32_t* vout,
                                                                uint64_t n, int shift,
                                                                const uint32_t* offs,
                                                                uint32_t nblocks) {
  __shared__ uint32_t wcnt[8][256];
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8 * 256; i += kSortThreads) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const uint64_t wbase = blockIdx.x * (uint64_t)kSortTile + warp * 256ull;
  uint32_t k[kSortItems], v[kSortItems];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    uint64_t e = wbase + i * 32 + lane;
    if (e < n) {
      k[i] = kin[e];
      v[i] = vin[e];
      atomicAdd(&wcnt[warp][(k[i] >> shift) & 0xFF], 1u);
    }
  }
  __syncthreads();
  {  // per digit: prefix over warps + global block offset
    const unsigned d = threadIdx.x;
    uint32_t run = offs[d * (uint64_t)nblocks + blockIdx.x];
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      uint32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    uint64_t e = wbase + i * 32 + lane;
    bool valid = e < n;
    unsigned active = __ballot_sync(0xffffffffu, valid);
    if (active == 0) break;
    uint32_t d = valid ? ((k[i] >> shift) & 0xFF) : 0x100u + lane;  // invalid lanes never match
    unsigned peers = __match_any_sync(0xffffffffu, d);
    uint32_t pos = 0;
    if (valid) pos = wcnt[warp][d] + __popc(peers & lt);
    __syncwarp();
    if (valid && (peers >> lane) == 1u) wcnt[warp][d] += __popc(peers);  // highest peer lane updates
    __syncwarp();
    if (valid) {
      kout[pos] = k[i];
      vout[pos] = v[i];
    }
  }
}

int radix_sort_pairs_u32(uint32_t* kin, uint32_t* vin, uint32_t* kout, uint32_t* vout, uint64_t n,
                         int bits, cudaStream_t s) {
  if (n == 0) return GEEK_OK;
  if (bits <= 0) bits = 1;
  const int passes = (bits + 7) / 8;
  const uint64_t nb64 = (n + kSortTile - 1) / kSortTile;
  GEEK_REQUIRE(nb64 * 256ull < 0xFFFFFFFFull, "radix sort input too large (%llu)", (unsigned long long)n);
  const uint32_t nb = static_cast<uint32_t>(nb64);
  Scratch counts, offs;
  GEEK_TRY(counts.alloc(256ull * nb * sizeof(uint32_t), s));
  GEEK_TRY(offs.alloc(256ull * nb * sizeof(uint32_t), s));
  uint32_t *ka = kin, *va = vin, *kb = kout, *vb = vout;
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    radix_upsweep<<<nb, kSortThreads, 0, s>>>(ka, n, shift, counts.as<uint32_t>(), nb);
    GEEK_CHECK_LAUNCH();
    GEEK_TRY(exclusive_scan_u32(counts.as<uint32_t>(), offs.as<uint32_t>(), 256ull * nb, s));
    radix_downsweep<<<nb, kSortThreads, 0, s>>>(ka, va, kb, vb, n, shift, offs.as<uint32_t>(), nb);
    GEEK_CHECK_LAUNCH();
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  if (ka != kout) {  // odd number of passes left the result in kin/vin
    GEEK_CHECK_CUDA(cudaMemcpyAsync(kout, ka, n * 4, cudaMemcpyDeviceToDevice, s));
    GEEK_CHECK_CUDA(cudaMemcpyAsync(vout, va, n * 4, cudaMemcpyDeviceToDevice, s));
  }
  return GEEK_OK;
}

__global__ void gather_col(const uint32_t* rows, int width, int col, const uint32_t* perm,
                           uint32_t* out, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = rows[(uint64_t)perm[i] * width + col];
}

int lex_argsort_rows(const uint32_t* rows, uint64_t n, int width, const int* bits, uint32_t* perm,
                     cudaStream_t s) {
  if (n == 0) return GEEK_OK;
  Scratch a, b, c;
  GEEK_TRY(a.alloc(n * 4, s));
  GEEK_TRY(b.alloc(n * 4, s));
  GEEK_TRY(c.alloc(n * 4, s));
  iota_u32<<<grid_for(n, 256), 256, 0, s>>>(perm, n);
  GEEK_CHECK_LAUNCH();
  for (int col = width - 1; col >= 0; --col) {
    int nb = bits ? bits[col] : 32;
    if (nb <= 0) continue;
    gather_col<<<grid_for(n, 256), 256, 0, s>>>(rows, width, col, perm, a.as<uint32_t>(), n);
    GEEK_CHECK_LAUNCH();
    GEEK_CHECK_CUDA(cudaMemcpyAsync(c.ptr, perm, n * 4, cudaMemcpyDeviceToDevice, s));
    GEEK_TRY(radix_sort_pairs_u32(a.as<uint32_t>(), c.as<uint32_t>(), b.as<uint32_t>(), perm, n,
                                  nb, s));
  }
  return GEEK_OK;
}

int argsort_cols(const uint32_t* const* cols, int ncols, const int* bits, uint64_t n, uint32_t* perm,
                 cudaStream_t s) {
  if (n == 0) return GEEK_OK;
  Scratch a, b, c;
  GEEK_TRY(a.alloc(n * 4, s));
  GEEK_TRY(b.alloc(n * 4, s));
  GEEK_TRY(c.alloc(n * 4, s));
  iota_u32<<<grid_for(n, 256), 256, 0, s>>>(perm, n);
  GEEK_CHECK_LAUNCH();
  for (int col = ncols - 1; col >= 0; --col) {
    int nb = bits ? bits[col] : 32;
    if (nb <= 0) continue;
    gather_col<<<grid_for(n, 256), 256, 0, s>>>(cols[col], 1, 0, perm, a.as<uint32_t>(), n);
    GEEK_CHECK_LAUNCH();
    GEEK_CHECK_CUDA(cudaMemcpyAsync(c.ptr, perm, n * 4, cudaMemcpyDeviceToDevice, s));
    GEEK_TRY(radix_sort_pairs_u32(a.as<uint32_t>(), c.as<uint32_t>(), b.as<uint32_t>(), perm, n,
                                  nb, s));
  }
  return GEEK_OK;
}

__global__ void row_boundaries(const uint32_t* rows, int width, const uint32_t* perm,
                               uint32_t* flag, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t f = 0;
    if (i > 0) {
      const uint32_t* a = rows + (uint64_t)perm[i] * width;
      const uint32_t* b = rows + (uint64_t)perm[i - 1] * width;
      for (int c = 0; c < width; ++c)
        if (a[c] != b[c]) {
          f = 1;
          break;
        }
    }
    flag[i] = f;
  }
}

__global__ void add_flag(uint32_t* gid, const uint32_t* flag, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    gid[i] += flag[i];
}

}  // namespace geek

using namespace geek;

extern "C" {

int geek_version(void) { return 1; }

const char* geek_last_error(void) { return geek::last_error(); }

int geek_device_sms(void) {
  int dev = 0, sms = 0;
  GEEK_CHECK_CUDA(cudaGetDevice(&dev));
  GEEK_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  return sms;
}

int geek_group_rows(const uint32_t* rows, uint64_t nrows, int width, const int* bits_host,
                    uint32_t* perm, uint32_t* gid, uint64_t* ngroups_host, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(width >= 1 && width <= 64, "width %d outside [1, 64]", width);
  if (nrows == 0) {
    if (ngroups_host) *ngroups_host = 0;
    return GEEK_OK;
  }
  GEEK_REQUIRE(nrows < 0xFFFFFFFFull, "too many rows");
  GEEK_TRY(lex_argsort_rows(rows, nrows, width, bits_host, perm, s));
  Scratch flag;
  GEEK_TRY(flag.alloc(nrows * 4, s));
  row_boundaries<<<grid_for(nrows, 256), 256, 0, s>>>(rows, width, perm, flag.as<uint32_t>(), nrows);
  GEEK_CHECK_LAUNCH();
  uint64_t tot = 0;
  GEEK_TRY(exclusive_scan_u32(flag.as<uint32_t>(), gid, nrows, s, &tot));
  add_flag<<<grid_for(nrows, 256), 256, 0, s>>>(gid, flag.as<uint32_t>(), nrows);
  GEEK_CHECK_LAUNCH();
  if (ngroups_host) *ngroups_host = tot + 1;
  return GEEK_OK;
}

}  // extern "C"
