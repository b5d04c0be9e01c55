// Shared helpers for libgeek: status handling, stream-ordered scratch,
// the MinHash permutation (forward / inverse) and device primitives.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/geek.h"

namespace geek {

void set_error(const char* fmt, ...);

struct Status {
  int code = GEEK_OK;
};

#define GEEK_CHECK_CUDA(expr)                                                      \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      ::geek::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,                 \
                        cudaGetErrorString(_e));                                   \
      return _e == cudaErrorMemoryAllocation ? GEEK_ENOMEM : GEEK_ECUDA;           \
    }                                                                              \
  } while (0)

#define GEEK_CHECK_LAUNCH() GEEK_CHECK_CUDA(cudaGetLastError())

#define GEEK_REQUIRE(cond, ...)          \
  do {                                   \
    if (!(cond)) {                       \
      ::geek::set_error(__VA_ARGS__);    \
      return GEEK_EINVAL;                \
    }                                    \
  } while (0)

#define GEEK_TRY(expr)          \
  do {                          \
    int _s = (expr);            \
    if (_s != GEEK_OK) return _s; \
  } while (0)

// keep the stream-ordered pool's memory cached across synchronisations
// (the default release threshold of 0 unmaps it at every sync)
void ensure_pool();

// Caller-provided workspace: while a WorkspaceScope is alive on this host
// thread, every Scratch carves its buffer out of the caller's device memory
// (256-byte aligned bump allocation, nothing freed until the scope ends)
// instead of the stream-ordered pool.
struct Workspace {
  char* base = nullptr;
  size_t size = 0, used = 0;
};
Workspace*& tls_workspace();
struct WorkspaceScope {
  Workspace ws;
  Workspace* prev;
  WorkspaceScope(void* base, size_t bytes) : prev(tls_workspace()) {
    ws.base = static_cast<char*>(base);
    ws.size = bytes;
    tls_workspace() = base ? &ws : nullptr;
  }
  ~WorkspaceScope() { tls_workspace() = prev; }
  WorkspaceScope(const WorkspaceScope&) = delete;
  WorkspaceScope& operator=(const WorkspaceScope&) = delete;
};

// Stream-ordered scratch buffer (cudaMallocAsync / cudaFreeAsync), or a slice
// of the caller's workspace inside a WorkspaceScope.
struct Scratch {
  void* ptr = nullptr;
  cudaStream_t stream = nullptr;
  bool pooled = false;
  Scratch() = default;
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  ~Scratch() {
    if (ptr && pooled) cudaFreeAsync(ptr, stream);
  }
  int alloc(size_t bytes, cudaStream_t s) {
    if (ptr && pooled) cudaFreeAsync(ptr, stream);
    ptr = nullptr;
    stream = s;
    if (bytes == 0) bytes = 16;
    if (Workspace* w = tls_workspace()) {
      const size_t off = (w->used + 255) & ~(size_t)255;
      if (off + bytes > w->size) {
        set_error("workspace of %zu bytes too small (needs more than %zu)", w->size, off + bytes);
        return GEEK_ERANGE;
      }
      ptr = w->base + off;
      w->used = off + bytes;
      pooled = false;
      return GEEK_OK;
    }
    pooled = true;
    ensure_pool();
    cudaError_t e = cudaMallocAsync(&ptr, bytes, s);
    if (e != cudaSuccess) {
      set_error("cudaMallocAsync(%zu): %s", bytes, cudaGetErrorString(e));
      ptr = nullptr;
      return e == cudaErrorMemoryAllocation ? GEEK_ENOMEM : GEEK_ECUDA;
    }
    return GEEK_OK;
  }
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(ptr);
  }
};

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 32u) {
  uint64_t g = (n + block - 1) / block;
  if (g == 0) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

// ---------------------------------------------------------------------------
// MinHash permutation (hashing.py:97-140)

__device__ __forceinline__ uint32_t perm_mix(const geek_perm_t& p, uint32_t x) {
  x = (x + p.a1) & p.mask;
  x ^= x >> p.s1;
  x = (x * p.c1) & p.mask;
  x ^= x >> p.s2;
  x = (x * p.c2) & p.mask;
  x ^= x >> p.s1;
  return x;
}

__device__ __forceinline__ uint32_t unxorshift(uint32_t y, uint32_t s) {
  // inverse of y = x ^ (x >> s) on w <= 32 bits
  uint32_t x = y;
  for (uint32_t k = s; k < 32; k += s) x = y ^ (x >> s);
  return x;
}

__device__ __forceinline__ uint32_t perm_unmix(const geek_perm_t& p, uint32_t y) {
  y = unxorshift(y, p.s1);
  y = (y * p.c2inv) & p.mask;
  y = unxorshift(y, p.s2);
  y = (y * p.c1inv) & p.mask;
  y = unxorshift(y, p.s1);
  return (y - p.a1) & p.mask;
}

__device__ __forceinline__ uint32_t perm_forward(const geek_perm_t& p, const uint32_t* tables,
                                                 uint32_t x) {
  if (p.table != GEEK_NONE) return tables[p.table + x];
  uint32_t y = perm_mix(p, x);
  while (y >= p.u) y = perm_mix(p, y);
  return y;
}

__device__ __forceinline__ uint32_t perm_inverse(const geek_perm_t& p, const uint32_t* tables,
                                                 uint32_t r) {
  if (p.inv_table != GEEK_NONE) return tables[p.inv_table + r];
  uint32_t y = perm_unmix(p, r);
  while (y >= p.u) y = perm_unmix(p, y);
  return y;
}

constexpr int kMaxPerms = 512;
int validate_perms(const geek_perm_t* perms, int nperm);

// ---------------------------------------------------------------------------
// even split (transform.py:95-100): slot of a rank

__device__ __forceinline__ uint32_t slot_of_rank(uint64_t rank, uint64_t n, uint64_t t) {
  uint64_t q = n / t, r = n % t;
  uint64_t big = r * (q + 1);
  if (rank < big) return static_cast<uint32_t>(rank / (q + 1));
  return static_cast<uint32_t>(r + (rank - big) / q);
}

// order-preserving uint64 image of a double; -0 == +0, NaN on top
__device__ __forceinline__ uint64_t f64_key(double v) {
  if (v != v) return ~0ull;
  if (v == 0.0) v = 0.0;
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// ---------------------------------------------------------------------------
// device primitives (prims.cu)

// exclusive scan; returns the total through *total_host if non-null (SYNC then)
int exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t s,
                       uint64_t* total_host = nullptr);
int exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, cudaStream_t s,
                       uint64_t* total_host = nullptr);

// stable LSD radix sort of (key, val) u32 pairs over the low `bits` bits of key.
// Result lands in (kout, vout); kin/vin are clobbered (used as ping-pong).
int radix_sort_pairs_u32(uint32_t* kin, uint32_t* vin, uint32_t* kout, uint32_t* vout, uint64_t n,
                         int bits, cudaStream_t s);

// lexicographic stable argsort of rows [n][width] (u32 columns) -> perm
int lex_argsort_rows(const uint32_t* rows, uint64_t n, int width, const int* bits, uint32_t* perm,
                     cudaStream_t s);

// lexicographic stable argsort over separate contiguous columns cols[c][n]
int argsort_cols(const uint32_t* const* cols, int ncols, const int* bits, uint64_t n, uint32_t* perm,
                 cudaStream_t s);

int bitlen_u64(uint64_t v);

// tensor-core assignment screen (tc_screen.cu)
int exponent_range_f32_device(const float* X, uint64_t total, int* out, cudaStream_t s);
// nprod: 1 / 3 TF32 products, 16 = FP16x3 over operands scaled by xscale (a
// power of two chosen by prepare; the kernel sets *ovf if a scaled point
// coordinate leaves the f16 range -- the caller then reruns with nprod 3)
int tc_screen_prepare(const double* C, uint64_t k, int d, int nprod, uint32_t lbo, uint32_t sbo, Scratch& img,
                      Scratch& c2, Scratch& mu, unsigned long long* cmax_dev, int& nct, float& xscale,
                      cudaStream_t s);
// C[n][m] = A[n][kk] . B[m][kk]^T in float64 through cuBLAS (blas.cu, loaded at run time)
int dgemm_nt(const double* A, const double* B, double* Cout, int n, int m, int kk, cudaStream_t s);
bool cublas_available();
// the same over f16 operands with fp32 accumulation and output (cublasGemmEx)
int hgemm_nt_f32(const void* A, const void* B, float* Cout, int n, int m, int kk, cudaStream_t s);
// mu and the FP16 scale {s, 2/s^2} of the wide-row FP16x3 screen (tc_screen.cu)
int tc_wide_prepare(const double* C, uint64_t k, int d, Scratch& mu, unsigned long long* cmax_dev, cudaStream_t s);
// {xscale, oscale} of a prepared screen (device memory inside its mu scratch)
const float* tc_scal(const Scratch& mu, int d);
// nprod 17 = tile-local FP16 (one product against each tile's origin center): see tc_screen.cu;
// nprod 16 with origins (no E table, with_E = false): the top-4 lists start at a bound from
// each tile's origin center instead of +inf
struct TcLocal {
  const float* cf;  // [k][d] float32 c'
  const int* j0;    // [ntiles] origin center per 128-point tile
  const float* Es;  // [k][nct * 192] origin table
  const unsigned long long* cmax;  // [0] |c'|max bits (from tc_screen_prepare)
  const float* dmin = nullptr;     // NPROD = 16: [k][nct] center-tile distance bounds (tile skipping)
  unsigned long long* tiles_done = nullptr;  // (point tile, center tile) pairs multiplied (device counter)
};
int tc_screen_launch(const float* X, uint64_t n, int d, int nprod, const Scratch& img, const Scratch& c2,
                     const Scratch& mu, uint64_t k, int nct, uint32_t lbo, uint32_t sbo, float* top_s, int* top_i,
                     double* xpart, float xscale, unsigned* ovf, cudaStream_t s, const TcLocal* loc = nullptr,
                     int xstride = 1, const unsigned* run_if = nullptr);
int tc_local_prepare(const double* C, uint64_t k, int d, const float* X, uint64_t n, uint32_t lbo, uint32_t sbo,
                     const Scratch& mu17, float xscale, int nct17, Scratch& cf, Scratch& Es, Scratch& j0, TcLocal& loc,
                     cudaStream_t s, bool with_E = true, Scratch* dmin = nullptr);

__global__ void iota_u32(uint32_t* p, uint64_t n);
__global__ void fill_u32(uint32_t* p, uint32_t v, uint64_t n);
__global__ void add_flag(uint32_t* gid, const uint32_t* flag, uint64_t n);

}  // namespace geek
