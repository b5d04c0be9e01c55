// MinHash kernels: forward permutation, segmented-min set signatures and the
// inverse-rank scan that produces SILK bucket signatures without touching
// bucket member lists (hashing.py:126-140, :265-282; engine.py:256-266).
#include "common.cuh"

#include <cstdlib>

#include <cmath>

namespace geek {

static int upload_perms(const geek_perm_t* perms_host, int nperm, Scratch& buf, cudaStream_t s) {
  GEEK_TRY(validate_perms(perms_host, nperm));
  GEEK_TRY(buf.alloc(sizeof(geek_perm_t) * nperm, s));
  GEEK_CHECK_CUDA(cudaMemcpyAsync(buf.ptr, perms_host, sizeof(geek_perm_t) * nperm,
                                  cudaMemcpyHostToDevice, s));
  return GEEK_OK;
}

__global__ void perm_forward_kernel(const geek_perm_t* perms, int nperm, const uint32_t* tables,
                                    const uint32_t* x, uint64_t count, uint32_t* out) {
  const int p = blockIdx.y;
  const geek_perm_t pm = perms[p];
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[(uint64_t)p * count + i] = perm_forward(pm, tables, x[i]);
}

__global__ void perm_inverse_kernel(const geek_perm_t* perms, int nperm, const uint32_t* tables,
                                    const uint32_t* r, uint64_t count, uint32_t* out) {
  const int p = blockIdx.y;
  const geek_perm_t pm = perms[p];
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[(uint64_t)p * count + i] = perm_inverse(pm, tables, r[i]);
}

__device__ __forceinline__ uint64_t find_segment(const uint64_t* off, uint64_t nseg, uint64_t e) {
  // largest s with off[s] <= e (segments non-empty)
  uint64_t lo = 0, hi = nseg;  // invariant off[lo] <= e < off[hi]
  while (hi - lo > 1) {
    uint64_t mid = (lo + hi) >> 1;
    if (off[mid] <= e) lo = mid;
    else hi = mid;
  }
  return lo;
}

__global__ void set_minhash_kernel(const geek_perm_t* perms, int nperm, const uint32_t* tables,
                                   const uint32_t* flat, const uint64_t* off, uint64_t nsets,
                                   uint64_t total, uint32_t* sig) {
  extern __shared__ geek_perm_t sp[];
  for (int i = threadIdx.x; i < nperm; i += blockDim.x) sp[i] = perms[i];
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u); base < total;
       base += stride) {
    const uint64_t e = base + lane;
    const bool valid = e < total;
    uint64_t s = valid ? find_segment(off, nsets, e) : ~0ull;
    uint32_t x = valid ? flat[e] : 0;
    unsigned peers = __match_any_sync(0xffffffffu, s);
    const bool leader = valid && (__ffs(peers) - 1 == (int)lane);
    for (int p = 0; p < nperm; ++p) {
      uint32_t v = valid ? perm_forward(sp[p], tables, x) : 0xFFFFFFFFu;
      uint32_t mn = __reduce_min_sync(peers, v);
      if (leader) atomicMin(&sig[s * nperm + p], mn);
    }
  }
}

// Rank-table regime (every function is a table over a universe u <= 4096,
// hashing.py:80-95): all nperm tables sit in shared memory, one warp per set
// keeps up to 4 of the set's ids per lane in registers, and each function's
// minimum is a shared-memory lookup per id plus one warp min-reduction --
// no segment search and no atomics.
constexpr int kTabSetRegs = 4;

__global__ void __launch_bounds__(256) set_minhash_tables_kernel(const geek_perm_t* perms, int nperm,
                                                                 const uint32_t* tables, uint32_t u,
                                                                 const uint32_t* __restrict__ flat,
                                                                 const uint64_t* __restrict__ off,
                                                                 uint64_t nsets, uint32_t* sig) {
  extern __shared__ uint32_t st[];  // [nperm][u]
  for (int p = 0; p < nperm; ++p)
    for (uint32_t i = threadIdx.x; i < u; i += blockDim.x) st[(size_t)p * u + i] = tables[perms[p].table + i];
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  const uint64_t wpb = blockDim.x >> 5;
  for (uint64_t s = blockIdx.x * wpb + (threadIdx.x >> 5); s < nsets; s += (uint64_t)gridDim.x * wpb) {
    const uint64_t b = off[s], e = off[s + 1];
    uint32_t x[kTabSetRegs];
#pragma unroll
    for (int r = 0; r < kTabSetRegs; ++r) {
      const uint64_t q = b + lane + 32ull * r;
      x[r] = q < e ? flat[q] : 0xFFFFFFFFu;
    }
    const bool more = e - b > 32ull * kTabSetRegs;
    for (int p = 0; p < nperm; ++p) {
      const uint32_t* tp = st + (size_t)p * u;
      uint32_t mn = 0xFFFFFFFFu;
#pragma unroll
      for (int r = 0; r < kTabSetRegs; ++r)
        if (x[r] != 0xFFFFFFFFu) mn = min(mn, tp[x[r]]);
      if (more)
        for (uint64_t q = b + lane + 32ull * kTabSetRegs; q < e; q += 32) mn = min(mn, tp[flat[q]]);
      mn = __reduce_min_sync(0xffffffffu, mn);
      if (lane == 0) sig[s * nperm + p] = mn;
    }
  }
}

// One thread per rank r of permutation p: id = pi_p^-1(r); every table's
// bucket of that id takes min(., r).  Blocks of finished permutations exit.
__global__ void __launch_bounds__(256) invscan_kernel(const uint32_t* __restrict__ codes, uint64_t n,
                                                      int m, uint64_t t, const geek_perm_t* perms,
                                                      const uint32_t* tables, uint32_t* sig,
                                                      unsigned long long* filled,
                                                      const int* active, uint64_t r0,
                                                      uint64_t r1) {
  // only permutations unfinished after the previous chunk are launched: a
  // permutation that completes inside this chunk must still scan all of it
  const int p = active[blockIdx.y];
  const geek_perm_t pm = perms[p];
  const uint64_t mt = (uint64_t)m * t;
  uint32_t* sp = sig + (uint64_t)p * mt;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = r0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < r1; r += stride) {
    const uint32_t id = perm_inverse(pm, tables, static_cast<uint32_t>(r));
    const uint32_t* row = codes + (uint64_t)id * m;
    unsigned long long newly = 0;
    for (int j = 0; j < m; ++j) {
      const uint32_t code = __ldg(row + j);
      uint32_t* a = sp + (uint64_t)j * t + code;
      if (__ldcg(a) > (uint32_t)r) {
        uint32_t old = atomicMin(a, (uint32_t)r);
        newly += (old == GEEK_NONE);
      }
    }
    if (newly) atomicAdd(&filled[p], newly);
  }
}

}  // namespace geek

using namespace geek;

extern "C" {

int geek_perm_forward(const geek_perm_t* perms_host, int nperm, const uint32_t* tables,
                      const uint32_t* x, uint64_t count, uint32_t* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (count == 0) return GEEK_OK;
  Scratch pb;
  GEEK_TRY(upload_perms(perms_host, nperm, pb, s));
  dim3 grid(grid_for(count, 256, 4096), nperm);
  perm_forward_kernel<<<grid, 256, 0, s>>>(pb.as<geek_perm_t>(), nperm, tables, x, count, out);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

int geek_perm_inverse(const geek_perm_t* perms_host, int nperm, const uint32_t* tables,
                      const uint32_t* r, uint64_t count, uint32_t* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (count == 0) return GEEK_OK;
  Scratch pb;
  GEEK_TRY(upload_perms(perms_host, nperm, pb, s));
  dim3 grid(grid_for(count, 256, 4096), nperm);
  perm_inverse_kernel<<<grid, 256, 0, s>>>(pb.as<geek_perm_t>(), nperm, tables, r, count, out);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

int geek_set_minhash(const geek_perm_t* perms_host, int nperm, const uint32_t* tables,
                     const uint32_t* flat, const uint64_t* offsets, uint64_t nsets, uint32_t* sig,
                     void* stream) {
  cudaStream_t s = as_stream(stream);
  if (nsets == 0) return GEEK_OK;
  Scratch pb;
  GEEK_TRY(upload_perms(perms_host, nperm, pb, s));
  uint64_t total = 0;
  GEEK_CHECK_CUDA(cudaMemcpyAsync(&total, offsets + nsets, 8, cudaMemcpyDeviceToHost, s));
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
  GEEK_CHECK_CUDA(cudaMemsetAsync(sig, 0xFF, nsets * nperm * 4ull, s));
  if (total == 0) return GEEK_OK;
  bool all_tables = nperm > 0;
  uint32_t u = nperm > 0 ? perms_host[0].u : 0;
  for (int p = 0; p < nperm; ++p) all_tables = all_tables && perms_host[p].table != GEEK_NONE && perms_host[p].u == u;
  const size_t tsm = (size_t)nperm * u * 4;
  if (all_tables && u <= 4096 && tsm <= 200 * 1024 && !getenv("GEEK_MINHASH_GENERIC")) {
    if (tsm > 48 * 1024)
      GEEK_CHECK_CUDA(cudaFuncSetAttribute(set_minhash_tables_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)tsm));
    set_minhash_tables_kernel<<<grid_for(nsets, 8, 148 * (tsm > 100 * 1024 ? 1 : 2) * 4), 256, tsm, s>>>(
        pb.as<geek_perm_t>(), nperm, tables, u, flat, offsets, nsets, sig);
    GEEK_CHECK_LAUNCH();
    return GEEK_OK;
  }
  size_t smem = sizeof(geek_perm_t) * nperm;
  set_minhash_kernel<<<grid_for(total, 256, 148 * 16), 256, smem, s>>>(pb.as<geek_perm_t>(), nperm,
                                                                      tables, flat, offsets, nsets,
                                                                      total, sig);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

int geek_silk_invscan(const uint32_t* codes, uint64_t n, int m, uint64_t t,
                      const geek_perm_t* perms_host, int nperm, const uint32_t* tables,
                      uint32_t* sig, const uint64_t* nonempty_host, uint64_t* draws_host,
                      void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(m >= 1 && t >= 1 && n >= 1, "invscan: empty partition");
  for (int p = 0; p < nperm; ++p)
    GEEK_REQUIRE(perms_host[p].u == n, "invscan: permutation %d universe %llu != n %llu", p,
                 (unsigned long long)perms_host[p].u, (unsigned long long)n);
  Scratch pb, ctr;
  GEEK_TRY(upload_perms(perms_host, nperm, pb, s));
  const uint64_t mt = (uint64_t)m * t;
  GEEK_TRY(ctr.alloc(12ull * nperm, s));
  unsigned long long* filled = ctr.as<unsigned long long>();
  int* active = reinterpret_cast<int*>(filled + nperm);
  std::vector<unsigned long long> tgt(nperm, nonempty_host ? *nonempty_host : mt);
  std::vector<int> act(nperm);
  for (int p = 0; p < nperm; ++p) act[p] = p;
  GEEK_CHECK_CUDA(cudaMemsetAsync(filled, 0, 8ull * nperm, s));
  GEEK_CHECK_CUDA(cudaMemsetAsync(sig, 0xFF, mt * nperm * 4ull, s));
  // coupon-collector estimate of the scan length for buckets of ~n/t ids
  double est = (double)t * (std::log((double)mt) + 2.0) * 1.5 + 1024.0;
  uint64_t r0 = 0, chunk = (uint64_t)est;
  std::vector<unsigned long long> got(nperm);
  const int sms = 148;
  int nact = nperm;
  while (r0 < n && nact > 0) {
    uint64_t r1 = r0 + chunk < n ? r0 + chunk : n;
    GEEK_CHECK_CUDA(cudaMemcpyAsync(active, act.data(), 4ull * nact, cudaMemcpyHostToDevice, s));
    dim3 grid(grid_for(r1 - r0, 256, sms * 8), nact);
    invscan_kernel<<<grid, 256, 0, s>>>(codes, n, m, t, pb.as<geek_perm_t>(), tables, sig, filled,
                                        active, r0, r1);
    GEEK_CHECK_LAUNCH();
    GEEK_CHECK_CUDA(cudaMemcpyAsync(got.data(), filled, 8ull * nperm, cudaMemcpyDeviceToHost, s));
    GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
    r0 = r1;
    nact = 0;
    for (int p = 0; p < nperm; ++p)
      if (got[p] < tgt[p]) act[nact++] = p;
    chunk *= 2;
  }
  if (draws_host) *draws_host = r0;
  return GEEK_OK;
}

}  // extern "C"
