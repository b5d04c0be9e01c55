// K2, shared-memory form: the exact even rank split of keys [m][n] into t
// buckets per table, ties by id (transform.py:95-109; engine.py:216-225) --
// the same result as np.lexsort((arange(n), values)) + even split, with every
// random lookup in shared memory instead of L2.
//
//   1. sample histogram of the top 13 key bits per table (sign, exponent,
//      one mantissa bit: half-octave cells); a sampled cell gets
//      ceil(count / target) fine bins (fine bin = cell base + the next 32 key
//      bits scaled into the cell's bins, monotone in the key), an unsampled
//      cell none (its keys join the next cell's first bin);
//   2. exact fine-bin histogram, table by table, with the table's cell map and
//      counters in shared memory (one global flush per block);
//   3. scan -> each bin's exact rank range; bins inside one bucket get that
//      slot, bins straddling a boundary become segments;
//   4. codes pass, table-major and coalesced: slot from the shared bin map, or
//      (key, id) staged into the bin's segment (warp-aggregated cursors);
//   5. every segment is sorted by (key, id) in shared memory (bitonic) and its
//      ids get the slot of their exact rank; larger segments (giant tie
//      classes) take a global lexicographic sort;
//   6. tiled transpose into the id-major (strided) code rows.
// Traffic: keys read twice + codes written twice (table-major, then rows),
// against round 1's L2-bound global-atomic histogram and dependent lookups.
#include "common.cuh"

#include <algorithm>
#include <cmath>
#include <vector>

namespace geek {

constexpr int kV2Cb = 13;        // coarse bits: half-octave cells
constexpr int kV2Cells = 1 << kV2Cb;  // the cell map (SMEM: 32 KB, (first bin << 16) | bins)
constexpr int kV2Bins = 16384;   // fine bins per table (SMEM counters / bin map: 64 KB): two blocks per SM
constexpr int kV2Seg = 16384;    // largest segment sorted in SMEM (12 B per entry: 192 KB)
constexpr uint32_t kV2Straddle = 0x80000000u;

struct V2Meta {
  uint32_t cmin, ncells, nbins, over;
};

__global__ void v2_sample_hist(const uint64_t* __restrict__ keys, uint64_t n, uint64_t stride, int cb,
                               uint32_t* hist) {
  const int j = blockIdx.y;
  const uint64_t ns = (n + stride - 1) / stride;
  uint32_t* h = hist + ((uint64_t)j << cb);
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < ns; s += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[keys[(uint64_t)j * n + s * stride] >> (64 - cb)], 1u);
}

// one block (1024 threads) per table: fine bins per cell (0 for unsampled cells), scan
__global__ void __launch_bounds__(1024) v2_layout(const uint32_t* hist, uint64_t stride, uint32_t target,
                                                  uint32_t* cinfo, V2Meta* meta) {
  const int j = blockIdx.x;
  const uint32_t* h = hist + (uint64_t)j * kV2Cells;
  __shared__ uint32_t s_run;
  __shared__ uint32_t warp_sums[32];
  if (threadIdx.x == 0) s_run = 0;
  __syncthreads();
  uint32_t* ci = cinfo + (uint64_t)j * kV2Cells;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint32_t base = 0; base < (uint32_t)kV2Cells; base += blockDim.x) {
    const uint32_t c = base + threadIdx.x;
    const uint64_t est = (uint64_t)h[c] * stride;
    const uint32_t nf = est ? (uint32_t)std::min<uint64_t>((est + target - 1) / target, 0xFFFFu) : 0u;
    uint32_t x = nf;  // block inclusive scan
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
      uint32_t v = warp_sums[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      warp_sums[lane] = v;
    }
    __syncthreads();
    const uint32_t incl = x + (w ? warp_sums[w - 1] : 0u) + s_run;
    ci[c] = ((incl - nf) << 16) | nf;  // bins < 2^16 (checked below)
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_run = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const uint32_t nb = s_run;
    meta[j] = V2Meta{0, (uint32_t)kV2Cells, nb, (nb > (uint32_t)kV2Bins || nb == 0) ? 1u : 0u};
  }
}

__device__ __forceinline__ uint32_t v2_bin(uint64_t key, int cb, const V2Meta& mt, const uint32_t* ci) {
  const uint32_t e = ci[(uint32_t)(key >> (64 - cb))];
  const uint32_t frac = (uint32_t)((key << cb) >> 32);
  const uint32_t b = (e >> 16) + (uint32_t)(((uint64_t)frac * (e & 0xFFFFu)) >> 32);
  return b < mt.nbins ? b : mt.nbins - 1;  // an unsampled cell past the last sampled one
}

// exact fine-bin counts, table blockIdx.y, counters in SMEM
__global__ void __launch_bounds__(512, 2) v2_hist(const uint64_t* __restrict__ keys, uint64_t n, int cb,
                                               const uint32_t* __restrict__ cinfo, const V2Meta* __restrict__ meta,
                                               const uint64_t* __restrict__ boff, uint32_t* fcnt) {
  extern __shared__ uint8_t smem[];
  const int j = blockIdx.y;
  const V2Meta mt = meta[j];
  uint32_t* ci = reinterpret_cast<uint32_t*>(smem);
  uint32_t* hc = ci + mt.ncells;
  for (uint32_t c = threadIdx.x; c < mt.ncells; c += blockDim.x) ci[c] = cinfo[(uint64_t)j * kV2Cells + c];
  for (uint32_t b = threadIdx.x; b < mt.nbins; b += blockDim.x) hc[b] = 0;
  __syncthreads();
  const uint64_t* kj = keys + (uint64_t)j * n;
  // 4 independent keys per thread in flight; lanes that hit the same bin (the
  // ids of a cluster-ordered table run in key runs) add once per warp
  const int lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x - lane; i0 < n; i0 += 8 * stride) {
    uint64_t key[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint64_t i = i0 + u * stride + lane;
      key[u] = i < n ? __ldg(kj + i) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool ok = i0 + u * stride + lane < n;
      const uint32_t b = ok ? v2_bin(key[u], cb, mt, ci) : 0xFFFFFFFFu;
      const unsigned grp = __match_any_sync(0xffffffffu, b);
      if (ok && lane == __ffs(grp) - 1) atomicAdd(&hc[b], (uint32_t)__popc(grp));
    }
  }
  __syncthreads();
  uint32_t* out = fcnt + boff[j];
  for (uint32_t b = threadIdx.x; b < mt.nbins; b += blockDim.x)
    if (hc[b]) atomicAdd(&out[b], hc[b]);
}

__global__ void widen_u32(const uint32_t* in, uint64_t* out, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

// bin -> slot (inside one bucket) or straddle flag; segment sizes and list
__global__ void v2_classify(const uint32_t* fcnt, const uint64_t* fstart, uint64_t totbins, const uint64_t* boff,
                            int m, uint64_t n, uint64_t t, uint32_t* bincode, uint64_t* segcnt, uint32_t* seglist,
                            unsigned long long* stats) {
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < totbins;
       b += (uint64_t)gridDim.x * blockDim.x) {
    int j = 0;
    while (j + 1 < m && boff[j + 1] <= b) ++j;
    const uint32_t c = fcnt[b];
    const uint64_t r0 = fstart[b] - (uint64_t)j * n;
    uint32_t code = 0;
    uint64_t sc = 0;
    if (c > 0) {
      code = slot_of_rank(r0, n, t);
      if (c > 1 && code != slot_of_rank(r0 + c - 1, n, t)) {
        code = kV2Straddle;
        sc = c;
        seglist[atomicAdd(&stats[4], 1ull)] = (uint32_t)b;
        atomicAdd(&stats[0], (unsigned long long)c);
        atomicMax(&stats[1], (unsigned long long)c);
        if (c > (uint32_t)kV2Seg) atomicAdd(&stats[2], (unsigned long long)c);
      }
    }
    bincode[b] = code;
    segcnt[b] = sc;
  }
}

// codes, table-major: slot from the SMEM bin map, or (key, id) staged
__global__ void __launch_bounds__(512, 2) v2_codes(const uint64_t* __restrict__ keys, uint64_t n, int cb,
                                                const uint32_t* __restrict__ cinfo, const V2Meta* __restrict__ meta,
                                                const uint64_t* __restrict__ boff, const uint32_t* __restrict__ bincode,
                                                const uint64_t* __restrict__ sbase, unsigned long long* sfill,
                                                uint32_t* codes_tm, uint64_t* st_key, uint32_t* st_id) {
  extern __shared__ uint8_t smem[];
  const int j = blockIdx.y;
  const V2Meta mt = meta[j];
  uint32_t* ci = reinterpret_cast<uint32_t*>(smem);
  uint32_t* bc = ci + mt.ncells;
  const uint64_t b0 = boff[j];
  for (uint32_t c = threadIdx.x; c < mt.ncells; c += blockDim.x) ci[c] = cinfo[(uint64_t)j * kV2Cells + c];
  for (uint32_t b = threadIdx.x; b < mt.nbins; b += blockDim.x) bc[b] = bincode[b0 + b];
  __syncthreads();
  const uint64_t* kj = keys + (uint64_t)j * n;
  uint32_t* cj = codes_tm + (uint64_t)j * n;
  const int lane = threadIdx.x & 31;
  const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
  // 4 independent keys per thread in flight (key -> SMEM cell -> SMEM bin map)
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u); i0 < n; i0 += 8 * step) {
    uint64_t key[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint64_t i = i0 + u * step + lane;
      key[u] = i < n ? __ldg(kj + i) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint64_t i = i0 + u * step + lane;
      const bool ok = i < n;
      const uint32_t bin = ok ? v2_bin(key[u], cb, mt, ci) : 0u;
      const uint32_t code = ok ? bc[bin] : 0u;
      const bool st = ok && (code & kV2Straddle);
      if (ok && !st) cj[i] = code;
      if (__ballot_sync(0xffffffffu, st)) {  // lanes of one straddling bin take consecutive slots of its segment
        const unsigned grp = __match_any_sync(0xffffffffu, st ? bin : 0xFFFFFFFFu);
        if (st) {
          const int leader = __ffs(grp) - 1;
          unsigned long long basepos = 0;
          if (lane == leader) basepos = atomicAdd(&sfill[b0 + bin], (unsigned long long)__popc(grp));
          basepos = __shfl_sync(grp, basepos, leader);
          const uint64_t pos = sbase[b0 + bin] + basepos + __popc(grp & ((1u << lane) - 1));
          st_key[pos] = key[u];
          st_id[pos] = (uint32_t)i;
        }
      }
    }
  }
}

// one block per segment (looping over the device list): SMEM bitonic sort of
// (key, id), exact ranks -> slots
__global__ void __launch_bounds__(1024) v2_resolve(const uint32_t* seglist, const unsigned long long* nseg,
                                                   const uint32_t* fcnt, const uint64_t* fstart,
                                                   const uint64_t* sbase, const uint64_t* boff, int m, uint64_t n,
                                                   uint64_t t, const uint64_t* st_key, const uint32_t* st_id,
                                                   uint32_t* codes_tm) {
  extern __shared__ uint8_t smem[];  // kV2Seg keys, then kV2Seg ids
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem);
  uint32_t* si = reinterpret_cast<uint32_t*>(sk + kV2Seg);
  const uint64_t ns = *nseg;
  for (uint64_t q = blockIdx.x; q < ns; q += gridDim.x) {
    const uint32_t b = seglist[q];
    const uint32_t c = fcnt[b];
    if (c > (uint32_t)kV2Seg) continue;  // global sort path
    int j = 0;
    while (j + 1 < m && boff[j + 1] <= b) ++j;
    uint32_t P = 1;
    while (P < c) P <<= 1;
    const uint64_t s0 = sbase[b];
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < P; e += blockDim.x) {
      sk[e] = e < c ? st_key[s0 + e] : ~0ull;
      si[e] = e < c ? st_id[s0 + e] : 0xFFFFFFFFu;
    }
    __syncthreads();
    for (uint32_t kk = 2; kk <= P; kk <<= 1)
      for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
        for (uint32_t e = threadIdx.x; e < P; e += blockDim.x) {
          const uint32_t p = e ^ jj;
          if (p > e) {
            const bool up = (e & kk) == 0;
            const uint64_t a = sk[e], bkey = sk[p];
            const uint32_t ia = si[e], ib = si[p];
            const bool gt = a > bkey || (a == bkey && ia > ib);
            if (gt == up) {
              sk[e] = bkey;
              sk[p] = a;
              si[e] = ib;
              si[p] = ia;
            }
          }
        }
        __syncthreads();
      }
    const uint64_t r0 = fstart[b] - (uint64_t)j * n;
    uint32_t* cj = codes_tm + (uint64_t)j * n;
    for (uint32_t e = threadIdx.x; e < c; e += blockDim.x) cj[si[e]] = slot_of_rank(r0 + e, n, t);
  }
}

// giant segments: rows (bin, key hi, key lo, id) of the staged entries
__global__ void v2_big_gather(const uint32_t* seglist, const unsigned long long* nseg, const uint32_t* fcnt,
                              const uint64_t* sbase, const uint64_t* st_key, const uint32_t* st_id, uint32_t* rows,
                              unsigned long long* cursor) {
  const uint64_t ns = *nseg;
  __shared__ unsigned long long base;
  for (uint64_t q = blockIdx.x; q < ns; q += gridDim.x) {
    const uint32_t b = seglist[q];
    const uint32_t c = fcnt[b];
    if (c <= (uint32_t)kV2Seg) continue;
    if (threadIdx.x == 0) base = atomicAdd(cursor, (unsigned long long)c);
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < c; e += blockDim.x) {
      uint32_t* r = rows + 4ull * (base + e);
      const uint64_t k = st_key[sbase[b] + e];
      r[0] = b;
      r[1] = (uint32_t)(k >> 32);
      r[2] = (uint32_t)k;
      r[3] = st_id[sbase[b] + e];
    }
    __syncthreads();
  }
}

__global__ void v2_big_rank(const uint32_t* rows, const uint32_t* perm, uint64_t nbig, const uint64_t* fstart,
                            const uint64_t* boff, int m, uint64_t n, uint64_t t, uint32_t* codes_tm) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nbig;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = rows[4ull * perm[q]];
    uint64_t lo = 0, hi = q;  // first sorted position of bin b
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (rows[4ull * perm[mid]] < b) lo = mid + 1;
      else hi = mid;
    }
    int j = 0;
    while (j + 1 < m && boff[j + 1] <= b) ++j;
    const uint64_t rank = fstart[b] - (uint64_t)j * n + (q - lo);
    codes_tm[(uint64_t)j * n + rows[4ull * perm[q] + 3]] = slot_of_rank(rank, n, t);
  }
}

// codes_tm [m][n] -> codes[i * stride + col + j]: tiles of 128 ids x 16 tables
__global__ void __launch_bounds__(256) v2_transpose(const uint32_t* __restrict__ codes_tm, uint64_t n, int m,
                                                    uint32_t* codes, uint64_t stride, uint64_t col) {
  __shared__ uint32_t tile[16][129];
  for (uint64_t i0 = (uint64_t)blockIdx.x * 128; i0 < n; i0 += (uint64_t)gridDim.x * 128) {
    for (int j0 = 0; j0 < m; j0 += 16) {
      const int jn = min(16, m - j0);
      __syncthreads();
      for (int e = threadIdx.x; e < jn * 128; e += 256) {
        const int jj = e >> 7, r = e & 127;
        if (i0 + r < n) tile[jj][r] = __ldg(codes_tm + (uint64_t)(j0 + jj) * n + i0 + r);
      }
      __syncthreads();
      for (int e = threadIdx.x; e < jn * 128; e += 256) {
        const int r = e / jn, jj = e - r * jn;
        if (i0 + r < n) codes[(i0 + r) * stride + col + j0 + jj] = tile[jj][r];
      }
    }
  }
}

// returns GEEK_OK, or 1 when the key distribution does not fit the SMEM maps
// (the caller then runs the global-memory split)
int rank_split_v2(const uint64_t* keys, uint64_t n, int m, uint64_t t, uint32_t* codes, uint64_t code_stride,
                  uint64_t col, uint64_t* stats_host, cudaStream_t s) {
  const int cb = kV2Cb;
  const uint64_t stride = n > (1ull << 18) ? n >> 18 : 1;
  const uint32_t target = (uint32_t)std::max<uint64_t>(256, (n + 13999) / 14000);
  Scratch hist, cinfo, meta;
  GEEK_TRY(hist.alloc((uint64_t)m << cb << 2, s));
  GEEK_CHECK_CUDA(cudaMemsetAsync(hist.ptr, 0, (uint64_t)m << cb << 2, s));
  GEEK_TRY(cinfo.alloc((uint64_t)m * kV2Cells * 4, s));
  GEEK_TRY(meta.alloc((uint64_t)m * sizeof(V2Meta), s));
  v2_sample_hist<<<dim3(grid_for((n + stride - 1) / stride, 256, 64), m), 256, 0, s>>>(keys, n, stride, cb,
                                                                                       hist.as<uint32_t>());
  GEEK_CHECK_LAUNCH();
  v2_layout<<<m, 1024, 0, s>>>(hist.as<uint32_t>(), stride, target, cinfo.as<uint32_t>(), meta.as<V2Meta>());
  GEEK_CHECK_LAUNCH();
  std::vector<V2Meta> mh(m);
  GEEK_CHECK_CUDA(cudaMemcpyAsync(mh.data(), meta.ptr, m * sizeof(V2Meta), cudaMemcpyDeviceToHost, s));
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));  // SMEM sizes and the bin offsets come from the layout
  uint32_t maxc = 0, maxb = 0;
  std::vector<uint64_t> bo(m + 1, 0);
  for (int j = 0; j < m; ++j) {
    if (mh[j].over) return 1;
    maxc = std::max(maxc, mh[j].ncells);
    maxb = std::max(maxb, mh[j].nbins);
    bo[j + 1] = bo[j] + mh[j].nbins;
  }
  const uint64_t totbins = bo[m];
  Scratch boff, fcnt, fcnt64, fstart, bincode, segcnt, sbase, sfill, seglist, stats, codes_tm;
  GEEK_TRY(boff.alloc((m + 1) * 8, s));
  GEEK_CHECK_CUDA(cudaMemcpyAsync(boff.ptr, bo.data(), (m + 1) * 8, cudaMemcpyHostToDevice, s));
  GEEK_TRY(fcnt.alloc(totbins * 4, s));
  GEEK_CHECK_CUDA(cudaMemsetAsync(fcnt.ptr, 0, totbins * 4, s));
  const size_t smem = (size_t)maxc * 4 + (size_t)maxb * 4;
  GEEK_CHECK_CUDA(cudaFuncSetAttribute(v2_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  GEEK_CHECK_CUDA(cudaFuncSetAttribute(v2_codes, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // blocks per table: enough to fill the SMs across the tables, each a long key stream
  const unsigned bx = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 4095) / 4096,
                                                                          (uint64_t)std::max(1, 2 * sms / m)));
  v2_hist<<<dim3(bx, m), 512, smem, s>>>(keys, n, cb, cinfo.as<uint32_t>(), meta.as<V2Meta>(), boff.as<uint64_t>(),
                                        fcnt.as<uint32_t>());
  GEEK_CHECK_LAUNCH();
  GEEK_TRY(fcnt64.alloc(totbins * 8, s));
  GEEK_TRY(fstart.alloc(totbins * 8, s));
  widen_u32<<<grid_for(totbins, 256), 256, 0, s>>>(fcnt.as<uint32_t>(), fcnt64.as<uint64_t>(), totbins);
  GEEK_CHECK_LAUNCH();
  GEEK_TRY(exclusive_scan_u64(fcnt64.as<uint64_t>(), fstart.as<uint64_t>(), totbins, s));
  GEEK_TRY(bincode.alloc(totbins * 4, s));
  GEEK_TRY(segcnt.alloc(totbins * 8, s));
  GEEK_TRY(seglist.alloc(totbins * 4, s));
  GEEK_TRY(stats.alloc(64, s));
  GEEK_CHECK_CUDA(cudaMemsetAsync(stats.ptr, 0, 64, s));
  unsigned long long* st = stats.as<unsigned long long>();  // [0] staged [1] max seg [2] big [4] nseg [5] cursor
  v2_classify<<<grid_for(totbins, 256), 256, 0, s>>>(fcnt.as<uint32_t>(), fstart.as<uint64_t>(), totbins,
                                                     boff.as<uint64_t>(), m, n, t, bincode.as<uint32_t>(),
                                                     segcnt.as<uint64_t>(), seglist.as<uint32_t>(), st);
  GEEK_CHECK_LAUNCH();
  uint64_t nstage = 0;
  GEEK_TRY(sbase.alloc(totbins * 8, s));
  GEEK_TRY(exclusive_scan_u64(segcnt.as<uint64_t>(), sbase.as<uint64_t>(), totbins, s, &nstage));  // SYNC
  GEEK_TRY(sfill.alloc(totbins * 8, s));
  GEEK_CHECK_CUDA(cudaMemsetAsync(sfill.ptr, 0, totbins * 8, s));
  Scratch skey, sid;
  GEEK_TRY(skey.alloc(std::max<uint64_t>(1, nstage) * 8, s));
  GEEK_TRY(sid.alloc(std::max<uint64_t>(1, nstage) * 4, s));
  GEEK_TRY(codes_tm.alloc((uint64_t)m * n * 4, s));
  v2_codes<<<dim3(bx, m), 512, smem, s>>>(keys, n, cb, cinfo.as<uint32_t>(), meta.as<V2Meta>(), boff.as<uint64_t>(),
                                         bincode.as<uint32_t>(), sbase.as<uint64_t>(),
                                         sfill.as<unsigned long long>(), codes_tm.as<uint32_t>(),
                                         skey.as<uint64_t>(), sid.as<uint32_t>());
  GEEK_CHECK_LAUNCH();
  const size_t rsm = (size_t)kV2Seg * 12;
  GEEK_CHECK_CUDA(cudaFuncSetAttribute(v2_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));
  v2_resolve<<<(unsigned)(2 * sms), 1024, rsm, s>>>(seglist.as<uint32_t>(), st + 4, fcnt.as<uint32_t>(),
                                                  fstart.as<uint64_t>(), sbase.as<uint64_t>(), boff.as<uint64_t>(), m,
                                                  n, t, skey.as<uint64_t>(), sid.as<uint32_t>(),
                                                  codes_tm.as<uint32_t>());
  GEEK_CHECK_LAUNCH();
  unsigned long long sh[3] = {0, 0, 0};
  GEEK_CHECK_CUDA(cudaMemcpyAsync(sh, st, 24, cudaMemcpyDeviceToHost, s));
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));  // giant segments need a host-sized sort
  const uint64_t nbig = sh[2];
  if (nbig) {
    Scratch rows, perm;
    GEEK_TRY(rows.alloc(nbig * 16, s));
    GEEK_TRY(perm.alloc(nbig * 4, s));
    v2_big_gather<<<(unsigned)sms, 256, 0, s>>>(seglist.as<uint32_t>(), st + 4, fcnt.as<uint32_t>(),
                                               sbase.as<uint64_t>(), skey.as<uint64_t>(), sid.as<uint32_t>(),
                                               rows.as<uint32_t>(), st + 5);
    GEEK_CHECK_LAUNCH();
    GEEK_TRY(lex_argsort_rows(rows.as<uint32_t>(), nbig, 4, nullptr, perm.as<uint32_t>(), s));
    v2_big_rank<<<grid_for(nbig, 256), 256, 0, s>>>(rows.as<uint32_t>(), perm.as<uint32_t>(), nbig,
                                                    fstart.as<uint64_t>(), boff.as<uint64_t>(), m, n, t,
                                                    codes_tm.as<uint32_t>());
    GEEK_CHECK_LAUNCH();
  }
  v2_transpose<<<grid_for((n + 127) / 128, 1, (unsigned)(sms * 8)), 256, 0, s>>>(codes_tm.as<uint32_t>(), n, m, codes,
                                                                             code_stride, col);
  GEEK_CHECK_LAUNCH();
  if (stats_host) {
    stats_host[0] = totbins;
    stats_host[1] = nstage;
    stats_host[2] = sh[1];
    stats_host[3] = nbig;
  }
  return GEEK_OK;
}

}  // namespace geek
