// SILK voting and dedup helpers (seeding.py:93-134; engine.py:242-295):
// membership emission for binned buckets, strict-majority vote with the
// delta filter, dedup representatives and the canonical group order.
#include "common.cuh"

#include <algorithm>

namespace geek {

__global__ void emit_members_kernel(const uint32_t* __restrict__ codes, uint64_t n, int m, uint64_t t,
                                    const uint32_t* __restrict__ bb_off,
                                    const uint32_t* __restrict__ bb_bins, uint32_t* out_bin,
                                    uint32_t* out_id, uint64_t cap, unsigned long long* cursor) {
  const uint64_t total = n * (uint64_t)m;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = e / m;
    const int j = static_cast<int>(e - i * m);
    const uint64_t b = (uint64_t)j * t + codes[e];
    const uint32_t lo = bb_off[b], hi = bb_off[b + 1];
    for (uint32_t k = lo; k < hi; ++k) {
      unsigned long long pos = atomicAdd(cursor, 1ull);
      if (pos < cap) {
        out_bin[pos] = bb_bins[k];
        out_id[pos] = static_cast<uint32_t>(i);
      }
    }
  }
}

// bit b set when bucket b belongs to at least one bin
__global__ void binned_bitmap_kernel(const uint32_t* bb_off, uint64_t nb, uint32_t* words) {
  const uint64_t nw = (nb + 31) / 32;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    for (int k = 0; k < 32; ++k) {
      const uint64_t b = w * 32 + k;
      if (b < nb && bb_off[b + 1] > bb_off[b]) v |= 1u << k;
    }
    words[w] = v;
  }
}

// One thread per id row: test each table's bucket against the bitmap
// (shared memory when it fits), count the row's pairs, take a warp-aggregated
// range of the output, then write.
__global__ void __launch_bounds__(256) emit_rows_kernel(const uint32_t* __restrict__ codes, uint64_t n, int m,
                                                        uint64_t t, const uint32_t* __restrict__ bb_off,
                                                        const uint32_t* __restrict__ bb_bins,
                                                        const uint32_t* __restrict__ gwords, uint64_t nwords,
                                                        int smem_words, uint32_t* out_bin, uint32_t* out_id,
                                                        uint64_t cap, unsigned long long* cursor) {
  extern __shared__ uint32_t sw[];
  const bool in_smem = smem_words > 0;
  if (in_smem)
    for (uint64_t w = threadIdx.x; w < nwords; w += blockDim.x) sw[w] = gwords[w];
  __syncthreads();
  const uint32_t* words = in_smem ? sw : gwords;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u); base < n; base += stride) {
    const uint64_t i = base + lane;
    const bool valid = i < n;
    const uint32_t* row = codes + (valid ? i : 0) * m;
    uint32_t cnt = 0;
    if (valid)
      for (int j = 0; j < m; ++j) {
        const uint64_t b = (uint64_t)j * t + row[j];
        if ((words[b >> 5] >> (b & 31)) & 1u) cnt += bb_off[b + 1] - bb_off[b];
      }
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (unsigned)o) incl += u;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) continue;
    unsigned long long wbase = 0;
    if (lane == 31) wbase = atomicAdd(cursor, (unsigned long long)total);
    wbase = __shfl_sync(0xffffffffu, wbase, 31);
    unsigned long long pos = wbase + incl - cnt;
    if (cnt)
      for (int j = 0; j < m; ++j) {
        const uint64_t b = (uint64_t)j * t + row[j];
        if ((words[b >> 5] >> (b & 31)) & 1u)
          for (uint32_t k = bb_off[b]; k < bb_off[b + 1]; ++k, ++pos)
            if (pos < cap) {
              out_bin[pos] = bb_bins[k];
              out_id[pos] = static_cast<uint32_t>(i);
            }
      }
  }
}

// Strict-majority vote fused into the emission (seeding.py:107-114): an id's
// count in a bin is the number of its m buckets that belong to the bin, all
// visible in the id's own code row, so each (bin, id) is decided in place and
// only the winners are written.
constexpr int kRowBins = 64;  // bins one id can reach through its m buckets (checked)

// per bucket: (first entry, entries) of its bin list; per entry: (bin, size),
// with bins of 2m or more buckets dropped -- an id's count in a bin is at most
// m (one bucket per table), so nobody can win them.  A bucket with exactly one
// entry carries it inline as (bin, size | kPackOne): one dependent load less.
constexpr uint32_t kPackOne = 0x80000000u;
__global__ void pack_bins_kernel(const uint32_t* bb_off, const uint32_t* bb_bins, const uint32_t* bin_size,
                                 uint64_t nbk, int m, uint2* pack, uint2* ent, uint32_t* words) {
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nbk; b += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t lo = bb_off[b], hi = bb_off[b + 1];
    uint32_t c = 0;
    for (uint32_t k = lo; k < hi; ++k) {
      const uint32_t bin = bb_bins[k], sz = bin_size[bin];
      if (sz < 2u * (uint32_t)m) ent[lo + c++] = make_uint2(bin, sz);
    }
    pack[b] = c == 1 ? make_uint2(ent[lo].x, ent[lo].y | kPackOne) : make_uint2(lo, c);
    if (c) atomicOr(&words[b >> 5], 1u << (b & 31));
  }
}

// One block = 256 consecutive ids: their code rows (contiguous, id-major) are
// staged in SMEM with coalesced 16-byte loads; each thread then walks its row
// from SMEM with the winnable-bin bitmap in SMEM too.
constexpr int kEwThreads = 256;
#ifndef GEEK_EW_GROUP
#define GEEK_EW_GROUP 8
#endif
constexpr int kEwGroup = GEEK_EW_GROUP;  // tables whose bucket words are fetched together
__global__ void __launch_bounds__(kEwThreads) emit_winners_kernel(
    const uint32_t* __restrict__ codes, uint64_t n, int m, uint64_t t, const uint2* __restrict__ pack,
    const uint2* __restrict__ ent, const uint32_t* __restrict__ gwords, uint64_t nwords, int smem_words,
    uint32_t* out_bin, uint32_t* out_id, uint64_t cap, unsigned long long* cursor, unsigned long long* overflow) {
  extern __shared__ uint32_t sm[];
  const int ld = m + 1;
  uint32_t* srow = sm;                     // [256][m+1]
  uint32_t* sw = sm + kEwThreads * ld;     // bitmap
  const int tid = threadIdx.x;
  if (smem_words > 0)
    for (uint64_t w = tid; w < nwords; w += kEwThreads) sw[w] = gwords[w];
  const unsigned lane = tid & 31;
  for (uint64_t base = blockIdx.x * (uint64_t)kEwThreads; base < n; base += (uint64_t)gridDim.x * kEwThreads) {
    const int rows = (int)(n - base < (uint64_t)kEwThreads ? n - base : (uint64_t)kEwThreads);
    __syncthreads();  // previous rows consumed (and the bitmap is in)
    const uint32_t* src = codes + base * m;
    if ((m & 3) == 0) {
      const int n4 = rows * m / 4;
      for (int e4 = tid; e4 < n4; e4 += kEwThreads) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(src) + e4);
        const int e = 4 * e4, r = e / m, j = e - r * m;
        uint32_t* d = srow + r * ld + j;
        d[0] = v.x;
        d[1] = v.y;
        d[2] = v.z;
        d[3] = v.w;
      }
    } else {
      for (int e = tid; e < rows * m; e += kEwThreads) {
        const int r = e / m;
        srow[r * ld + (e - r * m)] = __ldg(src + e);
      }
    }
    __syncthreads();
    const uint64_t i = base + tid;
    uint32_t rb[kRowBins], rs[kRowBins];
    int nb = 0;
    const uint32_t* bm = smem_words > 0 ? sw : gwords;  // winnable-bucket bitmap (SMEM when it fits)
    if (tid < rows) {
      const uint32_t* row = srow + tid * ld;
      // 8 tables at a time: their bucket lists and first entries are
      // fetched together instead of as one dependent chain per table
      const uint32_t t32 = (uint32_t)t;  // m * t < 2^32 (checked by the caller)
      for (int j0 = 0; j0 < m; j0 += kEwGroup) {
        uint2 pk[kEwGroup], e0[kEwGroup];
#pragma unroll
        for (int u = 0; u < kEwGroup; ++u) {
          pk[u] = make_uint2(0u, 0u);
          if (j0 + u < m) {
            const uint32_t b = (uint32_t)(j0 + u) * t32 + row[j0 + u];
            const uint32_t w = bm[b >> 5];
            if ((w >> (b & 31)) & 1u) pk[u] = __ldg(pack + b);
          }
        }
#pragma unroll
        for (int u = 0; u < kEwGroup; ++u)
          e0[u] = (pk[u].y & kPackOne) ? make_uint2(pk[u].x, pk[u].y & ~kPackOne)
                  : pk[u].y            ? __ldg(ent + pk[u].x)
                                       : make_uint2(0u, 0u);
#pragma unroll
        for (int u = 0; u < kEwGroup; ++u)
          for (uint32_t k = 0, ne = (pk[u].y & kPackOne) ? 1u : pk[u].y; k < ne; ++k) {
            const uint2 e = k == 0 ? e0[u] : __ldg(ent + pk[u].x + k);
            if (nb < kRowBins) {
              rb[nb] = e.x;
              rs[nb] = e.y;
            }
            ++nb;
          }
      }
    }
    if (nb > kRowBins) {  // cannot happen for m <= 64 with one bin per bucket and table; keep loud
      atomicAdd(overflow, 1ull);
      nb = kRowBins;
    }
    // winners: first occurrence of each bin whose multiplicity is a strict
    // majority -- one pass: each entry's later duplicates are counted once and
    // marked seen (kRowBins <= 64 entries: 64-bit masks), the winner mask is
    // kept for the emission
    static_assert(kRowBins <= 64, "winner masks are 64-bit");
    uint64_t win = 0, seen = 0;
    for (int a = 0; a < nb; ++a) {
      if ((seen >> a) & 1ull) continue;
      const uint32_t ba = rb[a], sz = rs[a];
      if (2u * (uint32_t)nb <= sz) continue;  // count <= nb cannot be a strict majority
      uint32_t c = 1;
      for (int q = a + 1; q < nb; ++q)
        if (rb[q] == ba) {
          ++c;
          seen |= 1ull << q;
        }
      if (2u * c > sz) win |= 1ull << a;
    }
    const uint32_t cnt = (uint32_t)__popcll(win);
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (unsigned)o) incl += u;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) continue;
    unsigned long long wbase = 0;
    if (lane == 31) wbase = atomicAdd(cursor, (unsigned long long)total);
    wbase = __shfl_sync(0xffffffffu, wbase, 31);
    unsigned long long pos = wbase + incl - cnt;
    for (uint64_t w = win; w; w &= w - 1) {
      const int a = __ffsll((long long)w) - 1;
      if (pos < cap) {
        out_bin[pos] = rb[a];
        out_id[pos] = static_cast<uint32_t>(i);
      }
      ++pos;
    }
  }
}

__global__ void gather_u32(const uint32_t* src, const uint32_t* perm, uint32_t* dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[perm[i]];
}

// run starts of the sorted (a, b) sequence
__global__ void run_flags2(const uint32_t* a, const uint32_t* b, uint32_t* flag, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0) || a[i] != a[i - 1] || (b && b[i] != b[i - 1]);
}

__global__ void scatter_run_start(const uint32_t* flag, const uint32_t* ridx, uint32_t* start, uint64_t n,
                                  uint64_t nruns) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (flag[i]) start[ridx[i]] = static_cast<uint32_t>(i);
  if (blockIdx.x == 0 && threadIdx.x == 0) start[nruns] = static_cast<uint32_t>(n);
}

// winner flag per (bin, id) run: 2*count > bin size (seeding.py:110)
__global__ void winner_flags(const uint32_t* start, const uint32_t* sbin, const uint32_t* bin_size,
                             uint64_t nruns, uint32_t* win) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < nruns;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t cnt = start[r + 1] - start[r];
    const uint32_t b = sbin[start[r]];
    win[r] = 2ull * cnt > (uint64_t)bin_size[b];
  }
}

__global__ void compact_winners(const uint32_t* start, const uint32_t* sbin, const uint32_t* sid,
                                const uint32_t* win, const uint32_t* wpos, uint64_t nruns,
                                uint32_t* wbin, uint32_t* wid) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < nruns;
       r += (uint64_t)gridDim.x * blockDim.x)
    if (win[r]) {
      wbin[wpos[r]] = sbin[start[r]];
      wid[wpos[r]] = sid[start[r]];
    }
}

// keep winners whose bin has >= delta of them
__global__ void bin_keep_flags(const uint32_t* gstart, uint64_t ng, uint64_t delta, uint32_t* keep) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < ng;
       r += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c = gstart[r + 1] - gstart[r];
    keep[r] = c >= delta && c > 0;
  }
}

__global__ void expand_keep(const uint32_t* gstart, const uint32_t* keep, uint64_t ng, uint32_t* ekeep) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < ng;
       r += (uint64_t)gridDim.x * blockDim.x)
    for (uint32_t e = gstart[r]; e < gstart[r + 1]; ++e) ekeep[e] = keep[r];
}

// element-parallel: element e belongs to run gidx[e] + flag[e] - 1
__global__ void expand_keep_elems(const uint32_t* gidx, const uint32_t* flag, const uint32_t* keep, uint64_t n,
                                  uint32_t* ekeep) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x)
    ekeep[e] = keep[gidx[e] + flag[e] - 1];
}

__global__ void compact_pairs(const uint32_t* a, const uint32_t* b, const uint32_t* keep,
                              const uint32_t* pos, uint64_t n, uint32_t* oa, uint32_t* ob) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (keep[i]) {
      oa[pos[i]] = a[i];
      ob[pos[i]] = b[i];
    }
}

__device__ int lex_cmp(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb) {
  uint64_t k = na < nb ? na : nb;
  for (uint64_t i = 0; i < k; ++i)
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  return na < nb ? -1 : (na > nb ? 1 : 0);
}

__global__ void pick_reps_kernel(const uint32_t* flat, const uint64_t* off, const uint32_t* perm,
                                 const uint32_t* gid, uint64_t n, uint8_t* keep) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
       r += (uint64_t)gridDim.x * blockDim.x) {
    if (r > 0 && gid[r] == gid[r - 1]) continue;  // keep[] was zeroed by the host
    uint32_t best = perm[r];
    for (uint64_t q = r + 1; q < n && gid[q] == gid[r]; ++q) {
      const uint32_t c = perm[q];
      const uint64_t nc = off[c + 1] - off[c], nbst = off[best + 1] - off[best];
      if (nc > nbst || (nc == nbst && lex_cmp(flat + off[c], nc, flat + off[best], nbst) < 0))
        best = c;
    }
    keep[best] = 2;  // marked after all zeroing below
  }
}

__global__ void fix_keep(uint8_t* keep, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    keep[i] = keep[i] == 2;
}

// value at position p of a group's member tuple: id + 1, or 0 past the end
__global__ void tuple_digit(const uint32_t* flat, const uint64_t* off, const uint32_t* order,
                            uint64_t n, uint64_t p, uint32_t* out) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t g = order[r];
    const uint64_t len = off[g + 1] - off[g];
    out[r] = p < len ? flat[off[g] + p] + 1u : 0u;
  }
}

// class = position of the first element of the tie run in the current order
__global__ void tie_class(const uint32_t* cls_sorted, const uint32_t* dig_sorted, uint32_t* flag,
                          uint64_t n) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
       r += (uint64_t)gridDim.x * blockDim.x)
    flag[r] = (r == 0) || cls_sorted[r] != cls_sorted[r - 1] || dig_sorted[r] != dig_sorted[r - 1];
}

}  // namespace geek

using namespace geek;

extern "C" {

int geek_emit_members_codes(const uint32_t* codes, uint64_t n, int m, uint64_t t, const uint32_t* bb_off,
                            const uint32_t* bb_bins, uint32_t* out_bin, uint32_t* out_id, uint64_t cap,
                            uint64_t* count_host, void* stream) {
  cudaStream_t s = as_stream(stream);
  Scratch cur, bm;
  GEEK_TRY(cur.alloc(8, s));
  GEEK_CHECK_CUDA(cudaMemsetAsync(cur.ptr, 0, 8, s));
  if (n) {
    const uint64_t nb = (uint64_t)m * t, nw = (nb + 31) / 32;
    GEEK_TRY(bm.alloc(nw * 4, s));
    binned_bitmap_kernel<<<grid_for(nw, 256), 256, 0, s>>>(bb_off, nb, bm.as<uint32_t>());
    GEEK_CHECK_LAUNCH();
    const int smem_words = nw * 4 <= 96 * 1024 ? (int)nw : 0;
    if (smem_words * 4 > 48 * 1024)
      GEEK_CHECK_CUDA(cudaFuncSetAttribute(emit_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           smem_words * 4));
    emit_rows_kernel<<<grid_for(n, 256, 148 * 8), 256, smem_words * 4, s>>>(
        codes, n, m, t, bb_off, bb_bins, bm.as<uint32_t>(), nw, smem_words, out_bin, out_id, cap,
        cur.as<unsigned long long>());
    GEEK_CHECK_LAUNCH();
  }
  unsigned long long c = 0;
  GEEK_CHECK_CUDA(cudaMemcpyAsync(&c, cur.ptr, 8, cudaMemcpyDeviceToHost, s));
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
  *count_host = c;
  if (c > cap) {
    set_error("emit_members: %llu pairs exceed capacity %llu", c, (unsigned long long)cap);
    return GEEK_ERANGE;
  }
  return GEEK_OK;
}

int geek_emit_winners_codes(const uint32_t* codes, uint64_t n, int m, uint64_t t, const uint32_t* bb_off,
                            const uint32_t* bb_bins, const uint32_t* bin_size, uint32_t* out_bin, uint32_t* out_id,
                            uint64_t cap, uint64_t* count_host, void* stream) {
  cudaStream_t s = as_stream(stream);
  Scratch cur, bm, pk, en;
  GEEK_TRY(cur.alloc(16, s));
  GEEK_CHECK_CUDA(cudaMemsetAsync(cur.ptr, 0, 16, s));
  unsigned long long* cursor = cur.as<unsigned long long>();
  if (n) {
    GEEK_REQUIRE(m <= 256, "emit_winners: m = %d tables per row exceeds 256", m);
    const uint64_t nb = (uint64_t)m * t, nw = (nb + 31) / 32;
    GEEK_REQUIRE(nb < 0xFFFFFFFFull, "emit_winners: %llu buckets exceed 32-bit indexing", (unsigned long long)nb);
    uint32_t nent = 0;
    GEEK_CHECK_CUDA(cudaMemcpyAsync(&nent, bb_off + nb, 4, cudaMemcpyDeviceToHost, s));
    GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
    GEEK_TRY(bm.alloc(nw * 4, s));
    GEEK_TRY(pk.alloc(nb * 8, s));
    GEEK_TRY(en.alloc((size_t)(nent ? nent : 1) * 8, s));
    GEEK_CHECK_CUDA(cudaMemsetAsync(bm.ptr, 0, nw * 4, s));
    pack_bins_kernel<<<grid_for(nb, 256), 256, 0, s>>>(bb_off, bb_bins, bin_size, nb, m, pk.as<uint2>(),
                                                       en.as<uint2>(), bm.as<uint32_t>());
    GEEK_CHECK_LAUNCH();
    const size_t fixed = (size_t)4 * kEwThreads * (m + 1);
    const int smem_words = fixed + nw * 4 <= 160 * 1024 ? (int)nw : 0;
    const size_t smem = fixed + (size_t)smem_words * 4;
    GEEK_CHECK_CUDA(
        cudaFuncSetAttribute(emit_winners_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    emit_winners_kernel<<<(unsigned)std::min<uint64_t>((n + kEwThreads - 1) / kEwThreads, 148 * 8), kEwThreads,
                          smem, s>>>(codes, n, m, t, pk.as<uint2>(), en.as<uint2>(), bm.as<uint32_t>(), nw,
                                     smem_words, out_bin, out_id, cap, cursor, cursor + 1);
    GEEK_CHECK_LAUNCH();
  }
  unsigned long long c[2] = {0, 0};
  GEEK_CHECK_CUDA(cudaMemcpyAsync(c, cursor, 16, cudaMemcpyDeviceToHost, s));
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
  *count_host = c[0];
  if (c[1]) {
    set_error("emit_winners: %llu ids reach more than %d bins; use the pair path", c[1], kRowBins);
    return GEEK_ERANGE;
  }
  if (c[0] > cap) {
    set_error("emit_winners: %llu winners exceed capacity %llu", c[0], (unsigned long long)cap);
    return GEEK_ERANGE;
  }
  return GEEK_OK;
}

int geek_group_winners(const uint32_t* win_bin, const uint32_t* win_id, uint64_t nwin, uint64_t nbins,
                       uint64_t id_bound, uint64_t delta, uint32_t* out_bin, uint32_t* out_id, uint64_t* nout_host,
                       void* stream) {
  cudaStream_t s = as_stream(stream);
  *nout_host = 0;
  if (nwin == 0) return GEEK_OK;
  GEEK_REQUIRE(nwin < 0xFFFFFFFFull, "too many winners");
  const uint64_t nw = nwin;
  Scratch perm, wb, wi, gflag, gidx, gstart, gkeep, ekeep, epos;
  GEEK_TRY(perm.alloc(nw * 4, s));
  GEEK_TRY(wb.alloc(nw * 4, s));
  GEEK_TRY(wi.alloc(nw * 4, s));
  const uint32_t* cols[2] = {win_bin, win_id};
  const int bits[2] = {bitlen_u64(nbins ? nbins - 1 : 0) ? bitlen_u64(nbins - 1) : 1,
                       bitlen_u64(id_bound ? id_bound - 1 : 0) ? bitlen_u64(id_bound - 1) : 1};
  GEEK_TRY(argsort_cols(cols, 2, bits, nw, perm.as<uint32_t>(), s));
  gather_u32<<<grid_for(nw, 256), 256, 0, s>>>(win_bin, perm.as<uint32_t>(), wb.as<uint32_t>(), nw);
  gather_u32<<<grid_for(nw, 256), 256, 0, s>>>(win_id, perm.as<uint32_t>(), wi.as<uint32_t>(), nw);
  GEEK_CHECK_LAUNCH();
  // delta filter per bin (engine.py:281)
  GEEK_TRY(gflag.alloc(nw * 4, s));
  GEEK_TRY(gidx.alloc(nw * 4, s));
  run_flags2<<<grid_for(nw, 256), 256, 0, s>>>(wb.as<uint32_t>(), nullptr, gflag.as<uint32_t>(), nw);
  GEEK_CHECK_LAUNCH();
  uint64_t ng = 0;
  GEEK_TRY(exclusive_scan_u32(gflag.as<uint32_t>(), gidx.as<uint32_t>(), nw, s, &ng));
  GEEK_TRY(gstart.alloc((ng + 1) * 4, s));
  scatter_run_start<<<grid_for(nw, 256), 256, 0, s>>>(gflag.as<uint32_t>(), gidx.as<uint32_t>(),
                                                      gstart.as<uint32_t>(), nw, ng);
  GEEK_TRY(gkeep.alloc(ng * 4, s));
  bin_keep_flags<<<grid_for(ng, 256), 256, 0, s>>>(gstart.as<uint32_t>(), ng, delta, gkeep.as<uint32_t>());
  GEEK_TRY(ekeep.alloc(nw * 4, s));
  GEEK_TRY(epos.alloc(nw * 4, s));
  expand_keep_elems<<<grid_for(nw, 256), 256, 0, s>>>(gidx.as<uint32_t>(), gflag.as<uint32_t>(),
                                                      gkeep.as<uint32_t>(), nw, ekeep.as<uint32_t>());
  GEEK_CHECK_LAUNCH();
  uint64_t nk = 0;
  GEEK_TRY(exclusive_scan_u32(ekeep.as<uint32_t>(), epos.as<uint32_t>(), nw, s, &nk));
  compact_pairs<<<grid_for(nw, 256), 256, 0, s>>>(wb.as<uint32_t>(), wi.as<uint32_t>(), ekeep.as<uint32_t>(),
                                                  epos.as<uint32_t>(), nw, out_bin, out_id);
  GEEK_CHECK_LAUNCH();
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
  *nout_host = nk;
  return GEEK_OK;
}

int geek_majority_vote(const uint32_t* pair_bin, const uint32_t* pair_id, uint64_t npairs,
                       const uint32_t* bin_size, uint64_t nbins, uint64_t delta, uint32_t* win_bin,
                       uint32_t* win_id, uint64_t* nwin_host, void* stream) {
  cudaStream_t s = as_stream(stream);
  *nwin_host = 0;
  if (npairs == 0) return GEEK_OK;
  GEEK_REQUIRE(npairs < 0xFFFFFFFFull, "too many vote pairs");
  (void)nbins;
  const uint64_t n = npairs;
  Scratch perm, sbin, sid, flag, ridx, start, win, wpos, wb, wi, gflag, gidx, gstart, gkeep, ekeep, epos;
  GEEK_TRY(perm.alloc(n * 4, s));
  GEEK_TRY(sbin.alloc(n * 4, s));
  GEEK_TRY(sid.alloc(n * 4, s));
  const uint32_t* cols[2] = {pair_bin, pair_id};
  GEEK_TRY(argsort_cols(cols, 2, nullptr, n, perm.as<uint32_t>(), s));
  gather_u32<<<grid_for(n, 256), 256, 0, s>>>(pair_bin, perm.as<uint32_t>(), sbin.as<uint32_t>(), n);
  gather_u32<<<grid_for(n, 256), 256, 0, s>>>(pair_id, perm.as<uint32_t>(), sid.as<uint32_t>(), n);
  GEEK_CHECK_LAUNCH();
  GEEK_TRY(flag.alloc(n * 4, s));
  GEEK_TRY(ridx.alloc(n * 4, s));
  run_flags2<<<grid_for(n, 256), 256, 0, s>>>(sbin.as<uint32_t>(), sid.as<uint32_t>(), flag.as<uint32_t>(), n);
  GEEK_CHECK_LAUNCH();
  uint64_t nruns = 0;
  GEEK_TRY(exclusive_scan_u32(flag.as<uint32_t>(), ridx.as<uint32_t>(), n, s, &nruns));
  GEEK_TRY(start.alloc((nruns + 1) * 4, s));
  scatter_run_start<<<grid_for(n, 256), 256, 0, s>>>(flag.as<uint32_t>(), ridx.as<uint32_t>(),
                                                     start.as<uint32_t>(), n, nruns);
  GEEK_CHECK_LAUNCH();
  GEEK_TRY(win.alloc(nruns * 4, s));
  GEEK_TRY(wpos.alloc(nruns * 4, s));
  winner_flags<<<grid_for(nruns, 256), 256, 0, s>>>(start.as<uint32_t>(), sbin.as<uint32_t>(), bin_size,
                                                    nruns, win.as<uint32_t>());
  GEEK_CHECK_LAUNCH();
  uint64_t nw = 0;
  GEEK_TRY(exclusive_scan_u32(win.as<uint32_t>(), wpos.as<uint32_t>(), nruns, s, &nw));
  if (nw == 0) return GEEK_OK;
  GEEK_TRY(wb.alloc(nw * 4, s));
  GEEK_TRY(wi.alloc(nw * 4, s));
  compact_winners<<<grid_for(nruns, 256), 256, 0, s>>>(start.as<uint32_t>(), sbin.as<uint32_t>(),
                                                       sid.as<uint32_t>(), win.as<uint32_t>(),
                                                       wpos.as<uint32_t>(), nruns, wb.as<uint32_t>(),
                                                       wi.as<uint32_t>());
  GEEK_CHECK_LAUNCH();
  // delta filter per bin (engine.py:281)
  GEEK_TRY(gflag.alloc(nw * 4, s));
  GEEK_TRY(gidx.alloc(nw * 4, s));
  run_flags2<<<grid_for(nw, 256), 256, 0, s>>>(wb.as<uint32_t>(), nullptr, gflag.as<uint32_t>(), nw);
  GEEK_CHECK_LAUNCH();
  uint64_t ng = 0;
  GEEK_TRY(exclusive_scan_u32(gflag.as<uint32_t>(), gidx.as<uint32_t>(), nw, s, &ng));
  GEEK_TRY(gstart.alloc((ng + 1) * 4, s));
  scatter_run_start<<<grid_for(nw, 256), 256, 0, s>>>(gflag.as<uint32_t>(), gidx.as<uint32_t>(),
                                                      gstart.as<uint32_t>(), nw, ng);
  GEEK_TRY(gkeep.alloc(ng * 4, s));
  bin_keep_flags<<<grid_for(ng, 256), 256, 0, s>>>(gstart.as<uint32_t>(), ng, delta, gkeep.as<uint32_t>());
  GEEK_TRY(ekeep.alloc(nw * 4, s));
  GEEK_TRY(epos.alloc(nw * 4, s));
  expand_keep_elems<<<grid_for(nw, 256), 256, 0, s>>>(gidx.as<uint32_t>(), gflag.as<uint32_t>(),
                                                      gkeep.as<uint32_t>(), nw, ekeep.as<uint32_t>());
  GEEK_CHECK_LAUNCH();
  uint64_t nk = 0;
  GEEK_TRY(exclusive_scan_u32(ekeep.as<uint32_t>(), epos.as<uint32_t>(), nw, s, &nk));
  compact_pairs<<<grid_for(nw, 256), 256, 0, s>>>(wb.as<uint32_t>(), wi.as<uint32_t>(), ekeep.as<uint32_t>(),
                                                  epos.as<uint32_t>(), nw, win_bin, win_id);
  GEEK_CHECK_LAUNCH();
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
  *nwin_host = nk;
  return GEEK_OK;
}

int geek_pick_representatives(const uint32_t* flat, const uint64_t* offsets, const uint32_t* perm,
                              const uint32_t* gid, uint64_t ngroups, uint8_t* keep, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (ngroups == 0) return GEEK_OK;
  GEEK_CHECK_CUDA(cudaMemsetAsync(keep, 0, ngroups, s));
  pick_reps_kernel<<<grid_for(ngroups, 128), 128, 0, s>>>(flat, offsets, perm, gid, ngroups, keep);
  GEEK_CHECK_LAUNCH();
  fix_keep<<<grid_for(ngroups, 256), 256, 0, s>>>(keep, ngroups);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

int geek_sort_groups(const uint32_t* flat, const uint64_t* offsets, uint64_t ngroups, uint32_t* order,
                     void* stream) {
  cudaStream_t s = as_stream(stream);
  if (ngroups == 0) return GEEK_OK;
  const uint64_t n = ngroups;
  // max length bounds the refinement rounds
  std::vector<uint64_t> off_host(n + 1);
  GEEK_CHECK_CUDA(cudaMemcpyAsync(off_host.data(), offsets, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
  uint64_t maxlen = 0;
  for (uint64_t g = 0; g < n; ++g) maxlen = std::max(maxlen, off_host[g + 1] - off_host[g]);
  Scratch cls, dig, perm, tmp_cls, tmp_dig, flag, neworder;
  GEEK_TRY(cls.alloc(n * 4, s));
  GEEK_TRY(dig.alloc(n * 4, s));
  GEEK_TRY(perm.alloc(n * 4, s));
  GEEK_TRY(tmp_cls.alloc(n * 4, s));
  GEEK_TRY(tmp_dig.alloc(n * 4, s));
  GEEK_TRY(flag.alloc(n * 4, s));
  GEEK_TRY(neworder.alloc(n * 4, s));
  iota_u32<<<grid_for(n, 256), 256, 0, s>>>(order, n);
  GEEK_CHECK_CUDA(cudaMemsetAsync(cls.ptr, 0, n * 4, s));
  for (uint64_t p = 0; p <= maxlen; ++p) {
    // order is sorted by (tuple prefix < p); refine by element p within classes
    tuple_digit<<<grid_for(n, 256), 256, 0, s>>>(flat, offsets, order, n, p, dig.as<uint32_t>());
    GEEK_CHECK_LAUNCH();
    const uint32_t* cols[2] = {cls.as<uint32_t>(), dig.as<uint32_t>()};
    GEEK_TRY(argsort_cols(cols, 2, nullptr, n, perm.as<uint32_t>(), s));
    gather_u32<<<grid_for(n, 256), 256, 0, s>>>(order, perm.as<uint32_t>(), neworder.as<uint32_t>(), n);
    gather_u32<<<grid_for(n, 256), 256, 0, s>>>(cls.as<uint32_t>(), perm.as<uint32_t>(), tmp_cls.as<uint32_t>(), n);
    gather_u32<<<grid_for(n, 256), 256, 0, s>>>(dig.as<uint32_t>(), perm.as<uint32_t>(), tmp_dig.as<uint32_t>(), n);
    GEEK_CHECK_LAUNCH();
    GEEK_CHECK_CUDA(cudaMemcpyAsync(order, neworder.ptr, n * 4, cudaMemcpyDeviceToDevice, s));
    tie_class<<<grid_for(n, 256), 256, 0, s>>>(tmp_cls.as<uint32_t>(), tmp_dig.as<uint32_t>(),
                                                flag.as<uint32_t>(), n);
    GEEK_CHECK_LAUNCH();
    uint64_t nb = 0;
    GEEK_TRY(exclusive_scan_u32(flag.as<uint32_t>(), cls.as<uint32_t>(), n, s, &nb));
    // inclusive count of run starts: equal within a tie run, increasing across
    add_flag<<<grid_for(n, 256), 256, 0, s>>>(cls.as<uint32_t>(), flag.as<uint32_t>(), n);
    GEEK_CHECK_LAUNCH();
    if (nb == n) break;  // every group in its own class
  }
  return GEEK_OK;
}

}  // extern "C"
