// K2: exact even rank split of n keys into t buckets per table, ties by id
// (transform.py:95-109; engine.py:216-225), without a full sort.
//
//   1. coarse histogram of the top `cb` key bits (sampled)        -> estimate
//   2. every coarse cell is cut into ~count/G fine bins by linear
//      interpolation on the next 32 key bits (monotone in the key)
//   3. exact fine-bin histogram + exclusive scan -> exact rank range per bin
//   4. bins whose rank range lies inside one bucket write that bucket's slot
//      directly; bins that straddle a bucket boundary (about G/(n/t) of the
//      ids) are staged and ranked exactly by (key, id) inside the bin.
//
// Every id gets the slot of its exact rank in the (key, id) order, so the
// result is bit-identical to np.lexsort((arange(n), values)) + even split.
#include "common.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>

namespace geek {

// ids per fine bin (G).  256 keeps the per-bin tables of a batch of 8 tables
// (~17 MB) L2-resident for the random lookups of fine_hist / codes; the
// straddling bins it stages (~G per boundary) are ranked in L1-broadcast loops.
constexpr uint32_t kFineTargetDefault = 256;
constexpr uint32_t kLocalRankMax = 2048; // larger straddling bins take the sort path

struct SplitGeom {
  uint64_t n, t;
  int m, j0, tb;  // key tables [j0, j0+tb) of keys[j][n]
  int c0;         // code column of key table j0 in codes[i*m + c]
  int cb;         // coarse bits
  uint32_t nc;    // coarse cells per table
  uint32_t fine_target;  // ids per fine bin
};

__device__ __forceinline__ uint32_t coarse_of(uint64_t key, int cb) {
  return static_cast<uint32_t>(key >> (64 - cb));
}
#define coarse_of_key coarse_of

// cinfo[cell] = (number of fine bins, first fine bin): one 8-byte lookup
__device__ __forceinline__ uint32_t fine_of(uint64_t key, int cb, const uint2* __restrict__ cinfo) {
  const uint2 ci = __ldg(cinfo + coarse_of_key(key, cb));
  const uint32_t frac = static_cast<uint32_t>((key << cb) >> 32);
  return ci.y + static_cast<uint32_t>(((uint64_t)frac * ci.x) >> 32);
}

__global__ void pack_cinfo_kernel(const uint32_t* nfine, const uint32_t* fbase, uint64_t total, uint2* cinfo) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < total;
       c += (uint64_t)gridDim.x * blockDim.x)
    cinfo[c] = make_uint2(nfine[c], fbase[c]);
}

__global__ void coarse_hist_kernel(const uint64_t* __restrict__ keys, SplitGeom g, uint64_t stride,
                                   uint32_t* hist) {
  const int jb = blockIdx.y;
  const uint64_t* kj = keys + (uint64_t)(g.j0 + jb) * g.n;
  uint32_t* h = hist + (uint64_t)jb * g.nc;
  const uint64_t ns = (g.n + stride - 1) / stride;
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < ns;
       s += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[coarse_of(kj[s * stride], g.cb)], 1u);
}

__global__ void fine_layout_kernel(const uint32_t* hist, uint64_t total, uint64_t stride, uint32_t target,
                                   uint32_t* nfine) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < total;
       c += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t est = (uint64_t)hist[c] * stride;
    uint64_t nf = (est + target - 1) / target;
    nfine[c] = static_cast<uint32_t>(nf < 1 ? 1 : (nf > (1u << 20) ? (1u << 20) : nf));
  }
}

// 4 ids per thread per round: the key -> cell -> counter chains of
// independent ids overlap instead of exposing three latencies each
__global__ void __launch_bounds__(256) fine_hist_kernel(const uint64_t* __restrict__ keys, SplitGeom g,
                                                        const uint2* __restrict__ cinfo, uint32_t* fcnt) {
  const int jb = blockIdx.y;
  const uint64_t* kj = keys + (uint64_t)(g.j0 + jb) * g.n;
  const uint2* ci = cinfo + (uint64_t)jb * g.nc;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i0 < g.n; i0 += 4 * stride) {
    uint64_t key[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) key[u] = i0 + u * stride < g.n ? __ldg(kj + i0 + u * stride) : 0ull;
    uint2 c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) c[u] = __ldg(ci + coarse_of(key[u], g.cb));
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * stride < g.n) {
        const uint32_t frac = static_cast<uint32_t>((key[u] << g.cb) >> 32);
        atomicAdd(&fcnt[c[u].y + static_cast<uint32_t>(((uint64_t)frac * c[u].x) >> 32)], 1u);
      }
  }
}

__device__ __forceinline__ int table_of_fine(const uint32_t* tb_first, int tb, uint32_t f) {
  int jb = 0;
  while (jb + 1 < tb && tb_first[jb + 1] <= f) ++jb;
  return jb;
}

// per fine bin: rank start within its table, straddle size (0 if inside one bucket)
// fcode[f] = the slot of every id of bin f, or GEEK_NONE when f straddles a boundary
__global__ void straddle_kernel(SplitGeom g, const uint32_t* fcnt, const uint32_t* fstart,
                                const uint32_t* tb_first, uint32_t nfbins, uint32_t* scnt, uint32_t* fcode,
                                unsigned long long* stats) {
  for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f < nfbins;
       f += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = fcnt[f];
    uint32_t s = 0, code = 0;
    if (c > 0) {
      const int jb = table_of_fine(tb_first, g.tb, (uint32_t)f);
      const uint64_t r0 = (uint64_t)fstart[f] - (uint64_t)jb * g.n;
      code = slot_of_rank(r0, g.n, g.t);
      if (c > 1 && code != slot_of_rank(r0 + c - 1, g.n, g.t)) {
        s = c;
        code = GEEK_NONE;
        atomicAdd(&stats[0], (unsigned long long)c);
        atomicMax(&stats[1], (unsigned long long)c);
        if (c > kLocalRankMax) atomicAdd(&stats[2], (unsigned long long)c);
      }
    }
    scnt[f] = s;
    fcode[f] = code;
  }
}

// Coarse cells whose non-empty fine bins all map to one slot are rewritten to
// (0, slot): codes_kernel then needs a single lookup for most ids.
// A cell's ids occupy the rank range of its fine bins, so the cell is
// uniform exactly when its first and last rank fall in the same slot: O(1).
__global__ void cell_shortcut_kernel(SplitGeom g, uint2* cinfo, const uint32_t* fcnt, const uint32_t* fstart,
                                     uint64_t ncell) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < ncell;
       c += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 ci = cinfo[c];
    const uint64_t base = (c / g.nc) * g.n;  // ranks of table jb start at jb * n in fstart
    const uint32_t fl = ci.y + ci.x - 1;
    const uint64_t r0 = (uint64_t)fstart[ci.y] - base;
    const uint64_t r1 = (uint64_t)fstart[fl] + fcnt[fl] - base;  // one past the last rank
    if (r1 > r0 && slot_of_rank(r0, g.n, g.t) == slot_of_rank(r1 - 1, g.n, g.t))
      cinfo[c] = make_uint2(0u, slot_of_rank(r0, g.n, g.t));
  }
}

// slot codes for ids in non-straddling bins; straddling ids are staged (their
// code word is written as GEEK_NONE here and fixed by resolve / big_rank).
// Tables go in groups of 8 with the three dependent loads (key, cell,
// fine-bin code) issued group-wide, and each id's 8 codes leave as one
// 32-byte row segment when the row layout allows it.
__global__ void __launch_bounds__(256, 4) codes_kernel(const uint64_t* __restrict__ keys, SplitGeom g,
                                                    const uint2* __restrict__ cinfo,
                                                    const uint32_t* __restrict__ fcode,
                                                    const uint32_t* __restrict__ sbase,
                                                    uint32_t* sfill, uint32_t* codes,
                                                    uint64_t* st_key, uint32_t* st_id,
                                                    uint32_t* st_bin) {
  const bool vec = (g.m % 4) == 0 && (g.c0 % 4) == 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < g.n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t* crow = codes + i * (uint64_t)g.m + g.c0;
    for (int jb0 = 0; jb0 < g.tb; jb0 += 8) {
      uint64_t key[8];
      uint2 ci[8];
      uint32_t f[8], code[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        key[u] = jb0 + u < g.tb ? __ldg(keys + (uint64_t)(g.j0 + jb0 + u) * g.n + i) : 0ull;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        ci[u] = jb0 + u < g.tb ? __ldg(cinfo + (uint64_t)(jb0 + u) * g.nc + coarse_of(key[u], g.cb))
                               : make_uint2(0u, 0u);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        f[u] = ci[u].y + static_cast<uint32_t>(((uint64_t)static_cast<uint32_t>((key[u] << g.cb) >> 32) * ci[u].x) >> 32);
        code[u] = ci[u].x == 0 ? ci[u].y : __ldg(fcode + f[u]);  // (0, slot): whole cell inside one bucket
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (jb0 + u < g.tb && code[u] == GEEK_NONE) {
          const uint32_t pos = sbase[f[u]] + atomicAdd(&sfill[f[u]], 1u);
          st_key[pos] = key[u];
          st_id[pos] = static_cast<uint32_t>(i);
          st_bin[pos] = f[u];
        }
      if (vec && jb0 + 8 <= g.tb) {
        uint4* dst = reinterpret_cast<uint4*>(crow + jb0);
        dst[0] = make_uint4(code[0], code[1], code[2], code[3]);
        dst[1] = make_uint4(code[4], code[5], code[6], code[7]);
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (jb0 + u < g.tb) crow[jb0 + u] = code[u];
      }
    }
  }
}

// ---- group-level codes ---------------------------------------------------------
// 64 consecutive fine bins of one table cover a contiguous rank range; when it
// lies inside one bucket (most groups: a bucket holds ~n/t ids, a group
// ~64 G) the group's slot is enough for all its ids.  mcode[q] = that slot as
// 16 bits (0xFFFF: the group straddles a boundary, crosses a table, or t >
// 65535), and codes_group_kernel reads it from an SMEM copy of the 8 tables'
// groups: the per-id fine-bin code is fetched from L2 only in straddling groups.
constexpr uint16_t kGroupNone = 0xFFFFu;

__global__ void group_code_kernel(SplitGeom g, const uint32_t* fcnt, const uint32_t* fstart,
                                  const uint32_t* tb_first, uint32_t nfbins, uint16_t* mcode, int kGroupShift) {
  const uint32_t ng = (nfbins + (1u << kGroupShift) - 1) >> kGroupShift;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < ng; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t f0 = (uint32_t)q << kGroupShift;
    const uint32_t f1 = min(nfbins, f0 + (1u << kGroupShift)) - 1;  // last bin of the group
    const int j0 = table_of_fine(tb_first, g.tb, f0), j1 = table_of_fine(tb_first, g.tb, f1);
    uint16_t code = kGroupNone;
    if (j0 == j1 && g.t < 0xFFFFull) {
      const uint64_t r0 = (uint64_t)fstart[f0] - (uint64_t)j0 * g.n;
      const uint64_t r1 = (uint64_t)fstart[f1] + fcnt[f1] - (uint64_t)j0 * g.n;  // one past the last rank
      if (r1 == r0) code = 0;  // an empty group: never looked up
      else if (slot_of_rank(r0, g.n, g.t) == slot_of_rank(r1 - 1, g.n, g.t)) code = (uint16_t)slot_of_rank(r0, g.n, g.t);
    }
    mcode[q] = code;
  }
}

// codes_kernel with the table groups outside the id loop: per chunk of ids
// and group of 8 tables the groups' codes [q_lo, q_lo + nq) sit in SMEM
template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) codes_group_kernel(const uint64_t* __restrict__ keys, SplitGeom g,
                                                            const uint2* __restrict__ cinfo,
                                                            const uint32_t* __restrict__ fcode,
                                                            const uint16_t* __restrict__ mcode,
                                                            const uint32_t* __restrict__ tb_first, uint32_t nfbins,
                                                            const uint32_t* __restrict__ sbase, uint32_t* sfill,
                                                            uint32_t* codes, uint64_t* st_key, uint32_t* st_id,
                                                            uint32_t* st_bin, uint64_t chunk, int kGroupShift) {
  extern __shared__ uint16_t smc[];
  const int tid = threadIdx.x;
  const bool vec = (g.m % 4) == 0 && (g.c0 % 4) == 0;
  for (uint64_t c0 = (uint64_t)blockIdx.x * chunk; c0 < g.n; c0 += (uint64_t)gridDim.x * chunk) {
    const uint64_t c1 = min(g.n, c0 + chunk);
    for (int jb0 = 0; jb0 < g.tb; jb0 += 8) {
      const int nt = min(8, g.tb - jb0);
      const uint32_t flo = tb_first[jb0];
      const uint32_t fhi = jb0 + nt < g.tb ? tb_first[jb0 + nt] : nfbins;
      const uint32_t qlo = flo >> kGroupShift, qhi = (fhi + (1u << kGroupShift) - 1) >> kGroupShift;
      __syncthreads();  // the previous group's readers are done
      {  // 16-byte copies from the 8-aligned group below qlo (mcode is padded to whole uint4s)
        const uint32_t q8 = qlo & ~7u, n16 = (qhi - q8 + 7) >> 3;
        const uint4* srcv = reinterpret_cast<const uint4*>(mcode + q8);
        uint4* dstv = reinterpret_cast<uint4*>(smc);
        for (uint32_t v = tid; v < n16; v += blockDim.x) dstv[v] = __ldg(srcv + v);
      }
      __syncthreads();
      for (uint64_t i = c0 + tid; i < c1; i += blockDim.x) {
        uint64_t key[8];
        uint2 ci[8];
        uint32_t f[8], code[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) key[u] = u < nt ? __ldg(keys + (uint64_t)(g.j0 + jb0 + u) * g.n + i) : 0ull;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          ci[u] = u < nt ? __ldg(cinfo + (uint64_t)(jb0 + u) * g.nc + coarse_of(key[u], g.cb)) : make_uint2(0u, 0u);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          f[u] = ci[u].y + static_cast<uint32_t>(((uint64_t)static_cast<uint32_t>((key[u] << g.cb) >> 32) * ci[u].x) >> 32);
          if (ci[u].x == 0) {
            code[u] = ci[u].y;  // (0, slot): whole cell inside one bucket
          } else {
            const uint16_t mc = smc[(f[u] >> kGroupShift) - (qlo & ~7u)];
            code[u] = mc != kGroupNone ? (uint32_t)mc : __ldg(fcode + f[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (u < nt && code[u] == GEEK_NONE) {
            const uint32_t pos = sbase[f[u]] + atomicAdd(&sfill[f[u]], 1u);
            st_key[pos] = key[u];
            st_id[pos] = static_cast<uint32_t>(i);
            st_bin[pos] = f[u];
          }
        uint32_t* crow = codes + i * (uint64_t)g.m + g.c0 + jb0;
        if (vec && nt == 8) {
          uint4* dst = reinterpret_cast<uint4*>(crow);
          dst[0] = make_uint4(code[0], code[1], code[2], code[3]);
          dst[1] = make_uint4(code[4], code[5], code[6], code[7]);
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (u < nt) crow[u] = code[u];
        }
      }
    }
  }
}

// ---- group-level counting ------------------------------------------------------
// Exact ranks are needed bin by bin only inside groups that straddle a bucket
// boundary.  The group counts come from SMEM counters (one table per block,
// flushed once per block), the fine-bin counts from L2 atomics only for keys
// in straddling groups, and every other group's count is lumped into its
// first fine bin -- the fine-bin scan then still yields every straddling
// bin's exact rank start and every group's exact rank range.
__global__ void __launch_bounds__(256) group_hist_kernel(const uint64_t* __restrict__ keys, SplitGeom g,
                                                         const uint2* __restrict__ cinfo,
                                                         const uint32_t* __restrict__ tb_first, uint32_t nfbins,
                                                         int gs, uint32_t* gcnt) {
  extern __shared__ uint32_t sg[];
  const int jb = blockIdx.y, tid = threadIdx.x;
  const uint32_t qlo = tb_first[jb] >> gs;
  const uint32_t fend = jb + 1 < g.tb ? tb_first[jb + 1] : nfbins;
  const uint32_t nq = ((fend + (1u << gs) - 1) >> gs) - qlo;
  for (uint32_t q = tid; q < nq; q += 256) sg[q] = 0u;
  __syncthreads();
  const uint64_t* kj = keys + (uint64_t)(g.j0 + jb) * g.n;
  const uint2* ci = cinfo + (uint64_t)jb * g.nc;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + tid; i0 < g.n; i0 += 4 * stride) {
    uint64_t key[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) key[u] = i0 + u * stride < g.n ? __ldg(kj + i0 + u * stride) : 0ull;
    uint2 c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) c[u] = __ldg(ci + coarse_of(key[u], g.cb));
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * stride < g.n) {
        const uint32_t frac = static_cast<uint32_t>((key[u] << g.cb) >> 32);
        const uint32_t f = c[u].y + static_cast<uint32_t>(((uint64_t)frac * c[u].x) >> 32);
        atomicAdd(&sg[(f >> gs) - qlo], 1u);
      }
  }
  __syncthreads();
  for (uint32_t q = tid; q < nq; q += 256) {
    const uint32_t v = sg[q];
    if (v) atomicAdd(&gcnt[qlo + q], v);
  }
}

// gstr[q] = 1 when group q's rank range crosses a bucket boundary or a table
__global__ void group_flag_kernel(SplitGeom g, const uint32_t* gcnt, const uint32_t* gstart,
                                  const uint32_t* tb_first, uint32_t nfbins, int gs, uint32_t ngrp, uint8_t* gstr) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < ngrp; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t f0 = (uint32_t)q << gs, f1 = min(nfbins, f0 + (1u << gs)) - 1;
    const int j0 = table_of_fine(tb_first, g.tb, f0), j1 = table_of_fine(tb_first, g.tb, f1);
    uint8_t st = 1;
    if (j0 == j1) {
      const uint32_t c = gcnt[q];
      const uint64_t r0 = (uint64_t)gstart[q] - (uint64_t)j0 * g.n;
      st = (c > 1 && slot_of_rank(r0, g.n, g.t) != slot_of_rank(r0 + c - 1, g.n, g.t)) ? 1 : 0;
    }
    gstr[q] = st;
  }
}

// fine_hist_kernel for the keys of straddling groups only
__global__ void __launch_bounds__(256) fine_hist_sel_kernel(const uint64_t* __restrict__ keys, SplitGeom g,
                                                            const uint2* __restrict__ cinfo,
                                                            const uint8_t* __restrict__ gstr, int gs,
                                                            uint32_t* fcnt) {
  const int jb = blockIdx.y;
  const uint64_t* kj = keys + (uint64_t)(g.j0 + jb) * g.n;
  const uint2* ci = cinfo + (uint64_t)jb * g.nc;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i0 < g.n; i0 += 4 * stride) {
    uint64_t key[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) key[u] = i0 + u * stride < g.n ? __ldg(kj + i0 + u * stride) : 0ull;
    uint2 c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) c[u] = __ldg(ci + coarse_of(key[u], g.cb));
    uint32_t f[4];
    uint8_t sel[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t frac = static_cast<uint32_t>((key[u] << g.cb) >> 32);
      f[u] = c[u].y + static_cast<uint32_t>(((uint64_t)frac * c[u].x) >> 32);
      sel[u] = i0 + u * stride < g.n ? __ldg(gstr + (f[u] >> gs)) : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (sel[u]) atomicAdd(&fcnt[f[u]], 1u);
  }
}

// every fine bin of a lumped counting group (its ids all in one bucket) takes
// the group's slot: the empty-looking bins behind the lump are looked up by
// ids of a straddling code group that contains the counting group
__global__ void group_fill_kernel(SplitGeom g, const uint32_t* gstart, const uint32_t* gcnt, const uint8_t* gstr,
                                  const uint32_t* tb_first, uint32_t nfbins, int cs, uint32_t* fcode) {
  for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f < nfbins; f += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t q = (uint32_t)f >> cs;
    if (gstr[q] || gcnt[q] == 0) continue;
    const int jb = table_of_fine(tb_first, g.tb, (uint32_t)f);
    fcode[f] = slot_of_rank((uint64_t)gstart[q] - (uint64_t)jb * g.n, g.n, g.t);
  }
}

__global__ void group_lump_kernel(const uint32_t* gcnt, const uint8_t* gstr, uint32_t ngrp, int gs, uint32_t* fcnt) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < ngrp; q += (uint64_t)gridDim.x * blockDim.x)
    if (!gstr[q]) fcnt[(uint32_t)q << gs] = gcnt[q];
}

// exact rank inside a small straddling bin by counting smaller (key, id)
__global__ void __launch_bounds__(256) resolve_kernel(SplitGeom g, const uint64_t* __restrict__ st_key,
                                                      const uint32_t* __restrict__ st_id,
                                                      const uint32_t* __restrict__ st_bin,
                                                      uint64_t nstage,
                                                      const uint32_t* __restrict__ fstart,
                                                      const uint32_t* __restrict__ scnt,
                                                      const uint32_t* __restrict__ sbase,
                                                      const uint32_t* __restrict__ tb_first,
                                                      uint32_t* codes) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nstage;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t f = st_bin[e];
    const uint32_t c = scnt[f];
    if (c > kLocalRankMax) continue;
    const uint64_t key = st_key[e];
    const uint32_t id = st_id[e];
    const uint32_t b0 = sbase[f];
    uint32_t below = 0;
    for (uint32_t q = 0; q < c; ++q) {
      const uint64_t k2 = st_key[b0 + q];
      const uint32_t i2 = st_id[b0 + q];
      below += (k2 < key) || (k2 == key && i2 < id);
    }
    const int jb = table_of_fine(tb_first, g.tb, f);
    const uint64_t rank = (uint64_t)fstart[f] - (uint64_t)jb * g.n + below;
    codes[(uint64_t)id * g.m + g.c0 + jb] = slot_of_rank(rank, g.n, g.t);
  }
}

// ---- fallback for large straddling bins: full (bin, key, id) sort --------

__global__ void big_gather_kernel(const uint64_t* st_key, const uint32_t* st_id, const uint32_t* st_bin,
                                  uint64_t nstage, const uint32_t* scnt, uint32_t* rows,
                                  uint32_t* cursor) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nstage;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t f = st_bin[e];
    if (scnt[f] <= kLocalRankMax) continue;
    const uint32_t p = atomicAdd(cursor, 1u);
    uint32_t* r = rows + 4ull * p;
    r[0] = f;
    r[1] = static_cast<uint32_t>(st_key[e] >> 32);
    r[2] = static_cast<uint32_t>(st_key[e]);
    r[3] = st_id[e];
  }
}

__global__ void big_rank_kernel(SplitGeom g, const uint32_t* rows, const uint32_t* perm, uint64_t nbig,
                                const uint32_t* fstart, const uint32_t* tb_first, uint32_t* codes) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nbig;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t f = rows[4ull * perm[q]];
    // first sorted position of bin f (bins are the major sort key)
    uint64_t lo = 0, hi = q;
    while (lo < hi) {
      uint64_t mid = (lo + hi) >> 1;
      if (rows[4ull * perm[mid]] < f) lo = mid + 1;
      else hi = mid;
    }
    const int jb = table_of_fine(tb_first, g.tb, f);
    const uint64_t rank = (uint64_t)fstart[f] - (uint64_t)jb * g.n + (q - lo);
    const uint32_t id = rows[4ull * perm[q] + 3];
    codes[(uint64_t)id * g.m + g.c0 + jb] = slot_of_rank(rank, g.n, g.t);
  }
}

// coarse-histogram sample stride: ~2^18 keys per table shape the fine bins
// (the fine counts are exact anyway)
static uint64_t sample_stride(uint64_t n) {
  const int sbits = getenv("GEEK_SAMPLE_BITS") ? atoi(getenv("GEEK_SAMPLE_BITS")) : 18;
  return n > (1ull << sbits) ? n >> sbits : 1;
}

static int coarse_bits(uint64_t n) {
  // 16 coarse bits (sign, exponent, 4 mantissa bits: 1/16-octave cells) keep
  // the per-cell tables of a 16-table batch at 8 MB: the random lookups of
  // fine_hist / codes stay in L2 next to the key stream
  const int cb = (int)std::ceil(std::log2((double)n / 16.0 + 1.0));
  int c = std::min(16, std::max(10, cb));
  if (const char* e = getenv("GEEK_COARSE_BITS")) c = std::min(24, std::max(8, atoi(e)));
  return c;
}

static uint32_t fine_target() {
  uint32_t f = kFineTargetDefault;
  if (const char* ft = getenv("GEEK_FINE_TARGET")) f = (uint32_t)std::max(1, atoi(ft));
  return f;
}

// hist_in / fcnt_in (may be null): this batch's coarse sample histogram
// [tb][nc] and exact fine-bin counts, computed elsewhere (the projection
// counts fine bins as it writes keys); *nfb_out = fine bins of the batch
static int rank_split_batch(const uint64_t* keys, SplitGeom g, uint32_t* codes, uint64_t* stats_acc,
                            const uint32_t* hist_in, const uint32_t* fcnt_in, uint64_t* nfb_out, cudaStream_t s) {
  const uint64_t ncell = (uint64_t)g.tb * g.nc;
  const uint64_t stride = sample_stride(g.n);
  Scratch hist, nfine, fbase;
  GEEK_TRY(hist.alloc(ncell * 4, s));
  GEEK_TRY(nfine.alloc(ncell * 4, s));
  GEEK_TRY(fbase.alloc(ncell * 4, s));
  if (hist_in) {
    GEEK_CHECK_CUDA(cudaMemcpyAsync(hist.ptr, hist_in, ncell * 4, cudaMemcpyDeviceToDevice, s));
  } else {
    GEEK_CHECK_CUDA(cudaMemsetAsync(hist.ptr, 0, ncell * 4, s));
    dim3 gs(grid_for((g.n + stride - 1) / stride, 256, 148 * 8), g.tb);
    coarse_hist_kernel<<<gs, 256, 0, s>>>(keys, g, stride, hist.as<uint32_t>());
    GEEK_CHECK_LAUNCH();
  }
  fine_layout_kernel<<<grid_for(ncell, 256), 256, 0, s>>>(hist.as<uint32_t>(), ncell, stride, g.fine_target,
                                                          nfine.as<uint32_t>());
  GEEK_CHECK_LAUNCH();
  uint64_t nfb = 0;
  GEEK_TRY(exclusive_scan_u32(nfine.as<uint32_t>(), fbase.as<uint32_t>(), ncell, s, &nfb));
  GEEK_REQUIRE(nfb < 0xFFFFFFF0ull, "too many fine bins");
  std::vector<uint32_t> tbf(g.tb);
  for (int jb = 0; jb < g.tb; ++jb)
    GEEK_CHECK_CUDA(cudaMemcpyAsync(&tbf[jb], fbase.as<uint32_t>() + (uint64_t)jb * g.nc, 4,
                                    cudaMemcpyDeviceToHost, s));
  Scratch fcnt, fstart, scnt, sbase, sfill, tbfirst, stats, cinfo, fcode;
  GEEK_TRY(cinfo.alloc(ncell * 8, s));
  GEEK_TRY(fcode.alloc(nfb * 4, s));
  pack_cinfo_kernel<<<grid_for(ncell, 256), 256, 0, s>>>(nfine.as<uint32_t>(), fbase.as<uint32_t>(), ncell,
                                                         cinfo.as<uint2>());
  GEEK_CHECK_LAUNCH();
  GEEK_TRY(fcnt.alloc(nfb * 4, s));
  GEEK_TRY(fstart.alloc(nfb * 4, s));
  GEEK_TRY(scnt.alloc(nfb * 4, s));
  GEEK_TRY(sbase.alloc(nfb * 4, s));
  GEEK_TRY(sfill.alloc(nfb * 4, s));
  GEEK_TRY(tbfirst.alloc(g.tb * 4, s));
  GEEK_TRY(stats.alloc(32, s));
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));  // tbf is host memory
  GEEK_CHECK_CUDA(cudaMemcpyAsync(tbfirst.ptr, tbf.data(), g.tb * 4, cudaMemcpyHostToDevice, s));
  GEEK_CHECK_CUDA(cudaMemsetAsync(sfill.ptr, 0, nfb * 4, s));
  GEEK_CHECK_CUDA(cudaMemsetAsync(stats.ptr, 0, 32, s));
  // groups of 2^gshift fine bins: the finest grouping whose 8-table SMEM copy
  // of group codes fits (2^7 at n = 1e8: codes 31 -> 22 ms; 2^8 23 ms);
  // GEEK_SPLIT_GROUPS=s forces 2^s, 0 the per-bin paths only
  const char* gsel = getenv("GEEK_SPLIT_GROUPS");
  auto group_smem = [&](int gs) {
    size_t b = 0;
    for (int jb0 = 0; jb0 < g.tb; jb0 += 8) {
      const uint64_t flo = tbf[jb0], fhi = jb0 + 8 < g.tb ? tbf[jb0 + 8] : nfb;
      b = std::max<size_t>(b, (size_t)((((fhi + (1u << gs) - 1) >> gs) - ((flo >> gs) & ~7ull) + 15) & ~7ull) * 2);
    }
    return b;
  };
  // SMEM budget of the code groups: 200 KB (one 1024-thread block per SM: 2^6
  // fine bins per group at n = 1e8, codes 20.4 ms) or, GEEK_SPLIT_BIG=0, 104 KB
  // (two 512-thread blocks: 2^7, 21.4 ms)
  const char* bsel = getenv("GEEK_SPLIT_BIG");
  const bool big = !(bsel && atoi(bsel) == 0);
  const size_t gcap = big ? 200 * 1024 : 104 * 1024;
  int gshift = gsel ? atoi(gsel) : 6;
  if (!gsel)
    while (gshift < 10 && group_smem(gshift) > gcap) ++gshift;
  const size_t gsmem = gshift > 0 ? group_smem(gshift) : 0;
  const bool grouped = gshift > 0 && gsmem <= gcap;
  // group-level counting (not with counts from the projection): SMEM group
  // counters, fine counts in straddling groups only (GEEK_SPLIT_GCOUNT=0: every key's fine count)
  const char* gcs = getenv("GEEK_SPLIT_GCOUNT");
  const bool gcount = grouped && !fcnt_in && !(gcs && atoi(gcs) == 0);
  // counting groups: 2^cshift fine bins (finer than the code groups: fewer keys in
  // straddling groups; the code groups' rank ranges stay exact because every
  // code-group boundary is a counting-group boundary; 2^5 at n = 1e8: group
  // counts 7.4 ms + straddling fine counts 5.6 ms, against 21 ms of per-key atomics)
  const char* ccs = getenv("GEEK_SPLIT_CSHIFT");
  const int cshift = std::min(gshift, ccs ? std::max(1, atoi(ccs)) : 5);
  const uint64_t ngrp = grouped ? (nfb + (1u << cshift) - 1) >> cshift : 0;
  Scratch gcnt, gstart, gstr;
  if (fcnt_in) {
    GEEK_CHECK_CUDA(cudaMemcpyAsync(fcnt.ptr, fcnt_in, nfb * 4, cudaMemcpyDeviceToDevice, s));
  } else if (gcount) {
    size_t hs = 0;  // SMEM of the largest table's groups
    for (int jb = 0; jb < g.tb; ++jb) {
      const uint64_t fe = jb + 1 < g.tb ? tbf[jb + 1] : nfb;
      hs = std::max<size_t>(hs, (size_t)(((fe + (1u << cshift) - 1) >> cshift) - (tbf[jb] >> cshift)) * 4);
    }
    GEEK_TRY(gcnt.alloc(ngrp * 4, s));
    GEEK_TRY(gstart.alloc(ngrp * 4, s));
    GEEK_TRY(gstr.alloc(ngrp, s));
    GEEK_CHECK_CUDA(cudaMemsetAsync(gcnt.ptr, 0, ngrp * 4, s));
    if (hs > 48 * 1024)
      GEEK_CHECK_CUDA(cudaFuncSetAttribute(group_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hs));
    dim3 gh(grid_for(g.n, 256, 148 * 4), g.tb);
    group_hist_kernel<<<gh, 256, hs, s>>>(keys, g, cinfo.as<uint2>(), tbfirst.as<uint32_t>(), (uint32_t)nfb, cshift,
                                          gcnt.as<uint32_t>());
    GEEK_CHECK_LAUNCH();
    GEEK_TRY(exclusive_scan_u32(gcnt.as<uint32_t>(), gstart.as<uint32_t>(), ngrp, s));
    group_flag_kernel<<<grid_for(ngrp, 256), 256, 0, s>>>(g, gcnt.as<uint32_t>(), gstart.as<uint32_t>(),
                                                           tbfirst.as<uint32_t>(), (uint32_t)nfb, cshift,
                                                           (uint32_t)ngrp, gstr.as<uint8_t>());
    GEEK_CHECK_LAUNCH();
    GEEK_CHECK_CUDA(cudaMemsetAsync(fcnt.ptr, 0, nfb * 4, s));
    dim3 gf(grid_for(g.n, 256, 148 * 8), g.tb);
    fine_hist_sel_kernel<<<gf, 256, 0, s>>>(keys, g, cinfo.as<uint2>(), gstr.as<uint8_t>(), cshift,
                                            fcnt.as<uint32_t>());
    GEEK_CHECK_LAUNCH();
    group_lump_kernel<<<grid_for(ngrp, 256), 256, 0, s>>>(gcnt.as<uint32_t>(), gstr.as<uint8_t>(), (uint32_t)ngrp,
                                                           cshift, fcnt.as<uint32_t>());
    GEEK_CHECK_LAUNCH();
  } else {
    GEEK_CHECK_CUDA(cudaMemsetAsync(fcnt.ptr, 0, nfb * 4, s));
    dim3 gf(grid_for(g.n, 256, 148 * 8), g.tb);
    fine_hist_kernel<<<gf, 256, 0, s>>>(keys, g, cinfo.as<uint2>(), fcnt.as<uint32_t>());
    GEEK_CHECK_LAUNCH();
  }
  GEEK_TRY(exclusive_scan_u32(fcnt.as<uint32_t>(), fstart.as<uint32_t>(), nfb, s));
  straddle_kernel<<<grid_for(nfb, 256), 256, 0, s>>>(g, fcnt.as<uint32_t>(), fstart.as<uint32_t>(),
                                                      tbfirst.as<uint32_t>(), (uint32_t)nfb,
                                                      scnt.as<uint32_t>(), fcode.as<uint32_t>(),
                                                      stats.as<unsigned long long>());
  GEEK_CHECK_LAUNCH();
  uint64_t nstage = 0;
  if (gcount && cshift < gshift) {
    group_fill_kernel<<<grid_for(nfb, 256), 256, 0, s>>>(g, gstart.as<uint32_t>(), gcnt.as<uint32_t>(), gstr.as<uint8_t>(),
                                                          tbfirst.as<uint32_t>(), (uint32_t)nfb, cshift,
                                                          fcode.as<uint32_t>());
    GEEK_CHECK_LAUNCH();
  }
  if (!gcount) {  // (lumped groups hide the rank starts of bins inside them: no whole-cell shortcut then)
    cell_shortcut_kernel<<<grid_for(ncell, 256), 256, 0, s>>>(g, cinfo.as<uint2>(), fcnt.as<uint32_t>(),
                                                               fstart.as<uint32_t>(), ncell);
    GEEK_CHECK_LAUNCH();
  }
  GEEK_TRY(exclusive_scan_u32(scnt.as<uint32_t>(), sbase.as<uint32_t>(), nfb, s, &nstage));
  unsigned long long st[4] = {0, 0, 0, 0};
  GEEK_CHECK_CUDA(cudaMemcpyAsync(st, stats.ptr, 24, cudaMemcpyDeviceToHost, s));
  Scratch skey, sid, sbin;
  GEEK_TRY(skey.alloc(nstage * 8, s));
  GEEK_TRY(sid.alloc(nstage * 4, s));
  GEEK_TRY(sbin.alloc(nstage * 4, s));
  if (getenv("GEEK_SPLIT_GROUPS_DBG")) fprintf(stderr, "[split] group shift %d: %zu bytes of SMEM\n", gshift, gsmem);
  if (grouped) {  // group-level codes: the 8-table SMEM copy of the group codes (<= 104 KB: two blocks per SM)
    Scratch mcode;
    const uint64_t ncg = (nfb + (1u << gshift) - 1) >> gshift;
    GEEK_TRY(mcode.alloc((ncg + 16) * 2, s));  // + slack: the SMEM copies read whole uint4s
    group_code_kernel<<<grid_for(ncg, 256), 256, 0, s>>>(g, fcnt.as<uint32_t>(), fstart.as<uint32_t>(),
                                                          tbfirst.as<uint32_t>(), (uint32_t)nfb, mcode.as<uint16_t>(),
                                                          gshift);
    GEEK_CHECK_LAUNCH();
    const uint64_t chunk = 65536;
    const unsigned nchunk = (unsigned)((g.n + chunk - 1) / chunk);
#define GEEK_CODES_GROUP(NT, MINB)                                                                                 \
  GEEK_CHECK_CUDA(cudaFuncSetAttribute(codes_group_kernel<NT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                       (int)gsmem));                                                                \
  codes_group_kernel<NT, MINB><<<std::min(nchunk, 148u * MINB), NT, gsmem, s>>>(                                   \
      keys, g, cinfo.as<uint2>(), fcode.as<uint32_t>(), mcode.as<uint16_t>(), tbfirst.as<uint32_t>(), (uint32_t)nfb, \
      sbase.as<uint32_t>(), sfill.as<uint32_t>(), codes, skey.as<uint64_t>(), sid.as<uint32_t>(), sbin.as<uint32_t>(), \
      chunk, gshift)
    if (gsmem > 104 * 1024) {
      GEEK_CODES_GROUP(1024, 1);
    } else {
      GEEK_CODES_GROUP(512, 2);
    }
#undef GEEK_CODES_GROUP
  } else {
    codes_kernel<<<grid_for(g.n, 256, 148 * 16), 256, 0, s>>>(
        keys, g, cinfo.as<uint2>(), fcode.as<uint32_t>(), sbase.as<uint32_t>(), sfill.as<uint32_t>(), codes,
        skey.as<uint64_t>(), sid.as<uint32_t>(), sbin.as<uint32_t>());
  }
  GEEK_CHECK_LAUNCH();
  if (nstage) {
    resolve_kernel<<<grid_for(nstage, 256, 148 * 16), 256, 0, s>>>(
        g, skey.as<uint64_t>(), sid.as<uint32_t>(), sbin.as<uint32_t>(), nstage, fstart.as<uint32_t>(),
        scnt.as<uint32_t>(), sbase.as<uint32_t>(), tbfirst.as<uint32_t>(), codes);
    GEEK_CHECK_LAUNCH();
  }
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
  const uint64_t nbig = st[2];
  if (nbig) {
    Scratch rows, perm, cur;
    GEEK_TRY(rows.alloc(nbig * 16, s));
    GEEK_TRY(perm.alloc(nbig * 4, s));
    GEEK_TRY(cur.alloc(4, s));
    GEEK_CHECK_CUDA(cudaMemsetAsync(cur.ptr, 0, 4, s));
    big_gather_kernel<<<grid_for(nstage, 256), 256, 0, s>>>(skey.as<uint64_t>(), sid.as<uint32_t>(),
                                                            sbin.as<uint32_t>(), nstage,
                                                            scnt.as<uint32_t>(), rows.as<uint32_t>(),
                                                            cur.as<uint32_t>());
    GEEK_CHECK_LAUNCH();
    GEEK_TRY(lex_argsort_rows(rows.as<uint32_t>(), nbig, 4, nullptr, perm.as<uint32_t>(), s));
    big_rank_kernel<<<grid_for(nbig, 256), 256, 0, s>>>(g, rows.as<uint32_t>(), perm.as<uint32_t>(),
                                                        nbig, fstart.as<uint32_t>(),
                                                        tbfirst.as<uint32_t>(), codes);
    GEEK_CHECK_LAUNCH();
    GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
  }
  if (nfb_out) *nfb_out = nfb;
  stats_acc[0] += nfb;
  stats_acc[1] += nstage;
  stats_acc[2] = std::max<uint64_t>(stats_acc[2], st[1]);
  stats_acc[3] += nbig;
  return GEEK_OK;
}

int rank_split_v2(const uint64_t* keys, uint64_t n, int m, uint64_t t, uint32_t* codes, uint64_t code_stride,
                  uint64_t col, uint64_t* stats_host, cudaStream_t s);  // ranksplit2.cu

static int rank_split_impl(const uint64_t* keys, uint64_t n, int m, uint64_t t, uint32_t* codes,
                           uint64_t code_stride, uint64_t col, uint64_t* stats_host, cudaStream_t s,
                           const uint32_t* hist_in = nullptr, const uint32_t* fcnt_in = nullptr) {
  GEEK_REQUIRE(t >= 1 && t <= n, "cannot split %llu objects into %llu buckets",
               (unsigned long long)n, (unsigned long long)t);
  GEEK_REQUIRE(n < 0xFFFFFFFFull, "n must be < 2^32");
  if (!hist_in && !fcnt_in && getenv("GEEK_SPLIT_V2")) {
    // experimental shared-memory split (ranksplit2.cu): exact, but on the
    // benchmark data its coarser bins stage 3-8 % of the ids and its histogram
    // and codes passes run latency-bound at one or two blocks per SM -- 125-145
    // ms against this split's 56 ms (profiles/r2_split_v2.md), so it is opt-in
    const int st = rank_split_v2(keys, n, m, t, codes, code_stride, col, stats_host, s);
    if (st != 1) return st;
  }
  SplitGeom g;
  g.n = n;
  g.t = t;
  g.m = static_cast<int>(code_stride);
  g.cb = coarse_bits(n);
  g.nc = 1u << g.cb;
  g.fine_target = fine_target();
  const double per_table = 4.0 * ((double)n / g.fine_target + 2.0 * g.nc) * 5.0;
  // batches of whole tables: codes rows are then written in tb-word runs
  // (8 tables = one 32-byte sector), counters stay u32 (tb * n < 2^32)
  int tb = (int)std::max(1.0, std::min((double)m, (1024.0 * (1 << 20)) / per_table));
  tb = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)tb, 0xFFFFFFF0ull / n));
  // at most 16 tables per batch: the cell and fine-bin tables of a batch
  // (~30 MB at n = 1e8) stay L2-resident for the random lookups
  const int tb_cap = getenv("GEEK_SPLIT_TB") ? std::max(1, atoi(getenv("GEEK_SPLIT_TB"))) : 16;
  tb = std::min(tb, tb_cap);
  if (tb >= 8 && tb < m) tb -= tb % 8;
  uint64_t acc[4] = {0, 0, 0, 0};
  uint64_t foff = 0;  // fine counts of the batches so far (precounted path)
  for (int j0 = 0; j0 < m; j0 += tb) {
    g.j0 = j0;
    g.c0 = static_cast<int>(col) + j0;
    g.tb = std::min(tb, m - j0);
    uint64_t nfb = 0;
    GEEK_TRY(rank_split_batch(keys, g, codes, acc, hist_in ? hist_in + (uint64_t)j0 * g.nc : nullptr,
                              fcnt_in ? fcnt_in + foff : nullptr, &nfb, s));
    foff += nfb;
  }
  if (stats_host)
    for (int i = 0; i < 4; ++i) stats_host[i] = acc[i];
  return GEEK_OK;
}

// hist[t][cell] += counts of the sample keys [m][ns] (every key counted)
__global__ void sample_hist_kernel(const uint64_t* __restrict__ keys, uint64_t ns, int cb, uint32_t nc,
                                   uint32_t* hist) {
  const int t = blockIdx.y;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ns; i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&hist[(uint64_t)t * nc + coarse_of(keys[(uint64_t)t * ns + i], cb)], 1u);
}

__global__ void table_offsets_kernel(const uint32_t* fbase, int m, uint32_t nc, uint64_t nfb, uint32_t* toff) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < m) toff[t] = fbase[(uint64_t)t * nc];
  if (t == m) toff[m] = (uint32_t)nfb;
}

}  // namespace geek

using namespace geek;

extern "C" {

int geek_rank_split(const uint64_t* keys, uint64_t n, int m, uint64_t t, uint32_t* codes,
                    uint64_t* stats_host, void* stream) {
  GEEK_REQUIRE(m >= 1, "need at least one table");
  return rank_split_impl(keys, n, m, t, codes, (uint64_t)m, 0, stats_host, as_stream(stream));
}

int geek_rank_split_strided(const uint64_t* keys, uint64_t n, uint64_t t, uint32_t* codes,
                            uint64_t stride, uint64_t col, void* stream) {
  GEEK_REQUIRE(col < stride, "column outside stride");
  return rank_split_impl(keys, n, 1, t, codes, stride, col, nullptr, as_stream(stream));
}


int geek_split_plan(uint64_t n, int* cb_out, uint64_t* stride_out) {
  GEEK_REQUIRE(n >= 1, "empty split");
  if (cb_out) *cb_out = coarse_bits(n);
  if (stride_out) *stride_out = sample_stride(n);
  return GEEK_OK;
}

int geek_coarse_hist(const uint64_t* keys, uint64_t ns, int m, int cb, uint32_t* hist, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(m >= 1 && cb >= 1 && cb <= 24, "bad coarse histogram shape");
  if (ns == 0) return GEEK_OK;
  dim3 gs(grid_for(ns, 256, 148 * 8), m);
  sample_hist_kernel<<<gs, 256, 0, s>>>(keys, ns, cb, 1u << cb, hist);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

int geek_fine_layout(const uint32_t* hist, int m, uint64_t n, uint32_t* cinfo, uint32_t* toff, uint64_t* nfb_host,
                     void* stream) {
  cudaStream_t s = as_stream(stream);
  const int cb = coarse_bits(n);
  const uint64_t nc = 1ull << cb, ncell = (uint64_t)m * nc;
  Scratch nfine, fbase;
  GEEK_TRY(nfine.alloc(ncell * 4, s));
  GEEK_TRY(fbase.alloc(ncell * 4, s));
  fine_layout_kernel<<<grid_for(ncell, 256), 256, 0, s>>>(hist, ncell, sample_stride(n), fine_target(),
                                                          nfine.as<uint32_t>());
  GEEK_CHECK_LAUNCH();
  uint64_t nfb = 0;
  GEEK_TRY(exclusive_scan_u32(nfine.as<uint32_t>(), fbase.as<uint32_t>(), ncell, s, &nfb));
  GEEK_REQUIRE(nfb < 0x7FFFFFF0ull, "too many fine bins");
  pack_cinfo_kernel<<<grid_for(ncell, 256), 256, 0, s>>>(nfine.as<uint32_t>(), fbase.as<uint32_t>(), ncell,
                                                         reinterpret_cast<uint2*>(cinfo));
  GEEK_CHECK_LAUNCH();
  table_offsets_kernel<<<1, m + 1 > 1024 ? 1024 : m + 1, 0, s>>>(fbase.as<uint32_t>(), m, (uint32_t)nc, nfb, toff);
  GEEK_CHECK_LAUNCH();
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
  if (nfb_host) *nfb_host = nfb;
  return GEEK_OK;
}

int geek_rank_split_counted(const uint64_t* keys, uint64_t n, int m, uint64_t t, const uint32_t* hist,
                            const uint32_t* fcnt, uint32_t* codes, uint64_t* stats_host, void* stream) {
  GEEK_REQUIRE(m >= 1 && m <= 1023, "need 1..1023 tables");
  GEEK_REQUIRE(hist && fcnt, "precounted split needs the sample histogram and the fine counts");
  return rank_split_impl(keys, n, m, t, codes, (uint64_t)m, 0, stats_host, as_stream(stream), hist, fcnt);
}

}  // extern "C"
