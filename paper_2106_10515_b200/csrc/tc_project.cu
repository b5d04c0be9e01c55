// K1 on the 5th-gen tensor cores: the random projections of transform.py:125 /
// engine.py:180 (X @ a for every table's direction a) as exact integer
// products on kind::i8 tcgen05 MMAs, within the float64 order bound of the
// reference's OpenBLAS keys.
//
// Digits.  Row r of X (float32) with max|x| < 2^e_r is the 40-bit two's
// complement integer F = floor(x 2^(39-e_r)) plus a remainder 0 <= rho <
// 2^(e_r-39); F's bytes are the x digits X_0 (signed top byte) and X_1..X_4
// (unsigned), so x = 2^(e_r-7) sum_s X_s 2^(-8s) + rho.  Table j's direction
// (float64, max|a| < 2^e_j) is trunc(a 2^(62-e_j)) written in 8 balanced
// signed base-256 digits A_0..A_7: a = 2^(e_j-6) sum_t A_t 2^(-8t) + alpha,
// |alpha| < 2^(e_j-62).  Then
//   x.a = 2^(e_r+e_j-13) sum_l 2^(-8l) D_l + sum_k rho_k a_k + err,
//   D_l = sum_{s+t=l} sum_k X_{s,k} A_{t,k}   (exact int32: |D_l| < 2^25)
// keeping the levels l <= 7.  err (the alpha terms and the dropped levels)
// is below 2^-6 of gamma_d 2^e_r |a|_1, the float64 order bound that
// transform.projection_tolerance doubles for the boundary accounting; the
// two roundings of the float64 combination add at most 2 ulps.  So every key
// is as close to the exact dot product as any float64 summation order (the
// reference's dgemv or the DMMA chains of project.cu), and the ids whose key
// could order differently are the ones split_boundary_stats counts.
//
// MMA shape.  The D columns are (level l, table j) = l*mp + j (mp = m rounded
// up to 8): 8 mp int32 columns in two blocks of 4 mp (levels 0-3, 4-7).  The
// A operand is x digit s of the 128-row tile (K = d, 32 bytes per MMA), the B
// operand the direction digits t = l - s for every column -- one image P of
// the digits, rows (t + 3) mp + j, read from row (block start - s mp + 3 mp):
// a shift of s levels is a shift of the B descriptor's start address, so the
// 20 MMAs per 32-dim K step (block 0: s <= 3, block 1: s <= 4) need one 55 KB
// image.  The remainders rho (only elements 2^15 below their row's maximum)
// go through float64 FMAs in the epilogue, from a per-row bit mask.
//
// Warps: 0-7 epilogue (lane group w % 4, column groups of 8 tables w / 4, 2
// + w/4, ...), 8-15 loaders (float32 rows -> digits in SMEM, two 8-row
// groups per warp and tile, the next group's loads in flight), 16 MMA.  The
// digit tile is double-buffered; the accumulator (8 mp <= 320 columns) is
// single-buffered, so a tile's MMAs wait for the previous tile's epilogue.
#include "common.cuh"
#include "project.cuh"
#include "tcgen05.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace geek {

constexpr int kPjM = 128;          // rows per tile = TMEM lanes
constexpr int kPjXd = 5;           // x digits (bytes of the 40-bit F)
constexpr int kPjAd = 8;           // direction digits
constexpr int kPjLv = 8;           // levels kept
constexpr int kPjEpiWarps = 8;
constexpr int kPjLoadWarps = 7;
constexpr int kPjLoadBase = 8;
constexpr int kPjMmaWarp = 15;
constexpr int kPjThreads = 16 * 32;  // 4 warps per SM sub-partition: 128 registers
constexpr int kPjStep = kPjM * 32;  // one 32-byte K step of 128 rows: 4 KB
constexpr int kPjSlots = 4;         // row-metadata ring (tiles in flight between loader and epilogue)
constexpr int kPjSpecialE = 0x7FFF;
constexpr int kPjMaxSmem = 232448;

struct PjParams {
  const float* X;
  uint64_t n;
  int d, kp, m, mp;
  const double* A;       // [m][d]
  const uint8_t* Pimg;   // [kp/32][11 mp / 8][2][8][16]: the B image
  const int* ej;         // [m]: e_j, or kPjSpecialE (table keys by float64 FMAs)
  KeyDst dst;
  int* exprange;
  unsigned* nonfinite;
  unsigned long long* tl;  // -DGEEK_DEBUG_KNOBS timeline of CTA 0 (tools/build_debug.py), else null
  int prof;                // -DGEEK_DEBUG_KNOBS: 1 = no key stores, 2 = no remainder terms, 3 = no keys at all
};

// issued by one elected lane of a converged warp (the descriptors are warp-uniform)
__device__ __forceinline__ void pj_mma(uint32_t dt, uint32_t alo, uint32_t blo, uint32_t dhi, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      ".reg .b64 ad, bd;\n"
      "mov.b64 ad, {%1, %3};\n"
      "mov.b64 bd, {%2, %3};\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %5, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], ad, bd, %4, p;\n"
      "}\n" ::"r"(dt),
      "r"(alo), "r"(blo), "r"(dhi), "r"(idesc), "r"(acc));
}

// kind::i8: D = s32 (2 at [4,6)), A = u8 (0) / s8 (1) at [7,10), B = s8 at
// [10,13), both K-major, N>>3 at [17,23), M>>4 at [24,29)
__host__ __device__ constexpr uint32_t pj_idesc(int N, bool a_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(kPjM >> 4) << 24);
}

__device__ __forceinline__ void pj_ld8(uint32_t taddr, int32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}

// frexp exponent of the float32 magnitude bits b (> 0): 2^(e-1) <= |x| < 2^e
__device__ __forceinline__ int pj_fexp(uint32_t b) {
  const int E = (int)(b >> 23);
  return E ? E - 126 : (32 - __clz((int)b)) - 149;
}

__device__ __forceinline__ double pj_pow2(int e) {  // e in [-1022, 1023]
  return __longlong_as_double((long long)(1023 + e) << 52);
}

// The B image: direction digits in the K-major core-matrix layout, row w =
// (t + 3) mp + j of the shifted level axis (t outside 0..7 or j >= m: zero).
__global__ void pj_prep_kernel(const double* __restrict__ A, int m, int d, int mp, int kp, uint8_t* __restrict__ img,
                               int* __restrict__ ej) {
  __shared__ int se[48];
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    double mx = 0.0;
    bool fin = true;
    for (int k = 0; k < d; ++k) {
      const double v = A[(uint64_t)j * d + k];
      fin &= isfinite(v);
      mx = fmax(mx, fabs(v));
    }
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);
    se[j] = (!fin || e < -400 || e > 400) ? kPjSpecialE : e;
    ej[j] = se[j];
  }
  __syncthreads();
  const int rows = 11 * mp;
  const uint32_t pk = (uint32_t)rows * 32;
  for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < rows * kp; e += blockDim.x * gridDim.x) {
    const int w = e / kp, k = e - w * kp;
    const int t = w / mp - 3, j = w - (w / mp) * mp;
    int8_t dig = 0;
    if (t >= 0 && t < kPjAd && j < m && k < d && se[j] != kPjSpecialE) {
      long long a = (long long)(A[(uint64_t)j * d + k] * pj_pow2(62 - se[j]));  // trunc, |a| < 2^62
      int8_t digs[kPjAd];
      for (int q = kPjAd - 1; q > 0; --q) {  // balanced base-256, least significant first
        const long long r = ((a + 128) & 255) - 128;
        digs[q] = (int8_t)r;
        a = (a - r) >> 8;
      }
      digs[0] = (int8_t)a;  // |a| <= 65 here
      dig = digs[t];
    }
    img[(uint32_t)(k >> 5) * pk + core_off_b(w, k & 31, 128, 256)] = (uint8_t)dig;
  }
}

__device__ __forceinline__ void pj_count(const KeyDst& dst, int j, uint64_t kk) {  // fused fine-bin count
  const uint2 ci = __ldg(dst.cinfo + ((uint64_t)j << dst.cb) + (uint32_t)(kk >> (64 - dst.cb)));
  const uint32_t frac = static_cast<uint32_t>((kk << dst.cb) >> 32);
  atomicAdd(dst.fcnt + ci.y + static_cast<uint32_t>(((uint64_t)frac * ci.x) >> 32), 1u);
}

// Keys of special rows / tables (non-finite or out-of-range exponents, or
// more than two remainder elements): float64 FMAs in dimension order.
__device__ __noinline__ uint64_t pj_fma_key(const float* X, const double* A, int d, uint64_t row, int j) {
  const float* x = X + row * d;
  const double* a = A + (uint64_t)j * d;
  double key = 0.0;
  for (int k = 0; k < d; ++k) key = fma((double)__ldg(x + k), __ldg(a + k), key);
  return f64_key(key);
}

#define PJ_T(ti, k)                                                                       \
  do {                                                                                    \
    if (P.tl && blockIdx.x == 0 && (ti) < 64) P.tl[(ti) * 8 + (k)] = clock64();           \
  } while (0)

template <int NKS>  // 32-dim K steps (d <= 32 NKS): compile-time digit-tile offsets
__global__ void __launch_bounds__(kPjThreads, 1) tc_project_kernel(const PjParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int nks = NKS;
  const int mp = P.mp;
  const uint32_t abytes = (uint32_t)kPjXd * nks * kPjStep;
  const uint32_t pk = (uint32_t)11 * mp * 32;  // bytes of one K step of the B image
  const uint32_t nb = 4 * mp;                  // accumulator columns of one level block
  const int nslot = 3 * nb <= 512 ? 3 : 2;     // TMEM block slots (a ring: tile i, block b -> slot (2i + b) % nslot)
  uint8_t* Abuf = smem;                        // [2][kPjXd][nks][4 KB]
  uint8_t* Pb = smem + 2 * abytes;             // [nks][11 mp rows]
  double* tsc = reinterpret_cast<double*>(Pb + nks * pk);           // [48]: 2^(e_j - 69), 0 = special table
  int* tse = reinterpret_cast<int*>(tsc + kMaxKeyTables);            // [48]: (e_j - 69) 2^20 (exponent-field add)
  uint64_t** tpp = reinterpret_cast<uint64_t**>(tse + kMaxKeyTables);  // [48]: the key destinations
  uint16_t* meta = reinterpret_cast<uint16_t*>(tpp + kMaxKeyTables);  // [slots][128]: e_r + 128 | nrem << 8 | fma << 10
  uint2* rems = reinterpret_cast<uint2*>(meta + kPjSlots * kPjM);  // [slots][128][2]: (k, rho_k as f32)
  uint64_t* bars = reinterpret_cast<uint64_t*>(rems + kPjSlots * kPjM * 2);
  uint64_t* afull = bars;       // [2] loaders -> MMA
  uint64_t* aempty = bars + 2;  // [2] MMA -> loaders
  uint64_t* dfull = bars + 4;   // MMA -> epilogue (both blocks of a tile)
  uint64_t* sfree = bars + 5;   // [3] epilogue -> MMA: a TMEM block slot was read
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  {
    const uint4* s = reinterpret_cast<const uint4*>(P.Pimg);
    uint4* dd = reinterpret_cast<uint4*>(Pb);
    for (uint32_t i = threadIdx.x; i < nks * pk / 16; i += blockDim.x) dd[i] = s[i];
    for (int j = threadIdx.x; j < kMaxKeyTables; j += blockDim.x) {
      const int e = j < P.m ? P.ej[j] : kPjSpecialE;
      tsc[j] = e == kPjSpecialE ? 0.0 : pj_pow2(e - 69);  // 2^(e_j - 13) 2^-56
      tse[j] = e == kPjSpecialE ? 0 : (e - 69) * (1 << 20);  // the exponent-field add, high word
      tpp[j] = P.dst.tptr[j];
    }
  }
  fence_proxy_async();
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&afull[b], kPjM / 8 * 32);  // one arrival per loader lane and 8-row group
      mbar_init(&aempty[b], 1);
    }
    mbar_init(dfull, 1);
    for (int q = 0; q < 3; ++q) mbar_init(&sfree[q], kPjEpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  bool anyspec = false;  // a table whose keys take float64 FMAs (non-finite or extreme direction)
  for (int j = 0; j < P.m; ++j) anyspec |= tsc[j] == 0.0;
  const uint64_t ntiles = (P.n + kPjM - 1) / kPjM;
  const uint64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (warp >= kPjLoadBase && warp < kPjLoadBase + kPjLoadWarps) {
    // ---- loaders: 8-row groups (16 per tile, dealt round-robin over the
    // loader warps); lane (row r8 = lane / 4, quarter q = lane % 4) holds
    // dims 16c + 4q .. +3 of its row; the next group's rows are in flight
    const int lw = warp - kPjLoadBase, r8 = lane >> 2, q = lane & 3;
    constexpr int nc = 2 * NKS;  // 16-dim chunks
    uint32_t amax = 0u, amin = 0xFFFFFFFFu;
    const uint64_t items = my_tiles * (kPjM / 8);
    float4 cur[8], nxt[8];
    auto load = [&](uint64_t it, float4* v) {
      const uint64_t tile = blockIdx.x + (it >> 4) * gridDim.x;
      const uint64_t row = tile * kPjM + (it & 15) * 8 + r8;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int k = 16 * c + 4 * q;
        v[c] = (c < nc && row < P.n && k < P.d) ? __ldg(reinterpret_cast<const float4*>(P.X + row * P.d + k))
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    if ((uint64_t)lw < items) load(lw, nxt);
    for (uint64_t it = lw; it < items; it += kPjLoadWarps) {
#pragma unroll
      for (int c = 0; c < 8; ++c) cur[c] = nxt[c];
      if (it + kPjLoadWarps < items) load(it + kPjLoadWarps, nxt);
      const uint64_t ti = it >> 4;
      const int b = (int)(ti & 1);
      const int rl = (int)(it & 15) * 8 + r8;
      uint32_t rmax = 0u;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float* f = reinterpret_cast<const float*>(&cur[c]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t ab = __float_as_uint(f[e]) & 0x7FFFFFFFu;
          rmax = max(rmax, ab);
          amin = min(amin, ab - 1u);  // 0 wraps to the top: zeros never count
        }
      }
      amax = max(amax, rmax);
      rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, 1));
      rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, 2));
      const int er = rmax ? pj_fexp(rmax) : 0;
      const bool special = rmax >= 0x7F800000u || er < -80 || er > 39;
      const float scale = special ? 0.f : __uint_as_float((uint32_t)(166 - er) << 23);  // 2^(39 - e_r)
      const uint32_t rthr = special ? 0u : ((uint32_t)(er + 111) << 23) - 1u;  // bits of 2^(e_r - 16), minus 1
      const float rback = special ? 0.f : __uint_as_float((uint32_t)(88 + er) << 23);  // 2^(e_r - 39)
      if (ti >= 2) mbar_wait(&aempty[b], (uint32_t)((ti - 2) >> 1) & 1u);
      if (lw == 0 && lane == 0 && (it & 15) == 0) PJ_T(ti, 0);
      uint8_t* Ab = Abuf + b * abytes;
      // x = 2^(e_r-39) F + rho, F = trunc(x 2^(39-e_r)) (any integer's two's
      // complement bytes are its digits); rho != 0 only for |x| < 2^(e_r-16),
      // and rho (the tail of x's significand) is exact in float32
      uint32_t rb = 0u;  // elements with a remainder (bit 4c + e), branch-free in the digit loop
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < nc) {
          const float* f = reinterpret_cast<const float*>(&cur[c]);
          uint32_t lo[4], hi[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const long long F = __float2ll_rz(f[e] * scale);
            lo[e] = (uint32_t)F;
            hi[e] = (uint32_t)((unsigned long long)F >> 32);
            // candidates only (|x| < 2^(e_r-16)); the rare pass below keeps those with rho != 0
            rb |= ((__float_as_uint(f[e]) & 0x7FFFFFFFu) - 1u < rthr ? 1u : 0u) << (c * 4 + e);
          }
          const uint32_t t0 = __byte_perm(lo[0], lo[1], 0x5140), t1 = __byte_perm(lo[0], lo[1], 0x7362);
          const uint32_t u0 = __byte_perm(lo[2], lo[3], 0x5140), u1 = __byte_perm(lo[2], lo[3], 0x7362);
          const uint32_t w[kPjXd] = {
              __byte_perm(__byte_perm(hi[0], hi[1], 0x0040), __byte_perm(hi[2], hi[3], 0x0040), 0x5410),
              __byte_perm(t1, u1, 0x7632),   // byte 3 of F
              __byte_perm(t1, u1, 0x5410),   // byte 2
              __byte_perm(t0, u0, 0x7632),   // byte 1
              __byte_perm(t0, u0, 0x5410)};  // byte 0
          const uint32_t off = (uint32_t)(c >> 1) * kPjStep + core_off_b(rl, (c & 1) * 16 + 4 * q, 128, 256);
#pragma unroll
          for (int s = 0; s < kPjXd; ++s) *reinterpret_cast<uint32_t*>(Ab + (uint32_t)(s * nks) * kPjStep + off) = w[s];
        }
      }
      // the rare remainder entries (x re-read from L2): at most 2 per lane kept
      int nrl = 0;
      uint2 re0 = make_uint2(0u, 0u), re1 = make_uint2(0u, 0u);
      if (rb && !special) {
        const uint64_t row = (blockIdx.x + ti * gridDim.x) * kPjM + rl;
#pragma unroll 1
        while (rb) {
          const int bi = __ffs(rb) - 1;
          rb &= rb - 1u;
          const int k = 16 * (bi >> 2) + 4 * q + (bi & 3);
          const float y = __ldg(P.X + row * P.d + k) * scale;
          const float rho = (y - truncf(y)) * rback;  // exact: the tail of x's significand
          if (rho != 0.f) {
            const uint2 en = make_uint2((uint32_t)k, __float_as_uint(rho));
            if (nrl == 0) re0 = en;
            else if (nrl == 1) re1 = en;
            ++nrl;
          }
        }
      }
      // the row's entries: exclusive scan over its 4 lanes, at most 2 kept
      const int qbase = lane & ~3;
      const int c1 = __shfl_sync(0xffffffffu, nrl, qbase), c2 = __shfl_sync(0xffffffffu, nrl, qbase + 1),
                c3 = __shfl_sync(0xffffffffu, nrl, qbase + 2), c4 = __shfl_sync(0xffffffffu, nrl, qbase + 3);
      const int pre = (q > 0 ? c1 : 0) + (q > 1 ? c2 : 0) + (q > 2 ? c3 : 0);
      const int tot = c1 + c2 + c3 + c4;
      const int slot = (int)(ti & (kPjSlots - 1));
      uint2* rrow = rems + (slot * kPjM + rl) * 2;
      if (tot <= 2) {
        if (nrl > 0) rrow[pre] = re0;
        if (nrl > 1) rrow[pre + 1] = re1;
      }
      if (q == 0)
        meta[slot * kPjM + rl] = (uint16_t)((special ? 128u : (uint32_t)(er + 128)) | (tot <= 2 ? (uint32_t)tot << 8 : 0u) |
                                            (special || tot > 2 ? 1u << 10 : 0u));
      fence_proxy_async();
      mbar_arrive(&afull[b]);
      if (lw == 0 && lane == 0 && (it & 15) + kPjLoadWarps > 15) PJ_T(ti, 1);
    }
    if (P.exprange) {
      amax = __reduce_max_sync(0xffffffffu, amax);
      amin = __reduce_min_sync(0xffffffffu, amin);
      if (lane == 0) {
        if (amax >= 0x7F800000u) atomicOr(P.nonfinite, 1u);
        if (amin != 0xFFFFFFFFu) {
          const int e = (int)(((amin + 1u) >> 23) & 0xFF);
          atomicMin(&P.exprange[0], e ? e - 150 : -172);
        }
        if (amax != 0u) {
          const int e = (int)((amax >> 23) & 0xFF);
          atomicMax(&P.exprange[1], e ? e - 126 : -148);
        }
      }
    }
  } else if (warp == kPjMmaWarp) {
    // ---- MMA issuer: block b of tile i into TMEM slot (2i + b) % nslot
    const uint32_t id_s = pj_idesc((int)nb, true), id_u = pj_idesc((int)nb, false);
    const uint64_t d0 = make_sdesc(smem_u32(Abuf), 128, 256);
    const uint32_t alo0 = (uint32_t)d0, dhi = (uint32_t)(d0 >> 32);
    const uint32_t blo0 = (uint32_t)make_sdesc(smem_u32(Pb), 128, 256);  // same high word (LBO/SBO/version)
    for (uint64_t ti = 0; ti < my_tiles; ++ti) {
      const int b = (int)(ti & 1);
      mbar_wait(&afull[b], (uint32_t)(ti >> 1) & 1u);
      if (lane == 0) PJ_T(ti, 2);
#pragma unroll 1
      for (int blk = 0; blk < 2; ++blk) {
        const uint64_t u = 2 * ti + blk;
        const int sl = (int)(u % nslot);
        if (u >= (uint64_t)nslot) mbar_wait(&sfree[sl], (uint32_t)((u / nslot) - 1) & 1u);
        if (lane == 0 && blk) PJ_T(ti, 3);
        fence_after();
        const int smax = blk ? kPjXd : kPjXd - 1;  // block 0 (levels 0-3) never meets digit 4
        const uint32_t dt = tmem + (uint32_t)sl * nb;
#pragma unroll 1
        for (int s = 0; s < smax; ++s) {
          const uint32_t w0 = (uint32_t)((4 * blk - s + 3) * mp);  // B image row of the block's first column
          uint32_t alo = alo0 + ((b * abytes + (uint32_t)(s * nks) * kPjStep) >> 4);
          uint32_t blo = blo0 + ((w0 * 32) >> 4);
#pragma unroll 1
          for (int kk = 0; kk < nks; ++kk) {
            pj_mma(dt, alo, blo, dhi, s ? id_u : id_s, (s | kk) ? 1u : 0u);
            alo += kPjStep >> 4;
            blo += pk >> 4;
          }
        }
      }
      if (elect_one()) {
        tc_commit(&aempty[b]);
        tc_commit(dfull);
      }
      __syncwarp();
      if (lane == 0) PJ_T(ti, 4);
    }
  } else if (warp < kPjEpiWarps) {
    // ---- epilogue: one row per thread; column groups of 8 tables
    const int g4 = warp & 3, half = warp >> 2;
    const int ng = mp >> 3;
    const int rl = g4 * 32 + lane;
    for (uint64_t ti = 0; ti < my_tiles; ++ti) {
      const uint64_t tile = blockIdx.x + ti * gridDim.x;
      const uint64_t row = tile * kPjM + rl;
      const int sl0 = (int)((2 * ti) % nslot), sl1 = (int)((2 * ti + 1) % nslot);
      mbar_wait(dfull, (uint32_t)ti & 1u);
      if (warp == 0 && lane == 0) PJ_T(ti, 5);
      fence_after();
      const int slot = (int)(ti & (kPjSlots - 1));
      const uint32_t mt = meta[slot * kPjM + rl];
      const int er = (int)(mt & 0xFF) - 128;
      const bool frow = (mt >> 10) & 1u;  // special row or > 2 remainder elements
      const double rs = pj_pow2(er);
      const uint32_t erb20 = (uint32_t)(er * (1 << 20));  // + tse[j]: the exponent-field add of the fast keys
      // drain: every group of 8 tables -> sum_l 2^(-8l) D_l as a float64 (one
      // rounding), then release both TMEM slots before the key stores
      constexpr int kMaxG = (kMaxKeyTables / 8 + 1) / 2;  // column groups per warp
      double v[kMaxG][8];
#pragma unroll
      for (int gi = 0; gi < kMaxG; ++gi) {
        const int gq = half + 2 * gi;
        if (gq < ng) {
          int32_t D[kPjLv][8];
          const uint32_t tl = tmem + ((uint32_t)(g4 * 32) << 16) + (uint32_t)gq * 8;
#pragma unroll
          for (int l = 0; l < kPjLv; ++l)
            pj_ld8(tl + (uint32_t)((l < 4 ? sl0 : sl1) * nb + (l & 3) * mp), D[l]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int qj = 0; qj < 8; ++qj) {
            const long long hi = (long long)D[0][qj] * 16777216LL + (long long)D[1][qj] * 65536LL +
                                 (long long)D[2][qj] * 256LL + (long long)D[3][qj];
            const long long lo = (long long)D[4][qj] * 16777216LL + (long long)D[5][qj] * 65536LL +
                                 (long long)D[6][qj] * 256LL + (long long)D[7][qj];
            v[gi][qj] = fma((double)hi, 0x1p32, (double)lo);  // 2^56 sum_l 2^(-8l) D_l, one rounding
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&sfree[sl0]);
        mbar_arrive(&sfree[sl1]);
      }
      if (warp == 0 && lane == 0) PJ_T(ti, 6);
      if (row < P.n) {
        // rows with remainder elements (at most 2; more: float64 FMAs):
        // key = 2^(e_r+e_j-69) v + sum rho_k a_jk, one more rounding
        const int nr = P.prof == 2 ? 0 : (int)(mt >> 8) & 3;
        const bool fma_row = frow || anyspec;
        int k0 = 0, k1 = 0;
        double r0 = 0.0, r1 = 0.0;
        if (nr) {
          const uint2 e0 = rems[(slot * kPjM + rl) * 2], e1 = rems[(slot * kPjM + rl) * 2 + 1];
          k0 = (int)e0.x;
          r0 = (double)__uint_as_float(e0.y);
          if (nr > 1) {
            k1 = (int)e1.x;
            r1 = (double)__uint_as_float(e1.y);
          }
        }
#pragma unroll 1
        for (int gi = 0; gi < kMaxG; ++gi) {  // one copy of the store code (instruction-cache footprint)
          const int gq = half + 2 * gi;
          if (gq >= ng || P.prof == 3) break;
          double w[8];
#pragma unroll
          for (int qj = 0; qj < 8; ++qj) w[qj] = gi == 0 ? v[0][qj] : gi == 1 ? v[1][qj] : v[2][qj];
          const bool full = gq * 8 + 8 <= P.m;
          double corr[8];
          if (nr) {  // the A entries of the 8 tables, loaded together
#pragma unroll
            for (int qj = 0; qj < 8; ++qj) {
              const int j = gq * 8 + qj;
              const double* a = P.A + (uint64_t)min(j, P.m - 1) * P.d;
              corr[qj] = r0 * __ldg(a + k0);
              if (nr > 1) corr[qj] = fma(r1, __ldg(a + k1), corr[qj]);
            }
          }
          // branch-free per table: the keys first, then predicated global stores
          uint64_t kk[8];
          if (!nr) {
#pragma unroll
            for (int qj = 0; qj < 8; ++qj) {
              // w is 0 or an integer-valued double >= 1 in magnitude: scaling by
              // 2^(e_r + e_j - 69) is an add to its exponent field (the result stays normal)
              // on the 32-bit halves: the exponent add touches the high word only (w is 0,
              // or >= 1 in magnitude so its high word is nonzero), then the order transform
              const uint32_t wl = (uint32_t)__double2loint(w[qj]), wh = (uint32_t)__double2hiint(w[qj]);
              const uint32_t h2 = wh ? wh + erb20 + (uint32_t)tse[gq * 8 + qj] : 0u;
              const uint32_t sg = (uint32_t)((int32_t)h2 >> 31);
              kk[qj] = ((uint64_t)(h2 ^ (sg | 0x80000000u)) << 32) | (uint64_t)(wl ^ sg);
            }
          } else {
#pragma unroll
            for (int qj = 0; qj < 8; ++qj) {
              const double key = w[qj] * (rs * tsc[gq * 8 + qj]) + corr[qj];
              const uint64_t bv = key == 0.0 ? 0ull : static_cast<uint64_t>(__double_as_longlong(key));
              kk[qj] = bv ^ (static_cast<uint64_t>(static_cast<long long>(bv) >> 63) | 0x8000000000000000ull);
            }
          }
#pragma unroll
          for (int qj = 0; qj < 8; ++qj)  // streaming global stores the compiler may schedule freely
            if (full || gq * 8 + qj < P.m)
              __stcs(reinterpret_cast<unsigned long long*>(tpp[gq * 8 + qj] + row), (unsigned long long)kk[qj]);
          if (P.dst.fcnt && !fma_row) {
#pragma unroll
            for (int qj = 0; qj < 8; ++qj)
              if (gq * 8 + qj < P.m) pj_count(P.dst, gq * 8 + qj, kk[qj]);
          }
          if (fma_row) {  // special rows / tables: float64 FMAs overwrite the keys
#pragma unroll
            for (int qj = 0; qj < 8; ++qj) {
              const int j = gq * 8 + qj;
              if (j < P.m) {
                const bool fm = frow || tsc[j] == 0.0;
                const uint64_t k2 = fm ? pj_fma_key(P.X, P.A, P.d, row, j) : kk[qj];
                if (fm) P.dst.tptr[j][row] = k2;
                if (P.dst.fcnt) pj_count(P.dst, j, k2);
              }
            }
          }
        }
      }
      if (warp == 0 && lane == 0) PJ_T(ti, 7);
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int tc_project_launch(const float* X, uint64_t n, int d, const double* A, int m, const KeyDst& dst, int* er,
                      unsigned* nf, cudaStream_t s, bool* used) {
  *used = false;
  // the default K1 where it fits; GEEK_TCPROJ=0 selects the DMMA stream kernel (K1t)
  const char* on = getenv("GEEK_TCPROJ");
  if ((on && !atoi(on)) || d < 4 || d > 128 || d % 4 || m < 1 || m > kMaxKeyTables) return GEEK_OK;
  const int mp = (m + 7) / 8 * 8, kp = (d + 31) / 32 * 32, nks = kp / 32;
  const size_t abytes = (size_t)kPjXd * nks * kPjStep, pk = (size_t)11 * mp * 32;
  const size_t smem = 2 * abytes + nks * pk + kMaxKeyTables * 20 + kPjSlots * kPjM * 2 + kPjSlots * kPjM * 16 + 8 * 8 + 16;
  if (smem > (size_t)kPjMaxSmem || 8 * mp > 512) return GEEK_OK;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  Scratch img;
  GEEK_TRY(img.alloc(nks * pk + 64 * 4, s));
  uint8_t* pimg = img.as<uint8_t>();
  int* ej = reinterpret_cast<int*>(pimg + nks * pk);
  pj_prep_kernel<<<std::max(1, std::min(64, (int)((11 * mp * kp + 255) / 256))), 256, 0, s>>>(A, m, d, mp, kp,
                                                                                               pimg, ej);
  GEEK_CHECK_LAUNCH();
  PjParams P;
  P.X = X;
  P.n = n;
  P.d = d;
  P.kp = kp;
  P.m = m;
  P.mp = mp;
  P.A = A;
  P.Pimg = pimg;
  P.ej = ej;
  P.dst = dst;
  P.exprange = er;
  P.nonfinite = nf;
  P.tl = nullptr;
  P.prof = 0;
#ifdef GEEK_DEBUG_KNOBS
  if (const char* e = getenv("GEEK_PJ_PROF")) P.prof = atoi(e);
  static unsigned long long* tl_buf = nullptr;
  if (getenv("GEEK_PJ_TIMELINE")) {
    if (!tl_buf) cudaMalloc(&tl_buf, 64 * 8 * 8);
    cudaMemsetAsync(tl_buf, 0, 64 * 8 * 8, s);
    P.tl = tl_buf;
  }
#endif
  const uint64_t ntiles = (n + kPjM - 1) / kPjM;
  const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)sms);
  auto go = [&](auto kern) -> int {
    GEEK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, kPjThreads, smem, s>>>(P);
    GEEK_CHECK_LAUNCH();
    return GEEK_OK;
  };
  switch (nks) {
    case 1: GEEK_TRY(go(tc_project_kernel<1>)); break;
    case 2: GEEK_TRY(go(tc_project_kernel<2>)); break;
    case 3: GEEK_TRY(go(tc_project_kernel<3>)); break;
    default: GEEK_TRY(go(tc_project_kernel<4>)); break;
  }
#ifdef GEEK_DEBUG_KNOBS
  if (P.tl) {  // per-tile phase durations of CTA 0 (clock64 deltas, tiles 8..63)
    unsigned long long h[64 * 8];
    cudaMemcpyAsync(h, P.tl, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double acc[8] = {0};
    int cnt = 0;
    for (int t = 8; t < 63; ++t) {
      if (!h[(t + 1) * 8 + 5]) break;
      const unsigned long long* r = h + t * 8;
      const double e[8] = {(double)(r[1] - r[0]), (double)(r[3] - r[2]), (double)(r[4] - r[3]),
                           (double)(r[5] - r[4]), (double)(r[6] - r[5]), (double)(r[7] - r[6]),
                           (double)(h[(t + 1) * 8 + 5] - r[5]), (double)(r[2] - h[(t - 1) * 8 + 4])};
      for (int q = 0; q < 8; ++q) acc[q] += e[q];
      ++cnt;
    }
    if (cnt)
      fprintf(stderr,
              "tc_project timeline (clk/tile, %d tiles): load %.0f | mma afull->blk1 %.0f, blk1 issue %.0f | "
              "commit->epi %.0f | drain %.0f | stores %.0f | epi period %.0f | mma gap %.0f\n",
              cnt, acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt, acc[5] / cnt, acc[6] / cnt,
              acc[7] / cnt);
  }
#endif
  *used = true;
  return GEEK_OK;
}

}  // namespace geek
