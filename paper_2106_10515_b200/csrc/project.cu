// K1: float64-accurate random projections of every point onto every table's
// direction (transform.py:125, engine.py:180), emitted as order-preserving
// uint64 keys for the rank split.  HBM-streaming: X is read once per table
// block through shared memory; directions stay resident in shared memory.
#include "common.cuh"
#include "project.cuh"

#include <algorithm>
#include <cstdlib>

namespace geek {

constexpr int kProjThreads = 128;
constexpr int kProjPts = 2;     // points per thread
constexpr int kProjTB = 8;      // tables per pass
constexpr int kProjTile = kProjThreads * kProjPts;

// Bounds of the binary exponent window of a value as the exact-sum kernel
// decomposes it (v = M * 2^L, |M| < 2^P; numeric.py:19-40): lo <= L, hi >= L + P.
// Subnormals take the most negative L their format allows.
__device__ __forceinline__ void exp_window(float v, int& lo, int& hi) {
  const uint32_t b = __float_as_uint(v);
  const int e = (b >> 23) & 0xFF;
  if (e == 0xFF || (b & 0x7FFFFFFFu) == 0) return;
  const int L = e ? e - 150 : -172;
  lo = min(lo, L);
  hi = max(hi, e ? e - 126 : -148);
}

__device__ __forceinline__ void exp_window(double v, int& lo, int& hi) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
  const int e = (int)((b >> 52) & 0x7FF);
  if (e == 0x7FF || (b & 0x7FFFFFFFFFFFFFFFull) == 0) return;
  lo = min(lo, e ? e - 1075 : -1127);
  hi = max(hi, e ? e - 1022 : -1074);
}

template <class T>
__global__ void __launch_bounds__(kProjThreads) project_kernel(const T* __restrict__ X, uint64_t n,
                                                               int d, const double* __restrict__ A,
                                                               int m, uint64_t* __restrict__ keys,
                                                               int* exprange) {
  constexpr int kProjKT = sizeof(T) == 4 ? 32 : 16;  // dims per shared-memory tile (<= 33 KB)
  __shared__ double sA[kProjTB][kProjKT];
  __shared__ T sX[kProjKT][kProjTile + 1];
  const uint64_t tile0 = blockIdx.x * (uint64_t)kProjTile;
  int elo = 1 << 30, ehi = -(1 << 30);
  for (int j0 = 0; j0 < m; j0 += kProjTB) {
    double acc[kProjPts][kProjTB];
#pragma unroll
    for (int p = 0; p < kProjPts; ++p)
#pragma unroll
      for (int j = 0; j < kProjTB; ++j) acc[p][j] = 0.0;
    for (int k0 = 0; k0 < d; k0 += kProjKT) {
      __syncthreads();
      for (int e = threadIdx.x; e < kProjTB * kProjKT; e += kProjThreads) {
        int j = e / kProjKT, k = e % kProjKT;
        sA[j][k] = (j0 + j < m && k0 + k < d) ? A[(uint64_t)(j0 + j) * d + k0 + k] : 0.0;
      }
      // coalesced: consecutive threads read consecutive dims of a row
      for (int e = threadIdx.x; e < kProjTile * kProjKT; e += kProjThreads) {
        int pt = e / kProjKT, k = e % kProjKT;
        uint64_t i = tile0 + pt;
        const T v = (i < n && k0 + k < d) ? X[i * d + k0 + k] : T(0);
        sX[k][pt] = v;
        if (j0 == 0) exp_window(v, elo, ehi);  // fused exponent window (first table pass)
      }
      __syncthreads();
#pragma unroll 8
      for (int k = 0; k < kProjKT; ++k) {
        double x[kProjPts];
#pragma unroll
        for (int p = 0; p < kProjPts; ++p) x[p] = (double)sX[k][threadIdx.x + p * kProjThreads];
#pragma unroll
        for (int j = 0; j < kProjTB; ++j) {
          const double a = sA[j][k];
#pragma unroll
          for (int p = 0; p < kProjPts; ++p) acc[p][j] = fma(x[p], a, acc[p][j]);
        }
      }
    }
#pragma unroll
    for (int p = 0; p < kProjPts; ++p) {
      uint64_t i = tile0 + threadIdx.x + p * kProjThreads;
      if (i < n) {
#pragma unroll
        for (int j = 0; j < kProjTB; ++j)
          if (j0 + j < m) keys[(uint64_t)(j0 + j) * n + i] = f64_key(acc[p][j]);
      }
    }
  }
  if (exprange) {
    for (int o = 16; o; o >>= 1) {
      elo = min(elo, __shfl_xor_sync(0xffffffffu, elo, o));
      ehi = max(ehi, __shfl_xor_sync(0xffffffffu, ehi, o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&exprange[0], elo);
      atomicMax(&exprange[1], ehi);
    }
  }
}

// Register-blocked float64 projection: a block owns 128 points and ALL m
// tables; thread (pg, tg) accumulates 4 points x 4 tables (16 DFMA per
// LDS.128 of x and two LDS.128 of directions).  X and A are staged through
// shared memory in 64-dim chunks, so every X byte is read from HBM once.
constexpr int kP2Pts = 128, kP2KC = 64;

template <class T>
__global__ void __launch_bounds__(512) project4x4_kernel(const T* __restrict__ X, uint64_t n, int d,
                                                          const double* __restrict__ A, int m,
                                                          uint64_t* __restrict__ keys, int* exprange) {
  extern __shared__ __align__(16) uint8_t smraw[];
  const int mg = (m + 3) / 4;                       // table groups
  double* sA = reinterpret_cast<double*>(smraw);    // [kP2KC][mg*4] (k-major, tables adjacent)
  float* sX = reinterpret_cast<float*>(sA + kP2KC * mg * 4);  // [kP2KC][kP2Pts + 4] (T = float)
  double* sXd = reinterpret_cast<double*>(sA + kP2KC * mg * 4);  // (T = double)
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int pg = tid & 31, tg = tid >> 5;           // 32 point groups x mg table groups
  const uint64_t p0 = blockIdx.x * (uint64_t)kP2Pts;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  int elo = 1 << 30, ehi = -(1 << 30);
  const int ldx = kP2Pts + 4;
  for (int k0 = 0; k0 < d; k0 += kP2KC) {
    const int kc = min(kP2KC, d - k0);
    __syncthreads();
    for (int e = tid; e < kP2KC * mg * 4; e += nthr) {
      const int k = e / (mg * 4), j = e - k * (mg * 4);
      sA[e] = (k < kc && j < m) ? A[(uint64_t)j * d + k0 + k] : 0.0;
    }
    for (int e = tid; e < kP2Pts * kP2KC; e += nthr) {
      const int p = e / kP2KC, k = e - p * kP2KC;  // consecutive threads: consecutive dims of a row
      const uint64_t i = p0 + p;
      const T v = (i < n && k < kc) ? X[i * d + k0 + k] : T(0);
      exp_window(v, elo, ehi);
      if (sizeof(T) == 4) sX[k * ldx + p] = (float)v;
      else sXd[k * ldx + p] = (double)v;
    }
    __syncthreads();
    if (tg < mg) {
#pragma unroll 4
      for (int k = 0; k < kc; ++k) {
        double xv[4];
        if (sizeof(T) == 4) {
          const float4 x4 = *reinterpret_cast<const float4*>(sX + k * ldx + pg * 4);
          xv[0] = x4.x; xv[1] = x4.y; xv[2] = x4.z; xv[3] = x4.w;
        } else {
          const double2 xa = *reinterpret_cast<const double2*>(sXd + k * ldx + pg * 4);
          const double2 xb = *reinterpret_cast<const double2*>(sXd + k * ldx + pg * 4 + 2);
          xv[0] = xa.x; xv[1] = xa.y; xv[2] = xb.x; xv[3] = xb.y;
        }
        const double2 aa = *reinterpret_cast<const double2*>(sA + k * mg * 4 + tg * 4);
        const double2 ab = *reinterpret_cast<const double2*>(sA + k * mg * 4 + tg * 4 + 2);
        const double av[4] = {aa.x, aa.y, ab.x, ab.y};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(xv[a], av[b], acc[a][b]);
      }
    }
  }
  if (tg < mg) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int j = tg * 4 + b;
      if (j >= m) break;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const uint64_t i = p0 + pg * 4 + a;
        if (i < n) keys[(uint64_t)j * n + i] = f64_key(acc[a][b]);
      }
    }
  }
  if (exprange) {
    for (int o = 16; o; o >>= 1) {
      elo = min(elo, __shfl_xor_sync(0xffffffffu, elo, o));
      ehi = max(ehi, __shfl_xor_sync(0xffffffffu, ehi, o));
    }
    if ((tid & 31) == 0) {
      atomicMin(&exprange[0], elo);
      atomicMax(&exprange[1], ehi);
    }
  }
}

// float64 projection on the DMMA tensor path (mma.sync m8n8k4 f64; FP64 on
// sm_100 has no tcgen05 kind): 4 warps x 32 points per block, each warp holds
// 4 x NT accumulator fragments (32 points x 8*NT tables); X (as stored) and
// the directions are staged in 64-dim chunks, X read from HBM once.
constexpr int kDmLdx = 136;  // 136: fragment loads are bank-conflict free

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <class T, int NT>
__global__ void __launch_bounds__(128) project_dmma_kernel(const T* __restrict__ X, uint64_t n, int d,
                                                           const double* __restrict__ A, int m,
                                                           uint64_t* __restrict__ keys, int* exprange) {
  constexpr int LDA = NT * 8 + 4;  // tables per k row (+pad)
  constexpr int kDmKC = sizeof(T) == 4 ? 32 : 16;  // dims per chunk: static smem <= 48 KB
  __shared__ __align__(16) T sX[kDmKC * kDmLdx];
  __shared__ __align__(16) double sA[kDmKC * LDA];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t p0 = blockIdx.x * 128ull;
  double acc[4][NT][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  int elo = 1 << 30, ehi = -(1 << 30);
  for (int k0 = 0; k0 < d; k0 += kDmKC) {
    const int kc = min(kDmKC, d - k0);
    __syncthreads();
    // consecutive threads take consecutive points for one dim: conflict-free stores
    for (int e = tid; e < 128 * kDmKC; e += 128) {
      const int k = e >> 7, p = e & 127;  // kDmKC rows of 128 points
      const uint64_t i = p0 + p;
      const T v = (i < n && k < kc) ? X[i * d + k0 + k] : T(0);
      exp_window(v, elo, ehi);
      sX[k * kDmLdx + p] = v;
    }
    for (int e = tid; e < kDmKC * NT * 8; e += 128) {
      const int k = e / (NT * 8), t = e - k * (NT * 8);
      sA[k * LDA + t] = (k < kc && t < m) ? A[(uint64_t)t * d + k0 + k] : 0.0;
    }
    __syncthreads();
    const int kr = lane & 3, rr = lane >> 2;
#pragma unroll 2
    for (int ks = 0; ks < kDmKC; ks += 4) {
      double a[4], b[NT];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = (double)sX[(ks + kr) * kDmLdx + warp * 32 + i * 8 + rr];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = sA[(ks + kr) * LDA + j * 8 + rr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma884(acc[i][j], a[i], b[j]);
    }
  }
  // D fragment: row (point) = lane>>2, columns (tables) 2*(lane&3) + {0,1}
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t pt = p0 + warp * 32 + i * 8 + (lane >> 2);
    if (pt >= n) continue;
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int t = j * 8 + (lane & 3) * 2 + h;
        if (t < m) keys[(uint64_t)t * n + pt] = f64_key(acc[i][j][h]);
      }
  }
  if (exprange) {
    for (int o = 16; o; o >>= 1) {
      elo = min(elo, __shfl_xor_sync(0xffffffffu, elo, o));
      ehi = max(ehi, __shfl_xor_sync(0xffffffffu, ehi, o));
    }
    if (lane == 0) {
      atomicMin(&exprange[0], elo);
      atomicMax(&exprange[1], ehi);
    }
  }
}

// Streaming DMMA projection for float32 X (d % 4 == 0, d <= 128): persistent
// CTAs (two per SM) keep the transposed directions resident in SMEM and pull
// 32-dim chunks of 128-point tiles through a 3-stage cp.async ring, so the
// HBM stream of X overlaps the DMMAs.  The k order of the accumulation is the
// one of project_dmma_kernel (chunks of 4 dims, ascending): same bits.
constexpr int kPsLdp = 36;     // floats per point row of a stage: fragment loads are conflict-free
constexpr int kPsStages = 3;
constexpr int kPsStageFloats = 128 * kPsLdp;
constexpr int kPsKeyLd = 34;   // u64 per table row of the per-warp key tile (16-byte aligned rows)

__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int NT>
__global__ void __launch_bounds__(128, 2) project_stream_kernel(const float* __restrict__ X, uint64_t n, int d,
                                                                const double* __restrict__ A, int m,
                                                                const KeyDst dst, int* exprange,
                                                                unsigned* nonfinite) {
  constexpr int LDA = NT * 8 + 4;
  extern __shared__ __align__(16) uint8_t smem[];
  double* sA = reinterpret_cast<double*>(smem);                      // [d][LDA]
  float* sX = reinterpret_cast<float*>(smem + (size_t)d * LDA * 8);  // [stages][128][kPsLdp]
  uint64_t* sK = reinterpret_cast<uint64_t*>(sX + kPsStages * kPsStageFloats);  // [4 warps][8][kPsKeyLd]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < d * NT * 8; e += 128) {
    const int k = e / (NT * 8), t = e - k * (NT * 8);
    sA[k * LDA + t] = t < m ? A[(uint64_t)t * d + k] : 0.0;
  }
  const int nck = (d + 31) / 32;
  const uint64_t ntiles = (n + 127) / 128;
  const uint64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint64_t total = my_tiles * nck;
  auto issue = [&](uint64_t q) {
    if (q < total) {
      const uint64_t tile = blockIdx.x + (q / nck) * gridDim.x;
      const int kc = (int)(q % nck);
      float* st = sX + (q % kPsStages) * kPsStageFloats;
      // each warp stages only its own 32 rows: the warps never wait for each other
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = warp * 32 + (lane >> 3) + 4 * u, c4 = lane & 7;
        const uint64_t row = tile * 128 + r;
        const int dim = kc * 32 + c4 * 4;
        const bool ok = row < n && dim < d;
        cp_async16(st + r * kPsLdp + c4 * 4, ok ? X + row * d + dim : X, ok ? 16u : 0u);
      }
    }
    cp_async_commit();  // empty groups keep the wait count uniform
  };
#pragma unroll
  for (int q = 0; q < kPsStages - 1; ++q) issue(q);
  double acc[4][NT][2];
  // exponent window from the extreme |x| bit patterns (4 integer ops per
  // element): the exponent field of the smallest nonzero and of the largest
  // |x| give exp_window's bounds; a non-finite value sends the caller to the
  // exact per-element pass instead
  uint32_t amax = 0u, amin = 0xFFFFFFFFu;
  const int kr = lane & 3, rr = lane >> 2;
  uint64_t* kdst[NT][2];  // this thread's tables (D fragment columns)
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = j * 8 + kr * 2 + h;
      kdst[j][h] = t < m ? dst.tptr[t] : nullptr;
    }
  __syncthreads();  // the directions are in SMEM
  for (uint64_t q = 0; q < total; ++q) {
    cp_async_wait<kPsStages - 2>();
    __syncwarp();                   // chunk q of this warp's rows landed; its rows of stage (q-1) % S are free
    issue(q + kPsStages - 1);
    const int kc = (int)(q % nck);
    if (kc == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    const float* st = sX + (q % kPsStages) * kPsStageFloats + (warp * 32 + rr) * kPsLdp + kr;
    const double* sa = sA + (kc * 32 + kr) * LDA + rr;
#pragma unroll
    for (int ks = 0; ks < 32; ks += 4) {
      double a[4], b[NT];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float v = st[i * 8 * kPsLdp + ks];
        const uint32_t ab = __float_as_uint(v) & 0x7FFFFFFFu;
        amax = max(amax, ab);
        amin = min(amin, ab - 1u);  // 0 wraps to the top: zeros never count
        a[i] = (double)v;
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = kc * 32 + ks < d ? sa[ks * LDA + j * 8] : 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma884(acc[i][j], a[i], b[j]);
    }
    if (kc == nck - 1 && dst.vec16 && !dst.fcnt) {
      // keys leave as 16-byte stores that make 256-byte runs per table: the
      // warp's 32 points x 8 tables of one column group are transposed
      // through a per-warp SMEM tile (NVLink-friendly when the owner is a peer)
      const uint64_t tile = blockIdx.x + (q / nck) * gridDim.x;
      uint64_t* sw = sK + warp * 8 * kPsKeyLd;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int h = 0; h < 2; ++h) sw[(kr * 2 + h) * kPsKeyLd + i * 8 + rr] = f64_key(acc[i][j][h]);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int tl = 2 * k + (lane >> 4), t = j * 8 + tl, qp = lane & 15;
          const uint64_t pt0 = tile * 128 + warp * 32 + 2 * qp;
          if (t < m && pt0 < n) {
            const uint64_t k0 = sw[tl * kPsKeyLd + 2 * qp], k1 = sw[tl * kPsKeyLd + 2 * qp + 1];
            uint64_t* dp = dst.tptr[t] + pt0;
            if (pt0 + 1 < n) *reinterpret_cast<ulonglong2*>(dp) = make_ulonglong2(k0, k1);
            else dp[0] = k0;
          }
        }
      }
    } else if (kc == nck - 1) {
      const uint64_t tile = blockIdx.x + (q / nck) * gridDim.x;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint64_t pt = tile * 128 + warp * 32 + i * 8 + rr;
        if (pt >= n) continue;
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int t = j * 8 + kr * 2 + h;
            if (t < m) {
              const uint64_t key = f64_key(acc[i][j][h]);
              kdst[j][h][pt] = key;
              if (dst.fcnt) {
                const uint2 ci = __ldg(dst.cinfo + ((uint64_t)t << dst.cb) + (uint32_t)(key >> (64 - dst.cb)));
                const uint32_t frac = static_cast<uint32_t>((key << dst.cb) >> 32);
                atomicAdd(dst.fcnt + ci.y + static_cast<uint32_t>(((uint64_t)frac * ci.x) >> 32), 1u);
              }
            }
          }
      }
    }
  }
  cp_async_wait<0>();
  if (exprange) {
    amax = __reduce_max_sync(0xffffffffu, amax);
    amin = __reduce_min_sync(0xffffffffu, amin);
    if (lane == 0) {
      if (amax >= 0x7F800000u) atomicOr(nonfinite, 1u);
      if (amin != 0xFFFFFFFFu) {
        const int e = (int)(((amin + 1u) >> 23) & 0xFF);
        atomicMin(&exprange[0], e ? e - 150 : -172);
      }
      if (amax != 0u) {
        const int e = (int)((amax >> 23) & 0xFF);
        atomicMax(&exprange[1], e ? e - 126 : -148);
      }
    }
  }
}

static void fill_table_ptrs(KeyDst& dst, int m) {
  dst.vec16 = 1;
  for (int t = 0; t < kMaxKeyTables; ++t) {
    dst.tptr[t] = t < m ? dst.ptr[t % dst.G] + (uint64_t)(t / dst.G) * dst.ntot + dst.row_lo : nullptr;
    if (t < m && (reinterpret_cast<uintptr_t>(dst.tptr[t]) & 15)) dst.vec16 = 0;
  }
}

template <int NT>
static int launch_stream(const float* X, uint64_t n, int d, const double* A, int m, const KeyDst& dst, int* er,
                         unsigned* nf, cudaStream_t s) {
  const size_t smem = (size_t)d * (NT * 8 + 4) * 8 + (size_t)kPsStages * kPsStageFloats * 4 + 4 * 8 * kPsKeyLd * 8;
  GEEK_CHECK_CUDA(cudaFuncSetAttribute(project_stream_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t ntiles = (n + 127) / 128;
  const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)sms * 2);
  project_stream_kernel<NT><<<grid, 128, smem, s>>>(X, n, d, A, m, dst, er, nf);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

static int launch_stream_any(const float* X, uint64_t n, int d, const double* A, int m, const KeyDst& keys,
                             int* er, cudaStream_t s) {
  Scratch flag;
  unsigned* nf = nullptr;
  if (er) {
    GEEK_TRY(flag.alloc(4, s));
    GEEK_CHECK_CUDA(cudaMemsetAsync(flag.ptr, 0, 4, s));
    nf = flag.as<unsigned>();
  }
  bool tc = false;
  GEEK_TRY(tc_project_launch(X, n, d, A, m, keys, er, nf, s, &tc));
  if (!tc) switch ((m + 7) / 8) {
    case 1: GEEK_TRY(launch_stream<1>(X, n, d, A, m, keys, er, nf, s)); break;
    case 2: GEEK_TRY(launch_stream<2>(X, n, d, A, m, keys, er, nf, s)); break;
    case 3: GEEK_TRY(launch_stream<3>(X, n, d, A, m, keys, er, nf, s)); break;
    case 4: GEEK_TRY(launch_stream<4>(X, n, d, A, m, keys, er, nf, s)); break;
    case 5: GEEK_TRY(launch_stream<5>(X, n, d, A, m, keys, er, nf, s)); break;
    default: GEEK_TRY(launch_stream<6>(X, n, d, A, m, keys, er, nf, s)); break;
  }
  if (er) {  // a non-finite value: redo the window exactly, value by value
    unsigned h = 0;
    GEEK_CHECK_CUDA(cudaMemcpyAsync(&h, nf, 4, cudaMemcpyDeviceToHost, s));
    GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
    if (h) GEEK_TRY(exponent_range_f32_device(X, n * (uint64_t)d, er, s));
  }
  return GEEK_OK;
}

template <class T>
static void launch_dmma(const T* X, uint64_t n, int d, const double* A, int m, uint64_t* keys, int* er,
                        cudaStream_t s) {
  const unsigned grid = (unsigned)((n + 127) / 128);
  switch ((m + 7) / 8) {
    case 1: project_dmma_kernel<T, 1><<<grid, 128, 0, s>>>(X, n, d, A, m, keys, er); break;
    case 2: project_dmma_kernel<T, 2><<<grid, 128, 0, s>>>(X, n, d, A, m, keys, er); break;
    case 3: project_dmma_kernel<T, 3><<<grid, 128, 0, s>>>(X, n, d, A, m, keys, er); break;
    case 4: project_dmma_kernel<T, 4><<<grid, 128, 0, s>>>(X, n, d, A, m, keys, er); break;
    case 5: project_dmma_kernel<T, 5><<<grid, 128, 0, s>>>(X, n, d, A, m, keys, er); break;
    case 6: project_dmma_kernel<T, 6><<<grid, 128, 0, s>>>(X, n, d, A, m, keys, er); break;
    default: break;
  }
}

template <class T>
__global__ void column_keys_kernel(const T* __restrict__ v, uint64_t n, uint64_t stride, uint64_t col,
                                   uint64_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = f64_key((double)v[i * stride + col]);
}

}  // namespace geek

using namespace geek;

extern "C" {

int geek_project_keys(const void* X, int dtype, uint64_t n, int d, const double* A, int m,
                      uint64_t* keys, int* exprange, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(dtype == 0 || dtype == 1, "dtype must be 0 (f32) or 1 (f64)");
  GEEK_REQUIRE(d >= 1 && m >= 1, "empty projection");
  if (n == 0) return GEEK_OK;
  if (m <= 48 && dtype == 0 && d % 4 == 0 && d <= 128 && !getenv("GEEK_NO_DMMA") && !getenv("GEEK_NO_PSTREAM"))
  {
    KeyDst dst{};
    dst.ptr[0] = keys;
    dst.G = 1;
    dst.ntot = n;
    dst.row_lo = 0;
    dst.cinfo = nullptr;
    dst.fcnt = nullptr;
    dst.cb = 0;
    fill_table_ptrs(dst, m);
    return launch_stream_any((const float*)X, n, d, A, m, dst, exprange, s);
  }
  if (m <= 48 && !getenv("GEEK_NO_DMMA")) {  // DMMA path (up to 6 column fragments)
    if (dtype == 0) launch_dmma<float>((const float*)X, n, d, A, m, keys, exprange, s);
    else launch_dmma<double>((const double*)X, n, d, A, m, keys, exprange, s);
    GEEK_CHECK_LAUNCH();
    return GEEK_OK;
  }
  const int mg = (m + 3) / 4;
  if (mg <= 16) {  // register-blocked path: 32 point groups x mg table groups per block
    const size_t smem = (size_t)kP2KC * mg * 4 * 8 + (size_t)kP2KC * (kP2Pts + 4) * (dtype == 0 ? 4 : 8);
    const unsigned grid = (unsigned)((n + kP2Pts - 1) / kP2Pts);
    if (dtype == 0) {
      if (smem > 48 * 1024)
        GEEK_CHECK_CUDA(cudaFuncSetAttribute(project4x4_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
      project4x4_kernel<float><<<grid, 32 * mg, smem, s>>>((const float*)X, n, d, A, m, keys, exprange);
    } else {
      if (smem > 48 * 1024)
        GEEK_CHECK_CUDA(cudaFuncSetAttribute(project4x4_kernel<double>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      project4x4_kernel<double><<<grid, 32 * mg, smem, s>>>((const double*)X, n, d, A, m, keys, exprange);
    }
    GEEK_CHECK_LAUNCH();
    return GEEK_OK;
  }
  unsigned grid = (unsigned)((n + kProjTile - 1) / kProjTile);
  if (dtype == 0)
    project_kernel<float><<<grid, kProjThreads, 0, s>>>((const float*)X, n, d, A, m, keys, exprange);
  else
    project_kernel<double><<<grid, kProjThreads, 0, s>>>((const double*)X, n, d, A, m, keys, exprange);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

int geek_project_keys_routed(const void* X, int dtype, uint64_t n, int d, const double* A, int m,
                             uint64_t* const* dst_host, int G, uint64_t ntot, uint64_t row_lo, int* exprange,
                             const uint32_t* fine_cinfo, int cb, uint32_t* fine_cnt, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(G >= 1 && G <= kMaxKeyDst, "routed projection supports 1..%d owners", kMaxKeyDst);
  GEEK_REQUIRE(dtype == 0 && d % 4 == 0 && d >= 4 && d <= 128 && m >= 1 && m <= 48,
               "routed projection needs float32 rows, d %% 4 == 0, d <= 128, m <= 48");
  GEEK_REQUIRE(row_lo + n <= ntot, "rows [%llu, %llu) outside the %llu-row key arrays",
               (unsigned long long)row_lo, (unsigned long long)(row_lo + n), (unsigned long long)ntot);
  if (n == 0) return GEEK_OK;
  KeyDst dst{};
  for (int q = 0; q < G; ++q) dst.ptr[q] = dst_host[q];
  dst.G = G;
  dst.ntot = ntot;
  dst.row_lo = row_lo;
  GEEK_REQUIRE(!fine_cnt || (fine_cinfo && cb >= 1 && cb <= 24), "fused fine counts need the cell layout");
  dst.cinfo = reinterpret_cast<const uint2*>(fine_cinfo);
  dst.fcnt = fine_cnt;
  dst.cb = cb;
  fill_table_ptrs(dst, m);
  return launch_stream_any((const float*)X, n, d, A, m, dst, exprange, s);
}

int geek_column_keys(const void* values, int dtype, uint64_t n, uint64_t stride, uint64_t col,
                     uint64_t* keys, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(dtype == 0 || dtype == 1, "dtype must be 0 (f32) or 1 (f64)");
  if (n == 0) return GEEK_OK;
  if (dtype == 0)
    column_keys_kernel<float><<<grid_for(n, 256), 256, 0, s>>>((const float*)values, n, stride, col, keys);
  else
    column_keys_kernel<double><<<grid_for(n, 256), 256, 0, s>>>((const double*)values, n, stride, col, keys);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

}  // extern "C"
