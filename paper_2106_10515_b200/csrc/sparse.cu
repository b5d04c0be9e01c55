// K9/K10: sparse-set and categorical kernels -- DOPH reduction
// (hashing.py:304-329), Jaccard assignment for categorical records and
// binary sparse sets (assignment.py:63-78), and the mode statistics behind
// categorical / sparse centers (seeding.py:180-194, engine.py:312-322).
#include "common.cuh"

#include <algorithm>
#include <cstdlib>

namespace geek {

// one warp per set: bin-minimum flags and tokens (bin + rel) mod r
__global__ void doph_tokens_kernel(const uint32_t* p, const uint64_t* off, uint64_t nsets, uint64_t width,
                                   uint64_t r, uint32_t* tok, uint8_t* ismin) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const unsigned lane = threadIdx.x & 31;
  for (uint64_t s = warp; s < nsets; s += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const uint64_t b = off[s], e = off[s + 1];
    for (uint64_t i = b + lane; i < e; i += 32) {
      const uint64_t pi = p[i], bi = pi / width;
      bool mn = true;
      for (uint64_t j = b; j < e; ++j) {
        const uint64_t pj = p[j];
        if (pj / width == bi && pj < pi) {
          mn = false;
          break;
        }
      }
      ismin[i] = mn;
      tok[i] = static_cast<uint32_t>((bi + (pi - bi * width)) % r);
    }
  }
}

// distinct sorted tokens of the bin minima
__global__ void doph_emit_kernel(const uint32_t* tok, const uint8_t* ismin, const uint64_t* off, uint64_t nsets,
                                 uint32_t* counts, const uint64_t* out_off, uint32_t* out_flat) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const unsigned lane = threadIdx.x & 31;
  for (uint64_t s = warp; s < nsets; s += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const uint64_t b = off[s], e = off[s + 1];
    uint32_t distinct = 0;
    for (uint64_t i = b + lane; i < e; i += 32) {
      if (!ismin[i]) continue;
      const uint32_t ti = tok[i];
      bool first = true;
      uint32_t below = 0;
      for (uint64_t j = b; j < e; ++j) {
        if (!ismin[j]) continue;
        const uint32_t tj = tok[j];
        if (tj == ti && j < i) first = false;
        // count distinct smaller tokens: only first occurrences
        if (tj < ti) {
          bool jfirst = true;
          for (uint64_t q = b; q < j; ++q)
            if (ismin[q] && tok[q] == tj) {
              jfirst = false;
              break;
            }
          below += jfirst;
        }
      }
      if (first) {
        ++distinct;
        if (out_flat) out_flat[out_off[s] + below] = ti;
      }
    }
    for (int o = 16; o; o >>= 1) distinct += __shfl_xor_sync(0xffffffffu, distinct, o);
    if (lane == 0 && counts) counts[s] = distinct;
  }
}

// One warp per set, r <= kDophSmemR: bin minima of the permuted ids by
// shared-memory atomicMin over r slots, then the tokens of the occupied bins
// set bits of an r-bit map, and the set's distinct tokens leave in ascending
// order by popcount prefix -- O(|set| + r/32) per set instead of the pairwise
// scans of doph_tokens / doph_emit.
constexpr uint32_t kDophSmemR = 4096;

__global__ void doph_smem_kernel(const uint32_t* __restrict__ p, const uint64_t* __restrict__ off,
                                 uint64_t nsets, uint64_t width, uint32_t r, uint32_t* counts,
                                 const uint64_t* out_off, uint32_t* out_flat) {
  extern __shared__ uint32_t sm[];
  const int wpb = blockDim.x >> 5, w = threadIdx.x >> 5;
  const unsigned lane = threadIdx.x & 31;
  const uint32_t words = (r + 31) / 32;
  uint32_t* bmin = sm + (size_t)w * (r + words);
  uint32_t* bits = bmin + r;
  for (uint64_t s = blockIdx.x * (uint64_t)wpb + w; s < nsets; s += (uint64_t)gridDim.x * wpb) {
    const uint64_t b = off[s], e = off[s + 1];
    for (uint32_t j = lane; j < r; j += 32) bmin[j] = 0xFFFFFFFFu;
    for (uint32_t j = lane; j < words; j += 32) bits[j] = 0u;
    __syncwarp();
    for (uint64_t i = b + lane; i < e; i += 32) {
      const uint32_t pi = p[i];
      atomicMin(&bmin[pi / width], pi);
    }
    __syncwarp();
    for (uint32_t j = lane; j < r; j += 32) {
      const uint32_t pm = bmin[j];
      if (pm != 0xFFFFFFFFu) {
        const uint32_t t = (uint32_t)(((uint64_t)j + (pm - (uint64_t)j * width)) % r);
        atomicOr(&bits[t >> 5], 1u << (t & 31));
      }
    }
    __syncwarp();
    uint32_t base = 0;
    for (uint32_t w0 = 0; w0 < words; w0 += 32) {
      const uint32_t wi = w0 + lane;
      const uint32_t v = wi < words ? bits[wi] : 0u;
      const uint32_t c = __popc(v);
      uint32_t incl = c;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane >= o) incl += y;
      }
      if (out_flat && v) {
        uint32_t pos = base + incl - c;
        uint32_t m = v;
        while (m) {
          const int bit = __ffs(m) - 1;
          out_flat[out_off[s] + pos++] = wi * 32 + bit;
          m &= m - 1;
        }
      }
      base += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0 && counts) counts[s] = base;
    __syncwarp();
  }
}

__global__ void assign_cat_kernel(const int32_t* __restrict__ codes, uint64_t n, int d,
                                  const int32_t* __restrict__ modes, uint64_t k, int64_t* labels, double* best) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const int32_t* x = codes + i * d;
    double bd = 0.0;
    int64_t bl = -1;
    for (uint64_t c = 0; c < k; ++c) {
      const int32_t* mo = modes + c * d;
      int mt = 0;
      for (int a = 0; a < d; ++a) mt += (x[a] == mo[a]);
      const double dist = __dsub_rn(1.0, __ddiv_rn((double)mt, (double)(2 * d - mt)));
      if (bl < 0 || dist < bd) {
        bd = dist;
        bl = (int64_t)c;
      }
    }
    labels[i] = bl;
    best[i] = bd;
  }
}

// Tiled categorical assignment (d <= 64, k < 2^24): every thread keeps one
// center's DP codes in registers, the block streams 256-point (128 for d > 40) tiles of codes
// through shared memory (a broadcast read per 4 attributes) and keeps each
// point's best key max(mt << 24 | (2^24 - 1 - c)) -- the largest match count
// mt, first center on ties -- in shared memory across the center chunks.
// The Jaccard-style distance 1 - mt / (2d - mt) decreases strictly with mt, so
// the key's order is the reference's `dist < best` scan order
// (assignment.py:63-67; numpy argmin's first index).
__device__ __forceinline__ void cat_match(int& m, int x, int c) {
  asm("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %1, %2;\n\t@p add.s32 %0, %0, 1;\n\t}" : "+r"(m) : "r"(x), "r"(c));
}

template <int DP>
constexpr int cat_pt() { return DP <= 40 ? 256 : 128; }  // points per tile: <= 41 KB static smem

template <int DP>
__global__ void __launch_bounds__(256) assign_cat_tiled_kernel(const int32_t* __restrict__ codes, uint64_t n, int d,
                                                                 const int32_t* __restrict__ modesT, uint64_t kpad,
                                                                 uint64_t k, int64_t* labels, double* best) {
  constexpr int PT = cat_pt<DP>();
  __shared__ __align__(16) int32_t sp[PT * DP];
  __shared__ unsigned sbest[PT];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint64_t ntiles = (n + PT - 1) / PT;
  const uint64_t nchunks = (k + 255) / 256;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t p0 = tile * PT;
    const int np = (int)((n - p0) < (uint64_t)PT ? (n - p0) : (uint64_t)PT);
    const int32_t* src = codes + p0 * (uint64_t)d;
    for (int e = tid; e < PT * DP; e += 256) {
      const int p = e / DP, a = e - p * DP;
      sp[e] = (p < np && a < d) ? src[(uint64_t)p * d + a] : 0;  // pad attributes read 0
    }
    if (tid < PT) sbest[tid] = 0;
    __syncthreads();
    for (uint64_t ch = 0; ch < nchunks; ++ch) {
      const uint64_t c = ch * 256 + tid;
      int32_t cm[DP];
#pragma unroll
      for (int a = 0; a < DP; ++a) cm[a] = modesT[(uint64_t)a * kpad + c];  // pad rows hold 1
      const unsigned tag = (c < k) ? (0xFFFFFFu - (unsigned)c) : 0u;
      const bool valid = c < k;
      for (int p = 0; p < np; ++p) {
        const int4* row = reinterpret_cast<const int4*>(sp + p * DP);
        int m0 = 0, m1 = 0;  // two chains: compare + predicated increment per attribute
#pragma unroll
        for (int q = 0; q < DP / 4; ++q) {
          const int4 v = row[q];
          cat_match(m0, v.x, cm[4 * q]);
          cat_match(m1, v.y, cm[4 * q + 1]);
          cat_match(m0, v.z, cm[4 * q + 2]);
          cat_match(m1, v.w, cm[4 * q + 3]);
        }
        const int mt = m0 + m1;
        const unsigned key = valid ? (((unsigned)mt << 24) | tag) : 0u;
        const unsigned wk = __reduce_max_sync(0xffffffffu, key);
        if (lane == 0) atomicMax(&sbest[p], wk);
      }
    }
    __syncthreads();
    if (tid < np) {
      const unsigned key = sbest[tid];
      const int mt = (int)(key >> 24);
      labels[p0 + tid] = (int64_t)(0xFFFFFFu - (key & 0xFFFFFFu));
      best[p0 + tid] = __dsub_rn(1.0, __ddiv_rn((double)mt, (double)(2 * d - mt)));
    }
    __syncthreads();
  }
}

__global__ void modes_transpose_kernel(const int32_t* modes, uint64_t k, int d, int DP, uint64_t kpad, int32_t* out) {
  const uint64_t total = (uint64_t)DP * kpad;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = e / kpad, c = e - a * kpad;
    out[e] = ((int)a < d && c < k) ? modes[c * d + a] : 1;  // pad rows/centers never meet a point's 0 pad
  }
}

__global__ void mode_sizes_kernel(const int32_t* modes, uint64_t k, uint64_t u, double* sz) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < k;
       c += (uint64_t)gridDim.x * blockDim.x) {
    long long t = 0;
    for (uint64_t e = 0; e < u; ++e) t += modes[c * u + e];
    sz[c] = (double)t;
  }
}

__global__ void assign_sparse_kernel(const uint32_t* flat, const uint64_t* off, uint64_t n, uint64_t u,
                                     const int32_t* modes, const double* msz, uint64_t k, int64_t* labels,
                                     double* best) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = off[i], e = off[i + 1];
    const double xs = (double)(e - b);
    double bd = 0.0;
    int64_t bl = -1;
    for (uint64_t c = 0; c < k; ++c) {
      const int32_t* mo = modes + c * u;
      long long inter = 0;
      for (uint64_t q = b; q < e; ++q) inter += (mo[flat[q]] != 0);
      const double in = (double)inter;
      const double uni = __dsub_rn(__dadd_rn(xs, msz[c]), in);
      const double sim = uni > 0.0 ? __ddiv_rn(in, uni) : 1.0;
      const double dist = __dsub_rn(1.0, sim);
      if (bl < 0 || dist < bd) {
        bd = dist;
        bl = (int64_t)c;
      }
    }
    labels[i] = bl;
    best[i] = bd;
  }
}

// Bitset Jaccard assignment for universes <= 32*WM ids: modes as bitsets
// staged in SMEM tiles, each thread's set as WM register words; per pair
// inter = sum popc(x & c), union = |x| + |c| - inter.  With |x|, |c| <= 2048
// distinct similarities inter/union differ by more than 2^-22, so comparing
// them exactly as fractions (inter * u' vs inter' * u) orders them as the
// reference's float64 1 - inter/union does, ties included (first index kept);
// the winner's distance is then evaluated with the reference's float64 ops.
constexpr int kBitTile = 256;

__global__ void mode_bits_kernel(const int32_t* modes, uint64_t k, uint64_t u, int W, uint32_t* bits,
                                 uint32_t* sizes) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < k; c += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t tot = 0;
    for (int w = 0; w < W; ++w) {
      uint32_t v = 0;
      for (int b = 0; b < 32; ++b) {
        const uint64_t e = (uint64_t)w * 32 + b;
        if (e < u && modes[c * u + e] != 0) v |= 1u << b;
      }
      bits[c * W + w] = v;
      tot += __popc(v);
    }
    sizes[c] = tot;
  }
}

template <int WM>
__global__ void __launch_bounds__(128) assign_sparse_bits_kernel(const uint32_t* __restrict__ flat,
                                                                 const uint64_t* __restrict__ off, uint64_t n,
                                                                 const uint32_t* __restrict__ mbits,
                                                                 const uint32_t* __restrict__ msize, uint64_t k,
                                                                 int W, int64_t* labels, double* best) {
  __shared__ uint32_t sb[kBitTile * WM];
  __shared__ uint32_t ss[kBitTile];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t first = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  // block-uniform trip count (the tiles are loaded cooperatively)
  const uint64_t iters = (n + stride - 1) / stride;
  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t i = first + it * stride;
    const bool valid = i < n;
    uint32_t x[WM];
#pragma unroll
    for (int w = 0; w < WM; ++w) x[w] = 0;
    uint32_t xs = 0;
    if (valid) {
      const uint64_t b = off[i], e = off[i + 1];
      xs = (uint32_t)(e - b);
      for (uint64_t q = b; q < e; ++q) {
        const uint32_t v = flat[q];
        const uint32_t wv = v >> 5, bit = 1u << (v & 31);
#pragma unroll
        for (int w = 0; w < WM; ++w) x[w] |= (wv == (uint32_t)w) ? bit : 0u;
      }
    }
    uint32_t bi = 0, bu = 1;
    long long bl = -1;
    for (uint64_t c0 = 0; c0 < k; c0 += kBitTile) {
      const int nc = (int)min((uint64_t)kBitTile, k - c0);
      __syncthreads();
      for (int e = threadIdx.x; e < nc * W; e += blockDim.x) {
        const int c = e / W, w = e - c * W;
        sb[c * WM + w] = mbits[(c0 + c) * W + w];
      }
      for (int c = threadIdx.x; c < nc; c += blockDim.x) ss[c] = msize[c0 + c];
      __syncthreads();
      if (!valid) continue;
      for (int c = 0; c < nc; ++c) {
        uint32_t in = 0;
#pragma unroll
        for (int w = 0; w < WM; ++w) in += __popc(x[w] & sb[c * WM + w]);
        const uint32_t un = xs + ss[c] - in;
        // similarity in/un strictly larger (un >= 1: sets are non-empty)
        if (bl < 0 || (unsigned long long)in * bu > (unsigned long long)bi * un) {
          bi = in;
          bu = un;
          bl = (long long)(c0 + c);
        }
      }
    }
    if (valid) {
      const double uni = __dsub_rn(__dadd_rn((double)xs, (double)(bu + bi - xs)), (double)bi);
      const double sim = uni > 0.0 ? __ddiv_rn((double)bi, uni) : 1.0;
      labels[i] = bl;
      best[i] = __dsub_rn(1.0, sim);
    }
  }
}

__global__ void mode_counts_kernel(const int32_t* codes, uint64_t nrows, int d, uint64_t row_lo, uint64_t cs,
                                   const uint32_t* flat, const uint64_t* off, uint64_t ngroups, uint64_t total,
                                   unsigned long long* counts) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total * d;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = e / d;
    const int c = (int)(e - k * d);
    const uint64_t id = flat[k];
    if (id < row_lo || id >= row_lo + nrows) continue;
    uint64_t lo = 0, hi = ngroups;
    while (hi - lo > 1) {
      uint64_t mid = (lo + hi) >> 1;
      if (off[mid] <= k) lo = mid;
      else hi = mid;
    }
    const int32_t v = codes[(id - row_lo) * d + c];
    atomicAdd(&counts[(lo * d + c) * cs + (uint64_t)v], 1ull);
  }
}

__global__ void sparse_counts_kernel(const uint32_t* set_flat, const uint64_t* set_off, uint64_t nrows,
                                     uint64_t row_lo, uint64_t u, const uint32_t* flat, const uint64_t* off,
                                     uint64_t ngroups, uint64_t total, unsigned long long* counts) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < total;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t id = flat[k];
    if (id < row_lo || id >= row_lo + nrows) continue;
    uint64_t lo = 0, hi = ngroups;
    while (hi - lo > 1) {
      uint64_t mid = (lo + hi) >> 1;
      if (off[mid] <= k) lo = mid;
      else hi = mid;
    }
    const uint64_t r = id - row_lo;
    for (uint64_t q = set_off[r]; q < set_off[r + 1]; ++q) atomicAdd(&counts[lo * u + set_flat[q]], 1ull);
  }
}

}  // namespace geek

using namespace geek;

extern "C" {

int geek_doph_reduce(const geek_perm_t* perm_host, const uint32_t* tables, const uint32_t* flat,
                     const uint64_t* offsets, uint64_t nsets, uint64_t D, uint64_t r, uint32_t* counts,
                     const uint64_t* out_off, uint32_t* out_flat, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(r >= 1 && r <= D, "need 1 <= target_dims <= universe");
  GEEK_REQUIRE(perm_host->u == D, "permutation universe must equal D");
  if (nsets == 0) return GEEK_OK;
  uint64_t total = 0;
  GEEK_CHECK_CUDA(cudaMemcpyAsync(&total, offsets + nsets, 8, cudaMemcpyDeviceToHost, s));
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
  Scratch p, tok, mn;
  GEEK_TRY(p.alloc(total * 4, s));
  GEEK_TRY(geek_perm_forward(perm_host, 1, tables, flat, total, p.as<uint32_t>(), stream));
  const uint64_t width = (D + r - 1) / r;
  if (r <= kDophSmemR && !getenv("GEEK_DOPH_PAIRWISE")) {
    const size_t per_warp = 4 * ((size_t)r + (r + 31) / 32);
    const int wpb = (int)std::max<size_t>(1, std::min<size_t>(8, (96 * 1024) / per_warp));
    const size_t smem = per_warp * wpb;
    if (smem > 48 * 1024)
      GEEK_CHECK_CUDA(cudaFuncSetAttribute(doph_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    doph_smem_kernel<<<grid_for(nsets, wpb, 148 * 16), 32 * wpb, smem, s>>>(p.as<uint32_t>(), offsets, nsets, width,
                                                                            (uint32_t)r, counts, out_off, out_flat);
    GEEK_CHECK_LAUNCH();
    GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
    return GEEK_OK;
  }
  GEEK_TRY(tok.alloc(total * 4, s));
  GEEK_TRY(mn.alloc(total, s));
  doph_tokens_kernel<<<grid_for(nsets * 32, 256), 256, 0, s>>>(p.as<uint32_t>(), offsets, nsets, width, r,
                                                               tok.as<uint32_t>(), mn.as<uint8_t>());
  GEEK_CHECK_LAUNCH();
  doph_emit_kernel<<<grid_for(nsets * 32, 256), 256, 0, s>>>(tok.as<uint32_t>(), mn.as<uint8_t>(), offsets,
                                                             nsets, counts, out_off, out_flat);
  GEEK_CHECK_LAUNCH();
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
  return GEEK_OK;
}

int geek_assign_categorical(const int32_t* codes, uint64_t n, int d, const int32_t* modes, uint64_t k,
                            int64_t* labels, double* best, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(k >= 1 && d >= 1, "cannot assign without centers");
  if (n == 0) return GEEK_OK;
  if (d > 64 || k >= (1ull << 24) || getenv("GEEK_CAT_NAIVE")) {
    assign_cat_kernel<<<grid_for(n, 128), 128, 0, s>>>(codes, n, d, modes, k, labels, best);
    GEEK_CHECK_LAUNCH();
    return GEEK_OK;
  }
  const int DP = (d + 7) / 8 * 8;
  const uint64_t kpad = (k + 255) / 256 * 256;
  Scratch mt;
  GEEK_TRY(mt.alloc((uint64_t)DP * kpad * 4, s));
  modes_transpose_kernel<<<grid_for((uint64_t)DP * kpad, 256), 256, 0, s>>>(modes, k, d, DP, kpad, mt.as<int32_t>());
  GEEK_CHECK_LAUNCH();
  const uint64_t ntiles = (n + 127) / 128;
  const unsigned grid = (unsigned)(ntiles < 148ull * 4 ? ntiles : 148ull * 4);
#define GEEK_CAT(DPV)                                                                                          \
  assign_cat_tiled_kernel<DPV><<<grid, 256, 0, s>>>(codes, n, d, mt.as<int32_t>(), kpad, k, labels, best)
  switch (DP) {
    case 8: GEEK_CAT(8); break;
    case 16: GEEK_CAT(16); break;
    case 24: GEEK_CAT(24); break;
    case 32: GEEK_CAT(32); break;
    case 40: GEEK_CAT(40); break;
    case 48: GEEK_CAT(48); break;
    case 56: GEEK_CAT(56); break;
    default: GEEK_CAT(64); break;
  }
#undef GEEK_CAT
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

int geek_assign_sparse(const uint32_t* flat, const uint64_t* offsets, uint64_t n, uint64_t universe,
                       const int32_t* modes, uint64_t k, int64_t* labels, double* best, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(k >= 1, "cannot assign without centers");
  if (n == 0) return GEEK_OK;
  if (universe <= 1024 && !getenv("GEEK_SPARSE_DENSE")) {
    const int W = (int)((universe + 31) / 32);
    Scratch mb, ms;
    GEEK_TRY(mb.alloc(k * W * 4, s));
    GEEK_TRY(ms.alloc(k * 4, s));
    mode_bits_kernel<<<grid_for(k, 128), 128, 0, s>>>(modes, k, universe, W, mb.as<uint32_t>(), ms.as<uint32_t>());
    GEEK_CHECK_LAUNCH();
    const unsigned grid = grid_for(n, 128, 148 * 8);
#define GEEK_BITS(WMV)                                                                                     \
  assign_sparse_bits_kernel<WMV><<<grid, 128, 0, s>>>(flat, offsets, n, mb.as<uint32_t>(), ms.as<uint32_t>(), k, \
                                                      W, labels, best)
    if (W <= 4) GEEK_BITS(4);
    else if (W <= 8) GEEK_BITS(8);
    else if (W <= 16) GEEK_BITS(16);
    else GEEK_BITS(32);
#undef GEEK_BITS
    GEEK_CHECK_LAUNCH();
    return GEEK_OK;
  }
  Scratch msz;
  GEEK_TRY(msz.alloc(k * 8, s));
  mode_sizes_kernel<<<grid_for(k, 128), 128, 0, s>>>(modes, k, universe, msz.as<double>());
  assign_sparse_kernel<<<grid_for(n, 128), 128, 0, s>>>(flat, offsets, n, universe, modes, msz.as<double>(), k,
                                                        labels, best);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

int geek_mode_counts(const int32_t* codes, uint64_t nrows, int d, uint64_t row_lo, uint64_t cs,
                     const uint32_t* flat, const uint64_t* offsets, uint64_t ngroups, int64_t* counts,
                     void* stream) {
  cudaStream_t s = as_stream(stream);
  if (ngroups == 0) return GEEK_OK;
  uint64_t total = 0;
  GEEK_CHECK_CUDA(cudaMemcpyAsync(&total, offsets + ngroups, 8, cudaMemcpyDeviceToHost, s));
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
  if (total == 0) return GEEK_OK;
  mode_counts_kernel<<<grid_for(total * d, 256), 256, 0, s>>>(codes, nrows, d, row_lo, cs, flat, offsets, ngroups,
                                                              total, reinterpret_cast<unsigned long long*>(counts));
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

int geek_sparse_counts(const uint32_t* set_flat, const uint64_t* set_off, uint64_t nrows, uint64_t row_lo,
                       uint64_t universe, const uint32_t* flat, const uint64_t* offsets, uint64_t ngroups,
                       int64_t* counts, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (ngroups == 0) return GEEK_OK;
  uint64_t total = 0;
  GEEK_CHECK_CUDA(cudaMemcpyAsync(&total, offsets + ngroups, 8, cudaMemcpyDeviceToHost, s));
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));
  if (total == 0) return GEEK_OK;
  sparse_counts_kernel<<<grid_for(total, 256), 256, 0, s>>>(set_flat, set_off, nrows, row_lo, universe, flat,
                                                            offsets, ngroups, total,
                                                            reinterpret_cast<unsigned long long*>(counts));
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

}  // extern "C"
