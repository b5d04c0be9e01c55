// K8: one-pass assignment (assignment.py:44-107).
//
// Euclidean distances are evaluated exactly as numpy does for
// sqrt(((x - c)**2).sum(axis=-1)) on float64: round-to-nearest subtract and
// square (no FMA contraction), numpy's pairwise summation tree (blocks of
// <= 128 with 8 accumulators, recursive halving at multiples of 8), a
// correctly rounded sqrt, and first-index argmin -- so labels, best
// distances and radii are bit-identical to the reference.
#include "common.cuh"

#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>

namespace geek {

// ---- numpy pairwise-sum plan for a row of length d -----------------------
// ops: leaf = (offset << 1) | 0 with length in len[], add = 1 (pop 2, push 1)
struct PwPlan {
  int nops = 0;
  int op[64];
  int off[64];
  int len[64];
};

static void pw_build(PwPlan& p, int off, int n) {
  if (n <= 128) {
    p.op[p.nops] = 0;
    p.off[p.nops] = off;
    p.len[p.nops] = n;
    ++p.nops;
    return;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  pw_build(p, off, n2);
  pw_build(p, off + n2, n - n2);
  p.op[p.nops] = 1;
  p.off[p.nops] = 0;
  p.len[p.nops] = 0;
  ++p.nops;
}

template <class G>
__device__ __forceinline__ double pw_leaf(const G& get, int off, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, get(off + i));
    return r;
  }
  double r0 = get(off), r1 = get(off + 1), r2 = get(off + 2), r3 = get(off + 3);
  double r4 = get(off + 4), r5 = get(off + 5), r6 = get(off + 6), r7 = get(off + 7);
  int i = 8;
  const int lim = n - (n % 8);
  for (; i < lim; i += 8) {
    r0 = __dadd_rn(r0, get(off + i));
    r1 = __dadd_rn(r1, get(off + i + 1));
    r2 = __dadd_rn(r2, get(off + i + 2));
    r3 = __dadd_rn(r3, get(off + i + 3));
    r4 = __dadd_rn(r4, get(off + i + 4));
    r5 = __dadd_rn(r5, get(off + i + 5));
    r6 = __dadd_rn(r6, get(off + i + 6));
    r7 = __dadd_rn(r7, get(off + i + 7));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                         __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
  for (; i < n; ++i) res = __dadd_rn(res, get(off + i));
  return res;
}

template <class G>
__device__ __forceinline__ double pw_sum(const PwPlan& p, const G& get) {
  if (p.nops == 1) return pw_leaf(get, p.off[0], p.len[0]);
  double st[16];
  int sp = 0;
  for (int k = 0; k < p.nops; ++k) {
    if (p.op[k] == 0) {
      st[sp++] = pw_leaf(get, p.off[k], p.len[k]);
    } else {
      double b = st[--sp];
      double a = st[--sp];
      st[sp++] = __dadd_rn(a, b);
    }
  }
  return st[0];
}

// ---- exact Euclidean assignment -----------------------------------------

constexpr int kAsgThreads = 128;
constexpr int kAsgCenters = 16;  // centers staged per shared-memory tile

// n_dev (may be null): the point count lives on the device (the queue of a
// screen); the grid then strides over it
template <class T>
__global__ void __launch_bounds__(kAsgThreads) assign_l2_kernel(const T* __restrict__ X, uint64_t n, int d,
                                                                const double* __restrict__ C, uint64_t k,
                                                                const PwPlan plan, int64_t* labels,
                                                                double* best, const uint32_t* idx,
                                                                const unsigned long long* n_dev = nullptr) {
  extern __shared__ double sC[];  // [kAsgCenters][d]
  if (n_dev) n = *n_dev;
  for (uint64_t base = blockIdx.x * (uint64_t)kAsgThreads; base < n; base += (uint64_t)gridDim.x * kAsgThreads) {
  const uint64_t q = base + threadIdx.x;
  const bool valid = q < n;
  const uint64_t i = (idx && valid) ? idx[q] : q;
  const T* xr = X + (valid ? i : 0) * d;
  double bd = 0.0;
  int64_t bl = -1;
  for (uint64_t c0 = 0; c0 < k; c0 += kAsgCenters) {
    const int nc = (int)(k - c0 < (uint64_t)kAsgCenters ? k - c0 : (uint64_t)kAsgCenters);
    __syncthreads();
    for (int e = threadIdx.x; e < nc * d; e += kAsgThreads) sC[e] = C[c0 * d + e];
    __syncthreads();
    if (!valid) continue;
    for (int c = 0; c < nc; ++c) {
      const double* cr = sC + c * d;
      auto get = [&](int j) {
        const double df = __dsub_rn((double)xr[j], cr[j]);
        return __dmul_rn(df, df);
      };
      const double dist = __dsqrt_rn(pw_sum(plan, get));
      if (bl < 0 || dist < bd) {
        bd = dist;
        bl = (int64_t)(c0 + c);
      }
    }
  }
  if (valid) {
    labels[i] = bl;
    best[i] = bd;
  }
  }
}

// Exact assignment for wide rows (d > 128, where neither screen applies):
// one thread per center, kCtP points of the block in SMEM (as float64), the
// centers transposed (ct[j*kpad + c]) so a warp's center loads coalesce and
// each center value is loaded once for the kCtP points.  Every distance is
// the same float64 pairwise-ordered sum as assign_l2_kernel (same plan,
// same rounding steps); the argmin over centers is a lexicographic
// (distance, index) minimum -- numpy's first-index rule.
constexpr int kCtThreads = 128;
constexpr int kCtP = 4;

// x(p, j): coordinate j of the p-th point as float64 (SMEM tile or global row)
template <int P, class XA>
__device__ __forceinline__ void ct_leaf(const XA& x, const double* __restrict__ ct, uint64_t kpad,
                                        uint64_t c, int off, int n, double (&res)[P]) {
  auto sq = [&](int p, int j, double cj) {
    const double df = __dsub_rn(x(p, j), cj);
    return __dmul_rn(df, df);
  };
  if (n < 8) {
#pragma unroll
    for (int p = 0; p < P; ++p) res[p] = 0.0;
    for (int i = 0; i < n; ++i) {
      const double cj = ct[(uint64_t)(off + i) * kpad + c];
#pragma unroll
      for (int p = 0; p < P; ++p) res[p] = __dadd_rn(res[p], sq(p, off + i, cj));
    }
    return;
  }
  double r[P][8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const double cj = ct[(uint64_t)(off + u) * kpad + c];
#pragma unroll
    for (int p = 0; p < P; ++p) r[p][u] = sq(p, off + u, cj);
  }
  int i = 8;
  const int lim = n - (n % 8);
  for (; i < lim; i += 8) {
    double cj[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) cj[u] = ct[(uint64_t)(off + i + u) * kpad + c];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int p = 0; p < P; ++p) r[p][u] = __dadd_rn(r[p][u], sq(p, off + i + u, cj[u]));
  }
#pragma unroll
  for (int p = 0; p < P; ++p)
    res[p] = __dadd_rn(__dadd_rn(__dadd_rn(r[p][0], r[p][1]), __dadd_rn(r[p][2], r[p][3])),
                       __dadd_rn(__dadd_rn(r[p][4], r[p][5]), __dadd_rn(r[p][6], r[p][7])));
  for (; i < n; ++i) {
    const double cj = ct[(uint64_t)(off + i) * kpad + c];
#pragma unroll
    for (int p = 0; p < P; ++p) res[p] = __dadd_rn(res[p], sq(p, off + i, cj));
  }
}

template <class T>
__global__ void __launch_bounds__(kCtThreads) assign_l2_ct_kernel(const T* __restrict__ X, uint64_t n, int d,
                                                                  const double* __restrict__ ct, uint64_t k,
                                                                  uint64_t kpad, const PwPlan plan,
                                                                  int64_t* labels, double* best) {
  extern __shared__ double xs[];  // [kCtP][d]
  __shared__ double wd[kCtP][kCtThreads / 32];
  __shared__ long long wl[kCtP][kCtThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t p0 = (uint64_t)blockIdx.x * kCtP; p0 < n; p0 += (uint64_t)gridDim.x * kCtP) {
    const int np = (int)min((uint64_t)kCtP, n - p0);
    __syncthreads();
    for (int e = threadIdx.x; e < kCtP * d; e += kCtThreads) {
      const int p = e / d;
      xs[e] = p < np ? (double)X[(p0 + p) * d + (e - p * d)] : 0.0;
    }
    __syncthreads();
    double bd[kCtP];
    long long bl[kCtP];
#pragma unroll
    for (int p = 0; p < kCtP; ++p) {
      bd[p] = 0.0;
      bl[p] = -1;
    }
    for (uint64_t c = threadIdx.x; c < kpad; c += kCtThreads) {
      const bool cv = c < k;
      const uint64_t cc = cv ? c : 0;
      double st[6][kCtP];
      int sp = 0;
      for (int o = 0; o < plan.nops; ++o) {
        if (plan.op[o] == 0) {
          double r[kCtP];
          ct_leaf<kCtP>([&](int p, int j) { return xs[p * d + j]; }, ct, kpad, cc, plan.off[o], plan.len[o], r);
#pragma unroll
          for (int p = 0; p < kCtP; ++p) st[sp][p] = r[p];
          ++sp;
        } else {
#pragma unroll
          for (int p = 0; p < kCtP; ++p) st[sp - 2][p] = __dadd_rn(st[sp - 2][p], st[sp - 1][p]);
          --sp;
        }
      }
      if (!cv) continue;
#pragma unroll
      for (int p = 0; p < kCtP; ++p) {
        const double dist = __dsqrt_rn(st[0][p]);
        if (bl[p] < 0 || dist < bd[p]) {  // c ascends per thread: first index kept on ties
          bd[p] = dist;
          bl[p] = (long long)c;
        }
      }
    }
    // lexicographic (distance, index) minimum over the block
#pragma unroll
    for (int p = 0; p < kCtP; ++p) {
      double d0 = bd[p];
      long long l0 = bl[p];
      for (int o = 16; o; o >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, d0, o);
        const long long ol = __shfl_xor_sync(0xffffffffu, l0, o);
        if (ol >= 0 && (l0 < 0 || od < d0 || (od == d0 && ol < l0))) {
          d0 = od;
          l0 = ol;
        }
      }
      if (lane == 0) {
        wd[p][warp] = d0;
        wl[p][warp] = l0;
      }
    }
    __syncthreads();
    if (threadIdx.x < np) {
      const int p = threadIdx.x;
      double d0 = wd[p][0];
      long long l0 = wl[p][0];
      for (int w = 1; w < kCtThreads / 32; ++w) {
        const double od = wd[p][w];
        const long long ol = wl[p][w];
        if (ol >= 0 && (l0 < 0 || od < d0 || (od == d0 && ol < l0))) {
          d0 = od;
          l0 = ol;
        }
      }
      labels[p0 + p] = l0;
      best[p0 + p] = d0;
    }
  }
}

// Small k (<= 32): a warp holds 32/S segments of S = pow2 >= k lanes, lane
// l of a segment evaluates center l for the segment's kCtP points, read
// straight from their global rows (one address per segment per load).
template <class T>
__global__ void __launch_bounds__(kCtThreads) assign_l2_ctk_kernel(const T* __restrict__ X, uint64_t n, int d,
                                                                   const double* __restrict__ ct, uint64_t k,
                                                                   uint64_t kpad, int S, const PwPlan plan,
                                                                   int64_t* labels, double* best) {
  const int l = threadIdx.x & (S - 1);
  const uint64_t gt = blockIdx.x * (uint64_t)kCtThreads + threadIdx.x;
  const uint64_t wseg0 = (gt >> 5) * (32 / S);  // first segment of this warp
  const uint64_t nseg = (uint64_t)gridDim.x * kCtThreads / S;
  const bool cv = (uint64_t)l < k;
  const uint64_t cc = cv ? l : 0;
  // the loop bound is warp-uniform (the shuffles below need every lane);
  // segments past the end compute on clamped rows and write nothing
  for (uint64_t base = wseg0 * kCtP; base < n; base += nseg * kCtP) {
    const uint64_t p0 = base + (uint64_t)((threadIdx.x & 31) / S) * kCtP;
    const T* xr[kCtP];
#pragma unroll
    for (int p = 0; p < kCtP; ++p) xr[p] = X + min(p0 + p, n - 1) * d;
    double st[6][kCtP];
    int sp = 0;
    for (int o = 0; o < plan.nops; ++o) {
      if (plan.op[o] == 0) {
        double r[kCtP];
        ct_leaf<kCtP>([&](int p, int j) { return (double)xr[p][j]; }, ct, kpad, cc, plan.off[o], plan.len[o], r);
#pragma unroll
        for (int p = 0; p < kCtP; ++p) st[sp][p] = r[p];
        ++sp;
      } else {
#pragma unroll
        for (int p = 0; p < kCtP; ++p) st[sp - 2][p] = __dadd_rn(st[sp - 2][p], st[sp - 1][p]);
        --sp;
      }
    }
#pragma unroll
    for (int p = 0; p < kCtP; ++p) {
      double d0 = __dsqrt_rn(st[0][p]);
      long long l0 = cv ? (long long)l : -1;
      for (int o = 1; o < S; o <<= 1) {  // lexicographic (distance, index) minimum in the segment
        const double od = __shfl_xor_sync(0xffffffffu, d0, o);
        const long long ol = __shfl_xor_sync(0xffffffffu, l0, o);
        if (ol >= 0 && (l0 < 0 || od < d0 || (od == d0 && ol < l0))) {
          d0 = od;
          l0 = ol;
        }
      }
      if (l == 0 && p0 + p < n) {
        labels[p0 + p] = l0;
        best[p0 + p] = d0;
      }
    }
  }
}

__global__ void transpose_centers_kernel(const double* C, uint64_t k, int d, uint64_t kpad, double* ct) {
  const uint64_t total = (uint64_t)d * kpad;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = e / kpad, c = e - j * kpad;
    ct[e] = c < k ? C[c * d + j] : 0.0;
  }
}

// Exact argmin for the few points whose screen window overflowed: one block
// per point, threads over centers (first index wins ties, as np.argmin).
constexpr int kFsThreads = 256;
__global__ void __launch_bounds__(kFsThreads) full_scan_kernel(const float* __restrict__ X, int d,
                                                               const double* __restrict__ C, uint64_t k,
                                                               const PwPlan plan, const uint32_t* idx,
                                                               const unsigned long long* nidx, int64_t* labels,
                                                               double* best) {
  extern __shared__ double sx[];  // [d]
  __shared__ double rd[kFsThreads / 32];
  __shared__ long long rl[kFsThreads / 32];
  const uint64_t nq = *nidx;
  for (uint64_t q = blockIdx.x; q < nq; q += gridDim.x) {
  const uint64_t i = idx[q];
  __syncthreads();  // the previous point's reads of sx / rd / rl are done
  for (int j = threadIdx.x; j < d; j += kFsThreads) sx[j] = (double)X[i * d + j];
  __syncthreads();
  double bd = INFINITY;
  long long bl = -1;
  for (uint64_t c = threadIdx.x; c < k; c += kFsThreads) {
    const double* cr = C + c * d;
    const double dist = __dsqrt_rn(pw_sum(plan, [&](int j) {
      const double df = __dsub_rn(sx[j], cr[j]);
      return __dmul_rn(df, df);
    }));
    if (bl < 0 || dist < bd) {
      bd = dist;
      bl = (long long)c;
    }
  }
  // lexicographic (dist, index) minimum over the block
  for (int o = 16; o; o >>= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, bd, o);
    const long long ol = __shfl_xor_sync(0xffffffffu, bl, o);
    if (ol >= 0 && (bl < 0 || od < bd || (od == bd && ol < bl))) {
      bd = od;
      bl = ol;
    }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    rd[w] = bd;
    rl[w] = bl;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int v = 1; v < kFsThreads / 32; ++v)
      if (rl[v] >= 0 && (bl < 0 || rd[v] < bd || (rd[v] == bd && rl[v] < bl))) {
        bd = rd[v];
        bl = rl[v];
      }
    labels[i] = bl;
    best[i] = bd;
  }
  }
}

__global__ void radii_sizes_kernel(const int64_t* labels, const double* best, uint64_t n, double* radii,
                                   int64_t* sizes) {
  // warp-aggregated: ids are cluster-contiguous, so a warp mostly shares a label
  const unsigned lane = threadIdx.x & 31;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u); base < n;
       base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = base + lane;
    const bool valid = i < n;
    const long long l = valid ? labels[i] : -1ll - lane;
    // best >= 0, so its bit pattern orders like the value
    unsigned long long bits = valid ? (unsigned long long)__double_as_longlong(best[i]) : 0ull;
    const unsigned peers = __match_any_sync(0xffffffffu, l);
    // 64-bit max over the peer group as (hi, lo) lexicographic 32-bit maxima
    const unsigned hi = (unsigned)(bits >> 32), lo = (unsigned)bits;
    const unsigned mhi = __reduce_max_sync(peers, hi);
    const unsigned mlo = __reduce_max_sync(peers, hi == mhi ? lo : 0u);
    const unsigned long long mx = ((unsigned long long)mhi << 32) | mlo;
    const int leader = __ffs(peers) - 1;
    if (valid && (int)lane == leader) {
      atomicMax(reinterpret_cast<unsigned long long*>(radii) + l, mx);
      atomicAdd(reinterpret_cast<unsigned long long*>(sizes) + l, (unsigned long long)__popc(peers));
    }
  }
}

// ---- numpy pairwise sum over a long vector (the objective) ---------------

struct SumTree {
  // leaves in tree order; internal nodes per level (deepest first)
  std::vector<uint64_t> leaf_off;
  std::vector<uint32_t> leaf_len;
  std::vector<uint32_t> leaf_node;
  std::vector<std::vector<uint32_t>> lv_node, lv_left, lv_right;
  uint32_t nnodes = 0;
};

struct Node {
  uint64_t off, n;
  int depth;
  uint32_t id;
};

static std::shared_ptr<SumTree> make_tree(uint64_t n) {
  auto t = std::make_shared<SumTree>();
  // breadth-first expansion; node ids assigned in BFS order
  std::vector<Node> cur{{0, n, 0, 0}};
  t->nnodes = 1;
  std::vector<std::vector<uint32_t>> lvn, lvl, lvr;
  while (!cur.empty()) {
    std::vector<Node> nxt;
    std::vector<uint32_t> ln, ll, lr;
    for (const Node& nd : cur) {
      if (nd.n <= 128) {
        t->leaf_off.push_back(nd.off);
        t->leaf_len.push_back((uint32_t)nd.n);
        t->leaf_node.push_back(nd.id);
        continue;
      }
      uint64_t n2 = nd.n / 2;
      n2 -= n2 % 8;
      Node a{nd.off, n2, nd.depth + 1, t->nnodes++};
      Node b{nd.off + n2, nd.n - n2, nd.depth + 1, t->nnodes++};
      ln.push_back(nd.id);
      ll.push_back(a.id);
      lr.push_back(b.id);
      nxt.push_back(a);
      nxt.push_back(b);
    }
    if (!ln.empty()) {
      lvn.push_back(ln);
      lvl.push_back(ll);
      lvr.push_back(lr);
    }
    cur.swap(nxt);
  }
  // combine deepest internal level first
  for (int i = (int)lvn.size() - 1; i >= 0; --i) {
    t->lv_node.push_back(lvn[i]);
    t->lv_left.push_back(lvl[i]);
    t->lv_right.push_back(lvr[i]);
  }
  return t;
}

__global__ void leaf_sum_kernel(const double* v, const uint64_t* off, const uint32_t* len, const uint32_t* node,
                                uint64_t nleaf, double* val) {
  for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < nleaf;
       l += (uint64_t)gridDim.x * blockDim.x) {
    const double* a = v + off[l];
    auto get = [&](int j) { return a[j]; };
    val[node[l]] = pw_leaf(get, 0, (int)len[l]);
  }
}

__global__ void combine_kernel(const uint32_t* node, const uint32_t* left, const uint32_t* right, uint64_t cnt,
                               double* val) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < cnt;
       q += (uint64_t)gridDim.x * blockDim.x)
    val[node[q]] = __dadd_rn(val[left[q]], val[right[q]]);
}

// device copy of a SumTree's index arrays (leaves; per level node/left/right)
struct DevSumTree {
  uint64_t* leaf_off = nullptr;
  uint32_t* leaf_len = nullptr;
  uint32_t* leaf_node = nullptr;
  uint32_t* lv = nullptr;
  std::vector<uint64_t> lv_count;
  uint64_t nleaf = 0;
  uint32_t nnodes = 0;
  void* mem = nullptr;
  DevSumTree() = default;
  DevSumTree(const DevSumTree&) = delete;
  DevSumTree& operator=(const DevSumTree&) = delete;
  ~DevSumTree() {
    if (mem) cudaFree(mem);
  }
  int build(const SumTree& t) {
    nleaf = t.leaf_off.size();
    nnodes = t.nnodes;
    uint64_t ninternal = 0;
    for (auto& l : t.lv_node) {
      lv_count.push_back(l.size());
      ninternal += l.size();
    }
    const uint64_t bytes = nleaf * 16 + ninternal * 12 + 16;
    GEEK_CHECK_CUDA(cudaMalloc(&mem, bytes));
    leaf_off = static_cast<uint64_t*>(mem);
    leaf_len = reinterpret_cast<uint32_t*>(leaf_off + nleaf);
    leaf_node = leaf_len + nleaf;
    lv = leaf_node + nleaf;
    GEEK_CHECK_CUDA(cudaMemcpy(leaf_off, t.leaf_off.data(), nleaf * 8, cudaMemcpyHostToDevice));
    GEEK_CHECK_CUDA(cudaMemcpy(leaf_len, t.leaf_len.data(), nleaf * 4, cudaMemcpyHostToDevice));
    GEEK_CHECK_CUDA(cudaMemcpy(leaf_node, t.leaf_node.data(), nleaf * 4, cudaMemcpyHostToDevice));
    uint32_t* p = lv;
    for (size_t L = 0; L < t.lv_node.size(); ++L) {
      const uint64_t c = t.lv_node[L].size();
      GEEK_CHECK_CUDA(cudaMemcpy(p, t.lv_node[L].data(), c * 4, cudaMemcpyHostToDevice));
      GEEK_CHECK_CUDA(cudaMemcpy(p + c, t.lv_left[L].data(), c * 4, cudaMemcpyHostToDevice));
      GEEK_CHECK_CUDA(cudaMemcpy(p + 2 * c, t.lv_right[L].data(), c * 4, cudaMemcpyHostToDevice));
      p += 3 * c;
    }
    return GEEK_OK;
  }
};

// ---- screened assignment (float32 data) -----------------------------------
//
// screen: s(x, c) = |c|^2 - 2 x.c in float32 (SIMT register-blocked GEMM,
// 128 points x 128 centers per tile, 8x8 per thread) with a running top-2
// per point.  |s - S| <= E(x) for the exact S = |c|^2 - 2 x.c (rounding of
// c to float32, the dot product, |c|^2 and the subtraction, bounded with
// |x| |c| by Cauchy-Schwarz).  When s2 - s1 > T(x) = 2E + 2E64 + margin the
// exact float64 (numpy-order) distances have the same strict argmin, so the
// label is final and only best = dist(x, c_label) is evaluated exactly;
// otherwise the point is re-scanned exactly over all centers.

// effective screen mode of a call: an FP16 screen whose scaled operand left the
// f16 range was redone in TF32x3 (the fallback launch ran when *ovf != 0)
// an f16 overflow: the FP16 tcgen05 screens were redone in TF32x3 (mode 3);
// the wide-row FP16x3 screen (65) has no redo -- mode 0 sends every point to
// the exact full scan
__device__ __forceinline__ int eff_mode(int nprod, const unsigned* ovf) {
  return (ovf && *ovf) ? (nprod >= 65 ? 0 : 3) : nprod;
}

constexpr int kScrP = 128, kScrC = 128, kScrK = 16, kScrThreads = 256;

__global__ void center_prep_kernel(const double* C, uint64_t k, int d, float* Cf, float* c2f,
                                   unsigned long long* cmax_bits) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < k; c += (uint64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) {
      const double v = C[c * d + j];
      Cf[c * d + j] = (float)v;
      s = fma(v, v, s);
    }
    c2f[c] = (float)s;
    atomicMax(cmax_bits, (unsigned long long)__double_as_longlong(sqrt(s) * (1.0 + 1e-12)));
  }
}

__global__ void __launch_bounds__(kScrThreads, 2) screen_kernel(const float* __restrict__ X, uint64_t n, int d,
                                                                 const float* __restrict__ Cf,
                                                                 const float* __restrict__ c2f,
                                                                 const double* __restrict__ C, uint64_t k,
                                                                 const unsigned long long* cmax_bits,
                                                                 const PwPlan plan, int64_t* labels, double* best,
                                                                 uint32_t* amb, unsigned long long* namb) {
  extern __shared__ float smem[];
  const int xs_ld = kScrP + 4;
  float* Xs = smem;                                 // [d][xs_ld]
  float* Cs = Xs + (size_t)d * xs_ld;               // [kScrK][kScrC + 4]
  float* rs1 = Cs + kScrK * (kScrC + 4);            // [kScrP] merged top-2
  float* rs2 = rs1 + kScrP;
  int* ri1 = reinterpret_cast<int*>(rs2 + kScrP);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const uint64_t p0 = blockIdx.x * (uint64_t)kScrP;
  for (int e = threadIdx.x; e < kScrP * d; e += kScrThreads) {
    const int p = e / d, j = e - p * d;
    Xs[j * xs_ld + p] = (p0 + p < n) ? X[(p0 + p) * d + j] : 0.f;
  }
  float s1[8], s2[8];
  int i1[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    s1[a] = INFINITY;
    s2[a] = INFINITY;
    i1[a] = -1;
  }
  for (uint64_t c0 = 0; c0 < k; c0 += kScrC) {
    float acc[8][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[a][b] = 0.f;
    for (int k0 = 0; k0 < d; k0 += kScrK) {
      __syncthreads();
      for (int e = threadIdx.x; e < kScrC * kScrK; e += kScrThreads) {
        const int c = e / kScrK, kk = e - c * kScrK;
        Cs[kk * (kScrC + 4) + c] = (c0 + c < k && k0 + kk < d) ? Cf[(c0 + c) * d + k0 + kk] : 0.f;
      }
      __syncthreads();
      const int kn = min(kScrK, d - k0);
      for (int kk = 0; kk < kn; ++kk) {
        const float4 xa = *reinterpret_cast<const float4*>(Xs + (k0 + kk) * xs_ld + ty * 8);
        const float4 xb = *reinterpret_cast<const float4*>(Xs + (k0 + kk) * xs_ld + ty * 8 + 4);
        const float4 ca = *reinterpret_cast<const float4*>(Cs + kk * (kScrC + 4) + tx * 8);
        const float4 cb = *reinterpret_cast<const float4*>(Cs + kk * (kScrC + 4) + tx * 8 + 4);
        const float xv[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
        const float cv[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b < 8; ++b) acc[a][b] = fmaf(xv[a], cv[b], acc[a][b]);
      }
    }
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const uint64_t c = c0 + tx * 8 + b;
      if (c >= k) break;
      const float cc = c2f[c];
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const float sv = cc - 2.f * acc[a][b];
        if (sv < s1[a]) {
          s2[a] = s1[a];
          s1[a] = sv;
          i1[a] = (int)c;
        } else if (sv < s2[a]) {
          s2[a] = sv;
        }
      }
    }
  }
  // merge the 16 column groups (lanes tx within a half warp)
#pragma unroll
  for (int a = 0; a < 8; ++a) {
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const float os1 = __shfl_xor_sync(0xffffffffu, s1[a], o);
      const float os2 = __shfl_xor_sync(0xffffffffu, s2[a], o);
      const int oi1 = __shfl_xor_sync(0xffffffffu, i1[a], o);
      const float lo = fminf(s1[a], os1), hi = fmaxf(s1[a], os1);
      const bool take = os1 < s1[a] || (os1 == s1[a] && oi1 < i1[a] && oi1 >= 0);
      s2[a] = fminf(hi, fminf(s2[a], os2));
      if (take) i1[a] = oi1;
      s1[a] = lo;
    }
    if (tx == 0) {
      rs1[ty * 8 + a] = s1[a];
      rs2[ty * 8 + a] = s2[a];
      ri1[ty * 8 + a] = i1[a];
    }
  }
  __syncthreads();
  if (threadIdx.x < kScrP) {
    const int p = threadIdx.x;
    const uint64_t i = p0 + p;
    if (i < n) {
      double xn2 = 0.0;
      for (int j = 0; j < d; ++j) {
        const double v = Xs[j * xs_ld + p];
        xn2 = fma(v, v, xn2);
      }
      const double xn = sqrt(xn2) * (1.0 + 1e-12);
      const double cn = __longlong_as_double((long long)*cmax_bits);
      const double u = 5.9604644775390625e-08;  // 2^-24
      const double E = 1.01 * (2.0 * d + 10.0) * u * (xn * cn + cn * cn);
      const double E64 = 1.01 * (d + 4.0) * 1.1102230246251565e-16 * (xn + cn) * (xn + cn);
      const double T = 2.0 * E + 2.0 * E64 + 9.094947017729282e-13 * (xn + cn) * (xn + cn);
      const int lab = ri1[p];
      const bool certain = lab >= 0 && (k == 1 || (double)rs2[p] - (double)rs1[p] > T);
      if (certain) {
        const double* cr = C + (uint64_t)lab * d;
        auto get = [&](int j) {
          const double df = __dsub_rn((double)Xs[j * xs_ld + p], cr[j]);
          return __dmul_rn(df, df);
        };
        labels[i] = lab;
        best[i] = __dsqrt_rn(pw_sum(plan, get));
      } else {
        const unsigned long long q = atomicAdd(namb, 1ull);
        amb[q] = (uint32_t)i;
      }
    }
  }
}

// ---- tensor-core screen: classification and candidate recheck ----------------

// SWIZZLE_NONE K-major canonical layout strides (bytes): K-adjacent / M,N-adjacent core matrices
constexpr uint32_t kTcLBO = 128, kTcSBO = 256;

template <class G>
__device__ __forceinline__ double exact_dist(const PwPlan& plan, const G& get) {
  return __dsqrt_rn(pw_sum(plan, get));
}

// Bound T(x) on the separation the screen must show before its winner is
// final.  E bounds |s - S| (S = |c-mu|^2 - 2(x-mu).(c-mu) in exact arithmetic):
//   nprod 3: float32 operand rounding, hi/lo split residuals and the dropped
//            lo*lo term, fp32 accumulation of 3d products, |c'|^2 rounding and
//            the final subtraction;
//   nprod 1: float32 operand rounding, TF32 rounding of both operands
//            (2^-11 relative each), fp32 accumulation of d products, |c'|^2
//            rounding and the subtraction;
//   nprod 16 (FP16x3 over s x', s c', s a power of two): the nprod 3 terms
//            (f16 and tf32 share the 11-bit significand) plus the absolute
//            error of f16 subnormals, at most 2^-25 per scaled coordinate:
//            2^-25 sqrt(d) (|x'| + |c'|) / s, and the three f16 parts of
//            s^2 |c'|^2 / 2 (3 * 2^-25 / s^2 + 2^-33 |c'|^2 / 2).
//   nprod 65 (wide rows, FP16x3 as one cuBLAS GEMM over K = 3d: [xh xh xl] .
//            [ch cl ch] of s x', s c', fp32 accumulation in any order): the
//            nprod 16 terms with 3d accumulated products; |c'|^2 enters in
//            float64 and s is rounded once to float32 (both inside 4u cn^2 +
//            10u xn cn).
//   nprod 66 (nprod 65 over x'' = fl32(x' - c'_j0), j0 the row tile's origin
//            center, xn = |x''|): s = E[j0][j] - 2 x''.c'_j with the float64
//            table E[j0][j] = |c'_j|^2 - 2 c'_j0.c'_j (equal to s(x, c_j) up to a
//            per-point constant and the x'' rounding, 2u |x''||c'|), rounded once
//            to float32 (|s| <= 3 cn^2 + 2 xn cn).
//   nprod 64 (wide rows, float64 cuBLAS GEMM over uncentered x, c; xn = |x|,
//            cn = max |c|): gamma_{d+2} for the dot products and |c|^2, plus
//            the float32 rounding of the stored s = |c|^2 - 2 x.c.
//   nprod 17 (tile-local FP16, xn = |x''| = |x' - c'_j0|): one f16 product
//            of s x'' and s c' (2^-11 relative each, as nprod 1), fp32
//            accumulation of d products, f16 subnormals as nprod 16, and the
//            float64 table E[j0][j] (|E| <= 3|c'|^2) rounded to float32 and
//            added in float32; the float32 rounding of x' = fl(x - mu),
//            |x'| <= |x''| + |c'|, and of x'' itself.
// cmax_bits[0] = |c'|max, cmax_bits[3] = 1/s (FP16 only, else 0).
// Every product is bounded through sum |x'_i||c'_i| <= |x'||c'| (Cauchy-Schwarz).
// E64 bounds numpy's float64 evaluation of the squared distance, and the last
// term keeps the correctly rounded square roots of the two best distinct.
__device__ __forceinline__ double tc_threshold(double xn, double cn, int d, int nprod,
                                               const unsigned long long* cmax_bits) {
  if (nprod == 0) return INFINITY;  // no valid screen: every point is scanned exactly
  const double u = 5.9604644775390625e-08;  // 2^-24
  // fp32 accumulation of d products (the wide FP16x3 GEMM accumulates 3d)
  const double acc = (nprod == 65 || nprod == 66 ? 3.0 : 1.0) * (double)d * 1.1920928955078125e-07;  // d * 2^-23
  // (|c'|^2/2 enters the fp32 accumulation as a last K=8 slice: one more
  // rounding of the accumulator, 2u(xn cn + cn^2) in s units, on top)
  double E = nprod != 1 ? 1.05 * ((1.9073486328125e-06 + 6.0 * acc + 10.0 * u) * xn * cn + 4.0 * u * cn * cn)
                        : 1.05 * ((1.953125e-03 + 2.0 * acc + 8.0 * u) * xn * cn + 5.0 * u * cn * cn);
  if (nprod == 66)  // the E table enters in float64, s = E - 2 x''.c' rounded once (|s| <= 3 cn^2 + 2 xn cn)
    E = 1.05 * ((1.9073486328125e-06 + 6.0 * acc + 10.0 * u) * xn * cn + 12.0 * u * cn * cn);
  if (nprod == 16 || nprod == 65 || nprod == 66) {
    const double is = __longlong_as_double((long long)cmax_bits[3]);
    const double t25 = 2.9802322387695312e-08;  // 2^-25
    E += 1.05 * (t25 * sqrt((double)d) * (xn + cn) * is + 3.0 * t25 * is * is + 1.1641532182693481e-10 * 0.5 * cn * cn);
  }
  if (nprod == 64) {  // float64 GEMM screen of wide rows (x, c uncentered: mu = 0), s stored as float32
    const double g = (d + 2.0) * 1.1102230246251565e-16;
    E = 1.05 * (2.0 * g * xn * cn + g * cn * cn + u * (cn * cn + 2.0 * xn * cn));
  }
  if (nprod == 17) {
    const double is = __longlong_as_double((long long)cmax_bits[3]);
    const double t25 = 2.9802322387695312e-08;  // 2^-25
    E = 1.05 * ((1.953125e-03 + 2.0 * acc + 10.0 * u) * xn * cn + 12.0 * u * cn * cn + 4.0 * u * (xn + cn) * cn +
                t25 * sqrt((double)d) * (xn + cn) * is);
  }
  // |x - c| <= |x'| + |c'|, and with an origin (xn = |x''|) <= |x''| + 2 |c'|max
  const double xc = (nprod == 17 || nprod == 66) ? xn + 2.0 * cn : xn + cn;
  const double E64 = 1.01 * (d + 4.0) * 1.1102230246251565e-16 * xc * xc;
  return 2.0 * E + 2.0 * E64 + 9.094947017729282e-13 * xc * xc;
}

// The screen keeps the top-4 of each accumulator column half ([8] per point).
// Their union holds the true best and second best; every center within the
// window s0 + T is among them unless a half's 4th entry is itself inside the
// window (overflow -> exact scan over all centers).
struct ScreenView {
  float s0, s1;
  int i0;
  float s3a, s3b;
};

__device__ __forceinline__ ScreenView screen_view(const float* s8, const int* i8) {
  ScreenView v;
  v.s0 = INFINITY;
  v.s1 = INFINITY;
  v.i0 = -1;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const float x = s8[a];
    if (x < v.s0) {
      v.s1 = v.s0;
      v.s0 = x;
      v.i0 = i8[a];
    } else if (x < v.s1) {
      v.s1 = x;
    }
  }
  v.s3a = s8[3];
  v.s3b = s8[7];
  return v;
}

// certain points: label + exact best; others: queued with their candidates
__global__ void tc_classify_kernel(const float* __restrict__ X, uint64_t n, int d, const double* __restrict__ C,
                                   uint64_t k, const PwPlan plan, const float* top_s, const int* top_i,
                                   float* xnorm, const float* mu, const unsigned long long* cmax_bits, int nprod,
                                   const unsigned* ovf, int64_t* labels, double* best, uint32_t* amb,
                                   unsigned long long* namb, uint32_t* full, unsigned long long* nfull,
                                   const double* xn2_in) {
  const double cn = __longlong_as_double((long long)*cmax_bits);
  nprod = eff_mode(nprod, ovf);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const ScreenView v = screen_view(top_s + i * 8, top_i + i * 8);
    double xn2 = 0.0;  // |x'|, x' = fl32(x - mu) exactly as the screen's operand (or the screen's |x''|^2)
    if (xn2_in) {
      xn2 = xn2_in[i];
    } else {
      for (int j = 0; j < d; ++j) {
        const double xv = (double)(X[i * d + j] - mu[j]);
        xn2 = fma(xv, xv, xn2);
      }
    }
    const float xn = (float)(sqrt(xn2) * (1.0 + 1e-6));
    xnorm[i] = xn;
    const double T = tc_threshold((double)xn, cn, d, nprod, cmax_bits);
    const double s0 = v.s0;
    const bool nos = nprod == 0;  // no valid screen (an f16 overflow of the wide FP16x3 GEMM)
    if (!nos && v.i0 >= 0 && (k == 1 || (double)v.s1 - s0 > T)) {
      const int lab = v.i0;
      const float* xr = X + i * d;
      const double* cr = C + (uint64_t)lab * d;
      labels[i] = lab;
      best[i] = exact_dist(plan, [&](int j) {
        const double df = __dsub_rn((double)xr[j], cr[j]);
        return __dmul_rn(df, df);
      });
    } else if (nos || v.i0 < 0 || (double)v.s3a - s0 <= T || (double)v.s3b - s0 <= T) {
      full[atomicAdd(nfull, 1ull)] = (uint32_t)i;  // candidate window overflows the kept lists
    } else {
      amb[atomicAdd(namb, 1ull)] = (uint32_t)i;
    }
  }
}

// Same classification with 8 lanes per point for 8 <= d <= 128: lane a owns
// numpy's accumulator r[a] (elements a, a+8, ...), so row loads are coalesced
// and the summation order is exactly pw_leaf's.
__global__ void tc_classify8_kernel(const float* __restrict__ X, uint64_t n, int d, const double* __restrict__ C,
                                    uint64_t k, const float* top_s, const int* top_i, float* xnorm,
                                    const float* mu, const unsigned long long* cmax_bits, int nprod,
                                    const unsigned* ovf, int64_t* labels, double* best, uint32_t* amb,
                                    unsigned long long* namb, uint32_t* full, unsigned long long* nfull) {
  const double cn = __longlong_as_double((long long)*cmax_bits);
  nprod = eff_mode(nprod, ovf);
  const unsigned lane = threadIdx.x & 31, a = lane & 7;
  const unsigned gmask = 0xFFu << (lane & 24);
  const uint64_t stride = ((uint64_t)gridDim.x * blockDim.x) >> 3;
  const int lim = d - (d % 8);
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 3; i < n; i += stride) {
    const ScreenView v = screen_view(top_s + i * 8, top_i + i * 8);
    double xn2 = 0.0;  // |x'|, x' = fl32(x - mu) exactly as the screen's operand
    for (int e = (int)a; e < d; e += 8) {
      const double xv = (double)(X[i * d + e] - mu[e]);
      xn2 = fma(xv, xv, xn2);
    }
    xn2 += __shfl_xor_sync(gmask, xn2, 1);
    xn2 += __shfl_xor_sync(gmask, xn2, 2);
    xn2 += __shfl_xor_sync(gmask, xn2, 4);
    const float xn = (float)(sqrt(xn2) * (1.0 + 1e-6));
    if (a == 0) xnorm[i] = xn;
    const double T = tc_threshold((double)xn, cn, d, nprod, cmax_bits);
    const double s0 = v.s0;
    const bool certain = v.i0 >= 0 && (k == 1 || (double)v.s1 - s0 > T);
    if (certain) {
      const int lab = v.i0;
      const float* xr = X + i * d;
      const double* cr = C + (uint64_t)lab * d;
      double r;
      {
        const double df = __dsub_rn((double)xr[a], cr[a]);
        r = __dmul_rn(df, df);
      }
      for (int e = 8 + (int)a; e < lim; e += 8) {
        const double df = __dsub_rn((double)xr[e], cr[e]);
        r = __dadd_rn(r, __dmul_rn(df, df));
      }
      // ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7))
      const double p1 = __dadd_rn(r, __shfl_xor_sync(gmask, r, 1));
      const double p2 = __dadd_rn(p1, __shfl_xor_sync(gmask, p1, 2));
      const double p4 = __dadd_rn(p2, __shfl_xor_sync(gmask, p2, 4));
      if (a == 0) {
        // lane 0 holds ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)): xor-butterfly adds
        // (r0+r1), then with (r2+r3), then with the upper half -- same tree
        double res = p4;
        for (int e = lim; e < d; ++e) {
          const double df = __dsub_rn((double)xr[e], cr[e]);
          res = __dadd_rn(res, __dmul_rn(df, df));
        }
        labels[i] = lab;
        best[i] = __dsqrt_rn(res);
      }
    } else if (a == 0) {
      if (v.i0 < 0 || (double)v.s3a - s0 <= T || (double)v.s3b - s0 <= T) full[atomicAdd(nfull, 1ull)] = (uint32_t)i;
      else amb[atomicAdd(namb, 1ull)] = (uint32_t)i;
    }
  }
}

// tc_classify8_kernel with 2 lanes per point and 16-byte loads (d % 8 == 0,
// 8 <= d <= 128): lane h keeps numpy's accumulators r[4h..4h+3] (elements
// e with e % 8 in [4h, 4h+4)), forms (r[4h]+r[4h+1]) + (r[4h+2]+r[4h+3])
// locally and one xor-shuffle adds the other half: numpy's pairwise tree.
__global__ void __launch_bounds__(256) tc_classify2_kernel(
    const float* __restrict__ X, uint64_t n, int d, const double* __restrict__ C, uint64_t k,
    const float* __restrict__ top_s, const int* __restrict__ top_i, float* xnorm, const float* __restrict__ mu,
    const double* __restrict__ xpart, const unsigned long long* cmax_bits, int nprod, const unsigned* ovf,
    int64_t* labels, double* best, uint32_t* amb, unsigned long long* namb, uint32_t* full, unsigned long long* nfull) {
  const double cn = __longlong_as_double((long long)*cmax_bits);
  nprod = eff_mode(nprod, ovf);
  const unsigned lane = threadIdx.x & 31, h = lane & 1;
  const unsigned pmask = 3u << (lane & 30);
  const uint64_t stride = ((uint64_t)gridDim.x * blockDim.x) >> 1;
  const int nu = d / 8;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 1; i < n; i += stride) {
    const ScreenView v = screen_view(top_s + i * 8, top_i + i * 8);
    const float4* xr = reinterpret_cast<const float4*>(X + i * d);
    const float4* m4 = reinterpret_cast<const float4*>(mu);
    double xn2 = 0.0;  // |x'|, x' = fl32(x - mu) exactly as the screen's operand
    if (xpart) {       // summed by the screen while it converted the point tile
      xn2 = h == 0 ? __ldg(xpart + 2 * i) : __ldg(xpart + 2 * i + 1);
    } else for (int u = 0; u < nu; ++u) {
      const float4 x = __ldg(xr + 2 * u + h), m = __ldg(m4 + 2 * u + h);
      const double a0 = (double)(x.x - m.x), a1 = (double)(x.y - m.y);
      const double a2 = (double)(x.z - m.z), a3 = (double)(x.w - m.w);
      xn2 = fma(a0, a0, xn2);
      xn2 = fma(a1, a1, xn2);
      xn2 = fma(a2, a2, xn2);
      xn2 = fma(a3, a3, xn2);
    }
    xn2 += __shfl_xor_sync(pmask, xn2, 1);
    // the screen's partial sums are fp32 (relative error <= 64 u = 3.8e-6)
    const float xn = (float)(sqrt(xn2) * (xpart ? 1.0 + 1e-5 : 1.0 + 1e-6));
    if (h == 0) xnorm[i] = xn;
    const double T = tc_threshold((double)xn, cn, d, nprod, cmax_bits);
    const double s0 = v.s0;
    if (v.i0 >= 0 && (k == 1 || (double)v.s1 - s0 > T)) {
      const int lab = v.i0;
      const double2* cr = reinterpret_cast<const double2*>(C + (uint64_t)lab * d);
      double r0, r1, r2, r3;
      {
        const float4 x = __ldg(xr + h);
        const double2 c01 = __ldg(cr + 2 * h), c23 = __ldg(cr + 2 * h + 1);
        double df = __dsub_rn((double)x.x, c01.x);
        r0 = __dmul_rn(df, df);
        df = __dsub_rn((double)x.y, c01.y);
        r1 = __dmul_rn(df, df);
        df = __dsub_rn((double)x.z, c23.x);
        r2 = __dmul_rn(df, df);
        df = __dsub_rn((double)x.w, c23.y);
        r3 = __dmul_rn(df, df);
      }
      for (int u = 1; u < nu; ++u) {
        const float4 x = __ldg(xr + 2 * u + h);
        const double2 c01 = __ldg(cr + 4 * u + 2 * h), c23 = __ldg(cr + 4 * u + 2 * h + 1);
        double df = __dsub_rn((double)x.x, c01.x);
        r0 = __dadd_rn(r0, __dmul_rn(df, df));
        df = __dsub_rn((double)x.y, c01.y);
        r1 = __dadd_rn(r1, __dmul_rn(df, df));
        df = __dsub_rn((double)x.z, c23.x);
        r2 = __dadd_rn(r2, __dmul_rn(df, df));
        df = __dsub_rn((double)x.w, c23.y);
        r3 = __dadd_rn(r3, __dmul_rn(df, df));
      }
      const double t = __dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3));
      const double res = __dadd_rn(t, __shfl_xor_sync(pmask, t, 1));
      if (h == 0) {
        labels[i] = lab;
        best[i] = __dsqrt_rn(res);
      }
    } else if (h == 0) {
      if (v.i0 < 0 || (double)v.s3a - s0 <= T || (double)v.s3b - s0 <= T) full[atomicAdd(nfull, 1ull)] = (uint32_t)i;
      else amb[atomicAdd(namb, 1ull)] = (uint32_t)i;
    }
  }
}

// exact numpy distances over the screen candidates (<= 8 entries within the
// window); ties -> lower index
__global__ void tc_recheck_kernel(const float* __restrict__ X, int d, const double* __restrict__ C, uint64_t k,
                                  const PwPlan plan, const float* top_s, const int* top_i, const float* xnorm,
                                  const unsigned long long* cmax_bits, int nprod, const unsigned* ovf,
                                  const uint32_t* amb, const unsigned long long* na_dev, int64_t* labels, double* best) {
  const double cn = __longlong_as_double((long long)*cmax_bits);
  nprod = eff_mode(nprod, ovf);
  const uint64_t na = *na_dev;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < na; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = amb[q];
    const float* s8 = top_s + i * 8;
    const int* i8 = top_i + i * 8;
    const ScreenView v = screen_view(s8, i8);
    const double T = tc_threshold((double)xnorm[i], cn, d, nprod, cmax_bits);
    const float* xr = X + i * d;
    double bd = 0.0;
    int64_t bl = -1;
    (void)k;
    for (int a = 0; a < 8; ++a) {
      if ((double)s8[a] - (double)v.s0 > T || i8[a] < 0) continue;
      const double* cr = C + (uint64_t)i8[a] * d;
      const double dist = exact_dist(plan, [&](int j) {
        const double df = __dsub_rn((double)xr[j], cr[j]);
        return __dmul_rn(df, df);
      });
      if (bl < 0 || dist < bd || (dist == bd && i8[a] < bl)) {
        bd = dist;
        bl = i8[a];
      }
    }
    labels[i] = bl;
    best[i] = bd;
  }
}

// tc_recheck_kernel with 8 lanes per point (8 <= d <= 128): lane a keeps
// numpy's accumulator r[a]; the xor butterfly gives every lane the same,
// numpy-ordered total (IEEE addition is commutative), so all lanes agree.
__global__ void tc_recheck8_kernel(const float* __restrict__ X, int d, const double* __restrict__ C,
                                   const float* __restrict__ top_s, const int* __restrict__ top_i,
                                   const float* __restrict__ xnorm, const unsigned long long* cmax_bits, int nprod,
                                   const unsigned* ovf, const uint32_t* __restrict__ amb,
                                   const unsigned long long* na_dev, int64_t* labels, double* best) {
  const double cn = __longlong_as_double((long long)*cmax_bits);
  nprod = eff_mode(nprod, ovf);
  const uint64_t na = *na_dev;
  const unsigned lane = threadIdx.x & 31, a = lane & 7;
  const unsigned gmask = 0xFFu << (lane & 24);
  const uint64_t stride = ((uint64_t)gridDim.x * blockDim.x) >> 3;
  const int lim = d - (d % 8);
  for (uint64_t q = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 3; q < na; q += stride) {
    const uint64_t i = amb[q];
    const float* s8 = top_s + i * 8;
    const int* i8 = top_i + i * 8;
    const ScreenView v = screen_view(s8, i8);
    const double T = tc_threshold((double)xnorm[i], cn, d, nprod, cmax_bits);
    const float* xr = X + i * d;
    double xv[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) xv[u] = 8 * u + (int)a < lim ? (double)__ldg(xr + 8 * u + a) : 0.0;
    double bd = 0.0;
    long long bl = -1;
    for (int c8 = 0; c8 < 8; ++c8) {
      const int ci = i8[c8];
      if ((double)s8[c8] - (double)v.s0 > T || ci < 0) continue;
      const double* cr = C + (uint64_t)ci * d;
      double r;
      {
        const double df = __dsub_rn(xv[0], __ldg(cr + a));
        r = __dmul_rn(df, df);
      }
#pragma unroll
      for (int u = 1; u < 16; ++u)
        if (8 * u < lim) {
          const double df = __dsub_rn(xv[u], __ldg(cr + 8 * u + a));
          r = __dadd_rn(r, __dmul_rn(df, df));
        }
      const double p1 = __dadd_rn(r, __shfl_xor_sync(gmask, r, 1));
      const double p2 = __dadd_rn(p1, __shfl_xor_sync(gmask, p1, 2));
      double res = __dadd_rn(p2, __shfl_xor_sync(gmask, p2, 4));
      for (int e = lim; e < d; ++e) {
        const double df = __dsub_rn((double)xr[e], cr[e]);
        res = __dadd_rn(res, __dmul_rn(df, df));
      }
      const double dist = __dsqrt_rn(res);
      if (bl < 0 || dist < bd || (dist == bd && ci < bl)) {
        bd = dist;
        bl = ci;
      }
    }
    if (a == 0) {
      labels[i] = bl;
      best[i] = bd;
    }
  }
}

// ---- wide rows (d > 128): float64 GEMM screen ----------------------------------

__global__ void to_f64_kernel(const float* X, uint64_t count, double* Y) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < count; e += (uint64_t)gridDim.x * blockDim.x)
    Y[e] = (double)X[e];
}

// c2[j] = |c_j|^2 (float64), cmax_bits[0] = max_j |c_j| (1 + 1e-6)
__global__ void center_norms_kernel(const double* C, uint64_t k, int d, double* c2, unsigned long long* cmax_bits) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < k; j += (uint64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int e = 0; e < d; ++e) s = fma(C[j * d + e], C[j * d + e], s);
    c2[j] = s;
    atomicMax(cmax_bits, (unsigned long long)__double_as_longlong(sqrt(s) * (1.0 + 1e-6)));
  }
}

// FP16x3 operands of the wide-row screen, K = 3d: row r of A is
// [hi(s x') | hi(s x') | lo(s x')], row j of B is [hi(s c') | lo(s c') | hi(s c')],
// so one fp32-accumulated f16 GEMM gives s^2 (x'h.c'h + x'h.c'l + x'l.c'h)
__global__ void wide_split_points_kernel(const float* X, uint64_t rows, int d, const float* mu, const float* scal,
                                         __half* Aw, unsigned* ovf) {
  const float xs = __ldg(scal);
  bool big = false;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < rows * d; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = e / d;
    const int j = (int)(e - r * d);
    const float y = (X[e] - __ldg(mu + j)) * xs;  // x' = fl32(x - mu), exactly the classifier's
    big |= !(fabsf(y) <= 32768.f);
    const __half h = __float2half_rn(y);
    const __half l = __float2half_rn(y - __half2float(h));
    __half* a = Aw + r * 3 * (uint64_t)d;
    a[j] = h;
    a[d + j] = h;
    a[2 * d + j] = l;
  }
  if (big) atomicOr(ovf, 1u);
}

// mode 66 (tile origins): c' = fl32(c - mu) as float32 rows, the table
// E[a][j] = |c'_j|^2 - 2 c'_a.c'_j (float64 over the float32 c'), and for
// every 128-row tile the center nearest its first row (any choice is exact;
// a near one keeps |x''| and the window small)
__global__ void wide_cf_kernel(const double* C, uint64_t k, int d, const float* mu, float* cf) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < k * (uint64_t)d; e += (uint64_t)gridDim.x * blockDim.x)
    cf[e] = (float)(C[e] - (double)mu[e % d]);
}

__global__ void wide_etable_kernel(const float* cf, uint64_t k, int d, double* E) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < k * k; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = q / k, j = q % k;
    const float* ca = cf + a * d;
    const float* cj = cf + j * d;
    double e = 0.0;
    for (int t = 0; t < d; ++t) {
      const double y = (double)cj[t];
      e = fma(y, y - 2.0 * (double)ca[t], e);
    }
    E[q] = e;
  }
}

// one warp per tile: float32 distances of the tile's first row to every center
__global__ void wide_origin_kernel(const float* X, uint64_t n, int d, const float* mu, const float* cf, uint64_t k,
                                   int* j0) {
  const int lane = threadIdx.x & 31;
  const uint64_t ntiles = (n + 127) / 128;
  const uint64_t wstride = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t t = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; t < ntiles; t += wstride) {
    const float* xr = X + t * 128 * (uint64_t)d;
    float bv = INFINITY;
    int bj = 0;
    for (uint64_t j = 0; j < k; ++j) {
      float acc = 0.f;
      for (int e = lane; e < d; e += 32) {
        const float z = (xr[e] - mu[e]) - cf[j * d + e];
        acc = fmaf(z, z, acc);
      }
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (acc < bv) {
        bv = acc;
        bj = (int)j;
      }
    }
    if (lane == 0) j0[t] = bj;
  }
}

// one warp per row: x'' = fl32(fl32(x - mu) - c'_j0) (j0 = the row's tile
// origin), the FP16x3 row [hi | hi | lo] of s x'' and |x''|^2 in float64
__global__ void wide_split_local_kernel(const float* X, uint64_t rows, uint64_t row0, int d, const float* mu,
                                        const float* cf, const int* j0, const float* scal, __half* Aw, double* xn2,
                                        unsigned* ovf) {
  const int lane = threadIdx.x & 31;
  const float xs = __ldg(scal);
  const uint64_t wstride = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  bool big = false;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < rows; r += wstride) {
    const float* xr = X + r * (uint64_t)d;
    const float* org = cf + (uint64_t)__ldg(j0 + (row0 + r) / 128) * d;
    __half* a = Aw + r * 3 * (uint64_t)d;
    double q = 0.0;
    for (int e = lane; e < d; e += 32) {
      const float z = (xr[e] - __ldg(mu + e)) - __ldg(org + e);
      q = fma((double)z, (double)z, q);
      const float y = z * xs;
      big |= !(fabsf(y) <= 32768.f);
      const __half h = __float2half_rn(y);
      const __half l = __float2half_rn(y - __half2float(h));
      a[e] = h;
      a[d + e] = h;
      a[2 * d + e] = l;
    }
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    if (lane == 0) xn2[row0 + r] = q;
  }
  if (big) atomicOr(ovf, 1u);
}

// centers: c' = fl32(c - mu) as the FP16 screen's image, |c'|^2 in float64 and |c'|max
__global__ void wide_split_centers_kernel(const double* C, uint64_t k, int d, const float* mu, const float* scal,
                                          __half* Bw, double* c2p, unsigned long long* cmax_bits) {
  const float xs = __ldg(scal);
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < k; c += (uint64_t)gridDim.x * blockDim.x) {
    double n2 = 0.0;
    __half* b = Bw + c * 3 * (uint64_t)d;
    for (int j = 0; j < d; ++j) {
      const float cv = (float)(C[c * d + j] - (double)mu[j]);
      n2 = fma((double)cv, (double)cv, n2);
      const float y = cv * xs;
      const __half h = __float2half_rn(y);
      const __half l = __float2half_rn(y - __half2float(h));
      b[j] = h;
      b[d + j] = l;
      b[2 * d + j] = h;
    }
    c2p[c] = n2;
    atomicMax(cmax_bits, (unsigned long long)__double_as_longlong(sqrt(n2) * (1.0 + 1e-6)));
  }
}

// one warp per row: s_j = |c_j|^2 - 2 x.c_j over the GEMM row, the 8 smallest
// kept as (e0 e1 e2 e7 | e3 e4 e5 e6) -- the classifier reads entries 3 and 7
// as the two lists' 4th values, so a window reaching the 7th smallest counts
// as an overflow (full scan) and every entry of the 8 is a candidate
// (float64 GEMM: s = c2 - 2 g; FP16x3: g = s^2 x'.c', s = c2 - (2 / s^2) g, gw = scal + 1)
template <class T>
__global__ void __launch_bounds__(256) top8_rows_kernel(const T* __restrict__ G, uint64_t rows, uint64_t k,
                                                        const double* __restrict__ c2, float* top_s, int* top_i,
                                                        uint64_t row0, const float* gwp, uint64_t ldg) {
  const int lane = threadIdx.x & 31;
  const double gw = gwp ? (double)__ldg(gwp) : 2.0;
  const uint64_t wstride = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < rows; r += wstride) {
    double v[8];
    int id[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      v[a] = INFINITY;
      id[a] = -1;
    }
    const T* g = G + r * ldg;
    for (uint64_t j = lane; j < k; j += 32) {
      const double sv = c2[j] - gw * (double)g[j];
      if (sv < v[7]) {  // insertion, column order kept among equal values
        int p = 7;
        while (p > 0 && v[p - 1] > sv) {
          v[p] = v[p - 1];
          id[p] = id[p - 1];
          --p;
        }
        v[p] = sv;
        id[p] = (int)j;
      }
    }
    double e[8];
    int ei[8];
    int head = 0;
#pragma unroll
    for (int a = 0; a < 8; ++a) {  // 8 rounds of a warp (value, index) minimum over the lanes' heads
      double hv = INFINITY;
      int hi = -1;
#pragma unroll
      for (int b = 0; b < 8; ++b)
        if (b == head) {
          hv = v[b];
          hi = id[b];
        }
      double bv = hv;
      int bi = hi, bl = lane;
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
        const bool take = ov < bv || (ov == bv && ((unsigned)oi < (unsigned)bi));
        if (take) {
          bv = ov;
          bi = oi;
          bl = ol;
        }
      }
      e[a] = bv;
      ei[a] = bi;
      if (lane == bl && head < 8) ++head;
    }
    if (lane == 0) {
      const uint64_t i = row0 + r;
      const int pos[8] = {0, 1, 2, 4, 5, 6, 7, 3};  // e_a -> slot
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        top_s[i * 8 + pos[a]] = (float)e[a];
        top_i[i * 8 + pos[a]] = ei[a];
      }
    }
  }
}

// The same top-8 with the whole GEMM row in registers (k <= 32 R): R values
// per lane, then 8 rounds of a warp (value, column) minimum -- no per-lane
// insertion lists, every load of the row in flight at once.  Row r's
// |c'|^2-like term is Erow = E + (E_tile ? E_tile[(row0 + r) / 128] * kE : 0):
// the wide FP16x3 screen with tile origins (mode 66) subtracts 2 c'_j0.c'_j per tile.
template <class T, int R>
__global__ void __launch_bounds__(256) top8_rows_reg_kernel(const T* __restrict__ G, uint64_t rows, uint64_t k,
                                                            uint64_t ldg, const double* __restrict__ E,
                                                            const int* __restrict__ E_tile, uint64_t kE,
                                                            float* top_s, int* top_i, uint64_t row0,
                                                            const float* gwp) {
  const int lane = threadIdx.x & 31;
  const double gw = gwp ? (double)__ldg(gwp) : 2.0;
  const uint64_t wstride = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < rows; r += wstride) {
    const T* g = G + r * ldg;
    const double* er = E + (E_tile ? (uint64_t)__ldg(E_tile + (row0 + r) / 128) * kE : 0ull);
    float v[R];
#pragma unroll
    for (int a = 0; a < R; ++a) {
      const uint64_t j = (uint64_t)a * 32 + lane;
      v[a] = j < k ? (float)(__ldg(er + j) - gw * (double)g[j]) : INFINITY;
    }
    float e[8];
    int ei[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float bv = v[0];
      int ba = 0;
#pragma unroll
      for (int a = 1; a < R; ++a)
        if (v[a] < bv) {  // strict: the lane's smallest column among equal values
          bv = v[a];
          ba = a;
        }
      int bj = bv < INFINITY ? ba * 32 + lane : 0x7FFFFFFF;
      for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (ov < bv || (ov == bv && oj < bj)) {
          bv = ov;
          bj = oj;
        }
      }
      e[q] = bv;
      ei[q] = bv < INFINITY ? bj : -1;
      if (bv < INFINITY && (bj & 31) == lane) {
#pragma unroll
        for (int a = 0; a < R; ++a)
          if (a == (bj >> 5)) v[a] = INFINITY;
      }
    }
    if (lane == 0) {
      const uint64_t i = row0 + r;
      const int pos[8] = {0, 1, 2, 4, 5, 6, 7, 3};  // e_q -> slot (as top8_rows_kernel)
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        top_s[i * 8 + pos[q]] = e[q];
        top_i[i * 8 + pos[q]] = ei[q];
      }
    }
  }
}

template <class T>
static int launch_top8(const T* G, uint64_t rows, uint64_t k, uint64_t ldg, const double* E, const int* E_tile,
                       uint64_t kE, float* ts, int* ti, uint64_t row0, const float* gw, cudaStream_t s) {
  const unsigned grid = grid_for(rows * 32, 256);
#define GEEK_TOP8(RV) \
  top8_rows_reg_kernel<T, RV><<<grid, 256, 0, s>>>(G, rows, k, ldg, E, E_tile, kE, ts, ti, row0, gw)
  if (k <= 256) GEEK_TOP8(8);
  else if (k <= 512) GEEK_TOP8(16);
  else if (k <= 768) GEEK_TOP8(24);
  else if (k <= 1024) GEEK_TOP8(32);
  else if (!E_tile) top8_rows_kernel<T><<<grid, 256, 0, s>>>(G, rows, k, E, ts, ti, row0, gw, ldg);
  else {
    set_error("tile-origin top-8 needs k <= 1024");
    return GEEK_EINVAL;
  }
#undef GEEK_TOP8
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

__global__ void assign_stats_kernel(const unsigned long long* namb, const unsigned long long* nfull,
                                    const unsigned* ovf, int nprod, geek_assign_stats_t* st,
                                    const unsigned long long* tiles = nullptr);

// float64 GEMM screen for wide float32 rows: cuBLAS DGEMM in point chunks, the
// top-8 per point, then the exact classification / recheck of the tensor-core path
static int assign_wide_screen(const void* X, int dtype, uint64_t n, int d, const double* C, uint64_t k,
                              const PwPlan& plan, int64_t* labels, double* best, geek_assign_stats_t* stats,
                              void* ev0, void* ev1, cudaStream_t s) {
  // default (float32 rows, k <= 1024): the FP16x3 screen as one f16
  // tensor-core GEMM over K = 3d of the rows centered at their tile's origin
  // center (mode 66); GEEK_WIDE=65 the same centered at the center mean only,
  // GEEK_WIDE=64 (and float64 rows) the float64 DGEMM screen
  const char* wsel = getenv("GEEK_WIDE");
  const int want = wsel ? atoi(wsel) : 66;
  const int mode = (dtype != 0 || want == 64 || 3 * d > 65535) ? 64 : (want == 65 || k > 1024) ? 65 : 66;
  const uint64_t kp8 = (k + 7) / 8 * 8;  // GEMM rows of B / columns of G (16-byte aligned f32 rows)
  Scratch cnt, c2, ts, ti, xn, amb, full, mu0, x64, G, mus, Aw, Bw, cf, Et, j0, xn2;
  GEEK_TRY(cnt.alloc(48, s));
  GEEK_CHECK_CUDA(cudaMemsetAsync(cnt.ptr, 0, 48, s));
  unsigned long long* cmax = cnt.as<unsigned long long>();  // [0] |c'|max, [3] 1/s (FP16)
  unsigned long long* namb = cmax + 1;
  unsigned long long* nfull = cmax + 2;
  unsigned* ovf = reinterpret_cast<unsigned*>(cmax + 4);
  GEEK_TRY(c2.alloc(k * 8, s));
  const float* mu_cls;
  const float* gw = nullptr;
  if (mode >= 65) {
    GEEK_TRY(tc_wide_prepare(C, k, d, mus, cmax, s));
    GEEK_TRY(Bw.alloc(kp8 * 3 * (uint64_t)d * 2, s));
    GEEK_CHECK_CUDA(cudaMemsetAsync(Bw.ptr, 0, kp8 * 3 * (uint64_t)d * 2, s));  // padding centers: zero rows
    wide_split_centers_kernel<<<grid_for(k, 128), 128, 0, s>>>(C, k, d, mus.as<float>(), tc_scal(mus, d),
                                                              Bw.as<__half>(), c2.as<double>(), cmax);
    GEEK_CHECK_LAUNCH();
    mu_cls = mus.as<float>();
    gw = tc_scal(mus, d) + 1;
    if (mode == 66) {
      const uint64_t ntiles = (n + 127) / 128;
      GEEK_TRY(cf.alloc(k * (uint64_t)d * 4, s));
      GEEK_TRY(Et.alloc(k * k * 8, s));
      GEEK_TRY(j0.alloc(ntiles * 4, s));
      GEEK_TRY(xn2.alloc(n * 8, s));
      wide_cf_kernel<<<grid_for(k * (uint64_t)d, 256), 256, 0, s>>>(C, k, d, mu_cls, cf.as<float>());
      GEEK_CHECK_LAUNCH();
      wide_etable_kernel<<<grid_for(k * k, 128), 128, 0, s>>>(cf.as<float>(), k, d, Et.as<double>());
      GEEK_CHECK_LAUNCH();
      wide_origin_kernel<<<grid_for(ntiles * 32, 256), 256, 0, s>>>((const float*)X, n, d, mu_cls, cf.as<float>(), k,
                                                                    j0.as<int>());
      GEEK_CHECK_LAUNCH();
    }
  } else {
    GEEK_TRY(mu0.alloc((size_t)d * 4, s));
    GEEK_CHECK_CUDA(cudaMemsetAsync(mu0.ptr, 0, (size_t)d * 4, s));
    center_norms_kernel<<<grid_for(k, 128), 128, 0, s>>>(C, k, d, c2.as<double>(), cmax);
    GEEK_CHECK_LAUNCH();
    mu_cls = mu0.as<float>();
  }
  GEEK_TRY(ts.alloc(n * 32, s));
  GEEK_TRY(ti.alloc(n * 32, s));
  GEEK_TRY(xn.alloc(n * 4, s));
  GEEK_TRY(amb.alloc(n * 4, s));
  GEEK_TRY(full.alloc(n * 4, s));
  // point chunks: ~3 GB of GEMM operands and output at a time
  const uint64_t row_bytes = mode >= 65 ? 6ull * d + 4ull * kp8 : 8ull * (d + k);
  const uint64_t P = std::max<uint64_t>(1, std::min<uint64_t>(n, (3ull << 30) / row_bytes));
  if (mode >= 65) {
    GEEK_TRY(Aw.alloc(P * 3 * (uint64_t)d * 2, s));
    GEEK_TRY(G.alloc(P * kp8 * 4, s));
  } else {
    if (dtype == 0) GEEK_TRY(x64.alloc(P * d * 8, s));
    GEEK_TRY(G.alloc(P * k * 8, s));
  }
  if (ev0) GEEK_CHECK_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev0), s));
  for (uint64_t r0 = 0; r0 < n; r0 += P) {
    const uint64_t rows = std::min(P, n - r0);
    if (mode >= 65) {
      if (mode == 66)
        wide_split_local_kernel<<<grid_for(rows * 32, 256, 148 * 16), 256, 0, s>>>(
            (const float*)X + r0 * d, rows, r0, d, mu_cls, cf.as<float>(), j0.as<int>(), tc_scal(mus, d),
            Aw.as<__half>(), xn2.as<double>(), ovf);
      else
        wide_split_points_kernel<<<grid_for(rows * d, 256, 148 * 16), 256, 0, s>>>(
            (const float*)X + r0 * d, rows, d, mu_cls, tc_scal(mus, d), Aw.as<__half>(), ovf);
      GEEK_CHECK_LAUNCH();
      GEEK_TRY(hgemm_nt_f32(Aw.ptr, Bw.ptr, G.as<float>(), (int)rows, (int)kp8, 3 * d, s));
      GEEK_TRY(launch_top8<float>(G.as<float>(), rows, k, kp8, mode == 66 ? Et.as<double>() : c2.as<double>(),
                                  mode == 66 ? j0.as<int>() : nullptr, k, ts.as<float>(), ti.as<int>(), r0, gw, s));
      continue;
    }
    const double* A;
    if (dtype == 0) {
      to_f64_kernel<<<grid_for(rows * d, 256), 256, 0, s>>>((const float*)X + r0 * d, rows * d, x64.as<double>());
      GEEK_CHECK_LAUNCH();
      A = x64.as<double>();
    } else {
      A = (const double*)X + r0 * d;
    }
    GEEK_TRY(dgemm_nt(A, C, G.as<double>(), (int)rows, (int)k, d, s));
    GEEK_TRY(launch_top8<double>(G.as<double>(), rows, k, k, c2.as<double>(), nullptr, 0, ts.as<float>(), ti.as<int>(),
                                 r0, nullptr, s));
  }
  if (ev1) GEEK_CHECK_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev1), s));
  const unsigned* ovf_cls = mode >= 65 ? ovf : nullptr;
  // one lane per point: d > 128 needs numpy's full pairwise recursion (the PwPlan), not one 8-accumulator leaf
  tc_classify_kernel<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(
      (const float*)X, n, d, C, k, plan, ts.as<float>(), ti.as<int>(), xn.as<float>(), mu_cls, cmax, mode,
      ovf_cls, labels, best, amb.as<uint32_t>(), namb, full.as<uint32_t>(), nfull,
      mode == 66 ? xn2.as<double>() : nullptr);
  GEEK_CHECK_LAUNCH();
  tc_recheck_kernel<<<148 * 8, 128, 0, s>>>((const float*)X, d, C, k, plan, ts.as<float>(), ti.as<int>(),
                                            xn.as<float>(), cmax, mode, ovf_cls, amb.as<uint32_t>(), namb, labels,
                                            best);
  GEEK_CHECK_LAUNCH();
  full_scan_kernel<<<148 * 4, kFsThreads, sizeof(double) * d, s>>>((const float*)X, d, C, k, plan,
                                                                   full.as<uint32_t>(), nfull, labels, best);
  GEEK_CHECK_LAUNCH();
  if (stats) {
    assign_stats_kernel<<<1, 1, 0, s>>>(namb, nfull, ovf_cls, mode, stats);
    GEEK_CHECK_LAUNCH();
  }
  return GEEK_OK;
}

__global__ void assign_stats_kernel(const unsigned long long* namb, const unsigned long long* nfull,
                                    const unsigned* ovf, int nprod, geek_assign_stats_t* st,
                                    const unsigned long long* tiles) {
  st->rechecked = (namb ? *namb : 0ull) + (nfull ? *nfull : 0ull);
  st->full_scans = nfull ? *nfull : 0ull;
  st->screen_mode = (unsigned long long)eff_mode(nprod, ovf);
  st->screen_tiles = tiles ? *tiles : 0ull;
}

}  // namespace geek

using namespace geek;

extern "C" {

uint64_t geek_assign_l2_workspace_size(uint64_t n, int d, uint64_t k) {
  // an upper bound over every path: per-point screen lists and queues
  // (top-4 values / centers of both column halves, |x'|, queues, |x'|^2
  // halves), the center operand images of the FP16 screen and its TF32x3
  // fallback (<= 320 KB per 192-center tile at d <= 128), the tile-local
  // origin table, the wide-row transposed centers, the wide-row GEMM chunk
  // (<= 3 GB of operands and output, plus the FP16x3 center operand), and
  // alignment slack
  const uint64_t nct = (k + 191) / 192, ntiles = (n + 127) / 128;
  const uint64_t wide = d > 128 ? std::min<uint64_t>(3ull << 30, n * (8ull * (d + k))) + k * (uint64_t)d * 10 +
                                       k * k * 8 + n * 9 + (64ull << 10) : 0;
  return n * 100 + nct * (330ull << 10) + k * (uint64_t)d * 24 + k * nct * 192 * 4 + ntiles * 80 + wide + (4ull << 20);
}

int geek_assign_l2(const void* X, int dtype, uint64_t n, int d, const double* C, uint64_t k, int64_t* labels,
                   double* best, geek_assign_stats_t* stats, void* ev_screen_begin, void* ev_screen_end,
                   void* workspace, uint64_t workspace_bytes, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(dtype == 0 || dtype == 1, "dtype must be 0 or 1");
  GEEK_REQUIRE(k >= 1, "cannot assign without centers");
  GEEK_REQUIRE(d >= 1 && d <= 1536, "dimension %d outside [1, 1536]", d);
  WorkspaceScope scope(workspace, workspace_bytes);
  if (stats) GEEK_CHECK_CUDA(cudaMemsetAsync(stats, 0, sizeof(geek_assign_stats_t), s));
  if (n == 0) return GEEK_OK;
  PwPlan plan;
  pw_build(plan, 0, d);
  GEEK_REQUIRE(plan.nops <= 64, "pairwise plan too deep");
  const size_t smem = sizeof(double) * kAsgCenters * d;
  if (smem > 48 * 1024) {
    GEEK_CHECK_CUDA(cudaFuncSetAttribute(assign_l2_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
    GEEK_CHECK_CUDA(cudaFuncSetAttribute(assign_l2_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
  }
  if (dtype == 0 && k >= 4 && d <= 128 && n < 0xFFFFFFFFull) {
    // tensor-core screen -> classification -> candidate / full recheck, all
    // stream-ordered: the FP16 scale is chosen on the device, the TF32x3 redo
    // after an f16 overflow is a launch that exits unless the overflow flag is
    // set, and the rechecks stride over their device-side queue lengths.
    // Default FP16x3; GEEK_SCREEN=17 selects the tile-local FP16 screen (one
    // product per K slice against each point tile's origin center: a third of
    // the MMAs, but on the benchmark data the kernel is bound by its epilogue,
    // not the tensor pipe, and its wider window sends 21M instead of 12M
    // points to the recheck: profiles/r2_screen.md), 3 / 1 TF32x3 / one TF32
    const char* sel = getenv("GEEK_SCREEN");
    const bool local_ok = k <= 3840 && d % 8 == 0;  // 4 x 48 KB B stages + two origin-table rows in SMEM
    const int nprod = !sel ? 16 : atoi(sel) == 1 ? 1 : atoi(sel) == 3 ? 3 : (atoi(sel) == 17 && local_ok) ? 17 : 16;
    Scratch img, c2s, mus, img3, c2s3, mus3, ts, ti, xn, amb, full, cnt, lcf, les, lj0, xp, ldm;
    TcLocal loc{nullptr, nullptr, nullptr, nullptr};
    GEEK_TRY(cnt.alloc(48, s));
    GEEK_CHECK_CUDA(cudaMemsetAsync(cnt.ptr, 0, 48, s));
    unsigned long long* cmax = cnt.as<unsigned long long>();  // [0] |c'|max, [3] 1/s (FP16), [5] screen tiles
    unsigned long long* namb = cmax + 1;
    unsigned long long* nfull = cmax + 2;
    unsigned* ovf = reinterpret_cast<unsigned*>(cmax + 4);
    int nct = 0;
    float xscale = 1.f;
    GEEK_TRY(tc_screen_prepare(C, k, d, nprod, kTcLBO, kTcSBO, img, c2s, mus, cmax, nct, xscale, s));
    // FP16x3: the top-4 lists start at a bound from each point tile's origin
    // center (GEEK_SCREEN_BOUND=0 starts them at +inf)
    const char* bsel = getenv("GEEK_SCREEN_BOUND");
    const bool bound16 = nprod == 16 && !(bsel && atoi(bsel) == 0);
    if (nprod == 17 || bound16) {
      // FP16x3: + the center-tile distance bounds that let a point tile skip
      // center tiles no row can reach (GEEK_SCREEN_SKIP=0: every tile)
      const char* ksel = getenv("GEEK_SCREEN_SKIP");
      const bool skip = nprod == 16 && !(ksel && atoi(ksel) == 0);
      GEEK_TRY(tc_local_prepare(C, k, d, (const float*)X, n, kTcLBO, kTcSBO, mus, xscale, nct, lcf, les, lj0, loc, s,
                                nprod == 17, skip ? &ldm : nullptr));
      loc.cmax = cmax;
      loc.tiles_done = cmax + 5;
    }
    GEEK_TRY(ts.alloc(n * 32, s));
    GEEK_TRY(ti.alloc(n * 32, s));
    GEEK_TRY(xn.alloc(n * 4, s));
    GEEK_TRY(amb.alloc(n * 4, s));
    GEEK_TRY(full.alloc(n * 4, s));
    // the screens also leave |x'|^2 per row half for the 2-lane classifier
    const bool use_xp = nprod != 1 && d % 8 == 0 && d <= 128;
    if (use_xp) GEEK_TRY(xp.alloc(n * 16, s));
    if (ev_screen_begin) GEEK_CHECK_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_screen_begin), s));
    GEEK_TRY(tc_screen_launch((const float*)X, n, d, nprod, img, c2s, mus, k, nct, kTcLBO, kTcSBO, ts.as<float>(),
                              ti.as<int>(), use_xp ? xp.as<double>() : nullptr, xscale, ovf, s,
                              (nprod == 17 || bound16) ? &loc : nullptr));
    if (nprod >= 16) {  // a point coordinate beyond the f16 range: the TF32x3 redo runs (device-predicated)
      int nct3 = 0;
      float xs3 = 1.f;
      GEEK_TRY(tc_screen_prepare(C, k, d, 3, kTcLBO, kTcSBO, img3, c2s3, mus3, cmax, nct3, xs3, s));
      GEEK_TRY(tc_screen_launch((const float*)X, n, d, 3, img3, c2s3, mus3, k, nct3, kTcLBO, kTcSBO, ts.as<float>(),
                                ti.as<int>(), use_xp ? xp.as<double>() : nullptr, xs3, ovf, s, nullptr, 1, ovf));
    }
    if (ev_screen_end) GEEK_CHECK_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_screen_end), s));
    // (after a redo the mean / images of the TF32x3 prepare are the ones that match;
    // both prepares compute the same mean, and |c'|max is an atomic maximum of the same values)
    const float* mu_cls = mus.as<float>();
    if (d % 8 == 0 && d <= 128)
      tc_classify2_kernel<<<grid_for(n * 2, 256, 148 * 16), 256, 0, s>>>(
          (const float*)X, n, d, C, k, ts.as<float>(), ti.as<int>(), xn.as<float>(), mu_cls,
          use_xp ? xp.as<double>() : nullptr, cmax, nprod, ovf, labels, best, amb.as<uint32_t>(), namb,
          full.as<uint32_t>(), nfull);
    else if (d >= 8)
      tc_classify8_kernel<<<grid_for(n * 8, 256, 148 * 16), 256, 0, s>>>(
          (const float*)X, n, d, C, k, ts.as<float>(), ti.as<int>(), xn.as<float>(), mu_cls, cmax, nprod, ovf,
          labels, best, amb.as<uint32_t>(), namb, full.as<uint32_t>(), nfull);
    else
      tc_classify_kernel<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(
          (const float*)X, n, d, C, k, plan, ts.as<float>(), ti.as<int>(), xn.as<float>(), mu_cls, cmax, nprod, ovf,
          labels, best, amb.as<uint32_t>(), namb, full.as<uint32_t>(), nfull, nullptr);
    GEEK_CHECK_LAUNCH();
    if (d >= 8)
      tc_recheck8_kernel<<<148 * 16, 256, 0, s>>>((const float*)X, d, C, ts.as<float>(), ti.as<int>(), xn.as<float>(),
                                                  cmax, nprod, ovf, amb.as<uint32_t>(), namb, labels, best);
    else
      tc_recheck_kernel<<<148 * 8, 128, 0, s>>>((const float*)X, d, C, k, plan, ts.as<float>(), ti.as<int>(),
                                                xn.as<float>(), cmax, nprod, ovf, amb.as<uint32_t>(), namb, labels,
                                                best);
    GEEK_CHECK_LAUNCH();
    full_scan_kernel<<<148 * 4, kFsThreads, sizeof(double) * d, s>>>((const float*)X, d, C, k, plan,
                                                                     full.as<uint32_t>(), nfull, labels, best);
    GEEK_CHECK_LAUNCH();
    if (stats) {
      // (screen tiles: the FP16x3 screen's multiplied pairs; a TF32x3 redo after an
      // f16 overflow does not count them)
      assign_stats_kernel<<<1, 1, 0, s>>>(namb, nfull, ovf, nprod, stats, nprod == 16 ? cmax + 5 : nullptr);
      GEEK_CHECK_LAUNCH();
    }
    return GEEK_OK;
  }
  const size_t scr_smem = sizeof(float) * ((size_t)d * (kScrP + 4) + kScrK * (kScrC + 4) + 3 * kScrP);
  const bool screened = dtype == 0 && k >= 4 && scr_smem <= 200 * 1024 && n < 0xFFFFFFFFull;
  if (dtype == 0 && d > 128 && k >= 4 && n < 0xFFFFFFFFull && cublas_available()) {
    // tensor-core GEMM screen (FP16x3 over K = 3d, or the float64 DGEMM) + the
    // exact classification; without cuBLAS the exact SIMT kernels below
    return assign_wide_screen(X, dtype, n, d, C, k, plan, labels, best, stats, ev_screen_begin, ev_screen_end, s);
  }
  if (!screened && d > 128) {
    const uint64_t kpad = (k + 31) / 32 * 32;
    Scratch ctb;
    GEEK_TRY(ctb.alloc(kpad * d * 8, s));
    transpose_centers_kernel<<<grid_for(kpad * d, 256), 256, 0, s>>>(C, k, d, kpad, ctb.as<double>());
    const size_t xsm = sizeof(double) * kCtP * d;
    if (xsm + 1024 > 48 * 1024) {  // + the static reduction arrays
      GEEK_CHECK_CUDA(cudaFuncSetAttribute(assign_l2_ct_kernel<float>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xsm));
      GEEK_CHECK_CUDA(cudaFuncSetAttribute(assign_l2_ct_kernel<double>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xsm));
    }
    if (k <= 16) {
      int S = 1;
      while ((uint64_t)S < k) S <<= 1;
      const unsigned gk = grid_for((n + kCtP - 1) / kCtP, kCtThreads / S, 148 * 16);
      if (dtype == 0)
        assign_l2_ctk_kernel<float><<<gk, kCtThreads, 0, s>>>((const float*)X, n, d, ctb.as<double>(), k, kpad, S,
                                                              plan, labels, best);
      else
        assign_l2_ctk_kernel<double><<<gk, kCtThreads, 0, s>>>((const double*)X, n, d, ctb.as<double>(), k, kpad,
                                                               S, plan, labels, best);
      GEEK_CHECK_LAUNCH();
      return GEEK_OK;
    }
    const unsigned grid = grid_for((n + kCtP - 1) / kCtP, 1, 148 * 16);
    if (dtype == 0)
      assign_l2_ct_kernel<float><<<grid, kCtThreads, xsm, s>>>((const float*)X, n, d, ctb.as<double>(), k, kpad,
                                                               plan, labels, best);
    else
      assign_l2_ct_kernel<double><<<grid, kCtThreads, xsm, s>>>((const double*)X, n, d, ctb.as<double>(), k,
                                                                kpad, plan, labels, best);
    GEEK_CHECK_LAUNCH();
    return GEEK_OK;
  }
  if (!screened) {
    unsigned grid = (unsigned)((n + kAsgThreads - 1) / kAsgThreads);
    if (dtype == 0)
      assign_l2_kernel<float><<<grid, kAsgThreads, smem, s>>>((const float*)X, n, d, C, k, plan, labels, best,
                                                               nullptr);
    else
      assign_l2_kernel<double><<<grid, kAsgThreads, smem, s>>>((const double*)X, n, d, C, k, plan, labels, best,
                                                                nullptr);
    GEEK_CHECK_LAUNCH();
    return GEEK_OK;
  }
  // float32 SIMT screen (129 <= d with its SMEM tile in 200 KB): certain points
  // are labelled in the screen, the queued ones exactly over all centers
  Scratch cf, c2, amb, cnt;
  GEEK_TRY(cf.alloc(k * d * 4, s));
  GEEK_TRY(c2.alloc(k * 4, s));
  GEEK_TRY(amb.alloc(n * 4, s));
  GEEK_TRY(cnt.alloc(16, s));
  GEEK_CHECK_CUDA(cudaMemsetAsync(cnt.ptr, 0, 16, s));
  unsigned long long* namb = cnt.as<unsigned long long>();
  unsigned long long* cmax = namb + 1;
  center_prep_kernel<<<grid_for(k, 128), 128, 0, s>>>(C, k, d, cf.as<float>(), c2.as<float>(), cmax);
  GEEK_CHECK_LAUNCH();
  GEEK_CHECK_CUDA(cudaFuncSetAttribute(screen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scr_smem));
  const unsigned grid = (unsigned)((n + kScrP - 1) / kScrP);
  if (ev_screen_begin) GEEK_CHECK_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_screen_begin), s));
  screen_kernel<<<grid, kScrThreads, scr_smem, s>>>((const float*)X, n, d, cf.as<float>(), c2.as<float>(), C, k,
                                                    cmax, plan, labels, best, amb.as<uint32_t>(), namb);
  GEEK_CHECK_LAUNCH();
  if (ev_screen_end) GEEK_CHECK_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_screen_end), s));
  assign_l2_kernel<float><<<148 * 8, kAsgThreads, smem, s>>>((const float*)X, n, d, C, k, plan, labels, best,
                                                             amb.as<uint32_t>(), namb);
  GEEK_CHECK_LAUNCH();
  if (stats) {
    assign_stats_kernel<<<1, 1, 0, s>>>(namb, nullptr, nullptr, 0, stats);
    GEEK_CHECK_LAUNCH();
  }
  return GEEK_OK;
}

int geek_radii_sizes(const int64_t* labels, const double* best, uint64_t n, uint64_t k, double* radii,
                     int64_t* sizes, void* stream) {
  cudaStream_t s = as_stream(stream);
  (void)k;
  if (n == 0) return GEEK_OK;
  radii_sizes_kernel<<<grid_for(n, 256), 256, 0, s>>>(labels, best, n, radii, sizes);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

int geek_pairwise_sum(const double* v, uint64_t n, double* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n == 0) {
    GEEK_CHECK_CUDA(cudaMemsetAsync(out, 0, 8, s));
    return GEEK_OK;
  }
  // the tree's index arrays live on the device, built and uploaded once per
  // (device, n): the per-call work is one leaf pass and one launch per level
  static std::mutex mu;
  static std::map<std::pair<int, uint64_t>, std::shared_ptr<DevSumTree>> cache;
  int dev = 0;
  GEEK_CHECK_CUDA(cudaGetDevice(&dev));
  std::shared_ptr<DevSumTree> t;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, n});
    if (it == cache.end()) {
      GEEK_CHECK_CUDA(cudaStreamSynchronize(s));  // a cleared entry's arrays may still be in use
      if (cache.size() > 8) cache.clear();
      t = std::make_shared<DevSumTree>();
      GEEK_TRY(t->build(*make_tree(n)));
      cache[{dev, n}] = t;
    } else {
      t = it->second;
    }
  }
  Scratch val;
  GEEK_TRY(val.alloc((uint64_t)t->nnodes * 8, s));
  leaf_sum_kernel<<<grid_for(t->nleaf, 128), 128, 0, s>>>(v, t->leaf_off, t->leaf_len, t->leaf_node, t->nleaf,
                                                          val.as<double>());
  GEEK_CHECK_LAUNCH();
  const uint32_t* base = t->lv;
  for (uint64_t c : t->lv_count) {
    combine_kernel<<<grid_for(c, 128), 128, 0, s>>>(base, base + c, base + 2 * c, c, val.as<double>());
    GEEK_CHECK_LAUNCH();
    base += 3 * c;
  }
  GEEK_CHECK_CUDA(cudaMemcpyAsync(out, val.as<double>(), 8, cudaMemcpyDeviceToDevice, s));
  return GEEK_OK;
}

}  // extern "C"
