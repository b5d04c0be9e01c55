// K8: one-pass assignment (assignment.py:44-107).
//
// Euclidean distances are evaluated exactly as numpy does for
// sqrt(((x - c)**2).sum(axis=-1)) on float64: round-to-nearest subtract and
// square (no FMA contraction), numpy's pairwise summation tree (blocks of
// <= 128 with 8 accumulators, recursive halving at multiples of 8), a
// correctly rounded sqrt, and first-index argmin -- so labels, best
// distances and radii are bit-identical to the reference.
#include "common.cuh"

#include <algorithm>
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

template <class T>
__global__ void __launch_bounds__(kAsgThreads) assign_l2_kernel(const T* __restrict__ X, uint64_t n, int d,
                                                                const double* __restrict__ C, uint64_t k,
                                                                const PwPlan plan, int64_t* labels,
                                                                double* best) {
  extern __shared__ double sC[];  // [kAsgCenters][d]
  const uint64_t i = blockIdx.x * (uint64_t)kAsgThreads + threadIdx.x;
  const bool valid = i < n;
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

__global__ void radii_sizes_kernel(const int64_t* labels, const double* best, uint64_t n, double* radii,
                                   int64_t* sizes) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const int64_t l = labels[i];
    atomicMax(reinterpret_cast<unsigned long long*>(radii) + l,
              (unsigned long long)__double_as_longlong(best[i]));  // best >= 0
    atomicAdd(reinterpret_cast<unsigned long long*>(sizes) + l, 1ull);
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

}  // namespace geek

using namespace geek;

extern "C" {

int geek_assign_l2(const void* X, int dtype, uint64_t n, int d, const double* C, uint64_t k, int64_t* labels,
                   double* best, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(dtype == 0 || dtype == 1, "dtype must be 0 or 1");
  GEEK_REQUIRE(k >= 1, "cannot assign without centers");
  GEEK_REQUIRE(d >= 1 && d <= 1536, "dimension %d outside [1, 1536]", d);
  if (n == 0) return GEEK_OK;
  PwPlan plan;
  pw_build(plan, 0, d);
  GEEK_REQUIRE(plan.nops <= 64, "pairwise plan too deep");
  size_t smem = sizeof(double) * kAsgCenters * d;
  unsigned grid = (unsigned)((n + kAsgThreads - 1) / kAsgThreads);
  if (dtype == 0) {
    if (smem > 48 * 1024)
      GEEK_CHECK_CUDA(cudaFuncSetAttribute(assign_l2_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
    assign_l2_kernel<float><<<grid, kAsgThreads, smem, s>>>((const float*)X, n, d, C, k, plan, labels, best);
  } else {
    if (smem > 48 * 1024)
      GEEK_CHECK_CUDA(cudaFuncSetAttribute(assign_l2_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
    assign_l2_kernel<double><<<grid, kAsgThreads, smem, s>>>((const double*)X, n, d, C, k, plan, labels, best);
  }
  GEEK_CHECK_LAUNCH();
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
  static std::mutex mu;
  static std::map<uint64_t, std::shared_ptr<SumTree>> cache;
  std::shared_ptr<SumTree> t;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(n);
    if (it == cache.end()) {
      t = make_tree(n);
      if (cache.size() > 8) cache.clear();
      cache[n] = t;
    } else {
      t = it->second;
    }
  }
  const uint64_t nleaf = t->leaf_off.size();
  uint64_t ninternal = 0;
  for (auto& l : t->lv_node) ninternal += l.size();
  Scratch val, lf, lv;
  GEEK_TRY(val.alloc((uint64_t)t->nnodes * 8, s));
  GEEK_TRY(lf.alloc(nleaf * 16, s));
  GEEK_TRY(lv.alloc(ninternal * 12 + 16, s));
  uint64_t* loff = lf.as<uint64_t>();
  uint32_t* llen = reinterpret_cast<uint32_t*>(loff + nleaf);
  uint32_t* lnode = llen + nleaf;
  GEEK_CHECK_CUDA(cudaMemcpyAsync(loff, t->leaf_off.data(), nleaf * 8, cudaMemcpyHostToDevice, s));
  GEEK_CHECK_CUDA(cudaMemcpyAsync(llen, t->leaf_len.data(), nleaf * 4, cudaMemcpyHostToDevice, s));
  GEEK_CHECK_CUDA(cudaMemcpyAsync(lnode, t->leaf_node.data(), nleaf * 4, cudaMemcpyHostToDevice, s));
  leaf_sum_kernel<<<grid_for(nleaf, 128), 128, 0, s>>>(v, loff, llen, lnode, nleaf, val.as<double>());
  GEEK_CHECK_LAUNCH();
  uint32_t* base = lv.as<uint32_t>();
  for (size_t L = 0; L < t->lv_node.size(); ++L) {
    const uint64_t c = t->lv_node[L].size();
    GEEK_CHECK_CUDA(cudaMemcpyAsync(base, t->lv_node[L].data(), c * 4, cudaMemcpyHostToDevice, s));
    GEEK_CHECK_CUDA(cudaMemcpyAsync(base + c, t->lv_left[L].data(), c * 4, cudaMemcpyHostToDevice, s));
    GEEK_CHECK_CUDA(cudaMemcpyAsync(base + 2 * c, t->lv_right[L].data(), c * 4, cudaMemcpyHostToDevice, s));
    combine_kernel<<<grid_for(c, 128), 128, 0, s>>>(base, base + c, base + 2 * c, c, val.as<double>());
    GEEK_CHECK_LAUNCH();
    base += 3 * c;
  }
  GEEK_CHECK_CUDA(cudaMemcpyAsync(out, val.as<double>(), 8, cudaMemcpyDeviceToDevice, s));
  GEEK_CHECK_CUDA(cudaStreamSynchronize(s));  // host plan vectors are cached; scratch freed in order
  return GEEK_OK;
}

}  // extern "C"
