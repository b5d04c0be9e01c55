// cuBLAS, loaded at run time, for the one plain library GEMM on the path: the
// float64 distance screen of wide rows (d > 128, where the tcgen05 screen's
// 128-dim point tile does not apply).  dlopen keeps libgeek.so free of a
// link-time cuBLAS dependency: in a PyTorch process the already-loaded
// libcublas.so.12 is reused, else the CUDA toolkit's.
#include "common.cuh"

#include <dlfcn.h>

#include <mutex>

namespace geek {

namespace {

typedef int (*create_fn)(void**);
typedef int (*set_stream_fn)(void*, cudaStream_t);
typedef int (*dgemm_fn)(void*, int, int, int, int, int, const double*, const double*, int, const double*, int,
                        const double*, double*, int);

struct Cublas {
  bool tried = false, ok = false;
  create_fn create = nullptr;
  set_stream_fn set_stream = nullptr;
  dgemm_fn dgemm = nullptr;
  void* handle[64] = {};
};

Cublas& api() {
  static Cublas c;
  return c;
}

std::mutex& mu() {
  static std::mutex m;
  return m;
}

}  // namespace

// C[n][m] (row-major) = A[n][kk] . B[m][kk]^T  in float64 on `s`
int dgemm_nt(const double* A, const double* B, double* Cout, int n, int m, int kk, cudaStream_t s) {
  Cublas& c = api();
  std::lock_guard<std::mutex> lk(mu());
  if (!c.tried) {
    c.tried = true;
    const char* names[] = {"libcublas.so.12", "/usr/local/cuda/lib64/libcublas.so.12", "libcublas.so"};
    void* lib = nullptr;
    for (const char* nm : names)
      if ((lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (lib) {
      c.create = (create_fn)dlsym(lib, "cublasCreate_v2");
      c.set_stream = (set_stream_fn)dlsym(lib, "cublasSetStream_v2");
      c.dgemm = (dgemm_fn)dlsym(lib, "cublasDgemm_v2");
      c.ok = c.create && c.set_stream && c.dgemm;
    }
  }
  if (!c.ok) {
    set_error("cuBLAS (libcublas.so.12) not loadable");
    return GEEK_ECUDA;
  }
  int dev = 0;
  GEEK_CHECK_CUDA(cudaGetDevice(&dev));
  GEEK_REQUIRE(dev >= 0 && dev < 64, "device index %d", dev);
  if (!c.handle[dev] && c.create(&c.handle[dev]) != 0) {
    set_error("cublasCreate failed");
    return GEEK_ECUDA;
  }
  if (c.set_stream(c.handle[dev], s) != 0) {
    set_error("cublasSetStream failed");
    return GEEK_ECUDA;
  }
  const double one = 1.0, zero = 0.0;
  // column-major: C^T (m x n) = op(B)=T (m x kk, B is kk x m col-major) . A (kk x n)
  const int st = c.dgemm(c.handle[dev], /*transa=T*/ 1, /*transb=N*/ 0, m, n, kk, &one, B, kk, A, kk, &zero, Cout, m);
  if (st != 0) {
    set_error("cublasDgemm failed (%d)", st);
    return GEEK_ECUDA;
  }
  return GEEK_OK;
}

}  // namespace geek
