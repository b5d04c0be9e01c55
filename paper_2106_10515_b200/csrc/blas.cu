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
typedef int (*gemmex_fn)(void*, int, int, int, int, int, const void*, const void*, int, int, const void*, int, int,
                         const void*, void*, int, int, int, int);

struct Cublas {
  bool tried = false, ok = false;
  create_fn create = nullptr;
  set_stream_fn set_stream = nullptr;
  dgemm_fn dgemm = nullptr;
  gemmex_fn gemmex = nullptr;
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

// the caller holds mu(): the per-device handle's stream stays set through its call
static int cublas_ready(Cublas& c, cudaStream_t s) {
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
      c.gemmex = (gemmex_fn)dlsym(lib, "cublasGemmEx");
      c.ok = c.create && c.set_stream && c.dgemm && c.gemmex;
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
  return GEEK_OK;
}

// cuBLAS loadable (the wide-row screens exist); false sends callers to their exact SIMT kernels
bool cublas_available() {
  Cublas& c = api();
  std::lock_guard<std::mutex> lk(mu());
  if (!c.tried) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    if (cublas_ready(c, 0) != GEEK_OK) return false;
  }
  return c.ok;
}

// C[n][m] (row-major) = A[n][kk] . B[m][kk]^T  in float64 on `s`
int dgemm_nt(const double* A, const double* B, double* Cout, int n, int m, int kk, cudaStream_t s) {
  Cublas& c = api();
  std::lock_guard<std::mutex> lk(mu());
  GEEK_TRY(cublas_ready(c, s));
  int dev = 0;
  GEEK_CHECK_CUDA(cudaGetDevice(&dev));
  const double one = 1.0, zero = 0.0;
  // column-major: C^T (m x n) = op(B)=T (m x kk, B is kk x m col-major) . A (kk x n)
  const int st = c.dgemm(c.handle[dev], /*transa=T*/ 1, /*transb=N*/ 0, m, n, kk, &one, B, kk, A, kk, &zero, Cout, m);
  if (st != 0) {
    set_error("cublasDgemm failed (%d)", st);
    return GEEK_ECUDA;
  }
  return GEEK_OK;
}

// C[n][m] (row-major, float32) = A[n][kk] . B[m][kk]^T over f16 operands,
// fp32 accumulation (CUDA_R_16F inputs, CUBLAS_COMPUTE_32F, CUDA_R_32F output)
int hgemm_nt_f32(const void* A, const void* B, float* Cout, int n, int m, int kk, cudaStream_t s) {
  Cublas& c = api();
  std::lock_guard<std::mutex> lk(mu());
  GEEK_TRY(cublas_ready(c, s));
  int dev = 0;
  GEEK_CHECK_CUDA(cudaGetDevice(&dev));
  const float one = 1.f, zero = 0.f;
  const int kR16F = 2, kR32F = 0, kCompute32F = 68, kGemmDefault = -1;
  const int st = c.gemmex(c.handle[dev], /*transa=T*/ 1, /*transb=N*/ 0, m, n, kk, &one, B, kR16F, kk, A, kR16F, kk,
                          &zero, Cout, kR32F, m, kCompute32F, kGemmDefault);
  if (st != 0) {
    set_error("cublasGemmEx failed (%d)", st);
    return GEEK_ECUDA;
  }
  return GEEK_OK;
}

}  // namespace geek
