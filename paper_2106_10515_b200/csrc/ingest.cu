// Vector-file ingestion (io.py:21-48): .fvecs / .bvecs records are a 4-byte
// little-endian dimension prefix followed by d float32 / uint8 values.  The
// host streams whole records into device memory; this kernel strips the
// prefixes into a row-major float32 [n][d] matrix (uint8 values are exact in
// float32, as they are in the reference's float64) and reports the first
// record whose prefix differs from d.  Byte work, HBM-bound: one read of the
// raw records and one write of the matrix.
#include "common.cuh"

namespace geek {

__global__ void unpack_fvecs_kernel(const uint32_t* __restrict__ raw, uint64_t nrec, int d,
                                    float* __restrict__ out, unsigned long long* bad) {
  const uint64_t rec = (uint64_t)d + 1;  // words per record
  const uint64_t total = nrec * rec;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < total;
       w += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = w / rec;
    const uint64_t c = w - i * rec;
    const uint32_t v = raw[w];
    if (c == 0) {
      if (v != (uint32_t)d) atomicMin(bad, (unsigned long long)i);
    } else {
      out[i * d + (c - 1)] = __uint_as_float(v);
    }
  }
}

__global__ void unpack_bvecs_kernel(const uint8_t* __restrict__ raw, uint64_t nrec, int d,
                                    float* __restrict__ out, unsigned long long* bad) {
  const uint64_t rec = (uint64_t)d + 4;  // bytes per record
  const uint64_t total = nrec * (uint64_t)d;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = e / d;
    const uint64_t c = e - i * d;
    const uint8_t* r = raw + i * rec;
    out[e] = (float)r[4 + c];
    if (c == 0) {
      const uint32_t p = (uint32_t)r[0] | ((uint32_t)r[1] << 8) | ((uint32_t)r[2] << 16) | ((uint32_t)r[3] << 24);
      if (p != (uint32_t)d) atomicMin(bad, (unsigned long long)i);
    }
  }
}

}  // namespace geek

using namespace geek;

extern "C" {

int geek_unpack_vecs(const void* raw, uint64_t nrec, int d, int elem_bytes, float* out, uint64_t* bad_rec,
                     void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(d > 0, "dimension must be positive");
  GEEK_REQUIRE(elem_bytes == 4 || elem_bytes == 1, "element size must be 4 (fvecs) or 1 (bvecs)");
  if (nrec == 0) return GEEK_OK;
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(bad_rec);
  if (elem_bytes == 4) {
    unpack_fvecs_kernel<<<grid_for(nrec * (uint64_t)(d + 1), 256), 256, 0, s>>>(
        static_cast<const uint32_t*>(raw), nrec, d, out, bad);
  } else {
    unpack_bvecs_kernel<<<grid_for(nrec * (uint64_t)d, 256), 256, 0, s>>>(static_cast<const uint8_t*>(raw), nrec,
                                                                           d, out, bad);
  }
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

}  // extern "C"
