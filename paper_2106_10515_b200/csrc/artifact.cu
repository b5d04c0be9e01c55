// LSHC v1 bucket artifacts (serialize.py:129-162): the byte image of
// dump_buckets written straight from the device bucket CSR.  Per bucket:
//   <q table><q slot>  then pack_array(members int64):
//   <q length = 2 + 8 + 8*size><B code 1 = int64><B ndim 1><q size><size x <q id>
// One block per bucket: thread 0 writes the 34-byte header, the block widens
// the uint32 member ids to int64 little-endian.  Offsets come from a prefix
// sum of the sizes (host side), so the file is one D2H copy.
#include "common.cuh"

namespace geek {

__device__ __forceinline__ void put64(uint8_t* p, uint64_t v) {
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}

__global__ void pack_buckets_kernel(const uint32_t* __restrict__ flat, const uint64_t* __restrict__ off,
                                    const uint64_t* __restrict__ toff, int ntables, uint64_t nbuckets,
                                    uint64_t base, uint8_t* __restrict__ out) {
  for (uint64_t b = blockIdx.x; b < nbuckets; b += gridDim.x) {
    const uint64_t m0 = off[b], size = off[b + 1] - m0;
    // byte offset: each bucket before b costs 34 header bytes + 8 per member
    uint8_t* p = out + base + 34 * b + 8 * m0;
    if (threadIdx.x == 0) {
      int t = 0;
      while (t + 1 < ntables && toff[t + 1] <= b) ++t;
      put64(p, (uint64_t)t);
      put64(p + 8, b - toff[t]);
      put64(p + 16, 2 + 8 + 8 * size);
      p[24] = 1;  // int64
      p[25] = 1;  // ndim
      put64(p + 26, size);
    }
    uint8_t* body = p + 34;
    for (uint64_t i = threadIdx.x; i < size; i += blockDim.x) put64(body + 8 * i, (uint64_t)flat[m0 + i]);
  }
}

}  // namespace geek

using namespace geek;

extern "C" {

int geek_pack_buckets(const uint32_t* flat, const uint64_t* offsets, const uint64_t* table_off, int ntables,
                      uint64_t nbuckets, uint64_t base, uint8_t* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  GEEK_REQUIRE(ntables > 0 || nbuckets == 0, "buckets without tables");
  if (nbuckets == 0) return GEEK_OK;
  pack_buckets_kernel<<<grid_for(nbuckets, 1, 148 * 32), 128, 0, s>>>(flat, offsets, table_off, ntables, nbuckets,
                                                                      base, out);
  GEEK_CHECK_LAUNCH();
  return GEEK_OK;
}

}  // extern "C"
