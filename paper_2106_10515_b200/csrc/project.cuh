// K1's key destinations (shared by the DMMA stream kernel, project.cu, and
// the tcgen05 projection, tc_project.cu).
#pragma once
#include "common.cuh"

namespace geek {

// Where table t's key of local point p goes: dst[t % G] + (t / G) * ntot +
// row_lo + p.  G = 1 is the local [m][n] array; G > 1 stores every key
// straight into its owner rank's buffer (peer memory over NVLink), which is
// the bucket synchronisation of engine.py:199-238 without a separate
// all-to-all.
constexpr int kMaxKeyDst = 8;
constexpr int kMaxKeyTables = 48;
struct KeyDst {
  uint64_t* ptr[kMaxKeyDst];
  int G;
  uint64_t ntot, row_lo;
  uint64_t* tptr[kMaxKeyTables];  // table t's row-0 address for this shard (host-computed)
  int vec16;                      // every tptr is 16-byte aligned: 16-byte stores
  // optional fused fine-bin histogram of the rank split (fine_hist_kernel's
  // count, done here while the key is in a register): cinfo [m][2^cb] of
  // (fine bins, first global fine bin) per coarse cell, counters fcnt
  const uint2* cinfo;
  uint32_t* fcnt;
  int cb;
};

// The tcgen05 integer-digit projection (tc_project.cu).  Returns GEEK_OK with
// *used = false when the shape is outside its range (the caller then runs the
// DMMA stream kernel).
int tc_project_launch(const float* X, uint64_t n, int d, const double* A, int m, const KeyDst& dst, int* er,
                      unsigned* nf, cudaStream_t s, bool* used);

}  // namespace geek
