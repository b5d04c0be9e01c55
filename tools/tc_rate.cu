// Microbenchmark: tcgen05.mma kind::tf32 issue rate for M=128 and N in
// {64, 128, 256}, A from SMEM or TMEM, B from SMEM; one CTA per SM issuing
// back-to-back MMAs into one accumulator (operands are zeros).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_rate.bin tools/tc_rate.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, bool ATMEM>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, unsigned long long* cyc, int commit_every) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, cbar[4];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (16 * 1024 + N * 32 * 4) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    for (int q = 0; q < 4; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&cbar[q])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    uint32_t pred;
    asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}\n" : "=r"(pred));
    const uint32_t id = idesc(128, N);
    const uint64_t a = sdesc(su32(sm)), b = sdesc(su32(sm + 16 * 1024));
    const uint32_t at = tmem + 256;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (pred) {
        if (ATMEM)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(tmem), "r"(at), "l"(b), "r"(id), "r"(1));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem), "l"(a), "l"(b), "r"(id), "r"(1));
      }
      if (commit_every && (it + 1) % commit_every == 0 && pred)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            su32(&cbar[(it / commit_every) & 3])) : "memory");
      __syncwarp();
    }
    if (pred) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    __syncwarp();
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)) : "memory");
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// the screen's operand mix: per K=8 slice hi*hi (A TMEM), hi*lo (A TMEM),
// lo*hi (A SMEM), walking 4 slices of a 32 KB B stage and 3 stages
__global__ void __launch_bounds__(288, 1) mix_kernel(int iters, int spread, int commit, int spin, const float* gsrc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, cb[4], never, tb;
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  for (int i = threadIdx.x; i < (64 * 1024 + 96 * 1024) / 4; i += blockDim.x) {
    uint32_t z = i * 2654435761u + 12345u;
    z ^= z >> 13;
    z *= 0x5bd1e995u;
    z ^= z >> 15;
    reinterpret_cast<float*>(sm)[i] = spread >= 2 ? __uint_as_float((z & 0x807FE000u) | 0x3F800000u) : 0.f;
  }
  if (threadIdx.x == 0) done = 0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    for (int q = 0; q < 4; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&cb[q])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&never)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&tb)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    uint32_t pred;
    asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}\n" : "=r"(pred));
    const uint32_t id = idesc(128, 128);
    const uint32_t alo = su32(sm), bb = su32(sm + 64 * 1024);
    for (int it = 0; it < iters; ++it) {
      const int st = spread ? it % 3 : 0;
      if (pred) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (spin == 3 && j == 0) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (spin == 4 && j == 0) {
              asm volatile("{\n.reg .pred p;\nW4: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 1;\n@!p bra W4;\n}\n" ::"r"(su32(&never)) : "memory");
              asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            const int ks = spread ? c * 4 + j : 0;
            const uint64_t bhi = sdesc(bb + st * 32768 + (spread ? j : 0) * 4096);
            const uint64_t blo = sdesc(bb + st * 32768 + 16384 + (spread ? j : 0) * 4096);
            const uint64_t a = sdesc(alo + ks * 4096);
            const uint32_t at = tmem + 256 + ks * 8;
            const uint32_t dd = tmem + ((spin == 5) ? (it & 1) * 128 : 0);
            const uint32_t en = (spin == 6 && c == 0 && j == 0) ? 0u : 1u;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dd), "r"(at), "l"(bhi), "r"(id), "r"(en));
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dd), "r"(at), "l"(blo), "r"(id));
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dd), "l"(a), "l"(bhi), "r"(id));
            if (commit && j == 3)
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&cb[c])) : "memory");
          }
      }
      __syncwarp();
    }
    if (pred) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    __syncwarp();
    asm volatile("{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W2;\n}\n" ::"r"(su32(&bar)) : "memory");
    if (threadIdx.x == 0) done = 1;
  } else if (spin == 1 && threadIdx.x >= 64) {  // 7 warps polling an mbarrier that stays open
    while (!done) {
      uint32_t ok;
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.b32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(su32(&never)) : "memory");
    }
  } else if (spin == 2 && threadIdx.x == 32) {  // bulk copies streaming 32 KB into a spare SMEM region
    uint32_t ph = 0;
    while (!done) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&tb)), "r"(32768) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sm + 128 * 1024)), "l"(gsrc), "r"(32768), "r"(su32(&tb)) : "memory");
      asm volatile("{\n.reg .pred p;\nW3: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W3;\n}\n" ::"r"(su32(&tb)), "r"(ph) : "memory");
      ph ^= 1;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

void run_mix(int sms, int spread, int commit, int spin = 0) {
  static float* g = nullptr;
  if (!g) cudaMalloc(&g, 1 << 20);
  const int iters = getenv("MIX_ITERS") ? atoi(getenv("MIX_ITERS")) : 500, smem = 160 * 1024 + 1024;
  cudaFuncSetAttribute(mix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mix_kernel<<<sms, 288, smem>>>(10, spread, commit, spin, g);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix_kernel<<<sms, 288, smem>>>(iters, spread, commit, spin, g);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 128 * 128 * 8 * 48.0 * iters * sms;
  printf("mix spread=%d commit=%d spin=%d: %.1f TFLOP/s (%.2f ms) err=%s\n", spread, commit, spin, flops / ms / 1e9, ms, cudaGetErrorString(err));
}

template <int N, bool ATMEM>
void run(int sms, int ce = 0) {
  const int iters = 20000;
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  const int smem = 16 * 1024 + N * 32 * 4 + 1024;
  cudaFuncSetAttribute(rate_kernel<N, ATMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  rate_kernel<N, ATMEM><<<sms, 128, smem>>>(100, d, ce);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  rate_kernel<N, ATMEM><<<sms, 128, smem>>>(iters, d, ce);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double flops = 2.0 * 128 * N * 8 * (double)iters * sms;
  printf("commit/%d N=%d A=%s: %.1f TFLOP/s (%.2f ms), %.1f cycles/MMA on SM0, err=%s\n", ce, N, ATMEM ? "tmem" : "smem",
         flops / ms / 1e9, ms, (double)h / iters, cudaGetErrorString(err));
  cudaFree(d);
}

int main_mix() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<128, true>(sms);
  run_mix(sms, 2, 1, 0);
  run_mix(sms, 2, 1, 5);
  run_mix(sms, 2, 1, 6);
  return 0;
}

// the screen's B-ring protocol without data: S stages, a producer warp that
// waits "empty" (MMA commit) and arrives "full", an MMA warp that waits
// "full", issues one chunk (12 MMAs) and commits "empty"
template <int S, int H>
__global__ void __launch_bounds__(128, 1) ring_kernel(int chunks) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[S], empty[S], done, accf[2], acce[2];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (64 * 1024 + 96 * 1024) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int q = 0; q < S; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[q])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[q])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&done)));
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&accf[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 64;" ::"r"(su32(&acce[b])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  const int warp = threadIdx.x >> 5;
  const int cts = chunks / 4;  // 4 chunks per accumulator tile
  uint32_t pred;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}\n" : "=r"(pred));
  if (warp == 1) {  // producer
    for (int q = 0; q < chunks; ++q) {
      const int s = q % S;
      if (q >= S)
        asm volatile("{\n.reg .pred p;\nWE: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WE;\n}\n" ::"r"(
                         su32(&empty[s])), "r"(((q / S) - 1) & 1) : "memory");
      if (pred) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
      __syncwarp();
    }
  } else if (warp >= 2) {  // epilogue stand-ins: wait for an accumulator, hand it back
    if (H)
      for (int g = 0; g < cts; ++g) {
        const int b = g & 1;
        asm volatile("{\n.reg .pred p;\nWA: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WA;\n}\n" ::"r"(
                         su32(&accf[b])), "r"((g >> 1) & 1) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&acce[b])) : "memory");
      }
  } else if (warp == 0) {  // MMA issuer
    const uint32_t id = idesc(128, 128);
    const uint32_t alo = su32(sm), bb = su32(sm + 64 * 1024);
    for (int q = 0; q < chunks; ++q) {
      const int s = q % S;
      const int g = q / 4, b = g & 1;
      if (H && (q & 3) == 0) {
        asm volatile("{\n.reg .pred p;\nWB: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WB;\n}\n" ::"r"(
                         su32(&acce[b])), "r"(((g >> 1) & 1) ^ 1) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      const uint32_t dacc = tmem + (H ? b * 128 : 0);
      asm volatile("{\n.reg .pred p;\nWF: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WF;\n}\n" ::"r"(
                       su32(&full[s])), "r"((q / S) & 1) : "memory");
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (pred) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t bhi = sdesc(bb + (s % 3) * 32768 + j * 4096), blo = sdesc(bb + (s % 3) * 32768 + 16384 + j * 4096);
          const uint64_t a = sdesc(alo + ((q & 3) * 4 + j) * 4096);
          const uint32_t at = tmem + 256 + ((q & 3) * 4 + j) * 8;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dacc), "r"(at), "l"(bhi), "r"(id));
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dacc), "r"(at), "l"(blo), "r"(id));
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dacc), "l"(a), "l"(bhi), "r"(id));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&empty[s])) : "memory");
        if (H && (q & 3) == 3)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&accf[b])) : "memory");
      }
      __syncwarp();
    }
    if (pred) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&done)) : "memory");
    __syncwarp();
    asm volatile("{\n.reg .pred p;\nWD: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra WD;\n}\n" ::"r"(su32(&done)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int S, int H>
void run_ring(int sms) {
  const int chunks = 20000, smem = 160 * 1024 + 1024;
  cudaFuncSetAttribute(ring_kernel<S, H>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  ring_kernel<S, H><<<sms, 128, smem>>>(100);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  ring_kernel<S, H><<<sms, 128, smem>>>(chunks);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 128 * 128 * 8 * 12.0 * chunks * sms;
  printf("ring stages=%d handshake=%d: %.1f TFLOP/s (%.2f ms) err=%s\n", S, H, flops / ms / 1e9, ms, cudaGetErrorString(err));
}

int main_ring() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run_ring<3, 0>(sms);
  run_ring<3, 1>(sms);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == 'r') return main_ring();
  return main_mix();
}
