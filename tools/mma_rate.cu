// mma_rate.cu -- raw tcgen05.mma throughput on B200 (tool, not the library).
// One CTA per SM; one thread issues back-to-back kind::f16 MMAs (bf16 -> fp32)
// from fixed 128B-swizzled smem operands into TMEM, committing to an mbarrier
// every `per_commit` MMAs.  Reports FLOP/clk/SM vs the 8192 nominal.
// Variants: N = 64/128/256, M halves (1 or 2 accumulators sharing B), K-major
// vs MN-major B.
#include <cstdio>
#include "tc_common.cuh"

using namespace spt::tc;

__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, int N, int MH, int bmn,
                                                      long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16(128, N, false, bmn != 0);
    const uint32_t sa = smem_u32(smem), sb = sa + 32768;
    const long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t bd = bmn ? sdesc_sw128(sb + k * 2048, 8192, 1024) : sdesc_sw128(sb + k * 32, 16, 1024);
        for (int h = 0; h < MH; ++h)
          mma_bf16(tmem + h * 256, sdesc_sw128(sa + h * 16384 + k * 32, 16, 1024), bd, idesc,
                   (it | k) != 0);
      }
      if ((it & 63) == 63) {  // commit + wait every 64 stages
        mma_commit(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, ph);
    cycles[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// CTA-pair variant: cluster of 2, M = 256 (128 rows per CTA), each CTA holds
// its half of A and N/2 rows of B at the same smem offsets; the leader issues
// tcgen05.mma.cta_group::2 and commits to both CTAs' barriers.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma2_kernel(int iters, int N, int MH, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t idesc = idesc_bf16(256, N, false, false);
    const uint32_t sa = smem_u32(smem), sb = sa + 32768;
    const long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t bd = sdesc_sw128(sb + k * 32, 16, 1024);
        for (int h = 0; h < MH; ++h) {
          const uint64_t ad = sdesc_sw128(sa + h * 16384 + k * 32, 16, 1024);
          const uint32_t acc = (it | k) != 0;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + h * 256),
              "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
              : "memory");
        }
      }
      if ((it & 63) == 63) {
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"((uint16_t)3)
            : "memory");
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)3)
        : "memory");
    mbar_wait(&bar, ph);
    cycles[blockIdx.x] = clock64() - t0;
  }
  if (threadIdx.x == 0 && rank == 1) {  // peer: consume the same commits to keep phases aligned
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it)
      if ((it & 63) == 63) { mbar_wait(&bar, ph); ph ^= 1; }
    mbar_wait(&bar, ph);
    cycles[blockIdx.x] = 0;
  }
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// Ring variant: the library's stage protocol without data.  `stages` stage
// barriers; producers (nprod threads of warps 2.., one arrival each, plus the
// optional cp.async-style noinc arrival) wait empty[s] then arrive on full[s];
// the MMA thread waits full[s], issues 4 x MH MMAs (N=256), commits empty[s].
// Every `tile_k` stages it commits to tfull and waits for it (accumulator drain).
__global__ void __launch_bounds__(512, 1) ring_kernel(int iters, int stages, int nprod, int MH,
                                                      int tile_k, int noinc, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[8], empty[8], tfull;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], nprod);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int pt = threadIdx.x - 64;
  if (threadIdx.x == 32) {
    const uint32_t idesc = idesc_bf16(128, 256, false, false);
    const uint32_t sa0 = smem_u32(smem);
    const long long t0 = clock64();
    int stage = 0;
    uint32_t ph = 0, tph = 0;
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&full[stage], ph);
      const uint32_t sa = sa0 + stage * 65536u, sb = sa + 32768;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t bd = sdesc_sw128(sb + k * 32, 16, 1024);
        for (int h = 0; h < MH; ++h)
          mma_bf16(tmem + h * 256, sdesc_sw128(sa + h * 16384 + k * 32, 16, 1024), bd, idesc,
                   (it | k) != 0);
      }
      mma_commit(&empty[stage]);
      if (++stage == stages) { stage = 0; ph ^= 1; }
      if (tile_k > 0 && (it % tile_k) == tile_k - 1) {
        mma_commit(&tfull);
        mbar_wait(&tfull, tph);
        tph ^= 1;
      }
    }
    mma_commit(&tfull);
    mbar_wait(&tfull, tph);
    cycles[blockIdx.x] = clock64() - t0;
  } else if (pt >= 0 && pt < nprod) {
    int stage = 0;
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&empty[stage], ph ^ 1);
      if (noinc) {
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[stage]))
                     : "memory");
      } else {
        mbar_arrive(&full[stage]);
      }
      if (++stage == stages) { stage = 0; ph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, nsm * sizeof(long long));
  {
    const int rsmem = 1024 + 3 * 65536;
    cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, rsmem);
    struct R { int stages, nprod, MH, tile_k, noinc; } rs[] = {
        {3, 1, 2, 0, 0},   {3, 1, 2, 64, 0},  {3, 131, 2, 64, 0}, {3, 131, 2, 64, 1},
        {2, 1, 2, 64, 0},  {3, 1, 1, 64, 0},  {3, 131, 1, 64, 1}};
    for (auto c : rs) {
      const int iters = 4096;
      ring_kernel<<<nsm, 512, rsmem>>>(64, c.stages, c.nprod, c.MH, c.tile_k, c.noinc, d);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      ring_kernel<<<nsm, 512, rsmem>>>(iters, c.stages, c.nprod, c.MH, c.tile_k, c.noinc, d);
      cudaEventRecord(e1);
      cudaError_t err = cudaEventSynchronize(e1);
      if (err != cudaSuccess) { printf("ring error %s\n", cudaGetErrorString(err)); return 1; }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      long long h[1024];
      cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int i = 0; i < nsm; ++i) cyc += h[i];
      cyc /= nsm;
      const double flop_sm = 2.0 * 128 * 256 * 64 * c.MH * iters;
      printf("RING stages=%d nprod=%3d MH=%d tile_k=%2d noinc=%d: %.0f%% of 8192 FLOP/clk/SM (%.3f ms)\n",
             c.stages, c.nprod, c.MH, c.tile_k, c.noinc, 100 * flop_sm / cyc / 8192, ms);
    }
  }
  const int smem = 1024 + 32768 + 32768;
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct C { int N, MH, bmn; } cs[] = {{64, 1, 0}, {128, 1, 0}, {256, 1, 0}, {128, 2, 0},
                                       {256, 2, 0}, {256, 1, 1}, {128, 2, 1}};
  for (auto c : cs) {
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    mma_kernel<<<nsm, 128, smem>>>(64, c.N, c.MH, c.bmn, d);
    cudaEventRecord(e0);
    mma_kernel<<<nsm, 128, smem>>>(iters, c.N, c.MH, c.bmn, d);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) { printf("error\n"); return 1; }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[1024];
    cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < nsm; ++i) cyc += h[i];
    cyc /= nsm;
    const double flop_sm = 2.0 * 128 * c.N * 64 * c.MH * iters;
    printf("N=%3d MH=%d Bmn=%d: %.1f FLOP/clk/SM (%.0f%% of 8192), %.0f TFLOP/s chip (%.3f ms)\n", c.N,
           c.MH, c.bmn, flop_sm / cyc, 100 * flop_sm / cyc / 8192, flop_sm * nsm / ms / 1e9, ms);
  }
  // CTA pairs: per SM work = 128 rows x N x K per instruction
  cudaFuncSetAttribute(mma2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct C2 { int N, MH; } c2s[] = {{128, 1}, {256, 1}, {256, 2}, {128, 2}};
  for (auto c : c2s) {
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    mma2_kernel<<<nsm, 128, smem>>>(64, c.N, c.MH, d);
    cudaEventRecord(e0);
    mma2_kernel<<<nsm, 128, smem>>>(iters, c.N, c.MH, d);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    if (err != cudaSuccess) { printf("pair error %s\n", cudaGetErrorString(err)); return 1; }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[1024];
    cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
    double cyc = 0;
    int n = 0;
    for (int i = 0; i < nsm; ++i) if (h[i] > 0) { cyc += h[i]; ++n; }
    cyc /= n;
    const double flop_sm = 2.0 * 128 * c.N * 64 * c.MH * iters;  // per SM
    printf("PAIR N=%3d MH=%d: %.1f FLOP/clk/SM (%.0f%% of 8192), %.0f TFLOP/s chip (%.3f ms)\n", c.N, c.MH,
           flop_sm / cyc, 100 * flop_sm / cyc / 8192, flop_sm * nsm / ms / 1e9, ms);
  }
  return 0;
}
