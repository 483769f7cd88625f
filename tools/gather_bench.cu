// gather_bench.cu -- throughput of the two row-gather engines on B200 (tool,
// not part of the library).  Each CTA (one per SM) streams NSTAGE stages of
// 256 random token rows x 64 bf16 (32 KB) into a 4-deep smem ring; a consumer
// thread releases each stage once it has landed.  Modes:
//   0: TMA tile::gather4, all ops issued by ONE lane (64 ops / stage)
//   1: TMA tile::gather4, ops spread over 3 warps' lanes (uniform-register waterfall)
//   2: cp.async 16 B, W warps (W = 2, 4, 6, 8)
//   3: TMA 2-D tile loads of 128 contiguous rows (reference, 2 ops / stage)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I../paper_2312_10365_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "tc_common.cuh"
#include "tmap.h"

using namespace spt;
using namespace spt::tc;

constexpr int RING = 4, STAGE = 32768, ROWS = 256;

__global__ void __launch_bounds__(512, 1)
    gather_kernel(const __grid_constant__ CUtensorMap tg, const __grid_constant__ CUtensorMap tt,
                  const __nv_bfloat16* __restrict__ X, int d, const int* __restrict__ idx, int T,
                  int nstage, int mode, int cp_warps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + RING * STAGE);
  uint64_t* empty = full + RING;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_cp = cp_warps * 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < RING; ++s) {
      int cnt = mode == 2 ? n_cp : (mode == 1 ? 3 : 1);
      mbar_init(&full[s], cnt);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int* my_idx = idx + (size_t)blockIdx.x * ROWS * 16;  // 16 row sets, cycled
  if (warp == 0 && mode == 3) {
    if (lane == 0) {
      for (int s = 0; s < nstage; ++s) {
        const int st = s % RING;
        mbar_wait(&empty[st], ((s / RING) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[st], STAGE);
        const int r0 = (my_idx[(s % 16) * ROWS] / 128) * 128 % (T - 256);
        tma_load_2d(smem + st * STAGE, &tt, &full[st], (s % (d / 64)) * 64, r0);
        tma_load_2d(smem + st * STAGE + 16384, &tt, &full[st], (s % (d / 64)) * 64, r0 + 128);
      }
    }
  } else if (mode == 0 && warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < nstage; ++s) {
        const int st = s % RING;
        mbar_wait(&empty[st], ((s / RING) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[st], STAGE);
        const int* ix = my_idx + (s % 16) * ROWS;
        for (int c = 0; c < 64; ++c)
          tma_gather4(smem + st * STAGE + c * 512, &tg, &full[st], (s % (d / 64)) * 64, ix[4 * c],
                      ix[4 * c + 1], ix[4 * c + 2], ix[4 * c + 3]);
      }
    }
  } else if (mode == 1 && warp < 3) {
    const int c0 = lane * 3 + warp;
    const int my = (64 - warp + 2) / 3;
    for (int s = 0; s < nstage; ++s) {
      const int st = s % RING;
      if (lane == 0) {
        mbar_wait(&empty[st], ((s / RING) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[st], my * 512);
      }
      __syncwarp();
      const int* ix = my_idx + (s % 16) * ROWS;
      if (c0 < 64)
        tma_gather4(smem + st * STAGE + c0 * 512, &tg, &full[st], (s % (d / 64)) * 64, ix[4 * c0],
                    ix[4 * c0 + 1], ix[4 * c0 + 2], ix[4 * c0 + 3]);
    }
  } else if (mode == 2 && warp < cp_warps) {
    const int t = threadIdx.x;
    for (int s = 0; s < nstage; ++s) {
      const int st = s % RING;
      if (lane == 0) mbar_wait(&empty[st], ((s / RING) & 1) ^ 1);
      __syncwarp();
      const int* ix = my_idx + (s % 16) * ROWS;
      const uint32_t base = smem_u32(smem + st * STAGE);
      for (int ci = t; ci < ROWS * 8; ci += n_cp) {
        const int r = ci >> 3, ch = ci & 7;
        const __nv_bfloat16* g = X + (size_t)ix[r] * d + (s % (d / 64)) * 64 + ch * 8;
        cp_async_16(base + (r >> 7) * 16384 + (r & 127) * 128 + ((ch ^ (r & 7)) << 4), g, 16);
      }
      cp_async_arrive_noinc(&full[st]);
    }
  } else if (warp == 15 && lane == 0) {  // consumer
    for (int s = 0; s < nstage; ++s) {
      const int st = s % RING;
      mbar_wait(&full[st], (s / RING) & 1);
      mbar_arrive(&empty[st]);
    }
  }
}

int main() {
  const int d = 4096;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int T : {4096, 32768}) {
    __nv_bfloat16* X;
    cudaMalloc(&X, (size_t)T * d * 2);
    cudaMemset(X, 0, (size_t)T * d * 2);
    std::vector<int> h((size_t)nsm * ROWS * 16);
    srand(7);
    for (auto& v : h) v = rand() % T;
    int* idx;
    cudaMalloc(&idx, h.size() * 4);
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap tg, tt;
    make_tmap_bf16_2d(&tg, X, T, d, d, 64, 1);
    make_tmap_bf16_2d(&tt, X, T, d, d, 64, 128);
    const int smem = RING * STAGE + 2048;
    cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int nstage = 512;
    struct Cfg { int mode, w; const char* name; };
    Cfg cfgs[] = {{0, 0, "tma gather4, 1 lane"}, {1, 0, "tma gather4, 3 warps"},
                  {2, 2, "cp.async, 2 warps"}, {2, 4, "cp.async, 4 warps"},
                  {2, 6, "cp.async, 6 warps"}, {2, 8, "cp.async, 8 warps"},
                  {3, 0, "tma 2-D tiles (contiguous)"}};
    for (auto& c : cfgs) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        gather_kernel<<<nsm, 512, smem>>>(tg, tt, X, d, idx, T, nstage, c.mode, c.w);
        cudaEventRecord(e1);
        cudaError_t e = cudaEventSynchronize(e1);
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)nsm * nstage * STAGE;
      int clk = 0;
      cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      printf("T=%6d %-28s %8.3f ms  %7.1f GB/s  %6.1f B/cyc/SM (@%.2f GHz)\n", T, c.name, ms,
             bytes / ms / 1e6, bytes / nsm / (ms * 1e-3 * clk * 1e3), clk / 1e6);
    }
    cudaFree(X);
    cudaFree(idx);
  }
  return 0;
}
