// tc_probe.cu -- hardware probe for the tcgen05 / TMA building blocks used by
// the product kernels (not part of the library).  Runs three single-CTA GEMMs
// D[128 x N] = A * B^T through tc_common.cuh and compares against a CPU loop:
//   mode 0: A K-major gathered rows (TMA gather4, one OOB row -> zeros), B K-major tile
//   mode 1: A K-major tile, B MN-major tile (N contiguous)
//   mode 2: A MN-major tile (M contiguous), B MN-major gathered along K (gather4)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O2 -I../paper_2312_10365_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "tc_common.cuh"
#include "tmap.h"

using namespace spt;
using namespace spt::tc;

constexpr int M = 128, N = 256, KB = 64;

template <int MODE>
__global__ void __launch_bounds__(128, 1)
    probe(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
          const int* idx, float* D, int K) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;              // 16 KB
  uint8_t* sB = smem + 16384;      // 32 KB
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16(M, N, MODE == 2, MODE >= 1);
    for (int kb = 0; kb < K / KB; ++kb) {
      mbar_arrive_expect_tx(&bar_load, 16384 + 32768);
      if (MODE == 0) {
        for (int r = 0; r < M; r += 4)
          tma_gather4(sA + r * 128, &ta, &bar_load, kb * KB, idx[r], idx[r + 1], idx[r + 2],
                      idx[r + 3]);
        tma_load_2d(sB, &tb, &bar_load, kb * KB, 0);
      } else if (MODE == 1) {
        tma_load_2d(sA, &ta, &bar_load, kb * KB, 0);
        for (int j = 0; j < N / 64; ++j) tma_load_2d(sB + j * 8192, &tb, &bar_load, j * 64, kb * KB);
      } else {
        for (int j = 0; j < M / 64; ++j) tma_load_2d(sA + j * 8192, &ta, &bar_load, j * 64, kb * KB);
        for (int j = 0; j < N / 64; ++j)
          for (int r = 0; r < KB; r += 4) {
            const int* ix = idx + kb * KB + r;
            tma_gather4(sB + j * 8192 + r * 128, &tb, &bar_load, j * 64, ix[0], ix[1], ix[2], ix[3]);
          }
      }
      mbar_wait(&bar_load, kb & 1);
      tc_fence_after();
      for (int k = 0; k < KB / 16; ++k) {
        uint64_t ad, bd;
        if (MODE == 2) ad = sdesc_sw128(smem_u32(sA) + k * 2048, 8192, 1024);
        else ad = sdesc_sw128(smem_u32(sA) + k * 32, 16, 1024);
        if (MODE == 0) bd = sdesc_sw128(smem_u32(sB) + k * 32, 16, 1024);
        else bd = sdesc_sw128(smem_u32(sB) + k * 2048, 8192, 1024);
        mma_bf16(tmem, ad, bd, idesc, (kb | k) != 0);
      }
      mma_commit(&bar_mma);
      mbar_wait(&bar_mma, kb & 1);
    }
  }
  __syncthreads();
  tc_fence_after();
  const int row = warp * 32 + (threadIdx.x & 31);
  for (int c = 0; c < N; c += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) D[row * N + c + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

static float bf(float v) {  // round to bf16
  __nv_bfloat16 b = __float2bfloat16(v);
  return __bfloat162float(b);
}

int run(int mode) {
  const int K = 256, R = 300;  // R rows in the gathered source
  // Host matrices (float holding bf16 values)
  std::vector<float> A, B;
  std::vector<int> idx;
  srand(1234 + mode);
  auto rnd = [] { return bf((rand() / (float)RAND_MAX - 0.5f) * 2.f); };
  int a_rows, a_cols, b_rows, b_cols;
  if (mode == 0) { a_rows = R; a_cols = K; b_rows = N; b_cols = K; }
  else if (mode == 1) { a_rows = M; a_cols = K; b_rows = K; b_cols = N; }
  else { a_rows = K; a_cols = M; b_rows = R; b_cols = N; }
  A.resize(a_rows * a_cols); B.resize(b_rows * b_cols);
  for (auto& v : A) v = rnd();
  for (auto& v : B) v = rnd();
  int nidx = mode == 0 ? M : K;
  idx.resize(nidx);
  for (int i = 0; i < nidx; ++i) idx[i] = (i * 37 + 11) % R;
  idx[5] = R + 3;  // out of bounds -> expect zero fill
  std::vector<__nv_bfloat16> Ab(A.size()), Bb(B.size());
  for (size_t i = 0; i < A.size(); ++i) Ab[i] = __float2bfloat16(A[i]);
  for (size_t i = 0; i < B.size(); ++i) Bb[i] = __float2bfloat16(B[i]);
  __nv_bfloat16 *dA, *dB; float* dD; int* didx;
  cudaMalloc(&dA, Ab.size() * 2); cudaMalloc(&dB, Bb.size() * 2);
  cudaMalloc(&dD, M * N * 4); cudaMalloc(&didx, nidx * 4);
  cudaMemcpy(dA, Ab.data(), Ab.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bb.data(), Bb.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(didx, idx.data(), nidx * 4, cudaMemcpyHostToDevice);
  CUtensorMap ta, tb;
  bool ok = true;
  if (mode == 0) {
    ok &= make_tmap_bf16_2d(&ta, dA, R, K, K, 64, 1);
    ok &= make_tmap_bf16_2d(&tb, dB, N, K, K, 64, N);
  } else if (mode == 1) {
    ok &= make_tmap_bf16_2d(&ta, dA, M, K, K, 64, M);
    ok &= make_tmap_bf16_2d(&tb, dB, K, N, N, 64, 64);
  } else {
    ok &= make_tmap_bf16_2d(&ta, dA, K, M, M, 64, 64);
    ok &= make_tmap_bf16_2d(&tb, dB, R, N, N, 64, 1);
  }
  if (!ok) { printf("mode %d: tensor map encode failed\n", mode); return 1; }
  // host copy of idx for the kernel (it reads idx from global)
  const int smem = 1024 + 16384 + 32768;
  void (*kern)(CUtensorMap, CUtensorMap, const int*, float*, int) =
      mode == 0 ? probe<0> : mode == 1 ? probe<1> : probe<2>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<1, 128, smem>>>(ta, tb, didx, dD, K);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e)); return 1; }
  std::vector<float> D(M * N);
  cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) {
        double a, b;
        if (mode == 0) { a = idx[m] < R ? A[idx[m] * K + k] : 0.0; b = B[n * K + k]; }
        else if (mode == 1) { a = A[m * K + k]; b = B[k * N + n]; }
        else { a = A[k * M + m]; b = idx[k] < R ? B[idx[k] * N + n] : 0.0; }
        s += a * b;
      }
      double err = fabs(s - D[m * N + n]);
      if (err > 1e-3 * (1 + fabs(s))) { if (bad < 5) printf("  m%d n%d ref %f got %f\n", m, n, s, D[m * N + n]); ++bad; }
      maxerr = fmax(maxerr, err); maxref = fmax(maxref, fabs(s));
    }
  printf("mode %d: %s  maxerr %.3e (maxref %.3f) bad %d\n", mode, bad ? "FAIL" : "PASS", maxerr, maxref, bad);
  return bad ? 1 : 0;
}

int main() {
  int fails = 0;
  for (int mode = 0; mode < 3; ++mode) fails += run(mode);
  printf(fails ? "PROBE FAILED\n" : "PROBE OK\n");
  return fails;
}
