// l2_reduce_bench.cu -- can the FWD2 / dX epilogue add its per-pair output rows
// straight into an L2-resident fp32 token-row accumulator instead of writing
// bf16 partial rows to HBM for a separate combine pass?  (tool, not part of the
// library).  Emulates the epilogue of the weight-resident grouped GEMM at
// LLaMA scale: T*k/128 m-tiles x d/256 N tiles, each tile 128 rows x 256 fp32
// columns, 8 epilogue warps per CTA (warp = 32 rows x 128 columns), one CTA per
// SM.  Tile rows map to token rows scattered inside a token window of Wt tokens
// (tiles ordered window-major, N-tile-major inside a window, as a windowed unit
// schedule would run them).  Modes:
//   0: 1-D bulk reduce-add f32 (cp.reduce.async.bulk .add.f32), one 256-B op per
//      (row, 64 columns), padded row-major staging (272-B rows, conflict-free)
//   1: 2-D tensor reduce-add f32 with tile::scatter4 (4 token rows x 32 columns
//      = 512 B per op), 128-B swizzled staging
//   2: mode 0 without the reduction (plain 1-D bulk stores, same addresses)
//   3: reference: bf16 2-D TMA tile stores of 32 contiguous partial rows x 64
//      columns (what the FWD2 epilogue does today; partials [T*k, d])
//   4: red.global.add.v4.f32 from registers after an smem transpose (16 lanes
//      per 256-B row segment)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I../paper_2312_10365_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"
#include "tmap.h"

using namespace spt;
using namespace spt::tc;

constexpr int kWarps = 8, kPad = 272;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

__global__ void __launch_bounds__(256, 1)
    red_kernel(const __grid_constant__ CUtensorMap tmr, const __grid_constant__ CUtensorMap tmp,
               float* __restrict__ acc, int T, int d, int ntiles, int tiles_per_win, int mtiles_per_win,
               int Wt, int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, half = warp >> 2;
  uint8_t* buf0 = smem + warp * 2 * 9216;  // two 32-row x 64-col fp32 buffers (padded, 1 KB aligned)
  int bi = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int w = tile / tiles_per_win, ti = tile % tiles_per_win;
    const int nt = ti / mtiles_per_win, mt = ti % mtiles_per_win;
    const int row = q * 32 + lane;
    const int tok = w * Wt + (int)(hash32((uint32_t)(tile * 128 + row) * 2654435761u) % (uint32_t)Wt);
    for (int c0 = half * 128; c0 < half * 128 + 128; c0 += 64) {
      uint8_t* buf = buf0 + bi * 9216;
      bulk_wait_read<1>();  // bulk groups are per thread: every issuing lane waits for its own
      __syncwarp();
      float v[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = (float)((tile + i + lane) & 7) * 0.25f;
      if (mode == 0 || mode == 2 || mode == 4) {
#pragma unroll
        for (int c = 0; c < 16; ++c)
          *reinterpret_cast<float4*>(buf + lane * kPad + c * 16) =
              make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
      } else if (mode == 1) {
        // two 32-row x 32-col swizzled boxes (128-B rows): chunk c of row r at r*128 + ((c ^ (r&7))<<4)
#pragma unroll
        for (int hb = 0; hb < 2; ++hb)
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<float4*>(buf + hb * 4096 + lane * 128 + ((c ^ (lane & 7)) << 4)) =
                make_float4(v[32 * hb + 4 * c], v[32 * hb + 4 * c + 1], v[32 * hb + 4 * c + 2],
                            v[32 * hb + 4 * c + 3]);
      } else {  // mode 3: bf16 32 x 64 swizzled box
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(buf + lane * 128 + ((c ^ (lane & 7)) << 4)) =
              make_uint4(pack_bf16(v[8 * c], v[8 * c + 1]), pack_bf16(v[8 * c + 2], v[8 * c + 3]),
                         pack_bf16(v[8 * c + 4], v[8 * c + 5]), pack_bf16(v[8 * c + 6], v[8 * c + 7]));
      }
      fence_proxy_async_smem();
      __syncwarp();
      const int col = nt * 256 + c0;
      if (mode == 0 || mode == 2) {
        float* g = acc + (int64_t)tok * d + col;
        const uint32_t s = smem_u32(buf + lane * kPad);
        if (mode == 0)
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 256;" ::"l"(g),
                       "r"(s) : "memory");
        else
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 256;" ::"l"(g), "r"(s)
                       : "memory");
        bulk_commit();
      } else if (mode == 1) {
        // lanes 0..7: scatter4 op for rows 4l..4l+3, box halves hb = lane>>3 & 1 ... 16 ops per chunk
        const int quad = lane & 7, hb = (lane >> 3) & 1;
        int t4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) t4[i] = __shfl_sync(0xffffffffu, tok, 4 * quad + i);
        if (lane < 16) {
          asm volatile(
              "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile::scatter4.bulk_group"
              " [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(&tmr),
              "r"(smem_u32(buf + hb * 4096 + quad * 512)), "r"(col + hb * 32), "r"(t4[0]), "r"(t4[1]),
              "r"(t4[2]), "r"(t4[3])
              : "memory");
          bulk_commit();
        }
      } else if (mode == 3) {
        if (lane == 0) {
          const int prow = (w * mtiles_per_win + mt) * 128 + q * 32;
          tma_store_2d(&tmp, buf, col, prow);
          bulk_commit();
        }
      } else {  // mode 4: transpose through smem, red.v4 (16 lanes per row segment)
#pragma unroll 4
        for (int r2 = 0; r2 < 32; r2 += 2) {
          const int rr = r2 + (lane >> 4), c = lane & 15;
          const int tr = __shfl_sync(0xffffffffu, tok, rr);
          const float4 x = *reinterpret_cast<const float4*>(buf + rr * kPad + c * 16);
          float* g = acc + (int64_t)tr * d + col + c * 4;
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(g), "f"(x.x), "f"(x.y),
                       "f"(x.z), "f"(x.w) : "memory");
        }
      }
      bi ^= 1;
    }
  }
  bulk_wait<0>();
}

int main(int argc, char** argv) {
  const int T = 32768, d = 4096, k = 22;
  const int rows = T * k;                       // pairs
  const int mtiles = rows / 128;                // 5632
  const int NT = d / 256;
  float* acc;
  __nv_bfloat16* part;
  cudaMalloc(&acc, (size_t)T * d * 4);
  cudaMalloc(&part, (size_t)(rows + 128) * d * 2);
  cudaMemset(acc, 0, (size_t)T * d * 4);
  CUtensorMap tmr, tmp;
  {
    auto fn = get_encode_fn();
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)T};
    cuuint64_t strides[1] = {(cuuint64_t)d * 4};
    cuuint32_t box[2] = {32, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(&tmr, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, acc, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("tmr encode failed %d\n", (int)r);
  }
  if (!make_tmap_bf16_2d(&tmp, part, rows + 128, d, d, 64, 32)) printf("tmp encode failed\n");
  const int smem = kWarps * 2 * 9216 + 1024;
  cudaFuncSetAttribute(red_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"bulk-reduce f32 256B", "tensor-reduce scatter4 f32", "bulk-store f32 256B",
                         "bf16 TMA store partials (today)", "red.global.add.v4.f32"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int wins[] = {1024, 2048, 4096, 8192, 32768};
  for (int mode = 0; mode < 5; ++mode) {
    for (int wi = 0; wi < 5; ++wi) {
      const int Wt = wins[wi];
      if (mode == 3 && wi > 0) break;
      const int mpw = mtiles / (T / Wt);  // m-tiles per window
      const int tpw = mpw * NT;
      const int ntiles = tpw * (T / Wt);
      float best = 1e9;
      for (int it = 0; it < 4; ++it) {
        cudaEventRecord(e0);
        red_kernel<<<nsm, 256, smem>>>(tmr, tmp, acc, T, d, ntiles, tpw, mpw, Wt, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it) best = ms < best ? ms : best;
      }
      cudaError_t e = cudaGetLastError();
      const double bytes = (double)ntiles * 128 * 256 * (mode == 3 ? 2 : 4);
      printf("mode %d %-32s window %5d tok (acc %4.0f MB/win-slice %5.1f MB): %.3f ms  %.0f GB/s  %s\n",
             mode, names[mode], Wt, (double)Wt * d * 4 / 1e6, (double)Wt * 256 * 4 / 1e6, best,
             bytes / best / 1e6, cudaGetErrorString(e));
    }
  }
  return 0;
}
