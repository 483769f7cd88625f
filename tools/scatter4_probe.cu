// scatter4_probe.cu -- checks the TMA tile::scatter4 reduce-add element layout
// (tool): one warp stages 32 rows x 32 fp32 (row = lane, 128-byte swizzle by
// row & 7) and lanes 0..7 each reduce-add 4 rows into token rows of acc.
#include <cstdio>
#include <vector>
#include "tc_common.cuh"
#include "tmap.h"
using namespace spt;
using namespace spt::tc;

__global__ void probe(const __grid_constant__ CUtensorMap m, int mode) {
  __shared__ __align__(1024) uint8_t buf[4096];
  const int lane = threadIdx.x;
  float v[32];
  for (int i = 0; i < 32; ++i) v[i] = lane * 100 + i;  // row lane, column i
  for (int c = 0; c < 8; ++c) {
    const int cc = mode == 1 ? c : (c ^ (lane & 7));
    *reinterpret_cast<float4*>(buf + lane * 128 + (cc << 4)) =
        make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  }
  fence_proxy_async_smem();
  __syncwarp();
  const int tok = 2 * lane + 1;  // token row of tile row `lane`
  int t4[4];
  for (int i = 0; i < 4; ++i) t4[i] = __shfl_sync(0xffffffffu, tok, 4 * (lane & 7) + i);
  if (lane < 8) {
    for (int rep = 0; rep < 3; ++rep) {  // three adds: acc = 3 x the row
      tma_reduce_add_scatter4(&m, buf + lane * 512, 32, t4[0], t4[1], t4[2], t4[3]);
      bulk_commit();
      bulk_wait<0>();
    }
  }
}

int main() {
  const int T = 80, d = 96;
  float* acc;
  cudaMalloc(&acc, T * d * 4);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(acc, 0, T * d * 4);
    CUtensorMap m;
    if (!make_tmap_f32_2d_sw128(&m, acc, T, d, d, 1)) { printf("encode failed\n"); return 1; }
    probe<<<1, 32>>>(m, mode);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> h(T * d);
    cudaMemcpy(h.data(), acc, T * d * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int t = 0; t < T; ++t)
      for (int c = 0; c < d; ++c) {
        float want = 0;
        if (t % 2 == 1 && t / 2 < 32 && c >= 32 && c < 64) want = 3.f * ((t / 2) * 100 + (c - 32));
        if (h[t * d + c] != want) {
          if (bad < 8) printf("mode %d t %d c %d got %g want %g\n", mode, t, c, h[t * d + c], want);
          ++bad;
        }
      }
    printf("mode %d (%s): %s, %d mismatches\n", mode, mode ? "unswizzled" : "swizzled",
           cudaGetErrorString(e), bad);
  }
  return 0;
}
