// combine.cu -- a6 weighted scatter-add combine and the a8 grad-input combine
// (SURVEY §8(a)).  HBM-bound: each token reads its k per-block partial rows and
// writes one output row; fp32 accumulation in ascending block order (reading
// c12), so results are deterministic and independent of the GEMM schedule.
//
//   y[t]  = sum_{j asc} P[prow(t,j)]                        (Alg. 4 line 5, c1)
//   dx[t] = sum_{j asc} dXp[prow(t,j)] + dlogit(t,j) * w_r[b_j]
// prow(t,j) = tile_offsets[b]*128 + pair_slot[t*k+j] - block_offsets[b] is the
// padded bucket row of pair (t, b = topk_idx[t,j]).
// One CTA of 128 threads per token; 16-byte vector loads/stores.
#include "internal.h"

namespace spt {

template <typename TIn>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int N = 4;
  __device__ static void load(const float* p, float (&v)[4]) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  }
  __device__ static void store(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static void load(const __nv_bfloat16* p, float (&v)[8]) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
  __device__ static void store(__nv_bfloat16* p, const float (&v)[8]) {
    uint4 q;
    uint32_t* w = &q.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = q;
  }
};

template <typename TIn, bool kBwd>
__global__ void __launch_bounds__(128) combine_kernel(int64_t T, int d, int k, RouteView r,
                                                      const TIn* __restrict__ part,
                                                      const float* __restrict__ dlogit,
                                                      const TIn* __restrict__ w_r,
                                                      const TIn* __restrict__ dense,
                                                      TIn* __restrict__ out) {
  pdl_wait();  // PDL: predecessor grid complete, its writes visible
  // successor launches as this grid's CTAs exit (an early trigger measured slower)
  constexpr int V = Vec<TIn>::N;
  __shared__ int64_t rows[kMaxBlocks];
  __shared__ int blk[kMaxBlocks];
  __shared__ float dl[kMaxBlocks];
  const int64_t t = blockIdx.x;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    rows[j] = pair_row(r, t, k, j);
    if (kBwd && dlogit) {  // sparse router term (dense mode passes no dlogit)
      blk[j] = r.topk_idx[t * k + j];
      dl[j] = dlogit[rows[j]];
    }
  }
  __syncthreads();
  for (int c = threadIdx.x * V; c < d; c += blockDim.x * V) {
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.f;
    int j = 0;
    for (; j + 4 <= k; j += 4) {  // 4 independent 16-byte loads in flight
      float v0[V], v1[V], v2[V], v3[V];
      Vec<TIn>::load(part + rows[j] * d + c, v0);
      Vec<TIn>::load(part + rows[j + 1] * d + c, v1);
      Vec<TIn>::load(part + rows[j + 2] * d + c, v2);
      Vec<TIn>::load(part + rows[j + 3] * d + c, v3);
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = (((acc[i] + v0[i]) + v1[i]) + v2[i]) + v3[i];
    }
    for (; j < k; ++j) {
      float v0[V];
      Vec<TIn>::load(part + rows[j] * d + c, v0);
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] += v0[i];
    }
    if (kBwd && dense) {  // router term precomputed densely (load-balancing loss on)
      float v[V];
      Vec<TIn>::load(dense + t * d + c, v);
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] += v[i];
    } else if (kBwd && w_r) {  // router term: sum_j dlogit_j * w_r[b_j]   (ascending j)
      for (int jj = 0; jj < k; ++jj) {
        float w[V];
        Vec<TIn>::load(w_r + (int64_t)blk[jj] * d + c, w);
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] = fmaf(dl[jj], w[i], acc[i]);
      }
    }
    Vec<TIn>::store(out + t * d + c, acc);
  }
}

cudaError_t launch_combine_fwd(const Geom& g, const RouteView& r, const void* part, void* y,
                               cudaStream_t s) {
  prof_begin("combine_fwd", s);
  if (g.dtype == SPT_BF16)
    (void)launch_pdl(combine_kernel<__nv_bfloat16, false>, dim3((unsigned)g.T), dim3(128), 0, s, 
        g.T, g.d, g.k, r, (const __nv_bfloat16*)part, nullptr, nullptr, nullptr,
        (__nv_bfloat16*)y);
  else
    (void)launch_pdl(combine_kernel<float, false>, dim3((unsigned)g.T), dim3(128), 0, s, g.T, g.d, g.k, r, (const float*)part,
                                                               nullptr, nullptr, nullptr, (float*)y);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_combine_bwd(const Geom& g, const RouteView& r, const void* part,
                               const float* dlogit, const void* w_r, void* dx, cudaStream_t s) {
  // GATE_NONE: dlogit == 0, the router term vanishes (no gradient path, reading c2)
  const void* wr = g.gate == SPT_GATE_SIGMOID ? w_r : nullptr;
  prof_begin("combine_bwd", s);
  if (g.dtype == SPT_BF16)
    (void)launch_pdl(combine_kernel<__nv_bfloat16, true>, dim3((unsigned)g.T), dim3(128), 0, s, 
        g.T, g.d, g.k, r, (const __nv_bfloat16*)part, dlogit, (const __nv_bfloat16*)wr, nullptr,
        (__nv_bfloat16*)dx);
  else
    (void)launch_pdl(combine_kernel<float, true>, dim3((unsigned)g.T), dim3(128), 0, s, 
        g.T, g.d, g.k, r, (const float*)part, dlogit, (const float*)wr, nullptr, (float*)dx);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_combine_bwd_dense(const Geom& g, const RouteView& r, const void* part,
                                     const void* dxr, void* dx, cudaStream_t s) {
  prof_begin("combine_bwd", s);
  if (g.dtype == SPT_BF16)
    (void)launch_pdl(combine_kernel<__nv_bfloat16, true>, dim3((unsigned)g.T), dim3(128), 0, s, 
        g.T, g.d, g.k, r, (const __nv_bfloat16*)part, nullptr, nullptr,
        (const __nv_bfloat16*)dxr, (__nv_bfloat16*)dx);
  else
    (void)launch_pdl(combine_kernel<float, true>, dim3((unsigned)g.T), dim3(128), 0, s, 
        g.T, g.d, g.k, r, (const float*)part, nullptr, nullptr, (const float*)dxr, (float*)dx);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

__global__ void gather_dgate_kernel(int64_t T, int k, RouteView r, const float* __restrict__ rows,
                                    float* __restrict__ out) {
  pdl_wait();  // PDL: predecessor grid complete, its writes visible
  // successor launches as this grid's CTAs exit (an early trigger measured slower)
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T * k) return;
  out[i] = rows[pair_row(r, i / k, k, (int)(i % k))];
}

cudaError_t launch_gather_dgate(const Geom& g, const RouteView& r, const float* dgate_rows,
                                float* dgate_out, cudaStream_t s) {
  prof_begin("gather_dgate", s);
  (void)launch_pdl(gather_dgate_kernel, dim3((unsigned)ceil_div(g.pairs, 256)), dim3(256), 0, s, g.T, g.k, r, dgate_rows,
                                                                       dgate_out);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

}  // namespace spt
