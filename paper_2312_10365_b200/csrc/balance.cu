// balance.cu -- the router's load-balancing loss and its gradient (SURVEY.md
// §8(f) f2).  The paper asks for "similar activation rates" (§4.2,
// PAPER.md:436) without a formula; SPEC S:342-349 defines
//   L = G * sum_g f_g * pbar_g,   f_g = n_g / (T k)   (reading c18)
//   pbar_g = (1/T) sum_t p_tg,    p_t = softmax(x_R[t])
// and, with f piecewise constant (no gradient through the selection, c11),
//   dL/dx_R[t,j] = (G/T) p_tj (f_j - sum_g f_g p_tg).
// One warp per token (lane holds blocks s*32 + lane), fp32, deterministic
// (fixed-order reductions; no atomics).
#include "internal.h"

namespace spt {

namespace {

// softmax of one token's G logits held in NSLOT lane slots (invalid slots -inf)
template <int NSLOT>
__device__ __forceinline__ void warp_softmax(const float* __restrict__ row, int G, int lane,
                                             float (&p)[NSLOT]) {
  float m = -INFINITY;
#pragma unroll
  for (int s = 0; s < NSLOT; ++s) {
    const int g = s * 32 + lane;
    p[s] = g < G ? row[g] : -INFINITY;
    m = fmaxf(m, p[s]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float sum = 0.f;
#pragma unroll
  for (int s = 0; s < NSLOT; ++s) {
    p[s] = s * 32 + lane < G ? __expf(p[s] - m) : 0.f;
    sum += p[s];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float inv = 1.f / sum;
#pragma unroll
  for (int s = 0; s < NSLOT; ++s) p[s] *= inv;
}

// per 256-token chunk: sum_t p_tg (warps over 32 tokens each in token order,
// then the 8 warps in order)
template <int NSLOT>
__global__ void __launch_bounds__(256) balance_probs_kernel(int64_t T, int G,
                                                            const float* __restrict__ logits,
                                                            float* __restrict__ part) {
  __shared__ float wsum[8][kMaxBlocks];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t0 = (int64_t)blockIdx.x * kRouteChunk + warp * (kRouteChunk / 8);
  float acc[NSLOT];
#pragma unroll
  for (int s = 0; s < NSLOT; ++s) acc[s] = 0.f;
  for (int i = 0; i < kRouteChunk / 8; ++i) {
    const int64_t t = t0 + i;
    if (t >= T) break;
    float p[NSLOT];
    warp_softmax<NSLOT>(logits + t * G, G, lane, p);
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) acc[s] += p[s];
  }
#pragma unroll
  for (int s = 0; s < NSLOT; ++s)
    if (s * 32 + lane < G) wsum[warp][s * 32 + lane] = acc[s];
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    float v = 0.f;
    for (int w = 0; w < 8; ++w) v += wsum[w][g];
    part[blockIdx.x * G + g] = v;
  }
}

// one CTA: pbar_g = sum over chunks (in order) / T, f_g from the bucket sizes,
// L = G sum_g f_g pbar_g (summed in block order by thread 0)
__global__ void __launch_bounds__(256) balance_loss_kernel(int64_t T, int64_t n_chunks, int G,
                                                           int k, const int32_t* __restrict__ bo,
                                                           const float* __restrict__ part,
                                                           float* __restrict__ loss) {
  __shared__ float c[kMaxBlocks];
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    float pb = 0.f;
    for (int64_t ch = 0; ch < n_chunks; ++ch) pb += part[ch * G + g];
    const float f = (float)(bo[g + 1] - bo[g]) / ((float)T * (float)k);
    c[g] = f * (pb / (float)T);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float L = 0.f;
    for (int g = 0; g < G; ++g) L += c[g];
    *loss = T > 0 ? (float)G * L : 0.f;
  }
}

// lambda dL/dx_R[t, j] for every block j: added to the dense hi/lo bf16
// dlogits of the dW_R / dX router GEMMs, or written as dense f32
template <int NSLOT>
__global__ void __launch_bounds__(256) balance_grad_kernel(int64_t T, int G, int k, float lbw,
                                                           int gpad, const float* __restrict__ logits,
                                                           const int32_t* __restrict__ bo,
                                                           __nv_bfloat16* __restrict__ dlg,
                                                           float* __restrict__ lbg) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T) return;
  float p[NSLOT], f[NSLOT];
  warp_softmax<NSLOT>(logits + t * G, G, lane, p);
  float fp = 0.f;
#pragma unroll
  for (int s = 0; s < NSLOT; ++s) {
    const int g = s * 32 + lane;
    f[s] = g < G ? (float)(bo[g + 1] - bo[g]) / ((float)T * (float)k) : 0.f;
    fp += f[s] * p[s];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) fp += __shfl_xor_sync(0xffffffffu, fp, o);
  const float scale = lbw * (float)G / (float)T;
#pragma unroll
  for (int s = 0; s < NSLOT; ++s) {
    const int g = s * 32 + lane;
    if (g >= G) continue;
    const float grad = scale * p[s] * (f[s] - fp);
    if (dlg) {
      __nv_bfloat16* hi = dlg + t * gpad + g;
      __nv_bfloat16* lo = dlg + (T + t) * gpad + g;
      const float v = __bfloat162float(*hi) + __bfloat162float(*lo) + grad;
      const __nv_bfloat16 h = __float2bfloat16(v);
      *hi = h;
      *lo = __float2bfloat16(v - __bfloat162float(h));
    } else {
      lbg[t * G + g] = grad;
    }
  }
}

template <typename TIn>
__device__ __forceinline__ float ldf(const TIn* p) {
  return static_cast<float>(*p);
}
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

// SIMT path (small configs): dw_r[g, c] += sum_t lbg[t, g] x[t, c]
template <typename TIn>
__global__ void __launch_bounds__(128) balance_dwr_kernel(int64_t T, int d, int G,
                                                          const float* __restrict__ lbg,
                                                          const TIn* __restrict__ x,
                                                          float* __restrict__ dw_r) {
  const int g = blockIdx.x;
  const int c = blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= d) return;
  float acc = 0.f;
  for (int64_t t = 0; t < T; ++t) acc = fmaf(lbg[t * G + g], ldf(x + t * d + c), acc);
  dw_r[(int64_t)g * d + c] += acc;
}

// SIMT path: dx[t, c] += sum_g lbg[t, g] w_r[g, c]
template <typename TIn>
__global__ void __launch_bounds__(128) balance_dx_kernel(int64_t T, int d, int G,
                                                         const float* __restrict__ lbg,
                                                         const TIn* __restrict__ w_r,
                                                         TIn* __restrict__ dx) {
  const int64_t t = blockIdx.x;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float acc = ldf(dx + t * d + c);
    for (int g = 0; g < G; ++g) acc = fmaf(lbg[t * G + g], ldf(w_r + (int64_t)g * d + c), acc);
    dx[t * d + c] = static_cast<TIn>(acc);
  }
}

}  // namespace

cudaError_t launch_balance_loss(const Geom& g, const RouteView& r, const Bufs& b, float* loss,
                                cudaStream_t s) {
  if (g.T > 0) {
    prof_begin("balance_probs", s);
    const int ns = (g.G + 31) / 32;
    const dim3 grid((unsigned)g.n_chunks);
    if (ns <= 1) balance_probs_kernel<1><<<grid, 256, 0, s>>>(g.T, g.G, r.logits, b.lb_part);
    else if (ns == 2) balance_probs_kernel<2><<<grid, 256, 0, s>>>(g.T, g.G, r.logits, b.lb_part);
    else if (ns == 3) balance_probs_kernel<3><<<grid, 256, 0, s>>>(g.T, g.G, r.logits, b.lb_part);
    else if (ns == 4) balance_probs_kernel<4><<<grid, 256, 0, s>>>(g.T, g.G, r.logits, b.lb_part);
    else balance_probs_kernel<8><<<grid, 256, 0, s>>>(g.T, g.G, r.logits, b.lb_part);
    prof_end(s);
    count_launch();
  }
  prof_begin("balance_loss", s);
  balance_loss_kernel<<<1, 256, 0, s>>>(g.T, g.n_chunks, g.G, g.k, r.block_offsets, b.lb_part, loss);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_balance_grad(const Geom& g, const RouteView& r, void* dlg, float* lbg,
                                cudaStream_t s) {
  if (g.T == 0) return cudaSuccess;
  prof_begin("balance_grad", s);
  const dim3 grid((unsigned)ceil_div(g.T, 8));
  const int ns = (g.G + 31) / 32;
  __nv_bfloat16* dl = (__nv_bfloat16*)dlg;
#define SPT_BG(NS) \
  balance_grad_kernel<NS><<<grid, 256, 0, s>>>(g.T, g.G, g.k, g.lbw, g.gpad, r.logits, r.block_offsets, dl, lbg)
  if (ns <= 1) SPT_BG(1);
  else if (ns == 2) SPT_BG(2);
  else if (ns == 3) SPT_BG(3);
  else if (ns == 4) SPT_BG(4);
  else SPT_BG(8);
#undef SPT_BG
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_balance_simt_dwr(const Geom& g, const float* lbg, const void* x, float* dw_r,
                                    cudaStream_t s) {
  if (g.T == 0) return cudaSuccess;
  prof_begin("balance_dwr", s);
  const dim3 grid((unsigned)g.G, (unsigned)ceil_div(g.d, 128));
  if (g.dtype == SPT_BF16)
    balance_dwr_kernel<__nv_bfloat16><<<grid, 128, 0, s>>>(g.T, g.d, g.G, lbg,
                                                            (const __nv_bfloat16*)x, dw_r);
  else
    balance_dwr_kernel<float><<<grid, 128, 0, s>>>(g.T, g.d, g.G, lbg, (const float*)x, dw_r);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_balance_simt_dx(const Geom& g, const float* lbg, const void* w_r, void* dx,
                                   cudaStream_t s) {
  if (g.T == 0) return cudaSuccess;
  prof_begin("balance_dx", s);
  if (g.dtype == SPT_BF16)
    balance_dx_kernel<__nv_bfloat16><<<(unsigned)g.T, 128, 0, s>>>(
        g.T, g.d, g.G, lbg, (const __nv_bfloat16*)w_r, (__nv_bfloat16*)dx);
  else
    balance_dx_kernel<float><<<(unsigned)g.T, 128, 0, s>>>(g.T, g.d, g.G, lbg, (const float*)w_r,
                                                           (float*)dx);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

}  // namespace spt
