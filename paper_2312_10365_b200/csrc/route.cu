// route.cu -- a2 per-token top-k selection and a3 token bucketing,
// plus the SIMT route network for the fp32 path.
//
// Route network x_R = x W_R, top-G' blocks by largest magnitude.
// Bucketing replaces Alg. 4's per-block masks Mask_T = eq(Indices, i) and the
// gathers X[Mask_T] by one device-side layout:
//   K-topk    : one warp per token; threshold select of the k largest
//               |logit| bit patterns (ties: lower id), emits ids ascending,
//               gates, and a per-chunk (256-token) block histogram in smem.
//   K-scan    : one CTA per block: exclusive scan of the chunk histograms.
//   K-scatter : one CTA per chunk: per-warp lane masks give each (token,block)
//               pair its stable rank -> bucket_token / bucket_gate / pair_slot.
// No atomics on global memory, no host synchronisation, deterministic.
#include "internal.h"

namespace spt {

template <typename TIn>
__device__ __forceinline__ float ldf(const TIn* p) {
  return static_cast<float>(*p);
}
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

// ---------------------------------------------------------------- SIMT router
template <typename TIn>
__global__ void router_simt_kernel(int64_t T, int d, int G, const TIn* __restrict__ x,
                                   const TIn* __restrict__ w_r, float* __restrict__ logits) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (t >= T) return;
  const TIn* xr = x + t * d;
  for (int b = 0; b < G; ++b) {
    const TIn* wr = w_r + (int64_t)b * d;
    float s = 0.f;
    for (int c = lane; c < d; c += 32) s = fmaf(ldf(xr + c), ldf(wr + c), s);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) logits[t * G + b] = s;
  }
}

cudaError_t launch_router_simt(const Geom& g, const void* x, const void* w_r, float* logits,
                               cudaStream_t s) {
  const int warps = 8;
  dim3 grid((unsigned)ceil_div(g.T, warps));
  prof_begin("router_simt", s);
  if (g.dtype == SPT_F32)
    router_simt_kernel<float><<<grid, warps * 32, 0, s>>>(g.T, g.d, g.G, (const float*)x,
                                                           (const float*)w_r, logits);
  else
    router_simt_kernel<__nv_bfloat16><<<grid, warps * 32, 0, s>>>(
        g.T, g.d, g.G, (const __nv_bfloat16*)x, (const __nv_bfloat16*)w_r, logits);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------- top-k
// Selection order: larger |logit| bit pattern first (sign cleared, so NaN >
// +Inf > finite), then lower block id (reading c4).  One warp per token; lane
// holds blocks s*32 + lane in slot s.  v = |logit| bits + 1 (0 = no block).
// Threshold select: a 32-step bitwise binary search (warp redux-add counts)
// finds tau = the k-th largest v; blocks with v > tau are taken, and the
// k - #(v > tau) lowest-id blocks with v == tau (slot-major ballots = id
// order).  Same set as k rounds of (key desc, id asc) argmax, ~6x fewer
// instructions (the round form was issue-bound: 2.5 K warp-instr per token).
template <int NSLOT>
__global__ void __launch_bounds__(256) topk_hist_kernel(int64_t T, int G, int k, int gate_mode,
                                                        const float* __restrict__ logits,
                                                        int32_t* __restrict__ topk_idx,
                                                        float* __restrict__ topk_gate,
                                                        int32_t* __restrict__ chunk_counts) {
  pdl_wait();  // PDL: predecessor grid complete, its writes visible
  // successor launches as this grid's CTAs exit (an early trigger measured slower)
  __shared__ int hist[kMaxBlocks];
  for (int b = threadIdx.x; b < G; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t chunk = blockIdx.x;
  constexpr int kPer = kTopkChunk / 8;  // tokens per warp (8 warps per CTA)
  const unsigned lt = (1u << lane) - 1u;
  // all kPer tokens' logits loaded, and their threshold searches run, together
  // (independent chains: the warp's latency is paid once, not kPer times)
  uint32_t vv[kPer][NSLOT];
  float lgv[kPer][NSLOT];
  uint32_t tauv[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int64_t t = chunk * kTopkChunk + warp * kPer + i;
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) {
      const int b = s * 32 + lane;
      vv[i][s] = 0u;
      lgv[i][s] = 0.f;
      if (t < T && b < G) {
        lgv[i][s] = logits[t * G + b];
        vv[i][s] = (__float_as_uint(lgv[i][s]) & 0x7fffffffu) + 1u;
      }
    }
    tauv[i] = 0u;
  }
  // tau = max { c : #(v >= c) >= k }, per token
#pragma unroll 2
  for (int bit = 31; bit >= 0; --bit) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const uint32_t c = tauv[i] | (1u << bit);
      uint32_t n = 0u;
#pragma unroll
      for (int s = 0; s < NSLOT; ++s) n += vv[i][s] >= c ? 1u : 0u;
      if (__reduce_add_sync(0xffffffffu, n) >= (uint32_t)k) tauv[i] = c;
    }
  }
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int64_t t = chunk * kTopkChunk + warp * kPer + i;
    if (t >= T) break;
    const uint32_t* v = vv[i];
    const float* lg = lgv[i];
    const uint32_t tau = tauv[i];
    uint32_t ngt = 0u;
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) ngt += v[s] > tau ? 1u : 0u;
    int need = k - (int)__reduce_add_sync(0xffffffffu, ngt);  // ties to take, >= 1
    // select + emit ascending block ids (slot-major ballots)
    int base = 0;
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) {
      const unsigned tie = __ballot_sync(0xffffffffu, v[s] == tau);
      const int trank = __popc(tie & lt);
      const bool sel = v[s] > tau || (v[s] == tau && trank < need);
      need -= __popc(tie);
      const unsigned m = __ballot_sync(0xffffffffu, sel);
      if (sel) {
        const int pos = base + __popc(m & lt);
        const int b = s * 32 + lane;
        topk_idx[t * k + pos] = b;
        topk_gate[t * k + pos] = gate_mode == SPT_GATE_SIGMOID ? 1.f / (1.f + expf(-lg[s])) : 1.f;
        atomicAdd(&hist[b], 1);
      }
      base += __popc(m);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < G; b += blockDim.x) chunk_counts[chunk * G + b] = hist[b];
}

// --------------------------------------------------------------- bucket scan
// CTA b: chunk_base[c][b] = sum_{c' < c} chunk_counts[c'][b]; n_b[b] = total.
__global__ void __launch_bounds__(256) bucket_scan_kernel(int64_t n_chunks, int G,
                                                          const int32_t* __restrict__ counts,
                                                          int32_t* __restrict__ chunk_base,
                                                          int32_t* __restrict__ n_b) {
  pdl_wait();  // PDL: predecessor grid complete, its writes visible
  // successor launches as this grid's CTAs exit (an early trigger measured slower)
  __shared__ int wsum[8];
  const int b = blockIdx.x;
  const int per = (int)ceil_div(n_chunks, blockDim.x);
  const int64_t c0 = (int64_t)threadIdx.x * per;
  int local = 0;
  for (int i = 0; i < per; ++i)
    if (c0 + i < n_chunks) local += counts[(c0 + i) * G + b];
  // block exclusive scan of `local`
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += wsum[w];
  int run = wpre + incl - local;
  for (int i = 0; i < per; ++i)
    if (c0 + i < n_chunks) {
      chunk_base[(c0 + i) * G + b] = run;
      run += counts[(c0 + i) * G + b];
    }
  if (threadIdx.x == blockDim.x - 1) n_b[b] = run;
}

// ------------------------------------------------------------ bucket scatter
__global__ void __launch_bounds__(256) bucket_scatter_kernel(
    int64_t T, int G, int k, const int32_t* __restrict__ n_b, const int32_t* __restrict__ chunk_base,
    const int32_t* __restrict__ topk_idx, const float* __restrict__ topk_gate,
    int32_t* __restrict__ block_offsets, int32_t* __restrict__ tile_offsets,
    int32_t* __restrict__ bucket_token, float* __restrict__ bucket_gate,
    int32_t* __restrict__ pair_slot) {
  pdl_wait();  // PDL: predecessor grid complete, its writes visible
  // successor launches as this grid's CTAs exit (an early trigger measured slower)
  __shared__ int boff[kMaxBlocks + 1];
  __shared__ int toff[kMaxBlocks + 1];
  __shared__ unsigned mask[8][kMaxBlocks];
  __shared__ int wbase[8][kMaxBlocks];
  __shared__ int wsum[8], wsum2[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t chunk = blockIdx.x;
  // exclusive scans over blocks of n_b and ceil(n_b / kTileM)
  {
    const int b = threadIdx.x;
    const int v = b < G ? n_b[b] : 0;
    const int vt = (int)ceil_div(v, kTileM);
    int inc = v, inct = vt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, inc, o);
      const int at = __shfl_up_sync(0xffffffffu, inct, o);
      if (lane >= o) { inc += a; inct += at; }
    }
    if (lane == 31) { wsum[warp] = inc; wsum2[warp] = inct; }
    __syncthreads();
    int p = 0, pt = 0;
    for (int w = 0; w < warp; ++w) { p += wsum[w]; pt += wsum2[w]; }
    if (b < G) { boff[b] = p + inc - v; toff[b] = pt + inct - vt; }
    if (b == G - 1) { boff[G] = p + inc; toff[G] = pt + inct; }
  }
  for (int i = threadIdx.x; i < 8 * kMaxBlocks; i += blockDim.x) (&mask[0][0])[i] = 0u;
  __syncthreads();
  if (chunk == 0)
    for (int b = threadIdx.x; b <= G; b += blockDim.x) {
      block_offsets[b] = boff[b];
      tile_offsets[b] = toff[b];
    }
  const int64_t t = chunk * kRouteChunk + warp * 32 + lane;
  const bool valid = t < T;
  if (valid)
    for (int j = 0; j < k; ++j) atomicOr(&mask[warp][topk_idx[t * k + j]], 1u << lane);
  __syncthreads();
  for (int b = threadIdx.x; b < G; b += blockDim.x) {
    int run = 0;
    for (int w = 0; w < 8; ++w) {
      wbase[w][b] = run;
      run += __popc(mask[w][b]);
    }
  }
  __syncthreads();
  if (valid) {
    const unsigned lt = (1u << lane) - 1u;
    for (int j = 0; j < k; ++j) {
      const int b = topk_idx[t * k + j];
      const int pos =
          boff[b] + chunk_base[chunk * (kRouteChunk / kTopkChunk) * G + b] + wbase[warp][b] +
          __popc(mask[warp][b] & lt);
      bucket_token[pos] = (int32_t)t;
      bucket_gate[pos] = topk_gate[t * k + j];
      pair_slot[t * k + j] = pos;
    }
  }
}

cudaError_t launch_topk_bucket(const Geom& g, const RouteView& r, const Bufs& b, cudaStream_t s) {
  const unsigned nch = (unsigned)g.n_chunks;
  prof_begin("topk_hist", s);
  const int nslot = (g.G + 31) / 32;
  cudaError_t e;
  // one CTA of 8 warps per kTopkChunk tokens (4 per warp): T / 32 CTAs, so even
  // 8 K-token batches spread over every SM (the selection is a serial 32-step
  // search per token)
#define SPT_TOPK(NS)                                                                        \
  e = launch_pdl(topk_hist_kernel<NS>, dim3((unsigned)g.n_sub), dim3(256), 0, s, g.T, g.G, g.k, \
                 g.gate, r.logits, r.topk_idx, r.topk_gate, b.chunk_counts)
  if (nslot <= 1) SPT_TOPK(1);
  else if (nslot == 2) SPT_TOPK(2);
  else if (nslot == 3) SPT_TOPK(3);
  else if (nslot == 4) SPT_TOPK(4);
  else SPT_TOPK(8);
#undef SPT_TOPK
  prof_end(s);
  if (e != cudaSuccess) return e;
  prof_begin("bucket_scan", s);
  e = launch_pdl(bucket_scan_kernel, dim3(g.G), dim3(256), 0, s, (int64_t)g.n_sub, g.G,
                 b.chunk_counts, b.chunk_base, b.n_b);
  prof_end(s);
  if (e != cudaSuccess) return e;
  prof_begin("bucket_scatter", s);
  e = launch_pdl(bucket_scatter_kernel, dim3(nch), dim3(256), 0, s, g.T, g.G, g.k,
                 (const int32_t*)b.n_b, (const int32_t*)b.chunk_base, (const int32_t*)r.topk_idx,
                 (const float*)r.topk_gate, r.block_offsets, r.tile_offsets, r.bucket_token,
                 r.bucket_gate, r.pair_slot);
  prof_end(s);
  count_launch(3);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace spt
