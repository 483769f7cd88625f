// simt_ffn.cu -- the fp32 path of the routed FFN: grouped GEMMs on CUDA cores
// (FFMA; no TF32, so fp32 results meet the 1e-4 relative bound), one 64x64
// output tile per CTA with a device-side bucket-tile schedule.
//
// Forward  (Alg. 4, per block b over its bucket rows):
//   F1  Z_b  = X[bucket_b] W1_b^T                  (gathered rows, line 3-4)
//   F1b H~_b = g * act(Z_b)                         (rowwise; line 4 + gate)
//   F2  P_b  = H~_b W2_b                            (line 5, partials)
//   combine  y[t] = sum_j P[prow(t,j)]              (combine.cu)
// Backward (routing fixed):
//   B1  dA_b = dY[bucket_b] W2_b^T ; B1b dgate, dZ_b, dlogit (rowwise)
//   B2  dXp_b = dZ_b W1_b ; combine dx (+ router term)
//   B4  dW1_b = dZ_b^T X[bucket_b] ; B5 dW2_b = H~_b^T dY[bucket_b] ; B6 dW_R
// Padded bucket row of the m-th entry of block b: tile_offsets[b]*128 + m.
#include "act.cuh"

namespace spt {

namespace {

template <typename T>
__device__ __forceinline__ float ld(const T* p);
template <>
__device__ __forceinline__ float ld<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
template <typename T>
__device__ __forceinline__ T cvt(float v);
template <>
__device__ __forceinline__ float cvt<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(float v) { return __float2bfloat16(v); }

// locate bucket tile `t128` (a 128-row tile index) -> block b (binary search)
__device__ __forceinline__ int find_block(const int32_t* tile_offsets, int G, int t128) {
  int lo = 0, hi = G - 1;
  while (lo < hi) {  // largest b with tile_offsets[b] <= t128
    const int mid = (lo + hi + 1) >> 1;
    if (tile_offsets[mid] <= t128) lo = mid; else hi = mid - 1;
  }
  return lo;
}

struct Tile {
  int b;        // block
  int m0;       // first row (entry index inside block b's bucket)
  int n_valid;  // rows of this tile that are real bucket entries (<= 64, may be <= 0)
  int64_t prow0;  // padded bucket row of m0
  int64_t pos0;   // bucket position of m0 (block_offsets[b] + m0)
  int n0;       // first output column
};

// bucket-row tiles: blockIdx.x = 64-row tile over padded rows, blockIdx.y = n tile
__device__ __forceinline__ bool row_tile(const RouteView& r, int G, Tile& t) {
  const int total = r.tile_offsets[G] * (kTileM / 64);
  if ((int)blockIdx.x >= total) return false;
  const int t128 = blockIdx.x / (kTileM / 64);
  t.b = find_block(r.tile_offsets, G, t128);
  t.m0 = (t128 - r.tile_offsets[t.b]) * kTileM + (blockIdx.x % (kTileM / 64)) * 64;
  const int nb = r.block_offsets[t.b + 1] - r.block_offsets[t.b];
  t.n_valid = nb - t.m0;
  t.prow0 = (int64_t)r.tile_offsets[t.b] * kTileM + t.m0;
  t.pos0 = r.block_offsets[t.b] + t.m0;
  t.n0 = blockIdx.y * 64;
  return true;
}

// 64x64 tile, BK = 16, 256 threads, 4x4 outputs per thread.
// Op: float a(const Tile&, int m, int k)  (m < 64, k < K)
//     float b(const Tile&, int n, int k)  (n = absolute column)
//     void  store(const Tile&, int m, int n, float v)
template <class Op>
__device__ __forceinline__ void gemm_tile(const Op& op, const Tile& t, int K, int N) {
  __shared__ float sA[16][68];
  __shared__ float sB[16][68];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + i * 256;  // 0..1023 : (m or n) = e / 16, kk = e % 16
      const int mn = e >> 4, kk = e & 15;
      const int k = k0 + kk;
      sA[kk][mn] = (k < K) ? op.a(t, mn, k) : 0.f;
      const int n = t.n0 + mn;
      sB[kk][mn] = (k < K && n < N) ? op.b(t, n, k) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { av[i] = sA[kk][ty * 4 + i]; bv[i] = sB[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = t.n0 + tx * 4 + j;
      if (n < N) op.store(t, ty * 4 + i, n, acc[i][j]);
    }
}

// ------------------------------------------------------------------ F1: Z
template <typename T>
struct OpZ {
  RouteView r; const T* x; const T* w1; T* z; int d, D, bw, mp;
  __device__ float a(const Tile& t, int m, int k) const {
    if (m >= t.n_valid) return 0.f;
    return ld(x + (int64_t)r.bucket_token[t.pos0 + m] * d + k);
  }
  __device__ float b(const Tile& t, int n, int k) const {
    const int64_t row = n < bw ? (int64_t)t.b * bw + n : (int64_t)D + (int64_t)t.b * bw + (n - bw);
    return ld(w1 + row * d + k);
  }
  __device__ void store(const Tile& t, int m, int n, float v) const {
    z[(t.prow0 + m) * (int64_t)(mp * bw) + n] = cvt<T>(m < t.n_valid ? v : 0.f);
  }
};
template <typename T>
__global__ void __launch_bounds__(256) k_f1(OpZ<T> op, int G) {
  Tile t;
  if (!row_tile(op.r, G, t)) return;
  gemm_tile(op, t, op.d, op.mp * op.bw);
}

// F1b: H~[row][u] = g * act(Z[row][u], Z[row][bw+u])   (0 on padding rows)
template <typename T>
__global__ void k_f1b(RouteView r, int G, int bw, int mp, int act, const T* __restrict__ z,
                      T* __restrict__ h) {
  Tile t;
  if (!row_tile(r, G, t)) return;
  for (int e = threadIdx.x; e < 64 * bw; e += blockDim.x) {
    const int m = e / bw, u = e % bw;
    const int64_t row = t.prow0 + m;
    float v = 0.f;
    if (m < t.n_valid) {
      const float g = r.bucket_gate[t.pos0 + m];
      const T* zr = z + row * (int64_t)(mp * bw);
      v = g * act_fwd(act, ld(zr + u), mp == 2 ? ld(zr + bw + u) : 0.f);
    }
    h[row * bw + u] = cvt<T>(v);
  }
}

// ------------------------------------------------------------------ F2: P
template <typename T>
struct OpP {
  const T* h; const T* w2; T* part; int d, bw;
  __device__ float a(const Tile& t, int m, int k) const { return ld(h + (t.prow0 + m) * bw + k); }
  __device__ float b(const Tile& t, int n, int k) const {
    return ld(w2 + ((int64_t)t.b * bw + k) * d + n);
  }
  __device__ void store(const Tile& t, int m, int n, float v) const {
    if (m < t.n_valid) part[(t.prow0 + m) * (int64_t)d + n] = cvt<T>(v);
  }
};
template <typename T>
__global__ void __launch_bounds__(256) k_f2(OpP<T> op, RouteView r, int G) {
  Tile t;
  if (!row_tile(r, G, t)) return;
  gemm_tile(op, t, op.bw, op.d);
}

// ------------------------------------------------------------------ B1: dA
template <typename T>
struct OpDA {
  RouteView r; const T* dy; const T* w2; float* da; int d, bw;
  __device__ float a(const Tile& t, int m, int k) const {
    if (m >= t.n_valid) return 0.f;
    return ld(dy + (int64_t)r.bucket_token[t.pos0 + m] * d + k);
  }
  __device__ float b(const Tile& t, int n, int k) const {
    return ld(w2 + ((int64_t)t.b * bw + n) * d + k);
  }
  __device__ void store(const Tile& t, int m, int n, float v) const {
    da[(t.prow0 + m) * bw + n] = v;
  }
};
template <typename T>
__global__ void __launch_bounds__(256) k_b1(OpDA<T> op, int G) {
  Tile t;
  if (!row_tile(op.r, G, t)) return;
  gemm_tile(op, t, op.d, op.bw);
}

// B1b: one warp per padded row: dgate = sum_u dA*a ; dZ = g dA act'(Z); dlogit
template <typename T>
__global__ void k_b1b(RouteView r, int G, int bw, int mp, int act, int gate_mode,
                      const T* __restrict__ z, const float* __restrict__ da, T* __restrict__ dz,
                      float* __restrict__ dgate_rows, float* __restrict__ dlogit_rows) {
  Tile t;
  if (!row_tile(r, G, t)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int m = warp; m < 64; m += blockDim.x / 32) {
    const int64_t row = t.prow0 + m;
    const bool valid = m < t.n_valid;
    const float g = valid ? r.bucket_gate[t.pos0 + m] : 0.f;
    const T* zr = z + row * (int64_t)(mp * bw);
    T* dzr = dz + row * (int64_t)(mp * bw);
    float dgs = 0.f;
    for (int u = lane; u < bw; u += 32) {
      float a = 0.f, dg = 0.f, du = 0.f, dA = 0.f;
      if (valid) {
        dA = da[row * bw + u];
        act_fwd_bwd(act, ld(zr + u), mp == 2 ? ld(zr + bw + u) : 0.f, a, dg, du);
      }
      dgs = fmaf(dA, a, dgs);
      dzr[u] = cvt<T>(g * dA * dg);
      if (mp == 2) dzr[bw + u] = cvt<T>(g * dA * du);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) dgs += __shfl_xor_sync(0xffffffffu, dgs, o);
    if (lane == 0) {
      dgate_rows[row] = valid ? dgs : 0.f;
      float dl = 0.f;
      if (valid && gate_mode == SPT_GATE_SIGMOID) {
        const int64_t tok = r.bucket_token[t.pos0 + m];
        dl = dgs * sigmoid_pair(r.logits[tok * G + t.b]);   // = dgate g (1 - g)
      }
      dlogit_rows[row] = dl;
    }
  }
}

// ------------------------------------------------------------------ B2: dXp
template <typename T>
struct OpDX {
  const T* dz; const T* w1; T* part; int d, D, bw, mp;
  __device__ float a(const Tile& t, int m, int k) const {
    return ld(dz + (t.prow0 + m) * (int64_t)(mp * bw) + k);
  }
  __device__ float b(const Tile& t, int n, int k) const {
    const int64_t row = k < bw ? (int64_t)t.b * bw + k : (int64_t)D + (int64_t)t.b * bw + (k - bw);
    return ld(w1 + row * d + n);
  }
  __device__ void store(const Tile& t, int m, int n, float v) const {
    if (m < t.n_valid) part[(t.prow0 + m) * (int64_t)d + n] = cvt<T>(v);
  }
};
template <typename T>
__global__ void __launch_bounds__(256) k_b2(OpDX<T> op, RouteView r, int G) {
  Tile t;
  if (!row_tile(r, G, t)) return;
  gemm_tile(op, t, op.mp * op.bw, op.d);
}

// ------------------------------------------------------ B4/B5: weight grads
// grid (ceil(M/64), d/64, G); K = n_b bucket entries of block b.
template <typename T>
struct OpDW {
  RouteView r; const T* act_rows;  // dz [rows, M] or h [rows, bw]
  const T* tok;                    // x or dy [T, d]
  float* dw; int d, D, bw, M, acc_mode, split_gate_up;
  int64_t prow_b;                  // padded row of entry 0 of block b
  __device__ float a(const Tile& t, int m, int k) const {
    const int mm = t.m0 + m;
    return mm < M ? ld(act_rows + (prow_b + k) * (int64_t)M + mm) : 0.f;
  }
  __device__ float b(const Tile& t, int n, int k) const {
    return ld(tok + (int64_t)r.bucket_token[t.pos0 + k] * d + n);
  }
  __device__ void store(const Tile& t, int m, int n, float v) const {
    const int mm = t.m0 + m;
    if (mm >= M) return;
    int64_t row;
    if (split_gate_up) row = mm < bw ? (int64_t)t.b * bw + mm : (int64_t)D + (int64_t)t.b * bw + (mm - bw);
    else row = (int64_t)t.b * bw + mm;
    float* p = dw + row * d + n;
    *p = acc_mode ? *p + v : v;
  }
};
template <typename T>
__global__ void __launch_bounds__(256) k_dw(OpDW<T> op) {
  Tile t;
  t.b = blockIdx.z;
  t.m0 = blockIdx.x * 64;
  t.n0 = blockIdx.y * 64;
  t.pos0 = op.r.block_offsets[t.b];
  t.n_valid = 0;
  t.prow0 = 0;
  op.prow_b = (int64_t)op.r.tile_offsets[t.b] * kTileM;
  const int nb = op.r.block_offsets[t.b + 1] - op.r.block_offsets[t.b];
  gemm_tile(op, t, nb, op.d);
}

// B6: dW_R[b][c] = sum over bucket entries of dlogit * x[token][c]
template <typename T>
__global__ void k_dwr(RouteView r, int d, const T* __restrict__ x,
                      const float* __restrict__ dlogit_rows, float* __restrict__ dw_r, int acc_mode) {
  const int b = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  const int p0 = r.block_offsets[b], nb = r.block_offsets[b + 1] - p0;
  const int64_t prow_b = (int64_t)r.tile_offsets[b] * kTileM;
  float s = 0.f;
  for (int m = 0; m < nb; ++m)
    s = fmaf(dlogit_rows[prow_b + m], ld(x + (int64_t)r.bucket_token[p0 + m] * d + c), s);
  float* p = dw_r + (int64_t)b * d + c;
  *p = acc_mode ? *p + s : s;
}

template <typename T>
cudaError_t fwd_impl(const Geom& g, const T* x, const T* w1, const T* w2, const RouteView& r, T* y,
                     const Bufs& b, cudaStream_t s) {
  const unsigned tiles64 = (unsigned)((ceil_div(g.pairs, kTileM) + g.G) * (kTileM / 64));
  OpZ<T> oz{r, x, w1, (T*)b.z, g.d, g.D, g.bw, g.mp};
  prof_begin("simt_f1", s);
  k_f1<T><<<dim3(tiles64, (unsigned)ceil_div(g.mp * g.bw, 64)), 256, 0, s>>>(oz, g.G);
  prof_end(s);
  prof_begin("simt_f1b", s);
  k_f1b<T><<<tiles64, 256, 0, s>>>(r, g.G, g.bw, g.mp, g.act, (const T*)b.z, (T*)b.h);
  prof_end(s);
  OpP<T> op{(const T*)b.h, w2, (T*)b.part, g.d, g.bw};
  prof_begin("simt_f2", s);
  k_f2<T><<<dim3(tiles64, (unsigned)ceil_div(g.d, 64)), 256, 0, s>>>(op, r, g.G);
  prof_end(s);
  count_launch(3);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_combine_fwd(g, r, b.part, y, s);
}

template <typename T>
cudaError_t bwd_impl(const Geom& g, const T* x, const T* w1, const T* w2, const T* w_r,
                     const RouteView& r, const T* dy, T* dx, float* dw1, float* dw2, float* dw_r,
                     float* dgate_out, bool acc, const Bufs& b, cudaEvent_t dw_ev, cudaStream_t s) {
  const unsigned tiles64 = (unsigned)((ceil_div(g.pairs, kTileM) + g.G) * (kTileM / 64));
  OpDA<T> oda{r, dy, w2, b.da, g.d, g.bw};
  prof_begin("simt_b1", s);
  k_b1<T><<<dim3(tiles64, (unsigned)ceil_div(g.bw, 64)), 256, 0, s>>>(oda, g.G);
  prof_end(s);
  prof_begin("simt_b1b", s);
  k_b1b<T><<<tiles64, 256, 0, s>>>(r, g.G, g.bw, g.mp, g.act, g.gate, (const T*)b.z, b.da,
                                   (T*)b.dz, b.dgate, b.dlogit);
  prof_end(s);
  const int M1 = g.mp * g.bw;
  OpDW<T> o1{r, (const T*)b.dz, x, dw1, g.d, g.D, g.bw, M1, acc ? 1 : 0, g.mp == 2 ? 1 : 0, 0};
  prof_begin("simt_dw", s);
  k_dw<T><<<dim3((unsigned)ceil_div(M1, 64), (unsigned)ceil_div(g.d, 64), g.G), 256, 0, s>>>(o1);
  prof_end(s);
  OpDW<T> o2{r, (const T*)b.h, dy, dw2, g.d, g.D, g.bw, g.bw, acc ? 1 : 0, 0, 0};
  prof_begin("simt_dw", s);
  k_dw<T><<<dim3((unsigned)ceil_div(g.bw, 64), (unsigned)ceil_div(g.d, 64), g.G), 256, 0, s>>>(o2);
  prof_end(s);
  prof_begin("simt_dwr", s);
  k_dwr<T><<<dim3((unsigned)ceil_div(g.d, 128), g.G), 128, 0, s>>>(r, g.d, x, b.dlogit, dw_r,
                                                                  acc ? 1 : 0);
  prof_end(s);
  count_launch(5);  // b1, b1b, dw x2, dwr
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  float* lbg = (float*)b.lb_x;  // f2: lambda dL_balance/dx_R [T, G] (every block)
  if (g.lbw != 0.f) {
    if ((e = launch_balance_grad(g, r, nullptr, lbg, s)) != cudaSuccess) return e;
    if ((e = launch_balance_simt_dwr(g, lbg, x, dw_r, s)) != cudaSuccess) return e;
  }
  if (dw_ev && cudaEventRecord(dw_ev, s) != cudaSuccess) return cudaErrorUnknown;
  OpDX<T> odx{(const T*)b.dz, w1, (T*)b.part, g.d, g.D, g.bw, g.mp};
  prof_begin("simt_b2", s);
  k_b2<T><<<dim3(tiles64, (unsigned)ceil_div(g.d, 64)), 256, 0, s>>>(odx, r, g.G);
  prof_end(s);
  count_launch(1);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = launch_combine_bwd(g, r, b.part, b.dlogit, w_r, dx, s)) != cudaSuccess) return e;
  if (g.lbw != 0.f && (e = launch_balance_simt_dx(g, lbg, w_r, dx, s)) != cudaSuccess) return e;
  if (dgate_out) return launch_gather_dgate(g, r, b.dgate, dgate_out, s);
  return cudaSuccess;
}

}  // namespace

cudaError_t simt_forward(const Geom& g, const void* x, const void* w1, const void* w2,
                         const RouteView& r, void* y, const Bufs& b, cudaStream_t s) {
  if (g.dtype == SPT_F32)
    return fwd_impl<float>(g, (const float*)x, (const float*)w1, (const float*)w2, r, (float*)y, b, s);
  return fwd_impl<__nv_bfloat16>(g, (const __nv_bfloat16*)x, (const __nv_bfloat16*)w1,
                                 (const __nv_bfloat16*)w2, r, (__nv_bfloat16*)y, b, s);
}

cudaError_t simt_backward(const Geom& g, const void* x, const void* w1, const void* w2,
                          const void* w_r, const RouteView& r, const void* dy, void* dx,
                          float* dw1, float* dw2, float* dw_r, float* dgate_out, bool accumulate,
                          const Bufs& b, cudaEvent_t dw_ev, cudaStream_t s) {
  if (g.dtype == SPT_F32)
    return bwd_impl<float>(g, (const float*)x, (const float*)w1, (const float*)w2,
                           (const float*)w_r, r, (const float*)dy, (float*)dx, dw1, dw2, dw_r,
                           dgate_out, accumulate, b, dw_ev, s);
  return bwd_impl<__nv_bfloat16>(g, (const __nv_bfloat16*)x, (const __nv_bfloat16*)w1,
                                 (const __nv_bfloat16*)w2, (const __nv_bfloat16*)w_r, r,
                                 (const __nv_bfloat16*)dy, (__nv_bfloat16*)dx, dw1, dw2, dw_r,
                                 dgate_out, accumulate, b, dw_ev, s);
}

}  // namespace spt
