// lora.cu -- the LoRA-wrapped routed FFN: the HBM-bound
// and skinny (rank-r) kernels around the tcgen05 GEMMs of tc_ffn.cu.
//
// LoRA (Eq. 5): Y = XW + XBC with W frozen; SPT wraps both
// FFN projections and routes the FFN (§4.2), so block b
// uses the columns [b bw, (b+1) bw) of W_I + B_I C_I and the same rows of
// W_O + B_O C_O.  Per token t, block b in S_t (storage: b1 = B_I^T [m',r,d],
// c1 = C_I^T [m',D,r], b2 = B_O [D,r], c2 = C_O [r,d]):
//   u_t = x_t B_I                               tc_router GEMM (N = m' r)
//   z   = x_t W_I[:,b] + u_t C_I[:,b]           FWD1 on X_aug = [x | hi(u) | lo(u) | 0],
//                                                        W1_aug = [w1 | c1 | c1 | 0]
//   h~  = g act(z);  P = h~ W_O[b]              FWD1 epilogue, FWD2 (unchanged)
//   q_t = sum_b h~ B_O[b]                       lora_rowproj (per pair) + combine
//   y_t = sum_b P + q_t C_O                     lora_combine_fwd
// Backward (W frozen; routing fixed):
//   v_t = dy_t C_O^T                            tc_router GEMM (N = r)
//   dA  = dy W_O[b]^T + v B_O[b]^T              dA kernel on dY_aug = [dy | hi(v) | lo(v) | 0],
//                                                           W2_aug = [w2 | b2 | b2 | 0]
//   dgate, dZ                                   dA epilogue (unchanged)
//   dB_O[b] = sum_{t in b} h~^T v_t             lora_colgrad (per tile) + lora_grad_reduce
//   dC_I[:,b]^T = sum_{t in b} dZ^T u_t         lora_colgrad + lora_grad_reduce
//   du_t = sum_b dZ C_I[:,b]^T                  lora_rowproj (per pair) + combine
//   dx_t = sum_b dZ W_I[:,b]^T + router + du_t B_I^T    DX (unchanged) + lora_combine_bwd
//   dB_I^T = du^T X,  dC_O = q^T dY             tcgen05 split-K GEMMs (the dW_R kernel)
// u and v enter the tensor-core GEMMs as bf16 hi + lo halves (~16 significant
// bits: the pre-activation z, and with it every ReLU sign decision, matches the
// plain path's accuracy); q and du are reduced in fp32 and split hi + lo for
// their GEMMs too.
// Sums over a token's blocks run in ascending block order (reading c12), and
// every per-block gradient is reduced over its tiles in tile order: results
// are deterministic.
#include "internal.h"

namespace spt {

namespace {

__device__ __forceinline__ float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 q = __ldg(reinterpret_cast<const uint4*>(p));
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

__device__ __forceinline__ uint4 pack8(const float (&v)[8]) {
  uint4 q;
  uint32_t* w = &q.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  return q;
}

// out[t] = [src[t, 0:d] | hi(u[t, 0:nu]) | lo(u[t, 0:nu]) | 0 ...] (width d + ka), with
// hi = bf16(u), lo = bf16(u - hi); ust[t] = u[t] (fp32, for the backward)
__global__ void __launch_bounds__(256) lora_aug_rows_kernel(int64_t T, int d, int ka,
                                                            const __nv_bfloat16* __restrict__ src,
                                                            const float* __restrict__ u, int nu,
                                                            __nv_bfloat16* __restrict__ out,
                                                            float* __restrict__ ust) {
  const int dv = d / 8;
  for (int64_t t = blockIdx.x; t < T; t += gridDim.x) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src + t * d);
    uint4* o4 = reinterpret_cast<uint4*>(out + t * (d + ka));
    for (int c = threadIdx.x; c < dv; c += blockDim.x) o4[c] = __ldg(s4 + c);
    if ((int)threadIdx.x < ka / 8) {
      const int c0 = threadIdx.x * 8;
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int c = c0 + i;
        float x = 0.f;
        if (c < nu) {
          x = __bfloat162float(__float2bfloat16(u[t * nu + c]));
        } else if (c < 2 * nu) {
          const float f = u[t * nu + c - nu];
          x = f - __bfloat162float(__float2bfloat16(f));
        }
        v[i] = x;
      }
      o4[dv + threadIdx.x] = pack8(v);
    }
    if (ust)
      for (int c = threadIdx.x; c < nu; c += blockDim.x) ust[t * nu + c] = u[t * nu + c];
  }
}

// out[i] = [w[i, 0:d] | P[i, 0:r] at columns d + m r and d + nu + m r (m = i / rows_half) | 0]
// (W1_aug: the gate rows' C_I^T against hi(u_gate), lo(u_gate), the up rows'
// against hi(u_up), lo(u_up); W2_aug: rows_half = D, P = B_O against hi(v), lo(v))
__global__ void __launch_bounds__(256) lora_aug_w_kernel(int64_t R, int d, int ka,
                                                         const __nv_bfloat16* __restrict__ w,
                                                         const __nv_bfloat16* __restrict__ P, int r,
                                                         int nu, int64_t rows_half,
                                                         __nv_bfloat16* __restrict__ out) {
  const int dv = d / 8;
  for (int64_t i = blockIdx.x; i < R; i += gridDim.x) {
    const uint4* s4 = reinterpret_cast<const uint4*>(w + i * d);
    uint4* o4 = reinterpret_cast<uint4*>(out + i * (d + ka));
    for (int c = threadIdx.x; c < dv; c += blockDim.x) o4[c] = __ldg(s4 + c);
    const int off = (int)(i / rows_half) * r;
    if ((int)threadIdx.x < ka) {
      const int c = threadIdx.x;
      const int q = (c < nu ? c : c - nu) - off;
      out[i * (d + ka) + d + c] =
          (c < 2 * nu && q >= 0 && q < r) ? P[i * r + q] : __float2bfloat16(0.f);
    }
  }
}

struct TileRows {
  int b, nvalid, pos0;  // block, live rows, bucket position of row 0
  int64_t prow0;        // padded bucket row of row 0
};
__device__ __forceinline__ TileRows tile_rows(const RouteView& rv, const int32_t* tile_block,
                                              int tile) {
  TileRows tr;
  tr.b = tile_block[tile];
  const int mt = tile - rv.tile_offsets[tr.b];
  const int nb = rv.block_offsets[tr.b + 1] - rv.block_offsets[tr.b];
  tr.nvalid = min(kTileM, nb - mt * kTileM);
  tr.pos0 = rv.block_offsets[tr.b] + mt * kTileM;
  tr.prow0 = (int64_t)tile * kTileM;
  return tr;
}

// Per pair (one thread per padded bucket row of a 128-row tile):
//   out[prow, m r + q] = sum_{i < bw} A[prow, m bw + i] P[m][b bw + i][q]
// fwd: A = h~ (m' = 1), P = B_O -> q rows;  bwd: A = dZ (m' halves), P = C_I^T -> du rows.
template <int RP>
__global__ void __launch_bounds__(128) lora_rowproj_kernel(int G, int bw, int mp, int r, int64_t D,
                                                           RouteView rv,
                                                           const int32_t* __restrict__ tile_block,
                                                           const __nv_bfloat16* __restrict__ A,
                                                           const __nv_bfloat16* __restrict__ P,
                                                           float* __restrict__ out) {
  const int tile = blockIdx.x;
  if (tile >= rv.tile_offsets[G]) return;
  const TileRows tr = tile_rows(rv, tile_block, tile);
  __shared__ float Ps[64][RP];
  const int64_t prow = tr.prow0 + threadIdx.x;
  const bool live = (int)threadIdx.x < tr.nvalid;
  const int aw = mp * bw;
  for (int m = 0; m < mp; ++m) {
    float acc[RP];
#pragma unroll
    for (int q = 0; q < RP; ++q) acc[q] = 0.f;
    for (int i0 = 0; i0 < bw; i0 += 64) {
      const int ni = min(64, bw - i0);  // bw % 16 == 0
      __syncthreads();
      for (int e = threadIdx.x; e < 64 * RP; e += blockDim.x) {
        const int i = e / RP, q = e % RP;
        Ps[i][q] = (i < ni && q < r) ? bf2f(P[((int64_t)m * D + (int64_t)tr.b * bw + i0 + i) * r + q])
                                     : 0.f;
      }
      __syncthreads();
      if (live) {
        const __nv_bfloat16* ar = A + prow * aw + m * bw + i0;
        for (int i = 0; i < ni; i += 8) {
          float a[8];
          load8(ar + i, a);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int q = 0; q < RP; ++q) acc[q] = fmaf(a[j], Ps[i + j][q], acc[q]);
          }
        }
      }
    }
    if (live) {
      float* o = out + prow * kLoraK + m * r;
      for (int q = 0; q < r; ++q) o[q] = acc[q];
    }
  }
}

// Per 128-row tile of block b, per feature i (one thread each):
//   part[tile][m][i][q] = sum_{rows} A[prow, m bw + i] E[t(row), eoff + m r + q]
// dC_I: A = dZ, E = the stashed u (f32, pitch m' r);  dB_O: A = h~, E = v (f32, pitch r).
template <int RP, typename TE>
__global__ void __launch_bounds__(128) lora_colgrad_kernel(int G, int bw, int mp, int r,
                                                           RouteView rv,
                                                           const int32_t* __restrict__ tile_block,
                                                           const __nv_bfloat16* __restrict__ A,
                                                           const TE* __restrict__ E, int epitch,
                                                           float* __restrict__ part) {
  const int tile = blockIdx.x;
  if (tile >= rv.tile_offsets[G]) return;
  const TileRows tr = tile_rows(rv, tile_block, tile);
  __shared__ float Es[kTileM][RP];
  __shared__ int tok[kTileM];
  if (threadIdx.x < kTileM)
    tok[threadIdx.x] = (int)threadIdx.x < tr.nvalid ? rv.bucket_token[tr.pos0 + threadIdx.x] : 0;
  const int aw = mp * bw;
  for (int m = 0; m < mp; ++m) {
    __syncthreads();
    for (int e = threadIdx.x; e < kTileM * RP; e += blockDim.x) {
      const int row = e / RP, q = e % RP;
      float v = 0.f;
      if (row < tr.nvalid && q < r) v = (float)E[(int64_t)tok[row] * epitch + m * r + q];
      Es[row][q] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < bw; i += blockDim.x) {
      float acc[RP];
#pragma unroll
      for (int q = 0; q < RP; ++q) acc[q] = 0.f;
      const __nv_bfloat16* ac = A + tr.prow0 * aw + m * bw + i;
      for (int row = 0; row < tr.nvalid; ++row) {
        const float a = bf2f(ac[(int64_t)row * aw]);
#pragma unroll
        for (int q = 0; q < RP; ++q) acc[q] = fmaf(a, Es[row][q], acc[q]);
      }
      float* o = part + (((int64_t)tile * mp + m) * bw + i) * r;
      for (int q = 0; q < r; ++q) o[q] = acc[q];
    }
  }
}

// out[m][b bw + i][q] (=|+=) sum over block b's tiles (ascending) of part[tile][m][i][q]
__global__ void __launch_bounds__(256) lora_grad_reduce_kernel(int G, int bw, int mp, int r,
                                                               int64_t D, RouteView rv,
                                                               const float* __restrict__ part,
                                                               float* __restrict__ out, int acc) {
  const int64_t n = (int64_t)mp * D * r;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  const int m = (int)(idx / (D * r));
  const int64_t rem = idx % (D * r);
  const int64_t unit = rem / r;
  const int q = (int)(rem % r);
  const int b = (int)(unit / bw), i = (int)(unit % bw);
  float s = 0.f;
  for (int tile = rv.tile_offsets[b]; tile < rv.tile_offsets[b + 1]; ++tile)
    s += part[(((int64_t)tile * mp + m) * bw + i) * r + q];
  out[idx] = acc ? out[idx] + s : s;
}

// Per token t (one CTA): s[c] = sum_{j asc} rowp[prow(t,j)][c] for c < ns (q or du),
// written as bf16 hi + lo halves [2, T, spitch] for the tcgen05 GEMM; then
//   out[t] = sum_{j asc} part[prow(t,j)] + router term + sum_c s[c] F[c, :]
// (fwd: F = C_O, no router term; bwd: F = B_I^T rows, router term as combine_bwd).
template <bool kBwd>
__global__ void __launch_bounds__(128) lora_combine_kernel(int64_t T, int d, int k, int ns,
                                                           int spitch, RouteView r,
                                                           const __nv_bfloat16* __restrict__ part,
                                                           const float* __restrict__ rowp,
                                                           const __nv_bfloat16* __restrict__ F,
                                                           const float* __restrict__ dlogit,
                                                           const __nv_bfloat16* __restrict__ w_r,
                                                           const __nv_bfloat16* __restrict__ dense,
                                                           __nv_bfloat16* __restrict__ out,
                                                           __nv_bfloat16* __restrict__ shl) {
  __shared__ int64_t rows[kMaxBlocks];
  __shared__ int blk[kMaxBlocks];
  __shared__ float dl[kMaxBlocks];
  __shared__ float sv[kLoraK];
  const int64_t t = blockIdx.x;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    rows[j] = pair_row(r, t, k, j);
    if (kBwd && dlogit) {
      blk[j] = r.topk_idx[t * k + j];
      dl[j] = dlogit[rows[j]];
    }
  }
  __syncthreads();
  if (threadIdx.x < spitch) {
    float v = 0.f;
    if ((int)threadIdx.x < ns)
      for (int j = 0; j < k; ++j) v += rowp[rows[j] * kLoraK + threadIdx.x];
    if ((int)threadIdx.x < kLoraK) sv[threadIdx.x] = v;
    const __nv_bfloat16 hi = __float2bfloat16(v);
    shl[t * spitch + threadIdx.x] = hi;
    shl[(T + t) * spitch + threadIdx.x] = __float2bfloat16(v - __bfloat162float(hi));
  }
  __syncthreads();
  for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    int j = 0;
    for (; j + 4 <= k; j += 4) {
      float v0[8], v1[8], v2[8], v3[8];
      load8(part + rows[j] * d + c, v0);
      load8(part + rows[j + 1] * d + c, v1);
      load8(part + rows[j + 2] * d + c, v2);
      load8(part + rows[j + 3] * d + c, v3);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = (((acc[i] + v0[i]) + v1[i]) + v2[i]) + v3[i];
    }
    for (; j < k; ++j) {
      float v0[8];
      load8(part + rows[j] * d + c, v0);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += v0[i];
    }
    if (kBwd && dense) {
      float v[8];
      load8(dense + t * d + c, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += v[i];
    } else if (kBwd && w_r) {
      for (int jj = 0; jj < k; ++jj) {
        float w[8];
        load8(w_r + (int64_t)blk[jj] * d + c, w);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fmaf(dl[jj], w[i], acc[i]);
      }
    }
    for (int q = 0; q < ns; ++q) {
      float f[8];
      load8(F + (int64_t)q * d + c, f);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fmaf(sv[q], f[i], acc[i]);
    }
    *reinterpret_cast<uint4*>(out + t * d + c) = pack8(acc);
  }
}

template <int RP>
cudaError_t rowproj(const Geom& g, const RouteView& r, const Bufs& b, int mp, int rk,
                    const void* A, const void* P, float* out, cudaStream_t s) {
  lora_rowproj_kernel<RP><<<(unsigned)(ceil_div(g.pairs, kTileM) + g.G), 128, 0, s>>>(
      g.G, g.bw, mp, rk, g.D, r, b.tile_block, (const __nv_bfloat16*)A, (const __nv_bfloat16*)P,
      out);
  return cudaGetLastError();
}

cudaError_t launch_rowproj(const Geom& g, const RouteView& r, const Bufs& b, int mp, int rk,
                           const void* A, const void* P, float* out, cudaStream_t s) {
  prof_begin("lora_rowproj", s);
  cudaError_t e = rk <= 8    ? rowproj<8>(g, r, b, mp, rk, A, P, out, s)
                  : rk <= 16 ? rowproj<16>(g, r, b, mp, rk, A, P, out, s)
                  : rk <= 32 ? rowproj<32>(g, r, b, mp, rk, A, P, out, s)
                             : rowproj<64>(g, r, b, mp, rk, A, P, out, s);
  prof_end(s);
  count_launch();
  return e;
}

template <int RP, typename TE>
cudaError_t colgrad(const Geom& g, const RouteView& r, const Bufs& b, int mp, int rk,
                    const void* A, const TE* E, int epitch, float* part, cudaStream_t s) {
  lora_colgrad_kernel<RP, TE><<<(unsigned)(ceil_div(g.pairs, kTileM) + g.G), 128, 0, s>>>(
      g.G, g.bw, mp, rk, r, b.tile_block, (const __nv_bfloat16*)A, E, epitch, part);
  return cudaGetLastError();
}

template <typename TE>
cudaError_t launch_colgrad(const Geom& g, const RouteView& r, const Bufs& b, int mp, int rk,
                           const void* A, const TE* E, int epitch, float* part, cudaStream_t s) {
  prof_begin("lora_colgrad", s);
  cudaError_t e = rk <= 8    ? colgrad<8, TE>(g, r, b, mp, rk, A, E, epitch, part, s)
                  : rk <= 16 ? colgrad<16, TE>(g, r, b, mp, rk, A, E, epitch, part, s)
                  : rk <= 32 ? colgrad<32, TE>(g, r, b, mp, rk, A, E, epitch, part, s)
                             : colgrad<64, TE>(g, r, b, mp, rk, A, E, epitch, part, s);
  prof_end(s);
  count_launch();
  return e;
}

cudaError_t launch_grad_reduce(const Geom& g, const RouteView& r, int mp, int rk,
                               const float* part, float* out, bool acc, cudaStream_t s) {
  const int64_t n = (int64_t)mp * g.D * rk;
  prof_begin("lora_grad_reduce", s);
  lora_grad_reduce_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(g.G, g.bw, mp, rk, g.D, r,
                                                                     part, out, acc ? 1 : 0);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

cudaError_t aug_rows(const Geom& g, int ka, const void* src, const float* u, int nu, void* out,
                     float* ust, cudaStream_t s) {
  prof_begin("lora_aug_rows", s);
  const unsigned grid = (unsigned)std::min<int64_t>(g.T, 148 * 16);
  lora_aug_rows_kernel<<<grid, 256, 0, s>>>(g.T, g.d, ka, (const __nv_bfloat16*)src, u, nu,
                                            (__nv_bfloat16*)out, ust);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

cudaError_t aug_w(const Geom& g, int ka, int64_t R, const void* w, const void* P, int rk, int nu,
                  void* out, cudaStream_t s) {
  prof_begin("lora_aug_w", s);
  const unsigned grid = (unsigned)std::min<int64_t>(R, 148 * 16);
  lora_aug_w_kernel<<<grid, 256, 0, s>>>(R, g.d, ka, (const __nv_bfloat16*)w,
                                         (const __nv_bfloat16*)P, rk, nu, g.D,
                                         (__nv_bfloat16*)out);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

// geometry of the rank-r dense GEMMs: N (router kind) / M (dense_tn kind) = n rows
Geom skinny(const Geom& g, int n) {
  Geom h = g;
  h.G = n;
  h.gpad = (int)ceil_div(n, 16) * 16;
  return h;
}

}  // namespace

cudaError_t lora_fwd_prep(const Geom& g, const void* x, const void* w1, const LoraArgs& lo,
                          cudaStream_t s) {
  const int nu = g.mp * lo.r;
  cudaError_t e = tc_router(skinny(g, nu), x, lo.b1, lo.uv, s);  // U = x B_I
  if (e != cudaSuccess) return e;
  if ((e = aug_rows(g, lo.ka, x, lo.uv, nu, lo.xaug, lo.ust, s)) != cudaSuccess) return e;
  return aug_w(g, lo.ka, (int64_t)g.mp * g.D, w1, lo.c1, lo.r, nu, lo.waug, s);
}

cudaError_t lora_fwd_finish(const Geom& g, const RouteView& r, const Bufs& b, const LoraArgs& lo,
                            void* y, cudaStream_t s) {
  cudaError_t e = launch_rowproj(g, r, b, 1, lo.r, b.h, lo.b2, lo.rowp, s);  // h~ B_O[b]
  if (e != cudaSuccess) return e;
  prof_begin("lora_combine_fwd", s);
  lora_combine_kernel<false><<<(unsigned)g.T, 128, 0, s>>>(
      g.T, g.d, g.k, lo.r, lora_qpad(lo.r), r, (const __nv_bfloat16*)b.part, lo.rowp,
      (const __nv_bfloat16*)lo.c2, nullptr, nullptr, nullptr, (__nv_bfloat16*)y,
      (__nv_bfloat16*)lo.qhl);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

cudaError_t lora_bwd_prep(const Geom& g, const void* dy, const void* w2, const LoraArgs& lo,
                          cudaStream_t s) {
  cudaError_t e = tc_router(skinny(g, lo.r), dy, lo.c2, lo.uv, s);  // V = dy C_O^T
  if (e != cudaSuccess) return e;
  if ((e = aug_rows(g, lo.ka, dy, lo.uv, lo.r, lo.xaug, nullptr, s)) != cudaSuccess) return e;
  return aug_w(g, lo.ka, g.D, w2, lo.b2, lo.r, lo.r, lo.waug, s);
}

cudaError_t lora_bwd_grads(const Geom& g, const RouteView& r, const Bufs& b, const LoraArgs& lo,
                           cudaStream_t s) {
  const int64_t tiles = ceil_div(g.pairs, kTileM) + g.G;
  float* pc1 = lo.gpart;                                     // [tiles, m', bw, r]
  float* pb2 = lo.gpart + tiles * g.mp * g.bw * lo.r;        // [tiles, 1, bw, r]
  cudaError_t e = launch_rowproj(g, r, b, g.mp, lo.r, b.dz, lo.c1, lo.rowp, s);  // du rows
  if (e != cudaSuccess) return e;
  e = launch_colgrad<float>(g, r, b, g.mp, lo.r, b.dz, lo.ust, g.mp * lo.r, pc1, s);
  if (e != cudaSuccess) return e;
  e = launch_colgrad<float>(g, r, b, 1, lo.r, b.h, lo.uv, lo.r, pb2, s);
  if (e != cudaSuccess) return e;
  if ((e = launch_grad_reduce(g, r, g.mp, lo.r, pc1, lo.dc1, lo.accumulate, s)) != cudaSuccess)
    return e;
  return launch_grad_reduce(g, r, 1, lo.r, pb2, lo.db2, lo.accumulate, s);
}

cudaError_t lora_bwd_finish(const Geom& g, const RouteView& r, const Bufs& b, const LoraArgs& lo,
                            const void* x, const void* dy, const void* dense, const void* w_r,
                            void* dx, cudaStream_t s) {
  const int nu = g.mp * lo.r;
  const void* wr = g.gate == SPT_GATE_SIGMOID ? w_r : nullptr;
  prof_begin("lora_combine_bwd", s);
  lora_combine_kernel<true><<<(unsigned)g.T, 128, 0, s>>>(
      g.T, g.d, g.k, nu, lora_upad(g, lo.r), r, (const __nv_bfloat16*)b.part, lo.rowp,
      (const __nv_bfloat16*)lo.b1, dense ? nullptr : b.dlogit, (const __nv_bfloat16*)wr,
      (const __nv_bfloat16*)dense, (__nv_bfloat16*)dx, (__nv_bfloat16*)lo.dhl);
  prof_end(s);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // dB_I^T [m' r, d] = dU^T X ;  dC_O [r, d] = q^T dY
  e = tc_dense_tn(skinny(g, nu), lo.dhl, x, lo.spart, lo.n_split_u, lo.db1, lo.accumulate, s);
  if (e != cudaSuccess) return e;
  return tc_dense_tn(skinny(g, lo.r), lo.qhl, dy, lo.spart, lo.n_split_v, lo.dc2, lo.accumulate,
                     s);
}

}  // namespace spt
