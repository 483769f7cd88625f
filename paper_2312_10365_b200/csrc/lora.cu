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
//   q_t = sum_b h~ B_O[b]                       lora_tile_mma (per pair rows) + token reduce
//   y_t = sum_b P + q_t C_O                     tc_dense_nn (q C_O) + lora_combine_fwd
// Backward (W frozen; routing fixed):
//   v_t = dy_t C_O^T                            tc_router GEMM (N = r)
//   dA  = dy W_O[b]^T + v B_O[b]^T              dA kernel on dY_aug = [dy | hi(v) | lo(v) | 0],
//                                                           W2_aug = [w2 | b2 | b2 | 0]
//   dgate, dZ                                   dA epilogue (unchanged)
//   dB_O[b] = sum_{t in b} h~^T v_t             lora_tile_mma (per tile) + lora_grad_reduce
//   dC_I[:,b]^T = sum_{t in b} dZ^T u_t         lora_tile_mma + lora_grad_reduce
//   du_t = sum_b dZ C_I[:,b]^T                  lora_tile_mma (per pair rows) + token reduce
//   dx_t = sum_b dZ W_I[:,b]^T + router + du_t B_I^T    DX (unchanged) + tc_dense_nn
//                                                       (du B_I^T) + lora_combine_bwd
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
// hi = bf16(u), lo = bf16(u - hi); ust[t] = u[t] (fp32, for the backward).
// One flat grid-stride loop over the 16-byte chunks of the output (a streaming copy
// with several chunks in flight per thread); the ka / 8 tail chunks of a row build
// the hi | lo columns.
__global__ void __launch_bounds__(256) lora_aug_rows_kernel(int64_t T, int d, int ka,
                                                            const __nv_bfloat16* __restrict__ src,
                                                            const float* __restrict__ u, int nu,
                                                            __nv_bfloat16* __restrict__ out,
                                                            float* __restrict__ ust) {
  const int dv = d / 8, wv = (d + ka) / 8;
  const int64_t n = T * wv;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* o4 = reinterpret_cast<uint4*>(out);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
    const int64_t t = e / wv;
    const int c = (int)(e - t * wv);
    if (c < dv) {
      o4[e] = __ldg(s4 + t * dv + c);
      continue;
    }
    const int c0 = (c - dv) * 8;  // tail column of the augmented K stage
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int cc = c0 + i;
      float x = 0.f;
      if (cc < nu) {
        const float f = u[t * nu + cc];
        x = __bfloat162float(__float2bfloat16(f));
        if (ust) ust[t * nu + cc] = f;
      } else if (cc < 2 * nu) {
        const float f = u[t * nu + cc - nu];
        x = f - __bfloat162float(__float2bfloat16(f));
      }
      v[i] = x;
    }
    o4[e] = pack8(v);
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
  // flat grid-stride loop over the 16-byte chunks of the output rows
  const int dv = d / 8, wv = (d + ka) / 8;
  const int64_t n = R * wv;
  const uint4* s4 = reinterpret_cast<const uint4*>(w);
  uint4* o4 = reinterpret_cast<uint4*>(out);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
    const int64_t i = e / wv;
    const int c = (int)(e - i * wv);
    if (c < dv) {
      o4[e] = __ldg(s4 + i * dv + c);
      continue;
    }
    const int off = (int)(i / rows_half) * r;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int cc = (c - dv) * 8 + j;  // augmented column
      const int q = (cc < nu ? cc : cc - nu) - off;
      v[j] = (cc < 2 * nu && q >= 0 && q < r) ? P[i * r + q] : __float2bfloat16(0.f);
    }
    o4[e] = *reinterpret_cast<const uint4*>(v);
  }
}

// out[m][b bw + i][q] (=|+=) sum over block b's tiles (ascending) of
// part[tile][slab0 + m][i][q] (per-tile partials with `slabs` slabs per tile)
__global__ void __launch_bounds__(256) lora_grad_reduce_kernel(int G, int bw, int mp, int r,
                                                               int64_t D, RouteView rv, int slabs,
                                                               int slab0,
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
    s += part[(((int64_t)tile * slabs + slab0 + m) * bw + i) * r + q];
  out[idx] = acc ? out[idx] + s : s;
}

// Per token t (one CTA):
//   out[t] = sum_{j asc} part[prow(t,j)] + router term + lora[t]
// router term as combine_bwd (dense [T,d] if `dense`, else sum_j dlogit w_r[b_j]
// when w_r; none in the forward); lora = the dense rank-r term (q C_O forward,
// du B_I^T backward) computed on tensor cores by tc_dense_nn.
template <bool kBwd>
__global__ void __launch_bounds__(128) lora_combine_kernel(int64_t T, int d, int k, RouteView r,
                                                           const __nv_bfloat16* __restrict__ part,
                                                           const float* __restrict__ dlogit,
                                                           const __nv_bfloat16* __restrict__ w_r,
                                                           const __nv_bfloat16* __restrict__ dense,
                                                           const __nv_bfloat16* __restrict__ lora,
                                                           __nv_bfloat16* __restrict__ out) {
  __shared__ int64_t rows[kMaxBlocks];
  __shared__ int blk[kMaxBlocks];
  __shared__ float dl[kMaxBlocks];
  const int64_t t = blockIdx.x;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    rows[j] = pair_row(r, t, k, j);
    if (kBwd && dlogit) {
      blk[j] = r.topk_idx[t * k + j];
      dl[j] = dlogit[rows[j]];
    }
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
    float v[8];
    load8(lora + t * d + c, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] += v[i];
    *reinterpret_cast<uint4*>(out + t * d + c) = pack8(acc);
  }
}

cudaError_t launch_grad_reduce(const Geom& g, const RouteView& r, int mp, int rk, int slabs,
                               int slab0, const float* part, float* out, bool acc, cudaStream_t s) {
  const int64_t n = (int64_t)mp * g.D * rk;
  prof_begin("lora_grad_reduce", s);
  lora_grad_reduce_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(
      g.G, g.bw, mp, rk, g.D, r, slabs, slab0, part, out, acc ? 1 : 0);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

cudaError_t aug_rows(const Geom& g, int ka, const void* src, const float* u, int nu, void* out,
                     float* ust, cudaStream_t s) {
  prof_begin("lora_aug_rows", s);
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(g.T * ((g.d + ka) / 8), 256), 148 * 32);
  lora_aug_rows_kernel<<<grid, 256, 0, s>>>(g.T, g.d, ka, (const __nv_bfloat16*)src, u, nu,
                                            (__nv_bfloat16*)out, ust);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

cudaError_t aug_w(const Geom& g, int ka, int64_t R, const void* w, const void* P, int rk, int nu,
                  void* out, cudaStream_t s) {
  prof_begin("lora_aug_w", s);
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(R * ((g.d + ka) / 8), 256), 148 * 32);
  lora_aug_w_kernel<<<grid, 256, 0, s>>>(R, g.d, ka, (const __nv_bfloat16*)w,
                                         (const __nv_bfloat16*)P, rk, nu, g.D,
                                         (__nv_bfloat16*)out);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Tensor-core (mma.sync m16n8k16 bf16 -> fp32) form of the rank-r per-tile
// products, one CTA (8 warps) per 128-row bucket tile of block b:
//   rows:  out[prow, m r + q]   = sum_i A[prow, m bw + i] P[m][b bw + i][q]       (q / du rows)
//   cols:  part[tile][m][i][q]  = sum_rows A[prow, m bw + i] E[t(row), m r + q]   (dC_I, dB_O)
// A tiles are staged in shared memory once per 128-feature chunk and feed
// both products (ldmatrix for the row product, ldmatrix.trans for the column
// product); E is split into bf16 hi + lo halves (two MMAs) so the gradient
// keeps ~16 significant bits.
constexpr int kMmaRows = 128;
constexpr int kMmaChunk = 128;                 // features per staged chunk
constexpr int kMmaPitch = kMmaChunk + 8;       // +16 B per row: conflict-free ldmatrix
constexpr int kMmaEPitch = kMmaRows + 8;

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Grid: (tile, 128-feature chunk of the block); each chunk writes its own
// partial row products (summed by the token reduce), so wide blocks
// (bw = 1024-2752) spread over bw/128 CTAs per tile.
// mode 0 (forward): rows only, A = h~ (m' = 1), P = B_O  -> q rows
// mode 1 (backward): A = dZ: rows (P = C_I^T -> du rows) and cols (E = u -> dC_I);
//                    then A = h~: cols (E = v -> dB_O)
template <int RP>
__global__ void __launch_bounds__(256) lora_tile_mma_kernel(
    int mode, int G, int bw, int mp, int r, int64_t D, RouteView rv,
    const int32_t* __restrict__ tile_block, const __nv_bfloat16* __restrict__ A,
    const __nv_bfloat16* __restrict__ P, const float* __restrict__ U, int upitch,
    const __nv_bfloat16* __restrict__ H, const float* __restrict__ V, float* __restrict__ rows_out,
    int64_t rows_stride, float* __restrict__ part) {
  constexpr int NT = RP / 8;  // n8 tiles
  extern __shared__ __align__(16) uint8_t mma_smem[];
  __nv_bfloat16* As = reinterpret_cast<__nv_bfloat16*>(mma_smem);   // [row][feature]
  __nv_bfloat16* Pt = As + kMmaRows * kMmaPitch;                     // [q][i]
  __nv_bfloat16* Eh = Pt + RP * kMmaPitch;                           // [q][row] hi
  __nv_bfloat16* El = Eh + RP * kMmaEPitch;                          // [q][row] lo
  __shared__ int tok[kMmaRows];
  const int tile = blockIdx.x;
  if (tile >= rv.tile_offsets[G]) return;
  const int b = tile_block[tile];
  const int mt = tile - rv.tile_offsets[b];
  const int nb = rv.block_offsets[b + 1] - rv.block_offsets[b];
  const int nvalid = min(kMmaRows, nb - mt * kMmaRows);
  const int pos0 = rv.block_offsets[b] + mt * kMmaRows;
  const int64_t prow0 = (int64_t)tile * kMmaRows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  if (threadIdx.x < kMmaRows)
    tok[threadIdx.x] = (int)threadIdx.x < nvalid ? rv.bucket_token[pos0 + threadIdx.x] : 0;

  // stage rows [0,128) x features [f0, f0 + ni) of X (pitch xw) into As (zero rows >= nvalid)
  // issue (cp.async, no wait) rows [0,128) x features [f0, f0 + ni) of X (pitch xw)
  // into As; rows >= nvalid are zero.  Completed by cp_async_wait_all + barrier.
  auto stage_a = [&](const __nv_bfloat16* X, int xw, int f0, int ni) {
    const int v8 = ni / 8;
    for (int e = threadIdx.x; e < kMmaRows * v8; e += blockDim.x) {
      const int row = e / v8, cc = (e % v8) * 8;
      __nv_bfloat16* dst = &As[row * kMmaPitch + cc];
      if (row < nvalid) cp_async16(dst, X + (prow0 + row) * xw + f0 + cc);
      else *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    }
  };
  // stage E[t(row)][eoff + q] (fp32) as bf16 hi / lo, transposed [q][row]
  auto stage_e = [&](const float* E, int epitch, int eoff) {
    for (int e = threadIdx.x; e < RP * kMmaRows; e += blockDim.x) {
      const int row = e / RP, q = e % RP;  // consecutive threads read one token's row
      float v = 0.f;
      if (row < nvalid && q < r) v = E[(int64_t)tok[row] * epitch + eoff + q];
      const __nv_bfloat16 hi = __float2bfloat16(v);
      Eh[q * kMmaEPitch + row] = hi;
      El[q * kMmaEPitch + row] = __float2bfloat16(v - __bfloat162float(hi));
    }
  };
  // column product over the staged chunk: part rows [f0, f0 + ni) of slab m
  auto cols = [&](int ni, float* dst) {
    // warp w: features [16w, 16w + 16) of the chunk (ni <= 128 -> <= 8 m16 tiles)
    if (warp * 16 < ni) {
      float acc[NT][4];
#pragma unroll
      for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
#pragma unroll 2
      for (int k0 = 0; k0 < kMmaRows; k0 += 16) {
        // A^T fragment (m = feature, k = row) from As[row][feature] via ldmatrix.trans
        const int mi = lane >> 3, rr = lane & 7;
        const int krow = k0 + rr + ((mi & 2) ? 8 : 0);
        const int mcol = warp * 16 + ((mi & 1) ? 8 : 0);
        uint32_t a[4];
        ldsm_x4_t(a, &As[krow * kMmaPitch + mcol]);
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const __nv_bfloat16* eh = &Eh[(n * 8 + g) * kMmaEPitch + k0 + 2 * c];
          const __nv_bfloat16* el = &El[(n * 8 + g) * kMmaEPitch + k0 + 2 * c];
          mma16816(acc[n], a, *reinterpret_cast<const uint32_t*>(eh),
                   *reinterpret_cast<const uint32_t*>(eh + 8));
          mma16816(acc[n], a, *reinterpret_cast<const uint32_t*>(el),
                   *reinterpret_cast<const uint32_t*>(el + 8));
        }
      }
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int q0 = n * 8 + 2 * c;
        const int i0 = warp * 16 + g;
        if (q0 < r) {
          dst[(int64_t)i0 * r + q0] = acc[n][0];
          dst[(int64_t)(i0 + 8) * r + q0] = acc[n][2];
        }
        if (q0 + 1 < r) {
          dst[(int64_t)i0 * r + q0 + 1] = acc[n][1];
          dst[(int64_t)(i0 + 8) * r + q0 + 1] = acc[n][3];
        }
      }
    }
  };

  const __nv_bfloat16* Arow = mode == 0 ? H : A;  // the row product's operand
  const int aw = mode == 0 ? bw : mp * bw;
  const int mrows = mode == 0 ? 1 : mp;
  for (int m = 0; m < mrows; ++m) {
    float racc[NT][4];  // row product: warp w owns rows [16w, 16w + 16)
#pragma unroll
    for (int n = 0; n < NT; ++n) racc[n][0] = racc[n][1] = racc[n][2] = racc[n][3] = 0.f;
    {  // this CTA's 128-feature chunk (blockIdx.y) of the block
      const int i0 = blockIdx.y * kMmaChunk;
      const int ni = min(kMmaChunk, bw - i0);
      __syncthreads();  // the previous stage's readers are done
      stage_a(Arow, aw, m * bw + i0, ni);  // async; overlaps the E / P staging below
      if (mode == 1) stage_e(U, upitch, m * r);
      for (int e = threadIdx.x; e < RP * ni; e += blockDim.x) {
        const int i = e / RP, q = e % RP;  // consecutive threads read one feature's r values
        Pt[q * kMmaPitch + i] =
            q < r ? P[((int64_t)m * D + (int64_t)b * bw + i0 + i) * r + q] : __float2bfloat16(0.f);
      }
      cp_async_wait_all();
      __syncthreads();
      // row product: M = rows, K = features of the chunk, N = RP
      for (int k0 = 0; k0 < ni; k0 += 16) {
        const int mi = lane >> 3, rr = lane & 7;
        uint32_t a[4];
        ldsm_x4(a, &As[(warp * 16 + rr + ((mi & 1) ? 8 : 0)) * kMmaPitch + k0 + ((mi & 2) ? 8 : 0)]);
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const __nv_bfloat16* pb = &Pt[(n * 8 + g) * kMmaPitch + k0 + 2 * c];
          mma16816(racc[n], a, *reinterpret_cast<const uint32_t*>(pb),
                   *reinterpret_cast<const uint32_t*>(pb + 8));
        }
      }
      if (mode == 1)  // dC_I^T rows [b bw + i0, +ni) of slab m
        cols(ni, part + (((int64_t)tile * (mp + 1) + m) * bw + i0) * r);
    }
    // rows out: [chunk][prow, m r + q] (the chunks' partial sums, added by the token reduce)
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int q0 = n * 8 + 2 * c;
      const int row = warp * 16 + g;
      float* rb = rows_out + blockIdx.y * rows_stride;
      float* o0 = rb + (prow0 + row) * kLoraK + m * r;
      float* o1 = rb + (prow0 + row + 8) * kLoraK + m * r;
      if (row < nvalid) {
        if (q0 < r) o0[q0] = racc[n][0];
        if (q0 + 1 < r) o0[q0 + 1] = racc[n][1];
      }
      if (row + 8 < nvalid) {
        if (q0 < r) o1[q0] = racc[n][2];
        if (q0 + 1 < r) o1[q0 + 1] = racc[n][3];
      }
    }
  }
  if (mode == 1) {  // dB_O: A = h~, E = v
    {
      const int i0 = blockIdx.y * kMmaChunk;
      const int ni = min(kMmaChunk, bw - i0);
      __syncthreads();
      stage_a(H, bw, i0, ni);
      stage_e(V, r, 0);
      cp_async_wait_all();
      __syncthreads();
      cols(ni, part + (((int64_t)tile * (mp + 1) + mp) * bw + i0) * r);
    }
  }
}

// Per token (one warp): s[c] = sum_{j asc} rowp[prow(t,j)][c] (c < ns) as bf16 hi|lo
// halves [2, T, spitch] -- the A operand of the du B_I^T GEMM.
__global__ void __launch_bounds__(256) lora_token_reduce_kernel(int64_t T, int k, int ns,
                                                                int spitch, RouteView r,
                                                                const float* __restrict__ rowp,
                                                                int nch, int64_t rows_stride,
                                                                __nv_bfloat16* __restrict__ shl) {
  __shared__ int64_t rows[8][kMaxBlocks];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * 8 + w;
  if (t >= T) return;  // whole warp
  for (int j = lane; j < k; j += 32) rows[w][j] = pair_row(r, t, k, j) * kLoraK;  // in parallel
  __syncwarp();
  for (int c = lane; c < spitch; c += 32) {
    float v = 0.f;
    if (c < ns)
#pragma unroll 4
      for (int j = 0; j < k; ++j) {  // ascending blocks (c12); independent loads
        const int64_t row = rows[w][j] + c;
        for (int ch = 0; ch < nch; ++ch) v += rowp[ch * rows_stride + row];
      }
    const __nv_bfloat16 hi = __float2bfloat16(v);
    shl[t * spitch + c] = hi;
    shl[(T + t) * spitch + c] = __float2bfloat16(v - __bfloat162float(hi));
  }
}

template <int RP>
constexpr size_t tile_mma_smem() {
  return (size_t)(kMmaRows * kMmaPitch + RP * kMmaPitch + 2 * RP * kMmaEPitch) * 2;
}

template <int RP>
cudaError_t tile_mma(int mode, const Geom& g, const RouteView& r, const Bufs& b, const LoraArgs& lo,
                     const void* P, cudaStream_t s) {
  constexpr size_t smem = tile_mma_smem<RP>();
  cudaError_t e = cudaFuncSetAttribute(lora_tile_mma_kernel<RP>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((unsigned)(ceil_div(g.pairs, kTileM) + g.G), (unsigned)lora_chunks(g));
  lora_tile_mma_kernel<RP><<<grid, 256, smem, s>>>(
      mode, g.G, g.bw, g.mp, lo.r, g.D, r, b.tile_block, (const __nv_bfloat16*)b.dz,
      (const __nv_bfloat16*)P, lo.ust, g.mp * lo.r, (const __nv_bfloat16*)b.h, lo.uv, lo.rowp,
      lora_rows_stride(g), lo.gpart);
  return cudaGetLastError();
}

// mode 0: q rows (h~ B_O[b]);  mode 1: du rows (dZ C_I[b]) + per-tile dC_I / dB_O partials
cudaError_t launch_tile_mma(int mode, const Geom& g, const RouteView& r, const Bufs& b,
                            const LoraArgs& lo, cudaStream_t s) {
  const void* P = mode == 0 ? lo.b2 : lo.c1;
  prof_begin(mode == 0 ? "lora_rows_fwd" : "lora_tiles_bwd", s);
  cudaError_t e = lo.r <= 8    ? tile_mma<8>(mode, g, r, b, lo, P, s)
                  : lo.r <= 16 ? tile_mma<16>(mode, g, r, b, lo, P, s)
                  : lo.r <= 32 ? tile_mma<32>(mode, g, r, b, lo, P, s)
                               : tile_mma<64>(mode, g, r, b, lo, P, s);
  prof_end(s);
  count_launch();
  return e;
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
  cudaError_t e = launch_tile_mma(0, g, r, b, lo, s);  // q rows: h~ B_O[b]
  if (e != cudaSuccess) return e;
  // q = sum_b q rows -> hi|lo (stashed for dC_O); the dense q C_O term on tensor
  // cores into the (now free) X_aug buffer; the combine adds it to the partials
  const int qpad = lora_qpad(lo.r);
  prof_begin("lora_token_reduce", s);
  lora_token_reduce_kernel<<<(unsigned)ceil_div(g.T, 8), 256, 0, s>>>(
      g.T, g.k, lo.r, qpad, r, lo.rowp, lora_chunks(g), lora_rows_stride(g),
      (__nv_bfloat16*)lo.qhl);
  prof_end(s);
  count_launch();
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = tc_dense_nn(skinny(g, lo.r), lo.qhl, lo.c2, lo.xaug, s)) != cudaSuccess) return e;
  prof_begin("lora_combine_fwd", s);
  lora_combine_kernel<false><<<(unsigned)g.T, 128, 0, s>>>(
      g.T, g.d, g.k, r, (const __nv_bfloat16*)b.part, nullptr, nullptr, nullptr,
      (const __nv_bfloat16*)lo.xaug, (__nv_bfloat16*)y);
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
  // du rows (dZ C_I[b]) and per-tile [m' + 1] slabs: dC_I^T (m' slabs), dB_O
  cudaError_t e = launch_tile_mma(1, g, r, b, lo, s);
  if (e != cudaSuccess) return e;
  const int slabs = g.mp + 1;
  if ((e = launch_grad_reduce(g, r, g.mp, lo.r, slabs, 0, lo.gpart, lo.dc1, lo.accumulate, s)) !=
      cudaSuccess)
    return e;
  return launch_grad_reduce(g, r, 1, lo.r, slabs, g.mp, lo.gpart, lo.db2, lo.accumulate, s);
}

cudaError_t lora_bwd_finish(const Geom& g, const RouteView& r, const Bufs& b, const LoraArgs& lo,
                            const void* x, const void* dy, const void* dense, const void* w_r,
                            void* dx, cudaStream_t s) {
  const int nu = g.mp * lo.r;
  const int upad = lora_upad(g, lo.r);
  const void* wr = g.gate == SPT_GATE_SIGMOID ? w_r : nullptr;
  // dU rows -> hi|lo; the dense du B_I^T term on tensor cores into the (now free)
  // dY_aug buffer; the combine adds it next to the partials and the router term
  prof_begin("lora_token_reduce", s);
  lora_token_reduce_kernel<<<(unsigned)ceil_div(g.T, 8), 256, 0, s>>>(
      g.T, g.k, nu, upad, r, lo.rowp, lora_chunks(g), lora_rows_stride(g),
      (__nv_bfloat16*)lo.dhl);
  prof_end(s);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  Geom gu = skinny(g, nu);
  if ((e = tc_dense_nn(gu, lo.dhl, lo.b1, lo.xaug, s)) != cudaSuccess) return e;
  prof_begin("lora_combine_bwd", s);
  lora_combine_kernel<true><<<(unsigned)g.T, 128, 0, s>>>(
      g.T, g.d, g.k, r, (const __nv_bfloat16*)b.part, dense ? nullptr : b.dlogit,
      (const __nv_bfloat16*)wr, (const __nv_bfloat16*)dense, (const __nv_bfloat16*)lo.xaug,
      (__nv_bfloat16*)dx);
  prof_end(s);
  count_launch();
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // dB_I^T [m' r, d] = dU^T X ;  dC_O [r, d] = q^T dY
  e = tc_dense_tn(gu, lo.dhl, x, lo.spart, lo.n_split_u, lo.db1, lo.accumulate, s);
  if (e != cudaSuccess) return e;
  return tc_dense_tn(skinny(g, lo.r), lo.qhl, dy, lo.spart, lo.n_split_v, lo.dc2, lo.accumulate,
                     s);
}

}  // namespace spt
