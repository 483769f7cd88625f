// topl.cu -- SPT's bucket-sort top-L selection for sparse MHA:
// Eq. 3 integer similarity s(q,k) = sum_m I[t^m_q = t^m_k] and
// Algorithm 3 with readings c20-c23.
//
// The paper runs one thread per query with M+1 buckets of L slots in shared
// memory (plus two helper threads).  On sm_100a the same
// result comes from counting instead of storing buckets:
//   * one CTA per (head, query chunk) stages the head's key codes in shared
//     memory once (4 codes per 32-bit word; 16-byte loads per key);
//   * one warp per query, keys on lanes: pass 1 scores every key (XOR + zero-
//     byte test + POPC per word), keeps the per-key score bytes in shared
//     memory and builds the M+1 bucket counts with warp-aggregated updates
//     (match.any + one leader per score value) plus each bucket's last key;
//   * a lane-parallel scan over the buckets (score M first) gives each
//     bucket's output base and how many of its slots retrieval reads
//     (min(count, L), cut at L total) -- Alg. 3 lines 9-16 as arithmetic;
//   * pass 2 walks the score bytes in key order and writes each bucket's first
//     keys to their final positions (rank inside the bucket from match.any);
//     slot L-1 of an overflowed bucket is its last key (line 7's overwrite, c21).
// Everything is integer: results are bit-exact and deterministic.
#include "internal.h"

namespace spt {

namespace {

constexpr int kToplWarps = 16;
constexpr int kToplThreads = kToplWarps * 32;
constexpr int kMaxScore = 31;  // M <= 31: M + 1 buckets fit one warp

template <int NW>  // 32-bit code words per vector (M <= 4 NW)
__device__ __forceinline__ int score_words(const uint32_t (&q)[NW], const uint32_t* k) {
  int diff = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t v = q[w] ^ k[w];  // byte is 0 iff the codewords agree
    // high bit of each byte set iff the byte is non-zero (no carry across bytes)
    const uint32_t t = ((v & 0x7f7f7f7fu) + 0x7f7f7f7fu) | v;
    diff += __popc(t & 0x80808080u);  // differing codebooks in this word
  }
  return diff;
}

template <int NW>
__global__ void __launch_bounds__(kToplThreads) topl_kernel(int H, int nq, int nk, int M, int L,
                                                           int causal, int qpb,
                                                           const uint8_t* __restrict__ cq,
                                                           const uint8_t* __restrict__ ck,
                                                           int32_t* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int KW = NW == 3 ? 4 : NW;  // smem words per key (16-byte aligned rows for NW = 3)
  uint32_t* kw = reinterpret_cast<uint32_t*>(smem);                         // [nk][KW]
  uint8_t* sc = smem + (size_t)nk * KW * 4;                                  // [warps][nk]
  __shared__ int hist[kToplWarps][kMaxScore + 1];
  __shared__ int last[kToplWarps][kMaxScore + 1];
  __shared__ int base[kToplWarps][kMaxScore + 1];
  __shared__ int take[kToplWarps][kMaxScore + 1];
  __shared__ int seen[kToplWarps][kMaxScore + 1];

  // CTA (h, c) takes the queries q = c, c + chunks, c + 2 chunks, ... of head h:
  // interleaved, so causal rows (work ~ q) are balanced across CTAs
  const int chunks = (nq + qpb - 1) / qpb;
  const int h = blockIdx.x / chunks;
  const int c = blockIdx.x % chunks;
  const int q_last = c + ((nq - 1 - c) / chunks) * chunks;  // this CTA's last query
  const int nk_used = causal ? min(nk, q_last + 1) : nk;   // causal: later keys unused
  const int pad = NW * 4 - M;                      // zero pad bytes compare equal: subtract
  // stage the head's key codes: key k -> words [k*KW, k*KW + NW), pad bytes 0
  {
    const uint8_t* src = ck + (size_t)h * nk * M;
    for (int e = threadIdx.x; e < nk_used * KW; e += blockDim.x) {
      const int k = e / KW, w = e % KW;
      uint32_t v = 0;
      if (w < NW) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int m = w * 4 + b;
          if (m < M) v |= (uint32_t)src[(size_t)k * M + m] << (8 * b);
        }
      }
      kw[e] = v;
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  uint8_t* my = sc + (size_t)warp * nk;
  for (int q = c + warp * chunks; q < nq; q += kToplWarps * chunks) {
    uint32_t qv[NW];
    {
      const uint8_t* src = cq + ((size_t)h * nq + q) * M;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int m = w * 4 + b;
          if (m < M) v |= (uint32_t)__ldg(src + m) << (8 * b);
        }
        qv[w] = v;
      }
    }
    const int nc = causal ? min(nk, q + 1) : nk;  // candidates (c23)
    if (lane <= M) {
      hist[warp][lane] = 0;
      seen[warp][lane] = 0;
    }
    __syncwarp();
    // pass 1 (Alg. 3 lines 3-8): scores, bucket counts, last key per bucket
    for (int k0 = 0; k0 < nc; k0 += 32) {
      const int k = k0 + lane;
      const bool ok = k < nc;
      int s = -1;
      if (ok) {
        uint32_t kv[KW];
        if (KW == 4) {
          const uint4 t = *reinterpret_cast<const uint4*>(kw + (size_t)k * KW);
          kv[0] = t.x; kv[1] = t.y; kv[2] = t.z; kv[3] = t.w;
        } else if (KW == 2) {
          const uint2 t = *reinterpret_cast<const uint2*>(kw + (size_t)k * KW);
          kv[0] = t.x; kv[1] = t.y;
        } else {
#pragma unroll
          for (int w = 0; w < KW; ++w) kv[w] = kw[(size_t)k * KW + w];
        }
        s = NW * 4 - pad - score_words<NW>(qv, kv);  // Eq. 3
        my[k] = (uint8_t)s;
      }
      const unsigned act = __ballot_sync(0xffffffffu, ok);
      if (ok) {
        const unsigned grp = __match_any_sync(act, s);
        if ((grp & lt) == 0) {  // group leader: lowest lane of this score value
          hist[warp][s] += __popc(grp);
          last[warp][s] = k0 + 31 - __clz(grp);  // highest key of the group so far
        }
      }
      __syncwarp();  // leaders' hist / last updates visible to the next chunk's leaders
    }
    // Alg. 3 lines 9-16 as a scan: bucket M first; bucket s is read for
    // min(count, L) slots (c21) until L keys are collected (c20)
    {
      const int s = M - lane;  // lane 0 = bucket M
      const int rd = s >= 0 ? min(hist[warp][s], L) : 0;
      int inc = rd;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
      }
      const int b = inc - rd;
      if (s >= 0) {
        base[warp][s] = b;
        take[warp][s] = max(0, min(rd, L - b));
      }
    }
    __syncwarp();
    int32_t* orow = out + ((size_t)h * nq + q) * L;
    // rows with fewer than L candidates: pad (c23)
    for (int i = min(nc, L) + lane; i < L; i += 32) orow[i] = -1;
    // slot L-1 of a bucket read to its end holds its last key (line 7 overwrite)
    if (lane <= M && take[warp][lane] == L) orow[base[warp][lane] + L - 1] = last[warp][lane];
    // pass 2: first keys of each bucket in key order -> positions base + rank
    for (int k0 = 0; k0 < nc; k0 += 32) {
      const int k = k0 + lane;
      const bool ok = k < nc;
      const int s = ok ? (int)my[k] : -1;
      const unsigned act = __ballot_sync(0xffffffffu, ok);
      if (ok) {
        const unsigned grp = __match_any_sync(act, s);
        const int pos = seen[warp][s] + __popc(grp & lt);
        const int lim = min(take[warp][s], L - 1);  // slot L-1 handled above
        if (pos < lim) orow[base[warp][s] + pos] = k;
        __syncwarp(act);
        if ((grp & lt) == 0) seen[warp][s] += __popc(grp);
      }
      __syncwarp();
    }
    __syncwarp();
  }
}

template <int NW>
cudaError_t launch_topl_nw(int H, int nq, int nk, int M, int L, int causal, const uint8_t* cq,
                           const uint8_t* ck, int32_t* out, size_t smem, int qpb, cudaStream_t s) {
  const int chunks = (nq + qpb - 1) / qpb;
  cudaError_t e = cudaFuncSetAttribute(topl_kernel<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  topl_kernel<NW><<<(unsigned)((int64_t)H * chunks), kToplThreads, smem, s>>>(H, nq, nk, M, L,
                                                                             causal, qpb, cq, ck, out);
  return cudaGetLastError();
}

}  // namespace

size_t topl_smem_bytes(int nk, int M) {
  const int NW = (M + 3) / 4;
  const int KW = NW == 3 ? 4 : NW;
  return (size_t)nk * KW * 4 + (size_t)kToplWarps * nk;
}

int topl_max_score() { return kMaxScore; }

cudaError_t launch_topl(int H, int nq, int nk, int M, int L, int causal, const uint8_t* cq,
                        const uint8_t* ck, int32_t* out, cudaStream_t s) {
  const size_t smem = topl_smem_bytes(nk, M);
  // queries per CTA: enough CTAs to fill the SMs, each staging its head's keys once
  int qpb = 64;
  while (qpb < 1024 && (int64_t)H * ((nq + 2 * qpb - 1) / (2 * qpb)) >= 2 * 148) qpb *= 2;
  prof_begin("topl_select", s);
  const int NW = (M + 3) / 4;
  cudaError_t e;
  switch (NW) {
    case 1: e = launch_topl_nw<1>(H, nq, nk, M, L, causal, cq, ck, out, smem, qpb, s); break;
    case 2: e = launch_topl_nw<2>(H, nq, nk, M, L, causal, cq, ck, out, smem, qpb, s); break;
    case 3: e = launch_topl_nw<3>(H, nq, nk, M, L, causal, cq, ck, out, smem, qpb, s); break;
    case 4: e = launch_topl_nw<4>(H, nq, nk, M, L, causal, cq, ck, out, smem, qpb, s); break;
    case 5: e = launch_topl_nw<5>(H, nq, nk, M, L, causal, cq, ck, out, smem, qpb, s); break;
    case 6: e = launch_topl_nw<6>(H, nq, nk, M, L, causal, cq, ck, out, smem, qpb, s); break;
    case 7: e = launch_topl_nw<7>(H, nq, nk, M, L, causal, cq, ck, out, smem, qpb, s); break;
    default: e = launch_topl_nw<8>(H, nq, nk, M, L, causal, cq, ck, out, smem, qpb, s); break;
  }
  prof_end(s);
  count_launch();
  return e;
}

}  // namespace spt
