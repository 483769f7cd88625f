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

// Codes are packed CPW per 32-bit word: 4 bytes, or 8 nibbles when every
// codebook has E <= 16 codewords (the paper's setting: half the
// words, half the ALU work).
template <int NW, int CPW>
__device__ __forceinline__ int score_words(const uint32_t (&q)[NW], const uint32_t* k) {
  constexpr uint32_t lo = CPW == 4 ? 0x7f7f7f7fu : 0x77777777u;
  constexpr uint32_t hi = CPW == 4 ? 0x80808080u : 0x88888888u;
  int diff = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t v = q[w] ^ k[w];  // field is 0 iff the codewords agree
    // top bit of each field set iff the field is non-zero (no carry across fields)
    const uint32_t t = ((v & lo) + lo) | v;
    diff += __popc(t & hi);  // differing codebooks in this word
  }
  return diff;
}

template <int CPW>
__device__ __forceinline__ uint32_t pack_codes(const uint8_t* src, int w, int M) {
  constexpr int SH = 32 / CPW;
  uint32_t v = 0;
#pragma unroll
  for (int b = 0; b < CPW; ++b) {
    const int m = w * CPW + b;
    // mask to the field width: an out-of-range code (>= E, "unspecified result"
    // per the header) must not spill into the next field, or a score could
    // exceed M and index the bucket arrays out of bounds
    if (m < M) v |= ((uint32_t)src[m] & (CPW == 8 ? 0xFu : 0xFFu)) << (SH * b);
  }
  return v;
}

template <int NW, int CPW>
__global__ void __launch_bounds__(kToplThreads) topl_kernel(int H, int nq, int nk, int M, int L,
                                                           int causal, int qpb,
                                                           const uint8_t* __restrict__ cq,
                                                           const uint8_t* __restrict__ ck,
                                                           int32_t* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int KW = NW == 3 ? 4 : NW;  // smem words per key (16-byte aligned rows for NW = 3)
  uint32_t* kw = reinterpret_cast<uint32_t*>(smem);                         // [nk][KW]
  uint8_t* sc = smem + (size_t)nk * KW * 4;                                  // [warps][nk]
  __shared__ __align__(16) uint16_t cnt[kToplWarps][kMaxScore + 1][32];  // per-lane counts
  // per bucket: {keys still to place, first keys to place, output base, -}
  __shared__ int4 bk[kToplWarps][kMaxScore + 1];

  // CTA (h, c) takes the queries q = c, c + chunks, c + 2 chunks, ... of head h:
  // interleaved, so causal rows (work ~ q) are balanced across CTAs
  const int chunks = (nq + qpb - 1) / qpb;
  const int h = blockIdx.x / chunks;
  const int c = blockIdx.x % chunks;
  const int q_last = c + ((nq - 1 - c) / chunks) * chunks;  // this CTA's last query
  const int nk_used = causal ? min(nk, q_last + 1) : nk;   // causal: later keys unused
  const int pad = NW * CPW - M;                    // zero pad fields compare equal: subtract
  // stage the head's key codes: key k -> words [k*KW, k*KW + NW), pad bytes 0
  {
    const uint8_t* src = ck + (size_t)h * nk * M;
    for (int e = threadIdx.x; e < nk_used * KW; e += blockDim.x) {
      const int k = e / KW, w = e % KW;
      kw[e] = w < NW ? pack_codes<CPW>(src + (size_t)k * M, w, M) : 0u;
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;  // lanes below this one
  uint8_t* my = sc + (size_t)warp * nk;
  for (int q = c + warp * chunks; q < nq; q += kToplWarps * chunks) {
    uint32_t qv[NW];
    {
      const uint8_t* src = cq + ((size_t)h * nq + q) * M;
#pragma unroll
      for (int w = 0; w < NW; ++w) qv[w] = pack_codes<CPW>(src, w, M);
    }
    const int nc = causal ? min(nk, q + 1) : nk;  // candidates (c23)
    for (int v = 0; v <= M; ++v) cnt[warp][v][lane] = 0;  // this lane's column
    // pass 1 (Alg. 3 lines 3-8): scores and bucket counts (per lane, no
    // cross-lane traffic: every lane counts the keys it scored).  Full 32-key
    // batches run unguarded; the ragged tail once.
    const int full_score = NW * CPW - pad;
    uint16_t* mycnt = &cnt[warp][0][lane];
    auto score_key = [&](int k) {
      uint32_t kv[KW];
      if (KW == 4) {
        const uint4 t = *reinterpret_cast<const uint4*>(kw + k * KW);
        kv[0] = t.x; kv[1] = t.y; kv[2] = t.z; kv[3] = t.w;
      } else if (KW == 2) {
        const uint2 t = *reinterpret_cast<const uint2*>(kw + k * KW);
        kv[0] = t.x; kv[1] = t.y;
      } else {
#pragma unroll
        for (int w = 0; w < KW; ++w) kv[w] = kw[k * KW + w];
      }
      const int s = full_score - score_words<NW, CPW>(qv, kv);  // Eq. 3
      my[k] = (uint8_t)s;
      mycnt[s * 32] += 1;
    };
    const int nfull = nc & ~31;
#pragma unroll 4
    for (int k0 = 0; k0 < nfull; k0 += 32) score_key(k0 + lane);
    if (nfull + lane < nc) score_key(nfull + lane);
    __syncwarp();
    // Alg. 3 lines 9-16 as a scan: bucket M first; bucket s is read for
    // min(count, L) slots (c21) until L keys are collected (c20)
    int s_over = -1;  // the bucket read to its slot L-1 (holds its last key), if any
    int remaining;    // keys pass 2 must place
    {
      const int s = M - lane;  // lane 0 = bucket M
      int count = 0;
      if (s >= 0) {
        const uint4* row = reinterpret_cast<const uint4*>(&cnt[warp][s][0]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint4 v = row[i];
          count += (int)(v.x & 0xffff) + (int)(v.x >> 16) + (int)(v.y & 0xffff) + (int)(v.y >> 16) +
                   (int)(v.z & 0xffff) + (int)(v.z >> 16) + (int)(v.w & 0xffff) + (int)(v.w >> 16);
        }
      }
      const int rd = min(count, L);
      int inc = rd;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
      }
      const int b = inc - rd;
      const int take = max(0, min(rd, L - b));
      const int lm = min(take, L - 1);  // slot L-1 is written separately
      if (s >= 0) bk[warp][s] = make_int4(lm, lm, b, 0);
      const unsigned ov = __ballot_sync(0xffffffffu, s >= 0 && take == L);
      if (ov) s_over = M - (__ffs(ov) - 1);
      remaining = lm;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) remaining += __shfl_xor_sync(0xffffffffu, remaining, o);
    }
    __syncwarp();
    int32_t* orow = out + ((size_t)h * nq + q) * L;
    // rows with fewer than L candidates: pad (c23)
    for (int i = min(nc, L) + lane; i < L; i += 32) orow[i] = -1;
    // slot L-1 of the bucket read to its end holds its last key (line 7 overwrite):
    // the highest key of that score, found scanning back from the end
    if (s_over >= 0) {
      for (int k0 = ((nc - 1) / 32) * 32; k0 >= 0; k0 -= 32) {
        const int k = k0 + lane;
        const unsigned hit = __ballot_sync(0xffffffffu, k < nc && (int)my[k] == s_over);
        if (hit) {
          if (lane == 0) orow[bk[warp][s_over].z + L - 1] = k0 + 31 - __clz(hit);
          break;
        }
      }
    }
    // pass 2: the first keys of each bucket, in key order, to base + rank; lanes
    // whose bucket is already placed (or not read) drop out before any ranking
    for (int k0 = 0; k0 < nc && remaining > 0; k0 += 32) {
      const int k = k0 + lane;
      const int s = k < nc ? (int)my[k] : 0;
      const int4 e = bk[warp][s];
      const bool need = k < nc && e.x > 0;
      const unsigned cand = __ballot_sync(0xffffffffu, need);
      if (!cand) continue;
      unsigned grp = 0;
      bool w = false;
      if (need) {
        grp = __match_any_sync(cand, s);
        const int rank = __popc(grp & lt);
        w = rank < e.x;
        if (w) orow[e.z + (e.y - e.x) + rank] = k;
      }
      const unsigned put = __ballot_sync(0xffffffffu, w);
      __syncwarp();  // every lane's read of bk (above) before the leaders update it
      if (need && (grp & lt) == 0) bk[warp][s].x = e.x - __popc(grp);
      remaining -= __popc(put);
      __syncwarp();
    }
    __syncwarp();
  }
}

template <int NW, int CPW>
cudaError_t launch_topl_nw(int H, int nq, int nk, int M, int L, int causal, const uint8_t* cq,
                           const uint8_t* ck, int32_t* out, size_t smem, int qpb, cudaStream_t s) {
  const int chunks = (nq + qpb - 1) / qpb;
  cudaError_t e = cudaFuncSetAttribute(topl_kernel<NW, CPW>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) {
    cudaGetLastError();  // do not leave the failure in the thread's error state
    return e;
  }
  topl_kernel<NW, CPW><<<(unsigned)((int64_t)H * chunks), kToplThreads, smem, s>>>(
      H, nq, nk, M, L, causal, qpb, cq, ck, out);
  return cudaGetLastError();
}

int code_fields(int E) { return E <= 16 ? 8 : 4; }

}  // namespace

size_t topl_smem_bytes(int nk, int M, int E) {
  const int cpw = code_fields(E);
  const int NW = (M + cpw - 1) / cpw;
  const int KW = NW == 3 ? 4 : NW;
  return (size_t)nk * KW * 4 + (size_t)kToplWarps * nk;
}

int topl_max_score() { return kMaxScore; }

// static shared memory of topl_kernel (per-lane bucket counts + bucket records):
// the dynamic part may use at most the 227 KB opt-in limit minus this
size_t topl_static_smem_bytes() {
  return sizeof(uint16_t) * kToplWarps * (kMaxScore + 1) * 32 + sizeof(int4) * kToplWarps * (kMaxScore + 1);
}

cudaError_t launch_topl(int H, int nq, int nk, int M, int E, int L, int causal,
                        const uint8_t* cq, const uint8_t* ck, int32_t* out, cudaStream_t s) {
  const size_t smem = topl_smem_bytes(nk, M, E);
  // queries per CTA: >= 8 waves of 2 CTAs per SM (small tail), each CTA
  // staging its head's keys once
  int qpb = 64;
  while (qpb < 1024 && (int64_t)H * ((nq + 2 * qpb - 1) / (2 * qpb)) >= 8 * 2 * 148) qpb *= 2;
  prof_begin("topl_select", s);
  const int cpw = code_fields(E);
  const int NW = (M + cpw - 1) / cpw;
  cudaError_t e;
#define TOPL_CASE(nw)                                                                       \
  case nw:                                                                                  \
    e = cpw == 8 ? launch_topl_nw<nw, 8>(H, nq, nk, M, L, causal, cq, ck, out, smem, qpb, s) \
                 : launch_topl_nw<nw, 4>(H, nq, nk, M, L, causal, cq, ck, out, smem, qpb, s); \
    break;
  switch (NW) {
    TOPL_CASE(1)
    TOPL_CASE(2)
    TOPL_CASE(3)
    TOPL_CASE(4)
    TOPL_CASE(5)
    TOPL_CASE(6)
    TOPL_CASE(7)
    default:
      e = launch_topl_nw<8, 4>(H, nq, nk, M, L, causal, cq, ck, out, smem, qpb, s);
      break;
  }
#undef TOPL_CASE
  prof_end(s);
  count_launch();
  return e;
}

}  // namespace spt
