// tc_ffn.cu -- bf16 path of the routed FFN on the 5th-generation tensor cores.
//
// One persistent, warp-specialised tcgen05 kernel template serves every GEMM
// on the hot path:
//   warp 0         TMA tile producer (weights / contiguous operands)
//                  gather4 loads (4 token rows x 128 B each) of a stage are spread
//                  over the lanes of all three warps (three SM sub-partitions);
//                  each producer warp arms the stage barrier for its own bytes.
//   warp 1         TMEM allocator (512 columns) + single-thread tcgen05.mma issuer
//   warps 2-9      epilogue: two warps per TMEM lane quarter (column halves),
//                  tcgen05.ld -> registers -> fused math -> global stores
// M tile = 128 bucket rows per accumulator (one TMEM lane per row), K stage = 64
// bf16 (one 128-byte swizzle row), N <= 256 per MMA, two TMEM accumulators so the
// epilogue of tile i overlaps the MMAs of tile i+1 (DW1 with m'*bw = 256 instead
// uses both accumulators for the gate and up halves of one tile, sharing the
// gathered X stage), 3-6 smem stages.
//
// Kinds (Alg. 4 of PAPER.md:564-579 as grouped GEMMs over the bucket layout):
//   ROUTER : logits = X W_R                    A = X tile,       B = w_r (K-major)
//   FWD1   : Z_b = X[bucket_b] W1_b^T          A = gather4(X),   B = w1 rows (K-major)
//            epilogue: Z stash, H~ = g * act(Z)     (Alg. 4 line 4, gate)
//   FWD2   : P_b = H~_b W2_b                   A = H~ rows,      B = w2 rows (MN-major)
//   DA     : dA_b = dY[bucket_b] W2_b^T        A = gather4(dY),  B = w2 rows (K-major)
//            epilogue: dgate = rowdot(dA, act(Z)), dZ = g dA act'(Z), dlogit
//   DAT    : dA_b^T = W2_b dY[bucket_b]^T      A = w2 rows,      B = gather4 / cp.async(dY)
//            (the default a7 for bw <= 128: N = 256 tokens instead of N = bw units;
//            epilogue_dat_rows transposes through smem and computes DA's epilogue)
//   DX     : dXp_b = dZ_b W1_b                 A = dZ rows,      B = w1 rows (MN-major)
//   DW1    : dW1_b = dZ_b^T X[bucket_b]        A = dZ (MN-major), B = gather4(X) along K
//   DW2    : dW2_b = H~_b^T dY[bucket_b]       A = H~ (MN-major), B = gather4(dY) along K
//   DWR    : dW_R = dLogits^T X  (split-K)     A = dense dlogits hi|lo (MN-major), B = X (MN-major)
// Padded bucket rows: tile t128 of the schedule covers rows [t128*128, +128);
// rows past a block's n_b are zero in every stash written here, which makes
// the K tails of the weight-gradient GEMMs exact.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "act.cuh"
#include "tc_common.cuh"
#include "tmap.h"

namespace spt {

using namespace tc;

enum Kind : int { K_ROUTER = 0, K_FWD1, K_FWD2, K_DA, K_DX, K_DW1, K_DW2, K_DWR, K_DAT, K_DXR };

struct TcArgs {
  CUtensorMap ta;  // A operand
  CUtensorMap tb;  // B operand
  CUtensorMap tc;  // FWD2/DX: partials [rows, d] bf16, box 64 cols x 32 rows (TMA store)
  // fp32 path on the bf16 tensor cores (Geom::split, reading c13'): every fp32
  // operand is carried as two bf16 tensors, x = hi + lo + O(2^-17 |x|), and each
  // GEMM runs its K loop three times -- hi*hi, hi*lo, lo*hi -- into the same
  // fp32 TMEM accumulator (the dropped lo*lo term is <= 2^-18 of each product).
  CUtensorMap ta2;  // lo half of the A operand (geometry of ta)
  CUtensorMap tb2;  // lo half of the B operand (geometry of tb)
  CUtensorMap tw2;  // fused FWD1 -> FWD2 kernel: W2 (the second GEMM's MN-major B), box 64 x 64
  RouteView r;
  int64_t T;
  int G, d, D, bw, mp, act, gate, gpad;
  int NT;          // N tiles of 256 (FWD2/DX/DW*/DWR)
  int MH;          // 128-row M halves per tile (DW*: ceil(M/128) <= 2), else 1
  int n_split;     // DWR split-K factor
  int ksplit;      // DWR tokens per split (multiple of 64)
  int acc_mode;    // DW*: accumulate into output
  int BN;          // MMA N
  void* out;       // kind-specific primary output
  void* out2;      // secondary output (FWD1: h; DA: dz)
  const void* aux; // DA: z stash
  const void* aux2;  // gathering kinds: the tensor whose rows are gathered (x or dy)
  float* rows_f;   // DA: dgate rows
  float* rows_g;   // DA: dlogit rows
  void* dlg;       // DA: dense dlogits [2][T][gpad] bf16
  const int32_t* tile_list;     // FWD1/DA: (mt << 8 | b) in m-tile-major order
  const int32_t* unit_offsets;  // FWD2/DX: weight-resident unit prefix per block
  int n_stg;                    // FWD2/DX: 4 KB staging buffers per epilogue warp (1-3)
  int unit_mt;                  // FWD2/DX: m-tiles per weight-resident unit
  int prefetch;                 // gathering kinds: L2 prefetch of gathered rows (SPT_FFN_PREFETCH)
  unsigned long long* trace;    // SPT_FFN_TRACE: per-CTA role cycle counters (diagnostics)
  // wide blocks (m' bw > 256, the paper's G = 4 / 8 blocks): FWD1 / DA tile
  // the block's units (bn_u per tile, nu tiles), DW1 / DW2 tile the features
  // (256 per tile, nu tiles), FWD2 / DX stream K instead of keeping the
  // weight slab resident (kstream).  nu = 1, kstream = 0 otherwise.
  int bn_u;                     // FWD1 / DA: units per tile (= bw when nu == 1)
  int nu;                       // FWD1 / DA: unit tiles; DW1 / DW2: feature tiles
  int kstream;                  // FWD2 / DX: K-streaming tiles (K > 256)
  float* dgp;                   // DA, nu > 1: per-unit-tile dgate partials [rows_cap][nu]
  int split;                    // 1: fp32 path, three K passes (see ta2 / tb2 above)
  const void* aux2_lo;          // split: lo half of the gathered rows (aux2)
  const void* aux_lo;           // split, DA: lo half of the Z stash (aux)
  void* out_lo;                 // split, FWD1: lo half of the Z stash (out)
  void* out2_lo;                // split: FWD1 lo half of H~ (out2); DA lo half of dZ (out2)
  int ablate;                   // SPT_FFN_ABLATE (timing experiments only; results wrong):
                                //  1 = skip gathered-row copies, 2 = skip FWD1 epilogue stores,
                                //  3 = no operand loads at all, 4 = 3 + no epilogue work,
                                //  5 = 4 + no proxy fence before the MMAs, 6 = 5 + no full waits
  // DW1 / DW2 side work: the a8 grad-input combine (combine.cu's sum, same order)
  // rides on the dW kernels' epilogue warps, which wait ~130 K-stages per tile.
  // Tokens are claimed one per warp from *cb_ctr; cb_drain: after its tiles the
  // whole CTA finishes the remaining tokens (the last host kernel).  cb_ctr == 0: off.
  const __nv_bfloat16* cb_part;  // dX partial rows [rows_cap, d]
  const float* cb_dlogit;        // dlogit per padded bucket row
  const __nv_bfloat16* cb_wr;    // w_r [G, d] (nullptr: no router term, GATE_NONE)
  __nv_bfloat16* cb_out;         // dx [T, d]
  int* cb_ctr;
  int cb_k;                      // top-k (<= 32: one lane per pair)
  int cb_drain;
  int dat_fused;                 // DAT: dgate / dZ / dlogit epilogue in-kernel (no da_post pass)
  int dw_ng;                     // DW*: N tiles per raster group (SPT_FFN_DW_NG; NT = block-major)
  int pair_rows;                 // tc_pair_gather_kernel: rows per CTA stage by TMA gather4 (rest cp.async)
  int mma_batch;                 // tc_pair_gather_kernel: K stages per MMA-issuer wait round (1 or 2)
  int g1_rows;                   // tc_gemm_kernel FWD1 / DA / DAT: rows of a 256-row stage by TMA gather4 (32..256)
  int pair_cpw;                  // tc_pair_gather_kernel: cp.async warps (4: 8 epilogue warps; 8: 4 epilogue warps)
};

// One warp computes 512 columns (two 256-column chunks, 16 bytes per lane each) of
// dx[t] = sum_{j asc} dXp[prow(t,j)] + sum_{j asc} dlogit_j w_r[b_j], in the order and
// rounding of combine_kernel<bf16, true> (combine.cu, reading c12: the partial rows
// added one after another in ascending j, then the router term's fmas in ascending j),
// so the two give bit-identical dx.  Loads go out eight rows x two chunks at a time.
__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ void add_row8(float (&acc)[8], const uint4& q) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    acc[2 * i] += bf16lo(w[i]);
    acc[2 * i + 1] += bf16hi(w[i]);
  }
}
__device__ __forceinline__ void fma_row8(float (&acc)[8], float s, const uint4& q) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    acc[2 * i] = fmaf(s, bf16lo(w[i]), acc[2 * i]);
    acc[2 * i + 1] = fmaf(s, bf16hi(w[i]), acc[2 * i + 1]);
  }
}
constexpr int kSideCols8 = 32;  // 16-byte vectors of one side-combine unit (256 columns)
// A warp claims whole tokens (one atomic per token) and works through the token's
// 256-column units one at a time, so an epilogue warp can stop between two units
// for its tile and resume the token afterwards (the claim lives in SideState).
struct SideState {
  int t;       // claimed token, -1: none
  int c;       // next unit of it
  int row;     // lane j < k: padded bucket row of pair j (< 2^31: ABI check)
  int blk;     // lane j < k: block of pair j
  float dl;    // lane j < k: dlogit of pair j
};
// Rows missing from a round of 16 load as zeros: acc is never -0 (it starts at +0 and
// x + (-x) rounds to +0), so adding +0 -- or fma(dl, +0, acc) -- leaves it unchanged.
__device__ __forceinline__ void side_combine_unit(const TcArgs& a, const SideState& st, int lane) {
  const int k = a.cb_k;
  const int d8 = a.d / 8;  // 16-byte vectors per row
  const int c0 = st.c * kSideCols8 + lane;
  if (c0 >= d8) return;
  const uint4* part = reinterpret_cast<const uint4*>(a.cb_part) + c0;
  const uint4 zero = make_uint4(0u, 0u, 0u, 0u);
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
#pragma unroll 1
  for (int j = 0; j < k; j += 16) {  // sixteen rows in flight
    uint4 p[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int rw = __shfl_sync(0xffffffffu, st.row, (j + u) & 31);
      p[u] = j + u < k ? __ldg(part + (int64_t)rw * d8) : zero;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) add_row8(acc, p[u]);
  }
  if (a.cb_wr) {
    const uint4* wr = reinterpret_cast<const uint4*>(a.cb_wr) + c0;
#pragma unroll 1
    for (int j = 0; j < k; j += 16) {
      uint4 w[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int bj = __shfl_sync(0xffffffffu, st.blk, (j + u) & 31);
        w[u] = j + u < k ? __ldg(wr + (int64_t)bj * d8) : zero;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) fma_row8(acc, __shfl_sync(0xffffffffu, st.dl, (j + u) & 31), w[u]);
    }
  }
  reinterpret_cast<uint4*>(a.cb_out)[(int64_t)st.t * d8 + c0] =
      make_uint4(pack_bf16(acc[0], acc[1]), pack_bf16(acc[2], acc[3]), pack_bf16(acc[4], acc[5]),
                 pack_bf16(acc[6], acc[7]));
}
// Work through units (claiming tokens as needed) until every token is claimed and
// the warp's own token is finished (returns true), or -- polling `poll` between
// units -- until the barrier phase completes (returns false, the claim kept).
// only_own: finish the claimed token, claim nothing new.
__device__ __forceinline__ bool side_combine_run(const TcArgs& a, int lane, SideState& st,
                                                 uint64_t* poll, uint32_t parity, bool only_own = false) {
  const int npass = (a.d / 8 + kSideCols8 - 1) / kSideCols8;
  for (;;) {
    if (st.t < 0) {
      if (only_own) return true;
      int t = 0;
      if (lane == 0) t = atomicAdd(a.cb_ctr, 1);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= a.T) return true;  // every token claimed
      st.t = t;
      st.c = 0;
      const int k = a.cb_k;
      if (lane < k) {
        st.blk = a.r.topk_idx[(int64_t)t * k + lane];
        st.row = a.r.tile_offsets[st.blk] * 128 +
                 (a.r.pair_slot[(int64_t)t * k + lane] - a.r.block_offsets[st.blk]);
        st.dl = a.cb_wr ? a.cb_dlogit[st.row] : 0.f;
      } else {
        st.blk = st.row = 0;
        st.dl = 0.f;
      }
    }
    if (poll && mbar_test(poll, parity)) return false;
    side_combine_unit(a, st, lane);
    if (++st.c == npass) st.t = -1;
  }
}

// 16 warps.  warp 0: TMA tile producer; warp 1: TMEM alloc + MMA issuer;
// warps 4-11: epilogue (two warps per TMEM lane quarter).  Row gathers use both
// copy engines (measured on B200, tools/gather_bench.cu: TMA gather4 from 3
// warps ~16-20 B/clk/SM, cp.async from 8 warps ~22-24 B/clk/SM; independent):
//  FWD1 / DA (rows of A gathered): rows [0,128) of a 256-row stage by TMA
//    tile::gather4 from warps 0, 2, 3 (each arms the stage barrier for its own
//    bytes), rows [128,256) by cp.async from warps 12-15.
//  DW1 / DW2 (rows of B gathered along K): cp.async from warps 2, 3, 12-15.
constexpr int kThreads = 512;
constexpr int kEpiWarps = 8;                  // warps 4..11
constexpr int kTmaGatherWarps = 3;            // FWD1 / DA: warps 0, 2, 3
constexpr int kG1TmaRows = 64;                // 1-CTA gathered kinds: default TMA rows of a 256-row stage (a.g1_rows)
constexpr int kCpThreadsA = 128;              // FWD1 / DA: cp.async warps 12..15
// DW*: cp.async warps 2, 3, 8..15 (10 warps).  The dW tiles run ~130 K stages per
// epilogue, so warps 8..11 gather instead of waiting as epilogue warps: the B rows
// (32 KB gathered per 512-1024 MMA clocks) are what bounds dW2 / dW1
constexpr int kGatherWarpsB = 10;
constexpr int kCpThreadsB = kGatherWarpsB * 32;
constexpr int kEpiWarpsDW = 4;                // DW*: epilogue warps 4..7 (one per TMEM lane quarter)
constexpr int kABytes = 16384;                // 128 rows x 64 bf16

// kinds whose 256 gathered token rows per stage come from the pair-tile list:
// FWD1 / DA gather them as the A (M) operand, DAT as the B (N) operand
__host__ __device__ constexpr bool kind_gather_a(int k) { return k == K_FWD1 || k == K_DA || k == K_DAT; }
__host__ __device__ constexpr bool kind_rows_on_b(int k) { return k == K_DAT; }
__host__ __device__ constexpr bool kind_gather_b(int k) { return k == K_DW1 || k == K_DW2; }
__host__ __device__ constexpr bool kind_a_mn(int k) { return k == K_DW1 || k == K_DW2 || k == K_DWR; }
__host__ __device__ constexpr bool kind_b_mn(int k) {
  return !(k == K_ROUTER || k == K_FWD1 || k == K_DA || k == K_DAT);
}
// FWD2 / DX keep one (block, 256-column) weight slab resident in smem and
// stream up to unit_mtiles() A tiles of that block through it
__host__ __device__ constexpr bool kind_bres(int k) { return k == K_FWD2 || k == K_DX; }
// K rows per smem stage (64 for every kind).  32-row stages for the dW kinds
// (twice the ring depth for their latency-bound gathers) are supported and
// parity-clean but measured slower on B200 (dW1 1.83 vs 1.45 ms, dW2 1.71 vs
// 1.05 ms): the per-stage protocol (193 arrivals, commit, wake) doubles.
__host__ __device__ constexpr int kind_bk(int) { return 64; }
__host__ __device__ constexpr int b_bytes(int kind, int BN, int kstream = 0) {
  return kind_bres(kind) && !kstream ? 0 : (kind_b_mn(kind) ? 512 * kind_bk(kind) : BN * 128);
}

__device__ __forceinline__ int find_block(const int32_t* tile_offsets, int G, int t128) {
  int lo = 0, hi = G - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tile_offsets[mid] <= t128) lo = mid; else hi = mid - 1;
  }
  return lo;
}

struct TileInfo {
  int b, nt;
  int n_valid;      // valid rows of the M tile (bucket-row kinds) / bucket size n_b (DW*)
  int64_t prow0;    // first padded bucket row of the M tile (bucket-row kinds)
  int64_t pos0;     // bucket position of row 0 (bucket-row kinds) / of block start (DW*)
  int nkb;          // K stages (split: 3 passes of kb1 stages)
  int kb1;          // K stages of one pass
  int64_t kbase;    // DW*: first padded row of the block; DWR: first token of the split
  int rows_pad;     // bucket-row kinds: padded rows of the block from prow0 on (write limit)
  int ut;           // FWD1 / DA: unit tile; DW1 / DW2: feature tile (wide blocks)
};

// split K loop: stage kb of pass p = kb / kb1 reads stage kk = kb % kb1 of
// (A, B) = (hi, hi) for p = 0, (hi, lo) for p = 1, (lo, hi) for p = 2
__device__ __forceinline__ int kpass(const TileInfo& ti, int kb, int& kk) {
  const int p = kb >= ti.kb1 ? (kb >= 2 * ti.kb1 ? 2 : 1) : 0;
  kk = kb - p * ti.kb1;
  return p;
}

// TMEM columns: accumulator buffer `acc`, M half `h` (each half holds BN <= 256
// columns at a stride of 128 or 256); two buffers alternate between tiles when
// they fit in the 512 allocated columns, else one buffer.
__host__ __device__ __forceinline__ int tm_half_stride(int BN) { return BN > 128 ? 256 : 128; }
__host__ __device__ __forceinline__ int tm_nacc(int BN, int MH) {
  return 2 * MH * tm_half_stride(BN) <= 512 ? 2 : 1;
}
__host__ __device__ __forceinline__ uint32_t tm_col(int BN, int MH, int acc, int h) {
  return (uint32_t)((acc * MH + h) * tm_half_stride(BN));
}

template <int KIND>
__device__ __forceinline__ int num_tiles(const TcArgs& a) {
  if (KIND == K_ROUTER) return (int)ceil_div(a.T, 128);
  if (kind_gather_a(KIND)) return a.unit_offsets[a.G + 1] * a.nu;  // 256-row pair tiles x unit tiles
  if (KIND == K_FWD2 || KIND == K_DX)  // weight-resident units, or (m-tile, N tile) when streaming K
    return a.kstream ? a.r.tile_offsets[a.G] * a.NT : a.unit_offsets[a.G];
  if (KIND == K_DW1 || KIND == K_DW2) return a.G * a.nu * a.NT;
  if (KIND == K_DXR) return (int)ceil_div(a.T, 128) * a.NT;
  return a.NT * a.n_split;  // DWR (G <= 128 rows: one M tile)
}

template <int KIND>
__device__ __forceinline__ TileInfo decode(const TcArgs& a, int tile) {
  TileInfo ti{};
  if (KIND == K_ROUTER) {
    ti.prow0 = (int64_t)tile * 128;
    ti.n_valid = (int)(a.T - ti.prow0 < 128 ? a.T - ti.prow0 : 128);
    ti.nkb = a.d / 64;
  } else if (kind_gather_a(KIND)) {
    // pair tiles (two 128-row m-tiles sharing each B stage) in the raster order
    // of tile_sched_kernel; unit tiles fastest (their A rows are shared in L2)
    ti.ut = tile % a.nu;
    const int e = a.tile_list[tile / a.nu];
    ti.b = e & 255;
    const int mt = 2 * (e >> 8);
    const int nb = a.r.block_offsets[ti.b + 1] - a.r.block_offsets[ti.b];
    ti.n_valid = nb - mt * 128;
    ti.prow0 = (int64_t)(a.r.tile_offsets[ti.b] + mt) * 128;
    ti.pos0 = a.r.block_offsets[ti.b] + mt * 128;
    ti.rows_pad = (a.r.tile_offsets[ti.b + 1] - a.r.tile_offsets[ti.b] - mt) * 128;
    ti.nkb = a.d / 64;
  } else if (KIND == K_FWD2 || KIND == K_DX) {  // K-streaming: (global m-tile, N tile)
    ti.nt = tile % a.NT;
    const int mg = tile / a.NT;
    ti.b = find_block(a.r.tile_offsets, a.G, mg);
    const int mt = mg - a.r.tile_offsets[ti.b];
    const int nb = a.r.block_offsets[ti.b + 1] - a.r.block_offsets[ti.b];
    ti.n_valid = nb - mt * 128;
    ti.prow0 = (int64_t)mg * 128;
    ti.pos0 = a.r.block_offsets[ti.b] + mt * 128;
    ti.nkb = KIND == K_FWD2 ? (a.bw + 63) / 64 : (a.mp * a.bw + 63) / 64;
  } else if (KIND == K_DXR) {  // (token tile, N tile); K = hi then lo dlogits
    ti.nt = tile % a.NT;
    ti.prow0 = (int64_t)(tile / a.NT) * 128;
    ti.n_valid = (int)(a.T - ti.prow0 < 128 ? a.T - ti.prow0 : 128);
    ti.nkb = 2 * (a.gpad / 64 + (a.gpad % 64 ? 1 : 0));
  } else if (KIND == K_DW1 || KIND == K_DW2) {
    // raster: groups of dw_ng N tiles; inside a group (block, unit tile, N tile)
    // order, so one wave of CTAs covers ~SMs / dw_ng blocks x dw_ng N tiles
    const int per = a.dw_ng * a.G * a.nu;
    const int grp = tile / per;
    const int r = tile - grp * per;
    const int sz = min(a.dw_ng, a.NT - grp * a.dw_ng);
    ti.nt = grp * a.dw_ng + r % sz;
    ti.ut = (r / sz) % a.nu;
    ti.b = r / sz / a.nu;
    ti.pos0 = a.r.block_offsets[ti.b];
    ti.n_valid = a.r.block_offsets[ti.b + 1] - a.r.block_offsets[ti.b];  // bucket size n_b
    ti.kbase = (int64_t)a.r.tile_offsets[ti.b] * 128;
    // rows past n_b up to the stage boundary are the block's zero padding
    ti.nkb = (ti.n_valid + kind_bk(KIND) - 1) / kind_bk(KIND);
  } else {  // DWR: tile = (split, nt)
    ti.nt = tile % a.NT;
    const int s = tile / a.NT;
    ti.b = s;
    ti.kbase = (int64_t)s * a.ksplit;
    const int64_t t1 = a.T < ti.kbase + a.ksplit ? a.T : ti.kbase + a.ksplit;
    const int nk = t1 > ti.kbase ? (int)ceil_div(t1 - ti.kbase, 64) : 0;
    ti.nkb = 2 * nk;  // hi part then lo part
  }
  ti.kb1 = ti.nkb;
  if (a.split) {
    if (KIND == K_DWR) {  // parts: dlogit hi x X hi, dlogit lo x X hi, dlogit hi x X lo
      ti.kb1 = ti.nkb / 2;
      ti.nkb = 3 * ti.kb1;
    } else {
      ti.nkb *= 3;
    }
  }
  return ti;
}

// FWD2 / DX work unit u -> (block b, m-tiles [mt0, mt1), N tile nt)
struct UnitInfo {
  int b, nt, mt0, mt1;
};
__device__ __forceinline__ UnitInfo decode_unit(const TcArgs& a, int u) {
  UnitInfo ui;
  ui.b = find_block(a.unit_offsets, a.G, u);
  const int r = u - a.unit_offsets[ui.b];
  ui.nt = r % a.NT;
  const int mc = r / a.NT;
  const int ntb = a.r.tile_offsets[ui.b + 1] - a.r.tile_offsets[ui.b];
  ui.mt0 = mc * a.unit_mt;
  ui.mt1 = min(ntb, ui.mt0 + a.unit_mt);
  return ui;
}
template <int KIND>
__device__ __forceinline__ TileInfo decode_mtile(const TcArgs& a, const UnitInfo& u, int mt) {
  TileInfo ti{};
  ti.b = u.b;
  ti.nt = u.nt;
  const int nb = a.r.block_offsets[u.b + 1] - a.r.block_offsets[u.b];
  ti.n_valid = nb - mt * 128;
  ti.prow0 = (int64_t)(a.r.tile_offsets[u.b] + mt) * 128;
  ti.pos0 = a.r.block_offsets[u.b] + mt * 128;
  ti.nkb = KIND == K_FWD2 ? (a.bw + 63) / 64 : (a.mp * a.bw + 63) / 64;
  return ti;
}

// bytes of the tile (non-gather) loads of one stage, issued by warp 0 lane 0
template <int KIND>
__device__ __forceinline__ uint32_t tile_tx_bytes(const TcArgs& a) {
  if (KIND == K_FWD1) return a.mp * a.bn_u * 128;
  if (KIND == K_DA) return a.bn_u * 128;
  if (KIND == K_DAT) return 128 * 128;  // the W2 box is always 128 unit rows (rows >= bw unused)
  if (KIND == K_ROUTER) return kABytes + a.gpad * 128;
  if (KIND == K_DW1 || KIND == K_DW2) return 128 * kind_bk(KIND) * 2 * a.MH;
  if (KIND == K_DWR) return kABytes * a.MH + 32768;
  return kABytes + 32768;  // FWD2, DX
}

// ---------------------------------------------------------------- producer
// Tile (non-gathered) loads of one stage.  Called by warp 0 lane 0 only.
template <int KIND>
__device__ __forceinline__ void produce_tiles(const TcArgs& a, const TileInfo& ti, int kb,
                                              uint8_t* sA, uint8_t* sB, uint64_t* bar) {
  int kk = kb;
  const int p = kpass(ti, kb, kk);
  const CUtensorMap* ma = p == 2 ? &a.ta2 : &a.ta;  // split passes (p = 0 without split)
  const CUtensorMap* mb = p == 1 ? &a.tb2 : &a.tb;
  if (KIND == K_ROUTER) {
    tma_load_2d(sA, ma, bar, kk * 64, (int)ti.prow0);
    tma_load_2d(sB, mb, bar, kk * 64, 0);
  } else if (KIND == K_DAT) {  // A = the block's W2 rows (units) x 64 columns
    tma_load_2d(sA, &a.tb, bar, kb * 64, ti.b * a.bw);
  } else if (KIND == K_FWD1 || KIND == K_DA) {  // B: the tile's bn_u units (+ up rows)
    const int u0 = ti.b * a.bw + ti.ut * a.bn_u;
    tma_load_2d(sB, mb, bar, kk * 64, u0);
    if (KIND == K_FWD1 && a.mp == 2) tma_load_2d(sB + a.bn_u * 128, mb, bar, kk * 64, a.D + u0);
  } else if (KIND == K_FWD2 || KIND == K_DX) {
    tma_load_2d(sA, ma, bar, kk * 64, (int)ti.prow0);
    int krow;
    if (KIND == K_FWD2) krow = ti.b * a.bw + kk * 64;
    else krow = kk * 64 < a.bw ? ti.b * a.bw + kk * 64 : a.D + ti.b * a.bw + (kk * 64 - a.bw);
#pragma unroll
    for (int j = 0; j < 4; ++j) tma_load_2d(sB + j * 8192, mb, bar, ti.nt * 256 + j * 64, krow);
  } else if (KIND == K_DXR) {  // A = dense dlogits (hi rows, then lo rows), B = w_r (MN-major)
    const int nkh = ti.nkb / 2, kh = kb % nkh;
    tma_load_2d(sA, &a.ta, bar, kh * 64, (int)((kb < nkh ? 0 : a.T) + ti.prow0));
#pragma unroll
    for (int j = 0; j < 4; ++j) tma_load_2d(sB + j * 8192, &a.tb, bar, ti.nt * 256 + j * 64, kh * 64);
  } else if (KIND == K_DW1 || KIND == K_DW2) {
    constexpr int BK = kind_bk(KIND);  // MN-major A: 64-feature chunks x BK bucket rows
    for (int j = 0; j < 2 * a.MH; ++j)  // features [256 ut + 64 j, +64)
      tma_load_2d(sA + j * (BK * 128), ma, bar, ti.ut * 256 + j * 64, (int)(ti.kbase + kk * BK));
  } else {  // DWR: part 0 = (dlogit hi, X), 1 = (dlogit lo, X), split: 2 = (dlogit hi, X lo)
    const int nk = a.split ? ti.kb1 : ti.nkb / 2;
    const int part = kb / nk;
    const int kd = kb - part * nk;
    const int trow = (int)(ti.kbase + kd * 64);
    const CUtensorMap* mx = part == 2 ? &a.tb2 : &a.tb;
    for (int j = 0; j < 2 * a.MH; ++j)  // blocks [64 j, 64 j + 64); MH = 2 when G > 128
      tma_load_2d(sA + j * 8192, &a.ta, bar, j * 64, (int)((part & 1) * a.T) + trow);
#pragma unroll
    for (int j = 0; j < 4; ++j) tma_load_2d(sB + j * 8192, mx, bar, ti.nt * 256 + j * 64, trow);
  }
}

// ---------------------------------------------------------------- epilogues
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&v)[64], bool two) {
  uint32_t (&lo)[32] = *reinterpret_cast<uint32_t(*)[32]>(&v[0]);
  uint32_t (&hi)[32] = *reinterpret_cast<uint32_t(*)[32]>(&v[32]);
  tmem_ld32(taddr, lo);
  if (two) tmem_ld32(taddr + 32, hi);
  tmem_ld_wait();
}

__device__ __forceinline__ void store_bf16_row(__nv_bfloat16* dst, const uint32_t* v, int n) {
  // n in {32, 64}: pack fp32 pairs to bf16, 16-byte stores (a full line per 64 columns)
  uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (q * 8 >= n) break;
    d4[q] = make_uint4(pack_bf16(__uint_as_float(v[8 * q + 0]), __uint_as_float(v[8 * q + 1])),
                       pack_bf16(__uint_as_float(v[8 * q + 2]), __uint_as_float(v[8 * q + 3])),
                       pack_bf16(__uint_as_float(v[8 * q + 4]), __uint_as_float(v[8 * q + 5])),
                       pack_bf16(__uint_as_float(v[8 * q + 6]), __uint_as_float(v[8 * q + 7])));
  }
}

// split: the lo halves of a packed bf16 pair, x - bf16(x) (exact in fp32), rounded to bf16
__device__ __forceinline__ uint32_t pack_bf16_lo(float x0, float x1, uint32_t hi) {
  return pack_bf16(x0 - __uint_as_float(hi << 16), x1 - __uint_as_float(hi & 0xffff0000u));
}
// value of the bf16 at half (i & 1) of word w, plus (split) its lo half from word wl
__device__ __forceinline__ float bf16_at(uint32_t w, int i) {
  return __uint_as_float((i & 1) ? (w & 0xffff0000u) : (w << 16));
}

// Row `row` of the tile is TMEM lane `row`; columns [c_lo, c_hi) of it belong
// to this thread (the other warp of the same lane quarter owns the rest).
// tacc: TMEM address of (this warp's lane quarter, column 0) of the accumulator.
// sh (FWD1 of the fused FWD1 -> FWD2 kernel): also write this row's H~ units
// into the K-major, 128-byte-swizzled smem A tile of the second GEMM
// (k-block u / 64 at +16 KB, row at +128 B, 16-byte chunk ((u % 64) / 8) ^ (row & 7)).
// ACT >= 0 (FWD1 / DA): the activation fixed at compile time (no per-element
// dispatch; m' = 2 exactly for SwiGLU); -1: a.act / a.mp at run time
template <int KIND, bool kSplit = false, int ACT = -1>
__device__ __forceinline__ void epilogue(const TcArgs& a, const TileInfo& ti, uint32_t tacc,
                                         int row, int half, float* dg_xchg, uint8_t* sh = nullptr) {
  const bool valid = row < ti.n_valid;
  const int act = ACT >= 0 ? ACT : a.act;
  const int mp = ACT >= 0 ? (ACT == SPT_ACT_SWIGLU ? 2 : 1) : a.mp;
  if (KIND == K_ROUTER) {
    const int64_t t = ti.prow0 + row;
    for (int c0 = half * 16; c0 < a.gpad; c0 += 32) {
      uint32_t v[16];
      tmem_ld16(tacc + c0, v);
      tmem_ld_wait();
      if (valid) {
        float* dst = (float*)a.out + t * a.G;
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (c0 + i < a.G) dst[c0 + i] = __uint_as_float(v[i]);
      }
    }
  } else if (KIND == K_FWD1) {
    // 16 units per step (register budget: the kernel runs 512 threads)
    const float g = valid ? a.r.bucket_gate[ti.pos0 + row] : 0.f;
    const int64_t prow = ti.prow0 + row;
    // this tile's units [ub, ub + nut) of the block: TMEM columns u (gate) and
    // bn_u + u (up); Z stash row = [gate bw | up bw], H row = [bw]
    const int ub = ti.ut * a.bn_u, nut = min(a.bn_u, a.bw - ub);
    __nv_bfloat16* zr = (__nv_bfloat16*)a.out + prow * (int64_t)(mp * a.bw) + ub;
    __nv_bfloat16* hr = (__nv_bfloat16*)a.out2 + prow * (int64_t)a.bw + ub;
    const int hw = ((a.bn_u / 2) + 15) & ~15;
    const int u_lo = half < 0 ? 0 : half * hw, u_hi = half < 0 ? nut : min(nut, u_lo + hw);
    for (int u0 = u_lo; u0 < u_hi; u0 += 16) {
      uint32_t vg[16], vu[16];
      tmem_ld16(tacc + u0, vg);
      if (mp == 2) tmem_ld16(tacc + a.bn_u + u0, vu);
      tmem_ld_wait();
      uint32_t pz[8], pu[8], ph[8];
      uint32_t lz[8], lu[8], lh[8];  // split: lo halves
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const float z0 = valid ? __uint_as_float(vg[i]) : 0.f;
        const float z1 = valid ? __uint_as_float(vg[i + 1]) : 0.f;
        float u0f = 0.f, u1f = 0.f;
        if (mp == 2) {
          u0f = valid ? __uint_as_float(vu[i]) : 0.f;
          u1f = valid ? __uint_as_float(vu[i + 1]) : 0.f;
          pu[i / 2] = pack_bf16(u0f, u1f);
          if (kSplit) lu[i / 2] = pack_bf16_lo(u0f, u1f, pu[i / 2]);
        }
        pz[i / 2] = pack_bf16(z0, z1);
        const float h0 = g * act_fwd<true>(act, z0, u0f), h1 = g * act_fwd<true>(act, z1, u1f);
        ph[i / 2] = pack_bf16(h0, h1);
        if (kSplit) {
          lz[i / 2] = pack_bf16_lo(z0, z1, pz[i / 2]);
          lh[i / 2] = pack_bf16_lo(h0, h1, ph[i / 2]);
        }
      }
      if (a.ablate == 2) continue;
      if (sh) {  // fused FWD2's A operand (this CTA's 128 rows x bw units)
        const int u = ub + u0;
        uint8_t* rowp = sh + (u >> 6) * 16384 + row * 128;
        const int c0 = (u & 63) >> 3;
#pragma unroll
        for (int q = 0; q < 2; ++q)
          *reinterpret_cast<uint4*>(rowp + (((c0 + q) ^ (row & 7)) << 4)) =
              make_uint4(ph[4 * q], ph[4 * q + 1], ph[4 * q + 2], ph[4 * q + 3]);
      }
      if (kSplit) {  // lo halves: same row layout, separate tensors
        uint4* zd = reinterpret_cast<uint4*>((__nv_bfloat16*)a.out_lo + prow * (int64_t)(mp * a.bw) + ub + u0);
        uint4* hd = reinterpret_cast<uint4*>((__nv_bfloat16*)a.out2_lo + prow * (int64_t)a.bw + ub + u0);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          zd[q] = make_uint4(lz[4 * q], lz[4 * q + 1], lz[4 * q + 2], lz[4 * q + 3]);
          hd[q] = make_uint4(lh[4 * q], lh[4 * q + 1], lh[4 * q + 2], lh[4 * q + 3]);
        }
        if (mp == 2) {
          uint4* ud = reinterpret_cast<uint4*>((__nv_bfloat16*)a.out_lo + prow * (int64_t)(mp * a.bw) + ub + a.bw + u0);
#pragma unroll
          for (int q = 0; q < 2; ++q) ud[q] = make_uint4(lu[4 * q], lu[4 * q + 1], lu[4 * q + 2], lu[4 * q + 3]);
        }
      }
      uint4* zd = reinterpret_cast<uint4*>(zr + u0);
      uint4* hd = reinterpret_cast<uint4*>(hr + u0);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        zd[q] = make_uint4(pz[4 * q], pz[4 * q + 1], pz[4 * q + 2], pz[4 * q + 3]);
        hd[q] = make_uint4(ph[4 * q], ph[4 * q + 1], ph[4 * q + 2], ph[4 * q + 3]);
      }
      if (mp == 2) {
        uint4* ud = reinterpret_cast<uint4*>(zr + a.bw + u0);
#pragma unroll
        for (int q = 0; q < 2; ++q) ud[q] = make_uint4(pu[4 * q], pu[4 * q + 1], pu[4 * q + 2], pu[4 * q + 3]);
      }
    }
  } else if (KIND == K_FWD2 || KIND == K_DX || KIND == K_DXR) {
    const int64_t prow = ti.prow0 + row;
    __nv_bfloat16* dst = (__nv_bfloat16*)a.out + prow * (int64_t)a.d + ti.nt * 256;
    float* dstf = (float*)a.out + prow * (int64_t)a.d + ti.nt * 256;  // split: fp32 rows
    const int ncols = min(256, a.d - ti.nt * 256);
    const int c_lo = half * 128, c_hi = min(ncols, c_lo + 128);
    for (int c0 = c_lo; c0 < c_hi; c0 += 64) {
      uint32_t v[64];
      const bool two = c0 + 32 < c_hi;
      tmem_ld64(tacc + c0, v, two);
      if (!valid) continue;
      if (kSplit) {
        uint4* d4 = reinterpret_cast<uint4*>(dstf + c0);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          if (q >= (two ? 16 : 8)) break;
          d4[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
      } else {
        store_bf16_row(dst + c0, v, two ? 64 : 32);
      }
    }
  } else if (KIND == K_DA) {
    const int64_t prow = ti.prow0 + row;
    const float g = valid ? a.r.bucket_gate[ti.pos0 + row] : 0.f;
    const int ub = ti.ut * a.bn_u, nut = min(a.bn_u, a.bw - ub);  // this tile's units
    const __nv_bfloat16* zr = (const __nv_bfloat16*)a.aux + prow * (int64_t)(mp * a.bw) + ub;
    __nv_bfloat16* dzr = (__nv_bfloat16*)a.out2 + prow * (int64_t)(mp * a.bw) + ub;
    // split: lo halves of the Z stash / dZ rows (same layout)
    const __nv_bfloat16* zrl = (const __nv_bfloat16*)a.aux_lo + prow * (int64_t)(mp * a.bw) + ub;
    __nv_bfloat16* dzrl = (__nv_bfloat16*)a.out2_lo + prow * (int64_t)(mp * a.bw) + ub;
    const int hw = ((a.bn_u / 2) + 15) & ~15;
    const int u_lo = half < 0 ? 0 : half * hw, u_hi = half < 0 ? nut : min(nut, u_lo + hw);
    float dgate = 0.f;
    for (int u0 = u_lo; u0 < u_hi; u0 += 16) {  // 16 units per step (register budget)
      // the Z stash loads are issued before the TMEM load so the two latencies overlap
      uint32_t zg4[8], zu4[8], zgl[8], zul[8];
      if (valid) {
        auto ld8 = [](const __nv_bfloat16* src, uint32_t (&w8)[8]) {
          const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const uint4 w = s4[q];
            w8[4 * q] = w.x; w8[4 * q + 1] = w.y; w8[4 * q + 2] = w.z; w8[4 * q + 3] = w.w;
          }
        };
        ld8(zr + u0, zg4);
        if (mp == 2) ld8(zr + a.bw + u0, zu4);
        if (kSplit) {
          ld8(zrl + u0, zgl);
          if (mp == 2) ld8(zrl + a.bw + u0, zul);
        }
      }
      uint32_t v[16];
      tmem_ld16(tacc + u0, v);
      tmem_ld_wait();
      uint32_t pg[8], pu[8], lg[8], lu[8];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float dA = 0.f, zg = 0.f, zu = 0.f;
        if (valid) {
          dA = __uint_as_float(v[i]);
          zg = bf16_at(zg4[i / 2], i);
          if (kSplit) zg += bf16_at(zgl[i / 2], i);
          if (mp == 2) {
            zu = bf16_at(zu4[i / 2], i);
            if (kSplit) zu += bf16_at(zul[i / 2], i);
          }
        }
        float av, dg, du;
        act_fwd_bwd<true>(act, zg, zu, av, dg, du);
        dgate = fmaf(dA, av, dgate);
        const float dzg = g * dA * dg, dzu = g * dA * du;
        const uint32_t bg = __bfloat16_as_ushort(__float2bfloat16(dzg));
        const uint32_t bu = __bfloat16_as_ushort(__float2bfloat16(dzu));
        if (i & 1) { pg[i / 2] |= bg << 16; pu[i / 2] |= bu << 16; }
        else { pg[i / 2] = bg; pu[i / 2] = bu; }
        if (kSplit) {
          const uint32_t cg = __bfloat16_as_ushort(__float2bfloat16(dzg - __uint_as_float(bg << 16)));
          const uint32_t cu = __bfloat16_as_ushort(__float2bfloat16(dzu - __uint_as_float(bu << 16)));
          if (i & 1) { lg[i / 2] |= cg << 16; lu[i / 2] |= cu << 16; }
          else { lg[i / 2] = cg; lu[i / 2] = cu; }
        }
      }
      uint4* d4 = reinterpret_cast<uint4*>(dzr + u0);
#pragma unroll
      for (int q = 0; q < 2; ++q) d4[q] = make_uint4(pg[4 * q], pg[4 * q + 1], pg[4 * q + 2], pg[4 * q + 3]);
      if (mp == 2) {
        uint4* u4 = reinterpret_cast<uint4*>(dzr + a.bw + u0);
#pragma unroll
        for (int q = 0; q < 2; ++q) u4[q] = make_uint4(pu[4 * q], pu[4 * q + 1], pu[4 * q + 2], pu[4 * q + 3]);
      }
      if (kSplit) {
        uint4* l4 = reinterpret_cast<uint4*>(dzrl + u0);
#pragma unroll
        for (int q = 0; q < 2; ++q) l4[q] = make_uint4(lg[4 * q], lg[4 * q + 1], lg[4 * q + 2], lg[4 * q + 3]);
        if (mp == 2) {
          uint4* m4 = reinterpret_cast<uint4*>(dzrl + a.bw + u0);
#pragma unroll
          for (int q = 0; q < 2; ++q) m4[q] = make_uint4(lu[4 * q], lu[4 * q + 1], lu[4 * q + 2], lu[4 * q + 3]);
        }
      }
    }
    // column-split epilogue: combine the two halves' partial dgate (half 1 ->
    // smem -> half 0); half < 0: this thread saw the whole row
    const int q = row >> 5;
    if (half >= 0) {
      if (half == 1) dg_xchg[row] = dgate;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
      if (half == 0) dgate = dgate + dg_xchg[row];
    }
    if (half <= 0 && a.nu > 1) {
      // unit-tiled block: this tile's partial dgate; dgate_reduce_kernel sums
      // the tiles and derives dlogit / the dense dlogits
      a.dgp[prow * a.nu + ti.ut] = valid ? dgate : 0.f;
    } else if (half <= 0) {
      // dlogit = dgate * g (1 - g) = dgate * sigma(z) sigma(-z): no cancellation in 1 - g
      float dlogit = 0.f;
      int64_t t = 0;
      if (valid && a.gate == SPT_GATE_SIGMOID) {
        t = a.r.bucket_token[ti.pos0 + row];
        dlogit = dgate * sigmoid_pair(a.r.logits[t * a.G + ti.b]);
      }
      a.rows_f[prow] = valid ? dgate : 0.f;
      a.rows_g[prow] = dlogit;
      if (valid && a.gate == SPT_GATE_SIGMOID) {
        __nv_bfloat16* dl = (__nv_bfloat16*)a.dlg;
        const __nv_bfloat16 hi = __float2bfloat16(dlogit);
        const __nv_bfloat16 lo = __float2bfloat16(dlogit - __bfloat162float(hi));
        dl[t * a.gpad + ti.b] = hi;
        dl[(a.T + t) * a.gpad + ti.b] = lo;
      }
    }
    if (half >= 0) asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");  // dg_xchg reuse
  } else {  // DW1, DW2, DWR: fp32 tiles
    // NOTE: tcgen05.ld is warp-collective (.sync.aligned): every lane executes
    // the loads; only the stores are predicated on the row being real.
    int64_t orow = 0;
    bool live;
    int c_lo, c_hi;
    const int ncols = min(256, a.d - ti.nt * 256);
    if (KIND == K_DWR) {  // split-K partial [split][G][d]; MH == 2 (G > 128): half = block half
      const int f = (a.MH == 2 ? half * 128 : 0) + row;
      live = f < a.G;
      orow = (int64_t)ti.b * a.G + f;
      if (a.MH == 2) { c_lo = 0; c_hi = ncols; }
      else { c_lo = half * 128; c_hi = min(ncols, c_lo + 128); }
    } else {
      // MH == 2: this warp's half owns accumulator `half` (features half*128 + row);
      // MH == 1: one accumulator, columns split between the halves
      const int f = ti.ut * 256 + (a.MH == 2 ? half * 128 : 0) + row;
      const int M = KIND == K_DW1 ? a.mp * a.bw : a.bw;
      live = f < M;
      if (KIND == K_DW1 && a.mp == 2)
        orow = f < a.bw ? (int64_t)ti.b * a.bw + f : (int64_t)a.D + (int64_t)ti.b * a.bw + (f - a.bw);
      else
        orow = (int64_t)ti.b * a.bw + f;
      if (a.MH == 2) { c_lo = 0; c_hi = ncols; }
      else { c_lo = half * 128; c_hi = min(ncols, c_lo + 128); }
    }
    float* dst = (float*)a.out + orow * a.d + ti.nt * 256;
    const bool acc = KIND != K_DWR && a.acc_mode;
    for (int c0 = c_lo; c0 < c_hi; c0 += 64) {
      uint32_t v[64];
      const bool two = c0 + 32 < c_hi;
      if (ti.nkb > 0) {
        tmem_ld64(tacc + c0, v, two);
      } else {
#pragma unroll
        for (int i = 0; i < 64; ++i) v[i] = 0u;
      }
      if (!live) continue;
      float4* d4 = reinterpret_cast<float4*>(dst + c0);
      const int nq = two ? 16 : 8;
#pragma unroll
      for (int qq = 0; qq < 16; ++qq) {
        if (qq >= nq) break;
        float4 o = make_float4(__uint_as_float(v[4 * qq]), __uint_as_float(v[4 * qq + 1]),
                               __uint_as_float(v[4 * qq + 2]), __uint_as_float(v[4 * qq + 3]));
        if (acc) {
          const float4 p = d4[qq];
          o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
        }
        d4[qq] = o;
      }
    }
  }
}

// FWD2 / DX epilogue: the 32 rows x 128 columns of this warp go out as two
// 32 x 64 TMA tensor stores from a 128-byte-swizzled smem staging buffer
// (full-line writes, no per-thread strided stores).  Padding rows of the tile
// are written too: they lie inside the block's own padded bucket rows, which
// no consumer reads.
__device__ __forceinline__ void epilogue_tma_store(const TcArgs& a, const TileInfo& ti,
                                                   uint32_t tacc, int q, int lane, int half,
                                                   uint8_t* stg, int& stg_i) {
  const int ncols = min(256, a.d - ti.nt * 256);
  const int c_lo = half * 128, c_hi = min(ncols, c_lo + 128);
  for (int c0 = c_lo; c0 < c_hi; c0 += 64) {
    uint32_t v[64];
    tmem_ld64(tacc + c0, v, true);
    uint8_t* buf = stg + stg_i * 4096;
    if (lane == 0) {
      if (a.n_stg == 3) bulk_wait_read<2>();
      else if (a.n_stg == 2) bulk_wait_read<1>();
      else bulk_wait_read<0>();
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 8; ++c) {  // 16-byte chunk c of this row, swizzled by row & 7
      const uint4 w = make_uint4(pack_bf16(__uint_as_float(v[8 * c + 0]), __uint_as_float(v[8 * c + 1])),
                                 pack_bf16(__uint_as_float(v[8 * c + 2]), __uint_as_float(v[8 * c + 3])),
                                 pack_bf16(__uint_as_float(v[8 * c + 4]), __uint_as_float(v[8 * c + 5])),
                                 pack_bf16(__uint_as_float(v[8 * c + 6]), __uint_as_float(v[8 * c + 7])));
      *reinterpret_cast<uint4*>(buf + lane * 128 + ((c ^ (lane & 7)) << 4)) = w;
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(&a.tc, buf, ti.nt * 256 + c0, (int)(ti.prow0 + q * 32));
      bulk_commit();
    }
    stg_i = (stg_i + 1) % a.n_stg;
  }
}

// DAT epilogue: the accumulator is dA^T (TMEM lane = unit of the block, column =
// token row of the pair tile).  Each warp stages 32 tokens x 32 units of fp32
// row-major in smem and TMA-stores the box into dA[row][unit]; dgate / dZ are
// computed from dA and the Z stash by da_post_kernel (a streaming pass).
__device__ __forceinline__ void epilogue_dat(const TcArgs& a, const TileInfo& ti, uint32_t tacc,
                                             int q, int lane, int half, uint8_t* stg) {
  const bool units_live = q * 32 < a.bw;
  float* buf = reinterpret_cast<float*>(stg);
  for (int c0 = half * 128; c0 < half * 128 + 128; c0 += 32) {
    uint32_t v[32];
    tmem_ld32(tacc + c0, v);
    tmem_ld_wait();
    if (!units_live || c0 >= ti.rows_pad) continue;  // warp-uniform
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) buf[j * 32 + lane] = __uint_as_float(v[j]);  // [token j][unit]
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(&a.tc, buf, q * 32, (int)(ti.prow0 + c0));
      bulk_commit();
    }
  }
}

// DAT fused epilogue (a7 with tokens on N; Alg. 4 line 10's dgate and the dZ of
// the activation, as the DA epilogue computes them): TMEM lane = unit u = 32 q +
// lane of the block, column = token row of the pair tile; this warp owns the 128
// rows of `half`.  Per 16 rows: the Z stash values of (row, u) are loaded before
// the TMEM load, dZ(row, u) is written at once (64-byte warp segments), and the
// per-row dgate partials dA * act(z) are summed over the warp's 32 units by a
// reduce-scatter (16 shuffles for 16 rows); the four unit quarters meet in smem
// (xq) and are added in ascending q, after which each warp finishes 32 rows:
// dgate, dlogit = dgate g (1 - g), the dense dlogits (hi | lo).  Rows past the
// block's n_b get zero dZ / dgate / dlogit up to its padded end (rows_pad).
template <int ACT>
__device__ __forceinline__ void epilogue_dat_fused(const TcArgs& a, const TileInfo& ti,
                                                   uint32_t tacc, int q, int lane, int half,
                                                   float* xchg) {
  constexpr bool kGlu = ACT == SPT_ACT_SWIGLU;  // m' = 2: Z / dZ rows hold gate | up
  const int u = q * 32 + lane;
  const bool ulive = u < a.bw;
  const int zs = (kGlu ? 2 : 1) * a.bw;  // Z / dZ row stride (elements)
  float* xq = xchg + half * 512;  // [4 quarters][128 rows] partial dgate of this half
  const int r_lo = half * 128;
  for (int c0 = r_lo; c0 < r_lo + 128; c0 += 16) {
    if (c0 >= ti.rows_pad) break;  // uniform over the half's four warps
    const int nv = ulive ? ti.n_valid - c0 : 0;   // rows j < nv are real
    const int np = ulive ? ti.rows_pad - c0 : 0;  // rows j < np get dZ (zeros past nv)
    const float gl = (lane < 16 && c0 + lane < ti.n_valid) ? a.r.bucket_gate[ti.pos0 + c0 + lane] : 0.f;
    const __nv_bfloat16* zrow = (const __nv_bfloat16*)a.aux + (ti.prow0 + c0) * (int64_t)zs + u;
    __nv_bfloat16* dzrow = (__nv_bfloat16*)a.out2 + (ti.prow0 + c0) * (int64_t)zs + u;
    uint32_t zg[16], zu[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      zg[j] = j < nv ? (uint32_t)__bfloat16_as_ushort(zrow[j * zs]) : 0u;
      if (kGlu) zu[j] = j < nv ? (uint32_t)__bfloat16_as_ushort(zrow[j * zs + a.bw]) : 0u;
    }
    uint32_t v[16];
    tmem_ld16(tacc + c0, v);
    tmem_ld_wait();
    float p[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float dA = j < nv ? __uint_as_float(v[j]) : 0.f;
      const float g = __shfl_sync(0xffffffffu, gl, j);
      float av, dg, du;
      act_fwd_bwd<true>(ACT, __uint_as_float(zg[j] << 16), kGlu ? __uint_as_float(zu[j] << 16) : 0.f,
                        av, dg, du);
      p[j] = dA * av;
      if (j < np) {
        dzrow[j * zs] = __float2bfloat16(g * dA * dg);
        if (kGlu) dzrow[j * zs + a.bw] = __float2bfloat16(g * dA * du);
      }
    }
    // reduce-scatter of p[0..16) over the 32 lanes: offsets 16, 8, 4, 2 halve the
    // values each lane keeps, a final xor-1 add completes them
    float h8[8], h4[4], h2[2];
    {
      const bool up = lane & 16;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        h8[i] = (up ? p[i + 8] : p[i]) + __shfl_xor_sync(0xffffffffu, up ? p[i] : p[i + 8], 16);
    }
    {
      const bool up = lane & 8;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        h4[i] = (up ? h8[i + 4] : h8[i]) + __shfl_xor_sync(0xffffffffu, up ? h8[i] : h8[i + 4], 8);
    }
    {
      const bool up = lane & 4;
#pragma unroll
      for (int i = 0; i < 2; ++i)
        h2[i] = (up ? h4[i + 2] : h4[i]) + __shfl_xor_sync(0xffffffffu, up ? h4[i] : h4[i + 2], 4);
    }
    const bool up2 = lane & 2;
    float h1 = (up2 ? h2[1] : h2[0]) + __shfl_xor_sync(0xffffffffu, up2 ? h2[0] : h2[1], 2);
    h1 += __shfl_xor_sync(0xffffffffu, h1, 1);
    const int jrow = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
    if ((lane & 1) == 0) xq[q * 128 + (c0 - r_lo) + jrow] = h1;
  }
  asm volatile("bar.sync %0, 128;" ::"r"(5 + half) : "memory");
  const int rr = r_lo + q * 32 + lane;  // this thread finishes row rr of the pair tile
  if (rr < ti.rows_pad) {
    const int i = rr - r_lo;
    const bool valid = rr < ti.n_valid;
    const float dgate = valid ? ((xq[i] + xq[128 + i]) + xq[256 + i]) + xq[384 + i] : 0.f;
    const int64_t prow = ti.prow0 + rr;
    float dlogit = 0.f;
    if (valid && a.gate == SPT_GATE_SIGMOID) {
      const int64_t t = a.r.bucket_token[ti.pos0 + rr];
      dlogit = dgate * sigmoid_pair(a.r.logits[t * a.G + ti.b]);
      __nv_bfloat16* dl = (__nv_bfloat16*)a.dlg;
      const __nv_bfloat16 hi = __float2bfloat16(dlogit);
      dl[t * a.gpad + ti.b] = hi;
      dl[(a.T + t) * a.gpad + ti.b] = __float2bfloat16(dlogit - __bfloat162float(hi));
    }
    a.rows_f[prow] = dgate;
    a.rows_g[prow] = dlogit;
  }
  asm volatile("bar.sync %0, 128;" ::"r"(5 + half) : "memory");  // xq reuse by the next tile
}

// DAT fused epilogue, row-major form: each 32-unit x 16-row TMEM chunk is
// transposed through a per-warp smem tile (16 x 33 floats, conflict-free), after
// which lane l works on row l / 2 and units 16 (l % 2) .. +16 of the warp's
// quarter -- 16-byte Z loads and dZ stores, a thread-local rowdot finished by one
// xor-1 shuffle -- instead of one 2-byte access per (row, unit) (measured 1.62
// vs 1.40 ms for the tokens-on-M dA).  Same outputs as epilogue_dat_fused.
template <int ACT>
__device__ __forceinline__ void epilogue_dat_rows(const TcArgs& a, const TileInfo& ti,
                                                  uint32_t tacc, int q, int lane, int half,
                                                  float* xchg, float* tbuf) {
  constexpr bool kGlu = ACT == SPT_ACT_SWIGLU;
  const int zs = (kGlu ? 2 : 1) * a.bw;
  float* xq = xchg + half * 512;
  const int r_lo = half * 128;
  const int jr = lane >> 1, uh = lane & 1;
  const int u0 = q * 32 + uh * 16;            // this lane's 16 units
  const bool ulive = u0 < a.bw;               // bw % 16 == 0: all 16 or none
  for (int c0 = r_lo; c0 < r_lo + 128; c0 += 16) {
    if (c0 >= ti.rows_pad) break;  // uniform over the half's four warps
    const int r = c0 + jr;
    const bool valid = ulive && r < ti.n_valid;
    const bool write = ulive && r < ti.rows_pad;
    // Z stash loads first (their latency overlaps the TMEM load and the transpose)
    uint4 zg4[2], zu4[2];
    const __nv_bfloat16* zr = (const __nv_bfloat16*)a.aux + (ti.prow0 + r) * (int64_t)zs + u0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      zg4[h] = valid ? reinterpret_cast<const uint4*>(zr)[h] : make_uint4(0u, 0u, 0u, 0u);
      zu4[h] = (kGlu && valid) ? reinterpret_cast<const uint4*>(zr + a.bw)[h] : make_uint4(0u, 0u, 0u, 0u);
    }
    const float g = valid ? a.r.bucket_gate[ti.pos0 + r] : 0.f;
    uint32_t v[16];
    tmem_ld16(tacc + c0, v);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; ++j) tbuf[j * 33 + lane] = __uint_as_float(v[j]);  // [row j][unit lane]
    __syncwarp();
    float dA[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) dA[i] = valid ? tbuf[jr * 33 + uh * 16 + i] : 0.f;
    __syncwarp();  // tbuf reuse by the next chunk
    const uint32_t zgw[8] = {zg4[0].x, zg4[0].y, zg4[0].z, zg4[0].w, zg4[1].x, zg4[1].y, zg4[1].z, zg4[1].w};
    const uint32_t zuw[8] = {zu4[0].x, zu4[0].y, zu4[0].z, zu4[0].w, zu4[1].x, zu4[1].y, zu4[1].z, zu4[1].w};
    uint32_t pg[8], pu[8];
    float p = 0.f;
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      float av0, dg0, du0, av1, dg1, du1;
      act_fwd_bwd<true>(ACT, bf16_at(zgw[i / 2], 0), kGlu ? bf16_at(zuw[i / 2], 0) : 0.f, av0, dg0, du0);
      act_fwd_bwd<true>(ACT, bf16_at(zgw[i / 2], 1), kGlu ? bf16_at(zuw[i / 2], 1) : 0.f, av1, dg1, du1);
      p = fmaf(dA[i], av0, p);
      p = fmaf(dA[i + 1], av1, p);
      pg[i / 2] = pack_bf16(g * dA[i] * dg0, g * dA[i + 1] * dg1);
      pu[i / 2] = pack_bf16(g * dA[i] * du0, g * dA[i + 1] * du1);
    }
    if (write) {
      uint4* dzr = reinterpret_cast<uint4*>((__nv_bfloat16*)a.out2 + (ti.prow0 + r) * (int64_t)zs + u0);
      dzr[0] = make_uint4(pg[0], pg[1], pg[2], pg[3]);
      dzr[1] = make_uint4(pg[4], pg[5], pg[6], pg[7]);
      if (kGlu) {
        uint4* dur = reinterpret_cast<uint4*>((__nv_bfloat16*)a.out2 + (ti.prow0 + r) * (int64_t)zs + a.bw + u0);
        dur[0] = make_uint4(pu[0], pu[1], pu[2], pu[3]);
        dur[1] = make_uint4(pu[4], pu[5], pu[6], pu[7]);
      }
    }
    p += __shfl_xor_sync(0xffffffffu, p, 1);  // the warp's 32 units of row jr
    if (uh == 0) xq[q * 128 + (c0 - r_lo) + jr] = p;
  }
  asm volatile("bar.sync %0, 128;" ::"r"(5 + half) : "memory");
  const int rr = r_lo + q * 32 + lane;
  if (rr < ti.rows_pad) {
    const int i = rr - r_lo;
    const bool valid = rr < ti.n_valid;
    const float dgate = valid ? ((xq[i] + xq[128 + i]) + xq[256 + i]) + xq[384 + i] : 0.f;
    const int64_t prow = ti.prow0 + rr;
    float dlogit = 0.f;
    if (valid && a.gate == SPT_GATE_SIGMOID) {
      const int64_t t = a.r.bucket_token[ti.pos0 + rr];
      dlogit = dgate * sigmoid_pair(a.r.logits[t * a.G + ti.b]);
      __nv_bfloat16* dl = (__nv_bfloat16*)a.dlg;
      const __nv_bfloat16 hi = __float2bfloat16(dlogit);
      dl[t * a.gpad + ti.b] = hi;
      dl[(a.T + t) * a.gpad + ti.b] = __float2bfloat16(dlogit - __bfloat162float(hi));
    }
    a.rows_f[prow] = dgate;
    a.rows_g[prow] = dlogit;
  }
  asm volatile("bar.sync %0, 128;" ::"r"(5 + half) : "memory");  // xq reuse by the next tile
}

// One K stage (4 x K=16) of MMAs into MH accumulator halves: descriptors are
// advanced by constant adds (start address field, 16-byte units; no carry:
// smem offsets < 256 KB), the A half h lives 16 KB after half 0.
template <int MH, int NK = 4>
__device__ __forceinline__ void issue_kstage(uint32_t dtm, uint32_t hstride, uint64_t ad,
                                             uint64_t bd, uint32_t a_kstep, uint32_t b_kstep,
                                             uint32_t idesc, bool accumulate,
                                             uint32_t a_hoff = 16384 >> 4) {
#pragma unroll
  for (int k = 0; k < NK; ++k)
#pragma unroll
    for (int h = 0; h < MH; ++h)
      mma_bf16(dtm + h * hstride, ad + h * a_hoff + k * a_kstep, bd + k * b_kstep, idesc,
               (accumulate || k != 0) ? 1u : 0u);
}

// diagnostics: cycles spent in an mbarrier wait, accumulated into trace slot
__device__ __forceinline__ void twait(uint64_t* bar, uint32_t parity, unsigned long long* tr, int slot) {
  if (tr) {
    const long long t0 = clock64();
    mbar_wait(bar, parity);
    tr[slot] += (unsigned long long)(clock64() - t0);
  } else {
    mbar_wait(bar, parity);
  }
}
// trace slots (per CTA, 8 x u64): 0 MMA wait full, 1 MMA wait tempty, 2 epi wait tfull,
// 3 epi busy, 4 TMA producer wait empty, 5 gather wait empty, 6 total cycles, 7 tiles
constexpr int kTraceSlots = 8;

// ------------------------------------------------------------------ kernel
template <int KIND, bool kSplit = false>
__global__ void __launch_bounds__(kThreads, 1) tc_gemm_kernel(const __grid_constant__ TcArgs a,
                                                               int n_stages) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr bool kAmn = kind_a_mn(KIND);
  constexpr bool kBmn = kind_b_mn(KIND);
  constexpr int BK = kind_bk(KIND);  // K rows per stage
  const int astride = kABytes * BK / 64 * a.MH;
  const int bstride = (b_bytes(KIND, a.BN, a.kstream) + 1023) & ~1023;
  const int sstride = astride + bstride;
  const bool resident = kind_bres(KIND) && !a.kstream;  // weight-resident units
  // barrier area after the stage ring (weight-resident kinds: after slab + ring)
  const int ring_bytes = resident
                             ? (KIND == K_FWD2 ? (a.bw + 63) / 64 : (a.mp * a.bw + 63) / 64) * 32768 +
                                   n_stages * kABytes
                             : n_stages * sstride;
  uint64_t* full = (uint64_t*)(smem + ring_bytes);
  uint64_t* empty = full + n_stages;
  uint64_t* tfull = empty + n_stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* bres_full = tempty + 2;
  uint64_t* bres_empty = bres_full + 1;
  uint32_t* tmem_slot = (uint32_t*)(bres_empty + 1);
  float* dg_xchg = (float*)(tmem_slot + 4);  // [128] DA half-row exchange
  uint8_t* stg_base = (uint8_t*)(((uintptr_t)(dg_xchg + 128) + 1023) & ~(uintptr_t)1023);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  SideState side{-1, 0, 0, 0, 0.f};  // DW*: grad-input combine claim of this warp
  // two accumulators alternate between tiles when both fit in TMEM
  const int n_acc = tm_nacc(a.BN, a.MH);
  constexpr bool kGather = kind_gather_a(KIND) || kind_gather_b(KIND);  // uses cp.async
  const int n_epi = kind_gather_b(KIND) ? kEpiWarpsDW : kEpiWarps;
  constexpr int g1_cp_w0 = 12;              // first cp.async warp (gathered-A kinds)
  constexpr int g1_ncp = (16 - g1_cp_w0) * 32;  // cp.async threads
  if (threadIdx.x == 0) {
    // stage barrier: warp 0's TMA arm (+ expected bytes); FWD1 / DA: one arm
    // per gather4 warp; DW*: one cp.async completion arrival per gather thread
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(&full[s], kind_gather_b(KIND) ? 1 + kCpThreadsB
                          : (kind_gather_a(KIND) ? kTmaGatherWarps + g1_ncp : 1));
      mbar_init(&empty[s], 1);
    }
    mbar_init(bres_full, 1);
    mbar_init(bres_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], n_epi);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&a.ta);
    tma_prefetch_desc(&a.tb);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // PDL: barriers / TMEM set up; now the predecessor's outputs are visible
  // successor launches as this grid's CTAs exit (an early trigger measured slower)
  const int ntiles = num_tiles<KIND>(a);
  unsigned long long* tr = a.trace ? a.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
  const long long t_start = clock64();

  if (resident) {
    // ============ weight-resident units (FWD2 / DX): B slab once per unit
    const int kbu = KIND == K_FWD2 ? (a.bw + 63) / 64 : (a.mp * a.bw + 63) / 64;  // K stages
    uint8_t* sBres = smem;                                   // kbu x 32 KB
    uint8_t* ring = smem + kbu * 32768;                      // A stages of 16 KB
    if (warp == 0) {
      if (lane == 0) {
        int stage = 0;
        uint32_t phase = 0, uph = 0;
        for (int u = blockIdx.x; u < ntiles; u += gridDim.x) {
          const UnitInfo ui = decode_unit(a, u);
          twait(bres_empty, uph ^ 1, tr, 4);
          mbar_arrive_expect_tx(bres_full, kbu * 32768u);
          for (int kb = 0; kb < kbu; ++kb) {
            int krow;
            if (KIND == K_FWD2) krow = ui.b * a.bw + kb * 64;
            else krow = kb * 64 < a.bw ? ui.b * a.bw + kb * 64 : a.D + ui.b * a.bw + (kb * 64 - a.bw);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              tma_load_2d(sBres + kb * 32768 + j * 8192, &a.tb, bres_full, ui.nt * 256 + j * 64, krow);
          }
          uph ^= 1;
          for (int mt = ui.mt0; mt < ui.mt1; ++mt) {
            const int64_t prow0 = decode_mtile<KIND>(a, ui, mt).prow0;
            for (int kb = 0; kb < kbu; ++kb) {
              twait(&empty[stage], phase ^ 1, tr, 4);
              mbar_arrive_expect_tx(&full[stage], kABytes);
              tma_load_2d(ring + stage * kABytes, &a.ta, &full[stage], kb * 64, (int)prow0);
              if (++stage == n_stages) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
    } else if (warp == 1) {
      // whole warp, one elected issuer (see the MMA issuer below)
      const uint32_t idesc = idesc_bf16(128, 256, false, true);
      const uint64_t adesc0 = sdesc_sw128(smem_u32(ring), 16, 1024);
      const uint64_t bdesc0 = sdesc_sw128(smem_u32(sBres), 8192, 1024);
      unsigned long long* trl = lane == 0 ? tr : nullptr;
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0, uph = 0;
      for (int u = blockIdx.x; u < ntiles; u += gridDim.x) {
        const UnitInfo ui = decode_unit(a, u);
        twait(bres_full, uph, trl, 5);
        uph ^= 1;
        for (int mt = ui.mt0; mt < ui.mt1; ++mt) {
          twait(&tempty[acc], aphase ^ 1, trl, 1);
          tc_fence_after();
          if (trl) trl[7] += 1;
          const uint32_t dtm = tmem + acc * 256;
          for (int kb = 0; kb < kbu; ++kb) {
            twait(&full[stage], phase, trl, 0);
            tc_fence_after();
            if (elect_one()) {
              issue_kstage<1>(dtm, 0, adesc0 + (uint64_t)((stage * kABytes) >> 4),
                              bdesc0 + (uint64_t)((kb * 32768) >> 4), 32 >> 4, 2048 >> 4, idesc,
                              kb != 0);
              mma_commit(&empty[stage]);
            }
            __syncwarp();
            if (++stage == n_stages) { stage = 0; phase ^= 1; }
          }
          if (elect_one()) mma_commit(&tfull[acc]);
          __syncwarp();
          if (++acc == 2) { acc = 0; aphase ^= 1; }
        }
        if (elect_one()) mma_commit(bres_empty);  // weight slab free once this unit's MMAs retire
        __syncwarp();
      }
    } else if (warp >= 4 && warp < 4 + kEpiWarps) {
      const int e = warp - 4;
      const int q = warp & 3;
      const int half = e >> 2;
      int acc = 0, stg_i = 0;
      uint32_t aphase = 0;
      for (int u = blockIdx.x; u < ntiles; u += gridDim.x) {
        const UnitInfo ui = decode_unit(a, u);
        for (int mt = ui.mt0; mt < ui.mt1; ++mt) {
          const TileInfo ti = decode_mtile<KIND>(a, ui, mt);
          twait(&tfull[acc], aphase, (tr && threadIdx.x == 4 * 32) ? tr : nullptr, 2);
          tc_fence_after();
          const long long te0 = clock64();
          epilogue_tma_store(a, ti, tmem + ((uint32_t)(q * 32) << 16) + acc * 256, q, lane, half,
                               stg_base + e * a.n_stg * 4096, stg_i);
          tc_fence_before();
          __syncwarp();
          if (tr && threadIdx.x == 4 * 32) tr[3] += (unsigned long long)(clock64() - te0);
          if (lane == 0) mbar_arrive(&tempty[acc]);
          if (++acc == 2) { acc = 0; aphase ^= 1; }
        }
      }
      if (lane == 0) bulk_wait<0>();  // all partial tiles written before exit
    }
  } else if (kind_gather_a(KIND) && (warp == 0 || warp == 2 || warp == 3)) {
    // ------------------------ FWD1 / DA: TMA tile::gather4 of 256 token rows
    const int p = warp == 0 ? 0 : warp - 1;   // 0, 1, 2
    const int c = lane * kTmaGatherWarps + p;  // gather call of this lane: rows 4c..4c+3
    const int n_calls = a.g1_rows / 4;  // rows [0, g1_rows) of each 256-row stage by TMA
    const bool has_call = c < n_calls;
    const int my_calls = n_calls > p ? (n_calls - p + kTmaGatherWarps - 1) / kTmaGatherWarps : 0;
    const uint32_t tx = (a.ablate == 1 || a.ablate >= 3 ? 0u : (uint32_t)my_calls * 512u) +
                        (p == 0 && a.ablate < 3 ? tile_tx_bytes<KIND>(a) : 0u);
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const TileInfo ti = decode<KIND>(a, tile);
      int rr[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = 4 * c + i;
        rr[i] = (has_call && r < ti.n_valid) ? a.r.bucket_token[ti.pos0 + r] : (int)a.T;
      }
      if (KIND == K_DA || (KIND == K_DAT && a.dat_fused)) {
        // the epilogue reads this tile's Z stash rows (m'*bw bf16 each, written by
        // the forward and long evicted): warm L2 now, a whole mainloop ahead
        const int zrow = a.mp * a.bw * 2;
        for (int r = lane * kTmaGatherWarps + p; r < 256 && r < ti.rows_pad; r += 32 * kTmaGatherWarps)
          prefetch_l2_bulk((const uint8_t*)a.aux + (ti.prow0 + r) * zrow, zrow);
      }
      for (int kb = 0; kb < ti.nkb; ++kb) {
        if (lane == 0) {
          twait(&empty[stage], phase ^ 1, (tr && warp == 0) ? tr : nullptr, 4);
          mbar_arrive_expect_tx(&full[stage], tx);
        }
        __syncwarp();
        uint8_t* sA = smem + stage * sstride;
        if (p == 0 && lane == 0 && a.ablate < 3)
          produce_tiles<KIND>(a, ti, kb, sA, sA + astride, &full[stage]);
        if (has_call && a.ablate != 1 && a.ablate < 3) {
          int kk = kb;
          const int ps = kpass(ti, kb, kk);
          tma_gather4((kind_rows_on_b(KIND) ? sA + astride : sA) + c * 512, ps == 2 ? &a.ta2 : &a.ta,
                      &full[stage], kk * 64, rr[0], rr[1], rr[2], rr[3]);
          // warm L2 with the next 256 columns of these rows in one 512-byte run per
          // row (DRAM-friendly), 4..7 stages ahead of their gathers
          if (a.prefetch && !kind_rows_on_b(KIND) && (kb & 3) == 0 && kb + 4 < ti.nkb)
            tma_prefetch_gather4(&a.tc, (kb + 4) * 64, rr[0], rr[1], rr[2], rr[3]);
        }
        if (++stage == n_stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 0) {
    // ------------------------------------------------- TMA tile producer
    if (lane == 0) {
      const uint32_t tx = a.ablate >= 3 ? 0u : tile_tx_bytes<KIND>(a);
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const TileInfo ti = decode<KIND>(a, tile);
        for (int kb = 0; kb < ti.nkb; ++kb) {
          twait(&empty[stage], phase ^ 1, tr, 4);
          mbar_arrive_expect_tx(&full[stage], tx);
          uint8_t* sA = smem + stage * sstride;
          if (a.ablate < 3) produce_tiles<KIND>(a, ti, kb, sA, sA + astride, &full[stage]);
          if (++stage == n_stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (kind_gather_a(KIND) && warp >= g1_cp_w0) {
    // ------------ FWD1 / DA / DAT: cp.async of rows [g1_rows, 256) of each stage
    // thread t: 16-byte piece (t & 7) of rows g1_rows + (t >> 3) + 16 i
    const int t = threadIdx.x - g1_cp_w0 * 32;  // 0..g1_ncp-1
    const int rstep = g1_ncp / 8;                // rows covered per i (16 or 32)
    const __nv_bfloat16* src = (const __nv_bfloat16*)a.aux2;
    const int ch = t & 7;
    constexpr int kRowsPer = 14;  // upper bound: g1_rows >= 32
    const int r0 = a.g1_rows;
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const TileInfo ti = decode<KIND>(a, tile);
      int tok[kRowsPer];
#pragma unroll
      for (int i = 0; i < kRowsPer; ++i) {
        const int r = r0 + (t >> 3) + rstep * i;
        tok[i] = (r < 256 && r < ti.n_valid) ? a.r.bucket_token[ti.pos0 + r] : -1;
      }
      for (int kb = 0; kb < ti.nkb; ++kb) {
        if (lane == 0) mbar_wait(&empty[stage], phase ^ 1);
        __syncwarp();
        const uint32_t sA = smem_u32(smem + stage * sstride + (kind_rows_on_b(KIND) ? astride : 0));
        int kk = kb;
        const __nv_bfloat16* srcp = kpass(ti, kb, kk) == 2 ? (const __nv_bfloat16*)a.aux2_lo : src;
#pragma unroll
        for (int i = 0; i < kRowsPer; ++i) {
          if (a.ablate == 1 || a.ablate >= 3) break;
          const int r = r0 + (t >> 3) + rstep * i;
          if (r >= 256) break;
          const uint32_t dst = sA + (r >> 7) * 16384 + (r & 127) * 128 + ((ch ^ (r & 7)) << 4);
          const __nv_bfloat16* g = srcp + (int64_t)(tok[i] < 0 ? 0 : tok[i]) * a.d + kk * 64 + ch * 8;
          cp_async_16(dst, g, tok[i] < 0 ? 0u : 16u);
        }
        cp_async_arrive_noinc(&full[stage]);
        if (++stage == n_stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (kind_gather_b(KIND) && (warp == 2 || warp == 3 || warp >= 8)) {
    // ------------------------- DW*: cp.async row gathers of B (10 warps)
    // B: BK bucket rows (K) x 256 columns (N) per stage, MN-major: 64-column
    // chunk j at +BK*128 B*j, K row r at +128 B*r, 16-byte piece p swizzled
    // by r.  This thread: piece (gt & 31) of rows r_i = (gt >> 5) + 10 i.  Its
    // arrival on the stage barrier fires when its copies have landed.
    constexpr int kRowsG = (BK + kGatherWarpsB - 1) / kGatherWarpsB;  // rows per thread (upper bound)
    const int gt = (warp < 4 ? warp - 2 : warp - 6) * 32 + lane;  // 0..319
    const __nv_bfloat16* src = (const __nv_bfloat16*)a.aux2;
    const int j = (gt & 31) >> 3, pc = gt & 7;
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const TileInfo ti = decode<KIND>(a, tile);
      int tk[kRowsG];  // this stage's token rows (loaded one stage ahead)
      auto load_idx = [&](int kb, int (&t)[kRowsG]) {
        int kk = kb;
        kpass(ti, kb, kk);
#pragma unroll
        for (int i = 0; i < kRowsG; ++i) {
          const int r = (gt >> 5) + kGatherWarpsB * i;
          const int e = kk * BK + r;
          t[i] = (r < BK && e < ti.n_valid) ? a.r.bucket_token[ti.pos0 + e] : -1;
        }
      };
      if (ti.nkb > 0) load_idx(0, tk);
      for (int kb = 0; kb < ti.nkb; ++kb) {
        if (a.prefetch && (gt & 31) == 0) {  // warm L2 with this stage's rows (opt-in)
#pragma unroll
          for (int i = 0; i < kRowsG; ++i)
            if (tk[i] >= 0) prefetch_l2_bulk(src + (int64_t)tk[i] * a.d + ti.nt * 256, 512);
        }
        if (lane == 0) mbar_wait(&empty[stage], phase ^ 1);
        __syncwarp();
        const uint32_t sB = smem_u32(smem + stage * sstride + astride);
        int kk = kb;
        const __nv_bfloat16* srcp = kpass(ti, kb, kk) == 1 ? (const __nv_bfloat16*)a.aux2_lo : src;
#pragma unroll
        for (int i = 0; i < kRowsG; ++i) {
          const int r = (gt >> 5) + kGatherWarpsB * i;
          if (r < BK && a.ablate != 1) {
            const uint32_t dst = sB + j * (BK * 128) + r * 128 + ((pc ^ (r & 7)) << 4);
            const __nv_bfloat16* g =
                srcp + (int64_t)(tk[i] < 0 ? 0 : tk[i]) * a.d + ti.nt * 256 + j * 64 + pc * 8;
            cp_async_16(dst, g, tk[i] < 0 ? 0u : 16u);
          }
        }
        cp_async_arrive_noinc(&full[stage]);
        if (kb + 1 < ti.nkb) load_idx(kb + 1, tk);
        if (++stage == n_stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    // The whole warp runs the loop (every value warp-uniform, so descriptors
    // live in uniform registers) and one elected lane issues: a lean issue
    // loop matters, at 8 MMAs per ~1024-clk k-stage a generic one is slower
    // than the tensor pipe (measured: 58% vs 90% of the MMA rate).
    const uint32_t idesc = idesc_bf16(128, a.BN, kAmn, kBmn);
    const uint32_t a_kstep = kAmn ? 2048 >> 4 : 32 >> 4;  // descriptor units (16 B)
    const uint32_t b_kstep = kBmn ? 2048 >> 4 : 32 >> 4;
    const uint32_t hstride = (uint32_t)tm_half_stride(a.BN);
    // MN-major LBO = stride of the 64-element MN chunks = BK rows x 128 B
    const uint64_t adesc0 = sdesc_sw128(smem_u32(smem), kAmn ? BK * 128 : 16, 1024);
    const uint64_t bdesc0 = kBmn ? sdesc_sw128(smem_u32(smem) + astride, BK * 128, 1024)
                                 : sdesc_sw128(smem_u32(smem) + astride, 16, 1024);
    const uint32_t a_hoff = (uint32_t)((astride / a.MH) >> 4);  // A half h at +astride/MH
    unsigned long long* trl = lane == 0 ? tr : nullptr;
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t aphase = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const TileInfo ti = decode<KIND>(a, tile);
      twait(&tempty[acc], aphase ^ 1, trl, 1);
      tc_fence_after();
      if (trl) trl[7] += 1;
      const uint32_t dtm = tmem + tm_col(a.BN, a.MH, acc, 0);
      for (int kb = 0; kb < ti.nkb; ++kb) {
        if (a.ablate < 6) twait(&full[stage], phase, trl, 0);
        const long long tf0 = trl ? clock64() : 0;
        // cp.async writes are generic-proxy: order them before the UMMA reads
        if (kGather && a.ablate < 5) fence_proxy_async_smem();
        tc_fence_after();
        if (trl) trl[5] += (unsigned long long)(clock64() - tf0);
        const uint64_t soff = (uint64_t)((stage * sstride) >> 4);
        if (elect_one()) {
          if (a.MH == 2)
            issue_kstage<2, BK / 16>(dtm, hstride, adesc0 + soff, bdesc0 + soff, a_kstep, b_kstep,
                                     idesc, kb != 0, a_hoff);
          else
            issue_kstage<1, BK / 16>(dtm, hstride, adesc0 + soff, bdesc0 + soff, a_kstep, b_kstep,
                                     idesc, kb != 0, a_hoff);
          mma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == n_stages) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) mma_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == n_acc) { acc = 0; aphase ^= 1; }
    }
  } else if (warp >= 4 && warp < 4 + n_epi) {
    // --------------------------------------------------------- epilogue
    const int e = warp - 4;
    const int q = warp & 3;   // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    int acc = 0;
    uint32_t aphase = 0;
    bool side_done = !(kind_gather_b(KIND) && a.cb_ctr);
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const TileInfo ti = decode<KIND>(a, tile);
      // DW*: grad-input combine units while this tile's accumulator fills
      if (kind_gather_b(KIND) && !side_done) side_done = side_combine_run(a, lane, side, &tfull[acc], aphase);
      twait(&tfull[acc], aphase, (tr && threadIdx.x == 4 * 32) ? tr : nullptr, 2);
      tc_fence_after();
      const long long te0 = clock64();
      const uint32_t lanes = (uint32_t)(q * 32) << 16;
      const int half = e >> 2;  // warp group: M half (pair tiles, DW1) or column half
      if (a.ablate >= 4) {
      } else if (kind_gather_a(KIND) && a.MH == 2) {
        // M half `half` of a pair tile: this warp group owns its rows, all columns
        TileInfo th = ti;
        th.n_valid -= half * 128;
        th.prow0 += half * 128;
        th.pos0 += half * 128;
        if (half * 128 < ti.rows_pad)  // the second m-tile may not exist: write nothing
          epilogue<KIND, kSplit>(a, th, tmem + lanes + tm_col(a.BN, a.MH, acc, half), row, -1, dg_xchg);
      } else if (KIND == K_DAT && a.dat_fused) {
        const uint32_t tacc = tmem + lanes + tm_col(a.BN, a.MH, acc, 0);
        float* xchg = reinterpret_cast<float*>(stg_base);
        float* tbuf = reinterpret_cast<float*>(stg_base + 4096) + e * (16 * 33);
        if (a.dat_fused == 2) {
          if (a.act == SPT_ACT_SWIGLU) epilogue_dat_fused<SPT_ACT_SWIGLU>(a, ti, tacc, q, lane, half, xchg);
          else if (a.act == SPT_ACT_GELU) epilogue_dat_fused<SPT_ACT_GELU>(a, ti, tacc, q, lane, half, xchg);
          else epilogue_dat_fused<SPT_ACT_RELU>(a, ti, tacc, q, lane, half, xchg);
        } else {
          if (a.act == SPT_ACT_SWIGLU) {
            epilogue_dat_rows<SPT_ACT_SWIGLU>(a, ti, tacc, q, lane, half, xchg, tbuf);
          } else if (a.act == SPT_ACT_GELU) {
            epilogue_dat_rows<SPT_ACT_GELU>(a, ti, tacc, q, lane, half, xchg, tbuf);
          } else {
            epilogue_dat_rows<SPT_ACT_RELU>(a, ti, tacc, q, lane, half, xchg, tbuf);
          }
        }
      } else if (KIND == K_DAT) {
        epilogue_dat(a, ti, tmem + lanes + tm_col(a.BN, a.MH, acc, 0), q, lane, half,
                     stg_base + e * 4096);
      } else if (kind_gather_b(KIND)) {  // DW*: 4 warps cover both halves (M or column)
        for (int hf = 0; hf < 2; ++hf) {
          const uint32_t col0 = tm_col(a.BN, a.MH, acc, a.MH == 2 ? hf : 0);
          epilogue<KIND, kSplit>(a, ti, tmem + lanes + col0, row, hf, dg_xchg);
        }
      } else {
        const uint32_t col0 = tm_col(a.BN, a.MH, acc, a.MH == 2 ? half : 0);
        epilogue<KIND, kSplit>(a, ti, tmem + lanes + col0, row, half, dg_xchg);
      }
      tc_fence_before();
      __syncwarp();
      if (tr && threadIdx.x == 4 * 32) tr[3] += (unsigned long long)(clock64() - te0);
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == n_acc) { acc = 0; aphase ^= 1; }
    }
    if (KIND == K_DAT && lane == 0) bulk_wait<0>();  // dA tiles written before exit
  }
  // last DW host kernel: every warp of the CTA, its own role finished, takes
  // the grad-input combine tokens nobody has claimed yet
  if (kind_gather_b(KIND) && a.cb_ctr) {
    __syncwarp();
    side_combine_run(a, lane, side, nullptr, 0, !a.cb_drain);  // not the last host: own token only
  }
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[6] += (unsigned long long)(clock64() - t_start);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// =========================================== CTA-pair gather GEMMs (FWD1 / DA)
// A pair tile (256 bucket rows of one block, the tile list of the 1-CTA
// kernel) runs on a 2-CTA cluster with M = 256 cta_group::2 MMAs: CTA r
// gathers rows [128r, 128r+128) and holds the N-half r of B (FWD1 SwiGLU: the
// gate rows in CTA 0, the up rows in CTA 1), and its TMEM receives its 128
// rows x N.  Two accumulators fit (N <= 256), so the epilogue of tile i
// overlaps the MMAs of tile i+1 -- the 1-CTA kernel needs all 512 columns for
// its 256-row tile and cannot overlap.  A stage is 32 KB per CTA (6 stages).
// Producers fill their own CTA's stage and arrive on their own `full`
// barrier; the peer's warp 1 relays its completed stage to the leader
// (proxy fence + remote arrive), whose `full` counts that relay.  `empty` /
// `tfull` are multicast by tcgen05.commit; `tempty` (leader) counts both
// CTAs' epilogue warps.
constexpr int kPairRows = 64;  // rows per CTA-stage gathered by TMA gather4 (rest: cp.async)
constexpr int kPairStage = 32768;

template <int KIND>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    tc_pair_gather_kernel(const __grid_constant__ TcArgs a, int n_stages) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + n_stages * kPairStage);
  uint64_t* empty = full + n_stages;
  uint64_t* tfull = empty + n_stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  float* dg_xchg = (float*)(tmem_slot + 4);  // [128] DA half-row exchange

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int nh = a.BN / 2;  // B rows (N columns) held by this CTA
  // warp roles: 0, 2, 3 TMA gather4 (+ B); 1 MMA / relay; epilogue 4..4+nepi-1;
  // cp.async the warps after it (a.pair_cpw = 4: epilogue 4..11, cp.async 12..15;
  // 8: epilogue 4..7 on whole rows, cp.async 8..15)
  const int ncpw = a.pair_cpw == 8 ? 8 : 4;
  const int nepi = 12 - ncpw;
  const int ncp = ncpw * 32;
  const int cp_w0 = 16 - ncpw;
  if (threadIdx.x == 0) {
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(&full[s], kTmaGatherWarps + ncp + (leader ? 1 : 0));
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * nepi);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&a.ta);
    tma_prefetch_desc(&a.tb);
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  pdl_wait();  // PDL: barriers / TMEM set up; now the predecessor's outputs are visible
  // successor launches as this grid's CTAs exit (an early trigger measured slower)
  const uint32_t tmem = *tmem_slot;
  const int ntiles = a.unit_offsets[a.G + 1] * a.nu;  // pair tiles x unit tiles
  unsigned long long* tr = a.trace ? a.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
  const long long t_start = clock64();

  // this CTA's 128-row half of pair tile `tile`
  auto my_half = [&](int tile) {
    TileInfo ti = decode<KIND>(a, tile);
    ti.n_valid -= (int)rank * 128;
    ti.prow0 += rank * 128;
    ti.pos0 += rank * 128;
    ti.rows_pad -= (int)rank * 128;
    return ti;
  };

  if (warp == 0 || warp == 2 || warp == 3) {
    // --------- TMA gather4 of rows [0, kPairRows); warp 0 lane 0 also loads B
    const int p = warp == 0 ? 0 : warp - 1;
    const int c = lane * kTmaGatherWarps + p;
    const int n_calls = a.pair_rows / 4;
    const bool has_call = c < n_calls;
    const int my_calls = n_calls > p ? (n_calls - p + kTmaGatherWarps - 1) / kTmaGatherWarps : 0;
    const uint32_t tx = (uint32_t)my_calls * 512u + (p == 0 ? (uint32_t)nh * 128u : 0u);
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = cid; tile < ntiles; tile += ncl) {
      const TileInfo ti = my_half(tile);
      int rr[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = 4 * c + i;
        rr[i] = (has_call && r < ti.n_valid) ? a.r.bucket_token[ti.pos0 + r] : (int)a.T;
      }
      if (KIND == K_DA) {  // warm L2 with this half's Z stash rows (read by the epilogue)
        const int zrow = a.mp * a.bw * 2;
        for (int r = lane * kTmaGatherWarps + p; r < 128 && r < ti.rows_pad; r += 32 * kTmaGatherWarps)
          prefetch_l2_bulk((const uint8_t*)a.aux + (ti.prow0 + r) * zrow, zrow);
      }
      const int u0 = ti.b * a.bw + ti.ut * a.bn_u;  // first unit of the tile
      const int brow = (KIND == K_FWD1 && a.mp == 2) ? (int)rank * a.D + u0 : u0 + (int)rank * nh;
      for (int kb = 0; kb < ti.nkb; ++kb) {
        if (lane == 0) {
          twait(&empty[stage], phase ^ 1, (tr && warp == 0) ? tr : nullptr, 4);
          mbar_arrive_expect_tx(&full[stage], tx);
        }
        __syncwarp();
        uint8_t* sA = smem + stage * kPairStage;
        if (p == 0 && lane == 0) tma_load_2d(sA + kABytes, &a.tb, &full[stage], kb * 64, brow);
        if (has_call) tma_gather4(sA + c * 512, &a.ta, &full[stage], kb * 64, rr[0], rr[1], rr[2], rr[3]);
        if (++stage == n_stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp >= cp_w0) {
    // ------------------------------- cp.async of rows [pair_rows, 128)
    const int t = threadIdx.x - cp_w0 * 32;  // 0..ncp-1
    const __nv_bfloat16* src = (const __nv_bfloat16*)a.aux2;
    const int ch = t & 7;
    const int pr = a.pair_rows;
    constexpr int kRowsPer = 8;  // upper bound (pair_rows = 0, 4 warps); rows pr + (t >> 3) + rstep i < 128
    const int rstep = ncp / 8;   // rows covered per i (16 or 32)
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = cid; tile < ntiles; tile += ncl) {
      const TileInfo ti = my_half(tile);
      int tok[kRowsPer];
#pragma unroll
      for (int i = 0; i < kRowsPer; ++i) {
        const int r = pr + (t >> 3) + rstep * i;
        tok[i] = (r < 128 && r < ti.n_valid) ? a.r.bucket_token[ti.pos0 + r] : -1;
      }
      for (int kb = 0; kb < ti.nkb; ++kb) {
        if (lane == 0) mbar_wait(&empty[stage], phase ^ 1);
        __syncwarp();
        const uint32_t sA = smem_u32(smem + stage * kPairStage);
#pragma unroll
        for (int i = 0; i < kRowsPer; ++i) {
          const int r = pr + (t >> 3) + rstep * i;
          if (r >= 128) break;
          const uint32_t dst = sA + r * 128 + ((ch ^ (r & 7)) << 4);
          const __nv_bfloat16* g = src + (int64_t)(tok[i] < 0 ? 0 : tok[i]) * a.d + kb * 64 + ch * 8;
          cp_async_16(dst, g, tok[i] < 0 ? 0u : 16u);
        }
        cp_async_arrive_noinc(&full[stage]);
        if (++stage == n_stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------- MMA issuer (leader)
      const uint32_t idesc = idesc_bf16(256, a.BN, false, false);
      const uint64_t adesc0 = sdesc_sw128(smem_u32(smem), 16, 1024);
      const uint64_t bdesc0 = sdesc_sw128(smem_u32(smem) + kABytes, 16, 1024);
      unsigned long long* trl = lane == 0 ? tr : nullptr;
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int tile = cid; tile < ntiles; tile += ncl) {
        const TileInfo ti = decode<KIND>(a, tile);
        twait(&tempty[acc], aphase ^ 1, trl, 1);
        tc_fence_after();
        if (trl) trl[7] += 1;
        const uint32_t dtm = tmem + acc * 256;
        if (a.mma_batch == 2) {
          // two K stages per wait / fence round: the per-stage issue overhead
          // (barrier wait, proxy + tcgen05 fences) halves against dA's 256-clock
          // (N = 128) stages
          for (int kb = 0; kb < ti.nkb; kb += 2) {
            const bool two = kb + 1 < ti.nkb;
            const int st1 = stage + 1 == n_stages ? 0 : stage + 1;
            const uint32_t ph1 = stage + 1 == n_stages ? phase ^ 1 : phase;
            twait(&full[stage], phase, trl, 0);
            if (two) twait(&full[st1], ph1, trl, 0);
            fence_proxy_async_smem();  // this CTA's cp.async rows -> async proxy
            tc_fence_after();
            if (elect_one()) {
              const uint64_t s0 = (uint64_t)((stage * kPairStage) >> 4);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16_pair(dtm, adesc0 + s0 + k * 2, bdesc0 + s0 + k * 2, idesc,
                              (kb != 0 || k != 0) ? 1u : 0u);
              mma_commit_pair(&empty[stage]);
              if (two) {
                const uint64_t s1 = (uint64_t)((st1 * kPairStage) >> 4);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  mma_bf16_pair(dtm, adesc0 + s1 + k * 2, bdesc0 + s1 + k * 2, idesc, 1u);
                mma_commit_pair(&empty[st1]);
              }
            }
            __syncwarp();
            stage = st1;
            phase = ph1;
            if (two && ++stage == n_stages) { stage = 0; phase ^= 1; }
          }
        } else {
        for (int kb = 0; kb < ti.nkb; ++kb) {
          twait(&full[stage], phase, trl, 0);
          fence_proxy_async_smem();  // this CTA's cp.async rows -> async proxy
          tc_fence_after();
          if (elect_one()) {
            const uint64_t soff = (uint64_t)((stage * kPairStage) >> 4);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_bf16_pair(dtm, adesc0 + soff + k * 2, bdesc0 + soff + k * 2, idesc,
                            (kb != 0 || k != 0) ? 1u : 0u);
            mma_commit_pair(&empty[stage]);
          }
          __syncwarp();
          if (++stage == n_stages) { stage = 0; phase ^= 1; }
        }
        }
        if (elect_one()) mma_commit_pair(&tfull[acc]);
        __syncwarp();
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
    } else if (lane == 0) {
      // ------------- relay (peer): this CTA's stage complete -> leader
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cid; tile < ntiles; tile += ncl) {
        const TileInfo ti = decode<KIND>(a, tile);
        for (int kb = 0; kb < ti.nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          fence_proxy_async_smem();  // cp.async rows -> async proxy before the leader's MMAs
          if (a.ablate == 9) mbar_arrive_remote(&full[stage], 0);
          else mbar_arrive_remote_relaxed(&full[stage], 0);
          if (++stage == n_stages) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 4 + nepi) {
    // ------------------------------------------- epilogue (both CTAs)
    const int e = warp - 4;
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int half = nepi == 4 ? -1 : e >> 2;  // column (unit) half of the tile; -1: whole rows
    int acc = 0;
    uint32_t aphase = 0;
    for (int tile = cid; tile < ntiles; tile += ncl) {
      const TileInfo ti = my_half(tile);
      twait(&tfull[acc], aphase, (tr && threadIdx.x == 4 * 32) ? tr : nullptr, 2);
      tc_fence_after();
      const long long te0 = clock64();
      if (ti.rows_pad > 0) {  // the pair's second m-tile may not exist: write nothing
        const uint32_t tacc = tmem + ((uint32_t)(q * 32) << 16) + acc * 256;
        // (compile-time activation variants of this call measured neutral at
        // every config: the epilogue is hidden behind the mainloop)
        epilogue<KIND>(a, ti, tacc, row, half, dg_xchg);
      }
      tc_fence_before();
      __syncwarp();
      if (tr && threadIdx.x == 4 * 32) tr[3] += (unsigned long long)(clock64() - te0);
      if (lane == 0) {
        if (leader) mbar_arrive(&tempty[acc]);
        else mbar_arrive_remote_relaxed(&tempty[acc], 0);  // its TMEM loads completed (wait::ld)
      }
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[6] = (unsigned long long)(clock64() - t_start);
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem);
  }
}

// ================================== fused FWD1 -> FWD2 on CTA pairs (a4 + a5)
// One pair tile (256 bucket rows of block b; CTA r owns rows [128r, 128r+128))
// runs FWD1 exactly as tc_pair_gather_kernel<FWD1> (gathered X rows, W1_b gate /
// up halves, M = 256 cta_group::2 MMAs into TMEM columns [0, 256)), then its
// epilogue writes the Z / H~ stash AND the tile's H~ rows into smem (sH, the
// K-major A operand of the second GEMM).  The second GEMM P = H~ W2_b runs in
// 128-column chunks (M = 256, N = 128, K = bw <= 128) into two alternating
// TMEM accumulators (columns [256, 384) / [384, 512)) whose bf16 rows the
// epilogue TMA-stores as the per-pair partial rows (Alg. 4 line 5; the combine
// sums them).  The leader interleaves the chunks of tile i with the FWD1
// stages of tile i+1, so the partial-row writes (the HBM-bound half of the
// separate FWD2 kernel) overlap the gather-bound FWD1 mainloop.
// Warps: 0, 2 TMA gather4 of rows [0, 64) (warp 0 lane 0 also W1_b); 3 lane 0
// W2_b chunk producer (both CTAs; bytes land on the leader's barrier); 1 MMA
// issuer (leader) / stage relay (peer); 4-11 epilogue; 12-15 cp.async rows
// [64, 128).  Epilogue order per tile: FWD1 epilogue, then its chunk drains --
// so tile i+1's FWD1 epilogue (which overwrites sH) starts only after every
// chunk MMA of tile i has completed (their t2full commits).
constexpr int kMlpGatherWarps = 2;  // warps 0, 2
constexpr int kMlpW2Slots = 2;      // W2_b chunk ring (16 KB per CTA each)
constexpr int kMlpChunkN = 128;     // N of one second-GEMM chunk (64 columns per CTA)

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    tc_pair_mlp_kernel(const __grid_constant__ TcArgs a, int n_stages) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sH = smem + n_stages * kPairStage;                 // 2 k-blocks x 16 KB
  uint8_t* sW2 = sH + 32768;                                   // kMlpW2Slots x 16 KB
  uint8_t* stg_base = sW2 + kMlpW2Slots * 16384;               // kEpiWarps x 4 KB (TMA-store staging)
  uint64_t* full = (uint64_t*)(stg_base + kEpiWarps * 4096);
  uint64_t* empty = full + n_stages;
  uint64_t* w2full = empty + n_stages;
  uint64_t* w2empty = w2full + kMlpW2Slots;
  // TMEM: two 256-column buffers used in turn by the tiles of this cluster (tile
  // n -> buffer n & 1): FWD1 accumulates there, and after its epilogue the same
  // buffer's halves [0, 128) / [128, 256) take the tile's second-GEMM chunks
  // (chunk c -> half c & 1) -- so the FWD1 of tile n+1 (other buffer) overlaps
  // the FWD1 epilogue of tile n.
  uint64_t* t1full = w2empty + kMlpW2Slots;   // [2] FWD1 accumulator of buffer x complete
  uint64_t* hready = t1full + 2;              // FWD1 epilogue done (sH written, buffer read)
  uint64_t* t2full = hready + 1;              // [2][2] chunk accumulator (buffer, half) complete
  uint64_t* t2empty = t2full + 4;             // [2][2] chunk accumulator drained
  uint32_t* tmem_slot = (uint32_t*)(t2empty + 4);
  float* dg_xchg = (float*)(tmem_slot + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int nh = a.BN / 2;                         // FWD1 B rows held by this CTA
  const int nchunks = (a.d + kMlpChunkN - 1) / kMlpChunkN;
  const int kb2 = (a.bw + 63) / 64;                // K blocks of the second GEMM (<= 2)
  if (threadIdx.x == 0) {
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(&full[s], kMlpGatherWarps + kCpThreadsA + (leader ? 1 : 0));
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < kMlpW2Slots; ++i) {
      mbar_init(&w2full[i], 1);
      mbar_init(&w2empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) mbar_init(&t1full[i], 1);
    mbar_init(hready, 2 * kEpiWarps);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&t2full[i], 1);
      mbar_init(&t2empty[i], 2 * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&a.ta);
    tma_prefetch_desc(&a.tb);
    tma_prefetch_desc(&a.tw2);
    tma_prefetch_desc(&a.tc);
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  pdl_wait();
  const uint32_t tmem = *tmem_slot;
  const int ntiles = a.unit_offsets[a.G + 1];  // pair tiles (nu == 1)
  // SPT_FFN_TRACE slots: 0 MMA wait stage, 1 MMA wait acc1 / H~, 2 epi wait acc1,
  // 3 epi wait chunk, 4 MMA wait W2 chunk, 5 MMA wait acc2, 6 total, 7 epi drain busy
  unsigned long long* tr = a.trace ? a.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
  const long long t_start = clock64();

  auto my_half = [&](int tile) {
    TileInfo ti = decode<K_FWD1>(a, tile);
    ti.n_valid -= (int)rank * 128;
    ti.prow0 += rank * 128;
    ti.pos0 += rank * 128;
    ti.rows_pad -= (int)rank * 128;
    return ti;
  };

  if (warp == 0 || warp == 2) {
    // --------- TMA gather4 of rows [0, kPairRows); warp 0 lane 0 also loads W1_b
    const int p = warp == 0 ? 0 : 1;
    const int c = lane * kMlpGatherWarps + p;
    constexpr int n_calls = kPairRows / 4;
    const bool has_call = c < n_calls;
    const int my_calls = n_calls > p ? (n_calls - p + kMlpGatherWarps - 1) / kMlpGatherWarps : 0;
    const uint32_t tx = (uint32_t)my_calls * 512u + (p == 0 ? (uint32_t)nh * 128u : 0u);
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = cid; tile < ntiles; tile += ncl) {
      const TileInfo ti = my_half(tile);
      int rr[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = 4 * c + i;
        rr[i] = (has_call && r < ti.n_valid) ? a.r.bucket_token[ti.pos0 + r] : (int)a.T;
      }
      const int u0 = ti.b * a.bw;
      const int brow = a.mp == 2 ? (int)rank * a.D + u0 : u0 + (int)rank * nh;
      for (int kb = 0; kb < ti.nkb; ++kb) {
        if (lane == 0) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], tx);
        }
        __syncwarp();
        uint8_t* sA = smem + stage * kPairStage;
        if (p == 0 && lane == 0) tma_load_2d(sA + kABytes, &a.tb, &full[stage], kb * 64, brow);
        if (has_call) tma_gather4(sA + c * 512, &a.ta, &full[stage], kb * 64, rr[0], rr[1], rr[2], rr[3]);
        if (++stage == n_stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 3) {
    // ------------- W2_b chunk producer (both CTAs): this CTA's 64 columns
    if (lane == 0) {
      int slot = 0;
      uint32_t wph = 0;
      for (int tile = cid; tile < ntiles; tile += ncl) {
        const TileInfo ti = decode<K_FWD1>(a, tile);
        for (int ch = 0; ch < nchunks; ++ch) {
          mbar_wait(&w2empty[slot], wph ^ 1);
          if (leader) mbar_arrive_expect_tx(&w2full[slot], 2u * (uint32_t)kb2 * 8192u);
          for (int k2 = 0; k2 < kb2; ++k2)
            tma_load_2d_pair(sW2 + slot * 16384 + k2 * 8192, &a.tw2, &w2full[slot],
                             ch * kMlpChunkN + (int)rank * 64, ti.b * a.bw + k2 * 64);
          if (++slot == kMlpW2Slots) { slot = 0; wph ^= 1; }
        }
      }
    }
  } else if (warp >= 12) {
    // ------------------------------- cp.async of rows [kPairRows, 128)
    const int t = threadIdx.x - 12 * 32;  // 0..127
    const __nv_bfloat16* src = (const __nv_bfloat16*)a.aux2;
    const int ch = t & 7;
    constexpr int kRowsPer = (128 - kPairRows) * 8 / kCpThreadsA;  // 4
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = cid; tile < ntiles; tile += ncl) {
      const TileInfo ti = my_half(tile);
      int tok[kRowsPer];
#pragma unroll
      for (int i = 0; i < kRowsPer; ++i) {
        const int r = kPairRows + (t >> 3) + 16 * i;
        tok[i] = r < ti.n_valid ? a.r.bucket_token[ti.pos0 + r] : -1;
      }
      for (int kb = 0; kb < ti.nkb; ++kb) {
        if (lane == 0) mbar_wait(&empty[stage], phase ^ 1);
        __syncwarp();
        const uint32_t sA = smem_u32(smem + stage * kPairStage);
#pragma unroll
        for (int i = 0; i < kRowsPer; ++i) {
          const int r = kPairRows + (t >> 3) + 16 * i;
          const uint32_t dst = sA + r * 128 + ((ch ^ (r & 7)) << 4);
          const __nv_bfloat16* g = src + (int64_t)(tok[i] < 0 ? 0 : tok[i]) * a.d + kb * 64 + ch * 8;
          cp_async_16(dst, g, tok[i] < 0 ? 0u : 16u);
        }
        cp_async_arrive_noinc(&full[stage]);
        if (++stage == n_stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------- MMA issuer (leader)
      const uint32_t idesc1 = idesc_bf16(256, a.BN, false, false);
      const uint32_t idesc2 = idesc_bf16(256, kMlpChunkN, false, true);
      const uint64_t adesc0 = sdesc_sw128(smem_u32(smem), 16, 1024);
      const uint64_t bdesc0 = sdesc_sw128(smem_u32(smem) + kABytes, 16, 1024);
      const uint64_t hdesc0 = sdesc_sw128(smem_u32(sH), 16, 1024);
      const uint64_t wdesc0 = sdesc_sw128(smem_u32(sW2), 8192, 1024);
      unsigned long long* trl = lane == 0 ? tr : nullptr;
      int stage = 0, slot = 0;
      uint32_t phase = 0, wph = 0, hph = 0;
      int chunk = 0, px = 0;  // next chunk of the previous tile (buffer px)
      // chunk `chunk` of the previous tile into buffer px, half chunk & 1: waits its
      // W2_b chunk and the drain of chunk - 2 (the same half; its completion index
      // on that barrier is chunk / 2 - 1 within the tile, 16 per tile -> parity)
      auto issue_chunk = [&]() {
        const int h = chunk & 1;
        twait(&w2full[slot], wph, trl, 4);
        if (chunk >= 2) twait(&t2empty[px * 2 + h], ((chunk >> 1) - 1) & 1, trl, 5);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t dtm = tmem + px * 256 + h * kMlpChunkN;
          const uint64_t wd = wdesc0 + (uint64_t)((slot * 16384) >> 4);
          for (int k2 = 0; k2 < kb2; ++k2) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_bf16_pair(dtm, hdesc0 + (uint64_t)((k2 * 16384) >> 4) + k * 2,
                            wd + (uint64_t)((k2 * 8192) >> 4) + k * 128, idesc2,
                            (k2 != 0 || k != 0) ? 1u : 0u);
          }
          mma_commit_pair(&w2empty[slot]);
          mma_commit_pair(&t2full[px * 2 + h]);
        }
        __syncwarp();
        if (++slot == kMlpW2Slots) { slot = 0; wph ^= 1; }
        ++chunk;
      };
      bool prev = false;
      int n = 0;  // this cluster's tile sequence number (buffer n & 1)
      for (int tile = cid;; tile += ncl, ++n) {
        const bool cur = tile < ntiles;
        if (!cur && !prev) break;
        const int x = n & 1;
        bool started = false;  // the previous tile's FWD1 epilogue is done (hready)
        int kb0 = 0;           // the stage at which it was seen
        chunk = 0;
        px = x ^ 1;
        if (cur) {
          const TileInfo ti = decode<K_FWD1>(a, tile);
          if (n >= 2) {  // buffer x: every chunk drain of tile n - 2 (the last of each half)
            twait(&t2empty[x * 2 + 0], 1u, trl, 1);
            twait(&t2empty[x * 2 + 1], 1u, trl, 1);
          }
          tc_fence_after();
          for (int kb = 0; kb < ti.nkb; ++kb) {
            if (prev && chunk < nchunks) {
              if (!started && mbar_test(hready, hph)) {
                started = true;
                kb0 = kb;
                hph ^= 1;
                tc_fence_after();
              }
              // spread the chunks evenly over the stages left once started
              if (started && chunk * (ti.nkb - kb0) <= (kb - kb0) * nchunks) issue_chunk();
            }
            twait(&full[stage], phase, trl, 0);
            fence_proxy_async_smem();  // this CTA's cp.async rows -> async proxy
            tc_fence_after();
            if (elect_one()) {
              const uint64_t soff = (uint64_t)((stage * kPairStage) >> 4);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16_pair(tmem + x * 256, adesc0 + soff + k * 2, bdesc0 + soff + k * 2, idesc1,
                              (kb != 0 || k != 0) ? 1u : 0u);
              mma_commit_pair(&empty[stage]);
            }
            __syncwarp();
            if (++stage == n_stages) { stage = 0; phase ^= 1; }
          }
          if (elect_one()) mma_commit_pair(&t1full[x]);
          __syncwarp();
        }
        if (prev && chunk < nchunks) {
          if (!started) {
            twait(hready, hph, trl, 1);
            hph ^= 1;
            tc_fence_after();
          }
          while (chunk < nchunks) issue_chunk();
        }
        prev = cur;
      }
    } else if (lane == 0) {
      // ------------- relay (peer): this CTA's stage complete -> leader
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cid; tile < ntiles; tile += ncl) {
        const TileInfo ti = decode<K_FWD1>(a, tile);
        for (int kb = 0; kb < ti.nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          fence_proxy_async_smem();
          mbar_arrive_remote_relaxed(&full[stage], 0);
          if (++stage == n_stages) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 4 + kEpiWarps) {
    // ------------------------------------------- epilogue (both CTAs)
    const int e = warp - 4;
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int half = e >> 2;  // FWD1: unit half (= k-block of sH); chunks: 64-column half
    uint8_t* stg = stg_base + e * 4096;
    int n = 0;
    for (int tile = cid; tile < ntiles; tile += ncl, ++n) {
      const TileInfo ti = my_half(tile);
      const int x = n & 1;
      // FWD1: Z / H~ stash + the smem H~ tile (sH is free: every chunk MMA of the
      // previous tile completed before this warp drained its last chunk)
      unsigned long long* tre = (tr && threadIdx.x == 4 * 32) ? tr : nullptr;
      twait(&t1full[x], (n >> 1) & 1, tre, 2);
      tc_fence_after();
      if (ti.rows_pad > 0)
        epilogue<K_FWD1>(a, ti, tmem + ((uint32_t)(q * 32) << 16) + x * 256, row, half, dg_xchg, sH);
      fence_proxy_async_smem();  // sH (generic writes) -> the async proxy of the chunk MMAs
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(hready);
        else mbar_arrive_remote_relaxed(hready, 0);
      }
      // second GEMM: this tile's partial rows, chunk by chunk
      for (int ch = 0; ch < nchunks; ++ch) {
        const int h = ch & 1;
        twait(&t2full[x * 2 + h], (ch >> 1) & 1, tre, 3);
        const long long td0 = tre ? clock64() : 0;
        tc_fence_after();
        const int col0 = ch * kMlpChunkN + half * 64;
        uint32_t v[64];
        tmem_ld64(tmem + ((uint32_t)(q * 32) << 16) + x * 256 + h * kMlpChunkN + half * 64, v, true);
        if (ti.rows_pad > 0 && col0 < a.d) {
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 w = make_uint4(pack_bf16(__uint_as_float(v[8 * c + 0]), __uint_as_float(v[8 * c + 1])),
                                       pack_bf16(__uint_as_float(v[8 * c + 2]), __uint_as_float(v[8 * c + 3])),
                                       pack_bf16(__uint_as_float(v[8 * c + 4]), __uint_as_float(v[8 * c + 5])),
                                       pack_bf16(__uint_as_float(v[8 * c + 6]), __uint_as_float(v[8 * c + 7])));
            *reinterpret_cast<uint4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) = w;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&a.tc, stg, col0, (int)(ti.prow0 + q * 32));
            bulk_commit();
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader) mbar_arrive(&t2empty[x * 2 + h]);
          else mbar_arrive_remote_relaxed(&t2empty[x * 2 + h], 0);
        }
        if (tre) tre[7] += (unsigned long long)(clock64() - td0);
      }
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[6] = (unsigned long long)(clock64() - t_start);
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem);
  }
}

// ============================================= CTA-pair weight-resident GEMMs
// FWD2 / DX on CTA pairs (cta_group::2): a unit (block b, 256 output columns,
// its m-tiles) runs on a 2-CTA cluster; CTA r computes m-tiles 2p + r, keeps
// the N-half [r*128, r*128+128) of the weight slab resident (half the smem of
// the 1-CTA kernel, so the A ring is twice as deep) and the leader issues
// M = 256, N = 256 MMAs.  Barriers: stage / slab "full" live in the leader
// (both CTAs' TMA bytes land there), "empty" / "tfull" are multicast to both
// CTAs by tcgen05.commit, "tempty" lives in the leader and counts the epilogue
// warps of both CTAs (the peer arrives remotely).
template <int KIND>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    tc_pair_kernel(const __grid_constant__ TcArgs a, int n_stages) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int kbu = KIND == K_FWD2 ? (a.bw + 63) / 64 : (a.mp * a.bw + 63) / 64;  // K stages
  uint8_t* sBres = smem;                       // kbu x 16 KB (this CTA's 128 columns)
  uint8_t* ring = smem + kbu * 16384;          // n_stages x 16 KB A stages
  uint64_t* full = (uint64_t*)(ring + n_stages * kABytes);
  uint64_t* empty = full + n_stages;
  uint64_t* tfull = empty + n_stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* bres_full = tempty + 2;
  uint64_t* bres_empty = bres_full + 1;
  uint32_t* tmem_slot = (uint32_t*)(bres_empty + 1);
  uint8_t* stg_base = (uint8_t*)(((uintptr_t)(tmem_slot + 4) + 1023) & ~(uintptr_t)1023);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * kEpiWarps);
    }
    mbar_init(bres_full, 1);
    mbar_init(bres_empty, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised before any cross-CTA traffic
  tc_fence_after();
  pdl_wait();  // PDL: barriers / TMEM set up; now the predecessor's outputs are visible
  // successor launches as this grid's CTAs exit (an early trigger measured slower)
  const uint32_t tmem = *tmem_slot;
  const int nunits = a.unit_offsets[a.G];
  unsigned long long* tr = a.trace ? a.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
  const long long t_start = clock64();

  if (warp == 0) {
    if (lane == 0) {  // producer (both CTAs): own slab half + own m-tile rows
      int stage = 0;
      uint32_t phase = 0, uph = 0;
      for (int u = cid; u < nunits; u += ncl) {
        const UnitInfo ui = decode_unit(a, u);
        twait(bres_empty, uph ^ 1, tr, 4);
        if (leader) mbar_arrive_expect_tx(bres_full, 2u * kbu * 16384u);
        for (int kb = 0; kb < kbu; ++kb) {
          int krow;
          if (KIND == K_FWD2) krow = ui.b * a.bw + kb * 64;
          else krow = kb * 64 < a.bw ? ui.b * a.bw + kb * 64 : a.D + ui.b * a.bw + (kb * 64 - a.bw);
#pragma unroll
          for (int j = 0; j < 2; ++j)
            tma_load_2d_pair(sBres + kb * 16384 + j * 8192, &a.tb, bres_full,
                             ui.nt * 256 + (int)rank * 128 + j * 64, krow);
        }
        uph ^= 1;
        for (int mt = ui.mt0; mt < ui.mt1; mt += 2) {
          const int64_t prow0 = decode_mtile<KIND>(a, ui, mt + (int)rank).prow0;
          for (int kb = 0; kb < kbu; ++kb) {
            twait(&empty[stage], phase ^ 1, tr, 4);
            if (leader) mbar_arrive_expect_tx(&full[stage], 2u * kABytes);
            tma_load_2d_pair(ring + stage * kABytes, &a.ta, &full[stage], kb * 64, (int)prow0);
            if (++stage == n_stages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // MMA issuer (leader only; whole warp, one elected lane issues)
      const uint32_t idesc = idesc_bf16(256, 256, false, true);
      const uint64_t adesc0 = sdesc_sw128(smem_u32(ring), 16, 1024);
      const uint64_t bdesc0 = sdesc_sw128(smem_u32(sBres), 8192, 1024);
      unsigned long long* trl = lane == 0 ? tr : nullptr;
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0, uph = 0;
      for (int u = cid; u < nunits; u += ncl) {
        const UnitInfo ui = decode_unit(a, u);
        twait(bres_full, uph, trl, 5);
        uph ^= 1;
        for (int mt = ui.mt0; mt < ui.mt1; mt += 2) {
          twait(&tempty[acc], aphase ^ 1, trl, 1);
          tc_fence_after();
          if (trl) trl[7] += 1;
          const uint32_t dtm = tmem + acc * 256;
          for (int kb = 0; kb < kbu; ++kb) {
            twait(&full[stage], phase, trl, 0);
            tc_fence_after();
            if (elect_one()) {
              const uint64_t ad = adesc0 + (uint64_t)((stage * kABytes) >> 4);
              const uint64_t bd = bdesc0 + (uint64_t)((kb * 16384) >> 4);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16_pair(dtm, ad + k * 2, bd + k * 128, idesc, (kb != 0 || k != 0) ? 1u : 0u);
              mma_commit_pair(&empty[stage]);
            }
            __syncwarp();
            if (++stage == n_stages) { stage = 0; phase ^= 1; }
          }
          if (elect_one()) mma_commit_pair(&tfull[acc]);
          __syncwarp();
          if (++acc == 2) { acc = 0; aphase ^= 1; }
        }
        if (elect_one()) mma_commit_pair(bres_empty);
        __syncwarp();
      }
    }
  } else if (warp >= 4 && warp < 4 + kEpiWarps) {  // epilogue (both CTAs): own m-tile
    const int e = warp - 4;
    const int q = warp & 3;
    const int half = e >> 2;
    int acc = 0, stg_i = 0;
    uint32_t aphase = 0;
    for (int u = cid; u < nunits; u += ncl) {
      const UnitInfo ui = decode_unit(a, u);
      for (int mt = ui.mt0; mt < ui.mt1; mt += 2) {
        const int my_mt = mt + (int)rank;
        twait(&tfull[acc], aphase, (tr && threadIdx.x == 4 * 32) ? tr : nullptr, 2);
        tc_fence_after();
        const long long te0 = clock64();
        if (my_mt < ui.mt1) {  // the pair's second m-tile may not exist
          const TileInfo ti = decode_mtile<KIND>(a, ui, my_mt);
          epilogue_tma_store(a, ti, tmem + ((uint32_t)(q * 32) << 16) + acc * 256, q, lane, half,
                               stg_base + e * a.n_stg * 4096, stg_i);
        }
        tc_fence_before();
        __syncwarp();
        if (tr && threadIdx.x == 4 * 32) tr[3] += (unsigned long long)(clock64() - te0);
        if (lane == 0) {
          if (leader) mbar_arrive(&tempty[acc]);
          else mbar_arrive_remote_relaxed(&tempty[acc], 0);  // its TMEM loads completed (wait::ld)
        }
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[6] = (unsigned long long)(clock64() - t_start);
  cluster_sync();  // the leader's MMAs into this CTA's TMEM / smem are done
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem);
  }
}

// ====================================================================== host
static bool debug_sync() {  // SPT_FFN_DEBUG_SYNC=1: synchronise + report after each GEMM launch
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPT_FFN_DEBUG_SYNC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// Per-device caches: kernel attributes, SM counts and occupancy are
// properties of the current device's context, so every cache is an array
// indexed by the device id, with atomic slots (first calls may race; the work
// they repeat is idempotent).
constexpr int kMaxDev = 64;
static int cur_dev() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) dev = 0;
  return dev;
}
static int num_sms() {
  static std::atomic<int> cache[kMaxDev];
  const int dev = cur_dev();
  int n = cache[dev].load(std::memory_order_relaxed);
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
template <typename K>
static cudaError_t set_smem_attr_once(K* kern, std::atomic<bool>* done) {
  const int dev = cur_dev();
  if (done[dev].load(std::memory_order_acquire)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return e;
  }
  done[dev].store(true, std::memory_order_release);
  return cudaSuccess;
}
// co-resident 2-CTA clusters of a cluster kernel at `smem` bytes (GPCs may hold
// odd SM counts), once per (kernel, device)
template <typename K>
static int max_pair_clusters(K* kern, int smem, std::atomic<int>* cache) {
  const int dev = cur_dev();
  int mc = cache[dev].load(std::memory_order_acquire);
  if (mc > 0) return mc;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(num_sms());
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = 2;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  if (cudaOccupancyMaxActiveClusters(&mc, kern, &cfg) != cudaSuccess || mc <= 0) {
    cudaGetLastError();
    mc = num_sms() / 2;
  }
  cache[dev].store(mc, std::memory_order_release);
  return mc;
}
static int gemm_sms() { return num_sms(); }

// SPT_FFN_TRACE=1: per-CTA role cycle counters (slots: kTraceSlots above),
// summed over the grid and printed after a synchronising readback
static unsigned long long* g_trace_buf = nullptr;
static bool trace_begin(TcArgs& a, cudaStream_t s) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SPT_FFN_TRACE");
    on = (e && e[0] == '1') ? 1 : 0;
    if (on) cudaMalloc(&g_trace_buf, 1024 * kTraceSlots * sizeof(unsigned long long));
  }
  if (!on) return false;
  cudaMemsetAsync(g_trace_buf, 0, 1024 * kTraceSlots * sizeof(unsigned long long), s);
  a.trace = g_trace_buf;
  return true;
}
static void trace_report(TcArgs& a, const char* name, int grid, cudaStream_t s) {
  unsigned long long h[1024 * kTraceSlots];
  cudaMemcpyAsync(h, g_trace_buf, sizeof(unsigned long long) * grid * kTraceSlots,
                  cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  double sum[kTraceSlots] = {0};
  for (int b = 0; b < grid; ++b)
    for (int i = 0; i < kTraceSlots; ++i) sum[i] += (double)h[b * kTraceSlots + i];
  const double tot = sum[6] > 0 ? sum[6] : 1;
  fprintf(stderr,
          "[spt-trace] %-16s tiles/cta %.1f | MMA wait full %.0f%% wait tempty %.0f%% slab/fences "
          "%.0f%% | epi wait %.0f%% busy %.0f%% | tma prod wait empty %.0f%% | cta cycles %.0f\n",
          name, sum[7] / grid, 100 * sum[0] / tot, 100 * sum[1] / tot, 100 * sum[5] / tot,
          100 * sum[2] / tot, 100 * sum[3] / tot, 100 * sum[4] / tot, tot / grid);
  a.trace = nullptr;
}

static int nstg_fwd2() {
  static int v = 0;
  if (!v) {
    const char* e = getenv("SPT_FFN_NSTG");
    v = e ? atoi(e) : 3;  // measured: FWD2 1.21 ms at 3 vs 1.31 ms at 2 (LLaMA-scale)
    if (v < 1 || v > 3) v = 3;
  }
  return v;
}

template <int KIND>
static cudaError_t launch(TcArgs& a, int tiles_upper, cudaStream_t s) {
  const int bst = (b_bytes(KIND, a.BN, a.kstream) + 1023) & ~1023;
  const int sst = kABytes * kind_bk(KIND) / 64 * a.MH + bst;
  const int extra = 1024 + 256 + 512;  // alignment slack + barriers + DA exchange
  const bool resident = kind_bres(KIND) && !a.kstream;
  // weight-resident kinds: the slab (K stages x 32 KB) is carved before the A ring
  const int slab = resident
                       ? (KIND == K_FWD2 ? (a.bw + 63) / 64 : (a.mp * a.bw + 63) / 64) * 32768
                       : 0;
  // FWD2 keeps 2 staging buffers per epilogue warp, DX (128 KB slab) keeps 1
  // (FWD2, K = bw <= 128: a 4-stage A ring covers two m-tiles, the rest of smem
  // keeps more partial-output stores in flight; SPT_FFN_NSTG overrides)
  if (resident) a.n_stg = slab > 65536 ? 1 : nstg_fwd2();
  const int stg = resident ? kEpiWarps * a.n_stg * 4096 + 1024
                           : (KIND == K_DAT ? kEpiWarps * 4096 + 1024 : 0);
  int stages = std::min(kind_bres(KIND) || kind_bk(KIND) < 64 ? 8 : 6,
                        (227 * 1024 - extra - slab - stg) / sst);
  const int smem = slab + stages * sst + extra + stg;
  // split (fp32 on tensor cores): its own instantiation, so the hi / lo epilogue
  // code costs the bf16 kernels no registers
  static std::atomic<bool> attr_set[2][kMaxDev];
  auto* kern = a.split ? tc_gemm_kernel<KIND, true> : tc_gemm_kernel<KIND, false>;
  if (cudaError_t e = set_smem_attr_once(kern, attr_set[a.split ? 1 : 0])) return e;
  const int grid = std::max(1, std::min(tiles_upper, gemm_sms()));
  static const char* kNames[] = {"tc_router", "tc_fwd1_gate_up", "tc_fwd2_down", "tc_bwd_dA",
                                 "tc_bwd_dX", "tc_bwd_dW1", "tc_bwd_dW2", "tc_bwd_dWR",
                                 "tc_bwd_dAT", "tc_bwd_dXR"};
  const bool trace_on = trace_begin(a, s);
  prof_begin(kNames[KIND], s);
  cudaError_t le = launch_pdl(kern, dim3(grid), dim3(kThreads), smem, s, a, stages);
  prof_end(s);
  if (trace_on) trace_report(a, kNames[KIND], grid, s);
  count_launch();
  cudaError_t e = le != cudaSuccess ? le : cudaGetLastError();
  if (debug_sync()) {
    e = cudaStreamSynchronize(s);
    fprintf(stderr, "[spt] tc kind %d grid %d stages %d smem %d BN %d MH %d: %s\n", KIND, grid,
            stages, smem, a.BN, a.MH, cudaGetErrorString(e));
  }
  return e;
}

// CTA-pair weight-resident kernel: default for DX (K = m'bw = 256: the
// 1-CTA slab leaves a 4-stage A ring, measured 1.45 vs 1.79 ms), not for FWD2
// (K = bw = 128: bound by the partial-output writes, where the pair's coupled
// epilogues lose, 1.54 vs 1.31 ms).  SPT_FFN_PAIR=0: neither, =1: both.
static bool use_pair(int kind) {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("SPT_FFN_PAIR");
    v = e ? (e[0] == '1' ? 1 : 0) : -1;
  }
  return v == 1 || (v == -1 && kind == K_DX);
}
template <int KIND>
static cudaError_t launch_pair(TcArgs& a, int units_upper, cudaStream_t s) {
  const int kbu = KIND == K_FWD2 ? (a.bw + 63) / 64 : (a.mp * a.bw + 63) / 64;
  const int slab = kbu * 16384;  // this CTA's 128-column half of the slab
  const int extra = 1024 + 256;
  {  // SPT_FFN_PAIR_NSTG overrides the staging depth of the pair kernel
    static int v = -1;
    if (v < 0) {
      const char* e = getenv("SPT_FFN_PAIR_NSTG");
      v = e ? atoi(e) : 0;
    }
    a.n_stg = (v >= 1 && v <= 3) ? v : (slab > 32768 ? 1 : 2);
  }
  const int stg = kEpiWarps * a.n_stg * 4096 + 1024;
  const int stages = std::min(8, (227 * 1024 - extra - slab - stg) / kABytes);
  const int smem = slab + stages * kABytes + extra + stg;
  static std::atomic<bool> attr_set[kMaxDev];
  static std::atomic<int> mc_cache[kMaxDev];
  if (cudaError_t e = set_smem_attr_once(tc_pair_kernel<KIND>, attr_set)) return e;
  const int max_clusters = max_pair_clusters(tc_pair_kernel<KIND>, smem, mc_cache);
  if (debug_sync()) fprintf(stderr, "[spt] pair kind %d: max active clusters %d\n", KIND, max_clusters);
  const int clusters = std::max(1, std::min(units_upper, max_clusters));
  const bool trace_on = trace_begin(a, s);
  const char* name = KIND == K_FWD2 ? "tc_fwd2_down" : "tc_bwd_dX";
  prof_begin(name, s);
  cudaError_t le = launch_pdl(tc_pair_kernel<KIND>, dim3(2 * clusters), dim3(kThreads), smem, s, a, stages);
  prof_end(s);
  if (trace_on) trace_report(a, name, 2 * clusters, s);
  count_launch();
  cudaError_t e = le != cudaSuccess ? le : cudaGetLastError();
  if (debug_sync()) {
    e = cudaStreamSynchronize(s);
    fprintf(stderr, "[spt] tc pair kind %d clusters %d stages %d smem %d: %s\n", KIND, clusters,
            stages, smem, cudaGetErrorString(e));
  }
  return e;
}

// SPT_FFN_PAIR_GATHER=0 selects the 1-CTA kernel for FWD1 / DA
static bool use_pair_gather() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPT_FFN_PAIR_GATHER");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
// pair gather kernel: N = BN split in halves of BN/2 B rows per CTA.  Used
// for N > 128 only: at N = 128 one M = 256 x N = 128 accumulator chain per CTA
// runs the tensor pipe at ~43 % and the 1-CTA kernel (two M halves in flight)
// wins (same-box A/B, LLaMA-scale dA: 1.18 vs 1.33 ms; OPT FWD1 114 vs 132 us),
// while at N = 256 the pair wins (LLaMA FWD1 1.31 vs 1.50 ms).
// N = 128 (dA at bw = 128) also maps onto pairs (B halves of 64 rows); measured
// before taking it by default (SPT_FFN_PAIR128=1)
static bool pair128() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPT_FFN_PAIR128");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}
static bool pair_gather_ok(int BN) {
  return (BN > 128 || (BN == 128 && pair128())) && BN <= 256 && BN % 32 == 0;
}

// rows of each 128-row CTA stage gathered by TMA gather4 (multiple of 4; the rest
// by the four cp.async warps).  Measured at LLaMA scale (FWD1 / dA ms): 32 rows
// 1.37 / 1.39, 40 1.38, 48 1.32-1.34 / 1.39-1.42, 56 1.38, 64 1.43-1.44 / 1.39-1.41,
// 80 1.49, 96 1.56, 128 1.82 / 1.37 -- FWD1 (N = 256: half the gathered bytes per
// MMA clock of dA) is best with the cp.async warps taking 80 of 128 rows; dA does
// not move (its bound is not the gather engines).  Default FWD1 48, dA 64;
// SPT_FFN_PAIR_ROWS overrides both.
static int pair_tma_rows(int kind) {
  static int v = -2;  // -2: not read yet, -1: default
  if (v == -2) {
    const char* e = getenv("SPT_FFN_PAIR_ROWS");
    v = e ? atoi(e) : -1;
    if (v < 0 || v > 128 || v % 4) v = -1;
  }
  if (v >= 0) return v;
  return kind == K_FWD1 ? 48 : kPairRows;
}
// cp.async warps of the pair gather kernel (SPT_FFN_PAIR_CPW=4|8).  FWD1 default 8
// (epilogue on 4 warps, whole rows): FWD1 1.36 -> 1.28-1.30 ms at LLaMA scale
// (the FWD1 epilogue was ~28 % busy on 8 warps; the gathered X rows are what
// the mainloop waits for).  The same split for the 1-CTA tokens-on-N dA
// measured neutral (1.24-1.25 ms) and was not kept.
static int pair_cp_warps(int kind) {
  static int v = -1;  // 0: default per kind
  if (v < 0) {
    const char* e = getenv("SPT_FFN_PAIR_CPW");
    v = (e && e[0] == '4') ? 4 : ((e && e[0] == '8') ? 8 : 0);
  }
  if (v) return v;
  // dA on wide blocks (the paper's G = 8: 256 units per tile, heavy per-row
  // epilogue) needs all 8 epilogue warps: 4 measured dA 0.80 -> 0.54 PFLOP/s
  return kind == K_FWD1 ? 8 : 4;
}
// K stages the pair kernel's MMA issuer consumes per wait / fence round
// (SPT_FFN_MMA_BATCH=1|2; default 1)
static int mma_batch(int kind) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPT_FFN_MMA_BATCH");
    v = (e && e[0] == '2') ? 2 : 1;
  }
  (void)kind;
  return v;
}
template <int KIND>
static cudaError_t launch_pair_gather(TcArgs& a, int tiles_upper, cudaStream_t s) {
  a.pair_rows = pair_tma_rows(KIND);
  a.mma_batch = mma_batch(KIND);
  a.pair_cpw = pair_cp_warps(KIND);
  const int stages = std::min(7, (227 * 1024 - 2048) / kPairStage);
  const int smem = stages * kPairStage + 2048;
  static std::atomic<bool> attr_set[kMaxDev];
  static std::atomic<int> mc_cache[kMaxDev];
  if (cudaError_t e = set_smem_attr_once(tc_pair_gather_kernel<KIND>, attr_set)) return e;
  const int max_clusters = max_pair_clusters(tc_pair_gather_kernel<KIND>, smem, mc_cache);
  const int clusters = std::max(1, std::min(tiles_upper, max_clusters));
  const bool trace_on = trace_begin(a, s);
  const char* name = KIND == K_FWD1 ? "tc_fwd1_gate_up" : "tc_bwd_dA";
  prof_begin(name, s);
  cudaError_t le = launch_pdl(tc_pair_gather_kernel<KIND>, dim3(2 * clusters), dim3(kThreads), smem, s, a, stages);
  prof_end(s);
  if (trace_on) trace_report(a, name, 2 * clusters, s);
  count_launch();
  cudaError_t e = le != cudaSuccess ? le : cudaGetLastError();
  if (debug_sync()) {
    e = cudaStreamSynchronize(s);
    fprintf(stderr, "[spt] tc pair-gather kind %d clusters %d stages %d smem %d BN %d: %s\n", KIND,
            clusters, stages, smem, a.BN, cudaGetErrorString(e));
  }
  return e;
}

// fused FWD1 -> FWD2 (tc_pair_mlp_kernel): SwiGLU blocks of 128 units on the
// CTA-pair gather path; SPT_FFN_MLP=0 runs the two GEMMs as separate kernels
// Measured on B200 (round 2), LLaMA shapes: parity-clean and 2-4 % slower than the
// two kernels (1.42 vs 1.38 ms at 16 K tokens, 2.84 vs 2.72 ms at 32 K): sH, the
// W2 ring and the store staging leave FWD1 a 4-stage (128 KB) operand ring instead
// of 7, and the gathered mainloop loses what the overlap gains -> opt-in
static bool mlp_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPT_FFN_MLP");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}
static bool mlp_ok(const Geom& g) { return g.mp == 2 && g.bw == 128 && !g.split && mlp_enabled(); }

static cudaError_t launch_pair_mlp(TcArgs& a, int tiles_upper, cudaStream_t s) {
  // sH, W2 ring, TMA-store staging, barriers
  const int fixed = 32768 + kMlpW2Slots * 16384 + kEpiWarps * 4096 + 2048;
  const int stages = std::min(6, (227 * 1024 - fixed) / kPairStage);
  const int smem = stages * kPairStage + fixed;
  static std::atomic<bool> attr_set[kMaxDev];
  static std::atomic<int> mc_cache[kMaxDev];
  if (cudaError_t e = set_smem_attr_once(tc_pair_mlp_kernel, attr_set)) return e;
  const int max_clusters = max_pair_clusters(tc_pair_mlp_kernel, smem, mc_cache);
  const int clusters = std::max(1, std::min(tiles_upper, max_clusters));
  const bool trace_on = trace_begin(a, s);
  prof_begin("tc_fwd1_fwd2", s);
  cudaError_t le = launch_pdl(tc_pair_mlp_kernel, dim3(2 * clusters), dim3(kThreads), smem, s, a, stages);
  prof_end(s);
  if (trace_on) {
    unsigned long long h[1024 * kTraceSlots];
    cudaMemcpyAsync(h, g_trace_buf, sizeof(unsigned long long) * 2 * clusters * kTraceSlots,
                    cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double sum[kTraceSlots] = {0};
    for (int b = 0; b < 2 * clusters; b += 2)  // leaders (MMA) and their epilogue
      for (int i = 0; i < kTraceSlots; ++i) sum[i] += (double)h[b * kTraceSlots + i];
    const double tot = sum[6] > 0 ? sum[6] : 1;
    fprintf(stderr,
            "[spt-trace] fused fwd1->fwd2 (leaders) | MMA wait stage %.0f%% acc1/H %.0f%% W2 %.0f%% "
            "acc2 %.0f%% | epi wait acc1 %.0f%% chunk %.0f%% drain busy %.0f%% | cta cycles %.0f\n",
            100 * sum[0] / tot, 100 * sum[1] / tot, 100 * sum[4] / tot, 100 * sum[5] / tot,
            100 * sum[2] / tot, 100 * sum[3] / tot, 100 * sum[7] / tot, tot / clusters);
    a.trace = nullptr;
  }
  count_launch();
  cudaError_t e = le != cudaSuccess ? le : cudaGetLastError();
  if (debug_sync()) {
    e = cudaStreamSynchronize(s);
    fprintf(stderr, "[spt] fused fwd1->fwd2 clusters %d stages %d smem %d: %s\n", clusters, stages,
            smem, cudaGetErrorString(e));
  }
  return e;
}

template <int KIND>
static cudaError_t launch_bres(TcArgs& a, int units_upper, cudaStream_t s) {
  const int kbu = KIND == K_FWD2 ? (a.bw + 63) / 64 : (a.mp * a.bw + 63) / 64;
  const bool fits = 227 * 1024 - 1280 - kbu * 16384 - (kEpiWarps * 4096 + 1024) >= 3 * kABytes;
  if (fits && use_pair(KIND)) return launch_pair<KIND>(a, units_upper, s);
  return launch<KIND>(a, units_upper, s);
}

// N tiles per dW raster group.  Every CTA of a wave streams its block's bucket
// rows in token order, so the wave re-reads from DRAM about |union of its blocks'
// tokens| x (its distinct N tiles) x 512 B of gathered rows plus (its distinct
// blocks) x the blocks' dZ / H~ rows: block-major order (all NT N tiles of ~9
// blocks per wave at LLaMA scale) over-weights the first term.  Measured
// (LLaMA scale): dW1 1.55 -> 1.44 ms at 8 N tiles per group (~18 blocks per
// wave), 1.42-1.46 at 4 / 2; dW2 (bw-wide A, half dW1's dZ bytes) 1.17 at 16 and 8,
// 1.20-1.23 at 4 / 2.  Default: dW1 8, dW2 block-major; SPT_FFN_DW_NG overrides both.
static int dw_group(int NT, int kind) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPT_FFN_DW_NG");
    v = e ? atoi(e) : 0;
  }
  const int ng = v >= 1 ? v : (kind == K_DW1 ? 8 : NT);
  return ng < NT ? ng : NT;
}
// tc_gemm_kernel gathered-row kinds: rows of each 256-row stage by TMA gather4
// (the rest by the four cp.async warps); SPT_FFN_G1_ROWS (multiple of 4, 32..256)
// Measured: tokens-on-N dA at LLaMA scale 1.81 / 1.54 / 1.42 / 1.28 / 1.16 / 1.15 ms
// at 256 / 192 / 160 / 128 / 96 / 64 rows (second box: 64 1.24, 80 1.24, 48 1.28,
// 32 1.28); the 1-CTA FWD1 (OPT, N = 128) 0.124 -> 0.109 ms at 64.  Default 64.
static int g1_tma_rows() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPT_FFN_G1_ROWS");
    v = e ? atoi(e) : kG1TmaRows;
    if (v < 32 || v > 256 || v % 4) v = kG1TmaRows;
  }
  return v;
}
static void base_args(TcArgs& a, const Geom& g, const RouteView& r) {
  a.g1_rows = g1_tma_rows();
  a.r = r;
  a.T = g.T;
  a.G = g.G;
  a.d = g.d;
  a.D = g.D;
  a.bw = g.bw;
  a.mp = g.mp;
  a.act = g.act;
  a.gate = g.gate;
  a.gpad = g.gpad;
  a.NT = (int)ceil_div(g.d, 256);
  a.MH = 1;
  a.nu = 1;
  a.bn_u = g.bw;
  a.kstream = 0;
  a.split = g.split ? 1 : 0;
  a.unit_mt = unit_mtiles();
  static int pf = -1;  // SPT_FFN_PREFETCH=1 enables the L2 prefetch of gathered rows
  if (pf < 0) {
    const char* e = getenv("SPT_FFN_PREFETCH");
    pf = (e && e[0] == '1') ? 1 : 0;  // measured slower on B200 (r01): off by default
  }
  a.prefetch = pf;
  static int abl = -1;
  if (abl < 0) {
    const char* e = getenv("SPT_FFN_ABLATE");
    abl = e ? atoi(e) : 0;
  }
  a.ablate = abl;

}

static int bucket_tiles_upper(const Geom& g) { return (int)(ceil_div(g.pairs, 128) + g.G); }

int unit_mtiles() {
  static int v = 0;
  if (!v) {
    const char* e = getenv("SPT_FFN_UNIT_MT");
    v = e ? atoi(e) : 128;  // measured r01: 128 (~ a whole block per unit) best at LLaMA scale
    if (v < 1) v = 128;
  }
  return v;
}

// a7 variant.  Default: the fused dA kernel (tokens on M, N = bw, dgate/dZ in the
// epilogue).  SPT_FFN_DAT=1: tokens on N (N = 256, transposed dA via TMA store)
// + da_post_kernel; measured at parity on B200 in round 1 (both ~1.7 ms at
// LLaMA scale: the gathered-row supply, not the MMA shape, bounds a7).
// SPT_FFN_SIDE=1 (opt-in): dX first, then the grad-input combine as side work of
// the dW kernels' epilogue warps.  Measured slower (LLaMA-scale 10.72-10.85 vs
// 10.29-10.41 ms): four warps per SM claim only 15 % of the tokens during dW1
// (latency-bound at ~3 us per dependent round under the GEMM's load) while
// slowing it 12 %, and the drain in dW2 streams at ~3.7 TB/s, below the
// stand-alone kernel's 6.4 TB/s.  Default: the stand-alone combine kernel.
static bool side_combine_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPT_FFN_SIDE");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// SPT_FFN_DAT (bf16, bw <= 128; else always 0): 0 = a7 with tokens on M (N = bw) and
// the fused epilogue (tc_pair_gather_kernel<DA>); 1 = tokens on N
// (N = 256) with the dA tile stored and da_post_kernel; 2 = tokens on N with the
// fused epilogue (epilogue_dat_fused); 3 = tokens on N, fused row-major epilogue
// (epilogue_dat_rows: smem transpose, 16-byte Z / dZ accesses)
// Default 3 (measured, LLaMA scale: dA 1.41-1.45 -> 1.15-1.24 ms; OPT 0.133 ->
// 0.111 ms; BERT 0.055 -> 0.053 ms): the tokens-on-N MMA shape (N = 256, not
// bw = 128) with the row-major epilogue.
static int dat_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPT_FFN_DAT");
    v = (e && e[0] >= '0' && e[0] <= '3') ? e[0] - '0' : 3;
  }
  return v;
}
static bool use_fused_da() { return dat_mode() == 0; }

bool tc_supported(const Geom& g) {
  if (g.d % 64) return false;
  // m' bw > 256 (wide blocks): FWD1 / DA tile the units, DW* the features,
  // FWD2 / DX stream K (no limit on bw beyond the ABI's bw % 16 == 0)
  if (g.mp == 2 && g.bw % 64) return false;     // DX K stages must not straddle gate/up
  if (g.gpad > 256) return false;               // router N / DWR M (two 128-block halves) <= 256
  return true;
}

// tensor-map encode status is checked BEFORE the launch: a kernel must never
// run with a map the driver rejected (its TMA loads would never complete)
#define TRY(x)                                                                    \
  do {                                                                            \
    if (!ok) {                                                                    \
      if (debug_sync()) fprintf(stderr, "[spt] tensor map encode failed (%s)\n", #x); \
      return cudaErrorInvalidValue;                                               \
    }                                                                             \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) return e_;                                             \
  } while (0)

// fp32 -> bf16 hi | lo (reading c13': hi = RNE(x), lo = RNE(x - hi), x - hi exact)
__global__ void __launch_bounds__(256) split_bf16_kernel(const float* __restrict__ src,
                                                         __nv_bfloat16* __restrict__ hi,
                                                         __nv_bfloat16* __restrict__ lo, int64_t n) {
  pdl_wait();  // PDL: predecessor grid complete, its writes visible
  // successor launches as this grid's CTAs exit (an early trigger measured slower)
  const int64_t n4 = n / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldcs(reinterpret_cast<const float4*>(src) + i);
    const uint32_t h0 = pack_bf16(v.x, v.y), h1 = pack_bf16(v.z, v.w);
    reinterpret_cast<uint2*>(hi)[i] = make_uint2(h0, h1);
    reinterpret_cast<uint2*>(lo)[i] = make_uint2(pack_bf16_lo(v.x, v.y, h0), pack_bf16_lo(v.z, v.w, h1));
  }
  for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const __nv_bfloat16 h = __float2bfloat16(src[i]);
    hi[i] = h;
    lo[i] = __float2bfloat16(src[i] - __bfloat162float(h));
  }
}

cudaError_t launch_split_bf16(const float* src, void* dst, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int grid = (int)std::min<int64_t>(ceil_div(n / 4 + 1, 256), (int64_t)num_sms() * 8);
  prof_begin("split_bf16", s);
  cudaError_t le = launch_pdl(split_bf16_kernel, dim3(grid), dim3(256), 0, s, src,
                              (__nv_bfloat16*)dst, (__nv_bfloat16*)lo_half(dst, n), n);
  prof_end(s);
  count_launch();
  return le != cudaSuccess ? le : cudaGetLastError();
}

bool simt_forced() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPT_FFN_SIMT");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

cudaError_t tc_router(const Geom& g, const void* x, const void* w_r, float* logits,
                      cudaStream_t s, const Bufs* b) {
  TcArgs a{};
  base_args(a, g, RouteView{});
  bool ok = true;
  if (g.split) {  // fp32 operands -> hi | lo copies in the workspace
    if (!b) return cudaErrorInvalidValue;
    cudaError_t e = launch_split_bf16((const float*)x, b->xs, g.T * g.d, s);
    if (e == cudaSuccess) e = launch_split_bf16((const float*)w_r, b->wrs, (int64_t)g.G * g.d, s);
    if (e != cudaSuccess) return e;
    x = b->xs;
    w_r = b->wrs;
    ok = make_tmap_bf16_2d(&a.ta2, lo_half(x, g.T * g.d), g.T, g.d, g.d, 64, 128) &&
         make_tmap_bf16_2d(&a.tb2, lo_half(w_r, (int64_t)g.G * g.d), g.G, g.d, g.d, 64, g.gpad);
  }
  ok = ok && make_tmap_bf16_2d(&a.ta, x, g.T, g.d, g.d, 64, 128) &&
       make_tmap_bf16_2d(&a.tb, w_r, g.G, g.d, g.d, 64, g.gpad);
  a.BN = g.gpad;
  a.out = logits;
  TRY(launch<K_ROUTER>(a, (int)ceil_div(g.T, 128), s));
  return cudaSuccess;
}

// Device-side tile schedules from the bucket layout (no host sync):
//  tile_list[P(mt) + rank_b(mt)] = mt << 8 | b, i.e. bucket tiles in (m-tile,
//  block) order with P(mt) = sum_b min(nt_b, mt) and rank_b(mt) = #{b' < b :
//  nt_b' > mt};  unit_offsets = prefix over blocks of ceil(nt_b/16) * NT.
__global__ void __launch_bounds__(256) tile_sched_kernel(int G, int NT, int unit_mt, int raster,
                                                         const int32_t* __restrict__ tile_offsets,
                                                         int32_t* __restrict__ tile_list,
                                                         int32_t* __restrict__ unit_offsets,
                                                         int32_t* __restrict__ tile_block) {
  pdl_wait();  // PDL: predecessor grid complete, its writes visible
  // successor launches as this grid's CTAs exit (an early trigger measured slower)
  __shared__ int ntb[kMaxBlocks];
  __shared__ int ntu[kMaxBlocks];  // 128-row tiles per block (units) ...
  for (int i = threadIdx.x; i < G; i += blockDim.x) {
    ntu[i] = tile_offsets[i + 1] - tile_offsets[i];
    ntb[i] = (ntu[i] + 1) / 2;  // ... and 256-row pair tiles (gathered-A kinds)
  }
  __syncthreads();
  // 2-D raster: groups of kRasterBlocks blocks, inside a group (m-tile, block)
  // order.  The group's weights (<= 32 MB of W1 rows) and the window of tokens
  // the in-flight m-levels gather both stay in L2.
  const int b = blockIdx.x;
  for (int t = tile_offsets[b] + threadIdx.x; t < tile_offsets[b + 1]; t += blockDim.x) tile_block[t] = b;
  const int g0 = (b / raster) * raster, g1 = min(G, g0 + raster);
  int base = 0;
  for (int bb = 0; bb < g0; ++bb) base += ntb[bb];
  for (int mt = threadIdx.x; mt < ntb[b]; mt += blockDim.x) {
    int P = base, rank = 0;
    for (int bb = g0; bb < g1; ++bb) {
      P += min(ntb[bb], mt);
      rank += (bb < b) && (ntb[bb] > mt);
    }
    tile_list[P + rank] = (mt << 8) | b;
  }
  if (b == 0 && threadIdx.x == 0) {
    int run = 0;
    for (int bb = 0; bb < G; ++bb) {
      unit_offsets[bb] = run;
      run += (int)ceil_div(ntu[bb], unit_mt) * NT;
    }
    unit_offsets[G] = run;
    int pairs = 0;
    for (int bb = 0; bb < G; ++bb) pairs += ntb[bb];
    unit_offsets[G + 1] = pairs;
  }
}

// blocks per L2 raster group of the gathered-A GEMMs (SPT_FFN_RASTER, default kRasterBlocks)
static int raster_blocks() {
  static int v = 0;
  if (!v) {
    const char* e = getenv("SPT_FFN_RASTER");
    v = e ? atoi(e) : kRasterBlocks;
    if (v < 1) v = kRasterBlocks;
  }
  return v;
}

static cudaError_t build_schedules(const Geom& g, const RouteView& r, const Bufs& b, cudaStream_t s) {
  prof_begin("tile_sched", s);
  (void)launch_pdl(tile_sched_kernel, dim3(g.G), dim3(256), 0, s, g.G, (int)ceil_div(g.d, 256), unit_mtiles(),
                                        raster_blocks(), r.tile_offsets,
                                        b.tile_list,
                                        b.unit_offsets, b.tile_block);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

static int units_upper(const Geom& g) {
  return (int)((ceil_div(bucket_tiles_upper(g), unit_mtiles()) + g.G) * ceil_div(g.d, 256));
}

cudaError_t tc_forward(const Geom& g, const void* x, const void* w1, const void* w2,
                       const RouteView& r, void* y, const Bufs& b, cudaStream_t s,
                       const LoraArgs* lo) {
  const int up = bucket_tiles_upper(g);
  cudaError_t e0 = build_schedules(g, r, b, s);
  if (e0 != cudaSuccess) return e0;
  const int64_t nz = g.rows_cap * g.mp * g.bw, nh = g.rows_cap * g.bw;  // split: lo offsets
  if (g.split) {  // fp32 operands -> bf16 hi | lo copies (reading c13')
    if ((e0 = launch_split_bf16((const float*)x, b.xs, g.T * g.d, s)) != cudaSuccess ||
        (e0 = launch_split_bf16((const float*)w1, b.w1s, (int64_t)g.mp * g.D * g.d, s)) != cudaSuccess ||
        (e0 = launch_split_bf16((const float*)w2, b.w2s, (int64_t)g.D * g.d, s)) != cudaSuccess)
      return e0;
    x = b.xs;
    w1 = b.w1s;
    w2 = b.w2s;
  }
  if (!lo && mlp_ok(g) && use_pair_gather()) {  // a4 + a5 in one kernel, then the combine
    TcArgs a{};
    base_args(a, g, r);
    a.tile_list = b.tile_list;
    a.bn_u = g.bw;
    a.nu = 1;
    bool ok = make_tmap_bf16_2d(&a.ta, x, g.T, g.d, g.d, 64, 1) &&
              make_tmap_bf16_2d(&a.tb, w1, (uint64_t)g.mp * g.D, g.d, g.d, 64, a.bn_u) &&
              make_tmap_bf16_2d(&a.tw2, w2, g.D, g.d, g.d, 64, 64) &&
              make_tmap_bf16_2d(&a.tc, b.part, g.rows_cap, g.d, g.d, 64, 32);
    a.BN = g.mp * a.bn_u;
    a.MH = 2;
    a.aux2 = x;
    a.out = b.z;
    a.out2 = b.h;
    a.unit_offsets = b.unit_offsets;
    TRY(launch_pair_mlp(a, up / 2 + g.G, s));
    return launch_combine_fwd(g, r, b.part, y, s);
  }
  {
    // LoRA: FWD1 runs on X_aug / W1_aug (K = d + 64: the u C_I term is one more K stage)
    Geom g1 = g;
    if (lo) {
      if ((e0 = lora_fwd_prep(g, x, w1, *lo, s)) != cudaSuccess) return e0;
      g1.d = g.d + lo->ka;
      x = lo->xaug;
      w1 = lo->waug;
    }
    const Geom& g = g1;  // the FWD1 geometry
    TcArgs a{};
    base_args(a, g, r);
    a.tile_list = b.tile_list;
    // wide blocks (m' bw > 256): tiles of 256 / m' units (N = 256)
    a.bn_u = g.mp * g.bw > 256 ? 256 / g.mp : g.bw;
    a.nu = (int)ceil_div(g.bw, a.bn_u);
    bool ok = make_tmap_bf16_2d(&a.ta, x, g.T, g.d, g.d, 64, 1) &&
              make_tmap_bf16_2d(&a.tb, w1, (uint64_t)g.mp * g.D, g.d, g.d, 64, a.bn_u) &&
              make_tmap_bf16_2d(&a.tc, x, g.T, g.d, g.d, 256, 1, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_SWIZZLE_NONE);  // L2 prefetch rows
    a.BN = g.mp * a.bn_u;
    a.MH = 2;
    a.aux2 = x;
    a.out = b.z;
    a.out2 = b.h;
    a.unit_offsets = b.unit_offsets;
    if (g.split) {
      ok = ok && make_tmap_bf16_2d(&a.ta2, lo_half(x, g.T * g.d), g.T, g.d, g.d, 64, 1) &&
           make_tmap_bf16_2d(&a.tb2, lo_half(w1, (int64_t)g.mp * g.D * g.d), (uint64_t)g.mp * g.D,
                             g.d, g.d, 64, a.bn_u);
      a.aux2_lo = lo_half(x, g.T * g.d);
      a.out_lo = lo_half(b.z, nz);
      a.out2_lo = lo_half(b.h, nh);
    }
    const int tiles = (up / 2 + g.G) * a.nu;
    if (use_pair_gather() && pair_gather_ok(a.BN) && !g.split) {
      // CTA r holds B rows of its N half: the gate (r = 0) / up (r = 1) rows
      // for SwiGLU (a box of bn_u rows), else rows [r BN/2, (r+1) BN/2) of the tile
      if (g.mp != 2) ok = ok && make_tmap_bf16_2d(&a.tb, w1, g.D, g.d, g.d, 64, a.BN / 2);
      TRY(launch_pair_gather<K_FWD1>(a, tiles, s));
    } else {
      TRY(launch<K_FWD1>(a, tiles, s));
    }
  }
  {
    TcArgs a{};
    base_args(a, g, r);
    bool ok = make_tmap_bf16_2d(&a.ta, b.h, g.rows_cap, g.bw, g.bw, 64, 128) &&
              make_tmap_bf16_2d(&a.tb, w2, g.D, g.d, g.d, 64, 64);
    ok = ok && make_tmap_bf16_2d(&a.tc, b.part, g.rows_cap, g.d, g.d, 64, 32);
    if (g.split)  // fp32 partial rows (generic epilogue), K streamed in three passes
      ok = ok && make_tmap_bf16_2d(&a.ta2, lo_half(b.h, nh), g.rows_cap, g.bw, g.bw, 64, 128) &&
           make_tmap_bf16_2d(&a.tb2, lo_half(w2, (int64_t)g.D * g.d), g.D, g.d, g.d, 64, 64);
    a.BN = 256;
    a.out = b.part;
    a.unit_offsets = b.unit_offsets;
    a.kstream = g.bw > 256 || g.split;  // the K = bw slab no longer fits smem: stream K
    if (a.kstream) {
      TRY(launch<K_FWD2>(a, up * a.NT, s));
    } else {
      TRY(launch_bres<K_FWD2>(a, units_upper(g), s));
    }
  }
  if (lo) return lora_fwd_finish(g, r, b, *lo, y, s);
  return launch_combine_fwd(g, r, b.part, y, s);
}

// a7 second half: per padded bucket row (one warp), from dA (fp32) and the Z
// stash: dgate = sum_u dA_u act(z_u); dZ = g dA act'(Z); dlogit = dgate g (1-g)
// (as sigma(z) sigma(-z)); dense hi/lo bf16 dlogits for the dW_R GEMM.  Padding
// rows get dZ = 0 (the K tails of the dW1 GEMM rely on it).
__global__ void __launch_bounds__(256, 4) da_post_kernel(int64_t T, int G, int bw, int mp, int act,
                                                      int gate, int gpad, RouteView r,
                                                      const int32_t* __restrict__ tile_block,
                                                      const float* __restrict__ da,
                                                      const __nv_bfloat16* __restrict__ z,
                                                      __nv_bfloat16* __restrict__ dz,
                                                      float* __restrict__ dgate_rows,
                                                      float* __restrict__ dlogit_rows,
                                                      __nv_bfloat16* __restrict__ dlg) {
  // one warp per 4 padded rows; lane covers units lane*4 + 128 i; all loads of
  // the 4 rows are issued before any math (memory-level parallelism)
  constexpr int R = 4;
  const int lane = threadIdx.x & 31;
  const int64_t row0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * R;
  const int64_t nrows = (int64_t)r.tile_offsets[G] * 128;
  if (row0 >= nrows) return;
  for (int u0 = lane * 4; u0 < ((bw + 127) / 128) * 128; u0 += 128) {
    const bool ul = u0 < bw;
    float4 dA[R];
    uint2 zg2[R], zu2[R];
    bool valid[R];
    float g[R];
    int bidx[R];
    int64_t pos[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int64_t row = row0 + i;
      valid[i] = false;
      g[i] = 0.f;
      bidx[i] = 0;
      pos[i] = 0;
      dA[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      zg2[i] = zu2[i] = make_uint2(0u, 0u);
      if (row < nrows) {
        const int b = tile_block[row >> 7];
        const int e = (int)(row - (int64_t)r.tile_offsets[b] * 128);
        bidx[i] = b;
        pos[i] = r.block_offsets[b] + e;
        valid[i] = e < r.block_offsets[b + 1] - r.block_offsets[b];
        if (valid[i]) {
          g[i] = r.bucket_gate[pos[i]];
          if (ul) {
            dA[i] = *reinterpret_cast<const float4*>(da + row * bw + u0);
            const __nv_bfloat16* zr = z + row * (int64_t)(mp * bw);
            zg2[i] = *reinterpret_cast<const uint2*>(zr + u0);
            if (mp == 2) zu2[i] = *reinterpret_cast<const uint2*>(zr + bw + u0);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int64_t row = row0 + i;
      float dgate = 0.f;
      if (row < nrows) {
        const float a4[4] = {dA[i].x, dA[i].y, dA[i].z, dA[i].w};
        const float zg[4] = {__uint_as_float(zg2[i].x << 16), __uint_as_float(zg2[i].x & 0xffff0000u),
                             __uint_as_float(zg2[i].y << 16), __uint_as_float(zg2[i].y & 0xffff0000u)};
        const float zu[4] = {__uint_as_float(zu2[i].x << 16), __uint_as_float(zu2[i].x & 0xffff0000u),
                             __uint_as_float(zu2[i].y << 16), __uint_as_float(zu2[i].y & 0xffff0000u)};
        float dzg[4], dzu[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float av, dg, du;
          act_fwd_bwd<true>(act, zg[j], zu[j], av, dg, du);
          dgate = fmaf(a4[j], av, dgate);
          dzg[j] = g[i] * a4[j] * dg;
          dzu[j] = g[i] * a4[j] * du;
        }
        if (ul) {
          __nv_bfloat16* dzr = dz + row * (int64_t)(mp * bw);
          *reinterpret_cast<uint2*>(dzr + u0) = make_uint2(pack_bf16(dzg[0], dzg[1]), pack_bf16(dzg[2], dzg[3]));
          if (mp == 2)
            *reinterpret_cast<uint2*>(dzr + bw + u0) =
                make_uint2(pack_bf16(dzu[0], dzu[1]), pack_bf16(dzu[2], dzu[3]));
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) dgate += __shfl_xor_sync(0xffffffffu, dgate, o);
      // bw <= 128 for the tensor-core path, so one pass covers the row
      if (lane == 0 && row < nrows) {
        float dlogit = 0.f;
        if (valid[i] && gate == SPT_GATE_SIGMOID) {
          const int64_t t = r.bucket_token[pos[i]];
          dlogit = dgate * sigmoid_pair(r.logits[t * G + bidx[i]]);
          const __nv_bfloat16 hi = __float2bfloat16(dlogit);
          const __nv_bfloat16 lo = __float2bfloat16(dlogit - __bfloat162float(hi));
          dlg[t * gpad + bidx[i]] = hi;
          dlg[(T + t) * gpad + bidx[i]] = lo;
        }
        dgate_rows[row] = valid[i] ? dgate : 0.f;
        dlogit_rows[row] = dlogit;
      }
    }
  }
}

__global__ void dwr_reduce_kernel(int n_split, int64_t n, const float* __restrict__ part,
                                  float* __restrict__ out, int acc) {
  pdl_wait();  // PDL: predecessor grid complete, its writes visible
  // successor launches as this grid's CTAs exit (an early trigger measured slower)
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s = acc ? out[i] : 0.f;
  for (int k = 0; k < n_split; ++k) s += part[k * n + i];
  out[i] = s;
}

// Wide blocks (bw > 256): dA is unit-tiled, so each pair's dgate arrives as
// nu partial sums (one per unit tile, dgp[prow][ut]).  One thread per (token,
// selected block): dgate = sum of the partials, dlogit = dgate sigma(z)
// sigma(-z) (SIGMOID), and the dense hi/lo bf16 dlogits of the dW_R GEMM --
// what the fused dA epilogue writes inline when nu == 1.
__global__ void __launch_bounds__(256) dgate_reduce_kernel(int64_t T, int G, int k, int nu, int gate,
                                                           int gpad, RouteView r,
                                                           const float* __restrict__ dgp,
                                                           float* __restrict__ rows_f,
                                                           float* __restrict__ rows_g,
                                                           __nv_bfloat16* __restrict__ dlg) {
  pdl_wait();  // PDL: predecessor grid complete, its writes visible
  // successor launches as this grid's CTAs exit (an early trigger measured slower)
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T * k) return;
  const int64_t t = i / k;
  const int b = r.topk_idx[i];
  const int64_t pos = r.pair_slot[i];
  const int64_t prow = (int64_t)r.tile_offsets[b] * 128 + (pos - r.block_offsets[b]);
  float dgate = 0.f;
  for (int u = 0; u < nu; ++u) dgate += dgp[prow * nu + u];
  float dlogit = 0.f;
  if (gate == SPT_GATE_SIGMOID) {
    dlogit = dgate * sigmoid_pair(r.logits[t * G + b]);
    const __nv_bfloat16 hi = __float2bfloat16(dlogit);
    const __nv_bfloat16 lo = __float2bfloat16(dlogit - __bfloat162float(hi));
    dlg[t * gpad + b] = hi;
    dlg[(T + t) * gpad + b] = lo;
  }
  rows_f[prow] = dgate;
  rows_g[prow] = dlogit;
}

int dense_tn_splits(const Geom& g) {
  // one wave: (N tiles) x (splits) <= #SMs (ceil gave 160 CTAs on 148 SMs at d = 4096)
  const int tiles = (int)ceil_div(g.d, 256);  // one M tile of blocks (two halves when G > 128)
  int s = std::max(1, num_sms() / tiles);
  const int max_s = (int)ceil_div(g.T, 64);
  if (s > max_s) s = max_s;
  return s < 1 ? 1 : s;
}

cudaError_t tc_dense_tn(const Geom& g, const void* ahl, const void* bmat, float* part, int n_split,
                        float* out, bool accumulate, cudaStream_t s, const void* bmat_lo) {
  TcArgs a{};
  base_args(a, g, RouteView{});
  a.split = bmat_lo ? 1 : 0;  // third part: dlogit hi x B lo
  bool ok = make_tmap_bf16_2d(&a.ta, ahl, (uint64_t)2 * g.T, g.gpad, g.gpad, 64, 64) &&
            make_tmap_bf16_2d(&a.tb, bmat, g.T, g.d, g.d, 64, 64) &&
            (!bmat_lo || make_tmap_bf16_2d(&a.tb2, bmat_lo, g.T, g.d, g.d, 64, 64));
  a.BN = 256;
  a.MH = g.gpad > 128 ? 2 : 1;  // G in 129..256: two 128-block M halves
  a.n_split = n_split;
  a.ksplit = (int)(ceil_div(ceil_div(g.T, n_split), 64) * 64);
  a.out = part;
  TRY(launch<K_DWR>(a, a.NT * a.n_split, s));
  const int64_t n = (int64_t)g.G * g.d;
  prof_begin("dwr_reduce", s);
  (void)launch_pdl(dwr_reduce_kernel, dim3((unsigned)ceil_div(n, 256)), dim3(256), 0, s, n_split, n, part, out,
                                                               accumulate ? 1 : 0);
  prof_end(s);
  count_launch();
  return cudaGetLastError();
}

cudaError_t tc_dense_nn(const Geom& g, const void* ahl, const void* bmat, void* out,
                        cudaStream_t s) {
  TcArgs a{};
  base_args(a, g, RouteView{});
  bool ok = make_tmap_bf16_2d(&a.ta, ahl, (uint64_t)2 * g.T, g.gpad, g.gpad, 64, 128) &&
            make_tmap_bf16_2d(&a.tb, bmat, g.G, g.d, g.d, 64, 64);
  a.BN = 256;
  a.out = out;
  TRY(launch<K_DXR>(a, (int)ceil_div(g.T, 128) * a.NT, s));
  return cudaSuccess;
}

// ---- side stream for the backward's weight-gradient branch (per device)
// Measured (graph steps): BERT 0.305 -> 0.277 ms, OPT 0.967 -> 0.950, opt2048_g8
// 0.943 -> 0.912 (dW1 96 / 512 / 256 tiles), but LLaMA 4.92 -> 5.04 and LLaMA
// scale 9.82 -> 9.95 (1376 tiles: every kernel already fills the GPU, the pair
// only contends).  Default (unset): fork when dW1 has <= 4 tiles per SM;
// SPT_FFN_BWD_STREAMS=1 / 0 forces it on / off.
static bool bwd_streams_enabled(const Geom& g) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPT_FFN_BWD_STREAMS");
    v = (e && e[0] == '1') ? 1 : ((e && e[0] == '0') ? 0 : 2);
  }
  if (v != 2) return v == 1;
  const int64_t dw1_tiles = (int64_t)g.G * ceil_div((int64_t)g.mp * g.bw, 256) * ceil_div(g.d, 256);
  return dw1_tiles <= 4 * (int64_t)num_sms();
}
// two side streams: dW1 + dW_R on `side`, dW2 on `side2`; side2 joins side once
// the weight gradients are final (dw_event), side joins the caller's stream last
struct ForkJoin {
  cudaStream_t side, side2;
  cudaEvent_t join, join2;
};
struct SideRes {
  cudaStream_t st[2];
  cudaEvent_t fork, join, join2;
};
static std::mutex g_side_mu;  // event record + wait pairs on the shared side streams
static cudaError_t fork_side(cudaStream_t s, ForkJoin& fj) {
  static std::atomic<SideRes*> res[kMaxDev];
  std::mutex& mu = g_side_mu;
  const int dev = cur_dev();
  if (!res[dev].load()) {
    std::lock_guard<std::mutex> lk0(mu);
    if (!res[dev].load()) {
      SideRes* r = new SideRes{};
      if (cudaStreamCreateWithFlags(&r->st[0], cudaStreamNonBlocking) != cudaSuccess ||
          cudaStreamCreateWithFlags(&r->st[1], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&r->fork, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&r->join, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&r->join2, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();  // do not leave the failure in the thread's error state
        for (cudaStream_t st : r->st)
          if (st) cudaStreamDestroy(st);
        for (cudaEvent_t ev : {r->fork, r->join, r->join2})
          if (ev) cudaEventDestroy(ev);
        delete r;
        return cudaErrorUnknown;
      }
      res[dev].store(r);  // lives for the process (one set per device)
    }
  }
  const SideRes* r = res[dev].load();
  fj.side = r->st[0];
  fj.side2 = r->st[1];
  fj.join = r->join;
  fj.join2 = r->join2;
  // record + wait as one step: calls from several host threads share the
  // device's side streams and events (their dW work then runs in call order)
  std::lock_guard<std::mutex> lk(mu);
  if (cudaEventRecord(r->fork, s) != cudaSuccess || cudaStreamWaitEvent(fj.side, r->fork, 0) != cudaSuccess ||
      cudaStreamWaitEvent(fj.side2, r->fork, 0) != cudaSuccess)
    return cudaErrorUnknown;
  return cudaSuccess;
}
static cudaError_t join_side2(const ForkJoin& fj) {
  std::lock_guard<std::mutex> lk(g_side_mu);
  if (cudaEventRecord(fj.join2, fj.side2) != cudaSuccess || cudaStreamWaitEvent(fj.side, fj.join2, 0) != cudaSuccess)
    return cudaErrorUnknown;
  return cudaSuccess;
}
static cudaError_t join_side(cudaStream_t s, const ForkJoin& fj) {
  std::lock_guard<std::mutex> lk(g_side_mu);
  if (cudaEventRecord(fj.join, fj.side) != cudaSuccess || cudaStreamWaitEvent(s, fj.join, 0) != cudaSuccess)
    return cudaErrorUnknown;
  return cudaSuccess;
}

cudaError_t tc_backward(const Geom& g, const void* x, const void* w1, const void* w2,
                        const void* w_r, const RouteView& r, const void* dy, void* dx, float* dw1,
                        float* dw2, float* dw_r, float* dgate_out, bool accumulate, const Bufs& b,
                        cudaEvent_t dw_ev, cudaStream_t s, const LoraArgs* lo) {
  const int up = bucket_tiles_upper(g);
  const bool sig = g.gate == SPT_GATE_SIGMOID;
  const bool lb = g.lbw != 0.f;  // load-balancing loss: dense router gradient (every block)
  // the tile schedules are the forward's (in the stash: same routing)
  cudaError_t e0 = cudaSuccess;
  if ((sig || lb) && cudaMemsetAsync(b.dlg, 0, (size_t)2 * g.T * g.gpad * 2, s) != cudaSuccess)
    return cudaErrorUnknown;
  const int64_t nz = g.rows_cap * g.mp * g.bw, nh = g.rows_cap * g.bw, ntd = g.T * g.d;
  if (g.split) {  // fp32 operands -> bf16 hi | lo copies (reading c13'); w_r stays fp32 (combine)
    if ((e0 = launch_split_bf16((const float*)dy, b.dys, ntd, s)) != cudaSuccess ||
        (e0 = launch_split_bf16((const float*)x, b.xs, ntd, s)) != cudaSuccess ||
        (e0 = launch_split_bf16((const float*)w1, b.w1s, (int64_t)g.mp * g.D * g.d, s)) != cudaSuccess ||
        (e0 = launch_split_bf16((const float*)w2, b.w2s, (int64_t)g.D * g.d, s)) != cudaSuccess)
      return e0;
    dy = b.dys;
    x = b.xs;
    w1 = b.w1s;
    w2 = b.w2s;
  }
  // LoRA: dA runs on dY_aug / W2_aug (K = d + 64: the (dy C_O^T) B_O^T term)
  Geom gda = g;
  const void* dy_da = dy;
  const void* w2_da = w2;
  if (lo) {
    if ((e0 = lora_bwd_prep(g, dy, w2, *lo, s)) != cudaSuccess) return e0;
    gda.d = g.d + lo->ka;
    dy_da = lo->xaug;
    w2_da = lo->waug;
  }
  if (!use_fused_da() && g.bw <= 128 && !g.split) {  // a7: dA^T = W2_b dY[bucket]^T (tokens on N), then dgate/dZ
    TcArgs a{};
    base_args(a, gda, r);
    bool ok = make_tmap_bf16_2d(&a.ta, dy_da, g.T, gda.d, gda.d, 64, 1) &&
              make_tmap_bf16_2d(&a.tb, w2_da, g.D, gda.d, gda.d, 64, 128) &&
              make_tmap_f32_2d(&a.tc, b.da, g.rows_cap, g.bw, g.bw, 32, 32);
    a.BN = 256;
    a.MH = 1;
    a.aux2 = dy_da;
    a.tile_list = b.tile_list;
    a.unit_offsets = b.unit_offsets;
    if (dat_mode() >= 2) {  // dgate / dZ / dlogit in the GEMM's epilogue
      a.dat_fused = dat_mode() == 2 ? 2 : 1;  // 2: per-(row, unit) form, 1: row-major (smem transpose)
      a.aux = b.z;
      a.out2 = b.dz;
      a.rows_f = b.dgate;
      a.rows_g = b.dlogit;
      a.dlg = b.dlg;
      TRY(launch<K_DAT>(a, up / 2 + g.G, s));
    } else {
    TRY(launch<K_DAT>(a, up / 2 + g.G, s));
    prof_begin("da_post", s);
    da_post_kernel<<<(unsigned)ceil_div(g.rows_cap, 32), 256, 0, s>>>(
        g.T, g.G, g.bw, g.mp, g.act, g.gate, g.gpad, r, b.tile_block, b.da, (const __nv_bfloat16*)b.z,
        (__nv_bfloat16*)b.dz, b.dgate, b.dlogit, (__nv_bfloat16*)b.dlg);
    prof_end(s);
    count_launch();
    }
  } else {  // a7 fused variant: dA = dY[bucket] W2_b^T with the dgate / dZ / dlogit epilogue
    TcArgs a{};
    base_args(a, gda, r);
    // wide blocks (bw > 256): tiles of 256 units (N = 256: the CTA-pair
    // kernel); dgate partials per tile
    a.bn_u = g.bw > 256 ? 256 : g.bw;
    a.nu = (int)ceil_div(g.bw, a.bn_u);
    a.dgp = b.da;  // [rows_cap][nu] fits the [rows_cap][bw] f32 scratch
    bool ok = make_tmap_bf16_2d(&a.ta, dy_da, g.T, gda.d, gda.d, 64, 1) &&
              make_tmap_bf16_2d(&a.tb, w2_da, g.D, gda.d, gda.d, 64, a.bn_u) &&
              make_tmap_bf16_2d(&a.tc, dy_da, g.T, gda.d, gda.d, 256, 1, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_SWIZZLE_NONE);  // L2 prefetch rows
    a.BN = a.bn_u;
    a.aux = b.z;
    a.out2 = b.dz;
    a.rows_f = b.dgate;
    a.rows_g = b.dlogit;
    a.dlg = b.dlg;
    a.tile_list = b.tile_list;
    a.MH = 2;
    a.aux2 = dy_da;
    a.unit_offsets = b.unit_offsets;
    if (g.split) {
      ok = ok && make_tmap_bf16_2d(&a.ta2, lo_half(dy, ntd), g.T, g.d, g.d, 64, 1) &&
           make_tmap_bf16_2d(&a.tb2, lo_half(w2, (int64_t)g.D * g.d), g.D, g.d, g.d, 64, a.bn_u);
      a.aux2_lo = lo_half(dy, ntd);
      a.aux_lo = lo_half(b.z, nz);
      a.out2_lo = lo_half(b.dz, nz);
    }
    const int tiles = (up / 2 + g.G) * a.nu;
    if (use_pair_gather() && pair_gather_ok(a.BN) && !g.split) {
      ok = ok && make_tmap_bf16_2d(&a.tb, w2_da, g.D, gda.d, gda.d, 64, a.BN / 2);
      TRY(launch_pair_gather<K_DA>(a, tiles, s));
    } else {
      TRY(launch<K_DA>(a, tiles, s));
    }
    if (a.nu > 1) {  // sum the unit tiles' dgate partials; dlogit, dense dlogits
      const int64_t n = g.T * g.k;
      prof_begin("dgate_reduce", s);
      (void)launch_pdl(dgate_reduce_kernel, dim3((unsigned)ceil_div(n, 256)), dim3(256), 0, s, 
          g.T, g.G, g.k, a.nu, g.gate, g.gpad, r, b.da, b.dgate, b.dlogit, (__nv_bfloat16*)b.dlg);
      prof_end(s);
      count_launch();
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
  }
  if (lo) {  // W frozen: the LoRA factor gradients dC_I, dB_O from dZ, h~ (no dW1 / dW2)
    if ((e0 = lora_bwd_grads(g, r, b, *lo, s)) != cudaSuccess) return e0;
  }
  // The grad-input combine rides on the dW kernels (side work of their epilogue
  // warps, tc_gemm_kernel) when dX runs before them: single-process calls (no
  // dw_event to overlap a gradient all-reduce with), the plain bf16 path, k <= 32.
  const bool side = side_combine_enabled() && !lo && !lb && !g.split && g.k <= 32 && !dw_ev;
  auto set_side = [&](TcArgs& a, bool drain) {
    if (!side) return;
    a.cb_part = (const __nv_bfloat16*)b.part;
    a.cb_dlogit = b.dlogit;
    a.cb_wr = g.gate == SPT_GATE_SIGMOID ? (const __nv_bfloat16*)w_r : nullptr;
    a.cb_out = (__nv_bfloat16*)dx;
    a.cb_ctr = b.side_ctr;
    a.cb_k = g.k;
    a.cb_drain = drain ? 1 : 0;
  };
  cudaStream_t sd = s;   // stream of the dW1 / dW_R launches (bwd_streams: side stream 1)
  cudaStream_t sd2 = s;  // stream of the dW2 launch (bwd_streams: side stream 2)
  auto run_dw = [&]() -> cudaError_t {
    {  // a9: dW1_b = dZ_b^T X[bucket_b]   (M = m'*bw features: <= 2 halves, or 256-feature tiles)
      TcArgs a{};
      base_args(a, g, r);
      set_side(a, false);
      bool ok = make_tmap_bf16_2d(&a.ta, b.dz, g.rows_cap, (uint64_t)g.mp * g.bw,
                                  (uint64_t)g.mp * g.bw, 64, kind_bk(K_DW1)) &&
                make_tmap_bf16_2d(&a.tb, x, g.T, g.d, g.d, 64, 1);
      if (g.split) {
        ok = ok && make_tmap_bf16_2d(&a.ta2, lo_half(b.dz, nz), g.rows_cap, (uint64_t)g.mp * g.bw,
                                     (uint64_t)g.mp * g.bw, 64, kind_bk(K_DW1));
        a.aux2_lo = lo_half(x, ntd);
      }
      a.BN = 256;
      a.MH = (int)std::min<int64_t>(2, ceil_div(g.mp * g.bw, 128));
      a.nu = (int)ceil_div(g.mp * g.bw, 256);
      a.dw_ng = dw_group(a.NT, K_DW1);
      a.aux2 = x;
      a.out = dw1;
      a.acc_mode = accumulate;
      TRY(launch<K_DW1>(a, g.G * a.nu * a.NT, sd));
      if (side && getenv("SPT_FFN_SIDE_DEBUG")) {  // diagnostics: tokens claimed during dW1
        int n = 0;
        cudaMemcpyAsync(&n, b.side_ctr, 4, cudaMemcpyDeviceToHost, sd);
        cudaStreamSynchronize(sd);
        fprintf(stderr, "[spt-side] tokens claimed during dW1: %d of %lld\n", n, (long long)g.T);
      }
    }
    {  // a9: dW2_b = H~_b^T dY[bucket_b]
      TcArgs a{};
      base_args(a, g, r);
      set_side(a, true);
      bool ok = make_tmap_bf16_2d(&a.ta, b.h, g.rows_cap, g.bw, g.bw, 64, kind_bk(K_DW2)) &&
                make_tmap_bf16_2d(&a.tb, dy, g.T, g.d, g.d, 64, 1);
      if (g.split) {
        ok = ok && make_tmap_bf16_2d(&a.ta2, lo_half(b.h, nh), g.rows_cap, g.bw, g.bw, 64,
                                     kind_bk(K_DW2));
        a.aux2_lo = lo_half(dy, ntd);
      }
      a.BN = 256;
      a.MH = (int)std::min<int64_t>(2, ceil_div(g.bw, 128));
      a.nu = (int)ceil_div(g.bw, 256);
      a.dw_ng = dw_group(a.NT, K_DW2);
      a.aux2 = dy;
      a.out = dw2;
      a.acc_mode = accumulate;
      TRY(launch<K_DW2>(a, g.G * a.nu * a.NT, sd2));
    }
    return cudaSuccess;
  };
  auto run_dwr = [&]() -> cudaError_t {
    // f2: + lambda dL_balance/dx_R for every (token, block), into the dense dlogits
    if (lb) {
      cudaError_t e = launch_balance_grad(g, r, b.dlg, nullptr, sd);
      if (e != cudaSuccess) return e;
    }
    // a10: dW_R = dLogits^T X  (split-K, hi + lo bf16 halves of dlogit)
    if (sig || lb)
      return tc_dense_tn(g, b.dlg, x, b.dwr_part, b.n_split, dw_r, accumulate, sd,
                         g.split ? lo_half(x, ntd) : nullptr);
    if (!accumulate && cudaMemsetAsync(dw_r, 0, (size_t)g.G * g.d * 4, sd) != cudaSuccess)
      return cudaErrorUnknown;
    return cudaSuccess;
  };
  auto run_dx = [&]() -> cudaError_t {  // a8: dXp = dZ W1_b (partials)
    TcArgs a{};
    base_args(a, g, r);
    bool ok = make_tmap_bf16_2d(&a.ta, b.dz, g.rows_cap, (uint64_t)g.mp * g.bw,
                                (uint64_t)g.mp * g.bw, 64, 128) &&
              make_tmap_bf16_2d(&a.tb, w1, (uint64_t)g.mp * g.D, g.d, g.d, 64, 64);
    ok = ok && make_tmap_bf16_2d(&a.tc, b.part, g.rows_cap, g.d, g.d, 64, 32);
    if (g.split)  // fp32 partial rows (generic epilogue), K streamed in three passes
      ok = ok && make_tmap_bf16_2d(&a.ta2, lo_half(b.dz, nz), g.rows_cap, (uint64_t)g.mp * g.bw,
                                   (uint64_t)g.mp * g.bw, 64, 128) &&
           make_tmap_bf16_2d(&a.tb2, lo_half(w1, (int64_t)g.mp * g.D * g.d), (uint64_t)g.mp * g.D,
                             g.d, g.d, 64, 64);
    a.BN = 256;
    a.out = b.part;
    a.unit_offsets = b.unit_offsets;
    a.kstream = g.mp * g.bw > 256 || g.split;  // the K = m' bw slab no longer fits smem: stream K
    if (a.kstream) {
      TRY(launch<K_DX>(a, up * a.NT, s));
    } else {
      TRY(launch_bres<K_DX>(a, units_upper(g), s));
    }
    return cudaSuccess;
  };
  cudaError_t e;
  if (side) {  // dX partials, then dW1 / dW2 (+ the combine as their side work), dW_R
    if ((e = run_dx()) != cudaSuccess) return e;
    if (cudaMemsetAsync(b.side_ctr, 0, 4, s) != cudaSuccess) return cudaErrorUnknown;
    if ((e = run_dw()) != cudaSuccess) return e;
    if ((e = run_dwr()) != cudaSuccess) return e;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (dgate_out) return launch_gather_dgate(g, r, b.dgate, dgate_out, s);
    return cudaSuccess;
  }
  // the weight gradients (dW1, dW2, dW_R) on a side stream concurrently with dX +
  // the grad-input combine (they share only dA's outputs) at small shapes, where
  // each kernel alone leaves SMs idle (bwd_streams_enabled)
  ForkJoin fj{};
  const bool fork = bwd_streams_enabled(g) && !lo && !lb;  // lb: dX reads the dlogits dW_R's branch adds to
  if (fork) {
    if ((e = fork_side(s, fj)) != cudaSuccess) return e;
    sd = fj.side;
    sd2 = fj.side2;
  }
  if (!lo && (e = run_dw()) != cudaSuccess) return e;
  if ((e = run_dwr()) != cudaSuccess) return e;
  if (fork && (e = join_side2(fj)) != cudaSuccess) return e;
  // all of dw1 | dw2 | dw_r are final here: a data-parallel caller can start the
  // gradient all-reduce at this event while dX is computed below
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (!lo && dw_ev && cudaEventRecord(dw_ev, sd) != cudaSuccess) return cudaErrorUnknown;
  sd = sd2 = s;
  if ((e = run_dx()) != cudaSuccess) return e;
  if (lb) {
    // router term of dx from the dense dlogits (task + balance): dXR = dLogits W_R
    TcArgs a{};
    base_args(a, g, r);
    bool ok = make_tmap_bf16_2d(&a.ta, b.dlg, (uint64_t)2 * g.T, g.gpad, g.gpad, 64, 128) &&
              make_tmap_bf16_2d(&a.tb, w_r, g.G, g.d, g.d, 64, 64);
    a.BN = 256;
    a.out = b.lb_x;
    TRY(launch<K_DXR>(a, (int)ceil_div(g.T, 128) * a.NT, s));
    e = lo ? lora_bwd_finish(g, r, b, *lo, x, dy, b.lb_x, nullptr, dx, s)
           : launch_combine_bwd_dense(g, r, b.part, b.lb_x, dx, s);
  } else {
    e = lo ? lora_bwd_finish(g, r, b, *lo, x, dy, nullptr, w_r, dx, s)
           : launch_combine_bwd(g, r, b.part, b.dlogit, w_r, dx, s);
  }
  if (e != cudaSuccess) return e;
  if (fork && (e = join_side(s, fj)) != cudaSuccess) return e;
  // LoRA: every gradient (dw_r and the factors) is final only here
  if (lo && dw_ev && cudaEventRecord(dw_ev, s) != cudaSuccess) return cudaErrorUnknown;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (dgate_out) return launch_gather_dgate(g, r, b.dgate, dgate_out, s);
  return cudaSuccess;
}

}  // namespace spt
