// internal.h -- shared declarations of libspt_ffn (not part of the ABI).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/spt_ffn.h"

namespace spt {

constexpr int kTileM = SPT_TILE_M;   // bucket tile height (rows of a grouped-GEMM M tile)
constexpr int kRouteChunk = 256;     // tokens per bucketing chunk (one CTA)
constexpr int kTopkChunk = 32;       // tokens per top-k CTA (= per bucket-count row)
constexpr int kMaxBlocks = 256;      // G limit (routing keeps 8 logits per lane)

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Problem geometry derived from spt_ffn_desc.
struct Geom {
  int64_t T;
  int d, D, G, k, bw, mp;  // mp = m' (2 for SwiGLU)
  int dtype, act, gate;
  int64_t pairs;     // T*k
  int64_t rows_cap;  // padded bucket rows: T*k + G*kTileM (>= sum_b ceil(n_b/128)*128)
  int64_t n_chunks;  // ceil(T / kRouteChunk)
  int64_t n_sub;     // ceil(T / kTopkChunk): rows of the per-chunk bucket counts
  int gpad;          // G rounded up to 16 (router GEMM N, dense dlogit width)
  int esize;         // bytes per act element
  float lbw;         // load-balancing loss weight lambda (desc->balance_weight; 0 = off)
  // fp32 path on the bf16 tensor cores (reading c13'): every fp32 operand is
  // split into bf16 hi + lo and each GEMM sums the hi*hi, hi*lo and lo*hi
  // products in fp32.  Intermediates (Z, H~, dZ) are stored as bf16 hi / lo
  // halves (esize 4 = both halves, hi first), per-pair partials as fp32.
  bool split;
  bool tc() const { return dtype == SPT_BF16 || split; }  // tcgen05 kernels (else SIMT)
};

// Device-resident views of the routing decision (= spt_route_buf).
struct RouteView {
  float* logits;
  int32_t* topk_idx;
  float* topk_gate;
  int32_t* block_offsets;
  int32_t* bucket_token;
  float* bucket_gate;
  int32_t* pair_slot;
  int32_t* tile_offsets;
};

// Carved workspace / stash pointers.
struct Bufs {
  // stash (forward -> backward)
  void* z;        // [rows_cap, mp*bw] act: pre-activations (SwiGLU: gate | up)
  void* h;        // [rows_cap, bw] act: gated hidden g*act(z) (operand of W2 GEMM)
  // scratch
  void* part;     // [rows_cap, d] act: per-pair partial outputs (fwd Y, bwd dX)
  void* dz;       // [rows_cap, mp*bw] act
  float* da;      // [rows_cap, bw] f32 (SIMT path only)
  float* dlogit;  // [rows_cap] f32: dL/dlogit per padded bucket row
  float* dgate;   // [rows_cap] f32: dL/dgate per padded bucket row
  void* dlg;      // [2, T, gpad] bf16 (hi, lo) dense dlogits (tcgen05 dW_R GEMM)
  float* dwr_part;// [n_split, G, d] f32 split-K partials of dW_R
  int n_split;
  int32_t* chunk_counts;  // [n_sub, G] bucket counts per kTopkChunk tokens
  int32_t* chunk_base;    // [n_sub, G] exclusive prefix over the sub-chunks
  int32_t* n_b;           // [G]
  int32_t* side_ctr;      // [64] work counters (dW kernels' grad-input combine side work)
  // device tile schedules (stash: built by the forward, reused by the backward)
  int32_t* tile_list;     // [ceil(T*k/128) + G]: bucket tiles in (m-tile, block) order
  int32_t* unit_offsets;  // [G+2]: prefix of weight-resident work units per block; [G+1] = pair tiles
  int32_t* tile_block;    // [ceil(T*k/128) + G]: block of each 128-row bucket tile
  float* lb_part;         // [n_chunks, G] f32: per-chunk softmax sums (balance loss)
  void* lb_x;             // lambda != 0: bf16 [T, d] dense router term of dx (tcgen05 path)
                          //              f32 [T, G] lambda dL_balance/dx_R (SIMT path)
  // split (fp32 on tensor cores): bf16 hi | lo copies of the fp32 operands
  void* xs;               // [2][T, d]
  void* dys;              // [2][T, d]
  void* w1s;              // [2][m' D, d]
  void* w2s;              // [2][D, d]
  void* wrs;              // [2][G, d]
};

// split: the lo half of a hi | lo pair of bf16 tensors of n elements each
inline const void* lo_half(const void* hi, int64_t n) { return (const uint8_t*)hi + n * 2; }
inline void* lo_half(void* hi, int64_t n) { return (uint8_t*)hi + n * 2; }
bool simt_forced();  // SPT_FFN_SIMT=1: fp32 runs on the SIMT kernels (A/B of the split path)

int unit_mtiles();  // m-tiles per weight-resident unit (FWD2 / DX); SPT_FFN_UNIT_MT, default 128
constexpr int kRasterBlocks = 16;  // blocks per L2 raster group of the gathered-A GEMMs

void count_launch(int n = 1);

// Programmatic dependent launch (PDL): hot-path kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's grid is
// scheduled while its predecessor drains (its CTAs take SMs as the
// predecessor's exit and run their prologue -- barrier init, TMEM alloc,
// tensor-map prefetch).  Every such kernel executes pdl_wait() before its
// first access to global memory another kernel wrote or reads (it returns once
// the predecessor grid has completed and its writes are visible; a no-op when
// launched without the attribute); successors launch as its CTAs exit.
// Measured on B200 (round 2): an early pdl_trigger() at kernel start made the
// step 3-5 % slower (BERT 0.321 vs 0.305 ms, OPT 1.045 vs 0.996 ms), the
// exit-time trigger is neutral -- so the attribute is opt-in (SPT_FFN_PDL=1).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
// optional per-kernel CUDA-event profiling (spt_ffn_profile_enable / _read)
void prof_begin(const char* name, cudaStream_t s);
void prof_end(cudaStream_t s);

// routing (route.cu)
cudaError_t launch_router_simt(const Geom& g, const void* x, const void* w_r, float* logits,
                               cudaStream_t s);
cudaError_t launch_topk_bucket(const Geom& g, const RouteView& r, const Bufs& b, cudaStream_t s);

// SIMT path (simt_ffn.cu), any dtype
cudaError_t simt_forward(const Geom& g, const void* x, const void* w1, const void* w2,
                         const RouteView& r, void* y, const Bufs& b, cudaStream_t s);
cudaError_t simt_backward(const Geom& g, const void* x, const void* w1, const void* w2,
                          const void* w_r, const RouteView& r, const void* dy, void* dx,
                          float* dw1, float* dw2, float* dw_r, float* dgate_out, bool accumulate,
                          const Bufs& b, cudaEvent_t dw_ev, cudaStream_t s);

// shared HBM-bound kernels (combine.cu)
cudaError_t launch_combine_fwd(const Geom& g, const RouteView& r, const void* part, void* y,
                               cudaStream_t s);
cudaError_t launch_combine_bwd(const Geom& g, const RouteView& r, const void* part,
                               const float* dlogit, const void* w_r, void* dx, cudaStream_t s);
cudaError_t launch_gather_dgate(const Geom& g, const RouteView& r, const float* dgate_rows,
                                float* dgate_out, cudaStream_t s);
// the combine of dx with the dense router term dxr [T,d] (act dtype) replacing
// the sparse sum_j dlogit_j w_r[b_j] (load-balancing loss active)
cudaError_t launch_combine_bwd_dense(const Geom& g, const RouteView& r, const void* part,
                                     const void* dxr, void* dx, cudaStream_t s);

// load-balancing loss (balance.cu, reading c18)
cudaError_t launch_balance_loss(const Geom& g, const RouteView& r, const Bufs& b, float* loss,
                                cudaStream_t s);
// adds lambda dL/dx_R to the dense hi/lo bf16 dlogits (dlg != NULL) or writes it
// to a dense f32 [T,G] buffer (lbg != NULL)
cudaError_t launch_balance_grad(const Geom& g, const RouteView& r, void* dlg, float* lbg,
                                cudaStream_t s);
// SIMT path: dw_r += lbg^T x ; dx += lbg w_r (f32)
cudaError_t launch_balance_simt_dwr(const Geom& g, const float* lbg, const void* x, float* dw_r,
                                    cudaStream_t s);
cudaError_t launch_balance_simt_dx(const Geom& g, const float* lbg, const void* w_r, void* dx,
                                   cudaStream_t s);

// LoRA-wrapped routed FFN (lora.cu).  The LoRA terms of fc1
// enter FWD1 as extra K columns: X_aug = [x | hi(u) | lo(u) | 0] against
// W1_aug = [w1 | C_I^T | C_I^T | 0] with u = x B_I split into two bf16 halves
// (z = x W_I + u C_I with u carried to ~16 bits, so a ReLU sign decision sees
// the same z as the plain path); those of fc2 enter dA the same way
// (dY_aug = [dy | hi(v) | lo(v) | 0], W2_aug = [w2 | B_O | B_O | 0], v = dy C_O^T).
constexpr int kLoraK = 64;  // max m' r (width of the per-pair projection rows)
// augmented K columns: one 64-wide stage when the hi|lo halves fit, else two
inline int lora_ka(int mp, int r) { return 2 * mp * r <= 64 ? 64 : 128; }
struct LoraArgs {
  int r;                              // rank
  int ka;                             // augmented K columns (lora_ka)
  const void *b1, *c1, *b2, *c2;      // factors (bf16): [m',r,d], [m',D,r], [D,r], [r,d]
  float *db1, *dc1, *db2, *dc2;       // factor gradients (fp32, same shapes)
  bool accumulate;                    // gradients += instead of =
  // workspace
  void* xaug;    // [T, d+ka] bf16: fwd X_aug, bwd dY_aug
  void* waug;    // [m'D, d+ka] bf16: fwd W1_aug, bwd W2_aug
  float* uv;     // [T, m'r] f32: fwd U = x B_I, bwd V = dy C_O^T ([T, r])
  float* rowp;   // [chunks, rows_cap, 64] f32 per pair and 128-feature chunk: fwd q rows
                 // (h~ B_O[b]), bwd du rows (dZ C_I[b]); summed over chunks by the token reduce
  float* gpart;  // [tiles, m'+1, bw, r] f32 per-tile partials of dC_I (m' slabs) and dB_O
  float* spart;  // split-K partials of dB_I / dC_O
  int n_split_u, n_split_v;
  void* dhl;     // [2, T, upad] bf16 (hi, lo) dU rows for the dB_I GEMM
  // stash
  float* ust;    // [T, m'r] f32: u = x B_I (for dC_I)
  void* qhl;     // [2, T, qpad] bf16 (hi, lo) q = sum_b h~ B_O[b] for the dC_O GEMM
};
inline int lora_upad(const Geom& g, int r) { return (int)ceil_div(g.mp * r, 16) * 16; }
// per-pair rank-r rows are produced per 128-feature chunk of a block
inline int lora_chunks(const Geom& g) { return (int)ceil_div(g.bw, 128); }
inline int64_t lora_rows_stride(const Geom& g) { return g.rows_cap * kLoraK; }
inline int lora_qpad(int r) { return (int)ceil_div(r, 16) * 16; }

cudaError_t lora_fwd_prep(const Geom& g, const void* x, const void* w1, const LoraArgs& lo,
                          cudaStream_t s);
cudaError_t lora_fwd_finish(const Geom& g, const RouteView& r, const Bufs& b, const LoraArgs& lo,
                            void* y, cudaStream_t s);
cudaError_t lora_bwd_prep(const Geom& g, const void* dy, const void* w2, const LoraArgs& lo,
                          cudaStream_t s);
cudaError_t lora_bwd_grads(const Geom& g, const RouteView& r, const Bufs& b, const LoraArgs& lo,
                           cudaStream_t s);
// dx = sum_j dXp rows + router term (dense [T,d] if `dense`, else sum_j dlogit w_r[b_j]
// when w_r) + dU B_I^T; then dB_I = dU^T x and dC_O = q^T dy (tcgen05 split-K GEMMs)
cudaError_t lora_bwd_finish(const Geom& g, const RouteView& r, const Bufs& b, const LoraArgs& lo,
                            const void* x, const void* dy, const void* dense, const void* w_r,
                            void* dx, cudaStream_t s);

// sparse-MHA top-L selection (topl.cu, Alg. 3)
size_t topl_smem_bytes(int nk, int M, int E);  // dynamic smem of the top-L kernel
size_t topl_static_smem_bytes();               // its static smem (bucket counts / records)
int topl_max_score();
cudaError_t launch_topl(int H, int nq, int nk, int M, int E, int L, int causal,
                        const uint8_t* cq, const uint8_t* ck, int32_t* out, cudaStream_t s);

// tcgen05 path (tc_ffn.cu), bf16 only
bool tc_supported(const Geom& g);
// split (g.split): x / w_r are fp32 and the hi | lo copies go to b.xs / b.wrs
cudaError_t tc_router(const Geom& g, const void* x, const void* w_r, float* logits,
                      cudaStream_t s, const Bufs* b = nullptr);
// fp32 -> bf16 hi | lo halves (hi at dst, lo at lo_half(dst, n)), RNE both
cudaError_t launch_split_bf16(const float* src, void* dst, int64_t n, cudaStream_t s);
// dense split-K  out[G, d] (=|+=) A^T B  with A given as bf16 hi|lo halves [2, T, gpad]
// and B [T, d] bf16 (the dW_R GEMM; also dB_I / dC_O of the LoRA path)
cudaError_t tc_dense_tn(const Geom& g, const void* ahl, const void* bmat, float* part, int n_split,
                        float* out, bool accumulate, cudaStream_t s, const void* bmat_lo = nullptr);
int dense_tn_splits(const Geom& g);
// dense  out[T, d] (bf16) = A B  with A given as bf16 hi|lo halves [2, T, gpad] and
// B [G, d] bf16 (the dx router term of the balance loss; the du B_I^T term of LoRA)
cudaError_t tc_dense_nn(const Geom& g, const void* ahl, const void* bmat, void* out,
                        cudaStream_t s);
// lo != NULL: the LoRA-wrapped FFN (FWD1 on X_aug / W1_aug; dA on dY_aug / W2_aug;
// no dW1 / dW2 -- W is frozen -- and the LoRA factor gradients instead)
cudaError_t tc_forward(const Geom& g, const void* x, const void* w1, const void* w2,
                       const RouteView& r, void* y, const Bufs& b, cudaStream_t s,
                       const LoraArgs* lo = nullptr);
cudaError_t tc_backward(const Geom& g, const void* x, const void* w1, const void* w2,
                        const void* w_r, const RouteView& r, const void* dy, void* dx, float* dw1,
                        float* dw2, float* dw_r, float* dgate_out, bool accumulate, const Bufs& b,
                        cudaEvent_t dw_ev, cudaStream_t s, const LoraArgs* lo = nullptr);


// padded bucket row of pair (t, b = topk_idx[t,j]):
// tile_offsets[b]*128 + pair_slot[t*k+j] - block_offsets[b]
__device__ __forceinline__ int64_t pair_row(const RouteView& r, int64_t t, int k, int j) {
  const int b = r.topk_idx[t * k + j];
  return (int64_t)r.tile_offsets[b] * kTileM + (r.pair_slot[t * k + j] - r.block_offsets[b]);
}

}  // namespace spt
