/*
 * spt_ffn.h -- C ABI of the B200 (sm_100a) routed-FFN library libspt_ffn.so.
 *
 * SPT's routed FFN (arXiv 2312.10365, §4.2 "Dynamic routing", PAPER.md:426-437,
 * and §5.2 Algorithm 4 "The procedure of BSpMV"):
 *   - the FFN H = act(X W_I), Y = H W_O (Eq. 4) is split into
 *     G blocks of bw = D/G adjacent hidden units (rows of W_I^T / rows of W_O,
 *     Fig. 6a);
 *   - a route network x_R = x W_R (W_R in R^{d x G}) picks, per token, the k
 *     blocks with the largest |x_R|;
 *   - tokens are batched per activated block, each block runs as a dense GEMM
 *     and the block outputs are accumulated per token (Alg. 4).
 * The three compute calls map to the paper's problem statement (Alg. 4 inputs:
 * token sequence X, weights W_I, W_O, Indices of activated blocks; output Y)
 * plus the route network and the backward pass the router training needs
 * ("trained along with the FFN").
 *
 * Conventions (all calls):
 *   - Every tensor pointer is a DEVICE pointer (cudaMalloc'd or equivalent),
 *     row-major and contiguous; 16-byte aligned.  The caller owns all memory;
 *     the library never allocates device memory and retains no pointer after
 *     a call returns.
 *   - `stream` is a cudaStream_t (passed as void*); every call only enqueues
 *     work on it and never synchronises the host.  NULL = legacy default stream.
 *   - Argument validation happens before any launch; on error nothing is
 *     enqueued.  Launch failures return SPT_ERR_CUDA; faults inside kernels
 *     surface at the caller's next synchronisation.  No C++ exception crosses
 *     the ABI.
 *   - NaN / Inf inputs are not checked; IEEE propagation applies.  Routing
 *     stays total-ordered (see spt_ffn_route).
 *
 * Shapes (T tokens, d = d_model, D = d_ff, G blocks, bw = D/G, k = top_k,
 * m' = 2 for SwiGLU (gate and up projections) else 1):
 *   x, y, dy, dx : [T, d]        act dtype (fp32 or bf16)
 *   w1           : [D, d]  (SwiGLU: [2, D, d] = gate rows then up rows)
 *                  = W_I^T of Eq. 4; block b = rows [b*bw, (b+1)*bw)
 *   w2           : [D, d]  = W_O; block b = rows [b*bw, (b+1)*bw)
 *   w_r          : [G, d]  = W_R^T (route network)
 *   dw1, dw2, dw_r : fp32, shapes of w1, w2, w_r
 */
#ifndef SPT_FFN_H_
#define SPT_FFN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPT_FFN_ABI_VERSION 5
/* Height of a bucket tile: tile_offsets counts ceil(n_b / SPT_TILE_M) per block. */
#define SPT_TILE_M 128

typedef enum {
  SPT_OK = 0,
  SPT_ERR_INVALID_ARGUMENT = 1, /* NULL pointer, T < 0, k < 1, k > G, D % G != 0, dims <= 0 */
  SPT_ERR_UNSUPPORTED = 2,      /* G > 256, d % 64, bw % 16, non-sm_100 device; bf16: SwiGLU
                                   with bw % 64 (fp32 then runs its SIMT kernels).  Any block width
                                   otherwise (m' bw > 256 -- the paper's G = 4 / 8 blocks,
                                   PAPER.md:436 -- runs unit / feature-tiled GEMMs) */
  SPT_ERR_WORKSPACE_TOO_SMALL = 3,
  SPT_ERR_CUDA = 4              /* a CUDA launch / API call failed */
} spt_status;

typedef enum { SPT_F32 = 0, SPT_BF16 = 1 } spt_dtype;
/* SPT_ACT_RELU: Eq. 4; SPT_ACT_GELU: z*Phi(z) (erf form); SPT_ACT_SWIGLU:
 * silu(x w_gate) * (x w_up), block b covers the gate and up rows of units in b. */
typedef enum { SPT_ACT_RELU = 0, SPT_ACT_GELU = 1, SPT_ACT_SWIGLU = 2 } spt_act;
/* SPT_GATE_SIGMOID: each activated block's output is scaled by sigmoid(x_R[b])
 * (gives the router a gradient); SPT_GATE_NONE: plain 0/1
 * masking exactly as Alg. 4, router receives no gradient. */
typedef enum { SPT_GATE_SIGMOID = 0, SPT_GATE_NONE = 1 } spt_gate;

typedef struct {
  int64_t n_tokens; /* T >= 0 (batch x sequence flattened) */
  int32_t d_model;  /* d */
  int32_t d_ff;     /* D, divisible by n_blocks */
  int32_t n_blocks; /* G <= 256 */
  int32_t top_k;    /* k = G' in [1, G] (beta = k/G) */
  int32_t dtype;    /* spt_dtype: storage dtype of x, y, dy, dx, w1, w2, w_r */
  int32_t act;      /* spt_act */
  int32_t gate;     /* spt_gate */
  /* lambda >= 0 (finite): spt_ffn_backward adds the gradient of lambda * L_balance
   * (spt_ffn_balance_loss) to dw_r and dx.  0 disables it.  (ABI 2) */
  float balance_weight;
  /* SPT_FFN_* option bits (ABI 5); unknown bits -> SPT_ERR_INVALID_ARGUMENT. */
  uint32_t flags;
} spt_ffn_desc;

/* desc.flags: option bits (ABI 5).  SPT_FFN_DETERMINISTIC requests bitwise
 * reproducible results; every path of this library already is (the k-way sum
 * of a token's per-block outputs, Alg. 4 line 5, runs in fp32 in ascending
 * block id), so the bit is accepted and changes nothing.  It
 * is reserved so that a future non-deterministic fast path stays opt-out. */
#define SPT_FFN_DETERMINISTIC 1u

/* Routing decision and bucket layout (all DEVICE buffers, caller-allocated).
 * Written by spt_ffn_route, read by spt_ffn_forward / spt_ffn_backward. */
typedef struct {
  float* logits;         /* [T, G] fp32: x_R = x W_R.  Output; input if SPT_ROUTE_LOGITS_IN */
  int32_t* topk_idx;     /* [T, k]: activated block ids of each token, ascending */
  float* topk_gate;      /* [T, k]: gate g of each (token, block) pair (1.0 for GATE_NONE) */
  int32_t* block_offsets;/* [G+1]: exclusive prefix sum of bucket sizes n_b; [G] = T*k */
  int32_t* bucket_token; /* [T*k]: block-major, ascending token id within a block
                            (the order X[Mask_T] of Alg. 4 line 3 visits tokens) */
  float* bucket_gate;    /* [T*k]: gate of each bucket entry */
  int32_t* pair_slot;    /* [T*k]: pair_slot[t*k+j] = bucket position of (t, topk_idx[t,j]) */
  int32_t* tile_offsets; /* [G+1]: exclusive prefix of ceil(n_b / SPT_TILE_M) (device tile schedule) */
} spt_route_buf;

#define SPT_ROUTE_LOGITS_IN 1u   /* spt_ffn_route: skip x W_R, route the given r->logits */
#define SPT_BWD_ACCUMULATE_DW 1u /* spt_ffn_backward: dw1/dw2/dw_r += grads instead of = */

/* Bytes of the stash (forward -> backward activations, must survive unchanged
 * between the two calls) and of the per-call scratch workspace, for `desc`.
 * Pure host function; needs no device.  Returns SPT_ERR_INVALID_ARGUMENT on a
 * bad descriptor or NULL out-pointer. */
spt_status spt_ffn_sizes(const spt_ffn_desc* desc, size_t* stash_bytes, size_t* workspace_bytes);

/* Route network + per-token top-k + token bucketing (Alg. 4
 * lines 2-3).  x: [T,d]; w_r: [G,d] (may be NULL with SPT_ROUTE_LOGITS_IN).
 * Selection: the k blocks with the largest |logit|, compared as the uint32 bit
 * pattern of |logit| (sign cleared; NaN ranks above +Inf), ties -> lower block
 * id; ids emitted ascending.  Gate = sigmoid(logit) (fp32) or 1.
 * Writes every field of *r.  ws: >= workspace_bytes from spt_ffn_sizes. */
spt_status spt_ffn_route(const spt_ffn_desc* desc, const void* x, const void* w_r,
                         unsigned flags, const spt_route_buf* r, void* ws, size_t ws_bytes,
                         void* stream);

/* Routed FFN forward (Alg. 4 with accumulation; Fig. 6a):
 *   y_t = sum_{b in S_t, ascending b} g_{t,b} * act(x_t W1_b^T) W2_b
 * Reads r (from spt_ffn_route); writes y [T,d] and stash (pre-activations and
 * gated hidden activations of every (token, block) pair, for the backward). */
spt_status spt_ffn_forward(const spt_ffn_desc* desc, const void* x, const void* w1,
                           const void* w2, const spt_route_buf* r, void* y, void* stash,
                           void* ws, size_t ws_bytes, void* stream);

/* Backward of spt_ffn_forward (routing held fixed; no gradient through the
 * top-k selection).  Given dy = dL/dy [T,d]:
 *   dx   [T,d]   = sum_b dZ_b W1_b + sum_b dlogit_b w_r[b]       (act dtype)
 *   dw1, dw2     = per-block weight gradients (fp32, rows of inactive blocks 0)
 *   dw_r [G,d]   = sum over pairs of dlogit * x_t  (fp32; 0 for GATE_NONE)
 *                  + lambda * sum_t dL_balance/dx_R[t,:]^T x_t  (lambda = balance_weight;
 *                  dx likewise gets + lambda * dL_balance/dx_R[t,:] w_r)
 *   dgate [T,k]  = dL/dg per pair (fp32, optional: may be NULL)
 * with dlogit = dgate * g (1 - g) for GATE_SIGMOID.  stash must be the one the
 * matching spt_ffn_forward wrote.  flags: SPT_BWD_ACCUMULATE_DW.
 * dw_event: optional cudaEvent_t (void*, may be NULL).  The weight gradients
 * dw1, dw2, dw_r are computed first; the library records dw_event on `stream`
 * as soon as all three are final and only then computes dx.  A data-parallel
 * caller can start the gradient all-reduce on another stream at that event so
 * it overlaps the grad-input kernels.
 * Streams: at small shapes (the dW1 GEMM has <= 4 tiles per SM; environment
 * SPT_FFN_BWD_STREAMS=1/0 forces it on / off) the weight-gradient kernels run on
 * two library-owned streams of the current device, forked from `stream` after
 * the dA kernel and joined back into `stream` before the call's last kernel;
 * dw_event is then recorded on the first of them once all three gradients are
 * final.  Every output is complete, as always, when `stream` reaches the point
 * after this call (the call stays capturable into a CUDA graph). */
spt_status spt_ffn_backward(const spt_ffn_desc* desc, const void* x, const void* w1,
                            const void* w2, const void* w_r, const spt_route_buf* r,
                            const void* stash, const void* dy, void* dx, float* dw1, float* dw2,
                            float* dw_r, float* dgate, unsigned flags, void* ws, size_t ws_bytes,
                            void* dw_event, void* stream);

/* Load-balancing loss of a routing decision (the paper
 * names "similar activation rates", without a formula; SPEC
 * S:342-349 defines it, reading c18):
 *   L = G * sum_g f_g * pbar_g,  f_g = n_g / (T k),  pbar_g = (1/T) sum_t softmax(x_R[t])_g
 * (L = 1 for perfectly uniform routing).  Reads r->logits and r->block_offsets
 * (written by spt_ffn_route); writes the fp32 scalar *loss (DEVICE pointer) on
 * `stream`.  Deterministic.  T = 0 writes 0.  Its gradient enters
 * spt_ffn_backward through desc->balance_weight (every block's logit, not
 * just the selected ones; f carries no gradient). */
spt_status spt_ffn_balance_loss(const spt_ffn_desc* desc, const spt_route_buf* r, float* loss,
                                void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * LoRA-wrapped routed FFN (ABI 3) -- the paper's
 * fine-tuning mode.  LoRA (Eq. 5) writes a projection
 * Y = XW as Y = XW + XBC with W frozen and B in R^{d x r}, C in R^{r x h}
 * trained; SPT wraps both FFN projections (Model Adapter log, PAPER.md:
 * 1323-1328; rank "d_lora", default 16) and routes the FFN
 * (§4.2): block b uses the hidden units [b bw, (b+1) bw) of W_I + B_I C_I and
 * W_O + B_O C_O (reading c19).  Per token t, block b in S_t:
 *   z = x_t W_I[:,b] + (x_t B_I) C_I[:,b],   h~ = g act(z)
 *   y_t = sum_b h~ W_O[b,:] + (sum_b h~ B_O[b,:]) C_O
 * Storage (all DEVICE, row-major, act dtype = bf16; m' = 2 for SwiGLU, whose
 * gate and up projections each carry their own factors):
 *   b1 : [m', r, d]  = B_I^T            c1 : [m', D, r] = C_I^T  (block b = rows)
 *   b2 : [D, r]      = B_O (block b = rows)     c2 : [r, d]  = C_O
 * Gradients (fp32, same shapes): db1, dc1, db2, dc2.
 * Support: bf16 only (SPT_ERR_UNSUPPORTED for fp32); 1 <= r and m' r <= 64.
 * Numerics: x B_I and dy C_O^T enter the tensor-core GEMMs rounded once to
 * bf16 (an extra 64-wide K stage of FWD1 / dA); the reductions over a token's
 * blocks (sum_b h~ B_O, sum_b dZ C_I^T) are fp32 in ascending block order. */
typedef struct {
  int32_t rank;   /* r */
  const void* b1; /* [m', r, d] */
  const void* c1; /* [m', D, r] */
  const void* b2; /* [D, r]     */
  const void* c2; /* [r, d]     */
} spt_lora;

typedef struct {
  float* db1; /* [m', r, d] */
  float* dc1; /* [m', D, r] */
  float* db2; /* [D, r]     */
  float* dc2; /* [r, d]     */
} spt_lora_grads;

/* Stash / workspace bytes of the LoRA-wrapped calls (>= spt_ffn_sizes').  Host only.
 * SPT_ERR_INVALID_ARGUMENT: bad desc, rank < 1, NULL out-pointer;
 * SPT_ERR_UNSUPPORTED: fp32 dtype or m' rank > 64. */
spt_status spt_ffn_lora_sizes(const spt_ffn_desc* desc, int32_t rank, size_t* stash_bytes,
                              size_t* workspace_bytes);

/* Forward of the LoRA-wrapped routed FFN (formula above; routing from
 * spt_ffn_route).  w1, w2 are the frozen W_I^T, W_O.  Writes y [T,d] and the
 * stash (must survive unchanged until spt_ffn_lora_backward). */
spt_status spt_ffn_lora_forward(const spt_ffn_desc* desc, const void* x, const void* w1,
                                const void* w2, const spt_lora* lora, const spt_route_buf* r,
                                void* y, void* stash, void* ws, size_t ws_bytes, void* stream);

/* Backward of spt_ffn_lora_forward (W_I, W_O frozen: no dW1 / dW2; routing
 * fixed).  Writes dx [T,d] (act dtype), the factor gradients *grads, dw_r
 * (router, as spt_ffn_backward incl. desc->balance_weight) and optionally
 * dgate [T,k].  flags: SPT_BWD_ACCUMULATE_DW adds into the factor gradients
 * and dw_r.  grad_event (optional cudaEvent_t) is recorded once every gradient
 * (factors and dw_r) is final -- for a data-parallel all-reduce. */
spt_status spt_ffn_lora_backward(const spt_ffn_desc* desc, const void* x, const void* w1,
                                 const void* w2, const void* w_r, const spt_lora* lora,
                                 const spt_route_buf* r, const void* stash, const void* dy,
                                 void* dx, const spt_lora_grads* grads, float* dw_r, float* dgate,
                                 unsigned flags, void* ws, size_t ws_bytes, void* grad_event,
                                 void* stream);

/* ---------------------------------------------------------------------------
 * Sparse-MHA top-L selection (ABI 4): SPT's bucket-sort
 * top-L over product-quantisation codes (§4.1, §5.1
 * Algorithm 3).  Each query / key vector is given as its M
 * codeword ids (one per codebook); similarity is the integer
 * count of shared codewords, Eq. 3:
 *   s(q, k) = sum_m I[codes_q[q, m] == codes_k[k, m]]  in {0..M}
 * and per query Algorithm 3 fills M+1 buckets of capacity L in ascending key
 * order (a full bucket's slot L-1 is overwritten by each further key, line 7),
 * then reads buckets from score M down until L keys are collected.  Readings
 * (DESIGN.md c20-c23): empty buckets are skipped (line 11 as `while`); a
 * bucket is read for min(#keys, L) slots; causal rows see keys k <= q only and
 * rows with fewer than L candidates are padded with -1.  The result is the
 * exact top-L by Eq. 3 (ties: a bucket's first keys, plus its last key when it
 * overflowed) -- integer, deterministic, bit-exact.
 * Layout (DEVICE, row-major): codes_q [H, n_q, M] uint8, codes_k [H, n_k, M]
 * uint8, indices [H, n_q, L] int32 (bucket M's keys first; = the CSR column
 * indices of Fig. 7 with indptr [0, L, 2L, ...]). */
typedef struct {
  int32_t n_heads;     /* H >= 0 independent (sequence, head) problems */
  int32_t n_q;         /* queries per head >= 0 */
  int32_t n_k;         /* keys per head >= 0 */
  int32_t n_codebooks; /* M in [1, 31] (the paper: head_dim / 8) */
  int32_t n_codewords; /* E in [1, 256]: every code is < E (the paper: 16);
                          E <= 16 packs 8 codes per 32-bit word (half the compare work).
                          Codes >= E are a caller error (results unspecified, no fault). */
  int32_t top_l;       /* L >= 1 (the paper: lambda n) */
  int32_t causal;      /* 0 | 1: look-ahead mask applied before bucketing */
} spt_topl_desc;

/* Top-L key indices of every query.  SPT_ERR_INVALID_ARGUMENT: NULL desc, a
 * negative size, M outside [1, 31], E outside [1, 256], L < 1, causal not 0/1,
 * a NULL pointer with a non-empty problem; SPT_ERR_UNSUPPORTED: the key codes
 * of one head plus the per-warp score rows plus the kernel's 40,960 bytes of
 * static bucket state exceed the 227 KB of shared memory of one CTA
 * (n_k (4 ceil(M/c) + 16) + 40960 bytes, c = 8 codes per word for E <= 16
 * else 4; ceil(M/c) = 3 is stored as 4), non-sm_100 device.  Asynchronous on
 * stream. */
spt_status spt_mha_topl(const spt_topl_desc* desc, const uint8_t* codes_q, const uint8_t* codes_k,
                        int32_t* indices, void* stream);

/* Static string for a status code (never NULL). */
const char* spt_status_string(spt_status s);

/* SPT_FFN_ABI_VERSION of the loaded library. */
int spt_ffn_abi_version(void);

/* Number of this library's kernels launched by the calling process so far
 * (host-side counter, for the benchmark's gpu_launches report). */
uint64_t spt_ffn_launch_count(void);

/* Optional instrumentation: when enabled, every kernel the library launches is
 * bracketed by a pair of CUDA events on its launch stream (small overhead).
 * spt_ffn_profile_enable(1) clears previous records; spt_ffn_profile_read
 * waits for the recorded events, writes "name count total_ms\n" lines (one per
 * kernel name, first-launch order, NUL-terminated, truncated to len) into buf,
 * clears the records and returns the full text length (or -1 on a CUDA error). */
spt_status spt_ffn_profile_enable(int on);
int64_t spt_ffn_profile_read(char* buf, size_t len);

#ifdef __cplusplus
}
#endif
#endif /* SPT_FFN_H_ */
