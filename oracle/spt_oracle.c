/*
 * spt_oracle.c -- CPU fp64 ORACLE for SPT's routed FFN (arXiv 2312.10365).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2312_10365_b200/csrc) and never reads anything produced by it.
 *
 * Plain, slow, obviously-correct loops in fp64.  Tensor inputs arrive as
 * double arrays (the fp32 / bf16 input bits widened exactly; fp64 lets the
 * finite-difference pins perturb them by 1e-6); every
 * arithmetic step below is done in double with NO intermediate rounding
 * (SURVEY.md §8(c) reading c13).  OpenMP only parallelises independent
 * outer loops (tokens, or blocks for weight gradients); the arithmetic inside
 * each loop body is written in the paper's order.
 *
 * Notation (Eq. 4; §4.2 "Dynamic routing", 433-437):
 *   X  [T,d]          token matrix, one row x_t per token
 *   W_I = w1^T,  w1 [D,d]   (SwiGLU: w1 [2,D,d] = gate rows, up rows)
 *   W_O = w2,    w2 [D,d]
 *   W_R = w_r^T, w_r[G,d]   route network x_R = x W_R
 *   block b = hidden units [b*bw, (b+1)*bw), bw = D/G    (c5)
 *
 * Readings of the paper used here:
 *   c1  Alg. 4 line 5 "Y[Mask_T] <- H W_O[i]" accumulates:
 *       y_t = sum over the token's activated blocks (Fig. 6a).
 *   c2  gate: SIGMOID g = sigma(x_R[b]) or NONE g = 1 (paper-literal).
 *   c3  selection by largest |x_R|, c4: ties by the uint32 bit
 *       pattern of |logit| (sign cleared) descending, then lower block id.
 *   c6  no activation after W_O (Eq. 4; PAPER.md:430's "ReLU(xW_O)" is a typo).
 *   c7  activation: ReLU (Eq. 4), GELU-erf, or SwiGLU silu(z_g)*z_u.
 *   c8  no biases.   c11  no gradient through the selection.
 *   c12 k-way sum in ascending block id.
 *
 * Parity pins: see tests/test_oracle_*.py (dense Eq. 4 special case, masked
 * dense O1 and Alg.4-literal O3 cross-checks, finite differences, Euler
 * identities, SPEC S:328 worked example, brute-force sort).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { ACT_RELU = 0, ACT_GELU = 1, ACT_SWIGLU = 2 };
enum { GATE_SIGMOID = 0, GATE_NONE = 1 };

int spt_oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ---------------------------------------------------------------- helpers */

static double sigmoid(double z) { return 1.0 / (1.0 + exp(-z)); }

/* GELU with the exact erf form z*Phi(z) (BERT's activation; reading c7). */
static double gelu(double z) { return 0.5 * z * (1.0 + erf(z / sqrt(2.0))); }
static double gelu_grad(double z) {
  const double pi = 3.14159265358979323846;
  return 0.5 * (1.0 + erf(z / sqrt(2.0))) + z * exp(-0.5 * z * z) / sqrt(2.0 * pi);
}
static double silu(double z) { return z * sigmoid(z); }
static double silu_grad(double z) {
  double s = sigmoid(z);
  return s * (1.0 + z * (1.0 - s));
}

/* |logit| as the uint32 bit pattern with the sign bit cleared (reading c4). */
static uint32_t abs_bits(float v) {
  uint32_t u;
  memcpy(&u, &v, 4);
  return u & 0x7fffffffu;
}

/* ------------------------------------------------------------ a1: router */
/* logits[t][b] = sum_c x[t][c] * w_r[b][c]   i.e. x_R = x W_R */
void spt_oracle_router(int64_t T, int d, int G, const double* x, const double* w_r,
                       double* logits) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t)
    for (int b = 0; b < G; ++b) {
      double s = 0.0;
      for (int c = 0; c < d; ++c) s += (double)x[t * d + c] * (double)w_r[(int64_t)b * d + c];
      logits[t * G + b] = s;
    }
}

/* ------------------------------------------------------- a2: top-k select */
/* "we set the top G' entries in x_R with the largest magnitude ... as
 * activated".  Decision made on fp32 logits (the kernel's
 * precision, reading c15).  Plain definition: sort all G (key, id) pairs by
 * key descending then id ascending, take the first k, emit ids ascending. */
typedef struct { uint32_t key; int id; } keyed_t;

static int cmp_desc_key_then_id(const void* pa, const void* pb) {
  const keyed_t* a = (const keyed_t*)pa;
  const keyed_t* b = (const keyed_t*)pb;
  if (a->key != b->key) return a->key > b->key ? -1 : 1; /* explicit compare: no unsigned negation */
  return a->id < b->id ? -1 : (a->id > b->id);
}
static int cmp_int(const void* pa, const void* pb) {
  int a = *(const int*)pa, b = *(const int*)pb;
  return (a > b) - (a < b);
}

int spt_oracle_topk(int64_t T, int G, int k, const float* logits, int32_t* topk_idx) {
  if (k < 1 || k > G) return 1; /* G' > G is a config error */
#pragma omp parallel
  {
    keyed_t* row = (keyed_t*)malloc(sizeof(keyed_t) * (size_t)G);
    int* sel = (int*)malloc(sizeof(int) * (size_t)k);
#pragma omp for schedule(static)
    for (int64_t t = 0; t < T; ++t) {
      for (int b = 0; b < G; ++b) {
        row[b].key = abs_bits(logits[t * G + b]);
        row[b].id = b;
      }
      qsort(row, (size_t)G, sizeof(keyed_t), cmp_desc_key_then_id);
      for (int j = 0; j < k; ++j) sel[j] = row[j].id;
      qsort(sel, (size_t)k, sizeof(int), cmp_int); /* emitted in ascending id */
      for (int j = 0; j < k; ++j) topk_idx[t * k + j] = sel[j];
    }
    free(row);
    free(sel);
  }
  return 0;
}

/* --------------------------------------------------- a3: token bucketing */
/* Alg. 4 lines 1-3: for block i, Mask_T = eq(Indices, i),
 * X_i = X[Mask_T].  Written out as the block-major list of (block, token)
 * pairs, tokens ascending inside a block (the order X[Mask_T] produces).
 *   block_offsets[b] = number of pairs in blocks < b  ([G] = T*k)
 *   bucket_token[p]  = token of pair p
 *   pair_slot[t*k+j] = p such that pair p is (topk_idx[t][j], t)
 *   tile_offsets[b]  = sum_{b'<b} ceil(n_b' / tile_m)                   */
int spt_oracle_bucket(int64_t T, int G, int k, const int32_t* topk_idx, int tile_m,
                      int32_t* block_offsets, int32_t* bucket_token, int32_t* pair_slot,
                      int32_t* tile_offsets) {
  int64_t p = 0, tiles = 0;
  for (int b = 0; b < G; ++b) {
    block_offsets[b] = (int32_t)p;
    tile_offsets[b] = (int32_t)tiles;
    int64_t n_b = 0;
    for (int64_t t = 0; t < T; ++t)       /* Mask_T = eq(Indices, b) */
      for (int j = 0; j < k; ++j)
        if (topk_idx[t * k + j] == b) {
          bucket_token[p] = (int32_t)t;
          pair_slot[t * k + j] = (int32_t)p;
          ++p;
          ++n_b;
        }
    tiles += (n_b + tile_m - 1) / tile_m;
  }
  block_offsets[G] = (int32_t)p;
  tile_offsets[G] = (int32_t)tiles;
  return p == T * k ? 0 : 1;
}

/* ------------------------------------------------- activation of a unit */
/* z: pre-activations of one hidden unit i (z[0]; SwiGLU: z[0]=gate, z[1]=up) */
static double act_value(int act, const double* z) {
  switch (act) {
    case ACT_RELU: return z[0] > 0.0 ? z[0] : 0.0;      /* Eq. 4 ReLU */
    case ACT_GELU: return gelu(z[0]);
    default: return silu(z[0]) * z[1];                  /* SwiGLU */
  }
}

/* pre-activation(s) z_i = x_t . w1[i] (and w1[D+i] for SwiGLU up) */
static void unit_preact(int act, int d, int D, const double* x_t, const double* w1, int64_t i,
                        double* z) {
  double s = 0.0;
  for (int c = 0; c < d; ++c) s += (double)x_t[c] * (double)w1[i * d + c];
  z[0] = s;
  if (act == ACT_SWIGLU) {
    s = 0.0;
    for (int c = 0; c < d; ++c) s += (double)x_t[c] * (double)w1[((int64_t)D + i) * d + c];
    z[1] = s;
  }
}

static double gate_of(int gate_mode, double logit) {
  return gate_mode == GATE_SIGMOID ? sigmoid(logit) : 1.0;
}

/* ---------------------------------------------- a4-a6: forward (O2 form) */
/* y_t = sum_{b in S_t, ascending} g_{t,b} * sum_{i in b} act(z_{t,i}) w2[i]
 * i.e. Eq. 4 restricted to the activated hidden units (Fig. 6a,
 * PAPER.md:430-431), each block's output accumulated (reading c1), scaled by
 * the gate (reading c2).  logits: [T,G] fp64 (router output or fixed input).
 * tokens: optional subset (NULL = all T), y rows written for those tokens only.
 * h_out (optional, [T*k*bw]) receives g*act(z) per (t,j,unit) for diagnostics. */
void spt_oracle_forward(int64_t T, int d, int D, int G, int k, int act, int gate_mode,
                        const double* x, const double* w1, const double* w2,
                        const double* logits, const int32_t* topk_idx,
                        const int64_t* tokens, int64_t n_tokens, double* y) {
  const int bw = D / G;
  const int64_t n = tokens ? n_tokens : T;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t s = 0; s < n; ++s) {
    const int64_t t = tokens ? tokens[s] : s;
    const double* x_t = x + t * d;
    double* y_t = y + t * d;
    for (int c = 0; c < d; ++c) y_t[c] = 0.0;
    for (int j = 0; j < k; ++j) {
      const int b = topk_idx[t * k + j];
      const double g = gate_of(gate_mode, logits[t * G + b]);
      for (int64_t i = (int64_t)b * bw; i < (int64_t)(b + 1) * bw; ++i) {
        double z[2];
        unit_preact(act, d, D, x_t, w1, i, z);
        const double h = g * act_value(act, z);
        for (int c = 0; c < d; ++c) y_t[c] += h * (double)w2[i * d + c];
      }
    }
  }
}

/* -------------------------------------------- a7-a10: backward (O2 form) */
/* Given dY = dL/dY, with routing fixed (reading c11):
 *   dA_{t,i}    = dy_t . w2[i]                     (dA = dY W_O^T)
 *   dgate_{t,b} = sum_{i in b} dA_{t,i} act(z_{t,i})
 *   dH_{t,i}    = g_{t,b} dA_{t,i}
 *   dZ_{t,i}    = dH_{t,i} act'(z_{t,i})   (SwiGLU: dZg = dH zu silu'(zg), dZu = dH silu(zg))
 *   dlogit_{t,b}= dgate_{t,b} g (1-g)  (SIGMOID)  |  0  (NONE)
 *   dx_t        = sum_{b,i} dZ_{t,i} w1[i]  +  sum_b dlogit_{t,b} w_r[b]
 *   dw1[i]     += dZ_{t,i} x_t ;  dw2[i] += g act(z_{t,i}) dy_t ;
 *   dw_r[b]    += dlogit_{t,b} x_t
 * Per-token quantities (dx rows, dgate) for `tokens` (NULL = all); weight
 * gradients for `blocks` (NULL = all), each summing over ALL tokens of T
 * that activated the block.  dw1/dw2/dw_r rows of other blocks untouched. */
static void pair_grads(int act, int d, int D, int bw, const double* x_t, const double* dy_t,
                       const double* w1, const double* w2, int b, double g,
                       double* dz /* [bw*m'] */, double* hval /* [bw] g*act */,
                       double* dgate_out) {
  double dgate = 0.0;
  for (int u = 0; u < bw; ++u) {
    const int64_t i = (int64_t)b * bw + u;
    double z[2];
    unit_preact(act, d, D, x_t, w1, i, z);
    double dA = 0.0;
    for (int c = 0; c < d; ++c) dA += (double)dy_t[c] * (double)w2[i * d + c];
    const double a = act_value(act, z);
    dgate += dA * a;
    const double dH = g * dA;
    hval[u] = g * a;
    if (act == ACT_RELU) {
      dz[u] = z[0] > 0.0 ? dH : 0.0; /* ReLU'(0) = 0 */
    } else if (act == ACT_GELU) {
      dz[u] = dH * gelu_grad(z[0]);
    } else {
      dz[u] = dH * z[1] * silu_grad(z[0]);   /* d/dz_gate */
      dz[bw + u] = dH * silu(z[0]);          /* d/dz_up   */
    }
  }
  *dgate_out = dgate;
}

static double dlogit_of(int gate_mode, double dgate, double logit) {
  if (gate_mode != GATE_SIGMOID) return 0.0;
  const double g = sigmoid(logit);
  return dgate * g * (1.0 - g);
}

void spt_oracle_backward_tokens(int64_t T, int d, int D, int G, int k, int act, int gate_mode,
                                const double* x, const double* w1, const double* w2,
                                const double* w_r, const double* logits,
                                const int32_t* topk_idx, const double* dy,
                                const int64_t* tokens, int64_t n_tokens,
                                double* dx, double* dgate /* [T,k] */) {
  const int bw = D / G;
  const int mp = act == ACT_SWIGLU ? 2 : 1;
  const int64_t n = tokens ? n_tokens : T;
#pragma omp parallel
  {
    double* dz = (double*)malloc(sizeof(double) * (size_t)bw * mp);
    double* hv = (double*)malloc(sizeof(double) * (size_t)bw);
#pragma omp for schedule(dynamic, 4)
    for (int64_t s = 0; s < n; ++s) {
      const int64_t t = tokens ? tokens[s] : s;
      double* dx_t = dx + t * d;
      for (int c = 0; c < d; ++c) dx_t[c] = 0.0;
      for (int j = 0; j < k; ++j) {
        const int b = topk_idx[t * k + j];
        const double logit = logits[t * G + b];
        double dg;
        pair_grads(act, d, D, bw, x + t * d, dy + t * d, w1, w2, b, gate_of(gate_mode, logit),
                   dz, hv, &dg);
        dgate[t * k + j] = dg;
        for (int u = 0; u < bw; ++u) {
          const int64_t i = (int64_t)b * bw + u;
          for (int c = 0; c < d; ++c) dx_t[c] += dz[u] * (double)w1[i * d + c];
          if (mp == 2)
            for (int c = 0; c < d; ++c) dx_t[c] += dz[bw + u] * (double)w1[((int64_t)D + i) * d + c];
        }
        const double dl = dlogit_of(gate_mode, dg, logit);
        for (int c = 0; c < d; ++c) dx_t[c] += dl * (double)w_r[(int64_t)b * d + c];
      }
    }
    free(dz);
    free(hv);
  }
}

void spt_oracle_backward_blocks(int64_t T, int d, int D, int G, int k, int act, int gate_mode,
                                const double* x, const double* w1, const double* w2,
                                const double* logits, const int32_t* topk_idx, const double* dy,
                                const int32_t* blocks, int n_blocks,
                                double* dw1 /* [m',D,d] */, double* dw2 /* [D,d] */,
                                double* dw_r /* [G,d] */) {
  const int bw = D / G;
  const int mp = act == ACT_SWIGLU ? 2 : 1;
  const int nb = blocks ? n_blocks : G;
  /* parallel over (block, unit-chunk) work items would change nothing in the
   * math; keep it per block: each block's gradient is owned by one thread */
#pragma omp parallel
  {
    double* dz = (double*)malloc(sizeof(double) * (size_t)bw * mp);
    double* hv = (double*)malloc(sizeof(double) * (size_t)bw);
#pragma omp for schedule(dynamic, 1)
    for (int s = 0; s < nb; ++s) {
      const int b = blocks ? blocks[s] : s;
      for (int m = 0; m < mp; ++m)
        for (int u = 0; u < bw; ++u)
          memset(dw1 + (((int64_t)m * D) + (int64_t)b * bw + u) * d, 0, sizeof(double) * d);
      for (int u = 0; u < bw; ++u) memset(dw2 + ((int64_t)b * bw + u) * d, 0, sizeof(double) * d);
      memset(dw_r + (int64_t)b * d, 0, sizeof(double) * d);
      for (int64_t t = 0; t < T; ++t) {
        int j = -1;
        for (int jj = 0; jj < k; ++jj)
          if (topk_idx[t * k + jj] == b) j = jj;
        if (j < 0) continue;
        const double logit = logits[t * G + b];
        const double g = gate_of(gate_mode, logit);
        double dg;
        const double* x_t = x + t * d;
        const double* dy_t = dy + t * d;
        pair_grads(act, d, D, bw, x_t, dy_t, w1, w2, b, g, dz, hv, &dg);
        for (int u = 0; u < bw; ++u) {
          const int64_t i = (int64_t)b * bw + u;
          for (int m = 0; m < mp; ++m) {
            double* r = dw1 + ((int64_t)m * D + i) * d;
            const double v = dz[m * bw + u];
            for (int c = 0; c < d; ++c) r[c] += v * (double)x_t[c];
          }
          double* r2 = dw2 + i * d;
          for (int c = 0; c < d; ++c) r2[c] += hv[u] * (double)dy_t[c];
        }
        const double dl = dlogit_of(gate_mode, dg, logit);
        double* rr = dw_r + (int64_t)b * d;
        for (int c = 0; c < d; ++c) rr[c] += dl * (double)x_t[c];
      }
    }
    free(dz);
    free(hv);
  }
}

/* --------------------------------------------- cost model */
/* FLOPs of the activated-block GEMMs for one forward pass: every pair
 * (t, b) costs (m'+1) * d * bw multiply-adds.  Exposed so the test can pin
 * the ratio to the dense FFN at exactly beta = k/G. */
double spt_oracle_forward_gemm_flops(int64_t T, int d, int D, int G, int k, int act) {
  const int mp = act == ACT_SWIGLU ? 2 : 1;
  return 2.0 * (double)T * k * (double)(mp + 1) * d * (double)(D / G);
}

/* ------------------------------ load-balancing loss */
/* SPEC S:342-349 load_balance_loss (the paper names "similar activation
 * rates" in §4.2, but gives no formula):
 *   L = G * sum_g f_g * pbar_g
 *   f_g    = n_g / (T k): the share of the T*k (token, block) activations on
 *            block g (reading c18: the normalisation under which perfectly
 *            uniform routing gives exactly 1);
 *   pbar_g = (1/T) sum_t p_tg,  p_t = softmax(x_R[t])  ("pre").
 * f is piecewise constant in the logits (no gradient through the selection,
 * reading c11), so the gradient flows through p only:
 *   dL/dx_R[t,j] = (G/T) sum_g f_g dp_tg/dx_R[t,j] = (G/T) p_tj (f_j - sum_g f_g p_tg).
 * Returns L; writes dL/dx_R [T,G] when dlogit != NULL.  T = 0 returns 0. */
double spt_oracle_balance(int64_t T, int G, int k, const double* logits,
                          const int32_t* topk_idx, double* dlogit) {
  if (T <= 0) return 0.0;
  double* f = (double*)calloc((size_t)G, sizeof(double));
  double* pbar = (double*)calloc((size_t)G, sizeof(double));
  double* p = (double*)malloc((size_t)G * sizeof(double));
  for (int64_t t = 0; t < T; ++t)
    for (int j = 0; j < k; ++j) f[topk_idx[t * k + j]] += 1.0;
  for (int g = 0; g < G; ++g) f[g] /= (double)T * (double)k;
  for (int64_t t = 0; t < T; ++t) {  /* softmax row t, max-subtracted */
    const double* l = logits + t * G;
    double m = l[0], s = 0.0;
    for (int g = 1; g < G; ++g) m = l[g] > m ? l[g] : m;
    for (int g = 0; g < G; ++g) { p[g] = exp(l[g] - m); s += p[g]; }
    double fp = 0.0;
    for (int g = 0; g < G; ++g) { p[g] /= s; pbar[g] += p[g] / (double)T; fp += f[g] * p[g]; }
    if (dlogit)
      for (int j = 0; j < G; ++j) dlogit[t * G + j] = (double)G / (double)T * p[j] * (f[j] - fp);
  }
  double L = 0.0;
  for (int g = 0; g < G; ++g) L += f[g] * pbar[g];
  L *= (double)G;
  free(f);
  free(pbar);
  free(p);
  return L;
}
