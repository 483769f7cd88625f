// act.cuh -- activations of the routed FFN in fp32 (device), with derivatives.
//   ReLU   : Eq. 4; relu'(0) = 0
//   GELU   : z * Phi(z), exact erf form (BERT; reading c7)
//   SwiGLU : silu(z_gate) * z_up, silu(z) = z * sigmoid(z) (LLaMA; reading c7)
#pragma once
#include "internal.h"

namespace spt {

__device__ __forceinline__ float sigmoidf_(float z) { return 1.f / (1.f + expf(-z)); }
// fast variant for the bf16 tensor-core epilogues (outputs are rounded to bf16;
// __expf / fast reciprocal are accurate to a few fp32 ulp)
__device__ __forceinline__ float sigmoid_fast(float z) { return __frcp_rn(1.f + __expf(-z)); }

// g (1 - g) for g = sigmoid(z), as sigmoid(z) * sigmoid(-z) (accurate for |z| >> 1)
__device__ __forceinline__ float sigmoid_pair(float z) {
  return 1.f / ((1.f + expf(-z)) * (1.f + expf(z)));
}

// value of the activation for unit pre-activations (zg, zu); zu unused unless SwiGLU
template <bool kFast = false>
__device__ __forceinline__ float act_fwd(int act, float zg, float zu) {
  if (act == SPT_ACT_RELU) return zg > 0.f ? zg : 0.f;
  if (act == SPT_ACT_GELU) return 0.5f * zg * (1.f + erff(zg * 0.70710678118654752f));
  return zg * (kFast ? sigmoid_fast(zg) : sigmoidf_(zg)) * zu;
}

// act value a, and d a / d zg (dg), d a / d zu (du)
template <bool kFast = false>
__device__ __forceinline__ void act_fwd_bwd(int act, float zg, float zu, float& a, float& dg,
                                            float& du) {
  if (act == SPT_ACT_RELU) {
    a = zg > 0.f ? zg : 0.f;
    dg = zg > 0.f ? 1.f : 0.f;
    du = 0.f;
  } else if (act == SPT_ACT_GELU) {
    const float cdf = 0.5f * (1.f + erff(zg * 0.70710678118654752f));
    a = zg * cdf;
    dg = cdf + zg * 0.39894228040143268f * expf(-0.5f * zg * zg);
    du = 0.f;
  } else {
    const float s = kFast ? sigmoid_fast(zg) : sigmoidf_(zg);
    const float silu = zg * s;
    a = silu * zu;
    dg = zu * s * (1.f + zg * (1.f - s));
    du = silu;
  }
}

}  // namespace spt
