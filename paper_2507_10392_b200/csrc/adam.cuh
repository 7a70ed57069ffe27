// AdamW element update shared by the standalone shard optimizer (adam.cu) and the
// fused reduce-scatter + AdamW kernel over NVLink peer memory (peer.cu).
// Update rule follows torch.optim.AdamW (decoupled weight decay, bias-corrected).
#pragma once
#include "common.cuh"

namespace zb {

struct AdamParams {
  float lr, beta1, beta2, eps, wd, grad_scale;
  float step_size;      // lr / (1 - beta1^t)
  float inv_bc2_sqrt;   // 1 / sqrt(1 - beta2^t)
  float decay;          // 1 - lr * wd
  const int* step_dev;  // if set: t is read on the device (CUDA-graph replay)
};

ZB_DEVICE void resolve_step(AdamParams& a) {
  if (a.step_dev) {
    const int t = *a.step_dev;
    const double bc1 = 1.0 - pow((double)a.beta1, t), bc2 = 1.0 - pow((double)a.beta2, t);
    a.step_size = (float)(a.lr / bc1);
    a.inv_bc2_sqrt = (float)(1.0 / sqrt(bc2));
  }
}

ZB_DEVICE void adam_elem(float& p, float& m, float& v, float g, const AdamParams& a) {
  p *= a.decay;
  m = m + (g - m) * (1.f - a.beta1);
  v = v * a.beta2 + (1.f - a.beta2) * g * g;
  const float denom = sqrtf(v) * a.inv_bc2_sqrt + a.eps;
  p = p - a.step_size * (m / denom);
}

// Host-side parameter setup; step < 1 with step_dev set: t is read on the device.
inline AdamParams make_adam_params(float lr, float beta1, float beta2, float eps, float wd,
                                   float grad_scale, int step, const int* step_dev) {
  AdamParams a;
  a.lr = lr; a.beta1 = beta1; a.beta2 = beta2; a.eps = eps; a.wd = wd;
  a.grad_scale = grad_scale;
  a.step_dev = step_dev;
  if (step < 1) step = 1;
  const double bc1 = 1.0 - pow((double)beta1, step), bc2 = 1.0 - pow((double)beta2, step);
  a.step_size = (float)(lr / bc1);
  a.inv_bc2_sqrt = (float)(1.0 / sqrt(bc2));
  a.decay = 1.f - lr * wd;
  return a;
}

}  // namespace zb
