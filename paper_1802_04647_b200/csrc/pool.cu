// pool.cu -- relu_maxpool, maxpool_bwd and bias_add kernels (HBM-bound, CUDA cores).
//
// relu_maxpool (readings R3 R5 R6 R7): one thread per pooled output;
// the window is scanned r-outer / s-inner with a strict '>' so the first
// position attaining the max wins; values are compared in fp32, which is exact
// (max and relu introduce no rounding), so argmax is bit-identical to the fp64
// oracle on identical fp32 inputs.
//
// maxpool_bwd (reading R9): gather form.  Each input element (n,c,h,w)
// visits the pooled outputs whose window covers it in ascending (p',q') order and
// sums dout where argmax == its column index (and out > 0 when masked).  This is
// the same set of terms, in the same order, as the scatter definition, without
// atomics; for stride >= window each dx receives at most one term (bit-exact).
#include "common.cuh"
#include "kernels.cuh"

namespace sysml {

__global__ void relu_maxpool_kernel(PoolArgs a, const float *__restrict__ x,
                                    float *__restrict__ out, int32_t *__restrict__ argmax) {
  const int64_t total = (int64_t)a.N * a.C * a.P * a.Q;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(o % a.Q);
    int64_t t = o / a.Q;
    const int p = (int)(t % a.P);
    t /= a.P;
    const int c = (int)(t % a.C);
    const int64_t n = t / a.C;
    const float *xp = x + n * ((int64_t)a.C * a.H * a.W);
    bool found = false;
    float best = 0.f;
    int arg = -1;
    for (int r = 0; r < a.R; ++r) {
      const int h = p * a.sh - a.ph + r;
      if (h < 0 || h >= a.H) continue;
      for (int s = 0; s < a.S; ++s) {
        const int w = q * a.sw - a.pw + s;
        if (w < 0 || w >= a.W) continue;
        const int col = (c * a.H + h) * a.W + w;
        float v = __ldg(xp + col);
        if (a.relu) v = v > 0.f ? v : 0.f;
        if (!found || v > best) {
          found = true;
          best = v;
          arg = col;
        }
      }
    }
    out[o] = found ? best : 0.f;
    if (argmax) argmax[o] = arg;
  }
}

__global__ void maxpool_bwd_kernel(PoolArgs a, const int32_t *__restrict__ argmax,
                                   const float *__restrict__ dout,
                                   const float *__restrict__ mask, float *__restrict__ dx) {
  const int64_t total = (int64_t)a.N * a.C * a.H * a.W;
  const int64_t CPQ = (int64_t)a.C * a.P * a.Q;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int w = (int)(i % a.W);
    int64_t t = i / a.W;
    const int h = (int)(t % a.H);
    t /= a.H;
    const int c = (int)(t % a.C);
    const int64_t n = t / a.C;
    const int col = (c * a.H + h) * a.W + w;
    // pooled rows p with p*sh - ph <= h <= p*sh - ph + R - 1
    const int hp = h + a.ph, wp = w + a.pw;
    int p_lo = hp - a.R + 1;
    p_lo = p_lo <= 0 ? 0 : (p_lo + a.sh - 1) / a.sh;
    int p_hi = hp / a.sh;
    if (p_hi > a.P - 1) p_hi = a.P - 1;
    int q_lo = wp - a.S + 1;
    q_lo = q_lo <= 0 ? 0 : (q_lo + a.sw - 1) / a.sw;
    int q_hi = wp / a.sw;
    if (q_hi > a.Q - 1) q_hi = a.Q - 1;
    float acc = 0.f;
    const int64_t base = n * CPQ + (int64_t)c * a.P * a.Q;
    for (int p = p_lo; p <= p_hi; ++p)
      for (int q = q_lo; q <= q_hi; ++q) {
        const int64_t j = base + p * a.Q + q;
        if (__ldg(argmax + j) != col) continue;
        if (mask && !(__ldg(mask + j) > 0.f)) continue;
        acc += __ldg(dout + j);
      }
    dx[i] = acc;
  }
}

// Specialisation for non-overlapping windows (stride == window, pad 0): each
// pooled output owns a disjoint RxS block; one thread per pooled output writes
// its whole block (dout at argmax, 0 elsewhere).  Bit-exact (one term each).
__global__ void maxpool_bwd_disjoint_kernel(PoolArgs a, const int32_t *__restrict__ argmax,
                                            const float *__restrict__ dout,
                                            const float *__restrict__ mask,
                                            float *__restrict__ dx) {
  const int64_t total = (int64_t)a.N * a.C * a.P * a.Q;
  const int64_t CHW = (int64_t)a.C * a.H * a.W;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(o % a.Q);
    int64_t t = o / a.Q;
    const int p = (int)(t % a.P);
    t /= a.P;
    const int c = (int)(t % a.C);
    const int64_t n = t / a.C;
    const int am = __ldg(argmax + o);
    float g = __ldg(dout + o);
    if (mask && !(__ldg(mask + o) > 0.f)) g = 0.f;
    float *dxp = dx + n * CHW;
    for (int r = 0; r < a.R; ++r) {
      const int h = p * a.R + r;
      if (h >= a.H) break;
      for (int s = 0; s < a.S; ++s) {
        const int w = q * a.S + s;
        if (w >= a.W) break;
        const int col = (c * a.H + h) * a.W + w;
        dxp[col] = (col == am) ? g : 0.f;
      }
    }
  }
}

__global__ void zero_kernel(float *__restrict__ p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0.f;
}

__global__ void bias_add_kernel(int32_t N, int32_t K, int32_t PQ, float *__restrict__ y,
                                const float *__restrict__ bias) {
  const int64_t total = (int64_t)N * K * PQ;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)((i / PQ) % K);
    y[i] += __ldg(bias + k);
  }
}

// maxpool_bwd to SPF: one thread per pooled output writes its whole (disjoint) window.
__global__ void maxpool_bwd_spf_kernel(PoolArgs a, const int32_t *__restrict__ argmax,
                                       const float *__restrict__ dout,
                                       const float *__restrict__ mask, float *__restrict__ dx,
                                       int64_t plane, int Wf, int Lf) {
  const int64_t total = (int64_t)a.N * a.C * a.P * a.Q;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(o % a.Q);
    int64_t t = o / a.Q;
    const int p = (int)(t % a.P);
    t /= a.P;
    const int c = (int)(t % a.C);
    const int n = (int)(t / a.C);
    const int am = __ldg(argmax + o);
    float g = __ldg(dout + o);
    if (mask && !(__ldg(mask + o) > 0.f)) g = 0.f;
    float *dxp = dx + (int64_t)c * plane + (int64_t)n * Lf;
    for (int r = 0; r < a.R; ++r) {
      const int h = p * a.R + r;
      if (h >= a.H) break;
      for (int s = 0; s < a.S; ++s) {
        const int w = q * a.S + s;
        if (w >= a.W) break;
        const int col = (c * a.H + h) * a.W + w;
        dxp[h * Wf + w] = (col == am) ? g : 0.f;
      }
    }
  }
}

__global__ void nchw_to_spf_kernel(int N, int C, int H, int W, const float *__restrict__ x,
                                   float *__restrict__ spf, int64_t plane, int Wf, int Lf, int off) {
  const int64_t total = (int64_t)N * C * H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int w = (int)(i % W);
    int64_t t = i / W;
    const int h = (int)(t % H);
    t /= H;
    const int c = (int)(t % C);
    const int n = (int)(t / C);
    spf[(int64_t)c * plane + (int64_t)n * Lf + (h + off) * Wf + (w + off)] = __ldg(x + i);
  }
}

static inline int grid_for(int64_t total, int threads) {
  int64_t b = ceil_div(total, threads);
  int64_t cap = (int64_t)sm_count() * 16;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

sysml_status launch_relu_maxpool(const PoolArgs &a, const float *x, float *out, int32_t *argmax,
                                 cudaStream_t st) {
  const int64_t total = (int64_t)a.N * a.C * a.P * a.Q;
  relu_maxpool_kernel<<<grid_for(total, 256), 256, 0, st>>>(a, x, out, argmax);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status launch_maxpool_bwd(const PoolArgs &a, const int32_t *argmax, const float *dout,
                                const float *mask, float *dx, cudaStream_t st) {
  const bool disjoint = a.sh == a.R && a.sw == a.S && a.ph == 0 && a.pw == 0;
  if (disjoint) {
    // Every input element belongs to at most one window; elements of trailing
    // rows/cols not covered by any window must be zero.
    const bool covered = a.P * a.R == a.H && a.Q * a.S == a.W;
    if (!covered) {
      const int64_t n = (int64_t)a.N * a.C * a.H * a.W;
      zero_kernel<<<grid_for(n, 256), 256, 0, st>>>(dx, n);
      SYSML_LAUNCH_CHECK();
    }
    const int64_t total = (int64_t)a.N * a.C * a.P * a.Q;
    maxpool_bwd_disjoint_kernel<<<grid_for(total, 256), 256, 0, st>>>(a, argmax, dout, mask, dx);
  } else {
    const int64_t total = (int64_t)a.N * a.C * a.H * a.W;
    maxpool_bwd_kernel<<<grid_for(total, 256), 256, 0, st>>>(a, argmax, dout, mask, dx);
  }
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status launch_bias_add(int32_t N, int32_t K, int32_t PQ, float *y, const float *bias,
                             cudaStream_t st) {
  const int64_t total = (int64_t)N * K * PQ;
  bias_add_kernel<<<grid_for(total, 256), 256, 0, st>>>(N, K, PQ, y, bias);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status launch_maxpool_bwd_spf(const PoolArgs &a, const int32_t *argmax, const float *dout,
                                    const float *mask, float *dx_spf, int64_t plane, int Wf,
                                    int Lf, cudaStream_t st) {
  const int64_t total = (int64_t)a.N * a.C * a.P * a.Q;
  maxpool_bwd_spf_kernel<<<grid_for(total, 256), 256, 0, st>>>(a, argmax, dout, mask, dx_spf, plane,
                                                               Wf, Lf);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status launch_nchw_to_spf(int N, int C, int H, int W, const float *x, float *spf,
                                int64_t plane, int Wf, int Lf, int off, cudaStream_t st) {
  const int64_t total = (int64_t)N * C * H * W;
  nchw_to_spf_kernel<<<grid_for(total, 256), 256, 0, st>>>(N, C, H, W, x, spf, plane, Wf, Lf, off);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status launch_zero(float *p, int64_t n, cudaStream_t st) {
  if (n <= 0) return SYSML_OK;
  zero_kernel<<<grid_for(n, 256), 256, 0, st>>>(p, n);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

}  // namespace sysml
