// phase.cu -- strided convolutions with R or S > 1 on the tcgen05 kernels by phase
// decomposition (the ResNet-50 7x7/2 stem and the stride-2 3x3 convs).
//
// Conv2d with stride (sh, sw) and padding (ph, pw) (floor extents R2):
//   Y[n,k,p,q] = b[k] + sum_{c,r,s} F[k,c,r,s] Xp[n,c, p*sh + r, q*sw + s]
// where Xp is X zero-padded by (ph, pw).  Split each tap r = r'*sh + a (a < sh, r' < R' =
// ceil(R/sh)) and s = s'*sw + b.  Then Xp[p*sh + r, q*sw + s] = X'[(a,b,c)][p + r'][q + s'] with
//   X'[n][(a*sw + b)*C + c][h'][w'] = Xp[n][c][h'*sh + a][w'*sw + b]     (0 outside Xp)
//   F'[k][(a*sw + b)*C + c][r'][s'] = F[k][c][r'*sh + a][s'*sw + b]       (0 when r >= R or s >= S)
// so Y = conv_{stride 1, pad 0}(X', F') with X' of extent H' = P + R' - 1, W' = Q + S' - 1: a
// stride-1 problem with sh*sw*C channels and ceil(R/sh) x ceil(S/sw) taps that the
// shifted-window tcgen05 kernels run.  The extra taps carry zero filters (9 -> 16 taps for
// 3x3/2, 49 -> 64 for 7x7/2), which is the price of keeping the MMAs dense.
//
// The two backward operators follow from the same linear map X -> X':
//   bwd_data:   dX = (X -> X')^T dX',  dX' = bwd_data_{s1,p0}(F', dY): every Xp position
//               (h, w) is exactly one (h', a) x (w', b), so the transpose is a gather; rows past
//               (P-1)*sh + R - 1 are read by no output (floor extent) and receive 0.
//   bwd_filter: dF[k,c,r,s] = dF'[k][(r%sh, s%sw, c)][r/sh][s/sw],  dF' = bwd_filter_{s1,p0}(X', dY);
//               db is unchanged.
// Every step is a kernel: four HBM-bound gathers here plus the tcgen05 kernels of conv_tc.cu.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace sysml {

namespace {

ConvArgs phase_args(const ConvArgs &a) {
  ConvArgs b{};
  b.N = a.N;
  b.K = a.K;
  b.C = a.sh * a.sw * a.C;
  b.R = (a.R + a.sh - 1) / a.sh;
  b.S = (a.S + a.sw - 1) / a.sw;
  b.P = a.P;
  b.Q = a.Q;
  b.H = a.P + b.R - 1;
  b.W = a.Q + b.S - 1;
  b.sh = b.sw = 1;
  b.ph = b.pw = 0;
  return b;
}

bool is_phase_shape(const ConvArgs &a) {
  static const bool off = getenv("SYSML_NO_PHASE") != nullptr;  // A/B switch: FP32 SIMT instead
  return !off && (a.sh > 1 || a.sw > 1) && (a.R > 1 || a.S > 1) && a.sh <= 4 && a.sw <= 4;
}

int grid_for(int64_t total) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 16ll * sm_count()));
}

// X (N x C*H*W) -> X' (N x C'*H'*W'), one write per X' element, zero outside the padded image
__global__ void phase_split_x_kernel(const float *__restrict__ x, float *__restrict__ xp, int C, int H,
                                     int W, int sh, int sw, int ph, int pw, int C2, int H2, int W2,
                                     int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int w2 = (int)(i % W2);
    int64_t t = i / W2;
    const int h2 = (int)(t % H2);
    t /= H2;
    const int c2 = (int)(t % C2);
    const int64_t n = t / C2;
    const int c = c2 % C, ab = c2 / C, a = ab / sw, b = ab - a * sw;
    const int h = h2 * sh + a - ph, w = w2 * sw + b - pw;
    float v = 0.f;
    if (h >= 0 && h < H && w >= 0 && w < W) v = __ldg(x + ((n * C + c) * H + h) * (int64_t)W + w);
    xp[i] = v;
  }
}

// F (K x C*R*S) -> F' (K x C'*R'*S'), zero for the padded taps
__global__ void phase_split_f_kernel(const float *__restrict__ f, float *__restrict__ fp, int C, int R,
                                     int S, int sh, int sw, int R2, int S2, int64_t total) {
  const int C2 = sh * sw * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int s2 = (int)(i % S2);
    int64_t t = i / S2;
    const int r2 = (int)(t % R2);
    t /= R2;
    const int c2 = (int)(t % C2);
    const int64_t k = t / C2;
    const int c = c2 % C, ab = c2 / C, a = ab / sw, b = ab - a * sw;
    const int r = r2 * sh + a, s = s2 * sw + b;
    fp[i] = (r < R && s < S) ? __ldg(f + ((k * C + c) * R + r) * (int64_t)S + s) : 0.f;
  }
}

// dX'(N x C'*H'*W') -> dX (N x C*H*W): the transpose of phase_split_x (a gather, each Xp
// position belongs to exactly one phase cell)
__global__ void phase_merge_dx_kernel(const float *__restrict__ dxp, float *__restrict__ dx, int C, int H,
                                      int W, int sh, int sw, int ph, int pw, int C2, int H2, int W2,
                                      int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int w = (int)(i % W);
    int64_t t = i / W;
    const int h = (int)(t % H);
    t /= H;
    const int c = (int)(t % C);
    const int64_t n = t / C;
    const int hp = h + ph, wp = w + pw;
    const int h2 = hp / sh, a = hp - h2 * sh, w2 = wp / sw, b = wp - w2 * sw;
    float v = 0.f;
    if (h2 < H2 && w2 < W2)
      v = __ldg(dxp + ((n * C2 + (int64_t)(a * sw + b) * C + c) * H2 + h2) * (int64_t)W2 + w2);
    dx[i] = v;
  }
}

// dF' (K x C'*R'*S') -> dF (K x C*R*S)
__global__ void phase_merge_df_kernel(const float *__restrict__ dfp, float *__restrict__ df, int C, int R,
                                      int S, int sh, int sw, int R2, int S2, int64_t total) {
  const int C2 = sh * sw * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(i % S);
    int64_t t = i / S;
    const int r = (int)(t % R);
    t /= R;
    const int c = (int)(t % C);
    const int64_t k = t / C;
    const int c2 = ((r % sh) * sw + (s % sw)) * C + c;
    df[i] = __ldg(dfp + ((k * C2 + c2) * R2 + r / sh) * (int64_t)S2 + s / sw);
  }
}

size_t x2_bytes(const ConvArgs &b) {
  return align_up((size_t)b.N * b.C * b.H * b.W * sizeof(float), 256);
}
size_t f2_bytes(const ConvArgs &b) {
  return align_up((size_t)b.K * b.C * b.R * b.S * sizeof(float), 256);
}

sysml_status split_x(const ConvArgs &a, const ConvArgs &b, const float *x, float *xp, cudaStream_t st) {
  const int64_t total = (int64_t)b.N * b.C * b.H * b.W;
  phase_split_x_kernel<<<grid_for(total), 256, 0, st>>>(x, xp, a.C, a.H, a.W, a.sh, a.sw, a.ph, a.pw,
                                                        b.C, b.H, b.W, total);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status split_f(const ConvArgs &a, const ConvArgs &b, const float *f, float *fp, cudaStream_t st) {
  const int64_t total = (int64_t)b.K * b.C * b.R * b.S;
  phase_split_f_kernel<<<grid_for(total), 256, 0, st>>>(f, fp, a.C, a.R, a.S, a.sh, a.sw, b.R, b.S,
                                                        total);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

}  // namespace

// ---------------------------------------------------------------- forward
bool phase_fwd_supported(const ConvArgs &a) {
  return is_phase_shape(a) && tc_fwd_supported(phase_args(a), nullptr);
}

size_t phase_fwd_ws(const ConvArgs &a) {
  const ConvArgs b = phase_args(a);
  return x2_bytes(b) + f2_bytes(b) + align_up(tc_fwd_ws(b), 256);
}

sysml_status phase_conv_fwd(const ConvArgs &a, const float *x, const float *f, const float *bias,
                            float *y, void *ws, cudaStream_t st) {
  const ConvArgs b = phase_args(a);
  WsCarve wc(ws, (size_t)-1);
  float *xp = wc.take<float>((size_t)b.N * b.C * b.H * b.W);
  float *fp = wc.take<float>((size_t)b.K * b.C * b.R * b.S);
  void *tws = wc.take<char>(tc_fwd_ws(b));
  SYSML_TRY(split_x(a, b, x, xp, st));
  SYSML_TRY(split_f(a, b, f, fp, st));
  return tc_conv_fwd(b, xp, fp, bias, y, nullptr, nullptr, nullptr, tws, st);
}

// ---------------------------------------------------------------- bwd_data
bool phase_bwd_data_supported(const ConvArgs &a) {
  return is_phase_shape(a) && tc_bwd_data_supported(phase_args(a));
}

size_t phase_bwd_data_ws(const ConvArgs &a) {
  const ConvArgs b = phase_args(a);
  return x2_bytes(b) + f2_bytes(b) + align_up(tc_bwd_data_ws(b), 256);
}

sysml_status phase_conv_bwd_data(const ConvArgs &a, const float *f, const float *dy, float *dx,
                                 void *ws, cudaStream_t st) {
  const ConvArgs b = phase_args(a);
  WsCarve wc(ws, (size_t)-1);
  float *dxp = wc.take<float>((size_t)b.N * b.C * b.H * b.W);
  float *fp = wc.take<float>((size_t)b.K * b.C * b.R * b.S);
  void *tws = wc.take<char>(tc_bwd_data_ws(b));
  SYSML_TRY(split_f(a, b, f, fp, st));
  SYSML_TRY(tc_conv_bwd_data(b, fp, dy, dxp, tws, st));
  const int64_t total = (int64_t)a.N * a.C * a.H * a.W;
  phase_merge_dx_kernel<<<grid_for(total), 256, 0, st>>>(dxp, dx, a.C, a.H, a.W, a.sh, a.sw, a.ph, a.pw,
                                                         b.C, b.H, b.W, total);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

// ---------------------------------------------------------------- bwd_filter
bool phase_bwd_filter_supported(const ConvArgs &a) {
  return is_phase_shape(a) && tc_bwd_filter_supported(phase_args(a));
}

size_t phase_bwd_filter_ws(const ConvArgs &a) {
  const ConvArgs b = phase_args(a);
  return x2_bytes(b) + f2_bytes(b) + align_up(tc_bwd_filter_ws(b), 256);
}

sysml_status phase_conv_bwd_filter(const ConvArgs &a, const float *x, const float *dy, float *df,
                                   float *db, void *ws, cudaStream_t st) {
  const ConvArgs b = phase_args(a);
  WsCarve wc(ws, (size_t)-1);
  float *xp = wc.take<float>((size_t)b.N * b.C * b.H * b.W);
  float *dfp = wc.take<float>((size_t)b.K * b.C * b.R * b.S);
  void *tws = wc.take<char>(tc_bwd_filter_ws(b));
  SYSML_TRY(split_x(a, b, x, xp, st));
  SYSML_TRY(tc_conv_bwd_filter(b, xp, dy, dfp, db, tws, st));
  const int64_t total = (int64_t)a.K * a.C * a.R * a.S;
  phase_merge_df_kernel<<<grid_for(total), 256, 0, st>>>(dfp, df, a.C, a.R, a.S, a.sh, a.sw, b.R, b.S,
                                                         total);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

}  // namespace sysml
