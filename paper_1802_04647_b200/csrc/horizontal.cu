// horizontal.cu -- horizontal fusion for shared inputs (NEXT-2; "horizontal fusion
// for shared inputs (e.g. reuse temporary im2col intermediates in presence of multiple
// convolution operators consuming the same input)").
//
// n_ops convolutions with one geometry (C, H, W, R, S, stride, pad) that read the SAME input
// X -- a ResNet bottleneck's first 1x1 conv and its 1x1 projection shortcut, or several
// 3x3 branches over one feature map -- are one convolution with the filter banks stacked:
//   Y_cat = conv(X, [F_0; F_1; ...])      (K = sum K_i output channels, op i's channels are
//                                           the slice [K_0 + ... + K_{i-1}, ... + K_i))
//   dX    = sum_i bwd_data(F_i, dY_i) = bwd_data([F_0; F_1; ...], dY_cat)
//   [dF_0; dF_1; ...] = bwd_filter(X, dY_cat)
// so the staged input tile (the implicit-GEMM operand: shifted-window halo, or the TMA box)
// is loaded once and feeds every op's filters: X is read once instead of n_ops times, and the
// tensor-core N dimension is the sum of the ops' widths.  The stacked bank (tiny) is packed
// into the workspace by one kernel; dF / db are scattered back by one kernel.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace sysml {
sysml_status conv_fwd_dispatch(const sysml_conv_desc &cd, const sysml_input &x, const float *f,
                               const float *bias, float *y, const sysml_pool_desc *pd,
                               float *pout, int32_t *parg, void *ws, size_t ws_bytes,
                               cudaStream_t st);
sysml_status conv_fwd_ws(const sysml_conv_desc &cd, const sysml_pool_desc *pd, int is_csr,
                         size_t *bytes);
sysml_status conv_bwd_filter_dispatch(const sysml_conv_desc &cd, const sysml_input &x,
                                      const float *dy, float *df, float *db, void *ws,
                                      size_t ws_bytes, cudaStream_t st);
sysml_status conv_bwd_filter_ws(const sysml_conv_desc &cd, int is_csr, size_t *bytes);
sysml_status conv_bwd_data_dispatch(const sysml_conv_desc &cd, const float *f, const float *dy,
                                    float *dx, void *ws, size_t ws_bytes, cudaStream_t st);
sysml_status conv_bwd_data_ws(const sysml_conv_desc &cd, size_t *bytes);

namespace {

constexpr int MAX_OPS = 8;

struct Segs {
  const float *src[MAX_OPS];
  float *dst[MAX_OPS];
  int64_t off[MAX_OPS + 1];  // element offsets of each op inside the stacked array
  int n;
};

// stacked[off[i] + j] = src[i][j] (gather) or dst[i][j] = stacked[off[i] + j] (scatter)
__global__ void stack_kernel(Segs s, float *stacked, const float *stacked_in, int gather) {
  const int64_t total = s.off[s.n];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int i = 0;
    while (e >= s.off[i + 1]) ++i;
    const int64_t j = e - s.off[i];
    if (gather) stacked[e] = s.src[i] ? s.src[i][j] : 0.f;
    else if (s.dst[i]) s.dst[i][j] = stacked_in[e];
  }
}

sysml_status launch_stack(const Segs &s, float *stacked, const float *stacked_in, int gather, cudaStream_t st) {
  const int64_t total = s.off[s.n];
  if (total == 0) return SYSML_OK;
  stack_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 4 * sm_count()), 256, 0, st>>>(s, stacked,
                                                                                                   stacked_in, gather);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status check_ops(const sysml_conv_desc *d, int32_t n_ops, const int32_t *k, int64_t *crs) {
  SYSML_CHECK_ARG(d && k, "NULL descriptor / k_counts");
  SYSML_CHECK_ARG(n_ops >= 1 && n_ops <= MAX_OPS, "n_ops %d must be in [1, %d]", n_ops, MAX_OPS);
  int64_t ksum = 0;
  for (int i = 0; i < n_ops; ++i) {
    SYSML_CHECK_ARG(k[i] >= 1, "k_counts[%d] = %d must be >= 1", i, k[i]);
    ksum += k[i];
  }
  SYSML_CHECK_SHAPE(ksum == d->K, "the descriptor's K = %d must equal the sum of k_counts (%lld)", d->K,
                    (long long)ksum);
  *crs = (int64_t)d->C * d->R * d->S;
  return SYSML_OK;
}

Segs make_segs(int32_t n_ops, const int32_t *k, int64_t per_k) {
  Segs s{};
  s.n = n_ops;
  s.off[0] = 0;
  for (int i = 0; i < n_ops; ++i) s.off[i + 1] = s.off[i] + (int64_t)k[i] * per_k;
  return s;
}

size_t stacked_bytes(const sysml_conv_desc &d, int64_t crs) {
  return align_up((size_t)d.K * crs * sizeof(float), 256) + align_up((size_t)d.K * sizeof(float), 256);
}

}  // namespace
}  // namespace sysml

using namespace sysml;

extern "C" {

sysml_status sysml_conv2d_multi_workspace_size(const sysml_conv_desc *d, int32_t n_ops, const int32_t *k_counts,
                                               int32_t op, int32_t is_csr, size_t *bytes) {
  int64_t crs = 0;
  SYSML_TRY(check_ops(d, n_ops, k_counts, &crs));
  SYSML_CHECK_ARG(bytes && op >= 0 && op <= 2, "bad op %d / NULL bytes", op);
  size_t inner = 0;
  if (op == 0) SYSML_TRY(conv_fwd_ws(*d, nullptr, is_csr, &inner));
  else if (op == 1) SYSML_TRY(conv_bwd_data_ws(*d, &inner));
  else SYSML_TRY(conv_bwd_filter_ws(*d, is_csr, &inner));
  *bytes = stacked_bytes(*d, crs) + inner;
  return SYSML_OK;
}

sysml_status sysml_conv2d_multi(const sysml_conv_desc *d, int32_t n_ops, const int32_t *k_counts,
                                const sysml_input *x, const float *const *f, const float *const *bias,
                                float *y_cat, void *workspace, size_t workspace_bytes, sysml_stream_t stream) {
  int64_t crs = 0;
  SYSML_TRY(check_ops(d, n_ops, k_counts, &crs));
  SYSML_CHECK_ARG(x && f && y_cat, "NULL argument");
  size_t need = 0;
  SYSML_TRY(sysml_conv2d_multi_workspace_size(d, n_ops, k_counts, 0, x->is_csr, &need));
  SYSML_CHECK_ARG(workspace_bytes >= need && (need == 0 || workspace), "workspace %zu < required %zu",
                  workspace_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  WsCarve wc(workspace, workspace_bytes);
  float *fcat = wc.take<float>((size_t)d->K * crs);
  float *bcat = wc.take<float>((size_t)d->K);
  bool any_bias = false;
  for (int i = 0; i < n_ops; ++i) {
    SYSML_CHECK_ARG(f[i], "f[%d] is NULL", i);
    any_bias |= bias && bias[i];
  }
  Segs sf = make_segs(n_ops, k_counts, crs);
  for (int i = 0; i < n_ops; ++i) sf.src[i] = f[i];
  SYSML_TRY(launch_stack(sf, fcat, nullptr, 1, st));
  if (any_bias) {  // a NULL bias of one op contributes zeros
    Segs sb = make_segs(n_ops, k_counts, 1);
    for (int i = 0; i < n_ops; ++i) sb.src[i] = bias[i];
    SYSML_TRY(launch_stack(sb, bcat, nullptr, 1, st));
  }
  SYSML_TRY(conv_fwd_dispatch(*d, *x, fcat, any_bias ? bcat : nullptr, y_cat, nullptr, nullptr, nullptr,
                              wc.base + wc.used(), workspace_bytes - wc.used(), st));
  route_note("horizontal fusion of %d ops (K = %d)", n_ops, d->K);
  return SYSML_OK;
}

sysml_status sysml_conv2d_multi_bwd_data(const sysml_conv_desc *d, int32_t n_ops, const int32_t *k_counts,
                                         const float *const *f, const float *dy_cat, float *dx, void *workspace,
                                         size_t workspace_bytes, sysml_stream_t stream) {
  int64_t crs = 0;
  SYSML_TRY(check_ops(d, n_ops, k_counts, &crs));
  SYSML_CHECK_ARG(f && dy_cat && dx, "NULL argument");
  size_t need = 0;
  SYSML_TRY(sysml_conv2d_multi_workspace_size(d, n_ops, k_counts, 1, 0, &need));
  SYSML_CHECK_ARG(workspace_bytes >= need && (need == 0 || workspace), "workspace %zu < required %zu",
                  workspace_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  WsCarve wc(workspace, workspace_bytes);
  float *fcat = wc.take<float>((size_t)d->K * crs);
  wc.take<float>((size_t)d->K);
  Segs sf = make_segs(n_ops, k_counts, crs);
  for (int i = 0; i < n_ops; ++i) {
    SYSML_CHECK_ARG(f[i], "f[%d] is NULL", i);
    sf.src[i] = f[i];
  }
  SYSML_TRY(launch_stack(sf, fcat, nullptr, 1, st));
  SYSML_TRY(conv_bwd_data_dispatch(*d, fcat, dy_cat, dx, wc.base + wc.used(), workspace_bytes - wc.used(), st));
  route_note("horizontal fusion of %d ops (K = %d)", n_ops, d->K);
  return SYSML_OK;
}

sysml_status sysml_conv2d_multi_bwd_filter(const sysml_conv_desc *d, int32_t n_ops, const int32_t *k_counts,
                                           const sysml_input *x, const float *dy_cat, float *const *df,
                                           float *const *db, void *workspace, size_t workspace_bytes,
                                           sysml_stream_t stream) {
  int64_t crs = 0;
  SYSML_TRY(check_ops(d, n_ops, k_counts, &crs));
  SYSML_CHECK_ARG(x && dy_cat && df, "NULL argument");
  size_t need = 0;
  SYSML_TRY(sysml_conv2d_multi_workspace_size(d, n_ops, k_counts, 2, x->is_csr, &need));
  SYSML_CHECK_ARG(workspace_bytes >= need && (need == 0 || workspace), "workspace %zu < required %zu",
                  workspace_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  WsCarve wc(workspace, workspace_bytes);
  float *dfcat = wc.take<float>((size_t)d->K * crs);
  float *dbcat = wc.take<float>((size_t)d->K);
  bool any_db = false;
  for (int i = 0; i < n_ops; ++i) {
    SYSML_CHECK_ARG(df[i], "df[%d] is NULL", i);
    any_db |= db && db[i];
  }
  SYSML_TRY(conv_bwd_filter_dispatch(*d, *x, dy_cat, dfcat, any_db ? dbcat : nullptr, wc.base + wc.used(),
                                     workspace_bytes - wc.used(), st));
  route_note("horizontal fusion of %d ops (K = %d)", n_ops, d->K);
  Segs sf = make_segs(n_ops, k_counts, crs);
  for (int i = 0; i < n_ops; ++i) sf.dst[i] = df[i];
  SYSML_TRY(launch_stack(sf, nullptr, dfcat, 0, st));
  if (any_db) {
    Segs sb = make_segs(n_ops, k_counts, 1);
    for (int i = 0; i < n_ops; ++i) sb.dst[i] = db[i];
    SYSML_TRY(launch_stack(sb, nullptr, dbcat, 0, st));
  }
  return SYSML_OK;
}

}  // extern "C"
