// api.cu -- the extern "C" entry points of include/sysml.h: validation and dispatch
// to the sm_100a kernels.  No CPU fallback exists (BJ north_star): every path
// below launches CUDA kernels on the caller's stream.
//
// Dispatch:
//   dense conv fwd / bwd_data / bwd_filter:
//     math == TF32 and the tcgen05 kernel covers the shape -> conv_tc.cu (K3/K5/K6)
//     TF32, strided with R or S > 1, stride-1 image covered -> phase.cu (phase split +
//                                                              the tcgen05 stride-1 kernels)
//     TF32 bwd_filter outside the TMA kernels' shapes             -> phase.cu im2col + 1x1 TMA GEMM
//     otherwise                                             -> conv_simt.cu (fp32 FMA)
//   CSR input: fwd -> csr.cu K7 (fused epilogue optional); bwd_filter -> csr.cu K8;
//     shapes beyond K7/K8's shared-memory budget are densified into the workspace
//     first (still on the GPU) and take the dense path.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace sysml {

thread_local int64_t g_launches = 0;

static bool fused_pool_ok(const ConvGeom &cg, const ConvGeom &pg, const sysml_pool_desc *pd) {
  return pg.N == cg.N && pg.C == cg.K && pg.H == cg.P && pg.W == cg.Q && pd->relu &&
         pd->R == pd->stride_h && pd->S == pd->stride_w && pd->pad_h == 0 && pd->pad_w == 0;
}

sysml_status conv_fwd_ws(const sysml_conv_desc &cd, const sysml_pool_desc *pd, int is_csr,
                         size_t *bytes) {
  ConvGeom g;
  SYSML_TRY(validate_conv(&cd, &g));
  const ConvArgs a = conv_args(g);
  size_t b = 0;
  const bool use_tc = cd.math == SYSML_MATH_TF32;
  PoolArgs pa{};
  const PoolArgs *pap = nullptr;
  if (pd) {
    ConvGeom pg;
    SYSML_TRY(validate_pool(pd, &pg));
    pa = pool_args(pg, 1);
    pap = &pa;
  }
  if (use_tc && pap && conv1_pool_supported(a, pap)) {
    b += conv1_pool_ws(a, pap);  // C = 1 conv + pool: window in the MMA N dimension
  } else if (is_csr && use_tc && tc_fwd_ks(a) && tc_fwd_supported(a, pap)) {
    b += tc_fwd_ws(a);  // CSR rows scattered straight into the tcgen05 operand
  } else if (is_csr) {
    if (!csr_fwd_supported(a)) {
      b += align_up((size_t)g.N * g.CHW() * sizeof(float), 256);  // densified input
      if (use_tc && tc_fwd_supported(a, pap)) b += tc_fwd_ws(a);
      else if (use_tc && !pap && phase_fwd_supported(a)) b += phase_fwd_ws(a);
      else if (pd) b += align_up((size_t)g.N * g.KPQ() * sizeof(float), 256);
    }
  } else if (use_tc && !pap && pair_conv_supported(a, 0)) {
    b += pair_conv_ws(a, 0);  // CTA-pair (cta_group::2) kernel for 256-wide filter banks (opt-in)
  } else if (use_tc && !pap && c1x1_supported(a, 0)) {
    b += c1x1_ws(a, 0);  // 1x1: activation transposed through TMEM
  } else if (use_tc && tc_fwd_supported(a, pap)) {
    b += tc_fwd_ws(a);
  } else if (use_tc && !pap && phase_fwd_supported(a)) {
    b += phase_fwd_ws(a);
  } else if (pd) {
    b += align_up((size_t)g.N * g.KPQ() * sizeof(float), 256);  // unfused z
  }
  *bytes = b;
  return SYSML_OK;
}

sysml_status conv_fwd_dispatch(const sysml_conv_desc &cd, const sysml_input &x, const float *f,
                               const float *bias, float *y, const sysml_pool_desc *pd,
                               float *pout, int32_t *parg, void *ws, size_t ws_bytes,
                               cudaStream_t st) {
  route_reset();
  ConvGeom g;
  SYSML_TRY(validate_conv(&cd, &g));
  SYSML_TRY(validate_input(&x, g));
  SYSML_CHECK_ARG(f != nullptr, "filter pointer is NULL");
  SYSML_CHECK_ALIGN16(f, "filter");
  SYSML_CHECK_ALIGN16(bias, "bias");
  SYSML_CHECK_ALIGN16(y, "output");
  SYSML_CHECK_ALIGN16(pout, "pooled output");
  SYSML_CHECK_ALIGN16(parg, "argmax");
  SYSML_CHECK_ALIGN16(ws, "workspace");
  const ConvArgs a = conv_args(g);
  PoolArgs pa{};
  const PoolArgs *pap = nullptr;
  if (pd) {
    ConvGeom pg;
    SYSML_TRY(validate_pool(pd, &pg));
    SYSML_CHECK_SHAPE(pg.N == g.N && pg.C == g.K && pg.H == g.P && pg.W == g.Q,
                      "pool input %lldx(%lld*%lld*%lld) must equal the conv output %lldx(%lld*%lld*%lld)",
                      (long long)pg.N, (long long)pg.C, (long long)pg.H, (long long)pg.W,
                      (long long)g.N, (long long)g.K, (long long)g.P, (long long)g.Q);
    if (!fused_pool_ok(g, pg, pd)) {
      set_error("fused conv+bias+relu+maxpool supports relu=1, window == stride, pad 0 "
                "(got window %dx%d stride %dx%d pad %dx%d relu %d)",
                pd->R, pd->S, pd->stride_h, pd->stride_w, pd->pad_h, pd->pad_w, pd->relu);
      return SYSML_ERR_UNSUPPORTED;
    }
    SYSML_CHECK_ARG(pout != nullptr, "pooled output pointer is NULL");
    pa = pool_args(pg, 1);
    pap = &pa;
  } else {
    SYSML_CHECK_ARG(y != nullptr, "output pointer is NULL");
  }
  size_t need = 0;
  SYSML_TRY(conv_fwd_ws(cd, pd, x.is_csr, &need));
  if (need > 0 && (ws == nullptr || ws_bytes < need)) {
    set_error("workspace too small: need %zu bytes, got %zu", need, ws ? ws_bytes : 0);
    return SYSML_ERR_WORKSPACE;
  }
  WsCarve wc(ws, ws_bytes);
  const bool use_tc = cd.math == SYSML_MATH_TF32 && tc_fwd_supported(a, pap);
  const float *xd = x.dense;
  if (cd.math == SYSML_MATH_TF32 && pap && conv1_pool_supported(a, pap)) {
    void *tws = wc.take<char>(conv1_pool_ws(a, pap));
    SYSML_WS_FITS(wc);
    return conv1_pool(a, pap, x.is_csr ? nullptr : x.dense, f, bias, pout, parg, tws, st, nullptr,
                      x.is_csr ? &x.csr : nullptr);
  }
  if (x.is_csr && use_tc && tc_fwd_ks(a)) {
    void *tws = wc.take<char>(tc_fwd_ws(a));
    SYSML_WS_FITS(wc);
    return tc_conv_fwd(a, nullptr, f, bias, y, pap, pout, parg, tws, st, &x.csr);
  }
  if (x.is_csr) {
    if (csr_fwd_supported(a)) return csr_conv_fwd(a, x.csr, f, bias, y, pap, pout, parg, st);
    route_note("csr_densify_kernel");
    float *dense = wc.take<float>((size_t)g.N * g.CHW());
    SYSML_WS_FITS(wc);
    SYSML_TRY(csr_densify(x.csr, dense, st));
    xd = dense;
  }
  if (cd.math == SYSML_MATH_TF32 && !pap && !x.is_csr && pair_conv_supported(a, 0)) {
    void *tws = wc.take<char>(pair_conv_ws(a, 0));
    SYSML_WS_FITS(wc);
    return pair_conv(a, 0, xd, f, bias, y, tws, st);
  }
  if (cd.math == SYSML_MATH_TF32 && !pap && !x.is_csr && c1x1_supported(a, 0)) {
    void *tws = wc.take<char>(c1x1_ws(a, 0));
    SYSML_WS_FITS(wc);
    return c1x1_conv(a, 0, xd, f, bias, y, tws, st);
  }
  if (use_tc) {
    void *tws = wc.take<char>(tc_fwd_ws(a));
    SYSML_WS_FITS(wc);
    return tc_conv_fwd(a, xd, f, bias, y, pap, pout, parg, tws, st);
  }
  if (cd.math == SYSML_MATH_TF32 && !pap && phase_fwd_supported(a)) {
    route_note("phase split");
    void *pws = wc.take<char>(phase_fwd_ws(a));
    SYSML_WS_FITS(wc);
    return phase_conv_fwd(a, xd, f, bias, y, pws, st);
  }
  if (pap) {
    float *z = wc.take<float>((size_t)g.N * g.KPQ());
    SYSML_WS_FITS(wc);
    SYSML_TRY(simt_conv_fwd(a, xd, f, bias, z, st));
    route_note("relu_maxpool_kernel");
    return launch_relu_maxpool(*pap, z, pout, parg, st);
  }
  return simt_conv_fwd(a, xd, f, bias, y, st);
}

// TF32 dense bwd_filter route, best first: the dedicated TMA kernels; the phase
// split when its stride-1 problem fits the frame kernel; im2col + the 1x1 GEMM (tiny channel
// counts, 7x7 planes, frames too wide for the frame kernel); the generic tcgen05 kernel; the
// phase split onto it; else FP32 SIMT.
enum class WgRoute { TC, PHASE, IM2COL, SIMT };

static WgRoute wgrad_route(const sysml_conv_desc &cd, const ConvArgs &a) {
  if (cd.math != SYSML_MATH_TF32) return WgRoute::SIMT;
  if (tc_bwd_filter_fast_supported(a)) return WgRoute::TC;
  if (phase_bwd_filter_frame_ok(a)) return WgRoute::PHASE;
  // im2col after the frame kernels: measured on the ResNet-50 sweep, it loses wherever a frame
  // kernel applies (its split-K partials scale with K x CRS), and wins by 4-7x where none does
  if (im2col_bwd_filter_supported(a)) return WgRoute::IM2COL;
  if (tc_bwd_filter_supported(a)) return WgRoute::TC;
  if (phase_bwd_filter_supported(a)) return WgRoute::PHASE;
  return WgRoute::SIMT;
}

sysml_status conv_bwd_filter_ws(const sysml_conv_desc &cd, int is_csr, size_t *bytes) {
  ConvGeom g;
  SYSML_TRY(validate_conv(&cd, &g));
  const ConvArgs a = conv_args(g);
  size_t b = 0;
  if (is_csr && csr_bwd_filter_supported(a)) {
    b = csr_bwd_filter_ws(a);
  } else {
    if (is_csr) b += align_up((size_t)g.N * g.CHW() * sizeof(float), 256);
    switch (wgrad_route(cd, a)) {
      case WgRoute::TC: b += tc_bwd_filter_ws(a); break;
      case WgRoute::PHASE: b += phase_bwd_filter_ws(a); break;
      case WgRoute::IM2COL: b += im2col_bwd_filter_ws(a); break;
      case WgRoute::SIMT: b += simt_bwd_filter_ws(a); break;
    }
  }
  *bytes = b;
  return SYSML_OK;
}

sysml_status conv_bwd_filter_dispatch(const sysml_conv_desc &cd, const sysml_input &x,
                                      const float *dy, float *df, float *db, void *ws,
                                      size_t ws_bytes, cudaStream_t st) {
  route_reset();
  ConvGeom g;
  SYSML_TRY(validate_conv(&cd, &g));
  SYSML_TRY(validate_input(&x, g));
  SYSML_CHECK_ARG(dy && df, "dy/df pointer is NULL");
  SYSML_CHECK_ALIGN16(dy, "dy");
  SYSML_CHECK_ALIGN16(df, "df");
  SYSML_CHECK_ALIGN16(db, "db");
  SYSML_CHECK_ALIGN16(ws, "workspace");
  const ConvArgs a = conv_args(g);
  size_t need = 0;
  SYSML_TRY(conv_bwd_filter_ws(cd, x.is_csr, &need));
  if (need > 0 && (ws == nullptr || ws_bytes < need)) {
    set_error("workspace too small: need %zu bytes, got %zu", need, ws ? ws_bytes : 0);
    return SYSML_ERR_WORKSPACE;
  }
  WsCarve wc(ws, ws_bytes);
  const float *xd = x.dense;
  if (x.is_csr) {
    if (csr_bwd_filter_supported(a)) return csr_conv_bwd_filter(a, x.csr, dy, df, db, ws, st);
    float *dense = wc.take<float>((size_t)g.N * g.CHW());
    xd = dense;
  }
  const WgRoute route = wgrad_route(cd, a);
  if (route == WgRoute::PHASE) route_note("phase split");
  if (route == WgRoute::IM2COL) route_note("im2col_kernel");
  size_t route_ws = 0;
  switch (route) {
    case WgRoute::TC: route_ws = tc_bwd_filter_ws(a); break;
    case WgRoute::PHASE: route_ws = phase_bwd_filter_ws(a); break;
    case WgRoute::IM2COL: route_ws = im2col_bwd_filter_ws(a); break;
    case WgRoute::SIMT: route_ws = simt_bwd_filter_ws(a); break;
  }
  void *rws = wc.take<char>(route_ws);
  SYSML_WS_FITS(wc);
  if (x.is_csr) {
    route_note("csr_densify_kernel");
    SYSML_TRY(csr_densify(x.csr, const_cast<float *>(xd), st));
  }
  switch (route) {
    case WgRoute::TC: return tc_conv_bwd_filter(a, xd, dy, df, db, rws, st);
    case WgRoute::PHASE: return phase_conv_bwd_filter(a, xd, dy, df, db, rws, st);
    case WgRoute::IM2COL: return im2col_conv_bwd_filter(a, xd, dy, df, db, rws, st);
    case WgRoute::SIMT: break;
  }
  void *sws = rws;
  return simt_conv_bwd_filter(a, xd, dy, df, db, sws, st);
}

sysml_status conv_bwd_data_ws(const sysml_conv_desc &cd, size_t *bytes) {
  ConvGeom g;
  SYSML_TRY(validate_conv(&cd, &g));
  const ConvArgs a = conv_args(g);
  *bytes = 0;
  if (cd.math == SYSML_MATH_TF32 && pair_conv_supported(a, 1)) *bytes = pair_conv_ws(a, 1);
  else if (cd.math == SYSML_MATH_TF32 && c1x1_supported(a, 1)) *bytes = c1x1_ws(a, 1);
  else if (cd.math == SYSML_MATH_TF32 && tc_bwd_data_supported(a)) *bytes = tc_bwd_data_ws(a);
  else if (cd.math == SYSML_MATH_TF32 && phase_bwd_data_supported(a)) *bytes = phase_bwd_data_ws(a);
  else if (phase_simt_bwd_data_supported(a)) *bytes = phase_simt_bwd_data_ws(a);
  return SYSML_OK;
}

sysml_status conv_bwd_data_dispatch(const sysml_conv_desc &cd, const float *f, const float *dy,
                                    float *dx, void *ws, size_t ws_bytes, cudaStream_t st) {
  route_reset();
  ConvGeom g;
  SYSML_TRY(validate_conv(&cd, &g));
  SYSML_CHECK_ARG(f && dy && dx, "f/dy/dx pointer is NULL");
  SYSML_CHECK_ALIGN16(f, "filter");
  SYSML_CHECK_ALIGN16(dy, "dy");
  SYSML_CHECK_ALIGN16(dx, "dx");
  SYSML_CHECK_ALIGN16(ws, "workspace");
  const ConvArgs a = conv_args(g);
  size_t need = 0;
  SYSML_TRY(conv_bwd_data_ws(cd, &need));
  if (need > 0 && (ws == nullptr || ws_bytes < need)) {
    set_error("workspace too small: need %zu bytes, got %zu", need, ws ? ws_bytes : 0);
    return SYSML_ERR_WORKSPACE;
  }
  if (cd.math == SYSML_MATH_TF32 && pair_conv_supported(a, 1)) return pair_conv(a, 1, dy, f, nullptr, dx, ws, st);
  if (cd.math == SYSML_MATH_TF32 && c1x1_supported(a, 1)) return c1x1_conv(a, 1, dy, f, nullptr, dx, ws, st);
  if (cd.math == SYSML_MATH_TF32 && tc_bwd_data_supported(a))
    return tc_conv_bwd_data(a, f, dy, dx, ws, st);
  if (cd.math == SYSML_MATH_TF32 && phase_bwd_data_supported(a)) {
    route_note("phase split");
    return phase_conv_bwd_data(a, f, dy, dx, ws, st);
  }
  if (phase_simt_bwd_data_supported(a)) {
    route_note("phase split");
    return phase_simt_conv_bwd_data(a, f, dy, dx, ws, st);
  }
  return simt_conv_bwd_data(a, f, dy, dx, st);
}

}  // namespace sysml

using namespace sysml;

extern "C" {

const char *sysml_version(void) { return "sysml-b200 0.1 (sm_100a; tcgen05 TF32 + fp32 SIMT + CSR)"; }
const char *sysml_last_error(void) { return get_error(); }
const char *sysml_last_route(void) { return route_get(); }
int32_t sysml_device_sm_count(void) { return sm_count(); }
int64_t sysml_launch_counter(void) { return g_launches; }

sysml_status sysml_conv2d_workspace_size(const sysml_conv_desc *d, int32_t is_csr, size_t *bytes) {
  SYSML_CHECK_ARG(d && bytes, "NULL argument");
  return conv_fwd_ws(*d, nullptr, is_csr, bytes);
}

sysml_status sysml_conv2d(const sysml_conv_desc *d, const sysml_input *x, const float *f,
                          const float *bias, float *y, void *workspace, size_t workspace_bytes,
                          sysml_stream_t stream) {
  SYSML_CHECK_ARG(d && x, "NULL descriptor or input");
  return conv_fwd_dispatch(*d, *x, f, bias, y, nullptr, nullptr, nullptr, workspace,
                           workspace_bytes, (cudaStream_t)stream);
}

sysml_status sysml_conv2d_bwd_filter_workspace_size(const sysml_conv_desc *d, int32_t is_csr,
                                                    size_t *bytes) {
  SYSML_CHECK_ARG(d && bytes, "NULL argument");
  return conv_bwd_filter_ws(*d, is_csr, bytes);
}

sysml_status sysml_conv2d_bwd_filter(const sysml_conv_desc *d, const sysml_input *x,
                                     const float *dy, float *df, float *db, void *workspace,
                                     size_t workspace_bytes, sysml_stream_t stream) {
  SYSML_CHECK_ARG(d && x, "NULL descriptor or input");
  return conv_bwd_filter_dispatch(*d, *x, dy, df, db, workspace, workspace_bytes,
                                  (cudaStream_t)stream);
}

sysml_status sysml_conv2d_bwd_data_workspace_size(const sysml_conv_desc *d, size_t *bytes) {
  SYSML_CHECK_ARG(d && bytes, "NULL argument");
  return conv_bwd_data_ws(*d, bytes);
}

sysml_status sysml_conv2d_bwd_data(const sysml_conv_desc *d, const float *f, const float *dy,
                                   float *dx, void *workspace, size_t workspace_bytes,
                                   sysml_stream_t stream) {
  SYSML_CHECK_ARG(d, "NULL descriptor");
  return conv_bwd_data_dispatch(*d, f, dy, dx, workspace, workspace_bytes, (cudaStream_t)stream);
}

sysml_status sysml_affine(int32_t M, int32_t N, int32_t K, const float *x, const float *W,
                          const float *b, int32_t relu, int32_t math, float *out, sysml_stream_t stream) {
  SYSML_CHECK_ARG(M >= 1 && N >= 1 && K >= 1, "affine dims must be >= 1 (M=%d N=%d K=%d)", M, N, K);
  SYSML_CHECK_ARG(x && W && out, "NULL pointer");
  SYSML_CHECK_ARG(math == SYSML_MATH_FP32 || math == SYSML_MATH_TF32, "bad math %d", math);
  SYSML_CHECK_ALIGN16(x, "x");
  SYSML_CHECK_ALIGN16(W, "W");
  SYSML_CHECK_ALIGN16(b, "b");
  SYSML_CHECK_ALIGN16(out, "out");
  cudaStream_t st = (cudaStream_t)stream;
  route_reset();
  if (math == SYSML_MATH_TF32) {
    if (!tc_gemm_supported(M, N, K, K, K)) {
      set_error("affine TF32: unsupported shape M=%d N=%d K=%d (needs N >= 16, K %% 4 == 0)", M, N, K);
      return SYSML_ERR_UNSUPPORTED;
    }
    GemmEpi e;
    e.bias = b;
    e.relu = relu ? 1 : 0;
    return tc_gemm(M, N, K, x, K, W, K, out, N, e, st);
  }
  // FP32: the 1x1 convolution of M one-pixel images with K channels and N filters
  const ConvArgs a{M, K, 1, 1, N, 1, 1, 1, 1, 0, 0, 1, 1};
  route_note("igemm_kernel<FwdOp> [FP32 CUDA cores, affine as 1x1 conv]");
  SYSML_TRY(simt_conv_fwd(a, x, W, b, out, st));
  if (relu) {
    if ((N & 3) != 0) {
      set_error("affine FP32 relu epilogue needs N %% 4 == 0 (N=%d)", N);
      return SYSML_ERR_UNSUPPORTED;
    }
    SYSML_TRY(launch_relu_dropout(out, M, N, 0, 0, nullptr, 0, 1.f, 0, st));
  }
  return SYSML_OK;
}

sysml_status sysml_bias_add(int32_t N, int32_t K, int32_t PQ, float *y, const float *bias,
                            sysml_stream_t stream) {
  SYSML_CHECK_ARG(N >= 1 && K >= 1 && PQ >= 1, "bias_add dims must be >= 1 (N=%d K=%d PQ=%d)", N,
                  K, PQ);
  SYSML_CHECK_ARG(y && bias, "NULL pointer");
  SYSML_CHECK_ALIGN16(y, "y");
  SYSML_CHECK_ALIGN16(bias, "bias");
  return launch_bias_add(N, K, PQ, y, bias, (cudaStream_t)stream);
}

sysml_status sysml_relu_maxpool(const sysml_pool_desc *d, const float *x, float *out,
                                int32_t *argmax, sysml_stream_t stream) {
  ConvGeom g;
  SYSML_TRY(validate_pool(d, &g));
  SYSML_CHECK_ARG(x && out, "NULL pointer");
  SYSML_CHECK_ALIGN16(x, "x");
  SYSML_CHECK_ALIGN16(out, "out");
  SYSML_CHECK_ALIGN16(argmax, "argmax");
  return launch_relu_maxpool(pool_args(g, d->relu ? 1 : 0), x, out, argmax, (cudaStream_t)stream);
}

sysml_status sysml_maxpool_bwd(const sysml_pool_desc *d, const int32_t *argmax,
                               const float *dout, const float *out_mask, float *dx,
                               sysml_stream_t stream) {
  ConvGeom g;
  SYSML_TRY(validate_pool(d, &g));
  SYSML_CHECK_ARG(argmax && dout && dx, "NULL pointer");
  SYSML_CHECK_ALIGN16(argmax, "argmax");
  SYSML_CHECK_ALIGN16(dout, "dout");
  SYSML_CHECK_ALIGN16(out_mask, "out_mask");
  SYSML_CHECK_ALIGN16(dx, "dx");
  return launch_maxpool_bwd(pool_args(g, d->relu ? 1 : 0), argmax, dout, out_mask, dx,
                            (cudaStream_t)stream);
}

sysml_status sysml_conv2d_bias_relu_maxpool_workspace_size(const sysml_conv_desc *cd,
                                                           const sysml_pool_desc *pd,
                                                           int32_t is_csr, size_t *bytes) {
  SYSML_CHECK_ARG(cd && pd && bytes, "NULL argument");
  return conv_fwd_ws(*cd, pd, is_csr, bytes);
}

sysml_status sysml_conv2d_bias_relu_maxpool(const sysml_conv_desc *cd, const sysml_pool_desc *pd,
                                            const sysml_input *x, const float *f,
                                            const float *bias, float *out, int32_t *argmax,
                                            void *workspace, size_t workspace_bytes,
                                            sysml_stream_t stream) {
  SYSML_CHECK_ARG(cd && pd && x, "NULL descriptor or input");
  SYSML_CHECK_ARG(bias != nullptr, "bias pointer is NULL");
  return conv_fwd_dispatch(*cd, *x, f, bias, nullptr, pd, out, argmax, workspace, workspace_bytes,
                           (cudaStream_t)stream);
}

sysml_status sysml_csr_check(const sysml_csr *m, int64_t *violations, sysml_stream_t stream) {
  SYSML_CHECK_ARG(m && violations && m->row_ptr, "NULL argument");
  return csr_check(*m, violations, (cudaStream_t)stream);
}

}  // extern "C"
