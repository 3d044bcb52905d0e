// kernels.cuh -- launcher declarations shared between the API layer and kernels.
#pragma once
#include "common.cuh"

namespace sysml {

struct PoolArgs {
  int N, C, H, W, R, S, sh, sw, ph, pw, P, Q, relu;
};

inline PoolArgs pool_args(const ConvGeom &g, int relu) {
  return PoolArgs{(int)g.N, (int)g.C, (int)g.H, (int)g.W, (int)g.R, (int)g.S, (int)g.sh,
                  (int)g.sw, (int)g.ph, (int)g.pw, (int)g.P, (int)g.Q, relu};
}

struct ConvArgs {
  int N, C, H, W, K, R, S, sh, sw, ph, pw, P, Q;
};

inline ConvArgs conv_args(const ConvGeom &g) {
  return ConvArgs{(int)g.N, (int)g.C, (int)g.H, (int)g.W, (int)g.K, (int)g.R, (int)g.S,
                  (int)g.sh, (int)g.sw, (int)g.ph, (int)g.pw, (int)g.P, (int)g.Q};
}

// pool.cu
sysml_status launch_relu_maxpool(const PoolArgs &a, const float *x, float *out, int32_t *argmax,
                                 cudaStream_t st);
sysml_status launch_maxpool_bwd(const PoolArgs &a, const int32_t *argmax, const float *dout,
                                const float *mask, float *dx, cudaStream_t st);
sysml_status launch_bias_add(int32_t N, int32_t K, int32_t PQ, float *y, const float *bias,
                             cudaStream_t st);
sysml_status launch_zero(float *p, int64_t n, cudaStream_t st);

// conv_simt.cu : fp32 CUDA-core implicit GEMM (all shapes; SYSML_MATH_FP32)
sysml_status simt_conv_fwd(const ConvArgs &a, const float *x, const float *f, const float *bias,
                           float *y, cudaStream_t st);
size_t simt_bwd_filter_ws(const ConvArgs &a);
sysml_status simt_conv_bwd_filter(const ConvArgs &a, const float *x, const float *dy, float *df,
                                  float *db, void *ws, cudaStream_t st);
sysml_status simt_conv_bwd_data(const ConvArgs &a, const float *f, const float *dy, float *dx,
                                cudaStream_t st);
sysml_status launch_bias_grad(const ConvArgs &a, const float *dy, float *db, float *part,
                              cudaStream_t st);
size_t bias_grad_ws(const ConvArgs &a);

// csr.cu : CSR-input kernels (CUDA cores, HBM-bound)
bool csr_fwd_supported(const ConvArgs &a);
sysml_status csr_conv_fwd(const ConvArgs &a, const sysml_csr &x, const float *f,
                          const float *bias, float *y, const PoolArgs *pool, float *pout,
                          int32_t *parg, cudaStream_t st);
bool csr_bwd_filter_supported(const ConvArgs &a);
size_t csr_bwd_filter_ws(const ConvArgs &a);
sysml_status csr_conv_bwd_filter(const ConvArgs &a, const sysml_csr &x, const float *dy,
                                 float *df, float *db, void *ws, cudaStream_t st);
sysml_status csr_densify(const sysml_csr &x, float *dense, cudaStream_t st);
sysml_status csr_check(const sysml_csr &m, int64_t *violations, cudaStream_t st);

// Stacked planar frame (SPF) conv geometry: tensors [C][G] (x) and [K][G] (dy) with
// G = N*Hs*Wf frame positions; stored position = frame position + shift.
struct SpfConv {
  int K, C, R, S, Wf;
  int64_t G, plane_x, plane_dy;
  int x_shift, dy_shift;
};

// SPF input / pooled-output options of the tcgen05 forward kernel (LeNet-internal layout)
struct TcSpfIO {
  int64_t in_plane = 0;  // > 0: input SPF, channel stride in_plane, stored pos = frame pos + in_shift
  int in_shift = 0;
  int64_t out_plane = 0;  // > 0: pooled output to SPF planes (pp + out_off) * out_Wf + pc + out_off
  int out_Wf = 0, out_Lf = 0, out_off = 0;
  uint64_t *code = nullptr;  // pooled argmax + relu mask as packed 4-bit window codes
  int64_t code_plane = 0;    // code[k/16][n*PpQp + pp*Qp + pc]: bits 4j..4j+3 of channel
                             // 16g + j = positive*4 + dr*2 + ds (window winner (2pp+dr, 2pc+ds))
  int out_nhwc = 0;          // SN epilogue (bwd_data): y channel-minor [n][P*Q][K], K % 4 == 0
  // Routed SPF input (NEXT-1 vertical fusion; LeNet conv2 backward): the input is NOT read
  // from planes -- the producer builds each unpooled gradient value from the pooled gradient
  // route_val[(n*PpQp + window)*route_C + c] and the window code of (c, n, window) in
  // route_code (layout of `code` above): value = positive && winner == (dr, ds) ? val : 0.
  // Frame geometry: in_plane / in_shift as for SPF input (output-frame convention, Lf
  // positions per image, Wf per row); windows 2x2/2 over route_Pp x route_Qp.
  const float *route_val = nullptr;
  const uint64_t *route_code = nullptr;
  int64_t route_cplane = 0;
  int route_C = 0, route_Pp = 0, route_Qp = 0, route_Wf = 0, route_Lf = 0;
};

// conv_tc.cu : tcgen05 TF32 implicit GEMM (SYSML_MATH_TF32)

// K5 1x1 (stride 1, pad 0): TMA-fed GEMM over positions (wgrad_gemm.cu)
bool tc_wgrad_1x1_supported(const ConvArgs &a);
size_t tc_wgrad_1x1_ws(const ConvArgs &a);
sysml_status tc_wgrad_1x1(const ConvArgs &a, const float *x, const float *dy, float *df,
                          float *db, void *ws, cudaStream_t st);
// fused conv(C = 1) + bias + relu + 2x2/2 pool with the window in N (conv1_pool.cu)
bool conv1_pool_supported(const ConvArgs &a, const PoolArgs *pool);
size_t conv1_pool_ws(const ConvArgs &a, const PoolArgs *pool);
sysml_status conv1_pool(const ConvArgs &a, const PoolArgs *pool, const float *x, const float *f,
                        const float *bias, float *pout, int32_t *parg, void *ws, cudaStream_t st,
                        const TcSpfIO *io = nullptr, const sysml_csr *csr = nullptr);
bool tc_fwd_supported(const ConvArgs &a, const PoolArgs *pool);
// single-channel convs (C == 1, S <= 8) use the KS operand mode, which also reads CSR input
bool tc_fwd_ks(const ConvArgs &a);
size_t tc_fwd_ws(const ConvArgs &a);
sysml_status tc_conv_fwd(const ConvArgs &a, const float *x, const float *f, const float *bias,
                         float *y, const PoolArgs *pool, float *pout, int32_t *parg, void *ws,
                         cudaStream_t st, const sysml_csr *csr = nullptr);
// phase-split modes of the forward kernel (conv_tc.cu): a = the strided conv, b = its
// stride-1 pad-0 phase problem (phase.cu); the gather / scatter of X' / dX' happens in-kernel
bool tc_fwd_phase_fused_ok(const ConvArgs &a, const ConvArgs &b);
sysml_status tc_conv_fwd_phase(const ConvArgs &a, const ConvArgs &b, const float *x, const float *fp,
                               const float *bias, float *y, void *ws, cudaStream_t st);
bool tc_bwd_data_phase_fused_ok(const ConvArgs &a, const ConvArgs &b);
sysml_status tc_conv_bwd_data_phase(const ConvArgs &a, const ConvArgs &b, const float *fp, const float *dy,
                                    float *dx, void *ws, cudaStream_t st);
// phase.cu : strided convs with R or S > 1 as stride-1 tcgen05 convs over the phase-split
// input (space-to-depth); DESIGN.md §7 "Strided convolutions"
bool phase_fwd_supported(const ConvArgs &a);
size_t phase_fwd_ws(const ConvArgs &a);
sysml_status phase_conv_fwd(const ConvArgs &a, const float *x, const float *f, const float *bias,
                            float *y, void *ws, cudaStream_t st);
bool phase_bwd_data_supported(const ConvArgs &a);
size_t phase_bwd_data_ws(const ConvArgs &a);
sysml_status phase_conv_bwd_data(const ConvArgs &a, const float *f, const float *dy, float *dx,
                                 void *ws, cudaStream_t st);
// C < 8 bwd_filter lowered to im2col + the 1x1 TMA GEMM (phase.cu)
bool im2col_bwd_filter_supported(const ConvArgs &a);
size_t im2col_bwd_filter_ws(const ConvArgs &a);
sysml_status im2col_conv_bwd_filter(const ConvArgs &a, const float *x, const float *dy, float *df, float *db,
                                    void *ws, cudaStream_t st);
bool phase_simt_bwd_data_supported(const ConvArgs &a);
size_t phase_simt_bwd_data_ws(const ConvArgs &a);
sysml_status phase_simt_conv_bwd_data(const ConvArgs &a, const float *f, const float *dy, float *dx,
                                      void *ws, cudaStream_t st);
bool phase_bwd_filter_frame_ok(const ConvArgs &a);  // the phase problem fits the TMA frame kernel
bool phase_bwd_filter_supported(const ConvArgs &a);
size_t phase_bwd_filter_ws(const ConvArgs &a);
sysml_status phase_conv_bwd_filter(const ConvArgs &a, const float *x, const float *dy, float *df,
                                   float *db, void *ws, cudaStream_t st);
bool tc_bwd_filter_fast_supported(const ConvArgs &a);  // 1x1 / strided 1x1 / framed TMA kernels
bool tc_bwd_data_supported(const ConvArgs &a);
size_t tc_bwd_data_ws(const ConvArgs &a);
sysml_status tc_conv_bwd_data(const ConvArgs &a, const float *f, const float *dy, float *dx,
                              void *ws, cudaStream_t st);
sysml_status tc_conv_fwd_spf(const ConvArgs &a, const TcSpfIO &io, const float *x, const float *f,
                             const float *bias, float *y, const PoolArgs *pool, float *pout,
                             int32_t *parg, void *ws, cudaStream_t st,
                             const sysml_csr *csr = nullptr);
// true when the SN epilogue serves this bwd_data, so TcSpfIO::out_nhwc may be set
bool tc_conv_bwd_data_spf_nhwc_ok(const ConvArgs &a);
sysml_status tc_conv_bwd_data_spf(const ConvArgs &a, const TcSpfIO &io, const float *f,
                                  const float *dy, float *dx, void *ws, cudaStream_t st);
bool tc_wgrad_spf_supported(const SpfConv &sc);
// TMA-fed variant (wgrad_spf_tma.cu): ring of X atoms, no halo re-fetch
bool tc_wgrad_spf_tma_supported(const SpfConv &sc);
size_t tc_wgrad_spf_tma_ws(const SpfConv &sc);
sysml_status tc_wgrad_spf_tma(const SpfConv &sc, const float *x_spf, const float *dy_spf,
                              float *df, float *db, void *ws, cudaStream_t st,
                              const float *db_src = nullptr, int db_count = 0);
// NCHW entry: framing pre-pass + the TMA kernel (stride 1, C % 8 == 0)
bool tc_wgrad_frame_supported(const ConvArgs &a);
size_t tc_wgrad_frame_ws(const ConvArgs &a);
// x_framed: x is already in the frame layout of tc_wgrad_frame_geom (planes [c][plane],
// image n at n*Hs*Wf, pixel (h, w) at (h + ph)*Wf + w + pw, zeros elsewhere)
sysml_status tc_wgrad_frame(const ConvArgs &a, const float *x, const float *dy, float *df,
                            float *db, void *ws, cudaStream_t st, bool x_framed = false);
void tc_wgrad_frame_geom(const ConvArgs &a, int *Hs, int *Wf, int64_t *plane);
size_t tc_wgrad_spf_ws(const SpfConv &sc);
sysml_status tc_wgrad_spf(const SpfConv &sc, const float *x_spf, const float *dy_spf, float *df,
                          float *db, void *ws, cudaStream_t st);
bool tc_bwd_filter_supported(const ConvArgs &a);
size_t tc_bwd_filter_ws(const ConvArgs &a);
sysml_status tc_conv_bwd_filter(const ConvArgs &a, const float *x, const float *dy, float *df,
                                float *db, void *ws, cudaStream_t st);

// fused_bwd.cu : maxpool_bwd + conv2d_bwd_filter for single-channel conv layers
bool fused_pool_bwd_wgrad_supported(const ConvArgs &c, const PoolArgs &pa);
size_t fused_pool_bwd_wgrad_ws(const ConvArgs &c);
sysml_status fused_pool_bwd_wgrad(const ConvArgs &c, const PoolArgs &pa, const float *x,
                                  const sysml_csr *xcsr, const float *dpool,
                                  const int32_t *argmax, const float *mask, float *df, float *db,
                                  void *ws, cudaStream_t st, const TcSpfIO *mask_spf = nullptr,
                                  int dpool_nhwc = 0);  // dpool [n][Pp*Qp][K] (window-code path)

// pool.cu : LeNet-internal layout helpers
// maxpool_bwd (non-overlapping windows) writing the unpooled gradient into SPF planes
// [C][plane], position n*Lf + h*Wf + w (only the window positions are written).
sysml_status launch_maxpool_bwd_spf(const PoolArgs &a, const int32_t *argmax, const float *dout,
                                    const float *mask, float *dx_spf, int64_t plane, int Wf,
                                    int Lf, cudaStream_t st);
// NCHW (N x C*H*W) -> SPF planes [C][plane] at n*Lf + (h+off)*Wf + (w+off)
sysml_status launch_nchw_to_spf(int N, int C, int H, int W, const float *x, float *spf,
                                int64_t plane, int Wf, int Lf, int off, cudaStream_t st);

// conv1x1_tmem.cu : 1x1 stride-1 conv fwd / bwd_data, activation transposed through TMEM
bool c1x1_supported(const ConvArgs &a, int bwd_data);
size_t c1x1_ws(const ConvArgs &a, int bwd_data);
sysml_status c1x1_conv(const ConvArgs &a, int bwd_data, const float *in, const float *f, const float *bias,
                       float *out, void *ws, cudaStream_t st);

// pair_conv.cu : stride-1 conv fwd / bwd_data on CTA pairs (cta_group::2, M = 256) for 256-wide
// filter banks; bwd_data = 1 computes dX = conv(dY, rot180(F)^T)
bool pair_conv_supported(const ConvArgs &a, int bwd_data);
size_t pair_conv_ws(const ConvArgs &a, int bwd_data);
sysml_status pair_conv(const ConvArgs &a, int bwd_data, const float *x, const float *f, const float *bias,
                       float *y, void *ws, cudaStream_t st);

// b1_tc.cu : LeNet conv1 wgrad + pool1 backward on the tensor cores (window candidates stacked)
bool b1_tc_supported(const ConvArgs &c, const PoolArgs &pa, bool has_codes, bool nhwc, bool csr);
sysml_status b1_tc(const ConvArgs &c, const float *x, const float *dpool, const uint64_t *code, int64_t code_plane,
                   float *part, int max_ctas, int *used, cudaStream_t st);

// snt_fwd.cu : LeNet conv2 forward + bias + relu + 2x2 pool, SN-T (T = 3) with resident filters
bool snt_fwd_pool_supported(const ConvArgs &a, const PoolArgs *pool, int Wf, int Lf);
size_t snt_fwd_pool_ws(const ConvArgs &a);
sysml_status snt_fwd_pool_spf(const ConvArgs &a, const TcSpfIO &io, const float *x, const float *f,
                              const float *bias, float *pout, void *ws, cudaStream_t st);

// sn_tmem.cu : narrow-filter SN bwd_data with the A operand in TMEM and resident filters
// (LeNet conv2 bwd_data on SPF planes; output frame Wf x (Lf / Wf))
bool sn_tmem_supported(const ConvArgs &a, int Wf, int Lf);
size_t sn_tmem_ws(const ConvArgs &a, int Wf, int Lf);
sysml_status sn_tmem_bwd_data_spf(const ConvArgs &a, const TcSpfIO &io, int Wf, int Lf, const float *f,
                                  const float *dy, float *dx, void *ws, cudaStream_t st);

// affine_gemm.cu : the affine layers of the LeNet-512 step (NEXT-4)
// Fused epilogue of tc_gemm: C = acc (+ bias[col]) (relu) (inverted dropout of unit col of
// global row row0 + row: Philox4x64-10 stream (seed, *step), kept iff (raw >> 32) < keep_T)
struct GemmEpi {
  const float *bias = nullptr;
  int relu = 0, dropout = 0;
  uint64_t keep_T = 0;
  float keep_p = 1.f;
  uint64_t seed = 0;
  const uint64_t *step = nullptr;  // device counter (advances once per training step)
  int64_t row0 = 0;
  int units = 0;                    // mask row length (= N)
};
bool tc_gemm_supported(int M, int N, int K, int64_t lda, int64_t ldb);
// C[M][N] (row stride ldc) = A[M][K] (lda) . B[N][K]^T (ldb), tcgen05 TF32, fp32 accumulate
sysml_status tc_gemm(int M, int N, int K, const float *A, int64_t lda, const float *B, int64_t ldb,
                     float *C, int64_t ldc, const GemmEpi &e, cudaStream_t st);
sysml_status launch_transpose(const float *in, int R, int Cc, int64_t ldi, float *out, int64_t ldo,
                              cudaStream_t st);
sysml_status launch_dz3(int n, int H, const float *ds, const float *W4, const float *h, float keep_p,
                        float *dz3, float *dz3T, int64_t ldt, cudaStream_t st);
sysml_status launch_relu_dropout(float *z, int n, int H, int64_t row0, uint64_t seed, const uint64_t *step,
                                 uint64_t T, float keep_p, int dropout, cudaStream_t st);
sysml_status launch_counter_inc(uint64_t *c, cudaStream_t st);
int route_da2_chunks(int n);
sysml_status launch_route_da2_spf(int n, const float *da2, const uint64_t *c2, int64_t cplane, float *dz2s,
                                  int64_t plane, float *dbpart, cudaStream_t st);

}  // namespace sysml
