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
#include "tc_ptx.cuh"

namespace sysml {

namespace {

constexpr int PH_SMEM_FLOATS = 8192;  // 32 KB of staged rows per block (gather kernels)

ConvArgs phase_args(const ConvArgs &a) {
  ConvArgs b{};
  b.N = a.N;
  b.K = a.K;
  b.C = (a.sh * a.sw * a.C + 7) / 8 * 8;  // pad channels (zero planes / zero filters): the
                                         // frame bwd_filter and the 8-channel chunks want C % 8 == 0
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
  if (off || !((a.sh > 1 || a.sw > 1) && (a.R > 1 || a.S > 1)) || a.sh > 4 || a.sw > 4) return false;
  // the gathers stage sh input rows / sh*sw phase rows per block in shared memory
  const ConvArgs b = phase_args(a);
  return (int64_t)a.sh * a.W <= PH_SMEM_FLOATS && (int64_t)a.sh * a.sw * b.W <= PH_SMEM_FLOATS;
}

// SYSML_PHASE_FUSED=0: materialise X' / dX' with the gather kernels instead of the in-kernel
// gather / scatter (A/B switch; also exercises the unfused path in tests)
bool fused_ok() {
  static const bool on = [] {
    const char *e = getenv("SYSML_PHASE_FUSED");
    return !(e && e[0] == '0');
  }();
  return on;
}

int grid_for(int64_t total) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 16ll * sm_count()));
}

// X (N x C*H*W) -> X' (N x C'*H'*W'), zero outside the padded image and in the pad channels.
// Block (n*C + c, chunk of `rows` h' rows) stages the input rows it needs, [h0*sh - ph,
// (h0 + rows)*sh - ph), in shared memory with coalesced loads, then writes every phase row
// (a, b, h') of the chunk with coalesced stores (the stride-sw reads hit shared memory).
// Pad-channel planes (C' rounded up to 8) are extra blocks past N*C that only write zeros.
// Output element (n, c', h', w') lives at c'*cstride + n*nstride + h'*Wrow + w' (NCHW: cstride =
// H'W', nstride = C'H'W', Wrow = W'; the framed bwd_filter layout: cstride = plane, nstride =
// H'*Wf, Wrow = Wf); columns W' .. Wrow-1 are written as zeros.

template <int SW>  // the column stride sw, compile-time so w <-> (w', b) needs no division
__global__ void __launch_bounds__(256) phase_split_x_kernel(const float *__restrict__ x, float *__restrict__ xp,
                                                            int N, int C, int H, int W, int sh, int ph,
                                                            int pw, int C2, int H2, int W2, int rows,
                                                            int64_t cstride, int64_t nstride, int Wrow, int vec) {
  __shared__ __align__(16) float srow[PH_SMEM_FLOATS];
  constexpr int sw = SW;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int h0 = blockIdx.y * rows, nrows = min(rows, H2 - h0);
  const int Cph = sh * sw * C;
  if (blockIdx.x >= (unsigned)N * C) {  // zero plane of a pad channel
    const int i = blockIdx.x - N * C, npad = C2 - Cph, n = i / npad, c2 = Cph + i % npad;
    float *dst = xp + c2 * cstride + n * nstride + (int64_t)h0 * Wrow;
    for (int e = tid; e < nrows * Wrow; e += 256) dst[e] = 0.f;
    return;
  }
  const int n = blockIdx.x / C, c = blockIdx.x - n * C;
  const float *xs = x + (int64_t)blockIdx.x * H * W;
  // stage input rows hin = h0*sh - ph + j, j < nrows*sh (zero rows outside the image): a warp
  // per row, lanes over w -- no per-element index division (the kernel is issue-bound otherwise)
  // 4-byte cp.async (zero-fill outside the image): every copy of the thread is in flight at
  // once (plain load -> st.shared chains left the kernel latency-bound at ~2 loads per warp)
  const int hbase = h0 * sh - ph;
  const uint32_t sbase = ptx::smem_u32(srow);
  if (vec) {
    // W % 4 == 0, 16-byte aligned planes: the staged rows are one contiguous span of the
    // plane, copied as 16-byte chunks (rows outside the image zero-filled)
    const int nq = nrows * sh * W / 4, q4w = W / 4;
    for (int e = tid; e < nq; e += 256) {
      const int j = e / q4w, h = hbase + j;
      const bool ok = h >= 0 && h < H;
      ptx::cp_async16(sbase + 16u * e, ok ? xs + (int64_t)h * W + 4 * (e - j * q4w) : xs, ok ? 16u : 0u);
    }
  } else {
    for (int j = threadIdx.y; j < nrows * sh; j += 8) {
      const int h = hbase + j;
      const bool ok = h >= 0 && h < H;
      const float *src = ok ? xs + (int64_t)h * W : xs;
      for (int w = threadIdx.x; w < W; w += 32)
        ptx::cp_async4(sbase + 4u * (j * W + w), ok ? src + w : xs, ok ? 4u : 0u);
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (vec && (Wrow & 3) == 0) {
    // 16-byte stores: thread -> (phase row, 4 consecutive w'); 4 strided shared reads each
    const int nq = Wrow / 4, per_ab = nrows * nq;
    for (int ab = 0; ab < sh * sw; ++ab) {
      const int a = ab / sw, b = ab - a * sw;
      float *dst0 = xp + (ab * C + c) * cstride + n * nstride + (int64_t)h0 * Wrow;
      const float *s0 = srow + a * W + b - pw;
      for (int e = tid; e < per_ab; e += 256) {
        const int hl = e / nq, q4 = e - hl * nq;
        const float *src = s0 + hl * sh * W;
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int w2 = 4 * q4 + k, w = w2 * sw + b - pw;
          v[k] = (w2 < W2 && (unsigned)w < (unsigned)W) ? src[w2 * sw] : 0.f;
        }
        *reinterpret_cast<float4 *>(dst0 + (int64_t)hl * Wrow + 4 * q4) = make_float4(v[0], v[1], v[2], v[3]);
      }
    }
    return;
  }
  // a warp per output row (a, b, h'), lanes over w'; nested loops keep index divisions out of
  // the row loop (rows are short, so per-row overhead is what the kernel issues)
  for (int ab = 0; ab < sh * sw; ++ab) {
    const int a = ab / sw, b = ab - a * sw;
    float *dst0 = xp + (ab * C + c) * cstride + n * nstride + (int64_t)h0 * Wrow;
    const float *s0 = srow + a * W + b - pw;
    for (int hl = threadIdx.y; hl < nrows; hl += 8) {
      const float *src = s0 + hl * sh * W;
      float *dst = dst0 + (int64_t)hl * Wrow;
      for (int w2 = threadIdx.x; w2 < Wrow; w2 += 32) {
        const int w = w2 * sw + b - pw;
        dst[w2] = (w2 < W2 && (unsigned)w < (unsigned)W) ? src[w2 * sw] : 0.f;
      }
    }
  }
}

// F (K x C*R*S) -> F' (K x C'*R'*S'), zero for the padded taps and the pad channels
__global__ void phase_split_f_kernel(const float *__restrict__ f, float *__restrict__ fp, int C, int R,
                                     int S, int sh, int sw, int C2, int R2, int S2, int64_t total) {
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
    fp[i] = (ab < sh * sw && r < R && s < S) ? __ldg(f + ((k * C + c) * R + r) * (int64_t)S + s) : 0.f;
  }
}

// dX'(N x C'*H'*W') -> dX (N x C*H*W): the transpose of phase_split_x (a gather, each Xp
// position belongs to exactly one phase cell).  Block (n*C + c, chunk of `rows` dX rows,
// rows % sh == 0 and (h0 + ph) % sh == 0 unless clipped) stages the phase rows it needs, h' in
// [(h0 + ph)/sh, .. + rows/sh), from all sh*sw phase planes with coalesced loads, then writes
// the dX rows coalesced.
template <int SW>
__global__ void __launch_bounds__(256) phase_merge_dx_kernel(const float *__restrict__ dxp, float *__restrict__ dx,
                                                             int C, int H, int W, int sh, int ph, int pw,
                                                             int C2, int H2, int W2, int rows) {
  __shared__ float srow[PH_SMEM_FLOATS];
  constexpr int sw = SW;
  // chunk in padded-row space: hp in [blockIdx.y*rows, +rows), rows a multiple of sh
  const int hp0 = blockIdx.y * rows, h2b = hp0 / sh, nh2 = min(rows / sh, H2 - h2b);
  const int n = blockIdx.x / C, c = blockIdx.x - n * C;
  // stage [ab][h2 - h2b][w2] for the sh*sw phase planes of channel c: a warp per phase row
  const int per = nh2 > 0 ? nh2 * W2 : 0;
  const uint32_t sbase = ptx::smem_u32(srow);
  for (int ab = 0; ab < sh * sw; ++ab) {
    const float *src0 = dxp + ((int64_t)(n * C2 + ab * C + c) * H2 + h2b) * W2;
    const uint32_t dst0 = sbase + 4u * (ab * per);
    for (int hl = threadIdx.y; hl < nh2; hl += 8)
      for (int w2 = threadIdx.x; w2 < W2; w2 += 32)
        ptx::cp_async4(dst0 + 4u * (hl * W2 + w2), src0 + hl * W2 + w2, 4u);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  float *out = dx + (int64_t)blockIdx.x * H * W;
  for (int a = 0; a < sh; ++a) {
    for (int hl = threadIdx.y; hl * sh < rows; hl += 8) {
      const int h = hp0 + hl * sh + a - ph;
      if (h < 0 || h >= H) continue;
      const float *src = srow + a * sw * per + hl * W2;
      float *o = out + (int64_t)h * W;
      for (int w = threadIdx.x; w < W; w += 32) {
        const int wp = w + pw, w2 = wp / sw, b = wp - w2 * sw;
        o[w] = (hl < nh2 && w2 < W2) ? src[b * per + w2] : 0.f;
      }
    }
  }
}

// dF' (K x C'*R'*S') -> dF (K x C*R*S)
__global__ void phase_merge_df_kernel(const float *__restrict__ dfp, float *__restrict__ df, int C, int R,
                                      int S, int sh, int sw, int C2, int R2, int S2, int64_t total) {
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
  size_t n = (size_t)b.N * b.C * b.H * b.W;
  if (tc_wgrad_frame_supported(b)) {  // bwd_filter may write the framed layout (>= NCHW size)
    int Hs, Wf;
    int64_t plane;
    tc_wgrad_frame_geom(b, &Hs, &Wf, &plane);
    n = std::max(n, (size_t)b.C * plane);
  }
  return align_up(n * sizeof(float), 256);
}
size_t f2_bytes(const ConvArgs &b) {
  return align_up((size_t)b.K * b.C * b.R * b.S * sizeof(float), 256);
}

// frame: write the framed bwd_filter layout (tc_wgrad_frame_geom) instead of NCHW
sysml_status split_x(const ConvArgs &a, const ConvArgs &b, const float *x, float *xp, cudaStream_t st,
                     bool frame = false) {
  int64_t cstride = (int64_t)b.H * b.W, nstride = (int64_t)b.C * b.H * b.W;
  int Wrow = b.W;
  if (frame) {
    int Hs, Wf;
    int64_t plane;
    tc_wgrad_frame_geom(b, &Hs, &Wf, &plane);
    cstride = plane;
    nstride = (int64_t)Hs * Wf;
    Wrow = Wf;
  }
  const int rows = std::max(1, std::min(b.H, PH_SMEM_FLOATS / (a.sh * a.W)));
  const dim3 grid((unsigned)((int64_t)b.N * (b.C - a.sh * a.sw * a.C) + (int64_t)a.N * a.C),
                  (unsigned)ceil_div(b.H, rows));
  // 16-byte paths: input rows 16-byte aligned; output rows too (frame: Wf % 8 == 0, plane % 4
  // == 0; NCHW: W' % 4 == 0 and H'W' % 4 == 0)
  const int vec = (a.W % 4 == 0) && (((uintptr_t)x & 15) == 0) && (((uintptr_t)xp & 15) == 0) &&
                  (Wrow % 4 == 0) && (cstride % 4 == 0) && (nstride % 4 == 0);
#define SYSML_PH_SPLIT(SWV)                                                                            \
  phase_split_x_kernel<SWV><<<grid, dim3(32, 8), 0, st>>>(x, xp, a.N, a.C, a.H, a.W, a.sh, a.ph, a.pw, b.C, b.H, \
                                                          b.W, rows, cstride, nstride, Wrow, vec)
  switch (a.sw) {
    case 1: SYSML_PH_SPLIT(1); break;
    case 2: SYSML_PH_SPLIT(2); break;
    case 3: SYSML_PH_SPLIT(3); break;
    default: SYSML_PH_SPLIT(4); break;
  }
#undef SYSML_PH_SPLIT
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status split_f(const ConvArgs &a, const ConvArgs &b, const float *f, float *fp, cudaStream_t st) {
  const int64_t total = (int64_t)b.K * b.C * b.R * b.S;
  phase_split_f_kernel<<<grid_for(total), 256, 0, st>>>(f, fp, a.C, a.R, a.S, a.sh, a.sw, b.C, b.R, b.S,
                                                        total);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

// ---------------------------------------------------------------- im2col bwd_filter (C < 8)
// For tiny channel counts (the ResNet-50 stem, C = 3) the shifted-window / frame kernels have
// too little reuse per staged row, so bwd_filter is lowered explicitly (P:171-174's im2col):
//   Xcol[n][(c,r,s)][p*Q + q] = Xp[n][c][p*sh + r][q*sw + s]
//   dF[k][(c,r,s)] = sum_{n,p,q} dY[n][k][p*Q + q] Xcol[n][(c,r,s)][p*Q + q]
// which is exactly the 1x1 bwd_filter (K x CRS, positions contiguous in both operands) of the
// TMA-fed tcgen05 GEMM (wgrad_gemm.cu).  Images are processed in chunks that bound Xcol to
// im2col_ws_cap(); chunk partials are summed in chunk order (deterministic).
// Xcol bound per chunk: 512 MB (SYSML_IM2COL_WS_MB overrides; tests force many chunks)
size_t im2col_ws_cap() {
  static const size_t cap = [] {
    const char *e = getenv("SYSML_IM2COL_WS_MB");
    const long mb = e ? atol(e) : 512;
    return (size_t)std::max(1l, mb) << 20;
  }();
  return cap;
}

__global__ void __launch_bounds__(256) im2col_kernel(const float *__restrict__ x, float *__restrict__ xcol, int C,
                                                     int H, int W, int R, int S, int sh, int sw, int ph, int pw,
                                                     int P, int Q, int rows, int PQp) {
  // block (n*CRS + crs, chunk of `rows` output rows), a warp per row, lanes over q
  const int CRS = C * R * S;
  const int n = blockIdx.x / CRS, crs = blockIdx.x - n * CRS;
  const int c = crs / (R * S), rs = crs - c * R * S, r = rs / S, s = rs - r * S;
  const float *xs = x + ((int64_t)n * C + c) * H * W;
  float *dst0 = xcol + (int64_t)blockIdx.x * PQp;  // rows padded to PQp (% 4 == 0) with zeros
  const int p0 = blockIdx.y * rows, p1 = min(P, p0 + rows);
  if (blockIdx.y == 0 && threadIdx.y == 0 && threadIdx.x < PQp - P * Q) dst0[P * Q + threadIdx.x] = 0.f;
  if ((Q & 3) == 0) {
    // float4 stores: thread -> 4 consecutive q of one row (one division per 4 outputs)
    const int nq = Q / 4, tid = threadIdx.y * 32 + threadIdx.x;
    for (int e = tid; e < (p1 - p0) * nq; e += 256) {
      const int pr = e / nq, q0 = 4 * (e - pr * nq), pp = p0 + pr;
      const int h = pp * sh + r - ph;
      const bool rowok = h >= 0 && h < H;
      const float *src = xs + (int64_t)h * W;
      float v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int w = (q0 + k) * sw + s - pw;
        v[k] = (rowok && w >= 0 && w < W) ? __ldg(src + w) : 0.f;
      }
      *reinterpret_cast<float4 *>(dst0 + (int64_t)pp * Q + q0) = make_float4(v[0], v[1], v[2], v[3]);
    }
    return;
  }
  for (int pp = p0 + threadIdx.y; pp < p1; pp += 8) {
    const int h = pp * sh + r - ph;
    const bool rowok = h >= 0 && h < H;
    const float *src = xs + (int64_t)h * W;
    float *dst = dst0 + (int64_t)pp * Q;
    for (int q = threadIdx.x; q < Q; q += 32) {
      const int w = q * sw + s - pw;
      dst[q] = (rowok && w >= 0 && w < W) ? __ldg(src + w) : 0.f;
    }
  }
}

// dY (rows of P*Q) -> dYp (rows of PQp, zero tail) for the 16-byte TMA strides of the GEMM
__global__ void pad_rows_kernel(const float *__restrict__ src, float *__restrict__ dst, int64_t rows, int L,
                                int Lp) {
  const int64_t total = rows * Lp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / Lp;
    const int e = (int)(i - r * Lp);
    dst[i] = e < L ? __ldg(src + r * L + e) : 0.f;
  }
}

__global__ void chunk_sum_kernel(const float *__restrict__ part, float *__restrict__ out, int64_t len,
                                 int nchunks) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int k = 0; k < nchunks; ++k) acc += part[(int64_t)k * len + i];
    out[i] = acc;
  }
}

struct Im2colPlan {
  int nb, nchunks;
  ConvArgs g;  // the 1x1 GEMM of one chunk: N = nb, C = CRS, H*W = P*Q
  int PQp;  // P*Q rounded up to a multiple of 4 (TMA strides); > P*Q pads dY too
  size_t col_bytes, dyp_bytes, part_bytes, dbpart_bytes, gemm_ws;
  bool ok;
};

Im2colPlan plan_im2col(const ConvArgs &a) {
  Im2colPlan pl{};
  pl.ok = false;
  const int64_t CRS = (int64_t)a.C * a.R * a.S, PQ = (int64_t)a.P * a.Q, PQp = (PQ + 3) / 4 * 4;
  const int64_t per_img = CRS * PQp * sizeof(float);
  pl.PQp = (int)PQp;
  if (per_img > (int64_t)im2col_ws_cap()) return pl;
  pl.nb = (int)std::min<int64_t>(a.N, (int64_t)im2col_ws_cap() / per_img);
  pl.nchunks = (a.N + pl.nb - 1) / pl.nb;
  ConvArgs g{};
  g.N = pl.nb; g.C = (int)CRS; g.K = a.K; g.R = g.S = 1; g.sh = g.sw = 1; g.ph = g.pw = 0;
  g.H = g.P = 1; g.W = g.Q = (int)PQp;
  pl.g = g;
  if (!tc_wgrad_1x1_supported(g)) return pl;
  pl.col_bytes = align_up((size_t)pl.nb * per_img, 256);
  pl.dyp_bytes = PQp != PQ ? align_up((size_t)pl.nb * a.K * PQp * sizeof(float), 256) : 0;
  pl.part_bytes = pl.nchunks > 1 ? align_up((size_t)pl.nchunks * a.K * CRS * sizeof(float), 256) : 0;
  pl.dbpart_bytes = pl.nchunks > 1 ? align_up((size_t)pl.nchunks * a.K * sizeof(float), 256) : 0;
  pl.gemm_ws = align_up(tc_wgrad_1x1_ws(g), 256);
  pl.ok = true;
  return pl;
}

sysml_status merge_dx(const ConvArgs &a, const ConvArgs &b, const float *dxp, float *dx, cudaStream_t st) {
  // rows of padded-image space per block: a multiple of sh whose phase rows fit in smem
  const int rows = a.sh * std::max(1, std::min((a.H + a.ph + a.sh - 1) / a.sh, PH_SMEM_FLOATS / (a.sh * a.sw * b.W)));
  const dim3 grid((unsigned)((int64_t)a.N * a.C), (unsigned)ceil_div(a.H + a.ph, rows));
#define SYSML_PH_MERGE(SWV)                                                                          \
  phase_merge_dx_kernel<SWV><<<grid, dim3(32, 8), 0, st>>>(dxp, dx, a.C, a.H, a.W, a.sh, a.ph, a.pw, b.C, b.H, \
                                                           b.W, rows)
  switch (a.sw) {
    case 1: SYSML_PH_MERGE(1); break;
    case 2: SYSML_PH_MERGE(2); break;
    case 3: SYSML_PH_MERGE(3); break;
    default: SYSML_PH_MERGE(4); break;
  }
#undef SYSML_PH_MERGE
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

}  // namespace

bool im2col_bwd_filter_supported(const ConvArgs &a) {
  static const bool off = getenv("SYSML_NO_IM2COL") != nullptr;  // A/B switch
  if (off || (int64_t)a.C * a.R * a.S < 16) return false;
  return plan_im2col(a).ok;
}

size_t im2col_bwd_filter_ws(const ConvArgs &a) {
  const Im2colPlan pl = plan_im2col(a);
  return pl.ok ? pl.col_bytes + pl.dyp_bytes + pl.part_bytes + pl.dbpart_bytes + pl.gemm_ws : 0;
}

sysml_status im2col_conv_bwd_filter(const ConvArgs &a, const float *x, const float *dy, float *df, float *db,
                                    void *ws, cudaStream_t st) {
  const Im2colPlan pl = plan_im2col(a);
  if (!pl.ok) {
    set_error("im2col bwd_filter: unsupported shape");
    return SYSML_ERR_UNSUPPORTED;
  }
  WsCarve wc(ws, im2col_bwd_filter_ws(a));
  float *xcol = reinterpret_cast<float *>(wc.take<char>(pl.col_bytes));
  float *dyp = pl.dyp_bytes ? reinterpret_cast<float *>(wc.take<char>(pl.dyp_bytes)) : nullptr;
  float *dfp = pl.part_bytes ? reinterpret_cast<float *>(wc.take<char>(pl.part_bytes)) : nullptr;
  float *dbp = pl.dbpart_bytes ? reinterpret_cast<float *>(wc.take<char>(pl.dbpart_bytes)) : nullptr;
  void *gws = wc.take<char>(pl.gemm_ws);
  SYSML_WS_FITS(wc);
  const int CRS = a.C * a.R * a.S;
  const int64_t PQ = (int64_t)a.P * a.Q;
  for (int i = 0; i < pl.nchunks; ++i) {
    ConvArgs g = pl.g;
    g.N = std::min(pl.nb, a.N - i * pl.nb);
    const float *xi = x + (int64_t)i * pl.nb * a.C * a.H * a.W;
    const float *dyi = dy + (int64_t)i * pl.nb * a.K * PQ;  // 16-byte aligned when PQ % 4 == 0
    const int rows = std::max(1, std::min(a.P, 4096 / std::max(1, a.Q)));
    const dim3 grid((unsigned)((int64_t)g.N * CRS), (unsigned)ceil_div(a.P, rows));
    im2col_kernel<<<grid, dim3(32, 8), 0, st>>>(xi, xcol, a.C, a.H, a.W, a.R, a.S, a.sh, a.sw, a.ph, a.pw, a.P,
                                                a.Q, rows, pl.PQp);
    SYSML_LAUNCH_CHECK();
    if (dyp) {
      pad_rows_kernel<<<grid_for((int64_t)g.N * a.K * pl.PQp), 256, 0, st>>>(dyi, dyp, (int64_t)g.N * a.K, (int)PQ,
                                                                            pl.PQp);
      SYSML_LAUNCH_CHECK();
      dyi = dyp;
    }
    float *dfo = pl.nchunks > 1 ? dfp + (int64_t)i * a.K * CRS : df;
    float *dbo = db ? (pl.nchunks > 1 ? dbp + (int64_t)i * a.K : db) : nullptr;
    SYSML_TRY(tc_wgrad_1x1(g, xcol, dyi, dfo, dbo, gws, st));
  }
  if (pl.nchunks > 1) {
    chunk_sum_kernel<<<grid_for((int64_t)a.K * CRS), 256, 0, st>>>(dfp, df, (int64_t)a.K * CRS, pl.nchunks);
    SYSML_LAUNCH_CHECK();
    if (db) {
      chunk_sum_kernel<<<grid_for(a.K), 256, 0, st>>>(dbp, db, a.K, pl.nchunks);
      SYSML_LAUNCH_CHECK();
    }
  }
  return SYSML_OK;
}

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
  WsCarve wc(ws, phase_fwd_ws(a));
  float *xp = wc.take<float>((size_t)b.N * b.C * b.H * b.W);
  float *fp = wc.take<float>((size_t)b.K * b.C * b.R * b.S);
  void *tws = wc.take<char>(tc_fwd_ws(b));
  SYSML_WS_FITS(wc);
  SYSML_TRY(split_f(a, b, f, fp, st));
  if (fused_ok() && tc_fwd_phase_fused_ok(a, b))  // X' gathered by the conv kernel's producer
    return tc_conv_fwd_phase(a, b, x, fp, bias, y, tws, st);
  SYSML_TRY(split_x(a, b, x, xp, st));
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
  WsCarve wc(ws, phase_bwd_data_ws(a));
  float *dxp = wc.take<float>((size_t)b.N * b.C * b.H * b.W);
  float *fp = wc.take<float>((size_t)b.K * b.C * b.R * b.S);
  void *tws = wc.take<char>(tc_bwd_data_ws(b));
  SYSML_WS_FITS(wc);
  SYSML_TRY(split_f(a, b, f, fp, st));
  if (fused_ok() && tc_bwd_data_phase_fused_ok(a, b))  // dX' scattered by the conv epilogue
    return tc_conv_bwd_data_phase(a, b, fp, dy, dx, tws, st);
  SYSML_TRY(tc_conv_bwd_data(b, fp, dy, dxp, tws, st));
  return merge_dx(a, b, dxp, dx, st);
}

// FP32 math (no tensor cores): the same split onto the stride-1 SIMT bwd_data.  The strided
// SIMT gather tests every (k, r, s) term for stride divisibility and skips (sh*sw - 1)/(sh*sw)
// of them; over the phases every term is real.
bool phase_simt_bwd_data_supported(const ConvArgs &a) { return is_phase_shape(a); }

size_t phase_simt_bwd_data_ws(const ConvArgs &a) {
  const ConvArgs b = phase_args(a);
  return align_up((size_t)b.N * b.C * b.H * b.W * sizeof(float), 256) + f2_bytes(b);
}

sysml_status phase_simt_conv_bwd_data(const ConvArgs &a, const float *f, const float *dy, float *dx,
                                      void *ws, cudaStream_t st) {
  const ConvArgs b = phase_args(a);
  WsCarve wc(ws, phase_simt_bwd_data_ws(a));
  float *dxp = wc.take<float>((size_t)b.N * b.C * b.H * b.W);
  float *fp = wc.take<float>((size_t)b.K * b.C * b.R * b.S);
  SYSML_WS_FITS(wc);
  SYSML_TRY(split_f(a, b, f, fp, st));
  SYSML_TRY(simt_conv_bwd_data(b, fp, dy, dxp, st));
  return merge_dx(a, b, dxp, dx, st);
}

// ---------------------------------------------------------------- bwd_filter
bool phase_bwd_filter_frame_ok(const ConvArgs &a) {
  return is_phase_shape(a) && tc_wgrad_frame_supported(phase_args(a));
}

bool phase_bwd_filter_supported(const ConvArgs &a) {
  return is_phase_shape(a) && tc_bwd_filter_supported(phase_args(a));
}

// the inner stride-1 problem runs on the frame kernel whenever it supports it (same test as
// phase_conv_bwd_filter below), else on tc_conv_bwd_filter's own route: size for that kernel
static size_t phase_inner_wgrad_ws(const ConvArgs &b) {
  return tc_wgrad_frame_supported(b) ? tc_wgrad_frame_ws(b) : tc_bwd_filter_ws(b);
}

size_t phase_bwd_filter_ws(const ConvArgs &a) {
  const ConvArgs b = phase_args(a);
  return x2_bytes(b) + f2_bytes(b) + align_up(phase_inner_wgrad_ws(b), 256);
}

sysml_status phase_conv_bwd_filter(const ConvArgs &a, const float *x, const float *dy, float *df,
                                   float *db, void *ws, cudaStream_t st) {
  const ConvArgs b = phase_args(a);
  WsCarve wc(ws, phase_bwd_filter_ws(a));
  float *xp = reinterpret_cast<float *>(wc.take<char>(x2_bytes(b)));
  float *dfp = wc.take<float>((size_t)b.K * b.C * b.R * b.S);
  void *tws = wc.take<char>(phase_inner_wgrad_ws(b));
  SYSML_WS_FITS(wc);
  if (tc_wgrad_frame_supported(b)) {  // X' written straight into the frame (no second pass)
    SYSML_TRY(split_x(a, b, x, xp, st, /*frame=*/true));
    SYSML_TRY(tc_wgrad_frame(b, xp, dy, dfp, db, tws, st, /*x_framed=*/true));
  } else {
    SYSML_TRY(split_x(a, b, x, xp, st));
    SYSML_TRY(tc_conv_bwd_filter(b, xp, dy, dfp, db, tws, st));
  }
  const int64_t total = (int64_t)a.K * a.C * a.R * a.S;
  phase_merge_df_kernel<<<grid_for(total), 256, 0, st>>>(dfp, df, a.C, a.R, a.S, a.sh, a.sw, b.C, b.R, b.S,
                                                         total);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

}  // namespace sysml
