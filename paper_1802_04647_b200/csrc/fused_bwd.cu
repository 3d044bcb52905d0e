// fused_bwd.cu -- vertically fused backward block for single-channel conv layers
// ("vertical fusion across layers"):
//
//   dF[k,r,s] = sum_n sum_{pooled (k,p',q')} g * x(n, h + r - ph, w + s - pw)
//   db[k]     = sum_n sum_{pooled (k,p',q')} g
//   with g = dpool[n,k,p',q'] if (mask == NULL or pooled_out > 0) else 0 and
//   (h, w) = the argmax position of the window (S:191-198 routing, reading R9).
//
// This is exactly conv2d_backward_filter(x, maxpool_backward(argmax, dpool, mask)),
// evaluated without materialising the N x (K*P*Q) unpooled gradient: each pooled
// output contributes to one conv-output position only (non-overlapping windows),
// so the work and the bytes scale with the pooled tensor.  Input x is dense or CSR
// (densified per image in shared memory with a zero border = the conv padding).
//
// Determinism: thread t owns filter k = t / TPK and a fixed strided subset of the
// pooled positions; it accumulates all R*S taps + db in registers in a fixed
// (image, position) order; the TPK partials of a filter are summed in a fixed tree,
// per-CTA partials are summed in CTA order by a second kernel.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"
#include "csr_dev.cuh"

namespace sysml {

namespace {

constexpr int FB_THREADS = 256;

struct FusedB1Args {
  int N, H, W, K, R, S, ph, pw, P, Q, Pp, Qp;  // conv (C = 1) + pooled extents
  int Hp, Wp;                                   // padded image in smem
  int P4;                                       // bulk kernel, dense input: row pitch of the 4
                                                //   shifted image copies (0 = one scalar copy)
  int tpk;                                      // threads per filter
  int n_per_cta;
  int64_t mask_plane;                           // > 0: mask is SPF [K][mask_plane]
  int mask_Wf, mask_Lf, mask_off;
  const uint64_t *code;                         // non-null: argmax + mask as 4-bit window codes
  int64_t code_plane;                           //   (TcSpfIO::code) -> the bulk kernel below
  int dpool_nhwc;                               // bulk kernel: dpool[n] is [Pp*Qp][K] (else [K][Pp*Qp])
};

template <int R_, int S_>
__global__ void __launch_bounds__(FB_THREADS)
    pool_bwd_wgrad_c1_kernel(FusedB1Args a, const float *__restrict__ x, sysml_csr xcsr,
                             int is_csr, const float *__restrict__ dpool,
                             const int32_t *__restrict__ argmax, const float *__restrict__ mask,
                             float *__restrict__ part) {
  extern __shared__ float img[];  // Hp x Wp (zero border); reused for the final reduction
  constexpr int RS = R_ * S_;
  const int t = threadIdx.x;
  const int k = t / a.tpk, j = t - k * a.tpk;
  const bool kok = k < a.K;
  const int PpQp = a.Pp * a.Qp, PQ = a.P * a.Q;
  const float invQp = 1.0f / (float)a.Qp;  // exact floor for pp < 2^20 with the +0.5 offset
  float acc[RS];
#pragma unroll
  for (int i = 0; i < RS; ++i) acc[i] = 0.f;
  float dbacc = 0.f;
  const int n0 = blockIdx.x * a.n_per_cta, n1 = min(a.N, n0 + a.n_per_cta);
  const int HpWp = a.Hp * a.Wp;
  for (int n = n0; n < n1; ++n) {
    __syncthreads();
    for (int i = t; i < HpWp; i += FB_THREADS) img[i] = 0.f;
    __syncthreads();
    if (!is_csr) {
      const float *xn = x + (int64_t)n * a.H * a.W;
      for (int i = t; i < a.H * a.W; i += FB_THREADS) {
        const int h = i / a.W, w = i - h * a.W;
        img[(h + a.ph) * a.Wp + w + a.pw] = __ldg(xn + i);
      }
    } else {
      const int j0 = __ldg(xcsr.row_ptr + n), j1 = __ldg(xcsr.row_ptr + n + 1);
      // duplicates summed in stored order (reading R15; csr_dev.cuh)
      csr_scatter_row(xcsr.col_idx, xcsr.val, j0, j1, t, FB_THREADS,
                      [&](int col) -> float * {
                        if (col < 0 || col >= a.H * a.W) return nullptr;
                        const int h = col / a.W, w = col - h * a.W;
                        return img + (h + a.ph) * a.Wp + w + a.pw;
                      },
                      [](bool b) { return __syncthreads_or(b) != 0; });
    }
    __syncthreads();
    if (!kok) continue;
    const int64_t base = (int64_t)n * a.K * PpQp + (int64_t)k * PpQp;
    const int64_t mask_base = (int64_t)k * a.mask_plane + (int64_t)n * a.mask_Lf;
    // 8 pooled outputs per batch: all 24 global loads in flight before any use
    for (int pb = j; pb < PpQp; pb += 8 * a.tpk) {
      float gv[8], mv[8];
      int av[8];
      // all global loads of the batch first; decoding happens after they are in flight
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int pp = pb + u * a.tpk;
        gv[u] = 0.f; mv[u] = 1.f; av[u] = -1;
        if (pp < PpQp) {
          gv[u] = __ldg(dpool + base + pp);
          av[u] = __ldg(argmax + base + pp);
          if (mask) {
            int64_t mi = base + pp;
            if (a.mask_plane > 0) {
              const int pr = __float2int_rz(((float)pp + 0.5f) * invQp), pc = pp - pr * a.Qp;
              mi = mask_base + (pr + a.mask_off) * a.mask_Wf + pc + a.mask_off;
            }
            mv[u] = __ldg(mask + mi);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float g0 = gv[u];
        if (!(mv[u] > 0.f) || g0 == 0.f) continue;  // masked (reading R9) or zero gradient
        const int am = av[u] - k * PQ;               // position inside plane k
        if (am < 0 || am >= PQ) continue;
        const int h = am / a.Q, w = am - h * a.Q;
        const float *win = img + h * a.Wp + w;       // padded coords of tap (0,0)
        dbacc += g0;
#pragma unroll
        for (int r = 0; r < R_; ++r)
#pragma unroll
          for (int s = 0; s < S_; ++s) acc[r * S_ + s] = fmaf(g0, win[r * a.Wp + s], acc[r * S_ + s]);
      }
    }
  }
  // fixed-order reduction of the tpk partials of each filter through shared memory
  __syncthreads();
  float *sred = img;  // reuse (Hp*Wp >= FB_THREADS*(RS+1) is checked on the host)
#pragma unroll
  for (int i = 0; i < RS; ++i) sred[i * FB_THREADS + t] = acc[i];
  sred[RS * FB_THREADS + t] = dbacc;
  __syncthreads();
  const int nout = a.K * (RS + 1);
  for (int o = t; o < nout; o += FB_THREADS) {
    const int kk = o / (RS + 1), i = o - kk * (RS + 1);
    float s = 0.f;
    for (int jj = 0; jj < a.tpk; ++jj) s += sred[i * FB_THREADS + kk * a.tpk + jj];
    part[(int64_t)blockIdx.x * nout + o] = s;
  }
}

// Window-code variant (LeNet TF32 path, 2x2/2 pooling): the pool-gradient plane dpool[n]
// (K x Pp*Qp, contiguous), the 4-bit window codes (positive*4 + dr*2 + ds: argmax and
// relu mask, TcSpfIO::code) and the dense image x[n] are streamed into shared memory by
// 1-D bulk async copies (2-stage ring, mbarrier completion) from a producer warp, so the
// 256 compute threads only touch shared memory.  CSR images are scattered by the
// compute threads from global memory.  Accumulation order as above (deterministic).
constexpr int FBB_STAGES = 2;
constexpr int FBB_THREADS = FB_THREADS + 32;

template <int R_, int S_>
__global__ void __launch_bounds__(FBB_THREADS, 2)
    pool_bwd_wgrad_c1_bulk_kernel(FusedB1Args a, const float *__restrict__ x, sysml_csr xcsr,
                                  int is_csr, const float *__restrict__ dpool,
                                  float *__restrict__ part) {
  extern __shared__ __align__(16) uint8_t fbb_smem[];
  constexpr int RS = R_ * S_;
  const int PpQp = a.Pp * a.Qp, HW = a.H * a.W;
  const int G = (a.K + 15) >> 4;
  const uint32_t g_bytes = (uint32_t)(a.K * PpQp * 4), c_bytes = (uint32_t)(PpQp * 8),
                 x_bytes = is_csr ? 0u : (uint32_t)(HW * 4);
  const uint32_t stage_bytes = (g_bytes + G * c_bytes + x_bytes + 15) & ~15u;
  float *img = reinterpret_cast<float *>(fbb_smem + FBB_STAGES * stage_bytes);  // Hp x Wp
  // dense input: four copies of the padded image, copy j shifted left by j columns, rows of
  // a.P4 floats (16-byte aligned), so every window row is one aligned float4 (+ a scalar for
  // S = 5) whatever its start column; copy bases staggered by 16 banks, a.P4 = 8 mod 32
  const int copy_stride = a.Hp * a.P4 + 16;
  const bool vec = !is_csr && a.P4 > 0;
  uint64_t *full = reinterpret_cast<uint64_t *>(img + (vec ? ((4 * copy_stride + 3) & ~3) : ((a.Hp * a.Wp + 3) & ~3)));
  uint64_t *empty = full + FBB_STAGES;
  const int t = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, t >> 5, 0), lane = t & 31;
  const int n0 = blockIdx.x * a.n_per_cta, n1 = min(a.N, n0 + a.n_per_cta);
  for (int i = t; i < (vec ? 4 * copy_stride : a.Hp * a.Wp); i += blockDim.x) img[i] = 0.f;  // zero border
  if (t == 0) {
    for (int s_ = 0; s_ < FBB_STAGES; ++s_) {
      ptx::mbar_init(full + s_, 1);
      ptx::mbar_init(empty + s_, FB_THREADS / 32);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (warp == FB_THREADS / 32) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int n = n0; n < n1; ++n) {
        ptx::mbar_wait(empty + st, ph ^ 1);
        ptx::mbar_arrive_expect_tx(full + st, g_bytes + G * c_bytes + x_bytes);
        uint8_t *dst = fbb_smem + st * stage_bytes;
        ptx::bulk_g2s(dst, dpool + (int64_t)n * a.K * PpQp, g_bytes, full + st);
        for (int g = 0; g < G; ++g)
          ptx::bulk_g2s(dst + g_bytes + g * c_bytes, a.code + g * a.code_plane + (int64_t)n * PpQp,
                        c_bytes, full + st);
        if (!is_csr)
          ptx::bulk_g2s(dst + g_bytes + G * c_bytes, x + (int64_t)n * HW, x_bytes, full + st);
        if (++st == FBB_STAGES) { st = 0; ph ^= 1; }
      }
    }
    return;
  }
  // lane = filter k (K <= 32), warp w = every 8th pooled position: the window reads of a
  // warp touch at most 4 distinct addresses (the 2x2 winners) -> broadcasts, no conflicts
  const int k = lane, wq = warp;
  const bool kok = k < a.K;
  const int kk = kok ? k : 0;
  const float invQ = 1.0f / (float)a.Qp, invW = 1.0f / (float)a.W;
  float acc[RS];
#pragma unroll
  for (int i = 0; i < RS; ++i) acc[i] = 0.f;
  float dbacc = 0.f;
  int st = 0;
  uint32_t ph = 0;
  for (int n = n0; n < n1; ++n) {
    ptx::mbar_wait(full + st, ph);
    const uint8_t *sb = fbb_smem + st * stage_bytes;
    const float *gs = reinterpret_cast<const float *>(sb);
    const unsigned long long *cs = reinterpret_cast<const unsigned long long *>(sb + g_bytes);
    ptx::named_bar_sync(1, FB_THREADS);  // previous image's window reads are done
    if (vec) {
      const float *xs = reinterpret_cast<const float *>(sb + g_bytes + G * c_bytes);
      for (int i = t; i < HW; i += FB_THREADS) {
        const int h = __float2int_rz(((float)i + 0.5f) * invW), w = i - h * a.W;
        const float v = xs[i];
        float *row = img + (h + a.ph) * a.P4 + w + a.pw;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (w + a.pw - j >= 0) row[j * copy_stride - j] = v;
      }
    } else if (!is_csr) {
      const float *xs = reinterpret_cast<const float *>(sb + g_bytes + G * c_bytes);
      for (int i = t; i < HW; i += FB_THREADS) {
        const int h = __float2int_rz(((float)i + 0.5f) * invW), w = i - h * a.W;
        img[(h + a.ph) * a.Wp + w + a.pw] = xs[i];
      }
    } else {
      for (int i = t; i < HW; i += FB_THREADS) {
        const int h = __float2int_rz(((float)i + 0.5f) * invW), w = i - h * a.W;
        img[(h + a.ph) * a.Wp + w + a.pw] = 0.f;
      }
      ptx::named_bar_sync(1, FB_THREADS);
      const int j0 = __ldg(xcsr.row_ptr + n), j1 = __ldg(xcsr.row_ptr + n + 1);
      // duplicates summed in stored order (reading R15; csr_dev.cuh)
      csr_scatter_row(xcsr.col_idx, xcsr.val, j0, j1, t, FB_THREADS,
                      [&](int col) -> float * {
                        if (col < 0 || col >= HW) return nullptr;
                        const int h = col / a.W, w = col - h * a.W;
                        return img + (h + a.ph) * a.Wp + w + a.pw;
                      },
                      [](bool b) { return named_bar_or(1, FB_THREADS, b); });
    }
    ptx::named_bar_sync(1, FB_THREADS);  // image ready
    {
      // pooled gradient of (k, pp): [K][PpQp] or, channel-minor, [PpQp][K] (lanes contiguous)
      const int gsk = a.dpool_nhwc ? 1 : PpQp, gsp = a.dpool_nhwc ? a.K : 1;
      const float *gk = gs + kk * gsk;
      const unsigned long long *ck = cs + (kk >> 4) * PpQp;
      const int sh = 4 * (kk & 15);
#pragma unroll 2
      for (int pp = wq; pp < PpQp; pp += FB_THREADS / 32) {
        const float g0 = gk[pp * gsp];
        const uint32_t cd = (uint32_t)(ck[pp] >> sh) & 15u;
        // masked (reading R9) lanes add g = 0: every lane stays on the same path
        const float g = (kok && (cd & 4u)) ? g0 : 0.f;
        const int pr = __float2int_rz(((float)pp + 0.5f) * invQ), pc = pp - pr * a.Qp;
        dbacc += g;
        if (vec) {
          const int row0 = 2 * pr + (int)((cd >> 1) & 1u), col0 = 2 * pc + (int)(cd & 1u), j = col0 & 3;
          const float *win = img + j * copy_stride + row0 * a.P4 + (col0 - j);  // 16-byte aligned
#pragma unroll
          for (int r = 0; r < R_; ++r) {
            const float4 q = *reinterpret_cast<const float4 *>(win + r * a.P4);
            acc[r * S_ + 0] = fmaf(g, q.x, acc[r * S_ + 0]);
            if (S_ > 1) acc[r * S_ + 1] = fmaf(g, q.y, acc[r * S_ + 1]);
            if (S_ > 2) acc[r * S_ + 2] = fmaf(g, q.z, acc[r * S_ + 2]);
            if (S_ > 3) acc[r * S_ + 3] = fmaf(g, q.w, acc[r * S_ + 3]);
            if (S_ == 5) acc[r * S_ + 4] = fmaf(g, win[r * a.P4 + 4], acc[r * S_ + 4]);
          }
        } else {
          const float *win = img + (2 * pr + (int)((cd >> 1) & 1u)) * a.Wp + 2 * pc + (int)(cd & 1u);
#pragma unroll
          for (int r = 0; r < R_; ++r)
#pragma unroll
            for (int s_ = 0; s_ < S_; ++s_) acc[r * S_ + s_] = fmaf(g, win[r * a.Wp + s_], acc[r * S_ + s_]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(empty + st);
    if (++st == FBB_STAGES) { st = 0; ph ^= 1; }
  }
  // fixed-order reduction of the tpk partials of each filter (reuses the stage ring)
  ptx::named_bar_sync(1, FB_THREADS);
  float *sred = reinterpret_cast<float *>(fbb_smem);
#pragma unroll
  for (int i = 0; i < RS; ++i) sred[i * FB_THREADS + t] = acc[i];
  sred[RS * FB_THREADS + t] = dbacc;
  ptx::named_bar_sync(1, FB_THREADS);
  const int nout = a.K * (RS + 1);
  for (int o = t; o < nout; o += FB_THREADS) {
    const int ko = o / (RS + 1), i = o - ko * (RS + 1);
    float sum = 0.f;
    for (int w = 0; w < FB_THREADS / 32; ++w) sum += sred[i * FB_THREADS + w * 32 + ko];  // warp order
    part[(int64_t)blockIdx.x * nout + o] = sum;
  }
}

// block (32, 8): lane x owns output o, row y sums the y-th contiguous eighth of the CTA
// partials in order; the row sums are added in row order (deterministic)
__global__ void fused_b1_reduce_kernel(const float *__restrict__ part, int parts, int K, int RS,
                                       float *__restrict__ df, float *__restrict__ db) {
  __shared__ float red[32][33];
  const int nout = K * (RS + 1);
  const int x = threadIdx.x, y = threadIdx.y;
  const int ny = blockDim.y;  // <= 32 slices of the partials, summed in slice order
  const int c0 = y * parts / ny, c1 = (y + 1) * parts / ny;
  for (int base = blockIdx.x * 32; base < nout; base += gridDim.x * 32) {
    const int o = base + x;
    float s = 0.f;
    if (o < nout)
      for (int c = c0; c < c1; ++c) s += __ldg(part + (int64_t)c * nout + o);
    red[y][x] = s;
    __syncthreads();
    if (y == 0 && o < nout) {
      float t = 0.f;
      for (int g = 0; g < ny; ++g) t += red[g][x];
      const int kk = o / (RS + 1), i = o - kk * (RS + 1);
      if (i < RS) df[kk * RS + i] = t;
      else if (db) db[kk] = t;
    }
    __syncthreads();
  }
}

int fused_b1_ctas(int N) {
  // at least 4 images per CTA (keeps the partial count, and the reduce, small at small
  // batches; 8 measured 2% slower at batch 1024, 2 as well), at most 4 CTAs per SM
  int ctas = std::min(4 * sm_count(), (N + 3) / 4);
  if (ctas > N) ctas = N;
  return ctas < 1 ? 1 : ctas;
}

}  // namespace

bool fused_pool_bwd_wgrad_supported(const ConvArgs &c, const PoolArgs &pa) {
  const int RS = c.R * c.S;
  return c.C == 1 && c.sh == 1 && c.sw == 1 && ((c.R == 5 && c.S == 5) || (c.R == 3 && c.S == 3)) &&
         c.K <= FB_THREADS &&
         pa.sh == pa.R && pa.sw == pa.S && pa.ph == 0 && pa.pw == 0 && pa.H == c.P && pa.W == c.Q &&
         (size_t)(c.H + 2 * c.ph) * (c.W + 2 * c.pw) * 4 <= 48 * 1024;
}

size_t fused_pool_bwd_wgrad_ws(const ConvArgs &c) {
  const int RS = c.R * c.S;
  return align_up((size_t)fused_b1_ctas(c.N) * c.K * (RS + 1) * sizeof(float), 256);
}

sysml_status fused_pool_bwd_wgrad(const ConvArgs &c, const PoolArgs &pa, const float *x,
                                  const sysml_csr *xcsr, const float *dpool,
                                  const int32_t *argmax, const float *mask, float *df, float *db,
                                  void *ws, cudaStream_t st, const TcSpfIO *mask_spf,
                                  int dpool_nhwc) {
  FusedB1Args a{};
  a.dpool_nhwc = dpool_nhwc;
  if (mask_spf) {
    a.mask_plane = mask_spf->out_plane;
    a.mask_Wf = mask_spf->out_Wf;
    a.mask_Lf = mask_spf->out_Lf;
    a.mask_off = mask_spf->out_off;
    a.code = mask_spf->code;
    a.code_plane = mask_spf->code_plane;
  }
  a.N = c.N; a.H = c.H; a.W = c.W; a.K = c.K; a.R = c.R; a.S = c.S; a.ph = c.ph; a.pw = c.pw;
  a.P = c.P; a.Q = c.Q; a.Pp = pa.P; a.Qp = pa.Q;
  a.Hp = c.H + 2 * c.ph;
  a.Wp = c.W + 2 * c.pw;
  a.tpk = FB_THREADS / c.K;
  const int ctas = fused_b1_ctas(c.N);
  a.n_per_cta = (int)ceil_div(c.N, ctas);
  const int used = (int)ceil_div(c.N, a.n_per_cta);
  const int RS = c.R * c.S;
  // the reduction reuses the image buffer: need FB_THREADS*(RS+1) floats
  size_t smem = std::max((size_t)a.Hp * a.Wp, (size_t)FB_THREADS * (RS + 1)) * sizeof(float);
  float *part = reinterpret_cast<float *>(ws);
  sysml_csr empty{};
  const sysml_csr &cs = xcsr ? *xcsr : empty;
  if (dpool_nhwc && !a.code) {
    set_error("fused pool-bwd + conv1 wgrad: a channel-minor pooled gradient needs the window-code path");
    return SYSML_ERR_UNSUPPORTED;
  }
  if (a.code) {
    if (c.K > 32 || pa.R != 2 || pa.S != 2 || ((uintptr_t)dpool & 15) || (!xcsr && ((uintptr_t)x & 15)) ||
        ((int64_t)c.K * pa.P * pa.Q) % 4 || (pa.P * pa.Q) % 2 || (c.H * c.W) % 4) {
      set_error("fused pool-bwd + conv1 wgrad: window codes need 2x2 pooling and 16-byte aligned planes");
      return SYSML_ERR_UNSUPPORTED;
    }
    // padded-image row pitch = 2 mod 32: the four 2x2-window candidates of a warp's window
    // reads ((dr, ds) offsets 0, 1, pitch, pitch+1) fall in four different banks
    a.Wp = (a.Wp + 31 - 2) / 32 * 32 + 2;
    static const int vec_env = getenv("SYSML_B1_VEC") ? atoi(getenv("SYSML_B1_VEC")) : 1;
    // four shifted copies, pitch = 8 mod 32 floats and >= Wp + 3 (a window row may start at
    // any column <= W + 2 pw - S and reads 8 floats from its aligned start)
    a.P4 = (!xcsr && vec_env && c.S <= 5) ? (c.W + 2 * c.pw + 3 + 31 - 8) / 32 * 32 + 8 : 0;
    const size_t img_bytes = a.P4 ? align_up((size_t)4 * (a.Hp * a.P4 + 16) * 4, 16)
                                  : align_up((size_t)a.Hp * a.Wp * 4, 16);
    const int G = (c.K + 15) / 16;
    const size_t stage = align_up((size_t)c.K * pa.P * pa.Q * 4 + (size_t)G * pa.P * pa.Q * 8 +
                                      (xcsr ? 0 : (size_t)c.H * c.W * 4), 16);
    const size_t smem_b = std::max(FBB_STAGES * stage, (size_t)FB_THREADS * (RS + 1) * 4) + img_bytes +
                          8 * 2 * FBB_STAGES;
    const size_t smem_bulk = FBB_STAGES * stage + img_bytes + 8 * 2 * FBB_STAGES;
    const size_t sm_need = std::max(smem_b, smem_bulk);
    if (b1_tc_supported(c, pa, true, dpool_nhwc != 0, xcsr != nullptr)) {  // tensor-core form (b1_tc.cu)
      int used_tc = 0;
      SYSML_TRY(b1_tc(c, x, dpool, a.code, a.code_plane, part, ctas, &used_tc, st));
      fused_b1_reduce_kernel<<<(unsigned)ceil_div((int64_t)c.K * (RS + 1), 32), dim3(32, 32), 0, st>>>(
          part, used_tc, c.K, RS, df, db);
      SYSML_LAUNCH_CHECK();
      return SYSML_OK;
    }
    auto kern = RS == 25 ? pool_bwd_wgrad_c1_bulk_kernel<5, 5> : pool_bwd_wgrad_c1_bulk_kernel<3, 3>;
    SYSML_TRY(smem_attr(kern, sm_need));
    kern<<<used, FBB_THREADS, sm_need, st>>>(a, x, cs, xcsr != nullptr, dpool, part);
    SYSML_LAUNCH_CHECK();
    fused_b1_reduce_kernel<<<(unsigned)ceil_div((int64_t)c.K * (RS + 1), 32), dim3(32, 32), 0, st>>>(
        part, used, c.K, RS, df, db);
    SYSML_LAUNCH_CHECK();
    return SYSML_OK;
  }
  if (RS == 25) {
    SYSML_TRY(smem_attr(pool_bwd_wgrad_c1_kernel<5, 5>, 64 * 1024));
    pool_bwd_wgrad_c1_kernel<5, 5><<<used, FB_THREADS, smem, st>>>(a, x, cs, xcsr != nullptr, dpool,
                                                                 argmax, mask, part);
  } else {
    SYSML_TRY(smem_attr(pool_bwd_wgrad_c1_kernel<3, 3>, 64 * 1024));
    pool_bwd_wgrad_c1_kernel<3, 3><<<used, FB_THREADS, smem, st>>>(a, x, cs, xcsr != nullptr, dpool,
                                                                argmax, mask, part);
  }
  SYSML_LAUNCH_CHECK();
  fused_b1_reduce_kernel<<<(unsigned)ceil_div((int64_t)c.K * (RS + 1), 32), dim3(32, 32), 0, st>>>(
      part, used, c.K, RS, df, db);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

}  // namespace sysml
