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

namespace sysml {

namespace {

constexpr int FB_THREADS = 256;

struct FusedB1Args {
  int N, H, W, K, R, S, ph, pw, P, Q, Pp, Qp;  // conv (C = 1) + pooled extents
  int Hp, Wp;                                   // padded image in smem
  int tpk;                                      // threads per filter
  int n_per_cta;
  int64_t mask_plane;                           // > 0: mask is SPF [K][mask_plane]
  int mask_Wf, mask_Lf, mask_off;
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
      for (int jj = j0 + t; jj < j1; jj += FB_THREADS) {
        const int col = __ldg(xcsr.col_idx + jj);
        if (col >= 0 && col < a.H * a.W) {
          const int h = col / a.W, w = col - h * a.W;
          atomicAdd(img + (h + a.ph) * a.Wp + w + a.pw, __ldg(xcsr.val + jj));  // duplicates summed
        }
      }
    }
    __syncthreads();
    if (!kok) continue;
    const int64_t base = (int64_t)n * a.K * PpQp + (int64_t)k * PpQp;
    // 8 pooled outputs per batch: all 24 global loads in flight before any use
    for (int pb = j; pb < PpQp; pb += 8 * a.tpk) {
      float gv[8], mv[8];
      int av[8];
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
              const int pr = pp / a.Qp, pc = pp - pr * a.Qp;
              mi = (int64_t)k * a.mask_plane + (int64_t)n * a.mask_Lf + (pr + a.mask_off) * a.mask_Wf +
                   pc + a.mask_off;
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

__global__ void fused_b1_reduce_kernel(const float *__restrict__ part, int parts, int K, int RS,
                                       float *__restrict__ df, float *__restrict__ db) {
  const int nout = K * (RS + 1);
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < nout; o += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < parts; ++c) s += part[(int64_t)c * nout + o];
    const int kk = o / (RS + 1), i = o - kk * (RS + 1);
    if (i < RS) df[kk * RS + i] = s;
    else if (db) db[kk] = s;
  }
}

int fused_b1_ctas(int N) {
  int ctas = 4 * sm_count();
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
                                  void *ws, cudaStream_t st, const TcSpfIO *mask_spf) {
  FusedB1Args a{};
  if (mask_spf) {
    a.mask_plane = mask_spf->out_plane;
    a.mask_Wf = mask_spf->out_Wf;
    a.mask_Lf = mask_spf->out_Lf;
    a.mask_off = mask_spf->out_off;
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
  if (RS == 25) {
    static bool attr = false;
    if (!attr) {
      SYSML_CUDA(cudaFuncSetAttribute(pool_bwd_wgrad_c1_kernel<5, 5>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
      attr = true;
    }
    pool_bwd_wgrad_c1_kernel<5, 5><<<used, FB_THREADS, smem, st>>>(a, x, cs, xcsr != nullptr, dpool,
                                                                 argmax, mask, part);
  } else {
    static bool attr = false;
    if (!attr) {
      SYSML_CUDA(cudaFuncSetAttribute(pool_bwd_wgrad_c1_kernel<3, 3>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
      attr = true;
    }
    pool_bwd_wgrad_c1_kernel<3, 3><<<used, FB_THREADS, smem, st>>>(a, x, cs, xcsr != nullptr, dpool,
                                                                argmax, mask, part);
  }
  SYSML_LAUNCH_CHECK();
  fused_b1_reduce_kernel<<<(unsigned)ceil_div((int64_t)c.K * (RS + 1), 256), 256, 0, st>>>(
      part, used, c.K, RS, df, db);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

}  // namespace sysml
