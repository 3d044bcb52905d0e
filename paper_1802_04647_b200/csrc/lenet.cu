// lenet.cu -- minibatch SGD-step driver (Listing 1; P:142 LeNet; P:187-192
// data-parallel plan) over the conv2d-family kernels, plus the step glue kernels:
// affine + softmax + cross-entropy, SGD and the NCCL
// gradient allreduce of the data-parallel plan.
//
// Step (SURVEY §8(c) def 8), local batch b, global batch Ng:
//   F1  conv1+bias+relu+pool    X[b x 784]      -> a1[b x 6272], i1
//   F2  conv2+bias+relu+pool    a1              -> a2[b x 3136], i2
//   F3  affine+softmax+CE       a2, W3, b3      -> ds[b x 10] = (p - onehot)/Ng, loss_n
//   B3  dW3 = ds^T a2 (split over samples, ordered sum); db3 = colsum ds; da2 = ds W3
//   B2p dz2 = maxpool_bwd(i2, da2, a2 > 0)
//   B2f dF2, db2 = bwd_filter(a1, dz2);  B2d da1 = bwd_data(F2, dz2)
//   B1p dz1 = maxpool_bwd(i1, da1, a1 > 0); B1f dF1, db1 = bwd_filter(X, dz1)
#include <dlfcn.h>

#include <algorithm>
#include <cmath>

#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

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
}  // namespace sysml

using namespace sysml;

namespace {

constexpr int OFF_F1 = 0, OFF_B1 = OFF_F1 + 32 * 25, OFF_F2 = OFF_B1 + 32,
              OFF_B2 = OFF_F2 + 64 * 800, OFF_W3 = OFF_B2 + 64, OFF_B3 = OFF_W3 + 10 * 3136,
              NUM_PARAMS = OFF_B3 + 10;
constexpr int D3 = 3136, NCLS = 10;

// F3, persistent: each CTA stages W3 (125 KB) in shared memory once (1-D bulk copies), then
// every warp takes samples two at a time -- lanes stride the 784 float4 columns, 8
// iterations of a2 loads in flight, W3 from smem serving both samples.  The 2 x 10 partial
// logits are summed over the warp by a halving reduce-scatter (masks 16, 8) and xor sums
// (4, 2, 1) -- a fixed order; one lane per sample does the softmax/CE.
// D = input features of the output affine layer: 3136 (LeNet-min), 512 (LeNet-512).
constexpr int F3_THREADS = 512, F3_WARPS = F3_THREADS / 32;
constexpr size_t f3_smem(int D) { return (size_t)NCLS * D * 4 + (size_t)F3_WARPS * 2 * NCLS * 4; }
template <int D3>
__global__ void __launch_bounds__(F3_THREADS) affine_softmax_ce_smem_kernel(
    int n, float inv_ng, const float *__restrict__ a2, const float *__restrict__ W3,
    const float *__restrict__ b3, const int32_t *__restrict__ labels, float *__restrict__ ds,
    float *__restrict__ loss_n) {
  extern __shared__ float4 f3s[];
  float4 *w3s = f3s;  // [NCLS][D3/4]
  float *lg = reinterpret_cast<float *>(f3s + NCLS * D3 / 4);
  __shared__ __align__(8) uint64_t w3bar;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    ptx::mbar_init(&w3bar, 1);
    ptx::fence_mbar_init();
    ptx::mbar_arrive_expect_tx(&w3bar, NCLS * D3 * 4);
#pragma unroll 1
    for (int j = 0; j < NCLS; ++j) ptx::bulk_g2s(w3s + j * (D3 / 4), W3 + j * D3, D3 * 4, &w3bar);
  }
  __syncthreads();
  float *mylg = lg + warp * 2 * NCLS;
  const int npair = (n + 1) >> 1;
  // pairs spread over the CTAs first (small batches use every SM), and the first batch of a2
  // loads is issued before waiting for this CTA's W3 copy (the copy's latency overlaps it)
  bool w3ready = false;
  for (int pr = warp * gridDim.x + blockIdx.x; pr < npair; pr += gridDim.x * F3_WARPS) {
    const int i0 = 2 * pr;
    const bool two = i0 + 1 < n;
    const float4 *r0 = reinterpret_cast<const float4 *>(a2 + (int64_t)i0 * D3);
    const float4 *r1 = two ? r0 + D3 / 4 : r0;
    float v[2 * NCLS];
#pragma unroll
    for (int i = 0; i < 2 * NCLS; ++i) v[i] = 0.f;
    // 8 iterations of loads in flight per batch (784 = 3 x 256 + 16 float4 columns)
#pragma unroll 1
    for (int base = 0; base < D3 / 4; base += 256) {
      float4 xa[8], xb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int d4 = base + u * 32 + lane;
        if (d4 < D3 / 4) {
          xa[u] = __ldcs(r0 + d4);
          xb[u] = __ldcs(r1 + d4);
        } else {
          xa[u] = xb[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      if (!w3ready) {
        ptx::mbar_wait(&w3bar, 0);
        w3ready = true;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int d4 = base + u * 32 + lane;
        if (base + u * 32 < D3 / 4) {
          const float4 x0 = xa[u], x1 = xb[u];
#pragma unroll
          for (int j = 0; j < NCLS; ++j) {
            const float4 w = w3s[j * (D3 / 4) + min(d4, D3 / 4 - 1)];
            v[j] = fmaf(x0.x, w.x, fmaf(x0.y, w.y, fmaf(x0.z, w.z, fmaf(x0.w, w.w, v[j]))));
            v[NCLS + j] =
                fmaf(x1.x, w.x, fmaf(x1.y, w.y, fmaf(x1.z, w.z, fmaf(x1.w, w.w, v[NCLS + j]))));
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < NCLS; ++i) {
      const bool hi = lane & 16;
      const float r = __shfl_xor_sync(0xffffffffu, hi ? v[i] : v[i + NCLS], 16);
      v[i] = (hi ? v[i + NCLS] : v[i]) + r;
    }
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const bool hi = lane & 8;
      const float r = __shfl_xor_sync(0xffffffffu, hi ? v[i] : v[i + 5], 8);
      v[i] = (hi ? v[i + 5] : v[i]) + r;
    }
#pragma unroll
    for (int m = 4; m > 0; m >>= 1)
#pragma unroll
      for (int i = 0; i < 5; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], m);
    if ((lane & 7) == 0) {
      const int base = ((lane & 16) ? NCLS : 0) + ((lane & 8) ? 5 : 0);
#pragma unroll
      for (int i = 0; i < 5; ++i) mylg[base + i] = v[i];
    }
    __syncwarp();
    if (lane < (two ? 2 : 1)) {
      const float *a = mylg + lane * NCLS;
      float z[NCLS];
      float m = -INFINITY;
#pragma unroll
      for (int j = 0; j < NCLS; ++j) {
        z[j] = a[j] + __ldg(b3 + j);
        m = fmaxf(m, z[j]);
      }
      float den = 0.f;
#pragma unroll
      for (int j = 0; j < NCLS; ++j) den += expf(z[j] - m);
      const int img = i0 + lane;
      const int y = labels[img];
      float lossv = 0.f;
#pragma unroll
      for (int j = 0; j < NCLS; ++j) {
        const float pj = expf(z[j] - m) / den;
        ds[img * NCLS + j] = (pj - (j == y ? 1.f : 0.f)) * inv_ng;
        if (j == y) lossv = -logf(fmaxf(pj, 1e-15f)) * inv_ng;
      }
      loss_n[img] = lossv;
    }
    __syncwarp();
  }
}

// Scoring (P:193-202 parfor-style row-partitioned scoring): warp per sample, logits =
// a2 . W3^T + b3 (lanes stride the 784 float4 columns, xor-tree reduction), then the
// max-shifted softmax probabilities and the first maximum as the predicted label.
template <int D3>
__global__ void lenet_predict_kernel(int n, const float *__restrict__ a2, const float *__restrict__ W3,
                                     const float *__restrict__ b3, int32_t *__restrict__ pred,
                                     float *__restrict__ probs) {
  const int sample = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (sample >= n) return;
  const float4 *row = reinterpret_cast<const float4 *>(a2 + (int64_t)sample * D3);
  float acc[NCLS];
#pragma unroll
  for (int j = 0; j < NCLS; ++j) acc[j] = 0.f;
  for (int d4 = lane; d4 < D3 / 4; d4 += 32) {
    const float4 v = __ldg(row + d4);
#pragma unroll
    for (int j = 0; j < NCLS; ++j) {
      const float4 w = __ldg(reinterpret_cast<const float4 *>(W3 + j * D3) + d4);
      acc[j] = fmaf(v.x, w.x, fmaf(v.y, w.y, fmaf(v.z, w.z, fmaf(v.w, w.w, acc[j]))));
    }
  }
#pragma unroll
  for (int j = 0; j < NCLS; ++j)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
  if (lane == 0) {
    float m = -INFINITY;
    int best = 0;
#pragma unroll
    for (int j = 0; j < NCLS; ++j) {
      acc[j] += __ldg(b3 + j);
      if (acc[j] > m) {  // strict: the first maximum wins
        m = acc[j];
        best = j;
      }
    }
    if (pred) pred[sample] = best;
    if (probs) {
      float den = 0.f;
#pragma unroll
      for (int j = 0; j < NCLS; ++j) den += expf(acc[j] - m);
#pragma unroll
      for (int j = 0; j < NCLS; ++j) probs[(int64_t)sample * NCLS + j] = expf(acc[j] - m) / den;
    }
  }
}

// ordered sum of v[0..n) into *out (single block, fixed tree)
__global__ void ordered_total_kernel(const float *__restrict__ v, int n, float *__restrict__ out) {
  __shared__ float red[1024];
  float s = 0.f;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int i0 = threadIdx.x * per, i1 = min(n, i0 + per);
  for (int i = i0; i < i1; ++i) s += v[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// B3 stage 1: partial dW3/db3 over a chunk of samples.  Block (196 threads) x = a quarter
// of the 784 float4 columns of a2 (thread owns 4 columns x 10 classes), y = sample chunk;
// 8 samples' float4 loads in flight per thread.  part[chunk][j][d] (j < 10), and
// part[chunk][10][j] = db3 partial (sum of ds over the chunk).
// Templated on the feature width D3 (3136: 4 blocks of 196 threads; 512: one of 128).
constexpr int dw3_threads(int D) { return D == 3136 ? 196 : D / 4; }
constexpr int dw3_len(int D) { return NCLS * D + NCLS; }              // W then b (grads layout)
constexpr int dw3_stride(int D) { return (dw3_len(D) + 3) / 4 * 4; }  // float4-aligned partials
constexpr int DW3_LEN = dw3_len(D3), DW3_STRIDE = dw3_stride(D3);
template <int D3, int DW3_T>
__global__ void __launch_bounds__(DW3_T) dw3_partial_kernel(int n, int n_per_chunk, const float *__restrict__ ds,
                                                            const float *__restrict__ a2,
                                                            float *__restrict__ part) {
  constexpr int DW3_STRIDE = dw3_stride(D3);
  const int d4 = blockIdx.x * DW3_T + threadIdx.x;  // < D3 / 4
  const int chunk = blockIdx.y;
  const int n0 = chunk * n_per_chunk, n1 = min(n, n0 + n_per_chunk);
  __shared__ float dss[64 * NCLS];
  float4 acc[NCLS];
#pragma unroll
  for (int j = 0; j < NCLS; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 *a24 = reinterpret_cast<const float4 *>(a2) + d4;
  for (int nb = n0; nb < n1; nb += 64) {
    const int cnt = min(64, n1 - nb);
    __syncthreads();
    for (int i = threadIdx.x; i < cnt * NCLS; i += DW3_T) dss[i] = ds[(int64_t)nb * NCLS + i];
    __syncthreads();
    for (int i0 = 0; i0 < cnt; i0 += 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        v[u] = i0 + u < cnt ? __ldg(a24 + (int64_t)(nb + i0 + u) * (D3 / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (i0 + u >= cnt) break;
#pragma unroll
        for (int j = 0; j < NCLS; ++j) {
          const float w = dss[(i0 + u) * NCLS + j];
          acc[j].x = fmaf(w, v[u].x, acc[j].x);
          acc[j].y = fmaf(w, v[u].y, acc[j].y);
          acc[j].z = fmaf(w, v[u].z, acc[j].z);
          acc[j].w = fmaf(w, v[u].w, acc[j].w);
        }
      }
    }
  }
  float *pc = part + (int64_t)chunk * DW3_STRIDE;
#pragma unroll
  for (int j = 0; j < NCLS; ++j) reinterpret_cast<float4 *>(pc + j * D3)[d4] = acc[j];
  if (blockIdx.x == 0 && threadIdx.x < NCLS) {
    float s = 0.f;
    for (int i = n0; i < n1; ++i) s += ds[(int64_t)i * NCLS + threadIdx.x];
    pc[NCLS * D3 + threadIdx.x] = s;
  }
}

// B3 stage 2: out[i] = sum over chunks (fixed order) of part[c][i].  Block (32 float4
// groups x 8 eighths of the chunks): thread (e, g) sums its eighth in chunk order, the
// eighths are added in order (deterministic); the len % 4 scalar tail by block 0.
__global__ void __launch_bounds__(256) dw3_reduce_kernel(const float *__restrict__ part, int chunks,
                                                         int64_t stride, int64_t len, float *__restrict__ out) {
  __shared__ float4 red[8][32];
  const int gl = threadIdx.x & 31, e = threadIdx.x >> 5;
  const int64_t g = blockIdx.x * 32 + gl, ng = len / 4;
  const int per = (chunks + 7) / 8, c0 = e * per, c1 = min(chunks, c0 + per);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (g < ng)
    for (int cb = c0; cb < c1; cb += 8) {  // 8 loads in flight, summed in chunk order
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        v[u] = cb + u < c1 ? __ldg(reinterpret_cast<const float4 *>(part + (int64_t)(cb + u) * stride) + g)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc.x += v[u].x;
        acc.y += v[u].y;
        acc.z += v[u].z;
        acc.w += v[u].w;
      }
    }
  red[e][gl] = acc;
  __syncthreads();
  if (e == 0 && g < ng) {
    float4 t = red[0][gl];
#pragma unroll
    for (int k = 1; k < 8; ++k) {
      t.x += red[k][gl].x;
      t.y += red[k][gl].y;
      t.z += red[k][gl].z;
      t.w += red[k][gl].w;
    }
    if (((uintptr_t)out & 15) == 0) {
      reinterpret_cast<float4 *>(out)[g] = t;
    } else {  // caller's gradient buffer not 16-byte aligned
      out[4 * g] = t.x;
      out[4 * g + 1] = t.y;
      out[4 * g + 2] = t.z;
      out[4 * g + 3] = t.w;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < len - 4 * ng) {
    const int64_t i = 4 * ng + threadIdx.x;
    float s = 0.f;
    for (int c = 0; c < chunks; ++c) s += part[(int64_t)c * stride + i];
    out[i] = s;
  }
}

__global__ void da2_kernel(int n, const float *__restrict__ ds, const float *__restrict__ W3,
                           float *__restrict__ da2) {
  const int64_t total = (int64_t)n * D3;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = i / D3;
    const int d = (int)(i - s * D3);
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < NCLS; ++j) acc = fmaf(__ldg(ds + s * NCLS + j), __ldg(W3 + j * D3 + d), acc);
    da2[i] = acc;
  }
}

// B3+B2p fused (SPF path): da2 = ds W3 evaluated per pooled output and routed straight
// through the 2x2 max-pool argmax (ReLU mask a2 > 0) into the unpooled gradient dz2 in
// SPF planes [64][plane] (output frame 16x16, position n*256 + h*16 + w): the da2 tensor
// is never materialised.  One thread per pooled output (n, k, pp, pc).
// B2p (TF32 path): da2 = ds W3 (P:58-84 affine backward) fused with the masked max-pool
// routing (reading R9) into the dz2 SPF planes.  Block = 256 feature indices d
// x a chunk of images: each thread keeps its W3 column (10 floats) in registers and walks
// the chunk's images (ds rows staged in shared memory), so W3 is read once per block.
constexpr int B2P_IMGS = 32;
__global__ void __launch_bounds__(256) affine_bwd_route_spf_kernel(
    int n, const float *__restrict__ ds, const float *__restrict__ W3,
    const uint64_t *__restrict__ c2, int64_t cplane, float *__restrict__ dz2s, int64_t plane,
    float *__restrict__ dbpart) {
  __shared__ float dss[B2P_IMGS * NCLS];
  const int d = blockIdx.x * 256 + threadIdx.x;  // = k*49 + pp*7 + pc
  const int s0 = blockIdx.y * B2P_IMGS, s1 = min(n, s0 + B2P_IMGS);
  for (int i = threadIdx.x; i < (s1 - s0) * NCLS; i += 256) dss[i] = __ldg(ds + (int64_t)s0 * NCLS + i);
  __syncthreads();
  if (d >= D3) return;
  float w[NCLS];
#pragma unroll
  for (int j = 0; j < NCLS; ++j) w[j] = __ldg(W3 + j * D3 + d);
  const int k = d / 49, r = d - k * 49, pp = r / 7, pc = r - pp * 7;
  const unsigned long long *cw = reinterpret_cast<const unsigned long long *>(c2) + (int64_t)(k >> 4) * cplane + r;
  const int sh = 4 * (k & 15);
  float *base = dz2s + (int64_t)k * plane + (2 * pp) * 16 + 2 * pc;
  float gsum = 0.f;  // db2 partial of this (k, window) over the chunk's images (image order)
  for (int sb = s0; sb < s1; sb += 4) {
    uint32_t cd[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)  // the batch's code loads in flight together
      cd[u] = sb + u < s1 ? (uint32_t)(__ldg(cw + (int64_t)(sb + u) * 49) >> sh) & 15u : 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int s = sb + u;
      if (s >= s1) break;
      // window code of the pool2 winner: positive*4 + dr*2 + ds (positive: a2 > 0, R9)
      float g = 0.f;
      if (cd[u] & 4u) {
        const float *dsr = dss + (s - s0) * NCLS;
#pragma unroll
        for (int j = 0; j < NCLS; ++j) g = fmaf(dsr[j], w[j], g);
      }
      gsum += g;
      const uint32_t wp = cd[u] & 3u;
      float *bs = base + (int64_t)s * 256;
      __stcs(reinterpret_cast<float2 *>(bs), make_float2(wp == 0 ? g : 0.f, wp == 1 ? g : 0.f));  // streaming
      __stcs(reinterpret_cast<float2 *>(bs + 16), make_float2(wp == 2 ? g : 0.f, wp == 3 ? g : 0.f));
      if (pc == 6) {  // the frame's zero columns 14-15 too: whole 32-byte sectors written
        __stcs(reinterpret_cast<float2 *>(bs + 2), make_float2(0.f, 0.f));
        __stcs(reinterpret_cast<float2 *>(bs + 18), make_float2(0.f, 0.f));
      }
    }
  }
  dbpart[(int64_t)blockIdx.y * D3 + d] = gsum;
}

// B2p, vertically fused form (NEXT-1): da2 = ds W3 (P:58-84 affine backward) in the
// window-major, channel-minor layout da2w[n][pp*7 + pc][64] that the conv2 backward producers
// route through the window codes themselves -- the unpooled dz2 is never written.  Values are
// masked by the relu bit of the window code (R9), so da2w holds exactly the gradient each
// window routes to its winner.  Block = 64 channels x 4 windows x a chunk of 32 images; each
// thread keeps its W3 column in registers.  dbpart[chunk][k*49 + window] = db2 partials.
__global__ void __launch_bounds__(256) affine_bwd_da2w_kernel(
    int n, const float *__restrict__ ds, const float *__restrict__ W3, const uint64_t *__restrict__ c2,
    int64_t cplane, float *__restrict__ da2w, float *__restrict__ dbpart) {
  __shared__ float dss[B2P_IMGS * NCLS];
  const int k = threadIdx.x & 63, win = blockIdx.x * 4 + (threadIdx.x >> 6);
  const int s0 = blockIdx.y * B2P_IMGS, s1 = min(n, s0 + B2P_IMGS);
  for (int i = threadIdx.x; i < (s1 - s0) * NCLS; i += 256) dss[i] = __ldg(ds + (int64_t)s0 * NCLS + i);
  __syncthreads();
  if (win >= 49) return;
  const int d = k * 49 + win;
  float w[NCLS];
#pragma unroll
  for (int j = 0; j < NCLS; ++j) w[j] = __ldg(W3 + j * D3 + d);
  const unsigned long long *cw = reinterpret_cast<const unsigned long long *>(c2) + (int64_t)(k >> 4) * cplane + win;
  const int sh = 4 * (k & 15);
  float gsum = 0.f;
  for (int s = s0; s < s1; ++s) {
    const uint32_t cd = (uint32_t)(__ldg(cw + (int64_t)s * 49) >> sh) & 15u;
    float g = 0.f;
    if (cd & 4u) {
      const float *dsr = dss + (s - s0) * NCLS;
#pragma unroll
      for (int j = 0; j < NCLS; ++j) g = fmaf(dsr[j], w[j], g);
    }
    gsum += g;
    __stcs(da2w + ((int64_t)s * 49 + win) * 64 + k, g);
  }
  dbpart[(int64_t)blockIdx.y * D3 + d] = gsum;
}

// db2[k] = fixed-order sum of the B2p partials: block k, thread t sums chunks t, t + 256, ...
// (each over the 49 windows in order), then a fixed shared-memory tree
__global__ void __launch_bounds__(256) db2_reduce_kernel(const float *__restrict__ dbpart, int chunks,
                                                         float *__restrict__ db) {
  __shared__ float red[256];
  const int k = blockIdx.x, t = threadIdx.x;
  float acc = 0.f;
  for (int c = t; c < chunks; c += 256) {
    const float *pr = dbpart + (int64_t)c * D3 + k * 49;
    float v = 0.f;
    for (int r = 0; r < 49; ++r) v += __ldg(pr + r);
    acc += v;
  }
  red[t] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (t < o) red[t] += red[t + o];
    __syncthreads();
  }
  if (t == 0) db[k] = red[0];
}

// The six optimizers (include/sysml.h): elementwise fp32, one thread per
// parameter; kind is a template argument so the loop carries no dispatch.  Adam's bias
// corrections arrive as reciprocals c1 = 1/(1 - b1^t), c2 = 1/(1 - b2^t) (host, in double).
template <int KIND>
__global__ void optimizer_kernel(float *__restrict__ p, const float *__restrict__ g, float *__restrict__ st,
                                 int64_t n, float lr, float mu, float rho, float eps, float b1, float b2,
                                 float c1, float c2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    if (KIND == SYSML_OPT_SGD) {
      p[i] = p[i] - lr * gi;
    } else if (KIND == SYSML_OPT_MOMENTUM) {
      const float v = mu * st[i] - lr * gi;
      st[i] = v;
      p[i] = p[i] + v;
    } else if (KIND == SYSML_OPT_NESTEROV) {
      const float v_prev = st[i];
      const float v = mu * v_prev - lr * gi;
      st[i] = v;
      p[i] = p[i] - mu * v_prev + (1.f + mu) * v;
    } else if (KIND == SYSML_OPT_ADAGRAD) {
      const float c = st[i] + gi * gi;
      st[i] = c;
      p[i] = p[i] - lr * gi / (sqrtf(c) + eps);
    } else if (KIND == SYSML_OPT_RMSPROP) {
      const float c = rho * st[i] + (1.f - rho) * gi * gi;
      st[i] = c;
      p[i] = p[i] - lr * gi / (sqrtf(c) + eps);
    } else {
      const float m = b1 * st[i] + (1.f - b1) * gi;
      const float v = b2 * st[n + i] + (1.f - b2) * gi * gi;
      st[i] = m;
      st[n + i] = v;
      p[i] = p[i] - lr * (m * c1) / (sqrtf(v * c2) + eps);
    }
  }
}

__global__ void sgd_kernel(float *__restrict__ p, const float *__restrict__ g, int64_t n,
                           float lr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = p[i] - lr * g[i];
}

// ---- NCCL (resolved at run time from the library the caller already loaded) ----
typedef int (*nccl_allreduce_fn)(const void *, void *, size_t, int, int, void *, cudaStream_t);
typedef const char *(*nccl_errstr_fn)(int);

struct NcclSyms {
  nccl_allreduce_fn allreduce = nullptr;
  nccl_errstr_fn errstr = nullptr;
};

NcclSyms &nccl_syms() {
  static NcclSyms s;
  static std::once_flag once;
  std::call_once(once, [] {
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    void *h = nullptr;
    for (const char *nm : names) {
      h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
      if (h) break;
    }
    if (!h) h = RTLD_DEFAULT;
    s.allreduce = (nccl_allreduce_fn)dlsym(h, "ncclAllReduce");
    s.errstr = (nccl_errstr_fn)dlsym(h, "ncclGetErrorString");
  });
  return s;
}

const char *STAGE_NAMES[] = {"F1_conv1_pool", "F2_conv2_pool", "F3_affine_softmax_ce",
                             "B3_affine_bwd", "B2p_maxpool_bwd2", "B2f_conv2_bwd_filter",
                             "B2d_conv2_bwd_data", "B1p_maxpool_bwd1", "B1f_conv1_bwd_filter",
                             "B1_fused_pool_bwd_conv1_wgrad", "F3h_affine_relu_dropout",
                             "B3h_affine_hidden_bwd"};
constexpr int NSTAGES = 12;

// LeNet-512 (NEXT-4; R22): F1, b1, F2, b2, W3[512x3136], b3[512], W4[10x512], b4[10]
constexpr int H5 = 512;
constexpr int OFF5_W3 = OFF_B2 + 64, OFF5_B3 = OFF5_W3 + H5 * D3, OFF5_W4 = OFF5_B3 + H5,
              OFF5_B4 = OFF5_W4 + NCLS * H5, NUM_PARAMS5 = OFF5_B4 + NCLS;

__global__ void counter_set_kernel(uint64_t *c, uint64_t v) { *c = v; }

}  // namespace

struct sysml_lenet {
  int max_b = 0, math = 0, csr = 0;
  int da1_nhwc = 0;  // SPF path: B2d writes da1 as [n][196][32] for the fused B1 (codes)
  // data-parallel gradient exchange overlapped with the tail of the backward pass: the
  // {F2, b2, W3, b3} bucket is all-reduced on ar_stream as soon as conv2 bwd_filter is done
  // (while conv2 bwd_data and the conv1 backward run), {F1, b1} after the conv1 backward
  void *ar_comm = nullptr;  // set by sysml_lenet_step for the duration of the call
  cudaStream_t ar_stream = nullptr;
  cudaEvent_t ev_b2 = nullptr, ev_b1 = nullptr, ev_ar = nullptr;
  int64_t max_nnz = 0;
  float *a1 = nullptr, *a2 = nullptr, *ds = nullptr, *lossn = nullptr, *da2 = nullptr,
        *dz2 = nullptr, *da1 = nullptr, *dz1 = nullptr, *part3 = nullptr;
  int32_t *i1 = nullptr, *i2 = nullptr;
  void *ws = nullptr;
  size_t ws_bytes = 0;
  // host-input path buffers
  float *x_dev = nullptr, *loss_dev = nullptr;
  int32_t *lab_dev = nullptr;
  // pipelined host input (sysml_lenet_step_host_pipelined): a second input buffer filled on
  // copy_stream while the current step computes; slot 0 = x_dev / lab_dev, slot 1 = below
  float *x_dev2 = nullptr;
  int32_t *lab_dev2 = nullptr;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_consumed[2] = {nullptr, nullptr};
  const void *pf_x = nullptr, *pf_lab = nullptr;  // host batch prefetched into slot pf_slot
  int pf_slot = -1, pf_n = 0;
  // timing
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool, pending[NSTAGES];
  double ms[NSTAGES] = {0};
  int64_t calls[NSTAGES] = {0};
  int launches = 0;
  int dw3_chunks = 1;
  bool fused_b1 = false;  // maxpool_bwd1 + conv1 bwd_filter in one kernel (fused_bwd.cu)
  // TF32 path: a1 and dz2 live in the stacked planar frame layout (SPF, 16x16 frames,
  // zero padding stored) so the tcgen05 producers stream aligned float4s
  bool spf = false;
  int64_t spf_plane = 0;
  float *a1s = nullptr, *dz2s = nullptr;
  // TF32 path: pool argmax as packed 2-bit window codes, one u32 per (16 channels, window)
  uint64_t *c1 = nullptr, *c2 = nullptr;  // [2][b*196], [4][b*49] (kernels.cuh TcSpfIO::code)
  float *db2part = nullptr;                // B2p's conv2 bias-gradient partials [chunks][3136]
  // NEXT-1 vertical fusion: the conv2 backward producers route the pooled gradient da2w
  // ([n][49 windows][64], relu-masked) through the window codes themselves
  int route = 0;                           // B2d routed (SYSML_ROUTE=1, opt-in)
  float *da2w = nullptr;
  // LeNet-512 (hidden = 512; 0 = LeNet-min): affine 3136->512 + relu + inverted dropout
  int hidden = 0;
  int64_t num_params = NUM_PARAMS;
  float keep_p = 1.f;
  uint64_t seed = 0, keep_T = 0;
  int64_t row0 = 0;                 // global index of local row 0 (the mask follows the global row)
  uint64_t *drop_step = nullptr;    // device step counter of the mask stream (R23)
  float *h3 = nullptr, *dz3 = nullptr, *dz3T = nullptr, *a2T = nullptr, *W3T = nullptr, *part4 = nullptr;
};

namespace {

sysml_conv_desc conv1_desc(int n, int math) {
  return sysml_conv_desc{n, 1, 28, 28, 32, 5, 5, 1, 1, 2, 2, math};
}
sysml_conv_desc conv2_desc(int n, int math) {
  return sysml_conv_desc{n, 32, 14, 14, 64, 5, 5, 1, 1, 2, 2, math};
}
sysml_pool_desc pool1_desc(int n) { return sysml_pool_desc{n, 32, 28, 28, 2, 2, 2, 2, 0, 0, 1}; }
sysml_pool_desc pool2_desc(int n) { return sysml_pool_desc{n, 64, 14, 14, 2, 2, 2, 2, 0, 0, 1}; }

// pool2 window-code plane stride (64-bit words per 16-channel group): even, so the routed
// producers' per-tile bulk copies of code words start 16-byte aligned
int64_t c2_plane_of(int64_t max_b) { return (max_b * 49 + 1) / 2 * 2; }

int dw3_chunks_for(int n) {
  // about 32 samples per chunk (16 measured slower at batch 1024: twice the partials to
  // reduce), at most one chunk per SM (x 4 column blocks)
  int64_t c = std::min<int64_t>(sm_count(), ceil_div(n, 32));
  return (int)(c < 1 ? 1 : c);
}

struct StageTimer {
  sysml_lenet *h;
  cudaStream_t st;
  int stage = -1;
  std::pair<cudaEvent_t, cudaEvent_t> ev{};
  StageTimer(sysml_lenet *h_, cudaStream_t st_) : h(h_), st(st_) {}
  sysml_status begin(int s) {
    stage = s;
    if (!h->timing) return SYSML_OK;
    if (h->pool.empty()) {
      cudaEvent_t a, b;
      SYSML_CUDA(cudaEventCreate(&a));
      SYSML_CUDA(cudaEventCreate(&b));
      h->pool.push_back({a, b});
    }
    ev = h->pool.back();
    h->pool.pop_back();
    SYSML_CUDA(cudaEventRecord(ev.first, st));
    return SYSML_OK;
  }
  sysml_status end() {
    if (!h->timing) return SYSML_OK;
    SYSML_CUDA(cudaEventRecord(ev.second, st));
    h->pending[stage].push_back(ev);
    return SYSML_OK;
  }
};

}  // namespace

extern "C" {

int64_t sysml_lenet_num_params(void) { return NUM_PARAMS; }

}  // extern "C"

static sysml_status lenet_create_impl(int32_t max_local_batch, int32_t math, int32_t input_is_csr,
                                      int64_t max_nnz, int hidden, float keep_p, uint64_t seed,
                                      sysml_lenet **out) {
  SYSML_CHECK_ARG(out != nullptr, "out is NULL");
  SYSML_CHECK_ARG(max_local_batch >= 1, "max_local_batch must be >= 1 (got %d)", max_local_batch);
  SYSML_CHECK_ARG(math == SYSML_MATH_FP32 || math == SYSML_MATH_TF32, "bad math %d", math);
  SYSML_CHECK_ARG(!input_is_csr || max_nnz >= 0, "max_nnz must be >= 0");
  sysml_lenet *h = new sysml_lenet();
  h->max_b = max_local_batch;
  if (cudaStreamCreateWithFlags(&h->ar_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_b2, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_b1, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_ar, cudaEventDisableTiming) != cudaSuccess) {
    set_error("creating the allreduce stream / events failed");
    delete h;
    return SYSML_ERR_CUDA;
  }
  h->math = math;
  h->csr = input_is_csr ? 1 : 0;
  h->hidden = hidden;
  h->num_params = hidden ? NUM_PARAMS5 : NUM_PARAMS;
  h->keep_p = keep_p;
  h->seed = seed;
  h->keep_T = (uint64_t)floor((double)keep_p * 4294967296.0);  // R23: kept iff (raw >> 32) < T
  h->max_nnz = max_nnz;
  const int64_t b = max_local_batch;
  h->dw3_chunks = dw3_chunks_for(max_local_batch);
  auto fail = [&](sysml_status s) {
    sysml_lenet_destroy(h);
    return s;
  };
#define ALLOC(ptr, count)                                                        \
  do {                                                                           \
    cudaError_t e_ = cudaMalloc((void **)&(ptr), sizeof(*(ptr)) * (size_t)(count)); \
    if (e_ != cudaSuccess) {                                                     \
      set_error("cudaMalloc(%s) failed: %s", #ptr, cudaGetErrorString(e_));      \
      return fail(SYSML_ERR_CUDA);                                               \
    }                                                                            \
  } while (0)
  ALLOC(h->a1, b * 6272);
  ALLOC(h->i1, b * 6272);
  ALLOC(h->a2, b * 3136);
  ALLOC(h->i2, b * 3136);
  ALLOC(h->ds, b * NCLS);
  ALLOC(h->lossn, b);
  ALLOC(h->da2, b * 3136);
  ALLOC(h->dz2, b * 12544);
  ALLOC(h->da1, b * 6272);
  ALLOC(h->dz1, b * 25088);
  ALLOC(h->part3, (int64_t)h->dw3_chunks * DW3_STRIDE);
  ALLOC(h->loss_dev, 1);
  ALLOC(h->lab_dev, b);
  if (!h->csr) ALLOC(h->x_dev, b * 784);
  if (!h->csr) {
    ALLOC(h->x_dev2, b * 784);
    ALLOC(h->lab_dev2, b);
    if (cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_copied[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_copied[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_consumed[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_consumed[1], cudaEventDisableTiming) != cudaSuccess) {
      set_error("creating the input copy stream / events failed");
      return fail(SYSML_ERR_CUDA);
    }
  }
  const int64_t ldt_max = (b + 3) / 4 * 4;
  if (hidden) {
    ALLOC(h->h3, b * H5);
    ALLOC(h->dz3, b * H5);
    ALLOC(h->dz3T, (int64_t)H5 * ldt_max);
    ALLOC(h->a2T, (int64_t)D3 * ldt_max);
    ALLOC(h->W3T, (int64_t)D3 * H5);
    ALLOC(h->part4, (int64_t)h->dw3_chunks * dw3_stride(H5));
    ALLOC(h->drop_step, 1);
    if (cudaMemset(h->drop_step, 0, sizeof(uint64_t)) != cudaSuccess) {
      set_error("cudaMemset of the dropout step counter failed");
      return fail(SYSML_ERR_CUDA);
    }
  }
  // workspace: max over the conv calls of the step
  size_t need = 0, w = 0;
  if (hidden) {
    sysml_status s5;
    if (math == SYSML_MATH_TF32) {
      const ConvArgs wa{1, D3, 1, (int)ldt_max, H5, 1, 1, 1, 1, 0, 0, 1, (int)ldt_max};
      need = std::max(need, tc_wgrad_1x1_ws(wa));
    } else {
      const sysml_conv_desc hd{(int32_t)b, D3, 1, 1, H5, 1, 1, 1, 1, 0, 0, math};
      if ((s5 = conv_fwd_ws(hd, nullptr, 0, &w)) != SYSML_OK) return fail(s5);
      need = std::max(need, w);
      if ((s5 = conv_bwd_filter_ws(hd, 0, &w)) != SYSML_OK) return fail(s5);
      need = std::max(need, w);
      if ((s5 = conv_bwd_data_ws(hd, &w)) != SYSML_OK) return fail(s5);
      need = std::max(need, w);
    }
  }
  const sysml_conv_desc c1 = conv1_desc(max_local_batch, math), c2 = conv2_desc(max_local_batch, math);
  const sysml_pool_desc p1 = pool1_desc(max_local_batch), p2 = pool2_desc(max_local_batch);
  sysml_status s;
  if ((s = conv_fwd_ws(c1, &p1, h->csr, &w)) != SYSML_OK) return fail(s);
  need = std::max(need, w);
  if ((s = conv_fwd_ws(c2, &p2, 0, &w)) != SYSML_OK) return fail(s);
  need = std::max(need, w);
  if ((s = conv_bwd_filter_ws(c2, 0, &w)) != SYSML_OK) return fail(s);
  need = std::max(need, w);
  if ((s = conv_bwd_data_ws(c2, &w)) != SYSML_OK) return fail(s);
  need = std::max(need, w);
  if ((s = conv_bwd_filter_ws(c1, h->csr, &w)) != SYSML_OK) return fail(s);
  need = std::max(need, w);
  {
    ConvGeom g1, gp1;
    if ((s = validate_conv(&c1, &g1)) != SYSML_OK) return fail(s);
    if ((s = validate_pool(&p1, &gp1)) != SYSML_OK) return fail(s);
    h->fused_b1 = fused_pool_bwd_wgrad_supported(conv_args(g1), pool_args(gp1, 1));
    if (h->fused_b1) need = std::max(need, fused_pool_bwd_wgrad_ws(conv_args(g1)));
  }
  if (math == SYSML_MATH_TF32 && h->fused_b1) {
    ConvGeom g1, g2, gp1, gp2;
    validate_conv(&c1, &g1); validate_conv(&c2, &g2);
    validate_pool(&p1, &gp1); validate_pool(&p2, &gp2);
    const ConvArgs a1a = conv_args(g1), a2a = conv_args(g2);
    const PoolArgs pa1 = pool_args(gp1, 1), pa2 = pool_args(gp2, 1);
    SpfConv sc{64, 32, 5, 5, 16, (int64_t)max_local_batch * 256, (int64_t)max_local_batch * 256,
               (int64_t)max_local_batch * 256, 0, 0};
    h->spf = tc_fwd_supported(a1a, &pa1) && tc_fwd_supported(a2a, &pa2) &&
             tc_bwd_data_supported(a2a) && tc_wgrad_spf_supported(sc);
    if (h->spf) {
      h->spf_plane = (int64_t)max_local_batch * 256;
      static const int nhwc_env = getenv("SYSML_DA1_NHWC") ? atoi(getenv("SYSML_DA1_NHWC")) : 1;
      h->da1_nhwc = nhwc_env && tc_conv_bwd_data_spf_nhwc_ok(a2a) ? 1 : 0;
      need = std::max(need, tc_fwd_ws(a1a));
      need = std::max(need, conv1_pool_ws(a1a, &pa1));
      need = std::max(need, tc_fwd_ws(a2a));
      need = std::max(need, tc_bwd_data_ws(a2a));
      need = std::max(need, sn_tmem_ws(a2a, 16, 256));
      need = std::max(need, snt_fwd_pool_ws(a2a));
      need = std::max(need, tc_wgrad_spf_ws(sc));
      if (tc_wgrad_spf_tma_supported(sc)) need = std::max(need, tc_wgrad_spf_tma_ws(sc));
      ALLOC(h->a1s, 32 * h->spf_plane);
      if (cudaMalloc(&h->db2part, sizeof(float) * D3 * (size_t)ceil_div(max_local_batch, B2P_IMGS)) !=
              cudaSuccess ||
          cudaMalloc(&h->c1, sizeof(uint64_t) * 2 * (size_t)max_local_batch * 196) != cudaSuccess ||
          cudaMalloc(&h->c2, sizeof(uint64_t) * (4 * (size_t)c2_plane_of(max_local_batch) + 2)) != cudaSuccess) {
        set_error("cudaMalloc failed for the window-code buffers");
        return fail(SYSML_ERR_CUDA);
      }
      ALLOC(h->dz2s, 64 * h->spf_plane);
      // opt-in (SYSML_ROUTE=1): measured slower (r02, batch 8192): B2d 1.01M -> 1.14M cycles per
      // CTA with register-pipelined global loads, 1.36M with per-tile smem staging (2 pipeline
      // stages left); its MMA loop is shared-memory-operand bound, so expanding the pooled
      // gradient in the producer costs more than writing dz2 once (DESIGN.md §7 NEXT-1)
      static const int route_env = getenv("SYSML_ROUTE") ? atoi(getenv("SYSML_ROUTE")) : 0;
      h->route = route_env ? 1 : 0;
      if (h->route) ALLOC(h->da2w, b * D3 + 64);  // + one window: the routed staging reads even counts
      if (cudaMemset(h->a1s, 0, sizeof(float) * 32 * h->spf_plane) != cudaSuccess ||
          cudaMemset(h->dz2s, 0, sizeof(float) * 64 * h->spf_plane) != cudaSuccess) {
        set_error("cudaMemset of the SPF activation buffers failed");
        return fail(SYSML_ERR_CUDA);
      }
    }
  }
  h->ws_bytes = need;
  if (need) {
    cudaError_t e = cudaMalloc(&h->ws, need);
    if (e != cudaSuccess) {
      set_error("cudaMalloc(workspace %zu) failed: %s", need, cudaGetErrorString(e));
      return fail(SYSML_ERR_CUDA);
    }
  }
#undef ALLOC
  *out = h;
  return SYSML_OK;
}

extern "C" {

sysml_status sysml_lenet_create(int32_t max_local_batch, int32_t math, int32_t input_is_csr,
                                int64_t max_nnz, sysml_lenet **out) {
  return lenet_create_impl(max_local_batch, math, input_is_csr, max_nnz, 0, 1.f, 0, out);
}

int64_t sysml_lenet512_num_params(void) { return NUM_PARAMS5; }

sysml_status sysml_lenet512_create(int32_t max_local_batch, int32_t math, int32_t input_is_csr,
                                   int64_t max_nnz, float keep_p, uint64_t seed, sysml_lenet **out) {
  SYSML_CHECK_ARG(keep_p > 0.f && keep_p <= 1.f, "keep_p %g must be in (0, 1]", (double)keep_p);
  return lenet_create_impl(max_local_batch, math, input_is_csr, max_nnz, H5, keep_p, seed, out);
}

sysml_status sysml_lenet_set_dropout(sysml_lenet *h, int64_t row0, int64_t step, sysml_stream_t stream) {
  SYSML_CHECK_ARG(h, "NULL handle");
  SYSML_CHECK_ARG(h->hidden, "sysml_lenet_set_dropout: the handle has no dropout layer (LeNet-min)");
  SYSML_CHECK_ARG(row0 >= 0 && step >= 0, "row0 / step must be >= 0");
  h->row0 = row0;
  counter_set_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(h->drop_step, (uint64_t)step);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status sysml_lenet_get_dropout_step(sysml_lenet *h, int64_t *step) {
  SYSML_CHECK_ARG(h && step, "NULL argument");
  SYSML_CHECK_ARG(h->hidden, "the handle has no dropout layer (LeNet-min)");
  uint64_t v = 0;
  SYSML_CUDA(cudaMemcpy(&v, h->drop_step, sizeof(v), cudaMemcpyDeviceToHost));
  *step = (int64_t)v;
  return SYSML_OK;
}

int64_t sysml_lenet_handle_num_params(const sysml_lenet *h) { return h ? h->num_params : -1; }

sysml_status sysml_lenet_destroy(sysml_lenet *h) {
  if (!h) return SYSML_OK;
  if (h->ar_stream) cudaStreamDestroy(h->ar_stream);
  if (h->ev_b2) cudaEventDestroy(h->ev_b2);
  if (h->ev_b1) cudaEventDestroy(h->ev_b1);
  if (h->ev_ar) cudaEventDestroy(h->ev_ar);
  cudaFree(h->a1); cudaFree(h->i1); cudaFree(h->a2); cudaFree(h->i2); cudaFree(h->ds);
  cudaFree(h->c1); cudaFree(h->c2); cudaFree(h->db2part);
  cudaFree(h->lossn); cudaFree(h->da2); cudaFree(h->dz2); cudaFree(h->da1); cudaFree(h->dz1);
  cudaFree(h->part3); cudaFree(h->loss_dev); cudaFree(h->lab_dev); cudaFree(h->x_dev);
  cudaFree(h->x_dev2); cudaFree(h->lab_dev2);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  for (int i = 0; i < 2; ++i) {
    if (h->ev_copied[i]) cudaEventDestroy(h->ev_copied[i]);
    if (h->ev_consumed[i]) cudaEventDestroy(h->ev_consumed[i]);
  }
  cudaFree(h->ws);
  cudaFree(h->a1s); cudaFree(h->dz2s);
  cudaFree(h->h3); cudaFree(h->dz3); cudaFree(h->dz3T); cudaFree(h->a2T); cudaFree(h->W3T);
  cudaFree(h->part4); cudaFree(h->drop_step); cudaFree(h->da2w);
  for (auto &e : h->pool) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  for (int i = 0; i < NSTAGES; ++i)
    for (auto &e : h->pending[i]) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  delete h;
  return SYSML_OK;
}

// all-reduce (sum) of grads[0, count) on the handle's allreduce stream once the main stream
// reaches this point (event `ev`); no-op unless a communicator is set for this step
static sysml_status ar_bucket(sysml_lenet *h, float *g, size_t count, cudaEvent_t ev, cudaStream_t st) {
  if (!h->ar_comm) return SYSML_OK;
  NcclSyms &s = nccl_syms();
  if (!s.allreduce) {
    set_error("ncclAllReduce could not be resolved (libnccl.so.2 not loaded in this process)");
    return SYSML_ERR_NCCL;
  }
  SYSML_CUDA(cudaEventRecord(ev, st));
  SYSML_CUDA(cudaStreamWaitEvent(h->ar_stream, ev, 0));
  const int r = s.allreduce(g, g, count, /*ncclFloat32*/ 7, /*ncclSum*/ 0, h->ar_comm, h->ar_stream);
  if (r != 0) {
    set_error("ncclAllReduce failed: %s", s.errstr ? s.errstr(r) : "?");
    return SYSML_ERR_NCCL;
  }
  return SYSML_OK;
}

// the forward (+ backward) of the local shard; predict mode (pred or probs non-NULL) stops
// after conv2 + pool and scores instead
static sysml_status lenet_run(sysml_lenet *h, const float *params, const sysml_input *x,
                              const int32_t *labels, int32_t n_local, int64_t n_global,
                              float *grads, float *loss_sum, sysml_stream_t stream, int32_t *pred,
                              float *probs) {
  SYSML_CHECK_ARG(h && params && x && ((labels && grads) || pred || probs), "NULL argument to sysml_lenet_fwd_bwd / predict");
  route_reset();  // sysml_last_route then lists this call's kernels
  SYSML_CHECK_ARG(n_local >= 1 && n_local <= h->max_b,
                  "n_local %d out of range [1, max_local_batch=%d]", n_local, h->max_b);
  SYSML_CHECK_ARG(n_global >= n_local, "n_global %lld < n_local %d", (long long)n_global, n_local);
  SYSML_CHECK_ARG((x->is_csr != 0) == (h->csr != 0),
                  "input is_csr=%d but the handle was created with input_is_csr=%d", x->is_csr,
                  h->csr);
  SYSML_CHECK_ALIGN16(params, "params");
  SYSML_CHECK_ALIGN16(grads, "grads");
  SYSML_CHECK_ALIGN(labels, 4, "labels");
  SYSML_CHECK_ALIGN(loss_sum, 4, "loss_sum");
  SYSML_CHECK_ALIGN(pred, 4, "pred");
  SYSML_CHECK_ALIGN16(probs, "probs");
  if (!x->is_csr) SYSML_CHECK_ALIGN16(x->dense, "dense input");
  if (x->is_csr) {
    SYSML_CHECK_ALIGN(x->csr.row_ptr, 4, "CSR row_ptr");
    SYSML_CHECK_ALIGN(x->csr.col_idx, 4, "CSR col_idx");
    SYSML_CHECK_ALIGN(x->csr.val, 4, "CSR val");
    SYSML_CHECK_SHAPE(x->csr.rows == n_local && x->csr.cols == 784,
                      "CSR input %lldx%lld must be n_local x 784 = %dx784",
                      (long long)x->csr.rows, (long long)x->csr.cols, n_local);
    SYSML_CHECK_SHAPE(x->csr.nnz <= h->max_nnz, "CSR nnz %lld exceeds max_nnz %lld",
                      (long long)x->csr.nnz, (long long)h->max_nnz);
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int n = n_local;
  const float inv_ng = (float)(1.0 / (double)n_global);
  const sysml_conv_desc c1 = conv1_desc(n, h->math), c2 = conv2_desc(n, h->math);
  const sysml_pool_desc p1 = pool1_desc(n), p2 = pool2_desc(n);
  StageTimer T(h, st);
  int launches0 = 0;

  ConvGeom g1, g2, gp1, gp2;
  SYSML_TRY(validate_conv(&c1, &g1));
  SYSML_TRY(validate_conv(&c2, &g2));
  SYSML_TRY(validate_pool(&p1, &gp1));
  SYSML_TRY(validate_pool(&p2, &gp2));
  const ConvArgs ca1 = conv_args(g1), ca2 = conv_args(g2);
  const PoolArgs pa1 = pool_args(gp1, 1), pa2 = pool_args(gp2, 1);
  // SPF geometry of conv2's 14x14 planes: 16x16 frames (pad 2 stored as zeros)
  TcSpfIO a1_io;  // a1 written / read in conv2's input-frame convention
  a1_io.out_plane = h->spf_plane;
  a1_io.out_Wf = 16;
  a1_io.out_Lf = 256;
  a1_io.out_off = 2;
  a1_io.code = h->c1;
  a1_io.code_plane = (int64_t)h->max_b * 196;
  sysml_input a1in{0, h->a1, {}};
  // F1
  SYSML_TRY(T.begin(0));
  if (h->spf && conv1_pool_supported(ca1, &pa1)) {
    // dense or CSR: pooling window in the MMA N dimension, lane-local pool epilogue
    SYSML_TRY(conv1_pool(ca1, &pa1, x->is_csr ? nullptr : x->dense, params + OFF_F1, params + OFF_B1,
                         h->a1s, nullptr, h->ws, st, &a1_io, x->is_csr ? &x->csr : nullptr));
  } else if (h->spf) {
    // dense or CSR (scattered straight into the KS operand): pooled a1 lands in SPF
    SYSML_TRY(tc_conv_fwd_spf(ca1, a1_io, x->is_csr ? nullptr : x->dense, params + OFF_F1,
                              params + OFF_B1, nullptr, &pa1, h->a1s, nullptr, h->ws, st,
                              x->is_csr ? &x->csr : nullptr));
  } else {
    SYSML_TRY(conv_fwd_dispatch(c1, *x, params + OFF_F1, params + OFF_B1, nullptr, &p1, h->a1, h->i1,
                                h->ws, h->ws_bytes, st));
    if (h->spf)
      SYSML_TRY(launch_nchw_to_spf(n, 32, 14, 14, h->a1, h->a1s, h->spf_plane, 16, 256, 2, st));
  }
  SYSML_TRY(T.end());
  // F2
  SYSML_TRY(T.begin(1));
  if (h->spf) {
    TcSpfIO io;
    io.in_plane = h->spf_plane;
    io.in_shift = 0;
    io.code = h->c2;
    io.code_plane = c2_plane_of(h->max_b);
    static const int snt_env = getenv("SYSML_F2_SNT") ? atoi(getenv("SYSML_F2_SNT")) : 1;
    if (snt_env && snt_fwd_pool_supported(ca2, &pa2, 16, 256))
      SYSML_TRY(snt_fwd_pool_spf(ca2, io, h->a1s, params + OFF_F2, params + OFF_B2, h->a2, h->ws, st));
    else
      SYSML_TRY(tc_conv_fwd_spf(ca2, io, h->a1s, params + OFF_F2, params + OFF_B2, nullptr, &pa2, h->a2,
                                nullptr, h->ws, st));
  } else {
    SYSML_TRY(conv_fwd_dispatch(c2, a1in, params + OFF_F2, params + OFF_B2, nullptr, &p2, h->a2,
                                h->i2, h->ws, h->ws_bytes, st));
  }
  SYSML_TRY(T.end());
  const bool hid = h->hidden != 0;
  const int OW = hid ? OFF5_W4 : OFF_W3, OB = hid ? OFF5_B4 : OFF_B3;  // output affine layer
  const float *feat = hid ? h->h3 : h->a2;                            // its input features
  const int64_t ldt = ((int64_t)n + 3) / 4 * 4;                       // batch-contiguous row stride
  const sysml_conv_desc hd{n, D3, 1, 1, H5, 1, 1, 1, 1, 0, 0, h->math};  // affine as a 1x1 conv (FP32)
  if (hid) {
    // F3h: h = dropout(relu(a2 W3^T + b3)) (train) / relu(a2 W3^T + b3) (scoring)
    const bool train = !(pred || probs);
    SYSML_TRY(T.begin(10));
    if (h->math == SYSML_MATH_TF32) {
      GemmEpi e;
      e.bias = params + OFF5_B3;
      e.relu = 1;
      e.dropout = train && h->keep_p < 1.f;
      e.keep_T = h->keep_T;
      e.keep_p = h->keep_p;
      e.seed = h->seed;
      e.step = h->drop_step;
      e.row0 = h->row0;
      e.units = H5;
      SYSML_TRY(tc_gemm(n, H5, D3, h->a2, D3, params + OFF5_W3, D3, h->h3, H5, e, st));
    } else {
      sysml_input ain{0, h->a2, {}};
      SYSML_TRY(conv_fwd_dispatch(hd, ain, params + OFF5_W3, params + OFF5_B3, h->h3, nullptr, nullptr,
                                  nullptr, h->ws, h->ws_bytes, st));
      SYSML_TRY(launch_relu_dropout(h->h3, n, H5, h->row0, h->seed, h->drop_step, h->keep_T, h->keep_p,
                                    train && h->keep_p < 1.f, st));
    }
    SYSML_TRY(T.end());
  }
  if (pred || probs) {  // scoring: logits, softmax, argmax
    if (hid)
      lenet_predict_kernel<H5><<<(unsigned)ceil_div((int64_t)n * 32, 256), 256, 0, st>>>(
          n, feat, params + OW, params + OB, pred, probs);
    else
      lenet_predict_kernel<D3><<<(unsigned)ceil_div((int64_t)n * 32, 256), 256, 0, st>>>(
          n, feat, params + OW, params + OB, pred, probs);
    SYSML_LAUNCH_CHECK();
    return SYSML_OK;
  }
  // F3
  SYSML_TRY(T.begin(2));
  {
    const int ctas = (int)std::min<int64_t>(sm_count(), (n + 1) / 2);
    if (hid) {
      SYSML_TRY(smem_attr(affine_softmax_ce_smem_kernel<H5>, f3_smem(H5)));
      affine_softmax_ce_smem_kernel<H5><<<(unsigned)ctas, F3_THREADS, f3_smem(H5), st>>>(
          n, inv_ng, feat, params + OW, params + OB, labels, h->ds, h->lossn);
    } else {
      SYSML_TRY(smem_attr(affine_softmax_ce_smem_kernel<D3>, f3_smem(D3)));
      affine_softmax_ce_smem_kernel<D3><<<(unsigned)ctas, F3_THREADS, f3_smem(D3), st>>>(
          n, inv_ng, feat, params + OW, params + OB, labels, h->ds, h->lossn);
    }
  }
  SYSML_LAUNCH_CHECK();
  if (loss_sum) {
    ordered_total_kernel<<<1, 1024, 0, st>>>(h->lossn, n, loss_sum);
    SYSML_LAUNCH_CHECK();
  }
  SYSML_TRY(T.end());
  // B3
  SYSML_TRY(T.begin(3));
  {
    const int chunks = std::min(h->dw3_chunks, dw3_chunks_for(n));
    const int npc = (int)ceil_div(n, chunks);
    const int used = (int)ceil_div(n, npc);
    if (hid) {  // dW4, db4
      constexpr int T5 = dw3_threads(H5);
      dw3_partial_kernel<H5, T5><<<dim3(H5 / 4 / T5, used), T5, 0, st>>>(n, npc, h->ds, feat, h->part4);
      SYSML_LAUNCH_CHECK();
      dw3_reduce_kernel<<<(unsigned)ceil_div(dw3_len(H5) / 4, 32), 256, 0, st>>>(
          h->part4, used, dw3_stride(H5), dw3_len(H5), grads + OFF5_W4);
      SYSML_LAUNCH_CHECK();
    } else {
      constexpr int T3 = dw3_threads(D3);
      dw3_partial_kernel<D3, T3><<<dim3(D3 / 4 / T3, used), T3, 0, st>>>(n, npc, h->ds, h->a2, h->part3);
      SYSML_LAUNCH_CHECK();
      // grads W3 and b3 are contiguous: [W3 (10*3136)][b3 (10)] == part layout
      dw3_reduce_kernel<<<(unsigned)ceil_div(DW3_LEN / 4, 32), 256, 0, st>>>(h->part3, used, DW3_STRIDE,
                                                                            DW3_LEN, grads + OFF_W3);
      SYSML_LAUNCH_CHECK();
      if (!h->spf) {
        da2_kernel<<<(unsigned)std::min<int64_t>(ceil_div((int64_t)n * D3, 256), 16 * sm_count()), 256,
                     0, st>>>(n, h->ds, params + OFF_W3, h->da2);
        SYSML_LAUNCH_CHECK();
      }
    }
  }
  SYSML_TRY(T.end());
  if (hid) {
    // B3h: dz3 = (ds W4) [h > 0] / keep_p; dW3 = dz3^T a2, db3 = colsum dz3; da2 = dz3 W3
    SYSML_TRY(T.begin(11));
    SYSML_TRY(launch_dz3(n, H5, h->ds, params + OFF5_W4, h->h3, h->keep_p, h->dz3, h->dz3T, ldt, st));
    if (h->math == SYSML_MATH_TF32) {
      // contraction over the batch: both operands batch-contiguous (K-major) for the TMA GEMM
      SYSML_TRY(launch_transpose(h->a2, n, D3, D3, h->a2T, ldt, st));
      const ConvArgs wa{1, D3, 1, (int)ldt, H5, 1, 1, 1, 1, 0, 0, 1, (int)ldt};
      SYSML_TRY(tc_wgrad_1x1(wa, h->a2T, h->dz3T, grads + OFF5_W3, grads + OFF5_B3, h->ws, st));
      SYSML_TRY(launch_transpose(params + OFF5_W3, H5, D3, D3, h->W3T, H5, st));
      SYSML_TRY(tc_gemm(n, D3, H5, h->dz3, H5, h->W3T, H5, h->da2, D3, GemmEpi{}, st));
    } else {
      sysml_input ain{0, h->a2, {}};
      SYSML_TRY(conv_bwd_filter_dispatch(hd, ain, h->dz3, grads + OFF5_W3, grads + OFF5_B3, h->ws,
                                         h->ws_bytes, st));
      SYSML_TRY(conv_bwd_data_dispatch(hd, params + OFF5_W3, h->dz3, h->da2, h->ws, h->ws_bytes, st));
    }
    SYSML_TRY(T.end());
  }
  if (h->spf) {
    // B2p: unpooled gradient straight into the SPF planes (output-frame convention)
    SYSML_TRY(T.begin(4));
    if (hid) {
      static_assert(B2P_IMGS == 32, "route_da2_spf_kernel chunks db2 partials by 32 images");
      SYSML_TRY(launch_route_da2_spf(n, h->da2, h->c2, c2_plane_of(h->max_b), h->dz2s, h->spf_plane,
                                     h->db2part, st));
    } else {
      if (h->route) {
        affine_bwd_da2w_kernel<<<dim3(13, (unsigned)ceil_div(n, B2P_IMGS)), 256, 0, st>>>(
            n, h->ds, params + OFF_W3, h->c2, c2_plane_of(h->max_b), h->da2w, h->db2part);
        SYSML_LAUNCH_CHECK();
      }
      affine_bwd_route_spf_kernel<<<dim3((unsigned)ceil_div(D3, 256), (unsigned)ceil_div(n, B2P_IMGS)),
                                    256, 0, st>>>(n, h->ds, params + OFF_W3, h->c2,
                                                  c2_plane_of(h->max_b), h->dz2s, h->spf_plane,
                                                  h->db2part);
      SYSML_LAUNCH_CHECK();
    }
    SYSML_TRY(T.end());
    // B2f
    SYSML_TRY(T.begin(5));
    SpfConv sc{64, 32, 5, 5, 16, (int64_t)n * 256, h->spf_plane, h->spf_plane, 0, 0};
    if (tc_wgrad_spf_tma_supported(sc))
    {
      // db2 came out of B2p; the bwd_filter kernel computes dF2 only
      SYSML_TRY(tc_wgrad_spf_tma(sc, h->a1s, h->dz2s, grads + OFF_F2, nullptr, h->ws, st));
      db2_reduce_kernel<<<64, 256, 0, st>>>(h->db2part, (int)ceil_div(n, B2P_IMGS), grads + OFF_B2);
      SYSML_LAUNCH_CHECK();
    } else
      SYSML_TRY(tc_wgrad_spf(sc, h->a1s, h->dz2s, grads + OFF_F2, grads + OFF_B2, h->ws, st));
    SYSML_TRY(T.end());
    SYSML_TRY(ar_bucket(h, grads + OFF_F2, h->num_params - OFF_F2, h->ev_b2, st));
    // B2d: input frame (pad 2) position = stored output-frame position + 34
    SYSML_TRY(T.begin(6));
    TcSpfIO io;
    io.in_plane = h->spf_plane;
    io.in_shift = -(2 * 16 + 2);
    io.out_nhwc = h->da1_nhwc;  // da1 channel-minor: whole-vector stores, read only by B1
    if (h->route && !hid) {  // NEXT-1: the producer routes da2w through the pool2 codes
      io.route_val = h->da2w;
      io.route_code = h->c2;
      io.route_cplane = c2_plane_of(h->max_b);
      io.route_C = 64;
      io.route_Pp = 7;
      io.route_Qp = 7;
      io.route_Wf = 16;
      io.route_Lf = 256;
    }
    static const int sn_tmem_env = getenv("SYSML_SN_TMEM") ? atoi(getenv("SYSML_SN_TMEM")) : 1;
    if (sn_tmem_env && !io.route_val && sn_tmem_supported(ca2, 16, 256))
      SYSML_TRY(sn_tmem_bwd_data_spf(ca2, io, 16, 256, params + OFF_F2, h->dz2s, h->da1, h->ws, st));
    else
      SYSML_TRY(tc_conv_bwd_data_spf(ca2, io, params + OFF_F2, h->dz2s, h->da1, h->ws, st));
    SYSML_TRY(T.end());
  } else {
    // B2p
    SYSML_TRY(T.begin(4));
    SYSML_TRY(launch_maxpool_bwd(pa2, h->i2, h->da2, h->a2, h->dz2, st));
    SYSML_TRY(T.end());
    // B2f
    SYSML_TRY(T.begin(5));
    SYSML_TRY(conv_bwd_filter_dispatch(c2, a1in, h->dz2, grads + OFF_F2, grads + OFF_B2, h->ws,
                                       h->ws_bytes, st));
    SYSML_TRY(T.end());
    SYSML_TRY(ar_bucket(h, grads + OFF_F2, h->num_params - OFF_F2, h->ev_b2, st));
    // B2d
    SYSML_TRY(T.begin(6));
    SYSML_TRY(conv_bwd_data_dispatch(c2, params + OFF_F2, h->dz2, h->da1, h->ws, h->ws_bytes, st));
    SYSML_TRY(T.end());
  }
  if (h->fused_b1) {
    // B1 fused: conv1 bwd_filter of maxpool_bwd(i1, da1, a1 > 0) without materialising dz1
    SYSML_TRY(T.begin(9));
    SYSML_TRY(fused_pool_bwd_wgrad(ca1, pa1, x->is_csr ? nullptr : x->dense,
                                   x->is_csr ? &x->csr : nullptr, h->da1, h->i1,
                                   h->spf ? h->a1s : h->a1, grads + OFF_F1, grads + OFF_B1, h->ws,
                                   st, h->spf ? &a1_io : nullptr, h->spf ? h->da1_nhwc : 0));
    SYSML_TRY(T.end());
  } else {
    // B1p
    SYSML_TRY(T.begin(7));
    SYSML_TRY(launch_maxpool_bwd(pa1, h->i1, h->da1, h->a1, h->dz1, st));
    SYSML_TRY(T.end());
    // B1f
    SYSML_TRY(T.begin(8));
    SYSML_TRY(conv_bwd_filter_dispatch(c1, *x, h->dz1, grads + OFF_F1, grads + OFF_B1, h->ws,
                                       h->ws_bytes, st));
    SYSML_TRY(T.end());
  }
  (void)launches0;
  if (h->ar_comm) {  // {F1, b1}, then the main stream joins the allreduce stream
    SYSML_TRY(ar_bucket(h, grads, OFF_F2, h->ev_b1, st));
    SYSML_CUDA(cudaEventRecord(h->ev_ar, h->ar_stream));
    SYSML_CUDA(cudaStreamWaitEvent(st, h->ev_ar, 0));
  }
  return SYSML_OK;
}

sysml_status sysml_lenet_fwd_bwd(sysml_lenet *h, const float *params, const sysml_input *x,
                                 const int32_t *labels, int32_t n_local, int64_t n_global,
                                 float *grads, float *loss_sum, sysml_stream_t stream) {
  SYSML_CHECK_ARG(labels && grads, "NULL labels / grads argument to sysml_lenet_fwd_bwd");
  return lenet_run(h, params, x, labels, n_local, n_global, grads, loss_sum, stream, nullptr, nullptr);
}

sysml_status sysml_lenet_predict(sysml_lenet *h, const float *params, const sysml_input *x, int32_t n_local,
                                 int32_t *pred, float *probs, sysml_stream_t stream) {
  SYSML_CHECK_ARG(pred || probs, "sysml_lenet_predict needs pred and/or probs");
  return lenet_run(h, params, x, nullptr, n_local, n_local, nullptr, nullptr, stream, pred, probs);
}

sysml_status sysml_sgd_update(float *params, const float *grads, int64_t n, float lr,
                              sysml_stream_t stream) {
  SYSML_CHECK_ARG(params && grads && n >= 0, "bad arguments to sysml_sgd_update");
  if (n == 0) return SYSML_OK;
  int blocks = (int)std::min<int64_t>(ceil_div(n, 256), 4 * sm_count());
  sgd_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(params, grads, n, lr);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

int32_t sysml_optimizer_state_floats(int32_t kind) {
  switch (kind) {
    case SYSML_OPT_SGD: return 0;
    case SYSML_OPT_MOMENTUM: case SYSML_OPT_NESTEROV: case SYSML_OPT_ADAGRAD: case SYSML_OPT_RMSPROP: return 1;
    case SYSML_OPT_ADAM: return 2;
    default: return -1;
  }
}

sysml_status sysml_optimizer_update(const sysml_optimizer_desc *d, float *params, const float *grads,
                                    float *state, int64_t n, int64_t t, sysml_stream_t stream) {
  SYSML_CHECK_ARG(d && params && grads, "NULL argument to sysml_optimizer_update");
  const int nst = sysml_optimizer_state_floats(d->kind);
  SYSML_CHECK_ARG(nst >= 0, "unknown optimizer kind %d", d->kind);
  SYSML_CHECK_ARG(nst == 0 || state, "optimizer kind %d needs a state buffer", d->kind);
  SYSML_CHECK_ARG(n >= 0, "n = %lld < 0", (long long)n);
  SYSML_CHECK_ARG(d->kind != SYSML_OPT_ADAM || t >= 1, "adam timestep t = %lld < 1", (long long)t);
  if (n == 0) return SYSML_OK;
  double c1 = 1.0, c2 = 1.0;
  if (d->kind == SYSML_OPT_ADAM) {
    c1 = 1.0 / (1.0 - pow((double)d->beta1, (double)t));
    c2 = 1.0 / (1.0 - pow((double)d->beta2, (double)t));
  }
  const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n, 256), 8 * sm_count());
  cudaStream_t st = (cudaStream_t)stream;
#define SYSML_OPT_LAUNCH(K)                                                                       \
  optimizer_kernel<K><<<blocks, 256, 0, st>>>(params, grads, state, n, d->lr, d->mu, d->rho, d->eps, \
                                              d->beta1, d->beta2, (float)c1, (float)c2)
  switch (d->kind) {
    case SYSML_OPT_SGD: SYSML_OPT_LAUNCH(SYSML_OPT_SGD); break;
    case SYSML_OPT_MOMENTUM: SYSML_OPT_LAUNCH(SYSML_OPT_MOMENTUM); break;
    case SYSML_OPT_NESTEROV: SYSML_OPT_LAUNCH(SYSML_OPT_NESTEROV); break;
    case SYSML_OPT_ADAGRAD: SYSML_OPT_LAUNCH(SYSML_OPT_ADAGRAD); break;
    case SYSML_OPT_RMSPROP: SYSML_OPT_LAUNCH(SYSML_OPT_RMSPROP); break;
    default: SYSML_OPT_LAUNCH(SYSML_OPT_ADAM); break;
  }
#undef SYSML_OPT_LAUNCH
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

// end of a training step: the dropout mask stream advances (device counter, graph-replayable)
static sysml_status step_done(sysml_lenet *h, sysml_stream_t stream) {
  if (!h->hidden) return SYSML_OK;
  return launch_counter_inc(h->drop_step, (cudaStream_t)stream);
}

sysml_status sysml_lenet_step(sysml_lenet *h, float *params, float *grads, const sysml_input *x,
                              const int32_t *labels, int32_t n_local, int64_t n_global,
                              float lr, void *nccl_comm, float *loss_sum, sysml_stream_t stream) {
  SYSML_CHECK_ARG(h, "NULL handle");
  // overlapped bucketed allreduce unless SYSML_AR_OVERLAP=0 (read per call)
  const char *ov = getenv("SYSML_AR_OVERLAP");
  if (nccl_comm && !(ov && ov[0] == '0')) {
    h->ar_comm = nccl_comm;
    const sysml_status r = sysml_lenet_fwd_bwd(h, params, x, labels, n_local, n_global, grads, loss_sum, stream);
    h->ar_comm = nullptr;
    SYSML_TRY(r);
    SYSML_TRY(sysml_sgd_update(params, grads, h->num_params, lr, stream));
    return step_done(h, stream);
  }
  SYSML_TRY(sysml_lenet_fwd_bwd(h, params, x, labels, n_local, n_global, grads, loss_sum, stream));
  if (nccl_comm) {
    NcclSyms &s = nccl_syms();
    if (!s.allreduce) {
      set_error("ncclAllReduce could not be resolved (libnccl.so.2 not loaded in this process)");
      return SYSML_ERR_NCCL;
    }
    const int r = s.allreduce(grads, grads, (size_t)h->num_params, /*ncclFloat32*/ 7, /*ncclSum*/ 0,
                              nccl_comm, (cudaStream_t)stream);
    if (r != 0) {
      set_error("ncclAllReduce failed: %s", s.errstr ? s.errstr(r) : "?");
      return SYSML_ERR_NCCL;
    }
  }
  SYSML_TRY(sysml_sgd_update(params, grads, h->num_params, lr, stream));
  return step_done(h, stream);
}

sysml_status sysml_lenet_step_opt(sysml_lenet *h, float *params, float *grads, float *state,
                                  const sysml_optimizer_desc *d, int64_t t, const sysml_input *x,
                                  const int32_t *labels, int32_t n_local, int64_t n_global,
                                  void *nccl_comm, float *loss_sum, sysml_stream_t stream) {
  SYSML_CHECK_ARG(h && d, "NULL argument to sysml_lenet_step_opt");
  SYSML_CHECK_ARG(sysml_optimizer_state_floats(d->kind) >= 0, "unknown optimizer kind %d", d->kind);
  h->ar_comm = nccl_comm;  // bucketed allreduce overlapped with the backward tail (may be NULL)
  const sysml_status r = sysml_lenet_fwd_bwd(h, params, x, labels, n_local, n_global, grads, loss_sum, stream);
  h->ar_comm = nullptr;
  SYSML_TRY(r);
  SYSML_TRY(sysml_optimizer_update(d, params, grads, state, h->num_params, t, stream));
  return step_done(h, stream);
}

sysml_status sysml_lenet_step_host(sysml_lenet *h, float *params, float *grads,
                                   const float *x_host, const int32_t *labels_host,
                                   int32_t n_local, int64_t n_global, float lr, void *nccl_comm,
                                   float *loss_host, sysml_stream_t stream) {
  SYSML_CHECK_ARG(h && x_host && labels_host && loss_host, "NULL argument to sysml_lenet_step_host");
  SYSML_CHECK_ARG(!h->csr, "sysml_lenet_step_host takes dense host input (handle is CSR)");
  SYSML_CHECK_ARG(n_local >= 1 && n_local <= h->max_b, "n_local %d out of range", n_local);
  cudaStream_t st = (cudaStream_t)stream;
  if (h->copy_stream) {  // a pipelined prefetch may still target slot 0: let it land first
    SYSML_CUDA(cudaStreamWaitEvent(st, h->ev_copied[0], 0));
    SYSML_CUDA(cudaStreamWaitEvent(st, h->ev_copied[1], 0));
    h->pf_slot = -1;
  }
  SYSML_CUDA(cudaMemcpyAsync(h->x_dev, x_host, sizeof(float) * (size_t)n_local * 784,
                             cudaMemcpyHostToDevice, st));
  SYSML_CUDA(cudaMemcpyAsync(h->lab_dev, labels_host, sizeof(int32_t) * (size_t)n_local,
                             cudaMemcpyHostToDevice, st));
  sysml_input xin{0, h->x_dev, {}};
  SYSML_TRY(sysml_lenet_step(h, params, grads, &xin, h->lab_dev, n_local, n_global, lr, nccl_comm,
                             h->loss_dev, stream));
  SYSML_CUDA(cudaMemcpyAsync(loss_host, h->loss_dev, sizeof(float), cudaMemcpyDeviceToHost, st));
  SYSML_CUDA(cudaStreamSynchronize(st));
  return SYSML_OK;
}

sysml_status sysml_lenet_step_host_pipelined(sysml_lenet *h, float *params, float *grads,
                                             const float *x_host, const int32_t *labels_host,
                                             int32_t n_local, const float *x_host_next,
                                             const int32_t *labels_host_next, int32_t n_next,
                                             int64_t n_global, float lr, void *nccl_comm,
                                             float *loss_host, sysml_stream_t stream) {
  SYSML_CHECK_ARG(h && x_host && labels_host && loss_host, "NULL argument to sysml_lenet_step_host_pipelined");
  SYSML_CHECK_ARG(!h->csr, "sysml_lenet_step_host_pipelined takes dense host input (handle is CSR)");
  SYSML_CHECK_ARG(n_local >= 1 && n_local <= h->max_b, "n_local %d out of range", n_local);
  SYSML_CHECK_ARG(!x_host_next || (labels_host_next && n_next >= 1 && n_next <= h->max_b),
                  "next batch: labels NULL or n_next %d out of range", n_next);
  cudaStream_t st = (cudaStream_t)stream;
  float *xs[2] = {h->x_dev, h->x_dev2};
  int32_t *ls[2] = {h->lab_dev, h->lab_dev2};
  int slot;
  if (h->pf_slot >= 0 && h->pf_x == x_host && h->pf_lab == labels_host && h->pf_n == n_local) {
    slot = h->pf_slot;  // prefetched by the previous call: wait for its copy only
  } else {
    slot = h->pf_slot >= 0 ? 1 - h->pf_slot : 0;  // miss: copy now on the copy stream
    SYSML_CUDA(cudaStreamWaitEvent(h->copy_stream, h->ev_consumed[slot], 0));
    SYSML_CUDA(cudaMemcpyAsync(xs[slot], x_host, sizeof(float) * (size_t)n_local * 784,
                               cudaMemcpyHostToDevice, h->copy_stream));
    SYSML_CUDA(cudaMemcpyAsync(ls[slot], labels_host, sizeof(int32_t) * (size_t)n_local,
                               cudaMemcpyHostToDevice, h->copy_stream));
    SYSML_CUDA(cudaEventRecord(h->ev_copied[slot], h->copy_stream));
  }
  SYSML_CUDA(cudaStreamWaitEvent(st, h->ev_copied[slot], 0));
  h->pf_slot = -1;
  if (x_host_next) {
    // the next batch goes to the other slot once the step that last read it is done; the
    // copy overlaps this step's kernels.  The host buffers must stay unchanged until then.
    const int ns = 1 - slot;
    SYSML_CUDA(cudaStreamWaitEvent(h->copy_stream, h->ev_consumed[ns], 0));
    SYSML_CUDA(cudaMemcpyAsync(xs[ns], x_host_next, sizeof(float) * (size_t)n_next * 784,
                               cudaMemcpyHostToDevice, h->copy_stream));
    SYSML_CUDA(cudaMemcpyAsync(ls[ns], labels_host_next, sizeof(int32_t) * (size_t)n_next,
                               cudaMemcpyHostToDevice, h->copy_stream));
    SYSML_CUDA(cudaEventRecord(h->ev_copied[ns], h->copy_stream));
    h->pf_slot = ns;
    h->pf_x = x_host_next;
    h->pf_lab = labels_host_next;
    h->pf_n = n_next;
  }
  sysml_input xin{0, xs[slot], {}};
  SYSML_TRY(sysml_lenet_step(h, params, grads, &xin, ls[slot], n_local, n_global, lr, nccl_comm,
                             h->loss_dev, stream));
  SYSML_CUDA(cudaEventRecord(h->ev_consumed[slot], st));
  SYSML_CUDA(cudaMemcpyAsync(loss_host, h->loss_dev, sizeof(float), cudaMemcpyDeviceToHost, st));
  SYSML_CUDA(cudaStreamSynchronize(st));
  return SYSML_OK;
}

sysml_status sysml_lenet_set_timing(sysml_lenet *h, int32_t enable) {
  SYSML_CHECK_ARG(h, "NULL handle");
  h->timing = enable != 0;
  return SYSML_OK;
}

sysml_status sysml_lenet_get_timing(sysml_lenet *h, int32_t max_stages, int32_t *n_stages,
                                    double *ms, int64_t *calls, const char **names) {
  SYSML_CHECK_ARG(h, "NULL handle");
  for (int s = 0; s < NSTAGES; ++s) {
    for (auto &e : h->pending[s]) {
      SYSML_CUDA(cudaEventSynchronize(e.second));
      float t = 0.f;
      SYSML_CUDA(cudaEventElapsedTime(&t, e.first, e.second));
      h->ms[s] += t;
      h->calls[s] += 1;
      h->pool.push_back(e);
    }
    h->pending[s].clear();
  }
  if (n_stages) *n_stages = NSTAGES;
  for (int s = 0; s < NSTAGES && s < max_stages; ++s) {
    if (ms) ms[s] = h->ms[s];
    if (calls) calls[s] = h->calls[s];
    if (names) names[s] = STAGE_NAMES[s];
  }
  if (max_stages < 0) {  // reset
    for (int s = 0; s < NSTAGES; ++s) { h->ms[s] = 0; h->calls[s] = 0; }
  }
  return SYSML_OK;
}

}  // extern "C"
