// csr.cu -- sparse-input (CSR) conv2d kernels: the "sparse input / dense filter"
// physical operator of P:171-174, sparse-safe per P:168-170 ("reduces the number
// of floating point operations and improves memory efficiency").
//
// K7 csr_conv_fwd: one CTA per image (grid-stride).  The CSR row is gathered into
// a zeroed shared-memory copy of the image (warp-cooperative, coalesced loads of
// col_idx/val), the filter bank sits in shared memory, and each thread produces
// output pixels for a chunk of filters, skipping zero taps (work ~ nnz).  Output
// stores are coalesced along (p,q).  Optional fused bias + relu + non-overlapping
// max-pool epilogue writes only the pooled output and its argmax.
//
// K8 csr_conv_bwd_filter: one CTA per contiguous chunk of images.  Each image's
// dY (K x P x Q) is streamed into shared memory with 16-byte loads, the CSR row is
// staged, and every thread accumulates its own (k, r, s) outputs over the
// non-zeros in CSR order into a shared-memory dF partial (disjoint ownership, no
// atomics).  db is summed from the staged dY.  Chunk partials are reduced in a
// fixed order (deterministic).
#include "common.cuh"
#include "kernels.cuh"

namespace sysml {

namespace {

constexpr int CSR_THREADS = 256;
constexpr int MAX_IMG_FLOATS = 8192;      // dense image in smem (32 KB)
constexpr int MAX_FILTER_FLOATS = 8192;   // filter bank in smem (32 KB)
constexpr int FWD_KC = 8;                 // filters per register chunk

__device__ __forceinline__ void stage_row_dense(const sysml_csr &m, int64_t row, float *img,
                                                int chw) {
  for (int i = threadIdx.x; i < chw; i += blockDim.x) img[i] = 0.f;
  __syncthreads();
  const int j0 = __ldg(m.row_ptr + row), j1 = __ldg(m.row_ptr + row + 1);
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    const int col = __ldg(m.col_idx + j);
    const float v = __ldg(m.val + j);
    if (col >= 0 && col < chw) atomicAdd(img + col, v);  // duplicates summed (reading R15)
  }
  __syncthreads();
}

__global__ void __launch_bounds__(CSR_THREADS)
    csr_fwd_kernel(ConvArgs a, sysml_csr m, const float *__restrict__ f,
                   const float *__restrict__ bias, float *__restrict__ y) {
  extern __shared__ float sm[];
  const int CHW = a.C * a.H * a.W, CRS = a.C * a.R * a.S, RS = a.R * a.S, PQ = a.P * a.Q;
  float *fs = sm;              // K x CRS
  float *img = sm + a.K * CRS; // C x H x W
  for (int i = threadIdx.x; i < a.K * CRS; i += blockDim.x) fs[i] = __ldg(f + i);
  for (int64_t n = blockIdx.x; n < a.N; n += gridDim.x) {
    stage_row_dense(m, n, img, CHW);
    float *yn = y + n * (int64_t)a.K * PQ;
    for (int pq = threadIdx.x; pq < PQ; pq += blockDim.x) {
      const int p = pq / a.Q, q = pq - p * a.Q;
      for (int k0 = 0; k0 < a.K; k0 += FWD_KC) {
        float acc[FWD_KC];
#pragma unroll
        for (int i = 0; i < FWD_KC; ++i) acc[i] = 0.f;
        for (int c = 0; c < a.C; ++c)
          for (int r = 0; r < a.R; ++r) {
            const int h = p * a.sh - a.ph + r;
            if (h < 0 || h >= a.H) continue;
            for (int s = 0; s < a.S; ++s) {
              const int w = q * a.sw - a.pw + s;
              if (w < 0 || w >= a.W) continue;
              const float v = img[(c * a.H + h) * a.W + w];
              if (v == 0.f) continue;  // sparse-safe: zero inputs do no work
              const float *fk = fs + (int64_t)k0 * CRS + c * RS + r * a.S + s;
#pragma unroll
              for (int i = 0; i < FWD_KC; ++i)
                if (k0 + i < a.K) acc[i] = fmaf(v, fk[i * CRS], acc[i]);
            }
          }
#pragma unroll
        for (int i = 0; i < FWD_KC; ++i)
          if (k0 + i < a.K) yn[(int64_t)(k0 + i) * PQ + pq] = acc[i] + (bias ? __ldg(bias + k0 + i) : 0.f);
      }
    }
    __syncthreads();
  }
}

// Fused: conv + bias + relu + max-pool (window == stride, pad 0).  One thread per
// pooled output (k-chunk); the window is scanned r-outer/s-inner with strict '>'
// on relu'd values (readings R5, R7), argmax = column in the conv-output row.
__global__ void __launch_bounds__(CSR_THREADS)
    csr_fwd_pool_kernel(ConvArgs a, PoolArgs pa, sysml_csr m, const float *__restrict__ f,
                        const float *__restrict__ bias, float *__restrict__ out,
                        int32_t *__restrict__ arg) {
  extern __shared__ float sm[];
  const int CHW = a.C * a.H * a.W, CRS = a.C * a.R * a.S, RS = a.R * a.S;
  const int PQo = pa.P * pa.Q;
  float *fs = sm;
  float *img = sm + a.K * CRS;
  for (int i = threadIdx.x; i < a.K * CRS; i += blockDim.x) fs[i] = __ldg(f + i);
  for (int64_t n = blockIdx.x; n < a.N; n += gridDim.x) {
    stage_row_dense(m, n, img, CHW);
    float *on = out + n * (int64_t)a.K * PQo;
    int32_t *an = arg ? arg + n * (int64_t)a.K * PQo : nullptr;
    for (int o = threadIdx.x; o < PQo; o += blockDim.x) {
      const int po = o / pa.Q, qo = o - po * pa.Q;
      for (int k0 = 0; k0 < a.K; k0 += FWD_KC) {
        float best[FWD_KC];
        int barg[FWD_KC];
#pragma unroll
        for (int i = 0; i < FWD_KC; ++i) { best[i] = 0.f; barg[i] = -1; }
        for (int wr = 0; wr < pa.R; ++wr)
          for (int ws = 0; ws < pa.S; ++ws) {
            const int p = po * pa.sh + wr, q = qo * pa.sw + ws;
            if (p >= a.P || q >= a.Q) continue;
            float acc[FWD_KC];
#pragma unroll
            for (int i = 0; i < FWD_KC; ++i) acc[i] = 0.f;
            for (int c = 0; c < a.C; ++c)
              for (int r = 0; r < a.R; ++r) {
                const int h = p * a.sh - a.ph + r;
                if (h < 0 || h >= a.H) continue;
                for (int s = 0; s < a.S; ++s) {
                  const int w = q * a.sw - a.pw + s;
                  if (w < 0 || w >= a.W) continue;
                  const float v = img[(c * a.H + h) * a.W + w];
                  if (v == 0.f) continue;
                  const float *fk = fs + (int64_t)k0 * CRS + c * RS + r * a.S + s;
#pragma unroll
                  for (int i = 0; i < FWD_KC; ++i)
                    if (k0 + i < a.K) acc[i] = fmaf(v, fk[i * CRS], acc[i]);
                }
              }
            const int col_in_plane = p * a.Q + q;
#pragma unroll
            for (int i = 0; i < FWD_KC; ++i) {
              if (k0 + i >= a.K) continue;
              float z = acc[i] + (bias ? __ldg(bias + k0 + i) : 0.f);
              z = z > 0.f ? z : 0.f;
              if (barg[i] < 0 || z > best[i]) {
                best[i] = z;
                barg[i] = (k0 + i) * a.P * a.Q + col_in_plane;
              }
            }
          }
#pragma unroll
        for (int i = 0; i < FWD_KC; ++i) {
          if (k0 + i >= a.K) continue;
          on[(int64_t)(k0 + i) * PQo + o] = barg[i] < 0 ? 0.f : best[i];
          if (an) an[(int64_t)(k0 + i) * PQo + o] = barg[i];
        }
      }
    }
    __syncthreads();
  }
}

constexpr int BWF_MAX_DY_FLOATS = 26 * 1024;  // 104 KB of dY per image in smem
constexpr int BWF_MAX_NNZ = 1024;              // staged per pass

__global__ void __launch_bounds__(CSR_THREADS)
    csr_bwd_filter_kernel(ConvArgs a, sysml_csr m, const float *__restrict__ dy,
                          int n_per_block, float *__restrict__ part, float *__restrict__ dbpart) {
  extern __shared__ __align__(16) float sm[];
  const int PQ = a.P * a.Q, KPQ = a.K * PQ, RS = a.R * a.S, CRS = a.C * RS;
  const int KCRS = a.K * CRS;
  float *dys = sm;                       // K*PQ (rounded to 4)
  float *dfs = dys + ((KPQ + 3) & ~3);   // K*CRS
  float *dbs = dfs + KCRS;               // K
  int *nz_col = (int *)(dbs + a.K);      // BWF_MAX_NNZ
  float *nz_val = (float *)(nz_col + BWF_MAX_NNZ);
  for (int i = threadIdx.x; i < KCRS; i += blockDim.x) dfs[i] = 0.f;
  for (int i = threadIdx.x; i < a.K; i += blockDim.x) dbs[i] = 0.f;
  const int n0 = blockIdx.x * n_per_block, n1 = min(a.N, n0 + n_per_block);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int n = n0; n < n1; ++n) {
    __syncthreads();
    const float *dyn = dy + (int64_t)n * KPQ;
    if ((KPQ & 3) == 0 && ((uintptr_t)dyn & 15) == 0) {
      const float4 *src = reinterpret_cast<const float4 *>(dyn);
      float4 *dst = reinterpret_cast<float4 *>(dys);
      for (int i = threadIdx.x; i < KPQ / 4; i += blockDim.x) dst[i] = __ldg(src + i);
    } else {
      for (int i = threadIdx.x; i < KPQ; i += blockDim.x) dys[i] = __ldg(dyn + i);
    }
    __syncthreads();
    // db: warp w sums planes k = w, w+nwarps, ... (fixed order)
    for (int k = warp; k < a.K; k += nwarps) {
      float s = 0.f;
      for (int j = lane; j < PQ; j += 32) s += dys[k * PQ + j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) dbs[k] += s;
    }
    const int j0 = __ldg(m.row_ptr + n), j1 = __ldg(m.row_ptr + n + 1);
    for (int jb = j0; jb < j1; jb += BWF_MAX_NNZ) {
      const int cnt = min(BWF_MAX_NNZ, j1 - jb);
      __syncthreads();
      for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
        nz_col[i] = __ldg(m.col_idx + jb + i);
        nz_val[i] = __ldg(m.val + jb + i);
      }
      __syncthreads();
      // thread owns outputs o = (k, r, s) (all c): o = t, t + blockDim, ...
      for (int o = threadIdx.x; o < a.K * RS; o += blockDim.x) {
        const int k = o / RS, rs = o - k * RS, r = rs / a.S, s = rs - r * a.S;
        const float *dyk = dys + k * PQ;
        float *dfk = dfs + k * CRS + rs;
        for (int i = 0; i < cnt; ++i) {
          const int col = nz_col[i];
          const int c = col / (a.H * a.W), hw = col - c * a.H * a.W;
          const int h = hw / a.W, w = hw - h * a.W;
          const int hp = h + a.ph - r, wp = w + a.pw - s;
          if (hp < 0 || wp < 0) continue;
          const int p = hp / a.sh, q = wp / a.sw;
          if (p * a.sh != hp || q * a.sw != wp || p >= a.P || q >= a.Q) continue;
          dfk[c * RS] = fmaf(nz_val[i], dyk[p * a.Q + q], dfk[c * RS]);
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < KCRS; i += blockDim.x) part[(int64_t)blockIdx.x * KCRS + i] = dfs[i];
  if (dbpart)
    for (int i = threadIdx.x; i < a.K; i += blockDim.x) dbpart[(int64_t)blockIdx.x * a.K + i] = dbs[i];
}

__global__ void ordered_sum_kernel(const float *__restrict__ part, int parts, int64_t n,
                                   float *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int z = 0; z < parts; ++z) acc += __ldg(part + (int64_t)z * n + i);
    out[i] = acc;
  }
}

__global__ void csr_densify_kernel(sysml_csr m, float *__restrict__ dense) {
  for (int64_t r = blockIdx.x; r < m.rows; r += gridDim.x) {
    float *row = dense + r * m.cols;
    for (int64_t i = threadIdx.x; i < m.cols; i += blockDim.x) row[i] = 0.f;
    __syncthreads();
    const int j0 = m.row_ptr[r], j1 = m.row_ptr[r + 1];
    for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
      const int c = m.col_idx[j];
      if (c >= 0 && c < m.cols) atomicAdd(row + c, m.val[j]);
    }
    __syncthreads();
  }
}

__global__ void csr_check_kernel(sysml_csr m, unsigned long long *bad) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m.rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int j0 = m.row_ptr[r], j1 = m.row_ptr[r + 1];
    bool ok = j0 <= j1 && j0 >= 0 && j1 <= m.nnz && (r != 0 || j0 == 0);
    for (int j = j0; ok && j < j1; ++j) {
      const int c = m.col_idx[j];
      const float v = m.val[j];
      if (c < 0 || c >= m.cols || v == 0.f || !isfinite(v)) ok = false;
      if (j > j0 && m.col_idx[j - 1] >= c) ok = false;
    }
    if (!ok) atomicAdd(bad, 1ull);
  }
}

size_t fwd_smem(const ConvArgs &a) {
  return sizeof(float) * ((size_t)a.K * a.C * a.R * a.S + (size_t)a.C * a.H * a.W);
}

size_t bwf_smem(const ConvArgs &a) {
  const size_t kpq = ((size_t)a.K * a.P * a.Q + 3) & ~(size_t)3;
  return sizeof(float) * (kpq + (size_t)a.K * a.C * a.R * a.S + a.K) +
         BWF_MAX_NNZ * (sizeof(int) + sizeof(float));
}

int bwf_blocks(const ConvArgs &a) {
  const size_t smem = bwf_smem(a);
  int per_sm = (int)(220 * 1024 / (smem + 1024));
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 4) per_sm = 4;
  int blocks = sm_count() * per_sm;
  if (blocks > a.N) blocks = a.N;
  return blocks < 1 ? 1 : blocks;
}

}  // namespace

bool csr_fwd_supported(const ConvArgs &a) {
  return (int64_t)a.C * a.H * a.W <= MAX_IMG_FLOATS &&
         (int64_t)a.K * a.C * a.R * a.S <= MAX_FILTER_FLOATS;
}

sysml_status csr_conv_fwd(const ConvArgs &a, const sysml_csr &x, const float *f,
                          const float *bias, float *y, const PoolArgs *pool, float *pout,
                          int32_t *parg, cudaStream_t st) {
  const size_t smem = fwd_smem(a);
  int blocks = a.N < 8 * sm_count() ? a.N : 8 * sm_count();
  if (pool) {
    static bool attr_set = false;
    if (!attr_set) {
      SYSML_CUDA(cudaFuncSetAttribute(csr_fwd_pool_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
      attr_set = true;
    }
    csr_fwd_pool_kernel<<<blocks, CSR_THREADS, smem, st>>>(a, *pool, x, f, bias, pout, parg);
  } else {
    static bool attr_set = false;
    if (!attr_set) {
      SYSML_CUDA(cudaFuncSetAttribute(csr_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      96 * 1024));
      attr_set = true;
    }
    csr_fwd_kernel<<<blocks, CSR_THREADS, smem, st>>>(a, x, f, bias, y);
  }
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

bool csr_bwd_filter_supported(const ConvArgs &a) {
  return (int64_t)a.K * a.P * a.Q <= BWF_MAX_DY_FLOATS &&
         (int64_t)a.K * a.C * a.R * a.S <= MAX_FILTER_FLOATS;
}

size_t csr_bwd_filter_ws(const ConvArgs &a) {
  const int blocks = bwf_blocks(a);
  return align_up((size_t)blocks * a.K * a.C * a.R * a.S * sizeof(float), 256) +
         align_up((size_t)blocks * a.K * sizeof(float), 256);
}

sysml_status csr_conv_bwd_filter(const ConvArgs &a, const sysml_csr &x, const float *dy,
                                 float *df, float *db, void *ws, cudaStream_t st) {
  const int blocks = bwf_blocks(a);
  const int npb = (int)ceil_div(a.N, blocks);
  const int used = (int)ceil_div(a.N, npb);
  WsCarve wc(ws, (size_t)-1);
  const int64_t kcrs = (int64_t)a.K * a.C * a.R * a.S;
  float *part = wc.take<float>((size_t)blocks * kcrs);
  float *dbpart = wc.take<float>((size_t)blocks * a.K);
  const size_t smem = bwf_smem(a);
  static bool attr_set = false;
  if (!attr_set) {
    SYSML_CUDA(cudaFuncSetAttribute(csr_bwd_filter_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_set = true;
  }
  csr_bwd_filter_kernel<<<used, CSR_THREADS, smem, st>>>(a, x, dy, npb, part, db ? dbpart : nullptr);
  SYSML_LAUNCH_CHECK();
  ordered_sum_kernel<<<(unsigned)ceil_div(kcrs, 256), 256, 0, st>>>(part, used, kcrs, df);
  SYSML_LAUNCH_CHECK();
  if (db) {
    ordered_sum_kernel<<<(unsigned)ceil_div(a.K, 256), 256, 0, st>>>(dbpart, used, a.K, db);
    SYSML_LAUNCH_CHECK();
  }
  return SYSML_OK;
}

sysml_status csr_densify(const sysml_csr &x, float *dense, cudaStream_t st) {
  int blocks = x.rows < 4 * sm_count() ? (int)x.rows : 4 * sm_count();
  if (blocks < 1) blocks = 1;
  csr_densify_kernel<<<blocks, 256, 0, st>>>(x, dense);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status csr_check(const sysml_csr &m, int64_t *violations, cudaStream_t st) {
  unsigned long long *d = nullptr;
  SYSML_CUDA(cudaMallocAsync(&d, sizeof(unsigned long long), st));
  SYSML_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), st));
  int blocks = (int)ceil_div(m.rows, 256);
  if (blocks < 1) blocks = 1;
  if (blocks > 4 * sm_count()) blocks = 4 * sm_count();
  csr_check_kernel<<<blocks, 256, 0, st>>>(m, d);
  SYSML_LAUNCH_CHECK();
  unsigned long long h = 0;
  SYSML_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
  SYSML_CUDA(cudaStreamSynchronize(st));
  SYSML_CUDA(cudaFreeAsync(d, st));
  *violations = (int64_t)h;
  return SYSML_OK;
}

}  // namespace sysml
