// sparse_filter.cu -- the sparse-filter physical convolution operators and the dense /
// sparse format decision.
//  * "four physical convolution operators ... dense input / dense filter, sparse
//    input / dense filter, dense input / sparse filter and sparse input / sparse filter".
//    The first two are sysml_conv2d; this file adds the filter bank as CSR (K rows x C*R*S
//    columns, column (c*R + r)*S + s), with dense or CSR input.
//  * P:163-165 "decides upon dense or sparse formats" (threshold 0.4): a non-zero
//    count and a deterministic dense -> CSR conversion.
// Oracle: oracle_conv2d_fwd_csr_filter / oracle_count_nonzeros (tests only).
#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "csr_dev.cuh"

namespace sysml {
namespace {

constexpr int SF_THREADS = 256;   // output positions per CTA
constexpr int SF_CHUNK = 1024;    // filter non-zeros decoded into shared memory per pass
constexpr int64_t SF_MAX_IMG = 48 * 1024;  // CSR input: C*H*W floats densified in smem

struct SfArgs {
  int N, C, H, W, K, R, S, sh, sw, ph, pw, P, Q, nchunk;
};

// CTA (image n x 256-position chunk, filter k).  The filter row's non-zeros are decoded into
// shared memory (plane offset c*H*W, r, s, value) SF_CHUNK at a time; every thread owns one
// output position and adds its taps in the stored order (deterministic).  CSR input: the
// image is densified in shared memory first (duplicate columns summed, R15).
__global__ void __launch_bounds__(SF_THREADS) conv_csr_filter_kernel(SfArgs a, const float *__restrict__ xd,
                                                                     sysml_csr xc, int is_csr, sysml_csr f,
                                                                     const float *__restrict__ bias,
                                                                     float *__restrict__ y) {
  extern __shared__ __align__(16) float sf_smem[];
  const int64_t HW = (int64_t)a.H * a.W, CHW = a.C * HW;
  int4 *fd = reinterpret_cast<int4 *>(sf_smem);          // [SF_CHUNK]
  float *img = sf_smem + 4 * SF_CHUNK;                   // [C*H*W] (CSR input)
  const int n = blockIdx.x / a.nchunk, chunk = blockIdx.x - n * a.nchunk, k = blockIdx.y;
  const int PQ = a.P * a.Q;
  const int pos = chunk * SF_THREADS + threadIdx.x;
  const bool valid = pos < PQ;
  const int p = valid ? pos / a.Q : 0, q = valid ? pos - p * a.Q : 0;
  const float *xn = xd + n * CHW;
  if (is_csr) {
    for (int64_t i = threadIdx.x; i < CHW; i += SF_THREADS) img[i] = 0.f;
    __syncthreads();
    const int j0 = xc.row_ptr[n], j1 = xc.row_ptr[n + 1];
    // duplicates summed in stored order (reading R15; csr_dev.cuh)
    csr_scatter_row(xc.col_idx, xc.val, j0, j1, threadIdx.x, SF_THREADS,
                    [&](int col) { return col >= 0 && col < CHW ? img + col : nullptr; },
                    [](bool b) { return __syncthreads_or(b) != 0; });
    xn = img;
  }
  const int RS = a.R * a.S, CRS = a.C * RS;
  float acc = bias ? __ldg(bias + k) : 0.f;
  const int j0 = f.row_ptr[k], j1 = f.row_ptr[k + 1];
  for (int jb = j0; jb < j1; jb += SF_CHUNK) {
    const int cnt = min(SF_CHUNK, j1 - jb);
    __syncthreads();  // the previous chunk's (or the densified image's) readers are done
    for (int t = threadIdx.x; t < cnt; t += SF_THREADS) {
      const int col = __ldg(f.col_idx + jb + t);
      const bool ok = col >= 0 && col < CRS;
      const int c = ok ? col / RS : 0, rem = ok ? col - c * RS : 0, r = rem / a.S, s = rem - r * a.S;
      fd[t] = make_int4(ok ? (int)(c * HW) : -1, r, s, __float_as_int(ok ? __ldg(f.val + jb + t) : 0.f));
    }
    __syncthreads();
    if (valid) {
      const int h0 = p * a.sh - a.ph, w0 = q * a.sw - a.pw;
      for (int t = 0; t < cnt; ++t) {
        const int4 e = fd[t];  // broadcast
        const int h = h0 + e.y, w = w0 + e.z;
        if (e.x >= 0 && h >= 0 && h < a.H && w >= 0 && w < a.W)
          acc = fmaf(__int_as_float(e.w), xn[e.x + h * a.W + w], acc);
      }
    }
  }
  if (valid) y[((int64_t)n * a.K + k) * PQ + pos] = acc;
}

// ---- format decision / conversion
__global__ void count_nonzeros_kernel(const float *__restrict__ x, int64_t n, unsigned long long *out) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += x[i] != 0.f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);  // integer sum: order-free
}

// warp per row: non-zeros of the row -> row_ptr[row + 1] (counts; scanned in place next)
__global__ void row_nnz_kernel(const float *__restrict__ x, int64_t rows, int64_t cols, int32_t *row_ptr) {
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float *xr = x + row * cols;
  int c = 0;
  for (int64_t j = lane; j < cols; j += 32) c += xr[j] != 0.f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) row_ptr[row + 1] = c;
}

// single CTA: row_ptr[0] = 0, row_ptr[i + 1] += row_ptr[i] (block-wide scan per 1024 rows,
// carried across blocks of rows)
__global__ void __launch_bounds__(1024) row_ptr_scan_kernel(int32_t *row_ptr, int64_t rows) {
  __shared__ int32_t sm[1024];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) {
    row_ptr[0] = 0;
    carry = 0;
  }
  __syncthreads();
  for (int64_t base = 0; base < rows; base += 1024) {
    const int64_t i = base + threadIdx.x;
    int v = i < rows ? row_ptr[i + 1] : 0;
    sm[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan
      const int t = threadIdx.x >= o ? sm[threadIdx.x - o] : 0;
      __syncthreads();
      sm[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < rows) row_ptr[i + 1] = sm[threadIdx.x] + carry;
    __syncthreads();
    if (threadIdx.x == 1023) carry += sm[1023];
    __syncthreads();
  }
}

// warp per row: the row's non-zeros in column order at row_ptr[row] (ballot prefix)
__global__ void csr_fill_kernel(const float *__restrict__ x, int64_t rows, int64_t cols,
                                const int32_t *__restrict__ row_ptr, int32_t *__restrict__ col_idx,
                                float *__restrict__ val) {
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float *xr = x + row * cols;
  int out = row_ptr[row];
  for (int64_t j0 = 0; j0 < cols; j0 += 32) {
    const int64_t j = j0 + lane;
    const float v = j < cols ? xr[j] : 0.f;
    const unsigned m = __ballot_sync(0xffffffffu, v != 0.f);
    if (v != 0.f) {
      const int o = out + __popc(m & ((1u << lane) - 1u));
      col_idx[o] = (int32_t)j;
      val[o] = v;
    }
    out += __popc(m);
  }
}

}  // namespace
}  // namespace sysml

using namespace sysml;

extern "C" {

sysml_status sysml_conv2d_csr_filter(const sysml_conv_desc *d, const sysml_input *x, const sysml_csr *f,
                                     const float *bias, float *y, sysml_stream_t stream) {
  SYSML_CHECK_ARG(d && x && f && y, "NULL argument to sysml_conv2d_csr_filter");
  ConvGeom g;
  SYSML_TRY(validate_conv(d, &g));
  SYSML_CHECK_SHAPE(f->rows == g.K && f->cols == g.C * g.R * g.S,
                    "sparse filter is %lldx%lld, expected K x C*R*S = %lldx%lld", (long long)f->rows,
                    (long long)f->cols, (long long)g.K, (long long)(g.C * g.R * g.S));
  SYSML_CHECK_ARG(f->row_ptr && (f->nnz == 0 || (f->col_idx && f->val)), "sparse filter arrays are NULL");
  if (x->is_csr) {
    SYSML_CHECK_SHAPE(x->csr.rows == g.N && x->csr.cols == g.C * g.H * g.W,
                      "CSR input is %lldx%lld, expected N x C*H*W = %lldx%lld", (long long)x->csr.rows,
                      (long long)x->csr.cols, (long long)g.N, (long long)(g.C * g.H * g.W));
    SYSML_CHECK_ARG(x->csr.row_ptr && (x->csr.nnz == 0 || (x->csr.col_idx && x->csr.val)), "CSR input arrays are NULL");
    if (g.C * g.H * g.W > SF_MAX_IMG) {
      set_error("sparse input / sparse filter: C*H*W = %lld exceeds %lld (the image is densified in shared memory)",
                (long long)(g.C * g.H * g.W), (long long)SF_MAX_IMG);
      return SYSML_ERR_UNSUPPORTED;
    }
  } else {
    SYSML_CHECK_ARG(x->dense, "NULL dense input");
  }
  if (g.N == 0 || g.K == 0) return SYSML_OK;
  SfArgs a{(int)g.N, (int)g.C, (int)g.H, (int)g.W, (int)g.K, (int)g.R, (int)g.S, (int)g.sh, (int)g.sw,
           (int)g.ph, (int)g.pw, (int)g.P, (int)g.Q, 0};
  a.nchunk = (int)ceil_div(g.P * g.Q, SF_THREADS);
  SYSML_CHECK_SHAPE((int64_t)a.nchunk * g.N < (1ll << 31) && g.K <= 65535, "sparse-filter conv grid too large");
  const size_t smem = sizeof(int4) * SF_CHUNK + (x->is_csr ? sizeof(float) * (size_t)(g.C * g.H * g.W) : 0);
  if (smem > 48 * 1024) SYSML_TRY(smem_attr(conv_csr_filter_kernel, smem));
  conv_csr_filter_kernel<<<dim3((unsigned)(a.nchunk * g.N), (unsigned)g.K), SF_THREADS, smem, (cudaStream_t)stream>>>(
      a, x->is_csr ? nullptr : x->dense, x->csr, x->is_csr, *f, bias, y);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status sysml_count_nonzeros(const float *x, int64_t n, int64_t *nnz_host, sysml_stream_t stream) {
  SYSML_CHECK_ARG(nnz_host && (x || n == 0) && n >= 0, "bad argument to sysml_count_nonzeros");
  *nnz_host = 0;
  if (n == 0) return SYSML_OK;
  cudaStream_t st = (cudaStream_t)stream;
  static thread_local unsigned long long *cnt = nullptr;
  static thread_local int cnt_dev = -1;
  int dev = 0;
  SYSML_CUDA(cudaGetDevice(&dev));
  if (!cnt || cnt_dev != dev) {
    SYSML_CUDA(cudaMalloc(&cnt, sizeof(unsigned long long)));
    cnt_dev = dev;
  }
  SYSML_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
  const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n, 256), 8 * sm_count());
  count_nonzeros_kernel<<<blocks, 256, 0, st>>>(x, n, cnt);
  SYSML_LAUNCH_CHECK();
  unsigned long long h = 0;
  SYSML_CUDA(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st));
  SYSML_CUDA(cudaStreamSynchronize(st));
  *nnz_host = (int64_t)h;
  return SYSML_OK;
}

sysml_status sysml_decide_format(const float *x, int64_t n, double threshold, int32_t *is_sparse,
                                 int64_t *nnz_host, sysml_stream_t stream) {
  SYSML_CHECK_ARG(is_sparse && nnz_host, "bad argument to sysml_decide_format");
  SYSML_TRY(sysml_count_nonzeros(x, n, nnz_host, stream));
  const double thr = threshold > 0.0 ? threshold : SYSML_SPARSITY_THRESHOLD;
  *is_sparse = (n > 0 && (double)*nnz_host <= thr * (double)n) ? 1 : 0;
  return SYSML_OK;
}

sysml_status sysml_dense_to_csr(const float *x, int64_t rows, int64_t cols, int32_t *row_ptr, int32_t *col_idx,
                                float *val, sysml_stream_t stream) {
  SYSML_CHECK_ARG(row_ptr && rows >= 0 && cols >= 0 && (x || rows * cols == 0), "bad argument to sysml_dense_to_csr");
  SYSML_CHECK_ARG(rows * cols < (1ll << 31), "dense_to_csr: rows*cols = %lld does not fit int32 indices",
                  (long long)(rows * cols));
  cudaStream_t st = (cudaStream_t)stream;
  if (rows == 0) {
    SYSML_CUDA(cudaMemsetAsync(row_ptr, 0, sizeof(int32_t), st));
    return SYSML_OK;
  }
  const unsigned blocks = (unsigned)ceil_div(rows, 8);
  row_nnz_kernel<<<blocks, 256, 0, st>>>(x, rows, cols, row_ptr);
  SYSML_LAUNCH_CHECK();
  row_ptr_scan_kernel<<<1, 1024, 0, st>>>(row_ptr, rows);
  SYSML_LAUNCH_CHECK();
  csr_fill_kernel<<<blocks, 256, 0, st>>>(x, rows, cols, row_ptr, col_idx, val);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

}  // extern "C"
