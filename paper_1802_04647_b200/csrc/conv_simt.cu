// conv_simt.cu -- fp32 CUDA-core implicit-GEMM convolution (SYSML_MATH_FP32 path).
//
// Lowering without materialising im2col ("lowering technique"):
// every operator is a GEMM whose operand tiles are gathered straight from the
// row-major N x (C*H*W) encoding into shared memory, zero-filling padding:
//   fwd        Y[k, (n,p,q)]   = sum_{(c,r,s)} F[k,(c,r,s)] * Xcol[(c,r,s),(n,p,q)]
//   bwd_data   dX[c, (n,h,w)]  = sum_{(k,r,s)} F[k,(c,r,s)] * dYcol[(k,r,s),(n,h,w)]
//   bwd_filter dF[k, (c,r,s)]  = sum_{(n,p,q)} dY[k,(n,p,q)] * Xcol[(c,r,s),(n,p,q)]
// 64x64x16 block tile, 256 threads, 4x4 register tile per thread, register
// prefetch of the next K-slice.  bwd_filter splits the (n,p,q) reduction over
// blockIdx.z and sums the partials in a fixed order (deterministic, no atomics).
#include "common.cuh"
#include "kernels.cuh"

namespace sysml {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

struct FwdOp {
  ConvArgs a;
  const float *x, *f, *bias;
  float *y;
  static constexpr bool A_ALONG_K = true;   // F rows contiguous along (c,r,s)
  static constexpr bool B_ALONG_K = false;  // pixels contiguous
  __device__ int M() const { return a.K; }
  __device__ int Ng() const { return a.N * a.P * a.Q; }
  __device__ int Kg() const { return a.C * a.R * a.S; }
  __device__ float A(int m, int kk) const { return __ldg(f + (int64_t)m * Kg() + kk); }
  __device__ float B(int kk, int col) const {
    const int PQ = a.P * a.Q, RS = a.R * a.S;
    const int n = col / PQ, pq = col - n * PQ, p = pq / a.Q, q = pq - p * a.Q;
    const int c = kk / RS, rs = kk - c * RS, r = rs / a.S, s = rs - r * a.S;
    const int h = p * a.sh - a.ph + r, w = q * a.sw - a.pw + s;
    if (h < 0 || h >= a.H || w < 0 || w >= a.W) return 0.f;
    return __ldg(x + (int64_t)n * a.C * a.H * a.W + ((int64_t)c * a.H + h) * a.W + w);
  }
  __device__ void store(int m, int col, float v, int) const {
    const int PQ = a.P * a.Q;
    const int n = col / PQ, pq = col - n * PQ;
    if (bias) v += __ldg(bias + m);
    y[(int64_t)n * a.K * PQ + (int64_t)m * PQ + pq] = v;
  }
};

struct BwdDataOp {
  ConvArgs a;
  const float *f, *dy;
  float *dx;
  static constexpr bool A_ALONG_K = false;
  static constexpr bool B_ALONG_K = false;
  __device__ int M() const { return a.C; }
  __device__ int Ng() const { return a.N * a.H * a.W; }
  __device__ int Kg() const { return a.K * a.R * a.S; }
  __device__ float A(int c, int kk) const {
    const int RS = a.R * a.S;
    const int k = kk / RS, rs = kk - k * RS;
    return __ldg(f + (int64_t)k * a.C * RS + (int64_t)c * RS + rs);
  }
  __device__ float B(int kk, int col) const {
    const int HW = a.H * a.W, RS = a.R * a.S;
    const int n = col / HW, hw = col - n * HW, h = hw / a.W, w = hw - h * a.W;
    const int k = kk / RS, rs = kk - k * RS, r = rs / a.S, s = rs - r * a.S;
    const int hp = h + a.ph - r, wp = w + a.pw - s;
    if (hp < 0 || wp < 0) return 0.f;
    const int p = hp / a.sh, q = wp / a.sw;
    if (p * a.sh != hp || q * a.sw != wp || p >= a.P || q >= a.Q) return 0.f;
    return __ldg(dy + (int64_t)n * a.K * a.P * a.Q + ((int64_t)k * a.P + p) * a.Q + q);
  }
  __device__ void store(int c, int col, float v, int) const {
    const int HW = a.H * a.W;
    const int n = col / HW, hw = col - n * HW;
    dx[(int64_t)n * a.C * HW + (int64_t)c * HW + hw] = v;
  }
};

struct BwdFilterOp {
  ConvArgs a;
  const float *x, *dy;
  float *part;  // [splits][K][CRS]
  static constexpr bool A_ALONG_K = true;  // dY contiguous along (p,q)
  static constexpr bool B_ALONG_K = true;  // X contiguous along (q)
  __device__ int M() const { return a.K; }
  __device__ int Ng() const { return a.C * a.R * a.S; }
  __device__ int Kg() const { return a.N * a.P * a.Q; }
  __device__ float A(int k, int kk) const {
    const int PQ = a.P * a.Q;
    const int n = kk / PQ, pq = kk - n * PQ;
    return __ldg(dy + (int64_t)n * a.K * PQ + (int64_t)k * PQ + pq);
  }
  __device__ float B(int kk, int crs) const {
    const int PQ = a.P * a.Q, RS = a.R * a.S;
    const int n = kk / PQ, pq = kk - n * PQ, p = pq / a.Q, q = pq - p * a.Q;
    const int c = crs / RS, rs = crs - c * RS, r = rs / a.S, s = rs - r * a.S;
    const int h = p * a.sh - a.ph + r, w = q * a.sw - a.pw + s;
    if (h < 0 || h >= a.H || w < 0 || w >= a.W) return 0.f;
    return __ldg(x + (int64_t)n * a.C * a.H * a.W + ((int64_t)c * a.H + h) * a.W + w);
  }
  __device__ void store(int k, int crs, float v, int split) const {
    part[((int64_t)split * a.K + k) * (a.C * a.R * a.S) + crs] = v;
  }
};

template <class Op>
__global__ void __launch_bounds__(NT) igemm_kernel(Op op, int k_per_split) {
  __shared__ __align__(16) float As[2][BK][BM + 4];
  __shared__ __align__(16) float Bs[2][BK][BN + 4];
  const int t = threadIdx.x;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int M = op.M(), Ng = op.Ng(), Kg = op.Kg();
  const int kbeg = blockIdx.z * k_per_split;
  const int kend = min(Kg, kbeg + k_per_split);

  // load mappings (4 elements per thread per operand per K-slice)
  int am[4], ak[4], bk[4], bn[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (Op::A_ALONG_K) { ak[i] = t % BK; am[i] = t / BK + 16 * i; }
    else               { am[i] = t % BM; ak[i] = (t / BM) * 4 + i; }
    if (Op::B_ALONG_K) { bk[i] = t % BK; bn[i] = t / BK + 16 * i; }
    else               { bn[i] = t % BN; bk[i] = (t / BN) * 4 + i; }
  }
  float ra[4], rb[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + am[i], kk = k0 + ak[i];
      ra[i] = (m < M && kk < kend) ? op.A(m, kk) : 0.f;
      const int col = n0 + bn[i], kb = k0 + bk[i];
      rb[i] = (col < Ng && kb < kend) ? op.B(kb, col) : 0.f;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      As[buf][ak[i]][am[i]] = ra[i];
      Bs[buf][bk[i]][bn[i]] = rb[i];
    }
  };

  const int tx = t % 16, ty = t / 16;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  if (kbeg < kend) {
    load(kbeg);
    stash(0);
    __syncthreads();
    int buf = 0;
    for (int k0 = kbeg; k0 < kend; k0 += BK) {
      const bool more = k0 + BK < kend;
      if (more) load(k0 + BK);
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        const float4 av = *reinterpret_cast<const float4 *>(&As[buf][kk][ty * 4]);
        const float4 bv = *reinterpret_cast<const float4 *>(&Bs[buf][kk][tx * 4]);
        const float a4[4] = {av.x, av.y, av.z, av.w};
        const float b4[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a4[i], b4[j], acc[i][j]);
      }
      if (more) {
        stash(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = n0 + tx * 4 + j;
      if (col < Ng) op.store(m, col, acc[i][j], blockIdx.z);
    }
  }
}

// Deterministic split-K reduction: out[i] = sum_{z=0..splits-1} part[z][i] (z ascending).
__global__ void splitk_reduce_kernel(const float *__restrict__ part, int splits, int64_t n,
                                     float *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int z = 0; z < splits; ++z) acc += __ldg(part + (int64_t)z * n + i);
    out[i] = acc;
  }
}

// db[k] = sum_{n,p,q} dY[n,k,p,q]: stage 1 sums a contiguous chunk of samples for
// one k per block (fixed tree order), stage 2 sums the chunk partials in order.
constexpr int BG_THREADS = 256;
__global__ void bias_grad_stage1(ConvArgs a, const float *__restrict__ dy, int n_per_chunk,
                                 float *__restrict__ part) {
  const int k = blockIdx.x, chunk = blockIdx.y;
  const int PQ = a.P * a.Q;
  const int n0 = chunk * n_per_chunk, n1 = min(a.N, n0 + n_per_chunk);
  float acc = 0.f;
  for (int n = n0; n < n1; ++n) {
    const float *row = dy + (int64_t)n * a.K * PQ + (int64_t)k * PQ;
    for (int j = threadIdx.x; j < PQ; j += BG_THREADS) acc += __ldg(row + j);
  }
  __shared__ float red[BG_THREADS];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = BG_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(int64_t)k * gridDim.y + chunk] = red[0];
}

__global__ void bias_grad_stage2(int K, int chunks, const float *__restrict__ part,
                                 float *__restrict__ db) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  float acc = 0.f;
  for (int c = 0; c < chunks; ++c) acc += part[(int64_t)k * chunks + c];
  db[k] = acc;
}

int bias_grad_chunks(const ConvArgs &a) {
  int64_t chunks = ceil_div(2 * sm_count(), a.K);
  if (chunks > a.N) chunks = a.N;
  if (chunks < 1) chunks = 1;
  return (int)chunks;
}

int bwd_filter_splits(const ConvArgs &a) {
  const int64_t tiles = ceil_div(a.K, BM) * ceil_div((int64_t)a.C * a.R * a.S, BN);
  const int64_t kg = (int64_t)a.N * a.P * a.Q;
  int64_t splits = ceil_div(2 * sm_count(), tiles);
  const int64_t max_splits = ceil_div(kg, 4 * BK);
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  if (splits > 1024) splits = 1024;
  return (int)splits;
}

}  // namespace

sysml_status simt_conv_fwd(const ConvArgs &a, const float *x, const float *f, const float *bias,
                           float *y, cudaStream_t st) {
  FwdOp op{a, x, f, bias, y};
  const int64_t ng = (int64_t)a.N * a.P * a.Q;
  dim3 grid((unsigned)ceil_div(ng, BN), (unsigned)ceil_div(a.K, BM), 1);
  route_note("igemm_kernel<Fwd> (FP32 SIMT)");
  igemm_kernel<FwdOp><<<grid, NT, 0, st>>>(op, a.C * a.R * a.S);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status simt_conv_bwd_data(const ConvArgs &a, const float *f, const float *dy, float *dx,
                                cudaStream_t st) {
  BwdDataOp op{a, f, dy, dx};
  const int64_t ng = (int64_t)a.N * a.H * a.W;
  dim3 grid((unsigned)ceil_div(ng, BN), (unsigned)ceil_div(a.C, BM), 1);
  route_note("igemm_kernel<BwdData> (FP32 SIMT)");
  igemm_kernel<BwdDataOp><<<grid, NT, 0, st>>>(op, a.K * a.R * a.S);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

size_t bias_grad_ws(const ConvArgs &a) {
  return align_up((size_t)a.K * bias_grad_chunks(a) * sizeof(float), 256);
}

size_t simt_bwd_filter_ws(const ConvArgs &a) {
  const int splits = bwd_filter_splits(a);
  size_t b = align_up((size_t)splits * a.K * a.C * a.R * a.S * sizeof(float), 256);
  b += align_up((size_t)a.K * bias_grad_chunks(a) * sizeof(float), 256);
  return b;
}

sysml_status launch_bias_grad(const ConvArgs &a, const float *dy, float *db, float *part,
                              cudaStream_t st) {
  const int chunks = bias_grad_chunks(a);
  const int npc = (int)ceil_div(a.N, chunks);
  bias_grad_stage1<<<dim3(a.K, chunks), BG_THREADS, 0, st>>>(a, dy, npc, part);
  SYSML_LAUNCH_CHECK();
  bias_grad_stage2<<<(unsigned)ceil_div(a.K, 128), 128, 0, st>>>(a.K, chunks, part, db);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status simt_conv_bwd_filter(const ConvArgs &a, const float *x, const float *dy, float *df,
                                  float *db, void *ws, cudaStream_t st) {
  const int splits = bwd_filter_splits(a);
  const int64_t kg = (int64_t)a.N * a.P * a.Q;
  int k_per_split = (int)align_up((size_t)ceil_div(kg, splits), BK);
  const int used_splits = (int)ceil_div(kg, k_per_split);
  WsCarve wc(ws, simt_bwd_filter_ws(a));
  float *part = wc.take<float>((size_t)splits * a.K * a.C * a.R * a.S);
  float *bpart = wc.take<float>((size_t)a.K * bias_grad_chunks(a));
  SYSML_WS_FITS(wc);
  BwdFilterOp op{a, x, dy, used_splits == 1 ? df : part};
  dim3 grid((unsigned)ceil_div((int64_t)a.C * a.R * a.S, BN), (unsigned)ceil_div(a.K, BM),
            (unsigned)used_splits);
  route_note("igemm_kernel<BwdFilter> (FP32 SIMT, %d splits)", used_splits);
  igemm_kernel<BwdFilterOp><<<grid, NT, 0, st>>>(op, k_per_split);
  SYSML_LAUNCH_CHECK();
  if (used_splits > 1) {
    const int64_t n = (int64_t)a.K * a.C * a.R * a.S;
    int blocks = (int)ceil_div(n, 256);
    if (blocks > 4 * sm_count()) blocks = 4 * sm_count();
    splitk_reduce_kernel<<<blocks, 256, 0, st>>>(part, used_splits, n, df);
    SYSML_LAUNCH_CHECK();
  }
  if (db) SYSML_TRY(launch_bias_grad(a, dy, db, bpart, st));
  return SYSML_OK;
}

}  // namespace sysml
