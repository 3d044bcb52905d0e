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
// K8 csr_wgrad_k32 (C == 1, stride 1, K <= 32, 5x5 or 3x3 -- the MNIST conv1 shape):
// one CTA per SM walks a contiguous chunk of images.  A producer warp streams each
// image's dY (K planes) into shared memory with 1-D bulk async copies (double
// buffered, mbarrier completion; plane stride padded so that lane-per-filter float4
// reads are bank-conflict free).  Sixteen compute warps split the image's non-zeros
// (non-zero j -> warp j mod 16); lane k keeps dF[k][r][s] in registers and, per
// non-zero (h, w, v) and filter row r, reads the S consecutive dY values it touches
// with two float4 loads: work ~ nnz * K * R * S (sparse-safe).  db is
// summed from the staged planes.  Warp partials are combined in a fixed order and
// CTA partials reduced in a fixed order (deterministic, no float atomics).
//
// K8 csr_conv_bwd_filter (general fallback): one CTA per contiguous chunk of images.  Each image's
// dY (K x P x Q) is streamed into shared memory with 16-byte loads, the CSR row is
// staged, and every thread accumulates its own (k, r, s) outputs over the
// non-zeros in CSR order into a shared-memory dF partial (disjoint ownership, no
// atomics).  db is summed from the staged dY.  Chunk partials are reduced in a
// fixed order (deterministic).
#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"
#include "csr_dev.cuh"

#include <algorithm>

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
  // duplicates summed in stored order (reading R15; csr_dev.cuh)
  csr_scatter_row(m.col_idx, m.val, j0, j1, threadIdx.x, blockDim.x,
                  [&](int col) { return col >= 0 && col < chw ? img + col : nullptr; },
                  [](bool b) { return __syncthreads_or(b) != 0; });
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
    csr_scatter_row(m.col_idx, m.val, j0, j1, threadIdx.x, blockDim.x,
                    [&](int c) { return c >= 0 && c < m.cols ? row + c : nullptr; },
                    [](bool b) { return __syncthreads_or(b) != 0; });
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


// ---------------------------------------------------------------- K8 fast path
constexpr int WG_WARPS = 16;                    // compute warps
constexpr int WG_THREADS = (WG_WARPS + 1) * 32; // + producer warp

struct WgK32 {
  int N, K, H, W, P, Q, ph, pw;
  int stride;          // padded plane stride of the raw staging buffer (floats)
  int n_per_block;
  float invW;
};

__device__ __forceinline__ float4 lds4(const float *p) {
  return *reinterpret_cast<const float4 *>(p);
}

// Per image: the producer bulk-copies the K dY planes into `raw` (plane stride padded
// so lane-per-plane float4 reads are conflict free); the compute warps transpose raw
// into T[pos][32] (filter-contiguous: one conflict-free 128-B wavefront per position
// for lane = k) while summing db, release raw (the next image's copy then overlaps the
// compute), and accumulate dF from T.
template <int R_, int S_>
__global__ void __launch_bounds__(WG_THREADS, 1)
    csr_wgrad_k32_kernel(WgK32 g, sysml_csr m, const float *__restrict__ dy,
                         float *__restrict__ part, float *__restrict__ dbpart) {
  extern __shared__ __align__(16) float sm[];
  const int PQ = g.P * g.Q;
  float *raw = sm;                          // [K][stride]
  float *T = raw + g.K * g.stride;          // [PQ][32]
  float *wpart = sm;                        // [WG_WARPS][32][R_*S_ + 1] (after the loop)
  uint64_t *full = reinterpret_cast<uint64_t *>(T + PQ * 32);
  uint64_t *empty = full + 1;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    ptx::mbar_init(full, 1);
    ptx::mbar_init(empty, WG_WARPS);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int n0 = blockIdx.x * g.n_per_block, n1 = min(g.N, n0 + g.n_per_block);

  if (warp == WG_WARPS) {
    // ---------------- producer: one image's K dY planes per stage
    if (lane == 0) {
      uint32_t ph = 0;
      for (int n = n0; n < n1; ++n, ph ^= 1) {
        ptx::mbar_wait(empty, ph ^ 1);
        ptx::mbar_arrive_expect_tx(full, (uint32_t)(g.K * PQ * 4));
        const float *src = dy + (int64_t)n * g.K * PQ;
        for (int k = 0; k < g.K; ++k)
          ptx::bulk_g2s(raw + k * g.stride, src + (int64_t)k * PQ, (uint32_t)(PQ * 4), full);
      }
    }
    return;
  }

  // ---------------- compute warps: lane = filter k
  const int kk = lane < g.K ? lane : g.K - 1;
  float acc[R_][S_];
#pragma unroll
  for (int r = 0; r < R_; ++r)
#pragma unroll
    for (int s_ = 0; s_ < S_; ++s_) acc[r][s_] = 0.f;
  float dbacc = 0.f;
  const int ng4 = PQ / 4;
  const int q0 = warp * ng4 / WG_WARPS, q1 = (warp + 1) * ng4 / WG_WARPS;
  const int HW = g.H * g.W;
  const float *Tk = T + lane;

  // non-zero j of image n is handled by warp (j - row_ptr[n]) % WG_WARPS; lane l holds
  // the l-th of this warp's non-zeros of the round (prefetched one image ahead)
  int j0 = n0 < n1 ? __ldg(m.row_ptr + n0) : 0;
  int j1 = n0 < n1 ? __ldg(m.row_ptr + n0 + 1) : 0;
  int j2 = n0 + 1 < n1 ? __ldg(m.row_ptr + n0 + 2) : 0;
  int cur_col = -1;
  float cur_val = 0.f;
  {
    const int idx = j0 + warp + WG_WARPS * lane;
    if (n0 < n1 && idx < j1) { cur_col = __ldg(m.col_idx + idx); cur_val = __ldg(m.val + idx); }
  }
  uint32_t ph = 0;
  for (int n = n0; n < n1; ++n, ph ^= 1) {
    int nxt_col = -1;
    float nxt_val = 0.f;
    int j3 = 0;
    if (n + 1 < n1) {
      const int idx = j1 + warp + WG_WARPS * lane;
      if (idx < j2) { nxt_col = __ldg(m.col_idx + idx); nxt_val = __ldg(m.val + idx); }
      if (n + 2 < n1) j3 = __ldg(m.row_ptr + n + 3);
    }
    // T is free once every compute warp finished the previous image
    ptx::named_bar_sync(1, WG_WARPS * 32);
    ptx::mbar_wait(full, ph);
    {
      const float *plane = raw + kk * g.stride;
      for (int q = q0; q < q1; ++q) {
        const float4 e = lds4(plane + 4 * q);
        dbacc += (e.x + e.y) + (e.z + e.w);  // db[k] partial, fixed order
        float *t = T + (4 * q) * 32 + lane;
        t[0] = e.x; t[32] = e.y; t[64] = e.z; t[96] = e.w;
      }
    }
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(empty);  // raw may be refilled (next image's copy)
    ptx::named_bar_sync(1, WG_WARPS * 32);   // T complete
    const int mine = j1 - j0 > warp ? (j1 - j0 - warp + WG_WARPS - 1) / WG_WARPS : 0;
    for (int base = 0; base < mine; base += 32) {
      int bcol = cur_col;
      float bval = cur_val;
      if (base > 0) {  // rare: more than 32 * WG_WARPS non-zeros in one image
        const int idx = j0 + warp + WG_WARPS * (base + lane);
        bcol = idx < j1 ? __ldg(m.col_idx + idx) : -1;
        bval = idx < j1 ? __ldg(m.val + idx) : 0.f;
      }
      const int cnt = min(32, mine - base);
      // lane-parallel decode: code >= 0 -> interior non-zero (every tap in range) whose
      // tap (0, S_-1) reads dY position code; code <= -2 -> boundary non-zero with column
      // -2 - code; -1 -> skip
      int code = -1;
      if (bcol >= 0 && bcol < HW) {
        int h = __float2int_rz(((float)bcol + 0.5f) * g.invW);
        int w = bcol - h * g.W;
        if (w < 0) { --h; w += g.W; } else if (w >= g.W) { ++h; w -= g.W; }
        const int hp = h + g.ph, wp = w + g.pw;
        const bool interior = hp >= R_ - 1 && hp < g.P && wp >= S_ - 1 && wp < g.Q;
        code = interior ? hp * g.Q + wp - (S_ - 1) : -2 - bcol;
      }
      for (int t = 0; t < cnt; ++t) {
        const int c = __shfl_sync(0xffffffffu, code, t);
        const float v = __shfl_sync(0xffffffffu, bval, t);
        if (c >= 0) {
#pragma unroll
          for (int r = 0; r < R_; ++r) {
            const float *row = Tk + (c - r * g.Q) * 32;  // dY(p = hp - r, q = wp - (S_-1) + i)
#pragma unroll
            for (int s_ = 0; s_ < S_; ++s_) acc[r][s_] = fmaf(v, row[(S_ - 1 - s_) * 32], acc[r][s_]);
          }
          continue;
        }
        if (c == -1) continue;  // out-of-range column: ignored
        const int col = -2 - c;
        int h = __float2int_rz(((float)col + 0.5f) * g.invW);
        int w = col - h * g.W;
        if (w < 0) { --h; w += g.W; } else if (w >= g.W) { ++h; w -= g.W; }
        const int hp = h + g.ph, wp = w + g.pw;
#pragma unroll
        for (int r = 0; r < R_; ++r) {
          const int p = hp - r;
          if (p < 0 || p >= g.P) continue;
#pragma unroll
          for (int s_ = 0; s_ < S_; ++s_) {
            const int q = wp - s_;
            if (q < 0 || q >= g.Q) continue;
            acc[r][s_] = fmaf(v, Tk[(p * g.Q + q) * 32], acc[r][s_]);
          }
        }
      }
    }
    cur_col = nxt_col; cur_val = nxt_val;
    j0 = j1; j1 = j2; j2 = j3;
  }
  // combine the warps' partials in a fixed order (the staging buffers are free once
  // every compute warp is past its last image)
  ptx::named_bar_sync(1, WG_WARPS * 32);
  float *wp_ = wpart + (warp * 32 + lane) * (R_ * S_ + 1);
#pragma unroll
  for (int r = 0; r < R_; ++r)
#pragma unroll
    for (int s_ = 0; s_ < S_; ++s_) wp_[r * S_ + s_] = acc[r][s_];
  wp_[R_ * S_] = dbacc;
  ptx::named_bar_sync(1, WG_WARPS * 32);
  const int RS = R_ * S_;
  for (int i = threadIdx.x; i < g.K * (RS + 1); i += WG_WARPS * 32) {
    const int k = i / (RS + 1), e = i - k * (RS + 1);
    float t = 0.f;
    for (int w = 0; w < WG_WARPS; ++w) t += wpart[(w * 32 + k) * (RS + 1) + e];
    if (e < RS) part[(int64_t)blockIdx.x * g.K * RS + k * RS + e] = t;
    else if (dbpart) dbpart[(int64_t)blockIdx.x * g.K + k] = t;
  }
}

WgK32 wgrad_k32_plan(const ConvArgs &a, int *blocks, size_t *smem) {
  WgK32 g{};
  g.N = a.N; g.K = a.K; g.H = a.H; g.W = a.W; g.P = a.P; g.Q = a.Q; g.ph = a.ph; g.pw = a.pw;
  const int PQ = a.P * a.Q;
  int st = (PQ + 3) & ~3;
  if (((st / 4) & 1) == 0) st += 4;  // stride/4 odd: lane-per-plane float4 reads conflict free
  g.stride = st;
  g.invW = 1.0f / (float)a.W;
  const size_t bytes = sizeof(float) * ((size_t)a.K * st + (size_t)PQ * 32) + 64;
  *smem = std::max(bytes, sizeof(float) * WG_WARPS * 32 * (a.R * a.S + 1) + 64);
  int b = sm_count();
  if (b > a.N) b = a.N;
  if (b < 1) b = 1;
  g.n_per_block = (int)ceil_div(a.N, b);
  *blocks = (int)ceil_div(a.N, g.n_per_block);
  return g;
}

bool wgrad_k32_ok(const ConvArgs &a) {
  if (a.C != 1 || a.sh != 1 || a.sw != 1 || a.K > 32 || a.K < 1) return false;
  if (!((a.R == 5 && a.S == 5) || (a.R == 3 && a.S == 3))) return false;
  if ((a.P * a.Q) % 4 != 0 || a.H * a.W >= (1 << 22)) return false;
  int blocks;
  size_t smem;
  wgrad_k32_plan(a, &blocks, &smem);
  return smem <= 220 * 1024;
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
    SYSML_TRY(smem_attr(csr_fwd_pool_kernel, 96 * 1024));
    route_note("csr_fwd_pool_kernel (FP32)");
    csr_fwd_pool_kernel<<<blocks, CSR_THREADS, smem, st>>>(a, *pool, x, f, bias, pout, parg);
  } else {
    SYSML_TRY(smem_attr(csr_fwd_kernel, 96 * 1024));
    route_note("csr_fwd_kernel (FP32)");
    csr_fwd_kernel<<<blocks, CSR_THREADS, smem, st>>>(a, x, f, bias, y);
  }
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

bool csr_bwd_filter_supported(const ConvArgs &a) {
  if (wgrad_k32_ok(a)) return true;
  return (int64_t)a.K * a.P * a.Q <= BWF_MAX_DY_FLOATS &&
         (int64_t)a.K * a.C * a.R * a.S <= MAX_FILTER_FLOATS;
}

static size_t csr_bwf_part_ws(const ConvArgs &a, int blocks) {
  return align_up((size_t)blocks * a.K * a.C * a.R * a.S * sizeof(float), 256) +
         align_up((size_t)blocks * a.K * sizeof(float), 256);
}

// both routes of csr_conv_bwd_filter fit (the K32 kernel also needs a 16-byte aligned dy)
size_t csr_bwd_filter_ws(const ConvArgs &a) {
  size_t b = csr_bwf_part_ws(a, bwf_blocks(a));
  if (wgrad_k32_ok(a)) {
    int blocks;
    size_t smem;
    wgrad_k32_plan(a, &blocks, &smem);
    b = std::max(b, csr_bwf_part_ws(a, blocks));
  }
  return b;
}

sysml_status csr_conv_bwd_filter(const ConvArgs &a, const sysml_csr &x, const float *dy,
                                 float *df, float *db, void *ws, cudaStream_t st) {
  if (wgrad_k32_ok(a) && ((uintptr_t)dy & 15) == 0) {
    int blocks;
    size_t smem;
    const WgK32 g = wgrad_k32_plan(a, &blocks, &smem);
    WsCarve wc(ws, csr_bwd_filter_ws(a));
    const int64_t kcrs = (int64_t)a.K * a.R * a.S;
    float *part = wc.take<float>((size_t)blocks * kcrs);
    float *dbpart = wc.take<float>((size_t)blocks * a.K);
    SYSML_WS_FITS(wc);
    auto kern = (a.R == 5) ? csr_wgrad_k32_kernel<5, 5> : csr_wgrad_k32_kernel<3, 3>;
    SYSML_TRY(smem_attr(kern, smem));
    route_note("csr_wgrad_k32_kernel<%d,%d> (FP32, %d CTAs)", a.R, a.S, blocks);
    kern<<<blocks, WG_THREADS, smem, st>>>(g, x, dy, part, db ? dbpart : nullptr);
    SYSML_LAUNCH_CHECK();
    ordered_sum_kernel<<<(unsigned)ceil_div(kcrs, 256), 256, 0, st>>>(part, blocks, kcrs, df);
    SYSML_LAUNCH_CHECK();
    if (db) {
      ordered_sum_kernel<<<(unsigned)ceil_div(a.K, 256), 256, 0, st>>>(dbpart, blocks, a.K, db);
      SYSML_LAUNCH_CHECK();
    }
    return SYSML_OK;
  }
  const int blocks = bwf_blocks(a);
  const int npb = (int)ceil_div(a.N, blocks);
  const int used = (int)ceil_div(a.N, npb);
  WsCarve wc(ws, csr_bwd_filter_ws(a));
  const int64_t kcrs = (int64_t)a.K * a.C * a.R * a.S;
  float *part = wc.take<float>((size_t)blocks * kcrs);
  float *dbpart = wc.take<float>((size_t)blocks * a.K);
  SYSML_WS_FITS(wc);
  const size_t smem = bwf_smem(a);
  SYSML_TRY(smem_attr(csr_bwd_filter_kernel, 200 * 1024));
  route_note("csr_bwd_filter_kernel (FP32, %d CTAs)", used);
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
