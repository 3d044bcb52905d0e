// affine_gemm.cu -- the affine (fully connected) layers of the LeNet-512 step (NEXT-4;
// S:236-243 affine_forward/backward; SystemML mnist_lenet topology, R22-R24):
//
//   tc_gemm_kernel   C[M][N] = A[M][K] . B[N][K]^T on tcgen05 (TF32, fp32 accumulate), both
//                    operands K-major straight from HBM by TMA (2-D tensor maps, 128-byte
//                    swizzle, 32-float K boxes), with a fused epilogue: + bias[col], relu and
//                    inverted dropout (Philox4x64-10 mask, reading R23), or a plain store.
//                    Used for z3 -> h = dropout(relu(a2 W3^T + b3)) and da2 = dz3 W3.
//   transpose        row-major [R][C] -> [C][ldo] with zero columns [R, ldo) (for the
//                    contractions over the batch, which need the batch contiguous: dW3).
//   dz3 kernel       dh = ds W4, dz3 = dh * [h > 0] / keep_p  (dropout + relu backward, S:279,
//                    S:300), written both [n][512] (da2 GEMM) and [512][n] (dW3 GEMM).
//   bias/relu/dropout elementwise (FP32 path) and the pool2 routing of a materialised da2
//   into the dz2 SPF planes (TF32 path).
//
// tc_gemm_kernel is persistent with two TMEM accumulators (the epilogue of one tile overlaps
// the MMAs of the next); warp roles at the kernel.
#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"
#include "tma.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace sysml {

// Philox4x64-10 (Salmon et al. SC'11) in numpy.random.Philox's output order: raw output e of
// key (k0, k1) is word e % 4 of the block for counter (e / 4 + 1, 0, 0, 0).  DESIGN.md R23.
__device__ __forceinline__ void philox4x64_10(uint64_t c0, uint64_t k0, uint64_t k1, uint64_t (&w)[4]) {
  uint64_t c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    const uint64_t hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0), lo0 = 0xD2E7470EE14C6C93ULL * c0;
    const uint64_t hi1 = __umul64hi(0xCA5A826395121157ULL, c2), lo1 = 0xCA5A826395121157ULL * c2;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  w[0] = c0; w[1] = c1; w[2] = c2; w[3] = c3;
}

// keep bits of the 4 units e0 .. e0+3 (e0 % 4 == 0) of the mask stream (seed, step)
__device__ __forceinline__ uint32_t dropout_keep4(uint64_t e0, uint64_t seed, uint64_t step, uint64_t T) {
  uint64_t w[4];
  philox4x64_10(e0 / 4 + 1, seed, step, w);
  return ((w[0] >> 32) < T ? 1u : 0u) | ((w[1] >> 32) < T ? 2u : 0u) | ((w[2] >> 32) < T ? 4u : 0u) |
         ((w[3] >> 32) < T ? 8u : 0u);
}

namespace {

constexpr int G_KB = 32;        // K floats per stage = one 128-byte swizzled row
constexpr int G_EPI_WARPS = 8;  // two per TMEM lane quadrant, each owning half the tile columns
constexpr int G_THREADS = 64 + 32 * G_EPI_WARPS;

struct GParams {
  int M, N, K;
  int NB, nN, tiles;
  int64_t ldc;
  float *C;
  GemmEpi e;
};

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return ptx::make_desc(saddr, 16, 1024) | ((uint64_t)2 << 61);
}

// Persistent GEMM: CTA b takes output tiles b, b + grid, ... (128 x NB each, n fastest so
// concurrently running CTAs share A rows in L2).  Warp 0 = TMA producer over a STAGES-deep
// ring, warp 1 = MMA issuer into one of two TMEM accumulators (NB columns each), warps 2..9 =
// epilogue, which drains tile t from one accumulator while the MMAs of tile t+1 fill the
// other.  With the dropout epilogue, the epilogue threads draw the Philox mask bits of their
// next tile (row m, 128 or fewer units: <= 4 words of keep bits) while they wait for its
// accumulator -- the generator cost is hidden under the MMAs.
template <int STAGES>
__global__ void __launch_bounds__(G_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const uint32_t a_bytes = 128 * 128;
  const uint32_t b_bytes = (uint32_t)p.NB * 128;
  const uint32_t stage_bytes = a_bytes + b_bytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * stage_bytes);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + STAGES;  // [2] accumulator ready (MMA commit)
  uint64_t *tempty = tfull + 2;      // [2] accumulator drained (one arrive per epilogue warp)
  uint32_t *tslot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int kiters = (p.K + G_KB - 1) / G_KB;
  const uint32_t ncols = 2 * p.NB <= 64 ? 64 : 2 * p.NB <= 128 ? 128 : 2 * p.NB <= 256 ? 256 : 512;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(full + s, 1);
      ptx::mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(tfull + b, 1);
      ptx::mbar_init(tempty + b, G_EPI_WARPS);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
  }
  if (warp == 1) ptx::tmem_alloc(tslot, ncols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t sbase = ptx::smem_u32(smem);

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
        const int m0 = (t / p.nN) * 128, n0 = (t % p.nN) * p.NB;
        for (int it = 0; it < kiters; ++it) {
          ptx::mbar_wait(empty + stage, ph ^ 1);
          ptx::mbar_arrive_expect_tx(full + stage, stage_bytes);
          const uint32_t A = sbase + stage * stage_bytes;
          ptx::tma_load_2d(A, &tmA, it * G_KB, m0, ptx::smem_u32(full + stage));
          ptx::tma_load_2d(A + a_bytes, &tmB, it * G_KB, n0, ptx::smem_u32(full + stage));
          if (++stage == STAGES) { stage = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = ptx::make_idesc_tf32(128, p.NB);
    const uint64_t d0 = sw128_desc(sbase);
    const uint64_t stage_d = stage_bytes >> 4, b_d = a_bytes >> 4;
    int stage = 0;
    uint32_t ph = 0;
    int buf = 0;
    uint32_t tph = 0;  // bit b = phase of accumulator b
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      ptx::mbar_wait(tempty + buf, ((tph >> buf) & 1u) ^ 1u);  // the epilogue drained this accumulator
      tph ^= 1u << buf;
      ptx::tc_fence_after();
      const uint32_t tacc = tmem + (uint32_t)(buf * p.NB);
      uint32_t acc = 0;
      for (int it = 0; it < kiters; ++it) {
        ptx::mbar_wait(full + stage, ph);
        ptx::tc_fence_after();
        const uint64_t ad = d0 + (uint64_t)stage * stage_d;
#pragma unroll
        for (int kk = 0; kk < G_KB / 8; ++kk) {  // 8 floats = 32 bytes = 2 descriptor units
          if (ptx::elect_one()) ptx::mma_tf32(tacc, ad + 2 * kk, ad + b_d + 2 * kk, idesc, acc);
          __syncwarp();
          acc = 1;
        }
        if (ptx::elect_one()) ptx::mma_commit(empty + stage);
        __syncwarp();
        if (++stage == STAGES) { stage = 0; ph ^= 1; }
      }
      if (ptx::elect_one()) ptx::mma_commit(tfull + buf);
      __syncwarp();
      buf ^= 1;
    }
  } else {
    const int ew = warp - 2, qd = warp & 3, half = ew >> 2;  // lane quadrant, column half
    const GemmEpi &e = p.e;
    const uint64_t step = e.dropout ? *e.step : 0;
    const int hc = p.NB / 2;  // columns per epilogue warp (multiple of 16 when NB % 32 == 0)
    int buf = 0;
    uint32_t tph = 0;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      const int m = (t / p.nN) * 128 + qd * 32 + lane;
      const int cbase = (t % p.nN) * p.NB + half * hc;
      // keep bits of this thread's row and column range, drawn while the MMAs run
      // (hc <= 128 columns -> 4 words, kept in scalars so nothing goes to local memory)
      uint32_t k0 = 0, k1 = 0, k2 = 0, k3 = 0;
      if (e.dropout && m < p.M) {
        const uint64_t e0 = (uint64_t)(e.row0 + m) * (uint64_t)e.units;
#pragma unroll 1
        for (int c4 = 0; c4 < hc && cbase + c4 < p.N; c4 += 4) {
          const uint32_t b = dropout_keep4(e0 + (uint64_t)(cbase + c4), e.seed, step, e.keep_T) << (c4 & 31);
          const int w = c4 >> 5;
          k0 |= w == 0 ? b : 0u; k1 |= w == 1 ? b : 0u; k2 |= w == 2 ? b : 0u; k3 |= w == 3 ? b : 0u;
        }
      }
      ptx::mbar_wait_sleep(tfull + buf, (tph >> buf) & 1u);
      tph ^= 1u << buf;
      ptx::tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(buf * p.NB + half * hc);
      for (int cb = 0; cb < hc; cb += 16) {
        float v[16];
        ptx::tmem_ld16(tbase + (uint32_t)cb, v);
        const int c = cbase + cb;
        __syncwarp();
        if (m < p.M && c < p.N) {
          if (kiters == 0) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0.f;
          }
          if (e.bias) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] += c + j < p.N ? __ldg(e.bias + c + j) : 0.f;
          }
          if (e.relu) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = v[j] > 0.f ? v[j] : 0.f;  // R7: +0.0
          }
          if (e.dropout) {  // inverted dropout (R23, R24)
            const int w = cb >> 5;
            const uint32_t kb = (w == 0 ? k0 : w == 1 ? k1 : w == 2 ? k2 : k3) >> (cb & 31);
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = (kb >> j) & 1u ? __fdiv_rn(v[j], e.keep_p) : 0.f;
          }
          float *dst = p.C + (int64_t)m * p.ldc + c;
          if (c + 16 <= p.N && (p.ldc & 3) == 0) {
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              *reinterpret_cast<float4 *>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (c + j < p.N) dst[j] = v[j];
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(tempty + buf);
      buf ^= 1;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, ncols);
  }
}

struct GPlan {
  int NB, nN, nM, stages, grid;
  size_t smem;
};

GPlan plan_gemm(int M, int N) {
  // 128 x NB tiles, NB <= 256 (two NB-column accumulators fill TMEM), persistent grid
  GPlan pl{};
  static const char *nb_env = getenv("SYSML_GEMM_NB");  // A/B measurement
  int nb = 256;
  if (nb_env && atoi(nb_env) >= 32 && atoi(nb_env) <= 256) nb = atoi(nb_env) / 32 * 32;
  nb = std::min(nb, (int)ceil_div(N, 32) * 32);
  pl.NB = nb;
  pl.nN = (int)ceil_div(N, nb);
  pl.nM = (int)ceil_div(M, 128);
  pl.grid = (int)std::min<int64_t>((int64_t)pl.nN * pl.nM, sm_count());
  const size_t stage = (size_t)128 * 128 + (size_t)nb * 128;
  static const int stages_env = getenv("SYSML_GEMM_STAGES") ? atoi(getenv("SYSML_GEMM_STAGES")) : 0;
  pl.stages = stage * 4 + 2048 <= 200 * 1024 ? 4 : 3;
  if (stages_env >= 2 && stages_env <= 4 && stage * stages_env + 2048 <= 220 * 1024) pl.stages = stages_env;
  pl.smem = 1024 + pl.stages * stage + 8 * (2 * pl.stages + 4) + 16;
  return pl;
}

}  // namespace

bool tc_gemm_supported(int M, int N, int K, int64_t lda, int64_t ldb) {
  if (device_cc_major() != 10) return false;
  return M >= 1 && N >= 16 && K >= 1 && (K % 4) == 0 && (lda % 4) == 0 && (ldb % 4) == 0 &&
         lda >= K && ldb >= K;
}

sysml_status tc_gemm(int M, int N, int K, const float *A, int64_t lda, const float *B, int64_t ldb,
                     float *C, int64_t ldc, const GemmEpi &e, cudaStream_t st) {
  if (((uintptr_t)A & 15) || ((uintptr_t)B & 15)) {
    set_error("tcgen05 GEMM: A / B must be 16-byte aligned");
    return SYSML_ERR_UNSUPPORTED;
  }
  if (!tc_gemm_supported(M, N, K, lda, ldb)) {
    set_error("tcgen05 GEMM: unsupported shape M=%d N=%d K=%d lda=%lld ldb=%lld", M, N, K,
              (long long)lda, (long long)ldb);
    return SYSML_ERR_UNSUPPORTED;
  }
  if (e.dropout && (e.units % 4 != 0 || N % 4 != 0)) {
    set_error("tcgen05 GEMM dropout epilogue needs units %% 4 == 0");
    return SYSML_ERR_UNSUPPORTED;
  }
  const GPlan pl = plan_gemm(M, N);
  GParams p{M, N, K, pl.NB, pl.nN, pl.nN * pl.nM, ldc, C, e};
  CUtensorMap tmA, tmB;
  {
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)M};
    const uint64_t strides[1] = {(uint64_t)lda * 4};
    const uint32_t box[2] = {G_KB, 128};
    if (!tmap_encode_f32(&tmA, A, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return SYSML_ERR_CUDA;
  }
  {
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)N};
    const uint64_t strides[1] = {(uint64_t)ldb * 4};
    const uint32_t box[2] = {G_KB, (uint32_t)pl.NB};
    if (!tmap_encode_f32(&tmB, B, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return SYSML_ERR_CUDA;
  }
  route_note("tc_gemm_kernel [TMA + tcgen05 TF32, persistent, 128x%d tiles x %d on %d CTAs%s]", pl.NB,
             p.tiles, pl.grid, e.dropout ? ", bias+relu+dropout epilogue" : "");
  if (pl.stages == 4) {
    SYSML_TRY(smem_attr(tc_gemm_kernel<4>, pl.smem));
    tc_gemm_kernel<4><<<pl.grid, G_THREADS, pl.smem, st>>>(tmA, tmB, p);
  } else if (pl.stages == 2) {
    SYSML_TRY(smem_attr(tc_gemm_kernel<2>, pl.smem));
    tc_gemm_kernel<2><<<pl.grid, G_THREADS, pl.smem, st>>>(tmA, tmB, p);
  } else {
    SYSML_TRY(smem_attr(tc_gemm_kernel<3>, pl.smem));
    tc_gemm_kernel<3><<<pl.grid, G_THREADS, pl.smem, st>>>(tmA, tmB, p);
  }
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

// ---------------------------------------------------------------------------------------
namespace {

// out[c][r] = in[r][c] for r < R, 0 for R <= r < ldo (32 x 32 tiles through shared memory)
__global__ void __launch_bounds__(256) transpose_kernel(const float *__restrict__ in, int R, int Cc,
                                                        int64_t ldi, float *__restrict__ out, int64_t ldo) {
  __shared__ float t[32][33];
  const int r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int i = ty; i < 32; i += 8) {
    const int r = r0 + i, c = c0 + tx;
    t[i][tx] = (r < R && c < Cc) ? __ldcs(in + (int64_t)r * ldi + c) : 0.f;
  }
  __syncthreads();
#pragma unroll
  for (int i = ty; i < 32; i += 8) {
    const int c = c0 + i, r = r0 + tx;
    if (c < Cc && r < ldo) out[(int64_t)c * ldo + r] = t[tx][i];
  }
}

// dz3 = (ds W4) * [h > 0] / keep_p: block = 32 samples x 32 units (256 threads); writes dz3
// [n][H] (lane = unit) and dz3T [H][ldt] (lane = sample), zeros in columns [n, ldt).
template <int NC>
__global__ void __launch_bounds__(256) dz3_kernel(int n, int H, const float *__restrict__ ds,
                                                  const float *__restrict__ W4, const float *__restrict__ h,
                                                  float keep_p, float *__restrict__ dz3,
                                                  float *__restrict__ dz3T, int64_t ldt) {
  __shared__ float t[32][33];
  __shared__ float w[NC][32];
  __shared__ float dsv[32][NC];
  const int s0 = blockIdx.x * 32, u0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < NC * 32; i += 256) w[i / 32][i % 32] = __ldg(W4 + (int64_t)(i / 32) * H + u0 + i % 32);
  for (int i = threadIdx.x; i < 32 * NC; i += 256) {
    const int s = s0 + i / NC;
    dsv[i / NC][i % NC] = s < n ? __ldg(ds + (int64_t)s * NC + i % NC) : 0.f;
  }
  __syncthreads();
#pragma unroll
  for (int i = ty; i < 32; i += 8) {
    const int s = s0 + i, u = u0 + tx;
    float g = 0.f;
    if (s < n) {
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < NC; ++j) acc = fmaf(dsv[i][j], w[j][tx], acc);
      const float hv = __ldg(h + (int64_t)s * H + u);
      g = hv > 0.f ? __fdiv_rn(acc, keep_p) : 0.f;  // dropout and relu' backward
      dz3[(int64_t)s * H + u] = g;
    }
    t[i][tx] = g;
  }
  __syncthreads();
#pragma unroll
  for (int i = ty; i < 32; i += 8) {
    const int u = u0 + i, s = s0 + tx;
    if (s < ldt) dz3T[(int64_t)u * ldt + s] = t[tx][i];
  }
}

// FP32 path: h = dropout(relu(z)) in place (bias already added by the conv)
__global__ void relu_dropout_kernel(float *__restrict__ z, int n, int H, int64_t row0, uint64_t seed,
                                    const uint64_t *__restrict__ stepp, uint64_t T, float keep_p, int dropout) {
  const int64_t total4 = (int64_t)n * H / 4;
  const uint64_t step = dropout ? *stepp : 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = reinterpret_cast<float4 *>(z)[i];
    float a[4] = {v.x, v.y, v.z, v.w};
    const int64_t s = (4 * i) / H, u = 4 * i - s * H;
    uint32_t keep = 15u;
    if (dropout) keep = dropout_keep4((uint64_t)(row0 + s) * (uint64_t)H + (uint64_t)u, seed, step, T);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float r = a[j] > 0.f ? a[j] : 0.f;
      a[j] = dropout ? ((keep >> j) & 1u ? __fdiv_rn(r, keep_p) : 0.f) : r;
    }
    reinterpret_cast<float4 *>(z)[i] = make_float4(a[0], a[1], a[2], a[3]);
  }
}

__global__ void counter_inc_kernel(uint64_t *c) { *c += 1; }

// B2p from a materialised da2 (TF32 LeNet-512 path): the masked max-pool routing of
// affine_bwd_route_spf_kernel (lenet.cu) with g = da2[s][d] read instead of computed.
constexpr int RT_IMGS = 32;
__global__ void __launch_bounds__(256) route_da2_spf_kernel(int n, const float *__restrict__ da2,
                                                            const uint64_t *__restrict__ c2, int64_t cplane,
                                                            float *__restrict__ dz2s, int64_t plane,
                                                            float *__restrict__ dbpart) {
  constexpr int D3 = 3136;
  const int d = blockIdx.x * 256 + threadIdx.x;  // = k*49 + pp*7 + pc
  const int s0 = blockIdx.y * RT_IMGS, s1 = min(n, s0 + RT_IMGS);
  if (d >= D3) return;
  const int k = d / 49, r = d - k * 49, pp = r / 7, pc = r - pp * 7;
  const unsigned long long *cw = reinterpret_cast<const unsigned long long *>(c2) + (int64_t)(k >> 4) * cplane + r;
  const int sh = 4 * (k & 15);
  float *base = dz2s + (int64_t)k * plane + (2 * pp) * 16 + 2 * pc;
  float gsum = 0.f;
  for (int sb = s0; sb < s1; sb += 4) {
    uint32_t cd[4];
    float gv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      cd[u] = sb + u < s1 ? (uint32_t)(__ldg(cw + (int64_t)(sb + u) * 49) >> sh) & 15u : 0u;
      gv[u] = sb + u < s1 ? __ldcs(da2 + (int64_t)(sb + u) * D3 + d) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int s = sb + u;
      if (s >= s1) break;
      const float g = (cd[u] & 4u) ? gv[u] : 0.f;  // window code: positive*4 + dr*2 + ds (R9)
      gsum += g;
      const uint32_t wp = cd[u] & 3u;
      float *bs = base + (int64_t)s * 256;
      __stcs(reinterpret_cast<float2 *>(bs), make_float2(wp == 0 ? g : 0.f, wp == 1 ? g : 0.f));
      __stcs(reinterpret_cast<float2 *>(bs + 16), make_float2(wp == 2 ? g : 0.f, wp == 3 ? g : 0.f));
      if (pc == 6) {
        __stcs(reinterpret_cast<float2 *>(bs + 2), make_float2(0.f, 0.f));
        __stcs(reinterpret_cast<float2 *>(bs + 18), make_float2(0.f, 0.f));
      }
    }
  }
  dbpart[(int64_t)blockIdx.y * D3 + d] = gsum;
}

}  // namespace

sysml_status launch_transpose(const float *in, int R, int Cc, int64_t ldi, float *out, int64_t ldo,
                              cudaStream_t st) {
  if (R <= 0 || Cc <= 0) return SYSML_OK;
  dim3 grid((unsigned)ceil_div(std::max<int64_t>(R, ldo), 32), (unsigned)ceil_div(Cc, 32));
  transpose_kernel<<<grid, 256, 0, st>>>(in, R, Cc, ldi, out, ldo);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status launch_dz3(int n, int H, const float *ds, const float *W4, const float *h, float keep_p,
                        float *dz3, float *dz3T, int64_t ldt, cudaStream_t st) {
  if (H % 32 != 0) {
    set_error("dz3: hidden width %d must be a multiple of 32", H);
    return SYSML_ERR_UNSUPPORTED;
  }
  dim3 grid((unsigned)ceil_div(std::max<int64_t>(n, ldt), 32), (unsigned)(H / 32));
  dz3_kernel<10><<<grid, 256, 0, st>>>(n, H, ds, W4, h, keep_p, dz3, dz3T, ldt);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status launch_relu_dropout(float *z, int n, int H, int64_t row0, uint64_t seed, const uint64_t *step,
                                 uint64_t T, float keep_p, int dropout, cudaStream_t st) {
  const int64_t total4 = (int64_t)n * H / 4;
  if (total4 == 0) return SYSML_OK;
  relu_dropout_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total4, 256), 8 * sm_count()), 256, 0, st>>>(
      z, n, H, row0, seed, step, T, keep_p, dropout);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

sysml_status launch_counter_inc(uint64_t *c, cudaStream_t st) {
  counter_inc_kernel<<<1, 1, 0, st>>>(c);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

int route_da2_chunks(int n) { return (int)ceil_div(n, RT_IMGS); }

sysml_status launch_route_da2_spf(int n, const float *da2, const uint64_t *c2, int64_t cplane, float *dz2s,
                                  int64_t plane, float *dbpart, cudaStream_t st) {
  route_da2_spf_kernel<<<dim3((unsigned)ceil_div(3136, 256), (unsigned)ceil_div(n, RT_IMGS)), 256, 0, st>>>(
      n, da2, c2, cplane, dz2s, plane, dbpart);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

}  // namespace sysml
