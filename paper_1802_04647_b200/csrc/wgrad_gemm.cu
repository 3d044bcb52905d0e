// wgrad_gemm.cu -- K5 conv2d_backward_filter for 1x1, stride-1, unpadded convolutions
// (the ResNet bottleneck projection shape, SURVEY §8(d) cfg 4(ii)):
//
//   dF[k][c] = sum_{n,pos} dY[n][k][pos] * X[n][c][pos]        (§8(c) def. 4)
//
// is a plain GEMM whose contraction runs over positions, which are contiguous in the
// NCHW planes of both operands -- so both are K-major tcgen05 operands straight from
// HBM, moved by TMA (3-D tensor maps over (pos, channel, image), 128-byte swizzle, one
// 32-position box per stage; the image tail is zero-filled by TMA).  One CTA owns an
// output tile of 256 filters x NB channels (two M=128 accumulators, 512 TMEM columns)
// and a contiguous slice of the (image, position-block) iterations (split-K); the
// split partials are summed in a fixed order by a second kernel (deterministic).
//
// Warp roles: warp 0 = TMA producer, warp 1 = MMA issuer (TMEM owner), warps 2-5 =
// epilogue (TMEM lane quadrant = warp % 4).
#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"
#include "tma.cuh"

#include <algorithm>

namespace sysml {

namespace {

constexpr int W1_STAGES = 3;
constexpr int W1_KB = 32;  // positions per stage = one 128-byte swizzled row
constexpr int W1_THREADS = 192;

struct W1Params {
  int K, C, HW, N;
  int nblk;     // position blocks per image
  int mtiles;   // M = 128-filter tiles per CTA (1 or 2)
  int NB;       // channels per CTA tile (multiple of 16, <= 256)
  int nN, nM;   // channel tiles, filter-pair tiles
  int splits;
  int64_t iters;  // N * nblk
  float *part;    // [splits][K][C]
  float *dbpart;  // [splits][K] (channel-tile-0 CTAs; nullptr: no db)
};

__device__ __forceinline__ void named_bar_sync_epi() { ptx::named_bar_sync(1, 128); }

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  // K-major, 128-byte swizzle: 8-row atoms of 1 KB (SBO), LBO unused
  return ptx::make_desc(saddr, 16, 1024) | ((uint64_t)2 << 61);
}

__global__ void __launch_bounds__(W1_THREADS, 1)
    tc_wgrad_1x1_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, const W1Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const uint32_t a_bytes = (uint32_t)p.mtiles * 128 * 128;
  const uint32_t b_bytes = (uint32_t)p.NB * 128;
  const uint32_t stage_bytes = a_bytes + b_bytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + W1_STAGES * stage_bytes);
  uint64_t *empty = full + W1_STAGES;
  uint64_t *accf = empty + W1_STAGES;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(accf + 1);

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int z = blockIdx.x % p.splits;
  const int nt = (blockIdx.x / p.splits) % p.nN;
  const int mp = blockIdx.x / (p.splits * p.nN);
  const int k0 = mp * 256, c0 = nt * p.NB;
  const int64_t it0 = z * p.iters / p.splits, it1 = (z + 1) * p.iters / p.splits;

  const bool do_db = p.dbpart != nullptr && nt == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < W1_STAGES; ++s) {
      ptx::mbar_init(full + s, 1);
      ptx::mbar_init(empty + s, do_db ? 2 : 1);  // MMA commit (+ the db warp group)
    }
    ptx::mbar_init(accf, 1);
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
  }
  if (warp == 1) ptx::tmem_alloc(tslot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t sbase = ptx::smem_u32(smem);

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      for (int64_t it = it0; it < it1; ++it) {
        const int n = (int)(it / p.nblk), b = (int)(it - (int64_t)n * p.nblk);
        ptx::mbar_wait(empty + stage, ph ^ 1);
        ptx::mbar_arrive_expect_tx(full + stage, stage_bytes);
        const uint32_t A = sbase + stage * stage_bytes;
        ptx::tma_load_3d(A, &tmA, b * W1_KB, k0, n, ptx::smem_u32(full + stage));
        ptx::tma_load_3d(A + a_bytes, &tmB, b * W1_KB, c0, n, ptx::smem_u32(full + stage));
        if (++stage == W1_STAGES) { stage = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = ptx::make_idesc_tf32(128, p.NB);
    int stage = 0;
    uint32_t ph = 0;
    uint32_t acc = 0;
    for (int64_t it = it0; it < it1; ++it) {
      ptx::mbar_wait(full + stage, ph);
      ptx::tc_fence_after();
      const uint32_t A = sbase + stage * stage_bytes, B = A + a_bytes;
#pragma unroll
      for (int kk = 0; kk < W1_KB / 8; ++kk) {  // 8 positions = 32 bytes per MMA
        const uint64_t bd = sw128_desc(B + kk * 32);
        for (int mt = 0; mt < p.mtiles; ++mt) {
          if (ptx::elect_one())
            ptx::mma_tf32(tmem + mt * 256, sw128_desc(A + mt * 16384 + kk * 32), bd, idesc, acc);
          __syncwarp();
        }
        acc = 1;
      }
      if (ptx::elect_one()) ptx::mma_commit(empty + stage);
      __syncwarp();
      if (++stage == W1_STAGES) { stage = 0; ph ^= 1; }
    }
    if (ptx::elect_one()) ptx::mma_commit(accf);
    __syncwarp();
  } else {
    const int qd = warp & 3;
    const int et = threadIdx.x - 64;  // 0..127
    // (1) while the MMAs run: db[k] partial = row sums of the staged dY tiles (channel
    // tile 0 only; fixed order -> deterministic).  Thread et owns filter rows et and
    // et + 128 of the A tile; a swizzled 128-byte row holds 32 positions.
    float db0 = 0.f, db1 = 0.f;
    if (do_db) {
      int stage = 0;
      uint32_t ph = 0;
      for (int64_t it = it0; it < it1; ++it) {
        ptx::mbar_wait(full + stage, ph);
        {
          const float4 *row0 = reinterpret_cast<const float4 *>(smem + stage * stage_bytes + et * 128);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 v = row0[q];
            db0 += (v.x + v.y) + (v.z + v.w);
          }
          if (p.mtiles > 1) {
            const float4 *row1 = row0 + 128 * 8;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 v = row1[q];
              db1 += (v.x + v.y) + (v.z + v.w);
            }
          }
        }
        named_bar_sync_epi();
        if (et == 0) ptx::mbar_arrive(empty + stage);
        if (++stage == W1_STAGES) { stage = 0; ph ^= 1; }
      }
    }
    if (do_db) {
      float *dbp = p.dbpart + (int64_t)z * p.K;
      if (k0 + et < p.K) dbp[k0 + et] = db0;
      if (p.mtiles > 1 && k0 + 128 + et < p.K) dbp[k0 + 128 + et] = db1;
    }
    // (2) epilogue: lane = filter row of this warp's TMEM quadrant, 16 channels per load
    const bool any = it1 > it0;
    if (any) ptx::mbar_wait_sleep(accf, 0);
    ptx::tc_fence_after();
    float *part = p.part + (int64_t)z * p.K * p.C;
    for (int mt = 0; mt < p.mtiles; ++mt) {
      const int k = k0 + mt * 128 + qd * 32 + lane;
      for (int cb = 0; cb < p.NB; cb += 16) {
        float v[16];
        ptx::tmem_ld16(tmem + ((uint32_t)(qd * 32) << 16) + mt * 256 + cb, v);
        if (!any) {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = 0.f;
        }
        const int c = c0 + cb;
        if (k < p.K) {
          float *dst = part + (int64_t)k * p.C + c;
          if (c + 16 <= p.C && (p.C & 3) == 0) {
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              *reinterpret_cast<float4 *>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (c + j < p.C) dst[j] = v[j];
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// Sum of the split partials (deterministic): each float4 output is owned by a group of
// 4 lanes; lane q of the group sums splits z = q, q + 4, ... in increasing order and the
// four partial sums are combined as (s0 + s1) + (s2 + s3).  Elements [0, n) are df,
// [n, n + nb) are db (separate partial arrays).
__global__ void w1_reduce_kernel(const float *__restrict__ part, const float *__restrict__ dbpart,
                                 int parts, int64_t n, int nb, float *__restrict__ df,
                                 float *__restrict__ db) {
  const int64_t n4 = n / 4, nb4 = (nb + 3) / 4;
  const int64_t total = n4 + (dbpart ? nb4 : 0) + (n % 4 ? 1 : 0);
  const int q = threadIdx.x & 3;
  for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 2; g < total;
       g += ((int64_t)gridDim.x * blockDim.x) >> 2) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const float *src;
    int64_t stride, idx;
    int cnt;
    if (g < n4) { src = part; stride = n; idx = 4 * g; cnt = 4; }
    else if (dbpart && g < n4 + nb4) { src = dbpart; stride = nb; idx = 4 * (g - n4); cnt = (int)(nb - idx < 4 ? nb - idx : 4); }
    else { src = part; stride = n; idx = 4 * n4; cnt = (int)(n - 4 * n4); }
    for (int z = q; z < parts; z += 4) {
      const float *s = src + (int64_t)z * stride + idx;
      if (cnt == 4 && src == part && (n & 3) == 0) {  // split partials 16-byte aligned
        const float4 v = __ldg(reinterpret_cast<const float4 *>(s));
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      } else {
        acc.x += __ldg(s);
        if (cnt > 1) acc.y += __ldg(s + 1);
        if (cnt > 2) acc.z += __ldg(s + 2);
        if (cnt > 3) acc.w += __ldg(s + 3);
      }
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {  // (s0 + s1) + (s2 + s3)
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
      acc.z += __shfl_xor_sync(0xffffffffu, acc.z, off);
      acc.w += __shfl_xor_sync(0xffffffffu, acc.w, off);
    }
    if (q == 0) {
      float *dst = (src == dbpart) ? db + idx : df + idx;
      dst[0] = acc.x;
      if (cnt > 1) dst[1] = acc.y;
      if (cnt > 2) dst[2] = acc.z;
      if (cnt > 3) dst[3] = acc.w;
    }
  }
}

struct W1Plan {
  W1Params p;
  size_t smem, part_bytes, dbpart_bytes;
  int grid;
};

W1Plan plan_w1(const ConvArgs &a) {
  W1Plan pl{};
  W1Params &p = pl.p;
  p.K = a.K; p.C = a.C; p.HW = a.H * a.W; p.N = a.N;
  p.nblk = (int)ceil_div(p.HW, W1_KB);
  p.mtiles = a.K > 128 ? 2 : 1;
  p.nM = (int)ceil_div(a.K, 256);
  p.NB = a.C >= 256 ? 256 : std::max(16, (int)((a.C + 15) / 16 * 16));
  p.nN = (int)ceil_div(a.C, p.NB);
  p.iters = (int64_t)a.N * p.nblk;
  const int tiles = p.nM * p.nN;
  int splits = std::max(1, sm_count() / tiles);
  if (splits > p.iters) splits = (int)p.iters;
  p.splits = splits;
  pl.grid = tiles * splits;
  const size_t stage = (size_t)p.mtiles * 128 * 128 + (size_t)p.NB * 128;
  pl.smem = 1024 + W1_STAGES * stage + 8 * (2 * W1_STAGES + 1) + 16;
  pl.part_bytes = align_up((size_t)splits * a.K * a.C * sizeof(float), 256);
  pl.dbpart_bytes = align_up((size_t)splits * a.K * sizeof(float), 256);
  return pl;
}

}  // namespace

bool tc_wgrad_1x1_supported(const ConvArgs &a) {
  if (device_cc_major() != 10) return false;
  if (a.R != 1 || a.S != 1 || a.ph != 0 || a.pw != 0 || a.sh != 1 || a.sw != 1) return false;
  if ((a.H * a.W) % 4 != 0 || a.C < 16 || a.K < 16) return false;
  return plan_w1(a).smem <= 227 * 1024;
}

size_t tc_wgrad_1x1_ws(const ConvArgs &a) {
  const W1Plan pl = plan_w1(a);
  return pl.part_bytes + pl.dbpart_bytes;
}

sysml_status tc_wgrad_1x1(const ConvArgs &a, const float *x, const float *dy, float *df,
                          float *db, void *ws, cudaStream_t st) {
  if (((uintptr_t)x & 15) || ((uintptr_t)dy & 15)) {
    set_error("tcgen05 1x1 bwd_filter: x / dy must be 16-byte aligned");
    return SYSML_ERR_UNSUPPORTED;
  }
  W1Plan pl = plan_w1(a);
  W1Params p = pl.p;
  p.part = reinterpret_cast<float *>(ws);
  p.dbpart = db ? reinterpret_cast<float *>(reinterpret_cast<char *>(ws) + pl.part_bytes) : nullptr;
  CUtensorMap tmA, tmB;
  const uint64_t hw = (uint64_t)p.HW;
  {
    const uint64_t dims[3] = {hw, (uint64_t)a.K, (uint64_t)a.N};
    const uint64_t strides[2] = {hw * 4, hw * 4 * a.K};
    const uint32_t box[3] = {W1_KB, (uint32_t)(p.mtiles * 128), 1};
    if (!tmap_encode_f32(&tmA, dy, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return SYSML_ERR_CUDA;
  }
  {
    const uint64_t dims[3] = {hw, (uint64_t)a.C, (uint64_t)a.N};
    const uint64_t strides[2] = {hw * 4, hw * 4 * a.C};
    const uint32_t box[3] = {W1_KB, (uint32_t)p.NB, 1};
    if (!tmap_encode_f32(&tmB, x, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return SYSML_ERR_CUDA;
  }
  SYSML_TRY(smem_attr(tc_wgrad_1x1_kernel, pl.smem));
  route_note("tc_wgrad_1x1_kernel [TMA + tcgen05 TF32, %d CTAs]", pl.grid);
  tc_wgrad_1x1_kernel<<<pl.grid, W1_THREADS, pl.smem, st>>>(tmA, tmB, p);
  SYSML_LAUNCH_CHECK();
  const int64_t total = (int64_t)a.K * a.C;
  const int64_t groups = total / 4 + (db ? (a.K + 3) / 4 : 0) + 1;
  w1_reduce_kernel<<<(unsigned)std::min<int64_t>(ceil_div(groups * 4, 256), 16 * sm_count()), 256, 0,
                     st>>>(p.part, db ? p.dbpart : nullptr, p.splits, total, a.K, df, db);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

}  // namespace sysml
