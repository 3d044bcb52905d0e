// pair_conv.cu -- stride-1 dense conv2d forward and bwd_data (A1 / A7) on
// CTA pairs: tcgen05 kind::tf32 with cta_group::2 (M = 256), for wide filter banks (the output
// channel count a multiple of 256: the ResNet-50 3x3 C = K = 256 and 1x1 1024 <-> 256 layers).
//
// Why: the single-CTA forward kernel (conv_tc.cu, K3) runs these layers at N = 256 with two
// M-tiles per CTA sharing each filter chunk; per N = 256 MMA it reads a 4 KB A tile and an 8 KB B
// tile from shared memory and bulk-writes 4 KB more of B, ~170 clocks against 128 of math (ncu /
// SYSML_TC_PROFILE: 3x3 C = K = 256 at 52% of the TF32 peak).  Here a cluster of two CTAs issues
// M = 256 MMAs: CTA rank h stages the A rows of its own 128 frame positions and HALF of every
// filter chunk (output channels [128h, 128h + 128) of the 256-wide tile), at the same
// shared-memory offsets.  Per MMA each CTA reads 4 KB of A + 4 KB of B and bulk-loads 2 KB of B:
// the loop is math bound, and the filter stream from L2 halves.
//
// GEMM (shifted-window implicit GEMM, as K3): frame of Wf = W + pw columns and
// Hs = H + ph rows per image (the right / bottom padding of one row / image is the left / top
// padding of the next); output frame position g, tap (r, s) reads input frame position
// g + r*Wf + s; D[g][k] += sum_c A[g + r*Wf + s][c] * B[k][(c, r, s)].  A: 8-channel halo of
// HALO = 128 + (R-1)*Wf + S-1 positions, K-major no-swizzle [quad][position][4 ch], gathered by
// 4-byte cp.async (zero fill = padding); B: packed [tap][quad][128 k][4 c] per CTA half.
//
// Work unit = (pair tile of 256 frame positions, 256-wide filter tile).  Warps: 0-3 producers,
// 4 MMA issuer (rank 0) / completion relay (rank 1: forwards its stage-full events to rank 0),
// 5-12 epilogue (quadrant = warp % 4, column half = (warp - 5) / 4): + bias, NCHW stores.
// TMEM: two 256-column accumulators per CTA (the epilogue of unit i overlaps the MMAs of i + 1).
#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace sysml {

namespace {

constexpr int PC_THREADS = 32 * (4 + 1 + 8);
constexpr int PC_MAXHALO = 384;
constexpr int PC_MAXNS = 8;

struct PcParams {
  const float *x;     // input NCHW [N][Cin][H][W]
  const float *fp;    // packed filters [nft][nchunk][2 halves][RS][2 quads][128][4]
  const float *bias;  // [Kout] or null
  float *y;           // output NCHW [N][Kout][P][Q]
  int N, Cin, H, W, Kout, R, S, ph, pw, P, Q;
  int Wf, Hs, Lf;
  int64_t G;          // N * Lf frame positions
  int64_t npt, nunits;
  int nft, nchunk, RS, HALO, ns;
  int NT;             // output channels per unit (256 or 128): NT / 2 per CTA
  uint32_t a_bytes, b_bytes, stage_bytes;
  long long *clk;
};

__device__ __forceinline__ void mma_pair_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_mc2(uint64_t *bar) {  // arrives on `bar` in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          ptx::smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void arrive_rank0_pc(uint64_t *bar) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(ra) : "r"(ptx::smem_u32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void wait_cluster_pc(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(ptx::smem_u32(bar)), "r"(parity)
        : "memory");
}

__global__ void __launch_bounds__(PC_THREADS, 1) pair_conv_kernel(const PcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *stages = smem;
  int *src_off = reinterpret_cast<int *>(smem + (size_t)p.ns * p.stage_bytes);  // [PC_MAXHALO]
  uint64_t *bars = reinterpret_cast<uint64_t *>(src_off + PC_MAXHALO);
  uint64_t *full = bars;                  // [ns] local: 128 cp.async arrivals + the B expect_tx
  uint64_t *pfull = full + PC_MAXNS;      // [ns] rank 0: rank 1's stage is full (relay)
  uint64_t *empty = pfull + PC_MAXNS;     // [ns] multicast commit
  uint64_t *accf = empty + PC_MAXNS;      // [2] multicast commit
  uint64_t *acce = accf + 2;              // [2] rank 0: the 16 epilogue warps of the pair
  uint32_t *tslot = reinterpret_cast<uint32_t *>(acce + 2);

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.ns; ++s) {
      ptx::mbar_init(full + s, 128 + 1);
      ptx::mbar_init(pfull + s, 1);
      ptx::mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(accf + b, 1);
      ptx::mbar_init(acce + b, 16);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(tslot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // both CTAs' barriers initialised before any remote arrive
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t rank = ptx::cluster_ctarank();
  const int64_t cid = blockIdx.x / 2, ncl = gridDim.x / 2;
  const int HW = p.H * p.W;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // packed filters ready (PDL)

  if (warp < 4) {
    // ================= producers: per unit, the src_off table of this CTA's halo, then per
    // chunk one bulk copy of this CTA's B half and 8 x 4-byte cp.async per halo position
    const int tid = threadIdx.x;
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t u = cid; u < p.nunits; u += ncl) {
      const int64_t pt = u / p.nft;
      const int ft = (int)(u - pt * p.nft);
      const int64_t g0 = pt * 256 + (int64_t)rank * 128;
      ptx::named_bar_sync(1, 128);  // every producer is done with the previous table
      for (int pos = tid; pos < p.HALO; pos += 128) {
        const int64_t q = g0 + pos;
        int off = -1;
        if (q < p.G) {
          const int n = (int)(q / p.Lf);
          const int rem = (int)(q - (int64_t)n * p.Lf);
          const int row = rem / p.Wf, col = rem - row * p.Wf;
          const int h = row - p.ph, w = col - p.pw;
          if (h >= 0 && h < p.H && w >= 0 && w < p.W) off = n * p.Cin * HW + h * p.W + w;
        }
        src_off[pos] = off;
      }
      ptx::named_bar_sync(1, 128);
      for (int ch = 0; ch < p.nchunk; ++ch) {
        ptx::mbar_wait(empty + stage, phase ^ 1);
        uint8_t *A = stages + (size_t)stage * p.stage_bytes;
        uint8_t *B = A + p.a_bytes;
        if (tid == 0) {
          ptx::mbar_arrive_expect_tx(full + stage, p.b_bytes);
          const float *bsrc = p.fp + (((size_t)ft * p.nchunk + ch) * 2 + rank) * (p.b_bytes / 4);
          ptx::bulk_g2s(B, bsrc, p.b_bytes, full + stage);
        }
        const uint32_t a0 = ptx::smem_u32(A), a1 = a0 + (uint32_t)p.HALO * 16;
        const float *xc = p.x + (int64_t)(ch * 8) * HW;
        for (int pos = tid; pos < p.HALO; pos += 128) {
          const int off = src_off[pos];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const bool ok = off >= 0;
            ptx::cp_async4((j < 4 ? a0 : a1) + pos * 16 + (j & 3) * 4, ok ? xc + off + j * HW : p.x, ok ? 4u : 0u);
          }
        }
        ptx::cp_async_mbar_arrive(full + stage);
        if (++stage == p.ns) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 4) {
    if (rank == 0) {
      // ================= MMA issuer: one elected lane per chunk (RS pair MMAs + the commit)
      const uint32_t idesc = ptx::make_idesc_tf32(256, p.NT);
      const uint32_t brow = (uint32_t)p.NT / 2;  // B rows per CTA and tap
      int stage = 0;
      uint32_t phase = 0, tcount = 0;
      const uint32_t sbase = ptx::smem_u32(stages);
      long long t_w = 0;
      const long long t_s = clock64();
      for (int64_t u = cid; u < p.nunits; u += ncl, ++tcount) {
        const uint32_t buf = tcount & 1u, bph = (tcount >> 1) & 1u;
        wait_cluster_pc(acce + buf, bph ^ 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem + buf * 256;  // NT <= 256 columns per buffer
        for (int ch = 0; ch < p.nchunk; ++ch) {
          const long long t0 = p.clk ? clock64() : 0;
          ptx::mbar_wait(full + stage, phase);
          wait_cluster_pc(pfull + stage, phase);
          if (p.clk) t_w += clock64() - t0;
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            const uint32_t A = sbase + (uint32_t)stage * p.stage_bytes, B = A + p.a_bytes;
            for (int tap = 0; tap < p.RS; ++tap) {
              const int r = tap / p.S, s_ = tap - r * p.S;
              const uint64_t ad = ptx::make_desc(A + (uint32_t)(r * p.Wf + s_) * 16u, (uint32_t)p.HALO * 16u, 128);
              const uint64_t bd = ptx::make_desc(B + (uint32_t)tap * brow * 32u, brow * 16u, 128);
              mma_pair_ss(d, ad, bd, idesc, (ch | tap) ? 1u : 0u);
            }
            commit_mc2(empty + stage);
          }
          __syncwarp();
          if (++stage == p.ns) { stage = 0; phase ^= 1; }
        }
        if (ptx::elect_one()) commit_mc2(accf + buf);
        __syncwarp();
      }
      if (p.clk && lane == 0) {
        p.clk[blockIdx.x * 2 + 0] = t_w;
        p.clk[blockIdx.x * 2 + 1] = clock64() - t_s;
      }
    } else if (lane == 0) {
      // ================= relay (rank 1): this CTA's stage is full -> tell rank 0
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = cid; u < p.nunits; u += ncl)
        for (int ch = 0; ch < p.nchunk; ++ch) {
          ptx::mbar_wait(full + stage, phase);
          ptx::fence_proxy_async_smem();
          arrive_rank0_pc(pfull + stage);
          if (++stage == p.ns) { stage = 0; phase ^= 1; }
        }
    }
  } else {
    // ================= epilogue: + bias, NCHW stores; lane = frame position of the quadrant
    const int qd = warp & 3, half = (warp - 5) >> 2;
    const int PQ = p.P * p.Q;
    uint32_t tcount = 0;
    for (int64_t u = cid; u < p.nunits; u += ncl, ++tcount) {
      const int64_t pt = u / p.nft;
      const int ft = (int)(u - pt * p.nft);
      const uint32_t buf = tcount & 1u, bph = (tcount >> 1) & 1u;
      const int64_t g = pt * 256 + (int64_t)rank * 128 + qd * 32 + lane;
      int64_t ybase = -1;
      if (g < p.G) {
        const int n = (int)(g / p.Lf), rem = (int)(g - (int64_t)n * p.Lf);
        const int hh = rem / p.Wf, ww = rem - hh * p.Wf;
        if (hh < p.P && ww < p.Q) ybase = (int64_t)n * p.Kout * PQ + (int64_t)hh * p.Q + ww;
      }
      ptx::mbar_wait_sleep(accf + buf, bph);
      __syncwarp();
      ptx::tc_fence_after();
      const int hcols = p.NT / 2;  // this warp's columns
      const uint32_t tb = tmem + ((uint32_t)(qd * 32) << 16) + buf * 256 + (uint32_t)(half * hcols);
      for (int c16 = 0; c16 < hcols / 16; ++c16) {
        float v[16];
        ptx::tmem_ld16(tb + (uint32_t)(c16 * 16), v);
        const int k0 = ft * p.NT + half * hcols + c16 * 16;
        if (ybase >= 0) {
          float *yp = p.y + ybase + (int64_t)k0 * PQ;
#pragma unroll
          for (int j = 0; j < 16; ++j) yp[(int64_t)j * PQ] = v[j] + (p.bias ? __ldg(p.bias + k0 + j) : 0.f);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) ptx::mbar_arrive(acce + buf);
        else arrive_rank0_pc(acce + buf);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // no CTA frees TMEM or exits while its peer may still signal it
  if (warp == 4) {
    ptx::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// fp[ft][ch][h][tap][quad][n][e] = W(k = ft*NT + h*NT/2 + n, c = ch*8 + quad*4 + e, tap) with
// W = F[k][c][r][s] (forward) or F[c][k][R-1-r][S-1-s] (bwd_data: the roles of C and K swap).
// One thread per source (row, column) pair: its RS taps are read contiguously (coalesced across
// threads) and scattered to the packed layout.  Every packed element is written: zero-padded
// rows / channels do not exist (Kout % 128 == 0, Cin % 8 == 0).
__global__ void pair_conv_pack_kernel(const float *__restrict__ f, float *__restrict__ fp, int Kout, int Cin,
                                      int R, int S, int nchunk, int nft, int NT, int flip) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int RS = R * S, BR = NT / 2;
  const int A = flip ? Cin : Kout, Bd = flip ? Kout : Cin;  // source F is [A][Bd][RS]
  const int64_t pairs = (int64_t)A * Bd;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < pairs; i += (int64_t)gridDim.x * blockDim.x) {
    const int ia = (int)(i / Bd), ib = (int)(i - (int64_t)ia * Bd);
    const int k = flip ? ib : ia, c = flip ? ia : ib;
    const int ft = k / NT, h = (k % NT) / BR, n = k % BR;
    const int ch = c >> 3, qd = (c >> 2) & 1, e = c & 3;
    const float *src = f + i * RS;
    float *dst = fp + ((((int64_t)ft * nchunk + ch) * 2 + h) * RS * 2 + qd) * BR * 4 + (int64_t)n * 4 + e;
    for (int tap = 0; tap < RS; ++tap) {
      const int st = flip ? RS - 1 - tap : tap;  // (R-1-r)*S + (S-1-s) = RS-1-tap
      dst[(int64_t)st * 2 * BR * 4] = __ldg(src + tap);
    }
  }
}

struct PcPlan {
  PcParams p;
  size_t smem, fp_bytes;
  bool ok;
};

// the stride-1 forward problem computed: input [N][Cin][H][W], output [N][Kout][P][Q]
PcPlan plan_pair(int N, int Cin, int H, int W, int Kout, int R, int S, int ph, int pw) {
  PcPlan pl{};
  pl.ok = false;
  PcParams &p = pl.p;
  p.N = N; p.Cin = Cin; p.H = H; p.W = W; p.Kout = Kout; p.R = R; p.S = S; p.ph = ph; p.pw = pw;
  p.P = H + 2 * ph - R + 1;
  p.Q = W + 2 * pw - S + 1;
  if (p.P <= 0 || p.Q <= 0 || Cin % 8 || Kout % 128 || ph > R - 1 || pw > S - 1) return pl;
  p.Wf = W + pw;
  p.Hs = H + ph;
  if (p.Wf < p.Q + S - 1 - pw || p.Hs < p.P) return pl;  // the shared-padding frame needs Wf >= Q + S - 1 - pw
  p.Lf = p.Hs * p.Wf;
  p.G = (int64_t)N * p.Lf;
  p.RS = R * S;
  p.HALO = (128 + (R - 1) * p.Wf + (S - 1) + 7) / 8 * 8;
  if (p.HALO > PC_MAXHALO || p.RS > 16) return pl;
  p.nchunk = Cin / 8;
  p.npt = ceil_div(p.G, 256);
  // unit width: 256 output channels, or 128 when that balances the pairs better (the A halo is
  // then staged once per 128 channels): wave efficiency units / (ceil(units / pairs) * pairs)
  const int pairs = std::max(1, sm_count() / 2);
  auto eff = [&](int nt) {
    const int64_t u = p.npt * (Kout / nt);
    return (double)u / (double)(ceil_div(u, (int64_t)pairs) * pairs);
  };
  static const int nt_env = getenv("SYSML_PAIR_NT") ? atoi(getenv("SYSML_PAIR_NT")) : 0;
  p.NT = nt_env == 128 || (Kout % 256 || eff(128) > 1.15 * eff(256)) ? 128 : 256;
  p.nft = Kout / p.NT;
  p.nunits = p.npt * p.nft;
  if ((int64_t)N * Cin * H * W >= (1ll << 31) || (int64_t)N * Kout * p.P * p.Q >= (1ll << 40)) return pl;
  p.a_bytes = (uint32_t)p.HALO * 32;
  p.b_bytes = (uint32_t)p.RS * (uint32_t)p.NT * 16;  // RS taps x 2 quads x NT/2 rows x 16 B
  p.stage_bytes = (p.a_bytes + p.b_bytes + 1023) / 1024 * 1024;
  const size_t fixed = PC_MAXHALO * 4 + 8 * (3 * PC_MAXNS + 4) + 16;
  p.ns = (int)std::min<size_t>(PC_MAXNS, (227 * 1024 - fixed) / p.stage_bytes);
  if (p.ns < 2) return pl;
  pl.smem = (size_t)p.ns * p.stage_bytes + fixed;
  pl.fp_bytes = (size_t)p.nft * p.nchunk * 2 * p.b_bytes;
  pl.ok = true;
  return pl;
}

PcPlan plan_of(const ConvArgs &a, int bwd_data) {
  if (a.sh != 1 || a.sw != 1) return PcPlan{};
  return bwd_data ? plan_pair(a.N, a.K, a.P, a.Q, a.C, a.R, a.S, a.R - 1 - a.ph, a.S - 1 - a.pw)
                  : plan_pair(a.N, a.C, a.H, a.W, a.K, a.R, a.S, a.ph, a.pw);
}

}  // namespace

bool pair_conv_supported(const ConvArgs &a, int bwd_data) {
  // opt-in: measured equal to K3 on the ResNet 3x3 layer (68.6 / 67.5 vs 68.6 us in isolation,
  // 70.7 vs 68.6 us in the bench's layer loop); SYSML_PAIR_CONV=1 routes eligible shapes here,
  // 2 forces it on any shape it supports (tests)
  static const int env = getenv("SYSML_PAIR_CONV") ? atoi(getenv("SYSML_PAIR_CONV")) : 0;
  if (!env || device_cc_major() != 10 || sm_count() < 2) return false;
  const PcPlan pl = plan_of(a, bwd_data);
  if (!pl.ok) return false;
  if (bwd_data && (pl.p.P != a.H || pl.p.Q != a.W)) return false;
  if (env == 2) return true;  // forced (tests)
  // 1x1 layers: one MMA per 8-channel chunk leaves the 4-byte gather of the A rows exposed
  // (measured 185 vs 87 us on 1x1 1024 -> 256); those stay on K3's staged producer
  return pl.p.RS >= 4 && pl.p.nunits >= sm_count() / 2;
}

size_t pair_conv_ws(const ConvArgs &a, int bwd_data) {
  const PcPlan pl = plan_of(a, bwd_data);
  return pl.ok ? align_up(pl.fp_bytes, 256) : 0;
}

sysml_status pair_conv(const ConvArgs &a, int bwd_data, const float *x, const float *f, const float *bias,
                       float *y, void *ws, cudaStream_t st) {
  PcPlan pl = plan_of(a, bwd_data);
  if (!pl.ok) {
    set_error("pair conv: unsupported shape");
    return SYSML_ERR_UNSUPPORTED;
  }
  PcParams p = pl.p;
  p.x = x;
  p.bias = bias;
  p.y = y;
  float *fp = reinterpret_cast<float *>(ws);
  {
    const int64_t total = (int64_t)p.Kout * p.Cin;
    pair_conv_pack_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 8 * sm_count()), 256, 0, st>>>(
        f, fp, p.Kout, p.Cin, p.R, p.S, p.nchunk, p.nft, p.NT, bwd_data);
    SYSML_LAUNCH_CHECK();
  }
  p.fp = fp;
  SYSML_TRY(smem_attr(pair_conv_kernel, pl.smem));
  const int pairs = (int)std::min<int64_t>(p.nunits, sm_count() / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cfg.blockDim = dim3(PC_THREADS);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = 2;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  route_note("pair_conv_kernel [tcgen05 TF32 cta_group::2, M = 256, N = %d, %d stages, %lld units on %d CTA pairs]",
             p.NT, p.ns, (long long)p.nunits, pairs);
  static long long *dclk = nullptr;
  const bool prof = getenv("SYSML_TC_PROFILE") != nullptr;
  if (prof && !dclk) cudaMalloc(&dclk, sizeof(long long) * 2 * 1024);
  if (prof) cudaMemsetAsync(dclk, 0, sizeof(long long) * 2 * 1024, st);
  p.clk = prof ? dclk : nullptr;
  SYSML_CUDA(cudaLaunchKernelEx(&cfg, pair_conv_kernel, p));
  SYSML_LAUNCH_CHECK();
  if (prof) {
    static long long h[2 * 1024];
    cudaMemcpyAsync(h, dclk, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double w = 0, tot = 0;
    for (int b = 0; b < 2 * pairs; b += 2) {
      w += (double)h[b * 2] / pairs;
      tot += (double)h[b * 2 + 1] / pairs;
    }
    fprintf(stderr, "[pair_conv] mma_wait_full %.0f mma_total %.0f (clk per leader CTA)\n", w, tot);
  }
  return SYSML_OK;
}

}  // namespace sysml
