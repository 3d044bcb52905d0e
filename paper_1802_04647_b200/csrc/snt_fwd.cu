// snt_fwd.cu -- LeNet conv2 forward + bias + relu + 2x2/2 max-pool (F2; S:154-163 conv2d,
// S:163 relu, S:185 max_pool with the pool-window codes of reading R9) with the column taps
// folded into the MMA N dimension and the filter bank resident in shared memory.
//
// Why: the general forward kernel (conv_tc.cu) runs F2 as 25 taps x N = 64 MMAs per 8-channel
// chunk with A and B streamed through shared memory; at N = 64 the MMA reads 6 KB of operands
// per 32 clocks of math, so it is shared-memory bound (ncu: tensor pipe 81% busy at ~68 clk per
// MMA, 45% of the TF32 peak).  Here, per tap row r and chunk:
//   MMA 1: N = 3*64 = 192 columns (s, k) for taps s = 0, 1, 2, A at frame offset r*Wf;
//   MMA 2: N = 2*64 = 128 columns (s - 3, k) for taps s = 3, 4, A shifted by 3 positions,
//          accumulated into the first 128 columns (SN-T, T = 3);
// so D'[pos][(j, k)] holds every tap with s = j or j + 3 and the epilogue adds
//   Y[pos][k] = D'[pos][(0,k)] + D'[pos+1][(1,k)] + D'[pos+2][(2,k)].
// With 16-column frames (14 outputs + 2 pad) the shifted rows pos+1, pos+2 of every valid output
// lie in the same frame row, hence in the same warp: two shuffles, no exchange, and linear
// 128-position tiles of 8 whole frame rows need no overlap.  A 2x2 pool window (rows 2i, 2i+1)
// is lanes l, l^1, l^16, l^17 of one warp (reduce-scatter butterfly as in conv_tc.cu).
// Operand bytes per tap row: 8 KB of A + 10 KB of B over 160 clocks of math (vs 30 KB over 160
// for five N = 64 MMAs).  The 205 KB packed bank is loaded once per CTA (bulk copies), so the only
// streamed operand is A: four 6.4 KB stages, K-major no-swizzle [quad][position][4 ch], gathered
// from the SPF planes by three producer sets (global loads -> 16-byte shared stores).
//
// Warps (persistent, 1 CTA/SM): 0-11 producers (set = warp / 4 takes chunks q % 3 == set), 12 MMA
// issuer, 13-20 epilogue (quadrant = warp % 4, channel half = (warp - 13) / 4).
#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace sysml {

namespace {

constexpr int SF_PSETS = 3;
constexpr int SF_PWARPS = 4 * SF_PSETS;
constexpr int SF_MMAW = SF_PWARPS;
constexpr int SF_THREADS = 32 * (SF_PWARPS + 1 + 8);
constexpr int SF_ASTAGES = 4;
static_assert(SF_PSETS <= SF_ASTAGES, "producer sets would run a full ring ahead");
constexpr int SF_T = 3;                 // taps s < T in MMA 1, s >= T in MMA 2 (A shifted by T)
constexpr int SF_NF = 64;               // output channels
constexpr int SF_S = 5, SF_R = 5, SF_WF = 16;
constexpr int SF_N1 = SF_T * SF_NF;           // 192
constexpr int SF_N2 = (SF_S - SF_T) * SF_NF;  // 128
constexpr int SF_NN = SF_N1 + SF_N2;          // 320 packed B rows per (chunk, r)
constexpr int SF_HALO = 200;            // staged positions: 128 + (R-1)*Wf + T = 195, rounded to 8
constexpr uint32_t SF_QUAD_BYTES = SF_HALO * 16;
constexpr uint32_t SF_STAGE_BYTES = 2 * SF_QUAD_BYTES;
constexpr uint32_t SF_ACC_STRIDE = 256;  // TMEM columns per accumulator buffer (N1 = 192 used)

struct SfParams {
  const float *x;       // SPF planes [Cin][plane], stored position = frame position + in_shift
  int64_t plane;
  int in_shift;
  const float *fp;      // packed B: [chunk][r][quad][SF_NN][4]
  const float *bias;    // [K] (nullable)
  float *pout;          // pooled output: NCHW [n][K][Pp][Qp]
  uint64_t *pcode;      // window codes [K/16][code_plane] (nullable)
  int64_t code_plane;
  int N, Cin, nchunk, Hs, Pp, Qp;
  int64_t ntiles;
  uint32_t b_bytes;
  long long *clk;
};

__global__ void __launch_bounds__(SF_THREADS, 1) snt_fwd_pool_kernel(const SfParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint8_t *Bs = smem;
  uint8_t *As = smem + p.b_bytes;  // b_bytes is a multiple of 1024
  float *bias_s = reinterpret_cast<float *>(As + SF_ASTAGES * SF_STAGE_BYTES);
  uint64_t *bars = reinterpret_cast<uint64_t *>(bias_s + SF_NF);
  uint64_t *bfull = bars;
  uint64_t *afull = bars + 1;               // [SF_ASTAGES]
  uint64_t *aempty = afull + SF_ASTAGES;    // [SF_ASTAGES]
  uint64_t *accf = aempty + SF_ASTAGES;     // [2]
  uint64_t *acce = accf + 2;                // [2]
  uint32_t *tslot = reinterpret_cast<uint32_t *>(acce + 2);

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    ptx::mbar_init(bfull, 1);
    for (int s = 0; s < SF_ASTAGES; ++s) {
      ptx::mbar_init(afull + s, 128);  // one producer set
      ptx::mbar_init(aempty + s, 1);   // tcgen05.commit
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(accf + b, 1);
      ptx::mbar_init(acce + b, 8);
    }
    ptx::fence_mbar_init();
  }
  if (warp == SF_MMAW) ptx::tmem_alloc(tslot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // packed filters and a1 ready (PDL)
  for (int k = threadIdx.x; k < SF_NF; k += blockDim.x) bias_s[k] = p.bias ? p.bias[k] : 0.f;
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(bfull, p.b_bytes);
    for (uint32_t off = 0; off < p.b_bytes; off += 32768u) {
      const uint32_t nb = min(32768u, p.b_bytes - off);
      ptx::bulk_g2s(const_cast<uint8_t *>(Bs) + off, reinterpret_cast<const uint8_t *>(p.fp) + off, nb, bfull);
    }
  }
  __syncthreads();  // bias_s visible to the epilogue

  if (warp < SF_PWARPS) {
    // ================= producers: thread t of the set stages positions t and t + 128 (< HALO)
    const int set = warp >> 2, t = (warp & 3) * 32 + lane;
    const int plane = (int)p.plane;  // Cin * plane < 2^31 (launcher)
    const int64_t my_tiles = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t qtot = my_tiles * p.nchunk;
    int coff[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) coff[c] = c * plane;
    int64_t tile = blockIdx.x;
    int ch = set;
    while (ch >= p.nchunk) { ch -= p.nchunk; tile += gridDim.x; }
    for (int64_t q = set; q < qtot; q += SF_PSETS) {
      const int stage = (int)(q % SF_ASTAGES);
      const uint32_t ph = (uint32_t)((q / SF_ASTAGES) & 1);
      const int g0 = (int)(tile * 128) + p.in_shift;
      const float *xc = p.x + (int64_t)(ch * 8) * plane;
      float v[2][8];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = t + 128 * h;
        const int sv = g0 + i;
        const bool ok = i < SF_HALO && sv >= 0 && sv < plane;
#pragma unroll
        for (int c = 0; c < 8; ++c) v[h][c] = (ok && ch * 8 + c < p.Cin) ? __ldg(xc + (sv + coff[c])) : 0.f;
      }
      ptx::mbar_wait(aempty + stage, ph ^ 1);
      uint8_t *A = As + (size_t)stage * SF_STAGE_BYTES;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = t + 128 * h;
        if (i < SF_HALO) {
          *reinterpret_cast<float4 *>(A + (size_t)i * 16) = make_float4(v[h][0], v[h][1], v[h][2], v[h][3]);
          *reinterpret_cast<float4 *>(A + SF_QUAD_BYTES + (size_t)i * 16) =
              make_float4(v[h][4], v[h][5], v[h][6], v[h][7]);
        }
      }
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(afull + stage);
      ch += SF_PSETS;
      while (ch >= p.nchunk) { ch -= p.nchunk; tile += gridDim.x; }
    }
  } else if (warp == SF_MMAW) {
    // ================= MMA issuer: one elected lane issues each chunk's 2*R MMAs and the commit
    ptx::mbar_wait(bfull, 0);
    ptx::tc_fence_after();
    const uint32_t idesc1 = ptx::make_idesc_tf32(128, SF_N1), idesc2 = ptx::make_idesc_tf32(128, SF_N2);
    const uint32_t bbase = ptx::smem_u32(Bs), abase = ptx::smem_u32(As);
    int64_t q = 0;
    uint32_t tcount = 0;
    long long t_acce = 0, t_afull = 0;
    const long long t_start = clock64();
    for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++tcount) {
      const uint32_t buf = tcount & 1u, bph = (tcount >> 1) & 1u;
      const long long t0 = clock64();
      ptx::mbar_wait(acce + buf, bph ^ 1);
      t_acce += clock64() - t0;
      ptx::tc_fence_after();
      const uint32_t d = tmem + buf * SF_ACC_STRIDE;
      for (int ch = 0; ch < p.nchunk; ++ch, ++q) {
        const int stage = (int)(q % SF_ASTAGES);
        const long long t1 = clock64();
        ptx::mbar_wait(afull + stage, (uint32_t)((q / SF_ASTAGES) & 1));
        t_afull += clock64() - t1;
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint32_t a0 = abase + (uint32_t)stage * SF_STAGE_BYTES;
          const uint32_t b0 = bbase + (uint32_t)(ch * SF_R) * (2u * SF_NN * 16u);
#pragma unroll
          for (int r = 0; r < SF_R; ++r) {
            const uint32_t ar = a0 + (uint32_t)(r * SF_WF) * 16u;
            const uint32_t br = b0 + (uint32_t)r * (2u * SF_NN * 16u);
            const uint64_t ad1 = ptx::make_desc(ar, SF_QUAD_BYTES, 128);
            const uint64_t ad2 = ptx::make_desc(ar + SF_T * 16u, SF_QUAD_BYTES, 128);
            const uint64_t bd1 = ptx::make_desc(br, SF_NN * 16u, 128);
            const uint64_t bd2 = ptx::make_desc(br + SF_N1 * 16u, SF_NN * 16u, 128);
            ptx::mma_tf32(d, ad1, bd1, idesc1, (ch | r) ? 1u : 0u);
            ptx::mma_tf32(d, ad2, bd2, idesc2, 1u);
          }
          ptx::mma_commit(aempty + stage);
        }
        __syncwarp();
      }
      if (ptx::elect_one()) ptx::mma_commit(accf + buf);
      __syncwarp();
    }
    if (p.clk && lane == 0) {
      p.clk[blockIdx.x * 4 + 0] = t_acce;
      p.clk[blockIdx.x * 4 + 1] = t_afull;
      p.clk[blockIdx.x * 4 + 2] = clock64() - t_start;
    }
  } else {
    // ================= epilogue: SN-T shift-add, bias, relu, 2x2 pool, codes
    const int qd = warp & 3, eh = (warp - SF_MMAW - 1) >> 2;  // channel half [32*eh, +32)
    const int PpQp = p.Pp * p.Qp;
    const uint32_t odd_c = lane & 1, odd_r = (lane >> 4) & 1;
    const int cb = (int)(odd_c * 8 + odd_r * 4);  // first of the 4 channels this lane ends with
    const int col = lane & 15;
    uint32_t tcount = 0;
    for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++tcount) {
      const uint32_t buf = tcount & 1u, bph = (tcount >> 1) & 1u;
      const int grow = (int)(tile * 8) + qd * 2 + (int)odd_r;  // global frame row
      const int n = grow / p.Hs, hh = grow - n * p.Hs;
      const int pp = hh >> 1, pc = col >> 1;
      const bool store = n < p.N && pp < p.Pp && pc < p.Qp;
      const int64_t wi = store ? (int64_t)n * PpQp + pp * p.Qp + pc : 0;  // window index
      ptx::mbar_wait_sleep(accf + buf, bph);
      __syncwarp();
      ptx::tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(qd * 32) << 16) + buf * SF_ACC_STRIDE;
#pragma unroll 1
      for (int g = 0; g < 2; ++g) {
        const int k0 = eh * 32 + g * 16;
        uint32_t r0[16], r1[16], r2[16];
        ptx::tmem_ld16_issue(tbase + (uint32_t)k0, r0);
        ptx::tmem_ld16_issue(tbase + (uint32_t)(SF_NF + k0), r1);
        ptx::tmem_ld16_issue(tbase + (uint32_t)(2 * SF_NF + k0), r2);
        ptx::tmem_ld_wait(r0);
        ptx::tmem_ld_pin(r1);
        ptx::tmem_ld_pin(r2);
        uint32_t u[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float y = __uint_as_float(r0[j]) + __shfl_down_sync(0xffffffffu, __uint_as_float(r1[j]), 1) +
                          __shfl_down_sync(0xffffffffu, __uint_as_float(r2[j]), 2) + bias_s[k0 + j];
          u[j] = __float_as_uint(y > 0.f ? y : 0.f);  // relu, +0.0 for non-positive (reading R7)
        }
        // reduce-scatter butterfly (conv_tc.cu epi_pool2): column partner lane ^ 1, row partner
        // lane ^ 16; relu'd values compare as unsigned integers, the earlier position wins ties
        uint32_t v8[8], sbit = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t send = odd_c ? u[j] : u[j + 8];
          const uint32_t mine = odd_c ? u[j + 8] : u[j];
          const uint32_t got = __shfl_xor_sync(0xffffffffu, send, 1);
          const bool take = got + odd_c > mine;
          v8[j] = take ? got : mine;
          sbit |= (odd_c ^ (uint32_t)take) << j;
        }
        uint32_t v4[4];
        const uint32_t psbit = __shfl_xor_sync(0xffffffffu, sbit, 16);
        uint32_t code = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t send = odd_r ? v8[j] : v8[j + 4];
          const uint32_t mine = odd_r ? v8[j + 4] : v8[j];
          const uint32_t got = __shfl_xor_sync(0xffffffffu, send, 16);
          const bool take = got + odd_r > mine;
          v4[j] = take ? got : mine;
          const int jj = (int)(odd_r * 4) + j;
          const uint32_t ds = ((take ? psbit : sbit) >> jj) & 1u;
          const uint32_t pos = v4[j] != 0u;  // window max > 0 (reading R9)
          code |= ((pos << 2) | ((odd_r ^ (uint32_t)take) << 1) | ds) << (4 * j);
        }
        if (store) {
          float *po = p.pout + (int64_t)n * SF_NF * PpQp + pp * p.Qp + pc + (int64_t)(k0 + cb) * PpQp;
#pragma unroll
          for (int j = 0; j < 4; ++j) po[j * PpQp] = __uint_as_float(v4[j]);
          if (p.pcode)
            reinterpret_cast<uint16_t *>(p.pcode + (int64_t)(k0 >> 4) * p.code_plane + wi)[cb >> 2] = (uint16_t)code;
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(acce + buf);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == SF_MMAW) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// packed(chunk, r, quad, n, e) = F[k][c = chunk*8 + quad*4 + e][r][s]: n < N1 -> (s = n / 64,
// k = n % 64); n >= N1 -> (s = T + (n - N1) / 64, k = (n - N1) % 64)
__global__ void snt_fwd_pack_kernel(const float *__restrict__ f, float *__restrict__ fp, int Cin, int nchunk) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t total = (int64_t)nchunk * SF_R * 2 * SF_NN * 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int e = (int)(t % 4); t /= 4;
    const int n = (int)(t % SF_NN); t /= SF_NN;
    const int g = (int)(t % 2); t /= 2;
    const int r = (int)(t % SF_R); t /= SF_R;
    const int ch = (int)t;
    const int s_ = n < SF_N1 ? n / SF_NF : SF_T + (n - SF_N1) / SF_NF;
    const int k = n < SF_N1 ? n % SF_NF : (n - SF_N1) % SF_NF;
    const int c = ch * 8 + g * 4 + e;
    fp[i] = c < Cin ? f[(((int64_t)k * Cin + c) * SF_R + r) * SF_S + s_] : 0.f;
  }
}

size_t sf_b_bytes(int Cin) { return (size_t)((Cin + 7) / 8) * SF_R * 2 * SF_NN * 16; }
size_t sf_smem(int Cin) {
  return sf_b_bytes(Cin) + SF_ASTAGES * SF_STAGE_BYTES + SF_NF * 4 + 8 * (1 + 2 * SF_ASTAGES + 4) + 16;
}

}  // namespace

// LeNet conv2 geometry only: 5x5 pad 2 stride 1, K = 64, 16-wide frames of 16 rows per image
// (SPF planes, 14x14 outputs), 2x2/2 pool, pooled output NCHW + window codes.
bool snt_fwd_pool_supported(const ConvArgs &a, const PoolArgs *pool, int Wf, int Lf) {
  if (device_cc_major() != 10 || getenv("SYSML_NO_SNT_FWD")) return false;
  if (!pool || pool->R != 2 || pool->S != 2 || pool->sh != 2 || pool->sw != 2 || pool->ph || pool->pw) return false;
  if (a.K != SF_NF || a.R != SF_R || a.S != SF_S || a.sh != 1 || a.sw != 1 || a.ph != 2 || a.pw != 2) return false;
  if (a.H != 14 || a.W != 14 || Wf != SF_WF || Lf != 256 || a.C > 64) return false;
  return sf_smem(a.C) <= 227 * 1024;
}

size_t snt_fwd_pool_ws(const ConvArgs &a) { return align_up(sf_b_bytes(a.C), 256); }

sysml_status snt_fwd_pool_spf(const ConvArgs &a, const TcSpfIO &io, const float *x, const float *f,
                              const float *bias, float *pout, void *ws, cudaStream_t st) {
  if (io.in_plane <= 0 || io.out_plane > 0 || (int64_t)a.C * io.in_plane >= (1ll << 31)) {
    set_error("SN-T forward: unsupported I/O layout");
    return SYSML_ERR_UNSUPPORTED;
  }
  SfParams p{};
  p.x = x;
  p.plane = io.in_plane;
  p.in_shift = io.in_shift;
  p.bias = bias;
  p.pout = pout;
  p.pcode = io.code;
  p.code_plane = io.code_plane;
  p.N = a.N;
  p.Cin = a.C;
  p.nchunk = (a.C + 7) / 8;
  p.Hs = 16;
  p.Pp = 7;
  p.Qp = 7;
  p.ntiles = (int64_t)a.N * 2;  // 256 frame positions per image
  p.b_bytes = (uint32_t)sf_b_bytes(a.C);
  float *fp = reinterpret_cast<float *>(ws);
  {
    const int64_t total = (int64_t)p.nchunk * SF_R * 2 * SF_NN * 4;
    snt_fwd_pack_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 4 * sm_count()), 256, 0, st>>>(
        f, fp, a.C, p.nchunk);
    SYSML_LAUNCH_CHECK();
  }
  p.fp = fp;
  const size_t smem = sf_smem(a.C);
  SYSML_TRY(smem_attr(snt_fwd_pool_kernel, smem));
  const int grid = (int)std::min<int64_t>(p.ntiles, sm_count());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(SF_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  route_note("snt_fwd_pool_kernel [tcgen05 TF32, SN-T T=3 (N = 192 + 128), resident filters, fused pool, %lld tiles on %d CTAs]",
             (long long)p.ntiles, grid);
  static long long *dclk = nullptr;
  const bool prof = getenv("SYSML_TC_PROFILE") != nullptr;
  if (prof && !dclk) cudaMalloc(&dclk, sizeof(long long) * 4 * 1024);
  p.clk = prof ? dclk : nullptr;
  SYSML_CUDA(cudaLaunchKernelEx(&cfg, snt_fwd_pool_kernel, p));
  SYSML_LAUNCH_CHECK();
  if (prof) {
    static long long h[4 * 1024];
    cudaMemcpyAsync(h, dclk, sizeof(long long) * 4 * 1024, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double s3[3] = {0, 0, 0};
    for (int b = 0; b < grid; ++b)
      for (int j = 0; j < 3; ++j) s3[j] += (double)h[b * 4 + j] / grid;
    fprintf(stderr, "[snt_fwd] mma_wait_acce %.0f mma_wait_afull %.0f mma_total %.0f\n", s3[0], s3[1], s3[2]);
  }
  return SYSML_OK;
}

}  // namespace sysml
