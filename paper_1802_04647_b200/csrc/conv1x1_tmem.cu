// conv1x1_tmem.cu -- 1x1, stride-1, unpadded conv2d forward and backward-data (the ResNet
// bottleneck's 1x1 layers, SURVEY §8(d) cfg 4(ii)) with the activation transposed through TMEM.
//
//   fwd:       Y[n][k][p]  = sum_c F[k][c] X[n][c][p] + b[k]      (§8(c) def. 1)
//   bwd_data:  dX[n][c][p] = sum_k F[k][c] dY[n][k][p]            (§8(c) def. 5)
//
// Both are D[m][o] = sum_i In[n][i][p] W[o][i] with m = (n, p) the flattened positions
// (fwd: In = X, W = F; bwd_data: In = dY, W = F^T, transposed once into the workspace).  The
// NCHW activation is MN-major for this GEMM (positions contiguous), and MN-major TF32 operands
// read as zeros on sm_100a (tools/mn_major_probe.cu), so the K3 path transposes it through
// shared memory.  Here it goes through registers into TMEM instead: the MMA's A operand may live
// in TMEM (lane = row m, one 32-bit column per k), and a warp's lane t loading In[n][i][p0 + t]
// for 32 consecutive i is one coalesced 128-byte load per i, stored with one tcgen05.st as its
// lane's 32 columns -- no shared memory on the activation path.  W is a K-major operand (i
// contiguous) moved by TMA with the 128-byte swizzle.
//
// Work unit: 128 positions x ON (<= 128) output channels; the units of one position tile are
// consecutive, so they run at about the same time and the activation tile is read from HBM once
// (the second read hits L2).  Persistent CTAs walk units round-robin.  Per unit: I / 32 chunks
// of 4 MMAs (M = 128, N = ON, K = 8), double-buffered accumulators so the epilogue of a unit
// overlaps the next unit's MMAs.
//
// Warps: 0 = W TMA producer, 1 = MMA issuer (TMEM owner), 2-17 = activation producers (four per
// TMEM lane quadrant, warp % 4, rotating chunks), 18-25 = epilogue (quadrant warp % 4, two
// halves taking alternate 16-column groups).
#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"
#include "tma.cuh"

#include <algorithm>
#include <cstdlib>

namespace sysml {

namespace {

constexpr int X1_AST = 4;                    // TMEM activation stages (32 columns each)
constexpr int X1_BST = 4;                    // shared-memory W stages
constexpr int X1_PW = 16;                    // activation producer warps (4 per lane quadrant)
constexpr int X1_EW = 8;                     // epilogue warps: two per lane quadrant (column-group halves)
constexpr int X1_THREADS = (2 + X1_PW + X1_EW) * 32;
constexpr uint32_t X1_ACOL = 256;            // first activation-stage column (accumulators: 2 x ON <= 256)

struct X1Params {
  const float *in;       // [N][I][HW]
  const float *bias;     // [O] or null
  float *out;            // [N][O][HW]
  int I, O, HW, ON, n_ot, nchunk;
  int Mtot, units;
  int mtl;               // M tiles (128 positions) per unit: 2 shares each W box between 256 positions
  int nbuf;              // accumulator buffers (2: the epilogue overlaps the next unit's MMAs)
  int blocked;           // 1: contiguous unit ranges per CTA
  int staged;            // HW % 4 == 0: epilogue through shared memory, 16-byte row stores
  int dbg;               // experiments: 1 = no output stores, 2 = no MMAs, 4 = no activation loads
};

__device__ __forceinline__ void x1_mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ uint64_t x1_sw128(uint32_t saddr) {
  return ptx::make_desc(saddr, 16, 1024) | ((uint64_t)2 << 61);
}

__global__ void __launch_bounds__(X1_THREADS, 1)
    c1x1_kernel(const __grid_constant__ CUtensorMap tmW, const X1Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const uint32_t b_bytes = (uint32_t)p.ON * 128;
  float *stg = reinterpret_cast<float *>(smem + X1_BST * b_bytes);  // [half][2][16][128] epilogue staging
  uint64_t *bars = reinterpret_cast<uint64_t *>(stg + 2 * 2 * 16 * 128);
  uint64_t *fullA = bars, *emptyA = bars + X1_AST, *fullB = bars + 2 * X1_AST, *emptyB = fullB + X1_BST;
  uint64_t *accf = emptyB + X1_BST, *acce = accf + 2;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(acce + 2);

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < X1_AST; ++s) {
      ptx::mbar_init(fullA + s, p.mtl == 2 ? 8 : 4);  // one producer warp per lane quadrant (and M tile)
      ptx::mbar_init(emptyA + s, 1);
    }
    for (int s = 0; s < X1_BST; ++s) {
      ptx::mbar_init(fullB + s, 1);
      ptx::mbar_init(emptyB + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(accf + b, 1);
      ptx::mbar_init(acce + b, X1_EW);  // the epilogue warps
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tslot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  asm volatile("griddepcontrol.wait;" ::: "memory");

  // units of this CTA: round-robin (u0 = blockIdx.x, step gridDim.x) or a contiguous block;
  // 32-bit unit / chunk / position arithmetic (c1x1_supported: N*H*W < 2^31), no divisions in
  // the per-element paths
  int u0 = blockIdx.x, ustep = gridDim.x;
  int nmine = p.units > (int)blockIdx.x ? (p.units - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  if (p.blocked) {
    u0 = (int)((int64_t)blockIdx.x * p.units / gridDim.x);
    nmine = (int)((int64_t)(blockIdx.x + 1) * p.units / gridDim.x) - u0;
    ustep = 1;
  }
  const int nj = nmine * p.nchunk;  // chunks of this CTA, in order

  if (warp == 0) {
    // ================= W producer: one 32-wide K box of ON rows per chunk
    if (lane == 0) {
      const uint32_t sB = ptx::smem_u32(smem);
      int lu = 0, ch = 0;
      for (int j = 0; j < nj; ++j) {
        const int ot = (int)((uint32_t)(u0 + lu * ustep) % (uint32_t)p.n_ot);
        const int sb = j % X1_BST;
        ptx::mbar_wait(emptyB + sb, (uint32_t)(((j / X1_BST) & 1) ^ 1));
        ptx::mbar_arrive_expect_tx(fullB + sb, b_bytes);
        ptx::tma_load_2d(sB + sb * b_bytes, &tmW, ch * 32, ot * p.ON, ptx::smem_u32(fullB + sb));
        if (++ch == p.nchunk) { ch = 0; ++lu; }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    const uint32_t idesc = ptx::make_idesc_tf32(128, p.ON);
    const uint32_t sB = ptx::smem_u32(smem);
    int j = 0;
    for (int lu = 0; lu < nmine; ++lu) {
      const int buf = p.nbuf == 2 ? (lu & 1) : 0;
      ptx::mbar_wait(acce + buf, (uint32_t)(((lu / p.nbuf) & 1) ^ 1));
      ptx::tc_fence_after();
      const uint32_t d = tmem + (uint32_t)(buf * p.ON);  // mtl = 2: tiles at columns 0, ON (nbuf 1)
      for (int ch = 0; ch < p.nchunk; ++ch, ++j) {
        const int s = j % X1_AST, sb = j % X1_BST;
        ptx::mbar_wait(fullA + s, (uint32_t)((j / X1_AST) & 1));
        ptx::mbar_wait(fullB + sb, (uint32_t)((j / X1_BST) & 1));
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint64_t bd = x1_sw128(sB + sb * b_bytes);
          for (int t = 0; t < p.mtl; ++t) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              if (!(p.dbg & 2))
                x1_mma_ts(d + (uint32_t)(t * p.ON), tmem + X1_ACOL + (uint32_t)((s * p.mtl + t) * 32 + kk * 8),
                          bd + (uint64_t)(kk * 2), idesc, (ch | kk) ? 1u : 0u);
          }
          ptx::mma_commit(emptyA + s);
          ptx::mma_commit(emptyB + sb);
          if (ch == p.nchunk - 1) ptx::mma_commit(accf + buf);
        }
        __syncwarp();
      }
    }
  } else if (warp < 2 + X1_PW) {
    // ================= activation producers: lane t of quadrant q holds position
    // m = mt * 128 + 32 q + t; chunk j's 32 values In[n][i0 .. i0 + 31][p] go to its lane's 32
    // columns of stage j % 4
    // mtl = 1: the four warps of a quadrant rotate chunks (four chunks in flight); mtl = 2: M tile
    // par % 2, chunks rotating over the two warps of that tile
    constexpr int NPQ = X1_PW / 4;  // producer warps per quadrant
    const int q = warp & 3, par = (warp - 2) >> 2;
    const int tile = p.mtl == 2 ? (par & 1) : 0;
    const int jstep = p.mtl == 2 ? NPQ / 2 : NPQ, j0 = p.mtl == 2 ? (par >> 1) : par;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + X1_ACOL + (uint32_t)(tile * 32);
    int lu = 0, ch = j0;
    while (ch >= p.nchunk && p.nchunk > 0) { ch -= p.nchunk; ++lu; }
    for (int j = j0; j < nj; j += jstep) {
      const uint32_t u = (uint32_t)(u0 + lu * ustep);
      const int m = (int)(u / (uint32_t)p.n_ot) * (128 * p.mtl) + tile * 128 + q * 32 + lane;
      float v[32];
      if (m < p.Mtot && !(p.dbg & 4)) {
        const int n = (int)((uint32_t)m / (uint32_t)p.HW);
        const int pp = m - n * p.HW;
        const float *src = p.in + ((int64_t)n * p.I + ch * 32) * (int64_t)p.HW + pp;
        if (ch * 32 + 32 <= p.I) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = __ldg(src + (int64_t)e * p.HW);
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = ch * 32 + e < p.I ? __ldg(src + (int64_t)e * p.HW) : 0.f;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0.f;
      }
      const int s = j % X1_AST;
      ptx::mbar_wait(emptyA + s, (uint32_t)(((j / X1_AST) & 1) ^ 1));
      ptx::tc_fence_after();
      float *h0 = v, *h1 = v + 16;
      ptx::tmem_st16(lane_base + (uint32_t)(s * 32 * p.mtl), *reinterpret_cast<float(*)[16]>(h0));
      ptx::tmem_st16(lane_base + (uint32_t)(s * 32 * p.mtl + 16), *reinterpret_cast<float(*)[16]>(h1));
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(fullA + s);
      ch += jstep;
      while (ch >= p.nchunk) { ch -= p.nchunk; ++lu; }
    }
  } else {
    // ================= epilogue: lane t of quadrant q = position m; columns = output channels
    // mtl = 1: half h takes the column groups g % 2 == h; mtl = 2: half h is M tile h (all groups)
    const int q = warp & 3, half = (warp - 2 - X1_PW) >> 2;
    const int tileE = p.mtl == 2 ? half : 0, cstart = p.mtl == 2 ? 0 : 16 * half, cstep = p.mtl == 2 ? 16 : 32;
    int grp = 0;  // 16-column groups done by this half (staging buffer parity)
    const int et = ((int)threadIdx.x - (2 + X1_PW) * 32) & 127;
    float *stg_h = stg + half * (2 * 16 * 128);
    for (int lu = 0; lu < nmine; ++lu) {
      const int buf = p.nbuf == 2 ? (lu & 1) : 0;
      const uint32_t u = (uint32_t)(u0 + lu * ustep);
      const int mt = (int)(u / (uint32_t)p.n_ot);
      const int o0 = (int)(u - (uint32_t)mt * (uint32_t)p.n_ot) * p.ON;
      const int mbase = mt * (128 * p.mtl) + tileE * 128;
      const int m = mbase + q * 32 + lane;
      ptx::mbar_wait_sleep(accf + buf, (uint32_t)((lu / p.nbuf) & 1));
      ptx::tc_fence_after();
      const bool mv = m < p.Mtot;
      const int n = mv ? (int)((uint32_t)m / (uint32_t)p.HW) : 0;
      const int pp = mv ? m - n * p.HW : 0;
      float *dst = p.out + ((int64_t)n * p.O + o0) * (int64_t)p.HW + pp;
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((buf + tileE) * p.ON);
      if (p.staged) {
        // 16 columns at a time through shared memory ([16 o][128 positions], two buffers), then
        // whole 512-byte output rows with 16-byte stores (HW % 4 == 0: a float4 never straddles
        // an image); one named barrier per group
        // this thread's float4 column (4 positions) is the same in every row it copies
        const int c4 = et & 31, e0 = et >> 5;
        const int mm = mbase + c4 * 4;
        const bool mmv = mm < p.Mtot;
        const int nn = mmv ? (int)((uint32_t)mm / (uint32_t)p.HW) : 0;
        float *orow = p.out + ((int64_t)nn * p.O + o0) * (int64_t)p.HW + (mm - nn * p.HW);
        for (int c0 = cstart; c0 < p.ON; c0 += cstep, ++grp) {
          float v[16];
          ptx::tmem_ld16(ta + (uint32_t)c0, v);
          float *sg = stg_h + (grp & 1) * (16 * 128);
#pragma unroll
          for (int e = 0; e < 16; ++e) sg[e * 128 + q * 32 + lane] = v[e];
          ptx::named_bar_sync(1 + half, 128);
          if (!(p.dbg & 1) && mmv) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const int e = e0 + 4 * r, o = o0 + c0 + e;
              if (o < p.O) {
                float4 w = *reinterpret_cast<const float4 *>(sg + e * 128 + c4 * 4);
                if (p.bias) {
                  const float bv = __ldg(p.bias + o);
                  w.x += bv; w.y += bv; w.z += bv; w.w += bv;
                }
                *reinterpret_cast<float4 *>(orow + (int64_t)(c0 + e) * p.HW) = w;
              }
            }
          }
        }
      } else {
        for (int c0 = cstart; c0 < p.ON; c0 += cstep) {
          float v[16];
          ptx::tmem_ld16(ta + (uint32_t)c0, v);
          if (mv && !(p.dbg & 1)) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int o = o0 + c0 + e;
              if (o < p.O) dst[(int64_t)(c0 + e) * p.HW] = v[e] + (p.bias ? __ldg(p.bias + o) : 0.f);
            }
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(acce + buf);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// Ft[c][k] = F[k][c] (32 x 32 tiles through shared memory)
__global__ void c1x1_transpose_kernel(const float *__restrict__ f, float *__restrict__ ft, int K, int C) {
  __shared__ float t[32][33];
  const int c0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int k = k0 + r, c = c0 + threadIdx.x;
    t[r][threadIdx.x] = (k < K && c < C) ? f[(int64_t)k * C + c] : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int c = c0 + r, k = k0 + threadIdx.x;
    if (c < C && k < K) ft[(int64_t)c * K + k] = t[threadIdx.x][r];
  }
}

size_t c1x1_smem(int ON) {
  return 1024 + (size_t)X1_BST * ON * 128 + 2 * 2 * 16 * 128 * 4 + 8 * (2 * X1_AST + 2 * X1_BST + 4) + 16;
}

}  // namespace

bool c1x1_supported(const ConvArgs &a, int bwd_data) {
  static const int env = getenv("SYSML_C1X1") ? atoi(getenv("SYSML_C1X1")) : 1;
  if (!env || device_cc_major() != 10) return false;
  if (a.R != 1 || a.S != 1 || a.sh != 1 || a.sw != 1 || a.ph != 0 || a.pw != 0) return false;
  const int I = bwd_data ? a.K : a.C, O = bwd_data ? a.C : a.K;
  // TMA: the W row stride (I floats) must be a multiple of 16 bytes.  Expansion layers on large
  // images (O >= 4 I, H*W >= 2048: ResNet-50 stage 1's 64 -> 256) are output-store bound and stay
  // on K3 (114 vs 135 us measured at N = 128); every other ResNet-50 1x1 shape is faster here.
  if (O >= 4 * I && a.H * a.W >= 2048) return false;
  return I % 4 == 0 && O >= 16 && (int64_t)a.N * a.H * a.W < (1ll << 30);
}

size_t c1x1_ws(const ConvArgs &a, int bwd_data) {
  return bwd_data ? align_up((size_t)a.C * a.K * sizeof(float), 256) : 0;
}

sysml_status c1x1_conv(const ConvArgs &a, int bwd_data, const float *in, const float *f, const float *bias,
                       float *out, void *ws, cudaStream_t st) {
  const int I = bwd_data ? a.K : a.C, O = bwd_data ? a.C : a.K;
  const float *w = f;
  if (bwd_data) {
    float *ft = reinterpret_cast<float *>(ws);
    c1x1_transpose_kernel<<<dim3((unsigned)ceil_div(a.C, 32), (unsigned)ceil_div(a.K, 32)), dim3(32, 8), 0, st>>>(
        f, ft, a.K, a.C);
    SYSML_LAUNCH_CHECK();
    w = ft;
  }
  X1Params p{};
  p.in = in;
  p.bias = bwd_data ? nullptr : bias;
  p.out = out;
  p.I = I;
  p.O = O;
  p.HW = a.H * a.W;
  static const int on_env = getenv("SYSML_C1X1_ON") ? atoi(getenv("SYSML_C1X1_ON")) : 128;
  p.ON = (int)std::min<int64_t>(std::max(16, std::min(256, on_env)), (O + 15) / 16 * 16);
  // two M tiles per unit (each W box serves 256 positions; single-buffered accumulators) when the
  // activation dominates: long K loops amortise the unhidden epilogue
  static const int mt2_env = getenv("SYSML_C1X1_MT2") ? atoi(getenv("SYSML_C1X1_MT2")) : 0;
  p.mtl = (mt2_env == 2 || (mt2_env == 1 && I >= 2 * O && I >= 256)) && p.ON <= 128 ? 2 : 1;
  p.nbuf = p.ON <= 128 && p.mtl == 1 ? 2 : 1;
  p.blocked = getenv("SYSML_C1X1_BLOCKED") ? atoi(getenv("SYSML_C1X1_BLOCKED")) : 0;
  p.n_ot = (int)ceil_div(O, p.ON);
  p.nchunk = (int)ceil_div(I, 32);
  p.Mtot = a.N * p.HW;
  p.staged = p.HW % 4 == 0 && !(getenv("SYSML_C1X1_DIRECT"));
  p.dbg = getenv("SYSML_C1X1_DBG") ? atoi(getenv("SYSML_C1X1_DBG")) : 0;
  p.units = (int)ceil_div(p.Mtot, 128 * p.mtl) * p.n_ot;
  CUtensorMap tmW;
  {
    const uint64_t dims[2] = {(uint64_t)I, (uint64_t)O};
    const uint64_t strides[1] = {(uint64_t)I * 4};
    const uint32_t box[2] = {32, (uint32_t)p.ON};  // columns beyond I / rows beyond O: zero-filled
    if (!tmap_encode_f32(&tmW, w, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return SYSML_ERR_CUDA;
  }
  const size_t smem = c1x1_smem(p.ON);
  SYSML_TRY(smem_attr(c1x1_kernel, smem));
  const int grid = (int)std::min<int64_t>(p.units, sm_count());
  route_note("c1x1_kernel [tcgen05 TF32, activation transposed through TMEM, %d units of %d x %d on %d CTAs]",
             p.units, 128 * p.mtl, p.ON, grid);
  c1x1_kernel<<<grid, X1_THREADS, smem, st>>>(tmW, p);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

}  // namespace sysml
