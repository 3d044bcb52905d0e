// b1_tc.cu -- LeNet conv1 weight gradient fused with the pool1 backward (B1; S:165-173 bwd_filter
// of maxpool_backward, reading R9) on the tensor cores.
//
//   dF1[k][r][s] = sum_{n, pp} g[n][pp][k] * x_n(2 pr + dr + r - 2, 2 pc + ds + s - 2)
//   db1[k]       = sum_{n, pp} g[n][pp][k]
// with g masked by the window code (positive bit) and (dr, ds) the window winner of (n, k, pp).
//
// The winner offset depends on k, so the sum is not one GEMM; it is four, one per candidate
// d = (dr, ds), stacked in M.  The image operand depends on (dr, r) and (ds, s) only through
// u = dr + r and v = ds + s (0..5), so N needs the 36 distinct offsets, not 4 x 25 columns:
//   D[(d, k)][(u, v)] = sum_pp A[(d, k)][pp] * B[(u, v)][pp]
//   A[(d, k)][pp] = g[pp][k] if code(k, pp) = (positive, d) else 0       (M = 4 x 32 = 128)
//   B[(u, v)][pp] = x(2 pr + u - 2, 2 pc + v - 2)                         (N = 36 -> 48)
// and dF1[k][r][s] = sum_d D[(d, k)][(dr + r, ds + s)].  The SIMT kernel spent ~45 instructions
// per 25 FMAs (fused_bwd.cu, latency bound on its window reads); here the builder warps write
// each operand element once (A: masked copies of g, B: a stride-2 gather of the image) and the
// MMAs do the arithmetic (TF32, like the rest of the TF32 step).
//
// Per CTA (persistent, a contiguous range of images): a 2-stage ring of image inputs (g NHWC
// 25 KB and the two 16-channel code words per window by bulk copy; x as a 40 x 32 TMA box after
// a zero prefix, its out-of-bounds part the zero border), and two operand buffers of 72 pooled
// positions (18 K quads); per image three chunks of 9 MMAs (M = 128, N = 48, K = 8) accumulate
// into one TMEM tile for the whole range.
// Warps: 0-15 builders (0-3 also read the accumulator at the end), 16 MMA issuer, 17 loader.
#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"
#include "tma.cuh"

#include <algorithm>
#include <cstdlib>

namespace sysml {

namespace {

constexpr int B1T_BUILD = 512;                      // builder threads (16 warps)
constexpr int B1T_THREADS = B1T_BUILD + 64;         // + MMA warp + loader warp
constexpr int B1T_K = 32, B1T_RS = 25, B1T_PP = 196;
constexpr int B1T_UV = 36;                          // distinct image offsets (u, v) = (dr + r, ds + s)
constexpr int B1T_N = 48;                           // 36 columns + zero padding (M = 128 needs N % 16 = 0)
constexpr int B1T_XP = 40;                          // zero-bordered image tile: 32 rows x 40 (TMA box)
constexpr int B1T_CHUNK = 72, B1T_KQ = B1T_CHUNK / 4, B1T_NCHUNK = 3;  // 216 >= 196 positions
constexpr int B1T_AITEMS = B1T_KQ * B1T_K, B1T_ITEMS = B1T_AITEMS + B1T_KQ * B1T_UV;
constexpr uint32_t B1T_G_BYTES = B1T_PP * B1T_K * 4;        // 25088
constexpr uint32_t B1T_C_BYTES = B1T_PP * 8;                // one 16-channel code word per window
constexpr uint32_t B1T_X_BYTES = 32 * B1T_XP * 4;           // 5120
// x(h, w) sits at float 96 + 40 h + w of the stage: a zero prefix of 96 floats covers h = -2, -1
// (TMA rejects negative box coordinates on sm_100a: tools/tma_box_probe.cu), w = -2, -1 wrap
// into the zero columns 38, 39 of the row above, and the box's out-of-bounds rows 28..31 and
// columns 28..39 arrive as zeros
constexpr uint32_t B1T_XPRE = 96 * 4;
constexpr uint32_t B1T_STAGE_TX = B1T_X_BYTES + B1T_G_BYTES + 2 * B1T_C_BYTES;   // 33344
constexpr uint32_t B1T_XG = B1T_XPRE + B1T_X_BYTES;               // g after the prefixed x box
constexpr uint32_t B1T_STAGE = (B1T_XG - B1T_X_BYTES + B1T_STAGE_TX + 127) / 128 * 128;
constexpr uint32_t B1T_ABYTES = B1T_KQ * 128 * 16, B1T_BBYTES = B1T_KQ * B1T_N * 16;
constexpr uint32_t B1T_OPB = B1T_ABYTES + B1T_BBYTES;       // one operand buffer
constexpr int B1T_NBUF = 3;                         // operand buffers in flight
static_assert(B1T_AITEMS % 32 == 0 && B1T_BUILD % 32 == 0, "warp-uniform A/B split");

struct B1tParams {
  const float *g;          // da1, [n][196][32]
  const uint64_t *code;    // window codes [2][code_plane], index n * 196 + pp
  int64_t code_plane;
  float *part;             // [cta][32 * 26]: 25 dF taps + db per filter
  int N, n_per_cta;
};

__global__ void __launch_bounds__(B1T_THREADS, 1)
    b1_tc_kernel(const __grid_constant__ CUtensorMap tmX, const B1tParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *ops = smem;                                  // [2] operand buffers (A then B)
  uint8_t *stage = ops + B1T_NBUF * B1T_OPB;            // [2] image inputs
  float *red = reinterpret_cast<float *>(ops);          // [4][32][48] (end; over the drained operands)
  float *dbr = reinterpret_cast<float *>(stage + 2 * B1T_STAGE);  // [16 warps][32]
  int *ppoff = reinterpret_cast<int *>(dbr + 16 * 32);  // [216]: x(2 pr - 2, 2 pc - 2) (-1: pad)
  uint64_t *bars = reinterpret_cast<uint64_t *>(ppoff + 216);
  uint64_t *sfull = bars, *sempty = bars + 2, *ofull = bars + 4, *oempty = bars + 4 + B1T_NBUF;
  uint64_t *accf = bars + 4 + 2 * B1T_NBUF;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(accf + 1);

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * p.n_per_cta, n1 = min(p.N, n0 + p.n_per_cta);
  const int nimg = n1 > n0 ? n1 - n0 : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(sfull + s, 1);
      ptx::mbar_init(sempty + s, B1T_BUILD / 32);
    }
    for (int b = 0; b < B1T_NBUF; ++b) {
      ptx::mbar_init(ofull + b, B1T_BUILD / 32);
      ptx::mbar_init(oempty + b, 1);
    }
    ptx::mbar_init(accf, 1);
    ptx::fence_mbar_init();
  }
  // zero the B padding rows 36..47 of every buffer (never written again)
  for (int i = threadIdx.x; i < B1T_NBUF * B1T_KQ * (B1T_N - B1T_UV) * 4; i += blockDim.x) {
    const int b = i / (B1T_KQ * (B1T_N - B1T_UV) * 4), rem = i % (B1T_KQ * (B1T_N - B1T_UV) * 4);
    const int q = rem / ((B1T_N - B1T_UV) * 4), r2 = rem % ((B1T_N - B1T_UV) * 4);
    reinterpret_cast<float *>(ops + b * B1T_OPB + B1T_ABYTES + q * (B1T_N * 16) + B1T_UV * 16)[r2] = 0.f;
  }
  for (int i = threadIdx.x; i < B1T_NCHUNK * B1T_CHUNK; i += blockDim.x)
    ppoff[i] = i < B1T_PP ? 96 - 2 * B1T_XP - 2 + 2 * (i / 14) * B1T_XP + 2 * (i % 14) : -1;
  for (int i = threadIdx.x; i < 2 * 96; i += blockDim.x)
    reinterpret_cast<float *>(stage + (i / 96) * B1T_STAGE)[i % 96] = 0.f;
  if (warp == B1T_BUILD / 32) ptx::tmem_alloc(tslot, 64);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == B1T_BUILD / 32 + 1) {
    // ================= loader: one image per stage (bulk copies; x as a TMA box whose
    // out-of-bounds part -- the border below / right and the pitch padding -- arrives as zeros)
    if (lane == 0) {
      for (int i = 0; i < nimg; ++i) {
        const int s = i & 1;
        const uint32_t ph = (uint32_t)((i >> 1) & 1);
        ptx::mbar_wait(sempty + s, ph ^ 1);
        const int n = n0 + i;
        uint8_t *st = stage + s * B1T_STAGE;
        ptx::mbar_arrive_expect_tx(sfull + s, B1T_STAGE_TX);
        ptx::bulk_g2s(st + B1T_XG, p.g + (int64_t)n * B1T_PP * B1T_K, B1T_G_BYTES, sfull + s);
        for (int w = 0; w < 2; ++w)
          ptx::bulk_g2s(st + B1T_XG + B1T_G_BYTES + w * B1T_C_BYTES, p.code + w * p.code_plane + (int64_t)n * B1T_PP,
                        B1T_C_BYTES, sfull + s);
        ptx::tma_load_3d(ptx::smem_u32(st + B1T_XPRE), &tmX, 0, 0, n, ptx::smem_u32(sfull + s));
      }
    }
  } else if (warp == B1T_BUILD / 32) {
    // ================= MMA issuer: 9 MMAs (M = 128, N = 48, K = 8) per chunk
    const uint32_t idesc = ptx::make_idesc_tf32(128, B1T_N);
    const uint32_t obase = ptx::smem_u32(ops);
    int q = 0;
    for (int i = 0; i < nimg; ++i)
      for (int ci = 0; ci < B1T_NCHUNK; ++ci, ++q) {
        const int b = q % B1T_NBUF;
        ptx::mbar_wait(ofull + b, (uint32_t)((q / B1T_NBUF) & 1));
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint32_t A = obase + b * B1T_OPB, B = A + B1T_ABYTES;
#pragma unroll
          for (int kk = 0; kk < B1T_KQ / 2; ++kk) {
            const uint64_t ad = ptx::make_desc(A + kk * 2 * (128 * 16), 128 * 16, 128);
            const uint64_t bd = ptx::make_desc(B + kk * 2 * (B1T_N * 16), B1T_N * 16, 128);
            ptx::mma_tf32(tmem, ad, bd, idesc, (q | kk) ? 1u : 0u);
          }
          ptx::mma_commit(oempty + b);
        }
        __syncwarp();
      }
    if (ptx::elect_one()) ptx::mma_commit(accf);
    __syncwarp();
  } else {
    // ================= builders
    const int t = threadIdx.x;
    const int kmine = t & 31;  // every A item of this thread has filter k = t % 32
    // the 4-bit code of (k, pp) sits in 32-bit half (k >> 3) & 1 of word k >> 4, at bit 4 (k & 7)
    const int cword = (kmine >> 4) * B1T_PP * 2 + ((kmine >> 3) & 1), cshift = 4 * (kmine & 7);
    // B item j = uv + 36 pq; threads 64.. (one A item each) take j = t - 64 and j + 448
    static_assert(B1T_AITEMS - B1T_BUILD == 64 && B1T_ITEMS - B1T_AITEMS <= 2 * (B1T_BUILD - 64), "B split");
    int bpq0 = -1, buv0 = 0, broff0 = 0, bpq1 = -1, buv1 = 0, broff1 = 0;
    if (t >= 64) {
      const int j0 = t - 64, j1 = j0 + (B1T_BUILD - 64);
      bpq0 = j0 / B1T_UV; buv0 = j0 - bpq0 * B1T_UV; broff0 = buv0 / 6 * B1T_XP + buv0 % 6;
      if (j1 < B1T_ITEMS - B1T_AITEMS) { bpq1 = j1 / B1T_UV; buv1 = j1 - bpq1 * B1T_UV; broff1 = buv1 / 6 * B1T_XP + buv1 % 6; }
    }
    float dbacc = 0.f;
    int q = 0;
    for (int i = 0; i < nimg; ++i) {
      const int s = i & 1;
      ptx::mbar_wait(sfull + s, (uint32_t)((i >> 1) & 1));
      const uint8_t *st = stage + s * B1T_STAGE;
      const float *gs = reinterpret_cast<const float *>(st + B1T_XG);
      const uint32_t *cs = reinterpret_cast<const uint32_t *>(st + B1T_XG + B1T_G_BYTES) + cword;
      const float *xs = reinterpret_cast<const float *>(st);
      for (int ci = 0; ci < B1T_NCHUNK; ++ci, ++q) {
        const int b = q % B1T_NBUF;
        ptx::mbar_wait(oempty + b, (uint32_t)(((q / B1T_NBUF) & 1) ^ 1));
        uint8_t *A = ops + b * B1T_OPB;
        uint8_t *Bm = A + B1T_ABYTES;
        const int pbase = ci * B1T_CHUNK;
        // A items (pq, k): the four candidates d get the masked g of their own winners
        for (int it = t; it < B1T_AITEMS; it += B1T_BUILD) {
          const int pq = it >> 5;
          float v[4][4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int pp = pbase + pq * 4 + e;
            float gv = 0.f;
            uint32_t cd = 0;
            if (pp < B1T_PP) {
              gv = gs[pp * B1T_K + kmine];
              cd = (cs[2 * pp] >> cshift) & 15u;
            }
            dbacc += (cd & 4u) ? gv : 0.f;  // window max > 0 (reading R9)
#pragma unroll
            for (int d = 0; d < 4; ++d) v[d][e] = (cd == 4u + (uint32_t)d) ? gv : 0.f;
          }
#pragma unroll
          for (int d = 0; d < 4; ++d)
            *reinterpret_cast<float4 *>(A + pq * (128 * 16) + (d * 32 + kmine) * 16) =
                make_float4(v[d][0], v[d][1], v[d][2], v[d][3]);
        }
        // B items (uv, pq): x at offset (u, v) = (dr + r, ds + s) from each window origin; the
        // threads with one A item take them (nb0 / nb1 = this thread's first / second, -1: none)
        {
          float v[2][4];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int pq = h ? bpq1 : bpq0;
            if (pq >= 0) {
              const int4 o = *reinterpret_cast<const int4 *>(ppoff + pbase + pq * 4);
              const int rf = h ? broff1 : broff0;
              v[h][0] = o.x >= 0 ? xs[o.x + rf] : 0.f;
              v[h][1] = o.y >= 0 ? xs[o.y + rf] : 0.f;
              v[h][2] = o.z >= 0 ? xs[o.z + rf] : 0.f;
              v[h][3] = o.w >= 0 ? xs[o.w + rf] : 0.f;
            }
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int pq = h ? bpq1 : bpq0;
            if (pq >= 0)
              *reinterpret_cast<float4 *>(Bm + pq * (B1T_N * 16) + (h ? buv1 : buv0) * 16) =
                  make_float4(v[h][0], v[h][1], v[h][2], v[h][3]);
          }
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(ofull + b);
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(sempty + s);  // this warp is done with the image's inputs
    }
    // ================= partials: D[(d, k)][(u, v)] (warps 0-3 = TMEM lane quadrants = d);
    // dF1[k][r][s] = sum_d D[(d, k)][(dr + r, ds + s)]
    dbr[(t >> 5) * 32 + kmine] = dbacc;
    if (warp < 4) {
      if (nimg > 0) ptx::mbar_wait_sleep(accf, 0);
      ptx::tc_fence_after();
      float v[3][16];
      const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
      if (nimg > 0) {
#pragma unroll
        for (int h = 0; h < 3; ++h) ptx::tmem_ld16(ta + 16 * h, v[h]);
      } else {
#pragma unroll
        for (int h = 0; h < 3; ++h)
#pragma unroll
          for (int j = 0; j < 16; ++j) v[h][j] = 0.f;
      }
      float *rw = red + (warp * 32 + lane) * B1T_N;  // [d][k][uv]
#pragma unroll
      for (int h = 0; h < 3; ++h)
#pragma unroll
        for (int j = 0; j < 16; ++j) rw[16 * h + j] = v[h][j];
    }
    ptx::named_bar_sync(1, B1T_BUILD);
    for (int o = t; o < B1T_K * (B1T_RS + 1); o += B1T_BUILD) {
      const int k = o / (B1T_RS + 1), j = o - k * (B1T_RS + 1);
      float sum = 0.f;
      if (j < B1T_RS) {
        const int r = j / 5, s_ = j - r * 5;
        for (int d = 0; d < 4; ++d) sum += red[(d * 32 + k) * B1T_N + ((d >> 1) + r) * 6 + (d & 1) + s_];
      } else {
        for (int w = 0; w < B1T_BUILD / 32; ++w) sum += dbr[w * 32 + k];  // warp order
      }
      p.part[(int64_t)blockIdx.x * B1T_K * (B1T_RS + 1) + o] = sum;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == B1T_BUILD / 32) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 64);
  }
}

size_t b1_tc_smem() {
  static_assert(4 * 32 * B1T_N * 4 <= B1T_NBUF * B1T_OPB, "red fits over the operand buffers");
  return B1T_NBUF * (size_t)B1T_OPB + 2 * (size_t)B1T_STAGE + 16 * 32 * 4 + 216 * 4 + 8 * (5 + 2 * B1T_NBUF) + 16;
}

}  // namespace

// LeNet conv1 geometry only: 28x28 input, 32 filters 5x5 pad 2, 2x2/2 pooling, window codes,
// channel-minor pooled gradient, dense input
bool b1_tc_supported(const ConvArgs &c, const PoolArgs &pa, bool has_codes, bool nhwc, bool csr) {
  static const int env = getenv("SYSML_B1_TC") ? atoi(getenv("SYSML_B1_TC")) : 1;
  if (!env || device_cc_major() != 10 || !has_codes || !nhwc || csr) return false;
  return c.C == 1 && c.H == 28 && c.W == 28 && c.K == 32 && c.R == 5 && c.S == 5 && c.ph == 2 && c.pw == 2 &&
         c.sh == 1 && c.sw == 1 && pa.R == 2 && pa.S == 2 && pa.sh == 2 && pa.sw == 2 && pa.P == 14 &&
         pa.Q == 14 && b1_tc_smem() <= 227 * 1024;
}

// part: >= ctas x 32 x 26 floats; returns the CTA count (the partials to reduce)
sysml_status b1_tc(const ConvArgs &c, const float *x, const float *dpool, const uint64_t *code, int64_t code_plane,
                   float *part, int max_ctas, int *used, cudaStream_t st) {
  if (((uintptr_t)x & 15) || ((uintptr_t)dpool & 15) || ((uintptr_t)code & 15) || (code_plane & 1)) {
    set_error("B1 tensor-core kernel: inputs must be 16-byte aligned");
    return SYSML_ERR_UNSUPPORTED;
  }
  B1tParams p{};
  p.g = dpool;
  p.code = code;
  p.code_plane = code_plane;
  p.part = part;
  p.N = c.N;
  const int ctas = std::max(1, std::min({sm_count(), max_ctas, c.N}));
  p.n_per_cta = (int)ceil_div(c.N, ctas);
  *used = (int)ceil_div(c.N, p.n_per_cta);
  CUtensorMap tmX;
  {
    // x as [N][28][28]; a 40 x 32 box at (0, 0): the image plus zero rows / columns
    const uint64_t dims[3] = {28, 28, (uint64_t)c.N};
    const uint64_t strides[2] = {28 * 4, 784 * 4};
    const uint32_t box[3] = {B1T_XP, 32, 1};
    if (!tmap_encode_f32(&tmX, x, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE)) return SYSML_ERR_CUDA;
  }
  const size_t smem = b1_tc_smem();
  SYSML_TRY(smem_attr(b1_tc_kernel, smem));
  route_note("b1_tc_kernel [tcgen05 TF32, window candidates stacked in M (4 x 32), N = 36 image offsets, %d CTAs]", *used);
  b1_tc_kernel<<<*used, B1T_THREADS, smem, st>>>(tmX, p);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

}  // namespace sysml
