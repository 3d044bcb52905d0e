// conv1_pool.cu -- fused conv2d(C = 1) + bias + relu + 2x2/2 max-pool on tcgen05 with the
// pooling window in the MMA's N dimension (LeNet conv1, BJ cfg 1-3; A1 + A3 of SURVEY §8).
//
// GEMM rows are POOLED windows m = (n, pp, pc).  The 2x2 window's conv outputs are
//   y(2pp+dr, 2pc+ds, k) = sum_{r,s} F[k][r][s] * x_f(2pp + dr + r, 2pc + ds + s)
// (x_f = zero-padded input).  With the row operand
//   A_t[m][e] = x_f(2pp + t, 2pc + e),  e = 0..7  (8 consecutive inputs of one row)
// and the filter operand  B_r[e][(ds, k)] = F[k][r][e - ds]  (0 <= e - ds < S),
//   D_dr[m][(ds, k)] = sum_r A_{r+dr}[m] . B_r      (dr = 0, 1: 2*R MMAs, N = 2*Kp)
// holds all four window values of every filter in ONE TMEM lane, so the epilogue's
// bias + relu + max + first-occurrence argmax (readings R5/R7/R8) is lane-local -- no
// shuffles -- and every lane stores one pooled output per filter.  No frame positions
// are wasted (rows are exactly the pooled windows).
//
// Producer: A_t rows are 8-byte cp.async chunks straight from the NCHW image (pad even,
// W even: a chunk is fully inside or fully padding -> zero-fill); B (all R taps, a few KB)
// is bulk-copied once per CTA.  Warp roles as in conv_tc.cu: 4 producer warps, 1 MMA
// warp, 8 epilogue warps (the two sets take the two M-tiles of a CTA tile).
#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

#include <algorithm>

namespace sysml {

namespace {

constexpr int C1P_THREADS = 544;  // 0-3 producers, 4 MMA, 5-12 epilogue, 13-16 extra CSR producers
constexpr int C1P_CSR_PW = 8;     // CSR producer warps (0-3 and 13-16), each filling every 8th M-tile
constexpr int C1P_MT = 2;  // M-tiles per CTA tile (one per epilogue warp set)

struct C1pParams {
  const float *x;
  const float *fp;    // packed B: [r][quad][NN][4]
  const float *bias;  // may be null
  float *pout;        // pooled output (NCHW, or SPF planes when out_plane > 0)
  int32_t *parg;      // int32 argmax (NCHW pooled layout) or null
  uint64_t *pcode;    // 4-bit window codes (TcSpfIO::code) or null
  int64_t code_plane;
  int N, H, W, K, R, S, ph, pw, P, Q, Pp, Qp;
  int Kp, NN;         // filters padded to 16 / 32; NN = 2*Kp
  int T;              // A row blocks per M-tile = R + 1
  int64_t nwin, ntiles;
  int64_t out_plane;
  int out_Wf, out_Lf, out_off;
  int nstage;
  uint32_t a_bytes, b_bytes;  // per stage (T blocks of 128 rows x 32 B), B total
  int is_csr;                 // CSR input: non-zeros scattered straight into the A_t rows
  sysml_csr csr;
};

__device__ __forceinline__ void st_shared_v4c1(uint32_t addr) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};" ::"r"(addr), "f"(0.f) : "memory");
}

// CSR producer: pixel `col` of image n (value v) into every (window, tap) slot of the M-tile
// at window w0 it feeds.  Window of slot (t, e): pp = (hf - t)/2, pc = (wf - e)/2 with
// t = hf & 1 + 2a, e = wf & 1 + 2b -> row offset m(a, b) = m00 - a*Qp - b.  ACC: add (the
// stored-order rebuild of a row with duplicate columns) instead of store (one writer).
template <bool ACC, class P>
__device__ __forceinline__ void c1p_scatter(const P &p, float *Af, int col, float v, int n, int PpQp,
                                            int64_t w0, float invW, int HW) {
  if (col < 0 || col >= HW) return;
  const int h = __float2int_rz(((float)col + 0.5f) * invW);
  const int wc = col - h * p.W;
  const int hf = h + p.ph, wf = wc + p.pw;
  const int t0 = hf & 1, e0 = wf & 1;
  const int pp0 = (hf - t0) >> 1, pc0 = (wf - e0) >> 1;
  const int m00 = n * PpQp + pp0 * p.Qp + pc0 - (int)w0;
#pragma unroll
  for (int a_ = 0; a_ < 4; ++a_) {
    const int t = t0 + 2 * a_, pp = pp0 - a_;
    if (t >= p.T || pp < 0 || pp >= p.Pp) continue;
#pragma unroll
    for (int b_ = 0; b_ < 4; ++b_) {
      const int e = e0 + 2 * b_, pc = pc0 - b_;
      const int m = m00 - a_ * p.Qp - b_;
      if (pc >= 0 && pc < p.Qp && m >= 0 && m < 128) {
        float *d = Af + t * 1024 + (e >> 2) * 512 + m * 4 + (e & 3);
        if (ACC) *d += v; else *d = v;
      }
    }
  }
}

// One 16-channel group of the pooled epilogue (kept small: the argmax variant is a
// template, not a branch in the unrolled loop, so the executing loop stays compact)
template <bool PARG>
__device__ __forceinline__ void c1p_group(const C1pParams &p, const uint32_t (&v00)[16], const uint32_t (&v01)[16],
                                          const uint32_t (&v10)[16], const uint32_t (&v11)[16],
                                          const float *bias_s, int k0, bool wok, float *poutp, int64_t vstride,
                                          int32_t *pargp, int PpQp, int argbase, int PQ, uint64_t &code) {
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const float b = bias_s[k0 + j];
    // relu (+0.0 for non-positive, R7) then the strict-'>' scan in r-outer / s-inner
    // order (R5): non-negative floats compare as unsigned integers
    const float z0 = __uint_as_float(v00[j]) + b, z1 = __uint_as_float(v01[j]) + b;
    const float z2 = __uint_as_float(v10[j]) + b, z3 = __uint_as_float(v11[j]) + b;
    uint32_t best = __float_as_uint(z0 > 0.f ? z0 : 0.f), c = 0;
    const uint32_t u1 = __float_as_uint(z1 > 0.f ? z1 : 0.f);
    const uint32_t u2 = __float_as_uint(z2 > 0.f ? z2 : 0.f);
    const uint32_t u3 = __float_as_uint(z3 > 0.f ? z3 : 0.f);
    if (u1 > best) { best = u1; c = 1; }
    if (u2 > best) { best = u2; c = 2; }
    if (u3 > best) { best = u3; c = 3; }
    if (wok && k0 + j < p.K) {
      poutp[(int64_t)j * vstride] = __uint_as_float(best);
      if (PARG) pargp[(int64_t)j * PpQp] = argbase + j * PQ + (int)(c >> 1) * p.Q + (int)(c & 1);
    }
    code |= (uint64_t)(((best != 0u) ? 4u : 0u) | c) << (4 * j);
  }
}

__global__ void __launch_bounds__(C1P_THREADS, 1) conv1_pool_kernel(const C1pParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *Bs = smem;                                // R taps x [quad][NN][4]
  uint8_t *stages = smem + ((p.b_bytes + 1023) & ~1023u);
  float *bias_s = reinterpret_cast<float *>(stages + (size_t)p.nstage * p.a_bytes);
  uint64_t *bars = reinterpret_cast<uint64_t *>(bias_s + 64);
  uint64_t *full = bars, *empty = bars + p.nstage;
  uint64_t *accf = bars + 2 * p.nstage, *acce = accf + 2, *bfull = acce + 2;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bfull + 1);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nstage; ++s) {
      ptx::mbar_init(full + s, p.is_csr ? 1 : 128);  // cp.async arrivals / the filling warp
      ptx::mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(accf + b, 1);
      ptx::mbar_init(acce + b, 8);
    }
    ptx::mbar_init(bfull, 1);
    ptx::fence_mbar_init();
  }
  for (int k = threadIdx.x; k < 64; k += blockDim.x)
    bias_s[k] = (p.bias && k < p.K) ? p.bias[k] : 0.f;
  if (warp == 4) ptx::tmem_alloc(tslot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  const int PpQp = p.Pp * p.Qp;

  if ((warp < 4 || warp >= 13) && p.is_csr) {
    // ---------------- CSR producers: producer pw fills every 8th M-tile alone -- zero the T
    // row blocks, then each non-zero (h, w, v) of the overlapping images adds v to the
    // (window, t, e) slots with 2pp + t = h + ph and 2pc + e = w + pw (work ~ nnz,
    // P:168-170; duplicates summed, reading R15)
    if (threadIdx.x == 0) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      ptx::mbar_arrive_expect_tx(bfull, p.b_bytes);
      ptx::bulk_g2s(Bs, p.fp, p.b_bytes, bfull);
    }
    const int HW = p.H * p.W;
    const float invW = 1.0f / (float)p.W;
    const int pw = warp < 4 ? warp : warp - 9;  // 0..7
    for (int64_t it = 0;; ++it) {
      const int64_t tile = blockIdx.x + it * gridDim.x;
      if (tile >= p.ntiles) break;
      for (int i = 0; i < C1P_MT; ++i) {
        const int mine = (int)(it * C1P_MT + i);
        if (mine % C1P_CSR_PW != pw) continue;
        const int stage = mine % p.nstage;
        const uint32_t phase = (uint32_t)((mine / p.nstage) & 1);
        ptx::mbar_wait(empty + stage, phase ^ 1);
        uint8_t *As = stages + (size_t)stage * p.a_bytes;
        const uint32_t A = ptx::smem_u32(As);
        for (int q = lane; q < (int)(p.a_bytes / 16); q += 32) st_shared_v4c1(A + q * 16);
        __syncwarp();
        const int64_t w0 = (tile * C1P_MT + i) * 128;
        if (w0 < p.nwin) {
          const int n_lo = (int)(w0 / PpQp);
          const int n_hi = (int)min((int64_t)p.N - 1, (w0 + 127) / PpQp);
          float *Af = reinterpret_cast<float *>(As);
          // one input pixel owns distinct (window, tap) slots, so a strictly increasing row
          // has one writer per slot: plain stores.  Rows that are not (unsorted or
          // duplicate columns, reading R15) flag the tile, which lane 0 then rebuilds by
          // summing in stored order: deterministic, no float atomics.
          bool bad = false;
          for (int n = n_lo; n <= n_hi; ++n) {
            const int j0 = __ldg(p.csr.row_ptr + n), j1 = __ldg(p.csr.row_ptr + n + 1);
            int last = -1;
            for (int base = j0; base < j1; base += 8 * 32) {
              int cols[8];
              float vals[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) {  // the batch's loads in flight together
                const int jj = base + lane + 32 * u;
                cols[u] = jj < j1 ? __ldg(p.csr.col_idx + jj) : -1;
                vals[u] = jj < j1 ? __ldg(p.csr.val + jj) : 0.f;
              }
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int up = __shfl_up_sync(0xffffffffu, cols[u], 1);
                const int prev = lane ? up : last;
                last = __shfl_sync(0xffffffffu, cols[u], 31);
                const int jj = base + lane + 32 * u;
                if (jj < j1 && jj > j0 && prev >= cols[u]) bad = true;
              }
              // not unrolled: the 8 x 16 guarded scatter body unrolled thrashed the
              // instruction cache (ncu: 37% of stalls no_instructions, profiles/r01_ncu_csr_pool.txt)
#pragma unroll 1
              for (int u = 0; u < 8; ++u)
                c1p_scatter<false>(p, Af, cols[u], vals[u], n, PpQp, w0, invW, HW);
            }
          }
          if (__any_sync(0xffffffffu, bad)) {  // rebuild in stored order (lane 0)
            __syncwarp();
            for (int q = lane; q < (int)(p.a_bytes / 16); q += 32) st_shared_v4c1(A + q * 16);
            __syncwarp();
            if (lane == 0)
              for (int n = n_lo; n <= n_hi; ++n) {
                const int j1 = __ldg(p.csr.row_ptr + n + 1);
                for (int jj = __ldg(p.csr.row_ptr + n); jj < j1; ++jj)
                  c1p_scatter<true>(p, Af, __ldg(p.csr.col_idx + jj), __ldg(p.csr.val + jj), n, PpQp, w0,
                                    invW, HW);
              }
          }
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(full + stage);
      }
    }
  } else if (warp >= 13) {
    // extra CSR producers: idle on dense input
  } else if (warp < 4) {
    // ---------------- producers: thread tid owns row m = tid of every stage
    const int tid = threadIdx.x;
    if (tid == 0) {
      asm volatile("griddepcontrol.wait;" ::: "memory");  // packed filters (PDL)
      ptx::mbar_arrive_expect_tx(bfull, p.b_bytes);
      ptx::bulk_g2s(Bs, p.fp, p.b_bytes, bfull);
    }
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
      for (int i = 0; i < C1P_MT; ++i) {
        ptx::mbar_wait(empty + stage, phase ^ 1);
        const uint32_t A = ptx::smem_u32(stages + (size_t)stage * p.a_bytes);
        const int64_t w = (tile * C1P_MT + i) * 128 + tid;
        int n = 0, pp = 0, pc = 0;
        const bool wok = w < p.nwin;
        if (wok) {
          n = (int)(w / PpQp);
          const int rem = (int)(w - (int64_t)n * PpQp);
          pp = rem / p.Qp;
          pc = rem - pp * p.Qp;
        }
        const float *xn = p.x + (int64_t)n * p.H * p.W;
        for (int t = 0; t < p.T; ++t) {
          const int h = 2 * pp + t - p.ph;
          const bool hok = wok && h >= 0 && h < p.H;
#pragma unroll
          for (int j = 0; j < 4; ++j) {  // 8-byte chunk j = inputs e = 2j, 2j + 1
            const int c0 = 2 * pc - p.pw + 2 * j;
            const bool ok = hok && c0 >= 0 && c0 + 1 < p.W;
            const uint32_t dst = A + (uint32_t)(t * 4096 + (j >> 1) * 2048 + tid * 16 + (j & 1) * 8);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst),
                         "l"(ok ? xn + (int64_t)h * p.W + c0 : p.x), "r"(ok ? 8u : 0u)
                         : "memory");
          }
        }
        ptx::cp_async_mbar_arrive(full + stage);
        if (++stage == p.nstage) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 4) {
    // ---------------- MMA issuer: D_dr[(ds, k)] = sum_r A_{r+dr} . B_r per M-tile
    const uint32_t idesc = ptx::make_idesc_tf32(128, p.NN);
    const uint32_t sB = ptx::smem_u32(Bs), sA0 = ptx::smem_u32(stages);
    const uint32_t b_tap = (uint32_t)(2 * p.NN * 16);  // bytes per tap r
    ptx::mbar_wait(bfull, 0);
    int stage = 0;
    uint32_t phase = 0, tcount = 0;
    for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++tcount) {
      const uint32_t buf = tcount & 1u, bphase = (tcount >> 1) & 1u;
      ptx::mbar_wait(acce + buf, bphase ^ 1);
      ptx::tc_fence_after();
      for (int i = 0; i < C1P_MT; ++i) {
        ptx::mbar_wait(full + stage, phase);
        ptx::tc_fence_after();
        const uint32_t A = sA0 + (uint32_t)stage * p.a_bytes;
        const uint64_t adesc = ptx::make_desc(A, 2048, 128);
        const uint64_t bdesc = ptx::make_desc(sB, (uint32_t)p.NN * 16, 128);
        for (int dr = 0; dr < 2; ++dr) {
          const uint32_t tm = tmem + buf * 256 + i * 128 + dr * (uint32_t)p.NN;
          for (int r = 0; r < p.R; ++r) {
            if (ptx::elect_one())
              ptx::mma_tf32(tm, adesc + (uint64_t)((r + dr) * 256), bdesc + (uint64_t)(r * (b_tap >> 4)),
                            idesc, r > 0 ? 1u : 0u);
            __syncwarp();
          }
        }
        if (ptx::elect_one()) ptx::mma_commit(empty + stage);
        __syncwarp();
        if (++stage == p.nstage) { stage = 0; phase ^= 1; }
      }
      if (ptx::elect_one()) ptx::mma_commit(accf + buf);
      __syncwarp();
    }
  } else {
    // ---------------- epilogue: set e = M-tile e of the CTA tile; lane = pooled window
    const int qd = warp & 3, eset = (warp - 5) >> 2;
    uint32_t tcount = 0;
    for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++tcount) {
      const uint32_t buf = tcount & 1u, bphase = (tcount >> 1) & 1u;
      ptx::mbar_wait_sleep(accf + buf, bphase);
      __syncwarp();
      ptx::tc_fence_after();
      const int64_t w = (tile * C1P_MT + eset) * 128 + qd * 32 + lane;
      const bool wok = w < p.nwin;
      int n = 0, pp = 0, pc = 0;
      if (wok) {
        n = (int)(w / PpQp);
        const int rem = (int)(w - (int64_t)n * PpQp);
        pp = rem / p.Qp;
        pc = rem - pp * p.Qp;
      }
      const int64_t vbase = p.out_plane > 0
                                ? (int64_t)n * p.out_Lf + (int64_t)(pp + p.out_off) * p.out_Wf + pc + p.out_off
                                : (int64_t)n * p.K * PpQp + (int64_t)pp * p.Qp + pc;
      const int64_t vstride = p.out_plane > 0 ? p.out_plane : PpQp;
      const int PQ = p.P * p.Q;
      const int idx_tl = (2 * pp) * p.Q + 2 * pc;
      const uint32_t tb = tmem + ((uint32_t)(qd * 32) << 16) + buf * 256 + eset * 128;
      for (int k0 = 0; k0 < p.Kp; k0 += 16) {
        uint32_t v00[16], v01[16], v10[16], v11[16];
        ptx::tmem_ld16_issue(tb + (uint32_t)k0, v00);                       // (dr 0, ds 0)
        ptx::tmem_ld16_issue(tb + (uint32_t)(p.Kp + k0), v01);              // (0, 1)
        ptx::tmem_ld16_issue(tb + (uint32_t)(p.NN + k0), v10);              // (1, 0)
        ptx::tmem_ld16_issue(tb + (uint32_t)(p.NN + p.Kp + k0), v11);       // (1, 1)
        ptx::tmem_ld_wait(v00);  // each wait ties its registers to the completed load
        ptx::tmem_ld_wait(v01);
        ptx::tmem_ld_wait(v10);
        ptx::tmem_ld_wait(v11);
        uint64_t code = 0;
        float *poutp = p.pout + vbase + (int64_t)k0 * vstride;
        if (p.parg)
          c1p_group<true>(p, v00, v01, v10, v11, bias_s, k0, wok, poutp, vstride,
                          p.parg + ((int64_t)n * p.K + k0) * PpQp + pp * p.Qp + pc, PpQp, k0 * PQ + idx_tl, PQ, code);
        else
          c1p_group<false>(p, v00, v01, v10, v11, bias_s, k0, wok, poutp, vstride, nullptr, PpQp, 0, PQ, code);
        if (p.pcode && wok) p.pcode[(int64_t)(k0 >> 4) * p.code_plane + w] = code;
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(acce + buf);
    }
  }
  __syncthreads();
  if (warp == 4) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// B_r[e][(ds, k)] = F[k][r][e - ds], packed [r][quad = e/4][NN][4]
__global__ void conv1_pool_pack_kernel(const float *__restrict__ f, float *__restrict__ fp, int K,
                                       int R, int S, int Kp) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int NN = 2 * Kp;
  const int total = R * 2 * NN * 4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int e4 = i & 3, nn = (i >> 2) % NN, q = (i >> 2) / NN % 2, r = (i >> 2) / NN / 2;
    const int e = q * 4 + e4, ds = nn / Kp, k = nn - ds * Kp, s = e - ds;
    fp[i] = (k < K && s >= 0 && s < S) ? f[(k * R + r) * S + s] : 0.f;
  }
}

struct C1pPlan {
  C1pParams p;
  size_t smem;
  size_t fp_bytes;
  bool ok;
};

C1pPlan plan_c1p(const ConvArgs &a, const PoolArgs *pool) {
  C1pPlan pl{};
  pl.ok = false;
  C1pParams &p = pl.p;
  if (!pool || a.C != 1 || a.sh != 1 || a.sw != 1 || a.K > 32 || a.R > 7 || a.S > 7) return pl;
  if (pool->R != 2 || pool->S != 2 || pool->sh != 2 || pool->sw != 2 || pool->ph || pool->pw) return pl;
  if ((a.pw & 1) || (a.W & 1)) return pl;  // 8-byte chunks fully inside or fully padding
  p.N = a.N; p.H = a.H; p.W = a.W; p.K = a.K; p.R = a.R; p.S = a.S; p.ph = a.ph; p.pw = a.pw;
  p.P = a.P; p.Q = a.Q; p.Pp = pool->P; p.Qp = pool->Q;
  p.Kp = a.K <= 16 ? 16 : 32;
  p.NN = 2 * p.Kp;
  p.T = a.R + 1;
  p.nwin = (int64_t)a.N * p.Pp * p.Qp;
  p.ntiles = ceil_div(p.nwin, 128 * C1P_MT);
  p.a_bytes = (uint32_t)(p.T * 4096);
  p.b_bytes = (uint32_t)(a.R * 2 * p.NN * 16);
  const size_t fixed = ((p.b_bytes + 1023) & ~1023u) + 64 * 4 + 8 * 24 + 64;
  p.nstage = (int)std::min<size_t>(8, (225 * 1024 - fixed) / p.a_bytes);
  if (p.nstage < 2) return pl;
  pl.smem = fixed + (size_t)p.nstage * p.a_bytes + 1024;
  pl.fp_bytes = align_up(p.b_bytes, 256);
  pl.ok = true;
  return pl;
}

}  // namespace

bool conv1_pool_supported(const ConvArgs &a, const PoolArgs *pool) {
  return device_cc_major() == 10 && plan_c1p(a, pool).ok && getenv("SYSML_NO_C1P") == nullptr;
}

size_t conv1_pool_ws(const ConvArgs &a, const PoolArgs *pool) {
  const C1pPlan pl = plan_c1p(a, pool);
  return pl.ok ? pl.fp_bytes : 0;
}

sysml_status conv1_pool(const ConvArgs &a, const PoolArgs *pool, const float *x, const float *f,
                        const float *bias, float *pout, int32_t *parg, void *ws, cudaStream_t st,
                        const TcSpfIO *io, const sysml_csr *csr) {
  C1pPlan pl = plan_c1p(a, pool);
  if (!pl.ok) {
    set_error("conv1+pool (pool-in-N) kernel: unsupported shape");
    return SYSML_ERR_UNSUPPORTED;
  }
  if (!csr && ((uintptr_t)x & 7)) {
    set_error("conv1+pool kernel: input must be 8-byte aligned");
    return SYSML_ERR_UNSUPPORTED;
  }
  C1pParams p = pl.p;
  p.x = x;
  if (csr) {
    p.is_csr = 1;
    p.csr = *csr;
  }
  p.fp = reinterpret_cast<const float *>(ws);
  p.bias = bias;
  p.pout = pout;
  p.parg = parg;
  if (io) {
    p.out_plane = io->out_plane;
    p.out_Wf = io->out_Wf;
    p.out_Lf = io->out_Lf;
    p.out_off = io->out_off;
    p.pcode = io->code;
    p.code_plane = io->code_plane;
  }
  conv1_pool_pack_kernel<<<8, 256, 0, st>>>(f, reinterpret_cast<float *>(ws), a.K, a.R, a.S, p.Kp);
  SYSML_LAUNCH_CHECK();
  SYSML_TRY(smem_attr(conv1_pool_kernel, pl.smem));
  const int grid = (int)std::min<int64_t>(p.ntiles, sm_count());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(C1P_THREADS);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  route_note("conv1_pool_kernel [tcgen05 TF32 pool-in-N%s]", p.is_csr ? ", CSR producer" : "");
  SYSML_CUDA(cudaLaunchKernelEx(&cfg, conv1_pool_kernel, p));
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

}  // namespace sysml
