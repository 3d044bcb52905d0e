// sn_tmem.cu -- narrow-filter shifted-window convolution with the A operand in TMEM: the
// LeNet step's conv2 bwd_data (B2d, S:174-181 = conv(dY, rot180(F)^T), the dominant stage).
//
// Why: with M = 128 and the A tile in shared memory, a tcgen05 TF32 MMA costs
// max(32 + N/4, N/2) clocks: the 4 KB A read dominates for N < 128, and the
// LeNet conv2 backward has only 32 output channels.  The SN fold (taps s in N: N = S*32 = 160)
// makes the MMA math bound, but the A and B tiles still stream through shared memory together
// with the producers' writes, and B2d ran its MMA loop at ~3x the math time.  Here
//   * A lives in TMEM: tcgen05.mma reads it from the tensor memory (kind::tf32, A "TS" form;
//     validated by tools/mma_tmemA.cu: N = 64..256 at the math rate).  The producers load the
//     input rows straight from the SPF planes into registers (coalesced 4-byte loads, thread =
//     TMEM lane = GEMM row) and write the R row-shifted copies of each 8-channel chunk with
//     tcgen05.st -- no shared memory on the A path at all;
//   * the whole packed filter bank stays resident in shared memory (loaded once per CTA), so
//     B costs no L2 traffic and only the MMA's own B reads touch shared memory;
//   * accumulators are double-buffered (2 x S*NFpad columns) next to a 4-stage ring of A
//     chunks (R*8 columns each), so the SN epilogue of tile t overlaps the MMAs of tile t+1.
//
// GEMM (SN mode, as in conv_tc.cu): D'[m][(s, k)] = sum_{chunk, r} A_r[m][c] . B_r[(s,k)][c],
// A_r[m][c] = x[c][g0 + m + r*Wf] (frame position, SPF plane, stored position = frame pos +
// in_shift), and the epilogue adds Y[g0 + l][k] = b[k] + sum_s D'[l + s][(s, k)] for
// l < 128 - (S-1) (tiles overlap by S-1 rows).
//
// Warps (persistent, 1 CTA/SM): 4*ST_PSETS producers (TMEM lane quadrant = warp % 4; set w/4
// fills the chunks q with q % ST_PSETS == set, so ST_PSETS chunks' loads are in flight), one MMA
// issuer, 8 epilogue warps (quadrant = warp % 4; the two sets split the 16-channel groups).
#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

#include <algorithm>

#ifndef SN_DIRECT13
#define SN_DIRECT13 1  // copies 1, 3 loaded directly (L1 hits) instead of half-warp shuffles: fewer MIO ops
#endif
#include <cstdio>
#include <cstdlib>

namespace sysml {

namespace {

constexpr int ST_PSETS = 4;                            // producer warp sets (chunks in flight)
constexpr int ST_PWARPS = 4 * ST_PSETS;
constexpr int ST_MMAW = ST_PWARPS;                     // MMA warp index
constexpr int ST_THREADS = 32 * (ST_PWARPS + 1 + 8);
constexpr int ST_ASTAGES = 4;
// a producer set reaches chunk j only after its chunk j - ST_PSETS, produced after the
// consumption of chunk j - ST_PSETS - ST_ASTAGES; the stage's parity wait is unambiguous only
// when that is >= j - 2 * ST_ASTAGES, i.e. ST_PSETS <= ST_ASTAGES
static_assert(ST_PSETS <= ST_ASTAGES, "producer sets would run a full ring ahead");
constexpr int ST_MAXR = 5;                          // A copies per chunk (R <= 5)
constexpr int ST_XCH = 2 * 4 * 4 * 4 * 16;          // [set][quadrant][s 1..4][row < 4][16]

struct StParams {
  const float *x;      // SPF planes [Cin][plane]
  int64_t plane;
  int in_shift;
  const float *fp;     // packed B: [chunk][r][quad][NN][4]
  const float *bias;   // nullable
  float *y;
  int y_nhwc;          // 1: y channel-minor [n][P*Q][K]
  int Cin, K, R, S, NFpad, NN, nchunk;
  int Wf, Lf, P, Q;
  int64_t G, ntiles;
  int cta_pos;
  uint32_t b_bytes;
  uint32_t acc_cols;   // first A-stage column (= 2 * NN rounded to 32)
  long long *clk;      // optional per-CTA cycle counters (SYSML_TC_PROFILE)
};

__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
               "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
               : "memory");
}

__global__ void __launch_bounds__(ST_THREADS, 1) sn_tmem_kernel(const StParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint8_t *Bs = smem;                                                   // resident filters
  float *xch = reinterpret_cast<float *>(smem + ((p.b_bytes + 15) & ~15u));   // epilogue exchange
  float *bias_s = xch + ST_XCH;                                               // [64]
  uint64_t *bars = reinterpret_cast<uint64_t *>(bias_s + 64);
  uint64_t *bfull = bars;                       // B resident
  uint64_t *afull = bars + 1;                   // [ST_ASTAGES]
  uint64_t *aempty = afull + ST_ASTAGES;        // [ST_ASTAGES]
  uint64_t *accf = aempty + ST_ASTAGES;         // [2]
  uint64_t *acce = accf + 2;                    // [2]
  uint32_t *tslot = reinterpret_cast<uint32_t *>(acce + 2);

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    ptx::mbar_init(bfull, 1);
    for (int s = 0; s < ST_ASTAGES; ++s) {
      ptx::mbar_init(afull + s, 128);  // one producer set: 4 warps x 32 threads
      ptx::mbar_init(aempty + s, 1);   // tcgen05.commit
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(accf + b, 1);
      ptx::mbar_init(acce + b, 8);     // the 8 epilogue warps
    }
    ptx::fence_mbar_init();
  }
  for (int k = threadIdx.x; k < 64; k += blockDim.x) bias_s[k] = (p.bias && k < p.K) ? p.bias[k] : 0.f;
  if (warp == ST_MMAW) ptx::tmem_alloc(tslot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // packed filters ready (PDL)
    ptx::mbar_arrive_expect_tx(bfull, p.b_bytes);
    for (uint32_t off = 0; off < p.b_bytes; off += 32768u) {
      const uint32_t n = min(32768u, p.b_bytes - off);
      ptx::bulk_g2s(const_cast<uint8_t *>(Bs) + off, reinterpret_cast<const uint8_t *>(p.fp) + off, n, bfull);
    }
  }
  const uint32_t acol = p.acc_cols;        // A stage s: columns acol + s*R*8 .. + R*8
  const uint32_t astride = (uint32_t)(p.R * 8);

  if (warp < ST_PWARPS) {
    // ================= producers: thread = GEMM row m of its quadrant; set = chunk % ST_PSETS
    const int qd = warp & 3, set = warp >> 2;
    const int m = qd * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qd * 32) << 16);
    const int plane = (int)p.plane;  // Cin * plane < 2^31 (launcher)
    const int64_t my_tiles = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t qtot = my_tiles * p.nchunk;  // this CTA's chunks, in MMA order
    if (p.Wf == 16 && p.R == 5) {
      // Wf = 16: copy r of row m is position m + 16 r, so copies 0, 2, 4 are the 32-position
      // blocks of this warp and the next two (one coalesced load each per channel) and copies
      // 1, 3 are half-block shifts of them (one shuffle each): 3 loads per channel, not 5.  The
      // set's next chunk is loaded before the current one is stored (two register buffers).
      // per-channel plane offsets (loop invariant); chunk -> (tile, channel block) is advanced
      // incrementally (no 64-bit division per chunk): the producers are issue bound
      int coff[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) coff[c] = c * plane;
#if SN_DIRECT13
      float d1[8], d3[8];
#endif
      auto load = [&](int64_t tile, int ch, float (&v)[3][8]) {
        const int gp = (int)(tile * p.cta_pos) + m + p.in_shift;  // plane position of copy 0
        const float *xc = p.x + (int64_t)(ch * 8) * plane;
        if (gp >= 0 && gp + 64 < plane && ch * 8 + 8 <= p.Cin) {
          const float *xb = xc + gp;
#pragma unroll
          for (int b = 0; b < 3; ++b)
#pragma unroll
            for (int c = 0; c < 8; ++c) v[b][c] = __ldg(xb + (32 * b + coff[c]));
#if SN_DIRECT13
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            d1[c] = __ldg(xb + (16 + coff[c]));
            d3[c] = __ldg(xb + (48 + coff[c]));
          }
#endif
        } else {
          const int nc = min(8, p.Cin - ch * 8);
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const int sv = gp + 32 * b;
            const bool ok = sv >= 0 && sv < plane;
#pragma unroll
            for (int c = 0; c < 8; ++c) v[b][c] = (ok && c < nc) ? __ldg(xc + (sv + coff[c])) : 0.f;
          }
#if SN_DIRECT13
          const int s1 = gp + 16, s3 = gp + 48;
          const bool ok1 = s1 >= 0 && s1 < plane, ok3 = s3 >= 0 && s3 < plane;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            d1[c] = (ok1 && c < nc) ? __ldg(xc + (s1 + coff[c])) : 0.f;
            d3[c] = (ok3 && c < nc) ? __ldg(xc + (s3 + coff[c])) : 0.f;
          }
#endif
        }
      };
      auto store = [&](int64_t q, const float (&v)[3][8]) {
        const int stage = (int)(q % ST_ASTAGES);
        const uint32_t ph = (uint32_t)((q / ST_ASTAGES) & 1);
#if SN_DIRECT13
        float (&w1)[8] = d1, (&w3)[8] = d3;
#else
        float w1[8], w3[8];
        const int src = (lane + 16) & 31;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          w1[c] = __shfl_sync(0xffffffffu, lane >= 16 ? v[0][c] : v[1][c], src);
          w3[c] = __shfl_sync(0xffffffffu, lane >= 16 ? v[1][c] : v[2][c], src);
        }
#endif
        ptx::mbar_wait(aempty + stage, ph ^ 1);
        ptx::tc_fence_after();
        const uint32_t ta = trow + acol + (uint32_t)stage * astride;
        tmem_st8(ta + 0, v[0]);
        tmem_st8(ta + 8, w1);
        tmem_st8(ta + 16, v[1]);
        tmem_st8(ta + 24, w3);
        tmem_st8(ta + 32, v[2]);
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(afull + stage);
      };
      int64_t tile = blockIdx.x;
      int ch = set;
      while (ch >= p.nchunk) { ch -= p.nchunk; tile += gridDim.x; }
      for (int64_t q = set; q < qtot; q += ST_PSETS) {
        float va[3][8];
        load(tile, ch, va);
        store(q, va);
        ch += ST_PSETS;
        while (ch >= p.nchunk) { ch -= p.nchunk; tile += gridDim.x; }
      }
    } else {
      int64_t q = 0;  // CTA-local chunk counter (over all tiles)
      for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
        const int64_t gm = tile * p.cta_pos + m;
        int si[ST_MAXR];
#pragma unroll
        for (int r = 0; r < ST_MAXR; ++r) {
          const int64_t v = gm + (int64_t)r * p.Wf + p.in_shift;
          si[r] = (r < p.R && gm < p.G && v >= 0 && v < p.plane) ? (int)v : -1;
        }
        for (int ch = 0; ch < p.nchunk; ++ch, ++q) {
          if ((int)(q % ST_PSETS) != set) continue;
          const int stage = (int)(q % ST_ASTAGES);
          const uint32_t ph = (uint32_t)((q / ST_ASTAGES) & 1);
          const int nc = min(8, p.Cin - ch * 8);
          const float *xc = p.x + (int64_t)(ch * 8) * plane;
          float v[ST_MAXR][8];
#pragma unroll
          for (int r = 0; r < ST_MAXR; ++r) {
            const float *xr = xc + (si[r] >= 0 ? si[r] : 0);
#pragma unroll
            for (int c = 0; c < 8; ++c) v[r][c] = (si[r] >= 0 && c < nc) ? __ldg(xr + c * plane) : 0.f;
          }
          ptx::mbar_wait(aempty + stage, ph ^ 1);
          ptx::tc_fence_after();
          const uint32_t ta = trow + acol + (uint32_t)stage * astride;
#pragma unroll
          for (int r = 0; r < ST_MAXR; ++r)
            if (r < p.R) tmem_st8(ta + (uint32_t)(r * 8), v[r]);
          ptx::tmem_st_wait();
          ptx::tc_fence_before();
          ptx::mbar_arrive(afull + stage);
        }
      }
    }
  } else if (warp == ST_MMAW) {
    // ================= MMA issuer (whole warp in the loop; one elected lane issues)
    ptx::mbar_wait(bfull, 0);
    const uint32_t idesc = ptx::make_idesc_tf32(128, p.NN);
    const uint64_t b0 = ptx::make_desc(ptx::smem_u32(Bs), (uint32_t)p.NN * 16, 128);
    const uint64_t bstep = (uint64_t)((2u * (uint32_t)p.NN * 16u) >> 4);  // next (chunk, r) block
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
      const uint32_t d = tmem + buf * (uint32_t)p.NN;
      uint64_t bd = b0;
      uint32_t acc = 0;
      for (int ch = 0; ch < p.nchunk; ++ch, ++q) {
        const int stage = (int)(q % ST_ASTAGES);
        const long long t1 = clock64();
        ptx::mbar_wait(afull + stage, (uint32_t)((q / ST_ASTAGES) & 1));
        t_afull += clock64() - t1;
        ptx::tc_fence_after();
        const uint32_t ta = tmem + acol + (uint32_t)stage * astride;
        for (int r = 0; r < p.R; ++r) {
          if (ptx::elect_one()) mma_tf32_ts(d, ta + (uint32_t)(r * 8), bd, idesc, acc);
          __syncwarp();
          acc = 1u;
          bd += bstep;
        }
        if (ptx::elect_one()) ptx::mma_commit(aempty + stage);
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
    // ================= epilogue: SN shift-add, lane = accumulator row of its quadrant
    const int qd = warp & 3, eset = (warp - ST_MMAW - 1) >> 2;
    const int nc16 = p.NFpad / 16, PQ = p.P * p.Q;
    float *xs = xch + eset * (4 * 4 * 4 * 16);
    auto xidx = [&](int qq, int s_, int row) { return ((qq * 4 + (s_ - 1)) * 4 + row) * 16; };
    uint32_t tcount = 0;
    for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++tcount) {
      const uint32_t buf = tcount & 1u, bph = (tcount >> 1) & 1u;
      const int64_t g0 = tile * p.cta_pos;
      ptx::mbar_wait_sleep(accf + buf, bph);
      __syncwarp();
      ptx::tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(qd * 32) << 16) + buf * (uint32_t)p.NN;
      for (int c16 = eset; c16 < nc16; c16 += 2) {
        // rows l + s of this quadrant by shuffles; lanes < S-1 publish their s >= 1 values for
        // the quadrant above (every block is loaded once), whose rows l + s >= 32 come from it
        const int k0 = c16 * 16;
        float acc[16];
        ptx::tmem_ld16(tbase + (uint32_t)(c16 * 16), acc);
        for (int s_ = 1; s_ < p.S; ++s_) {
          float t[16];
          ptx::tmem_ld16(tbase + (uint32_t)(s_ * p.NFpad + c16 * 16), t);
          if (lane < p.S - 1) {
            float4 *dst = reinterpret_cast<float4 *>(xs + xidx(qd, s_, lane));
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) dst[j4] = make_float4(t[4 * j4], t[4 * j4 + 1], t[4 * j4 + 2], t[4 * j4 + 3]);
          }
          const bool from_next = lane + s_ >= 32;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float vv = __shfl_down_sync(0xffffffffu, t[j], s_);
            if (!from_next) acc[j] += vv;
          }
        }
        ptx::named_bar_sync(2 + eset, 128);
        if (qd < 3) {  // quadrant 3: rows >= cta_pos need no next-quadrant terms
          for (int s_ = 1; s_ < p.S; ++s_) {
            if (lane + s_ >= 32) {
              const float4 *src = reinterpret_cast<const float4 *>(xs + xidx(qd + 1, s_, lane + s_ - 32));
#pragma unroll
              for (int j4 = 0; j4 < 4; ++j4) {
                const float4 u = src[j4];
                acc[4 * j4] += u.x; acc[4 * j4 + 1] += u.y; acc[4 * j4 + 2] += u.z; acc[4 * j4 + 3] += u.w;
              }
            }
          }
        }
        const int l = qd * 32 + lane;
        const int64_t g = g0 + l;
        if (l < p.cta_pos && g < p.G) {
          const int n = (int)(g / p.Lf), rem = (int)(g - (int64_t)n * p.Lf);
          const int hh = rem / p.Wf, qq = rem - hh * p.Wf;
          if (hh < p.P && qq < p.Q) {
            if (p.y_nhwc) {
              float4 *yp = reinterpret_cast<float4 *>(p.y + ((int64_t)n * PQ + (int64_t)hh * p.Q + qq) * p.K + k0);
#pragma unroll
              for (int j4 = 0; j4 < 4; ++j4)
                if (k0 + 4 * j4 + 4 <= p.K)
                  yp[j4] = make_float4(acc[4 * j4] + bias_s[k0 + 4 * j4], acc[4 * j4 + 1] + bias_s[k0 + 4 * j4 + 1],
                                       acc[4 * j4 + 2] + bias_s[k0 + 4 * j4 + 2], acc[4 * j4 + 3] + bias_s[k0 + 4 * j4 + 3]);
            } else {
              float *yp = p.y + (int64_t)n * p.K * PQ + (int64_t)hh * p.Q + qq + (int64_t)k0 * PQ;
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (k0 + j < p.K) yp[(int64_t)j * PQ] = acc[j] + bias_s[k0 + j];
            }
          }
        }
        ptx::named_bar_sync(2 + eset, 128);  // before the next group overwrites the dump
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(acce + buf);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == ST_MMAW) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// packed(chunk, r, quad, n = s*NFpad + k, e) = W[k][c = chunk*8 + quad*4 + e][r][s] of the conv
// being computed (flip: W[k][c][r][s] = F[c][k][R-1-r][S-1-s], the bwd_data filters)
__global__ void sn_tmem_pack_kernel(const float *__restrict__ f, float *__restrict__ fp, int Kout, int Cin,
                                    int R, int S, int NFpad, int nchunk, int flip) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int NN = S * NFpad;
  const int64_t total = (int64_t)nchunk * R * 2 * NN * 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int e = (int)(t % 4); t /= 4;
    const int n = (int)(t % NN); t /= NN;
    const int g = (int)(t % 2); t /= 2;
    const int r = (int)(t % R); t /= R;
    const int ch = (int)t;
    const int s_ = n / NFpad, j = n % NFpad, c = ch * 8 + g * 4 + e;
    float v = 0.f;
    if (j < Kout && c < Cin)
      v = flip ? f[(((int64_t)c * Kout + j) * R + (R - 1 - r)) * S + (S - 1 - s_)]
               : f[(((int64_t)j * Cin + c) * R + r) * S + s_];
    fp[i] = v;
  }
}

struct StPlan {
  StParams p;
  size_t smem, fp_bytes;
  bool ok;
};

// a = the bwd_data problem (fwd geometry); the conv computed is dX = conv(dY, W), Cin = a.K,
// Kout = a.C, pad R-1-ph, on the output frame of the SPF layout (Wf, Lf)
StPlan plan_sn_tmem(const ConvArgs &a, int Wf, int Lf) {
  StPlan pl{};
  pl.ok = false;
  StParams &p = pl.p;
  if (a.sh != 1 || a.sw != 1 || a.R > ST_MAXR || a.S < 2 || a.S > 5 || a.C > 32) return pl;
  p.Cin = a.K;
  p.K = a.C;
  p.R = a.R;
  p.S = a.S;
  p.NFpad = a.C <= 16 ? 16 : 32;
  p.NN = p.S * p.NFpad;
  p.nchunk = (p.Cin + 7) / 8;
  p.Wf = Wf;
  p.Lf = Lf;
  p.P = a.H;
  p.Q = a.W;
  p.G = (int64_t)a.N * Lf;
  p.cta_pos = 128 - (p.S - 1);
  p.ntiles = ceil_div(p.G, p.cta_pos);
  p.acc_cols = (uint32_t)((2 * p.NN + 31) / 32 * 32);
  if (p.acc_cols + (uint32_t)(ST_ASTAGES * p.R * 8) > 512) return pl;
  p.b_bytes = (uint32_t)((size_t)p.nchunk * p.R * 2 * p.NN * 16);
  pl.fp_bytes = align_up(p.b_bytes, 256);
  pl.smem = ((p.b_bytes + 15) & ~15u) + (size_t)ST_XCH * 4 + 64 * 4 + 8 * (1 + 2 * ST_ASTAGES + 4) + 16;
  if (pl.smem > 227 * 1024) return pl;
  pl.ok = true;
  return pl;
}

}  // namespace

bool sn_tmem_supported(const ConvArgs &a, int Wf, int Lf) {
  if (device_cc_major() != 10 || getenv("SYSML_NO_SN_TMEM")) return false;
  return plan_sn_tmem(a, Wf, Lf).ok;
}

size_t sn_tmem_ws(const ConvArgs &a, int Wf, int Lf) {
  const StPlan pl = plan_sn_tmem(a, Wf, Lf);
  return pl.ok ? pl.fp_bytes : 0;
}

sysml_status sn_tmem_bwd_data_spf(const ConvArgs &a, const TcSpfIO &io, int Wf, int Lf, const float *f,
                                  const float *dy, float *dx, void *ws, cudaStream_t st) {
  StPlan pl = plan_sn_tmem(a, Wf, Lf);
  if (!pl.ok || io.in_plane <= 0 || (int64_t)pl.p.Cin * io.in_plane >= (1ll << 31)) {
    set_error("SN/TMEM bwd_data: unsupported shape");
    return SYSML_ERR_UNSUPPORTED;
  }
  StParams p = pl.p;
  p.x = dy;
  p.plane = io.in_plane;
  p.in_shift = io.in_shift;
  p.y = dx;
  p.y_nhwc = io.out_nhwc;
  p.bias = nullptr;
  if (p.y_nhwc && ((p.K & 3) || ((uintptr_t)dx & 15))) {
    set_error("SN/TMEM bwd_data: channel-minor output needs K %% 4 == 0 and a 16-byte aligned dx");
    return SYSML_ERR_UNSUPPORTED;
  }
  float *fp = reinterpret_cast<float *>(ws);
  {
    const int64_t total = (int64_t)p.nchunk * p.R * 2 * p.NN * 4;
    sn_tmem_pack_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 4 * sm_count()), 256, 0, st>>>(
        f, fp, p.K, p.Cin, p.R, p.S, p.NFpad, p.nchunk, 1);
    SYSML_LAUNCH_CHECK();
  }
  p.fp = fp;
  SYSML_TRY(smem_attr(sn_tmem_kernel, pl.smem));
  const int grid = (int)std::min<int64_t>(p.ntiles, sm_count());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(ST_THREADS);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap the pack kernel
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  route_note("sn_tmem_kernel [tcgen05 TF32, A in TMEM, resident filters, SN N=%d, %lld tiles on %d CTAs]", p.NN,
             (long long)p.ntiles, grid);
  static long long *dclk = nullptr;
  const bool prof = getenv("SYSML_TC_PROFILE") != nullptr;
  if (prof && !dclk) cudaMalloc(&dclk, sizeof(long long) * 5 * 1024);
  p.clk = prof ? dclk : nullptr;
  SYSML_CUDA(cudaLaunchKernelEx(&cfg, sn_tmem_kernel, p));
  SYSML_LAUNCH_CHECK();
  if (prof) {
    static long long h[5 * 1024];
    cudaMemcpyAsync(h, dclk, sizeof(long long) * 5 * 1024, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double a[5] = {0, 0, 0, 0, 0};
    for (int b = 0; b < grid; ++b) {
      for (int j = 0; j < 4; ++j) a[j] += (double)h[b * 4 + j] / grid;
      a[4] += (double)h[4 * 1024 + b] / grid;
    }
    fprintf(stderr, "[sn_tmem] mma_wait_acce %.0f mma_wait_afull %.0f mma_total %.0f prod_load %.0f prod_store %.0f\n",
            a[0], a[1], a[2], a[3], a[4]);
  }
  return SYSML_OK;
}

}  // namespace sysml
