// conv_tc.cu -- tcgen05 TF32 implicit-GEMM convolution for sm_100a:
//   K3 forward (+ fused bias / relu / max-pool epilogue), K6 bwd_data, K5 bwd_filter.
//
// The paper's GPU backend lowers conv2d to GEMMs via im2col (cuDNN);
// here the lowering is implicit and "shifted-window": no im2col is built, not even
// in shared memory.
//
// Frame.  Output positions are laid out in a stacked, padded frame: image n owns
// Hs rows of Wf = W + pw columns (Hs >= H + ph), so output (n,p,q) is frame
// position g = (n*Hs + p)*Wf + q, and the input value feeding it through tap (r,s)
// sits at frame position g + (r*Wf + s) of the input frame (same geometry; zero
// padding comes from frame rows/columns that decode outside the image: the right
// padding of a row is the left padding of the next row, the bottom padding of an
// image is the top padding of the next).  Every tap of the convolution is the SAME
// matrix shifted by a constant number of rows.
//
// Forward GEMM.  D[m = position][n = out channel] += sum_{tap,c} A[m + d_tap][c] B[n][(tap,c)]
//   A: a halo of the input frame for 8 channels, staged once per K-chunk in shared
//      memory in the UMMA K-major no-swizzle layout [channel quad][position][4 ch]
//      (16 B per position).  Tap t is the same bytes with the descriptor start
//      advanced by 16*d_tap, so each staged element feeds R*S MMAs.  The 8-row
//      group stride (SBO) is 16 B x 8 in "linear" M-tiles (128 consecutive
//      positions) or one frame row (16 B x Wf) in "2-D" M-tiles (16 rows x 8
//      columns), which puts each 2x2 pool window inside one warp (lanes l, l+1,
//      l+8, l+9) so the fused max-pool is four shuffles.
//   B: filters, repacked once into [filter tile][chunk][tap][quad][filter][4 ch] and
//      streamed per chunk with one bulk async copy (cp.async.bulk, TMA 1-D).
//   D: fp32 accumulators in TMEM; MT M-tiles share every B chunk (MT*NF <= 512 cols).
//   Roles (TC_FWD_THREADS = 416 threads, persistent, 1 CTA/SM): warps 0-3 stage A and
//   issue the B copy (the staged modes split them into 16-byte loaders and transposers);
//   warp 4 issues tcgen05.mma (the whole warp runs the loop, one elected lane issues);
//   warps 5-12 drain TMEM in the epilogue, two per lane quadrant.
// bwd_data = the forward kernel on dY with the filter bank transposed and
// rotated 180 degrees, padding R-1-ph (stride 1).
//
// bwd_filter GEMM.  For tap (r,s): D_rs[k][c] = sum_g dY[k][g] X[c][g + d_rs]
//   over output frame positions g.  M = filters: A = dY chunk, K-major [pos quad]
//   [row][4 pos]; when K < 128 the 128 TMEM lanes hold 128/K copies of the filters,
//   copy j being dY shifted by j*Wf, so one MMA yields taps (r,s),(r+1,s),... (the
//   shift by a frame row moves the tap down one row).  N = channels: B = the X halo
//   in the MN-major layout [channel quad][position][4 ch], the tap shift again being
//   a descriptor offset.  One accumulator per tap group; the position range is split
//   over CTAs and the partials are summed in a fixed order (deterministic).
#include <stdio.h>

#include <cmath>
#include <mutex>
#include <string.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace sysml {

namespace {

constexpr int TC_THREADS = 256;      // bwd_filter kernel: 4 producer warps + MMA/epilogue warps
constexpr int TC_FWD_THREADS = 416;  // forward kernel: 4 producer, 1 MMA, 8 epilogue warps
constexpr int TC_EPI_WARPS = 8;      // two per TMEM lane quadrant; they split the M-tiles
constexpr int SMEM_BUDGET = 225 * 1024;
// routed SPF input (NEXT-1): per-tile staging of the pooled gradient rows [<=RT_MAXW][64] and
// the window codes [4][RT_MAXW], double-buffered across tiles
constexpr int RT_MAXW = 96;
constexpr int RT_SLOT = RT_MAXW * 64 * 4 + 4 * RT_MAXW * 8;  // 27,648 B
constexpr int RT_BYTES = 2 * RT_SLOT;

__device__ __forceinline__ void st_shared_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

// =====================================================================================
// Forward kernel
// =====================================================================================
struct TcFwdParams {
  const float *x;
  const float *fp;    // packed filters
  const float *bias;  // may be null
  float *y;           // plain output (N x K*P*Q) or null
  float *pout;        // pooled output or null
  int32_t *parg;      // pooled argmax or null
  uint64_t *pcode;    // packed 4-bit window codes (LeNet-internal) or null: pcode[k/16][n*PpQp + pp*Qp + pc]
  int64_t code_plane; // stride (64-bit words) of a 16-channel code group
  long long *clk;     // optional per-CTA cycle counters (SYSML_TC_PROFILE instrumentation)
  int N, C, H, W, K, R, S, ph, pw, P, Q;
  int sh, sw;          // stride: 1, or > 1 for 1x1 filters (frame = the output grid)
  // phase-split mode (phase.cu; phs > 0): this is the stride-1 pad-0 problem over the phase
  // planes X'[n][(a*phw + b)*phC + c][h'][w'] = X[n][c][h'*phs + a - php][w'*phw + b - phpw] of an
  // original phH x phW image with phC channels.  in_phase: the producer gathers X' straight from
  // the original X (fwd); out_phase: the plain epilogue writes channel (ab, c), position
  // (h', w') to dX[n][c][h'*phs + a - php][w'*phw + b - phpw] (bwd_data)
  int phs, phw, phC, phH, phW, php, phpw, in_phase, out_phase;
  int yH, yW, ysh, ysw;  // plain epilogue: output image yH x yW, row (p, q) -> (p*ysh, q*ysw)
                         // (strided 1x1 bwd_data writes every ysh-th row / ysw-th column)
  int Wf, Hs, Lf;
  int64_t G;
  int NFpad, nft, nchunk;
  int MT, HALO, nstage;
  int tile2d;          // 0: linear 128-position M-tiles; 1: 16x8 2-D M-tiles
  int CT, BB;          // 2-D: column tiles per band, bands per CTA tile (MT = CT*BB)
  int64_t cta_pos;     // positions advanced per CTA tile (linear: MT*128; 2-D: BB*16*Wf)
  int pool, PR, PS, Pp, Qp;
  int bias_smem;       // bias staged in shared memory (K floats)
  int ks;              // C == 1: the S column taps fill the MMA K slots (s = 4*half + e)
  int sn;              // narrow filter banks: the S column taps fold into N (D'[pos][(s,k)]),
                       // the epilogue adds Y[pos][k] = sum_s D'[pos + s][(s,k)]
  int snt;             // SN: taps s < snt in N (MMA 1, A unshifted); taps s = snt .. S-1 come
                       // from MMA 2 with A shifted by snt positions, accumulated into columns
                       // (s - snt, k).  snt == S: one MMA; snt < S: the accumulator is snt*NFpad
                       // wide, so two tiles fit TMEM and the epilogue overlaps the MMAs
  int NN;              // accumulator width per M-tile: NFpad, or snt*NFpad in SN mode
  int is_csr;          // KS mode only: input rows are CSR (scattered straight into the operand)
  sysml_csr csr;
  const float *route_val;       // routed SPF input (TcSpfIO::route_*): producer builds the values
  const uint64_t *route_code;
  int64_t route_cplane;
  int route_C, route_Pp, route_Qp, route_Wf, route_Lf;
  int64_t in_plane;    // > 0: input is SPF [C][in_plane], stored position = frame pos + in_shift
  int in_shift;
  int64_t out_plane;   // > 0: pooled output to SPF [K][out_plane] at (pp+out_off)*out_Wf + pc+out_off
  int out_Wf, out_Lf, out_off;
  int y_nhwc;          // SN epilogue: y written channel-minor [n][P*Q][K] (else NCHW)
  uint32_t a_bytes, b_bytes, stage_bytes, a_sbo;
  int64_t ntiles;
  uint32_t tmem_cols;
  uint32_t tbuf;       // TMEM accumulator buffer stride: 256 (double buffer) or 0 (single, MT*NFpad <= 512)
  int cl2;             // CTA-pair cluster: each CTA bulk-loads half of every filter chunk and
                       // multicasts it to both (halves the L2 -> SMEM filter stream)
  int64_t iters;       // tile iterations per CTA (cl2: equal in both CTAs, padded with empty tiles)
  int abulk;          // 1: 1x1 / pad 0 / NCHW input, 2: SPF input (any R, S): each chunk's 8
                      // channel rows are staged MN-major by 16-byte copies, then transposed
  int stg_row;        // floats per staged channel row (HALO; HALO + 4 for SPF: unaligned start)
                       //   ([8][HALO], 16-byte cp.async) behind the stage and transposed to the
                       //   K-major A operand by the producer threads
  int sk;              // stream-K: CTA b runs the global chunk iterations [b*I/G, (b+1)*I/G),
                       //   I = ntiles*nchunk, G = grid; tiles split across CTAs are combined below
  float *sk_part;      // stream-K partial accumulators [grid][MT][NN/16][128 rows][16] (workspace)
  int *sk_flag;        // [grid] ready flags of this launch (library-owned, reset by their consumer)
};

struct TcPlan {
  TcFwdParams p;
  size_t smem;
  size_t fp_bytes;
  bool ok;
};

constexpr uint32_t TMEM_BUF = 256;  // accumulator double buffer: columns [0,256) and [256,512)


// ---------------------------------------------------------------- epilogues
// Both drain the CTA tile's accumulators (MT M-tiles x NFpad columns) from TMEM in
// 16-column chunks with one tcgen05.ld in flight while the previous chunk is stored.
// Bias comes from shared memory as float4s; full chunks (all 16 filters < K) take a
// branch-free path.

__device__ __forceinline__ void load_bias16(const TcFwdParams &p, const float *bias_s, int k0,
                                            float (&b)[16]) {
  if (!p.bias) {
#pragma unroll
    for (int j = 0; j < 16; ++j) b[j] = 0.f;
  } else if (p.bias_smem && k0 + 16 <= p.K && (k0 & 3) == 0) {
    const float4 *b4 = reinterpret_cast<const float4 *>(bias_s + k0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 v = b4[j];
      b[4 * j] = v.x; b[4 * j + 1] = v.y; b[4 * j + 2] = v.z; b[4 * j + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) b[j] = (k0 + j < p.K) ? __ldg(p.bias + k0 + j) : 0.f;
  }
}

// phase mode gather offset of frame position gi (phase-problem frame, pad 0) for phase ab:
// n*phC*phH*phW + h*phW + w of the original image, -1 outside it (zero-filled)
__device__ __forceinline__ int phase_off(const TcFwdParams &p, int64_t gi, int ab) {
  if (gi >= p.G || ab >= p.phs * p.phw) return -1;
  const int n = (int)(gi / p.Lf), rem = (int)(gi - (int64_t)n * p.Lf);
  const int hh = rem / p.Wf, ww = rem - hh * p.Wf;
  const int a = ab / p.phw, b = ab - a * p.phw;
  const int h = hh * p.phs + a - p.php, w = ww * p.phw + b - p.phpw;
  if (hh >= p.H || ww >= p.W || h < 0 || h >= p.phH || w < 0 || w >= p.phW) return -1;
  return (n * p.phC) * p.phH * p.phW + h * p.phW + w;
}

// phase-split bwd_data epilogue store (out of line: keeps the common epilogue's registers)
__device__ __forceinline__ void phase_store16(const TcFwdParams &p, int64_t g, int a, int bb, int c,
                                              const float *v) {
  const int n = (int)(g / p.Lf), r2 = (int)(g - (int64_t)n * p.Lf), hh = r2 / p.Wf, q = r2 - hh * p.Wf;
  const int h = hh * p.phs + a - p.php, w = q * p.phw + bb - p.phpw;
  if (h < 0 || h >= p.phH || w < 0 || w >= p.phW) return;
  const int64_t HWo = (int64_t)p.phH * p.phW;
  float *yo = p.y + ((int64_t)n * p.phC + c) * HWo + (int64_t)h * p.phW + w;
#pragma unroll
  for (int j = 0; j < 16; ++j) yo[(int64_t)j * HWo] = v[j];
}

// plain conv output: lane -> position (linear or 2-D M-tile), 16 filters per chunk
template <bool PH>  // PH: phase-split modes compiled in (a separate kernel instance, so the
                   // common instance keeps its register allocation)
__device__ __forceinline__ void epi_plain(const TcFwdParams &p, uint32_t tbase, int64_t g0, int ft,
                                          int qd, int lane, const float *bias_s, int i0, int istep) {
  const int64_t PQ = (int64_t)p.yH * p.yW;  // output plane (= P*Q unless strided bwd_data)
  const int nc16 = p.NFpad / 16;
  float *__restrict__ y = p.y;
  for (int i = i0; i < p.MT; i += istep) {
    const uint32_t trow = tbase + (uint32_t)(i * p.NFpad);
    uint32_t r0[16], r1[16];
    ptx::tmem_ld16_issue(trow, r0);
    int64_t g;
    if (!p.tile2d) g = g0 + i * 128 + qd * 32 + lane;
    else {
      const int bb = i / p.CT, ct = i - bb * p.CT;
      g = g0 + (int64_t)bb * 16 * p.Wf + ct * 8 + (qd * 4 + (lane >> 3)) * p.Wf + (lane & 7);
    }
    bool valid = g < p.G;
    int64_t ybase = 0;
    if (valid) {
      int n, rem;
      if (p.G < (1ll << 31)) {  // 32-bit position arithmetic (the common case)
        n = (int)((uint32_t)g / (uint32_t)p.Lf);
        rem = (int)((uint32_t)g - (uint32_t)n * (uint32_t)p.Lf);
      } else {
        n = (int)(g / p.Lf);
        rem = (int)(g - (int64_t)n * p.Lf);
      }
      const int hh = rem / p.Wf, q = rem - hh * p.Wf;
      valid = hh < p.P && q < p.Q;
      ybase = (int64_t)n * p.K * PQ + (int64_t)hh * p.ysh * p.yW + (int64_t)q * p.ysw;
    }
    auto process = [&](const uint32_t(&cur)[16], int c16) {
      const int k0 = ft * p.NFpad + c16 * 16;
      float b[16];
      load_bias16(p, bias_s, k0, b);
      if (!valid) return;
      float *yp = y + ybase + (int64_t)k0 * PQ;
      if (PH && p.out_phase) {  // phase-split bwd_data: 16 channels of one phase (phC % 16 == 0)
        const int ab = k0 / p.phC, c = k0 - ab * p.phC, a = ab / p.phw, bb = ab - a * p.phw;
        if (ab >= p.phs * p.phw) return;  // pad channels
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(cur[j]) + b[j];
        phase_store16(p, g, a, bb, c, v);
        return;
      }
      if (k0 + 16 <= p.K) {
#pragma unroll
        for (int j = 0; j < 16; ++j) yp[(int64_t)j * PQ] = __uint_as_float(cur[j]) + b[j];
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (k0 + j < p.K) yp[(int64_t)j * PQ] = __uint_as_float(cur[j]) + b[j];
      }
    };
    for (int c16 = 0; c16 < nc16; c16 += 2) {
      ptx::tmem_ld_wait(r0);
      if (c16 + 1 < nc16) ptx::tmem_ld16_issue(trow + (c16 + 1) * 16, r1);
      process(r0, c16);
      if (c16 + 1 < nc16) {
        ptx::tmem_ld_wait(r1);
        if (c16 + 2 < nc16) ptx::tmem_ld16_issue(trow + (c16 + 2) * 16, r0);
        process(r1, c16 + 1);
      }
    }
  }
}

// Fused bias + relu + 2x2/2 max-pool on a 2-D M-tile (16 rows x 8 cols: the window of
// lane l is lanes l, l^1 (next column), l^8 (next row), l^9, all in this warp) with a
// reduce-scatter butterfly: round 1 (column partner, lane ^ 1) leaves each lane the pair-max of 8 of the
// 16 channels, round 2 (row partner, lane ^ 8) the window max of 4 -- so each of the
// window's four lanes owns 4 channels: 4 value stores plus either 4 int32 argmax
// indices (column of the pool-input row, reading R6) or 16 bits of 4-bit codes
// (LeNet-internal: positive*4 + dr*2 + ds, positive = window max > 0).  Ties -> the
// earlier position in r-outer / s-inner order (readings R5/R7/R9).  relu'd values are >= +0.0, so they compare as unsigned integers; the later
// position takes the partner's value when it is >= (u + 1 > u), the earlier when >.
__device__ __forceinline__ void epi_pool2(const TcFwdParams &p, uint32_t tbase, int64_t g0,
                                               int ft, int qd, int lane, const float *bias_s,
                                               int i0, int istep) {
  const int PpQp = p.Pp * p.Qp;
  const int nc16 = p.NFpad / 16;
  const int rl = qd * 4 + (lane >> 3), cl = lane & 7;
  const uint32_t odd_c = cl & 1, odd_r = rl & 1;
  const int cb = (int)(odd_c * 8 + odd_r * 4);  // first of the 4 channels this lane ends with
  float *__restrict__ pout = p.pout;
  for (int i = i0; i < p.MT; i += istep) {
    const uint32_t trow = tbase + (uint32_t)(i * p.NFpad);
    uint32_t r0[16], r1[16];
    ptx::tmem_ld16_issue(trow, r0);
    const int bb = i / p.CT, ct = i - bb * p.CT;
    const int grow = (int)(g0 / p.Wf) + bb * 16 + rl;  // global frame row
    const int col = ct * 8 + cl;
    const int n = grow / p.Hs;
    const int hh = grow - n * p.Hs;
    const int pp = hh >> 1, pc = col >> 1;
    const bool store = n < p.N && pp < p.Pp && pc < p.Qp;
    const int vstride = p.out_plane > 0 ? (int)p.out_plane : PpQp;
    const int64_t vbase = !store ? 0
                          : p.out_plane > 0 ? (int64_t)n * p.out_Lf + (int64_t)(pp + p.out_off) * p.out_Wf +
                                                  (pc + p.out_off)
                                            : (int64_t)n * p.K * PpQp + (int64_t)pp * p.Qp + pc;
    float *const pout_t = pout + vbase + (int64_t)cb * vstride;
    uint16_t *const code_t = p.pcode ? reinterpret_cast<uint16_t *>(p.pcode + (store ? (int64_t)n * PpQp + pp * p.Qp + pc : 0)) +
                                           (cb >> 2)
                                     : nullptr;
    // int32 argmax (NCHW pooled layout): plane index of the window's top-left conv output
    int32_t *const parg_t = p.parg ? p.parg + (store ? (int64_t)n * p.K * PpQp + pp * p.Qp + pc : 0) +
                                         (int64_t)cb * PpQp
                                   : nullptr;
    const int idx_tl = (2 * pp) * p.Q + 2 * pc;
    auto process = [&](const uint32_t(&cur)[16], int c16) {
      const int k0 = ft * p.NFpad + c16 * 16;
      float b[16];
      uint32_t u[16];
      load_bias16(p, bias_s, k0, b);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float t = __uint_as_float(cur[j]) + b[j];
        u[j] = __float_as_uint(t > 0.f ? t : 0.f);  // relu, +0.0 for non-positive (reading R7)
      }
      // round 1: keep channels [8*odd_c, +8), send the other half to the column partner
      uint32_t v8[8], sbit = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t send = odd_c ? u[j] : u[j + 8];
        const uint32_t mine = odd_c ? u[j + 8] : u[j];
        const uint32_t got = __shfl_xor_sync(0xffffffffu, send, 1);
        const bool take = got + odd_c > mine;  // partner is the even (earlier) column iff odd_c
        v8[j] = take ? got : mine;
        sbit |= (odd_c ^ (uint32_t)take) << j;  // winner's column
      }
      // round 2: keep channels [cb, +4) of those 8, send the other 4 to the row partner
      uint32_t v4[4];
      const uint32_t psbit = __shfl_xor_sync(0xffffffffu, sbit, 8);
      uint32_t code = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t send = odd_r ? v8[j] : v8[j + 4];
        const uint32_t mine = odd_r ? v8[j + 4] : v8[j];
        const uint32_t got = __shfl_xor_sync(0xffffffffu, send, 8);
        const bool take = got + odd_r > mine;
        v4[j] = take ? got : mine;
        const int jj = (int)(odd_r * 4) + j;  // index among this lane's 8 channels
        const uint32_t ds = ((take ? psbit : sbit) >> jj) & 1u;
        const uint32_t pos = v4[j] != 0u;  // window max > 0: the relu/pool gradient mask (R9)
        code |= ((pos << 2) | ((odd_r ^ (uint32_t)take) << 1) | ds) << (4 * j);
      }
      if (store) {
        float *po = pout_t + (int64_t)k0 * vstride;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (k0 + cb + j < p.K) po[j * vstride] = __uint_as_float(v4[j]);
        if (code_t) code_t[(int64_t)(k0 >> 4) * p.code_plane * 4] = (uint16_t)code;
        if (parg_t) {
          const int PQ = p.P * p.Q;
          int32_t *pa = parg_t + (int64_t)k0 * PpQp;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t cj = code >> (4 * j);
            if (k0 + cb + j < p.K)
              pa[j * PpQp] = (k0 + cb + j) * PQ + idx_tl + (int)((cj >> 1) & 1u) * p.Q + (int)(cj & 1u);
          }
        }
      }
    };
    for (int c16 = 0; c16 < nc16; c16 += 2) {
      ptx::tmem_ld_wait(r0);
      if (c16 + 1 < nc16) ptx::tmem_ld16_issue(trow + (c16 + 1) * 16, r1);
      process(r0, c16);
      if (c16 + 1 < nc16) {
        ptx::tmem_ld_wait(r1);
        if (c16 + 2 < nc16) ptx::tmem_ld16_issue(trow + (c16 + 2) * 16, r0);
        process(r1, c16 + 1);
      }
    }
  }
}

constexpr int SN_MAXMT = 4;
constexpr int SN_XCH_FLOATS = 2 * SN_MAXMT * 4 * 8 * 4 * 16;  // [set][M-tile][warp][s][row < S-1 <= 4][16]

// SN epilogue (column taps in N): accumulator row l = i*128 + qd*32 + lane holds
// D'[g0 + l][(s', k)], s' < T = snt; output Y[g0 + l][k] = b[k] + sum_s' D'[g0 + l + s'][(s', k)]
// for l < cta_pos = MT*128 - (T-1) (CTA tiles overlap by T-1 rows).  Rows l + s of the same warp come by shfl_down; the
// first S-1 rows of the next 32-row group (next quadrant, or quadrant 0 of the next
// M-tile) are dumped to shared memory first.  The two warp sets split the 16-channel
// chunks.
__device__ __forceinline__ void epi_sn(const TcFwdParams &p, uint32_t tbase, int64_t g0, int qd,
                                       int lane, const float *bias_s, int eset, float *xch_all) {
  const int PQ = p.P * p.Q;
  const int nc16 = p.NFpad / 16;
  float *__restrict__ y = p.y;
  float *xch = xch_all + eset * (SN_MAXMT * 4 * 8 * 4 * 16);
  auto xidx = [&](int i, int q, int s_, int row) { return (((i * 4 + q) * 8 + s_) * 4 + row) * 16; };
  const bool g32 = p.G < (1ll << 31);
  for (int c16 = eset; c16 < nc16; c16 += 2) {
    // 1) dump the first S-1 rows of every 32-row group for s >= 1
    for (int i = 0; i < p.MT; ++i)
      for (int s_ = 1; s_ < p.snt; ++s_) {
        float t[16];
        ptx::tmem_ld16(tbase + (uint32_t)(i * p.NN + s_ * p.NFpad + c16 * 16), t);
        if (lane < p.snt - 1) {
          float *dst = xch + xidx(i, qd, s_, lane);
#pragma unroll
          for (int j = 0; j < 16; ++j) dst[j] = t[j];
        }
      }
    ptx::named_bar_sync(2 + eset, 128);
    const int k0 = c16 * 16;
    float b[16];
    load_bias16(p, bias_s, k0, b);
    // 2) shift-add per M-tile
    for (int i = 0; i < p.MT; ++i) {
      const int l = i * 128 + qd * 32 + lane;
      const int ni = qd == 3 ? i + 1 : i, nq = (qd + 1) & 3;  // next 32-row group
      float acc[16];
      ptx::tmem_ld16(tbase + (uint32_t)(i * p.NN + c16 * 16), acc);
      for (int s_ = 1; s_ < p.snt; ++s_) {
        float t[16];
        ptx::tmem_ld16(tbase + (uint32_t)(i * p.NN + s_ * p.NFpad + c16 * 16), t);
        const bool from_next = lane + s_ >= 32;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float v = __shfl_down_sync(0xffffffffu, t[j], s_);
          if (!from_next) acc[j] += v;
        }
        if (from_next) {  // the last s lanes: rows of the next 32-row group (4 x 16 B loads)
          const float4 *src =
              reinterpret_cast<const float4 *>(xch + xidx(ni < p.MT ? ni : 0, nq, s_, lane + s_ - 32));
#pragma unroll
          for (int j4 = 0; j4 < 4; ++j4) {
            const float4 u = src[j4];
            acc[4 * j4] += u.x;
            acc[4 * j4 + 1] += u.y;
            acc[4 * j4 + 2] += u.z;
            acc[4 * j4 + 3] += u.w;
          }
        }
      }
      const int64_t g = g0 + l;
      if (l < (int)p.cta_pos && g < p.G) {
        int n, rem;
        if (g32) {
          n = (int)((uint32_t)g / (uint32_t)p.Lf);
          rem = (int)((uint32_t)g - (uint32_t)n * (uint32_t)p.Lf);
        } else {
          n = (int)(g / p.Lf);
          rem = (int)(g - (int64_t)n * p.Lf);
        }
        const int hh = rem / p.Wf, q = rem - hh * p.Wf;
        if (hh < p.P && q < p.Q) {
          if (p.y_nhwc) {
            // channel-minor [n][P*Q][K]: 16 channels = 64 contiguous bytes per row
            float4 *yp = reinterpret_cast<float4 *>(y + ((int64_t)n * PQ + (int64_t)hh * p.Q + q) * p.K + k0);
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4)
              if (k0 + 4 * j4 + 4 <= p.K)
                yp[j4] = make_float4(acc[4 * j4] + b[4 * j4], acc[4 * j4 + 1] + b[4 * j4 + 1],
                                     acc[4 * j4 + 2] + b[4 * j4 + 2], acc[4 * j4 + 3] + b[4 * j4 + 3]);
          } else {
            float *yp = y + (int64_t)n * p.K * PQ + (int64_t)hh * p.Q + q + (int64_t)k0 * PQ;
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (k0 + j < p.K) yp[(int64_t)j * PQ] = acc[j] + b[j];
          }
        }
      }
    }
    ptx::named_bar_sync(2 + eset, 128);  // before the next chunk overwrites the dump
  }
}

// ---------------------------------------------------------------- work distribution
// Round-robin whole tiles (tile = blockIdx.x + it*gridDim.x), or stream-K: the
// ntiles*nchunk chunk iterations are cut into gridDim.x equal contiguous ranges, so a
// tile may be split across consecutive CTAs.  A segment is (tile, chunks [c0, c1)).
// The CTA holding a split tile's first segment (c0 = 0) computes it LAST in its range and
// owns the tile: it adds the other segments' partial accumulators, which their CTAs
// computed FIRST in their ranges and published (partial slot + release flag), in segment
// order -- a fixed order, so results are deterministic -- then runs the normal epilogue.
struct TcWork {
  int64_t i, i1, it;
};
__device__ __forceinline__ int64_t sk_begin(const TcFwdParams &p, int b) {
  return (int64_t)b * (p.ntiles * p.nchunk) / gridDim.x;
}
__device__ __forceinline__ TcWork tc_work_init(const TcFwdParams &p) {
  TcWork w;
  w.it = 0;
  w.i = p.sk ? sk_begin(p, blockIdx.x) : 0;
  w.i1 = p.sk ? sk_begin(p, blockIdx.x + 1) : 0;
  return w;
}
__device__ __forceinline__ bool tc_next_raw(const TcFwdParams &p, TcWork &w, int64_t &tile, int &c0,
                                            int &c1) {
  if (p.sk) {
    if (w.i >= w.i1) return false;
    tile = w.i / p.nchunk;
    c0 = (int)(w.i - tile * p.nchunk);
    c1 = (int)min((int64_t)p.nchunk, (int64_t)c0 + (w.i1 - w.i));
    w.i += c1 - c0;
    return true;
  }
  if (w.it >= p.iters) return false;
  tile = blockIdx.x + w.it * gridDim.x;  // >= ntiles: empty (cl2 padding)
  ++w.it;
  if (tile >= p.ntiles && !p.cl2) return false;
  c0 = 0;
  c1 = p.nchunk;
  return true;
}
// the segment, broadcast from lane 0: provably warp-uniform, so the MMA issue loop keeps
// its descriptors on the uniform datapath
__device__ __forceinline__ bool tc_next(const TcFwdParams &p, TcWork &w, int64_t &tile, int &c0, int &c1) {
  const bool ok = tc_next_raw(p, w, tile, c0, c1);
  if (!__shfl_sync(0xffffffffu, (int)ok, 0)) return false;
  tile = __shfl_sync(0xffffffffu, tile, 0);
  c0 = __shfl_sync(0xffffffffu, c0, 0);
  c1 = __shfl_sync(0xffffffffu, c1, 0);
  return true;
}

// stream-K contributor: this thread's accumulator row (all MT x NN columns; the two warp
// sets of a quadrant split the 16-column groups) -> the CTA's partial slot
__device__ __forceinline__ void sk_dump(const TcFwdParams &p, uint32_t tb, int row, int eset) {
  const int ng = p.NN / 16;
  float *slot = p.sk_part + (size_t)blockIdx.x * p.MT * ng * 128 * 16;
  for (int i = 0; i < p.MT; ++i)
    for (int c16 = eset; c16 < ng; c16 += 2) {
      float v[16];
      ptx::tmem_ld16(tb + (uint32_t)(i * p.NN + c16 * 16), v);
      float4 *o = reinterpret_cast<float4 *>(slot + ((size_t)(i * ng + c16) * 128 + row) * 16);
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
}

// stream-K owner: add the partials of the CTAs holding segments [c1, nchunk) of this tile
// (CTAs blockIdx.x + 1, + 2, ... in segment order) into the accumulator in TMEM
__device__ __forceinline__ void sk_fixup(const TcFwdParams &p, uint32_t tb, int row, int eset, int c1) {
  const int ng = p.NN / 16;
  int nj = 0;
  for (int cur = c1, j = blockIdx.x + 1; cur < p.nchunk && j < (int)gridDim.x; ++j, ++nj) {
    cur += (int)(sk_begin(p, j + 1) - sk_begin(p, j));
    while (ptx::ld_acquire_gpu(p.sk_flag + j) == 0) __nanosleep(64);
  }
  for (int i = 0; i < p.MT; ++i)
    for (int c16 = eset; c16 < ng; c16 += 2) {
      float v[16];
      ptx::tmem_ld16(tb + (uint32_t)(i * p.NN + c16 * 16), v);
      for (int jj = 1; jj <= nj; ++jj) {
        const float4 *src = reinterpret_cast<const float4 *>(
            p.sk_part + (size_t)(blockIdx.x + jj) * p.MT * ng * 128 * 16 + ((size_t)(i * ng + c16) * 128 + row) * 16);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 u = __ldcg(src + j);
          v[4 * j] += u.x;
          v[4 * j + 1] += u.y;
          v[4 * j + 2] += u.z;
          v[4 * j + 3] += u.w;
        }
      }
      ptx::tmem_st16(tb + (uint32_t)(i * p.NN + c16 * 16), v);
    }
  ptx::tmem_st_wait();
}

// Routed SPF input (NEXT-1): the staged window range of the tile starting at frame position g0 --
// first window (even, for 16-byte aligned code copies) and the even window count covering
// every position of the halo.
__device__ __forceinline__ int64_t rt_win_at(const TcFwdParams &p, int64_t si, int after) {
  const int64_t n = si / p.route_Lf;
  const int row = (int)((si - n * p.route_Lf) / p.route_Wf);
  const int pp = min((row >> 1) + after, p.route_Pp);
  return (n * p.route_Pp + pp) * p.route_Qp;
}
__device__ __forceinline__ int64_t rt_w0(const TcFwdParams &p, int64_t g0) {
  const int64_t si0 = max(g0 + (int64_t)p.in_shift, (int64_t)0);
  if (si0 >= p.in_plane) return 0;
  return rt_win_at(p, si0, 0) & ~(int64_t)1;
}
__device__ __forceinline__ void rt_issue(const TcFwdParams &p, int64_t g0, uint8_t *buf, uint64_t *bar) {
  const int64_t w0 = rt_w0(p, g0);
  const int64_t si0 = max(g0 + (int64_t)p.in_shift, (int64_t)0);
  const int64_t si1 = min(g0 + (int64_t)p.in_shift + p.HALO - 1, p.in_plane - 1);
  int cnt = 0;
  if (si0 <= si1 && si0 < p.in_plane) {
    const int64_t total = (int64_t)p.N * p.route_Pp * p.route_Qp;
    const int64_t w1 = min(rt_win_at(p, si1, 1), total);
    cnt = (int)max((int64_t)0, (w1 - w0 + 1) & ~(int64_t)1);
    cnt = min(cnt, RT_MAXW);
  }
  const int ng = (p.C + 15) / 16;
  ptx::fence_proxy_async_smem();  // the previous tile's generic reads of this slot are ordered first
  ptx::mbar_arrive_expect_tx(bar, (uint32_t)(cnt * p.route_C * 4 + ng * cnt * 8));
  if (cnt > 0) {
    ptx::bulk_g2s(buf, p.route_val + w0 * p.route_C, (uint32_t)(cnt * p.route_C * 4), bar);
    for (int g = 0; g < ng; ++g)
      ptx::bulk_g2s(buf + RT_MAXW * 64 * 4 + g * RT_MAXW * 8, p.route_code + g * p.route_cplane + w0,
                    (uint32_t)(cnt * 8), bar);
  }
}

// MODE 0: common instance; 1: phase-split modes compiled in; 2: routed SPF input (NEXT-1).
// Separate instances so the common one keeps its register allocation.
template <int MODE>
__global__ void __launch_bounds__(TC_FWD_THREADS, 1) tc_conv_fwd_kernel(const TcFwdParams p) {
  constexpr bool PH = MODE == 1, RT = MODE == 2;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *stage_base = smem;
  uint8_t *rt_buf = smem + (size_t)p.nstage * p.stage_bytes;  // RT: [2][RT_SLOT] tile staging
  int *src_off = reinterpret_cast<int *>(rt_buf + (RT ? RT_BYTES : 0));
  float *bias_s = reinterpret_cast<float *>(src_off + p.HALO + 8);
  // SN epilogue exchange: [set 2][warp 4][s 8][row 4][16] floats (rows 0..3 of each warp)
  float *sn_xch = reinterpret_cast<float *>(
      (reinterpret_cast<uintptr_t>(bias_s + (p.bias_smem ? p.K : 0)) + 15) & ~(uintptr_t)15);
  uint64_t *bars = reinterpret_cast<uint64_t *>(sn_xch + (p.sn ? SN_XCH_FLOATS : 0));
  uint64_t *full = bars;
  uint64_t *empty = bars + p.nstage;
  uint64_t *accf = bars + 2 * p.nstage;  // [2]
  uint64_t *acce = accf + 2;             // [2]
  uint64_t *staged = acce + 2;           // [nstage] abulk: staging buffer filled
  uint64_t *rtfull = staged + p.nstage;  // [2] RT: tile staging landed
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(rtfull + 2);

  // warp index via shuffle: provably warp-uniform, so role branches keep the uniform datapath
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nstage; ++s) {
      // dense: 128 producer threads (cp.async arrivals) + the expect_tx arrival;
      // CSR: one warp fills a whole stage and arrives once with the expect_tx
      ptx::mbar_init(full + s, p.is_csr ? 1 : (p.abulk ? 64 : 128) + 1);
      ptx::mbar_init(empty + s, p.cl2 ? 2 : 1);  // tcgen05.commit (of both CTAs of a pair)
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(accf + b, 1);
      ptx::mbar_init(acce + b, TC_EPI_WARPS);
    }
    for (int s = 0; s < p.nstage; ++s) ptx::mbar_init(staged + s, 64);  // abulk: loader cp.async arrivals
    ptx::mbar_init(rtfull, 1);
    ptx::mbar_init(rtfull + 1, 1);
    ptx::fence_mbar_init();
  }
  if (p.bias_smem)
    for (int k = threadIdx.x; k < p.K; k += blockDim.x) bias_s[k] = p.bias[k];
  if (warp == 4) ptx::tmem_alloc(tmem_slot, p.tmem_cols);  // warp 4 = MMA warp
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (p.cl2) ptx::cluster_sync();  // the peer's barriers are initialised before any multicast
  const uint32_t crank = p.cl2 ? ptx::cluster_ctarank() : 0u;
  const int HW = p.H * p.W;
  const long long t_kernel0 = clock64();

  if (warp < 4 && p.is_csr) {
    // ================= CSR producers (KS mode, one chunk per tile): each warp owns every
    // 4th tile of this CTA and fills its stage alone -- zero-fill, scatter the non-zeros
    // of the images overlapping the tile into their S slots, fence, then one arrival
    // with the filter chunk's expect_tx.  Four tiles' load-latency chains overlap.
    if (lane == 0) asm volatile("griddepcontrol.wait;" ::: "memory");  // packed filters ready
    int tl = warp;  // CTA-local tile counter of this warp
    for (int64_t tile = blockIdx.x + (int64_t)warp * gridDim.x; tile < p.ntiles;
         tile += 4 * (int64_t)gridDim.x, tl += 4) {
      const int ft = (int)(tile % p.nft);
      const int64_t g0 = (tile / p.nft) * p.cta_pos;
      const int stage = tl % p.nstage;
      const uint32_t phase = (uint32_t)((tl / p.nstage) & 1);
      ptx::mbar_wait(empty + stage, phase ^ 1);
      uint8_t *A = stage_base + (size_t)stage * p.stage_bytes;
      const uint32_t a0 = ptx::smem_u32(A);
      // the row pointers of the (at most a few) images overlapping [g0, g0 + HALO + 8)
      const int64_t last = g0 + p.HALO + 7;
      const int n_lo = (int)(g0 / p.Lf);
      const int n_hi = (int)min((int64_t)p.N - 1, last / p.Lf);
      const int nimg = n_hi - n_lo + 1;
      const int rp = lane <= nimg ? __ldg(p.csr.row_ptr + n_lo + lane) : 0;
      for (int i = lane; i < 2 * p.HALO; i += 32) st_shared_v4(a0 + i * 16, 0.f, 0.f, 0.f, 0.f);
      __syncwarp();
      float *Af = reinterpret_cast<float *>(A);
      // Every input position owns distinct (pos, s) slots, so a strictly increasing row (the
      // S:31-32 contract) has one writer per slot: plain stores.  A row that is not strictly
      // increasing (unsorted, or duplicate columns -- reading R15) flags the tile, which is
      // then rebuilt by lane 0 summing in stored order: deterministic, no float atomics.
      bool bad = false;
      const int jA = __shfl_sync(0xffffffffu, rp, 0);
      const int jB = nimg <= 31 ? __shfl_sync(0xffffffffu, rp, nimg) : __ldg(p.csr.row_ptr + n_hi + 1);
      if (nimg <= 31) {
        // the overlapping images' non-zeros are one contiguous CSR range: 4 (col, val)
        // pairs per lane in flight, each entry's image from the row pointers (uniform loop)
        int last = -1;  // column of the entry before this batch (lane 31 of the last one)
        for (int base = jA; base < jB; base += 128) {
          int col[4], img[4];
          float val[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int jj = base + u * 32 + lane;
            const bool ok = jj < jB;
            col[u] = ok ? __ldg(p.csr.col_idx + jj) : -1;
            val[u] = ok ? __ldg(p.csr.val + jj) : 0.f;
            img[u] = 0;
          }
          for (int ii = 1; ii < nimg; ++ii) {
            const int b = __shfl_sync(0xffffffffu, rp, ii);
#pragma unroll
            for (int u = 0; u < 4; ++u) img[u] += (base + u * 32 + lane >= b) ? 1 : 0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int up = __shfl_up_sync(0xffffffffu, col[u], 1);
            const int prev = lane ? up : last;
            last = __shfl_sync(0xffffffffu, col[u], 31);
            const int rs = __shfl_sync(0xffffffffu, rp, img[u]);
            const int jj = base + u * 32 + lane;
            if (jj < jB && jj > rs && prev >= col[u]) bad = true;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (col[u] < 0 || col[u] >= HW) continue;
            const int h = col[u] / p.W, w = col[u] - h * p.W;
            const int64_t gi = (int64_t)(n_lo + img[u]) * p.Lf + (int64_t)(h + p.ph) * p.Wf + (w + p.pw);
            for (int s_ = 0; s_ < p.S; ++s_) {
              const int64_t pos = gi - g0 - s_;
              if (pos >= 0 && pos < p.HALO) Af[(s_ >> 2) * p.HALO * 4 + pos * 4 + (s_ & 3)] = val[u];
            }
          }
        }
      } else
      for (int ii = 0; ii < nimg; ++ii) {  // more than 31 images in one tile (tiny images)
        const int n = n_lo + ii;
        const int j0 = __ldg(p.csr.row_ptr + n), j1 = __ldg(p.csr.row_ptr + n + 1);
        int last = -1;
        for (int base = j0; base < j1; base += 32) {
          const int jj = base + lane;
          const int col = jj < j1 ? __ldg(p.csr.col_idx + jj) : -1;
          const float v = jj < j1 ? __ldg(p.csr.val + jj) : 0.f;
          const int up = __shfl_up_sync(0xffffffffu, col, 1);
          const int prev = lane ? up : last;
          last = __shfl_sync(0xffffffffu, col, 31);
          if (jj < j1 && jj > j0 && prev >= col) bad = true;
          if (col < 0 || col >= HW) continue;
          const int h = col / p.W, w = col - h * p.W;
          const int64_t gi = (int64_t)n * p.Lf + (int64_t)(h + p.ph) * p.Wf + (w + p.pw);
          for (int s_ = 0; s_ < p.S; ++s_) {
            const int64_t pos = gi - g0 - s_;
            if (pos >= 0 && pos < p.HALO) Af[(s_ >> 2) * p.HALO * 4 + pos * 4 + (s_ & 3)] = v;
          }
        }
      }
      if (__any_sync(0xffffffffu, bad)) {  // rebuild the tile in stored order (lane 0)
        __syncwarp();
        for (int i = lane; i < 2 * p.HALO; i += 32) st_shared_v4(a0 + i * 16, 0.f, 0.f, 0.f, 0.f);
        __syncwarp();
        if (lane == 0) {
          int n = n_lo, jn = __ldg(p.csr.row_ptr + n_lo + 1);
          for (int jj = jA; jj < jB; ++jj) {
            while (jj >= jn) jn = __ldg(p.csr.row_ptr + (++n) + 1);
            const int col = __ldg(p.csr.col_idx + jj);
            if (col < 0 || col >= HW) continue;
            const float v = __ldg(p.csr.val + jj);
            const int h = col / p.W, w = col - h * p.W;
            const int64_t gi = (int64_t)n * p.Lf + (int64_t)(h + p.ph) * p.Wf + (w + p.pw);
            for (int s_ = 0; s_ < p.S; ++s_) {
              const int64_t pos = gi - g0 - s_;
              if (pos >= 0 && pos < p.HALO) Af[(s_ >> 2) * p.HALO * 4 + pos * 4 + (s_ & 3)] += v;
            }
          }
        }
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive_expect_tx(full + stage, p.b_bytes);
        ptx::bulk_g2s(A + p.a_bytes, p.fp + (size_t)ft * p.nchunk * (p.b_bytes / 4), p.b_bytes,
                      full + stage);
      }
    }
  } else if (warp < 4) {
    // ================= producers: A halo (ld.global -> st.shared) + B chunk (bulk copy)
    const int tid = threadIdx.x;
    int stage = 0;
    uint32_t phase = 0;
    // programmatic dependent launch: everything up to the first packed-filter read
    // (barriers, TMEM, gather tables, A copies) overlaps the filter-pack kernel
    if (tid == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
    TcWork wk = tc_work_init(p);
    int64_t tile;
    int c0, c1;
    int ist = 0;  // abulk issuer (tid 0): stage cursor, runs up to L chunks ahead
    int64_t rt_tl = 0;  // RT: CTA-local tile counter (tile staging slot = rt_tl & 1)
    uint32_t iph = 0;
    while (tc_next(p, wk, tile, c0, c1)) {
      const int ft = (int)(tile % p.nft);
      const int64_t g0 = (tile / p.nft) * p.cta_pos;
      if (p.abulk) {
        // ---- 1x1 / pad 0: frame position = image position g = n*HW + hw.  Warps 0-1 stage
        // chunk ch's 8 channel rows MN-major ([8][HALO]) by 16-byte cp.async of 4-position
        // groups (groups never straddle an image as HW % 4 == 0; lanes take consecutive
        // groups: coalesced, conflict-free) plus the filter chunk, running ahead on the
        // empty barriers; warps 2-3 transpose staging -> A[quad][pos][4 ch] (4-byte reads
        // of consecutive positions, 16-byte row writes: conflict-free), fence generic ->
        // async proxy (their own stores only: a fence behind in-flight cp.async of the same
        // thread would wait for them), and arrive on the stage's full barrier.
        // SPF input (abulk 2): the halo of every channel is the contiguous run of stored
        // positions [g0 + in_shift, + HALO) of its plane; it is staged from the 16-byte
        // aligned position below it, and the transposers skip the first `dl` floats
        const int64_t s0 = p.abulk == 2 ? g0 + p.in_shift : 0;
        const int dl = p.abulk == 2 ? (int)(((s0 % 4) + 4) % 4) : 0;
        const int ngrp = (p.HALO + dl + 3) / 4;
        const int ROW = p.stg_row;
        if (tid < 64) {
          // per-segment group offsets n*C*HW + hw (int: N*C*H*W < 2^31, plan), -1 past G
          ptx::named_bar_sync(5, 64);  // the previous segment's copies have read the table
          for (int gq = tid; gq < ngrp; gq += 64) {
            int off = -1;
            if (p.abulk == 2) {
              const int64_t sp = s0 - dl + 4 * gq;  // planes hold whole 4-position groups
              if (sp >= 0 && sp + 4 <= p.in_plane) off = (int)sp;
            } else {
              const int64_t g = g0 + 4 * gq;
              if (g < p.G) {
                const int64_t n = g / HW;
                off = (int)(n * p.C * HW + (g - n * HW));
              }
            }
            src_off[gq] = off;
          }
          ptx::named_bar_sync(5, 64);
          const int64_t cstr = p.abulk == 2 ? p.in_plane : (int64_t)HW;
          for (int ch = c0; ch < c1; ++ch) {
            ptx::mbar_wait(empty + ist, iph ^ 1);
            uint8_t *A = stage_base + (size_t)ist * p.stage_bytes;
            uint8_t *B = A + p.a_bytes;
            const uint32_t stg = ptx::smem_u32(B + p.b_bytes);
            if (tid == 0) {
              ptx::mbar_arrive_expect_tx(full + ist, p.b_bytes);
              ptx::bulk_g2s(B, p.fp + ((size_t)ft * p.nchunk + ch) * (p.b_bytes / 4), p.b_bytes, full + ist);
            }
            const int cc0 = ch * 8, nc = min(8, p.C - cc0);
            const float *xc = p.x + (int64_t)cc0 * cstr;
            // item = (channel half jh, group gq): four channel rows share offset and address
            for (int base = tid; base < 2 * ngrp; base += 64) {
              const int jh = base >= ngrp ? 1 : 0, gq = base - jh * ngrp;
              const int off = src_off[gq];
              const uint32_t dst = stg + (uint32_t)(4 * jh * ROW + 4 * gq) * 4;
              const float *src = xc + off + (int64_t)(4 * jh) * cstr;
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                const bool ok = off >= 0 && 4 * jh + jj < nc;
                ptx::cp_async16(dst + (uint32_t)(jj * ROW) * 4, ok ? src + (int64_t)jj * cstr : p.x, ok ? 16u : 0u);
              }
            }
            ptx::cp_async_mbar_arrive(staged + ist);
            if (++ist == p.nstage) { ist = 0; iph ^= 1; }
          }
        } else {
          const int tt = tid - 64;
          for (int ch = c0; ch < c1; ++ch) {
            ptx::mbar_wait(staged + stage, phase);
            const uint8_t *A = stage_base + (size_t)stage * p.stage_bytes;
            const float *stg = reinterpret_cast<const float *>(A + p.a_bytes + p.b_bytes);
            const uint32_t a0 = ptx::smem_u32(A);
            for (int it = tt; it < 2 * p.HALO; it += 64) {
              const int q = it >= p.HALO ? 1 : 0, pos = it - q * p.HALO;
              const float *sr = stg + (4 * q) * ROW + pos + dl;
              st_shared_v4(a0 + (uint32_t)(q * p.HALO + pos) * 16, sr[0], sr[ROW], sr[2 * ROW], sr[3 * ROW]);
            }
            ptx::fence_proxy_async_smem();
            ptx::mbar_arrive(full + stage);
            if (++stage == p.nstage) { stage = 0; phase ^= 1; }
          }
        }
        continue;
      }
      ptx::named_bar_sync(1, 128);
      const int ntab = p.ks ? p.HALO + 8 : p.HALO;
      // phase mode: the table holds the gather offsets of phase cur_ab (recomputed below when
      // the chunk loop crosses into the next phase's channels)
      int cur_ab = (PH && p.in_phase) ? (c0 * 8) / p.phC : 0;
      for (int pos = tid; pos < ntab; pos += 128) {
        const int64_t gi = g0 + pos;
        int off = -1;
        if (PH && p.in_phase) {
          off = phase_off(p, gi, cur_ab);
        } else if (RT) {
          // routed: (window index - the tile's first staged window) * 4 + position in the window
          const int64_t si = gi + p.in_shift;
          if (gi < p.G && si >= 0 && si < p.in_plane) {
            const int n = (int)(si / p.route_Lf), rem = (int)(si - (int64_t)n * p.route_Lf);
            const int row = rem / p.route_Wf, col = rem - row * p.route_Wf;
            if (row < 2 * p.route_Pp && col < 2 * p.route_Qp)
              off = ((int)(((int64_t)n * p.route_Pp + (row >> 1)) * p.route_Qp + (col >> 1) - rt_w0(p, g0))) * 4 +
                    (row & 1) * 2 + (col & 1);
          }
        } else if (p.in_plane > 0) {
          const int64_t si = gi + p.in_shift;  // SPF: zeros are stored, no decoding
          if (gi < p.G && si >= 0 && si < p.in_plane) off = (int)si;
        } else if (gi < p.G) {
          const int n = (int)(gi / p.Lf);
          const int rem = (int)(gi - (int64_t)n * p.Lf);
          const int hh = rem / p.Wf, ww = rem - hh * p.Wf;
          const int h = hh * p.sh - p.ph, w = ww * p.sw - p.pw;  // stride > 1: output-grid frame
          if (h >= 0 && h < p.H && w >= 0 && w < p.W) off = n * p.C * HW + h * p.W + w;
        }
        src_off[pos] = off;
      }
      ptx::named_bar_sync(1, 128);
      if (RT) {
        // NEXT-1 vertical fusion: the unpooled gradient is built here from the
        // pooled gradient (route_val, window-major, channel-minor) and the pool window codes
        // -- dz2 never exists in HBM.  The tile's window rows and code words are staged in
        // shared memory by bulk copies (issued one tile ahead, double-buffered); each chunk
        // then expands them smem -> smem: two 16-byte loads + one code word per (position,
        // 8 channels), two 16-byte row stores into the K-major [quad][pos][4] operand.
        const int slot = (int)(rt_tl & 1);
        if (tid == 0) {
          if (rt_tl == 0) rt_issue(p, g0, rt_buf, rtfull);  // first tile: nobody prefetched it
          const int64_t nxt = tile + gridDim.x;             // round-robin tiles (no stream-K)
          if (nxt < p.ntiles) rt_issue(p, (nxt / p.nft) * p.cta_pos, rt_buf + (1 - slot) * RT_SLOT, rtfull + (1 - slot));
        }
        ptx::mbar_wait(rtfull + slot, (uint32_t)((rt_tl >> 1) & 1));
        const float *rv = reinterpret_cast<const float *>(rt_buf + slot * RT_SLOT);
        const unsigned long long *rc =
            reinterpret_cast<const unsigned long long *>(rt_buf + slot * RT_SLOT + RT_MAXW * 64 * 4);
        for (int ch = c0; ch < c1; ++ch) {
          ptx::mbar_wait(empty + stage, phase ^ 1);
          uint8_t *A = stage_base + (size_t)stage * p.stage_bytes;
          if (tid == 0) {
            ptx::mbar_arrive_expect_tx(full + stage, p.b_bytes);
            ptx::bulk_g2s(A + p.a_bytes, p.fp + ((size_t)ft * p.nchunk + ch) * (p.b_bytes / 4), p.b_bytes,
                          full + stage);
          }
          const uint32_t a0 = ptx::smem_u32(A), a1 = a0 + (uint32_t)p.HALO * 16;
          const int cc = ch * 8, nc = min(8, p.C - cc), csh = (cc & 15) * 4;
          const unsigned long long *rcg = rc + (cc >> 4) * RT_MAXW;
          for (int pos = tid; pos < p.HALO; pos += 128) {
            const int off = src_off[pos];
            float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (off >= 0) {
              const int lw = off >> 2, sub = off & 3;
              const float4 v0 = *reinterpret_cast<const float4 *>(rv + lw * 64 + cc);
              const float4 v1 = *reinterpret_cast<const float4 *>(rv + lw * 64 + cc + 4);
              const uint32_t nib = (uint32_t)(rcg[lw] >> csh);
              const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const uint32_t cd = (nib >> (4 * j)) & 15u;  // positive*4 + dr*2 + ds (R9)
                o[j] = (j < nc && (cd & 4u) && (int)(cd & 3u) == sub) ? v[j] : 0.f;
              }
            }
            st_shared_v4(a0 + pos * 16, o[0], o[1], o[2], o[3]);
            st_shared_v4(a1 + pos * 16, o[4], o[5], o[6], o[7]);
          }
          ptx::fence_proxy_async_smem();
          ptx::mbar_arrive(full + stage);
          if (++stage == p.nstage) { stage = 0; phase ^= 1; }
        }
        ++rt_tl;
        continue;
      }
      for (int ch = c0; ch < c1; ++ch) {
        const long long t_e0 = clock64();
        ptx::mbar_wait(empty + stage, phase ^ 1);
        const long long t_f0 = clock64();
        if (p.clk && tid == 0) p.clk[blockIdx.x * 16 + 0] += t_f0 - t_e0;
        uint8_t *A = stage_base + (size_t)stage * p.stage_bytes;
        uint8_t *B = A + p.a_bytes;
        if (tid == 0) {
          ptx::mbar_arrive_expect_tx(full + stage, p.b_bytes);
          const float *bsrc = p.fp + ((size_t)ft * p.nchunk + ch) * (p.b_bytes / 4);
          if (p.cl2) {
            const uint32_t half = p.b_bytes / 2;
            ptx::bulk_g2s_mc(B + crank * half, bsrc + crank * (half / 4), half, full + stage, 0x3);
          } else {
            ptx::bulk_g2s(B, bsrc, p.b_bytes, full + stage);
          }
        }
        const uint32_t a0 = ptx::smem_u32(A);
        const uint32_t a1 = a0 + (uint32_t)p.HALO * 16;
        if (p.ks) {
          // dense C == 1 input: element (pos, s) = x(pos + s) for s < S, 0 for S <= s < 8;
          // 4-byte async copies (zero-filled where padded) -> no register round trip
          for (int pos = tid; pos < p.HALO; pos += 128) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int off = e < p.S ? src_off[pos + e] : -1;
              ptx::cp_async4((e < 4 ? a0 : a1) + pos * 16 + (e & 3) * 4, off >= 0 ? p.x + off : p.x,
                             off >= 0 ? 4u : 0u);
            }
          }
        } else {
          int c0 = ch * 8;
          int nc = min(8, p.C - c0);
          int64_t cstride = p.in_plane > 0 ? p.in_plane : (int64_t)HW;
          if (PH && p.in_phase) {
            const int ab = c0 / p.phC;
            if (ab != cur_ab) {  // next phase: every producer has issued from the old table
              ptx::named_bar_sync(1, 128);
              for (int pos = tid; pos < p.HALO; pos += 128) src_off[pos] = phase_off(p, g0 + pos, ab);
              ptx::named_bar_sync(1, 128);
              cur_ab = ab;
            }
            c0 -= ab * p.phC;  // channel of the original image (phC % 8 == 0)
            nc = ab < p.phs * p.phw ? 8 : 0;  // pad channels: zero-fill
            cstride = (int64_t)p.phH * p.phW;
          }
          const float *xc = p.x + c0 * cstride;
          for (int pos = tid; pos < p.HALO; pos += 128) {
            const int off = src_off[pos];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const bool ok = off >= 0 && j < nc;
              ptx::cp_async4((j < 4 ? a0 : a1) + pos * 16 + (j & 3) * 4,
                             ok ? xc + off + j * cstride : p.x, ok ? 4u : 0u);
            }
          }
        }
        ptx::cp_async_mbar_arrive(full + stage);  // arrives when this thread's copies land
        if (p.clk && tid == 0) p.clk[blockIdx.x * 16 + 1] += clock64() - t_f0;
        if (++stage == p.nstage) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ================= MMA issuer (warp 4) | epilogue (warps 5-12, TMEM quadrant warp % 4)
    const int qd = warp & 3;
    const uint32_t idesc = ptx::make_idesc_tf32(128, p.NN);
    int stage = 0;
    uint32_t phase = 0;
    const int PQ = p.P * p.Q;
    const int nc16 = p.NFpad / 16;
    uint32_t tcount = 0;
    TcWork wk = tc_work_init(p);
    int64_t tile;
    int c0, c1;
    for (; tc_next(p, wk, tile, c0, c1); ++tcount) {
      const int ft = (int)(tile % p.nft);
      const int64_t g0 = (tile / p.nft) * p.cta_pos;
      // double buffer: buffers alternate; single buffer (tbuf 0): buffer 0 every tile
      const uint32_t buf = p.tbuf ? (tcount & 1u) : 0u;
      const uint32_t bphase = p.tbuf ? ((tcount >> 1) & 1u) : (tcount & 1u);
      if (warp == 4) {
        // Whole warp runs the issue loop: descriptors stay warp-uniform (uniform
        // registers, no per-MMA conversions).  TMEM columns are addressed from 0:
        // the CTA owns all 512 columns (1 CTA / SM); buffer `buf` = [buf*256, +256).
        const long long t_a0 = clock64();
        ptx::mbar_wait(acce + buf, bphase ^ 1);
        const long long t_a1 = clock64();
        if (p.clk && lane == 0) p.clk[blockIdx.x * 16 + 3] += t_a1 - t_a0;
        ptx::tc_fence_after();
        const int n_inner = p.tile2d ? p.CT : 1;
        const uint32_t step_outer = p.tile2d ? (uint32_t)(16 * p.Wf) : 128u;
        const uint32_t jump_outer = step_outer - 8u * (uint32_t)(n_inner - 1);
        const uint32_t nf = (uint32_t)p.NN;
        const uint32_t sbase = ptx::smem_u32(stage_base);
        for (int ch = c0; ch < c1; ++ch) {
          const long long t_w1 = clock64();
          ptx::mbar_wait(full + stage, phase);
          if (p.clk && lane == 0) p.clk[blockIdx.x * 16 + 2] += clock64() - t_w1;
          ptx::tc_fence_after();
          const uint32_t A = sbase + (uint32_t)stage * p.stage_bytes;
          const uint64_t adesc0 = ptx::make_desc(A, p.HALO * 16, p.a_sbo);
          uint64_t bdesc = ptx::make_desc(A + p.a_bytes, nf * 16, 128);
          uint32_t acc = ch != c0 ? 1u : 0u;
          uint32_t drow = 0;
          if (p.sn && p.snt < p.S) {
            // SN-T: per tap row, MMA 1 (taps s < T, N = T*NF, A unshifted) then MMA 2 (taps
            // s >= T, N = (S-T)*NF, A shifted by T positions) into the same accumulator columns
            const uint32_t n1 = (uint32_t)(p.snt * p.NFpad), n2 = (uint32_t)((p.S - p.snt) * p.NFpad);
            const uint32_t idesc2 = ptx::make_idesc_tf32(128, (int)n2);
            const uint32_t bsrow = A + p.a_bytes;
            for (int r = 0; r < p.R; ++r, drow += (uint32_t)p.Wf) {
              const uint32_t br = bsrow + (uint32_t)r * 2u * (n1 + n2) * 16u;
              const uint64_t bd1 = ptx::make_desc(br, n1 * 16, 128);
              const uint64_t bd2 = ptx::make_desc(br + 2u * n1 * 16u, n2 * 16, 128);
              uint64_t ad = adesc0 + (uint64_t)drow;
              uint32_t tm = buf * p.tbuf;
              for (int i = 0; i < p.MT; ++i) {
                if (ptx::elect_one()) ptx::mma_tf32(tm, ad, bd1, idesc, acc);
                __syncwarp();
                if (ptx::elect_one()) ptx::mma_tf32(tm, ad + (uint64_t)p.snt, bd2, idesc2, 1u);
                __syncwarp();
                tm += nf;
                ad += (uint64_t)jump_outer;  // next M-tile: 128 positions (linear tiles)
              }
              acc = 1u;
            }
          } else {
          // KS: all S column taps are in the K slots; SN: in the N columns
          const int s_taps = (p.ks || p.sn) ? 1 : p.S;
          for (int r = 0; r < p.R; ++r, drow += (uint32_t)p.Wf) {
            for (int s_ = 0; s_ < s_taps; ++s_) {
              uint64_t ad = adesc0 + (uint64_t)(drow + (uint32_t)s_);
              uint32_t tm = buf * p.tbuf;
              int ct = 0;
              for (int i = 0; i < p.MT; ++i) {
                if (ptx::elect_one()) ptx::mma_tf32(tm, ad, bdesc, idesc, acc);
                __syncwarp();
                tm += nf;
                if (++ct == n_inner) { ct = 0; ad += (uint64_t)jump_outer; }
                else ad += 8u;
              }
              acc = 1u;
              bdesc += (uint64_t)(2 * nf);  // next tap: 2 quads x NFpad x 16 B
            }
          }
          }
          if (ptx::elect_one()) {
            if (p.cl2) ptx::mma_commit_mc(empty + stage, 0x3);  // frees the stage in both CTAs
            else ptx::mma_commit(empty + stage);
          }
          __syncwarp();
          if (++stage == p.nstage) { stage = 0; phase ^= 1; }
        }
        if (ptx::elect_one()) ptx::mma_commit(accf + buf);
        __syncwarp();
        if (p.clk && lane == 0) p.clk[blockIdx.x * 16 + 6] += clock64() - t_a1;
        continue;  // the MMA warp goes straight on to the next tile
      }
      ptx::mbar_wait_sleep(accf + buf, bphase);
      __syncwarp();
      const long long t_epi0 = clock64();
      ptx::tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(qd * 32) << 16) + buf * p.tbuf;
      const int eset = (warp - 5) >> 2;  // epilogue warp set 0 / 1 -> even / odd M-tiles
      if (p.sk && (c0 > 0 || c1 < p.nchunk)) {
        if (c0 > 0) {
          // stream-K contributor: publish the raw partial accumulator, no epilogue
          sk_dump(p, tbase, qd * 32 + lane, eset);
          ptx::named_bar_sync(4, 32 * TC_EPI_WARPS);
          if (warp == 5 && lane == 0) {
            __threadfence();
            ptx::st_release_gpu(p.sk_flag + blockIdx.x, 1);
          }
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(acce + buf);
          continue;
        }
        // stream-K owner: add the later segments' partials, then the normal epilogue
        sk_fixup(p, tbase, qd * 32 + lane, eset, c1);
        ptx::tc_fence_before();
        ptx::named_bar_sync(4, 32 * TC_EPI_WARPS);  // both sets' columns are complete
        ptx::tc_fence_after();
        if (warp == 5 && lane == 0)  // reset the consumed flags for the next launch
          for (int cur = c1, j = blockIdx.x + 1; cur < p.nchunk && j < (int)gridDim.x; ++j) {
            cur += (int)(sk_begin(p, j + 1) - sk_begin(p, j));
            p.sk_flag[j] = 0;
          }
      }
      if (p.sn) {
        epi_sn(p, tbase, g0, qd, lane, bias_s, eset, sn_xch);
      } else if (p.pool) {
        epi_pool2(p, tbase, g0, ft, qd, lane, bias_s, eset, 2);
      } else {
        epi_plain<PH>(p, tbase, g0, ft, qd, lane, bias_s, eset, 2);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(acce + buf);
      if (p.clk && lane == 0 && warp == 5) p.clk[blockIdx.x * 16 + 4] += clock64() - t_epi0;
    }
  }
  if (p.clk && threadIdx.x == 160) p.clk[blockIdx.x * 16 + 5] = clock64() - t_kernel0;
  if (p.clk && threadIdx.x == 0) p.clk[blockIdx.x * 16 + 7] = clock64() - t_kernel0;
  __syncthreads();
  if (warp == 4) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, p.tmem_cols);
  }
  if (p.cl2) ptx::cluster_sync();  // no CTA leaves while its peer may still signal it
}

// Repack filters into [ftile][chunk][tap][quad][NFpad][4] (zero padded).
//  flip == 0: packed(k, c, t) = F[k][c][t]        (F is Kout x (Cin*RS))
//  flip == 1: packed(k, c, t) = F[c][k][RS-1-t]   (F is Cin x (Kout*RS): bwd_data)
constexpr int PACK_JB = 32;       // filters per pack block
constexpr int PACK_MAX_RS = 40;   // taps supported by the staged pack (else per-element)

// Block = (32-filter group, chunk, ftile): the filter rows it needs are contiguous in
// F (8*RS floats per filter; for flip, 32*RS per input channel), so they are read
// coalesced into shared memory and written out as [tap][quad][j][4] slabs.
__global__ void __launch_bounds__(256) tc_pack_filters_kernel(
    const float *__restrict__ f, float *__restrict__ fp, int Kout, int Cin, int RS, int NFpad,
    int nft, int nchunk, int flip) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // PDL: the conv may start
  __shared__ float sm[PACK_JB * 8 * PACK_MAX_RS];  // [j][c8 * RS + t]
  const int njb = NFpad / PACK_JB;
  const int jb = blockIdx.x % njb, ch = (blockIdx.x / njb) % nchunk, f_ = blockIdx.x / (njb * nchunk);
  const int k0 = f_ * NFpad + jb * PACK_JB, c0 = ch * 8;
  const int row = 8 * RS;
  // 8 independent loads in flight per thread before the shared-memory stores
  const int total = PACK_JB * row;
  for (int base = threadIdx.x; base < total; base += 8 * blockDim.x) {
    float v[8];
    int dst[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = base + u * blockDim.x;
      v[u] = 0.f;
      dst[u] = -1;
      if (i < total) {
        if (!flip) {
          const int j = i / row, r = i - j * row;
          const int k = k0 + j, c = c0 + r / RS;
          dst[u] = i;
          if (k < Kout && c < Cin) v[u] = __ldg(f + ((size_t)k * Cin + c0) * RS + r);
        } else {
          const int crow = PACK_JB * RS;  // F[c][k0 .. k0+32)[*] is contiguous
          const int cc = i / crow, r = i - cc * crow;
          const int j = r / RS, t = r - j * RS;
          const int k = k0 + j, c = c0 + cc;
          dst[u] = j * row + cc * RS + t;
          if (k < Kout && c < Cin) v[u] = __ldg(f + ((size_t)c * Kout + k0) * RS + r);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (dst[u] >= 0) sm[dst[u]] = v[u];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < RS * 2 * PACK_JB * 4; i += blockDim.x) {
    const int e = i & 3, j = (i >> 2) % PACK_JB, g = (i >> 2) / PACK_JB % 2, tap = i / (2 * PACK_JB * 4);
    const int src_t = flip ? RS - 1 - tap : tap;
    const size_t slab = ((size_t)f_ * nchunk + ch) * RS + tap;
    fp[slab * (8 * NFpad) + (size_t)(g * NFpad + jb * PACK_JB + j) * 4 + e] = sm[j * row + (g * 4 + e) * RS + src_t];
  }
}

// fallback for RS > PACK_MAX_RS: one thread per packed element
__global__ void tc_pack_filters_elem_kernel(const float *__restrict__ f, float *__restrict__ fp,
                                            int Kout, int Cin, int RS, int NFpad, int nft,
                                            int nchunk, int flip) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t total = (int64_t)nft * nchunk * RS * 2 * NFpad * 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int e = (int)(t % 4); t /= 4;
    const int j = (int)(t % NFpad); t /= NFpad;
    const int g = (int)(t % 2); t /= 2;
    const int tap = (int)(t % RS); t /= RS;
    const int ch = (int)(t % nchunk); t /= nchunk;
    const int k = (int)t * NFpad + j, c = ch * 8 + g * 4 + e;
    float v = 0.f;
    if (k < Kout && c < Cin)
      v = flip ? f[((int64_t)c * Kout + k) * RS + (RS - 1 - tap)] : f[((int64_t)k * Cin + c) * RS + tap];
    fp[i] = v;
  }
}

// SN packing: per (chunk, r) the taps s < T as [quad][T*NFpad][4] (column n = s*NFpad + j,
// MMA 1), then the taps s >= T as [quad][(S-T)*NFpad][4] (column n = (s-T)*NFpad + j, MMA 2):
//  packed(j, c, r, s) = F[j][c][r][s] (flip 0) or F[c][j][R-1-r][S-1-s] (flip 1, bwd_data)
__global__ void tc_pack_filters_sn_kernel(const float *__restrict__ f, float *__restrict__ fp,
                                          int Kout, int Cin, int R, int S, int NFpad, int nchunk,
                                          int flip, int T) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int NN = S * NFpad, N1 = T * NFpad;
  const int64_t total = (int64_t)nchunk * R * 2 * NN * 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int e = (int)(t % 4); t /= 4;
    int w = (int)(t % (2 * NN)); t /= 2 * NN;   // position inside the (chunk, r) block
    const int r = (int)(t % R); t /= R;
    const int ch = (int)t;
    int g, n, s0;
    if (w < 2 * N1) { g = w / N1; n = w - g * N1; s0 = 0; }                       // MMA 1 block
    else { w -= 2 * N1; g = w / (NN - N1); n = w - g * (NN - N1); s0 = T; }       // MMA 2 block
    const int s_ = s0 + n / NFpad, j = n % NFpad, c = ch * 8 + g * 4 + e;
    float v = 0.f;
    if (j < Kout && c < Cin)
      v = flip ? f[(((int64_t)c * Kout + j) * R + (R - 1 - r)) * S + (S - 1 - s_)]
               : f[(((int64_t)j * Cin + c) * R + r) * S + s_];
    fp[i] = v;
  }
}

// KS packing (C == 1): [ftile][r][half][NFpad][4] with packed(k, r, 4*half + e) = F[k][0][r][s]
__global__ void tc_pack_filters_ks_kernel(const float *__restrict__ f, float *__restrict__ fp,
                                          int Kout, int R, int S, int NFpad, int nft) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t total = (int64_t)nft * R * 2 * NFpad * 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int e = (int)(t % 4); t /= 4;
    const int j = (int)(t % NFpad); t /= NFpad;
    const int g = (int)(t % 2); t /= 2;
    const int r = (int)(t % R); t /= R;
    const int k = (int)t * NFpad + j, s = g * 4 + e;
    fp[i] = (k < Kout && s < S) ? f[((int64_t)k * R + r) * S + s] : 0.f;
  }
}

int round_up(int a, int b) { return (a + b - 1) / b * b; }

// Plan the forward kernel for a stride-1 conv: input (N,C,H,W), K output channels.
TcPlan plan_fwd(int N, int C, int H, int W, int K, int R, int S, int ph, int pw,
                const PoolArgs *pool, bool allow_ks = true, int sh = 1, int sw = 1, int spf_in = 0,
                int route = 0) {
  TcPlan pl{};
  TcFwdParams &p = pl.p;
  p.N = N; p.C = C; p.H = H; p.W = W; p.K = K; p.R = R; p.S = S; p.ph = ph; p.pw = pw;
  p.sh = sh; p.sw = sw;
  p.ysh = p.ysw = 1;
  pl.ok = false;
  const bool strided = sh != 1 || sw != 1;
  // a strided conv has no shifted-window reuse: only 1x1 filters, on the output grid
  if (sh < 1 || sw < 1 || (strided && (R != 1 || S != 1 || pool))) return pl;
  p.P = (H + 2 * ph - R) / sh + 1;
  p.Q = (W + 2 * pw - S) / sw + 1;
  if (H + 2 * ph - R < 0 || W + 2 * pw - S < 0 || p.P < 1 || p.Q < 1) return pl;
  p.Wf = strided ? p.Q : W + pw;
  p.yH = p.P;
  p.yW = p.Q;
  p.pool = pool ? 1 : 0;
  p.PR = pool ? pool->R : 1;
  p.PS = pool ? pool->S : 1;
  if (pool) {
    // 2-D tiles: window rows must tile the 16-row tile and columns the 8-column tile
    if (p.PR != 2 || p.PS != 2) return pl;  // the fused epilogue implements 2x2/2 windows
    p.Pp = pool->P;
    p.Qp = pool->Q;
  }
  p.Hs = strided ? p.P : round_up(H + ph, p.PR);
  p.Lf = p.Hs * p.Wf;
  p.G = (int64_t)N * p.Lf;
  if (p.G + 4096 >= (1ll << 31)) return pl;
  p.tile2d = pool ? 1 : 0;
  static const int abulk_env = getenv("SYSML_TC_ABULK") ? atoi(getenv("SYSML_TC_ABULK")) : -1;
  p.abulk = (abulk_env != 0 && !pool && R == 1 && S == 1 && ph == 0 && pw == 0 && !strided &&
             ((int64_t)H * W) % 4 == 0 && C > 1 && (int64_t)N * C * H * W < (1ll << 31)) ? 1 : 0;
  // SPF input (LeNet-internal planes, zeros stored): every channel's halo is one contiguous
  // run, so the staged 16-byte producer applies to any R, S.  Opt-in (SYSML_TC_SPF_STAGE=1):
  // measured on the LeNet step (r02) B2d 1011K -> 982K and F2 808K -> 788K cycles per CTA, but
  // the step 1879 -> 1910 us -- the producers were not the limit (the MMA loop is, mma_wait_full
  // is 9% of B2d) and the staging buffer costs pipeline stages.
  static const int spf_stage_env = getenv("SYSML_TC_SPF_STAGE") ? atoi(getenv("SYSML_TC_SPF_STAGE")) : 0;
  if (spf_in && spf_stage_env != 0 && abulk_env != 0 && !strided && C > 1) p.abulk = 2;
  if (K <= 256) {
    p.NFpad = std::max(16, round_up(K, 16));
    p.nft = 1;
  } else {
    // K > 256: 256-wide filter tiles.  SYSML_TC_BALANCE_NF=1 balances the widths instead
    // (K = 320 -> 2 x 160): measured on the horizontally fused bottleneck convs, 320 filters
    // 239 -> 198 us but 640 filters 247 -> 316 us (the 224-wide tiles drop to MT = 1)
    static const int bal_env = getenv("SYSML_TC_BALANCE_NF") ? atoi(getenv("SYSML_TC_BALANCE_NF")) : 0;
    p.nft = (K + 255) / 256;
    p.NFpad = bal_env ? round_up((K + p.nft - 1) / p.nft, 16) : 256;
  }
  p.ks = (allow_ks && C == 1 && S <= 8) ? 1 : 0;
  // SN: narrow filter banks (N = NFpad <= 64 keeps the MMA SMEM-operand bound) fold
  // the column taps into N when S * NFpad still fits one 256-column accumulator
  static const int sn_env = getenv("SYSML_TC_SN") ? atoi(getenv("SYSML_TC_SN")) : -1;
  // (NFpad <= 32 by default: at NFpad = 64 the N = 64 MMAs are only 1.5x SMEM-bound and the
  // SN epilogue costs more than it saves -- ResNet-50 stem (phase) fwd 528 -> 235 us without it;
  // SYSML_TC_SN=2 restores the 64-wide rule)
  const int sn_max = sn_env == 2 ? 64 : 32;
  p.sn = (sn_env != 0 && !p.ks && !pool && p.nft == 1 && S >= 2 && S <= 5 && p.NFpad <= sn_max &&
          S * p.NFpad <= 256 && p.NFpad % 16 == 0)
             ? 1 : 0;
  // SN-T (default): at most 96 accumulator columns per M-tile, so two tiles of 2+ M-tiles fit
  // TMEM and the epilogue of one tile overlaps the MMAs of the next (B2d profile r02: the MMA
  // warp waited 37% of the kernel on the single-buffered 480-column SN accumulator).
  // SYSML_TC_SNT=0 restores all taps in N (single buffer); SYSML_TC_SNT=t forces t.
  static const int snt_env = getenv("SYSML_TC_SNT") ? atoi(getenv("SYSML_TC_SNT")) : -1;
  p.snt = S;
  if (p.sn) {
    if (snt_env < 0) p.snt = std::min(S, std::max(3, 96 / p.NFpad));
    else if (snt_env >= 3) p.snt = std::min(S, snt_env);  // T = 2 (MT = 4) is not supported
  }
  p.NN = p.sn ? p.snt * p.NFpad : p.NFpad;
  p.nchunk = p.ks ? 1 : (C + 7) / 8;
  const int RS = R * S;
  const int b_taps = (p.ks || p.sn) ? R : RS;
  // KS / SN: the S window is in K / N (SN-T: MMA 2 reads A shifted by snt positions)
  const int s_halo = p.ks ? 0 : p.sn ? S - p.snt : S - 1;
  p.b_bytes = (uint32_t)(b_taps * 2 * (p.sn ? S * p.NFpad : p.NN) * 16);
  const int nsm = sm_count();
  const int64_t rows_total = (int64_t)N * p.Hs;
  // TMEM double buffer (epilogue overlaps the next tile's MMAs) unless B-heavy wide
  // tiles want two M-tiles sharing each filter chunk (halves the L2 -> SMEM filter
  // stream) -- then one 512-column accumulator
  static const int single_env = getenv("SYSML_TC_SINGLEBUF") ? atoi(getenv("SYSML_TC_SINGLEBUF")) : -1;
  static const int cluster_env = getenv("SYSML_TC_CLUSTER") ? atoi(getenv("SYSML_TC_CLUSTER")) : -1;
  // 256-wide filter tiles: either a CTA pair sharing every filter chunk by multicast
  // (double-buffered accumulators, MT = 1) or two M-tiles per CTA sharing it (single buffer)
  p.cl2 = (cluster_env == 1) && p.NFpad == 256 && p.nft == 1 && !pool && !p.ks ? 1 : 0;
  const bool single = (!p.cl2 && (single_env < 0 || single_env == 1) && p.NFpad == 256 && !pool) ||
                      (p.sn && p.snt == S);
  p.tbuf = single ? 0u : TMEM_BUF;
  int mt_cap = p.sn ? std::min(SN_MAXMT, (single ? 512 : (int)TMEM_BUF) / p.NN)
                    : std::min(16, (single ? 512 : (int)TMEM_BUF) / p.NFpad);
  static const int mtcap_env = getenv("SYSML_TC_MTCAP") ? atoi(getenv("SYSML_TC_MTCAP")) : 0;
  if (mtcap_env > 0) mt_cap = std::min(mt_cap, mtcap_env);
  p.CT = (p.Q + 7) / 8;
  if (p.tile2d && p.CT > mt_cap) return pl;
  for (int attempt = 0; attempt < 2; ++attempt) {
    int mt = mt_cap;
    for (; mt >= 1; --mt) {
      int bb = 1, halo;
      int64_t cta_pos, ntiles;
      if (p.tile2d) {
        bb = mt / p.CT;
        if (bb < 1) continue;
        cta_pos = (int64_t)bb * 16 * p.Wf;
        halo = (bb - 1) * 16 * p.Wf + (p.CT - 1) * 8 + 15 * p.Wf + 7 + (R - 1) * p.Wf + s_halo + 1;
        halo = round_up(halo, 8);  // LBO multiple of 128 B
        ntiles = ceil_div(rows_total, (int64_t)bb * 16) * p.nft;
      } else {
        // SN: tiles overlap by T-1 rows (output row l needs accumulator rows l .. l+T-1)
        cta_pos = p.sn ? (int64_t)mt * 128 - (p.snt - 1) : (int64_t)mt * 128;
        halo = round_up(mt * 128 + (R - 1) * p.Wf + s_halo, 8);  // LBO multiple of 128 B
        ntiles = ceil_div(p.G, cta_pos) * p.nft;
      }
      if (attempt == 0 && mt > 1 && ntiles < nsm && !single) continue;  // keep the SMs busy first
      const uint32_t a_bytes = (uint32_t)(2 * halo * 16);
      const int stg_row = halo + (p.abulk == 2 ? 4 : 0);
      const uint32_t stage = a_bytes + p.b_bytes + (p.abulk ? (uint32_t)(8 * stg_row * 4) : 0u);
      p.bias_smem = K <= 4096 ? 1 : 0;
      const size_t fixed = (size_t)(halo + 8) * 4 + (p.bias_smem ? (size_t)K * 4 : 0) + 16 + 8 * 24 + 16 + 16 +
                           (route ? (size_t)RT_BYTES : 0) +
                           (p.sn ? (size_t)SN_XCH_FLOATS * 4 : 0);
      const int nst = (int)((SMEM_BUDGET - (int64_t)fixed) / (int64_t)stage);
      if (nst < 2) continue;
      p.MT = p.tile2d ? bb * p.CT : mt;
      p.BB = bb;
      p.HALO = halo;
      p.stg_row = stg_row;
      p.cta_pos = cta_pos;
      p.ntiles = ntiles;
      p.a_bytes = a_bytes;
      p.stage_bytes = stage;
      p.nstage = std::min(nst, 8);
      p.a_sbo = p.tile2d ? (uint32_t)(p.Wf * 16) : 128u;
      pl.smem = (size_t)p.nstage * stage + fixed + 8 * (3 * p.nstage + 4);
      pl.ok = true;
      break;
    }
    if (pl.ok) break;
  }
  if (!pl.ok) return pl;
  if (p.tile2d && (uint32_t)p.Wf * 16 >= (1u << 18)) { pl.ok = false; return pl; }
  if (p.MT * p.NN > (p.tbuf ? (int)p.tbuf : 512)) { pl.ok = false; return pl; }
  p.tmem_cols = 512;  // whole TMEM: base column 0 (1 CTA per SM), issue loops address from 0
  pl.fp_bytes = align_up((size_t)p.nft * p.nchunk * b_taps * 8 * (p.sn ? S * p.NFpad : p.NN) * sizeof(float), 256);
  return pl;
}


// stream-K hand-off flags: per device a ring of TC_SK_SETS sets of TC_SK_MAX_GRID ints,
// zeroed once; each launch takes the next set (a captured graph keeps its set, and its
// replays on one stream are sequential); every flag is reset by the CTA that consumes it.
constexpr int TC_SK_SETS = 64, TC_SK_MAX_GRID = 256;
static int *sk_flag_set(cudaStream_t st) {
  static std::mutex mu;
  static int *base[64] = {};
  static unsigned ctr[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!base[dev]) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
    int *b = nullptr;
    if (cudaMalloc(&b, sizeof(int) * TC_SK_SETS * TC_SK_MAX_GRID) != cudaSuccess) return nullptr;
    if (cudaMemset(b, 0, sizeof(int) * TC_SK_SETS * TC_SK_MAX_GRID) != cudaSuccess) return nullptr;
    base[dev] = b;
  }
  return base[dev] + (ctr[dev]++ % TC_SK_SETS) * TC_SK_MAX_GRID;
}

// workspace for the stream-K partial accumulators: one slot of <= 512 TMEM columns x 128
// rows per CTA (behind the packed filters)
static size_t sk_ws_bytes() {
  static const bool on = getenv("SYSML_TC_SK") && atoi(getenv("SYSML_TC_SK")) == 1;
  return on ? align_up((size_t)sm_count() * 512 * 128 * sizeof(float), 256) : 0;
}

sysml_status run_fwd(TcPlan &pl, const float *x, const float *f, int flip, int f_cin,
                     const float *bias, float *y, float *pout, int32_t *parg, void *ws,
                     cudaStream_t st, const TcSpfIO *io = nullptr, const sysml_csr *csr = nullptr) {
  TcFwdParams p = pl.p;
  if (csr) {
    if (!p.ks) {
      set_error("tcgen05 forward: CSR input needs the single-channel (KS) mode");
      return SYSML_ERR_UNSUPPORTED;
    }
    p.is_csr = 1;
    p.csr = *csr;
  }
  if (io) {
    p.in_plane = io->in_plane;
    p.in_shift = io->in_shift;
    p.route_val = io->route_val;
    p.route_code = io->route_code;
    p.route_cplane = io->route_cplane;
    p.route_C = io->route_C;
    p.route_Pp = io->route_Pp;
    p.route_Qp = io->route_Qp;
    p.route_Wf = io->route_Wf;
    p.route_Lf = io->route_Lf;
    if (p.route_val && (p.ks || p.is_csr || p.in_plane <= 0 || (p.route_C != 64) || p.C > p.route_C || p.HALO > 384 || p.sk || (p.route_cplane & 1) ||
                        ((uintptr_t)p.route_val & 15))) {
      set_error("tcgen05 forward: routed SPF input needs C %% 8 == 0 planes and 16-byte aligned values");
      return SYSML_ERR_UNSUPPORTED;
    }
    p.out_plane = io->out_plane;
    p.out_Wf = io->out_Wf;
    p.out_Lf = io->out_Lf;
    p.out_off = io->out_off;
    p.pcode = io->code;
    p.code_plane = io->code_plane;
    p.y_nhwc = io->out_nhwc;
    if (p.y_nhwc && (!p.sn || (p.K & 3) || ((uintptr_t)y & 15))) {
      set_error("tcgen05 forward: channel-minor output needs the SN epilogue, K %% 4 == 0 and a 16-byte aligned y");
      return SYSML_ERR_UNSUPPORTED;
    }
    if (p.pcode && !(p.pool && p.tile2d)) {
      set_error("tcgen05 forward: packed window codes need the fused 2x2 pool epilogue");
      return SYSML_ERR_UNSUPPORTED;
    }
  }
  if (p.abulk == 1 && (p.cl2 || p.in_plane > 0 || p.is_csr || ((uintptr_t)x & 15))) p.abulk = 0;  // NCHW only
  if (p.abulk == 2 && (p.cl2 || p.in_plane <= 0 || (p.in_plane & 3) || p.in_phase || p.is_csr ||
                       ((uintptr_t)x & 15) || p.route_val))
    p.abulk = 0;  // SPF only

  float *fp = reinterpret_cast<float *>(ws);
  if (p.ks) {
    if (flip) {
      set_error("tcgen05 KS mode does not implement the flipped (bwd_data) packing");
      return SYSML_ERR_UNSUPPORTED;
    }
    const int64_t total = (int64_t)p.nft * p.R * 2 * p.NFpad * 4;
    const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 4 * sm_count());
    tc_pack_filters_ks_kernel<<<blocks, 256, 0, st>>>(f, fp, p.K, p.R, p.S, p.NFpad, p.nft);
    SYSML_LAUNCH_CHECK();
  } else if (p.sn) {
    const int64_t total = (int64_t)p.nchunk * p.R * 2 * p.S * p.NFpad * 4;
    const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 8 * sm_count());
    tc_pack_filters_sn_kernel<<<blocks, 256, 0, st>>>(f, fp, p.K, f_cin, p.R, p.S, p.NFpad, p.nchunk, flip, p.snt);
    SYSML_LAUNCH_CHECK();
  } else {
    const int RS = p.R * p.S;
    const int slab_blocks = p.nft * p.nchunk * (p.NFpad / PACK_JB);
    if (RS <= PACK_MAX_RS && p.NFpad % PACK_JB == 0 && slab_blocks >= sm_count()) {
      tc_pack_filters_kernel<<<p.nft * p.nchunk * (p.NFpad / PACK_JB), 256, 0, st>>>(
          f, fp, p.K, f_cin, RS, p.NFpad, p.nft, p.nchunk, flip);
    } else {
      const int64_t total = (int64_t)p.nft * p.nchunk * RS * 2 * p.NFpad * 4;
      const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 8 * sm_count());
      tc_pack_filters_elem_kernel<<<blocks, 256, 0, st>>>(f, fp, p.K, f_cin, RS, p.NFpad, p.nft,
                                                           p.nchunk, flip);
    }
    SYSML_LAUNCH_CHECK();
  }
  p.x = x;
  p.fp = fp;
  p.bias = bias;
  p.y = y;
  p.pout = pout;
  p.parg = parg;
  if (!bias) p.bias_smem = 0;
  const bool ph = p.in_phase || p.out_phase;
  if (ph) {
    SYSML_TRY(smem_attr(tc_conv_fwd_kernel<1>, pl.smem));
  } else if (p.route_val) {
    SYSML_TRY(smem_attr(tc_conv_fwd_kernel<2>, pl.smem));
  } else {
    SYSML_TRY(smem_attr(tc_conv_fwd_kernel<0>, pl.smem));
  }
  int grid = (int)std::min<int64_t>(p.ntiles, sm_count());
  // stream-K (opt-in, SYSML_TC_SK=1): even chunk-iteration ranges per CTA instead of whole
  // tiles.  Measured slower on every shape of this build -- single-buffered accumulators
  // serialise the contributor's partial dump with its next segment's MMAs, and short tiles
  // (LeNet conv2: 4 chunks) pay a second halo prologue and epilogue per split tile -- so the
  // default stays round-robin whole tiles.
  p.sk = 0;
  p.sk_part = nullptr;
  p.sk_flag = nullptr;
  {
    static const int sk_env = getenv("SYSML_TC_SK") ? atoi(getenv("SYSML_TC_SK")) : 0;
    const int nsm = sm_count();
    if (sk_env == 1 && !p.cl2 && !p.is_csr &&
        p.ntiles * (int64_t)p.nchunk >= 2 * nsm && nsm <= TC_SK_MAX_GRID) {
      int *flags = sk_flag_set(st);
      if (flags) {
        p.sk = 1;
        p.sk_flag = flags;
        p.sk_part = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(ws) + align_up(pl.fp_bytes, 256));
        grid = nsm;
      }
    }
  }
  if (p.cl2) {
    if (grid < 2) p.cl2 = 0;
    else grid &= ~1;
  }
  p.iters = ceil_div(p.ntiles, grid);
  static long long *dclk = nullptr;
  const bool prof = getenv("SYSML_TC_PROFILE") != nullptr;
  p.clk = nullptr;
  if (prof) {
    if (!dclk) cudaMalloc(&dclk, sizeof(long long) * 16 * 1024);
    cudaMemsetAsync(dclk, 0, sizeof(long long) * 16 * 1024, st);
    p.clk = dclk;
  }
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(TC_FWD_THREADS);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap the pack kernel
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
    if (p.cl2) {
      at[na].id = cudaLaunchAttributeClusterDimension;
      at[na].val.clusterDim.x = 2;
      at[na].val.clusterDim.y = 1;
      at[na].val.clusterDim.z = 1;
      ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    route_note("tc_conv_fwd_kernel%s [tcgen05 TF32, %s%s, MT=%d, N=%d, %d tiles on %d CTAs%s]", ph ? "<phase>" : "",
               p.ks ? "KS" : p.sn ? (p.snt < p.S ? "SN-T" : "SN") : "standard",
               p.is_csr ? " CSR" : p.abulk == 2 ? " staged-SPF" : p.abulk ? " staged" : "", p.MT, p.NN, (int)p.ntiles, grid,
               p.pool ? ", pool epilogue" : "");
    SYSML_CUDA(cudaLaunchKernelEx(&cfg, ph ? tc_conv_fwd_kernel<1> : p.route_val ? tc_conv_fwd_kernel<2> : tc_conv_fwd_kernel<0>, p));
  }
  SYSML_LAUNCH_CHECK();
  if (prof) {
    static long long h[16 * 1024];
    cudaMemcpyAsync(h, dclk, sizeof(long long) * 16 * grid, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double a[16] = {0};
    for (int b = 0; b < grid; ++b)
      for (int j = 0; j < 16; ++j) a[j] += (double)h[b * 16 + j] / grid;
    fprintf(stderr, "[tc_fwd N=%d C=%d K=%d MT=%d nstage=%d tiles=%lld] prod_wait_empty %.0f prod_fill %.0f "
            "mma_wait_full %.0f mma_wait_acce %.0f epilogue %.0f total_warp4 %.0f mma_loop %.0f total_prod %.0f\n",
            p.N, p.C, p.K, p.MT, p.nstage, (long long)p.ntiles, a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7]);
    if (p.sn)
      fprintf(stderr, "  [sn epi] dump %.0f bar1 %.0f tmem_ld %.0f shfl_add %.0f store %.0f bar2 %.0f\n", a[8], a[9],
              a[10], a[11], a[12], a[13]);
  }
  return SYSML_OK;
}

bool pool_fusable(const PoolArgs *pool) {
  return !pool || (pool->sh == pool->R && pool->sw == pool->S && pool->ph == 0 && pool->pw == 0);
}

// =====================================================================================
// bwd_filter (weight gradient) kernel
// =====================================================================================
// Frame width Wf4 = round_up(W + pw, 4), so a tap shift d = rg*copies*Wf4 + s splits
// into a whole number of 4-position quads (a = d >> 2) plus a phase (s mod 4): the X
// halo is staged K-major ([pos quad][channel][4 pos]) once per phase (X shifted by
// phi = 0..nph-1 positions) and every tap is a descriptor offset into its phase copy.
struct TcWgParams {
  const float *x, *dy;
  float *part;    // [split][wt][tgc][128][NC]
  float *dbpart;  // [split][K] (or null)
  int N, C, H, W, K, R, S, ph, pw, P, Q;
  int Wf, Hs, Lf;
  int64_t G, Gext;
  int Kc, copies, nkt;   // filters per copy, copies (128/Kc), filter tiles of 128
  int NC, nct;           // channels per tile (mult of 16), channel tiles
  int RG, TGt, TGc, ntg; // tap row groups, tap groups total / per CTA, tap-group tiles
  int nwt;               // work types = nkt*nct*ntg
  int splits;
  int64_t pos_per_split;
  int KC;                // positions per stage (multiple of 8)
  int nph, HBq, XT;      // phases, B quads per phase, X offset table length
  int dmax;              // max tap shift
  int YT;                // dY offset table length = KC + (copies-1)*Wf
  int nstage;
  uint32_t a_bytes, b_bytes, phase_bytes, stage_bytes;
  uint32_t tmem_cols;
};

struct TcWgPlan {
  TcWgParams p;
  size_t smem, part_bytes, dbpart_bytes;
  bool ok;
};

__global__ void __launch_bounds__(TC_THREADS, 1) tc_conv_wgrad_kernel(const TcWgParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *stage_base = smem;
  int *ytab = reinterpret_cast<int *>(smem + (size_t)p.nstage * p.stage_bytes);  // [nstage][YT]
  int *xtab = ytab + p.nstage * p.YT;                                            // [nstage][XT]
  float *dbs = reinterpret_cast<float *>(xtab + p.nstage * p.XT);                 // [128]
  uint64_t *bars = reinterpret_cast<uint64_t *>(
      (reinterpret_cast<uintptr_t>(dbs + 128) + 15) & ~(uintptr_t)15);
  uint64_t *full = bars;
  uint64_t *empty = bars + p.nstage;
  uint64_t *accf = bars + 2 * p.nstage;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accf + 1);

  // warp index via shuffle: provably warp-uniform, so role branches keep the uniform datapath
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  // work decomposition: blockIdx.x = split * nwt + wt; wt = (kt * nct + ct) * ntg + tgt
  const int wt = blockIdx.x % p.nwt;
  const int split = blockIdx.x / p.nwt;
  const int tgt = wt % p.ntg;
  const int ct = (wt / p.ntg) % p.nct;
  const int kt = wt / (p.ntg * p.nct);
  const int tg0 = tgt * p.TGc;
  const int tgn = min(p.TGc, p.TGt - tg0);
  const int64_t gs = (int64_t)split * p.pos_per_split;
  const int64_t ge = min(p.Gext, gs + p.pos_per_split);
  const int64_t span = ge > gs ? ge - gs : 0;
  const int nchunks = (int)((span + p.KC - 1) / p.KC);
  const bool do_db = p.dbpart != nullptr && ct == 0 && tgt == 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nstage; ++s) {
      ptx::mbar_init(full + s, 4);
      ptx::mbar_init(empty + s, 1);
    }
    ptx::mbar_init(accf, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 4) ptx::tmem_alloc(tmem_slot, p.tmem_cols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int HW = p.H * p.W, PQ = p.P * p.Q;

  if (warp < 4) {
    // ================= producers
    const int tid = threadIdx.x;
    // A row owned by this thread: copy j = tid / Kc, filter k = kt*128 + tid % Kc
    const int arow = tid;
    const int aj = arow / p.Kc;
    const int ak = kt * 128 + (arow - aj * p.Kc);
    const bool arow_ok = aj < p.copies && ak < p.K;
    float db_acc = 0.f;
    int stage = 0;
    uint32_t phase = 0;
    for (int ch = 0; ch < nchunks; ++ch) {
      const int64_t u0 = gs + (int64_t)ch * p.KC;
      ptx::mbar_wait_sleep(empty + stage, phase ^ 1);
      int *yt = ytab + stage * p.YT;
      int *xt = xtab + stage * p.XT;
      // dY offsets for output-frame positions u0 - (copies-1)*Wf + e, e < YT
      for (int e = tid; e < p.YT; e += 128) {
        const int64_t g = u0 - (int64_t)(p.copies - 1) * p.Wf + e;
        int off = -1;
        if (g >= 0 && g < p.G) {
          const int n = (int)(g / p.Lf);
          const int rem = (int)(g - (int64_t)n * p.Lf);
          const int hh = rem / p.Wf, q = rem - hh * p.Wf;
          if (hh < p.P && q < p.Q) off = n * p.K * PQ + hh * p.Q + q;
        }
        yt[e] = off;
      }
      // X offsets for input-frame positions u0 + e, e < XT
      for (int e = tid; e < p.XT; e += 128) {
        const int64_t gi = u0 + e;
        int off = -1;
        if (gi < p.G) {
          const int n = (int)(gi / p.Lf);
          const int rem = (int)(gi - (int64_t)n * p.Lf);
          const int hh = rem / p.Wf, ww = rem - hh * p.Wf;
          const int h = hh - p.ph, w = ww - p.pw;
          if (h >= 0 && h < p.H && w >= 0 && w < p.W) off = n * p.C * HW + h * p.W + w;
        }
        xt[e] = off;
      }
      ptx::named_bar_sync(1, 128);
      const uint32_t A = ptx::smem_u32(stage_base + (size_t)stage * p.stage_bytes);
      const uint32_t B = A + p.a_bytes;
      
// ---- A: row = (copy j, filter k); K-major [pos quad][128 rows][4 pos]
      {
        const int shift = (p.copies - 1 - aj) * p.Wf;  // yt index of position u0 + u - j*Wf
        const float *dyk = p.dy + (size_t)(arow_ok ? ak : 0) * PQ;
        for (int qb = 0; qb < p.KC / 4; qb += 4) {
          float v[4][4];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int u = (qb + a) * 4 + e;
              // positions at or past this CTA's range end belong to the next CTA
              const int off = (arow_ok && qb + a < p.KC / 4 && u0 + u < ge) ? yt[shift + u] : -1;
              v[a][e] = off >= 0 ? __ldg(dyk + off) : 0.f;
            }
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            if (qb + a < p.KC / 4) {
              st_shared_v4(A + (uint32_t)(((qb + a) * 128 + arow) * 16), v[a][0], v[a][1], v[a][2], v[a][3]);
              if (do_db && aj == 0) {
#pragma unroll
                for (int e = 0; e < 4; ++e) db_acc += v[a][e];
              }
            }
          }
        }
      }
      // ---- B: X halo, K-major per phase: [phase][pos quad][NC][4 pos]
      {
        const int c0 = ct * p.NC;
        const int ntask = p.NC * p.HBq;
        for (int t0 = tid; t0 < ntask; t0 += 2 * 128) {
          float v[2][7];
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            const int t = t0 + a * 128;
            const int cq = t / p.HBq;  // channel (within tile)
            const int qd_ = t - cq * p.HBq;
            const int c = c0 + cq;
            const bool ok = t < ntask && c < p.C;
            const float *xc = p.x + (size_t)(ok ? c : 0) * HW;
#pragma unroll
            for (int e = 0; e < 7; ++e) {
              const int off = (ok && e < 3 + p.nph) ? xt[qd_ * 4 + e] : -1;
              v[a][e] = off >= 0 ? __ldg(xc + off) : 0.f;
            }
          }
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            const int t = t0 + a * 128;
            if (t < ntask) {
              const int cq = t / p.HBq;
              const int qd_ = t - cq * p.HBq;
              const uint32_t dst = B + (uint32_t)((qd_ * p.NC + cq) * 16);
#pragma unroll
              for (int f = 0; f < 4; ++f)
                if (f < p.nph)
                  st_shared_v4(dst + f * p.phase_bytes, v[a][f], v[a][f + 1], v[a][f + 2], v[a][f + 3]);
            }
          }
        }
      }
      ptx::fence_proxy_async_smem();
      ptx::named_bar_sync(1, 128);
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(full + stage);
      if (++stage == p.nstage) { stage = 0; phase ^= 1; }
    }
    if (do_db) {
      // fixed-order reduction: thread arow (copy 0 rows only) owns filter ak
      dbs[arow] = db_acc;
      ptx::named_bar_sync(1, 128);
      if (tid < p.Kc && ak < p.K) p.dbpart[(size_t)split * p.K + ak] = dbs[tid];
    }
  } else {
    const int qd = warp - 4;
    if (warp == 4) {
      const uint32_t idesc = ptx::make_idesc_tf32(128, p.NC);  // A, B K-major
      int stage = 0;
      uint32_t phase = 0;
      // tap groups handled by this CTA, in (rg, s) order from tg0
      const int rg0 = tg0 / p.S, s0 = tg0 - rg0 * p.S;
      for (int ch = 0; ch < nchunks; ++ch) {
        ptx::mbar_wait(full + stage, phase);
        ptx::tc_fence_after();
        const uint32_t A = ptx::smem_u32(stage_base + (size_t)stage * p.stage_bytes);
        const uint32_t B = A + p.a_bytes;
        const uint64_t adesc0 = ptx::make_desc(A, 128 * 16, 128);
        const uint64_t bdesc0 = ptx::make_desc(B, (uint32_t)p.NC * 16, 128);
        for (int kk = 0; kk < p.KC / 8; ++kk) {
          const uint64_t adesc = adesc0 + (uint64_t)(kk * 2 * 128);  // 2 pos quads x 2048 B
          int rg = rg0, s_ = s0;
          uint32_t tm = 0;  // CTA owns all 512 TMEM columns
          const uint32_t acc = (ch | kk) != 0 ? 1u : 0u;
          for (int tl = 0; tl < tgn; ++tl) {
            const uint32_t d = (uint32_t)(rg * p.copies * p.Wf + s_);
            const uint64_t bdesc = bdesc0 + (uint64_t)((d & 3u) * (p.phase_bytes >> 4)) +
                                   (uint64_t)((2 * kk + (int)(d >> 2)) * p.NC);
            if (ptx::elect_one()) ptx::mma_tf32(tm, adesc, bdesc, idesc, acc);
            __syncwarp();
            tm += (uint32_t)p.NC;
            if (++s_ == p.S) { s_ = 0; ++rg; }
          }
        }
        if (ptx::elect_one()) ptx::mma_commit(empty + stage);
        __syncwarp();
        if (++stage == p.nstage) { stage = 0; phase ^= 1; }
      }
      if (ptx::elect_one()) ptx::mma_commit(accf);
      __syncwarp();
    }
    ptx::mbar_wait_sleep(accf, 0);
    __syncwarp();
    ptx::tc_fence_after();
    // epilogue: partial[split][wt][tl][row][NC]; zero if no chunk ran
    const int row = qd * 32 + lane;
    float *dst = p.part + (((size_t)split * p.nwt + wt) * p.TGc) * 128 * p.NC;
    for (int tl = 0; tl < p.TGc; ++tl) {
      for (int c16 = 0; c16 < p.NC / 16; ++c16) {
        float v[16];
        if (tl < tgn && nchunks > 0) {
          ptx::tmem_ld16(tmem_base + ((uint32_t)(qd * 32) << 16) + (uint32_t)(tl * p.NC + c16 * 16), v);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = 0.f;
        }
        float4 *o = reinterpret_cast<float4 *>(dst + ((size_t)tl * 128 + row) * p.NC + c16 * 16);
        o[0] = make_float4(v[0], v[1], v[2], v[3]);
        o[1] = make_float4(v[4], v[5], v[6], v[7]);
        o[2] = make_float4(v[8], v[9], v[10], v[11]);
        o[3] = make_float4(v[12], v[13], v[14], v[15]);
      }
    }
    ptx::tc_fence_before();
  }
  __syncthreads();
  if (warp == 4) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// dF[k][c][r][s] = sum_{split} part[split][wt(k,c,r,s)][tl][row][col]  (split ascending)
__global__ void tc_wgrad_reduce_kernel(const TcWgParams p, float *__restrict__ df,
                                       float *__restrict__ db) {
  const int RS = p.R * p.S;
  const int64_t total = (int64_t)p.K * p.C * RS;
  const size_t split_stride = (size_t)p.nwt * p.TGc * 128 * p.NC;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / ((int64_t)p.C * RS));
    const int rem = (int)(i - (int64_t)k * p.C * RS);
    const int c = rem / RS, t = rem - c * RS, r = t / p.S, s = t - r * p.S;
    const int kt = k / 128, kk = k - kt * 128;
    const int ct = c / p.NC, col = c - ct * p.NC;
    const int rg = r / p.copies, j = r - rg * p.copies;
    const int tg = rg * p.S + s;
    const int tgt = tg / p.TGc, tl = tg - tgt * p.TGc;
    const int wt = (kt * p.nct + ct) * p.ntg + tgt;
    const int row = j * p.Kc + kk;
    const size_t off = (((size_t)wt * p.TGc + tl) * 128 + row) * p.NC + col;
    float acc = 0.f;
    for (int sp = 0; sp < p.splits; ++sp) acc += p.part[(size_t)sp * split_stride + off];
    df[i] = acc;
  }
  if (db) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < p.K;
         k += (int64_t)gridDim.x * blockDim.x) {
      float acc = 0.f;
      for (int sp = 0; sp < p.splits; ++sp) acc += p.dbpart[(size_t)sp * p.K + k];
      db[k] = acc;
    }
  }
}

TcWgPlan plan_wgrad(const ConvArgs &a) {
  TcWgPlan pl{};
  TcWgParams &p = pl.p;
  pl.ok = false;
  if (a.sh != 1 || a.sw != 1) return pl;
  p.N = a.N; p.C = a.C; p.H = a.H; p.W = a.W; p.K = a.K; p.R = a.R; p.S = a.S;
  p.ph = a.ph; p.pw = a.pw; p.P = a.P; p.Q = a.Q;
  p.Wf = round_up(a.W + a.pw, 4);
  p.Hs = a.H + a.ph;
  p.Lf = p.Hs * p.Wf;
  p.G = (int64_t)a.N * p.Lf;
  if (p.G + 8192 >= (1ll << 31)) return pl;
  if (a.K >= 128) { p.Kc = 128; p.copies = 1; p.nkt = (a.K + 127) / 128; }
  else {
    p.Kc = a.K <= 16 ? 16 : a.K <= 32 ? 32 : a.K <= 64 ? 64 : 128;
    p.copies = 128 / p.Kc;
    if (p.copies > a.R) p.copies = std::max(1, a.R);  // extra copies would compute nothing
    while (128 % (p.Kc * p.copies) != 0) --p.copies;
    p.nkt = 1;
  }
  p.nph = std::min(a.S, 4);
  p.RG = (a.R + p.copies - 1) / p.copies;
  p.TGt = p.RG * a.S;
  p.dmax = (p.RG - 1) * p.copies * p.Wf + (a.S - 1);
  p.Gext = p.G + (int64_t)(p.copies - 1) * p.Wf;
  // channel tile: as wide as TMEM allows for >= min(TGt, 8) tap groups, >= 16
  int nc = std::min(256, round_up(std::max(a.C, 16), 16));
  while (nc > 16 && std::min(p.TGt, 8) * nc > 512) nc -= 16;
  bool planned = false;
  for (; nc >= 16 && !planned; nc -= 16) {
    p.NC = nc;
    p.nct = (a.C + p.NC - 1) / p.NC;
    p.TGc = std::min(p.TGt, 512 / p.NC);
    p.ntg = (p.TGt + p.TGc - 1) / p.TGc;
    p.nwt = p.nkt * p.nct * p.ntg;
    for (p.KC = 64; p.KC >= 8; p.KC /= 2) {
      p.HBq = p.KC / 4 + (p.dmax >> 2);
      p.XT = p.HBq * 4 + 4;
      p.YT = p.KC + (p.copies - 1) * p.Wf;
      p.a_bytes = (uint32_t)(p.KC * 128 * 4);
      p.phase_bytes = (uint32_t)(p.HBq * p.NC * 16);
      p.b_bytes = (uint32_t)p.nph * p.phase_bytes;
      p.stage_bytes = p.a_bytes + p.b_bytes;
      const size_t per_stage = p.stage_bytes + 4 * (size_t)(p.YT + p.XT);
      const size_t fixed = 128 * 4 + 16 + 8 * 20 + 16;
      const int nst = (int)((SMEM_BUDGET - (int64_t)fixed) / (int64_t)per_stage);
      if (nst >= 2) {
        p.nstage = std::min(nst, 4);
        pl.smem = (size_t)p.nstage * per_stage + fixed + 8 * (2 * p.nstage + 1);
        planned = true;
        break;
      }
    }
  }
  if (!planned) return pl;
  // split the position range: ~2 CTAs per SM worth of work items
  const int64_t target = 2ll * sm_count();
  int64_t splits = std::max<int64_t>(1, target / p.nwt);
  const int64_t max_splits = std::max<int64_t>(1, ceil_div(p.Gext, 4 * p.KC));
  splits = std::min(splits, max_splits);
  p.pos_per_split = align_up((size_t)ceil_div(p.Gext, splits), (size_t)p.KC);
  p.splits = (int)ceil_div(p.Gext, p.pos_per_split);
  uint32_t cols = 32;
  while (cols < (uint32_t)(p.TGc * p.NC)) cols <<= 1;
  if (cols > 512) return pl;
  p.tmem_cols = 512;  // whole TMEM: base column 0 (1 CTA per SM), issue loops address from 0
  pl.part_bytes = align_up((size_t)p.splits * p.nwt * p.TGc * 128 * p.NC * sizeof(float), 256);
  pl.dbpart_bytes = align_up((size_t)p.splits * p.K * sizeof(float), 256);
  pl.ok = true;
  return pl;
}

// =====================================================================================
// bwd_filter on stacked-planar-frame (SPF) tensors -- the LeNet step's internal layout
// =====================================================================================
// SPF: tensor [C][G] with G = N * Hs * Wf stacked frame positions (Wf % 4 == 0), zeros in
// every padding / garbage position, plane stride a multiple of 4 floats.  Every 4
// consecutive positions are one aligned float4, so producers stream with 16-byte loads
// and no index decoding.
//   A rows (j, k): dY[k][g - j*Wf]              (copy j -> tap row r + j)
//   B rows (s, c): X[c][g + s]                  (all S column taps in one MMA: N = S*C)
//   D_rg[(j,k)][(s,c)] += A . B shifted by rg*copies*Wf  ->  dF[k][c][rg*copies + j][s]
// One K-step (8 positions) issues RG MMAs of N = S*C instead of R*S small ones.
struct TcWgSpfParams {
  const float *x, *dy;   // SPF planes
  int64_t plane_x, plane_dy;
  int x_shift, dy_shift;  // stored position = frame position + shift
  float *part;            // [split][RG][128][NB]
  float *dbpart;          // [split][K] or null
  int64_t G, Gext;
  int K, C, R, S, Wf;
  int Kc, copies, RG, NB;
  int KC, HBq, nstage;
  int splits;
  int64_t pos_per_split;
  uint32_t a_bytes, b_bytes, stage_bytes;
  long long *clk;  // optional per-CTA cycle counters (SYSML_TC_PROFILE)
};

constexpr int WG_THREADS = 288;  // 8 producer/epilogue warps + 1 MMA warp

__device__ __forceinline__ float4 ld_f4(const float *p) { return __ldg(reinterpret_cast<const float4 *>(p)); }

template <int S_>
__global__ void __launch_bounds__(WG_THREADS, 1) tc_wgrad_spf_kernel(const TcWgSpfParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *stage_base = smem;
  float *dbs = reinterpret_cast<float *>(smem + (size_t)p.nstage * p.stage_bytes);  // [256]
  uint64_t *bars = reinterpret_cast<uint64_t *>(dbs + 256);
  uint64_t *full = bars;
  uint64_t *empty = bars + p.nstage;
  uint64_t *accf = bars + 2 * p.nstage;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accf + 1);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int split = blockIdx.x;
  const int64_t gs = (int64_t)split * p.pos_per_split;
  const int64_t ge = min(p.Gext, gs + p.pos_per_split);
  const int64_t span = ge > gs ? ge - gs : 0;
  const int nchunks = (int)((span + p.KC - 1) / p.KC);
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nstage; ++s) {
      ptx::mbar_init(full + s, 8);
      ptx::mbar_init(empty + s, 1);
    }
    ptx::mbar_init(accf, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 8) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < 8) {
    const int tid = threadIdx.x;
    // A task: fixed row (tid / 2) and quad half (tid % 2) of the KC/4 quads
    const int arow = tid >> 1, ahalf = tid & 1;
    const int aj = arow / p.Kc, ak = arow - aj * p.Kc;
    const bool arow_ok = aj < p.copies && ak < p.K;
    const int nq = p.KC / 4, qper = (nq + 1) / 2;  // KC <= 32: at most 4 quads per half
    const float *dyk = p.dy + (arow_ok ? (int64_t)ak * p.plane_dy : 0);
    float db_acc = 0.f;
    // B task: channel c, group of 4 quads
    const int ngrp = (p.HBq + 3) / 4;
    const int ntask = p.C * ngrp;
    struct Regs {
      float4 va[4];
      float vb[2][20];
    };
    // global -> registers for chunk ch (A: 4 float4, B: up to 2 x 5 float4)
    auto load = [&](int ch, Regs &R) {
      const int64_t u0 = gs + (int64_t)ch * p.KC;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int q = ahalf * qper + i;
        R.va[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < qper && q < nq && arow_ok) {
          const int64_t pos = u0 + 4 * q;          // CTA-range position of this quad
          const int64_t src = pos - (int64_t)aj * p.Wf;
          if (pos < ge && src >= 0 && src < p.G) R.va[i] = ld_f4(dyk + src + p.dy_shift);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int t = tid + u * 256;
        const int c = t % p.C, q0 = (t / p.C) * 4;
        const float *xc = p.x + (int64_t)c * p.plane_x + p.x_shift;
#pragma unroll
        for (int i = 0; i < 5; ++i) {
          const int64_t pos = u0 + 4 * (q0 + i);
          float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
          if (t < ntask && q0 + i < p.HBq + 1 && pos < p.G) f = ld_f4(xc + pos);
          R.vb[u][4 * i] = f.x; R.vb[u][4 * i + 1] = f.y; R.vb[u][4 * i + 2] = f.z; R.vb[u][4 * i + 3] = f.w;
        }
      }
    };
    // registers -> the stage's shared-memory operands (A rows (j,k); B rows (s,c) with
    // lanes on consecutive channels: conflict-free 16-byte stores)
    auto store = [&](const Regs &R, uint32_t A, uint32_t B) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int q = ahalf * qper + i;
        if (i < qper && q < nq) {
          st_shared_v4(A + (uint32_t)((q * 128 + arow) * 16), R.va[i].x, R.va[i].y, R.va[i].z, R.va[i].w);
          if (aj == 0) db_acc += (R.va[i].x + R.va[i].y) + (R.va[i].z + R.va[i].w);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int t = tid + u * 256;
        if (t >= ntask) continue;
        const int c = t % p.C, q0 = (t / p.C) * 4;
#pragma unroll
        for (int qi = 0; qi < 4; ++qi) {
          const int q = q0 + qi;
          if (q < p.HBq) {
#pragma unroll
            for (int s_ = 0; s_ < S_; ++s_)
              st_shared_v4(B + (uint32_t)(((q * p.NB) + s_ * p.C + c) * 16), R.vb[u][4 * qi + s_],
                           R.vb[u][4 * qi + s_ + 1], R.vb[u][4 * qi + s_ + 2], R.vb[u][4 * qi + s_ + 3]);
          }
        }
      }
    };
    int stage = 0;
    uint32_t phase = 0;
    auto publish = [&](const Regs &R) {
      const long long t0 = clock64();
      ptx::mbar_wait(empty + stage, phase ^ 1);
      if (p.clk && tid == 0) p.clk[blockIdx.x * 8 + 0] += clock64() - t0;
      const uint32_t A = ptx::smem_u32(stage_base + (size_t)stage * p.stage_bytes);
      store(R, A, A + p.a_bytes);
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(full + stage);
      if (++stage == p.nstage) { stage = 0; phase ^= 1; }
    };
    // software pipeline: the loads of chunk ch+1 are in flight while chunk ch is stored
    Regs R0, R1;
    const long long tp0 = clock64();
    if (nchunks > 0) load(0, R0);
    for (int ch = 0; ch < nchunks; ch += 2) {
      if (ch + 1 < nchunks) load(ch + 1, R1);
      publish(R0);
      if (ch + 1 < nchunks) {
        if (ch + 2 < nchunks) load(ch + 2, R0);
        publish(R1);
      }
    }
    if (p.clk && tid == 0) p.clk[blockIdx.x * 8 + 1] = clock64() - tp0;
    if (p.dbpart) {
      dbs[tid] = db_acc;
      ptx::named_bar_sync(1, 256);
      if (tid < p.Kc && tid < p.K) p.dbpart[(int64_t)split * p.K + tid] = dbs[2 * tid] + dbs[2 * tid + 1];
    }
  } else {
    // ================= MMA warp
    const uint32_t idesc = ptx::make_idesc_tf32(128, p.NB);
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t sbase = ptx::smem_u32(stage_base);
    const uint32_t rg_step = (uint32_t)(p.copies * p.Wf / 4 * p.NB);  // quads x NB rows (16-B units)
    const long long tm0 = clock64();
    for (int ch = 0; ch < nchunks; ++ch) {
      const long long tw = clock64();
      ptx::mbar_wait(full + stage, phase);
      if (p.clk && lane == 0) p.clk[blockIdx.x * 8 + 2] += clock64() - tw;
      ptx::tc_fence_after();
      const uint32_t A = sbase + (uint32_t)stage * p.stage_bytes;
      uint64_t adesc = ptx::make_desc(A, 128 * 16, 128);
      uint64_t bdesc = ptx::make_desc(A + p.a_bytes, (uint32_t)p.NB * 16, 128);
      for (int kk = 0; kk < p.KC / 8; ++kk) {
        uint64_t bd = bdesc;
        uint32_t tm = 0;
        const uint32_t acc = (ch | kk) != 0 ? 1u : 0u;
        for (int rg = 0; rg < p.RG; ++rg) {
          if (ptx::elect_one()) ptx::mma_tf32(tm, adesc, bd, idesc, acc);
          __syncwarp();
          tm += (uint32_t)p.NB;
          bd += (uint64_t)rg_step;
        }
        adesc += 2 * 128;                 // 2 quads of 128 rows x 16 B
        bdesc += (uint64_t)(2 * p.NB);    // 2 quads of NB rows x 16 B
      }
      if (ptx::elect_one()) ptx::mma_commit(empty + stage);
      __syncwarp();
      if (++stage == p.nstage) { stage = 0; phase ^= 1; }
    }
    if (ptx::elect_one()) ptx::mma_commit(accf);
    __syncwarp();
    if (p.clk && lane == 0) p.clk[blockIdx.x * 8 + 3] = clock64() - tm0;
  }
  // ================= epilogue: warps 0-7 (quadrant warp % 4, column chunk parity warp / 4)
  if (warp < 8) {
    ptx::mbar_wait_sleep(accf, 0);
    __syncwarp();
    ptx::tc_fence_after();
    const int qd = warp & 3, half = warp >> 2;
    const int row = qd * 32 + lane;
    float *dst = p.part + (int64_t)split * p.RG * 128 * p.NB;
    const int nc16 = p.NB / 16;
    for (int rg = 0; rg < p.RG; ++rg)
      for (int c16 = half; c16 < nc16; c16 += 2) {
        float v[16];
        if (nchunks > 0) {
          ptx::tmem_ld16(tmem_base + ((uint32_t)(qd * 32) << 16) + (uint32_t)(rg * p.NB + c16 * 16), v);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = 0.f;
        }
        float4 *o = reinterpret_cast<float4 *>(dst + ((int64_t)rg * 128 + row) * p.NB + c16 * 16);
        o[0] = make_float4(v[0], v[1], v[2], v[3]);
        o[1] = make_float4(v[4], v[5], v[6], v[7]);
        o[2] = make_float4(v[8], v[9], v[10], v[11]);
        o[3] = make_float4(v[12], v[13], v[14], v[15]);
      }
    ptx::tc_fence_before();
  }
  __syncthreads();
  if (warp == 8) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, 512);
  }
}

__global__ void tc_wgrad_spf_reduce_kernel(const TcWgSpfParams p, float *__restrict__ df,
                                           float *__restrict__ db) {
  const int RS = p.R * p.S;
  const int64_t total = (int64_t)p.K * p.C * RS;
  const int64_t split_stride = (int64_t)p.RG * 128 * p.NB;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / ((int64_t)p.C * RS));
    const int rem = (int)(i - (int64_t)k * p.C * RS);
    const int c = rem / RS, t = rem - c * RS, r = t / p.S, s = t - r * p.S;
    const int rg = r / p.copies, j = r - rg * p.copies;
    const int64_t off = ((int64_t)rg * 128 + j * p.Kc + k) * p.NB + s * p.C + c;
    float acc = 0.f;
    for (int sp = 0; sp < p.splits; ++sp) acc += p.part[sp * split_stride + off];
    df[i] = acc;
  }
  if (db) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < p.K;
         k += (int64_t)gridDim.x * blockDim.x) {
      float acc = 0.f;
      for (int sp = 0; sp < p.splits; ++sp) acc += p.dbpart[(int64_t)sp * p.K + k];
      db[k] = acc;
    }
  }
}

struct TcWgSpfPlan {
  TcWgSpfParams p;
  size_t smem, part_bytes, dbpart_bytes;
  bool ok;
};

TcWgSpfPlan plan_wgrad_spf(const SpfConv &sc) {
  TcWgSpfPlan pl{};
  TcWgSpfParams &p = pl.p;
  pl.ok = false;
  p.K = sc.K; p.C = sc.C; p.R = sc.R; p.S = sc.S; p.Wf = sc.Wf;
  p.G = sc.G;
  p.plane_x = sc.plane_x; p.plane_dy = sc.plane_dy;
  p.x_shift = sc.x_shift; p.dy_shift = sc.dy_shift;
  if (sc.Wf % 4 || sc.plane_x % 4 || sc.plane_dy % 4 || sc.G % 4 || sc.x_shift % 4 || sc.dy_shift % 4) return pl;
  if (!(sc.S == 5 || sc.S == 3) || sc.K > 128) return pl;
  p.Kc = sc.K <= 16 ? 16 : sc.K <= 32 ? 32 : sc.K <= 64 ? 64 : 128;
  p.copies = 128 / p.Kc;
  if (p.copies > sc.R) p.copies = std::max(1, sc.R);
  while (128 % (p.Kc * p.copies) != 0) --p.copies;
  p.RG = (sc.R + p.copies - 1) / p.copies;
  p.NB = sc.S * sc.C;
  if (p.NB % 16 || p.NB > 256 || p.RG * p.NB > 512) return pl;
  p.Gext = p.G + (int64_t)(p.copies - 1) * p.Wf;
  p.KC = 32;
  p.HBq = p.KC / 4 + (p.RG - 1) * p.copies * p.Wf / 4;
  p.a_bytes = (uint32_t)(p.KC / 4 * 128 * 16);
  p.b_bytes = (uint32_t)(p.HBq * p.NB * 16);
  p.stage_bytes = p.a_bytes + p.b_bytes;
  if ((int64_t)sc.C * ((p.HBq + 3) / 4) > 512) return pl;  // producer B tasks: <= 2 per thread
  const size_t fixed = 256 * 4 + 8 * 12 + 16;
  p.nstage = (int)std::min<int64_t>(4, (SMEM_BUDGET - (int64_t)fixed) / p.stage_bytes);
  if (p.nstage < 2) return pl;
  pl.smem = (size_t)p.nstage * p.stage_bytes + fixed;
  const int64_t target = 2ll * sm_count();
  int64_t splits = std::min<int64_t>(target, std::max<int64_t>(1, ceil_div(p.Gext, 8 * p.KC)));
  p.pos_per_split = align_up((size_t)ceil_div(p.Gext, splits), (size_t)p.KC);
  p.splits = (int)ceil_div(p.Gext, p.pos_per_split);
  pl.part_bytes = align_up((size_t)p.splits * p.RG * 128 * p.NB * sizeof(float), 256);
  pl.dbpart_bytes = align_up((size_t)p.splits * p.K * sizeof(float), 256);
  pl.ok = true;
  return pl;
}

}  // namespace

// ------------------------------------------------------------------ forward (K3)
bool tc_fwd_ks(const ConvArgs &a) { return a.C == 1 && a.S <= 8; }

bool tc_fwd_supported(const ConvArgs &a, const PoolArgs *pool) {
  if (device_cc_major() != 10) return false;
  if (((a.sh != 1 || a.sw != 1) && (a.R != 1 || a.S != 1 || pool)) || !pool_fusable(pool)) return false;
  return plan_fwd(a.N, a.C, a.H, a.W, a.K, a.R, a.S, a.ph, a.pw, pool, true, a.sh, a.sw).ok;
}

size_t tc_fwd_ws(const ConvArgs &a) {
  // the packed filter bank only depends on (K, C, R, S)
  const int nfpad = a.K <= 256 ? std::max(16, round_up(a.K, 16)) : 256;
  const int nft = a.K <= 256 ? 1 : (a.K + 255) / 256;
  if (a.C == 1 && a.S <= 8)  // KS packing: [ftile][r][2 halves][NFpad][4]
    return align_up((size_t)nft * a.R * 8 * nfpad * sizeof(float), 256) + sk_ws_bytes();
  return align_up((size_t)nft * ((a.C + 7) / 8) * a.R * a.S * 8 * nfpad * sizeof(float), 256) + sk_ws_bytes();
}

sysml_status tc_conv_fwd(const ConvArgs &a, const float *x, const float *f, const float *bias,
                         float *y, const PoolArgs *pool, float *pout, int32_t *parg, void *ws,
                         cudaStream_t st, const sysml_csr *csr) {
  TcPlan pl = plan_fwd(a.N, a.C, a.H, a.W, a.K, a.R, a.S, a.ph, a.pw, pool, true, a.sh, a.sw);
  if (!pl.ok) {
    set_error("tcgen05 forward: unsupported shape");
    return SYSML_ERR_UNSUPPORTED;
  }
  return run_fwd(pl, x, f, 0, a.C, bias, pool ? nullptr : y, pout, parg, ws, st, nullptr, csr);
}

// ------------------------------------------------------------------ bwd_data (K6)
static bool strided_1x1(const ConvArgs &a) {
  return (a.sh != 1 || a.sw != 1) && a.R == 1 && a.S == 1 && a.ph == 0 && a.pw == 0;
}

static TcPlan plan_bwd_data(const ConvArgs &a, int spf_in = 0, int route = 0) {
  if (strided_1x1(a)) {
    // strided 1x1: dX[n, c, p*sh, q*sw] = sum_k F[k, c] dY[n, k, p, q], zero elsewhere -- a
    // stride-1 1x1 "forward" on dY's grid whose rows land on every sh-th row / sw-th column
    TcPlan pl = plan_fwd(a.N, a.K, a.P, a.Q, a.C, 1, 1, 0, 0, nullptr, /*allow_ks=*/false);
    pl.p.yH = a.H;
    pl.p.yW = a.W;
    pl.p.ysh = a.sh;
    pl.p.ysw = a.sw;
    return pl;
  }
  // dX = conv(dY, rot180(F)^T), pad R-1-ph; input (N, K, P, Q) -> output (N, C, H, W)
  return plan_fwd(a.N, a.K, a.P, a.Q, a.C, a.R, a.S, a.R - 1 - a.ph, a.S - 1 - a.pw, nullptr,
                  /*allow_ks=*/false, 1, 1, spf_in, route);
}

bool tc_bwd_data_supported(const ConvArgs &a) {
  if (device_cc_major() != 10) return false;
  if (strided_1x1(a)) return plan_bwd_data(a).ok && !plan_bwd_data(a).p.sn;
  if (a.sh != 1 || a.sw != 1 || a.ph > a.R - 1 || a.pw > a.S - 1) return false;
  TcPlan pl = plan_bwd_data(a);
  return pl.ok && pl.p.P == a.H && pl.p.Q == a.W;
}

size_t tc_bwd_data_ws(const ConvArgs &a) {
  TcPlan pl = plan_bwd_data(a);
  return pl.ok ? align_up(pl.fp_bytes, 256) + sk_ws_bytes() : 0;
}

sysml_status tc_conv_bwd_data(const ConvArgs &a, const float *f, const float *dy, float *dx,
                              void *ws, cudaStream_t st) {
  TcPlan pl = plan_bwd_data(a);
  if (!pl.ok) {
    set_error("tcgen05 bwd_data: unsupported shape");
    return SYSML_ERR_UNSUPPORTED;
  }
  if (strided_1x1(a))  // positions off the stride grid receive no contribution
    SYSML_CUDA(cudaMemsetAsync(dx, 0, sizeof(float) * (size_t)a.N * a.C * a.H * a.W, st));
  // filter bank F is (K x C*RS) = (Cin_of_this_conv x Kout*RS) -> flip = 1
  return run_fwd(pl, dy, f, 1, a.K, nullptr, dx, nullptr, nullptr, ws, st);
}

// ------------------------------------------------------------------ phase-split entry points
// (phase.cu): `b` is the stride-1 pad-0 phase problem of the strided conv `a`; X' is gathered
// from X by the producer (fwd) and dX' scattered to dX by the epilogue (bwd_data), so neither
// phase tensor exists in HBM.
static void set_phase(TcFwdParams &p, const ConvArgs &a) {
  p.phs = a.sh; p.phw = a.sw; p.phC = a.C; p.phH = a.H; p.phW = a.W; p.php = a.ph; p.phpw = a.pw;
}

bool tc_fwd_phase_fused_ok(const ConvArgs &a, const ConvArgs &b) {
  if (a.C % 8 || (int64_t)a.N * a.C * a.H * a.W >= (1ll << 31)) return false;
  const TcPlan pl = plan_fwd(b.N, b.C, b.H, b.W, b.K, b.R, b.S, 0, 0, nullptr, true);
  return pl.ok && !pl.p.ks && !pl.p.abulk;
}

sysml_status tc_conv_fwd_phase(const ConvArgs &a, const ConvArgs &b, const float *x, const float *fp,
                               const float *bias, float *y, void *ws, cudaStream_t st) {
  TcPlan pl = plan_fwd(b.N, b.C, b.H, b.W, b.K, b.R, b.S, 0, 0, nullptr, true);
  if (!pl.ok || pl.p.ks || pl.p.abulk) {
    set_error("tcgen05 phase forward: unsupported shape");
    return SYSML_ERR_UNSUPPORTED;
  }
  set_phase(pl.p, a);
  pl.p.in_phase = 1;
  return run_fwd(pl, x, fp, 0, b.C, bias, y, nullptr, nullptr, ws, st);
}

bool tc_bwd_data_phase_fused_ok(const ConvArgs &a, const ConvArgs &b) {
  if (a.C % 16 || (int64_t)a.N * a.C * a.H * a.W >= (1ll << 31) || !tc_bwd_data_supported(b)) return false;
  const TcPlan pl = plan_bwd_data(b);
  return pl.ok && !pl.p.sn && !pl.p.tile2d && !pl.p.pool;
}

sysml_status tc_conv_bwd_data_phase(const ConvArgs &a, const ConvArgs &b, const float *fp, const float *dy,
                                    float *dx, void *ws, cudaStream_t st) {
  TcPlan pl = plan_bwd_data(b);
  if (!pl.ok || pl.p.sn || pl.p.tile2d) {
    set_error("tcgen05 phase bwd_data: unsupported shape");
    return SYSML_ERR_UNSUPPORTED;
  }
  // positions no phase cell reaches (floor extent) receive no contribution
  if ((int64_t)b.H * a.sh - a.ph < a.H || (int64_t)b.W * a.sw - a.pw < a.W)
    SYSML_CUDA(cudaMemsetAsync(dx, 0, sizeof(float) * (size_t)a.N * a.C * a.H * a.W, st));
  set_phase(pl.p, a);
  pl.p.out_phase = 1;
  return run_fwd(pl, dy, fp, 1, b.K, nullptr, dx, nullptr, nullptr, ws, st);
}

// ------------------------------------------------------------------ SPF-layout entry points
sysml_status tc_conv_fwd_spf(const ConvArgs &a, const TcSpfIO &io, const float *x, const float *f,
                             const float *bias, float *y, const PoolArgs *pool, float *pout,
                             int32_t *parg, void *ws, cudaStream_t st, const sysml_csr *csr) {
  TcPlan pl = plan_fwd(a.N, a.C, a.H, a.W, a.K, a.R, a.S, a.ph, a.pw, pool, true, 1, 1, 1);
  if (!pl.ok) pl = plan_fwd(a.N, a.C, a.H, a.W, a.K, a.R, a.S, a.ph, a.pw, pool);
  if (!pl.ok || a.sh != 1 || a.sw != 1) {
    set_error("tcgen05 SPF forward: unsupported shape");
    return SYSML_ERR_UNSUPPORTED;
  }
  return run_fwd(pl, x, f, 0, a.C, bias, pool ? nullptr : y, pout, parg, ws, st, &io, csr);
}

bool tc_conv_bwd_data_spf_nhwc_ok(const ConvArgs &a) {
  if (!tc_bwd_data_supported(a)) return false;
  const TcPlan pl = plan_bwd_data(a);
  return pl.ok && pl.p.sn && (pl.p.K & 3) == 0;
}

sysml_status tc_conv_bwd_data_spf(const ConvArgs &a, const TcSpfIO &io, const float *f,
                                  const float *dy, float *dx, void *ws, cudaStream_t st) {
  if (!tc_bwd_data_supported(a)) {
    set_error("tcgen05 SPF bwd_data: unsupported shape");
    return SYSML_ERR_UNSUPPORTED;
  }
  const int route = io.route_val ? 1 : 0;
  TcPlan pl = plan_bwd_data(a, route ? 0 : 1, route);
  if (!route && (!pl.ok || pl.fp_bytes > plan_bwd_data(a).fp_bytes)) pl = plan_bwd_data(a);  // ws sized by the plain plan
  if (!pl.ok || pl.fp_bytes > plan_bwd_data(a).fp_bytes) {
    set_error("tcgen05 SPF bwd_data: no plan for this shape%s", route ? " with routed input" : "");
    return SYSML_ERR_UNSUPPORTED;
  }
  return run_fwd(pl, dy, f, 1, a.K, nullptr, dx, nullptr, nullptr, ws, st, &io);
}

// ------------------------------------------------------------------ bwd_filter on SPF
bool tc_wgrad_spf_supported(const SpfConv &sc) {
  return device_cc_major() == 10 && plan_wgrad_spf(sc).ok;
}

size_t tc_wgrad_spf_ws(const SpfConv &sc) {
  TcWgSpfPlan pl = plan_wgrad_spf(sc);
  return pl.ok ? pl.part_bytes + pl.dbpart_bytes : 0;
}

sysml_status tc_wgrad_spf(const SpfConv &sc, const float *x_spf, const float *dy_spf, float *df,
                          float *db, void *ws, cudaStream_t st) {
  TcWgSpfPlan pl = plan_wgrad_spf(sc);
  if (!pl.ok) {
    set_error("tcgen05 SPF bwd_filter: unsupported shape");
    return SYSML_ERR_UNSUPPORTED;
  }
  TcWgSpfParams p = pl.p;
  p.x = x_spf;
  p.dy = dy_spf;
  p.part = reinterpret_cast<float *>(ws);
  p.dbpart = db ? reinterpret_cast<float *>(reinterpret_cast<char *>(ws) + pl.part_bytes) : nullptr;
  static long long *dclk = nullptr;
  const bool prof = getenv("SYSML_TC_PROFILE") != nullptr;
  p.clk = nullptr;
  if (prof) {
    if (!dclk) cudaMalloc(&dclk, sizeof(long long) * 8 * 4096);
    cudaMemsetAsync(dclk, 0, sizeof(long long) * 8 * 4096, st);
    p.clk = dclk;
  }
  if (p.S == 5) {
      SYSML_TRY(smem_attr(tc_wgrad_spf_kernel<5>, pl.smem));
    route_note("tc_wgrad_spf_kernel<5> [tcgen05 TF32, %d splits]", p.splits);
    tc_wgrad_spf_kernel<5><<<p.splits, WG_THREADS, pl.smem, st>>>(p);
  } else {
      SYSML_TRY(smem_attr(tc_wgrad_spf_kernel<3>, pl.smem));
    route_note("tc_wgrad_spf_kernel<3> [tcgen05 TF32, %d splits]", p.splits);
    tc_wgrad_spf_kernel<3><<<p.splits, WG_THREADS, pl.smem, st>>>(p);
  }
  SYSML_LAUNCH_CHECK();
  if (prof) {
    static long long h[8 * 4096];
    cudaMemcpyAsync(h, dclk, sizeof(long long) * 8 * p.splits, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double a[8] = {0};
    for (int b = 0; b < p.splits; ++b)
      for (int j = 0; j < 8; ++j) a[j] += (double)h[b * 8 + j] / p.splits;
    fprintf(stderr, "[tc_wgrad_spf splits=%d nstage=%d KC=%d] prod_wait_empty %.0f prod_total %.0f "
            "mma_wait_full %.0f mma_total %.0f\n", p.splits, p.nstage, p.KC, a[0], a[1], a[2], a[3]);
  }
  const int64_t total = (int64_t)p.K * p.C * p.R * p.S;
  const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 8 * sm_count());
  tc_wgrad_spf_reduce_kernel<<<blocks, 256, 0, st>>>(p, df, db);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

// ------------------------------------------------------------------ bwd_filter (K5)
// strided 1x1 bwd_filter: dF[k][c] = sum_{n,p,q} dY[n,k,p,q] X[n,c,p*sh,q*sw] is the stride-1
// 1x1 bwd_filter of the subsampled X (N x C x P x Q, gathered into the workspace first)
static ConvArgs subsampled_1x1(const ConvArgs &a) {
  ConvArgs b = a;
  b.H = a.P;
  b.W = a.Q;
  b.sh = b.sw = 1;
  return b;
}

__global__ void subsample_kernel(const float *__restrict__ x, float *__restrict__ xs, int64_t NC, int H, int W,
                                 int P, int Q, int sh, int sw) {
  const int64_t total = NC * P * Q;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t nc = i / (P * Q);
    const int pq = (int)(i - nc * P * Q), pp = pq / Q, qq = pq - pp * Q;
    xs[i] = __ldg(x + nc * H * W + (int64_t)pp * sh * W + (int64_t)qq * sw);
  }
}

// the dedicated TMA kernels (1x1 GEMM, strided 1x1 via subsampling, framed shifted rows)
bool tc_bwd_filter_fast_supported(const ConvArgs &a) {
  if (device_cc_major() != 10) return false;
  if (strided_1x1(a)) return tc_wgrad_1x1_supported(subsampled_1x1(a));
  return tc_wgrad_1x1_supported(a) || tc_wgrad_frame_supported(a);
}

bool tc_bwd_filter_supported(const ConvArgs &a) {
  if (device_cc_major() != 10) return false;
  if (strided_1x1(a)) return tc_wgrad_1x1_supported(subsampled_1x1(a));
  if (tc_wgrad_1x1_supported(a)) return true;
  if (tc_wgrad_frame_supported(a)) return true;
  if (a.C < 8) return false;  // tiny channel counts waste N; CUDA-core / CSR kernels instead
  return plan_wgrad(a).ok;
}

size_t tc_bwd_filter_ws(const ConvArgs &a) {
  if (strided_1x1(a))
    return align_up((size_t)a.N * a.C * a.P * a.Q * sizeof(float), 256) + tc_wgrad_1x1_ws(subsampled_1x1(a));
  if (tc_wgrad_1x1_supported(a)) return tc_wgrad_1x1_ws(a);
  if (tc_wgrad_frame_supported(a)) return tc_wgrad_frame_ws(a);
  TcWgPlan pl = plan_wgrad(a);
  return pl.ok ? pl.part_bytes + pl.dbpart_bytes : 0;
}

sysml_status tc_conv_bwd_filter(const ConvArgs &a, const float *x, const float *dy, float *df,
                                float *db, void *ws, cudaStream_t st) {
  if (strided_1x1(a)) {
    const ConvArgs b = subsampled_1x1(a);
    if (!tc_wgrad_1x1_supported(b)) {
      set_error("tcgen05 bwd_filter: unsupported strided 1x1 shape");
      return SYSML_ERR_UNSUPPORTED;
    }
    float *xs = reinterpret_cast<float *>(ws);
    const int64_t total = (int64_t)a.N * a.C * a.P * a.Q;
    route_note("subsample_kernel");
    subsample_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 16 * sm_count()), 256, 0, st>>>(
        x, xs, (int64_t)a.N * a.C, a.H, a.W, a.P, a.Q, a.sh, a.sw);
    SYSML_LAUNCH_CHECK();
    return tc_wgrad_1x1(b, xs, dy, df, db,
                        reinterpret_cast<char *>(ws) + align_up((size_t)total * sizeof(float), 256), st);
  }
  if (tc_wgrad_1x1_supported(a)) return tc_wgrad_1x1(a, x, dy, df, db, ws, st);
  if (tc_wgrad_frame_supported(a)) return tc_wgrad_frame(a, x, dy, df, db, ws, st);
  TcWgPlan pl = plan_wgrad(a);
  if (!pl.ok) {
    set_error("tcgen05 bwd_filter: unsupported shape");
    return SYSML_ERR_UNSUPPORTED;
  }
  TcWgParams p = pl.p;
  p.x = x;
  p.dy = dy;
  p.part = reinterpret_cast<float *>(ws);
  p.dbpart = db ? reinterpret_cast<float *>(reinterpret_cast<char *>(ws) + pl.part_bytes) : nullptr;
  SYSML_TRY(smem_attr(tc_conv_wgrad_kernel, pl.smem));
  route_note("tc_conv_wgrad_kernel [tcgen05 TF32, %d CTAs]", p.splits * p.nwt);
  tc_conv_wgrad_kernel<<<p.splits * p.nwt, TC_THREADS, pl.smem, st>>>(p);
  SYSML_LAUNCH_CHECK();
  const int64_t total = (int64_t)a.K * a.C * a.R * a.S;
  const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 8 * sm_count());
  tc_wgrad_reduce_kernel<<<blocks, 256, 0, st>>>(p, df, db);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

}  // namespace sysml
