// wgrad_spf_tma.cu -- K5 conv2d_backward_filter on stacked-planar-frame (SPF) tensors
// (the LeNet step's conv2 bwd_filter, §8(c) def. 4), fed by TMA.
//
//   dF[k][c][r][s] = sum_g dY[k][g] * X[c][g + r*Wf + s]        (g: frame position)
//
// GEMM over frame positions g (contiguous in SPF planes -> K-major tcgen05 operands
// straight from HBM with 128-byte-swizzled TMA boxes of 32 positions = one "atom"):
//   A rows (j, k): dY[k][g - j*Wf]          j < copies (= 128 / Kc): TMA box at g - j*Wf
//   B rows (s, c): X[c][g + s]              s < S: one TMA box per s
//   D_rb[(j,k)][(s,c)] = sum_g A . B(g + rb*copies*Wf)  ->  r = rb*copies + j
// The rb shift (copies*Wf positions) is a whole number of atoms, so it is a descriptor
// offset into a ring of B atoms: each X atom is loaded once and used by RG MMAs of
// consecutive A atoms (no halo re-fetch).  All RG accumulators (RG * S*C columns) live
// in TMEM; split-K over positions, partials reduced in a fixed order.
//
// Warp roles (W2_THREADS = 352): warp 0 = dY (A) TMA producer, warp 6 = X (B) TMA producer
// of the s % 4 == 0 column taps, warp 1 = MMA issuer, warps 2-5 and 7-10 = helpers that build
// the other column shifts of each X atom in shared memory; warps 2-5 also sum db from the
// staged dY atoms during the loop and run the epilogue (TMEM quadrant warp % 4).
#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"
#include "tma.cuh"

#include <algorithm>

namespace sysml {

namespace {

constexpr int W2_MAXS = 8;  // column taps (plan: S <= 8)
constexpr int W2_NA = 6;          // A ring (dY atoms)
constexpr int W2_THREADS = 352;  // warps 0 A producer, 1 MMA, 2-5 + 7-10 helpers, 6 B producer
constexpr int W2_HELP_WARPS = 8;
constexpr int W2_ATOM = 32;       // positions per atom (128-byte swizzled row)
constexpr int W2_MAXL = 7;        // B lookahead (atoms): descriptors of atoms ai .. ai + 7

struct W2Params {
  int K, C, R, S, Wf;
  int Kc, copies, RG, N;          // A rows per copy; N = S*Ct
  int Ct, nct, nkt;               // channels per CTA tile, channel tiles, filter tiles
  int shift;                      // positions per rb shift (copies*Wf, multiple of 8)
  int L;                          // B lookahead in atoms
  int nbr;                        // B ring slots
  int64_t atoms;                  // ceil(G / 32)
  int splits;
  float *part;                    // [split][RG][128][N]
  float *dbpart;                  // [split][K] or null
  int dbg;                        // debug: 1 = skip the MMAs
  const float *x;                 // X plane base (+ x_shift) for the shifted B rows
  int64_t G, plane_x;
  int ntma_s;                     // column taps s with s % 4 == 0 (TMA-loaded)
  int hcopy;                      // 1: A copies j >= 1 built by the helpers ((copies - 1) * Wf <= 32)
  int hb4;                        // 1: B tap s = 4 built by the helpers (else TMA-loaded)
  long long *clk;                 // optional per-CTA cycle counters (SYSML_TC_PROFILE)
};

__device__ __forceinline__ void st_shared_v4_w2(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

__device__ __forceinline__ float4 ld_shared_v4_w2(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint64_t sw128(uint32_t saddr) {
  return ptx::make_desc(saddr, 16, 1024) | ((uint64_t)2 << 61);
}

template <int SHIFT>  // positions per rb shift (compile-time: 16 or 32), 0 = runtime p.shift
__global__ void __launch_bounds__(W2_THREADS, 1)
    tc_wgrad_spf_tma_kernel(const __grid_constant__ CUtensorMap tmDy,
                            const __grid_constant__ CUtensorMap tmX, const W2Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const uint32_t a_slot = 128 * 128;                  // 16 KB
  const uint32_t b_slot = (uint32_t)p.N * 128;        // N rows x 128 B
  uint8_t *Aring = smem, *Bring = smem + W2_NA * a_slot;
  uint64_t *fullA = reinterpret_cast<uint64_t *>(Bring + p.nbr * b_slot);  // A atom complete (helpers)
  uint64_t *emptyA = fullA + W2_NA;
  uint64_t *fullAt = emptyA + W2_NA;   // TMA part of an A atom landed
  uint64_t *fullB = fullAt + W2_NA;    // B atom complete (helper warps)
  uint64_t *emptyB = fullB + p.nbr;
  uint64_t *fullBt = emptyB + p.nbr;   // TMA part of a B atom landed
  uint64_t *accf = fullBt + p.nbr;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(accf + 1);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int z = blockIdx.x % p.splits;
  const int ct = (blockIdx.x / p.splits) % p.nct, kt = blockIdx.x / (p.splits * p.nct);
  const int k0 = kt * p.Kc, c0 = ct * p.Ct;
  const int64_t a0 = z * p.atoms / p.splits, a1 = (z + 1) * p.atoms / p.splits;
  const int L = p.L;  // B lookahead (atoms)
  const bool do_db = p.dbpart != nullptr && !(p.dbg & 4) && ct == 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < W2_NA; ++i) {
      // A copies j >= 1 (dY shifted by j frame rows) are built by the helper warps from the
      // TMA-loaded copy 0 of this atom and the previous one (fewer TMA row requests: the TMA
      // engine handles ~1 128-byte row per 9-10 clocks here, which paced the whole kernel)
      ptx::mbar_init(fullA + i, W2_HELP_WARPS);
      ptx::mbar_init(fullAt + i, 1);
      ptx::mbar_init(emptyA + i, 1 + (p.copies > 1 && p.hcopy ? W2_HELP_WARPS : 0) + (do_db ? 1 : 0));
    }
    for (int i = 0; i < p.nbr; ++i) {
      ptx::mbar_init(fullB + i, W2_HELP_WARPS);  // the helper warps (after they saw the TMA part)
      ptx::mbar_init(fullBt + i, 1);  // expect_tx
      ptx::mbar_init(emptyB + i, 1);
    }
    ptx::mbar_init(accf, 1);
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tmDy);
    ptx::tma_prefetch_desc(&tmX);
  }
  if (warp == 1) ptx::tmem_alloc(tslot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t sA = ptx::smem_u32(Aring), sB = ptx::smem_u32(Bring);
  const int64_t nA = a1 - a0, nB = a1 > a0 ? nA + L : 0;

  const long long tk0 = clock64();
  if (warp == 0) {
    if (lane == 0) {
      // B atom bi (= a0 + bi) goes to slot bi % nbr; A atom ai to slot ai % NA.  (No
      // lambdas here: the tensor-map parameters must be addressed in param space.)
      // A producer (dY atoms); the B producer is warp 6 so neither blocks the other.
      // Ring cursors advance incrementally (no divisions in the issue loops).
      int sa = 0;
      uint32_t pa = 0;
      for (int ia = 0; ia < (int)nA; ++ia) {
        const long long t0 = p.clk ? clock64() : 0;
        ptx::mbar_wait(emptyA + sa, pa ^ 1);
        if (p.clk) p.clk[blockIdx.x * 8 + 4] += clock64() - t0;
        // the bytes the copies below deliver: copies x Kc rows (< 128 rows when copies*Kc < 128;
        // the slot's other rows only feed accumulator rows the reduce skips)
        // copy 0 only, except for the CTA's first atom (no previous atom to build the rest from)
        const int ncp = (ia == 0 || !p.hcopy) ? p.copies : 1;
        ptx::mbar_arrive_expect_tx(fullAt + sa, (uint32_t)(ncp * p.Kc * 128));
        const int g = (int)((a0 + ia) * W2_ATOM);
        for (int j = 0; j < ncp; ++j)
          ptx::tma_load_3d(sA + sa * a_slot + j * p.Kc * 128, &tmDy, g - j * p.Wf, k0, 0,
                           ptx::smem_u32(fullAt + sa));
        if (++sa == W2_NA) { sa = 0; pa ^= 1; }
      }
    }
  } else if (warp == 6) {
    if (lane == 0) {
      // B producer: the s % 4 == 0 column taps of X atoms 0 .. nB (atom nB feeds the
      // tail of the last shifted rows) as fast as ring slots free up.  TMA needs
      // 16-byte aligned inner coordinates, so the helper warps build the other shifts.
      const int nBt = nA > 0 ? (int)nB + 1 : 0;
      int sb = 0;
      uint32_t pb = 0;
      for (int ib = 0; ib < nBt; ++ib) {
        const long long t0 = p.clk ? clock64() : 0;
        ptx::mbar_wait(emptyB + sb, pb ^ 1);
        if (p.clk) p.clk[blockIdx.x * 8 + 5] += clock64() - t0;
        // the s = 0 rows (and s = 4 unless the helpers build it): helpers build the others
        const bool t4 = !p.hb4 && p.S > 4;
        ptx::mbar_arrive_expect_tx(fullBt + sb, (uint32_t)((t4 ? 2 : 1) * p.Ct * 128));
        const int g = (int)((a0 + ib) * W2_ATOM);
        ptx::tma_load_3d(sB + sb * b_slot, &tmX, g, c0, 0, ptx::smem_u32(fullBt + sb));
        if (t4) ptx::tma_load_3d(sB + sb * b_slot + 4 * p.Ct * 128, &tmX, g + 4, c0, 0, ptx::smem_u32(fullBt + sb));
        if (++sb == p.nbr) { sb = 0; pb ^= 1; }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = ptx::make_idesc_tf32(128, p.N);
    int sbw = 0;  // B ring cursor of the waits (atoms 0, 1, ... in order)
    uint32_t pbw = 0;
    for (int bi = 0; bi < (int)std::min<int64_t>(L, nB); ++bi) {
      ptx::mbar_wait(fullB + sbw, pbw);
      if (++sbw == p.nbr) { sbw = 0; pbw ^= 1; }
    }
    int sa = 0, s_ai = 0;  // A cursor; B slot of atom ai
    uint32_t pa = 0;
    // per (kk, rb): the B atom offset and the 32-byte step inside the swizzled row of
    // positions 8*kk + rb*shift (constant across atoms)
    const int shift = SHIFT ? SHIFT : p.shift;
    for (int ai = 0; ai < (int)nA; ++ai) {
      const long long t0 = p.clk ? clock64() : 0;
      ptx::mbar_wait(fullA + sa, pa);
      const long long t1 = p.clk ? clock64() : 0;
      ptx::mbar_wait(fullB + sbw, pbw);  // newest B atom this group needs (ai + L)
      if (++sbw == p.nbr) { sbw = 0; pbw ^= 1; }
      if (p.clk && lane == 0) {
        p.clk[blockIdx.x * 8 + 0] += t1 - t0;
        p.clk[blockIdx.x * 8 + 1] += clock64() - t1;
      }
      ptx::tc_fence_after();
      // descriptors built once per atom; K-steps / sub-atom shifts are start-address
      // increments (16-byte units) -- keeps the issue loop to a few uniform adds per MMA
      const uint64_t adesc = sw128(sA + sa * a_slot);
      uint64_t bdesc[W2_MAXL + 1];
#pragma unroll
      for (int a = 0; a <= W2_MAXL; ++a) {
        int sl = s_ai + a;
        if (sl >= p.nbr) sl -= p.nbr;
        if (sl >= p.nbr) sl -= p.nbr;  // a > L (unused) with a small ring
        bdesc[a] = sw128(sB + (uint32_t)sl * b_slot);
      }
      // one elected lane issues the atom's MMAs and commits as one block (a per-MMA elect /
      // __syncwarp round trip costs more than an N = 160 MMA: tools/mma_snstream.cu)
      if (ptx::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < W2_ATOM / 8; ++kk) {
          const uint32_t acc = (ai | kk) != 0 ? 1u : 0u;
#pragma unroll
          for (int rb = 0; rb < 4; ++rb) {
            if (rb < p.RG) {
              const int t = 8 * kk + rb * shift;  // compile-time when SHIFT != 0
              const uint64_t bd = bdesc[(t >> 5) & W2_MAXL] + (uint64_t)((t & 31) >> 2);
              if (!p.dbg) ptx::mma_tf32(tmem + rb * p.N, adesc + (uint64_t)(kk * 2), bd, idesc, acc);
            }
          }
        }
        ptx::mma_commit(emptyA + sa);
        ptx::mma_commit(emptyB + s_ai);  // B atom ai has no later user
      }
      __syncwarp();
      if (++sa == W2_NA) { sa = 0; pa ^= 1; }
      if (++s_ai == p.nbr) s_ai = 0;
    }
    if (ptx::elect_one()) ptx::mma_commit(accf);
    __syncwarp();
  } else {
    // helpers: warps 2-5 (et 0..127: also db and the epilogue) and 7-10 (et 128..255)
    const bool main_helper = warp <= 5;
    const int et = main_helper ? (int)threadIdx.x - 64 : 128 + (int)threadIdx.x - 224;
    const int qd = warp & 3;
    // Merged loop in the producer's order: (1) the B rows of column taps s % 4 != 0 of
    // atom bi -- X[c][g + s] from two aligned float4 loads, shifted in registers, stored
    // into the 128-byte-swizzled row (16-byte chunk q ^ (row % 8)); (2) db[k] over this
    // CTA's dY atoms (rows k of copy j = 0), two threads per row.
    float dbv = 0.f;
    const int npre = (int)std::min<int64_t>(L, nB);
    // db rows: Kc <= 64 -> two threads per row (64-byte halves); Kc = 128 -> one per row
    const bool dsplit = p.Kc <= 64;
    const int drow = dsplit ? et >> 1 : et, dhalf = dsplit ? et & 1 : 0, dq = dsplit ? 4 : 8;
    // shift tasks (channel c, 16-byte chunk q) of this thread: t = et + 128u (Ct*8 <= 384).
    // Source: the TMA-loaded s = 0 tile of atom bi (chunk q) and, for q = 7, chunk 0 of
    // atom bi + 1 (next ring slot); both rows are 128-byte swizzled (chunk q at q ^ (c & 7)).
    const int ntask = p.S > 1 ? p.Ct * 8 : 0;  // S = 1: no shifted taps to build
    int sb = 0, sa = 0;
    uint32_t pb = 0, pa = 0;
    for (int step = -npre; step < (int)nA; ++step) {
      const int bi = step + npre;
      if (bi < nB) {
        const int slot = sb, slot1 = sb + 1 == p.nbr ? 0 : sb + 1;
        const uint32_t ph1 = sb + 1 == p.nbr ? pb ^ 1 : pb;
        const long long t0 = p.clk ? clock64() : 0;
        ptx::mbar_wait(fullBt + slot, pb);
        ptx::mbar_wait(fullBt + slot1, ph1);
        if (p.clk && et == 0) p.clk[blockIdx.x * 8 + 2] += clock64() - t0;
        if (++sb == p.nbr) { sb = 0; pb ^= 1; }
        const uint32_t Bs = sB + slot * b_slot, B1s = sB + slot1 * b_slot;
        // all 16-byte loads of this thread's (up to) two tasks first, then the shifts; explicit
        // ld.shared.v4 (a generic pointer here compiled to split generic loads: 2.7x the
        // shared-memory wavefronts)
        float4 v0[2], v1[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int t = et + u * 256;
          if (t < ntask) {
            const int c = t >> 3, q = t & 7;
            v0[u] = ld_shared_v4_w2(Bs + (uint32_t)(c * 128 + ((q ^ (c & 7)) << 4)));
            v1[u] = ld_shared_v4_w2(q < 7 ? Bs + (uint32_t)(c * 128 + (((q + 1) ^ (c & 7)) << 4))
                                          : B1s + (uint32_t)(c * 128 + ((c & 7) << 4)));
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int t = et + u * 256;
          if (t >= ntask) continue;
          const int c = t >> 3, q = t & 7;
          const float e[8] = {v0[u].x, v0[u].y, v0[u].z, v0[u].w, v1[u].x, v1[u].y, v1[u].z, v1[u].w};
          // taps s = 1 .. S-1 (S <= 5): positions 4q + s .. 4q + s + 3 of the s = 0 row
#pragma unroll
          for (int s_ = 1; s_ < 5; ++s_) {
            if (s_ >= p.S || (s_ == 4 && !p.hb4)) break;
            const int row = s_ * p.Ct + c;
            const uint32_t dst = Bs + row * 128 + ((q ^ (row & 7)) << 4);
            st_shared_v4_w2(dst, e[s_], e[s_ + 1], e[s_ + 2], e[s_ + 3]);
          }
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(fullB + slot);
      }
      if (step >= 0) {
        // A atom `step`: wait its TMA rows; build copies j >= 1 (rows j*Kc + k) from copy 0 of
        // this atom and the previous one: copy j = positions g - 16j .. g - 16j + 31 = the last
        // j * Wf / 4 16-byte chunks of the previous atom's row, then the first ones of this row
        const int slotA = sa, slotP = sa == 0 ? W2_NA - 1 : sa - 1;
        const long long t0 = p.clk ? clock64() : 0;
        ptx::mbar_wait(fullAt + slotA, pa);
        if (p.clk && et == 0) p.clk[blockIdx.x * 8 + 3] += clock64() - t0;
        if (step > 0 && p.copies > 1 && p.hcopy) {
          const uint32_t As = sA + slotA * a_slot, Ps = sA + slotP * a_slot;
          const int nrow = (p.copies - 1) * p.Kc;
          for (int t = et; t < nrow * 8; t += 256) {
            const int rr = t >> 3, q = t & 7;
            const int j = 1 + rr / p.Kc, k = rr - (j - 1) * p.Kc;
            const int sh = j * p.Wf / 4;  // chunks (Wf % 4 == 0)
            const int srow = k;           // copy 0 row of filter k ((srow & 7) == (row & 7): Kc % 8 == 0)
            const float4 v = q < sh ? ld_shared_v4_w2(Ps + srow * 128 + (((q + 8 - sh) ^ (srow & 7)) << 4))
                                    : ld_shared_v4_w2(As + srow * 128 + (((q - sh) ^ (srow & 7)) << 4));
            const int row = j * p.Kc + k;
            st_shared_v4_w2(As + row * 128 + ((q ^ (row & 7)) << 4), v.x, v.y, v.z, v.w);
          }
          ptx::fence_proxy_async_smem();
        }
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive(fullA + slotA);
          if (step > 0 && p.copies > 1 && p.hcopy) ptx::mbar_arrive(emptyA + slotP);  // previous atom no longer read
        }
      }
      if (step >= 0 && do_db && main_helper) {
        const int slotA = sa;
        if (drow < p.Kc) {
          const float4 *rp = reinterpret_cast<const float4 *>(Aring + slotA * a_slot + drow * 128) + dhalf * 4;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (q < dq) {
              const float4 v = rp[q];
              dbv += (v.x + v.y) + (v.z + v.w);
            }
          }
        }
        ptx::named_bar_sync(1, 128);
        if (et == 0) ptx::mbar_arrive(emptyA + slotA);
      }
      if (step >= 0) {
        if (++sa == W2_NA) { sa = 0; pa ^= 1; }
      }
    }
    if (do_db && main_helper) {
      if (dsplit) dbv += __shfl_xor_sync(0xffffffffu, dbv, 1);
      if ((!dsplit || (et & 1) == 0) && drow < p.Kc && k0 + drow < p.K)
        p.dbpart[(int64_t)z * p.K + k0 + drow] = dbv;
    }
    {
    // accumulator dump by both helper sets (TMEM quadrant = warp % 4): set main takes the even
    // 16-column groups, the other set the odd ones; rows whose tap r = rb*copies + j is past R
    // (R = 5 in row groups of two) are skipped -- the reduce skips them too
    if (nA > 0) ptx::mbar_wait_sleep(accf, 0);
    ptx::tc_fence_after();
    const int row = qd * 32 + lane;
    const int jrow = row / p.Kc;
    float *dst = p.part + (int64_t)blockIdx.x * p.RG * 128 * p.N;
    for (int rb = 0; rb < p.RG; ++rb) {
      const bool dead = rb * p.copies + jrow >= p.R || jrow >= p.copies;
      if (__all_sync(0xffffffffu, dead)) continue;  // tcgen05.ld is warp-collective
      for (int cb = main_helper ? 0 : 16; cb < p.N; cb += 32) {
        float v[16];
        if (nA > 0) {
          ptx::tmem_ld16(tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(rb * p.N + cb), v);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = 0.f;
        }
        if (dead) continue;
        float4 *o = reinterpret_cast<float4 *>(dst + ((int64_t)rb * 128 + row) * p.N + cb);
        o[0] = make_float4(v[0], v[1], v[2], v[3]);
        o[1] = make_float4(v[4], v[5], v[6], v[7]);
        o[2] = make_float4(v[8], v[9], v[10], v[11]);
        o[3] = make_float4(v[12], v[13], v[14], v[15]);
      }
    }
    }
  }
  if (p.clk && threadIdx.x == 32) p.clk[blockIdx.x * 8 + 6] = clock64() - tk0;
  if (p.clk && threadIdx.x == 64) p.clk[blockIdx.x * 8 + 7] = clock64() - tk0;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// dF[k][c][r][s] = sum over splits (fixed order) of D_rb[(j,k')][(s,c')] of the CTA tile
// (kt, ct) holding k = kt*Kc + k', c = ct*Ct + c', r = rb*copies + j
// few splits: one thread per output, splits summed in order
__global__ void w2_reduce_kernel(const W2Params p, float *__restrict__ df, float *__restrict__ db,
                                 const float *__restrict__ dbsrc, int dbcount) {
  const int RS = p.R * p.S;
  const int64_t total = (int64_t)p.K * p.C * RS;
  const int64_t cta_stride = (int64_t)p.RG * 128 * p.N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / ((int64_t)p.C * RS));
    const int rem = (int)(i - (int64_t)k * p.C * RS);
    const int c = rem / RS, t = rem - c * RS, r = t / p.S, s = t - r * p.S;
    const int rb = r / p.copies, j = r - rb * p.copies;
    const int kt = k / p.Kc, kk = k - kt * p.Kc, ct = c / p.Ct, cc = c - ct * p.Ct;
    const int64_t off = ((int64_t)rb * 128 + j * p.Kc + kk) * p.N + s * p.Ct + cc;
    const float *src = p.part + ((int64_t)(kt * p.nct + ct) * p.splits) * cta_stride + off;
    float acc = 0.f;
    for (int sp0 = 0; sp0 < p.splits; sp0 += 8) {  // 8 loads in flight, summed in split order
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = sp0 + u < p.splits ? __ldg(src + (sp0 + u) * cta_stride) : 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
    df[i] = acc;
  }
  if (db)
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < p.K;
         k += (int64_t)gridDim.x * blockDim.x) {
      float acc = 0.f;
      for (int sp = 0; sp < dbcount; ++sp) acc += __ldg(dbsrc + (int64_t)sp * p.K + k);
      db[k] = acc;
    }
}

// many splits: a CTA covers 32 float4 groups of partial offsets (the CTA-tile partial
// layout, so each split's reads are contiguous) x 8 eighths of the splits; thread (q, g)
// sums its eighth in split order, 8 float4 loads in flight, then the eight partial sums are
// added in order and scattered to dF[k][c][r][s] (valid rows / columns only).
// Fixed order throughout: deterministic.
constexpr int W2R_GROUPS = 32, W2R_Q = 8;
__global__ void __launch_bounds__(W2R_GROUPS * W2R_Q) w2_reduce_wide_kernel(
    const W2Params p, float *__restrict__ df, float *__restrict__ db, const float *__restrict__ dbsrc,
    int dbcount) {
  __shared__ float4 red[W2R_Q][W2R_GROUPS];
  const int64_t per_cta = (int64_t)p.RG * 128 * p.N;  // multiple of 4
  const int64_t groups = (int64_t)p.nkt * p.nct * per_cta / 4;
  const int gl = threadIdx.x % W2R_GROUPS, q = threadIdx.x / W2R_GROUPS;
  const int64_t g = blockIdx.x * (int64_t)W2R_GROUPS + gl;
  const int sq = (p.splits + W2R_Q - 1) / W2R_Q;
  const int sp_lo = q * sq, sp_hi = min(p.splits, sp_lo + sq);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int tile = 0;
  int64_t w = 0;
  bool live = false;
  if (g < groups) {
    tile = (int)(g * 4 / per_cta);
    w = g * 4 - (int64_t)tile * per_cta;
    // a group of 4 lies in one accumulator row; rows of taps past R were never written
    const int rb = (int)(w / (128 * p.N)), row = (int)(w - (int64_t)rb * 128 * p.N) / p.N;
    live = rb * p.copies + row / p.Kc < p.R && row / p.Kc < p.copies;
  }
  if (live) {
    const float4 *src =
        reinterpret_cast<const float4 *>(p.part + (int64_t)tile * p.splits * per_cta + w);
    const int64_t stride4 = per_cta / 4;
    for (int sp0 = sp_lo; sp0 < sp_hi; sp0 += 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        v[u] = sp0 + u < sp_hi ? __ldg(src + (int64_t)(sp0 + u) * stride4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc.x += v[u].x;
        acc.y += v[u].y;
        acc.z += v[u].z;
        acc.w += v[u].w;
      }
    }
  }
  red[q][gl] = acc;
  __syncthreads();
  if (q == 0 && live) {
    float4 t = red[0][gl];
#pragma unroll
    for (int qq = 1; qq < W2R_Q; ++qq) {
      const float4 u = red[qq][gl];
      t.x += u.x;
      t.y += u.y;
      t.z += u.z;
      t.w += u.w;
    }
    const float tv[4] = {t.x, t.y, t.z, t.w};
    const int kt = tile / p.nct, ct = tile - kt * p.nct;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t we = w + e;
      const int rb = (int)(we / (128 * p.N));
      const int rem = (int)(we - (int64_t)rb * 128 * p.N);
      const int row = rem / p.N, col = rem - row * p.N;
      const int j = row / p.Kc, kk = row - j * p.Kc;
      const int s = col / p.Ct, cc = col - s * p.Ct;
      const int k = kt * p.Kc + kk, c = ct * p.Ct + cc, r = rb * p.copies + j;
      if (kk >= p.Kc || k >= p.K || c >= p.C || r >= p.R || j >= p.copies || s >= p.S) continue;
      df[(((int64_t)k * p.C + c) * p.R + r) * p.S + s] = tv[e];
    }
  }
  if (db)
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < p.K;
         k += (int64_t)gridDim.x * blockDim.x) {
      float a = 0.f;
      for (int sp = 0; sp < dbcount; ++sp) a += __ldg(dbsrc + (int64_t)sp * p.K + k);
      db[k] = a;
    }
}

struct W2Plan {
  W2Params p;
  size_t smem, part_bytes, dbpart_bytes;
  int grid;
  bool ok;
};

W2Plan plan_w2(const SpfConv &sc) {
  W2Plan pl{};
  W2Params &p = pl.p;
  pl.ok = false;
  p.K = sc.K; p.C = sc.C; p.R = sc.R; p.S = sc.S; p.Wf = sc.Wf;
  if (sc.C % 8 || sc.x_shift % 4 || sc.dy_shift % 4 || sc.plane_x % 4 || sc.plane_dy % 4 ||
      sc.G <= 0 || sc.Wf % 8 || sc.S > 5)  // taps s = 1 .. 4 are built from the s = 0 rows
    return pl;
  // A rows (j, k): Kc filters per copy, copies of dY shifted by j frame rows
  p.Kc = sc.K <= 16 ? 16 : sc.K <= 32 ? 32 : sc.K <= 64 ? 64 : 128;
  p.copies = std::min(128 / p.Kc, sc.R);
  p.nkt = (int)ceil_div(sc.K, p.Kc);
  p.RG = (sc.R + p.copies - 1) / p.copies;
  p.shift = p.copies * sc.Wf;
  {
    // helper-built A copies: exact but slower (457 vs 392 us on LeNet B2f), opt-in
    static const int hc_env = getenv("SYSML_W2_HCOPY") ? atoi(getenv("SYSML_W2_HCOPY")) : 0;
    static const int hb_env = getenv("SYSML_W2_HB4") ? atoi(getenv("SYSML_W2_HB4")) : 1;
    p.hcopy = hc_env && (p.copies - 1) * sc.Wf <= 32 ? 1 : 0;
    p.hb4 = hb_env;
  }
  // channel tile: Ct <= 48 (3 helper tasks per thread), S*Ct % 16 == 0, RG*S*Ct TMEM
  // columns <= 512; the fewest tiles win, then the narrowest such tile (least zero-filled
  // padding in the ragged last one: C = 64 takes 2 x 32, not 2 x 48)
  // S = 1 has no helper-built taps, so the tile may be as wide as the MMA (N <= 256): fewer TMA
  // rows per unit of work (1x1 convs on planes whose rows are not 16-byte multiples, 7x7)
  p.Ct = 0;
  for (int ct = std::min(sc.S == 1 ? 256 : 48, (sc.C + 7) / 8 * 8); ct >= 8; ct -= 8)
    if ((sc.S * ct) % 16 == 0 && sc.S * ct <= 256 && p.RG * sc.S * ct <= 512) {
      if (p.Ct && ceil_div(sc.C, ct) > ceil_div(sc.C, p.Ct)) break;
      p.Ct = ct;
    }
  if (!p.Ct || p.RG > 4) return pl;
  p.nct = (int)ceil_div(sc.C, p.Ct);
  p.N = sc.S * p.Ct;
  p.L = (24 + (p.RG - 1) * p.shift) / W2_ATOM;
  if (p.L > W2_MAXL) return pl;  // B descriptors of atoms ai .. ai + W2_MAXL
  // B ring: >= L + 2 (atom bi + 1 resident while bi is shifted) plus run-ahead slots
  size_t smem = 0;
  for (p.nbr = p.L + 6; p.nbr >= p.L + 3; --p.nbr) {
    smem = 1024 + (size_t)W2_NA * 128 * 128 + (size_t)p.nbr * p.N * 128 +
           8 * (2 * W2_NA + 3 * p.nbr + 1) + 16;
    if (smem <= 227 * 1024) break;
  }
  if (smem > 227 * 1024) return pl;
  p.atoms = ceil_div(sc.G, W2_ATOM);
  const int tiles = p.nkt * p.nct;
  int splits = std::max(1, sm_count() / tiles);
  if (splits > p.atoms) splits = (int)p.atoms;
  p.splits = std::max(1, splits);
  pl.grid = tiles * p.splits;
  pl.smem = smem;
  pl.part_bytes = align_up((size_t)pl.grid * p.RG * 128 * p.N * sizeof(float), 256);
  pl.dbpart_bytes = align_up((size_t)p.splits * p.K * sizeof(float), 256);
  pl.ok = true;
  return pl;
}

}  // namespace

bool tc_wgrad_spf_tma_supported(const SpfConv &sc) {
  return device_cc_major() == 10 && plan_w2(sc).ok && getenv("SYSML_NO_TMA_WGRAD") == nullptr;
}

size_t tc_wgrad_spf_tma_ws(const SpfConv &sc) {
  const W2Plan pl = plan_w2(sc);
  return pl.ok ? pl.part_bytes + pl.dbpart_bytes : 0;
}

sysml_status tc_wgrad_spf_tma(const SpfConv &sc, const float *x_spf, const float *dy_spf,
                              float *df, float *db, void *ws, cudaStream_t st,
                              const float *db_src, int db_count) {
  W2Plan pl = plan_w2(sc);
  if (!pl.ok) {
    set_error("tcgen05 TMA SPF bwd_filter: unsupported shape");
    return SYSML_ERR_UNSUPPORTED;
  }
  const float *xb = x_spf + sc.x_shift, *dyb = dy_spf + sc.dy_shift;
  if (((uintptr_t)xb & 15) || ((uintptr_t)dyb & 15)) {
    set_error("tcgen05 TMA SPF bwd_filter: planes must be 16-byte aligned");
    return SYSML_ERR_UNSUPPORTED;
  }
  W2Params p = pl.p;
  p.dbg = getenv("SYSML_W2_DBG") ? atoi(getenv("SYSML_W2_DBG")) : 0;
  p.x = xb;
  p.G = sc.G;
  p.plane_x = sc.plane_x;
  p.ntma_s = (sc.S + 3) / 4;
  p.part = reinterpret_cast<float *>(ws);
  // db either from the staged dY atoms (dbpart) or precomputed per-image partials (db_src)
  p.dbpart = (db && !db_src) ? reinterpret_cast<float *>(reinterpret_cast<char *>(ws) + pl.part_bytes)
                             : nullptr;
  CUtensorMap tmDy, tmX;
  {
    const uint64_t dims[3] = {(uint64_t)sc.G, (uint64_t)sc.K, 1};
    const uint64_t strides[2] = {(uint64_t)sc.plane_dy * 4, (uint64_t)sc.plane_dy * 4 * sc.K};
    const uint32_t box[3] = {W2_ATOM, (uint32_t)p.Kc, 1};  // rows beyond K: zero-filled
    if (!tmap_encode_f32(&tmDy, dyb, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return SYSML_ERR_CUDA;
  }
  {
    const uint64_t dims[3] = {(uint64_t)sc.G, (uint64_t)sc.C, 1};
    const uint64_t strides[2] = {(uint64_t)sc.plane_x * 4, (uint64_t)sc.plane_x * 4 * sc.C};
    const uint32_t box[3] = {W2_ATOM, (uint32_t)p.Ct, 1};
    if (!tmap_encode_f32(&tmX, xb, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return SYSML_ERR_CUDA;
  }
  auto kern = p.shift == 32 ? tc_wgrad_spf_tma_kernel<32>
              : p.shift == 16 ? tc_wgrad_spf_tma_kernel<16>
                              : tc_wgrad_spf_tma_kernel<0>;
  SYSML_TRY(smem_attr(kern, pl.smem));
  static long long *dclk = nullptr;
  const bool prof = getenv("SYSML_TC_PROFILE") != nullptr;
  p.clk = nullptr;
  if (prof) {
    if (!dclk) cudaMalloc(&dclk, sizeof(long long) * 8 * 4096);
    cudaMemsetAsync(dclk, 0, sizeof(long long) * 8 * 4096, st);
    p.clk = dclk;
  }
  route_note("tc_wgrad_spf_tma_kernel<%d> [TMA + tcgen05 TF32, %d CTAs]", p.shift, pl.grid);
  kern<<<pl.grid, W2_THREADS, pl.smem, st>>>(tmDy, tmX, p);
  SYSML_LAUNCH_CHECK();
  if (prof) {
    static long long h[8 * 4096];
    cudaMemcpyAsync(h, dclk, sizeof(long long) * 8 * pl.grid, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double a[8] = {0};
    for (int b = 0; b < pl.grid; ++b)
      for (int j = 0; j < 8; ++j) a[j] += (double)h[b * 8 + j] / pl.grid;
    fprintf(stderr, "[w2 splits=%d atoms/cta=%.0f] mma_wait_A %.0f mma_wait_B %.0f help_wait_emptyB %.0f "
            "help_wait_fullA %.0f prod_wait_emptyA %.0f prod_wait_emptyB %.0f mma_total %.0f help_total %.0f\n",
            p.splits, (double)p.atoms / p.splits, a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7]);
  }
  const int64_t total = (int64_t)p.K * p.C * p.R * p.S;
  if (p.splits >= 32)
    w2_reduce_wide_kernel<<<(unsigned)ceil_div((int64_t)p.nkt * p.nct * p.RG * 128 * p.N / 4, W2R_GROUPS),
                            W2R_GROUPS * W2R_Q, 0, st>>>(
        p, df, db_src ? db : (p.dbpart ? db : nullptr), db_src ? db_src : p.dbpart,
        db_src ? db_count : p.splits);
  else
  w2_reduce_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 8 * sm_count()), 256, 0, st>>>(
      p, df, db_src ? db : (p.dbpart ? db : nullptr), db_src ? db_src : p.dbpart,
      db_src ? db_count : p.splits);
  SYSML_LAUNCH_CHECK();
  return SYSML_OK;
}

}  // namespace sysml

// =====================================================================================
// NCHW entry (public conv2d_backward_filter, K5): copy X and dY into stacked frames
// (HBM-bound pre-pass) and run the TMA kernel above.
//   X frame:  X_f[c][n*Hs*Wf + (h+ph)*Wf + (w+pw)] = X[n][c][h][w], zeros elsewhere
//   dY frame: dY_f[k][n*Hs*Wf + p*Wf + q] = dY[n][k][p][q], zeros elsewhere
// sum_g dY_f[g] X_f[g + r*Wf + s] equals the definition when the column /
// row wrap lands in zero padding: Wf >= max(W + pw, Q + S - 1 - pw) and
// Hs >= max(H + ph, P + R - 1 - ph); Wf is rounded up to a multiple of 8 so the tap-row
// shifts are whole 32-byte steps of the swizzled rows.
// =====================================================================================
namespace sysml {
namespace {

// four float4s of frame rows per thread iteration (Wf % 4 == 0): independent loads in
// flight; index decoding per float4
__global__ void nchw_to_frame_kernel(const float *__restrict__ src, float *__restrict__ dst, int N,
                                     int C, int H, int W, int Hs, int Wf, int oh, int ow,
                                     int64_t plane) {
  const int q4 = Wf >> 2;
  const int NHs = N * Hs;
  const int64_t total = (int64_t)C * NHs * q4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t0 < total; t0 += 4 * stride) {
    float v[4][4];
    int64_t dsti[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = t0 + u * stride;
      dsti[u] = -1;
#pragma unroll
      for (int e = 0; e < 4; ++e) v[u][e] = 0.f;
      if (t < total) {
        const int64_t row = t / q4;
        const int w0 = (int)(t - row * q4) * 4 - ow;
        const int c = (int)(row / NHs);
        const int rem = (int)(row - (int64_t)c * NHs);
        const int n = rem / Hs, hh = rem - n * Hs;
        const int h = hh - oh;
        dsti[u] = (int64_t)c * plane + (int64_t)rem * Wf + (t - row * q4) * 4;
        if (h >= 0 && h < H) {
          const float *srow = src + (((int64_t)n * C + c) * H + h) * W;
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (w0 + e >= 0 && w0 + e < W) v[u][e] = __ldg(srow + w0 + e);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (dsti[u] >= 0)
        *reinterpret_cast<float4 *>(dst + dsti[u]) = make_float4(v[u][0], v[u][1], v[u][2], v[u][3]);
  }
}

// dY framing, one warp per (k, n) plane, also writing the plane's sum (db partial
// psum[n][k], warp butterfly in a fixed order -> deterministic)
__global__ void nchw_to_frame_sum_kernel(const float *__restrict__ src, float *__restrict__ dst,
                                         float *__restrict__ psum, int N, int C, int H, int W,
                                         int Hs, int Wf, int64_t plane) {
  const int lane = threadIdx.x & 31;
  const int q4 = Wf >> 2, nf4 = Hs * q4;
  const int64_t planes = (int64_t)C * N;
  const int64_t wstep = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t pl = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; pl < planes; pl += wstep) {
    const int n = (int)(pl / C), c = (int)(pl - (int64_t)n * C);
    const float *sp = src + ((int64_t)n * C + c) * H * W;
    float *dp = dst + (int64_t)c * plane + (int64_t)n * Hs * Wf;
    float sum = 0.f;
    for (int f4 = lane; f4 < nf4; f4 += 32) {
      const int hh = f4 / q4, w0 = (f4 - hh * q4) * 4;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (hh < H) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (w0 + e < W) v[e] = __ldg(sp + hh * W + w0 + e);
      }
      sum += (v[0] + v[1]) + (v[2] + v[3]);
      reinterpret_cast<float4 *>(dp)[f4] = make_float4(v[0], v[1], v[2], v[3]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0 && psum) psum[(int64_t)n * C + c] = sum;
  }
}

struct FramePlan {
  int Hs, Wf;
  int64_t G, plane;
  SpfConv sc;
  size_t x_bytes, dy_bytes;
  bool ok;
};

FramePlan plan_frame(const ConvArgs &a) {
  FramePlan f{};
  f.ok = false;
  if (a.sh != 1 || a.sw != 1 || a.C % 8 || a.R > 8 || a.S > 8) return f;
  f.Wf = (int)std::max<int64_t>(a.W + a.pw, a.Q + a.S - 1 - a.pw);
  f.Wf = (f.Wf + 7) / 8 * 8;
  f.Hs = (int)std::max<int64_t>(a.H + a.ph, a.P + a.R - 1 - a.ph);
  f.G = (int64_t)a.N * f.Hs * f.Wf;
  f.plane = (f.G + 3) / 4 * 4;
  if (f.G >= (1ll << 31)) return f;
  f.sc = SpfConv{(int)a.K, (int)a.C, (int)a.R, (int)a.S, f.Wf, f.G, f.plane, f.plane, 0, 0};
  f.x_bytes = align_up((size_t)a.C * f.plane * sizeof(float), 256);
  f.dy_bytes = align_up((size_t)a.K * f.plane * sizeof(float), 256) +
               align_up((size_t)a.N * a.K * sizeof(float), 256);  // + per-image db partials
  f.ok = plan_w2(f.sc).ok;
  return f;
}

}  // namespace

bool tc_wgrad_frame_supported(const ConvArgs &a) {
  if (device_cc_major() != 10 || getenv("SYSML_NO_TMA_WGRAD")) return false;
  return plan_frame(a).ok;
}

size_t tc_wgrad_frame_ws(const ConvArgs &a) {
  const FramePlan f = plan_frame(a);
  return f.ok ? f.x_bytes + f.dy_bytes + tc_wgrad_spf_tma_ws(f.sc) : 0;
}

void tc_wgrad_frame_geom(const ConvArgs &a, int *Hs, int *Wf, int64_t *plane) {
  const FramePlan f = plan_frame(a);
  *Hs = f.Hs;
  *Wf = f.Wf;
  *plane = f.plane;
}

sysml_status tc_wgrad_frame(const ConvArgs &a, const float *x, const float *dy, float *df,
                            float *db, void *ws, cudaStream_t st, bool x_framed) {
  const FramePlan f = plan_frame(a);
  if (!f.ok) {
    set_error("tcgen05 framed bwd_filter: unsupported shape");
    return SYSML_ERR_UNSUPPORTED;
  }
  float *xf = reinterpret_cast<float *>(ws);
  float *dyf = reinterpret_cast<float *>(reinterpret_cast<char *>(ws) + f.x_bytes);
  void *ws2 = reinterpret_cast<char *>(ws) + f.x_bytes + f.dy_bytes;
  const int blocks = 8 * sm_count();
  if (x_framed) {
    xf = const_cast<float *>(x);  // caller wrote X in the frame layout already (phase.cu)
  } else {
    nchw_to_frame_kernel<<<blocks, 256, 0, st>>>(x, xf, (int)a.N, (int)a.C, (int)a.H, (int)a.W, f.Hs,
                                                 f.Wf, (int)a.ph, (int)a.pw, f.plane);
    SYSML_LAUNCH_CHECK();
  }
  float *psum = reinterpret_cast<float *>(reinterpret_cast<char *>(dyf) +
                                          align_up((size_t)a.K * f.plane * sizeof(float), 256));
  nchw_to_frame_sum_kernel<<<blocks, 256, 0, st>>>(dy, dyf, db ? psum : nullptr, (int)a.N, (int)a.K,
                                                   (int)a.P, (int)a.Q, f.Hs, f.Wf, f.plane);
  SYSML_LAUNCH_CHECK();
  return tc_wgrad_spf_tma(f.sc, xf, dyf, df, db, ws2, st, db ? psum : nullptr, (int)a.N);
}

}  // namespace sysml
