// mma_bench4.cu -- issue-loop shapes matching conv_tc's forward loop (runtime taps x M-tiles)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../paper_1802_04647_b200/csrc/tc_ptx.cuh"
using namespace sysml;

struct P { int R, S, Wf, MT, N, reps, rnd; int halo = 1096; int kernel_layout = 0; };

template <int V>
__global__ void bench(P p, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) { uint32_t h = (uint32_t)i * 2654435761u; h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15; ((float *)smem)[i] = p.rnd ? ((float)(h & 0xFFFFFF) / 16777216.0f - 0.5f) : 0.001f * (i & 7); }
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc(&tslot, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t A = ptx::smem_u32(smem);
  const uint32_t B = A + 128 * 1024;
  const uint32_t idesc = ptx::make_idesc_tf32(128, p.N);
  const uint32_t halo = p.halo;
  uint64_t adesc0 = ptx::make_desc(A, halo * 16, 128);
  const uint32_t nf = p.N;
  if (threadIdx.x < 32) {
    __syncwarp();
    unsigned long long t0 = clock64();
    for (int rep = 0; rep < p.reps; ++rep) {
      uint64_t bdesc = ptx::make_desc(B, nf * 16, 128);
      if (p.kernel_layout) {  // the conv kernel's stage layout: [A halo | B taps] x 2 stages
        const uint32_t a_bytes = 2 * halo * 16, stage_bytes = a_bytes + 25 * 2 * nf * 16;
        const uint32_t As = A + (uint32_t)(rep & 1) * stage_bytes;
        adesc0 = ptx::make_desc(As, halo * 16, 128);
        bdesc = ptx::make_desc(As + a_bytes, nf * 16, 128);
      }
      if (V == 3 || V == 4) {  // kernel style + per-chunk fence/commit (+ acc=0 start for V4)
        ptx::tc_fence_after();
        uint32_t drow = 0;
        uint32_t acc = (V == 4 && rep == 0) ? 0u : 1u;
        for (int r = 0; r < p.R; ++r, drow += p.Wf)
          for (int s = 0; s < p.S; ++s) {
            const uint64_t ad_t = adesc0 + drow + s;
            uint32_t tm = 0;
            for (int i = 0; i < p.MT; ++i) {
              if (ptx::elect_one()) ptx::mma_tf32(tm, ad_t + (uint64_t)(i * 128), bdesc, idesc, acc);
              __syncwarp();
              tm += nf;
            }
            acc = 1u;
            bdesc += 2 * nf;
          }
        if (ptx::elect_one()) ptx::mma_commit(&bar);
        __syncwarp();
      } else if (V == 0) {  // current kernel style: nested runtime loops, elect per MMA
        uint32_t drow = 0;
        for (int r = 0; r < p.R; ++r, drow += p.Wf)
          for (int s = 0; s < p.S; ++s) {
            const uint64_t ad_t = adesc0 + drow + s;
            uint32_t tm = 0;
            for (int i = 0; i < p.MT; ++i) {
              if (ptx::elect_one()) ptx::mma_tf32(tm, ad_t + (uint64_t)(i * 128), bdesc, idesc, 1u);
              __syncwarp();
              tm += nf;
            }
            bdesc += 2 * nf;
          }
      } else if (V == 1) {  // unrolled M-tile loop (guarded), elect per MMA
        uint32_t drow = 0;
        for (int r = 0; r < p.R; ++r, drow += p.Wf)
          for (int s = 0; s < p.S; ++s) {
            const uint64_t ad_t = adesc0 + drow + s;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if (i < p.MT) {
                if (ptx::elect_one()) ptx::mma_tf32(i * nf, ad_t + (uint64_t)(i * 128), bdesc, idesc, 1u);
                __syncwarp();
              }
            }
            bdesc += 2 * nf;
          }
      } else {  // one elected thread issues the whole tap loop, M-tiles unrolled
        if (ptx::elect_one()) {
          uint32_t drow = 0;
          for (int r = 0; r < p.R; ++r, drow += p.Wf)
            for (int s = 0; s < p.S; ++s) {
              const uint64_t ad_t = adesc0 + drow + s;
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (i < p.MT) ptx::mma_tf32(i * nf, ad_t + (uint64_t)(i * 128), bdesc, idesc, 1u);
              bdesc += 2 * nf;
            }
        }
        __syncwarp();
      }
    }
    unsigned long long t1 = clock64();
    if (ptx::elect_one()) ptx::mma_commit(&bar);
    __syncwarp();
    ptx::mbar_wait(&bar, (V == 3 || V == 4) ? (p.reps & 1) : 0);
    unsigned long long t2 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(tslot, 512); }
}

template <int V> void run(const char *nm, P p) {
  unsigned long long *d, h[2];
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  bench<V><<<1, 128, 200 * 1024>>>(p, d);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); exit(1); }
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double n = (double)p.reps * p.R * p.S * p.MT;
  printf("%-28s R=%d MT=%d N=%3d rnd=%d: %.1f clk/mma (issue %.1f)\n", nm, p.R, p.MT, p.N, p.rnd, h[1] / n, h[0] / n);
}

int main() {
  P cases[4] = {P{5, 5, 16, 8, 64, 20, 1}, P{5, 5, 16, 8, 64, 20, 1}, P{5, 5, 16, 8, 64, 20, 1}, P{5, 5, 16, 8, 64, 20, 1}};
  cases[1].halo = 1092; cases[2].kernel_layout = 1; cases[3].halo = 1092; cases[3].kernel_layout = 1;
  for (P p : cases) {
    printf("halo %d kernel_layout %d\n", p.halo, p.kernel_layout);
    run<0>("nested/elect-per-mma", p);
    run<3>("kernel-style+fence+commit", p);
    run<4>("kernel-style+acc0", p);
    run<1>("unrolled16/elect-per-mma", p);
    run<2>("single-thread/unrolled16", p);
  }
}
