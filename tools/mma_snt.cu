// mma_snt.cu -- the conv kernel's SN-T issue loop (per tap row: MMA N=T*32 unshifted, MMA
// N=(S-T)*32 on A shifted by T, MT M-tiles) in isolation: clocks per MMA without producers
// or epilogue, to separate the issue loop from smem / TMEM contention.
#include <cstdio>
#include <cstdint>
#include "../paper_1802_04647_b200/csrc/tc_ptx.cuh"
using namespace sysml;

struct P { int R, S, snt, NFpad, MT, Wf, HALO, reps; int n2override, shift2; };

template <int V>
__global__ void bench(P p, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 180 * 1024 / 4; i += blockDim.x) ((float *)smem)[i] = 0.001f * (i & 7);
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc(&tslot, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t A = ptx::smem_u32(smem);
  const uint32_t n1 = p.snt * p.NFpad, n2 = p.n2override ? p.n2override : (p.S - p.snt) * p.NFpad;
  const uint32_t idesc = ptx::make_idesc_tf32(128, n1), idesc2 = ptx::make_idesc_tf32(128, n2);
  const uint32_t a_bytes = 2 * p.HALO * 16;
  const uint64_t adesc0 = ptx::make_desc(A, p.HALO * 16, 128);
  const uint32_t nf = n1;
  if (threadIdx.x < 32) {
    unsigned long long t0 = clock64();
    if (V == 0) {
    for (int rep = 0; rep < p.reps; ++rep) {
      uint32_t drow = 0, acc = 1;
      const uint32_t bsrow = A + a_bytes;
      for (int r = 0; r < p.R; ++r, drow += (uint32_t)p.Wf) {
        const uint32_t br = bsrow + (uint32_t)r * 2u * (n1 + n2) * 16u;
        const uint64_t bd1 = ptx::make_desc(br, n1 * 16, 128);
        const uint64_t bd2 = ptx::make_desc(br + 2u * n1 * 16u, n2 * 16, 128);
        uint64_t ad = adesc0 + (uint64_t)drow;
        uint32_t tm = 0;
        for (int i = 0; i < p.MT; ++i) {
          if (ptx::elect_one()) ptx::mma_tf32(tm, ad, bd1, idesc, acc);
          __syncwarp();
          if (ptx::elect_one()) ptx::mma_tf32(tm, ad + (uint64_t)p.shift2, bd2, idesc2, 1u);
          __syncwarp();
          tm += nf;
          ad += 128u;
        }
      }
    }
    } else {
    // descriptors by adds only, M-tile loop unrolled (MT <= 4, guarded)
    const uint64_t bd1_0 = ptx::make_desc(A + a_bytes, n1 * 16, 128);
    const uint64_t bd2_0 = ptx::make_desc(A + a_bytes + 2u * n1 * 16u, n2 * 16, 128);
    const uint64_t bstep = (uint64_t)((2u * (n1 + n2) * 16u) >> 4);
    const uint64_t rstep = (uint64_t)p.Wf;
    const uint32_t sh2 = (uint32_t)p.shift2;
    for (int rep = 0; rep < p.reps; ++rep) {
      uint64_t bd1 = bd1_0, bd2 = bd2_0, ad = adesc0;
      for (int r = 0; r < p.R; ++r) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i < p.MT) {
            if (ptx::elect_one()) ptx::mma_tf32((uint32_t)i * nf, ad + (uint64_t)(i * 128), bd1, idesc, 1u);
            __syncwarp();
            if (ptx::elect_one()) ptx::mma_tf32((uint32_t)i * nf, ad + (uint64_t)(i * 128 + sh2), bd2, idesc2, 1u);
            __syncwarp();
          }
        }
        ad += rstep;
        bd1 += bstep;
        bd2 += bstep;
      }
    }
    }
    unsigned long long t1 = clock64();
    if (ptx::elect_one()) ptx::mma_commit(&bar);
    __syncwarp();
    ptx::mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(tslot, 512); }
}

int main() {
  unsigned long long *d, h[2];
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024);
  cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024);
  P cases[] = {{5, 5, 3, 32, 2, 16, 328, 400, 0, 3}, {5, 5, 3, 32, 2, 16, 328, 400, 0, 0},
               {5, 5, 3, 32, 2, 16, 328, 400, 96, 3}, {5, 5, 3, 32, 2, 16, 328, 400, 96, 0},
               {5, 5, 3, 32, 2, 16, 328, 400, 64, 0}, {5, 5, 2, 32, 2, 16, 328, 400, 64, 0}};
  for (int v = 0; v < 2; ++v)
  for (P p : cases) {
    if (v == 0) bench<0><<<148, 128, 180 * 1024>>>(p, d); else bench<1><<<148, 128, 180 * 1024>>>(p, d);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const int per = p.snt < p.S ? 2 : 1;
    const double n = (double)p.reps * p.R * p.MT * per;
    printf("V%d n1=%d n2=%d shift2=%d MT=%d: %.1f clk/mma, %.1f clk per (r, M-tile)\n", v, p.snt * p.NFpad,
           p.n2override ? p.n2override : (p.S - p.snt) * p.NFpad, p.shift2, p.MT, h[1] / n,
           h[1] / ((double)p.reps * p.R * p.MT));
  }
  return 0;
}
