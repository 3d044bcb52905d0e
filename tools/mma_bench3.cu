// mma_bench3.cu -- tcgen05.mma tf32 M=128 throughput vs operand/accumulator variation.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../paper_1802_04647_b200/csrc/tc_ptx.cuh"
using namespace sysml;

__global__ void bench(int N, int nmma, int vary_a, int vary_d, int vary_b, int a_shift16, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) ((float *)smem)[i] = 0.001f * (i & 7);
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc(&tslot, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t A = ptx::smem_u32(smem);
  const uint32_t B = A + 128 * 1024;
  const uint32_t idesc = ptx::make_idesc_tf32(128, N);
  // A: 8 M-tiles of 128 rows (linear positions, 16 B each) for 2 quads: quad stride = 8*128*16 = 16 KB
  const uint32_t halo = 1100;
  uint64_t ad = ptx::make_desc(A, halo * 16, 128);
  uint64_t bd = ptx::make_desc(B, (uint32_t)N * 16, 128);
  if (threadIdx.x < 32) {
    __syncwarp();
    unsigned long long t0 = clock64();
    for (int i = 0; i < nmma; i += 8) {
      const uint64_t b_i = bd + (vary_b ? (uint64_t)(((i >> 3) % 25) * 2 * N) % 2048 : 0);
      const uint64_t shift = a_shift16 ? (uint64_t)((i >> 3) % 25) : 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (ptx::elect_one())
          ptx::mma_tf32(vary_d ? (uint32_t)((j * N) % 512) : 0u, ad + (vary_a ? (uint64_t)(j * 128) : 0) + shift, b_i, idesc, 1u);
        __syncwarp();
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

int GRID = 1;
int main(int argc, char **argv) {
  if (argc > 1) GRID = atoi(argv[1]);
  unsigned long long *d, h[2];
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct V { int a, dd, b, sh; const char *n; } vs[] = {
    {0, 0, 0, 0, "same A/B/D"}, {1, 0, 0, 0, "vary A"}, {0, 1, 0, 0, "vary D"}, {0, 0, 1, 0, "vary B"},
    {1, 1, 0, 0, "vary A+D"}, {1, 1, 1, 0, "vary A+D+B"}, {1, 1, 1, 1, "vary all + A shift"}};
  for (auto v : vs)
    for (int N : {64, 256}) {
      int nmma = 4000;
      bench<<<GRID, 128, 200 * 1024>>>(N, nmma, v.a, v.dd, v.b, v.sh, d);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("%-22s N=%3d: issue %.1f, complete %.1f clk/mma\n", v.n, N, (double)h[0] / nmma, (double)h[1] / nmma);
    }
  return 0;
}
