// mma_bench.cu -- microbenchmark: cycles per tcgen05.mma.kind::tf32 (M=128) issued
// back to back from one thread, for smem operand layouts SWIZZLE_NONE / 32B / 128B,
// K-major A and B, several N; plus aligned vs shifted A start addresses.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mma_bench.cu -o /tmp/mma_bench
#include <cstdio>
#include <cstdint>
#include "../paper_1802_04647_b200/csrc/tc_ptx.cuh"

using namespace sysml;

__device__ uint64_t desc_layout(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout,
                                uint32_t base_off) {
  uint64_t d = ptx::make_desc(saddr, lbo, sbo);
  d |= (uint64_t)(base_off & 7) << 49;
  d |= (uint64_t)layout << 61;
  return d;
}

// layout: 0 none, 6 = SW32, 2 = SW128
__global__ void bench(int layout, int N, int nmma, int shift_rows, int use_commit_each,
                      unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  // fill smem with small values
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((float *)smem)[i] = 0.001f * (i & 7);
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc(&tslot, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t A = ptx::smem_u32(smem);
  const uint32_t B = A + 64 * 1024;
  uint32_t lbo, sbo;
  if (layout == 0) { lbo = 128 * 16; sbo = 128; }      // A: [khalf][row][16B]
  else if (layout == 6) { lbo = 16; sbo = 256; }       // 32B rows
  else { lbo = 16; sbo = 1024; }                       // 128B rows
  uint32_t rowb = layout == 0 ? 16 : (layout == 6 ? 32 : 128);
  const uint32_t idesc = ptx::make_idesc_tf32(128, N);
  if (threadIdx.x == 0) {
    unsigned long long t0 = clock64();
    for (int i = 0; i < nmma; ++i) {
      uint32_t aoff = shift_rows ? (uint32_t)((i % 7) * rowb) : 0;
      uint32_t astart = A + aoff;
      uint32_t boff = layout == 6 ? ((astart >> 8) & 7) : ((astart >> 7) & 7);
      uint64_t ad = desc_layout(astart, lbo, sbo, layout, layout == 0 ? 0 : boff);
      uint32_t blbo = layout == 0 ? (uint32_t)N * 16 : 16;
      uint64_t bd = desc_layout(B, blbo, sbo, layout, 0);
      ptx::mma_tf32(tmem + (i & 1) * 256 * 0, ad, bd, idesc, i > 0);
      if (use_commit_each) ptx::mma_commit(&bar);
    }
    ptx::mma_commit(&bar);
    // wait for the final commit (phase parity toggles once per commit arrival)
    unsigned long long t1 = clock64();
    int commits = use_commit_each ? nmma + 1 : 1;
    ptx::mbar_wait(&bar, (commits - 1) & 1);
    unsigned long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

int main() {
  unsigned long long *d, h[2];
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int layouts[3] = {0, 6, 2};
  const char *names[3] = {"NONE", "SW32", "SW128"};
  for (int li = 0; li < 3; ++li)
    for (int N : {32, 64, 128, 256})
      for (int shift : {0, 1}) {
        int nmma = 2000;
        bench<<<1, 128, 160 * 1024>>>(layouts[li], N, nmma, shift, 0, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("layout %-5s N=%3d shift=%d: issue %.1f clk/mma, complete %.1f clk/mma (ideal %d)\n",
               names[li], N, shift, (double)h[0] / nmma, (double)h[1] / nmma, 128 * N / 256);
      }
  return 0;
}
