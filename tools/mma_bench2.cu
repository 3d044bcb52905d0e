// mma_bench2.cu -- issue-loop styles for tcgen05.mma (cycles per MMA, one CTA).
#include <cstdio>
#include <cstdint>
#include "../paper_1802_04647_b200/csrc/tc_ptx.cuh"
using namespace sysml;

template <int VARIANT>
__global__ void bench(int N, int nmma, uint32_t layout, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
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
  const uint32_t idesc = ptx::make_idesc_tf32(128, N);
  uint64_t ad = ptx::make_desc(A, 128 * 16, 128) | ((uint64_t)layout << 61);
  uint64_t bd = ptx::make_desc(B, (uint32_t)N * 16, 128) | ((uint64_t)layout << 61);
  if (threadIdx.x < 32) {
    __syncwarp();
    unsigned long long t0 = clock64();
    if (VARIANT == 0) {
      // warp-wide loop, elect per MMA, uniform descriptor increments
      for (int i = 0; i < nmma; ++i) {
        if (ptx::elect_one()) ptx::mma_tf32(tmem, ad + (uint64_t)((i & 7) * 2), bd, idesc, 1u);
        __syncwarp();
      }
    } else if (VARIANT == 1) {
      // warp-wide loop, one elect per 8 MMAs, unrolled constant offsets
      for (int i = 0; i < nmma; i += 8) {
        if (ptx::elect_one()) {
#pragma unroll
          for (int j = 0; j < 8; ++j) ptx::mma_tf32(tmem + j * 0, ad + (uint64_t)(j * 2), bd, idesc, 1u);
        }
        __syncwarp();
      }
    } else {
      // single thread, unrolled by 8
      if (threadIdx.x == 0) {
        for (int i = 0; i < nmma; i += 8) {
#pragma unroll
          for (int j = 0; j < 8; ++j) ptx::mma_tf32(tmem, ad + (uint64_t)(j * 2), bd, idesc, 1u);
        }
      }
      __syncwarp();
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
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

template <int V>
void run(const char *name) {
  unsigned long long *d, h[2];
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  for (uint32_t layout : {0u, 2u})
    for (int N : {32, 64, 128, 256}) {
      int nmma = 4096;
      bench<V><<<1, 128, 160 * 1024>>>(N, nmma, layout, d);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return; }
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("%-22s layout %u N=%3d: issue %.1f, complete %.1f clk/mma (ideal %d)\n", name, layout, N,
             (double)h[0] / nmma, (double)h[1] / nmma, 128 * N / 256);
    }
}

int main() {
  run<0>("warp elect/mma");
  run<1>("warp elect/8mma");
  run<2>("thread unroll8");
  return 0;
}
