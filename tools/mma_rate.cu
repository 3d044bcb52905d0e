// mma_rate.cu -- clocks per tcgen05.mma kind::tf32 (M=128) by N, operand layout (no swizzle /
// 128-byte swizzle K-major) and data (constant / random): is the MMA itself the limit?
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../paper_1802_04647_b200/csrc/tc_ptx.cuh"
using namespace sysml;

__global__ void bench(int N, int sw, int rnd, int reps, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u; h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    ((float *)smem)[i] = rnd ? ((float)(h & 0xFFFFFF) / 16777216.0f - 0.5f) : 0.001f * (i & 7);
  }
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc(&tslot, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t A = ptx::smem_u32(smem), B = A + 64 * 1024;
  const uint32_t idesc = ptx::make_idesc_tf32(128, N);
  if (threadIdx.x < 32) {
    unsigned long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad, bd;
        if (sw) {
          ad = (ptx::make_desc(A + kk * 32, 16, 1024) | ((uint64_t)2 << 61));
          bd = (ptx::make_desc(B + kk * 32, 16, 1024) | ((uint64_t)2 << 61));
        } else {
          ad = ptx::make_desc(A + kk * 128 * 32, 128 * 16, 128);
          bd = ptx::make_desc(B + kk * N * 32, N * 16, 128);
        }
        if (ptx::elect_one()) ptx::mma_tf32(0, ad, bd, idesc, 1u);
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

int main() {
  unsigned long long *d, h[2];
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  const int reps = 2000;
  for (int sw = 0; sw < 2; ++sw)
    for (int rnd = 0; rnd < 2; ++rnd)
      for (int N : {64, 128, 256}) {
        for (int grid : {1, 148}) {
          bench<<<grid, 128, 170 * 1024>>>(N, sw, rnd, reps, d);
          if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
          cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
          const double n = reps * 4.0;
          printf("sw128=%d rnd=%d N=%3d grid=%3d: %.1f clk/mma (ideal %.1f at 2048 FMA/clk)\n", sw, rnd, N, grid,
                 h[1] / n, 128.0 * N * 8 / 2048);
        }
      }
  return 0;
}
