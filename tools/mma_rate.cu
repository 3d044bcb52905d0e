// mma_rate.cu -- clocks per tcgen05.mma kind::tf32 (M=128) by N, operand layout (no swizzle /
// 128-byte swizzle K-major) and data (constant / random): is the MMA itself the limit?
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../paper_1802_04647_b200/csrc/tc_ptx.cuh"
using namespace sysml;

template <int NACC>
__global__ void bench(int N, int sw, int rnd, int reps, unsigned long long *out, int aoff, int halo, int boff) {
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
  const uint32_t A = ptx::smem_u32(smem), B = A + (boff ? boff : 64 * 1024);
  const uint32_t idesc = ptx::make_idesc_tf32(128, N);
  uint32_t tm[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) tm[k] = (uint32_t)((k % NACC) * N);
  uint64_t adv[4], bdv[4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    if (sw) {
      adv[kk] = (ptx::make_desc(A + kk * 32, 16, 1024) | ((uint64_t)2 << 61));
      bdv[kk] = (ptx::make_desc(B + kk * 32, 16, 1024) | ((uint64_t)2 << 61));
    } else {
      adv[kk] = halo ? ptx::make_desc(A + kk * 16 * 16 + aoff * 16, halo * 16, 128) : ptx::make_desc(A + kk * 128 * 32 + aoff * 16, 128 * 16, 128);
      bdv[kk] = ptx::make_desc(B + kk * N * 32, N * 16, 128);
    }
  }
  if (threadIdx.x < 32) {
    unsigned long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (ptx::elect_one()) ptx::mma_tf32(tm[kk], adv[kk], bdv[kk], idesc, 1u);
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
  cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  cudaFuncSetAttribute(bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  cudaFuncSetAttribute(bench<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  const int reps = 2000;
  for (int cfg = 0; cfg < 4; ++cfg)
  for (int sw = 0; sw < 1; ++sw)
    for (int nacc : {1})
      for (int N : {64, 96, 160}) {
        const int aoff = 0, halo = (cfg & 1) ? 328 : 0, boff = (cfg & 2) ? 2 * 328 * 16 : 0;
        if (nacc * N > 512) continue;
        const int rnd = 1;
        for (int grid : {148}) {
          if (nacc == 1) bench<1><<<grid, 128, 170 * 1024>>>(N, sw, rnd, reps, d, aoff, halo, boff);
          else if (nacc == 2) bench<2><<<grid, 128, 170 * 1024>>>(N, sw, rnd, reps, d, aoff, halo, boff);
          else bench<4><<<grid, 128, 170 * 1024>>>(N, sw, rnd, reps, d, aoff, halo, boff);
          if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
          cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
          const double n = reps * 4.0;
          printf("halo=%d boff=%d sw128=%d nacc=%d N=%3d grid=%3d: %.1f clk/mma (ideal %.1f at 2048 FMA/clk)\n", halo, boff, sw, nacc, N, grid,
                 h[1] / n, 128.0 * N * 8 / 2048);
        }
      }
  return 0;
}
