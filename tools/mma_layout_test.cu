// mma_layout_test.cu -- correctness probe for tcgen05.mma.kind::tf32 operand layouts:
// A (128 x 8) and B (16 x 8) written to shared memory in a chosen layout, one MMA,
// D read back and compared with a host reference.  Used to establish which
// MN-major / swizzled layouts the hardware accepts for TF32.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/mma_layout_test.cu -o /tmp/mlt
#include <cstdio>
#include <cstdint>
#include <cmath>
#include "../paper_1802_04647_b200/csrc/tc_ptx.cuh"
using namespace sysml;

// modes for A: 0 K-major none, 1 MN-major none (SBO=MN grp, LBO=K grp), 2 MN-major none swapped,
// 3 MN-major SW128 (LBO=MN atom, SBO=K atom), 4 MN-major SW128 swapped, 5 MN-major SW32, 6 SW64
__device__ uint32_t a_off(int mode, int m, int k) {
  switch (mode) {
    case 0: return (k / 4) * 2048 + (m / 8) * 128 + (m % 8) * 16 + (k % 4) * 4;
    case 1: case 2: return (m / 4) * 128 + (k / 8) * 4096 + (k % 8) * 16 + (m % 4) * 4;
    case 3: case 4: {  // atom 8 K-rows x 128 B (32 m)
      const int row = k % 8, chunk = (m % 32) / 4;
      return (m / 32) * 1024 + row * 128 + ((chunk ^ row) * 16) + (m % 4) * 4;
    }
    case 5: {  // SW32: atom 8 K-rows x 32 B (8 m), swizzle chunk ^= (row>>2)&1 ... Swizzle<1,4,3>
      const int row = k % 8, chunk = (m % 8) / 4;
      const uint32_t lin = row * 32 + chunk * 16;
      const uint32_t sw = lin ^ (((lin >> 7) & 1) << 4);
      return (m / 8) * 256 + sw + (m % 4) * 4;
    }
    case 7: {  // K-major SW128: row m = 128 B (32 k), 16-B chunk ^= (m % 8); atoms of 8 rows at 1024 B
      const int chunk = k / 4;
      return m * 128 + ((chunk ^ (m % 8)) * 16) + (k % 4) * 4;
    }
    case 8: {  // K-major SW128, K offset 8 (second K-step inside the 128-B row): data at k+8
      const int kk = k + 8, chunk = kk / 4;
      return m * 128 + ((chunk ^ (m % 8)) * 16) + (kk % 4) * 4;
    }
    case 9: {  // K-major SW64: row m = 64 B (16 k), chunk ^= (m/2)%4 (Swizzle<2,4,3> on byte addr)
      const uint32_t lin = m * 64 + (k / 4) * 16;
      const uint32_t sw = lin ^ (((lin >> 7) & 3) << 4);
      return sw + (k % 4) * 4;
    }
    default: {  // SW64: atom 8 rows x 64 B (16 m), Swizzle<2,4,3>
      const int row = k % 8, chunk = (m % 16) / 4;
      const uint32_t lin = row * 64 + chunk * 16;
      const uint32_t sw = lin ^ (((lin >> 7) & 3) << 4);
      return (m / 16) * 512 + sw + (m % 4) * 4;
    }
  }
}
__device__ uint64_t a_desc(int mode, uint32_t A) {
  uint64_t d;
  switch (mode) {
    case 0: d = ptx::make_desc(A, 2048, 128); break;
    case 1: d = ptx::make_desc(A, 4096, 128); break;
    case 2: d = ptx::make_desc(A, 128, 4096); break;
    case 3: d = ptx::make_desc(A, 1024, 4096) | ((uint64_t)2 << 61); break;
    case 4: d = ptx::make_desc(A, 4096, 1024) | ((uint64_t)2 << 61); break;
    case 5: d = ptx::make_desc(A, 256, 4096) | ((uint64_t)6 << 61); break;
    case 7: d = ptx::make_desc(A, 16, 1024) | ((uint64_t)2 << 61); break;
    case 8: d = ptx::make_desc(A + 32, 16, 1024) | ((uint64_t)2 << 61); break;
    case 9: d = ptx::make_desc(A, 16, 512) | ((uint64_t)4 << 61); break;
    default: d = ptx::make_desc(A, 512, 4096) | ((uint64_t)4 << 61); break;
  }
  return d;
}

__global__ void probe(int mode, float *D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) ((float *)smem)[i] = 0.f;
  __syncthreads();
  const uint32_t A = ptx::smem_u32(smem), B = A + 32 * 1024;
  float *Af = (float *)smem, *Bf = (float *)(smem + 32 * 1024);
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) {
    const int m = i / 8, k = i % 8;
    Af[a_off(mode, m, k) / 4] = (float)((m * 3 + k * 7) % 11 - 5);
  }
  for (int i = threadIdx.x; i < 16 * 8; i += blockDim.x) {  // B K-major none: [khalf][n][16B]
    const int n = i / 8, k = i % 8;
    Bf[((k / 4) * 16 * 16 + (n / 8) * 128 + (n % 8) * 16 + (k % 4) * 4) / 4] = (float)((n * 5 + k * 3) % 7 - 3);
  }
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc(&tslot, 32);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t idesc = (mode == 0 || mode >= 7) ? ptx::make_idesc_tf32(128, 16) : ptx::make_idesc_tf32_amn(128, 16);
  if (threadIdx.x == 0) {
    ptx::mma_tf32(tmem, a_desc(mode, A), ptx::make_desc(B, 16 * 16, 128), idesc, 0);
    ptx::mma_commit(&bar);
  }
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  float v[16];
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  ptx::tmem_ld16(tmem + ((uint32_t)(w * 32) << 16), v);
  for (int j = 0; j < 16; ++j) D[(w * 32 + l) * 16 + j] = v[j];
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tmem, 32);
}

int main() {
  float *D;
  cudaMalloc(&D, 128 * 16 * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int mode = 0; mode < 10; ++mode) {
    cudaMemset(D, 0, 128 * 16 * 4);
    probe<<<1, 128, 64 * 1024>>>(mode, D);
    cudaError_t e = cudaDeviceSynchronize();
    float h[128 * 16];
    cudaMemcpy(h, D, sizeof(h), cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 16; ++n) {
        double ref = 0;
        for (int k = 0; k < 8; ++k) ref += (double)((m * 3 + k * 7) % 11 - 5) * ((n * 5 + k * 3) % 7 - 3);
        err = fmax(err, fabs(ref - h[m * 16 + n]));
        mx = fmax(mx, fabs(h[m * 16 + n]));
      }
    printf("mode %d: %s max_err %.1f max|D| %.1f\n", mode, cudaGetErrorString(e), err, mx);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
