// mma_tmemA.cu -- tcgen05.mma kind::tf32 with A in TMEM (written by tcgen05.st): checks the
// layout (lane = row m, columns = K) against a CPU product and measures clocks per MMA by N.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include "../paper_1802_04647_b200/csrc/tc_ptx.cuh"
using namespace sysml;

__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a_tmem), "l"(bdesc),
               "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
               "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
               : "memory");
}

// A: 128 x 8 (row m, k), B: N x 8 (row n, k), D = A B^T (128 x N).  K-step 8 = one MMA.
__global__ void check(const float *A, const float *B, float *D, int N, int reps, unsigned long long *clk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // B in smem, K-major no swizzle: [quad][n][4]
  float *Bs = reinterpret_cast<float *>(smem);
  for (int i = threadIdx.x; i < N * 8; i += blockDim.x) {
    const int n = i / 8, k = i % 8;
    Bs[(k / 4) * N * 4 + n * 4 + (k % 4)] = B[i];
  }
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(&tslot, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  // A into TMEM columns [256, 264): thread (warp w, lane t) -> lane 32w+t, 8 columns
  {
    const int m = warp * 32 + lane;
    float v[8];
    for (int k = 0; k < 8; ++k) v[k] = A[m * 8 + k];
    tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + 256, v);
    ptx::tmem_st_wait();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t idesc = ptx::make_idesc_tf32(128, N);
  const uint64_t bdesc = ptx::make_desc(ptx::smem_u32(Bs), N * 16, 128);
  if (warp == 0) {
    unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (ptx::elect_one()) mma_tf32_ts(tmem, tmem + 256, bdesc, idesc, r == 0 ? 0u : 1u);
      __syncwarp();
    }
    if (ptx::elect_one()) ptx::mma_commit(&bar);
    __syncwarp();
    ptx::mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (lane == 0) *clk = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  {
    const int m = warp * 32 + lane;
    for (int c = 0; c < N; c += 16) {
      float v[16];
      ptx::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
      for (int j = 0; j < 16; ++j) D[m * N + c + j] = v[j];
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

int main() {
  for (int N : {32, 64, 80, 96, 160, 256}) {
    std::vector<float> A(128 * 8), B(N * 8), D(128 * N);
    for (int i = 0; i < 128 * 8; ++i) A[i] = (float)((i * 37) % 17 - 8) / 8.0f;
    for (int i = 0; i < N * 8; ++i) B[i] = (float)((i * 53) % 13 - 6) / 4.0f;
    float *dA, *dB, *dD; unsigned long long *dclk, clk;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dclk, 8);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(check, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int reps = 1;
    check<<<1, 128, 64 * 1024>>>(dA, dB, dD, N, reps, dclk);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("N=%d: CUDA error %s\n", N, cudaGetErrorString(cudaGetLastError())); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < 8; ++k) ref += (double)A[m * 8 + k] * B[n * 8 + k];
        maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
      }
    // rate: many reps on 148 CTAs
    check<<<148, 128, 64 * 1024>>>(dA, dB, dD, N, 4000, dclk);
    cudaDeviceSynchronize();
    cudaMemcpy(&clk, dclk, 8, cudaMemcpyDeviceToHost);
    printf("A-in-TMEM tf32 N=%3d: max|err| %.3g  %.1f clk/mma (ideal %.1f)\n", N, maxerr, clk / 4000.0, 128.0 * N * 8 / 2048);
    cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dclk);
  }
  return 0;
}
