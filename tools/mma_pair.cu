// mma_pair.cu -- tcgen05.mma.cta_group::2 kind::tf32 with A in TMEM (each CTA of the pair holds
// its 128 rows) and B split by N (each CTA holds N/2 rows of B at the same smem offset):
// checks D (each CTA reads its 128 rows x N columns) against a CPU product, and clocks/MMA.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include "../paper_1802_04647_b200/csrc/tc_ptx.cuh"
using namespace sysml;

__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a_tmem), "l"(bdesc),
               "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit2_mc(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(ptx::smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
               "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
               : "memory");
}
__device__ __forceinline__ void remote_arrive(uint64_t *bar, uint32_t rank) {
  uint32_t la = ptx::smem_u32(bar), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ bool try_wait_cluster(uint64_t *bar, uint32_t parity) {
  uint32_t done;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(ptx::smem_u32(bar)), "r"(parity) : "memory");
  return done != 0;
}

// A: 256 x 8 (rows 0-127 in CTA 0, 128-255 in CTA 1), B: N x 8 (rows [0,N/2) in CTA 0, [N/2,N) in CTA 1)
__global__ void __cluster_dims__(2, 1, 1) check(const float *A, const float *B, float *D, int N, int reps,
                                                unsigned long long *clk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t ready, done;
  __shared__ uint32_t tslot;
  const uint32_t rank = ptx::cluster_ctarank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NH = N / 2;
  float *Bs = reinterpret_cast<float *>(smem);  // [quad][NH][4]
  for (int i = threadIdx.x; i < NH * 8; i += blockDim.x) {
    const int n = i / 8, k = i % 8;
    Bs[(k / 4) * NH * 4 + n * 4 + (k % 4)] = B[(rank * NH + n) * 8 + k];
  }
  if (threadIdx.x == 0) {
    ptx::mbar_init(&ready, 2 * 128);  // both CTAs' 128 threads (leader's barrier)
    ptx::mbar_init(&done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(&tslot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  {  // A rows of this CTA into TMEM columns [256, 264)
    const int m = warp * 32 + lane;
    float v[8];
    for (int k = 0; k < 8; ++k) v[k] = A[(rank * 128 + m) * 8 + k];
    tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + 256, v);
    ptx::tmem_st_wait();
    ptx::tc_fence_before();
    remote_arrive(&ready, 0);  // arrive on the leader's barrier (also for the leader itself)
  }
  if (rank == 0 && warp == 0) {
    while (!try_wait_cluster(&ready, 0)) {}
    ptx::tc_fence_after();
    const uint32_t idesc = ptx::make_idesc_tf32(256, N);
    const uint64_t bdesc = ptx::make_desc(ptx::smem_u32(Bs), NH * 16, 128);
    unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (ptx::elect_one()) mma2_ts(tmem, tmem + 256, bdesc, idesc, r == 0 ? 0u : 1u);
      __syncwarp();
    }
    if (ptx::elect_one()) commit2_mc(&done);
    __syncwarp();
    while (!ptx::mbar_try_wait(&done, 0)) {}
    if (lane == 0) *clk = clock64() - t0;
  }
  // every CTA waits for its own copy of `done` (multicast commit)
  while (!ptx::mbar_try_wait(&done, 0)) {}
  ptx::tc_fence_after();
  {
    const int m = warp * 32 + lane;
    for (int c = 0; c < N; c += 16) {
      float v[16];
      ptx::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
      for (int j = 0; j < 16; ++j) D[(rank * 128 + m) * N + c + j] = v[j];
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  if (warp == 0) {
    ptx::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

int main() {
  for (int N : {64, 160, 256}) {
    std::vector<float> A(256 * 8), B(N * 8), D(256 * N);
    for (int i = 0; i < 256 * 8; ++i) A[i] = (float)((i * 37) % 17 - 8) / 8.0f;
    for (int i = 0; i < N * 8; ++i) B[i] = (float)((i * 53) % 13 - 6) / 4.0f;
    float *dA, *dB, *dD; unsigned long long *dclk, clk = 0;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dclk, 8);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(check, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    check<<<2, 128, 64 * 1024>>>(dA, dB, dD, N, 1, dclk);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("N=%d: CUDA error %s\n", N, cudaGetErrorString(cudaGetLastError())); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < 256; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < 8; ++k) ref += (double)A[m * 8 + k] * B[n * 8 + k];
        maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
      }
    check<<<148, 128, 64 * 1024>>>(dA, dB, dD, N, 4000, dclk);
    cudaDeviceSynchronize();
    cudaMemcpy(&clk, dclk, 8, cudaMemcpyDeviceToHost);
    printf("pair tf32 A-in-TMEM N=%3d: max|err| %.3g  %.1f clk/mma (M=256; ideal per SM %.1f)\n", N, maxerr, clk / 4000.0,
           128.0 * N * 8 / 2048);
  }
  return 0;
}
