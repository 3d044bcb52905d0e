// mma_snstream.cu -- the MMA stream of sn_tmem_kernel without producers or epilogue: M = 128,
// N = NN, K = 8 TF32 MMAs with A in TMEM (one of 4 stages x R copies), B walking a resident
// filter bank of nb blocks in shared memory, D alternating between two accumulators every
// tile of nchunk * R MMAs.  Prints clocks per MMA next to the math rate (128 * N * 8 / 2048).
// usage: mma_snstream [NN=160] [bank_kb=200] [commit_every=5] [flags]
//   flags: 1 = A fixed, 2 = B fixed, 4 = D fixed, 8 = A from shared memory (SS form),
//          16 = one elected lane issues the 5 MMAs of a chunk in one unrolled block,
//          32 = one elected lane runs a runtime-count loop over the chunk's MMAs
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../paper_1802_04647_b200/csrc/tc_ptx.cuh"
using namespace sysml;

__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a_tmem), "l"(bdesc),
               "r"(idesc), "r"(acc) : "memory");
}

__global__ void stream(int NN, int nblocks, int commit_every, int nmma, int flags, int nrt, unsigned long long *clk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < nblocks * NN * 8; i += blockDim.x) reinterpret_cast<float *>(smem)[i] = 0.25f;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(&tslot, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t acol = (uint32_t)((2 * NN + 31) / 32 * 32);
  const uint32_t idesc = ptx::make_idesc_tf32(128, NN);
  const uint64_t b0 = ptx::make_desc(ptx::smem_u32(smem), NN * 16, 128);
  const uint64_t bstep = (uint64_t)((2u * NN * 16u) >> 4);
  if (warp == 0) {
    unsigned long long t0 = clock64();
    uint64_t bd = b0;
    int blk = 0;
    const int per_tile = 40;
    if (flags & 16) {
      for (int i = 0; i < nmma; i += 5) {
        const int tile = i / per_tile, in = i % per_tile;
        const uint32_t d = tmem + (uint32_t)(tile & 1) * NN;
        const uint32_t a = tmem + acol + (uint32_t)(((i / 5) & 3) * 40);
        if (ptx::elect_one()) {
          if (flags & 32) {
            for (int j = 0; j < nrt; ++j) {
              if (flags & 8) {
                const uint64_t ad = ptx::make_desc(ptx::smem_u32(smem) + (uint32_t)j * 4096u, 128 * 16, 128);
                ptx::mma_tf32(d, ad, bd + (uint64_t)j * bstep, idesc, (in == 0 && j == 0) ? 0u : 1u);
              } else {
                mma_tf32_ts(d, a + 8 * j, bd + (uint64_t)j * bstep, idesc, (in == 0 && j == 0) ? 0u : 1u);
              }
            }
          } else if (flags & 8) {
#pragma unroll
            for (int j = 0; j < 5; ++j) {
              const uint64_t ad = ptx::make_desc(ptx::smem_u32(smem) + (uint32_t)j * 4096u, 128 * 16, 128);
              ptx::mma_tf32(d, ad, bd + (uint64_t)j * bstep, idesc, (in == 0 && j == 0) ? 0u : 1u);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 5; ++j)
              mma_tf32_ts(d, a + 8 * j, bd + (uint64_t)j * bstep, idesc, (in == 0 && j == 0) ? 0u : 1u);
          }
          if (commit_every > 0) ptx::mma_commit(&bar);
        }
        __syncwarp();
        blk += 5;
        if (blk >= nblocks) { blk = 0; bd = b0; } else bd += 5 * bstep;
      }
    } else
    for (int i = 0; i < nmma; ++i) {
      const int tile = i / per_tile, in = i % per_tile;
      const uint32_t d = tmem + ((flags & 4) ? 0u : (uint32_t)(tile & 1) * NN);
      const uint32_t aoff = (flags & 1) ? 0u : (uint32_t)(((i / 5) & 3) * 40 + (i % 5) * 8);
      const uint64_t bb = (flags & 2) ? b0 : bd;
      if (flags & 8) {
        // A from shared memory: 128 rows x 8 k, K-major no swizzle, in the first 4 KB x 20 slots
        const uint64_t ad = ptx::make_desc(ptx::smem_u32(smem) + aoff / 8 * 4096u % (16 * 4096u), 128 * 16, 128);
        if (ptx::elect_one()) ptx::mma_tf32(d, ad, bb, idesc, in == 0 ? 0u : 1u);
      } else if (ptx::elect_one()) {
        mma_tf32_ts(d, tmem + acol + aoff, bb, idesc, in == 0 ? 0u : 1u);
      }
      __syncwarp();
      if (commit_every > 0 && (i + 1) % commit_every == 0) {
        if (ptx::elect_one()) ptx::mma_commit(&bar);
        __syncwarp();
      }
      if (++blk == nblocks) { blk = 0; bd = b0; } else bd += bstep;
    }
    if (ptx::elect_one()) ptx::mma_commit(&bar);
    __syncwarp();
    // wait for the last commit: phases alternate, so poll until every MMA has drained
    ptx::tc_fence_before();
    unsigned long long t1;
    {
      // a final fresh barrier round-trip
      __shared__ uint64_t bar2;
      if (threadIdx.x == 0) { ptx::mbar_init(&bar2, 1); ptx::fence_mbar_init(); }
      __syncwarp();
      if (ptx::elect_one()) ptx::mma_commit(&bar2);
      __syncwarp();
      ptx::mbar_wait(&bar2, 0);
      t1 = clock64();
    }
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

int main(int argc, char **argv) {
  const int NN = argc > 1 ? atoi(argv[1]) : 160;
  const int bank_kb = argc > 2 ? atoi(argv[2]) : 200;
  const int commit_every = argc > 3 ? atoi(argv[3]) : 5;
  const int flags = argc > 4 ? atoi(argv[4]) : 0;
  const int nblocks = bank_kb * 1024 / (NN * 32);
  const int smem = nblocks * NN * 32;
  unsigned long long *dclk;
  cudaMalloc(&dclk, 148 * 8);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int nmma = 40 * 200;
  stream<<<148, 128, smem>>>(NN, nblocks, commit_every, nmma, flags, 5, dclk);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
  unsigned long long h[148];
  cudaMemcpy(h, dclk, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += (double)h[i];
  printf("NN=%d bank %d KB (%d blocks) commit every %d flags %d: %.1f clk/mma (math %.1f)\n", NN, bank_kb, nblocks,
         commit_every, flags, s / 148 / nmma, 128.0 * NN * 8 / 2048);
  return 0;
}
