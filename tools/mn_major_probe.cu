// mn_major_probe.cu -- does tcgen05.mma accept MN-major (transposed) TF32 operands on sm_100a?
// (round 1's tools/mma_layout_test.cu saw zeros.)  One CTA builds A (128 x K)
// and B (16 x K) in shared memory in a chosen canonical layout (cute::UMMA make_umma_desc<MN>
// forms, mma_traits_sm100.hpp:171-175), issues ONE MMA, and compares D with a host reference.
// A bf16 run of the same MN-major layouts is the control: CUTLASS uses MN-major bf16 routinely,
// so if bf16 passes and tf32 does not, the limitation is the hardware / ISA, not the probe.
//
// MN-major canonical layouts, element (mn, k), T = 16 / sizeof(elem) elements per 16 B:
//   INTERLEAVE: byte = (mn%T)*e + (k%8)*16 + (mn/T)*SBO + (k/8)*LBO
//   SW{32,64,128}: atom = W bytes of MN (W/e elements) x 8 K-rows; byte inside the atom
//     lin = (k%8)*W + (mn%(W/e))*e, swizzled lin ^ (((lin >> 7) & (W/16 - 1)) << 4);
//     MN atoms LBO apart, 8-row K groups SBO apart.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/mn_major_probe.cu -o /tmp/mnp
#include <cmath>
#include <cstdint>
#include <cstdio>

#include "../paper_1802_04647_b200/csrc/tc_ptx.cuh"
using namespace sysml;

__device__ __host__ inline float aval(int m, int k) { return (float)((m * 3 + k * 7) % 11 - 5); }
__device__ __host__ inline float bval(int n, int k) { return (float)((n * 5 + k * 3) % 7 - 3); }

// layout: 0 K-major INTERLEAVE (reference), 1 MN INTERLEAVE, 2 MN SW32, 3 MN SW64, 4 MN SW128
__device__ uint32_t off_mn(int layout, int esz, int mn, int k, int MNext, uint32_t *lbo, uint32_t *sbo) {
  const int T = 16 / esz;
  if (layout == 0) {  // K-major interleave: rows of 16 B (T k), 8-row core matrices
    *lbo = (uint32_t)(MNext * 16);  // next T-wide K chunk
    *sbo = 128;                     // next 8-row group
    return (uint32_t)((k / T) * MNext * 16 + (mn / 8) * 128 + (mn % 8) * 16 + (k % T) * esz);
  }
  if (layout == 1) {
    *sbo = 128;                          // next T-element MN group (8 K-rows of 16 B)
    *lbo = (uint32_t)(MNext / T) * 128;  // next 8-row K group
    return (uint32_t)((mn % T) * esz + (k % 8) * 16 + (mn / T) * 128 + (k / 8) * (*lbo));
  }
  const int W = layout == 2 ? 32 : layout == 3 ? 64 : 128;
  const int per = W / esz;              // MN elements per atom row
  *lbo = (uint32_t)(W * 8);             // next MN atom
  *sbo = (uint32_t)((MNext / per) * W * 8);  // next 8-row K group
  const uint32_t lin = (uint32_t)((k % 8) * W + (mn % per) * esz);
  const uint32_t sw = lin ^ (((lin >> 7) & (uint32_t)(W / 16 - 1)) << 4);
  return (uint32_t)((mn / per) * W * 8) + (uint32_t)((k / 8) * (*sbo)) + sw;
}

__device__ uint64_t desc_for(uint32_t addr, int layout, uint32_t lbo, uint32_t sbo, int swap) {
  uint64_t d = ptx::make_desc(addr, swap ? sbo : lbo, swap ? lbo : sbo);
  const uint64_t lt = layout == 2 ? 6 : layout == 3 ? 4 : layout == 4 ? 2 : 0;  // SW32=6, SW64=4, SW128=2
  return d | (lt << 61);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc)
      : "memory");
}

// la / lb: layouts of A / B; bf16: kind::f16 with bf16 operands (K = 16) else kind::tf32 (K = 8)
__global__ void probe(int la, int lb, int bf16, int swap, float *D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int esz = bf16 ? 2 : 4, K = bf16 ? 16 : 8, M = 128, N = 16;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((float *)smem)[i] = 0.f;
  __syncthreads();
  uint8_t *As = smem, *Bs = smem + 32 * 1024;
  uint32_t alb = 0, asb = 0, blb = 0, bsb = 0;
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    const uint32_t o = off_mn(la, esz, m, k, M, &alb, &asb);
    if (bf16) ((__nv_bfloat16_raw *)(As + o))->x = (unsigned short)(__float_as_uint(aval(m, k)) >> 16);
    else *(float *)(As + o) = aval(m, k);
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    const uint32_t o = off_mn(lb, esz, n, k, N, &blb, &bsb);
    if (bf16) ((__nv_bfloat16_raw *)(Bs + o))->x = (unsigned short)(__float_as_uint(bval(n, k)) >> 16);
    else *(float *)(Bs + o) = bval(n, k);
  }
  // every thread computed the same strides; thread 0's are used below
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc(&tslot, 32);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    off_mn(la, esz, 0, 0, M, &alb, &asb);
    off_mn(lb, esz, 0, 0, N, &blb, &bsb);
    const uint64_t ad = desc_for(ptx::smem_u32(As), la, alb, asb, swap && la);
    const uint64_t bd = desc_for(ptx::smem_u32(Bs), lb, blb, bsb, swap && lb);
    uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    idesc |= bf16 ? ((1u << 7) | (1u << 10)) : ((2u << 7) | (2u << 10));
    if (la) idesc |= 1u << 15;
    if (lb) idesc |= 1u << 16;
    if (bf16) mma_f16(tmem, ad, bd, idesc);
    else ptx::mma_tf32(tmem, ad, bd, idesc, 0);
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
  const char *names[] = {"Kmaj", "MN-INTER", "MN-SW32", "MN-SW64", "MN-SW128"};
  for (int bf16 = 1; bf16 >= 0; --bf16)
    for (int which = 0; which < 2; ++which)      // 0: A varies (B K-major), 1: B varies (A K-major)
      for (int lay = 0; lay < 5; ++lay)
        for (int swap = 0; swap < (lay ? 2 : 1); ++swap) {
          const int la = which == 0 ? lay : 0, lb = which == 1 ? lay : 0;
          cudaMemset(D, 0, 128 * 16 * 4);
          probe<<<1, 128, 64 * 1024>>>(la, lb, bf16, swap, D);
          cudaError_t e = cudaDeviceSynchronize();
          float h[128 * 16];
          cudaMemcpy(h, D, sizeof(h), cudaMemcpyDeviceToHost);
          const int K = bf16 ? 16 : 8;
          double err = 0, mx = 0;
          for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 16; ++n) {
              double ref = 0;
              for (int k = 0; k < K; ++k) ref += (double)aval(m, k) * bval(n, k);
              err = fmax(err, fabs(ref - h[m * 16 + n]));
              mx = fmax(mx, fabs(h[m * 16 + n]));
            }
          printf("%s %s=%-8s swap=%d: %s max_err %.1f max|D| %.1f %s\n", bf16 ? "bf16" : "tf32", which ? "B" : "A",
                 names[lay], swap, cudaGetErrorString(e), err, mx, err == 0 ? "OK" : "");
          if (e != cudaSuccess) return 1;
        }
  return 0;
}
