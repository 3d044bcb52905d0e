// tma_box_probe.cu -- which tiled TMA boxes over a [N][28][28] fp32 tensor are legal on sm_100a:
// box larger than the tensor's extent, negative start coordinates (out-of-bounds zero fill).
// usage: tma_box_probe bx by cx cy   (prints the 32x? tile's corner values or dies)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__global__ void probe(const __grid_constant__ CUtensorMap tm, int cx, int cy, int bytes, float *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(bytes));
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"((uint64_t)&tm), "r"(cx), "r"(cy), "r"(1), "r"(b) : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(b));
    for (int i = 0; i < bytes / 4; ++i) out[i] = reinterpret_cast<float *>(smem)[i];
  }
}

int main(int argc, char **argv) {
  const int bx = atoi(argv[1]), by = atoi(argv[2]), cx = atoi(argv[3]), cy = atoi(argv[4]);
  float *x, *out;
  cudaMalloc(&x, 4 * 784 * 4);
  cudaMalloc(&out, 64 * 64 * 4);
  float h[4 * 784];
  for (int i = 0; i < 4 * 784; ++i) h[i] = 1.0f + i;
  cudaMemcpy(x, h, sizeof(h), cudaMemcpyHostToDevice);
  typedef CUresult (*encode_fn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t d[3] = {28, 28, 4}, st[2] = {112, 3136};
  cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1}, es[3] = {1, 1, 1};
  CUresult r = ((encode_fn)p)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("box %dx%d at (%d,%d): encode %d", bx, by, cx, cy, (int)r);
  const int bytes = bx * by * 4;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<<<1, 32, 64 * 1024>>>(tm, cx, cy, bytes, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf(" -> %s\n", cudaGetErrorString(e)); return 1; }
  float o[64 * 64];
  cudaMemcpy(o, out, bytes, cudaMemcpyDeviceToHost);
  printf(" -> ok: [0][0]=%g [2][2]=%g [2][29]=%g (x[1][0][0]=%g)\n", o[0], o[2 * bx + 2], by > 2 && bx > 29 ? o[2 * bx + 29] : -1.f, h[784]);
  return 0;
}
