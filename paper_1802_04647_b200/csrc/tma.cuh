// tma.cuh -- tensor-map (TMA) support for sm_100a: host-side encoding through the
// driver entry point (libsysml links no libcuda) and the device-side tiled bulk
// tensor copy into shared memory with mbarrier completion.
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "common.cuh"

namespace sysml {

// Encode a tiled fp32 tensor map.  dims[0] is the contiguous dimension;
// strides_bytes[i] is the byte stride of dims[i + 1] (multiples of 16).  Returns
// false (with the error set) if the driver rejects the description.
bool tmap_encode_f32(CUtensorMap *map, const void *base, int rank, const uint64_t *dims,
                     const uint64_t *strides_bytes, const uint32_t *box,
                     CUtensorMapSwizzle swizzle);

namespace ptx {

__device__ __forceinline__ void tma_load_3d(uint32_t dst_smem, const CUtensorMap *map, int c0,
                                            int c1, int c2, uint32_t bar_smem) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst_smem),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar_smem)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst_smem, const CUtensorMap *map, int c0,
                                            int c1, uint32_t bar_smem) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(dst_smem),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_smem)
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

}  // namespace ptx
}  // namespace sysml
