// csr_dev.cuh -- deterministic CSR row scatter used by the kernels that densify one CSR row
// (one image) into shared or global memory (product path only).
//
// Reading R15: the kernels accept unsorted rows and duplicate
// columns, and duplicates are summed.  The sum must not depend on scheduling (sysml.h:
// "bitwise run-to-run reproducible ... no floating-point atomics"), so:
//   * a strictly increasing row (the S:31-32 contract, every well-formed input) has exactly
//     one writer per destination slot -- the threads store in parallel;
//   * any other row is accumulated by thread 0 in stored order.
// The test for "strictly increasing" is itself parallel (each entry against its
// predecessor) and is combined with a barrier reduction (`bar_or`).
#pragma once

#include <stdint.h>

namespace sysml {

// OR-reduce a predicate over the threads of named barrier `id` (nthreads threads).
__device__ __forceinline__ bool named_bar_or(int id, int nthreads, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "bar.red.or.pred q, %2, %3, p;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)pred), "r"(id), "r"(nthreads)
      : "memory");
  return r != 0;
}

// Scatter entries [j0, j1) of a CSR row: dst(col) returns the destination slot of column
// `col` (nullptr to skip it); the slot holds 0 beforehand.  bar_or(pred) must be a barrier
// over exactly the threads tid in [0, nthr) that returns the OR of pred.  The caller
// synchronises again before reading the slots.
template <class Dst, class BarOr>
__device__ __forceinline__ void csr_scatter_row(const int32_t *__restrict__ col_idx,
                                                const float *__restrict__ val, int j0, int j1, int tid,
                                                int nthr, Dst dst, BarOr bar_or) {
  bool bad = false;
  for (int j = j0 + tid; j < j1; j += nthr)
    if (j > j0 && __ldg(col_idx + j - 1) >= __ldg(col_idx + j)) bad = true;
  if (!bar_or(bad)) {
    for (int j = j0 + tid; j < j1; j += nthr) {
      float *d = dst(__ldg(col_idx + j));
      if (d) *d = __ldg(val + j);
    }
  } else if (tid == 0) {
    for (int j = j0; j < j1; ++j) {
      float *d = dst(__ldg(col_idx + j));
      if (d) *d += __ldg(val + j);
    }
  }
}

}  // namespace sysml
