// common.cuh -- shared host/device helpers of libsysml (product path only).
// No code here is shared with the oracle (oracle/oracle.c).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/sysml.h"

namespace sysml {

// Thread-local route log (sysml_last_route): the main kernels the last dispatch launched,
// so a bench line or test can report which implementation an op took.
void route_reset();
void route_note(const char *fmt, ...) __attribute__((format(printf, 1, 2)));
const char *route_get();

// Thread-local last error message (sysml_last_error).
void set_error(const char *fmt, ...) __attribute__((format(printf, 1, 2)));
const char *get_error();

#define SYSML_CHECK_ARG(cond, ...)   \
  do {                               \
    if (!(cond)) {                   \
      ::sysml::set_error(__VA_ARGS__); \
      return SYSML_ERR_ARG;          \
    }                                \
  } while (0)

#define SYSML_CHECK_SHAPE(cond, ...) \
  do {                               \
    if (!(cond)) {                   \
      ::sysml::set_error(__VA_ARGS__); \
      return SYSML_ERR_SHAPE;        \
    }                                \
  } while (0)

// sysml.h "Conventions": dense tensors and workspaces are 16-byte aligned (the kernels move
// them with 16-byte vector, cp.async and bulk/TMA copies); int32 index arrays (CSR, labels)
// need their natural 4-byte alignment.  A view that breaks this is rejected, not faulted on.
#define SYSML_CHECK_ALIGN(ptr, bytes, name)                                                   \
  do {                                                                                        \
    if ((ptr) != nullptr && ((uintptr_t)(ptr) & ((bytes) - 1)) != 0) {                        \
      ::sysml::set_error("%s pointer %p is not %d-byte aligned", name, (const void *)(ptr),    \
                         (int)(bytes));                                                       \
      return SYSML_ERR_UNSUPPORTED;                                                          \
    }                                                                                         \
  } while (0)
#define SYSML_CHECK_ALIGN16(ptr, name) SYSML_CHECK_ALIGN(ptr, 16, name)

#define SYSML_CUDA(call)                                                           \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      ::sysml::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(e_),        \
                         __FILE__, __LINE__, cudaGetErrorString(e_));              \
      return SYSML_ERR_CUDA;                                                       \
    }                                                                              \
  } while (0)

extern thread_local int64_t g_launches;  // kernels launched by this thread (api.cu)

// After a kernel launch: count it and report launch-configuration errors.
#define SYSML_LAUNCH_CHECK()               \
  do {                                     \
    ++::sysml::g_launches;                 \
    SYSML_CUDA(cudaPeekAtLastError());     \
  } while (0)

#define SYSML_TRY(expr)                     \
  do {                                      \
    sysml_status s_ = (expr);               \
    if (s_ != SYSML_OK) return s_;          \
  } while (0)

inline int64_t out_extent(int64_t in, int64_t pad, int64_t k, int64_t stride) {
  int64_t num = in + 2 * pad - k;
  if (num < 0 || stride <= 0) return 0;
  return num / stride + 1;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t a, size_t b) { return (a + b - 1) / b * b; }

int sm_count();              // cached per device

// Opt `func` (a __global__ function) into `bytes` of dynamic shared memory on the CURRENT
// device.  The attribute is per device, so the cache is keyed by (function, device) and
// guarded by a mutex (reentrant, multi-GPU processes).
sysml_status ensure_smem_attr(const void *func, size_t bytes);
template <class K>
inline sysml_status smem_attr(K *kernel, size_t bytes) {
  return ensure_smem_attr(reinterpret_cast<const void *>(kernel), bytes);
}
int device_cc_major();       // cached per device

// Derived geometry of a conv descriptor.
struct ConvGeom {
  int64_t N, C, H, W, K, R, S, sh, sw, ph, pw, P, Q;
  int64_t CHW() const { return C * H * W; }
  int64_t CRS() const { return C * R * S; }
  int64_t KPQ() const { return K * P * Q; }
  int64_t PQ() const { return P * Q; }
  int64_t HW() const { return H * W; }
};

sysml_status validate_conv(const sysml_conv_desc *d, ConvGeom *g);
sysml_status validate_input(const sysml_input *x, const ConvGeom &g);
sysml_status validate_pool(const sysml_pool_desc *d, ConvGeom *g /* R,S,sh,... P,Q; K unused */);

// Simple bump allocator over a caller workspace.
struct WsCarve {
  char *base;
  size_t size, off = 0;
  WsCarve(void *b, size_t s) : base((char *)b), size(s) {}
  template <class T>
  T *take(size_t count) {
    off = align_up(off, 256);
    T *p = (T *)(base ? base + off : nullptr);
    off += count * sizeof(T);
    return p;
  }
  size_t used() const { return align_up(off, 256); }
  // false once the carved regions run past the declared size (a sizing/dispatch mismatch)
  bool fits() const { return off <= size; }
};

// Carve check: every internal path that carves a caller workspace is given the size its
// own *_ws() function declared and must stay inside it (sizing and dispatch
// disagreed once and the kernel wrote past the caller's buffer).
#define SYSML_WS_FITS(wc)                                                                  \
  do {                                                                                     \
    if (!(wc).fits()) {                                                                    \
      ::sysml::set_error("internal: workspace carve %zu bytes exceeds declared %zu at %s:%d", \
                         (wc).off, (wc).size, __FILE__, __LINE__);                          \
      return SYSML_ERR_WORKSPACE;                                                          \
    }                                                                                      \
  } while (0)

}  // namespace sysml
