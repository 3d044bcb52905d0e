// common.cu -- error reporting, device queries and descriptor validation.
#include <stdarg.h>
#include <string.h>

#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "tma.cuh"

namespace sysml {

static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

const char *get_error() { return g_err; }

static thread_local char g_route[512] = "";

void route_reset() { g_route[0] = 0; }

void route_note(const char *fmt, ...) {
  size_t len = strlen(g_route);
  if (len + 4 >= sizeof(g_route)) return;
  if (len) {
    strcpy(g_route + len, " + ");
    len += 3;
  }
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_route + len, sizeof(g_route) - len, fmt, ap);
  va_end(ap);
}

const char *route_get() { return g_route; }

static int query_attr(cudaDeviceAttr a) {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&v, a, dev) != cudaSuccess) return 0;
  return v;
}

sysml_status ensure_smem_attr(const void *func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, size_t> done;  // (kernel, device) -> bytes set
  int dev = 0;
  SYSML_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t &cur = done[{func, dev}];
  if (bytes > cur) {
    SYSML_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    cur = bytes;
  }
  return SYSML_OK;
}

int sm_count() {
  static thread_local int dev_cached = -1, val = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != dev_cached) {
    val = query_attr(cudaDevAttrMultiProcessorCount);
    dev_cached = dev;
  }
  return val > 0 ? val : 148;
}

int device_cc_major() {
  static thread_local int dev_cached = -1, val = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != dev_cached) {
    val = query_attr(cudaDevAttrComputeCapabilityMajor);
    dev_cached = dev;
  }
  return val;
}

sysml_status validate_conv(const sysml_conv_desc *d, ConvGeom *g) {
  SYSML_CHECK_ARG(d != nullptr, "conv descriptor is NULL");
  SYSML_CHECK_ARG(d->N >= 1 && d->C >= 1 && d->H >= 1 && d->W >= 1 && d->K >= 1 && d->R >= 1 &&
                      d->S >= 1,
                  "conv dims must be >= 1 (N=%d C=%d H=%d W=%d K=%d R=%d S=%d)", d->N, d->C,
                  d->H, d->W, d->K, d->R, d->S);
  SYSML_CHECK_ARG(d->stride_h >= 1 && d->stride_w >= 1 && d->pad_h >= 0 && d->pad_w >= 0,
                  "conv stride must be >= 1 and pad >= 0 (stride %dx%d pad %dx%d)", d->stride_h,
                  d->stride_w, d->pad_h, d->pad_w);
  SYSML_CHECK_ARG(d->math == SYSML_MATH_FP32 || d->math == SYSML_MATH_TF32,
                  "conv math must be SYSML_MATH_FP32 (0) or SYSML_MATH_TF32 (1), got %d", d->math);
  g->N = d->N; g->C = d->C; g->H = d->H; g->W = d->W; g->K = d->K; g->R = d->R; g->S = d->S;
  g->sh = d->stride_h; g->sw = d->stride_w; g->ph = d->pad_h; g->pw = d->pad_w;
  g->P = out_extent(g->H, g->ph, g->R, g->sh);
  g->Q = out_extent(g->W, g->pw, g->S, g->sw);
  SYSML_CHECK_SHAPE(g->P >= 1 && g->Q >= 1,
                    "conv output extent < 1: input %lldx%lld, kernel %lldx%lld, pad %lldx%lld",
                    (long long)g->H, (long long)g->W, (long long)g->R, (long long)g->S,
                    (long long)g->ph, (long long)g->pw);
  SYSML_CHECK_SHAPE(g->N * g->CHW() < (1ll << 31) && g->N * g->KPQ() < (1ll << 31) &&
                        g->K * g->CRS() < (1ll << 31),
                    "tensor with >= 2^31 elements is unsupported (N x CHW = %lld, N x KPQ = %lld)",
                    (long long)(g->N * g->CHW()), (long long)(g->N * g->KPQ()));
  return SYSML_OK;
}

sysml_status validate_input(const sysml_input *x, const ConvGeom &g) {
  SYSML_CHECK_ARG(x != nullptr, "input is NULL");
  if (!x->is_csr) {
    SYSML_CHECK_ARG(x->dense != nullptr, "dense input pointer is NULL");
    SYSML_CHECK_ALIGN16(x->dense, "dense input");
    return SYSML_OK;
  }
  const sysml_csr &m = x->csr;
  SYSML_CHECK_ARG(m.row_ptr && (m.nnz == 0 || (m.col_idx && m.val)), "CSR arrays are NULL");
  SYSML_CHECK_ALIGN(m.row_ptr, 4, "CSR row_ptr");
  SYSML_CHECK_ALIGN(m.col_idx, 4, "CSR col_idx");
  SYSML_CHECK_ALIGN(m.val, 4, "CSR val");
  SYSML_CHECK_SHAPE(m.rows == g.N && m.cols == g.CHW(),
                    "CSR shape %lldx%lld does not match input N x (C*H*W) = %lldx%lld",
                    (long long)m.rows, (long long)m.cols, (long long)g.N, (long long)g.CHW());
  SYSML_CHECK_SHAPE(m.nnz >= 0 && m.nnz < (1ll << 31), "CSR nnz %lld out of range",
                    (long long)m.nnz);
  return SYSML_OK;
}

sysml_status validate_pool(const sysml_pool_desc *d, ConvGeom *g) {
  SYSML_CHECK_ARG(d != nullptr, "pool descriptor is NULL");
  SYSML_CHECK_ARG(d->N >= 1 && d->C >= 1 && d->H >= 1 && d->W >= 1 && d->R >= 1 && d->S >= 1,
                  "pool dims must be >= 1 (N=%d C=%d H=%d W=%d R=%d S=%d)", d->N, d->C, d->H,
                  d->W, d->R, d->S);
  SYSML_CHECK_ARG(d->stride_h >= 1 && d->stride_w >= 1 && d->pad_h >= 0 && d->pad_w >= 0,
                  "pool stride must be >= 1 and pad >= 0");
  SYSML_CHECK_SHAPE(d->pad_h < d->R && d->pad_w < d->S,
                    "pool pad (%d,%d) must be smaller than the window (%d,%d)", d->pad_h,
                    d->pad_w, d->R, d->S);
  g->N = d->N; g->C = d->C; g->H = d->H; g->W = d->W; g->K = d->C; g->R = d->R; g->S = d->S;
  g->sh = d->stride_h; g->sw = d->stride_w; g->ph = d->pad_h; g->pw = d->pad_w;
  g->P = out_extent(g->H, g->ph, g->R, g->sh);
  g->Q = out_extent(g->W, g->pw, g->S, g->sw);
  SYSML_CHECK_SHAPE(g->P >= 1 && g->Q >= 1, "pool output extent < 1 (input %dx%d window %dx%d)",
                    d->H, d->W, d->R, d->S);
  SYSML_CHECK_SHAPE(g->N * g->CHW() < (1ll << 31), "pool tensor with >= 2^31 elements");
  return SYSML_OK;
}

}  // namespace sysml

namespace sysml {

bool tmap_encode_f32(CUtensorMap *map, const void *base, int rank, const uint64_t *dims,
                     const uint64_t *strides_bytes, const uint32_t *box,
                     CUtensorMapSwizzle swizzle) {
  typedef CUresult (*encode_fn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static encode_fn fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p) {
      set_error("cuTensorMapEncodeTiled is not available from the driver");
      return false;
    }
    fn = reinterpret_cast<encode_fn>(p);
  }
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = 1;
    if (i + 1 < rank) st[i] = strides_bytes[i];
  }
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, const_cast<void *>(base),
                        d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
    return false;
  }
  return true;
}

}  // namespace sysml
