/*
 * sysml.h -- C ABI of the B200-native conv2d-family hot path of arXiv 1802.04647
 * ("Deep Learning with Apache SystemML"; the paper's GPU backend, §3).
 *
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n (reference text).
 *
 * Tensor encoding: a tensor [N, C, H, W] is the row-major matrix
 * N x (C*H*W); element (n,c,h,w) is at  n*(C*H*W) + (c*H + h)*W + w.
 * All floating point data is IEEE fp32; all index data is int32.
 *
 * Conventions common to every entry point
 * ---------------------------------------
 *  * Pointers named x, f, bias, y, dy, dx, df, db, out, argmax, workspace, params,
 *    grads, labels and the sysml_csr arrays are DEVICE pointers (cudaMalloc /
 *    torch CUDA tensors) on the current CUDA device.  fp32 tensors, argmax
 *    outputs and workspaces must be 16-byte aligned; int32 index arrays (the
 *    sysml_csr arrays, labels, pred) and the loss scalar need 4-byte alignment.
 *    A pointer that breaks this returns SYSML_ERR_UNSUPPORTED (nothing is
 *    launched).  The caller owns every buffer; the library never frees them.
 *  * Outputs are fully overwritten (never accumulated into), except
 *    sysml_bias_add, which updates y in place.  Inputs are not modified and
 *    must not alias outputs.
 *  * Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *    default stream), does not allocate device memory, does not synchronize,
 *    and is CUDA-graph capturable.  Scratch memory is the caller's
 *    `workspace` of at least the size the matching *_workspace_size query
 *    returns.
 *  * Results are bitwise run-to-run reproducible for fixed inputs, device and
 *    math mode (no floating-point atomics; split reductions are summed in a
 *    fixed order; duplicate CSR columns are summed in stored order).
 *  * Errors: a non-zero sysml_status; sysml_last_error() returns a
 *    thread-local message naming the offending argument / both shapes
 *    ("shape error naming both shapes").  Nothing is launched on error.
 *    There is no CPU fallback (BJ north_star).
 *  * Output extents use the floor reading (reading R2):
 *        P = floor((H + 2*pad_h - R)/stride_h) + 1,  Q likewise;  P,Q >= 1.
 */
#ifndef SYSML_H_
#define SYSML_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SYSML_API __attribute__((visibility("default")))
#else
#define SYSML_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *sysml_stream_t; /* == cudaStream_t */

typedef enum {
  SYSML_OK = 0,
  SYSML_ERR_ARG = 1,         /* NULL pointer, negative/zero dimension, bad enum        */
  SYSML_ERR_SHAPE = 2,       /* inconsistent shapes, P or Q < 1, pool pad >= window    */
  SYSML_ERR_UNSUPPORTED = 3, /* valid but not implemented by any kernel (message says)  */
  SYSML_ERR_CUDA = 4,        /* a CUDA runtime error (message carries cudaGetErrorString) */
  SYSML_ERR_NCCL = 5,        /* NCCL not loadable or ncclAllReduce failed               */
  SYSML_ERR_WORKSPACE = 6    /* workspace NULL or smaller than the queried size         */
} sysml_status;

/* Arithmetic of the convolution contractions.
 *  SYSML_MATH_FP32: fp32 operands, fp32 fused multiply-add on CUDA cores
 *                   (parity: max|err| <= 1e-4 * max|ref| vs the fp64 oracle).
 *  SYSML_MATH_TF32: operands rounded to TF32 by the tcgen05 tensor cores,
 *                   fp32 accumulation in TMEM (parity: <= 5e-3 * max|ref|).   */
typedef enum { SYSML_MATH_FP32 = 0, SYSML_MATH_TF32 = 1 } sysml_math;

/* ConvParams: input N x (C*H*W), filter K x (C*R*S) (row k holds
 * F[k,c,r,s] at (c*R + r)*S + s), output N x (K*P*Q).                           */
typedef struct {
  int32_t N, C, H, W;     /* input tensor                        */
  int32_t K, R, S;        /* K filters of R x S                  */
  int32_t stride_h, stride_w;
  int32_t pad_h, pad_w;   /* zero padding (reading R3)           */
  int32_t math;           /* sysml_math                          */
} sysml_conv_desc;

/* PoolParams: max-pool window R x S over input N x (C*H*W);
 * relu != 0 applies relu before the max (SystemML relu_maxpooling).
 * Padding is excluded from the max (-inf); pad must be < window.        */
typedef struct {
  int32_t N, C, H, W;
  int32_t R, S;
  int32_t stride_h, stride_w;
  int32_t pad_h, pad_w;
  int32_t relu;
} sysml_pool_desc;

/* CSR matrix ("various sparse formats (COO, CSR and Modified CSR)";
 * S:28-34): rows x cols, row_ptr[rows+1] (row_ptr[0] == 0, non-decreasing),
 * col_idx[nnz] in [0, cols), val[nnz].  Kernels do not rely on sorted or
 * duplicate-free columns (duplicates are summed), but sysml_csr_check reports
 * violations of S:31-32 (sorted, unique, no explicit zeros, finite).            */
typedef struct {
  int64_t rows, cols, nnz;
  const int32_t *row_ptr;
  const int32_t *col_idx;
  const float *val;
} sysml_csr;

/* Dense-or-CSR input (P:171-174 physical operators "dense input / dense filter,
 * sparse input / dense filter").  is_csr = 0: `dense` is N x (C*H*W);
 * is_csr = 1: `csr` with rows == N and cols == C*H*W.                           */
typedef struct {
  int32_t is_csr;
  const float *dense;
  sysml_csr csr;
} sysml_input;

/* Library identity / diagnostics ------------------------------------------- */
SYSML_API const char *sysml_version(void);
SYSML_API const char *sysml_last_error(void); /* thread-local; never NULL               */
/* Thread-local route of the last conv2d / conv2d_bias_relu_maxpool / bwd_filter /
 * bwd_data call on this thread: the main kernels it launched, " + "-separated, with their
 * operand mode (e.g. "tc_conv_fwd_kernel [tcgen05 TF32, SN, ...]").  Never NULL.        */
SYSML_API const char *sysml_last_route(void);
/* Number of SMs of the current device, as the kernels size their grids.      */
SYSML_API int32_t sysml_device_sm_count(void);

/* conv2d (P:138-140 builtin conv2d; SURVEY §8(c) def 2):
 *   y[n,(k*P+p)*Q+q] = [bias[k]] + sum_{c,r,s} f[k,(c*R+r)*S+s] * x(n,c,p*sh-ph+r,q*sw-pw+s)
 * bias == NULL: plain conv2d; else conv2d_bias_add (bias fp32[K]).
 * x: dense or CSR input (dense: N x CHW). y: N x (K*P*Q).                         */
SYSML_API sysml_status sysml_conv2d_workspace_size(const sysml_conv_desc *d, int32_t is_csr, size_t *bytes);
SYSML_API sysml_status sysml_conv2d(const sysml_conv_desc *d, const sysml_input *x, const float *f,
                          const float *bias, float *y, void *workspace, size_t workspace_bytes,
                          sysml_stream_t stream);

/* conv2d_backward_filter ("their respective backward functions";
 * S:165-173; SURVEY §8(c) def 4):
 *   df[k,(c*R+r)*S+s] = sum_{n,p,q} dy[n,(k*P+p)*Q+q] * x(n,c,p*sh-ph+r,q*sw-pw+s)
 *   db[k] = sum_{n,p,q} dy[n,(k*P+p)*Q+q]        (db may be NULL)
 * x: dense or CSR (N x CHW); dy: N x KPQ; df: K x CRS; db: fp32[K].              */
SYSML_API sysml_status sysml_conv2d_bwd_filter_workspace_size(const sysml_conv_desc *d, int32_t is_csr,
                                                    size_t *bytes);
SYSML_API sysml_status sysml_conv2d_bwd_filter(const sysml_conv_desc *d, const sysml_input *x,
                                     const float *dy, float *df, float *db, void *workspace,
                                     size_t workspace_bytes, sysml_stream_t stream);

/* conv2d_backward_data (SURVEY §8(c) def 5): the adjoint of conv2d in x
 *   dx[n,(c*H+h)*W+w] = sum_{k,r,s,p,q: p*sh-ph+r=h, q*sw-pw+s=w} f[k,(c*R+r)*S+s]*dy[n,(k*P+p)*Q+q]
 * f: K x CRS; dy: N x KPQ; dx: N x CHW.                                          */
SYSML_API sysml_status sysml_conv2d_bwd_data_workspace_size(const sysml_conv_desc *d, size_t *bytes);
SYSML_API sysml_status sysml_conv2d_bwd_data(const sysml_conv_desc *d, const float *f, const float *dy,
                                   float *dx, void *workspace, size_t workspace_bytes,
                                   sysml_stream_t stream);

/* Horizontal fusion for shared inputs (NEXT-2; "horizontal fusion for shared
 * inputs (e.g. reuse temporary im2col intermediates in presence of multiple convolution
 * operators consuming the same input)").  n_ops (1..8) convolutions with ONE geometry
 * (d's N, C, H, W, R, S, stride, pad, math) read the same input x; op i has k_counts[i]
 * filters f[i] (k_counts[i] x C*R*S, device) and d->K must equal sum(k_counts).  They run
 * as one convolution over the stacked bank [f[0]; f[1]; ...], so the staged input feeds
 * every op and x is read once:
 *   sysml_conv2d_multi           y_cat = N x (K*P*Q): op i's output channels are the slice
 *                                [k_0 + ... + k_{i-1}, ... + k_i) of each row (channel
 *                                concatenation); bias[i] nullable (bias itself nullable).
 *   sysml_conv2d_multi_bwd_data  dx = sum_i conv2d_bwd_data(f[i], dy_i), dy_cat laid out as
 *                                y_cat (the input gradient of all consumers of x, summed).
 *   sysml_conv2d_multi_bwd_filter df[i] (k_i x CRS) and db[i] (nullable) of each op from
 *                                x and dy_cat.
 * Workspace: sysml_conv2d_multi_workspace_size(d, n_ops, k_counts, op = 0 fwd / 1 bwd_data /
 * 2 bwd_filter, is_csr).  Errors: SYSML_ERR_ARG (n_ops, k_counts, NULL), SYSML_ERR_SHAPE
 * (d->K != sum k_counts), otherwise as the single-op calls.                              */
SYSML_API sysml_status sysml_conv2d_multi_workspace_size(const sysml_conv_desc *d, int32_t n_ops,
                                                         const int32_t *k_counts, int32_t op,
                                                         int32_t is_csr, size_t *bytes);
SYSML_API sysml_status sysml_conv2d_multi(const sysml_conv_desc *d, int32_t n_ops, const int32_t *k_counts,
                                          const sysml_input *x, const float *const *f,
                                          const float *const *bias, float *y_cat, void *workspace,
                                          size_t workspace_bytes, sysml_stream_t stream);
SYSML_API sysml_status sysml_conv2d_multi_bwd_data(const sysml_conv_desc *d, int32_t n_ops,
                                                   const int32_t *k_counts, const float *const *f,
                                                   const float *dy_cat, float *dx, void *workspace,
                                                   size_t workspace_bytes, sysml_stream_t stream);
SYSML_API sysml_status sysml_conv2d_multi_bwd_filter(const sysml_conv_desc *d, int32_t n_ops,
                                                     const int32_t *k_counts, const sysml_input *x,
                                                     const float *dy_cat, float *const *df,
                                                     float *const *db, void *workspace,
                                                     size_t workspace_bytes, sysml_stream_t stream);

/* affine layer forward (S:236-243 affine_forward; P:48-49 NN library; the hidden layer of
 * LeNet-512, NEXT-4): out[m][j] = sum_k x[m][k] * W[j][k] + b[j] (b nullable), then relu
 * (R7) if relu != 0.  x: M x K, W: N x K (out features x in features), out: M x N, all
 * row-major device fp32, 16-byte aligned.  math TF32: tcgen05 GEMM (TMA-fed, fused
 * epilogue; N >= 16, K % 4 == 0); FP32: CUDA cores (relu needs N % 4 == 0).
 * Errors: SYSML_ERR_ARG (dims < 1, NULL), SYSML_ERR_UNSUPPORTED (alignment, shape).    */
SYSML_API sysml_status sysml_affine(int32_t M, int32_t N, int32_t K, const float *x, const float *W,
                                    const float *b, int32_t relu, int32_t math, float *out,
                                    sysml_stream_t stream);

/* bias_add (P:132 broadcasting; reading R10): y[n, k*PQ + j] += bias[k], in place.
 * y: N x (K*PQ).                                                                  */
SYSML_API sysml_status sysml_bias_add(int32_t N, int32_t K, int32_t PQ, float *y, const float *bias,
                            sysml_stream_t stream);

/* relu_maxpool (P:138-140 pooling builtin; SystemML relu_maxpooling):
 * for each window, v = relu ? max(x,+0) : x scanned r-outer/s-inner over valid
 * (unpadded) positions; out = max, argmax = first position attaining it, encoded
 * as the column index (c*H+h)*W+w of the pool-input row (readings R5, R6).
 * x: N x (C*H*W); out: N x (C*P*Q); argmax: int32 N x (C*P*Q) or NULL.            */
SYSML_API sysml_status sysml_relu_maxpool(const sysml_pool_desc *d, const float *x, float *out,
                                int32_t *argmax, sysml_stream_t stream);

/* maxpooling_backward: dx = 0; dx[n, argmax[n,j]] += dout[n,j] for every
 * pooled output j (collisions summed in ascending j; exact when stride >= window);
 * if out_mask != NULL, only where out_mask[n,j] > 0 (the fused ReLU backward,
 * reading R9).  argmax from sysml_relu_maxpool (same desc).
 * argmax, dout, out_mask: N x (C*P*Q); dx: N x (C*H*W).                           */
SYSML_API sysml_status sysml_maxpool_bwd(const sysml_pool_desc *d, const int32_t *argmax,
                               const float *dout, const float *out_mask, float *dx,
                               sysml_stream_t stream);

/* Fused forward block: conv2d + bias + relu + maxpool in ONE kernel (P:206-207
 * "vertical fusion"; BJ north_star fused epilogue).  Equals
 *   sysml_relu_maxpool(pd with relu=1, sysml_conv2d(cd, x, f, bias))
 * with pd.{N,C,H,W} == (cd.N, cd.K, P, Q).  Supported: pool window == stride
 * (non-overlapping), pad 0.  out: N x (K*P'*Q'); argmax: N x (K*P'*Q').          */
SYSML_API sysml_status sysml_conv2d_bias_relu_maxpool_workspace_size(const sysml_conv_desc *cd,
                                                           const sysml_pool_desc *pd,
                                                           int32_t is_csr, size_t *bytes);
SYSML_API sysml_status sysml_conv2d_bias_relu_maxpool(const sysml_conv_desc *cd, const sysml_pool_desc *pd,
                                            const sysml_input *x, const float *f,
                                            const float *bias, float *out, int32_t *argmax,
                                            void *workspace, size_t workspace_bytes,
                                            sysml_stream_t stream);

/* Debug validation of a device CSR matrix against S:31-32.  Synchronizes
 * `stream`; *violations receives the number of offending rows (0 = valid).       */
SYSML_API sysml_status sysml_csr_check(const sysml_csr *m, int64_t *violations, sysml_stream_t stream);

/* Sparse-filter convolution: the third and fourth of the paper's physical convolution
 * operators ("dense input / sparse filter and sparse input / sparse filter").
 * f: the filter bank as CSR, f->rows = K, f->cols = C*R*S, column (c*R + r)*S + s;
 * only stored entries contribute, duplicate columns are summed (R15).  x: dense
 * N x (C*H*W) or CSR (then C*H*W <= 49152: each image is densified in shared memory).
 * y (device, N x (K*P*Q)) = conv2d(x, densify(f)) (+ bias[K] if non-NULL), fp32, each
 * output summed in the filter's stored order (deterministic).  Errors: SYSML_ERR_SHAPE
 * for mismatched extents, SYSML_ERR_UNSUPPORTED for a CSR image larger than the limit.  */
SYSML_API sysml_status sysml_conv2d_csr_filter(const sysml_conv_desc *d, const sysml_input *x,
                                               const sysml_csr *f, const float *bias, float *y,
                                               sysml_stream_t stream);

/* Format decision ("decides upon dense or sparse formats"): a matrix
 * is stored sparse iff nnz / (rows*cols) <= 0.4.  sysml_count_nonzeros counts the entries
 * != 0 (+0.0 and -0.0 are not stored) of x[0, n) and synchronizes `stream`.
 * sysml_dense_to_csr encodes the dense rows x cols matrix x as CSR: row_ptr int32[rows+1],
 * col_idx int32 / val fp32 [nnz] (sized by sysml_count_nonzeros), columns ascending per row
 * (deterministic); rows*cols < 2^31.  Caller-owned device buffers.                      */
SYSML_API sysml_status sysml_count_nonzeros(const float *x, int64_t n, int64_t *nnz_host,
                                            sysml_stream_t stream);
SYSML_API sysml_status sysml_dense_to_csr(const float *x, int64_t rows, int64_t cols, int32_t *row_ptr,
                                          int32_t *col_idx, float *val, sysml_stream_t stream);
/* The decision itself: *is_sparse = 1 iff n > 0 and
 * nnz / n <= threshold (threshold <= 0 selects the default SYSML_SPARSITY_THRESHOLD),
 * else 0; *nnz_host = nnz of x[0, n).  Synchronizes `stream` (a host decision).         */
#define SYSML_SPARSITY_THRESHOLD 0.4
SYSML_API sysml_status sysml_decide_format(const float *x, int64_t n, double threshold, int32_t *is_sparse,
                                           int64_t *nnz_host, sysml_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Minibatch SGD-step driver (Listing 1: batch -> forward -> backward ->
 * sgd::update, lr = 0.01; P:142 LeNet; P:187-192 data-parallel plan).
 * LeNet-min = [conv5x5(32,p2)+relu+pool2] -> [conv5x5(64,p2)+relu+pool2]
 *             -> affine(3136->10) -> softmax -> cross-entropy.
 * Flat parameter order: F1[32x25], b1[32], F2[64x800], b2[64], W3[10x3136], b3[10]
 * (83,466 floats).                                                               */
typedef struct sysml_lenet sysml_lenet;

SYSML_API int64_t sysml_lenet_num_params(void);
/* max_local_batch: largest n_local a call may pass.  input_is_csr selects the
 * CSR conv1 kernels; max_nnz bounds CSR nnz per call (ignored when dense).
 * The handle owns activations and scratch (allocated here, once).               */
SYSML_API sysml_status sysml_lenet_create(int32_t max_local_batch, int32_t math, int32_t input_is_csr,
                                int64_t max_nnz, sysml_lenet **out);
SYSML_API sysml_status sysml_lenet_destroy(sysml_lenet *h);

/* LeNet-512 (NEXT-4; SystemML's mnist_lenet topology, R22-R24; "20+
 * pre-implemented layers", S:275-281 dropout):
 *   [conv5x5(32,p2)+relu+pool2] -> [conv5x5(64,p2)+relu+pool2] -> affine(3136->512) -> relu
 *   -> inverted dropout(keep_p) -> affine(512->10) -> softmax -> cross-entropy.
 * Flat parameter order: F1[32x25], b1[32], F2[64x800], b2[64], W3[512x3136], b3[512],
 * W4[10x512], b4[10] (1,663,370 floats).  The returned handle serves sysml_lenet_fwd_bwd /
 * _predict / _step / _step_opt / _step_host* exactly as a LeNet-min handle, with this
 * parameter vector.  Dropout mask (R23): unit j of GLOBAL sample row g is kept iff the high
 * 32 bits of raw output e = g*512 + j of Philox4x64-10 with key (seed, t) are below
 * floor(keep_p * 2^32) (numpy.random.Philox order), where t is the handle's device step
 * counter: 0 at creation, +1 at the end of every sysml_lenet_step* call (so CUDA-graph
 * replays draw fresh masks); fwd_bwd alone does not advance it.  Kept units are scaled by
 * 1/keep_p.  Scoring (predict) applies no dropout.
 * Errors: SYSML_ERR_ARG if keep_p is not in (0, 1]; others as sysml_lenet_create.        */
SYSML_API int64_t sysml_lenet512_num_params(void);
SYSML_API sysml_status sysml_lenet512_create(int32_t max_local_batch, int32_t math, int32_t input_is_csr,
                                             int64_t max_nnz, float keep_p, uint64_t seed,
                                             sysml_lenet **out);
/* row0 = global index of the local shard's first row (rank * local batch in the
 * data-parallel plan; the mask follows the global row, so sharding does not change it);
 * step = new value of the device step counter, set on `stream`.  LeNet-512 handles only.  */
SYSML_API sysml_status sysml_lenet_set_dropout(sysml_lenet *h, int64_t row0, int64_t step,
                                               sysml_stream_t stream);
/* Reads the device step counter (synchronous).                                           */
SYSML_API sysml_status sysml_lenet_get_dropout_step(sysml_lenet *h, int64_t *step);
/* Parameter count of this handle's model (83,466 or 1,663,370).                          */
SYSML_API int64_t sysml_lenet_handle_num_params(const sysml_lenet *h);

/* Forward + backward of the local shard (rows of the global batch):
 * grads (device, fp32[83466]) receive sum over local samples of dLoss/dtheta
 * with Loss = (1/n_global) sum_global CE, i.e. already scaled by 1/n_global
 * so that the sum over ranks is the full-batch gradient.
 * loss_sum (device scalar, may be NULL) receives (1/n_global) sum_local CE.
 * labels: int32[n_local] in [0,10).                                               */
SYSML_API sysml_status sysml_lenet_fwd_bwd(sysml_lenet *h, const float *params, const sysml_input *x,
                                 const int32_t *labels, int32_t n_local, int64_t n_global,
                                 float *grads, float *loss_sum, sysml_stream_t stream);

/* Scoring (parfor-style row-partitioned scoring; replicas need no collective):
 * the forward of the local rows (conv-relu-pool x2, affine) -> pred int32[n_local] = the
 * first maximal class (nullable) and probs fp32[n_local x 10] = softmax (nullable; one of
 * the two required).  x: dense or CSR as the handle was created.                      */
SYSML_API sysml_status sysml_lenet_predict(sysml_lenet *h, const float *params, const sysml_input *x,
                                           int32_t n_local, int32_t *pred, float *probs,
                                           sysml_stream_t stream);

/* SGD (S:282-290 sgd: p - lr*g): params[i] -= lr * grads[i], i < n.              */
SYSML_API sysml_status sysml_sgd_update(float *params, const float *grads, int64_t n, float lr,
                              sysml_stream_t stream);

/* One data-parallel step = fwd_bwd + (if nccl_comm != NULL) ncclAllReduce(sum, fp32)
 * of grads over the communicator + sgd_update.  nccl_comm is an ncclComm_t of the
 * NCCL library already loaded in the process (e.g. torch's ProcessGroupNCCL);
 * ncclAllReduce is resolved from it at run time (SYSML_ERR_NCCL if absent).      */
SYSML_API sysml_status sysml_lenet_step(sysml_lenet *h, float *params, float *grads, const sysml_input *x,
                              const int32_t *labels, int32_t n_local, int64_t n_global,
                              float lr, void *nccl_comm, float *loss_sum, sysml_stream_t stream);

/* The six optimizers of the NN library ("Adagrad, Adam, RMSprop, SGD, SGD with
 * momentum, and SGD with Nesterov momentum"; S:282-290 optimizer_update).  One update of
 * params[0, n) with grads (device fp32).  `state` (device, caller-owned, zero before the
 * first update; NULL for SGD) holds sysml_optimizer_state_floats(kind) * n floats: the
 * velocity (momentum, nesterov), the squared-gradient cache (adagrad, rmsprop), or the
 * first moments then the second moments (adam).  t = adam timestep of this update, >= 1
 * (ignored by the others).  Rules, elementwise in fp32 (oracle: oracle_optimizer_update):
 *   sgd       p -= lr g
 *   momentum  v = mu v - lr g;  p += v
 *   nesterov  v' = mu v - lr g;  p += -mu v + (1 + mu) v'
 *   adagrad   c += g^2;  p -= lr g / (sqrt(c) + eps)
 *   rmsprop   c = rho c + (1 - rho) g^2;  p -= lr g / (sqrt(c) + eps)
 *   adam      m = b1 m + (1 - b1) g;  v = b2 v + (1 - b2) g^2;
 *             p -= lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)
 * Errors: SYSML_ERR_ARG for an unknown kind, NULL pointers, n < 0, t < 1 (adam). */
typedef enum {
  SYSML_OPT_SGD = 0, SYSML_OPT_MOMENTUM = 1, SYSML_OPT_NESTEROV = 2,
  SYSML_OPT_ADAGRAD = 3, SYSML_OPT_RMSPROP = 4, SYSML_OPT_ADAM = 5
} sysml_optimizer_kind;
typedef struct {
  int32_t kind;
  float lr, mu, rho, eps, beta1, beta2;
} sysml_optimizer_desc;
SYSML_API int32_t sysml_optimizer_state_floats(int32_t kind); /* 0, 1 or 2 per parameter; -1 unknown */
SYSML_API sysml_status sysml_optimizer_update(const sysml_optimizer_desc *d, float *params,
                                              const float *grads, float *state, int64_t n, int64_t t,
                                              sysml_stream_t stream);

/* sysml_lenet_step with any of the six optimizers: fwd_bwd + (if nccl_comm) the bucketed
 * gradient allreduce + sysml_optimizer_update(d, params, grads, state, 83466, t).        */
SYSML_API sysml_status sysml_lenet_step_opt(sysml_lenet *h, float *params, float *grads, float *state,
                                  const sysml_optimizer_desc *d, int64_t t, const sysml_input *x,
                                  const int32_t *labels, int32_t n_local, int64_t n_global,
                                  void *nccl_comm, float *loss_sum, sysml_stream_t stream);

/* End-to-end variant with HOST inputs: x_host (dense fp32 n_local x 784, pinned
 * for overlap) and labels_host are copied into handle-owned device buffers on
 * `stream`, the step runs as sysml_lenet_step, and the loss is copied back to
 * *loss_host.  Synchronizes `stream` before returning (the loss is valid).     */
SYSML_API sysml_status sysml_lenet_step_host(sysml_lenet *h, float *params, float *grads,
                                   const float *x_host, const int32_t *labels_host,
                                   int32_t n_local, int64_t n_global, float lr, void *nccl_comm,
                                   float *loss_host, sysml_stream_t stream);

/* Pipelined variant of sysml_lenet_step_host for a training loop over host batches: the
 * step on (x_host, labels_host) runs while the NEXT batch (x_host_next, labels_host_next,
 * n_next; NULL = none) is copied host->device on the handle's copy stream into its second
 * input buffer.  A call whose batch is the one the previous call prefetched (same host
 * pointers and size) only waits for that copy; otherwise it copies now.  The next batch's
 * host memory (pinned for overlap) must stay unchanged until the following call.  Every
 * call performs one batch H2D and reads the loss back; synchronizes `stream` on return.  */
SYSML_API sysml_status sysml_lenet_step_host_pipelined(sysml_lenet *h, float *params, float *grads,
                                             const float *x_host, const int32_t *labels_host,
                                             int32_t n_local, const float *x_host_next,
                                             const int32_t *labels_host_next, int32_t n_next,
                                             int64_t n_global, float lr, void *nccl_comm,
                                             float *loss_host, sysml_stream_t stream);

/* Per-stage device timing of the step (bench instrumentation).  When enabled,
 * fwd_bwd records CUDA events around each stage on `stream`; get_timing returns
 * accumulated milliseconds, launch counts and stage names (stage i < *n_stages),
 * after synchronizing the recorded events.  reset clears the accumulators.      */
SYSML_API sysml_status sysml_lenet_set_timing(sysml_lenet *h, int32_t enable);
SYSML_API sysml_status sysml_lenet_get_timing(sysml_lenet *h, int32_t max_stages, int32_t *n_stages,
                                    double *ms, int64_t *calls, const char **names);
/* Total number of CUDA kernels this library has launched from the calling thread
 * (monotonic; the bench reads it around its timed region).                       */
SYSML_API int64_t sysml_launch_counter(void);

#ifdef __cplusplus
}
#endif
#endif /* SYSML_H_ */
