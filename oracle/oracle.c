/*
 * oracle.c -- fp64 CPU oracle for the conv2d-family hot path of
 * arXiv 1802.04647 ("Deep Learning with Apache SystemML", SysML'18).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA library
 * (paper_1802_04647_b200/csrc); neither includes nor links the other.
 *
 * Every operator is the plain definition written out as direct nested loops
 * in double precision (SURVEY.md §8(c) "Definitions").
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n.
 *
 * Tensor layout ("a 4-dimensional tensor of shape [N, C, H, W] is
 * represented as a matrix with N rows and C*H*W columns"): element (n,c,h,w)
 * lives at X[n*(C*H*W) + (c*H + h)*W + w]  (S:100 nchw_to_flat).
 *
 * Readings of the paper where it is silent (listed in DESIGN.md "Readings"):
 *   R1 cross-correlation (no filter flip), S:159 f . im2col(x)
 *   R2 output extent P = floor((H + 2ph - R)/sh) + 1
 *   R3 conv padding contributes 0; pool padding is excluded (-inf)
 *   R4 fully padded pool window -> out 0, argmax -1
 *   R5 pool ties -> first position in row-major window order (strict >)
 *   R6 argmax = column index (c*H+h)*W+w into the pool-input row
 *   R7 relu(x) = x > 0 ? x : +0.0
 *   R9 maxpool_bwd with relu mask routes dout iff pooled out > 0
 *   R11 loss = -(1/N_global) sum log(max(p[y], 1e-15)); dscores = (p - onehot)/N_global
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

static inline int64_t out_extent(int64_t in, int64_t pad, int64_t k, int64_t stride) {
  /* R2: floor((in + 2 pad - k) / stride) + 1 ; <1 means invalid */
  int64_t num = in + 2 * pad - k;
  if (num < 0) return 0;
  return num / stride + 1;
}

EXPORT int64_t oracle_out_extent(int64_t in, int64_t pad, int64_t k, int64_t stride) {
  return out_extent(in, pad, k, stride);
}

/* ------------------------------------------------------------------------ */
/* conv2d forward  (P:138-140 builtin conv2d; SURVEY §8(c) def 2)
 *   Y[n,(k*P+p)*Q+q] = [b[k]] + sum_{c,r,s} F[k,(c*R+r)*S+s] * x(n,c,p*sh-ph+r,q*sw-pw+s)
 * Summation order: for each output plane (n,k): start from b[k] (or 0), then
 * c ascending, r ascending, s ascending, each term added to every (p,q). */
EXPORT void oracle_conv2d_fwd(int64_t N, int64_t C, int64_t H, int64_t W, int64_t K,
                              int64_t R, int64_t S, int64_t sh, int64_t sw, int64_t ph,
                              int64_t pw, const double *x, const double *f,
                              const double *bias, double *y) {
  const int64_t P = out_extent(H, ph, R, sh), Q = out_extent(W, pw, S, sw);
  const int64_t CHW = C * H * W, CRS = C * R * S, KPQ = K * P * Q;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t n = 0; n < N; ++n) {
    for (int64_t k = 0; k < K; ++k) {
      double *plane = y + n * KPQ + k * P * Q;
      const double b0 = bias ? bias[k] : 0.0;
      for (int64_t i = 0; i < P * Q; ++i) plane[i] = b0;
      for (int64_t c = 0; c < C; ++c)
        for (int64_t r = 0; r < R; ++r)
          for (int64_t s = 0; s < S; ++s) {
            const double wgt = f[k * CRS + (c * R + r) * S + s];
            for (int64_t p = 0; p < P; ++p) {
              const int64_t h = p * sh - ph + r;
              if (h < 0 || h >= H) continue;
              const double *xrow = x + n * CHW + (c * H + h) * W;
              double *yrow = plane + p * Q;
              for (int64_t q = 0; q < Q; ++q) {
                const int64_t w = q * sw - pw + s;
                if (w < 0 || w >= W) continue;
                yrow[q] += wgt * xrow[w];
              }
            }
          }
    }
  }
}

/* ------------------------------------------------------------------------ */
/* bias_add ("broadcasting operations over scalars and vectors";
 * reading R10: bias is fp32[K], added to all P*Q outputs of filter k)
 *   Y[n, k*PQ + j] += b[k] */
EXPORT void oracle_bias_add(int64_t N, int64_t K, int64_t PQ, double *y, const double *b) {
  for (int64_t n = 0; n < N; ++n)
    for (int64_t k = 0; k < K; ++k)
      for (int64_t j = 0; j < PQ; ++j) y[(n * K + k) * PQ + j] += b[k];
}

/* ------------------------------------------------------------------------ */
/* conv2d_backward_filter ("their respective backward functions";
 * S:165-173; SURVEY §8(c) def 4)
 *   dF[k,(c*R+r)*S+s] = sum_n sum_p sum_q dY[n,(k*P+p)*Q+q] * x(n,c,p*sh-ph+r,q*sw-pw+s)
 *   db[k] = sum_{n,p,q} dY[n,(k*P+p)*Q+q]
 * Summation order: n, p, q ascending. */
EXPORT void oracle_conv2d_bwd_filter(int64_t N, int64_t C, int64_t H, int64_t W, int64_t K,
                                     int64_t R, int64_t S, int64_t sh, int64_t sw, int64_t ph,
                                     int64_t pw, const double *x, const double *dy, double *df,
                                     double *db) {
  const int64_t P = out_extent(H, ph, R, sh), Q = out_extent(W, pw, S, sw);
  const int64_t CHW = C * H * W, CRS = C * R * S, KPQ = K * P * Q;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t k = 0; k < K; ++k) {
    for (int64_t c = 0; c < C; ++c) {
      for (int64_t r = 0; r < R; ++r)
        for (int64_t s = 0; s < S; ++s) {
          double acc = 0.0;
          for (int64_t n = 0; n < N; ++n)
            for (int64_t p = 0; p < P; ++p) {
              const int64_t h = p * sh - ph + r;
              if (h < 0 || h >= H) continue;
              for (int64_t q = 0; q < Q; ++q) {
                const int64_t w = q * sw - pw + s;
                if (w < 0 || w >= W) continue;
                acc += dy[n * KPQ + (k * P + p) * Q + q] * x[n * CHW + (c * H + h) * W + w];
              }
            }
          df[k * CRS + (c * R + r) * S + s] = acc;
        }
    }
  }
  if (db) {
    for (int64_t k = 0; k < K; ++k) {
      double acc = 0.0;
      for (int64_t n = 0; n < N; ++n)
        for (int64_t j = 0; j < P * Q; ++j) acc += dy[n * KPQ + k * P * Q + j];
      db[k] = acc;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* conv2d_backward_data (SURVEY §8(c) def 5): the exact adjoint
 * (transpose) of conv2d_fwd in X, written as the forward loop nest with the
 * multiply-add redirected into dX:
 *   dX[n,(c*H+h)*W+w] = sum_{k,r,s,p,q : p*sh-ph+r=h, q*sw-pw+s=w} F[k,c,r,s] dY[n,k,p,q]
 * Summation order per dX element: k, r, s, p, q ascending (loop nest order). */
EXPORT void oracle_conv2d_bwd_data(int64_t N, int64_t C, int64_t H, int64_t W, int64_t K,
                                   int64_t R, int64_t S, int64_t sh, int64_t sw, int64_t ph,
                                   int64_t pw, const double *f, const double *dy, double *dx) {
  const int64_t P = out_extent(H, ph, R, sh), Q = out_extent(W, pw, S, sw);
  const int64_t CHW = C * H * W, CRS = C * R * S, KPQ = K * P * Q;
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < N; ++n) {
    double *dxn = dx + n * CHW;
    for (int64_t i = 0; i < CHW; ++i) dxn[i] = 0.0;
    for (int64_t c = 0; c < C; ++c)
      for (int64_t k = 0; k < K; ++k)
        for (int64_t r = 0; r < R; ++r)
          for (int64_t s = 0; s < S; ++s) {
            const double wgt = f[k * CRS + (c * R + r) * S + s];
            for (int64_t p = 0; p < P; ++p) {
              const int64_t h = p * sh - ph + r;
              if (h < 0 || h >= H) continue;
              for (int64_t q = 0; q < Q; ++q) {
                const int64_t w = q * sw - pw + s;
                if (w < 0 || w >= W) continue;
                dxn[(c * H + h) * W + w] += wgt * dy[n * KPQ + (k * P + p) * Q + q];
              }
            }
          }
  }
}

/* ------------------------------------------------------------------------ */
/* relu_maxpool (P:138-140 pooling builtin; SURVEY §8(c) def 6)
 * For each (n,c,p',q'): scan r outer, s inner over the window; skip padded
 * positions (R3); v = relu ? (x>0 ? x : +0.0) : x (R7); first valid position or
 * v > best (strict, R5) updates best and arg = (c*H+h)*W+w (R6).
 * Fully padded window: out 0, argmax -1 (R4). */
EXPORT void oracle_relu_maxpool(int64_t N, int64_t C, int64_t H, int64_t W, int64_t R,
                                int64_t S, int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                                int64_t relu, const double *x, double *out, int32_t *argmax) {
  const int64_t P = out_extent(H, ph, R, sh), Q = out_extent(W, pw, S, sw);
  const int64_t CHW = C * H * W, CPQ = C * P * Q;
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < N; ++n)
    for (int64_t c = 0; c < C; ++c)
      for (int64_t p = 0; p < P; ++p)
        for (int64_t q = 0; q < Q; ++q) {
          int found = 0;
          double best = 0.0;
          int64_t arg = -1;
          for (int64_t r = 0; r < R; ++r)
            for (int64_t s = 0; s < S; ++s) {
              const int64_t h = p * sh - ph + r, w = q * sw - pw + s;
              if (h < 0 || h >= H || w < 0 || w >= W) continue;
              double v = x[n * CHW + (c * H + h) * W + w];
              if (relu) v = v > 0.0 ? v : 0.0;
              if (!found || v > best) {
                found = 1;
                best = v;
                arg = (c * H + h) * W + w;
              }
            }
          const int64_t o = n * CPQ + (c * P + p) * Q + q;
          out[o] = found ? best : 0.0;
          if (argmax) argmax[o] = (int32_t)arg;
        }
}

/* ------------------------------------------------------------------------ */
/* maxpool_backward (SURVEY §8(c) def 7)
 *   dX = 0; for each window in ascending (c,p',q') order: if argmax >= 0 and
 *   (no mask or out > 0, R9): dX[n, argmax] += dout[n, (c*P'+p')*Q'+q'] */
EXPORT void oracle_maxpool_bwd(int64_t N, int64_t C, int64_t H, int64_t W, int64_t P,
                               int64_t Q, const int32_t *argmax, const double *dout,
                               const double *out_mask, double *dx) {
  const int64_t CHW = C * H * W, CPQ = C * P * Q;
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < N; ++n) {
    double *dxn = dx + n * CHW;
    for (int64_t i = 0; i < CHW; ++i) dxn[i] = 0.0;
    for (int64_t j = 0; j < CPQ; ++j) {
      const int32_t a = argmax[n * CPQ + j];
      if (a < 0) continue;
      if (out_mask && !(out_mask[n * CPQ + j] > 0.0)) continue;
      dxn[a] += dout[n * CPQ + j];
    }
  }
}

/* ------------------------------------------------------------------------ */
/* CSR densify ("various sparse formats (COO, CSR and Modified CSR)";
 * S:28-34).  The CSR input case of every operator is defined as the operator
 * on this densification (duplicates summed). */
EXPORT void oracle_csr_densify(int64_t rows, int64_t cols, const int32_t *row_ptr,
                               const int32_t *col_idx, const double *val, double *dense) {
  memset(dense, 0, sizeof(double) * (size_t)(rows * cols));
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t j = row_ptr[r]; j < row_ptr[r + 1]; ++j) dense[r * cols + col_idx[j]] += val[j];
}

/* ------------------------------------------------------------------------ */
/* LeNet-min minibatch SGD step (Listing 1 loop body: forward, backward,
 * sgd::update with lr = 0.01; "LeNet"; SURVEY §8(c) def 8):
 *   z1 = conv(X; F1,b1, 5x5 p2 s1);  a1,i1 = relu_maxpool(z1, 2x2/2)
 *   z2 = conv(a1; F2,b2, 5x5 p2 s1); a2,i2 = relu_maxpool(z2, 2x2/2)
 *   s  = a2 W3^T + b3;  p = softmax(s) (max shift)
 *   L  = -(1/Ng) sum_n log(max(p[n,y_n], 1e-15))       (R11)
 *   ds = (p - onehot(y)) / Ng
 *   dW3 = ds^T a2; db3 = colsum(ds); da2 = ds W3
 *   dz2 = maxpool_bwd(i2, da2, a2>0); dF2,db2 = bwd_filter(a1,dz2); da1 = bwd_data(F2,dz2)
 *   dz1 = maxpool_bwd(i1, da1, a1>0); dF1,db1 = bwd_filter(X,dz1)
 * Parameter order (flat): F1[32x25], b1[32], F2[64x800], b2[64], W3[10x3136], b3[10]. */
#define L_F1 0
#define L_B1 (L_F1 + 32 * 25)
#define L_F2 (L_B1 + 32)
#define L_B2 (L_F2 + 64 * 800)
#define L_W3 (L_B2 + 64)
#define L_B3 (L_W3 + 10 * 3136)
#define L_NP (L_B3 + 10)

EXPORT int64_t oracle_lenet_num_params(void) { return L_NP; }

EXPORT void oracle_lenet_forward(int64_t n, const double *x, const double *prm, double *a1,
                                 int32_t *i1, double *a2, int32_t *i2, double *scores) {
  double *z1 = (double *)malloc(sizeof(double) * (size_t)(n * 32 * 784));
  double *z2 = (double *)malloc(sizeof(double) * (size_t)(n * 64 * 196));
  oracle_conv2d_fwd(n, 1, 28, 28, 32, 5, 5, 1, 1, 2, 2, x, prm + L_F1, prm + L_B1, z1);
  oracle_relu_maxpool(n, 32, 28, 28, 2, 2, 2, 2, 0, 0, 1, z1, a1, i1);
  oracle_conv2d_fwd(n, 32, 14, 14, 64, 5, 5, 1, 1, 2, 2, a1, prm + L_F2, prm + L_B2, z2);
  oracle_relu_maxpool(n, 64, 14, 14, 2, 2, 2, 2, 0, 0, 1, z2, a2, i2);
  const double *W3 = prm + L_W3, *b3 = prm + L_B3;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < 10; ++j) {
      double acc = b3[j];
      for (int64_t d = 0; d < 3136; ++d) acc += a2[i * 3136 + d] * W3[j * 3136 + d];
      scores[i * 10 + j] = acc;
    }
  free(z1);
  free(z2);
}

/* Scoring (P:193-202 parfor-style scoring; Listing 1 "probs = softmax::forward(scores)",
 * S:252-258 softmax with the max shift): probs[i,j] = exp(s_ij - m_i) / sum_j' exp(s_ij' - m_i),
 * m_i = max_j s_ij; pred[i] = the first j with s_ij == m_i (first maximal class).          */
EXPORT void oracle_lenet_predict(int64_t n, const double *x, const double *prm, int32_t *pred,
                                 double *probs) {
  double *a1 = (double *)malloc(sizeof(double) * (size_t)(n * 6272));
  double *a2 = (double *)malloc(sizeof(double) * (size_t)(n * 3136));
  int32_t *i1 = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n * 6272));
  int32_t *i2 = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n * 3136));
  double *sc = (double *)malloc(sizeof(double) * (size_t)(n * 10));
  oracle_lenet_forward(n, x, prm, a1, i1, a2, i2, sc);
  for (int64_t i = 0; i < n; ++i) {
    double m = sc[i * 10];
    int32_t arg = 0;
    for (int j = 1; j < 10; ++j)
      if (sc[i * 10 + j] > m) { m = sc[i * 10 + j]; arg = j; }
    double den = 0.0;
    for (int j = 0; j < 10; ++j) den += exp(sc[i * 10 + j] - m);
    for (int j = 0; j < 10; ++j) probs[i * 10 + j] = exp(sc[i * 10 + j] - m) / den;
    pred[i] = arg;
  }
  free(a1); free(a2); free(i1); free(i2); free(sc);
}

EXPORT void oracle_lenet_fwd_bwd(int64_t n, int64_t n_global, const double *x,
                                 const int32_t *labels, const double *prm, double *grads,
                                 double *loss_sum) {
  double *a1 = (double *)malloc(sizeof(double) * (size_t)(n * 6272));
  double *a2 = (double *)malloc(sizeof(double) * (size_t)(n * 3136));
  int32_t *i1 = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n * 6272));
  int32_t *i2 = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n * 3136));
  double *sc = (double *)malloc(sizeof(double) * (size_t)(n * 10));
  double *ds = (double *)malloc(sizeof(double) * (size_t)(n * 10));
  double *da2 = (double *)malloc(sizeof(double) * (size_t)(n * 3136));
  double *dz2 = (double *)malloc(sizeof(double) * (size_t)(n * 12544));
  double *da1 = (double *)malloc(sizeof(double) * (size_t)(n * 6272));
  double *dz1 = (double *)malloc(sizeof(double) * (size_t)(n * 25088));
  oracle_lenet_forward(n, x, prm, a1, i1, a2, i2, sc);

  double loss = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double m = sc[i * 10];
    for (int j = 1; j < 10; ++j) m = sc[i * 10 + j] > m ? sc[i * 10 + j] : m;
    double den = 0.0;
    for (int j = 0; j < 10; ++j) den += exp(sc[i * 10 + j] - m);
    for (int j = 0; j < 10; ++j) {
      const double pj = exp(sc[i * 10 + j] - m) / den;
      ds[i * 10 + j] = (pj - (j == labels[i] ? 1.0 : 0.0)) / (double)n_global;
      if (j == labels[i]) loss += -log(pj > 1e-15 ? pj : 1e-15);
    }
  }
  if (loss_sum) *loss_sum = loss / (double)n_global;

  const double *W3 = prm + L_W3;
  double *dW3 = grads + L_W3, *db3 = grads + L_B3;
  for (int j = 0; j < 10; ++j) {
    double accb = 0.0;
    for (int64_t i = 0; i < n; ++i) accb += ds[i * 10 + j];
    db3[j] = accb;
    for (int64_t d = 0; d < 3136; ++d) {
      double acc = 0.0;
      for (int64_t i = 0; i < n; ++i) acc += ds[i * 10 + j] * a2[i * 3136 + d];
      dW3[j * 3136 + d] = acc;
    }
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t d = 0; d < 3136; ++d) {
      double acc = 0.0;
      for (int j = 0; j < 10; ++j) acc += ds[i * 10 + j] * W3[j * 3136 + d];
      da2[i * 3136 + d] = acc;
    }
  oracle_maxpool_bwd(n, 64, 14, 14, 7, 7, i2, da2, a2, dz2);
  oracle_conv2d_bwd_filter(n, 32, 14, 14, 64, 5, 5, 1, 1, 2, 2, a1, dz2, grads + L_F2,
                           grads + L_B2);
  oracle_conv2d_bwd_data(n, 32, 14, 14, 64, 5, 5, 1, 1, 2, 2, prm + L_F2, dz2, da1);
  oracle_maxpool_bwd(n, 32, 28, 28, 14, 14, i1, da1, a1, dz1);
  oracle_conv2d_bwd_filter(n, 1, 28, 28, 32, 5, 5, 1, 1, 2, 2, x, dz1, grads + L_F1,
                           grads + L_B1);
  free(a1); free(a2); free(i1); free(i2); free(sc); free(ds);
  free(da2); free(dz2); free(da1); free(dz1);
}

/* SGD ("lr = 0.01", P:80-81 sgd::update): theta <- theta - lr * g */
EXPORT void oracle_sgd_update(int64_t n, double *params, const double *grads, double lr) {
  for (int64_t i = 0; i < n; ++i) params[i] = params[i] - lr * grads[i];
}

/* The six optimizers of the NN library ("6 optimizers (namely Adagrad, Adam, RMSprop,
 * SGD, SGD with momentum, and SGD with Nesterov momentum)"; S:282-290 optimizer_update).
 * kind: 0 sgd, 1 sgd_momentum, 2 sgd_nesterov, 3 adagrad, 4 rmsprop, 5 adam.
 * state: kinds 1-4 one accumulator per parameter (velocity v / squared-gradient cache);
 * adam two, first moments m[0..n) then second moments v[n..2n).  t = adam timestep of
 * this update (>= 1).  One update, written out in the order of the rules:
 *   sgd       p <- p - lr g
 *   momentum  v <- mu v - lr g;  p <- p + v
 *   nesterov  v_prev <- v;  v <- mu v - lr g;  p <- p - mu v_prev + (1 + mu) v
 *             (the look-ahead form of momentum; reading R19)
 *   adagrad   c <- c + g^2;  p <- p - lr g / (sqrt(c) + eps)
 *   rmsprop   c <- rho c + (1 - rho) g^2;  p <- p - lr g / (sqrt(c) + eps)
 *   adam      m <- b1 m + (1 - b1) g;  v <- b2 v + (1 - b2) g^2;
 *             mh = m / (1 - b1^t);  vh = v / (1 - b2^t);  p <- p - lr mh / (sqrt(vh) + eps)
 *             (bias-corrected moments; eps outside the correction as in S:290's
 *             worked example p = -lr * 1 / (sqrt(1) + eps) at t = 1)                    */
EXPORT void oracle_optimizer_update(int64_t kind, int64_t n, double *p, const double *g, double *state,
                                    double lr, double mu, double rho, double eps, double b1, double b2,
                                    int64_t t) {
  for (int64_t i = 0; i < n; ++i) {
    const double gi = g[i];
    if (kind == 0) {
      p[i] = p[i] - lr * gi;
    } else if (kind == 1) {
      state[i] = mu * state[i] - lr * gi;
      p[i] = p[i] + state[i];
    } else if (kind == 2) {
      const double v_prev = state[i];
      state[i] = mu * state[i] - lr * gi;
      p[i] = p[i] - mu * v_prev + (1.0 + mu) * state[i];
    } else if (kind == 3) {
      state[i] = state[i] + gi * gi;
      p[i] = p[i] - lr * gi / (sqrt(state[i]) + eps);
    } else if (kind == 4) {
      state[i] = rho * state[i] + (1.0 - rho) * gi * gi;
      p[i] = p[i] - lr * gi / (sqrt(state[i]) + eps);
    } else {
      double *m = state, *v = state + n;
      m[i] = b1 * m[i] + (1.0 - b1) * gi;
      v[i] = b2 * v[i] + (1.0 - b2) * gi * gi;
      const double mh = m[i] / (1.0 - pow(b1, (double)t));
      const double vh = v[i] / (1.0 - pow(b2, (double)t));
      p[i] = p[i] - lr * mh / (sqrt(vh) + eps);
    }
  }
}

/* Dense input / sparse filter convolution (the third of the four physical
 * convolution operators): the filter bank is CSR with K rows and C*R*S columns
 * (column (c*R + r)*S + s, the row-major index of S:100), and only its stored non-zeros
 * contribute: y[n,k,p,q] = b[k] + sum over stored (col, v) of row k of
 *                          v * x(n, c, p*sh - ph + r, q*sw - pw + s)   (0 outside).
 * Duplicate columns of a row are summed (reading R15).  Sparse input / sparse filter is
 * this with x densified (oracle_csr_densify).                                         */
EXPORT void oracle_conv2d_fwd_csr_filter(int64_t N, int64_t C, int64_t H, int64_t W, int64_t K,
                                         int64_t R, int64_t S, int64_t sh, int64_t sw, int64_t ph,
                                         int64_t pw, const double *x, const int32_t *f_row_ptr,
                                         const int32_t *f_col_idx, const double *f_val,
                                         const double *bias, double *y) {
  const int64_t P = out_extent(H, ph, R, sh), Q = out_extent(W, pw, S, sw);
  const int64_t CHW = C * H * W, KPQ = K * P * Q;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t n = 0; n < N; ++n) {
    for (int64_t k = 0; k < K; ++k) {
      double *plane = y + n * KPQ + k * P * Q;
      const double b0 = bias ? bias[k] : 0.0;
      for (int64_t i = 0; i < P * Q; ++i) plane[i] = b0;
      for (int64_t j = f_row_ptr[k]; j < f_row_ptr[k + 1]; ++j) {
        const int64_t col = f_col_idx[j];
        const int64_t c = col / (R * S), r = (col / S) % R, s = col % S;
        const double v = f_val[j];
        for (int64_t p = 0; p < P; ++p) {
          const int64_t h = p * sh - ph + r;
          if (h < 0 || h >= H) continue;
          for (int64_t q = 0; q < Q; ++q) {
            const int64_t w = q * sw - pw + s;
            if (w < 0 || w >= W) continue;
            plane[p * Q + q] += v * x[n * CHW + (c * H + h) * W + w];
          }
        }
      }
    }
  }
}

/* decide_format ("decides upon dense or sparse formats"): a matrix is
 * stored sparse iff nnz / (rows * cols) <= threshold (0.4 by default, S's design decision).
 * Returns the number of non-zeros (exact zeros, +0.0 and -0.0, are not stored).          */
EXPORT int64_t oracle_count_nonzeros(int64_t n, const double *a) {
  int64_t nnz = 0;
  for (int64_t i = 0; i < n; ++i) nnz += a[i] != 0.0;
  return nnz;
}

/* ------------------------------------------------------------------------ */
/* NEXT-4: the SystemML LeNet with a 512-unit hidden affine layer and dropout
 * ("20+ pre-implemented layers"; S:275-281 dropout; SURVEY §8(f) NEXT-4;
 * DESIGN.md readings R22-R24).
 *
 * Dropout's random numbers come from a counter-based generator so that the GPU and this
 * oracle draw the same mask without sharing code (R23): Philox4x64-10 (Salmon et al.,
 * SC'11), the generator numpy exposes as numpy.random.Philox, in numpy's output order:
 * raw 64-bit output e of key (k0, k1) is word e % 4 of the block for counter value
 * (e / 4 + 1, 0, 0, 0).  (numpy increments the counter before each block.)           */
static inline void philox_mulhilo(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
  const unsigned __int128 p = (unsigned __int128)a * b;
  *hi = (uint64_t)(p >> 64);
  *lo = (uint64_t)p;
}

static void philox4x64_10(const uint64_t ctr_in[4], uint64_t k0, uint64_t k1, uint64_t out[4]) {
  uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { /* key schedule: Weyl sequence bump between rounds */
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    uint64_t hi0, lo0, hi1, lo1;
    philox_mulhilo(0xD2E7470EE14C6C93ULL, c0, &hi0, &lo0);
    philox_mulhilo(0xCA5A826395121157ULL, c2, &hi1, &lo1);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* raw outputs e = start .. start + n - 1 of the stream with key (k0, k1) */
EXPORT void oracle_philox_raw(uint64_t k0, uint64_t k1, int64_t start, int64_t n, uint64_t *out) {
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t e = (uint64_t)(start + i);
    const uint64_t ctr[4] = {e / 4 + 1, 0, 0, 0};
    uint64_t w[4];
    philox4x64_10(ctr, k0, k1, w);
    out[i] = w[e % 4];
  }
}

/* Dropout keep mask ("Bernoulli(keep_p) mask from the seeded generator"; R23):
 * unit j of global sample row g, step t: e = g * units + j, key = (seed, t);
 * kept  <=>  (raw_e >> 32) < floor(keep_p * 2^32)   (keep_p in (0, 1]; keep_p = 1 keeps all). */
static inline uint64_t keep_threshold(double keep_p) { return (uint64_t)floor(keep_p * 4294967296.0); }

EXPORT void oracle_dropout_mask(uint64_t seed, uint64_t step, int64_t row0, int64_t rows, int64_t units,
                                double keep_p, uint8_t *mask) {
  const uint64_t T = keep_threshold(keep_p);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < units; ++j) {
      uint64_t raw;
      oracle_philox_raw(seed, step, (row0 + i) * units + j, 1, &raw);
      mask[i * units + j] = (raw >> 32) < T ? 1 : 0;
    }
}

/* inverted dropout: out = x * mask / keep_p;  backward: dx = dout * mask / keep_p */
EXPORT void oracle_dropout_fwd(int64_t n, const double *x, const uint8_t *mask, double keep_p, double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = mask[i] ? x[i] / keep_p : 0.0;
}

EXPORT void oracle_dropout_bwd(int64_t n, const double *dout, const uint8_t *mask, double keep_p, double *dx) {
  for (int64_t i = 0; i < n; ++i) dx[i] = mask[i] ? dout[i] / keep_p : 0.0;
}

/* LeNet-512 (SystemML's mnist_lenet.dml topology, SURVEY §8(c) reading 12 [ext]; R22):
 *   z1 = conv(X; F1,b1, 5x5 p2);  a1,i1 = relu_maxpool(z1, 2x2/2)
 *   z2 = conv(a1; F2,b2, 5x5 p2); a2,i2 = relu_maxpool(z2, 2x2/2)
 *   z3 = a2 W3^T + b3  (3136 -> 512);  r3 = relu(z3);  h = dropout(r3; mask, keep_p)
 *   s  = h W4^T + b4   (512 -> 10);    p = softmax(s);  L = -(1/Ng) sum log(max(p[y], 1e-15))
 * backward:  ds = (p - onehot(y)) / Ng;  dW4 = ds^T h;  db4 = colsum(ds);  dh = ds W4
 *   dr3 = dropout_bwd(dh; mask);  dz3 = dr3 * [z3 > 0];  dW3 = dz3^T a2;  db3 = colsum(dz3)
 *   da2 = dz3 W3;  then exactly the LeNet-min tail (dz2, dF2, db2, da1, dz1, dF1, db1).
 * train = 0 (scoring) skips dropout (h = r3).  row0 = global index of local row 0 (the
 * mask is a function of the global sample row, so any sharding draws the same masks).
 * Flat parameter order: F1[32x25], b1[32], F2[64x800], b2[64], W3[512x3136], b3[512],
 * W4[10x512], b4[10]  (1,663,370 floats).                                             */
#define L5_H 512
#define L5_F1 0
#define L5_B1 (L5_F1 + 32 * 25)
#define L5_F2 (L5_B1 + 32)
#define L5_B2 (L5_F2 + 64 * 800)
#define L5_W3 (L5_B2 + 64)
#define L5_B3 (L5_W3 + L5_H * 3136)
#define L5_W4 (L5_B3 + L5_H)
#define L5_B4 (L5_W4 + 10 * L5_H)
#define L5_NP (L5_B4 + 10)

EXPORT int64_t oracle_lenet512_num_params(void) { return L5_NP; }

/* forward; writes a1, i1, a2, i2 (as oracle_lenet_forward), z3 [n x 512], h [n x 512],
 * mask [n x 512] (all ones when train = 0) and scores [n x 10]. */
EXPORT void oracle_lenet512_forward(int64_t n, int64_t row0, const double *x, const double *prm,
                                    int64_t train, uint64_t seed, uint64_t step, double keep_p,
                                    double *a1, int32_t *i1, double *a2, int32_t *i2, double *z3,
                                    double *h, uint8_t *mask, double *scores) {
  double *z1 = (double *)malloc(sizeof(double) * (size_t)(n * 32 * 784));
  double *z2 = (double *)malloc(sizeof(double) * (size_t)(n * 64 * 196));
  double *r3 = (double *)malloc(sizeof(double) * (size_t)(n * L5_H));
  oracle_conv2d_fwd(n, 1, 28, 28, 32, 5, 5, 1, 1, 2, 2, x, prm + L5_F1, prm + L5_B1, z1);
  oracle_relu_maxpool(n, 32, 28, 28, 2, 2, 2, 2, 0, 0, 1, z1, a1, i1);
  oracle_conv2d_fwd(n, 32, 14, 14, 64, 5, 5, 1, 1, 2, 2, a1, prm + L5_F2, prm + L5_B2, z2);
  oracle_relu_maxpool(n, 64, 14, 14, 2, 2, 2, 2, 0, 0, 1, z2, a2, i2);
  const double *W3 = prm + L5_W3, *b3 = prm + L5_B3, *W4 = prm + L5_W4, *b4 = prm + L5_B4;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t u = 0; u < L5_H; ++u) {
      double acc = b3[u];
      for (int64_t d = 0; d < 3136; ++d) acc += a2[i * 3136 + d] * W3[u * 3136 + d];
      z3[i * L5_H + u] = acc;
      r3[i * L5_H + u] = acc > 0.0 ? acc : 0.0; /* R7 */
    }
  if (train) {
    oracle_dropout_mask(seed, step, row0, n, L5_H, keep_p, mask);
    oracle_dropout_fwd(n * L5_H, r3, mask, keep_p, h);
  } else {
    memset(mask, 1, (size_t)(n * L5_H));
    memcpy(h, r3, sizeof(double) * (size_t)(n * L5_H));
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < 10; ++j) {
      double acc = b4[j];
      for (int64_t u = 0; u < L5_H; ++u) acc += h[i * L5_H + u] * W4[j * L5_H + u];
      scores[i * 10 + j] = acc;
    }
  free(z1); free(z2); free(r3);
}

EXPORT void oracle_lenet512_fwd_bwd(int64_t n, int64_t n_global, int64_t row0, const double *x,
                                    const int32_t *labels, const double *prm, uint64_t seed,
                                    uint64_t step, double keep_p, double *grads, double *loss_sum) {
  double *a1 = (double *)malloc(sizeof(double) * (size_t)(n * 6272));
  double *a2 = (double *)malloc(sizeof(double) * (size_t)(n * 3136));
  int32_t *i1 = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n * 6272));
  int32_t *i2 = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n * 3136));
  double *z3 = (double *)malloc(sizeof(double) * (size_t)(n * L5_H));
  double *h = (double *)malloc(sizeof(double) * (size_t)(n * L5_H));
  uint8_t *mask = (uint8_t *)malloc((size_t)(n * L5_H));
  double *sc = (double *)malloc(sizeof(double) * (size_t)(n * 10));
  double *ds = (double *)malloc(sizeof(double) * (size_t)(n * 10));
  double *dh = (double *)malloc(sizeof(double) * (size_t)(n * L5_H));
  double *dz3 = (double *)malloc(sizeof(double) * (size_t)(n * L5_H));
  double *da2 = (double *)malloc(sizeof(double) * (size_t)(n * 3136));
  double *dz2 = (double *)malloc(sizeof(double) * (size_t)(n * 12544));
  double *da1 = (double *)malloc(sizeof(double) * (size_t)(n * 6272));
  double *dz1 = (double *)malloc(sizeof(double) * (size_t)(n * 25088));
  oracle_lenet512_forward(n, row0, x, prm, 1, seed, step, keep_p, a1, i1, a2, i2, z3, h, mask, sc);

  double loss = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double m = sc[i * 10];
    for (int j = 1; j < 10; ++j) m = sc[i * 10 + j] > m ? sc[i * 10 + j] : m;
    double den = 0.0;
    for (int j = 0; j < 10; ++j) den += exp(sc[i * 10 + j] - m);
    for (int j = 0; j < 10; ++j) {
      const double pj = exp(sc[i * 10 + j] - m) / den;
      ds[i * 10 + j] = (pj - (j == labels[i] ? 1.0 : 0.0)) / (double)n_global;
      if (j == labels[i]) loss += -log(pj > 1e-15 ? pj : 1e-15);
    }
  }
  if (loss_sum) *loss_sum = loss / (double)n_global;

  const double *W3 = prm + L5_W3, *W4 = prm + L5_W4;
  double *dW4 = grads + L5_W4, *db4 = grads + L5_B4, *dW3 = grads + L5_W3, *db3 = grads + L5_B3;
  for (int j = 0; j < 10; ++j) {
    double accb = 0.0;
    for (int64_t i = 0; i < n; ++i) accb += ds[i * 10 + j];
    db4[j] = accb;
    for (int64_t u = 0; u < L5_H; ++u) {
      double acc = 0.0;
      for (int64_t i = 0; i < n; ++i) acc += ds[i * 10 + j] * h[i * L5_H + u];
      dW4[j * L5_H + u] = acc;
    }
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t u = 0; u < L5_H; ++u) {
      double acc = 0.0;
      for (int j = 0; j < 10; ++j) acc += ds[i * 10 + j] * W4[j * L5_H + u];
      dh[i * L5_H + u] = acc;
    }
  oracle_dropout_bwd(n * L5_H, dh, mask, keep_p, dz3);            /* dr3 */
  for (int64_t e = 0; e < n * L5_H; ++e) dz3[e] = z3[e] > 0.0 ? dz3[e] : 0.0; /* relu' */
#pragma omp parallel for schedule(static)
  for (int64_t u = 0; u < L5_H; ++u) {
    double accb = 0.0;
    for (int64_t i = 0; i < n; ++i) accb += dz3[i * L5_H + u];
    db3[u] = accb;
    for (int64_t d = 0; d < 3136; ++d) {
      double acc = 0.0;
      for (int64_t i = 0; i < n; ++i) acc += dz3[i * L5_H + u] * a2[i * 3136 + d];
      dW3[u * 3136 + d] = acc;
    }
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t d = 0; d < 3136; ++d) {
      double acc = 0.0;
      for (int64_t u = 0; u < L5_H; ++u) acc += dz3[i * L5_H + u] * W3[u * 3136 + d];
      da2[i * 3136 + d] = acc;
    }
  oracle_maxpool_bwd(n, 64, 14, 14, 7, 7, i2, da2, a2, dz2);
  oracle_conv2d_bwd_filter(n, 32, 14, 14, 64, 5, 5, 1, 1, 2, 2, a1, dz2, grads + L5_F2, grads + L5_B2);
  oracle_conv2d_bwd_data(n, 32, 14, 14, 64, 5, 5, 1, 1, 2, 2, prm + L5_F2, dz2, da1);
  oracle_maxpool_bwd(n, 32, 28, 28, 14, 14, i1, da1, a1, dz1);
  oracle_conv2d_bwd_filter(n, 1, 28, 28, 32, 5, 5, 1, 1, 2, 2, x, dz1, grads + L5_F1, grads + L5_B1);
  free(a1); free(a2); free(i1); free(i2); free(z3); free(h); free(mask); free(sc); free(ds);
  free(dh); free(dz3); free(da2); free(dz2); free(da1); free(dz1);
}

/* scoring of LeNet-512 (no dropout at inference): first maximal class + softmax */
EXPORT void oracle_lenet512_predict(int64_t n, const double *x, const double *prm, int32_t *pred,
                                    double *probs) {
  double *a1 = (double *)malloc(sizeof(double) * (size_t)(n * 6272));
  double *a2 = (double *)malloc(sizeof(double) * (size_t)(n * 3136));
  int32_t *i1 = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n * 6272));
  int32_t *i2 = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n * 3136));
  double *z3 = (double *)malloc(sizeof(double) * (size_t)(n * L5_H));
  double *h = (double *)malloc(sizeof(double) * (size_t)(n * L5_H));
  uint8_t *mask = (uint8_t *)malloc((size_t)(n * L5_H));
  double *sc = (double *)malloc(sizeof(double) * (size_t)(n * 10));
  oracle_lenet512_forward(n, 0, x, prm, 0, 0, 0, 1.0, a1, i1, a2, i2, z3, h, mask, sc);
  for (int64_t i = 0; i < n; ++i) {
    double m = sc[i * 10];
    int32_t arg = 0;
    for (int j = 1; j < 10; ++j)
      if (sc[i * 10 + j] > m) { m = sc[i * 10 + j]; arg = j; }
    double den = 0.0;
    for (int j = 0; j < 10; ++j) den += exp(sc[i * 10 + j] - m);
    for (int j = 0; j < 10; ++j) probs[i * 10 + j] = exp(sc[i * 10 + j] - m) / den;
    pred[i] = arg;
  }
  free(a1); free(a2); free(i1); free(i2); free(z3); free(h); free(mask); free(sc);
}
