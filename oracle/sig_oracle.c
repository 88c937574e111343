/*
 * oracle/sig_oracle.c -- CPU restatement of the reference `sigkit` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path and the CPU baseline timed by bench.py (`cpu_baseline` leg and
 * `--impl reference`).  Nothing in paper_2602_24066_b200/ links or calls it.
 *
 * Every routine restates one reference routine (paths relative to
 * /root/reference/pkg/src/sigkit):
 *   ora_increments        sigcore.py:80-88   PathBatch.increments
 *   ora_letters           wordsets.py:176-188  WordSet.letters
 *   ora_factor_table      wordsets.py:205-228  WordSet._factor_table (prefix/suffix)
 *   ora_forward_{f32,f64} _kernels.py:40-58    forward_kernel  (+ sigcore.py:201-206 inv)
 *   ora_windows_{f32,f64} _kernels.py:61-82    windows_kernel
 *   ora_backward_f64      _kernels.py:85-183   backward_kernel (+ backward.py:186-200 buffers)
 *   ora_sample_grads      backward.py:130-147  increment_to_sample_grads
 *
 * Numerics follow the numba kernels operation by operation: in the float32
 * forward the Horner accumulator `h` is float64 (numba unifies `h = 0.0` with
 * the float64 product), the scratch stack and inv[] are float32, and
 * `scratch[m] += h` rounds the float64 sum back to float32.  The backward is
 * float64 throughout (backward.py:166-167).  OpenMP parallelises over the same
 * units as numba's prange ((path, word) forward, path backward), so results
 * are bitwise independent of the thread count, as in the reference.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EPSILON_INDEX (-1)
#define MISSING_INDEX (-2)

static uint64_t upow(uint64_t d, int64_t e) {
  uint64_t p = 1;
  for (int64_t i = 0; i < e; ++i) p *= d;
  return p;
}

/* sigcore.py:80-88 -- per-path X[1:] - X[:-1] in the sample dtype. */
void ora_increments_f64(const double* X, int64_t B, int64_t L, int64_t d, double* out) {
  int64_t M = L - 1;
  for (int64_t b = 0; b < B; ++b)
    for (int64_t j = 0; j < M; ++j)
      for (int64_t i = 0; i < d; ++i)
        out[(b * M + j) * d + i] = X[(b * L + j + 1) * d + i] - X[(b * L + j) * d + i];
}
void ora_increments_f32(const float* X, int64_t B, int64_t L, int64_t d, float* out) {
  int64_t M = L - 1;
  for (int64_t b = 0; b < B; ++b)
    for (int64_t j = 0; j < M; ++j)
      for (int64_t i = 0; i < d; ++i)
        out[(b * M + j) * d + i] = X[(b * L + j + 1) * d + i] - X[(b * L + j) * d + i];
}

/* wordsets.py:176-188 -- letters[i, j] = (code // d^(n-1-j)) % d, zero padded. */
void ora_letters(const uint64_t* codes, const int64_t* lengths, int64_t W, int64_t d,
                 int64_t max_len, int64_t* letters) {
  for (int64_t i = 0; i < W; ++i) {
    int64_t n = lengths[i];
    for (int64_t j = 0; j < max_len; ++j) {
      letters[i * max_len + j] =
          (j < n) ? (int64_t)((codes[i] / upow((uint64_t)d, n - 1 - j)) % (uint64_t)d) : 0;
    }
  }
}

/* Position of (len, code) in the canonical (length asc, code asc) arrays, or
 * MISSING_INDEX: the reference's global_index dict lookup (wordsets.py:155-161,
 * :221-227) restated as a binary search over the sorted arrays. */
static int64_t find_word(const uint64_t* codes, const int64_t* lengths, int64_t W, int64_t len,
                         uint64_t code) {
  int64_t lo = 0, hi = W;
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (lengths[mid] < len || (lengths[mid] == len && codes[mid] < code))
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo < W && lengths[lo] == len && codes[lo] == code) return lo;
  return MISSING_INDEX;
}

/* wordsets.py:205-228 -- prefix (suffix=0) or suffix (suffix=1) table,
 * shape (W, max_len+1); both the full-truncation arithmetic path and the
 * lookup path produce the same entries, so one lookup restatement suffices. */
void ora_factor_table(const uint64_t* codes, const int64_t* lengths, int64_t W, int64_t d,
                      int64_t max_len, int suffix, int64_t* table) {
  int64_t C = max_len + 1;
  for (int64_t i = 0; i < W; ++i) {
    int64_t n = lengths[i];
    table[i * C] = EPSILON_INDEX;
    for (int64_t k = 1; k < C; ++k) {
      if (k > n) { table[i * C + k] = MISSING_INDEX; continue; }
      uint64_t sub = suffix ? codes[i] % upow((uint64_t)d, k) : codes[i] / upow((uint64_t)d, n - k);
      table[i * C + k] = find_word(codes, lengths, W, k, sub);
    }
  }
}

/* _kernels.py:40-58 with sigcore.py:201-206 (inv in the path dtype). */
void ora_forward_f64(const double* incr, int64_t B, int64_t M, int64_t d, const int64_t* letters,
                     const int64_t* lengths, int64_t W, int64_t max_len, double* out) {
  double* inv = (double*)calloc((size_t)max_len + 1, sizeof(double));
  for (int64_t k = 1; k <= max_len; ++k) inv[k] = 1.0 / (double)k;
#pragma omp parallel
  {
    double* scratch = (double*)malloc(sizeof(double) * ((size_t)max_len + 1));
#pragma omp for schedule(static)
    for (int64_t unit = 0; unit < B * W; ++unit) {
      int64_t b = unit / W, wi = unit % W, n = lengths[wi];
      const int64_t* lw = letters + wi * max_len;
      scratch[0] = 1.0;
      for (int64_t k = 1; k <= n; ++k) scratch[k] = 0.0;
      for (int64_t j = 0; j < M; ++j) {
        const double* dx = incr + (b * M + j) * d;
        for (int64_t m = n; m >= 1; --m) {
          double h = 0.0;
          for (int64_t k = 0; k < m; ++k) h = dx[lw[k]] * inv[m - k] * (scratch[k] + h);
          scratch[m] += h;
        }
      }
      out[b * W + wi] = scratch[n];
    }
    free(scratch);
  }
  free(inv);
}

void ora_forward_f32(const float* incr, int64_t B, int64_t M, int64_t d, const int64_t* letters,
                     const int64_t* lengths, int64_t W, int64_t max_len, float* out) {
  float* inv = (float*)calloc((size_t)max_len + 1, sizeof(float));
  for (int64_t k = 1; k <= max_len; ++k) inv[k] = 1.0f / (float)k;
#pragma omp parallel
  {
    float* scratch = (float*)malloc(sizeof(float) * ((size_t)max_len + 1));
#pragma omp for schedule(static)
    for (int64_t unit = 0; unit < B * W; ++unit) {
      int64_t b = unit / W, wi = unit % W, n = lengths[wi];
      const int64_t* lw = letters + wi * max_len;
      scratch[0] = 1.0f;
      for (int64_t k = 1; k <= n; ++k) scratch[k] = 0.0f;
      for (int64_t j = 0; j < M; ++j) {
        const float* dx = incr + (b * M + j) * d;
        for (int64_t m = n; m >= 1; --m) {
          double h = 0.0; /* numba types h as float64 */
          for (int64_t k = 0; k < m; ++k) {
            float a = dx[lw[k]] * inv[m - k]; /* float32 * float32 */
            h = (double)a * ((double)scratch[k] + h);
          }
          scratch[m] = (float)((double)scratch[m] + h);
        }
      }
      out[b * W + wi] = scratch[n];
    }
    free(scratch);
  }
  free(inv);
}

/* _kernels.py:61-82 -- bounds (K, 2) sample indices; out (B, K, W). */
void ora_windows_f64(const double* incr, int64_t B, int64_t M, int64_t d, const int64_t* letters,
                     const int64_t* lengths, int64_t W, int64_t max_len, const int64_t* bounds,
                     int64_t K, double* out) {
  double* inv = (double*)calloc((size_t)max_len + 1, sizeof(double));
  for (int64_t k = 1; k <= max_len; ++k) inv[k] = 1.0 / (double)k;
#pragma omp parallel
  {
    double* scratch = (double*)malloc(sizeof(double) * ((size_t)max_len + 1));
#pragma omp for schedule(static)
    for (int64_t unit = 0; unit < B * K * W; ++unit) {
      int64_t b = unit / (K * W), rest = unit % (K * W), kw = rest / W, wi = rest % W;
      int64_t n = lengths[wi];
      const int64_t* lw = letters + wi * max_len;
      scratch[0] = 1.0;
      for (int64_t k = 1; k <= n; ++k) scratch[k] = 0.0;
      for (int64_t j = bounds[2 * kw]; j < bounds[2 * kw + 1]; ++j) {
        const double* dx = incr + (b * M + j) * d;
        for (int64_t m = n; m >= 1; --m) {
          double h = 0.0;
          for (int64_t k = 0; k < m; ++k) h = dx[lw[k]] * inv[m - k] * (scratch[k] + h);
          scratch[m] += h;
        }
      }
      out[(b * K + kw) * W + wi] = scratch[n];
    }
    free(scratch);
  }
  free(inv);
}

void ora_windows_f32(const float* incr, int64_t B, int64_t M, int64_t d, const int64_t* letters,
                     const int64_t* lengths, int64_t W, int64_t max_len, const int64_t* bounds,
                     int64_t K, float* out) {
  float* inv = (float*)calloc((size_t)max_len + 1, sizeof(float));
  for (int64_t k = 1; k <= max_len; ++k) inv[k] = 1.0f / (float)k;
#pragma omp parallel
  {
    float* scratch = (float*)malloc(sizeof(float) * ((size_t)max_len + 1));
#pragma omp for schedule(static)
    for (int64_t unit = 0; unit < B * K * W; ++unit) {
      int64_t b = unit / (K * W), rest = unit % (K * W), kw = rest / W, wi = rest % W;
      int64_t n = lengths[wi];
      const int64_t* lw = letters + wi * max_len;
      scratch[0] = 1.0f;
      for (int64_t k = 1; k <= n; ++k) scratch[k] = 0.0f;
      for (int64_t j = bounds[2 * kw]; j < bounds[2 * kw + 1]; ++j) {
        const float* dx = incr + (b * M + j) * d;
        for (int64_t m = n; m >= 1; --m) {
          double h = 0.0;
          for (int64_t k = 0; k < m; ++k) {
            float a = dx[lw[k]] * inv[m - k];
            h = (double)a * ((double)scratch[k] + h);
          }
          scratch[m] = (float)((double)scratch[m] + h);
        }
      }
      out[(b * K + kw) * W + wi] = scratch[n];
    }
    free(scratch);
  }
  free(inv);
}

/* _kernels.py:85-183 -- float64 reverse sweep per path, words sequential.
 * upstream (B, W) float64; stride 0 = no checkpoints (backward.py:193-199);
 * inc_grads (B, M, d) is accumulated (+=) and must be zero on entry. */
void ora_backward_f64(const double* incr, int64_t B, int64_t M, int64_t d, const int64_t* letters,
                      const int64_t* lengths, int64_t W, int64_t max_len, const double* upstream,
                      int64_t stride, double* inc_grads) {
  int64_t C = max_len + 1;
  int64_t n_ckpt = stride > 0 ? M / stride + 1 : 1;
  double* inv = (double*)calloc((size_t)C, sizeof(double));
  for (int64_t k = 1; k <= max_len; ++k) inv[k] = 1.0 / (double)k;
#pragma omp parallel
  {
    double* left = (double*)malloc(sizeof(double) * C);
    double* right = (double*)malloc(sizeof(double) * C);
    double* dh = (double*)malloc(sizeof(double) * d);
    double* acc = (double*)malloc(sizeof(double) * d);
    double* ckpt = (double*)malloc(sizeof(double) * n_ckpt * C);
#pragma omp for schedule(dynamic, 1)
    for (int64_t b = 0; b < B; ++b) {
      const double* inc = incr + b * M * d;
      double* ig = inc_grads + b * M * d;
      for (int64_t wi = 0; wi < W; ++wi) {
        double g = upstream[b * W + wi];
        if (g == 0.0) continue;
        int64_t n = lengths[wi];
        const int64_t* lw = letters + wi * max_len;
        left[0] = 1.0;
        for (int64_t k = 1; k <= n; ++k) left[k] = 0.0;
        if (stride > 0)
          for (int64_t k = 0; k <= n; ++k) ckpt[k] = left[k];
        for (int64_t j = 0; j < M; ++j) {
          for (int64_t m = n; m >= 1; --m) {
            double h = 0.0;
            for (int64_t k = 0; k < m; ++k) h = inc[j * d + lw[k]] * inv[m - k] * (left[k] + h);
            left[m] += h;
          }
          if (stride > 0 && (j + 1) % stride == 0)
            for (int64_t k = 0; k <= n; ++k) ckpt[((j + 1) / stride) * C + k] = left[k];
        }
        right[0] = 1.0;
        for (int64_t k = 1; k <= n; ++k) right[k] = 0.0;
        for (int64_t j = M - 1; j >= 0; --j) {
          if (stride > 0 && j % stride == 0) {
            for (int64_t k = 0; k <= n; ++k) left[k] = ckpt[(j / stride) * C + k];
          } else {
            for (int64_t m = n; m >= 1; --m) {
              double h = 0.0;
              for (int64_t k = 0; k < m; ++k)
                h = -inc[j * d + lw[k]] * inv[m - k] * (left[k] + h);
              left[m] += h;
            }
          }
          for (int64_t i = 0; i < d; ++i) acc[i] = 0.0;
          for (int64_t q = 1; q <= n; ++q) {
            double h = 0.0;
            for (int64_t i = 0; i < d; ++i) dh[i] = 0.0;
            for (int64_t k = 0; k < q; ++k) {
              int64_t lett = lw[k];
              double a = inc[j * d + lett];
              double s = inv[q - k];
              double tmp = left[k] + h;
              for (int64_t i = 0; i < d; ++i) dh[i] = s * a * dh[i];
              dh[lett] += s * tmp;
              h = s * a * tmp;
            }
            double rv = right[n - q];
            for (int64_t i = 0; i < d; ++i) acc[i] += rv * dh[i];
          }
          for (int64_t i = 0; i < d; ++i) ig[j * d + i] += g * acc[i];
          for (int64_t m = n; m >= 1; --m) {
            double h = 0.0;
            for (int64_t p = m; p >= 1; --p)
              h = inc[j * d + lw[n - m + p - 1]] * inv[p] * (right[m - p] + h);
            right[m] += h;
          }
        }
      }
    }
    free(left); free(right); free(dh); free(acc); free(ckpt);
  }
  free(inv);
}

/* backward.py:130-147 -- dX_j = dDelta_j - dDelta_{j+1}, one-sided ends. */
void ora_sample_grads(const double* inc_grads, int64_t B, int64_t M, int64_t d, double* out) {
  int64_t L = M + 1;
  memset(out, 0, sizeof(double) * (size_t)(B * L * d));
  for (int64_t b = 0; b < B; ++b) {
    for (int64_t j = 0; j < M; ++j)
      for (int64_t i = 0; i < d; ++i) out[(b * L + j + 1) * d + i] += inc_grads[(b * M + j) * d + i];
    for (int64_t j = 0; j < M; ++j)
      for (int64_t i = 0; i < d; ++i) out[(b * L + j) * d + i] -= inc_grads[(b * M + j) * d + i];
  }
}
