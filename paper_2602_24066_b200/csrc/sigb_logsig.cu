// Consumers of the signature on the device: the Lyndon log-series polynomial
// (logsig.py:139-192) and the dense truncated tensor algebra behind
// tensor_log / tensor_exp / chen_concat / signature_inverse
// (logsig.py:42-72, sigcore.py:297-352).
//
// All three are HBM/L2-bound gathers over one path's coefficient row, so the
// kernels put a path's row per CTA column block and keep every reduction in a
// fixed order (no atomics): the polynomial's gradient is a gather over the
// column -> (term, factor) inverted index the host builds once per (d, N).
#include <algorithm>

#include "sigb_internal.h"

namespace sigb {
namespace {

constexpr int64_t kMaxGridY = 65535;  // batch rows per launch (grid.y)

// out[b, i] = sum_{t in terms(i)} coef[t] * prod_k sig[b, cols[t][k]]
template <typename T>
__global__ void logsig_poly_kernel(const T* __restrict__ sig, int64_t B, int64_t sig_ld,
                                   const int64_t* __restrict__ term_off, const int32_t* __restrict__ cols,
                                   const double* __restrict__ coef, int64_t n_out, int F, T* __restrict__ out,
                                   int64_t out_ld) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t b = blockIdx.y;
  if (i >= n_out || b >= B) return;
  const T* row = sig + b * sig_ld;
  T acc = T(0);
  for (int64_t t = term_off[i]; t < term_off[i + 1]; ++t) {
    const int32_t* c = cols + t * F;
    T p = row[c[0]];
    for (int k = 1; k < F && c[k] >= 0; ++k) p *= row[c[k]];
    acc += T(coef[t]) * p;
  }
  out[b * out_ld + i] = acc;
}

// up[b, c] = sum over entries (t, k) of column c of
//            g[b, word[t]] * coef[t] * prod_{k' != k} sig[b, cols[t][k']]
template <typename T>
__global__ void logsig_poly_grad_kernel(const T* __restrict__ sig, int64_t B, int64_t sig_ld,
                                        const T* __restrict__ g, int64_t g_ld, const int64_t* __restrict__ col_off,
                                        const int64_t* __restrict__ ent, const int64_t* __restrict__ term_word,
                                        const int32_t* __restrict__ cols, const double* __restrict__ coef, int F,
                                        int64_t ncols, T* __restrict__ up, int64_t up_ld) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t b = blockIdx.y;
  if (c >= ncols || b >= B) return;
  const T* row = sig + b * sig_ld;
  const T* grow = g + b * g_ld;
  T acc = T(0);
  for (int64_t e = col_off[c]; e < col_off[c + 1]; ++e) {
    const int64_t t = ent[e] >> 8;
    const int k0 = (int)(ent[e] & 0xff);
    const int32_t* cc = cols + t * F;
    T p = grow[term_word[t]] * T(coef[t]);
    for (int k = 0; k < F && cc[k] >= 0; ++k)
      if (k != k0) p *= row[cc[k]];
    acc += p;
  }
  up[b * up_ld + c] = acc;
}

// Graded product of dense truncated tensors (epsilon-first layout, width
// sum_{n<=N} d^n): out_n[c] = scale * sum_{m=0..n} x_m[c / d^(n-m)] * y_{n-m}[c % d^(n-m)],
// then out[0] += add0.  One thread per output coefficient, m ascending.
template <typename T>
__global__ void tensor_mul_kernel(const T* __restrict__ x, const T* __restrict__ y, int64_t B, int64_t d, int N,
                                  int64_t width, T scale, T add0, T* __restrict__ out) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t b = blockIdx.y;
  if (o >= width || b >= B) return;
  // level n of o and its offset
  int n = 0;
  int64_t off = 0, pw = 1;
  while (o >= off + pw) {
    off += pw;
    pw *= d;
    ++n;
  }
  const int64_t c = o - off;
  const T* xr = x + b * width;
  const T* yr = y + b * width;
  int64_t pm = 1, offm = 0;           // d^m, offset of level m
  int64_t pr = pw, offr = off;        // d^(n-m), offset of level n-m
  T acc = T(0);
  for (int m = 0; m <= n; ++m) {
    acc += xr[offm + c / pr] * yr[offr + c % pr];
    offm += pm;
    pm *= d;
    if (m < n) {
      pr /= d;
      offr -= pr;
    }
  }
  acc *= scale;
  if (o == 0) acc += add0;
  out[b * width + o] = acc;
}

}  // namespace
}  // namespace sigb

using namespace sigb;

extern "C" int sigb_logsig_forward(int dtype, const void* d_sig, int64_t B, int64_t sig_ld, const int64_t* d_term_off,
                                   const int32_t* d_cols, const double* d_coef, int64_t n_out, int max_factors,
                                   void* d_out, int64_t out_ld, void* stream) {
  if (dtype != SIGB_F32 && dtype != SIGB_F64) return fail(SIGB_ERR_SHAPE, "unsupported dtype; use float64 or float32");
  if (B < 0 || n_out < 0 || max_factors < 1) return fail(SIGB_ERR_SHAPE, "bad logsig polynomial shape");
  if (B == 0 || n_out == 0) return SIGB_OK;
  const size_t es = dtype == SIGB_F32 ? 4 : 8;
  for (int64_t b0 = 0; b0 < B; b0 += kMaxGridY) {
    const int64_t Bc = std::min<int64_t>(kMaxGridY, B - b0);
    const char* sig = (const char*)d_sig + es * b0 * sig_ld;
    char* out = (char*)d_out + es * b0 * out_ld;
    const dim3 grid((unsigned)((n_out + 127) / 128), (unsigned)Bc);
    count_launch();
    if (dtype == SIGB_F32)
      logsig_poly_kernel<float><<<grid, 128, 0, (cudaStream_t)stream>>>(
          (const float*)sig, Bc, sig_ld, d_term_off, d_cols, d_coef, n_out, max_factors, (float*)out, out_ld);
    else
      logsig_poly_kernel<double><<<grid, 128, 0, (cudaStream_t)stream>>>(
          (const double*)sig, Bc, sig_ld, d_term_off, d_cols, d_coef, n_out, max_factors, (double*)out, out_ld);
    SIGB_CUDA_TRY(cudaGetLastError());
  }
  return SIGB_OK;
}

extern "C" int sigb_logsig_backward(int dtype, const void* d_sig, int64_t B, int64_t sig_ld, const void* d_g,
                                    int64_t g_ld, const int64_t* d_col_off, const int64_t* d_entries,
                                    const int64_t* d_term_word, const int32_t* d_cols, const double* d_coef,
                                    int max_factors, int64_t ncols, void* d_up, int64_t up_ld, void* stream) {
  if (dtype != SIGB_F32 && dtype != SIGB_F64) return fail(SIGB_ERR_SHAPE, "unsupported dtype; use float64 or float32");
  if (B < 0 || ncols < 0 || max_factors < 1) return fail(SIGB_ERR_SHAPE, "bad logsig polynomial shape");
  if (B == 0 || ncols == 0) return SIGB_OK;
  const size_t es = dtype == SIGB_F32 ? 4 : 8;
  for (int64_t b0 = 0; b0 < B; b0 += kMaxGridY) {
    const int64_t Bc = std::min<int64_t>(kMaxGridY, B - b0);
    const char* sig = (const char*)d_sig + es * b0 * sig_ld;
    const char* g = (const char*)d_g + es * b0 * g_ld;
    char* up = (char*)d_up + es * b0 * up_ld;
    const dim3 grid((unsigned)((ncols + 127) / 128), (unsigned)Bc);
    count_launch();
    if (dtype == SIGB_F32)
      logsig_poly_grad_kernel<float><<<grid, 128, 0, (cudaStream_t)stream>>>(
          (const float*)sig, Bc, sig_ld, (const float*)g, g_ld, d_col_off, d_entries, d_term_word, d_cols, d_coef,
          max_factors, ncols, (float*)up, up_ld);
    else
      logsig_poly_grad_kernel<double><<<grid, 128, 0, (cudaStream_t)stream>>>(
          (const double*)sig, Bc, sig_ld, (const double*)g, g_ld, d_col_off, d_entries, d_term_word, d_cols,
          d_coef, max_factors, ncols, (double*)up, up_ld);
    SIGB_CUDA_TRY(cudaGetLastError());
  }
  return SIGB_OK;
}

extern "C" int sigb_tensor_mul(int dtype, const void* d_x, const void* d_y, int64_t B, int64_t d, int N, double scale,
                               double add0, void* d_out, void* stream) {
  if (dtype != SIGB_F32 && dtype != SIGB_F64) return fail(SIGB_ERR_SHAPE, "unsupported dtype; use float64 or float32");
  if (B < 0 || d < 1 || N < 0) return fail(SIGB_ERR_SHAPE, "bad truncated tensor shape");
  int64_t width = 0, pw = 1;
  for (int n = 0; n <= N; ++n) {
    width += pw;
    if (width > (int64_t(1) << 40)) return fail(SIGB_ERR_CAPACITY, "truncated tensor too wide");
    pw *= d;
  }
  if (B == 0) return SIGB_OK;
  const size_t es = dtype == SIGB_F32 ? 4 : 8;
  for (int64_t b0 = 0; b0 < B; b0 += kMaxGridY) {
    const int64_t Bc = std::min<int64_t>(kMaxGridY, B - b0);
    const size_t o = es * b0 * width;
    const dim3 grid((unsigned)((width + 255) / 256), (unsigned)Bc);
    count_launch();
    if (dtype == SIGB_F32)
      tensor_mul_kernel<float><<<grid, 256, 0, (cudaStream_t)stream>>>(
          (const float*)((const char*)d_x + o), (const float*)((const char*)d_y + o), Bc, d, N, width, (float)scale,
          (float)add0, (float*)((char*)d_out + o));
    else
      tensor_mul_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>(
          (const double*)((const char*)d_x + o), (const double*)((const char*)d_y + o), Bc, d, N, width, scale, add0,
          (double*)((char*)d_out + o));
    SIGB_CUDA_TRY(cudaGetLastError());
  }
  return SIGB_OK;
}
