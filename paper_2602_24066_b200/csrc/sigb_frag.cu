// Instantiations and dispatch of the fragment kernels (sigb_frag.cuh).
#include <algorithm>

#include "sigb_frag.cuh"

namespace sigb {
namespace frag {
namespace {


FragDev dev_of(const sigb_plan* p) {
  FragDev f;
  f.letter = p->frag.letter;
  f.cidx = p->frag.cidx;
  f.eidx = p->frag.eidx;
  f.sidx = p->frag.sidx;
  f.pos = p->frag.pos;
  f.red_off = p->frag.red_off;
  f.pstride = p->frag.pstride;
  f.Fp = p->frag.Fp;
  f.cpp = p->frag.cpp;
  f.d = (int)p->d;
  return f;
}

template <typename T, int NC, int G, int K>
int fwd(const sigb_plan* p, const T* X, int64_t B, int64_t L, const int64_t* bounds, int64_t nwin, T* out,
        int64_t out_ld, int64_t out_col0, int include_empty, T* state, cudaStream_t stream) {
  const int d = (int)p->d;
  const int64_t grid = B * p->frag.cpp;
  if (grid == 0) return SIGB_OK;
  const size_t smem = sizeof(T) * (2 * (size_t)(kChunkF + 1) * d + (size_t)kChunkF * (d + 1));
  if (smem > 48 * 1024)
    SIGB_CUDA_TRY(cudaFuncSetAttribute(frag_forward_kernel<T, NC, G, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
  count_launch();
  timing_begin(0, stream);
  frag_forward_kernel<T, NC, G, K><<<(unsigned)grid, kTPB, smem, stream>>>(dev_of(p), X, L, bounds, nwin, out, out_ld,
                                                                            out_col0, include_empty, state, p->Wc);
  timing_end(0, stream);
  SIGB_CUDA_TRY(cudaGetLastError());
  return SIGB_OK;
}

// checkpoint rows per path (checkpoint_stride > 0): the chain and mid slots of every fragment at
// k = 0, stride, 2 stride, ... (frag_ckpt_kernel)
size_t ckpt_elems(const sigb_plan* p, int64_t L, int64_t stride, int NS) {
  return stride > 0 ? (size_t)((L - 1) / stride + 1) * NS * p->frag.Fp : 0;
}

template <typename T>
int64_t bwd_chunk(const sigb_plan* p, int64_t B, int64_t L, int64_t stride = 0) {
  const size_t per_path = sizeof(T) * ((size_t)p->frag.cpp * (size_t)(L - 1) * p->d +
                                       ckpt_elems(p, L, stride, p->frag.NC + p->frag.G));
  int64_t c = per_path ? (int64_t)(partial_budget() / 2 / per_path) : B;
  return std::max<int64_t>(1, std::min(c, B));
}

template <typename T>
__global__ void frag_sample_grads(const T* __restrict__ partial, int64_t Bc, int64_t P, int64_t M, int64_t d,
                                  int64_t b0, T* __restrict__ dX, T* __restrict__ dinc) {
  const int64_t L = M + 1;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= Bc * L * d) return;
  const int64_t z = i % d, t = (i / d) % L, bl = i / (d * L);
  auto inc = [&](int64_t j) {
    T s = T(0);
    for (int64_t q = 0; q < P; ++q) s += partial[((bl * P + q) * M + j) * d + z];
    return s;
  };
  T v = T(0);
  if (t >= 1) v += inc(t - 1);
  if (t < M) {
    const T it = inc(t);
    v -= it;
    if (dinc) dinc[((b0 + bl) * M + t) * d + z] = it;
  }
  dX[((b0 + bl) * L + t) * d + z] = v;
}

template <typename T, int NC, int G, int K>
int bwd(const sigb_plan* p, const T* X, int64_t B, int64_t L, const T* S, int64_t s_ld, int64_t s_col0, const T* g,
        int64_t g_ld, int64_t g_col0, void* work, size_t work_bytes, T* dX, T* dinc, cudaStream_t stream,
        int64_t stride) {
  const int d = (int)p->d;
  const int64_t M = L - 1;
  const int cpp = p->frag.cpp;
  const int64_t chunk = bwd_chunk<T>(p, B, L, stride);
  const size_t part = (size_t)chunk * cpp * M * d;
  const size_t need = sizeof(T) * (part + (size_t)chunk * ckpt_elems(p, L, stride, NC + G));
  if (!work || work_bytes < need) return fail(SIGB_ERR_DOMAIN, "backward workspace too small");
  const size_t smem = sizeof(T) * bwd_smem_elems<NC, G, K>(d, p->frag.pstride);
  auto kern = stride > 0 ? frag_backward_kernel<T, NC, G, K, true> : frag_backward_kernel<T, NC, G, K, false>;
  SIGB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const size_t csmem = sizeof(T) * (2 * (size_t)(kChunkF + 1) * d + (size_t)kChunkF * (d + 1));
  if (stride > 0 && csmem > 48 * 1024)
    SIGB_CUDA_TRY(cudaFuncSetAttribute(frag_ckpt_kernel<T, NC, G, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)csmem));
  T* partial = (T*)work;
  T* ckpt = stride > 0 ? partial + part : nullptr;
  for (int64_t b0 = 0; b0 < B; b0 += chunk) {
    const int64_t Bc = std::min(chunk, B - b0);
    if (stride > 0) {
      count_launch();
      frag_ckpt_kernel<T, NC, G, K><<<(unsigned)(Bc * cpp), kTPB, csmem, stream>>>(dev_of(p), X, L, b0, stride, ckpt);
      SIGB_CUDA_TRY(cudaGetLastError());
    }
    count_launch(2);
    timing_begin(1, stream);
    kern<<<(unsigned)(Bc * cpp), kTPB, smem, stream>>>(dev_of(p), X, L, b0, S, s_ld, s_col0, g, g_ld, g_col0, partial,
                                                       ckpt, stride);
    timing_end(1, stream);
    SIGB_CUDA_TRY(cudaGetLastError());
    const int64_t n = Bc * L * d;
    frag_sample_grads<T><<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(partial, Bc, cpp, M, d, b0, dX, dinc);
    SIGB_CUDA_TRY(cudaGetLastError());
  }
  return SIGB_OK;
}

#define SIGB_FRAG_GK(X, NC) X(NC, 5, 5) X(NC, 4, 4) X(NC, 2, 8) X(NC, 1, 16)
#define SIGB_FRAG_CASES(X) SIGB_FRAG_GK(X, 1) SIGB_FRAG_GK(X, 2) SIGB_FRAG_GK(X, 3) SIGB_FRAG_GK(X, 4) SIGB_FRAG_GK(X, 5)

}  // namespace

bool supported(int NC, int G, int K) {
#define X(a, b, c) \
  if (NC == a && G == b && K == c) return true;
  SIGB_FRAG_CASES(X)
#undef X
  return false;
}

int forward(const sigb_plan* p, int dtype, const void* Xv, int64_t B, int64_t L, const int64_t* bounds, int64_t nwin,
            void* out, int64_t out_ld, int64_t out_col0, int include_empty, void* state, cudaStream_t stream) {
  const int NC = p->frag.NC, G = p->frag.G, K = p->frag.K;
#define X(a, b, c)                                                                                               \
  if (NC == a && G == b && K == c) {                                                                             \
    if (dtype == SIGB_F32)                                                                                       \
      return fwd<float, a, b, c>(p, (const float*)Xv, B, L, bounds, nwin, (float*)out, out_ld, out_col0,            \
                                 include_empty, (float*)state, stream);                                          \
    return fwd<double, a, b, c>(p, (const double*)Xv, B, L, bounds, nwin, (double*)out, out_ld, out_col0,           \
                                include_empty, (double*)state, stream);                                          \
  }
  SIGB_FRAG_CASES(X)
#undef X
  return fail(SIGB_ERR_UNSUPPORTED, "no fragment kernel for this shape");
}

size_t backward_workspace(const sigb_plan* p, int dtype, int64_t B, int64_t L, int64_t stride) {
  const size_t es = dtype == SIGB_F32 ? 4 : 8;
  const int64_t chunk = dtype == SIGB_F32 ? bwd_chunk<float>(p, B, L, stride) : bwd_chunk<double>(p, B, L, stride);
  return es * (size_t)chunk *
         ((size_t)p->frag.cpp * (size_t)(L - 1) * p->d + ckpt_elems(p, L, stride, p->frag.NC + p->frag.G));
}

int backward(const sigb_plan* p, int dtype, const void* Xv, int64_t B, int64_t L, const void* S, int64_t s_ld,
             int64_t s_col0, const void* g, int64_t g_ld, int64_t g_col0, void* work, size_t work_bytes, void* dX,
             void* dinc, cudaStream_t stream, int64_t stride) {
  const int NC = p->frag.NC, G = p->frag.G, K = p->frag.K;
#define X(a, b, c)                                                                                                 \
  if (NC == a && G == b && K == c) {                                                                               \
    if (dtype == SIGB_F32)                                                                                         \
      return bwd<float, a, b, c>(p, (const float*)Xv, B, L, (const float*)S, s_ld, s_col0, (const float*)g, g_ld,  \
                                 g_col0, work, work_bytes, (float*)dX, (float*)dinc, stream, stride);              \
    return bwd<double, a, b, c>(p, (const double*)Xv, B, L, (const double*)S, s_ld, s_col0, (const double*)g,      \
                                g_ld, g_col0, work, work_bytes, (double*)dX, (double*)dinc, stream, stride);       \
  }
  SIGB_FRAG_CASES(X)
#undef X
  return fail(SIGB_ERR_UNSUPPORTED, "no fragment kernel for this shape");
}

}  // namespace frag
}  // namespace sigb
