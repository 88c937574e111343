// Instantiations and dispatch of the level-slot kernels (sigb_slot.cuh).
#include <algorithm>

#include "sigb_slot.cuh"

namespace sigb {
namespace slot {
namespace {

constexpr size_t kPartialBudget = size_t(4) << 30;

SlotDev dev_of(const sigb_plan* p) {
  const SlotHost& h = p->slot.h;
  SlotDev s;
  s.tinfo = p->slot.tinfo;
  s.meta0 = p->slot.meta0;
  s.meta1 = p->slot.meta1;
  s.pos = p->slot.pos;
  s.cidx = p->slot.cidx;
  s.eidx = p->slot.eidx;
  s.lvl = p->slot.lvl;
  s.red_off = p->slot.red_off;
  s.TPB = h.TPB;
  s.d = (int)p->d;
  s.N = h.N;
  s.t_size = h.t_size;
  s.p_size = h.p_size;
  s.a_off = h.a_off;
  s.t_off = h.t_off;
  s.tm_off = h.tm_off;
  s.p_off = h.p_off;
  s.park_off = h.park_off;
  s.pstride = h.pstride;
  s.smem_floats = h.bwd_smem;
  return s;
}

template <typename T, int N>
int fwd(const sigb_plan* p, const T* X, int64_t B, int64_t L, T* out, int64_t out_ld, int64_t out_col0,
        int include_empty, T* state, cudaStream_t stream) {
  if (B == 0) return SIGB_OK;
  const size_t smem = sizeof(T) * (size_t)p->slot.h.fwd_smem;
  SIGB_CUDA_TRY(cudaFuncSetAttribute(slot_forward_kernel<T, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  count_launch();
  timing_begin(0, stream);
  slot_forward_kernel<T, N><<<(unsigned)B, p->slot.h.TPB, smem, stream>>>(dev_of(p), X, L, out, out_ld, out_col0,
                                                                          include_empty, state, p->Wc);
  timing_end(0, stream);
  SIGB_CUDA_TRY(cudaGetLastError());
  return SIGB_OK;
}

template <typename T>
int64_t bwd_chunk(const sigb_plan* p, int64_t B, int64_t L) {
  const size_t per_path = sizeof(T) * (size_t)(L - 1) * p->d;
  int64_t c = per_path ? (int64_t)(kPartialBudget / per_path) : B;
  return std::max<int64_t>(1, std::min(c, B));
}

template <typename T>
__global__ void slot_sample_grads(const T* __restrict__ partial, int64_t Bc, int64_t M, int64_t d, int64_t b0,
                                  T* __restrict__ dX, T* __restrict__ dinc) {
  const int64_t L = M + 1;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= Bc * L * d) return;
  const int64_t z = i % d, t = (i / d) % L, bl = i / (d * L);
  T v = T(0);
  if (t >= 1) v += partial[(bl * M + t - 1) * d + z];
  if (t < M) {
    const T it = partial[(bl * M + t) * d + z];
    v -= it;
    if (dinc) dinc[((b0 + bl) * M + t) * d + z] = it;
  }
  dX[((b0 + bl) * L + t) * d + z] = v;
}

template <typename T, int N>
int bwd(const sigb_plan* p, const T* X, int64_t B, int64_t L, const T* S, int64_t s_ld, int64_t s_col0, const T* g,
        int64_t g_ld, int64_t g_col0, void* work, size_t work_bytes, T* dX, T* dinc, cudaStream_t stream) {
  const int d = (int)p->d;
  const int64_t M = L - 1;
  const int64_t chunk = bwd_chunk<T>(p, B, L);
  if (!work || work_bytes < sizeof(T) * (size_t)chunk * M * d) return fail(SIGB_ERR_DOMAIN, "backward workspace too small");
  const size_t smem = sizeof(T) * (size_t)p->slot.h.bwd_smem;
  SIGB_CUDA_TRY(cudaFuncSetAttribute(slot_backward_kernel<T, N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  T* partial = (T*)work;
  for (int64_t b0 = 0; b0 < B; b0 += chunk) {
    const int64_t Bc = std::min(chunk, B - b0);
    count_launch(2);
    timing_begin(1, stream);
    slot_backward_kernel<T, N><<<(unsigned)Bc, p->slot.h.TPB, smem, stream>>>(dev_of(p), X, L, b0, S, s_ld, s_col0, g,
                                                                              g_ld, g_col0, partial);
    timing_end(1, stream);
    SIGB_CUDA_TRY(cudaGetLastError());
    const int64_t n = Bc * L * d;
    slot_sample_grads<T><<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(partial, Bc, M, d, b0, dX, dinc);
    SIGB_CUDA_TRY(cudaGetLastError());
  }
  return SIGB_OK;
}

#define SIGB_SLOT_CASES(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7)

}  // namespace

bool supported(int N) { return N >= 1 && N <= 7; }

int forward(const sigb_plan* p, int dtype, const void* Xv, int64_t B, int64_t L, void* out, int64_t out_ld,
            int64_t out_col0, int include_empty, void* state, cudaStream_t stream) {
  const int N = p->slot.h.N;
#define X(n)                                                                                                      \
  if (N == n) {                                                                                                   \
    if (dtype == SIGB_F32)                                                                                        \
      return fwd<float, n>(p, (const float*)Xv, B, L, (float*)out, out_ld, out_col0, include_empty, (float*)state, \
                           stream);                                                                               \
    return fwd<double, n>(p, (const double*)Xv, B, L, (double*)out, out_ld, out_col0, include_empty,              \
                          (double*)state, stream);                                                                \
  }
  SIGB_SLOT_CASES(X)
#undef X
  return fail(SIGB_ERR_UNSUPPORTED, "no level-slot kernel for this depth");
}

size_t backward_workspace(const sigb_plan* p, int dtype, int64_t B, int64_t L) {
  const size_t es = dtype == SIGB_F32 ? 4 : 8;
  const int64_t chunk = dtype == SIGB_F32 ? bwd_chunk<float>(p, B, L) : bwd_chunk<double>(p, B, L);
  return es * (size_t)chunk * (size_t)(L - 1) * p->d;
}

int backward(const sigb_plan* p, int dtype, const void* Xv, int64_t B, int64_t L, const void* S, int64_t s_ld,
             int64_t s_col0, const void* g, int64_t g_ld, int64_t g_col0, void* work, size_t work_bytes, void* dX,
             void* dinc, cudaStream_t stream) {
  const int N = p->slot.h.N;
#define X(n)                                                                                                         \
  if (N == n) {                                                                                                      \
    if (dtype == SIGB_F32)                                                                                           \
      return bwd<float, n>(p, (const float*)Xv, B, L, (const float*)S, s_ld, s_col0, (const float*)g, g_ld, g_col0, \
                           work, work_bytes, (float*)dX, (float*)dinc, stream);                                      \
    return bwd<double, n>(p, (const double*)Xv, B, L, (const double*)S, s_ld, s_col0, (const double*)g, g_ld,      \
                          g_col0, work, work_bytes, (double*)dX, (double*)dinc, stream);                             \
  }
  SIGB_SLOT_CASES(X)
#undef X
  return fail(SIGB_ERR_UNSUPPORTED, "no level-slot kernel for this depth");
}

}  // namespace slot
}  // namespace sigb
