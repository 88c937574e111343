// Instantiations and dispatch of the register-resident truncated kernels.
// A plan whose closure is a full truncation (all D^n words of every length
// 1..N) is routed here when (D, N) has an instantiation; everything else
// runs the generic trie kernels of sigb_level.cu.
#include <cstdlib>

#include <type_traits>

#include "sigb_trunc.cuh"
#include "sigb_trunc_tc.cuh"
#include "sigb_trunc_pq.cuh"

namespace sigb {
// Bytes of per-part gradient partials (+ checkpoints) per batch chunk of the backward: 1/16 of the
// device's memory, at most 8 GiB (SIGB_PARTIAL_BUDGET_MB overrides).  Fixed per process, so the
// workspace query and the launch always agree on the chunking.
size_t partial_budget() {
  static const size_t budget = [] {
    if (const char* e = getenv("SIGB_PARTIAL_BUDGET_MB")) return std::max<size_t>(64, (size_t)atoll(e)) << 20;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess || total_b == 0) {
      cudaGetLastError();
      return size_t(8) << 30;
    }
    return std::min<size_t>(size_t(8) << 30, std::max<size_t>(size_t(256) << 20, total_b / 16));
  }();
  return budget;
}

namespace trunc {
namespace {



template <typename T, int D, int N, int G>
int fwd(const T* X, int64_t B, int64_t L, const int64_t* bounds, int64_t K, T* out, int64_t out_ld, int64_t out_col0,
        int include_empty, cudaStream_t stream) {
  using C = Cfg<D, N, G>;
  const int64_t grid = C::CPP > 1 ? B * C::CPP : (B + C::PPC - 1) / C::PPC;
  if (grid == 0) return SIGB_OK;
  if constexpr (std::is_same<T, float>::value && D == 16 && N == 4) {
    // leaf level on the tensor cores (sigb_trunc_tc.cuh): c5 fwd 127.4 -> 65 ms.  (The kernel
    // also builds for d = 8, depth 5 with the MMA's N padded to 16; config 2 measured 2.0 ->
    // 2.3 ms per 1,024 paths there, so that set keeps the register kernel.)
    // SIGB_TRUNC_TC=0 selects the register kernel (A/B experiments, parity tests).
    const char* e = getenv("SIGB_TRUNC_TC");
    const int64_t grid_tc = B * Cfg<D, N, 4>::CPP;  // the tensor-core kernel's fragment: 4 parents per thread
    if (g_tensor_cores && !(e && atoi(e) == 0) && !bounds) {
      SIGB_CUDA_TRY(cudaFuncSetAttribute(tc::trunc_tc_forward_kernel<D, N>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc::kFwdSmem));
      count_launch();
      timing_begin(0, stream);
      tc::trunc_tc_forward_kernel<D, N><<<(unsigned)grid_tc, tc::kThreadsTc, tc::kFwdSmem, stream>>>(
          X, B, L, out, out_ld, out_col0, include_empty);
      timing_end(0, stream);
      SIGB_CUDA_TRY(cudaGetLastError());
      return SIGB_OK;
    }
  }
  constexpr size_t smem = 0;  // static shared memory only
  count_launch();
  timing_begin(0, stream);
  trunc_forward_kernel<T, D, N, G><<<(unsigned)grid, C::THREADS, smem, stream>>>(X, B, L, bounds, K, out, out_ld,
                                                                                out_col0, include_empty);
  timing_end(0, stream);
  SIGB_CUDA_TRY(cudaGetLastError());
  return SIGB_OK;
}

// checkpoint words per path for checkpoint_stride > 0: levels 1..N-1 at M / stride + 1 steps
template <int D, int N, int G>
size_t ckpt_words(int64_t L, int64_t stride) {
  return stride > 0 ? (size_t)((L - 1) / stride + 1) * (size_t)Cfg<D, N, G>::off(N) : 0;
}

template <typename T, int D, int N, int G>
int64_t bwd_chunk(int64_t B, int64_t L, int64_t stride = 0) {
  using C = Cfg<D, N, G>;
  const size_t per_path = sizeof(T) * ((size_t)C::CPP * (L - 1) * D + ckpt_words<D, N, G>(L, stride));
  int64_t chunk = per_path ? (int64_t)(partial_budget() / per_path) : B;
  chunk = std::max<int64_t>(C::PPC, chunk - chunk % C::PPC);
  return std::min<int64_t>(chunk, ((B + C::PPC - 1) / C::PPC) * C::PPC);
}

template <typename T, int D, int N, int G>
size_t bwd_workspace(int64_t B, int64_t L, int64_t stride = 0) {
  using C = Cfg<D, N, G>;
  return sizeof(T) * (size_t)bwd_chunk<T, D, N, G>(B, L, stride) *
         ((size_t)C::CPP * (L - 1) * D + ckpt_words<D, N, G>(L, stride));
}

// dL/dX from the per-part partials: dInc_j = sum_p partial[p][j] (parts in ascending order), then
// the telescoping dX_0 = -dInc_0, dX_t = dInc_{t-1} - dInc_t, dX_M = dInc_{M-1} (backward.py:130-147).
// A thread walks kSeg consecutive samples of one (path, channel), so each dInc is summed once
// (the per-sample form summed every increment twice); same arithmetic, same bits.
constexpr int kSeg = 32;
// 16-byte vectors of the partial / gradient rows (d is 4, 8 or 16 here): 4 floats or 2 doubles
template <typename T> struct Vec16;
template <> struct Vec16<float> { using V = float4; static constexpr int W = 4; };
template <> struct Vec16<double> { using V = double2; static constexpr int W = 2; };
__device__ __forceinline__ float4 vadd(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
__device__ __forceinline__ float4 vsub(float4 a, float4 b) { return make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w); }
__device__ __forceinline__ double2 vadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 vsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
template <typename V> __device__ __forceinline__ V vzero();
template <> __device__ __forceinline__ float4 vzero<float4>() { return make_float4(0.f, 0.f, 0.f, 0.f); }
template <> __device__ __forceinline__ double2 vzero<double2>() { return make_double2(0.0, 0.0); }

// Scalar fallback for buffers the caller did not 16-byte align: thread = (path, segment, letter)
template <typename T>
__global__ void trunc_sample_grads_scalar(const T* __restrict__ partial, int64_t Bc, int64_t P, int64_t M,
                                          int64_t d, int64_t b0, int64_t B, T* __restrict__ dX,
                                          T* __restrict__ dinc) {
  const int64_t L = M + 1, nseg = (L + kSeg - 1) / kSeg;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= Bc * nseg * d) return;
  const int64_t z = i % d, sg = (i / d) % nseg, bl = i / (d * nseg);
  if (b0 + bl >= B) return;
  auto inc = [&](int64_t j) {
    T s = T(0);
    for (int64_t p = 0; p < P; ++p) s += partial[((bl * P + p) * M + j) * d + z];
    return s;
  };
  const int64_t t0 = sg * kSeg, t1 = t0 + kSeg < L ? t0 + kSeg : L;
  T prev = t0 >= 1 ? inc(t0 - 1) : T(0);
  for (int64_t t = t0; t < t1; ++t) {
    T v = t >= 1 ? prev : T(0);
    if (t < M) {
      const T it = inc(t);
      v -= it;
      if (dinc) dinc[((b0 + bl) * M + t) * d + z] = it;
      prev = it;
    }
    dX[((b0 + bl) * L + t) * d + z] = v;
  }
}

// dX[t] = inc(t-1) - inc(t), inc(j) = sum over the path's CTA parts of partial[part][j] (fixed
// part order); thread = (path, 32-sample segment, 16-byte group of letters), vector loads/stores
template <typename T>
__global__ void trunc_sample_grads(const T* __restrict__ partial, int64_t Bc, int64_t P, int64_t M, int64_t d,
                                   int64_t b0, int64_t B, T* __restrict__ dX, T* __restrict__ dinc) {
  using V = typename Vec16<T>::V;
  constexpr int W = Vec16<T>::W;
  const int64_t L = M + 1, nseg = (L + kSeg - 1) / kSeg, dv = d / W;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= Bc * nseg * dv) return;
  const int64_t zv = i % dv, sg = (i / dv) % nseg, bl = i / (dv * nseg);
  if (b0 + bl >= B) return;
  const V* pv = reinterpret_cast<const V*>(partial);
  auto inc = [&](int64_t j) {
    V s = vzero<V>();
    for (int64_t p = 0; p < P; ++p) s = vadd(s, pv[((bl * P + p) * M + j) * dv + zv]);
    return s;
  };
  V* xv = reinterpret_cast<V*>(dX);
  V* iv = reinterpret_cast<V*>(dinc);
  const int64_t t0 = sg * kSeg, t1 = t0 + kSeg < L ? t0 + kSeg : L;
  V prev = t0 >= 1 ? inc(t0 - 1) : vzero<V>();
  for (int64_t t = t0; t < t1; ++t) {
    V v = t >= 1 ? prev : vzero<V>();
    if (t < M) {
      const V it = inc(t);
      v = vsub(v, it);
      if (dinc) iv[((b0 + bl) * M + t) * dv + zv] = it;
      prev = it;
    }
    xv[((b0 + bl) * L + t) * dv + zv] = v;
  }
}

template <typename T, int D, int N, int G>
int bwd(const T* X, int64_t B, int64_t L, const T* S, int64_t s_ld, int64_t s_col0, const T* g, int64_t g_ld,
        int64_t g_col0, void* work, size_t work_bytes, T* dX, T* dinc, cudaStream_t stream, int64_t stride) {
  using C = Cfg<D, N, G>;
  using RG = RedGeom<D, N, G>;
  const int64_t M = L - 1;
  const int64_t chunk = bwd_chunk<T, D, N, G>(B, L, stride);
  if (work_bytes < bwd_workspace<T, D, N, G>(B, L, stride) || !work)
    return fail(SIGB_ERR_DOMAIN, "backward workspace too small");
  size_t smem = RG::template smem_bytes<T>();
  // experiment knob: SIGB_TRUNC_ASYNC=0/1 forces the staging mode (default: D >= 16)
  static const int force_async = getenv("SIGB_TRUNC_ASYNC") ? atoi(getenv("SIGB_TRUNC_ASYNC")) : -1;
  const bool async = force_async < 0 ? (D >= 16) : force_async != 0;
  auto kern = stride > 0 ? (async ? trunc_backward_kernel<T, D, N, G, true, false, true>
                                  : trunc_backward_kernel<T, D, N, G, false, false, true>)
                         : (async ? trunc_backward_kernel<T, D, N, G, true> : trunc_backward_kernel<T, D, N, G, false>);
  // leaf level on the tensor cores (fp32, d = 16 depth 4 and d = 8 depth 5).  SIGB_TRUNC_TC_BWD
  // selects: 2 (default) the P/Q kernel (sigb_trunc_pq.cuh, both leaf sums on tcgen05), 1 the
  // parent pull-back only on tcgen05 (TcBwd, d = 16 only), 0 the CUDA-core kernel (A/B
  // experiments, parity tests); checkpoints and sigb_set_tensor_cores(0) take the CUDA cores
  constexpr bool kPQ = std::is_same<T, float>::value && ((D == 16 && N == 4) || (D == 8 && N == 5));
  bool pq_kernel = false;
  if constexpr (kPQ) {
    const char* e = getenv("SIGB_TRUNC_TC_BWD");
    const int mode = (stride > 0 || !g_tensor_cores) ? 0 : (e ? atoi(e) : 2);
    if (mode == 2) {
      static_assert(pq::PQ<D, N>::CPP == C::CPP, "the P/Q kernel fills the same partial layout");
      pq_kernel = true;
      smem = pq::PQ<D, N>::kSmem;
      SIGB_CUDA_TRY(cudaFuncSetAttribute(pq::trunc_pq_backward_kernel<D, N>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    } else if constexpr (D == 16 && G == 4) {
      if (mode == 1 && force_async != 0) {
        kern = trunc_backward_kernel<T, D, N, G, true, true>;
        smem += TcBwd::bytes;
      }
    }
  }
  if (!pq_kernel) SIGB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  T* partial = (T*)work;
  T* ckpt = stride > 0 ? partial + (size_t)chunk * C::CPP * M * D : nullptr;
  for (int64_t b0 = 0; b0 < B; b0 += chunk) {
    const int64_t Bc = std::min(chunk, B - b0);
    const int64_t grid = C::CPP > 1 ? Bc * C::CPP : (Bc + C::PPC - 1) / C::PPC;
    if (stride > 0) {
      count_launch();
      trunc_ckpt_kernel<T, D, N, G><<<(unsigned)grid, C::THREADS, 0, stream>>>(X, B, L, b0, stride, ckpt);
      SIGB_CUDA_TRY(cudaGetLastError());
    }
    count_launch(2);
    timing_begin(1, stream);
    if constexpr (kPQ) {
      if (pq_kernel)
        pq::trunc_pq_backward_kernel<D, N><<<(unsigned)grid, pq::kBlock, smem, stream>>>(X, B, L, b0, S, s_ld, s_col0,
                                                                                           g, g_ld, g_col0, partial);
      else
        kern<<<(unsigned)grid, C::THREADS, smem, stream>>>(X, B, L, b0, S, s_ld, s_col0, g, g_ld, g_col0, partial,
                                                           ckpt, stride);
    } else {
      kern<<<(unsigned)grid, C::THREADS, smem, stream>>>(X, B, L, b0, S, s_ld, s_col0, g, g_ld, g_col0, partial,
                                                         ckpt, stride);
    }
    timing_end(1, stream);
    SIGB_CUDA_TRY(cudaGetLastError());
    if ((((uintptr_t)partial | (uintptr_t)dX | (uintptr_t)dinc) & 15) == 0) {
      const int64_t n = Bc * ((L + kSeg - 1) / kSeg) * (D / Vec16<T>::W);
      trunc_sample_grads<T><<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(partial, Bc, C::CPP, M, D, b0, B, dX,
                                                                             dinc);
    } else {
      const int64_t n = Bc * ((L + kSeg - 1) / kSeg) * D;
      trunc_sample_grads_scalar<T><<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(partial, Bc, C::CPP, M, D, b0,
                                                                                    B, dX, dinc);
    }
    SIGB_CUDA_TRY(cudaGetLastError());
  }
  return SIGB_OK;
}

// (D, N) -> (G forward, G backward).  The forward and backward kernels share
// only the output layout, so each picks its own fragment width: G = D where
// the fragment fits the register budget, smaller where occupancy pays more
// (d=8, N=5 backward: 168 registers at G=8 leave 8 warps per SM).
#define SIGB_TRUNC_CASES(X) \
  X(4, 4, 4, 4)             \
  X(4, 5, 4, 4)             \
  X(4, 6, 4, 4)             \
  X(8, 4, 8, 8)             \
  X(8, 5, 8, 4)             \
  X(16, 3, 4, 4)            \
  X(16, 4, 4, 4)

}  // namespace

int64_t forward_ctas(int64_t d, int depth, int64_t B) {
#define X(D_, N_, GF_, GB_)                                                      \
  if (d == D_ && depth == N_) {                                                  \
    using C = Cfg<D_, N_, GF_>;                                                  \
    return C::CPP > 1 ? B * C::CPP : (B + C::PPC - 1) / C::PPC;                  \
  }
  SIGB_TRUNC_CASES(X)
#undef X
  return -1;
}

bool supported(int64_t d, int depth) {
#define X(D_, N_, GF_, GB_) \
  if (d == D_ && depth == N_) return true;
  SIGB_TRUNC_CASES(X)
#undef X
  return false;
}

int forward(int dtype, int64_t d, int depth, const void* X, int64_t B, int64_t L, const int64_t* bounds, int64_t K,
            void* out, int64_t out_ld, int64_t out_col0, int include_empty, cudaStream_t stream) {
#define X(D_, N_, GF_, GB_)                                                                                \
  if (d == D_ && depth == N_) {                                                                            \
    if (dtype == SIGB_F32)                                                                                 \
      return fwd<float, D_, N_, GF_>((const float*)X, B, L, bounds, K, (float*)out, out_ld, out_col0,       \
                                     include_empty, stream);                                               \
    return fwd<double, D_, N_, GF_>((const double*)X, B, L, bounds, K, (double*)out, out_ld, out_col0,     \
                                    include_empty, stream);                                                \
  }
  SIGB_TRUNC_CASES(X)
#undef X
  return fail(SIGB_ERR_UNSUPPORTED, "no truncated kernel for this (d, depth)");
}

size_t backward_workspace(int dtype, int64_t d, int depth, int64_t B, int64_t L, int64_t stride) {
#define X(D_, N_, GF_, GB_)                                                                                \
  if (d == D_ && depth == N_)                                                                              \
    return dtype == SIGB_F32 ? bwd_workspace<float, D_, N_, GB_>(B, L, stride)                             \
                             : bwd_workspace<double, D_, N_, GB_>(B, L, stride);
  SIGB_TRUNC_CASES(X)
#undef X
  return 0;
}

int backward(int dtype, int64_t d, int depth, const void* X, int64_t B, int64_t L, const void* S, int64_t s_ld,
             int64_t s_col0, const void* g, int64_t g_ld, int64_t g_col0, void* work, size_t work_bytes, void* dX,
             void* dinc, cudaStream_t stream, int64_t stride) {
#define X(D_, N_, GF_, GB_)                                                                                       \
  if (d == D_ && depth == N_) {                                                                                   \
    if (dtype == SIGB_F32)                                                                                        \
      return bwd<float, D_, N_, GB_>((const float*)X, B, L, (const float*)S, s_ld, s_col0, (const float*)g, g_ld,  \
                                    g_col0, work, work_bytes, (float*)dX, (float*)dinc, stream, stride);          \
    return bwd<double, D_, N_, GB_>((const double*)X, B, L, (const double*)S, s_ld, s_col0, (const double*)g,     \
                                   g_ld, g_col0, work, work_bytes, (double*)dX, (double*)dinc, stream, stride);   \
  }
  SIGB_TRUNC_CASES(X)
#undef X
  return fail(SIGB_ERR_UNSUPPORTED, "no truncated kernel for this (d, depth)");
}

}  // namespace trunc
}  // namespace sigb
