// Register-resident Chen kernels for ARBITRARY prefix-closed tries
// (anisotropic truncations, user word sets: configs 3 and 4 of BASELINE.json,
// and full truncations without a dedicated sigb_trunc instantiation).
//
// Work decomposition (built by the planner in sigb_plan.cu).  Every thread
// owns one FRAGMENT of the trie for the whole time sweep, in registers:
//   - an anchor node a (any internal node whose children are not all leaves,
//     or the empty word) and its chain of ancestors,
//   - up to G "mids": children of a whose own children are all leaves,
//   - for every mid, up to K leaf children drawn from one fragment-wide list
//     of K letters LL (a mid that lacks LL[k] simply carries a dead register),
//   - up to K leaf children of a itself ("anchor leaves", letters AL).
// The generalisation of sigb_trunc's fragment is the chain: its length (the
// anchor's level) varies per thread, so chains are RIGHT-ALIGNED to a common
// length NC and padded at the front with identity nodes (S = 1, increment 0),
// for which the Horner recursion reproduces T(eps, m) = 1 exactly.  All levels
// are then "virtual" (real level + NC - |a|); the Horner factors 1/(m-|u|+1)
// only see level differences, so they are unchanged.
//
// Forward step per thread (PAPER.md:190-216 in the shared-prefix form of
// sigb_level.cu):  sum_{k<NC} (NV-k) chain + 2G mid + G*K leaf + K anchor-leaf
// FMAs, NV = NC + 2.  Increments are gathered per step from a shared-memory row
// (one LDS per letter slot; the row carries a zero column at index d for empty
// slots).
//
// Backward: the memory-lean reverse sweep of sigb_trunc (rebuild S by
// exp(-dX), partials, reverse mode; leaf adjoints are constant in time).  The
// per-step gradient terms of a thread belong to letters known only at run
// time, so they are parked in shared memory (slot-major, conflict-free) and
// summed per letter through the plan's fixed-order CSR lists: deterministic,
// no atomics.
#pragma once

#include "sigb_internal.h"

namespace sigb {
namespace frag {

constexpr int kTPB = 128;      // threads (fragments) per CTA
constexpr int kChunkF = 16;    // steps of samples staged per chunk
constexpr int kRedSteps = 4;   // steps per gradient-reduction round (bwd)

template <int NC, int G, int K>
struct Shape {
  static constexpr int NV = NC + 2;                 // virtual depth
  static constexpr int NS = NC + G + G * K + K;     // state slots
  static constexpr int NGS = NC + G + 2 * K;        // letter / gradient slots
  // slot order (state): chain [0,NC) | mids [NC,NC+G) | leaves [.., +G*K) g-major | anchor leaves
  // slot order (letters): chain | mids | LL[K] | AL[K]
};

template <typename T, int NC, int G, int K>
struct FState {
  T ch[NC];
  T mid[G];
  T leaf[G][K];
  T al[K];
};

template <typename T, int NC, int G, int K>
struct FIncr {
  T dc[NC];
  T dy[G];
  T dz[K];
  T da[K];
};

template <typename T>
__device__ __forceinline__ T rinv(int r) {
  return T(1) / T(r);
}

// Per-thread letter offsets into the staged increment row (letter d = zero column).
template <int NC, int G, int K>
struct Letters {
  int c[NC], y[G], z[K], a[K];
};

template <typename T, int NC, int G, int K>
__device__ __forceinline__ void gather(const T* __restrict__ row, const Letters<NC, G, K>& lt, T sign,
                                       FIncr<T, NC, G, K>& in) {
#pragma unroll
  for (int k = 0; k < NC; ++k) in.dc[k] = sign * row[lt.c[k]];
#pragma unroll
  for (int g = 0; g < G; ++g) in.dy[g] = sign * row[lt.y[g]];
#pragma unroll
  for (int k = 0; k < K; ++k) in.dz[k] = sign * row[lt.z[k]];
#pragma unroll
  for (int k = 0; k < K; ++k) in.da[k] = sign * row[lt.a[k]];
}

// tch[k][m] = T(chain_k, m), m = k+1 .. NV (virtual levels).
template <typename T, int NC, int G, int K>
__device__ __forceinline__ void chain_partials(const FState<T, NC, G, K>& st, const FIncr<T, NC, G, K>& in,
                                               T (&tch)[NC][NC + 3]) {
  constexpr int NV = NC + 2;
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int lv = k + 1;
#pragma unroll
    for (int m = lv; m <= NV; ++m) {
      const T a = (m == lv) ? in.dc[k] : in.dc[k] * rinv<T>(m - lv + 1);
      tch[k][m] = (k == 0) ? st.ch[k] + a : fma(a, tch[k > 0 ? k - 1 : 0][m], st.ch[k]);
    }
  }
}

// Leaves = false (backward reconstruction): leaf values are never read there.
template <typename T, int NC, int G, int K, bool Leaves = true>
__device__ __forceinline__ void chen_step(FState<T, NC, G, K>& st, const FIncr<T, NC, G, K>& in) {
  constexpr int NV = NC + 2;
  T tch[NC][NC + 3];
  chain_partials<T, NC, G, K>(st, in, tch);
  const T tN1 = tch[NC - 1][NV - 1];
  const T tN = tch[NC - 1][NV];
#pragma unroll
  for (int k = 0; k < NC; ++k) st.ch[k] = tch[k][k + 1];
  const T tNh = tN * T(0.5);  // dX/2 . T(anchor, NV) as dX . (T/2): exact, one scaling per step
  if constexpr (!Leaves && sizeof(T) == 4) {
    // the backward's reconstruction (no leaves): two mids' S += dX . T(anchor, NV-1) per packed
    // f32x2 FMA
#pragma unroll
    for (int g = 0; g + 1 < G; g += 2) {
      const float2 n2 = __ffma2_rn(make_float2(in.dy[g], in.dy[g + 1]), make_float2(tN1, tN1),
                                   make_float2(st.mid[g], st.mid[g + 1]));
      st.mid[g] = n2.x;
      st.mid[g + 1] = n2.y;
    }
    if constexpr (G % 2) st.mid[G - 1] = fma(in.dy[G - 1], tN1, st.mid[G - 1]);
    return;
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if constexpr (Leaves) {
      const T tm = fma(in.dy[g], tNh, st.mid[g]);  // T(mid_g, NV)
      if constexpr (sizeof(T) == 4) {
        // packed f32x2 FMAs for pairs of leaves (half the issue slots)
        const float2 tm2 = make_float2(tm, tm);
#pragma unroll
        for (int k = 0; k + 1 < K; k += 2) {
          const float2 r = __ffma2_rn(make_float2(in.dz[k], in.dz[k + 1]), tm2,
                                      make_float2(st.leaf[g][k], st.leaf[g][k + 1]));
          st.leaf[g][k] = r.x;
          st.leaf[g][k + 1] = r.y;
        }
        if constexpr (K % 2) st.leaf[g][K - 1] = fma(in.dz[K - 1], tm, st.leaf[g][K - 1]);
      } else {
#pragma unroll
        for (int k = 0; k < K; ++k) st.leaf[g][k] = fma(in.dz[k], tm, st.leaf[g][k]);
      }
    }
    st.mid[g] = fma(in.dy[g], tN1, st.mid[g]);
  }
  if constexpr (Leaves) {
#pragma unroll
    for (int k = 0; k < K; ++k) st.al[k] = fma(in.da[k], tN1, st.al[k]);
  }
}

// Device view of a fragment plan.  Per-fragment arrays are slot-major
// ([slot][Fp]) so that a warp's loads are coalesced.
struct FragDev {
  const unsigned char* letter;  // [NGS][Fp] letter of the slot, d = none
  const int* cidx;              // [NS][Fp] closure index to read S (-1 empty, -2 identity)
  const int* eidx;              // [NS][Fp] emitted index in I (owner only) or -1
  const int* sidx;              // [NS][Fp] closure index to write state (owner only) or -1
  const unsigned short* pos;    // [NGS][Fp] parking offset of the slot's gradient term (bwd)
  const int* red_off;           // [cpp][d + 1] letter blocks of the parking buffer, float4 units
  int Fp, cpp, d, pstride;
};

template <int NC, int G, int K>
__device__ __forceinline__ void load_letters(const FragDev& fd, int f, Letters<NC, G, K>& lt) {
  using SH = Shape<NC, G, K>;
  const unsigned char* L = fd.letter + f;
#pragma unroll
  for (int k = 0; k < NC; ++k) lt.c[k] = L[(size_t)k * fd.Fp];
#pragma unroll
  for (int g = 0; g < G; ++g) lt.y[g] = L[(size_t)(NC + g) * fd.Fp];
#pragma unroll
  for (int k = 0; k < K; ++k) lt.z[k] = L[(size_t)(NC + G + k) * fd.Fp];
#pragma unroll
  for (int k = 0; k < K; ++k) lt.a[k] = L[(size_t)(NC + G + K + k) * fd.Fp];
  (void)SH::NS;
}

// Visit every state slot with its flat index (slot order of Shape).
template <typename T, int NC, int G, int K, typename F>
__device__ __forceinline__ void for_slots(FState<T, NC, G, K>& st, F&& fn) {
#pragma unroll
  for (int k = 0; k < NC; ++k) fn(k, st.ch[k]);
#pragma unroll
  for (int g = 0; g < G; ++g) fn(NC + g, st.mid[g]);
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int k = 0; k < K; ++k) fn(NC + G + g * K + k, st.leaf[g][k]);
#pragma unroll
  for (int k = 0; k < K; ++k) fn(NC + G + G * K + k, st.al[k]);
}

// Stage samples [j0, j0+cs] of path b and write increments Dl[s][z] (row
// stride d+1, zero at column d).
template <typename T>
__device__ __forceinline__ void stage(const T* __restrict__ Xb, int d, int j0, int cs, T* __restrict__ Xs,
                                      T* __restrict__ Dl) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const T* src = Xb + (int64_t)j0 * d;
  for (int i = tid; i < (cs + 1) * d; i += nt) Xs[i] = src[i];
  __syncthreads();
  const int rs = d + 1;
  for (int i = tid; i < cs * rs; i += nt) {
    const int s = i / rs, z = i % rs;
    Dl[i] = z < d ? Xs[(s + 1) * d + z] - Xs[s * d + z] : T(0);
  }
  __syncthreads();
}

// Asynchronous staging: element cp.async of samples [j0, j0+cs] into Xs (one
// commit group); diff_rows turns a landed buffer into Dl.  The kernels issue
// chunk c+1 (forward) / c-1 (backward) while chunk c computes.
template <typename T>
__device__ __forceinline__ void issue_rows(const T* __restrict__ Xb, int d, int j0, int cs, T* __restrict__ Xs) {
  const T* src = Xb + (int64_t)j0 * d;
  for (int i = threadIdx.x; i < (cs + 1) * d; i += blockDim.x) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(Xs + i);
    if (sizeof(T) == 4) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(src + i) : "memory");
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src + i) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <typename T>
__device__ __forceinline__ void diff_rows(const T* __restrict__ Xs, int d, int cs, T* __restrict__ Dl) {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();  // the chunk landed for every thread; nobody reads Dl any more
  const int rs = d + 1;
  for (int i = threadIdx.x; i < cs * rs; i += blockDim.x) {
    const int s = i / rs, z = i % rs;
    Dl[i] = z < d ? Xs[(s + 1) * d + z] - Xs[s * d + z] : T(0);
  }
  __syncthreads();
}

template <typename T, int NC, int G, int K>
__global__ void __launch_bounds__(kTPB) frag_forward_kernel(FragDev fd, const T* __restrict__ X, int64_t L,
                                                            const int64_t* __restrict__ bounds, int64_t nwin,
                                                            T* __restrict__ out, int64_t out_ld, int64_t out_col0,
                                                            int include_empty, T* __restrict__ state, int64_t Wc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Xs = reinterpret_cast<T*>(smem_raw);
  T* Dl = Xs + (kChunkF + 1) * fd.d;
  const int64_t b = blockIdx.x / fd.cpp;  // virtual path: window b % nwin of path b / nwin
  const int f = (int)(blockIdx.x % fd.cpp) * kTPB + threadIdx.x;
  Letters<NC, G, K> lt;
  load_letters<NC, G, K>(fd, f, lt);
  FState<T, NC, G, K> st;
  for_slots<T, NC, G, K>(st, [&](int i, T& v) { v = fd.cidx[(size_t)i * fd.Fp + f] == -2 ? T(1) : T(0); });
  int64_t M = L - 1;
  const T* Xb = X + b * L * fd.d;
  if (bounds) {
    const int64_t k = b % nwin, lo = bounds[2 * k];
    M = bounds[2 * k + 1] - lo;
    Xb = X + ((b / nwin) * L + lo) * fd.d;
  }
  T* Xs2 = Dl + kChunkF * (fd.d + 1);  // second sample buffer
  if (M > 0) issue_rows<T>(Xb, fd.d, 0, (int)(M < kChunkF ? M : kChunkF), Xs);
  for (int64_t j0 = 0, c = 0; j0 < M; j0 += kChunkF, ++c) {
    const int cs = (int)(M - j0 < kChunkF ? M - j0 : kChunkF);
    T* Xc = (c & 1) ? Xs2 : Xs;
    diff_rows<T>(Xc, fd.d, cs, Dl);
    const int64_t j1 = j0 + kChunkF;
    if (j1 < M) issue_rows<T>(Xb, fd.d, (int)j1, (int)(M - j1 < kChunkF ? M - j1 : kChunkF), (c & 1) ? Xs : Xs2);
#pragma unroll 2
    for (int s = 0; s < cs; ++s) {
      FIncr<T, NC, G, K> in;
      gather<T, NC, G, K>(Dl + s * (fd.d + 1), lt, T(1), in);
      chen_step<T, NC, G, K>(st, in);
    }
  }
  T* orow = out ? out + b * out_ld + out_col0 : nullptr;
  T* srow = state ? state + b * Wc : nullptr;
  for_slots<T, NC, G, K>(st, [&](int i, T& v) {
    const int e = fd.eidx[(size_t)i * fd.Fp + f];
    if (orow && e >= 0) orow[e] = v;
    if (srow) {
      const int si = fd.sidx[(size_t)i * fd.Fp + f];
      if (si >= 0) srow[si] = v;
    }
  });
  if (orow && include_empty && f == 0) orow[-1] = T(1);
}

// Checkpoint replay for checkpoint_stride > 0 (reference backward.py:183-199, _kernels.py:122-141):
// the fragment forward without its leaves, storing every fragment's chain and mid values
// S_{0,t_k} at k = 0, stride, 2 stride, ... into ckpt[path][k / stride][slot][fragment] (slot-major:
// a warp's stores are coalesced).  The backward reloads them instead of its exp(-dX)
// reconstruction at those steps (frag_backward_kernel, CK).
template <typename T, int NC, int G, int K>
__global__ void __launch_bounds__(kTPB) frag_ckpt_kernel(FragDev fd, const T* __restrict__ X, int64_t L, int64_t b0,
                                                         int64_t stride, T* __restrict__ ckpt) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Xs = reinterpret_cast<T*>(smem_raw);
  T* Dl = Xs + (kChunkF + 1) * fd.d;
  const int64_t bl = blockIdx.x / fd.cpp, b = b0 + bl;
  const int f = (int)(blockIdx.x % fd.cpp) * kTPB + threadIdx.x;
  Letters<NC, G, K> lt;
  load_letters<NC, G, K>(fd, f, lt);
  FState<T, NC, G, K> st;
  for_slots<T, NC, G, K>(st, [&](int i, T& v) { v = fd.cidx[(size_t)i * fd.Fp + f] == -2 ? T(1) : T(0); });
  const int64_t M = L - 1, nck = M / stride + 1;
  constexpr int NS = NC + G;  // the slots the backward reloads
  T* cb = ckpt + bl * nck * NS * fd.Fp + f;
  auto store = [&](int64_t k) {
    T* row = cb + k * NS * fd.Fp;
#pragma unroll
    for (int c = 0; c < NC; ++c) row[(size_t)c * fd.Fp] = st.ch[c];
#pragma unroll
    for (int g = 0; g < G; ++g) row[(size_t)(NC + g) * fd.Fp] = st.mid[g];
  };
  store(0);
  const T* Xb = X + b * L * fd.d;
  T* Xs2 = Dl + kChunkF * (fd.d + 1);  // second sample buffer
  if (M > 0) issue_rows<T>(Xb, fd.d, 0, (int)(M < kChunkF ? M : kChunkF), Xs);
  for (int64_t j0 = 0, c = 0; j0 < M; j0 += kChunkF, ++c) {
    const int cs = (int)(M - j0 < kChunkF ? M - j0 : kChunkF);
    T* Xc = (c & 1) ? Xs2 : Xs;
    diff_rows<T>(Xc, fd.d, cs, Dl);
    const int64_t j1 = j0 + kChunkF;
    if (j1 < M) issue_rows<T>(Xb, fd.d, (int)j1, (int)(M - j1 < kChunkF ? M - j1 : kChunkF), (c & 1) ? Xs : Xs2);
    for (int s = 0; s < cs; ++s) {
      FIncr<T, NC, G, K> in;
      gather<T, NC, G, K>(Dl + s * (fd.d + 1), lt, T(1), in);
      chen_step<T, NC, G, K, false>(st, in);
      if ((j0 + s + 1) % stride == 0) store((j0 + s + 1) / stride);
    }
  }
}

// 16-byte aligned shared-memory load of four consecutive elements.
__device__ __forceinline__ void load4(const float* p, float& a, float& b, float& c, float& d) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  a = v.x; b = v.y; c = v.z; d = v.w;
}
__device__ __forceinline__ void load4(const double* p, double& a, double& b, double& c, double& d) {
  const double2 u = *reinterpret_cast<const double2*>(p);
  const double2 v = *reinterpret_cast<const double2*>(p + 2);
  a = u.x; b = u.y; c = v.x; d = v.y;
}

template <int NC, int G, int K>
__host__ __device__ constexpr size_t bwd_smem_elems(int d, int pstride) {
  return (((size_t)(kChunkF + 1) * d + (size_t)kChunkF * (d + 1) + 3) / 4) * 4 + (size_t)kRedSteps * pstride +
         (size_t)(kChunkF + 1) * d;  // + second sample buffer
}

// Backward over paths [b0, b0 + gridDim.x / cpp).  partial layout:
// [(b - b0) * cpp + cip][M][d] (fixed-order sums of this CTA's fragments).
template <typename T, int NC, int G, int K, bool CK = false>
__global__ void __launch_bounds__(kTPB) frag_backward_kernel(FragDev fd, const T* __restrict__ X, int64_t L,
                                                             int64_t b0, const T* __restrict__ Sin, int64_t s_ld,
                                                             int64_t s_col0, const T* __restrict__ gup,
                                                             int64_t g_ld, int64_t g_col0, T* __restrict__ partial,
                                                             const T* __restrict__ ckpt = nullptr, int64_t stride = 0) {
  using SH = Shape<NC, G, K>;
  constexpr int NV = SH::NV;
  constexpr int NGS = SH::NGS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int d = fd.d;
  T* Xs = reinterpret_cast<T*>(smem_raw);
  T* Dl = Xs + (kChunkF + 1) * d;
  // parking buffer [kRedSteps][pstride], letter-major (16-byte aligned)
  T* buf = Xs + (((size_t)(kChunkF + 1) * d + (size_t)kChunkF * (d + 1) + 3) / 4) * 4;
  const int cip = (int)(blockIdx.x % fd.cpp);
  const int64_t bl = blockIdx.x / fd.cpp, b = b0 + bl;
  const int tid = threadIdx.x;
  const int f = cip * kTPB + tid;
  const int64_t M = L - 1;
  Letters<NC, G, K> lt;
  load_letters<NC, G, K>(fd, f, lt);
  FState<T, NC, G, K> st, lam;
  {
    const T* srow = Sin + b * s_ld + s_col0;
    const T* grow = gup + b * g_ld + g_col0;
    for_slots<T, NC, G, K>(st, [&](int i, T& v) {
      const int c = fd.cidx[(size_t)i * fd.Fp + f];
      v = c == -2 ? T(1) : (c >= 0 ? srow[c] : T(0));
    });
    for_slots<T, NC, G, K>(lam, [&](int i, T& v) {
      const int e = fd.eidx[(size_t)i * fd.Fp + f];
      v = e >= 0 ? grow[e] : T(0);
    });
  }
  const int* roff = fd.red_off + cip * (d + 1);
  int pos[NGS];
#pragma unroll
  for (int i = 0; i < NGS; ++i) pos[i] = fd.pos[(size_t)i * fd.Fp + f];
  // zero the parking buffer once: letter blocks are padded to float4s that are never written
  for (int i = tid; i < kRedSteps * fd.pstride; i += kTPB) buf[i] = T(0);
  // reduction geometry: segments (parked step, letter), lps lanes per segment
  int lps = 1;
  while (lps * 2 <= 32 && lps * 2 * kRedSteps * d <= kTPB) lps *= 2;
  const T* Xb = X + b * L * d;
  T* pout = partial + (bl * fd.cpp + cip) * M * d;
  const int nchunks = (int)((M + kChunkF - 1) / kChunkF);
  T* Xs2 = buf + (size_t)kRedSteps * fd.pstride;  // second sample buffer
  // checkpoint_stride (CK): the chain / mid values of the next checkpoint at or below the current
  // step, prefetched one reload ahead; ck_rem = j mod stride and ck_k = j / stride are carried down
  // the sweep (no 64-bit division per step)
  T ck_ch[NC], ck_mid[G];
  int ck_rem = 0;
  int64_t ck_k = 0;
  const T* ck_base = nullptr;
  auto ck_load = [&](int64_t k) {
    const T* row = ck_base + k * (NC + G) * fd.Fp;
#pragma unroll
    for (int c = 0; c < NC; ++c) ck_ch[c] = row[(size_t)c * fd.Fp];
#pragma unroll
    for (int g = 0; g < G; ++g) ck_mid[g] = row[(size_t)(NC + g) * fd.Fp];
  };
  if constexpr (CK) {
    if (M > 0) {
      ck_rem = (int)((M - 1) % stride);  // the sweep's first step j = M - 1
      ck_k = (M - 1) / stride;
      ck_base = ckpt + bl * (M / stride + 1) * (NC + G) * fd.Fp + f;
      ck_load(ck_k);
    }
  }
  if (nchunks > 0) issue_rows<T>(Xb, d, (nchunks - 1) * kChunkF, (int)(M - (nchunks - 1) * kChunkF), Xs);
  for (int c = nchunks - 1; c >= 0; --c) {
    const int j0 = c * kChunkF;
    const int cs = (int)(M - j0 < kChunkF ? M - j0 : kChunkF);
    T* Xc = ((nchunks - 1 - c) & 1) ? Xs2 : Xs;
    diff_rows<T>(Xc, d, cs, Dl);
    if (c > 0) issue_rows<T>(Xb, d, j0 - kChunkF, kChunkF, Xc == Xs ? Xs2 : Xs);
    int nbuf = 0;  // steps parked in buf
#pragma unroll 1
    for (int s = cs - 1; s >= 0; --s) {
      const T* row = Dl + s * (d + 1);
      FIncr<T, NC, G, K> in;
      // (a) S_{0,t_{j+1}} -> S_{0,t_j} (chain and mids; leaf values are never read)
      gather<T, NC, G, K>(row, lt, T(-1), in);
      chen_step<T, NC, G, K, false>(st, in);
      if constexpr (CK) {  // S_{0,t_j} from the forward replay at the checkpoint steps
        if (ck_rem == 0) {
#pragma unroll
          for (int c = 0; c < NC; ++c) st.ch[c] = ck_ch[c];
#pragma unroll
          for (int g = 0; g < G; ++g) st.mid[g] = ck_mid[g];
        }
        const int nrem = ck_rem == 0 ? (int)stride - 1 : ck_rem - 1;
        const int64_t nk = ck_rem == 0 ? ck_k - 1 : ck_k;
        if (nrem == 0 && nk >= 0) ck_load(nk);
        ck_rem = nrem;
        ck_k = nk;
      }
      // (b) forward partials from S_{0,t_j}
      gather<T, NC, G, K>(row, lt, T(1), in);
      T tch[NC][NC + 3];
      chain_partials<T, NC, G, K>(st, in, tch);
      const T tN1 = tch[NC - 1][NV - 1];
      const T tN = tch[NC - 1][NV];
      const T tNh = tN * T(0.5);  // halvings folded per step (exact: bitwise the same results)
      // (c) reverse: leaves, mids, anchor leaves, chain
      T gl[K];
#pragma unroll
      for (int k = 0; k < K; ++k) gl[k] = T(0);
      T gm[G];
      T tbp1 = T(0), tbp2 = T(0);  // Tbar(anchor, NV-1), Tbar(anchor, NV)
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const T tm = fma(in.dy[g], tNh, st.mid[g]);
        T tb = T(0);
        if constexpr (sizeof(T) == 4 && K >= 2) {
          // packed f32x2: leaf pairs; the adjoint dot product keeps two partial sums
          float2 tb2 = make_float2(0.f, 0.f);
          const float2 tm2 = make_float2(tm, tm);
#pragma unroll
          for (int k = 0; k + 1 < K; k += 2) {
            const float2 lz = make_float2(lam.leaf[g][k], lam.leaf[g][k + 1]);
            tb2 = __ffma2_rn(make_float2(in.dz[k], in.dz[k + 1]), lz, tb2);
            const float2 r = __ffma2_rn(lz, tm2, make_float2(gl[k], gl[k + 1]));
            gl[k] = r.x;
            gl[k + 1] = r.y;
          }
          if constexpr (K % 2) {
            tb2.x = fma(in.dz[K - 1], lam.leaf[g][K - 1], tb2.x);
            gl[K - 1] = fma(lam.leaf[g][K - 1], tm, gl[K - 1]);
          }
          tb = tb2.x + tb2.y;
        } else {
#pragma unroll
          for (int k = 0; k < K; ++k) {
            tb = fma(in.dz[k], lam.leaf[g][k], tb);
            gl[k] = fma(lam.leaf[g][k], tm, gl[k]);
          }
        }
        const T lm = lam.mid[g];
        tbp1 = fma(in.dy[g], lm, tbp1);
        tbp2 = fma(in.dy[g], tb, tbp2);  // halved below
        gm[g] = fma(lm, tN1, tb * tNh);
        lam.mid[g] = lm + tb;
      }
      T ga[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        tbp1 = fma(in.da[k], lam.al[k], tbp1);
        ga[k] = lam.al[k] * tN1;
      }
      T gch[NC];
      {
        T tbc[NV + 1];
#pragma unroll
        for (int m = 0; m <= NV; ++m) tbc[m] = T(0);
        tbc[NV - 1] = tbp1;
        tbc[NV] = tbp2 * T(0.5);
#pragma unroll
        for (int k = NC - 1; k >= 0; --k) {
          const int lv = k + 1;
          T tbn[NV + 1];
#pragma unroll
          for (int m = 0; m <= NV; ++m) tbn[m] = (m == lv) ? lam.ch[k] : tbc[m];
          T lsum = tbn[lv];
          T gs = T(0);
#pragma unroll
          for (int m = lv; m <= NV; ++m) {
            if (m > lv) lsum += tbn[m];
            const T par = (k == 0) ? T(1) : tch[k > 0 ? k - 1 : 0][m];
            gs = (m == lv) ? fma(tbn[m], par, gs) : fma(tbn[m] * rinv<T>(m - lv + 1), par, gs);
          }
          lam.ch[k] = lsum;
          gch[k] = gs;
#pragma unroll
          for (int m = 0; m <= NV; ++m)
            tbc[m] = (m >= lv) ? ((m == lv) ? in.dc[k] : in.dc[k] * rinv<T>(m - lv + 1)) * tbn[m] : T(0);
        }
      }
      // (d) park this step's gradient terms at their letter-major offsets
      T* pb = buf + (size_t)nbuf * fd.pstride;
#pragma unroll
      for (int k = 0; k < NC; ++k)
        if (pos[k] != 0xFFFF) pb[pos[k]] = gch[k];
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (pos[NC + g] != 0xFFFF) pb[pos[NC + g]] = gm[g];
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (pos[NC + G + k] != 0xFFFF) pb[pos[NC + G + k]] = gl[k];
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (pos[NC + G + K + k] != 0xFFFF) pb[pos[NC + G + K + k]] = ga[k];
      ++nbuf;
      if (nbuf == kRedSteps || s == 0) {
        __syncthreads();
        // each (parked step r, letter z) block is a contiguous run of float4s:
        // lps lanes stride over it, then a fixed xor tree -- deterministic
        for (int sg0 = 0; sg0 < kRedSteps * d; sg0 += kTPB / lps) {
          const int sg = sg0 + tid / lps, sub = tid % lps;
          const int r = sg / d, z = sg % d;
          T acc = T(0);
          if (sg < kRedSteps * d && r < nbuf) {
            const T* pr = buf + (size_t)r * fd.pstride;
            // two float4 accumulators and four loads in flight per lane (the
            // run is ~60 float4s at c4: latency, not bandwidth, bound this loop)
            T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0), b0 = T(0), b1 = T(0), b2 = T(0), b3 = T(0);
            const int q1 = roff[z + 1];
            int q = roff[z] + sub;
#pragma unroll 1
            for (; q + 3 * lps < q1; q += 4 * lps) {
              T v0, v1, v2, v3, w0, w1, w2, w3, x0, x1, x2, x3, y0, y1, y2, y3;
              load4(pr + 4 * q, v0, v1, v2, v3);
              load4(pr + 4 * (q + lps), w0, w1, w2, w3);
              load4(pr + 4 * (q + 2 * lps), x0, x1, x2, x3);
              load4(pr + 4 * (q + 3 * lps), y0, y1, y2, y3);
              a0 += v0 + x0;
              a1 += v1 + x1;
              a2 += v2 + x2;
              a3 += v3 + x3;
              b0 += w0 + y0;
              b1 += w1 + y1;
              b2 += w2 + y2;
              b3 += w3 + y3;
            }
#pragma unroll 1
            for (; q < q1; q += lps) {
              T v0, v1, v2, v3;
              load4(pr + 4 * q, v0, v1, v2, v3);
              a0 += v0;
              a1 += v1;
              a2 += v2;
              a3 += v3;
            }
            acc = ((a0 + b0) + (a1 + b1)) + ((a2 + b2) + (a3 + b3));
          }
          for (int o = lps / 2; o > 0; o /= 2) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if (sg < kRedSteps * d && r < nbuf && sub == 0) {
            const int jstep = j0 + s + (nbuf - 1 - r);  // buf[0] holds the latest (largest) step
            pout[(int64_t)jstep * d + z] = acc;
          }
        }
        __syncthreads();
        nbuf = 0;
      }
    }
  }
}

}  // namespace frag
}  // namespace sigb
