// Register-resident Chen kernels for fully truncated word sets (all words of
// length 1..N over D letters): configs 1, 2 and 5 of BASELINE.json.
//
// Work decomposition.  A truncated trie is perfectly regular, so each thread
// owns a fixed FRAGMENT for the whole time sweep, held in registers:
//   - G sibling "mid" words u_g (length N-1) sharing the grand-parent gp,
//   - their G*D leaf children u_g∘z (length N),
//   - the chain of gp's prefixes (lengths 1..N-2), recomputed redundantly by
//     the Q = D/G threads that share gp (and by every gp below them).
// One step of Chen's relation in the shared-prefix Horner form (see
// sigb_level.cu) then costs, per thread,
//   sum_{k=1}^{N-2} (N-k+1) chain FMAs + 2G mid FMAs + G*D leaf FMAs
// with no shared memory traffic except the broadcast increments and no
// barrier inside a chunk of kChunkT steps.  For D=16, N=4, G=4 that is 79
// FMAs for 68.5 words (the reference executes sum |w|(|w|+1)/2 ~ 680 Horner
// steps for the same words, _kernels.py:52-57).
//
// Backward: the same fragment, with the adjoints lambda.  Leaf adjoints are
// constant in time (a leaf has a single Horner node), so the reverse step
// per leaf is two FMAs (adjoint to the parent, gradient).  Per-step
// gradients dL/d(dX_j) are reduced across the warp by a transposing
// shuffle butterfly, across warps through shared memory once per chunk, and
// across the CTAs of a path by sample_grads_kernel, all in fixed order.
#pragma once

#include "sigb_internal.h"
#include "sigb_tc_util.cuh"

namespace sigb {
namespace trunc {

constexpr int kChunkT = 32;  // backward steps staged per chunk (16 where the reduction buffers would not fit)
constexpr int kThreadsT = 256;

// iterative (not recursive): with an unrolled loop index as exponent it inlines and folds to a
// constant instead of compiling to a device-function call, whose CALL waits on every load in flight
__host__ __device__ constexpr int ipow(int b, int e) {
  int r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

template <int D, int N, int G>
struct Cfg {
  static_assert(N >= 2, "truncated kernel needs depth >= 2");
  static_assert(D % G == 0, "G must divide D");
  static constexpr int Q = D / G;                       // threads per grand-parent
  static constexpr int NC = N - 2;                      // chain length
  static constexpr int NGP = ipow(D, N - 2);            // grand-parents per path
  static constexpr int TPP = NGP * Q;                   // threads per path
  static constexpr int PPC = TPP >= kThreadsT ? 1 : kThreadsT / TPP;  // paths per CTA
  static constexpr int CPP = TPP >= kThreadsT ? TPP / kThreadsT : 1;  // CTAs per path
  static constexpr int THREADS = TPP >= kThreadsT ? kThreadsT : PPC * TPP;
  static constexpr int RW = TPP < 32 ? TPP : 32;        // reduction width (lanes of one path)
  static constexpr int NW = THREADS / 32 > 0 ? THREADS / 32 : 1;
  static_assert(TPP % 32 == 0 || 32 % TPP == 0, "threads per path must tile warps");
  static_assert(D <= (TPP < 32 ? TPP : 32), "letters must not exceed the reduction width");
  static_assert(TPP < kThreadsT ? kThreadsT % TPP == 0 : TPP % kThreadsT == 0, "CTA tiling");
  // level offsets in canonical order: O[l] = sum_{k=1}^{l-1} D^k
  __host__ __device__ static constexpr int64_t off(int l) {
    int64_t o = 0;
    for (int k = 1; k < l; ++k) o += ipow(D, k);
    return o;
  }
};

template <typename T, int R>
__device__ __forceinline__ constexpr T inv() {
  return T(1) / T(R);
}

template <typename T>
__device__ __forceinline__ T shfl_xor(T v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}

// Per-thread fragment geometry.
template <int D, int N, int G>
struct Frag {
  using C = Cfg<D, N, G>;
  int64_t b;    // path
  int cip;      // CTA index within the path
  int t;        // thread index within the path
  int q;        // which G-slice of gp's children
  int gp;       // grand-parent code (level N-2)
  int pc;       // path slot within the CTA
  int chain_letter[C::NC > 0 ? C::NC : 1];

  __device__ __forceinline__ Frag(int64_t cta, int tid) {
    if (C::CPP > 1) {
      b = cta / C::CPP;
      cip = (int)(cta % C::CPP);
      t = cip * kThreadsT + tid;
      pc = 0;
    } else {
      pc = tid / C::TPP;
      b = cta * C::PPC + pc;
      cip = 0;
      t = tid % C::TPP;
    }
    q = t % C::Q;
    gp = t / C::Q;
    int code = gp;
#pragma unroll
    for (int k = C::NC - 1; k >= 0; --k) {
      chain_letter[k] = code % D;
      code /= D;
    }
  }
  // canonical index of chain node k (length k+1)
  __device__ __forceinline__ int64_t chain_index(int k) const {
    return C::off(k + 1) + gp / ipow(D, C::NC - 1 - k);
  }
  // this thread emits / seeds chain node k iff it is the first thread below it
  __device__ __forceinline__ bool chain_owner(int k) const {
    return q == 0 && gp % ipow(D, C::NC - 1 - k) == 0;
  }
  __device__ __forceinline__ int64_t mid_index(int g) const { return C::off(N - 1) + (int64_t)gp * D + q * G + g; }
  __device__ __forceinline__ int64_t leaf_index(int g, int z) const {
    return C::off(N) + ((int64_t)gp * D + q * G + g) * D + z;
  }
};

// Stage samples of paths of this CTA for steps [j0, j0+cs] and write the
// increments dX[s][z] (s < cs) to shared memory: layout Dl[pc][s][D].
template <typename T, int D, int PPC, int CH>
__device__ __forceinline__ void stage_increments(const T* __restrict__ X, int64_t b_first, int64_t B, int64_t L,
                                                 int j0, int cs, T* __restrict__ Xs, T* __restrict__ Dl) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int rows = cs + 1;
  for (int i = tid; i < PPC * rows * D; i += nt) {
    const int pc = i / (rows * D), r = i % (rows * D);
    const int64_t b = b_first + pc;
    Xs[pc * (CH + 1) * D + r] = b < B ? X[(b * L + j0) * D + r] : T(0);
  }
  __syncthreads();
  for (int i = tid; i < PPC * cs * D; i += nt) {
    const int pc = i / (cs * D), r = i % (cs * D);
    const T* xs = Xs + pc * (CH + 1) * D;
    Dl[pc * CH * D + r] = xs[r + D] - xs[r];
  }
  __syncthreads();
}

// Backward staging, asynchronous: element cp.async of the samples of steps
// [j0, j0+cs] into Xb (layout of stage_increments); one commit group.  The
// backward issues chunk c-1 while chunk c computes.
template <typename T, int D, int PPC, int CH>
__device__ __forceinline__ void issue_samples(const T* __restrict__ X, int64_t b_first, int64_t B, int64_t L, int j0,
                                              int cs, T* __restrict__ Xb) {
  const int rows = cs + 1;
  for (int i = threadIdx.x; i < PPC * rows * D; i += blockDim.x) {
    const int pc = i / (rows * D), r = i % (rows * D);
    const int64_t b = b_first + pc;
    T* dst = Xb + pc * (CH + 1) * D + r;
    if (b < B) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
      if (sizeof(T) == 4)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(X + (b * L + j0) * D + r) : "memory");
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(X + (b * L + j0) * D + r) : "memory");
    } else {
      *dst = T(0);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Register prefetch of the samples of the next chunk (forward): issued before
// the current chunk's steps so the global-load latency hides behind them.
template <typename T, int D, int PPC, int CH, int NT>
struct Prefetch {
  static constexpr int PF = (PPC * (CH + 1) * D + NT - 1) / NT;
  T v[PF];
  // Virtual path v = b_first + pc is window (v % K) of path v / K (K = 1, bounds
  // = NULL: the whole path).  Samples past the window's end are clamped to its
  // last sample, so their increments are exactly zero and the Chen step a no-op.
  __device__ __forceinline__ void load(const T* __restrict__ X, int64_t b_first, int64_t B, int64_t L,
                                       const int64_t* __restrict__ bounds, int64_t K, int64_t t0, int cs) {
    const int rows = cs + 1;
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const int i = threadIdx.x + k * NT;
      const int pc = i / (rows * D), r = i % (rows * D);
      const int64_t vp = b_first + pc;
      T val = T(0);
      if (pc < PPC && vp < B) {
        int64_t b = vp, lo = 0, len = L - 1;
        if (bounds) {
          b = vp / K;
          lo = bounds[2 * (vp % K)];
          len = bounds[2 * (vp % K) + 1] - lo;
        }
        const int64_t t = t0 + r / D;
        val = X[(b * L + lo + (t < len ? t : len)) * D + r % D];
      }
      v[k] = val;
    }
  }
  // Xs[pc][r] layout with row pitch (CH + 1) * D, as stage_increments.
  __device__ __forceinline__ void commit(T* __restrict__ Xs, int cs) const {
    const int rows = cs + 1;
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const int i = threadIdx.x + k * NT;
      const int pc = i / (rows * D), r = i % (rows * D);
      if (pc < PPC) Xs[pc * (CH + 1) * D + r] = v[k];
    }
  }
};

template <typename T, int D>
__device__ __forceinline__ void load_row(const T* __restrict__ src, T (&v)[D], T sign) {
  if constexpr (sizeof(T) == 4 && D % 4 == 0) {
#pragma unroll
    for (int i = 0; i < D; i += 4) {
      const float4 f = *reinterpret_cast<const float4*>(src + i);
      v[i] = sign * f.x; v[i + 1] = sign * f.y; v[i + 2] = sign * f.z; v[i + 3] = sign * f.w;
    }
  } else if constexpr (sizeof(T) == 8 && D % 2 == 0) {
#pragma unroll
    for (int i = 0; i < D; i += 2) {
      const double2 f = *reinterpret_cast<const double2*>(src + i);
      v[i] = sign * f.x; v[i + 1] = sign * f.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < D; ++i) v[i] = sign * src[i];
  }
}

// The thread's fragment state.
template <typename T, int D, int N, int G>
struct State {
  using C = Cfg<D, N, G>;
  T ch[C::NC > 0 ? C::NC : 1];
  T mid[G];
  T leaf[G][D];
};

// Increments needed by the fragment at one step: all D letters (leaves), the
// G mid letters and the chain letters.
template <typename T, int D, int N, int G>
struct StepIncr {
  using C = Cfg<D, N, G>;
  T dz[D];
  T dy[G];
  T dc[C::NC > 0 ? C::NC : 1];

  __device__ __forceinline__ void load(const T* __restrict__ row, const Frag<D, N, G>& f, T sign) {
    load_row<T, D>(row, dz, sign);
    if constexpr (G == D) {
#pragma unroll
      for (int g = 0; g < G; ++g) dy[g] = dz[g];
    } else {
#pragma unroll
      for (int g = 0; g < G; ++g) dy[g] = sign * row[f.q * G + g];
    }
#pragma unroll
    for (int k = 0; k < C::NC; ++k) dc[k] = sign * row[f.chain_letter[k]];
  }
};

// Forward partials of the chain: tch[k][m] = T(chain_k, m) for m = k+1..N.
template <typename T, int D, int N, int G>
__device__ __forceinline__ void chain_partials(const State<T, D, N, G>& st, const StepIncr<T, D, N, G>& in,
                                               T (&tch)[Cfg<D, N, G>::NC > 0 ? Cfg<D, N, G>::NC : 1][N + 1]) {
  constexpr int NC = Cfg<D, N, G>::NC;
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int lv = k + 1;
#pragma unroll
    for (int m = lv; m <= N; ++m) {
      const T a = in.dc[k] * (T(1) / T(m - lv + 1));
      tch[k][m] = (k == 0) ? st.ch[k] + a : fma(a, tch[k > 0 ? k - 1 : 0][m], st.ch[k]);
    }
  }
}

// One forward Chen step S <- S ⊗ exp(dX) on the fragment (in.* already signed).
// Leaves = false skips the leaf values: the backward never reads a leaf's S
// (a leaf's adjoint is constant in time and its gradient term uses its
// parent's partial), so its reconstruction would be pure waste (G*D FMAs/step).
template <typename T, int D, int N, int G, bool Leaves = true>
__device__ __forceinline__ void chen_step(State<T, D, N, G>& st, const StepIncr<T, D, N, G>& in) {
  constexpr int NC = Cfg<D, N, G>::NC;
  T tch[NC > 0 ? NC : 1][N + 1];
  chain_partials<T, D, N, G>(st, in, tch);
  const T tN1 = NC > 0 ? tch[NC > 0 ? NC - 1 : 0][N - 1] : T(1);
  const T tN = NC > 0 ? tch[NC > 0 ? NC - 1 : 0][N] : T(1);
#pragma unroll
  for (int k = 0; k < NC; ++k) st.ch[k] = tch[k][k + 1];
  // dX/2 . T(gp, N) as dX . (T(gp, N)/2): one scaling per step instead of one per parent (exact, so
  // bitwise the same)
  const T tNh = tN * inv<T, 2>();
  if constexpr (!Leaves && sizeof(T) == 4 && G % 2 == 0) {
    // the backward's reconstruction (no leaves): two parents' S(u) += dX . T(gp, N-1) per packed
    // f32x2 FMA (pairs in the layout of the increment row and the state).  (With the leaves, the
    // forward measured slower packed: c5 register forward 127 -> 144 ms, register pressure.)
#pragma unroll
    for (int g = 0; g < G; g += 2) {
      const float2 n2 = __ffma2_rn(make_float2(in.dy[g], in.dy[g + 1]), make_float2(tN1, tN1),
                                   make_float2(st.mid[g], st.mid[g + 1]));
      st.mid[g] = n2.x;
      st.mid[g + 1] = n2.y;
    }
    return;
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if constexpr (Leaves) {
      const T tm = fma(in.dy[g], tNh, st.mid[g]);  // T(u_g, N)
      if constexpr (sizeof(T) == 4 && D % 2 == 0) {
        // packed f32x2 FMAs: half the issue slots for the leaf level (the FMA
        // pipe still does one lane-FMA per cycle, see tools/ubench_fma.cu)
        const float2 tm2 = make_float2(tm, tm);
#pragma unroll
        for (int z = 0; z < D; z += 2) {
          const float2 r = __ffma2_rn(make_float2(in.dz[z], in.dz[z + 1]), tm2,
                                      make_float2(st.leaf[g][z], st.leaf[g][z + 1]));
          st.leaf[g][z] = r.x;
          st.leaf[g][z + 1] = r.y;
        }
      } else {
#pragma unroll
        for (int z = 0; z < D; ++z) st.leaf[g][z] = fma(in.dz[z], tm, st.leaf[g][z]);
      }
    }
    st.mid[g] = fma(in.dy[g], tN1, st.mid[g]);
  }
}

constexpr int kChunkFwd = 32;  // forward steps per staged chunk

template <typename T, int D, int N, int G>
__global__ void __launch_bounds__(Cfg<D, N, G>::THREADS)
    trunc_forward_kernel(const T* __restrict__ X, int64_t B, int64_t L, const int64_t* __restrict__ bounds,
                         int64_t K, T* __restrict__ out, int64_t out_ld, int64_t out_col0, int include_empty) {
  using C = Cfg<D, N, G>;
  constexpr int CH = kChunkFwd;
  __shared__ __align__(16) T Xs[C::PPC * (CH + 1) * D];
  __shared__ __align__(16) T Dl[C::PPC * CH * D];
  const Frag<D, N, G> f(blockIdx.x, threadIdx.x);
  const int64_t b_first = C::CPP > 1 ? f.b : (int64_t)blockIdx.x * C::PPC;
  State<T, D, N, G> st;
#pragma unroll
  for (int k = 0; k < C::NC; ++k) st.ch[k] = T(0);
#pragma unroll
  for (int g = 0; g < G; ++g) {
    st.mid[g] = T(0);
#pragma unroll
    for (int z = 0; z < D; ++z) st.leaf[g][z] = T(0);
  }
  // steps of this CTA: the longest window among its (virtual) paths
  int64_t M = L - 1;
  if (bounds) {
    M = 0;
    for (int pc = 0; pc < C::PPC; ++pc) {
      const int64_t vp = b_first + pc;
      if (vp < B) M = max(M, bounds[2 * (vp % K) + 1] - bounds[2 * (vp % K)]);
    }
  }
  Prefetch<T, D, C::PPC, CH, C::THREADS> pf;
  if (M > 0) pf.load(X, b_first, B, L, bounds, K, 0, (int)(M < CH ? M : CH));
  for (int64_t j0 = 0; j0 < M; j0 += CH) {
    const int cs = (int)(M - j0 < CH ? M - j0 : CH);
    pf.commit(Xs, cs);
    __syncthreads();  // samples visible; every thread is past the previous chunk's steps
    for (int i = threadIdx.x; i < C::PPC * cs * D; i += blockDim.x) {
      const int pc = i / (cs * D), r = i % (cs * D);
      const T* xs = Xs + pc * (CH + 1) * D;
      Dl[pc * CH * D + r] = xs[r + D] - xs[r];
    }
    __syncthreads();
    const int64_t j1 = j0 + CH;
    if (j1 < M) pf.load(X, b_first, B, L, bounds, K, j1, (int)(M - j1 < CH ? M - j1 : CH));  // in flight during steps
    const T* rows = Dl + f.pc * CH * D;
    // next steps' increment loads overlap this step's FMAs: by 4 at D = 16 (c5 fwd
    // 134.0 -> 129.4 -> 127.7 ms for 1 / 2 / 4), by 2 below (c2: 4 measured slower)
    constexpr int kUnrollF = D >= 16 ? 4 : 2;
#pragma unroll kUnrollF
    for (int s = 0; s < cs; ++s) {
      StepIncr<T, D, N, G> in;
      in.load(rows + s * D, f, T(1));
      chen_step<T, D, N, G>(st, in);
    }
  }
  if (f.b >= B) return;
  T* orow = out + f.b * out_ld + out_col0;
#pragma unroll
  for (int k = 0; k < C::NC; ++k)
    if (f.chain_owner(k)) orow[f.chain_index(k)] = st.ch[k];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    orow[f.mid_index(g)] = st.mid[g];
#pragma unroll
    for (int z = 0; z < D; ++z) orow[f.leaf_index(g, z)] = st.leaf[g][z];
  }
  if (include_empty && f.t == 0) orow[-1] = T(1);
}

// Checkpoint replay for checkpoint_stride > 0 (reference backward.py:183-199, _kernels.py:122-141):
// the forward sweep without the leaf level, storing S_{0,t_k} of every non-leaf word (levels
// 1..N-1, canonical indices [0, off(N))) at k = 0, stride, 2 stride, ... into
// ckpt[(b - b0)][k / stride][word].  The reverse sweep reloads these instead of its
// exp(-dX) reconstruction at those steps.
template <typename T, int D, int N, int G>
__global__ void __launch_bounds__(Cfg<D, N, G>::THREADS)
    trunc_ckpt_kernel(const T* __restrict__ X, int64_t B, int64_t L, int64_t b0, int64_t stride,
                      T* __restrict__ ckpt) {
  using C = Cfg<D, N, G>;
  constexpr int CH = kChunkFwd;
  constexpr int64_t NW = C::off(N);  // non-leaf words per checkpoint
  __shared__ __align__(16) T Xs[C::PPC * (CH + 1) * D];
  __shared__ __align__(16) T Dl[C::PPC * CH * D];
  const int64_t cta = blockIdx.x + (C::CPP > 1 ? b0 * C::CPP : b0 / C::PPC);
  const Frag<D, N, G> f(cta, threadIdx.x);
  const int64_t b_first = C::CPP > 1 ? f.b : cta * C::PPC;
  const int64_t M = L - 1, nck = M / stride + 1;
  const bool live = f.b < B;
  State<T, D, N, G> st;
#pragma unroll
  for (int k = 0; k < C::NC; ++k) st.ch[k] = T(0);
#pragma unroll
  for (int g = 0; g < G; ++g) st.mid[g] = T(0);
  T* cb = ckpt + (live ? f.b - b0 : 0) * nck * NW;
  auto store = [&](int64_t k) {
    if (!live) return;
    T* row = cb + k * NW;
#pragma unroll
    for (int c = 0; c < C::NC; ++c)
      if (f.chain_owner(c)) row[f.chain_index(c)] = st.ch[c];
#pragma unroll
    for (int g = 0; g < G; ++g) row[f.mid_index(g)] = st.mid[g];
  };
  store(0);
  Prefetch<T, D, C::PPC, CH, C::THREADS> pf;  // the next chunk's samples load under this chunk's steps
  if (M > 0) pf.load(X, b_first, B, L, nullptr, 1, 0, (int)(M < CH ? M : CH));
  for (int64_t j0 = 0; j0 < M; j0 += CH) {
    const int cs = (int)(M - j0 < CH ? M - j0 : CH);
    pf.commit(Xs, cs);
    __syncthreads();
    for (int i = threadIdx.x; i < C::PPC * cs * D; i += blockDim.x) {
      const int pc = i / (cs * D), r = i % (cs * D);
      Dl[pc * CH * D + r] = Xs[pc * (CH + 1) * D + r + D] - Xs[pc * (CH + 1) * D + r];
    }
    __syncthreads();
    if (j0 + CH < M) pf.load(X, b_first, B, L, nullptr, 1, j0 + CH, (int)(M - j0 - CH < CH ? M - j0 - CH : CH));
    const T* rows = Dl + f.pc * CH * D;
    for (int s = 0; s < cs; ++s) {
      StepIncr<T, D, N, G> in;
      in.load(rows + s * D, f, T(1));
      chen_step<T, D, N, G, false>(st, in);
      if ((j0 + s + 1) % stride == 0) store((j0 + s + 1) / stride);
    }
  }
}

// Transposing butterfly: V values over the WIDTH lanes of each aligned group.
// On return v[0] holds the group sum of value index `idx` (returned); lanes
// that differ only in the plain-sum bits hold the same index.
template <typename T, int V, int WIDTH>
__device__ __forceinline__ int transpose_reduce(T (&v)[V], int lane) {
  int idx = 0;
  int cnt = V;
#pragma unroll
  for (int mask = WIDTH / 2; mask >= 1; mask /= 2) {
    if (cnt > 1) {
      const int half = cnt / 2;
      const bool upper = (lane & mask) != 0;
#pragma unroll
      for (int i = 0; i < V / 2; ++i) {
        if (i < half) {
          const T send = upper ? v[i] : v[i + half];
          const T keep = upper ? v[i + half] : v[i];
          v[i] = keep + shfl_xor(send, mask);
        }
      }
      if (upper) idx += half;
      cnt = half;
    } else {
      v[0] += shfl_xor(v[0], mask);
    }
  }
  // V > WIDTH: remaining values stay in v[0..cnt) (not used by the configs here)
  return idx;
}

// The same reduction for V = 16 or 8 values over 32 lanes whose registers
// are XOR-permuted by f = 4 * (lane & (V/4 - 1)) (register p holds letter
// p ^ f): the stages over the low lane bits then keep the low half and send
// the high half in every lane -- no select pairs -- and leave letters
// f..f+3 in v[0..3]; lane bits 4 and 3 finish with selects, the remaining
// bits are plain sums (lanes differing only there hold the same letter).
// With G = 4 a thread's mid letters (quad lane & (V/4 - 1)) sit in
// registers 0..3 of that order.
template <typename T, int V>
__device__ __forceinline__ int transpose_reduce_perm(T (&v)[V], int lane) {
  static_assert(V == 16 || V == 8, "quad-permuted butterfly for 8 or 16 letters");
  if constexpr (V == 16) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += shfl_xor(v[i + 8], 2);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] += shfl_xor(v[i + 4], 1);
  int idx = 4 * (lane & (V / 4 - 1));
  {
    const bool upper = (lane & 16) != 0;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const T send = upper ? v[i] : v[i + 2];
      const T keep = upper ? v[i + 2] : v[i];
      v[i] = keep + shfl_xor(send, 16);
    }
    if (upper) idx += 2;
  }
  {
    const bool upper = (lane & 8) != 0;
    const T send = upper ? v[0] : v[1];
    const T keep = upper ? v[1] : v[0];
    v[0] = keep + shfl_xor(send, 8);
    if (upper) idx += 1;
  }
  v[0] += shfl_xor(v[0], 4);
  if constexpr (V == 8) v[0] += shfl_xor(v[0], 2);
  return idx;
}

template <int D, int N, int G>
struct RedGeom {
  using C = Cfg<D, N, G>;
  static constexpr int GPW = C::RW / C::Q > 0 ? C::RW / C::Q : 1;  // gp groups per reduction group
  static constexpr int RGW = 32 / C::RW;                              // reduction groups per warp
  static constexpr int NE = C::NW * RGW * GPW * (C::NC > 0 ? C::NC : 1);  // chain terms per parked step
  static constexpr int NKEY = C::PPC * D;                                 // (path slot, letter)
  // reduction-buffer elements for a chunk of ch steps (+ staging)
  static constexpr size_t elems(int ch) {
    return (size_t)C::PPC * (ch + 1) * D * 2 + (size_t)C::PPC * ch * D + (size_t)C::NW * RGW * ch * D +
           (size_t)C::NW * RGW * ch * GPW * (C::NC > 0 ? C::NC : 1);
  }
  static constexpr int CH = elems(kChunkT) * 8 <= 160 * 1024 ? kChunkT : 16;  // steps per chunk
  template <typename T>
  static constexpr size_t smem_bytes() {
    return sizeof(T) * ((size_t)C::PPC * (CH + 1) * D + (size_t)C::PPC * CH * D +
                        (size_t)C::NW * RGW * CH * D + (size_t)C::NW * RGW * CH * GPW * (C::NC > 0 ? C::NC : 1)) +
           sizeof(int) * (NKEY + 1) + sizeof(unsigned short) * NE + 16 +
           sizeof(T) * (size_t)C::PPC * (CH + 1) * D;  // second sample buffer (async staging)
  }
};

// Tensor-core leaf term of the backward (TC = true; fp32, D = 16, N = 4, G = 4):
// tb[u, j] = sum_z Lambda[u z] dX_j[z] for the CTA's 1,024 leaf parents u over
// a 32-step chunk is one (1024 x 16) . (16 x 32) product, eight tcgen05.mma
// kind::f16 tiles of M = 128 parents, N = 32 steps, K = 16 letters.  The leaf
// adjoints Lambda are constant over the sweep, so A is written to shared memory
// once; B (the chunk's increments) is rebuilt per chunk.  fp32 accuracy: every A
// row (per thread: its 4 parents) and every B column (step) is scaled by a power
// of two into [2^13, 2^14) and split into fp16 hi + lo; D = A_hi B_hi + A_lo B_hi
// + A_hi B_lo (3 MMAs per tile), fp32 accumulation in TMEM (7.6e-8 relative to
// |a||b|K on rows spanning 2^+-20, tools/ubench_tc_f16.cu); the scales come off
// exactly.  TMEM: 8 tiles x 32 steps = 256 columns, two CTAs per SM.
struct TcBwd {
  static constexpr int kTiles = 8;
  static constexpr int kRows = 128;
  static constexpr int kSteps = 32;                        // N of the MMA = the chunk
  static constexpr int kAHalves = kTiles * kRows * 16;     // per hi / lo
  static constexpr int kBHalves = kSteps * 16;             // per hi / lo
  static constexpr size_t bytes = 2 * (2 * kAHalves + 2 * kBHalves) + 4 * kSteps + 16 + 1024;  // + align slack
};

// Backward.  grid: one CTA per (CTA-part of a path) -- paths [b0, b0 + nb).
// partial layout: [(b - b0) * CPP + cip][M][D].
template <typename T, int D, int N, int G, bool ASYNC = (D >= 16), bool TC = false, bool CK = false>
__global__ void __launch_bounds__(Cfg<D, N, G>::THREADS, (TC || (sizeof(T) == 4 && D == 16)) ? 2 : 1)
    trunc_backward_kernel(const T* __restrict__ X, int64_t B, int64_t L, int64_t b0, const T* __restrict__ Sin,
                          int64_t s_ld, int64_t s_col0, const T* __restrict__ gup, int64_t g_ld, int64_t g_col0,
                          T* __restrict__ partial, const T* __restrict__ ckpt = nullptr, int64_t stride = 0) {
  using C = Cfg<D, N, G>;
  using RG = RedGeom<D, N, G>;
  constexpr int NC = C::NC;
  constexpr int NCc = NC > 0 ? NC : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Xs = reinterpret_cast<T*>(smem_raw);
  T* Dl = Xs + C::PPC * (RG::CH + 1) * D;
  // per-warp per-step reduced gradients: leaf/mid letters, and chain terms per gp group
  T(*red_leaf)[RG::RGW][RG::CH][D] = reinterpret_cast<T(*)[RG::RGW][RG::CH][D]>(Dl + C::PPC * RG::CH * D);
  T(*red_chain)[RG::RGW][RG::CH][RG::GPW][NCc] = reinterpret_cast<T(*)[RG::RGW][RG::CH][RG::GPW][NCc]>(
      Dl + C::PPC * RG::CH * D + C::NW * RG::RGW * RG::CH * D);
  // per-(path slot, letter) lists of this CTA's parked chain terms, built once:
  // replaces a per-element scan of every chain term in the chunk epilogue
  int* key_off = reinterpret_cast<int*>(Dl + C::PPC * RG::CH * D + C::NW * RG::RGW * RG::CH * D +
                                        C::NW * RG::RGW * RG::CH * RG::GPW * NCc);
  unsigned short* key_idx = reinterpret_cast<unsigned short*>(key_off + RG::NKEY + 1);
  T* Xs2 = reinterpret_cast<T*>(
      smem_raw + ((((size_t)(reinterpret_cast<unsigned char*>(key_idx + RG::NE) - smem_raw)) + 15) & ~size_t(15)));
  static_assert(!TC || (sizeof(T) == 4 && D == 16 && N == 4 && G == 4 && C::CPP == 4 && ASYNC && RG::CH == 32),
                "tensor-core leaf term: fp32, d = 16, depth 4, four CTAs of 1,024 leaf parents per path");
  // TC region (after the second sample buffer): A hi/lo, B hi/lo (fp16), 1/sigma per step, mbarrier, TMEM slot
  __half* Ah = reinterpret_cast<__half*>(
      smem_raw + ((((size_t)(reinterpret_cast<unsigned char*>(Xs2 + C::PPC * (RG::CH + 1) * D) - smem_raw)) + 1023) &
                  ~size_t(1023)));
  __half* Al = Ah + TcBwd::kAHalves;
  __half* Bh = Al + TcBwd::kAHalves;
  __half* Bl = Bh + TcBwd::kBHalves;
  float* inv_sig = reinterpret_cast<float*>(Bl + TcBwd::kBHalves);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(inv_sig + TcBwd::kSteps);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + 1);
  const int64_t cta = blockIdx.x + (C::CPP > 1 ? b0 * C::CPP : b0 / C::PPC);
  const Frag<D, N, G> f(cta, threadIdx.x);
  const int64_t b_first = C::CPP > 1 ? f.b : cta * C::PPC;
  const int64_t M = L - 1;
  const bool live = f.b < B;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rg = lane / C::RW;  // reduction group inside the warp
  State<T, D, N, G> st, lam;
  // PERM (D = 16, G = 4, full warps of one path): leaf-letter registers XOR-permuted
  // per lane so the gradient butterfly's first two stages need no selects and the
  // thread's mid letters land in registers 0..3 (transpose_reduce_perm16)
  constexpr bool PERM = (D == 16 || D == 8) && C::RW == 32 && G == 4 && C::Q == D / 4 && sizeof(T) == 4;
  const int pperm = PERM ? 4 * (lane & (D / 4 - 1)) : 0;
  // terminal state and adjoint seeds
  {
    const T* srow = Sin + (live ? f.b : 0) * s_ld + s_col0;
    const T* grow = gup + (live ? f.b : 0) * g_ld + g_col0;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      st.ch[k] = live ? srow[f.chain_index(k)] : T(0);
      lam.ch[k] = (live && f.chain_owner(k)) ? grow[f.chain_index(k)] : T(0);
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      st.mid[g] = live ? srow[f.mid_index(g)] : T(0);
      lam.mid[g] = live ? grow[f.mid_index(g)] : T(0);
#pragma unroll
      for (int z = 0; z < D; ++z) {
        st.leaf[g][z] = T(0);  // never read by the backward
        lam.leaf[g][z] = live ? grow[f.leaf_index(g, PERM ? (z ^ pperm) : z)] : T(0);
      }
    }
  }
  if (threadIdx.x == 0) {
    // entry e = ((w * RGW + r) * GPW + gg) * NCc + k; its letter is digit k of its grand-parent
    auto key_of = [&](int e) {
      const int k = e % NCc, gg = (e / NCc) % RG::GPW, wr = e / (NCc * RG::GPW);
      const int first_thread = (wr / RG::RGW) * 32 + (wr % RG::RGW) * C::RW;
      const int pc = C::CPP > 1 ? 0 : first_thread / C::TPP;
      const int tt = (C::CPP > 1 ? f.cip * kThreadsT : 0) + (first_thread % C::TPP) + gg * C::Q;
      int code = tt / C::Q;
      for (int q = NC - 1; q > k; --q) code /= D;
      return pc * D + code % D;
    };
    for (int i = 0; i <= RG::NKEY; ++i) key_off[i] = 0;
    for (int e = 0; e < RG::NE; ++e) key_off[key_of(e) + 1]++;
    for (int i = 0; i < RG::NKEY; ++i) key_off[i + 1] += key_off[i];
    int fill[RG::NKEY > 0 ? RG::NKEY : 1];
    for (int i = 0; i < RG::NKEY; ++i) fill[i] = key_off[i];
    for (int e = 0; e < RG::NE; ++e) {
      const int k = e % NCc, gg = (e / NCc) % RG::GPW, wr = e / (NCc * RG::GPW);
      // offset of red_chain[w][r][0][gg][k]
      key_idx[fill[key_of(e)]++] = (unsigned short)((wr * RG::CH * RG::GPW + gg) * NCc + k);
    }
  }
  // TC: TMEM, the mbarrier and the A operand (this thread's 4 rows: tiles mt0 + g, row = its TMEM lane)
  uint32_t tmem = 0, mma_phase = 0;
  float inv_s = 1.f;
  const int mt0 = (warp >> 2) * G;
  const uint32_t lane_addr = (uint32_t)(32 * (warp & 3)) << 16;
  if constexpr (TC) {
    if (warp == 0) tcu::tmem_alloc<256>(tmem_slot);
    if (threadIdx.x == 32) tcu::mbar_init(mbar, 1);
    float amax = 0.f;
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int z = 0; z < D; ++z) amax = fmaxf(amax, fabsf(lam.leaf[g][z]));
    const float sc = tcu::pow2_scale(amax);
    inv_s = 1.f / sc;  // exact: a power of two
    const int r = 32 * (warp & 3) + lane;
    const T* grow = gup + (live ? f.b : 0) * g_ld + g_col0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int kg = 0; kg < 2; ++kg) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = live ? grow[f.leaf_index(g, 8 * kg + i)] : 0.f;
        const int off = (mt0 + g) * TcBwd::kRows * 16 + tcu::kmajor_off16<2>(r, 8 * kg);
        tcu::split8_store(v, sc, Ah + off, Al + off);
      }
    }
    tcu::fence_before();
    __syncthreads();
    tcu::fence_after();
    tmem = *tmem_slot;
  }
  const int nchunks = (int)((M + RG::CH - 1) / RG::CH);
  T ck_ch[NCc], ck_mid[G];  // checkpoint_stride (CK): the next reload, prefetched
  int ck_rem = 0;
  int64_t ck_k = 0;
  const T* ck_base = nullptr;
  if (CK) {
    ck_rem = (int)((M - 1) % stride);  // the sweep's first step j = M - 1
    ck_k = (M - 1) / stride;
    ck_base = ckpt + (live ? f.b - b0 : 0) * ((L - 1) / stride + 1) * Cfg<D, N, G>::off(N);
    if (live) {
      const T* row = ck_base + ck_k * Cfg<D, N, G>::off(N);
#pragma unroll
      for (int k = 0; k < NC; ++k) ck_ch[k] = row[f.chain_index(k)];
#pragma unroll
      for (int g = 0; g < G; ++g) ck_mid[g] = row[f.mid_index(g)];
    }
  }
  // ASYNC: double-buffered cp.async staging of chunk c-1 while chunk c computes
  if (ASYNC && nchunks > 0)
    issue_samples<T, D, C::PPC, RG::CH>(X, b_first, B, L, (nchunks - 1) * RG::CH,
                                (int)(M - (nchunks - 1) * RG::CH), Xs);
  for (int c = nchunks - 1; c >= 0; --c) {
    const int j0 = c * RG::CH;
    const int cs = (int)(M - j0 < RG::CH ? M - j0 : RG::CH);
    if constexpr (ASYNC) {
      T* Xb = ((nchunks - 1 - c) & 1) ? Xs2 : Xs;
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();  // chunk c landed (every thread's copies); Dl free
      for (int i = threadIdx.x; i < C::PPC * cs * D; i += blockDim.x) {
        const int pc = i / (cs * D), r = i % (cs * D);
        const T* xs = Xb + pc * (RG::CH + 1) * D;
        Dl[pc * RG::CH * D + r] = xs[r + D] - xs[r];
      }
      __syncthreads();
      if (c > 0) issue_samples<T, D, C::PPC, RG::CH>(X, b_first, B, L, j0 - RG::CH, RG::CH, Xb == Xs ? Xs2 : Xs);
      if constexpr (TC) {
        // B operand: one thread per step row (rows past the chunk are zero), scaled per step
        if (threadIdx.x < TcBwd::kSteps) {
          const int sr = threadIdx.x;
          float v[16];
#pragma unroll
          for (int z = 0; z < 16; ++z) v[z] = sr < cs ? Dl[sr * D + z] : 0.f;
          float amax = 0.f;
#pragma unroll
          for (int z = 0; z < 16; ++z) amax = fmaxf(amax, fabsf(v[z]));
          const float sc = tcu::pow2_scale(amax);
          inv_sig[sr] = 1.f / sc;
#pragma unroll
          for (int kg = 0; kg < 2; ++kg) {
            float w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = v[8 * kg + i];
            const int off = tcu::kmajor_off16<2>(sr, 8 * kg);
            tcu::split8_store(w, sc, Bh + off, Bl + off);
          }
        }
        tcu::fence_async_smem();  // generic-proxy writes of A / B -> the tensor core's async proxy
        tcu::fence_before();      // the previous chunk's tcgen05.ld before the MMAs overwrite D
        __syncthreads();
        tcu::fence_after();
        if (warp == 0) {
          constexpr uint32_t id = tcu::idesc_f16(128, TcBwd::kSteps);
          const uint64_t bh = tcu::smem_desc(tcu::su32(Bh), 128, 256), bl = tcu::smem_desc(tcu::su32(Bl), 128, 256);
#pragma unroll
          for (int mt = 0; mt < TcBwd::kTiles; ++mt) {
            const uint64_t ah = tcu::smem_desc(tcu::su32(Ah + mt * TcBwd::kRows * 16), 128, 256);
            const uint64_t al = tcu::smem_desc(tcu::su32(Al + mt * TcBwd::kRows * 16), 128, 256);
            const uint32_t d = tmem + TcBwd::kSteps * mt;
            tcu::mma_ss_f16(d, ah, bh, id, 0u);  // A_hi B_hi
            tcu::mma_ss_f16(d, al, bh, id, 1u);  // A_lo B_hi
            tcu::mma_ss_f16(d, ah, bl, id, 1u);  // A_hi B_lo
          }
          tcu::mma_commit(mbar);
        }
        tcu::mbar_wait(mbar, mma_phase);
        mma_phase ^= 1u;
        tcu::fence_after();
      }
    } else {
      stage_increments<T, D, C::PPC, RG::CH>(X, b_first, B, L, j0, cs, Xs, Dl);
    }
    const T* rows = Dl + f.pc * RG::CH * D;
    // unrolled by 2 where the registers allow (c2: 10.26 -> 10.05 ms); at D = 16
    // the unrolled loop needs 134 registers and halves the resident CTAs
    constexpr int kUnrollB = D >= 16 ? 1 : 2;
#pragma unroll kUnrollB
    for (int s = cs - 1; s >= 0; --s) {
      StepIncr<T, D, N, G> in;
      // (a) rebuild S_{0,t_j} = S_{0,t_{j+1}} ⊗ exp(-dX_j) (chain and mids only)
      if constexpr (TC) {  // the leaf letters' increments only feed the MMA: mid and chain letters here
        const T* row = rows + s * D;
        const float4 y = *reinterpret_cast<const float4*>(row + f.q * G);
        in.dy[0] = -y.x; in.dy[1] = -y.y; in.dy[2] = -y.z; in.dy[3] = -y.w;
#pragma unroll
        for (int k = 0; k < NC; ++k) in.dc[k] = -row[f.chain_letter[k]];
      } else {
        in.load(rows + s * D, f, T(-1));
      }
      if constexpr (PERM && !TC) {  // leaf increments in the lane's permuted letter order (quad-level XOR)
        const T* row = rows + s * D;
#pragma unroll
        for (int k = 0; k < D / 4; ++k) {
          const float4 q4 = *reinterpret_cast<const float4*>(row + 4 * (k ^ (pperm >> 2)));
          in.dz[4 * k] = -q4.x; in.dz[4 * k + 1] = -q4.y; in.dz[4 * k + 2] = -q4.z; in.dz[4 * k + 3] = -q4.w;
        }
      }
      chen_step<T, D, N, G, false>(st, in);
      if (CK) {
        // checkpoint_stride: S_{0,t_j} from the forward replay instead of the reconstruction,
        // loaded one step ahead (ck_*) so the reload does not stall the sweep.  ck_rem = j mod
        // stride and ck_k = j / stride are carried down the sweep (no 64-bit division per step).
        if (ck_rem == 0) {
#pragma unroll
          for (int k = 0; k < NC; ++k) st.ch[k] = ck_ch[k];
#pragma unroll
          for (int g = 0; g < G; ++g) st.mid[g] = ck_mid[g];
        }
        const int nrem = ck_rem == 0 ? (int)stride - 1 : ck_rem - 1;
        const int64_t nk = ck_rem == 0 ? ck_k - 1 : ck_k;
        if (nrem == 0 && nk >= 0 && live) {
          const T* row = ck_base + nk * Cfg<D, N, G>::off(N);
#pragma unroll
          for (int k = 0; k < NC; ++k) ck_ch[k] = row[f.chain_index(k)];
#pragma unroll
          for (int g = 0; g < G; ++g) ck_mid[g] = row[f.mid_index(g)];
        }
        ck_rem = nrem;
        ck_k = nk;
      }
      // (b) forward partials from S_{0,t_j}
      if constexpr (!TC) {
#pragma unroll
        for (int i = 0; i < D; ++i) in.dz[i] = -in.dz[i];
      }
#pragma unroll
      for (int g = 0; g < G; ++g) in.dy[g] = -in.dy[g];
#pragma unroll
      for (int k = 0; k < NC; ++k) in.dc[k] = -in.dc[k];
      T tch[NCc][N + 1];
      chain_partials<T, D, N, G>(st, in, tch);
      const T tN1 = NC > 0 ? tch[NCc - 1][N - 1] : T(1);
      const T tN = NC > 0 ? tch[NCc - 1][N] : T(1);
      const T tNh = tN * inv<T, 2>();  // halvings folded per step (exact: bitwise the same results)
      // (c) reverse: leaves, mids, chain
      T gl[D];
#pragma unroll
      for (int z = 0; z < D; ++z) gl[z] = T(0);
      T gm[G];
      T tbp1 = T(0), tbp2 = T(0);  // Tbar(gp, N-1), Tbar(gp, N) from the mids
      T tbv[G];  // TC: Tbar(u_g, N) = sum_z Lambda[u_g z] dX[z], from the chunk's MMAs
      if constexpr (TC) {
        const float kf = inv_s * inv_sig[s];
        uint32_t rr[G];
#pragma unroll
        for (int g = 0; g < G; ++g) rr[g] = tcu::tmem_ld1(tmem + lane_addr + TcBwd::kSteps * (mt0 + g) + s);
        tcu::tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < G; ++g) tbv[g] = __uint_as_float(rr[g]) * kf;
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const T tm = fma(in.dy[g], tNh, st.mid[g]);  // T(u_g, N)
        T tb0 = T(0), tb1 = T(0);
        if constexpr (TC) {
          const float2 tm2 = make_float2(tm, tm);
#pragma unroll
          for (int z = 0; z < D; z += 2) {
            const float2 r = __ffma2_rn(make_float2(lam.leaf[g][z], lam.leaf[g][z + 1]), tm2,
                                        make_float2(gl[z], gl[z + 1]));
            gl[z] = r.x;
            gl[z + 1] = r.y;
          }
          tb0 = tbv[g];
        } else if constexpr (sizeof(T) == 4 && D % 2 == 0) {
          // packed f32x2: even/odd letters in the two halves (as the scalar split)
          float2 tb2 = make_float2(0.f, 0.f);
          const float2 tm2 = make_float2(tm, tm);
#pragma unroll
          for (int z = 0; z < D; z += 2) {
            const float2 lz = make_float2(lam.leaf[g][z], lam.leaf[g][z + 1]);
            tb2 = __ffma2_rn(make_float2(in.dz[z], in.dz[z + 1]), lz, tb2);
            const float2 r = __ffma2_rn(lz, tm2, make_float2(gl[z], gl[z + 1]));
            gl[z] = r.x;
            gl[z + 1] = r.y;
          }
          tb0 = tb2.x;
          tb1 = tb2.y;
        } else {
#pragma unroll
          for (int z = 0; z < D; z += 2) {
            tb0 = fma(in.dz[z], lam.leaf[g][z], tb0);
            gl[z] = fma(lam.leaf[g][z], tm, gl[z]);
            if (z + 1 < D) {
              tb1 = fma(in.dz[z + 1], lam.leaf[g][z + 1], tb1);
              gl[z + 1] = fma(lam.leaf[g][z + 1], tm, gl[z + 1]);
            }
          }
        }
        const T tb = TC ? tb0 : tb0 + tb1;  // Tbar(u_g, N)
        const T lm = lam.mid[g];  // Tbar(u_g, N-1)
        tbp1 = fma(in.dy[g], lm, tbp1);
        tbp2 = fma(in.dy[g], tb, tbp2);  // halved after the loop
        gm[g] = fma(lm, tN1, tb * tNh);
        lam.mid[g] = lm + tb;
      }
      // mids' gradient terms join the leaf letters (letter q*G + g).  A separate
      // butterfly over the grand-parent lanes was measured slower (more SHFL).
      if constexpr (G == D) {
#pragma unroll
        for (int g = 0; g < G; ++g) gl[g] += gm[g];
      } else if constexpr (PERM) {
#pragma unroll
        for (int g = 0; g < G; ++g) gl[g] += gm[g];  // letter quad f.q = lane & 3 sits at registers 0..3
      } else {
#pragma unroll
        for (int qq = 0; qq < C::Q; ++qq)
#pragma unroll
          for (int g = 0; g < G; ++g) gl[qq * G + g] += (f.q == qq) ? gm[g] : T(0);
      }
      // chain, deepest first: tbc[m] = Tbar(node, m) contributed by its child
      T gch[NCc] = {};
      {
        T tbc[N + 1];
#pragma unroll
        for (int m = 0; m <= N; ++m) tbc[m] = T(0);
        tbc[N - 1] = tbp1;
        tbc[N] = tbp2 * inv<T, 2>();
#pragma unroll
        for (int k = NC - 1; k >= 0; --k) {
          const int lv = k + 1;
          T tbn[N + 1];
#pragma unroll
          for (int m = 0; m <= N; ++m) tbn[m] = (m == lv) ? lam.ch[k] : tbc[m];
          T lsum = tbn[lv];
          T gs = T(0);
#pragma unroll
          for (int m = lv; m <= N; ++m) {
            if (m > lv) lsum += tbn[m];
            const T par = (k == 0) ? T(1) : tch[k > 0 ? k - 1 : 0][m];
            gs = fma(tbn[m] * (T(1) / T(m - lv + 1)), par, gs);
          }
          lam.ch[k] = lsum;
          gch[k] = gs;
#pragma unroll
          for (int m = 0; m <= N; ++m)
            tbc[m] = (m >= lv) ? in.dc[k] * (T(1) / T(m - lv + 1 > 0 ? m - lv + 1 : 1)) * tbn[m] : T(0);
        }
      }
      // (d) reduce within the path's lanes; park per-warp results in shared memory
      int idx;
      if constexpr (PERM) idx = transpose_reduce_perm<T, D>(gl, lane);
      else idx = transpose_reduce<T, D, C::RW>(gl, lane);
      constexpr int plain_bits = C::RW / (D < C::RW ? D : C::RW);  // lanes sharing one letter
      // one writer per letter: the plain (duplicating) stages are lane bits 2 (and 1 for
      // D = 8) for PERM, the low bits otherwise
      const bool writer = PERM ? (lane & (D == 16 ? 4 : 6)) == 0 : (lane % C::RW) % plain_bits == 0;
      if (writer && D <= C::RW) red_leaf[warp][rg][s][idx] = gl[0];
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        T v = gch[k];
#pragma unroll
        for (int msk = 1; msk < C::Q; msk *= 2) v += shfl_xor(v, msk);
        if (f.q == 0) red_chain[warp][rg][s][(lane % C::RW) / C::Q][k] = v;
      }
    }
    __syncthreads();
    // chunk epilogue: sum warps (and chain terms by letter) -> partial[path-part][j][z]
    for (int i = threadIdx.x; i < C::PPC * cs * D; i += blockDim.x) {
      const int pc = i / (cs * D), s = (i / D) % cs, z = i % D;
      const int64_t b = b_first + pc;
      if (b >= B) continue;
      T acc = T(0);
      // leaf letters: the warps / reduction groups belonging to path slot pc
#pragma unroll
      for (int w = 0; w < C::NW; ++w) {
#pragma unroll
        for (int r = 0; r < RG::RGW; ++r) {
          const int first_thread = w * 32 + r * C::RW;
          if (first_thread / C::TPP != pc && C::CPP == 1) continue;
          acc += red_leaf[w][r][s][z];
        }
      }
      // chain terms whose letter is z, in the fixed list order; four independent
      // partial sums so the list's dependent loads pipeline
      const T* rc = &red_chain[0][0][s][0][0];
      const int key = pc * D + z;
      T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
      int e = key_off[key];
      const int e1 = key_off[key + 1];
#pragma unroll 1
      for (; e + 4 <= e1; e += 4) {
        a0 += rc[key_idx[e]];
        a1 += rc[key_idx[e + 1]];
        a2 += rc[key_idx[e + 2]];
        a3 += rc[key_idx[e + 3]];
      }
      for (; e < e1; ++e) a0 += rc[key_idx[e]];
      acc += (a0 + a1) + (a2 + a3);
      partial[(((b - b0) * C::CPP + f.cip) * M + j0 + s) * D + z] = acc;
    }
    __syncthreads();
  }
  if constexpr (TC) {
    tcu::fence_before();
    __syncthreads();
    if (warp == 0) tcu::tmem_dealloc<256>(tmem);
  }
}

}  // namespace trunc
}  // namespace sigb
