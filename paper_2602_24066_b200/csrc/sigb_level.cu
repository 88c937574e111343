// Generic Chen-update kernels over an arbitrary prefix-closed trie part
// (north_star subsystems 2 and 3; any word set: truncated, anisotropic, custom).
//
// One CTA owns one (path, part).  The part's signature state S lives in
// shared memory for the whole time sweep; increments are staged kChunk steps
// at a time, already multiplied by inv[r] = 1/r (the reference's `inv` table,
// sigcore.py:201-206).
//
// Forward step (Chen's relation in Horner form, Alg. 1).
// The reference recomputes, for every word, the Horner chain of every prefix
// (_kernels.py:52-57: sum_|w| |w|(|w|+1)/2 multiply-adds).  Words that share
// a prefix share the head of that chain, so each (node u, target length m)
// pair is evaluated once:
//     T(u, m) = a[letter(u)][m - |u| + 1] * T(parent(u), m) + S_old(u),   T(eps, m) = 1
//     S_new(u) = T(u, |u|)
// which is exactly the reference's h-recursion (h_k = a * (s_k + h_{k-1})
// with T = s + h), one FMA per (node, target length).  Levels are processed
// in order with a CTA barrier between them.
//
// Backward step (memory-lean): walking j = M-1..0 the CTA
//   (a) rebuilds S_{0,t_j} from S_{0,t_{j+1}} with the same recursion and
//       -dX_j (exp(-dX) is the group inverse),
//   (b) recomputes the forward partials T(u, m) from S_{0,t_j},
//   (c) runs reverse-mode through the recursion, children before parents:
//         Tbar(u, |u|)  = lambda(u)
//         Tbar(u, m)    = sum_children a[letter(c)][m-|u|] * Tbar(c, m)   (m > |u|)
//         lambda'(u)    = sum_m Tbar(u, m)
//         dL/dX_j[letter(u)] += sum_m Tbar(u, m) * T(parent(u), m) / (m - |u| + 1)
//   (d) reduces the per-node gradient terms per letter in a fixed order.
// The adjoint lambda = dL/dS_{0,t} is the reference's "right" state
// contracted with the upstream.
#include "sigb_internal.h"

namespace sigb {

template <typename T>
__device__ __forceinline__ T inv_of(int r) {
  return T(1) / T(r);
}

struct SmemLayout {
  int xs, a, s, tv, lam, g, tb, total;  // element offsets
};

__host__ __device__ inline SmemLayout smem_layout(int d, int N, int n, int tv, int tb, bool backward) {
  SmemLayout L;
  int o = 0;
  L.xs = o; o += (kChunk + 1) * d;
  L.a = o; o += kChunk * N * d;
  L.s = o; o += n;
  L.tv = o; o += tv > 0 ? tv : 1;
  if (backward) {
    L.lam = o; o += n;
    L.g = o; o += n;
    L.tb = o; o += tb;
  } else {
    L.lam = L.g = L.tb = o;
  }
  L.total = o;
  return L;
}

// Stage samples j0..j0+cs of path b and the scaled increments
// A[s][r-1][z] = (X[j0+s+1][z] - X[j0+s][z]) * (1/r).
template <typename T>
__device__ __forceinline__ void stage_chunk(const T* __restrict__ Xb, int j0, int cs, int d, int N,
                                            T* __restrict__ Xs, T* __restrict__ A) {
  const int nthreads = blockDim.x, tid = threadIdx.x;
  const T* src = Xb + (int64_t)j0 * d;
  for (int i = tid; i < (cs + 1) * d; i += nthreads) Xs[i] = src[i];
  __syncthreads();
  const int per = N * d;
  for (int i = tid; i < cs * per; i += nthreads) {
    int s = i / per, r = (i / d) % N, z = i % d;
    A[i] = (Xs[(s + 1) * d + z] - Xs[s * d + z]) * inv_of<T>(r + 1);
  }
  __syncthreads();
}

// One Chen step over the part, levels 1..depth, in place.  sign = +1 forward,
// -1 rebuilds the previous state (multiplication by exp(-dX)).
template <typename T>
__device__ __forceinline__ void chen_step(const PartDesc& pd, const int4* __restrict__ nodeA,
                                          const T* __restrict__ As, int d, T sign, T* __restrict__ S,
                                          T* __restrict__ Tv) {
  const int nthreads = blockDim.x, tid = threadIdx.x;
  for (int l = 1; l <= pd.depth; ++l) {
    const int hi = pd.lvl[l + 1];
    for (int w = pd.lvl[l] + tid; w < hi; w += nthreads) {
      const int4 na = __ldg(&nodeA[w]);
      const int lw = na.y & 255, md = (na.y >> 16) & 255;
      const T s = S[w];
      const T* arow = As + lw;
      T tp = na.x >= 0 ? Tv[na.x] : T(1);
      S[w] = fma(sign * arow[0], tp, s);
      for (int m = l + 1; m <= md; ++m) {
        tp = na.x >= 0 ? Tv[na.x + (m - l)] : T(1);
        Tv[na.z + (m - l - 1)] = fma(sign * arow[(m - l) * d], tp, s);
      }
    }
    __syncthreads();
  }
}

// grid: one CTA per (path, window, part); bounds == nullptr means the whole path.
template <typename T>
__global__ void __launch_bounds__(256) forward_kernel(PlanDev plan, const T* __restrict__ X, int64_t L,
                                                      const int64_t* __restrict__ bounds, int64_t K,
                                                      T* __restrict__ out, int64_t out_ld, int64_t out_col0,
                                                      int include_empty, T* __restrict__ state, int64_t Wc,
                                                      T* __restrict__ ckpt, int64_t stride, int64_t nck,
                                                      int64_t plan_max_n) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  const int P = plan.num_parts, d = plan.d, N = plan.max_len;
  const int64_t cta = blockIdx.x;
  const int part = (int)(cta % P);
  const int64_t bk = cta / P;  // path * K + window
  const int64_t b = bk / K;
  const PartDesc pd = plan.parts[part];
  const int4* nodeA = plan.nodeA + pd.node_off;
  const int4* nodeB = plan.nodeB + pd.node_off;
  const SmemLayout lay = smem_layout(d, N, pd.n, pd.tv_size, pd.tb_size, false);
  T *Xs = smem + lay.xs, *A = smem + lay.a, *S = smem + lay.s, *Tv = smem + lay.tv;
  const int tid = threadIdx.x, nthreads = blockDim.x;
  for (int w = tid; w < pd.n; w += nthreads) S[w] = T(0);
  int64_t jlo = 0, jhi = L - 1;
  if (bounds) { jlo = bounds[2 * (bk % K)]; jhi = bounds[2 * (bk % K) + 1]; }
  const T* Xb = X + b * L * d;
  if (ckpt)
    for (int w = tid; w < pd.n; w += nthreads) ckpt[(int64_t)cta * nck * plan_max_n + w] = T(0);
  for (int64_t j0 = jlo; j0 < jhi; j0 += kChunk) {
    const int cs = (int)(jhi - j0 < kChunk ? jhi - j0 : kChunk);
    stage_chunk<T>(Xb, (int)j0, cs, d, N, Xs, A);
    for (int s = 0; s < cs; ++s) {
      chen_step<T>(pd, nodeA, A + s * N * d, d, T(1), S, Tv);
      const int64_t j = j0 + s + 1;
      if (ckpt && j % stride == 0) {  // checkpoint S_{0,t_j} (backward.py:183-199)
        T* dst = ckpt + ((int64_t)cta * nck + j / stride) * plan_max_n;
        for (int w = tid; w < pd.n; w += nthreads) dst[w] = S[w];
        __syncthreads();
      }
    }
  }
  __syncthreads();
  // emit (owner parts only) + closure state
  T* orow = out + bk * out_ld + out_col0;
  for (int w = tid; w < pd.n; w += nthreads) {
    const int4 na = __ldg(&nodeA[w]);
    if (!((na.y >> 24) & 1)) continue;
    const int4 nb = __ldg(&nodeB[w]);
    if (out && nb.y >= 0) orow[nb.y] = S[w];
    if (state) state[b * Wc + nb.x] = S[w];
  }
  if (out && include_empty && part == 0 && tid == 0) orow[-1] = T(1);
}

// grid: one CTA per (path in this batch chunk, part).  Writes the per-part,
// per-step, per-letter gradient partials; sample_grads_kernel sums the parts
// in a fixed order and telescopes.
template <typename T>
__global__ void __launch_bounds__(256) backward_kernel(PlanDev plan, const T* __restrict__ X, int64_t L,
                                                       int64_t b0, const T* __restrict__ Sin, int64_t s_ld,
                                                       int64_t s_col0, int s_is_state, int64_t Wc,
                                                       const T* __restrict__ g, int64_t g_ld, int64_t g_col0,
                                                       const T* __restrict__ ckpt, int64_t stride, int64_t nck,
                                                       int64_t plan_max_n, T* __restrict__ partial) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  const int P = plan.num_parts, d = plan.d, N = plan.max_len;
  const int64_t cta = blockIdx.x;
  const int part = (int)(cta % P);
  const int64_t bl = cta / P, b = b0 + bl;
  const int64_t M = L - 1;
  const PartDesc pd = plan.parts[part];
  const int4* nodeA = plan.nodeA + pd.node_off;
  const int4* nodeB = plan.nodeB + pd.node_off;
  const int* perm = plan.perm + pd.node_off;
  const int* lseg = plan.lseg + pd.lseg_off;
  const SmemLayout lay = smem_layout(d, N, pd.n, pd.tv_size, pd.tb_size, true);
  T *Xs = smem + lay.xs, *A = smem + lay.a, *S = smem + lay.s, *Tv = smem + lay.tv;
  T *Lam = smem + lay.lam, *G = smem + lay.g, *Tb = smem + lay.tb;
  const int tid = threadIdx.x, nthreads = blockDim.x;
  // terminal state and upstream seeds (only the owner part seeds a shared ancestor)
  for (int w = tid; w < pd.n; w += nthreads) {
    const int4 na = __ldg(&nodeA[w]);
    const int4 nb = __ldg(&nodeB[w]);
    S[w] = s_is_state ? Sin[b * Wc + nb.x] : Sin[b * s_ld + s_col0 + nb.y];
    const bool seed = ((na.y >> 24) & 1) && nb.y >= 0;
    Lam[w] = seed ? g[b * g_ld + g_col0 + nb.y] : T(0);
  }
  // letter-reduction geometry: tpl lanes per letter, a power of two <= 32
  int tpl = 1;
  while (tpl * 2 <= 32 && tpl * 2 * d <= nthreads) tpl *= 2;
  const int my_z = tid / tpl, my_lane = tid % tpl;
  const T* Xb = X + b * L * d;
  T* part_out = partial + (bl * P + part) * M * d;
  const int nchunks = (int)((M + kChunk - 1) / kChunk);
  for (int c = nchunks - 1; c >= 0; --c) {
    const int j0 = c * kChunk;
    const int cs = (int)(M - j0 < kChunk ? M - j0 : kChunk);
    stage_chunk<T>(Xb, j0, cs, d, N, Xs, A);
    for (int s = cs - 1; s >= 0; --s) {
      const int j = j0 + s;
      const T* As = A + s * N * d;
      // (a) S_{0,t_{j+1}} -> S_{0,t_j}
      if (ckpt && j % stride == 0) {
        const T* src = ckpt + ((int64_t)cta * nck + j / stride) * plan_max_n;
        for (int w = tid; w < pd.n; w += nthreads) S[w] = src[w];
        __syncthreads();
      } else {
        chen_step<T>(pd, nodeA, As, d, T(-1), S, Tv);
      }
      // (b) forward partials T(u, m), m > |u|, from S_{0,t_j}
      for (int l = 1; l < pd.depth; ++l) {
        const int hi = pd.lvl[l + 1];
        for (int w = pd.lvl[l] + tid; w < hi; w += nthreads) {
          const int4 na = __ldg(&nodeA[w]);
          const int lw = na.y & 255, md = (na.y >> 16) & 255;
          if (md <= l) continue;
          const T sv = S[w];
          for (int m = l + 1; m <= md; ++m) {
            const T tp = na.x >= 0 ? Tv[na.x + (m - l)] : T(1);
            Tv[na.z + (m - l - 1)] = fma(As[(m - l) * d + lw], tp, sv);
          }
        }
        __syncthreads();
      }
      // (c) reverse sweep, deepest level first
      for (int l = pd.depth; l >= 1; --l) {
        const int hi = pd.lvl[l + 1];
        for (int w = pd.lvl[l] + tid; w < hi; w += nthreads) {
          const int4 na = __ldg(&nodeA[w]);
          const int4 nb = __ldg(&nodeB[w]);
          const int md = (na.y >> 16) & 255;
          const T lam0 = Lam[w];
          T lam = lam0;
          T gs = lam0 * (na.x >= 0 ? Tv[na.x] : T(1));  // r = 1: inv = 1
          Tb[na.w] = lam0;
          for (int m = l + 1; m <= md; ++m) {
            T tb = T(0);
            for (int ch = nb.z; ch < nb.z + nb.w; ++ch) {
              const int4 nc = __ldg(&nodeA[ch]);
              if (((nc.y >> 16) & 255) >= m)
                tb = fma(As[(m - l - 1) * d + (nc.y & 255)], Tb[nc.w + (m - l - 1)], tb);
            }
            Tb[na.w + (m - l)] = tb;
            lam += tb;
            const T tp = na.x >= 0 ? Tv[na.x + (m - l)] : T(1);
            gs = fma(tb * inv_of<T>(m - l + 1), tp, gs);
          }
          Lam[w] = lam;
          G[w] = gs;
        }
        __syncthreads();
      }
      // (d) dL/d(dX_j)[z] = sum over nodes with last letter z, fixed order
      for (int z0 = 0; z0 < d; z0 += nthreads / tpl) {
        const int z = z0 + my_z;
        T acc = T(0);
        if (z < d && my_z < nthreads / tpl)
          for (int k = lseg[z] + my_lane; k < lseg[z + 1]; k += tpl) acc += G[perm[k]];
        for (int off = tpl / 2; off > 0; off /= 2) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (z < d && my_lane == 0 && my_z < nthreads / tpl) part_out[(int64_t)j * d + z] = acc;
      }
    }
  }
}

// dL/dX_t = inc(t-1) - inc(t) with inc(j) = sum_parts partial (backward.py:130-147).
template <typename T>
__global__ void sample_grads_kernel(const T* __restrict__ partial, int64_t Bc, int64_t P, int64_t M, int64_t d,
                                    int64_t b0, T* __restrict__ dX, T* __restrict__ dinc) {
  const int64_t L = M + 1;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= Bc * L * d) return;
  const int64_t z = i % d, t = (i / d) % L, bl = i / (d * L);
  auto inc = [&](int64_t j) {
    T s = T(0);
    for (int64_t p = 0; p < P; ++p) s += partial[((bl * P + p) * M + j) * d + z];
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

}  // namespace sigb
