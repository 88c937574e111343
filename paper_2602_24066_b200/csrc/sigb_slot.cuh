// Level-slot Chen kernels for SMALL sparse tries (whole closure per CTA; e.g.
// config 3's random 2,048-word set), where the fragment kernels replicate too
// much ancestor work (sigb_frag.cuh: ~24 issue slots of chain per ~7 words).
//
// One CTA = one path.  Every closure node is owned by exactly one thread; a
// thread owns up to KS consecutive (canonical-order) nodes of ONE level, so
// warps are level-pure and siblings mostly share their parent's data.  Node
// values S live in registers for the whole sweep; the Horner partials
//     T(u, m) = (dX[letter(u)] / (m-|u|+1)) * T(parent(u), m) + S(u),  m > |u|
// of internal nodes are published in shared memory, level by level, one CTA
// barrier per level and step (the reference recomputes every
// prefix chain per word instead, _kernels.py:52-57).  Scaled increments
// A[z][r] = dX[z] / r are staged per chunk so a node reads all its factors with
// vector loads.
//
// Backward per step (memory-lean):
//   top-down    internal nodes rebuild S_{0,t_j} with -dX (T^- partials) and
//               republish the forward partials T from it;
//   bottom-up   Tbar(u, m) = sum_children P(c, m), P(c, m) = a_c[m-|c|+1] *
//               Tbar(c, m) published per level; lambda += sum_{m>|u|} Tbar(u, m);
//               gradient term G(u) = sum_m Tbar(u,m) T(parent,m) / (m-|u|+1);
//   reduction   G(u) parked at letter-major offsets and summed per letter in a
//               fixed order every kRedS steps (no atomics).
#pragma once

#include "sigb_internal.h"

namespace sigb {
namespace slot {

constexpr int KS = 8;        // nodes per thread
constexpr int AW = 8;        // scaled-increment row width (r = 1..AW)
constexpr int kChunkS = 16;  // steps staged per chunk
constexpr int kRedS = 4;     // steps per gradient-reduction round

struct SlotDev {
  const int* tinfo;             // [TPB] level | cnt << 4 | first << 8  (level 0: idle thread)
  const unsigned* meta0;        // [KS][TPB] pT (16) | letter (8) | nT (8)
  const unsigned* meta1;        // [KS][TPB] child first (16, local in next level) | child count (16)
  const unsigned short* pos;    // [KS][TPB] parking offset (0xFFFF: none)
  const int* cidx;              // [KS][TPB] closure index (-1: empty slot)
  const int* eidx;              // [KS][TPB] emitted index in I or -1
  const int* lvl;               // [N + 2] per level: T base, (N + 2) P base, (N + 2) node count
  const int* red_off;           // [d + 1] letter blocks of the parking buffer, float4 units
  int TPB, d, N;
  int t_size, p_size, a_off, t_off, tm_off, p_off, park_off, pstride, smem_floats;
};

// Per-level geometry helpers (lvl table layout: [0..N+1] T base, [N+2..2N+3] P base,
// [2N+4..3N+5] counts).
__device__ __forceinline__ int tbase(const int* lv, int l) { return lv[l]; }
__device__ __forceinline__ int pbase(const int* lv, int N, int l) { return lv[N + 2 + l]; }
__host__ __device__ __forceinline__ int t_stride(int N, int l) { return ((N - l) + 3) / 4 * 4; }
__host__ __device__ __forceinline__ int p_stride(int N, int l) { return ((N - l + 1) + 3) / 4 * 4; }

template <typename T>
__device__ __forceinline__ void ld8(const T* p, T (&v)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = p[i];
}

// Stage samples [j0, j0+cs] of one path and the scaled increments A[s][z][r].
template <typename T>
__device__ __forceinline__ void stage_scaled(const T* __restrict__ Xb, int d, int j0, int cs, T* __restrict__ Xs,
                                             T* __restrict__ A) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const T* src = Xb + (int64_t)j0 * d;
  for (int i = tid; i < (cs + 1) * d; i += nt) Xs[i] = src[i];
  __syncthreads();
  for (int i = tid; i < cs * d * AW; i += nt) {
    const int s = i / (d * AW), z = (i / AW) % d, r = i % AW;
    A[i] = (Xs[(s + 1) * d + z] - Xs[s * d + z]) / T(r + 1);
  }
  __syncthreads();
}

template <typename T, int N>
__global__ void __launch_bounds__(512) slot_forward_kernel(SlotDev sd, const T* __restrict__ X, int64_t L,
                                                            T* __restrict__ out, int64_t out_ld, int64_t out_col0,
                                                            int include_empty, T* __restrict__ state, int64_t Wc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const int tid = threadIdx.x, d = sd.d;
  const int64_t b = blockIdx.x;
  const int info = sd.tinfo[tid];
  const int lv = info & 15, cnt = (info >> 4) & 15, first = info >> 8;
  unsigned m0[KS];
  T S[KS];
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    m0[k] = sd.meta0[k * sd.TPB + tid];
    S[k] = T(0);
  }
  for (int i = tid; i < 8; i += blockDim.x) sm[i] = T(1);  // T(eps, m) = 1
  const int tb = lv > 0 ? sd.lvl[lv] : 0, ts = t_stride(N, lv);
  T* Xs = sm + sd.park_off;  // forward: the parking area holds the raw samples
  T* A = sm + sd.a_off;
  const int64_t M = L - 1;
  const T* Xb = X + b * L * d;
  for (int64_t j0 = 0; j0 < M; j0 += kChunkS) {
    const int cs = (int)(M - j0 < kChunkS ? M - j0 : kChunkS);
    stage_scaled<T>(Xb, d, (int)j0, cs, Xs, A);
#pragma unroll 1
    for (int s = 0; s < cs; ++s) {
      const T* As = A + s * d * AW;
#pragma unroll 1
      for (int l = 1; l <= N; ++l) {
        if (lv == l) {
#pragma unroll
          for (int k = 0; k < KS; ++k) {
            if (k < cnt) {
              const int pT = m0[k] & 0xFFFF, letter = (m0[k] >> 16) & 0xFF, nT = m0[k] >> 24;
              const T* a = As + letter * AW;
              const T* par = sm + pT;
              const T s0 = S[k];
              if (nT == 1) {
                S[k] = fma(a[0], par[0], s0);
              } else {
                T av[8], pv[8];
                ld8(a, av);
                ld8(par, pv);
                S[k] = fma(av[0], pv[0], s0);
                T* ot = sm + tb + (first + k) * ts;
#pragma unroll
                for (int r = 1; r < N; ++r)
                  if (r < nT) ot[r - 1] = fma(av[r], pv[r], s0);
              }
            }
          }
        }
        __syncthreads();
      }
    }
  }
  T* orow = out ? out + b * out_ld + out_col0 : nullptr;
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    if (k < cnt) {
      const int e = sd.eidx[k * sd.TPB + tid];
      if (orow && e >= 0) orow[e] = S[k];
      if (state) state[b * Wc + sd.cidx[k * sd.TPB + tid]] = S[k];
    }
  }
  if (orow && include_empty && tid == 0) orow[-1] = T(1);
}

template <typename T, int N>
__global__ void __launch_bounds__(512) slot_backward_kernel(SlotDev sd, const T* __restrict__ X, int64_t L,
                                                             int64_t b0, const T* __restrict__ Sin, int64_t s_ld,
                                                             int64_t s_col0, const T* __restrict__ gup, int64_t g_ld,
                                                             int64_t g_col0, T* __restrict__ partial) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const int tid = threadIdx.x, d = sd.d;
  const int64_t bl = blockIdx.x, b = b0 + bl;
  const int info = sd.tinfo[tid];
  const int lv = info & 15, cnt = (info >> 4) & 15, first = info >> 8;
  unsigned m0[KS], m1[KS];
  unsigned short pos[KS];
  T S[KS], lam[KS];
  {
    const T* srow = Sin + b * s_ld + s_col0;
    const T* grow = gup + b * g_ld + g_col0;
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      m0[k] = sd.meta0[k * sd.TPB + tid];
      m1[k] = sd.meta1[k * sd.TPB + tid];
      pos[k] = sd.pos[k * sd.TPB + tid];
      const int c = sd.cidx[k * sd.TPB + tid], e = sd.eidx[k * sd.TPB + tid];
      S[k] = (k < cnt && c >= 0) ? srow[c] : T(0);
      lam[k] = (k < cnt && e >= 0) ? grow[e] : T(0);
    }
  }
  for (int i = tid; i < 8; i += blockDim.x) sm[i] = T(1);  // T(eps, m) = T^-(eps, m) = 1
  T* A = sm + sd.a_off;
  T* buf = sm + sd.park_off;  // [kRedS][pstride]
  T* Xs = buf;                // staging shares the parking area (disjoint phases)
  for (int i = tid; i < kRedS * sd.pstride; i += blockDim.x) buf[i] = T(0);
  // P entries past a node's last target are never written and must read as 0
  for (int i = tid; i < sd.p_size; i += blockDim.x) sm[sd.p_off + i] = T(0);
  const int tsl = t_stride(N, lv), psl = p_stride(N, lv), pschild = p_stride(N, lv + 1);
  const int tb = lv > 0 ? sd.lvl[lv] : 0;
  const int tmb = tb - sd.t_off + sd.tm_off;
  const int pb = lv > 0 ? sd.lvl[N + 2 + lv] : 0;
  const int pbc = lv > 0 && lv < N ? sd.lvl[N + 2 + lv + 1] : 0;
  int lps = 1;
  while (lps * 2 <= 32 && lps * 2 * kRedS * d <= (int)blockDim.x) lps *= 2;
  const int64_t M = L - 1;
  const T* Xb = X + b * L * d;
  T* pout = partial + bl * M * d;
  const int nchunks = (int)((M + kChunkS - 1) / kChunkS);
  for (int c = nchunks - 1; c >= 0; --c) {
    const int j0 = c * kChunkS;
    const int cs = (int)(M - j0 < kChunkS ? M - j0 : kChunkS);
    // the staging reuses the parking area: it is clean (zero) between rounds
    // except for the letter blocks, which are rewritten before being read
    stage_scaled<T>(Xb, d, j0, cs, Xs, A);
    for (int i = tid; i < kRedS * sd.pstride; i += blockDim.x) buf[i] = T(0);
    __syncthreads();
    int nbuf = 0;
#pragma unroll 1
    for (int s = cs - 1; s >= 0; --s) {
      const T* As = A + s * d * AW;
      // -- top-down: internal nodes rebuild S_{0,t_j} and republish T^-, T ------
#pragma unroll 1
      for (int l = 1; l < N; ++l) {
        if (lv == l) {
#pragma unroll
          for (int k = 0; k < KS; ++k) {
            const int nT = m0[k] >> 24;
            if (k < cnt && nT > 1) {
              const int pT = m0[k] & 0xFFFF, letter = (m0[k] >> 16) & 0xFF;
              const int pTm = pT == 0 ? 0 : pT - sd.t_off + sd.tm_off;
              T av[8], pv[8], pm[8];
              ld8(As + letter * AW, av);
              ld8(sm + pT, pv);
              ld8(sm + pTm, pm);
              const T sn = S[k];
              const T sj = fma(-av[0], pm[0], sn);
              T* otm = sm + tmb + (first + k) * tsl;
              T* ot = sm + tb + (first + k) * tsl;
#pragma unroll
              for (int r = 1; r < N; ++r)
                if (r < nT) {
                  otm[r - 1] = fma(-av[r], pm[r], sn);
                  ot[r - 1] = fma(av[r], pv[r], sj);
                }
              S[k] = sj;
            }
          }
        }
        __syncthreads();
      }
      // -- bottom-up: adjoints, children's P contributions, gradient terms -------
      T* pk = buf + nbuf * sd.pstride;
#pragma unroll 1
      for (int l = N; l >= 1; --l) {
        if (lv == l) {
#pragma unroll
          for (int k = 0; k < KS; ++k) {
            if (k < cnt) {
              const int pT = m0[k] & 0xFFFF, letter = (m0[k] >> 16) & 0xFF, nT = m0[k] >> 24;
              T av[8], pv[8], tbv[8];
              ld8(As + letter * AW, av);
              ld8(sm + pT, pv);
              tbv[0] = lam[k];
#pragma unroll
              for (int r = 1; r < 8; ++r) tbv[r] = T(0);
              if (nT > 1) {
                const int cf = m1[k] & 0xFFFF, cc = m1[k] >> 16;
                const T* pc = sm + pbc + cf * pschild;
#pragma unroll 1
                for (int ch = 0; ch < cc; ++ch) {
                  const T* v = pc + ch * pschild;
#pragma unroll
                  for (int r = 1; r < N; ++r)
                    if (r < nT) tbv[r] += v[r - 1];
                }
              }
              T lsum = tbv[0], g = tbv[0] * pv[0];
#pragma unroll
              for (int r = 1; r < N; ++r)
                if (r < nT) {
                  lsum += tbv[r];
                  g = fma(tbv[r] * (T(1) / T(r + 1)), pv[r], g);
                }
              lam[k] = lsum;
              T* op = sm + pb + (first + k) * psl;
#pragma unroll
              for (int r = 0; r < N; ++r)
                if (r < nT) op[r] = av[r] * tbv[r];
              if (pos[k] != 0xFFFF) pk[pos[k]] = g;
            }
          }
        }
        __syncthreads();
      }
      ++nbuf;
      if (nbuf == kRedS || s == 0) {
        for (int sg0 = 0; sg0 < kRedS * d; sg0 += (int)blockDim.x / lps) {
          const int sg = sg0 + tid / lps, sub = tid % lps;
          const int r = sg / d, z = sg % d;
          T acc = T(0);
          if (sg < kRedS * d && r < nbuf) {
            const T* pr = buf + r * sd.pstride;
            T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
            for (int q = sd.red_off[z] + sub; q < sd.red_off[z + 1]; q += lps) {
              a0 += pr[4 * q];
              a1 += pr[4 * q + 1];
              a2 += pr[4 * q + 2];
              a3 += pr[4 * q + 3];
            }
            acc = (a0 + a1) + (a2 + a3);
          }
          for (int o = lps / 2; o > 0; o /= 2) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if (sg < kRedS * d && r < nbuf && sub == 0) pout[(int64_t)(j0 + s + (nbuf - 1 - r)) * d + z] = acc;
        }
        __syncthreads();
        nbuf = 0;
      }
    }
  }
}

}  // namespace slot
}  // namespace sigb
