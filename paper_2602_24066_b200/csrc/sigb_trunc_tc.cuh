// Truncated forward with the leaf level on the tensor cores (tcgen05, sm_100a).
//
// For a full truncation the leaf update of one Chen step is rank one per
// parent: S(w z) += A_w(j) * dX_j[z], with A_w(j) = T(w, N) the Horner partial
// of the length-(N-1) word w that the register kernel already forms
// (sigb_trunc.cuh chen_step).  Over 8 steps the CTA's 1,024 leaf parents give
// the product (A: 1,024 x 8) . (dX: 8 x 16), i.e. eight tcgen05.mma
// kind::tf32 tiles of M = 128 parents, N = 16 letters, K = 8 steps, with the
// 1,024 x 16 leaf accumulators living in TMEM instead of 64 registers per
// thread.  fp32 accuracy comes from the 3xTF32 split
// (A_hi dX_hi + A_lo dX_hi + A_hi dX_lo, fp32 accumulation; measured 3.9e-7
// relative on random data, tools/ubench_tc_tf32.cu).
//
// Roles: warps 0-7 run the fragment kernel's chain and level-(N-1) updates
// (one thread = G = 4 parents, the register kernel's fragment) and write
// their 8 steps of A_hi / A_lo into TMEM with tcgen05.st (thread = TMEM lane,
// so the A operand needs no transpose); warp 8 issues the 24 MMAs of a chunk
// and commits them to an mbarrier.  The A buffer is single: the compute warps
// stage the next chunk in registers while the tensor core runs the current
// one, and wait for it only before their tcgen05.st.
//
// TMEM (256 columns per CTA, two CTAs per SM): D tile mt at columns
// [16 mt, 16 mt + 16); A tile mt at 128 + 16 mt (+8 for the lo part).
#pragma once

#include "sigb_tc_util.cuh"
#include "sigb_trunc.cuh"

namespace sigb {
namespace trunc {
namespace tc {

constexpr int kStepsPerMma = 8;  // tf32 K per tcgen05.mma
constexpr int kComputeThreads = 256;
constexpr int kThreadsTc = kComputeThreads + 32;  // + the MMA warp
constexpr int kTmemCols = 256;
constexpr int kACol = 128;
constexpr int kChunkTc = 32;  // steps of samples staged per round

using tcu::bar_arrive;
using tcu::bar_sync;
using tcu::idesc_tf32;
using tcu::mbar_wait;
using tcu::mma_commit;
using tcu::smem_desc;
using tcu::su32;

// high part of the 3xTF32 split: the top 19 bits (truncation; one LOP3 -- cvt.rna.tf32
// is emulated with ~8 integer instructions on sm_100a).  x - hi is exact, and the
// MMA's own truncation of lo costs < 2^-20 |x|.
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  tcu::mma_ts_tf32(d, a, bdesc, idesc, acc);
}

__device__ __forceinline__ int kmajor_off(int row, int k) { return tcu::kmajor_off32<2>(row, k); }  // rows x 8 steps

template <int D, int N>
__global__ void __launch_bounds__(kThreadsTc, 2)
    trunc_tc_forward_kernel(const float* __restrict__ X, int64_t B, int64_t L, float* __restrict__ out,
                            int64_t out_ld, int64_t out_col0, int include_empty) {
  constexpr int G = 4;
  using C = Cfg<D, N, G>;
  static_assert(D == 16 && C::PPC == 1 && C::THREADS == kComputeThreads, "one path per CTA, 16 letters");
  constexpr int NC = C::NC;
  constexpr int CH = kChunkTc;
  __shared__ __align__(16) float Xs[(CH + 1) * D];
  __shared__ __align__(16) float Dl[CH * D];
  __shared__ __align__(128) float Bs[2 * D * kStepsPerMma];  // rows 0-15 dX_hi, 16-31 dX_lo; K = 8 steps
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t M = L - 1;
  const int nch = (int)((M + kStepsPerMma - 1) / kStepsPerMma);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == kComputeThreads / 32) {
    // ---- MMA warp ----
    constexpr uint32_t id16 = idesc_tf32(128, 16);
    const uint64_t b_hi = smem_desc(su32(Bs), 128, 256);
    const uint64_t b_lo = smem_desc(su32(Bs + 16 * kStepsPerMma), 128, 256);
    for (int c = 0; c < nch; ++c) {
      bar_sync(1, kThreadsTc);  // A and B of chunk c written
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        const uint32_t d = tmem + 16 * mt, a = tmem + kACol + 16 * mt;
        mma_ts(d, a, b_hi, id16, c > 0 ? 1u : 0u);  // A_hi dX_hi
        mma_ts(d, a + 8, b_hi, id16, 1u);           // A_lo dX_hi
        mma_ts(d, a, b_lo, id16, 1u);               // A_hi dX_lo
      }
      mma_commit(&mbar);
    }
  } else {
    // ---- compute warps: the register kernel's fragment without its leaves ----
    const Frag<D, N, G> f(blockIdx.x, tid);
    float ch[NC > 0 ? NC : 1], mid[G];
#pragma unroll
    for (int k = 0; k < NC; ++k) ch[k] = 0.f;
#pragma unroll
    for (int g = 0; g < G; ++g) mid[g] = 0.f;
    const uint32_t lane_addr = (uint32_t)(32 * (warp & 3)) << 16;
    const int mt0 = (warp >> 2) * G;  // this thread's parents g sit in tiles mt0 + g
    Prefetch<float, D, 1, CH, kComputeThreads> pf;
    if (M > 0) pf.load(X, f.b, B, L, nullptr, 1, 0, (int)(M < CH ? M : CH));
    int c = 0;
    for (int64_t j0 = 0; j0 < M; j0 += CH) {
      const int cs = (int)(M - j0 < CH ? M - j0 : CH);
      const int cs8 = (cs + kStepsPerMma - 1) / kStepsPerMma * kStepsPerMma;
      pf.commit(Xs, cs);
      bar_sync(2, kComputeThreads);
      for (int i = tid; i < cs8 * D; i += kComputeThreads) Dl[i] = i < cs * D ? Xs[i + D] - Xs[i] : 0.f;
      bar_sync(2, kComputeThreads);
      const int64_t j1 = j0 + CH;
      if (j1 < M) pf.load(X, f.b, B, L, nullptr, 1, j1, (int)(M - j1 < CH ? M - j1 : CH));
      for (int s0 = 0; s0 < cs8; s0 += kStepsPerMma, ++c) {
        float ah[G][kStepsPerMma], al[G][kStepsPerMma];
#pragma unroll
        for (int s = 0; s < kStepsPerMma; ++s) {
          const float* row = Dl + (s0 + s) * D;
          StepIncr<float, D, N, G> in;
          const float4 y = *reinterpret_cast<const float4*>(row + f.q * G);
          in.dy[0] = y.x; in.dy[1] = y.y; in.dy[2] = y.z; in.dy[3] = y.w;
#pragma unroll
          for (int k = 0; k < NC; ++k) in.dc[k] = row[f.chain_letter[k]];
          float tch[NC > 0 ? NC : 1][N + 1];
          State<float, D, N, G> st;  // chain only (leaves unused)
#pragma unroll
          for (int k = 0; k < NC; ++k) st.ch[k] = ch[k];
          chain_partials<float, D, N, G>(st, in, tch);
          const float tN1 = NC > 0 ? tch[NC > 0 ? NC - 1 : 0][N - 1] : 1.f;
          const float tN = NC > 0 ? tch[NC > 0 ? NC - 1 : 0][N] : 1.f;
#pragma unroll
          for (int k = 0; k < NC; ++k) ch[k] = tch[k][k + 1];
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float tm = fmaf(in.dy[g] * 0.5f, tN, mid[g]);  // T(u_g, N): the leaves' multiplier
            mid[g] = fmaf(in.dy[g], tN1, mid[g]);
            const float h = tf32_hi(tm);
            ah[g][s] = h;
            al[g][s] = tm - h;
          }
        }
        if (c > 0) mbar_wait(&mbar, (uint32_t)((c - 1) & 1));  // chunk c-1's MMAs have read A and B
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (tid < 128) {
          const int n = tid & 15, k = tid >> 4;
          const float x = Dl[(s0 + k) * D + n], h = tf32_hi(x);
          Bs[kmajor_off(n, k)] = h;
          Bs[kmajor_off(16 + n, k)] = x - h;
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint32_t a = tmem + lane_addr + kACol + 16 * (mt0 + g);
          asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a),
                       "f"(ah[g][0]), "f"(ah[g][1]), "f"(ah[g][2]), "f"(ah[g][3]), "f"(ah[g][4]), "f"(ah[g][5]),
                       "f"(ah[g][6]), "f"(ah[g][7]));
          asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a + 8),
                       "f"(al[g][0]), "f"(al[g][1]), "f"(al[g][2]), "f"(al[g][3]), "f"(al[g][4]), "f"(al[g][5]),
                       "f"(al[g][6]), "f"(al[g][7]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        bar_arrive(1, kThreadsTc);
      }
    }
    float leaf[G][D];
    if (nch > 0) {
      mbar_wait(&mbar, (uint32_t)((nch - 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int g = 0; g < G; ++g) {
        uint32_t r[D];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(tmem + lane_addr + 16 * (mt0 + g)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int z = 0; z < D; ++z) leaf[g][z] = __uint_as_float(r[z]);
      }
    } else {
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int z = 0; z < D; ++z) leaf[g][z] = 0.f;
    }
    if (f.b < B) {
      float* orow = out + f.b * out_ld + out_col0;
#pragma unroll
      for (int k = 0; k < NC; ++k)
        if (f.chain_owner(k)) orow[f.chain_index(k)] = ch[k];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        orow[f.mid_index(g)] = mid[g];
#pragma unroll
        for (int z = 0; z < D; ++z) orow[f.leaf_index(g, z)] = leaf[g][z];
      }
      if (include_empty && f.t == 0) orow[-1] = 1.f;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
}

}  // namespace tc
}  // namespace trunc
}  // namespace sigb
