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
constexpr int kThreadsTc = kComputeThreads + 64;  // + the MMA warp + the staging warp
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

// shared memory of the forward (dynamic): samples, increments and B operands are double-buffered
// by chunk; the output staging tile (the CTA's 1,024 x 16 leaves, then its parents) reuses nothing
constexpr int kRounds = kChunkTc / kStepsPerMma;   // MMA rounds per chunk (4)
constexpr int fXs = 0;                              // [2][(CH + 1) * 16] samples
constexpr int fDl = fXs + 2 * 4 * (kChunkTc + 1) * 16;   // [2][CH * 16] increments
constexpr int fB = fDl + 2 * 4 * kChunkTc * 16;    // [2][kRounds][hi | lo][16 x 8] tf32 (128-byte aligned)
constexpr int fBar = fB + 2 * kRounds * 2 * 4 * 16 * kStepsPerMma;  // mbarriers: MMA done, ready[2]
constexpr int fSlot = fBar + 32;
constexpr int fOut = (fSlot + 16 + 1023) & ~1023;  // [1,024 parents][16] leaves, staged for coalesced stores
constexpr size_t kFwdSmem = fOut + 4 * 1024 * 16;

// Forward.  Warps 0-7 (compute): the register fragment without its leaves, A = the parents'
// partials per 8-step round via tcgen05.st.  Warp 8 (producer): stages the samples two chunks
// ahead (cp.async), forms each chunk's increments and the four rounds' B operands (dX hi / lo)
// one chunk ahead, and issues each round's 24 MMAs once the compute warps have stored A.
template <int D, int N>
__global__ void __launch_bounds__(kThreadsTc, 2)
    trunc_tc_forward_kernel(const float* __restrict__ X, int64_t B, int64_t L, float* __restrict__ out,
                            int64_t out_ld, int64_t out_col0, int include_empty) {
  constexpr int G = 4;
  using C = Cfg<D, N, G>;
  static_assert((D == 16 || D == 8) && C::PPC == 1 && C::CPP == 4 && C::THREADS == kComputeThreads,
                "a quarter path per CTA (1,024 leaf parents); d < 16 pads the MMA's N with zero letters");
  constexpr int NC = C::NC;
  constexpr int CH = kChunkTc;
  extern __shared__ __align__(1024) unsigned char smf[];
  auto Xsb = [&](int db) { return reinterpret_cast<float*>(smf + fXs) + db * (CH + 1) * D; };
  auto Dlb = [&](int db) { return reinterpret_cast<float*>(smf + fDl) + db * CH * D; };
  auto Bsb = [&](int db, int r, int lo) {
    return reinterpret_cast<float*>(smf + fB) + ((db * kRounds + r) * 2 + lo) * 16 * kStepsPerMma;
  };
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smf + fBar);  // [0] MMA round done, [1 + db] chunk ready
  uint32_t* slot = reinterpret_cast<uint32_t*>(smf + fSlot);
  float* stage_out = reinterpret_cast<float*>(smf + fOut);

  // warp index through a shuffle: provably warp-uniform, so the role branches are uniform and the
  // MMA issue compiles to plain uniform-datapath UTCHMMAs
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  const bool producer = warp == kComputeThreads / 32;      // issues the MMAs
  const bool stager = warp == kComputeThreads / 32 + 1;    // samples, increments, B operands
  const int64_t M = L - 1;
  const int nch = (int)((M + kStepsPerMma - 1) / kStepsPerMma);  // MMA rounds
  const int nchunks = (int)((M + CH - 1) / CH);
  const int64_t bpath = blockIdx.x / C::CPP;
  if (producer) {
    tcu::tmem_alloc<kTmemCols>(slot);
    if (lane == 0) {
      tcu::mbar_init(&mbar[0], 1);
      tcu::mbar_init(&mbar[1], 32);
      tcu::mbar_init(&mbar[2], 32);
    }
  }
  tcu::fence_before();
  __syncthreads();
  tcu::fence_after();
  const uint32_t tmem = *slot;

  if (stager) {
    auto chunk_len = [&](int c) { return (int)(M - (int64_t)c * CH < CH ? M - (int64_t)c * CH : CH); };
    auto stage = [&](int c) {  // cp.async of chunk c's samples into Xs[c & 1]
      const int rows = chunk_len(c) + 1;
      const float* src = X + (bpath * L + (int64_t)c * CH) * D;
      float* dst = Xsb(c & 1);
      if (((uintptr_t)src & 15) == 0) {  // rows of D floats: 16-byte copies when X is 16-byte aligned
        for (int i = 4 * lane; i < rows * D; i += 128)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + i)), "l"(src + i) : "memory");
      } else {
        for (int i = lane; i < rows * D; i += 32)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(su32(dst + i)), "l"(src + i) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto prepare = [&](int c, bool newest_in_flight) {  // Dl and the 4 rounds' B of chunk c, then "ready"
      if (newest_in_flight) asm volatile("cp.async.wait_group 1;" ::: "memory");
      else asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      const int cs = chunk_len(c), db = c & 1;
      // one pass over float4s (a step's four letters): increments into Dl, and their hi / lo
      // split into the round's B operand (rows = letters, hi 0-15 and lo in its own tile, K = 8
      // steps); steps past the chunk are zero.  (~110 instructions per lane per chunk: the
      // stager shares its scheduler with four compute warps and must stay a chunk ahead.)
      const float4* xs4 = reinterpret_cast<const float4*>(Xsb(db));
      float4* dl4 = reinterpret_cast<float4*>(Dlb(db));
      for (int i = lane; i < CH * D / 4; i += 32) {
        const int sidx = i / (D / 4), n0 = (i % (D / 4)) * 4, r = sidx / kStepsPerMma, k = sidx % kStepsPerMma;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (sidx < cs) {
          const float4 a = xs4[i + D / 4], b = xs4[i];
          x = make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
        }
        dl4[i] = x;
        float* bh = Bsb(db, r, 0);
        float* bl = Bsb(db, r, 1);
        const float v[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int off = kmajor_off(n0 + j, k);
          const float h = tf32_hi(v[j]);
          bh[off] = h;
          bl[off] = v[j] - h;
        }
      }
      tcu::fence_async_smem();
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(&mbar[1 + db])) : "memory");
    };
    if constexpr (D < 16) {  // the B rows of letters D..15 stay zero
      for (int db = 0; db < 2; ++db)
        for (int r = 0; r < kRounds; ++r)
          for (int lo = 0; lo < 2; ++lo)
            for (int i = lane; i < (16 - D) * kStepsPerMma; i += 32)
              Bsb(db, r, lo)[kmajor_off(D + i / kStepsPerMma, i % kStepsPerMma)] = 0.f;
    }
    if (nchunks > 0) {
      stage(0);
      if (nchunks > 1) stage(1);
      prepare(0, nchunks > 1);
      if (nchunks > 2) stage(2);
    }
    for (int ck = 1; ck < nchunks; ++ck) {
      // chunk ck's buffers are free once the compute warps have stored round 0 of chunk ck-1
      // (they read chunk ck-2's increments no more) and its MMAs read B of chunk ck-2 no more
      bar_sync(3, kComputeThreads + 32);
      prepare(ck, ck + 1 < nchunks);
      if (ck + 2 < nchunks) stage(ck + 2);
    }
  } else if (producer) {
    constexpr uint32_t id16 = idesc_tf32(128, 16);
    for (int c = 0; c < nch; ++c) {
      const int ck = c / kRounds, r = c % kRounds, db = ck & 1;
      const uint64_t b_hi = smem_desc(su32(Bsb(db, r, 0)), 128, 256);
      const uint64_t b_lo = smem_desc(su32(Bsb(db, r, 1)), 128, 256);
      bar_sync(1, kComputeThreads + 32);  // A of round c stored
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        const uint32_t d = tmem + 16 * mt, a = tmem + kACol + 16 * mt;
        mma_ts(d, a, b_hi, id16, c > 0 ? 1u : 0u);  // A_hi dX_hi
        mma_ts(d, a + 8, b_hi, id16, 1u);           // A_lo dX_hi
        mma_ts(d, a, b_lo, id16, 1u);               // A_hi dX_lo
      }
      mma_commit(&mbar[0]);
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
    int c = 0;
    for (int ck = 0; ck < nchunks; ++ck) {
      const int db = ck & 1;
      const int cs = (int)(M - (int64_t)ck * CH < CH ? M - (int64_t)ck * CH : CH);
      const int cs8 = (cs + kStepsPerMma - 1) / kStepsPerMma * kStepsPerMma;
      mbar_wait(&mbar[1 + db], (uint32_t)((ck >> 1) & 1));  // increments of chunk ck ready
      const float* Dl = Dlb(db);
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
          const float tNh = 0.5f * tN;  // dX/2 . T(gp, N) as dX . (T(gp, N)/2): exact, one scaling per step
          // two parents per packed f32x2 FMA: (dX_g, dX_g+1) . T/2 + (S_g, S_g+1) gives their
          // T(u, N) (the leaves' multipliers), . T(gp, N-1) their update (the pairs stay in the
          // layout of the float4 increment load and of the state)
#pragma unroll
          for (int g = 0; g < G; g += 2) {
            const float2 dy2 = make_float2(in.dy[g], in.dy[g + 1]), m2 = make_float2(mid[g], mid[g + 1]);
            const float2 tm = __ffma2_rn(dy2, make_float2(tNh, tNh), m2);
            const float2 nm = __ffma2_rn(dy2, make_float2(tN1, tN1), m2);
            mid[g] = nm.x;
            mid[g + 1] = nm.y;
            const float h0 = tf32_hi(tm.x), h1 = tf32_hi(tm.y);
            ah[g][s] = h0;
            ah[g + 1][s] = h1;
            al[g][s] = tm.x - h0;
            al[g + 1][s] = tm.y - h1;
          }
        }
        if (c > 0) mbar_wait(&mbar[0], (uint32_t)((c - 1) & 1));  // round c-1's MMAs have read A
        asm volatile("tcgen05.fence::after_thread_sync;");
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
        asm volatile("tcgen05.fence::before_thread_sync;");
        bar_arrive(1, kComputeThreads + 32);
        // round 0 of chunk ck stored: the stager may refill the buffers of chunk ck-1 with chunk ck+1
        if (s0 == 0 && ck + 1 < nchunks) bar_arrive(3, kComputeThreads + 32);
      }
    }
    // epilogue: leaves from TMEM, staged in shared memory [parent within the CTA][letter], then
    // written with consecutive threads on consecutive words (the CTA's leaves are one contiguous
    // block of 16,384 words; its parents one block of 1,024)
    const int pl0 = (f.gp - (int)(f.cip * (kComputeThreads / C::Q))) * D + f.q * G;  // first parent in the CTA
    // staged position of (parent row, letter z): at d = 16 the 16-byte chunk is XOR-swizzled by row/4 and
    // odd row quads of 16 swap row parity, so the eight 16-byte stores of a phase (rows 4 apart) and
    // the linear read-back both hit distinct banks
    auto spos = [](int row, int z) {
      if constexpr (D == 16) return ((row ^ ((row >> 4) & 1)) << 4) + ((((z >> 2) ^ (row >> 2)) & 3) << 2) + (z & 3);
      else return row * D + z;
    };
    if (nch > 0) {
      mbar_wait(&mbar[0], (uint32_t)((nch - 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int g = 0; g < G; ++g) {
        uint32_t rg[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(rg[0]), "=r"(rg[1]), "=r"(rg[2]), "=r"(rg[3]), "=r"(rg[4]), "=r"(rg[5]), "=r"(rg[6]), "=r"(rg[7]),
              "=r"(rg[8]), "=r"(rg[9]), "=r"(rg[10]), "=r"(rg[11]), "=r"(rg[12]), "=r"(rg[13]), "=r"(rg[14]),
              "=r"(rg[15])
            : "r"(tmem + lane_addr + 16 * (mt0 + g)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int z = 0; z < D; z += 4)
          *reinterpret_cast<float4*>(stage_out + spos(pl0 + g, z)) =
              make_float4(__uint_as_float(rg[z]), __uint_as_float(rg[z + 1]), __uint_as_float(rg[z + 2]),
                          __uint_as_float(rg[z + 3]));
      }
    } else {
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int z = 0; z < D; ++z) stage_out[spos(pl0 + g, z)] = 0.f;
    }
    bar_sync(2, kComputeThreads);  // the CTA's leaf block is staged
    if (f.b < B) {
      float* orow = out + f.b * out_ld + out_col0;
      float* leaves = orow + C::off(N) + (int64_t)f.cip * (kComputeThreads / C::Q) * D * D;
      for (int i = tid; i < (kComputeThreads / C::Q) * D * D; i += kComputeThreads) leaves[i] = stage_out[spos(i / D, i % D)];
#pragma unroll
      for (int k = 0; k < NC; ++k)
        if (f.chain_owner(k)) orow[f.chain_index(k)] = ch[k];
#pragma unroll
      for (int g = 0; g < G; ++g) orow[f.mid_index(g)] = mid[g];
      if (include_empty && f.t == 0) orow[-1] = 1.f;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (producer) tcu::tmem_dealloc<kTmemCols>(tmem);
}

}  // namespace tc
}  // namespace trunc
}  // namespace sigb
