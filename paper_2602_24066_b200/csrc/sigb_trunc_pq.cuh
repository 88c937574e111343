// Truncated backward for d = 16, depth 4, fp32 (config 5) with the whole leaf
// level on the tensor cores: the "P/Q" form.
//
// The leaves (words gp.y.z of length 4; gp a length-2 grand-parent, y the
// parent's last letter, z the leaf letter) carry constant adjoints
// Lambda[gp, y, z] (the upstream gradient; a leaf is a single Horner node).  They
// enter the reverse sweep twice per step j (_kernels.py:152-173):
//   (1) the pull-back to their parent u = gp.y:   tb[u]   = sum_z Lambda[gp,y,z] dX_j[z]
//   (2) the gradient of letter z:                 gl[gp,z] = sum_y Lambda[gp,y,z] T(gp.y, 4)_j
// with T(gp.y, 4)_j = S_j(gp.y) + dX_j[y]/2 T(gp, 4)_j the parent's Horner partial.
// On CUDA cores both are 16-term sums per (word, step): 2 x 65,536 FMAs per
// path-step plus a 16-letter butterfly per thread-step (round 1's kernel).
//
// (1) is a (1024 x 16) . (16 x 32-step) product per CTA and chunk -- D1 on tcgen05.
// (2) splits by linearity into
//   gl[gp,z] = P_j[gp,z] + T(gp,4)_j / 2 * Q_j[gp,z],
//   Q_j[gp,z] = sum_y Lambda[gp,y,z] dX_j[y]            (the transposed product -- D2 on tcgen05)
//   P_j[gp,z] = sum_y Lambda[gp,y,z] S_j(gp.y)          (kept as state: one FMA per step)
// because the memory-lean reconstruction S_j(gp.y) = S_{j+1}(gp.y) - dX_j[y] Tr(gp, 3)_j
// (Tr: the partial of the exp(-dX) step) gives P_j = P_{j+1} - Tr(gp,3)_j Q_j.
// So the CUDA cores keep two FMAs per (grand-parent, letter) and step for the
// leaves instead of 32, no 64-register Lambda block, and a 4-letter reduction
// per thread instead of 16.
//
// Tensor-core operands (kind::f16, M = 128 rows, N = 16 steps, K = 16 letters):
// A1 rows = parents u (K = z), A2 rows = (gp, z) pairs (K = y), both constant
// over the sweep and written to shared memory once; B = the chunk's increments
// (K = letter, N = step), rebuilt per chunk.  fp32 accuracy from a scaled 3-pass
// fp16 split (A rows scaled per grand-parent at depth 4, per thread at depth 5, and
// B columns per step, by powers of two into [2^13, 2^14), x = hi + lo,
// D = A_hi B_hi + A_lo B_hi + A_hi B_lo; tools/ubench_tc_f16.cu: 7.6e-8 relative).
// Steps 16-31 and 0-15 of a chunk are two MMA groups with their own mbarrier, so
// the second group runs while the sweep walks the first.  TMEM: {D1, D2} x 8 tiles
// x 16 steps x 2 groups = 512 columns; one CTA (a quarter path) per SM (220 KB of
// shared memory at depth 4).
//
// Thread (grand-parent gp, letter quad q) owns: parents gp.y for y in the quad's
// letters (adjoint, D1 rows) and pairs (gp, z) for z in them (P state, D2 rows).
// At depth 4 the grand-parent's chain is walked once per warp and MMA group
// (chain_pre) and its reverse mode deferred to a per-chunk sweep (chain_sweep);
// at depth 5 the quad computes the chain in the step.  The letter sums of the
// quad's letters are reduced over the warp's grand-parents by a transposing
// shuffle butterfly, parked per warp in shared memory, and summed over the 8 warps
// in fixed order per chunk into the partial buffer trunc_sample_grads telescopes.
#pragma once

#include "sigb_tc_util.cuh"
#include "sigb_trunc.cuh"

namespace sigb {
namespace trunc {
namespace pq {

// Geometry shared by the instantiations (d = 16, depth 4: config 5; d = 8, depth 5: config 2):
// a CTA holds 1,024 leaf parents (four per compute thread), i.e. a quarter path in both.
constexpr int kThreads = 256;          // compute threads
constexpr int kBlock = kThreads + 32;  // + the producer warp
constexpr int CH = 32;                 // steps per chunk
constexpr int NG = 16;                 // steps per MMA group (MMA N)
constexpr int kTiles = 8;              // 1,024 rows per operand / 128
constexpr int kRowHalves = 128 * 16;   // one A tile: 128 rows x K = 16 fp16 (d < 16 pads with zeros)
constexpr int kAHalves = kTiles * kRowHalves;

template <int D, int N>
struct PQ {
  static_assert(D == 16 || D == 8, "letter quads: d = 8 or 16");
  static constexpr int QPG = D / 4;                    // threads per grand-parent (letter quads)
  static constexpr int GPC = kThreads / QPG;           // grand-parents per CTA
  static constexpr int NGP = trunc::ipow(D, N - 2);    // grand-parents per path
  static constexpr int CPP = NGP / GPC;                // CTAs per path
  static constexpr int NC = N - 2;                     // chain nodes (levels 1 .. N-2)
  static_assert(GPC * D == 1024 && NGP % GPC == 0, "1,024 leaf parents per CTA");
  // canonical word offsets of a full truncation: level l starts at sum_{k<l} D^k
  __host__ __device__ static constexpr int64_t off(int l) { return trunc::Cfg<D, N, 4>::off(l); }
  // shared memory (bytes); B, increments, parked sums and 1/sigma are double-buffered by chunk parity
  static constexpr int oA1h = 0, oA1l = oA1h + 2 * kAHalves, oA2h = oA1l + 2 * kAHalves;
  static constexpr int oA2l = oA2h + 2 * kAHalves;
  static constexpr int kBBytes = 2 * CH * 16;            // one of hi / lo
  static constexpr int oB = oA2l + 2 * kAHalves;         // [2 buffers][hi, lo]
  static constexpr int oXs = oB + 2 * 2 * kBBytes;       // two sample buffers (CH + 1) x D
  static constexpr int oDl = oXs + 2 * 4 * (CH + 1) * D; // [2][CH][D] increments
  static constexpr int oRed = oDl + 2 * 4 * CH * D;      // [2][8 warps][CH][D] per-warp letter sums
  static constexpr int oSig = oRed + 2 * 4 * 8 * CH * D; // [2][CH] 1 / sigma per step
  // depth 4 (NC == 2): per warp and step, the grand-parents' parent-adjoint sums and chain inputs
  // for the deferred chain sweep, [8 warps][CH][8 grand-parents][T1, T2, d1, S (even gp) / d0 (odd)]
  static constexpr bool kDeferChain = NC == 2;
  static constexpr int oPark = oSig + 2 * 4 * CH;
  // depth 4: per warp, the chain values of its 8 grand-parents for the steps of one MMA group,
  // [8 warps][NG steps][8 grand-parents] float4 (chain_pre)
  static constexpr int oCb = oPark + (kDeferChain ? 8 * CH * 32 * 4 : 0);
  static constexpr int oBar = oCb + (kDeferChain ? 8 * NG * 8 * 16 : 0);  // mbarriers: MMA groups 0, 1; ready 0, 1
  static constexpr int oSlot = oBar + 32;
  static constexpr size_t kSmem = oSlot + 16;
};

__device__ __forceinline__ void ld_wait8(uint32_t (&r)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]));
}
__device__ __forceinline__ void ld_wait16(uint32_t (&a)[8], uint32_t (&b)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
                 "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]), "+r"(b[7]));
}

template <int D, int N>
__global__ void __launch_bounds__(kBlock, 1)
    trunc_pq_backward_kernel(const float* __restrict__ X, int64_t B, int64_t L, int64_t b0,
                             const float* __restrict__ Sin, int64_t s_ld, int64_t s_col0,
                             const float* __restrict__ gup, int64_t g_ld, int64_t g_col0,
                             float* __restrict__ partial) {
  using Q_ = PQ<D, N>;
  constexpr int QPG = Q_::QPG, GPC = Q_::GPC, CPP = Q_::CPP, NC = Q_::NC;
  extern __shared__ __align__(1024) unsigned char sm[];
  __half* A1h = reinterpret_cast<__half*>(sm + Q_::oA1h);
  __half* A1l = reinterpret_cast<__half*>(sm + Q_::oA1l);
  __half* A2h = reinterpret_cast<__half*>(sm + Q_::oA2h);
  __half* A2l = reinterpret_cast<__half*>(sm + Q_::oA2l);
  auto Bhi = [&](int db) { return reinterpret_cast<__half*>(sm + Q_::oB + db * 2 * Q_::kBBytes); };
  auto Blo = [&](int db) { return reinterpret_cast<__half*>(sm + Q_::oB + db * 2 * Q_::kBBytes + Q_::kBBytes); };
  auto Xsb = [&](int db) { return reinterpret_cast<float*>(sm + Q_::oXs) + db * (CH + 1) * D; };
  auto Dlb = [&](int db) { return reinterpret_cast<float*>(sm + Q_::oDl) + db * CH * D; };
  float(*red)[8][CH][D] = reinterpret_cast<float(*)[8][CH][D]>(sm + Q_::oRed);
  auto isig = [&](int db) { return reinterpret_cast<float*>(sm + Q_::oSig) + db * CH; };
  float* park = reinterpret_cast<float*>(sm + Q_::oPark);
  float4* cbuf = reinterpret_cast<float4*>(sm + Q_::oCb) + (threadIdx.x >> 5) * NG * 8;  // this warp's chain values
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + Q_::oBar);
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + Q_::oSlot);

  // warp index through a shuffle: provably warp-uniform, so the producer branch is uniform and the
  // MMA issue inside it compiles to plain uniform-datapath UTCHMMAs (no per-MMA collective sequence)
  const int tid = threadIdx.x, lane = tid & 31, warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const bool producer = warp == kThreads / 32;
  const int64_t b = b0 + blockIdx.x / CPP;  // the grid covers live paths only
  const int cip = blockIdx.x % CPP;
  const int q = lane & (QPG - 1);  // letter quad
  // grand-parent (level N-2 word, 0 .. D^(N-2)-1); the producer warp's value is unused but valid
  const int gp = ((cip * kThreads + tid) / QPG) % Q_::NGP;
  int cl[NC];  // the chain's letters: node k (level k+1) ends with letter cl[k]
  {
    int code = gp;
#pragma unroll
    for (int k = NC - 1; k >= 0; --k) {
      cl[k] = code % D;
      code /= D;
    }
  }
  auto chain_index = [&](int k) { return Q_::off(k + 1) + gp / trunc::ipow(D, NC - 1 - k); };
  auto par_index = [&](int y) { return Q_::off(N - 1) + (int64_t)gp * D + y; };
  const int64_t M = L - 1;
  const int r = 32 * (warp & 3) + lane;       // this thread's row in every tile = its TMEM lane
  const int mt0 = (warp >> 2) * 4;            // its tiles mt0 .. mt0 + 3
  const uint32_t lane_addr = (uint32_t)(32 * (warp & 3)) << 16;

  if (producer) {
    tcu::tmem_alloc<512>(slot);
    if (lane == 0) {
      tcu::mbar_init(&mbar[0], 1);  // MMA groups: one tcgen05.commit each per chunk
      tcu::mbar_init(&mbar[1], 1);
      tcu::mbar_init(&mbar[2], 32);  // increments / B of buffer 0, 1 ready: the producer's 32 lanes
      tcu::mbar_init(&mbar[3], 32);
    }
  }

  const int nchunks = (int)((M + CH - 1) / CH);
  auto chunk_len = [&](int c) { return (int)(M - (int64_t)c * CH < CH ? M - (int64_t)c * CH : CH); };
  auto stage = [&](int c, int db) {  // producer: cp.async of chunk c's samples into Xs[db]
    const int rows = chunk_len(c) + 1;
    const float* src = X + (b * L + (int64_t)c * CH) * D;
    float* dst = Xsb(db);
    for (int i = lane; i < rows * D; i += 32)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tcu::su32(dst + i)), "l"(src + i) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto prepare = [&](int c, int db, bool newest_in_flight) {  // producer: Dl[db], B[db], 1/sigma[db] of chunk c
    if (newest_in_flight) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    const int cs = chunk_len(c);
    const float4* xs = reinterpret_cast<const float4*>(Xsb(db));
    float4* dl = reinterpret_cast<float4*>(Dlb(db));
    for (int i = lane; i < cs * D / 4; i += 32) {
      const float4 a = xs[i], n = xs[i + D / 4];
      dl[i] = make_float4(n.x - a.x, n.y - a.y, n.z - a.z, n.w - a.w);
    }
    __syncwarp();
    float v[16];  // lane = step row of B; rows past the chunk are zero
#pragma unroll
    for (int z4 = 0; z4 < 4; ++z4) {
      const float4 t = (lane < cs && 4 * z4 < D) ? dl[lane * (D / 4) + z4 % (D / 4)] : make_float4(0.f, 0.f, 0.f, 0.f);
      v[4 * z4] = t.x; v[4 * z4 + 1] = t.y; v[4 * z4 + 2] = t.z; v[4 * z4 + 3] = t.w;
    }
    float amax = 0.f;
#pragma unroll
    for (int z = 0; z < 16; ++z) amax = fmaxf(amax, fabsf(v[z]));
    const float sc = tcu::pow2_scale(amax);
    isig(db)[lane] = 1.f / sc;
#pragma unroll
    for (int kg = 0; kg < 2; ++kg) {
      float w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = v[8 * kg + i];
      const int off = tcu::kmajor_off16<2>(lane, 8 * kg);
      tcu::split8_store(w, sc, Bhi(db) + off, Blo(db) + off);
    }
    tcu::fence_async_smem();  // generic-proxy writes of B -> the tensor core
    __syncwarp();
  };
  // ---- terminal state, adjoint seeds, P, and the constant A operands ----
  // The CTA's 1,024 x D leaf adjoints (contiguous in the upstream row: the leaves of its GPC
  // grand-parents) and 1,024 parent values are staged in shared memory first (all 288 threads,
  // coalesced cp.async; the A2 region and the parked-sums region are free until the sweep), so
  // each thread reads its A1 rows / A2 columns / P terms from shared memory.
  const float* srow = Sin + b * s_ld + s_col0;
  const float* grow = gup + b * g_ld + g_col0;
  float* lstage = reinterpret_cast<float*>(sm + Q_::oA2h);  // [GPC][D y][D z] fp32 (<= 64 KB = A2 hi + lo)
  float* sstage = reinterpret_cast<float*>(sm + Q_::oRed);  // [GPC][D y] parent values
  // Staged positions.  At d = 16 the 16-byte chunks are XOR-swizzled so that every read below is
  // bank-conflict free: row y of grand-parent gl sits in bank half (y ^ gl) & 1 and its chunk z/4
  // at slot (z/4) ^ (y/4) (the P terms read chunk q of one row across a warp's 8 grand-parents x 4
  // quads, the A1 rows read chunk j of rows 4q+g); a grand-parent's parent values are spread over
  // the banks by (gl/2) & 3.  Chunks stay whole, so 16-byte copies still apply.
  auto lidx = [](int gl, int y, int z) {
    if constexpr (D == 16) return gl * 256 + ((y ^ (gl & 1)) << 4) + ((((z >> 2) ^ (y >> 2)) & 3) << 2) + (z & 3);
    else return (gl * D + y) * D + z;
  };
  auto sidx = [](int gl, int y) {
    if constexpr (D == 16) return gl * 16 + (y ^ (((gl >> 1) & 3) << 2));
    else return gl * D + y;
  };
  {
    // 16-byte copies when the source rows are 16-byte aligned (no epsilon column, aligned tensors;
    // config 5's leaf block starts at word 4,369, so usually not), else 4-byte ones
    auto copy = [&](float* dst, const float* src, int n, auto pos) {
      if (((uintptr_t)src & 15) == 0) {
        for (int i = 4 * tid; i < n; i += 4 * kBlock)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tcu::su32(dst + pos(i))), "l"(src + i)
                       : "memory");
      } else {
        for (int i = tid; i < n; i += kBlock)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tcu::su32(dst + pos(i))), "l"(src + i)
                       : "memory");
      }
    };
    copy(lstage, grow + Q_::off(N) + (int64_t)cip * GPC * D * D, GPC * D * D,
         [&](int i) { return lidx(i / (D * D), (i / D) % D, i % D); });
    copy(sstage, srow + Q_::off(N - 1) + (int64_t)cip * GPC * D, GPC * D, [&](int i) { return sidx(i / D, i % D); });
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (producer && nchunks > 0) {  // the first two chunks' samples load under the setup
    stage(nchunks - 1, 0);
    if (nchunks > 1) stage(nchunks - 2, 1);
  }
  // chain values S_j and (partial) adjoints; a node is seeded once (the owner).  Depth 4: sc holds
  // the chain of the grand-parent this lane walks in chain_pre, (gp & ~7) + (lane & 7)
  float sc[NC], lc[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    if constexpr (Q_::kDeferChain) {
      const int gps = (gp & ~7) + (lane & 7);
      sc[k] = srow[k == 0 ? Q_::off(1) + gps / D : Q_::off(2) + gps];
    } else {
      sc[k] = srow[chain_index(k)];
    }
    const bool owner = q == 0 && gp % trunc::ipow(D, NC - 1 - k) == 0;
    lc[k] = owner ? grow[chain_index(k)] : 0.f;
  }
  // deferred chain (depth 4): the swept grand-parent (gp & ~7) + (lane & 7)'s adjoints -- level 2
  // (its own node) and its share of level 1 (seeded by the first grand-parent under that letter)
  float sw1 = 0.f, sw0 = 0.f;
  if constexpr (Q_::kDeferChain) {
    const int gps = (gp & ~7) + (lane & 7);
    sw1 = grow[Q_::off(2) + gps];
    sw0 = gps % D == 0 ? grow[Q_::off(1) + gps / D] : 0.f;
  }
  float lm_[4], P[4] = {0.f, 0.f, 0.f, 0.f};  // (the P/Q form never reads the parents' S_j)
#pragma unroll
  for (int g = 0; g < 4; ++g) lm_[g] = grow[par_index(4 * q + g)];
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const int gl_ = (gp - GPC * cip) & (GPC - 1);  // grand-parent within the CTA (valid for the producer too)
  // Lambda[gl_, y, 4j .. 4j+3] as a float4
  auto lchunk = [&](int y, int j) { return *reinterpret_cast<const float4*>(lstage + lidx(gl_, y, 4 * j)); };
  float a2v[4][D];  // Lambda[gp, y, 4q + i]: this thread's A2 rows (held across the barrier below)
  float amax1 = 0.f, amax2 = 0.f;
#pragma unroll
  for (int y = 0; y < D; ++y) {
    const float sy = sstage[sidx(gl_, y)];
    const float4 l4 = lchunk(y, q);
    a2v[0][y] = l4.x; a2v[1][y] = l4.y; a2v[2][y] = l4.z; a2v[3][y] = l4.w;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      P[i] = fmaf(a2v[i][y], sy, P[i]);
      amax2 = fmaxf(amax2, fabsf(a2v[i][y]));
    }
  }
#pragma unroll
  for (int g = 0; g < 4; ++g)
#pragma unroll
    for (int j = 0; j < D / 4; ++j) {
      const float4 t = lchunk(4 * q + g, j);
      amax1 = fmaxf(fmaxf(amax1, fmaxf(fabsf(t.x), fabsf(t.y))), fmaxf(fabsf(t.z), fabsf(t.w)));
    }
  // depth 4: one scale per grand-parent (the quad's max over both operands), so chain_pre can fold
  // it into the step's chain values; elsewhere one per thread and operand
  if constexpr (Q_::kDeferChain) {
    amax1 = fmaxf(amax1, amax2);
    amax1 = fmaxf(amax1, __shfl_xor_sync(0xffffffffu, amax1, 1));
    amax1 = fmaxf(amax1, __shfl_xor_sync(0xffffffffu, amax1, 2));
    amax2 = amax1;
  }
  const float s1 = tcu::pow2_scale(amax1), s2 = tcu::pow2_scale(amax2);
  const float inv_s1 = 1.f / s1, inv_s2 = 1.f / s2;  // exact: powers of two
  const float inv_s1h = 0.5f * inv_s1;
  // the scale of the grand-parent this lane walks in chain_pre, (gp & ~7) + (lane & 7)
  const float inv_sp = __shfl_sync(0xffffffffu, inv_s1, 4 * (lane & 7));
  if (!producer) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {  // A1 row (tile mt0 + g) = parent gp.(4q+g), K = leaf letter z (zero-padded)
#pragma unroll
      for (int kg = 0; kg < 2; ++kg) {
        float v[8];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float4 t = 8 * kg + 4 * h < D ? lchunk(4 * q + g, 2 * kg + h) : make_float4(0.f, 0.f, 0.f, 0.f);
          v[4 * h] = t.x; v[4 * h + 1] = t.y; v[4 * h + 2] = t.z; v[4 * h + 3] = t.w;
        }
        const int off = (mt0 + g) * kRowHalves + tcu::kmajor_off16<2>(r, 8 * kg);
        tcu::split8_store(v, s1, A1h + off, A1l + off);
      }
    }
  }
  if (producer && nchunks > 0) {  // chunk 0's increments and B, prepared while the A operands are built
    prepare(nchunks - 1, 0, false);
    if (nchunks > 2) stage(nchunks - 3, 0);
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(tcu::su32(&mbar[2])) : "memory");
  }
  __syncthreads();  // the staged leaf adjoints are read: their region becomes A2
  if (!producer) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // A2 row (tile mt0 + i) = pair (gp, 4q+i), K = parent letter y (zero-padded)
#pragma unroll
      for (int kg = 0; kg < 2; ++kg) {
        float v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = 8 * kg + k < D ? a2v[i][(8 * kg + k) % D] : 0.f;
        const int off = (mt0 + i) * kRowHalves + tcu::kmajor_off16<2>(r, 8 * kg);
        tcu::split8_store(v, s2, A2h + off, A2l + off);
      }
    }
  }
  tcu::fence_async_smem();  // the A operands (generic-proxy stores) -> the tensor core's async proxy
  tcu::fence_before();
  __syncthreads();
  tcu::fence_after();
  // the CTA owns all 512 columns, so the allocator can only return lane 0 / column 0: the TMEM
  // addresses below are compile-time constants (uniform-datapath MMA issue, no per-MMA R2UR)
  if (*slot != 0u) __trap();
  constexpr uint32_t tmem = 0u;
  // chain letters' home lanes: mk[k][i] selects slot i (letter 4q+i) of the lane whose quad holds cl[k]
  // (the in-loop chain of depth > 4 only)
  float mk[NC][4];
#pragma unroll
  for (int k = 0; k < NC; ++k)
#pragma unroll
    for (int i = 0; i < 4; ++i) mk[k][i] = (q == (cl[k] >> 2) && i == (cl[k] & 3)) ? 1.f : 0.f;
  const int my_letter = 4 * q + ((lane & 16) ? 2 : 0) + ((lane & 8) ? 1 : 0);
  // lanes summed plainly in the letter reduction (the grand-parent bits below bit 3)
  constexpr int kPlainMask = (8 - 1) & ~(QPG - 1);

  // ---- chunk pipeline (chunk k = the k-th processed, c = nchunks-1-k; buffers by k & 1).
  // The producer warp stages samples two chunks ahead (cp.async), forms increments, B and
  // 1/sigma one chunk ahead (mbarrier "ready" per buffer), issues each MMA group of chunk k+1
  // as soon as the compute warps release that TMEM half in chunk k (named barriers 1, 2), and
  // runs the chunk epilogue; the compute warps never wait on a CTA-wide barrier.
  auto issue = [&](int h, int db) {  // producer: the 48 MMAs of group h (steps 16h .. 16h+15) from B[db]
    constexpr uint32_t id = tcu::idesc_f16(128, NG);
    const uint64_t bh = tcu::smem_desc(tcu::su32(Bhi(db) + h * NG * 16), 128, 256);
    const uint64_t bl = tcu::smem_desc(tcu::su32(Blo(db) + h * NG * 16), 128, 256);
#pragma unroll
    for (int mt = 0; mt < kTiles; ++mt) {
      const uint32_t d1 = tmem + h * 256 + mt * NG, d2 = d1 + 128;
      const uint64_t a1h = tcu::smem_desc(tcu::su32(A1h + mt * kRowHalves), 128, 256);
      const uint64_t a1l = tcu::smem_desc(tcu::su32(A1l + mt * kRowHalves), 128, 256);
      const uint64_t a2h = tcu::smem_desc(tcu::su32(A2h + mt * kRowHalves), 128, 256);
      const uint64_t a2l = tcu::smem_desc(tcu::su32(A2l + mt * kRowHalves), 128, 256);
      tcu::mma_ss_f16(d1, a1h, bh, id, 0u);
      tcu::mma_ss_f16(d1, a1l, bh, id, 1u);
      tcu::mma_ss_f16(d1, a1h, bl, id, 1u);
      tcu::mma_ss_f16(d2, a2h, bh, id, 0u);
      tcu::mma_ss_f16(d2, a2l, bh, id, 1u);
      tcu::mma_ss_f16(d2, a2h, bl, id, 1u);
    }
    tcu::mma_commit(&mbar[h]);
  };

  // one reverse step s of the current chunk; rr = the TMEM products of step s (D1 then D2)
  // a step's increments (its quad's 4 letters, the chain letters) and 1/sigma, fetched one step
  // ahead so the next step's shared loads sit above this step's parked-sum store
  // (depth 4: the chain values come precomputed per step from chain_pre instead, cb)
  struct Inc {
    float4 y;
    float dc[NC];
    float is;
    float4 cb;  // depth 4: (Tr(gp,3) / sigma, T(gp,3), T(gp,4) / (2 sigma), 1 / sigma)
  };
  auto fetch = [&](int s, const float* dl, const float* isg, int lo) {
    const float* row = dl + s * D;
    Inc in;
    in.y = *reinterpret_cast<const float4*>(row + 4 * q);
    if constexpr (Q_::kDeferChain) {
      in.cb = cbuf[(s - lo) * 8 + (lane >> 2)];
    } else {
#pragma unroll
      for (int k = 0; k < NC; ++k) in.dc[k] = row[cl[k]];
      in.is = isg[s];
    }
    return in;
  };
  // a step's letter sums before the cross-lane reduction: the reduction of step s is issued after
  // the arithmetic of step s-1 (source order), so its shuffle latency overlaps that arithmetic
  struct Sums {
    float v[4], gc[NC];  // depth 4: gc[0], gc[1] = this lane's parent-adjoint sums T1, T2 (see park)
  };
  float* park_w = park + warp * CH * 32;
  auto reduce = [&](Sums& u, int s, float(*redw)[D]) {
    float* v = u.v;
    if constexpr (Q_::kDeferChain) {
      // park the grand-parent's T1 = Tbar(gp, 3), T2 = Tbar(gp, 4) contributions (summed over the quad:
      // transposing over lane bit 0, then plain over bit 1) for the deferred sweep (quad lanes 2, 3
      // of the park row hold the chain inputs, written by chain_pre)
      const bool b0 = (lane & 1) != 0;
      float keep = b0 ? u.gc[1] : u.gc[0];
      keep += __shfl_xor_sync(0xffffffffu, b0 ? u.gc[0] : u.gc[1], 1);
      keep += __shfl_xor_sync(0xffffffffu, keep, 2);
      if (!(lane & 2)) park_w[s * 32 + lane] = keep;
    } else {
      // the quad group's partial chain terms -> full per grand-parent, added at the lane of their letter
#pragma unroll
      for (int msk = 1; msk < QPG; msk *= 2)
#pragma unroll
        for (int k = 0; k < NC; ++k) u.gc[k] += __shfl_xor_sync(0xffffffffu, u.gc[k], msk);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int k = 0; k < NC; ++k) v[i] = fmaf(mk[k][i], u.gc[k], v[i]);
    }
    // sum over the warp's grand-parents: transposing over lane bits 4 and 3 (one letter per lane
    // group), plain over the grand-parent bits below
    const bool u4 = (lane & 16) != 0, u3 = (lane & 8) != 0;
    {
      const float s0 = u4 ? v[0] : v[2], s1v = u4 ? v[1] : v[3];
      const float k0 = u4 ? v[2] : v[0], k1v = u4 ? v[3] : v[1];
      v[0] = k0 + __shfl_xor_sync(0xffffffffu, s0, 16);
      v[1] = k1v + __shfl_xor_sync(0xffffffffu, s1v, 16);
    }
    {
      const float snd = u3 ? v[0] : v[1], kp = u3 ? v[1] : v[0];
      v[0] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
    }
#pragma unroll
    for (int msk = 4; msk >= QPG; msk /= 2) v[0] += __shfl_xor_sync(0xffffffffu, v[0], msk);
    if ((lane & kPlainMask) == 0) redw[s][my_letter] = v[0];
  };
  auto step = [&](const Inc& in, const uint32_t (&rr)[8]) -> Sums {
    const float dy[4] = {in.y.x, in.y.y, in.y.z, in.y.w};
    float is = 0.f, trN1, tN1, tN;
    float tp[NC][N + 1];  // forward partials T(chain_k, m) from S_j (m = k+1 .. N)
    float pq, gq, gt, k1;  // the MMA products carry the operand scales: D1 = Tbar(u, N) / k1, D2 = Q / k2
    if constexpr (Q_::kDeferChain) {
      // chain_pre folded the grand-parent's scale (k1 = k2 = 1 / (s sigma)): cb = (-Tr(gp,3) k, T(gp,3),
      // T(gp,4)/2 k, k)
      pq = in.cb.x;
      tN1 = in.cb.y;
      gq = gt = in.cb.z;
      k1 = in.cb.w;
    } else {
      // (a) reconstruct S_j = S_{j+1} (x) exp(-dX_j) on the chain: partials of the exp(-dX) step
      // (targets up to N-1; Tr(gp, N-1) drives the parents' and P's reconstruction)
      float tn[NC][N];
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const int lv = k + 1;
#pragma unroll
        for (int m = lv; m < N; ++m) {
          const float a = -in.dc[k] * (1.f / (float)(m - lv + 1));
          tn[k][m] = (k == 0) ? sc[k] + a : fmaf(a, tn[k > 0 ? k - 1 : 0][m], sc[k]);
        }
      }
      trN1 = tn[NC - 1][N - 1];  // Tr(gp, N-1)
#pragma unroll
      for (int k = 0; k < NC; ++k) sc[k] = tn[k][k + 1];
      // (b) forward partials from S_j
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const int lv = k + 1;
#pragma unroll
        for (int m = lv; m <= N; ++m) {
          const float a = in.dc[k] * (1.f / (float)(m - lv + 1));
          tp[k][m] = (k == 0) ? sc[k] + a : fmaf(a, tp[k > 0 ? k - 1 : 0][m], sc[k]);
        }
      }
      tN1 = tp[NC - 1][N - 1];  // T(gp, N-1)
      tN = tp[NC - 1][N];       // T(gp, N)
      is = in.is;
      const float k2 = inv_s2 * is;
      pq = -trN1 * k2;
      gq = 0.5f * tN * k2;
      k1 = inv_s1 * is;
      gt = 0.5f * tN * k1;
    }
    Sums out;
    float* v = out.v;
    float tbp1 = 0.f, tbp2u = 0.f;  // Tbar(gp, N-1), Tbar(gp, N) / k1 from the parents
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      // leaf pairs: P_j = P_{j+1} - Tr(gp,N-1) Q_j;  gl = P_j + T(gp,N)/2 Q_j
      const float Di = __uint_as_float(rr[4 + i]);
      P[i] = fmaf(pq, Di, P[i]);
      // parent u = gp.(4q+i): adjoint pull-back from its leaves, gradient of its letter
      const float Du = __uint_as_float(rr[i]);  // Tbar(u, N) / k1
      const float lm = lm_[i];                  // Tbar(u, N-1)
      tbp1 = fmaf(dy[i], lm, tbp1);
      tbp2u = fmaf(dy[i], Du, tbp2u);
      // letter 4q+i: leaf term P_j + T(gp,N)/2 Q_j, parent term Tbar(u,N-1) T(gp,N-1) + Tbar(u,N) T(gp,N)/2
      v[i] = fmaf(gt, Du, fmaf(lm, tN1, fmaf(gq, Di, P[i])));
      lm_[i] = fmaf(Du, k1, lm);
    }
    // Tbar(gp, N): depth 4 parks it doubled (the sweep halves it once per grand-parent)
    const float tbp2 = Q_::kDeferChain ? k1 * tbp2u : (inv_s1h * is) * tbp2u;
    // chain, deepest first (trunc_backward_kernel (c)): tbc[m] = Tbar contributed by the child
    if constexpr (Q_::kDeferChain) {
      // the chain's reverse is a pure sink (its adjoints feed only the chain letters' gradients):
      // swept once per grand-parent after the chunk (chain_sweep), from the parked T1, T2, S_j
      out.gc[0] = tbp1;
      out.gc[1] = tbp2;
    } else {
      float tbc[N + 1];
#pragma unroll
      for (int m = 0; m <= N; ++m) tbc[m] = 0.f;
      tbc[N - 1] = tbp1;
      tbc[N] = tbp2;
#pragma unroll
      for (int k = NC - 1; k >= 0; --k) {
        const int lv = k + 1;
        float tbn[N + 1];
#pragma unroll
        for (int m = 0; m <= N; ++m) tbn[m] = (m == lv) ? lc[k] : tbc[m];
        float lsum = tbn[lv], gs = 0.f;
#pragma unroll
        for (int m = lv; m <= N; ++m) {
          if (m > lv) lsum += tbn[m];
          const float par = (k == 0) ? 1.f : tp[k > 0 ? k - 1 : 0][m];
          gs = fmaf(tbn[m] * (1.f / (float)(m - lv + 1)), par, gs);
        }
        lc[k] = lsum;
        out.gc[k] = gs;
#pragma unroll
        for (int m = 0; m <= N; ++m)
          tbc[m] = (m >= lv) ? in.dc[k] * (1.f / (float)(m - lv + 1 > 0 ? m - lv + 1 : 1)) * tbn[m] : 0.f;
      }
    }
    return out;
  };

  // Depth 4: the chain values of the warp's 8 grand-parents for the steps lo..hi of one MMA group,
  // computed before the group's steps (under its MMA wait) instead of by every quad lane per step.
  // Lane (g = lane & 7, quarter qq = lane >> 3) walks grand-parent (gp & ~7) + g over steps
  // lo+4qq+3 .. lo+4qq; the state entering its quarter comes from a suffix scan of the quarter maps
  //   (S1, S2) -> (S1 - A, S2 - S1 Bs + C),  A = sum d0, Bs = sum d1, C = sum d1 (a + d0 / 2)
  // (S1 = S_j(la), S2 = S_j(gp), a = the quarter's d0 after the step), composed upper then lower as
  //   (A_u + A_l, Bs_u + Bs_l, C_u + C_l + A_u Bs_l).
  // Writes cbuf[s - lo][g] for the steps and the park row's chain inputs (quad lanes 2, 3: d1, and
  // S_j(la) for even / d0 for odd grand-parents), and carries sc below the group.
  auto chain_pre = [&](const float* dl, const float* isg, int lo, int hi) {
    if constexpr (Q_::kDeferChain) {
      __syncwarp();  // the previous group's steps have read cbuf
      const int g = lane & 7, qq = lane >> 3;
      const int gps = (gp & ~7) + g, c0 = gps / D, c1 = gps % D;
      float d0v[4], d1v[4], A = 0.f, Bs = 0.f, C = 0.f;
#pragma unroll
      for (int i = 3; i >= 0; --i) {
        const int st = lo + 4 * qq + i;
        d0v[i] = st <= hi ? dl[st * D + c0] : 0.f;
        d1v[i] = st <= hi ? dl[st * D + c1] : 0.f;
        C = fmaf(d1v[i], A + 0.5f * d0v[i], C);
        A += d0v[i];
        Bs += d1v[i];
      }
#pragma unroll
      for (int off = 8; off <= 16; off *= 2) {  // inclusive suffix scan over the quarters
        const float oA = __shfl_down_sync(0xffffffffu, A, off);
        const float oB = __shfl_down_sync(0xffffffffu, Bs, off);
        const float oC = __shfl_down_sync(0xffffffffu, C, off);
        if (qq + off / 8 <= 3) {
          C = fmaf(oA, Bs, C + oC);
          A += oA;
          Bs += oB;
        }
      }
      float eA = __shfl_down_sync(0xffffffffu, A, 8);  // exclusive: the quarters above this one
      float eB = __shfl_down_sync(0xffffffffu, Bs, 8);
      float eC = __shfl_down_sync(0xffffffffu, C, 8);
      if (qq == 3) eA = eB = eC = 0.f;
      float s0 = sc[0] - eA, s1 = fmaf(-sc[0], eB, sc[1] + eC);
#pragma unroll
      for (int i = 3; i >= 0; --i) {
        const int st = lo + 4 * qq + i;
        const float d0 = d0v[i], d1 = d1v[i];
        const float trN1 = fmaf(-0.5f * d1, s0 - d0 * (1.f / 3.f), s1);  // Tr(gp, 3): the exp(-dX) partial
        const float ns1 = fmaf(-d1, s0 - 0.5f * d0, s1);
        s0 = s0 - d0;
        s1 = ns1;
        const float tN1 = fmaf(0.5f * d1, fmaf(1.f / 3.f, d0, s0), s1);        // T(gp, 3)
        const float tN = fmaf(d1 * (1.f / 3.f), fmaf(0.25f, d0, s0), s1);      // T(gp, 4)
        if (st <= hi) {
          const float is = isg[st];
          const float k = inv_sp * is;
          cbuf[(st - lo) * 8 + g] = make_float4(-trN1 * k, tN1, 0.5f * tN * k, k);
          *reinterpret_cast<float2*>(park_w + st * 32 + 4 * g + 2) = make_float2(d1, (g & 1) ? d0 : s0);
        }
      }
      sc[0] = __shfl_sync(0xffffffffu, s0, g);  // the state below the group: quarter 0's walk
      sc[1] = __shfl_sync(0xffffffffu, s1, g);
      __syncwarp();
    }
  };

  // chunk epilogue: fixed-order sum over the 8 compute warps' parked letter sums of chunk c (buffer
  // db) -> partial[path part][step][letter], four letters per float4
  auto sum_parked = [&](int db, int cs, int c, int t0, int nt) {
    float4* dst = reinterpret_cast<float4*>(partial + (((b - b0) * CPP + cip) * M + (int64_t)c * CH) * D);
    for (int i = t0; i < cs * D / 4; i += nt) {
      float4 w[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) w[k] = reinterpret_cast<const float4*>(&red[db][k][0][0])[i];
      auto add = [](float4 a, float4 b) {  // two packed f32x2 adds (the producer shares a scheduler)
        const float2 lo = __fadd2_rn(make_float2(a.x, a.y), make_float2(b.x, b.y));
        const float2 hi = __fadd2_rn(make_float2(a.z, a.w), make_float2(b.z, b.w));
        return make_float4(lo.x, lo.y, hi.x, hi.y);
      };
      dst[i] = add(add(add(w[0], w[1]), add(w[2], w[3])), add(add(w[4], w[5]), add(w[6], w[7])));
    }
  };

  // Deferred chain sweep of one chunk (depth 4), per compute warp after its steps: lane (g, quarter
  // qq) walks grand-parent g's chain over steps 8qq+7 .. 8qq (high to low, as the reverse sweep),
  // the carried adjoints entering each quarter through a suffix scan over the quad:
  //   Tbar(gp,2): n2 <- n2 + T1 + T2,  gl[cl1] += n2 T(la,2) + T1/2 T(la,3) + T2/3 T(la,4)
  //   Tbar(la,1): m1 <- m1 + c2 + c3 + c4 (c = d1 n2, d1 T1/2, d1 T2/3),
  //               gl[cl0] += m1 + c2/2 + c3/3 + c4/4           (trunc_backward_kernel (c), depth 4)
  // with T(la, m) = S_j(la) + d0/m.  The chain letters' sums are added to the warp's parked letter
  // sums (cl1 per grand-parent; cl0 is common to the warp's 8 grand-parents: summed over them first).
  auto chain_sweep = [&](int db, int cs, float(*redw)[D]) {
    if constexpr (Q_::kDeferChain) {
      __syncwarp();  // the parked values and the steps' letter sums of this warp
      // lane = (grand-parent g = lane & 7, quarter qq = lane >> 3): a quarter's 8 grand-parents read
      // one 128-byte park row per step (conflict-free)
      const int g = lane & 7, qq = lane >> 3;
      const int gps = (gp & ~7) + g;  // the swept grand-parent
      const int c0 = gps / D, c1 = gps % D;
      float t1[8], t2[8], s0[8], d0[8], d1[8];
      float A = 0.f;
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        const int st = 8 * qq + i;
        float4 pk = make_float4(0.f, 0.f, 0.f, 0.f);
        if (st < cs) pk = *reinterpret_cast<const float4*>(park_w + st * 32 + 4 * g);
        const float other = __shfl_xor_sync(0xffffffffu, pk.w, 1);
        t1[i] = pk.x; t2[i] = 0.5f * pk.y; d1[i] = pk.z;  // T2 was parked doubled
        s0[i] = (g & 1) ? other : pk.w;
        d0[i] = (g & 1) ? pk.w : other;
        A += t1[i] + t2[i];
      }
      // suffix scan over the quarters (quarter 3 is swept first): carry-in and chunk total
      auto scan = [&](float x, float& carry_in, float& total) {
        float inc = x;
        float o = __shfl_down_sync(0xffffffffu, inc, 8);
        if (qq < 3) inc += o;
        o = __shfl_down_sync(0xffffffffu, inc, 16);
        if (qq < 2) inc += o;
        o = __shfl_down_sync(0xffffffffu, inc, 8);
        carry_in = qq < 3 ? o : 0.f;
        total = __shfl_sync(0xffffffffu, inc, g);
      };
      float in1, tot1;
      scan(A, in1, tot1);
      float n2 = sw1 + in1, C = 0.f;
      float cg[8], csum[8];
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        // with T(la, m) = S + d0/m the terms regroup into u = n2 + n3/2 + n4/3 and
        // w = n2/2 + n3/6 + n4/12:  gl[cl1] += S u + d0 w,  c2 + c3 + c4 = d1 u,  c2/2 + c3/3 + c4/4 = d1 w
        const float n3 = t1[i], n4 = t2[i];
        const float u = fmaf(0.5f, n3, fmaf(1.f / 3.f, n4, n2));
        const float w = fmaf(0.5f, n2, fmaf(1.f / 6.f, n3, (1.f / 12.f) * n4));
        const float gc1 = fmaf(s0[i], u, d0[i] * w);
        n2 = n2 + n3 + n4;
        cg[i] = d1[i] * w;
        csum[i] = d1[i] * u;
        C += csum[i];
        const int st = 8 * qq + i;
        if (st < cs) redw[st][c1] += gc1;
      }
      float in2, tot2;
      scan(C, in2, tot2);
      __syncwarp();  // the cl1 additions above may target a cl0 entry added below
      float m1 = sw0 + in2;
      float t[8];
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        t[i] = m1 + cg[i];
        m1 += csum[i];
      }
      // sum over the 8 grand-parents transposing over lane bits 2, 1, 0: lane g ends with step 8qq+g
      float u[4], w[2];
      const bool b2 = (g & 4) != 0, b1 = (g & 2) != 0, b0 = (g & 1) != 0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        u[k] = (b2 ? t[4 + k] : t[k]) + __shfl_xor_sync(0xffffffffu, b2 ? t[k] : t[4 + k], 4);
#pragma unroll
      for (int k = 0; k < 2; ++k)
        w[k] = (b1 ? u[2 + k] : u[k]) + __shfl_xor_sync(0xffffffffu, b1 ? u[k] : u[2 + k], 2);
      const float tg = (b0 ? w[1] : w[0]) + __shfl_xor_sync(0xffffffffu, b0 ? w[0] : w[1], 1);
      if (8 * qq + g < cs) redw[8 * qq + g][c0] += tg;
      sw1 += tot1;
      sw0 += tot2;
    }
  };

  if (producer) {
    if (nchunks > 0) {  // chunk 0 was staged and prepared during the setup
      issue(1, 0);
      issue(0, 0);
    }
    for (int k = 0; k < nchunks; ++k) {
      const int c = nchunks - 1 - k, db = k & 1;
      if (k + 1 < nchunks) {  // increments / B of chunk k+1 (its samples were staged two chunks ago)
        prepare(c - 1, db ^ 1, k + 2 < nchunks);
        if (k + 3 < nchunks) stage(c - 3, db ^ 1);
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(tcu::su32(&mbar[2 + (db ^ 1)]))
                     : "memory");
      }
      tcu::bar_sync(1, kBlock);  // chunk k's group 1 is read: its TMEM half takes chunk k+1's group 1
      tcu::fence_after();
      if (k + 1 < nchunks) issue(1, db ^ 1);
      tcu::bar_sync(2, kBlock);  // chunk k's group 0 is read and red[db] is complete
      tcu::fence_after();
      if (k + 1 < nchunks) issue(0, db ^ 1);
      // chunk epilogue (the last chunk's is summed by the compute warps, which have nothing else
      // left to do)
      if (k + 1 < nchunks) sum_parked(db, chunk_len(c), c, lane, 32);
    }
  } else {
    for (int k = 0; k < nchunks; ++k) {
      const int c = nchunks - 1 - k, db = k & 1;
      const int cs = chunk_len(c);
      tcu::mbar_wait(&mbar[2 + db], (uint32_t)((k >> 1) & 1));  // increments of chunk k ready
      const float* dl = Dlb(db);
      const float* is = isig(db);
      float(*redw)[D] = red[db][warp];
#pragma unroll 1
      for (int h = 1; h >= 0; --h) {
        const int lo = NG * h, hi = (cs < NG * (h + 1) ? cs : NG * (h + 1)) - 1;
        if (hi >= lo) chain_pre(dl, is, lo, hi);
        tcu::mbar_wait(&mbar[h], (uint32_t)(k & 1));  // group h's products are in TMEM
        tcu::fence_after();
        if (hi >= lo) {
          const uint32_t base = tmem + lane_addr + h * 256 - lo;
          // TMEM products of one step (x1) or of two consecutive steps in one load per tile (x2:
          // column c -> rlo, c + 1 -> rhi)
          auto load1 = [&](uint32_t (&rr)[8], int c) {
#pragma unroll
            for (int g = 0; g < 4; ++g) rr[g] = tcu::tmem_ld1(base + (mt0 + g) * NG + c);
#pragma unroll
            for (int i = 0; i < 4; ++i) rr[4 + i] = tcu::tmem_ld1(base + 128 + (mt0 + i) * NG + c);
          };
          auto load2 = [&](uint32_t (&rlo)[8], uint32_t (&rhi)[8], int c) {
#pragma unroll
            for (int g = 0; g < 4; ++g) tcu::tmem_ld2(base + (mt0 + g) * NG + c, rlo[g], rhi[g]);
#pragma unroll
            for (int i = 0; i < 4; ++i) tcu::tmem_ld2(base + 128 + (mt0 + i) * NG + c, rlo[4 + i], rhi[4 + i]);
          };
          // step hi alone; then pairs (s, s-1) whose products land in one register-set pair while the
          // previous pair computes; each step's arithmetic precedes the previous step's reduction
          uint32_t ra[8], rb[8], rc[8], rd[8];
          Inc ia, ib, ic, id;
          load1(ra, hi);
          ia = fetch(hi, dl, is, lo);
          int s = hi - 1;
          auto issue_next = [&](uint32_t (&rlo)[8], uint32_t (&rhi)[8], Inc& ilo, Inc& ihi, int top) {
            if (top - 1 >= lo) {
              load2(rlo, rhi, top - 1);
              ihi = fetch(top, dl, is, lo);
              ilo = fetch(top - 1, dl, is, lo);
            } else if (top >= lo) {
              load1(rhi, top);
              ihi = fetch(top, dl, is, lo);
            }
          };
          issue_next(rc, rd, ic, id, s);
          ld_wait8(ra);
          Sums pend = step(ia, ra);
          bool in_second = false;
#pragma unroll 1
          for (;;) {
            if (s - 1 < lo) break;
            ld_wait16(rc, rd);
            issue_next(ra, rb, ia, ib, s - 2);
            {
              Sums cur = step(id, rd);
              reduce(pend, s + 1, redw);
              pend = step(ic, rc);
              reduce(cur, s, redw);
            }
            s -= 2;
            if (s - 1 < lo) {
              in_second = true;
              break;
            }
            ld_wait16(ra, rb);
            issue_next(rc, rd, ic, id, s - 2);
            {
              Sums cur = step(ib, rb);
              reduce(pend, s + 1, redw);
              pend = step(ia, ra);
              reduce(cur, s, redw);
            }
            s -= 2;
          }
          if (s == lo) {  // one step left, in rd (or rb)
            Sums cur;
            if (in_second) {
              ld_wait8(rb);
              cur = step(ib, rb);
            } else {
              ld_wait8(rd);
              cur = step(id, rd);
            }
            reduce(pend, s + 1, redw);
            pend = cur;
            s -= 1;
          }
          reduce(pend, s + 1, redw);
        }
        if (h == 0) chain_sweep(db, cs, redw);  // before red[db] is released to the epilogue
        tcu::fence_before();
        tcu::bar_arrive(h == 1 ? 1 : 2, kBlock);
      }
    }
    if (nchunks > 0) {  // the last chunk's epilogue (chunk c = 0), in the same fixed order
      tcu::bar_sync(4, kThreads);
      sum_parked((nchunks - 1) & 1, chunk_len(0), 0, tid, kThreads);
    }
  }
  tcu::fence_before();
  __syncthreads();
  if (producer) tcu::tmem_dealloc<512>(tmem);
}

}  // namespace pq
}  // namespace trunc
}  // namespace sigb
