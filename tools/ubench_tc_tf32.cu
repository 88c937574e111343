// Microbenchmark / correctness probe for the tensor-core leaf level planned for
// the truncated kernels (DESIGN.md §9 item 1): tcgen05.mma kind::tf32 with
// M = 128 words, N = 16 letters, K = 8 steps per instruction, accumulators in
// TMEM, fp32 operands split hi/lo into tf32 (3xTF32: hi*hi + hi*lo + lo*hi).
//
// Checks, against an fp64 host product:
//   1. A and B from shared memory (SS form), canonical K-major no-swizzle
//      layout, both LBO/SBO assignments (prints which one is right);
//   2. A from TMEM (TS form: the producer threads tcgen05.st their rows);
//   3. 1xTF32 vs 3xTF32 error;
// then times back-to-back N=16 MMAs (cycles per instruction).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tc_tf32 tools/ubench_tc_tf32.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int M = 128, N = 16, KT = 8;   // one MMA
constexpr int KS = 32;                   // K steps in the test (4 MMAs)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  return d;                // base offset 0, layout SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4)            // D f32
         | (2u << 7)          // A tf32
         | (2u << 10)         // B tf32
         | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_ss(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_ts_warp(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}

// issued by a converged warp: one elected lane runs the MMA
__device__ __forceinline__ void mma_ss_warp(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar))
               : "memory");
}

__device__ __forceinline__ bool mbar_wait(uint64_t* mbar, uint32_t phase) {
  const uint32_t a = smem_u32(mbar);
  for (int it = 0; it < (1 << 22); ++it) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(a), "r"(phase)
        : "memory");
    if (ok) return true;
  }
  return false;
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// canonical K-major, no swizzle: core matrix = 8 rows x 16 B (4 tf32), stored
// contiguously (128 B); core matrices laid out [row group][k group].
__device__ __forceinline__ int kmajor_off(int row, int k, int kgroups) {
  return ((row >> 3) * kgroups + (k >> 2)) * 32 + (row & 7) * 4 + (k & 3);
}

// mode 0: SS, 1xTF32; 1: SS 3xTF32; 2: TS 3xTF32.  swap: exchange LBO/SBO.
__global__ void k_check(const float* A, const float* B, float* D, int mode, int swap, int* err) {
  __shared__ __align__(1024) float As[2][M * KS];  // hi, lo
  __shared__ __align__(1024) float Bs[2][N * KS];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  // A[m][k] row-major in global, B[n][k] (i.e. B^T, K-major)
  for (int i = tid; i < M * KS; i += blockDim.x) {
    const int m = i / KS, k = i % KS;
    const float x = A[i], h = tf32_hi(x);
    As[0][kmajor_off(m, k, KS / 4)] = h;
    As[1][kmajor_off(m, k, KS / 4)] = tf32_hi(x - h);
  }
  for (int i = tid; i < N * KS; i += blockDim.x) {
    const int n = i / KS, k = i % KS;
    const float x = B[i], h = tf32_hi(x);
    Bs[0][kmajor_off(n, k, KS / 4)] = h;
    Bs[1][kmajor_off(n, k, KS / 4)] = tf32_hi(x - h);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  const uint32_t td = tm;            // D: columns [0, 16)
  const uint32_t ta = tm + 32;       // A (TS mode): columns [32, 32 + 2*KS) hi then lo
  const uint32_t lane_base = (uint32_t)(warp & 3) * 32;
  if (mode == 2) {
    // each thread writes its row (lane) of A hi / lo: row m = tid (128 threads)
    const int m = tid;
    for (int part = 0; part < 2; ++part)
      for (int k0 = 0; k0 < KS; k0 += 8) {
        uint32_t v[8];
        for (int j = 0; j < 8; ++j) {
          const float x = A[m * KS + k0 + j], h = tf32_hi(x);
          v[j] = __float_as_uint(part ? tf32_hi(x - h) : h);
        }
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                ta + (lane_base << 16) + part * KS + k0),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
      }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  if (tid == 0) {
    const uint32_t id = idesc_tf32(M, N);
    const uint32_t lbo = swap ? 256 : 128, sbo = swap ? 128 : 256;  // A: 2 k-groups per MMA
    // per MMA (K = 8): A k-groups kk, kk+1 of the row-group stride KS/4 core matrices
    const uint32_t lboA = swap ? (KS / 4) * 128 : 128, sboA = swap ? 128 : (KS / 4) * 128;
    const uint32_t lboB = lboA, sboB = sboA;
    (void)lbo; (void)sbo;
    uint32_t acc = 0;
    for (int k0 = 0; k0 < KS; k0 += KT) {
      const int pairs = mode == 0 ? 1 : 3;
      for (int p = 0; p < pairs; ++p) {
        const int ah = (p == 2) ? 1 : 0, bh = (p == 1) ? 1 : 0;  // hi*hi, hi*lo, lo*hi
        const uint64_t db = smem_desc(smem_u32(&Bs[bh][kmajor_off(0, k0, KS / 4)]), lboB, sboB);
        if (mode == 2) {
          mma_ts(td, ta + ah * KS + k0, db, id, acc);
        } else {
          const uint64_t da = smem_desc(smem_u32(&As[ah][kmajor_off(0, k0, KS / 4)]), lboA, sboA);
          mma_ss(td, da, db, id, acc);
        }
        acc = 1;
      }
    }
    mma_commit(&mbar);
  }
  __syncwarp();
  if (!mbar_wait(&mbar, 0)) {
    if ((tid & 31) == 0) atomicAdd(err, 1);
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(td + (lane_base << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int n = 0; n < N; ++n) D[tid * N + n] = __uint_as_float(r[n]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

// back-to-back SS MMAs M=128 N=16 K=8 (operands fixed): cycles per instruction
template <int ROT>
__global__ void k_rate(int iters, long long* cyc, int* err) {
  __shared__ __align__(1024) float As[M * KT];
  __shared__ __align__(1024) float Bs[N * KT];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * KT; i += blockDim.x) As[i] = 1e-3f * (i & 7);
  for (int i = tid; i < N * KT; i += blockDim.x) Bs[i] = 1e-3f * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    const uint32_t id = idesc_tf32(M, N);
    const uint64_t da = smem_desc(smem_u32(As), 128, 256), db = smem_desc(smem_u32(Bs), 128, 256);
    const long long t0 = clock64();
    mma_ss(tm, da, db, id, 0);
    for (int i = 1; i < ROT; ++i) mma_ss(tm + i * 16, da, db, id, 0);
    for (int i = ROT; i < iters; i += ROT) {
#pragma unroll
      for (int r = 0; r < ROT; ++r) mma_ss(tm + r * 16, da, db, id, 1);
    }
    mma_commit(&mbar);
    if (!mbar_wait(&mbar, 0)) atomicAdd(err, 1);
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

// TS form: A (128 x 8 tf32) from TMEM columns [256, 264), B from smem, N = NN
template <int ROT, int NN, bool TS>
__global__ void k_rate2(int iters, long long* cyc, int* err) {
  __shared__ __align__(1024) float As[M * KT];
  __shared__ __align__(1024) float Bs[256 * KT];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * KT; i += blockDim.x) As[i] = 1e-3f * (i & 7);
  for (int i = tid; i < 256 * KT; i += blockDim.x) Bs[i] = 1e-3f * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    const uint32_t id = idesc_tf32(M, NN);
    const uint64_t da = smem_desc(smem_u32(As), 128, 256), db = smem_desc(smem_u32(Bs), 128, 256);
    const uint32_t ta = tm + 448;
    const long long t0 = clock64();
    for (int i = 0; i < iters; i += ROT) {
#pragma unroll
      for (int r = 0; r < ROT; ++r) {
        if (TS) mma_ts(tm + r * NN, ta, db, id, i > 0);
        else mma_ss(tm + r * NN, da, db, id, i > 0);
      }
    }
    mma_commit(&mbar);
    if (!mbar_wait(&mbar, 0)) atomicAdd(err, 1);
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// whole warp 0 runs the issue loop; elect.sync inside the asm
template <int ROT, int NN, bool TS = false>
__global__ void k_rate3(int iters, long long* cyc, int* err) {
  __shared__ __align__(1024) float As[M * KT];
  __shared__ __align__(1024) float Bs[256 * KT];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * KT; i += blockDim.x) As[i] = 1e-3f * (i & 7);
  for (int i = tid; i < 256 * KT; i += blockDim.x) Bs[i] = 1e-3f * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  if (warp == 0) {
    const uint32_t id = idesc_tf32(M, NN);
    const uint64_t da = smem_desc(smem_u32(As), 128, 256), db = smem_desc(smem_u32(Bs), 128, 256);
    const long long t0 = clock64();
    for (int i = 0; i < iters; i += ROT) {
#pragma unroll
      for (int r = 0; r < ROT; ++r) {
        if (TS) mma_ts_warp(tm + r * NN, tm + 448 + 8 * r, db, id, i > 0);
        else mma_ss_warp(tm + r * NN, da, db, id, i > 0);
      }
    }
    if (tid == 0) {
      mma_commit(&mbar);
      if (!mbar_wait(&mbar, 0)) atomicAdd(err, 1);
      cyc[blockIdx.x] = clock64() - t0;
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int ROT, int NN, bool TS = false>
void run_rate3(long long* cyc, int* err) {
  *err = 0;
  k_rate3<ROT, NN, TS><<<148, 128>>>(8192, cyc, err);
  cudaDeviceSynchronize();
  printf("rate3 (warp-issued, elect.sync): %s M=128 N=%d K=8 tf32, %d accumulators: %.2f cycles/MMA = %.0f MAC/cycle (timeouts %d)\n",
         TS ? "TS" : "SS", NN, ROT, (double)cyc[0] / 8192, 128.0 * NN * 8 * 8192 / cyc[0], *err);
}

template <int ROT, int NN, bool TS>
void run_rate2(long long* cyc, int* err) {
  *err = 0;
  k_rate2<ROT, NN, TS><<<148, 128>>>(8192, cyc, err);
  cudaDeviceSynchronize();
  printf("rate2: %s M=128 N=%d K=8 tf32, %d accumulators: %.2f cycles/MMA = %.0f MAC/cycle (timeouts %d)\n",
         TS ? "TS" : "SS", NN, ROT, (double)cyc[0] / 8192, 128.0 * NN * 8 * 8192 / cyc[0], *err);
}

int main() {
  float *A, *B, *D;
  int* err;
  long long* cyc;
  cudaMallocManaged(&A, sizeof(float) * M * KS);
  cudaMallocManaged(&B, sizeof(float) * N * KS);
  cudaMallocManaged(&D, sizeof(float) * M * N);
  cudaMallocManaged(&err, sizeof(int));
  cudaMallocManaged(&cyc, sizeof(long long) * 148);
  srand(1);
  for (int i = 0; i < M * KS; ++i) A[i] = (float)rand() / RAND_MAX * 2.f - 1.f;
  for (int i = 0; i < N * KS; ++i) B[i] = ((float)rand() / RAND_MAX * 2.f - 1.f) * 0.01f;
  const char* names[3] = {"SS 1xTF32", "SS 3xTF32", "TS 3xTF32"};
  for (int mode = 0; mode < 3; ++mode)
    for (int swap = 0; swap < 2; ++swap) {
      *err = 0;
      for (int i = 0; i < M * N; ++i) D[i] = NAN;
      k_check<<<1, 128>>>(A, B, D, mode, swap, err);
      const cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("%s swap=%d: CUDA error %s\n", names[mode], swap, cudaGetErrorString(e));
        return 1;
      }
      double maxerr = 0, maxref = 0;
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
          double s = 0;
          for (int k = 0; k < KS; ++k) s += (double)A[m * KS + k] * (double)B[n * KS + k];
          maxref = fmax(maxref, fabs(s));
          maxerr = fmax(maxerr, fabs(s - (double)D[m * N + n]));
        }
      printf("%s swap=%d: timeout=%d max|D-ref|/max|ref| = %.3e\n", names[mode], swap, *err, maxerr / maxref);
    }
  void (*kr[5])(int, long long*, int*) = {k_rate<1>, k_rate<2>, k_rate<4>, k_rate<8>, k_rate<16>};
  for (int ri = 0; ri < 5; ++ri)
    for (int iters : {1024, 8192}) {
      const int rot = 1 << ri;
      *err = 0;
      kr[ri]<<<148, 128>>>(iters, cyc, err);
      cudaDeviceSynchronize();
      printf("rate: %d MMAs (128x16x8 tf32) over %d accumulators: %.2f cycles/MMA (timeouts %d)\n", iters, rot,
             (double)cyc[0] / iters, *err);
    }
  run_rate2<4, 16, false>(cyc, err);
  run_rate2<4, 16, true>(cyc, err);
  run_rate2<1, 16, true>(cyc, err);
  run_rate2<4, 32, false>(cyc, err);
  run_rate2<4, 32, true>(cyc, err);
  run_rate2<4, 64, false>(cyc, err);
  run_rate2<4, 64, true>(cyc, err);
  run_rate2<2, 128, false>(cyc, err);
  run_rate2<2, 128, true>(cyc, err);
  run_rate3<4, 16>(cyc, err);
  run_rate3<4, 32>(cyc, err);
  run_rate3<4, 64>(cyc, err);
  run_rate3<4, 16, true>(cyc, err);
  run_rate3<4, 32, true>(cyc, err);
  run_rate3<4, 64, true>(cyc, err);
  run_rate3<4, 128, true>(cyc, err);
  return 0;
}
