// Probe for the tensor-core leaf term of the truncated backward:
// tb[w, j] = sum_z Lambda[w, z] * dX_j[z] as tcgen05.mma kind::f16, M = 128
// words, N = 16 steps, K = 16 letters (one instruction), A = Lambda and
// B = dX from shared memory (SS), canonical K-major no-swizzle layout,
// accumulator in TMEM.  fp32 accuracy from a scaled 3-pass fp16 split:
// each A row and each B column is scaled by a power of two into
// [2^13, 2^14), split x = hi + lo (both fp16, round to nearest), and
// D = A_hi B_hi + A_lo B_hi + A_hi B_lo; the scales come off exactly.
//
// Checks against an fp64 host product (random rows spanning 2^-20..2^20):
//   1. the 3-pass result (relative error vs max |D| per row);
//   2. 1-pass fp16 for comparison;
// then times back-to-back SS MMAs (M=128, K=16) at N = 16 / 32 / 64.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tc_f16 tools/ubench_tc_f16.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

constexpr int M = 128, N = 16, K = 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);
}

__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);  // D f32, A/B f16, K-major
}

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* mbar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(mbar))
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

// K-major no swizzle, f16: core matrix = 8 rows x 8 halves (128 B), [row group][k group]
__device__ __forceinline__ int kmaj(int row, int k) { return ((row >> 3) * 2 + (k >> 3)) * 64 + (row & 7) * 8 + (k & 7); }

__device__ __forceinline__ float pow2_scale(float amax) {  // 2^e with amax * 2^e in [2^13, 2^14)
  if (!(amax > 0.f)) return 1.f;
  int e;
  frexpf(amax, &e);  // amax = f * 2^e, f in [0.5, 1)
  return ldexpf(1.f, 14 - e);
}

// mode 0: 1 pass, 1: 3 passes.  A[m][k] fp32, B[n][k] fp32 (B^T).
__global__ void k_check(const float* A, const float* B, float* D, int mode, int* err) {
  __shared__ __align__(1024) __half As[2][M * K];
  __shared__ __align__(1024) __half Bs[2][N * K];
  __shared__ float sa[M], sb[N];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid < M) {
    float mx = 0.f;
    for (int k = 0; k < K; ++k) mx = fmaxf(mx, fabsf(A[tid * K + k]));
    const float s = pow2_scale(mx);
    sa[tid] = 1.f / s;
    for (int k = 0; k < K; ++k) {
      const float x = A[tid * K + k] * s;
      const __half h = __float2half_rn(x);
      As[0][kmaj(tid, k)] = h;
      As[1][kmaj(tid, k)] = __float2half_rn(x - __half2float(h));
    }
  }
  if (tid < N) {
    float mx = 0.f;
    for (int k = 0; k < K; ++k) mx = fmaxf(mx, fabsf(B[tid * K + k]));
    const float s = pow2_scale(mx);
    sb[tid] = 1.f / s;
    for (int k = 0; k < K; ++k) {
      const float x = B[tid * K + k] * s;
      const __half h = __float2half_rn(x);
      Bs[0][kmaj(tid, k)] = h;
      Bs[1][kmaj(tid, k)] = __float2half_rn(x - __half2float(h));
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
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
  const uint32_t td = tmem_base;
  if (warp == 0) {
    const uint32_t id = idesc_f16(M, N);
    const int passes = mode == 0 ? 1 : 3;
    for (int p = 0; p < passes; ++p) {
      const int ah = (p == 1) ? 1 : 0, bh = (p == 2) ? 1 : 0;  // hi*hi, lo*hi, hi*lo
      mma_ss(td, smem_desc(smem_u32(As[ah]), 128, 256), smem_desc(smem_u32(Bs[bh]), 128, 256), id, p > 0);
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
      : "r"(td + ((uint32_t)(warp & 3) * 32 << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int n = 0; n < N; ++n) D[tid * N + n] = __uint_as_float(r[n]) * sa[tid] * sb[n];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(td));
}

// back-to-back SS MMAs at width n: cycles per instruction
template <int NN>
__global__ void k_rate(int iters, long long* cycles, int* err) {
  __shared__ __align__(1024) __half As[M * K];
  __shared__ __align__(1024) __half Bs[256 * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) As[i] = __float2half(0.001f * (i % 7));
  for (int i = tid; i < 256 * K; i += blockDim.x) Bs[i] = __float2half(0.001f * (i % 5));
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
  const uint32_t td = tmem_base;
  if (warp == 0) {
    const uint32_t id = idesc_f16(M, NN);
    const uint64_t da = smem_desc(smem_u32(As), 128, 256), db = smem_desc(smem_u32(Bs), 128, 256);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) mma_ss(td + (i & 1) * 128, da, db, id, 1u);
    mma_commit(&mbar);
    if (!mbar_wait(&mbar, 0)) atomicAdd(err, 1);
    const long long t1 = clock64();
    if (tid == 0) *cycles = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(td));
}

int main() {
  float *A, *B, *D;
  int* err;
  long long* cyc;
  cudaMallocManaged(&A, M * K * 4);
  cudaMallocManaged(&B, N * K * 4);
  cudaMallocManaged(&D, M * N * 4);
  cudaMallocManaged(&err, 4);
  cudaMallocManaged(&cyc, 8);
  srand(7);
  for (int m = 0; m < M; ++m) {
    const double rs = std::ldexp(1.0, (m % 41) - 20);  // rows spanning 2^-20 .. 2^20
    for (int k = 0; k < K; ++k) A[m * K + k] = (float)(rs * (2.0 * rand() / RAND_MAX - 1.0));
  }
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) B[n * K + k] = (float)(0.05 * (2.0 * rand() / RAND_MAX - 1.0) * (n == 3 ? 1e-6 : 1.0));
  for (int mode = 0; mode < 2; ++mode) {
    *err = 0;
    k_check<<<1, 128>>>(A, B, D, mode, err);
    cudaError_t e = cudaDeviceSynchronize();
    double worst = 0;
    for (int m = 0; m < M; ++m) {
      double ref[N], mx = 0;
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
        ref[n] = s;
        mx = fmax(mx, fabs(s));
      }
      // error relative to the row's magnitude (A row norm x B column norm)
      double an = 0;
      for (int k = 0; k < K; ++k) an = fmax(an, fabs((double)A[m * K + k]));
      for (int n = 0; n < N; ++n) {
        double bn = 0;
        for (int k = 0; k < K; ++k) bn = fmax(bn, fabs((double)B[n * K + k]));
        worst = fmax(worst, fabs(D[m * N + n] - ref[n]) / (an * bn * K));
      }
    }
    printf("{\"probe\": \"f16 SS M=128 N=16 K=16\", \"passes\": %d, \"cuda\": \"%s\", \"timeouts\": %d, "
           "\"max_err_rel_to_|a||b|K\": %.3e}\n",
           mode ? 3 : 1, cudaGetErrorString(e), *err, worst);
  }
  auto rate = [&](auto kern, int nn) {
    *err = 0;
    kern<<<1, 128>>>(4096, cyc, err);
    cudaError_t e = cudaDeviceSynchronize();
    printf("{\"probe\": \"f16 SS back-to-back\", \"N\": %d, \"cycles_per_mma\": %.1f, \"cuda\": \"%s\", \"timeouts\": %d}\n",
           nn, (double)*cyc / 4096, cudaGetErrorString(e), *err);
  };
  rate(k_rate<16>, 16);
  rate(k_rate<32>, 32);
  rate(k_rate<64>, 64);
  rate(k_rate<128>, 128);
  return 0;
}
