// Microbenchmark: FP32 FMA-pipe throughput on sm_100a for the leaf-update shape
// S[i] = fma(D[i % 16], T, S[i]) (scalar FFMA) versus the packed f32x2 form
// (__ffma2_rn).  Used once to pick the inner-loop instruction for the Chen kernels.
#include <cstdio>
#include <string>
#include <cuda_runtime.h>

template <int NACC>
__global__ void k_ffma(const float* in, float* out, int iters) {
  float S[NACC], D[16];
  float T = in[threadIdx.x & 7];
#pragma unroll
  for (int i = 0; i < 16; ++i) D[i] = in[(i + threadIdx.x) & 15] * 1e-3f;
#pragma unroll
  for (int i = 0; i < NACC; ++i) S[i] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) S[i] = fmaf(D[i & 15], T, S[i]);
    T = T * 0.999f;  // one extra dependent op per iteration
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += S[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void k_ffma2(const float* in, float* out, int iters) {
  float2 S[NACC / 2], D[8];
  float t = in[threadIdx.x & 7];
  float2 T = make_float2(t, t);
#pragma unroll
  for (int i = 0; i < 8; ++i) D[i] = make_float2(in[(2 * i + threadIdx.x) & 15] * 1e-3f, in[(2 * i + 1 + threadIdx.x) & 15] * 1e-3f);
#pragma unroll
  for (int i = 0; i < NACC / 2; ++i) S[i] = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC / 2; ++i) S[i] = __ffma2_rn(D[i & 7], T, S[i]);
    T.x = T.x * 0.999f; T.y = T.x;
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NACC / 2; ++i) s += S[i].x + S[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(const double* in, double* out, int iters) {
  double S[32], D[16];
  double T = in[threadIdx.x & 7];
#pragma unroll
  for (int i = 0; i < 16; ++i) D[i] = in[(i + threadIdx.x) & 15] * 1e-3;
#pragma unroll
  for (int i = 0; i < 32; ++i) S[i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) S[i] = fma(D[i & 15], T, S[i]);
    T = T * 0.999;
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += S[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main(int argc, char** argv) {
  const bool peak_only = argc > 1 && std::string(argv[1]) == "--peak";
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *in, *out; double *din, *dout;
  cudaMalloc(&in, 64 * 4); cudaMalloc(&out, 1 << 26); cudaMalloc(&din, 64 * 8); cudaMalloc(&dout, 1 << 27);
  float h[64]; for (int i = 0; i < 64; ++i) h[i] = 1.0f + i * 0.01f;
  double hd[64]; for (int i = 0; i < 64; ++i) hd[i] = 1.0 + i * 0.01;
  cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice); cudaMemcpy(din, hd, sizeof hd, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096;
  if (peak_only) {  // best of 5 at 256 threads x 8 CTAs/SM: {"ffma_tflops": .., "dfma_tflops": ..}
    double best[2] = {0, 0};
    const int grid = sms * 8;
    for (int rep = 0; rep < 6; ++rep)
      for (int v = 0; v < 2; ++v) {
        cudaEventRecord(a);
        if (v == 0) k_ffma<64><<<grid, 256>>>(in, out, iters);
        else k_dfma<<<grid, 256>>>(din, dout, iters);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double tf = 2.0 * grid * 256.0 * iters * (v ? 32 : 64) / ms / 1e9;
        if (rep > 0 && tf > best[v]) best[v] = tf;
      }
    printf("{\"ffma_tflops\": %.3f, \"dfma_tflops\": %.3f, \"sms\": %d, \"err\": \"%s\"}\n", best[0], best[1], sms,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
  }
  for (int threads : {128, 256, 512}) {
    for (int per_sm : {1, 2, 4}) {
      int grid = sms * per_sm * (512 / threads);
      for (int variant = 0; variant < 3; ++variant) {
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(a);
          if (variant == 0) k_ffma<64><<<grid, threads>>>(in, out, iters);
          else if (variant == 1) k_ffma2<64><<<grid, threads>>>(in, out, iters);
          else k_dfma<<<grid, threads>>>(din, dout, iters);
          cudaEventRecord(b); cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b);
          double nfma = (double)grid * threads * iters * (variant == 2 ? 32 : 64);
          if (rep == 1)
            printf("%s threads=%d grid=%d  %.3f ms  %.2f TFLOP/s (fma=2 flop)\n",
                   variant == 0 ? "FFMA " : variant == 1 ? "FFMA2" : "DFMA ", threads, grid, ms, 2 * nfma / ms / 1e9);
        }
      }
    }
  }
  printf("sms=%d clock_khz=%d err=%s\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
