// FP64 FMA throughput microbenchmark (the "alu" roofline denominator of the batched action,
// "the builder must measure it").
//
//   fp64_peak            the peak: 148 SMs x 8 blocks x 256 threads, 8 independent DFMA chains
//                        per thread; prints one JSON line {"fp64_fma_tflops": ...}
//   fp64_peak sweep      DFMA rate vs resident warps per SM and independent chains per thread
//                        (what a latency-bound FP64 kernel can reach), one JSON line per point,
//                        and the dependent-DFMA latency in cycles (one warp, one chain, clock64)
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

template <int C>
__global__ void k_fma(double* out, int iters, double a, double b) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

__global__ void k_latency(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x * 1e-3;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) x = fma(x, a, b);
  const long long t1 = clock64();
  if (x == 12345.678) out[0] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int C>
double run(int sms, int blocks_per_sm, int threads, int iters, double* out) {
  const int blocks = sms * blocks_per_sm;
  k_fma<C><<<blocks, threads>>>(out, 64, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_fma<C><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return 2.0 * C * (double)iters * blocks * threads / (best * 1e-3) / 1e12;
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  if (argc > 1 && std::strcmp(argv[1], "sweep") == 0) {
    long long* cyc;
    cudaMalloc(&cyc, 8);
    const int li = 1 << 16;
    k_latency<<<1, 32>>>(out, cyc, li, 0.999999, 1e-7);
    k_latency<<<1, 32>>>(out, cyc, li, 0.999999, 1e-7);
    long long hc = 0;
    cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"dfma_dependent_latency_cycles\": %.2f}\n", (double)hc / li);
    for (int wps : {4, 8, 16, 32, 64})
      for (int c : {1, 2, 4, 8, 16}) {
        // one block of wps warps per SM
        const int thr = 32 * wps > 1024 ? 1024 : 32 * wps, bps = 32 * wps / thr;
        double tf = 0;
        const int it = (1 << 16) / c;
        switch (c) {
          case 1: tf = run<1>(sms, bps, thr, it, out); break;
          case 2: tf = run<2>(sms, bps, thr, it, out); break;
          case 4: tf = run<4>(sms, bps, thr, it, out); break;
          case 8: tf = run<8>(sms, bps, thr, it, out); break;
          default: tf = run<16>(sms, bps, thr, it, out); break;
        }
        printf("{\"warps_per_sm\": %d, \"chains\": %d, \"fp64_fma_tflops\": %.3f}\n", wps, c, tf);
      }
    return 0;
  }
  const double tf = run<8>(sms, 8, 256, 1 << 14, out);
  printf("{\"fp64_fma_tflops\": %.3f, \"sms\": %d}\n", tf, sms);
  return 0;
}
