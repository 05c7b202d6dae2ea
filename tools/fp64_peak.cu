// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) and DFMA.
// Used to establish the FP64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dmma_m16n8k4(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-9, a1 = a0 * 0.5, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <typename K>
double run(K kernel, int blocks, int threads, int iters, double flop_per_iter_per_warp_or_thread, bool per_warp) {
  double* out; cudaMalloc(&out, 4096 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kernel<<<blocks, threads>>>(out, iters);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double units = per_warp ? (double)blocks * threads / 32 : (double)blocks * threads;
  double flops = units * iters * flop_per_iter_per_warp_or_thread;
  cudaFree(out);
  return flops / (best * 1e-3) / 1e12;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  const int iters = 20000;
  for (int tpb : {128, 256, 512}) {
    double t1 = run(dmma_m8n8k4<8>, sms * 4, tpb, iters, 8 * 2.0 * 8 * 8 * 4, true);
    double t2 = run(dmma_m16n8k4<8>, sms * 4, tpb, iters, 8 * 2.0 * 16 * 8 * 4, true);
    double t3 = run(dfma<8>, sms * 4, tpb, iters, 8 * 2.0, false);
    printf(", \"tpb%d\": {\"dmma_m8n8k4_tflops\": %.2f, \"dmma_m16n8k4_tflops\": %.2f, \"dfma_tflops\": %.2f}", tpb, t1, t2, t3);
  }
  printf("}\n");
  return 0;
}
