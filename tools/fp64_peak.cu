// FP64 peak probes for B200 (sm_100a): DMMA (mma.sync f64, m8n8k4 and m16n8k16) and DFMA.
// Each kernel runs a register-only dependent-free loop on every SM; the host divides
// algorithmic flops by CUDA-event time. Used once to record the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = 0.0; c[t][1] = 0.0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0; 
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int t = 0; t < 8; ++t) a[t] = threadIdx.x * 1e-3 + t;
#pragma unroll
  for (int t = 0; t < 4; ++t) b[t] = 1.0 + t * 1e-6;
  double c[4][4];
#pragma unroll
  for (int t = 0; t < 4; ++t) for (int u = 0; u < 4; ++u) c[t][u] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  if (s == 12345.678) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double x[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) x[t] = threadIdx.x * 1e-9 + t;
  const double m = 0.999999, a = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 16; ++t) x[t] = fma(x[t], m, a);
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 16; ++t) s += x[t];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
float timeit(K kern, int blocks, int threads, int iters, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters);  // warm
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  double* out; cudaMalloc(&out, 8);
  int iters = 20000;
  for (int warps : {4, 8, 16}) {
    int blocks = sms * 2, threads = warps * 32;
    float ms = timeit(dmma_m8n8k4, blocks, threads, iters, out);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)blocks * warps;
    printf("{\"probe\":\"dmma_m8n8k4\",\"warps_per_cta\":%d,\"ctas\":%d,\"tflops\":%.2f}\n", warps, blocks, flops / ms / 1e9);
    ms = timeit(dmma_m16n8k16, blocks, threads, iters / 4, out);
    flops = 2.0 * 16 * 8 * 16 * 4.0 * (iters / 4) * (double)blocks * warps;
    printf("{\"probe\":\"dmma_m16n8k16\",\"warps_per_cta\":%d,\"ctas\":%d,\"tflops\":%.2f}\n", warps, blocks, flops / ms / 1e9);
    ms = timeit(dfma_loop, blocks, threads, iters, out);
    flops = 2.0 * 16.0 * iters * (double)blocks * threads;
    printf("{\"probe\":\"dfma\",\"warps_per_cta\":%d,\"ctas\":%d,\"tflops\":%.2f}\n", warps, blocks, flops / ms / 1e9);
  }
  cudaError_t e = cudaGetLastError();
  printf("{\"probe\":\"status\",\"err\":\"%s\",\"sms\":%d}\n", cudaGetErrorString(e), sms);
  return 0;
}
