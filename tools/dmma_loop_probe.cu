// Mainloop probes for the FP64 DMMA GEMM kernels (what limits gram_kernel at ~74% pipe?):
//   mode 0: fragments from shared memory every k-step, no barriers (pure LDS + DMMA)
//   mode 1: + __syncthreads() every stage of 4 k-steps
//   mode 2: + a cp.async ring refilling each stage from global memory (the real loop)
// 64x64 CTA tile, 4 warps of WM x WN DMMA tiles (4x4 = 32x32 warp tile), BK = 16.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_loop_probe tools/dmma_loop_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int BK = 16, LD = 68;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(void* s, const void* g) {
  unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
}

template <int MODE, int WM, int WN, int ST = 4, int MINB = 3>
__global__ void __launch_bounds__(128, MINB) loop(const double* __restrict__ g, double* out, int stages) {
  extern __shared__ double sm[];
  double* Xs = sm;
  double* Ys = sm + ST * BK * LD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 2 * ST * BK * LD; e += 128) sm[e] = 1e-3 * (e % 97);
  __syncthreads();
  const int wm = warp >> 1, wn = warp & 1;
  const int fr = lane & 3, fc = lane >> 2;
  double acc[WM][WN][2];
#pragma unroll
  for (int a = 0; a < WM; ++a)
#pragma unroll
    for (int b = 0; b < WN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const double* gsrc = g + (int64_t)blockIdx.x * 1024;
  for (int s = 0; s < stages; ++s) {
    const int st = s % ST;
    if (MODE >= 2) {
      asm volatile("cp.async.wait_group %0;\n" ::"n"(ST - 2));
    }
    if (MODE >= 1) __syncthreads();
    if (MODE == 2) {  // refill stage (s+3)%ST: 16 x 64 doubles for each operand
      const int sn = (s + ST - 1) % ST;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = tid + 128 * i, r = e >> 5, c = (e & 31) * 2;
        cp16(Xs + sn * BK * LD + r * LD + c, gsrc + ((s * 16 + r) & 1023) * 0 + c);
        cp16(Ys + sn * BK * LD + r * LD + c, gsrc + 512 + c);
      }
      asm volatile("cp.async.commit_group;\n" ::);
    }
    if (MODE == 3) {  // the Gram's real stream: rows of a tall row-major matrix (ld 524),
      // CTA = (tile, chunk): X cols tile*64 mod 512, Y cols (tile*7)*64 mod 512, chunk rows
      const int sn = (s + ST - 1) % ST;
      const int tile = blockIdx.x % 81, chunk = blockIdx.x / 81;
      const int xc0 = (tile % 9) * 56, yc0 = (tile / 9) * 56;
      const int64_t row0 = (int64_t)chunk * stages * 16 + (int64_t)(s + ST - 1) * 16;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = tid + 128 * i, r = e >> 5, c = (e & 31) * 2;
        const int64_t row = (row0 + r) % 110592;
        cp16(Xs + sn * BK * LD + r * LD + c, g + row * 524 + xc0 + c);
        cp16(Ys + sn * BK * LD + r * LD + c, g + row * 524 + yc0 + c);
      }
      asm volatile("cp.async.commit_group;\n" ::);
    }
    const double* xs = Xs + st * BK * LD + fr * LD + wm * 8 * WM + fc;
    const double* ys = Ys + st * BK * LD + fr * LD + wn * 8 * WN + fc;
#pragma unroll
    for (int kq = 0; kq < BK / 4; ++kq) {
      double af[WM], bf[WN];
#pragma unroll
      for (int a = 0; a < WM; ++a) af[a] = xs[kq * 4 * LD + a * 8];
#pragma unroll
      for (int b = 0; b < WN; ++b) bf[b] = ys[kq * 4 * LD + b * 8];
#pragma unroll
      for (int a = 0; a < WM; ++a)
#pragma unroll
        for (int b = 0; b < WN; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  double t = 0.0;
#pragma unroll
  for (int a = 0; a < WM; ++a)
#pragma unroll
    for (int b = 0; b < WN; ++b) t += acc[a][b][0] + acc[a][b][1];
  if (t == 1234.5) out[0] = t;
}

// mode 4: the same HBM stream as mode 3, fed by bulk async copies (one 512 B row per
// cp.async.bulk, completing on a per-stage mbarrier) from a dedicated producer warp; the four
// MMA warps wait on "full" barriers and release stages through "empty" barriers -- no
// cp.async/LDGSTS issue slots and no __syncthreads in the MMA warps.
__device__ __forceinline__ unsigned sa32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(bar),
      "r"(parity));
}
template <int WM, int WN, int ST, int MINB>
__global__ void __launch_bounds__(160, MINB) loop_bulk(const double* __restrict__ g, double* out, int stages) {
  extern __shared__ __align__(128) double sm[];
  double* Xs = sm;
  double* Ys = sm + ST * BK * LD;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + 2 * ST * BK * LD);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < ST; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa32(bars + i)), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa32(bars + ST + i)), "r"(4));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::);
  }
  __syncthreads();
  const int tile = blockIdx.x % 81, chunk = blockIdx.x / 81;
  const int xc0 = (tile % 9) * 56, yc0 = (tile / 9) * 56;
  if (warp == 4) {  // producer
    for (int s = 0; s < stages; ++s) {
      const int st = s % ST;
      if (s >= ST) mb_wait(sa32(bars + ST + st), ((s / ST) - 1) & 1);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa32(bars + st)),
                     "r"(2 * BK * 64 * 8));
      __syncwarp();
      const int r = lane & 15;
      const int64_t row = ((int64_t)chunk * stages * 16 + (int64_t)s * 16 + r) % 110592;
      const double* src = g + row * 524 + (lane < 16 ? xc0 : yc0);
      double* dst = (lane < 16 ? Xs : Ys) + st * BK * LD + r * LD;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa32(dst)),
                   "l"(src), "r"(512), "r"(sa32(bars + st))
                   : "memory");
    }
    return;
  }
  const int wm = warp >> 1, wn = warp & 1;
  const int fr = lane & 3, fc = lane >> 2;
  double acc[WM][WN][2];
#pragma unroll
  for (int a = 0; a < WM; ++a)
#pragma unroll
    for (int b = 0; b < WN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int s = 0; s < stages; ++s) {
    const int st = s % ST;
    mb_wait(sa32(bars + st), (s / ST) & 1);
    const double* xs = Xs + st * BK * LD + fr * LD + wm * 8 * WM + fc;
    const double* ys = Ys + st * BK * LD + fr * LD + wn * 8 * WN + fc;
#pragma unroll
    for (int kq = 0; kq < BK / 4; ++kq) {
      double af[WM], bf[WN];
#pragma unroll
      for (int a = 0; a < WM; ++a) af[a] = xs[kq * 4 * LD + a * 8];
#pragma unroll
      for (int b = 0; b < WN; ++b) bf[b] = ys[kq * 4 * LD + b * 8];
#pragma unroll
      for (int a = 0; a < WM; ++a)
#pragma unroll
        for (int b = 0; b < WN; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa32(bars + ST + st)) : "memory");
  }
  double t = 0.0;
#pragma unroll
  for (int a = 0; a < WM; ++a)
#pragma unroll
    for (int b = 0; b < WN; ++b) t += acc[a][b][0] + acc[a][b][1];
  if (t == 1234.5) out[0] = t;
}

// mode 5: bulk copies issued by warp 0 of the four MMA warps (no producer warp): at stage s
// warp 0 waits until every warp released stage s-1 and refills it with stage s+ST-1.
template <int WM, int WN, int ST, int MINB>
__global__ void __launch_bounds__(128, MINB) loop_bulk_inl(const double* __restrict__ g, double* out, int stages) {
  extern __shared__ __align__(128) double sm[];
  double* Xs = sm;
  double* Ys = sm + ST * BK * LD;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + 2 * ST * BK * LD);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < ST; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa32(bars + i)), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa32(bars + ST + i)), "r"(4));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::);
  }
  __syncthreads();
  const int tile = blockIdx.x % 81, chunk = blockIdx.x / 81;
  const int xc0 = (tile % 9) * 56, yc0 = (tile / 9) * 56;
  auto produce = [&](int s) {
    const int st = s % ST;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa32(bars + st)),
                   "r"(2 * BK * 64 * 8));
    __syncwarp();
    const int r = lane & 15;
    const int64_t row = ((int64_t)chunk * stages * 16 + (int64_t)s * 16 + r) % 110592;
    const double* src = g + row * 524 + (lane < 16 ? xc0 : yc0);
    double* dst = (lane < 16 ? Xs : Ys) + st * BK * LD + r * LD;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa32(dst)),
                 "l"(src), "r"(512), "r"(sa32(bars + st))
                 : "memory");
  };
  if (warp == 0)
    for (int s = 0; s < ST - 1 && s < stages; ++s) produce(s);
  const int wm = warp >> 1, wn = warp & 1;
  const int fr = lane & 3, fc = lane >> 2;
  double acc[WM][WN][2];
#pragma unroll
  for (int a = 0; a < WM; ++a)
#pragma unroll
    for (int b = 0; b < WN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int s = 0; s < stages; ++s) {
    const int st = s % ST;
    if (warp == 0 && s + ST - 1 < stages) {
      const int sn = s + ST - 1;  // refills stage (s-1)%ST: wait until all warps released it
      if (sn >= ST) mb_wait(sa32(bars + ST + sn % ST), ((sn / ST) - 1) & 1);
      produce(sn);
    }
    mb_wait(sa32(bars + st), (s / ST) & 1);
    const double* xs = Xs + st * BK * LD + fr * LD + wm * 8 * WM + fc;
    const double* ys = Ys + st * BK * LD + fr * LD + wn * 8 * WN + fc;
#pragma unroll
    for (int kq = 0; kq < BK / 4; ++kq) {
      double af[WM], bf[WN];
#pragma unroll
      for (int a = 0; a < WM; ++a) af[a] = xs[kq * 4 * LD + a * 8];
#pragma unroll
      for (int b = 0; b < WN; ++b) bf[b] = ys[kq * 4 * LD + b * 8];
#pragma unroll
      for (int a = 0; a < WM; ++a)
#pragma unroll
        for (int b = 0; b < WN; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa32(bars + ST + st)) : "memory");
  }
  double t = 0.0;
#pragma unroll
  for (int a = 0; a < WM; ++a)
#pragma unroll
    for (int b = 0; b < WN; ++b) t += acc[a][b][0] + acc[a][b][1];
  if (t == 1234.5) out[0] = t;
}

template <int ST, int MINB>
void run_bulk_inl(const char* name, int blocks, const double* g, double* out, int stages) {
  const int smem = 2 * ST * BK * LD * 8 + 2 * ST * 8;
  cudaFuncSetAttribute(loop_bulk_inl<4, 4, ST, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  loop_bulk_inl<4, 4, ST, MINB><<<blocks, 128, smem>>>(g, out, stages);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    loop_bulk_inl<4, 4, ST, MINB><<<blocks, 128, smem>>>(g, out, stages);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 64 * 64 * BK * (double)stages * blocks;
  printf("{\"probe\":\"%s\",\"ctas\":%d,\"tflops\":%.2f,\"err\":\"%s\"}\n", name, blocks, flops / best / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

template <int ST, int MINB>
void run_bulk(const char* name, int blocks, const double* g, double* out, int stages) {
  const int smem = 2 * ST * BK * LD * 8 + 2 * ST * 8;
  cudaFuncSetAttribute(loop_bulk<4, 4, ST, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  loop_bulk<4, 4, ST, MINB><<<blocks, 160, smem>>>(g, out, stages);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    loop_bulk<4, 4, ST, MINB><<<blocks, 160, smem>>>(g, out, stages);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 64 * 64 * BK * (double)stages * blocks;
  printf("{\"probe\":\"%s\",\"ctas\":%d,\"tflops\":%.2f,\"err\":\"%s\"}\n", name, blocks, flops / best / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

template <int MODE, int WM, int WN, int ST = 4, int MINB = 3>
void run(const char* name, int blocks, const double* g, double* out, int stages) {
  const int smem = 2 * ST * BK * LD * 8;
  cudaFuncSetAttribute(loop<MODE, WM, WN, ST, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  loop<MODE, WM, WN, ST, MINB><<<blocks, 128, smem>>>(g, out, stages);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    loop<MODE, WM, WN, ST, MINB><<<blocks, 128, smem>>>(g, out, stages);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 64 * 64 * BK * (double)stages * blocks;
  printf("{\"probe\":\"%s\",\"ctas\":%d,\"tflops\":%.2f,\"err\":\"%s\"}\n", name, blocks, flops / best / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  double *g, *out;
  const size_t gbytes = sizeof(double) * 110592 * 524;
  cudaMalloc(&g, gbytes);
  cudaMemset(g, 0, gbytes);
  cudaMalloc(&out, 8);
  const int stages = 20000;
  for (int per : {2, 3}) {
    run<0, 4, 4>(per == 2 ? "lds_only_2cta" : "lds_only_3cta", sms * per, g, out, stages);
    run<1, 4, 4>(per == 2 ? "lds_barrier_2cta" : "lds_barrier_3cta", sms * per, g, out, stages);
    run<2, 4, 4>(per == 2 ? "cpasync_ring_2cta" : "cpasync_ring_3cta", sms * per, g, out, stages);
  }
  // the config-2 Gram's stream: 81 tiles x 16 chunks of 432 stages, 3 CTAs/SM
  run<3, 4, 4>("hbm_stream_gram_shape", 81 * 16, g, out, 432);
  run<3, 4, 4>("hbm_stream_gram_shape_8waves", 81 * 44, g, out, 157);
  run<3, 4, 4, 6, 2>("hbm_stream_st6_2cta", 81 * 44, g, out, 157);
  run<3, 4, 4, 3, 3>("hbm_stream_st3_3cta", 81 * 44, g, out, 157);
  run<3, 4, 4, 8, 1>("hbm_stream_st8_1cta", 81 * 44, g, out, 157);
  run<3, 4, 4, 5, 2>("hbm_stream_st5_2cta", 81 * 44, g, out, 157);
  run<3, 4, 4, 3, 4>("hbm_stream_st3_4cta", 81 * 44, g, out, 157);
  run<1, 4, 4, 3, 4>("lds_barrier_st3_4cta", sms * 4, g, out, 20000);
  run_bulk<4, 3>("bulk_st4_3cta", 81 * 44, g, out, 157);
  run_bulk<6, 2>("bulk_st6_2cta", 81 * 44, g, out, 157);
  run_bulk<3, 4>("bulk_st3_4cta", 81 * 44, g, out, 157);
  run_bulk<8, 2>("bulk_st8_2cta", 81 * 44, g, out, 157);
  run_bulk<5, 3>("bulk_st5_3cta", 81 * 44, g, out, 157);
  run_bulk_inl<4, 3>("bulk_inline_st4_3cta", 81 * 44, g, out, 157);
  run_bulk_inl<5, 3>("bulk_inline_st5_3cta", 81 * 44, g, out, 157);
  run_bulk_inl<3, 4>("bulk_inline_st3_4cta", 81 * 44, g, out, 157);
  run_bulk_inl<4, 4>("bulk_inline_st4_4cta", 81 * 44, g, out, 157);
  return 0;
}
