// FP64 peak microbenchmark for B200 (sm_100a): DFMA (SIMT) and DMMA (mma.sync .f64).
// Writes one JSON line per variant. The measured DMMA number is the roofline
// denominator for every FP64 tensor fraction this repo reports.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dmma884_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c0[CHAINS], c1[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { c0[c] = 0; c1[c] = c; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0[c]), "+d"(c1[c]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += c0[c] + c1[c];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dmma16816_loop(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = threadIdx.x * 2e-3 + i;
  double c[CHAINS][4];
#pragma unroll
  for (int ch = 0; ch < CHAINS; ++ch)
#pragma unroll
    for (int i = 0; i < 4; ++i) c[ch][i] = ch + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int ch = 0; ch < CHAINS; ++ch)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[ch][0]), "+d"(c[ch][1]), "+d"(c[ch][2]), "+d"(c[ch][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int ch = 0; ch < CHAINS; ++ch) s += c[ch][0] + c[ch][1] + c[ch][2] + c[ch][3];
  if (s == 1234.5) out[threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 1024 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch, double fma_per_iter_per_thread_block) {
    for (int w = 0; w < 2; ++w) launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double tf = 2.0 * fma_per_iter_per_thread_block / (best * 1e-3) / 1e12;
    printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"tflops\": %.3f}\n", name, best, tf);
    cudaError_t err = cudaGetLastError(); if (err != cudaSuccess) printf("err %s\n", cudaGetErrorString(err));
  };
  const int iters = 20000;
  for (int bpsm : {1, 2, 4}) {
    for (int threads : {128, 256, 512}) {
      int blocks = sms * bpsm;
      char nm[128];
      snprintf(nm, sizeof nm, "dfma8 b/sm=%d thr=%d", bpsm, threads);
      run(nm, [&] { dfma_loop<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-7); },
          (double)blocks * threads * iters * 8);
      snprintf(nm, sizeof nm, "dmma884x4 b/sm=%d thr=%d", bpsm, threads);
      run(nm, [&] { dmma884_loop<4><<<blocks, threads>>>(out, iters); },
          (double)blocks * (threads / 32) * iters * 4 * 256);
      snprintf(nm, sizeof nm, "dmma884x8 b/sm=%d thr=%d", bpsm, threads);
      run(nm, [&] { dmma884_loop<8><<<blocks, threads>>>(out, iters); },
          (double)blocks * (threads / 32) * iters * 8 * 256);
      snprintf(nm, sizeof nm, "dmma16816x2 b/sm=%d thr=%d", bpsm, threads);
      run(nm, [&] { dmma16816_loop<2><<<blocks, threads>>>(out, iters / 4); },
          (double)blocks * (threads / 32) * (iters / 4) * 2 * 2048);
    }
  }
  printf("{\"sms\": %d, \"clock_khz\": %d, \"name\": \"%s\"}\n", sms, p.clockRate, p.name);
  return 0;
}
