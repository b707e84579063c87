// Dependent-chain latency of FP64 ops on one warp (cycles per op):
// DFMA, DADD, DMUL, sqrt(), 1/x, x/y, rsqrt approx, __shfl_sync of a double.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_latency fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, double x0, long long* cyc, int iters) {
    double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (OP == 0) x = fma(x, y, 1e-30);
        if (OP == 1) x = x + y * 0.0 + 1e-300;  // dadd (the mul folds)
        if (OP == 2) x = sqrt(x + 1.0) ;
        if (OP == 3) x = 1.0 / (x + 1.0);
        if (OP == 4) x = (x + 2.0) / y;
        if (OP == 5) x = rsqrt(x + 1.0);
        if (OP == 6) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-300;
        if (OP == 7) x = __drcp_rn(x + 1.0);
        if (OP == 8) {  // MUFU.RSQ64H (the Jacobi rotation's seed) alone
            double y;
            asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x + 1.0));
            x = y;
        }
        if (OP == 9) {  // MUFU.RCP64H alone
            double y;
            asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x + 1.0));
            x = y;
        }
        if (OP == 10) x = __shfl_sync(0xffffffffu, x, 3) + 1e-300;  // broadcast shuffle
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * 8);
    cudaMallocManaged(&cyc, 8);
    const char* names[] = {"dfma", "dadd", "sqrt", "1/x", "x/y", "rsqrt", "shfl+dadd", "__drcp_rn",
                           "rsqrt.approx.f64 (+dadd)", "rcp.approx.f64 (+dadd)", "shfl.idx+dadd"};
    const int iters = 4096;
    for (int op = 0; op < 11; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            switch (op) {
                case 0: chain<0><<<1, 32>>>(out, 0.5, cyc, iters); break;
                case 1: chain<1><<<1, 32>>>(out, 0.5, cyc, iters); break;
                case 2: chain<2><<<1, 32>>>(out, 0.5, cyc, iters); break;
                case 3: chain<3><<<1, 32>>>(out, 0.5, cyc, iters); break;
                case 4: chain<4><<<1, 32>>>(out, 0.5, cyc, iters); break;
                case 5: chain<5><<<1, 32>>>(out, 0.5, cyc, iters); break;
                case 6: chain<6><<<1, 32>>>(out, 0.5, cyc, iters); break;
                case 7: chain<7><<<1, 32>>>(out, 0.5, cyc, iters); break;
                case 8: chain<8><<<1, 32>>>(out, 0.5, cyc, iters); break;
                case 9: chain<9><<<1, 32>>>(out, 0.5, cyc, iters); break;
                case 10: chain<10><<<1, 32>>>(out, 0.5, cyc, iters); break;
            }
            cudaDeviceSynchronize();
        }
        printf("{\"op\": \"%s\", \"cycles_per_op\": %.1f}\n", names[op], double(*cyc) / iters);
    }
    return 0;
}
