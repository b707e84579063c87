// H2D bandwidth from pinned memory: one 1-D copy, row-chunk 2-D copies (the
// upload_and_sketch pattern: nr rows x n columns of a column-major matrix),
// and the same 2-D chunks split over two copy streams.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)
int main() {
    const size_t m = 50000, n = 20000;  // 8 GB
    double *h, *d;
    CK(cudaMallocHost(&h, m * n * 8));
    CK(cudaMalloc(&d, m * n * 8));
    for (size_t i = 0; i < m * n; i += 4096) h[i] = 1.0;
    cudaStream_t s[2];
    CK(cudaStreamCreate(&s[0]));
    CK(cudaStreamCreate(&s[1]));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0, s[0]);
        CK(cudaMemcpyAsync(d, h, m * n * 8, cudaMemcpyHostToDevice, s[0]));
        cudaEventRecord(e1, s[0]);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("1-D: %.1f GB/s\n", m * n * 8 / ms / 1e6);
        for (int streams = 1; streams <= 2; ++streams) {
            const size_t nr = 3200;
            CK(cudaDeviceSynchronize());
            cudaEventRecord(e0, s[0]);
            cudaStreamWaitEvent(s[1], e0, 0);
            int c = 0;
            for (size_t r0 = 0; r0 < m; r0 += nr, ++c) {
                const size_t rows = r0 + nr <= m ? nr : m - r0;
                CK(cudaMemcpy2DAsync(d + r0, m * 8, h + r0, m * 8, rows * 8, n, cudaMemcpyHostToDevice, s[c % streams]));
            }
            cudaEvent_t e2;
            cudaEventCreate(&e2);
            cudaEventRecord(e2, s[1]);
            cudaStreamWaitEvent(s[0], e2, 0);
            cudaEventRecord(e1, s[0]);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("2-D row chunks, %d stream(s): %.1f GB/s\n", streams, m * n * 8 / ms / 1e6);
        }
    }
    return 0;
}
