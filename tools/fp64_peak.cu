// fp64_peak.cu -- measured DFMA and DMMA (mma.sync m8n8k4 f64) throughput of this B200, the
// denominator check for the implicit Q~p roofline.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    if (s == 123.456) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters, double a, double b) {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-3 + i;
    double A = a + threadIdx.x * 1e-9, B = b;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(A), "d"(B));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 123.456) out[0] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
        for (int bps : {1, 2, 4}) {
            dim3 grid(sms * bps), block(256);
            cudaEventRecord(e0);
            dfma_kernel<<<grid, block>>>(out, iters, 1.0000001, 1e-7);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double flops = 2.0 * 16 * iters * (double)grid.x * block.x;
            printf("DFMA  blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", bps, flops / ms / 1e9, ms);
            cudaEventRecord(e0);
            dmma_kernel<<<grid, block>>>(out, iters / 4, 1.0000001, 1e-7);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            flops = 2.0 * 256 * 8 * (iters / 4) * (double)grid.x * (block.x / 32);
            printf("DMMA  blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", bps, flops / ms / 1e9, ms);
        }
    }
    printf("SMs=%d\n", sms);
    return 0;
}
