// Host cost of the CUDA runtime calls a training call makes around its kernels (stream-ordered
// pool allocations, events, elapsed-time queries), to size the non-product time of a bench step.
//   nvcc -O2 -o /tmp/hac tools/host_api_cost.cu && /tmp/hac
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
int main() {
    cudaSetDevice(0);
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, 0);
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    for (int rep = 0; rep < 3; ++rep) {
        std::vector<void *> p(30);
        auto t0 = now();
        for (int i = 0; i < 30; ++i) cudaMallocAsync(&p[i], (size_t(1) << 20) * (i + 1), s);
        auto t1 = now();
        for (int i = 0; i < 30; ++i) cudaFreeAsync(p[i], s);
        auto t2 = now();
        cudaStreamSynchronize(s);
        cudaEvent_t ev[16];
        auto t3 = now();
        for (auto &e : ev) cudaEventCreate(&e);
        auto t4 = now();
        for (auto &e : ev) cudaEventRecord(e, s);
        cudaStreamSynchronize(s);
        auto t5 = now();
        float ms;
        for (int i = 0; i + 1 < 16; ++i) cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
        auto t6 = now();
        for (auto &e : ev) cudaEventDestroy(e);
        auto t7 = now();
        int dev;
        for (int i = 0; i < 100; ++i) cudaSetDevice(0), cudaGetDevice(&dev);
        auto t8 = now();
        cudaMemPool_t pl;
        for (int i = 0; i < 100; ++i) cudaDeviceGetDefaultMemPool(&pl, 0), cudaMemPoolSetAttribute(pl, cudaMemPoolAttrReleaseThreshold, &thr);
        auto t9 = now();
        std::printf("rep %d: 30 mallocAsync %.1f us, 30 freeAsync %.1f us, 16 eventCreate %.1f us, 15 elapsed %.1f us, "
                    "16 eventDestroy %.1f us, setDevice+getDevice %.2f us each, mempool setup %.2f us each\n",
                    rep, us(t0, t1), us(t1, t2), us(t3, t4), us(t5, t6), us(t6, t7), us(t7, t8) / 100, us(t8, t9) / 100);
    }
    return 0;
}
