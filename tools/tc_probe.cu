// tc_probe.cu -- standalone validation of the tcgen05 kind::tf32 building blocks used by the
// fp32 3xTF32 engine: SWIZZLE_128B K-major smem operands written by cp.async, UMMA smem and
// instruction descriptors, TMEM alloc / tcgen05.mma / commit->mbarrier / tcgen05.ld.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_probe tools/tc_probe.cu && tools/tc_probe
// Computes S = A B^T for A, B: 128 x K fp32 (K-major), plain TF32 and 3xTF32, against fp64.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                       \
    do {                                                                                            \
        cudaError_t e = (x);                                                                        \
        if (e != cudaSuccess) {                                                                     \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);          \
            exit(1);                                                                                \
        }                                                                                           \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t make_desc_sw128(const void *smem_ptr) {
    const uint64_t addr = smem_u32(smem_ptr);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;          // start address
    d |= (uint64_t)(0) << 16;              // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;      // SBO: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                // version (sm100)
    d |= (uint64_t)2 << 61;                // SWIZZLE_128B
    return d;
}

template <int MBIT>
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << MBIT);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// one CTA, 128 threads; K multiple of 32; mode 0 = plain tf32 (hi only), 1 = 3xTF32
template <int MBIT>
__global__ void probe(const float *A, const float *B, int K, float *C, int mode) {
    extern __shared__ __align__(1024) unsigned char sm[];
    // 4 operand tiles of 128 rows x 128 B (32 fp32), each 16 KiB, 1024-B aligned
    float *sAh = reinterpret_cast<float *>(sm), *sAl = sAh + 4096, *sBh = sAl + 4096, *sBl = sBh + 4096;
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base_sh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_sh;
    const uint32_t idesc = idesc_tf32<MBIT>(128, 128);
    uint32_t phase = 0;
    for (int k0 = 0; k0 < K; k0 += 32) {
        // each thread: one row (tid) of A and B, 8 chunks of 16 B (4 fp32), swizzled
        for (int c = 0; c < 8; ++c) {
            const int r = tid;
            float4 a = *reinterpret_cast<const float4 *>(A + (size_t)r * K + k0 + 4 * c);
            float4 b = *reinterpret_cast<const float4 *>(B + (size_t)r * K + k0 + 4 * c);
            float4 ah = make_float4(to_tf32(a.x), to_tf32(a.y), to_tf32(a.z), to_tf32(a.w));
            float4 bh = make_float4(to_tf32(b.x), to_tf32(b.y), to_tf32(b.z), to_tf32(b.w));
            float4 al = make_float4(to_tf32(a.x - ah.x), to_tf32(a.y - ah.y), to_tf32(a.z - ah.z), to_tf32(a.w - ah.w));
            float4 bl = make_float4(to_tf32(b.x - bh.x), to_tf32(b.y - bh.y), to_tf32(b.z - bh.z), to_tf32(b.w - bh.w));
            const int off = r * 32 + ((c ^ (r & 7)) * 4);
            *reinterpret_cast<float4 *>(sAh + off) = ah;
            *reinterpret_cast<float4 *>(sAl + off) = al;
            *reinterpret_cast<float4 *>(sBh + off) = bh;
            *reinterpret_cast<float4 *>(sBl + off) = bl;
        }
        asm volatile("fence.proxy.async.shared::cta;");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            for (int kk = 0; kk < 4; ++kk) {  // 4 x K=8 per 32-wide slab; +32 B per step
                const uint64_t dah = make_desc_sw128(sAh) + (uint64_t)(kk * 2);
                const uint64_t dal = make_desc_sw128(sAl) + (uint64_t)(kk * 2);
                const uint64_t dbh = make_desc_sw128(sBh) + (uint64_t)(kk * 2);
                const uint64_t dbl = make_desc_sw128(sBl) + (uint64_t)(kk * 2);
                const uint32_t acc0 = (k0 > 0 || kk > 0) ? 1u : 0u;
                mma_tf32(tmem, dah, dbh, idesc, acc0);
                if (mode == 1) {
                    mma_tf32(tmem, dah, dbl, idesc, 1u);
                    mma_tf32(tmem, dal, dbh, idesc, 1u);
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&mbar)));
        }
        // wait for the MMAs (they read smem) before overwriting it
        asm volatile(
            "{\n.reg .pred P1;\nWAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
            "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(&mbar)),
            "r"(phase));
        phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;");
        __syncthreads();
    }
    // epilogue: warp w reads TMEM lanes 32w..32w+31 (rows), 128 columns in chunks of 16
    for (int c0 = 0; c0 < 128; c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; ++j) C[(size_t)(warp * 32 + lane) * 128 + c0 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

template <int MBIT>
void run(int K) {
    std::vector<float> A(128 * K), B(128 * K), C(128 * 128);
    srand(1);
    for (auto &x : A) x = (rand() / (float)RAND_MAX) * 2 - 1;
    for (auto &x : B) x = (rand() / (float)RAND_MAX) * 2 - 1;
    float *dA, *dB, *dC;
    CK(cudaMalloc(&dA, A.size() * 4));
    CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&dC, C.size() * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(probe<MBIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024));
    for (int mode = 0; mode < 2; ++mode) {
        CK(cudaMemset(dC, 0, C.size() * 4));
        probe<MBIT><<<1, 128, 65536 + 1024>>>(dA, dB, K, dC, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("MBIT=%d mode=%d: kernel error %s\n", MBIT, mode, cudaGetErrorString(e));
            exit(1);
        }
        CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
        double num = 0, den = 0, mx = 0;
        for (int i = 0; i < 128; ++i)
            for (int j = 0; j < 128; ++j) {
                double s = 0;
                for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * (double)B[j * K + k];
                const double dlt = C[i * 128 + j] - s;
                num += dlt * dlt;
                den += s * s;
                mx = fmax(mx, fabs(dlt));
            }
        printf("MBIT=%d K=%d mode=%s: rel err %.3e  max abs %.3e  C[0]=%f C[129]=%f\n", MBIT, K,
               mode ? "3xTF32" : "tf32", sqrt(num / den), mx, C[0], C[129]);
    }
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
}


// ---- SWIZZLE_64B, N = 256 variant: 16 fp32 (64 B) per row, A 128 rows, B 256 rows --------------
// 64-byte swizzle atom (8 rows x 64 B = 512 B): 16-byte chunk c (0..3) of row r at c ^ ((r >> 1) & 3).
__device__ __forceinline__ uint64_t make_desc_sw64(const void *smem_ptr) {
    const uint64_t addr = smem_u32(smem_ptr);
    return ((addr >> 4) & 0x3FFFull) | ((uint64_t)(512 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}

__global__ void probe_n256(const float *A, const float *B, int K, float *C) {
    extern __shared__ __align__(1024) unsigned char sm[];
    float *sAh = reinterpret_cast<float *>(sm), *sAl = sAh + 128 * 16, *sBh = sAl + 128 * 16, *sBl = sBh + 256 * 16;
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base_sh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_sh;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    uint32_t phase = 0;
    for (int k0 = 0; k0 < K; k0 += 16) {
        for (int rr = tid; rr < 256; rr += 128) {
            for (int c = 0; c < 4; ++c) {
                const int off = rr * 16 + ((c ^ ((rr >> 1) & 3)) * 4);
                float4 b = *reinterpret_cast<const float4 *>(B + (size_t)rr * K + k0 + 4 * c);
                float4 bh = make_float4(to_tf32(b.x), to_tf32(b.y), to_tf32(b.z), to_tf32(b.w));
                float4 bl = make_float4(to_tf32(b.x - bh.x), to_tf32(b.y - bh.y), to_tf32(b.z - bh.z), to_tf32(b.w - bh.w));
                *reinterpret_cast<float4 *>(sBh + off) = bh;
                *reinterpret_cast<float4 *>(sBl + off) = bl;
                if (rr < 128) {
                    float4 a = *reinterpret_cast<const float4 *>(A + (size_t)rr * K + k0 + 4 * c);
                    float4 ah = make_float4(to_tf32(a.x), to_tf32(a.y), to_tf32(a.z), to_tf32(a.w));
                    float4 al = make_float4(to_tf32(a.x - ah.x), to_tf32(a.y - ah.y), to_tf32(a.z - ah.z), to_tf32(a.w - ah.w));
                    *reinterpret_cast<float4 *>(sAh + off) = ah;
                    *reinterpret_cast<float4 *>(sAl + off) = al;
                }
            }
        }
        asm volatile("fence.proxy.async.shared::cta;");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            for (int kk = 0; kk < 2; ++kk) {
                const uint64_t o = (uint64_t)(kk * 2);
                const uint32_t acc0 = (k0 > 0 || kk > 0) ? 1u : 0u;
                mma_tf32(tmem, make_desc_sw64(sAh) + o, make_desc_sw64(sBh) + o, idesc, acc0);
                mma_tf32(tmem, make_desc_sw64(sAh) + o, make_desc_sw64(sBl) + o, idesc, 1u);
                mma_tf32(tmem, make_desc_sw64(sAl) + o, make_desc_sw64(sBh) + o, idesc, 1u);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
        }
        asm volatile(
            "{\n.reg .pred P1;\nWAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
            "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(&mbar)),
            "r"(phase));
        phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;");
        __syncthreads();
    }
    for (int c0 = 0; c0 < 256; c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; ++j) C[(size_t)(warp * 32 + lane) * 256 + c0 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

void run_n256(int K) {
    std::vector<float> A(128 * K), B(256 * K), C(128 * 256);
    srand(2);
    for (auto &x : A) x = (rand() / (float)RAND_MAX) * 2 - 1;
    for (auto &x : B) x = (rand() / (float)RAND_MAX) * 2 - 1;
    float *dA, *dB, *dC;
    CK(cudaMalloc(&dA, A.size() * 4));
    CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&dC, C.size() * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(probe_n256, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152 + 1024));
    probe_n256<<<1, 128, 49152 + 1024>>>(dA, dB, K, dC);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("n256: kernel error %s\n", cudaGetErrorString(e)); exit(1); }
    CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
    double num = 0, den = 0;
    for (int i = 0; i < 128; ++i)
        for (int j = 0; j < 256; ++j) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * (double)B[j * K + k];
            num += (C[i * 256 + j] - s) * (C[i * 256 + j] - s);
            den += s * s;
        }
    printf("SW64 N=256 K=%d 3xTF32: rel err %.3e\n", K, sqrt(num / den));
}

int main(int argc, char **argv) {
    if (argc > 1 && atoi(argv[1]) == 256) { run_n256(256); return 0; }
    const int mbit = argc > 1 ? atoi(argv[1]) : 24;
    if (mbit == 23) run<23>(256);
    else run<24>(256);
    return 0;
}
