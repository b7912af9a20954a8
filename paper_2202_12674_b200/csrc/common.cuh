// common.cuh -- shared helpers of the B200 CUDA path (no method arithmetic here).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace plssvm {

constexpr int kTile = 128;         // Q~ tile edge (rows = cols), CTA tile of the tile engine
constexpr int kThreads = 256;      // threads of the tile-engine CTA (16 x 16 grid, 8x8 micro-tile)
constexpr int kVecThreads = 256;   // threads of the vector (CG) kernels
constexpr int kVecBlocks = 296;    // 2 x 148 SMs: grid of the vector kernels (fixed => deterministic)

enum Kernel : int { LINEAR = 0, POLYNOMIAL = 1, RBF = 2 };

// Error carrying a plssvm_status_t code.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &msg) : std::runtime_error(msg), code(c) {}
};

#define PLS_CUDA(call)                                                                       \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess) {                                                             \
            if (e_ == cudaErrorMemoryAllocation)                                             \
                throw ::plssvm::Error(3, std::string("CUDA OOM: ") + #call + " -> " +        \
                                             cudaGetErrorString(e_));                         \
            throw ::plssvm::Error(4, std::string(#call) + " -> " + cudaGetErrorString(e_) +  \
                                         " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
        }                                                                                    \
    } while (0)

#define PLS_CHECK_LAUNCH() PLS_CUDA(cudaGetLastError())

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Kernel-function parameters passed by value to device code.
template <typename T>
struct KParams {
    int kernel;
    T gamma;
    int degree;
    T coef0;
};

}  // namespace plssvm
