// Shared device helpers for the sm_100a kernels of libblockeig_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "../../include/bk_kernels.h"

#define BK_RET(expr)                                  \
    do {                                              \
        cudaError_t _e = (expr);                      \
        if (_e != cudaSuccess) return static_cast<int>(_e); \
    } while (0)

#define BK_LAUNCHED() return static_cast<int>(cudaGetLastError())

namespace bk {
constexpr int kMaxDevices = 64;
// Function attributes (dynamic shared memory, cluster size) and occupancy
// queries are per device: evaluate once per (call site, current device), so a
// host thread that moves between GPUs configures each of them.
struct OncePerDevice {
    std::once_flag flag[kMaxDevices];
    cudaError_t err[kMaxDevices] = {};
    template <class F>
    cudaError_t operator()(F&& f) {
        int dev = 0;
        const cudaError_t g = cudaGetDevice(&dev);
        if (g != cudaSuccess) return g;
        if (dev < 0 || dev >= kMaxDevices) return f();
        std::call_once(flag[dev], [&] { err[dev] = f(); });
        return err[dev];
    }
};
}  // namespace bk
#define BK_ONCE_PER_DEVICE(expr) \
    ([&]() -> cudaError_t { static ::bk::OncePerDevice _once; return _once([&]() -> cudaError_t { return (expr); }); }())

namespace bk {

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col) — SASS DMMA.8x8x4.
// Fragment ownership (lane = 4*g + t): a = A[g][t], b = B[t][g],
// c0/c1 = C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// 8-byte async global->shared copy (cp.async.ca); zero-fill when !pred
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int sz = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
// 4-byte variant
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
// 16-byte variant (cp.async.cg, L2 only); both addresses 16-byte aligned
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int sz = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace bk
