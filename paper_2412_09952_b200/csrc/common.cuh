// Shared helpers for the b200moe CUDA library (sm_100a only).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <atomic>

#include "../../include/b200moe.h"

#ifndef __CUDACC__
#error "compile with nvcc"
#endif

namespace b200moe {

// Thread-local error message behind b200moe_last_error().
void set_error(const char* fmt, ...);

// Make the current device's primary context current on this thread (for
// driver-API calls on a thread that has made no runtime call yet).
bool bind_current_context();

// 2-D bf16 TMA map over a row-major [outer, inner] tensor (row pitch ld
// elements), box {box_inner, box_outer}, no swizzle (rows land contiguous in
// shared memory) or the 128-byte swizzle of K-major tcgen05 operands,
// out-of-bounds rows zero-filled.  Returns a B200MOE_* code.
int make_tmap_bf16_2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                      uint32_t box_inner, uint32_t box_outer, bool sw128 = false);

#define B200_CHECK_ARG(cond, code, ...)          \
    do {                                         \
        if (!(cond)) {                           \
            ::b200moe::set_error(__VA_ARGS__);   \
            return (code);                       \
        }                                        \
    } while (0)

#define B200_CHECK_LAUNCH(what)                                                     \
    do {                                                                            \
        cudaError_t _e = cudaGetLastError();                                        \
        if (_e != cudaSuccess) {                                                    \
            ::b200moe::set_error("%s: %s", (what), cudaGetErrorString(_e));          \
            return B200MOE_ERR_CUDA;                                                \
        }                                                                           \
    } while (0)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: set it once
// per (kernel, device) the first time a launch lands on that device (thread-safe;
// a process driving several GPUs sets it on each).
template <class Kernel>
inline cudaError_t ensure_smem_attr(Kernel kern, int bytes, std::atomic<uint64_t>& done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

constexpr int kNumSMs = 148;     // B200
constexpr int kSegPad = 128;     // expert segments are zero-padded to this many rows

__host__ __device__ inline int round_up(int a, int b) { return (a + b - 1) / b * b; }
__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

__device__ __forceinline__ float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }

// 8 bf16 packed in a uint4 -> 8 floats
__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 t = __bfloat1622float2(p[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

__device__ __forceinline__ uint4 pack8(const float* f) {
    uint4 u;
    __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    return u;
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

__device__ __forceinline__ void st_v4(void* p, const uint4& v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// Two fp32 FMAs in one FFMA2 (sm_100 packed fp32 pipe): acc.{x,y} = fma(a.{x,y}, b.{x,y}, acc.{x,y}),
// each rounded exactly like fmaf (no FTZ), so results are bit-identical to two scalar fmaf.
__device__ __forceinline__ void ffma2(float2& acc, float2 a, float2 b) {
    unsigned long long r, x, y;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b.x), "f"(b.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(acc.x), "f"(acc.y));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(r) : "l"(x), "l"(y));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(acc.x), "=f"(acc.y) : "l"(r));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Importance (CV^2) loss from the per-expert gate masses (tensor.py:509-514):
// mean, population variance, var / mean^2; err_flag (nullable) set when mean <= 0.
__device__ __forceinline__ void importance_cv2(const volatile float* imp, int E, float* loss, int32_t* err_flag) {
    float mean = 0.f;
    for (int e = 0; e < E; ++e) mean += imp[e];
    mean /= (float)E;
    float var = 0.f;
    for (int e = 0; e < E; ++e) {
        const float dd = imp[e] - mean;
        var += dd * dd;
    }
    var /= (float)E;
    if (!(mean > 0.f) && err_flag) atomicExch(err_flag, 1);
    loss[0] = var / (mean * mean);
}

// Segment table: where each expert segment of the permuted activation buffer
// lives.  base[s] = first row, count[s] = valid rows (device), expert[s] =
// local expert index.  Rows [count, round_up(count,128)) are zero-filled.
struct SegTable {
    const int* base;
    const int* count;
    const int* expert;
    int nseg;
};

}  // namespace b200moe
