// Online upcycling copy (K12): replicate one dense SwiGLU FFN into E_local
// experts in the kernel's K-major weight layout.
//
// Reference: moefold/upcycle.py:104-112 (upcycle_full: every expert is a bitwise
// copy of the dense w1/w2/w3) and :216-224 (upcycle_shard: each EP rank copies its
// local FFN into the experts it owns).  Source layout is the reference's
// [in, out] (w1, w3: [H, F]; w2: [F, H]); destination is W1, W3: [E, F, H] and
// W2: [E, H, F] (bf16), i.e. a tiled transpose written E_local times.  The
// fp32 -> bf16 conversion is round-to-nearest-even (identical to torch's cast).
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "common.cuh"

namespace b200moe {

constexpr int kTile = 64;
constexpr int kTPad = 8;   // row stride 72 bf16 = 144 B: 16-byte aligned rows, 4-way conflicts on the transposed fill

// src [R, C] (fp32 or bf16) -> dst[e] [C, R] bf16 for e < E_local.  The tile
// is transposed on its way into shared memory, so each output row segment is
// 8 contiguous bf16 there and goes out as one 16-byte store per expert copy
// (the E_local-fold write stream is what bounds this kernel).
template <typename T>
__global__ void __launch_bounds__(256) transpose_replicate(const T* __restrict__ src, int R, int C, int E_local,
                                                           __nv_bfloat16* __restrict__ dst) {
    __shared__ __align__(16) __nv_bfloat16 tile[kTile][kTile + kTPad];   // tile[c][r]
    const int r0 = blockIdx.y * kTile, c0 = blockIdx.x * kTile;
    for (int i = threadIdx.x; i < kTile * kTile; i += blockDim.x) {
        const int r = i / kTile, c = i % kTile;   // coalesced along c in the source
        __nv_bfloat16 v = __float2bfloat16_rn(0.f);
        if (r0 + r < R && c0 + c < C) {
            if constexpr (sizeof(T) == 4) v = __float2bfloat16_rn(src[(size_t)(r0 + r) * C + c0 + c]);
            else v = src[(size_t)(r0 + r) * C + c0 + c];
        }
        tile[c][r] = v;
    }
    __syncthreads();
    const size_t plane = (size_t)R * C;
    const bool vec = (R % 8) == 0;
    for (int i = threadIdx.x; i < kTile * (kTile / 8); i += blockDim.x) {
        const int c = i / (kTile / 8), r = (i % (kTile / 8)) * 8;   // 8 consecutive destination columns
        if (c0 + c >= C || r0 + r >= R) continue;
        __nv_bfloat16* out = dst + (size_t)(c0 + c) * R + r0 + r;
        if (vec && r0 + r + 8 <= R) {
            const uint4 v = *reinterpret_cast<const uint4*>(&tile[c][r]);
            for (int e = 0; e < E_local; ++e) *reinterpret_cast<uint4*>(out + e * plane) = v;
        } else {
            for (int j = 0; j < 8 && r0 + r + j < R; ++j) {
                const __nv_bfloat16 v = tile[c][r + j];
                for (int e = 0; e < E_local; ++e) out[e * plane + j] = v;
            }
        }
    }
}

template <typename T>
static void launch_t(const void* src, int R, int C, int E_local, void* dst, cudaStream_t s) {
    dim3 grid(ceil_div(C, kTile), ceil_div(R, kTile));
    transpose_replicate<T><<<grid, 256, 0, s>>>((const T*)src, R, C, E_local, (__nv_bfloat16*)dst);
}

}  // namespace b200moe

using namespace b200moe;

extern "C" int b200moe_upcycle_copy(const void* w1, const void* w2, const void* w3, int src_is_fp32, int H, int F,
                                    int E_local, void* W1, void* W2, void* W3, cudaStream_t stream) {
    B200_CHECK_ARG(H >= 1 && F >= 1, B200MOE_ERR_SHAPE, "bad FFN shape (%d, %d)", H, F);
    B200_CHECK_ARG(E_local >= 1, B200MOE_ERR_CONFIG, "upcycling needs at least one local expert");
    if (src_is_fp32) {
        launch_t<float>(w1, H, F, E_local, W1, stream);
        launch_t<float>(w3, H, F, E_local, W3, stream);
        launch_t<float>(w2, F, H, E_local, W2, stream);
    } else {
        launch_t<__nv_bfloat16>(w1, H, F, E_local, W1, stream);
        launch_t<__nv_bfloat16>(w3, H, F, E_local, W3, stream);
        launch_t<__nv_bfloat16>(w2, F, H, E_local, W2, stream);
    }
    B200_CHECK_LAUNCH("upcycle_copy");
    return B200MOE_OK;
}
