// Router backward (K10 + K11), router weight gradients, importance penalty.
//
// Reference: softmax backward tensor.py:292-295, st top-k mask product
// moe.py:186 (mul backward), softplus backward tensor.py:224, take_rows
// backward tensor.py:375-378 (np.add.at), router matmul backward tensor.py:203,
// importance_penalty tensor.py:503-521.
//
//   dg_total = dg (expert path, kept slots) + dgates_ext (e.g. aux loss)
//   mixtral: dh = keep*p*(dg_total - sum(p*dg_total))       (p = gates)
//   st:      ds = dg_total*topk; dh = s*(ds - sum(s*ds))    (s = probs)
//   dn = dh * z * sigmoid(x.W_noise)          (noise only)
//   dx = sum_{kept e asc} dxp[row] + dh.W_g^T + dn.W_noise^T
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <math.h>

#include "common.cuh"

namespace b200moe {

template <int EP>
__global__ void swizzle_w_kernel_bwd(const float* __restrict__ w, int H, int E, float4* __restrict__ out) {
    const int n = (H / 4) * 4 * (EP / 4);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int hb = i % (H / 4);
        const int rest = i / (H / 4);
        const int e4 = rest % (EP / 4);
        const int j = rest / (EP / 4);
        const int h = hb * 4 + j;
        float v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int e = e4 * 4 + c;
            v[c] = (e < E) ? w[(size_t)h * E + e] : 0.f;
        }
        out[i] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

constexpr int kRbThreads = 512;

template <int EP, bool kNoise, bool kSmemW>
__global__ void __launch_bounds__(kRbThreads, 1)
router_bwd_kernel(const __nv_bfloat16* __restrict__ dxp, const int32_t* __restrict__ slot_rank,
                  const int32_t* __restrict__ seg_base, const float* __restrict__ dg,
                  const float* __restrict__ dgx, int64_t sx_t, int64_t sx_e, const float* __restrict__ gates,
                  const float* __restrict__ probs, const float4* __restrict__ wsw, const float4* __restrict__ wnsw,
                  const float* __restrict__ z, const float* __restrict__ noise_act, int T, int H, int E,
                  int router_type, __nv_bfloat16* __restrict__ dx, float* __restrict__ dh_out,
                  float* __restrict__ dn_out) {
    constexpr int TT = 32 / EP;
    extern __shared__ float4 smem_w[];
    const float4* W = wsw;
    if constexpr (kSmemW) {
        for (int i = threadIdx.x; i < H * EP / 4; i += blockDim.x) smem_w[i] = wsw[i];
        __syncthreads();
        W = smem_w;
    }
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    const int HB = H / 4;
    const int tt_mine = lane / EP, e_mine = lane % EP;

    for (int t0 = (blockIdx.x * (blockDim.x >> 5) + warp) * TT; t0 < T; t0 += nwarps * TT) {
        // ---- per (token, expert) lane: dh, dn
        const int t = t0 + tt_mine;
        const bool live = (t < T) && (e_mine < E);
        float gt = 0.f, pv = 0.f, topk = 0.f;
        int rank = -1;
        if (live) {
            const size_t i = (size_t)t * E + e_mine;
            gt = dg[i];
            if (dgx) gt += dgx[(int64_t)t * sx_t + (int64_t)e_mine * sx_e];
            const float gv = gates[i];
            pv = (router_type == B200MOE_ROUTER_MIXTRAL) ? gv : probs[i];
            topk = (gv > 0.f) ? 1.f : 0.f;
            rank = slot_rank[i];
        }
        const float geff = (router_type == B200MOE_ROUTER_MIXTRAL) ? ((pv > 0.f) ? gt : 0.f) : gt * topk;
        float dot = pv * geff;
#pragma unroll
        for (int o = 1; o < EP; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        float dhv = live ? pv * (geff - dot) : 0.f;
        if (router_type == B200MOE_ROUTER_MIXTRAL && !(pv > 0.f)) dhv = 0.f;
        float dnv = 0.f;
        if constexpr (kNoise) {
            if (live) {
                const size_t i = (size_t)t * E + e_mine;
                const float an = noise_act[i];
                const float sg = 1.0f / (1.0f + expf(-an));
                dnv = dhv * z[i] * sg;
                dn_out[i] = dnv;
            }
        }
        if (live) dh_out[(size_t)t * E + e_mine] = dhv;
        // broadcast all (token, expert) values to every lane
        float dhall[32], dnall[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            dhall[i] = __shfl_sync(0xffffffffu, dhv, i);
            if constexpr (kNoise) dnall[i] = __shfl_sync(0xffffffffu, dnv, i);
        }
        // rows of the kept experts for each token (ascending expert order)
        const int row = (rank >= 0) ? seg_base[e_mine] + rank : -1;
        int rr[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) rr[i] = __shfl_sync(0xffffffffu, row, i);

        for (int hb = lane; hb < HB; hb += 32) {
            float acc[TT][4];
#pragma unroll
            for (int tt = 0; tt < TT; ++tt)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[tt][j] = 0.f;
            // expert-path contributions, ascending expert order
#pragma unroll
            for (int tt = 0; tt < TT; ++tt) {
#pragma unroll
                for (int e = 0; e < EP; ++e) {
                    const int r = rr[tt * EP + e];
                    if (r >= 0) {
                        const uint2 u = *reinterpret_cast<const uint2*>(dxp + (size_t)r * H + hb * 4);
                        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
                        const float2 f0 = __bfloat1622float2(b[0]), f1 = __bfloat1622float2(b[1]);
                        acc[tt][0] += f0.x; acc[tt][1] += f0.y; acc[tt][2] += f1.x; acc[tt][3] += f1.y;
                    }
                }
            }
            // router path: dh . W_g^T (+ dn . W_noise^T)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
#pragma unroll
                for (int e4 = 0; e4 < EP / 4; ++e4) {
                    const float4 w = W[(j * (EP / 4) + e4) * HB + hb];
#pragma unroll
                    for (int tt = 0; tt < TT; ++tt) {
                        const float* d = dhall + tt * EP + e4 * 4;
                        acc[tt][j] = fmaf(d[0], w.x, acc[tt][j]);
                        acc[tt][j] = fmaf(d[1], w.y, acc[tt][j]);
                        acc[tt][j] = fmaf(d[2], w.z, acc[tt][j]);
                        acc[tt][j] = fmaf(d[3], w.w, acc[tt][j]);
                    }
                    if constexpr (kNoise) {
                        const float4 wn = __ldg(&wnsw[(j * (EP / 4) + e4) * HB + hb]);
#pragma unroll
                        for (int tt = 0; tt < TT; ++tt) {
                            const float* d = dnall + tt * EP + e4 * 4;
                            acc[tt][j] = fmaf(d[0], wn.x, acc[tt][j]);
                            acc[tt][j] = fmaf(d[1], wn.y, acc[tt][j]);
                            acc[tt][j] = fmaf(d[2], wn.z, acc[tt][j]);
                            acc[tt][j] = fmaf(d[3], wn.w, acc[tt][j]);
                        }
                    }
                }
            }
#pragma unroll
            for (int tt = 0; tt < TT; ++tt) {
                if (t0 + tt < T) {
                    uint2 u;
                    u.x = pack2(acc[tt][0], acc[tt][1]);
                    u.y = pack2(acc[tt][2], acc[tt][3]);
                    *reinterpret_cast<uint2*>(dx + (size_t)(t0 + tt) * H + hb * 4) = u;
                }
            }
        }
    }
}

// dW[h, e] = sum_t x[t, h] * d[t, e]: per (H/1024 block, 128-token chunk) partials,
// then a fixed-order reduction over chunks.
constexpr int kWgTok = 128;

template <int EP>
__global__ void __launch_bounds__(256)
router_wgrad_partial(const __nv_bfloat16* __restrict__ x, const float* __restrict__ d, int T, int H, int E,
                     float* __restrict__ part) {
    __shared__ float ds[kWgTok * EP];
    const int chunk = blockIdx.y;
    const int t0 = chunk * kWgTok;
    for (int i = threadIdx.x; i < kWgTok * EP; i += blockDim.x) {
        const int tt = i / EP, e = i % EP;
        const int t = t0 + tt;
        ds[i] = (t < T && e < E) ? d[(size_t)t * E + e] : 0.f;
    }
    __syncthreads();
    const int h0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (h0 >= H) return;
    float acc[4][EP];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < EP; ++e) acc[j][e] = 0.f;
    const int tn = min(kWgTok, T - t0);
    for (int tt = 0; tt < tn; ++tt) {
        const uint2 u = *reinterpret_cast<const uint2*>(x + (size_t)(t0 + tt) * H + h0);
        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
        const float2 f0 = __bfloat1622float2(b[0]), f1 = __bfloat1622float2(b[1]);
        const float xv[4] = {f0.x, f0.y, f1.x, f1.y};
#pragma unroll
        for (int e = 0; e < EP; ++e) {
            const float dv = ds[tt * EP + e];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j][e] = fmaf(xv[j], dv, acc[j][e]);
        }
    }
    float* p = part + (size_t)chunk * H * E;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < EP; ++e)
            if (e < E) p[(size_t)(h0 + j) * E + e] = acc[j][e];
}

__global__ void reduce_partials(const float* __restrict__ part, int nchunks, size_t n, float* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float s = 0.f;
        for (int c = 0; c < nchunks; ++c) s += part[(size_t)c * n + i];
        out[i] = s;
    }
}

// Importance penalty forward: one block.  imp_e = sum_t g[t,e] (fixed order),
// mean, population variance, loss = var / mean^2 (tensor.py:509-514).
__global__ void importance_fwd_kernel(const float* __restrict__ g, int T, int E, float* __restrict__ imp,
                                      float* __restrict__ loss, int32_t* __restrict__ err_flag) {
    __shared__ float part[32][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;  // 32 warps
    for (int e0 = 0; e0 < E; e0 += 32) {
        const int e = e0 + lane;
        float s = 0.f;
        if (e < E)
            for (int t = warp; t < T; t += 32) s += g[(size_t)t * E + e];
        part[warp][lane] = s;
        __syncthreads();
        if (warp == 0 && e < E) {
            float r = 0.f;
            for (int w = 0; w < 32; ++w) r += part[w][lane];
            imp[e] = r;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        float mean = 0.f;
        for (int e = 0; e < E; ++e) mean += ((volatile float*)imp)[e];
        mean /= (float)E;
        float var = 0.f;
        for (int e = 0; e < E; ++e) {
            const float d = ((volatile float*)imp)[e] - mean;
            var += d * d;
        }
        var /= (float)E;
        if (!(mean > 0.f)) atomicExch(err_flag, 1);
        loss[0] = var / (mean * mean);
    }
}

// dimp_e = gscale * (2 (imp_e - mean) / (E mean^2) - 2 var / (E mean^3))  (tensor.py:517-518)
__global__ void importance_bwd_kernel(const float* __restrict__ imp, const float* __restrict__ gscale, int E,
                                      float* __restrict__ dimp) {
    if (threadIdx.x != 0) return;
    float mean = 0.f;
    for (int e = 0; e < E; ++e) mean += imp[e];
    mean /= (float)E;
    float var = 0.f;
    for (int e = 0; e < E; ++e) {
        const float d = imp[e] - mean;
        var += d * d;
    }
    var /= (float)E;
    const float gs = gscale ? gscale[0] : 1.0f;
    const float n = (float)E;
    for (int e = 0; e < E; ++e)
        dimp[e] = gs * (2.0f * (imp[e] - mean) / (n * mean * mean) - 2.0f * var / (n * mean * mean * mean));
}

}  // namespace b200moe

using namespace b200moe;

namespace {
template <int EP>
int router_bwd_impl(const void* dxp, const int32_t* slot_rank, const int32_t* seg_base, const float* dg,
                    const float* dgx, int64_t sx_t, int64_t sx_e, const float* gates, const float* probs,
                    const float* w_g, const float* w_noise, const float* z, const float* noise_act, int T, int H,
                    int E, int router_type, void* dx, float* dh, float* dn, float* workspace, cudaStream_t stream) {
    float4* wsw = reinterpret_cast<float4*>(workspace);
    float4* wnsw = reinterpret_cast<float4*>(workspace + (size_t)H * EP);
    swizzle_w_kernel_bwd<EP><<<64, 256, 0, stream>>>(w_g, H, E, wsw);
    const bool noise = z != nullptr;
    if (noise) swizzle_w_kernel_bwd<EP><<<64, 256, 0, stream>>>(w_noise, H, E, wnsw);
    const size_t wbytes = (size_t)H * EP * sizeof(float);
    const bool smem_w = wbytes <= 160 * 1024;
    constexpr int TT = 32 / EP;
    int grid = ceil_div(ceil_div(T, TT), kRbThreads / 32);
    if (grid > kNumSMs) grid = kNumSMs;
#define LAUNCH(NZ, SM)                                                                                         \
    do {                                                                                                       \
        auto kern = router_bwd_kernel<EP, NZ, SM>;                                                             \
        const size_t sh = SM ? wbytes : 0;                                                                     \
        if (SM) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh);              \
        kern<<<grid, kRbThreads, sh, stream>>>((const __nv_bfloat16*)dxp, slot_rank, seg_base, dg, dgx, sx_t, \
                                               sx_e, gates, probs, wsw, wnsw, z, noise_act, T, H, E,          \
                                               router_type, (__nv_bfloat16*)dx, dh, dn);                       \
    } while (0)
    if (noise) {
        if (smem_w) LAUNCH(true, true); else LAUNCH(true, false);
    } else {
        if (smem_w) LAUNCH(false, true); else LAUNCH(false, false);
    }
#undef LAUNCH
    B200_CHECK_LAUNCH("router_bwd");
    return B200MOE_OK;
}

template <int EP>
int wgrad_impl(const void* x, const float* d, int T, int H, int E, float* out, float* part, cudaStream_t stream) {
    const int nch = ceil_div(T, kWgTok);
    dim3 grid(ceil_div(H, 1024), nch);
    router_wgrad_partial<EP><<<grid, 256, 0, stream>>>((const __nv_bfloat16*)x, d, T, H, E, part);
    const size_t n = (size_t)H * E;
    reduce_partials<<<(int)((n + 255) / 256), 256, 0, stream>>>(part, nch, n, out);
    B200_CHECK_LAUNCH("router_wgrad");
    return B200MOE_OK;
}
}  // namespace

extern "C" {

int b200moe_router_bwd(const void* dxp, const int32_t* slot_rank, const int32_t* seg_base, const float* dg,
                       const float* dgates_ext, int64_t dgates_stride_t, int64_t dgates_stride_e, const float* gates,
                       const float* probs, const float* w_g, const float* w_noise, const float* z,
                       const float* noise_act, int T, int H, int E, int router_type, void* dx, float* dh, float* dn,
                       float* workspace, cudaStream_t stream) {
    B200_CHECK_ARG(T >= 1 && E >= 1 && E <= 32, B200MOE_ERR_CONFIG, "bad T/E (%d, %d)", T, E);
    B200_CHECK_ARG(H % 4 == 0, B200MOE_ERR_SHAPE, "hidden must be a multiple of 4");
    B200_CHECK_ARG(router_type != B200MOE_ROUTER_ST || probs != nullptr, B200MOE_ERR_CONFIG, "st needs probs");
    B200_CHECK_ARG(z == nullptr || (w_noise && noise_act && dn), B200MOE_ERR_CONFIG, "noise args missing");
#define CALL(EP) router_bwd_impl<EP>(dxp, slot_rank, seg_base, dg, dgates_ext, dgates_stride_t, dgates_stride_e, \
                                     gates, probs, w_g, w_noise, z, noise_act, T, H, E, router_type, dx, dh, dn,  \
                                     workspace, stream)
    if (E <= 4) return CALL(4);
    if (E <= 8) return CALL(8);
    if (E <= 16) return CALL(16);
    return CALL(32);
#undef CALL
}

int b200moe_router_wgrad(const void* x, const float* dh, const float* dn, int T, int H, int E, float* dw_g,
                         float* dw_noise, float* workspace, cudaStream_t stream) {
    B200_CHECK_ARG(T >= 1 && E >= 1 && E <= 32, B200MOE_ERR_CONFIG, "bad T/E (%d, %d)", T, E);
    B200_CHECK_ARG(H % 4 == 0, B200MOE_ERR_SHAPE, "hidden must be a multiple of 4");
#define CALL(EP, D, O) wgrad_impl<EP>(x, D, T, H, E, O, workspace, stream)
    int rc;
    if (E <= 4) rc = CALL(4, dh, dw_g);
    else if (E <= 8) rc = CALL(8, dh, dw_g);
    else if (E <= 16) rc = CALL(16, dh, dw_g);
    else rc = CALL(32, dh, dw_g);
    if (rc || dn == nullptr) return rc;
    if (E <= 4) return CALL(4, dn, dw_noise);
    if (E <= 8) return CALL(8, dn, dw_noise);
    if (E <= 16) return CALL(16, dn, dw_noise);
    return CALL(32, dn, dw_noise);
#undef CALL
}

int b200moe_importance_fwd(const float* gates, int T, int E, float* imp, float* loss, int32_t* err_flag,
                           cudaStream_t stream) {
    B200_CHECK_ARG(T >= 1 && E >= 1, B200MOE_ERR_SHAPE, "importance penalty needs a [T, E] gate matrix");
    importance_fwd_kernel<<<1, 1024, 0, stream>>>(gates, T, E, imp, loss, err_flag);
    B200_CHECK_LAUNCH("importance_fwd");
    return B200MOE_OK;
}

int b200moe_importance_bwd(const float* imp, const float* gscale, int E, float* dimp, cudaStream_t stream) {
    B200_CHECK_ARG(E >= 1, B200MOE_ERR_SHAPE, "E >= 1");
    importance_bwd_kernel<<<1, 32, 0, stream>>>(imp, gscale, E, dimp);
    B200_CHECK_LAUNCH("importance_bwd");
    return B200MOE_OK;
}

}  // extern "C"
