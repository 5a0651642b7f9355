// Kernels of the transformer step around the MoE layer:
// fused residual-add + RMSNorm forward/backward, embedding gather / segmented
// scatter-add, fused cross-entropy forward/backward, and the multi-tensor
// Adam / SGD-momentum optimizer step.  All of them are HBM-bound row or
// elementwise passes; the dense projections around them are plain library
// GEMMs and attention is the library SDPA.
//
// Reference: moefold/tensor.py:307-364 (rmsnorm, embedding, cross_entropy),
// moefold/train.py:146-179 (_Optimizer), moefold/model.py:135-169 (the block).
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <math.h>

#include "common.cuh"
#include "ptx.cuh"

namespace b200moe {

using bf16 = __nv_bfloat16;

constexpr int kRowThreads = 256;

// Block-wide sum (fixed order: warp shuffles, then warp 0 over the partials).
__device__ __forceinline__ float block_sum(float v, float* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    float t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.f;
    if (w == 0) t = warp_sum(t);
    if (threadIdx.x == 0) red[32] = t;
    __syncthreads();
    return red[32];
}

__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    float t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : -INFINITY;
    if (w == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t = fmaxf(t, __shfl_xor_sync(0xffffffffu, t, o));
    }
    if (threadIdx.x == 0) red[32] = t;
    __syncthreads();
    return red[32];
}

__device__ __forceinline__ float4 ld_bf16x4(const bf16* p) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ void st_bf16x4(bf16* p, float4 v) {
    uint2 u;
    u.x = pack2(v.x, v.y);
    u.y = pack2(v.z, v.w);
    *reinterpret_cast<uint2*>(p) = u;
}

// ---------------------------------------------------------------------------
// RMSNorm (tensor.py:307-321): ms = mean(x^2) + eps, r = ms^-1/2,
// y = (x * r) * gain.  Fused with the residual add x_out = x + delta so the
// block's two residual updates cost one pass each.  One block per row.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kRowThreads) rmsnorm_fwd_kernel(const float* __restrict__ x,
                                                                  const bf16* __restrict__ delta,
                                                                  const float* __restrict__ gain, int H, float eps,
                                                                  float* __restrict__ x_out, bf16* __restrict__ y,
                                                                  float* __restrict__ rstd) {
    __shared__ float red[33];
    const size_t row = blockIdx.x;
    const float* xr = x + row * H;
    float ss = 0.f;
    for (int c = threadIdx.x * 4; c < H; c += kRowThreads * 4) {
        float4 v = *reinterpret_cast<const float4*>(xr + c);
        if (delta != nullptr) {
            const float4 d = ld_bf16x4(delta + row * H + c);
            v.x += d.x; v.y += d.y; v.z += d.z; v.w += d.w;
            *reinterpret_cast<float4*>(x_out + row * H + c) = v;
        }
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    const float ms = block_sum(ss, red) / (float)H + eps;
    const float r = 1.0f / sqrtf(ms);
    const float* src = delta != nullptr ? x_out + row * H : xr;
    for (int c = threadIdx.x * 4; c < H; c += kRowThreads * 4) {
        const float4 v = *reinterpret_cast<const float4*>(src + c);
        const float4 g = *reinterpret_cast<const float4*>(gain + c);
        st_bf16x4(y + row * H + c, make_float4(v.x * r * g.x, v.y * r * g.y, v.z * r * g.z, v.w * r * g.w));
    }
    if (threadIdx.x == 0) rstd[row] = r;
}

// Backward (tensor.py:314-319): gg = dy * gain, dot = sum(gg * x),
// dx = r * gg - (r^3 / H) * x * dot (+ the residual stream's gradient),
// dgain = sum_rows dy * x * r.  Each block owns kBwdRows rows and all columns
// (NV float4 per thread), so the dgain partial sums stay in registers; a
// second kernel reduces the per-block partials in fixed order.
constexpr int kBwdRows = 8;

// Two block sums in one pass (same fixed order as block_sum for each).
__device__ __forceinline__ float2 block_sum2(float a, float b, float* red) {
    a = warp_sum(a);
    b = warp_sum(b);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) { red[w] = a; red[16 + w] = b; }
    __syncthreads();
    float ta = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.f;
    float tb = (threadIdx.x < (blockDim.x >> 5)) ? red[16 + threadIdx.x] : 0.f;
    if (w == 0) { ta = warp_sum(ta); tb = warp_sum(tb); }
    if (threadIdx.x == 0) { red[32] = ta; red[33] = tb; }
    __syncthreads();
    return make_float2(red[32], red[33]);
}

// Rows are taken two at a time with every load of both rows (dy, x and the
// residual gradient) issued before the row reductions: the kernel is bound by
// load latency, not bandwidth, at one row per step (measured 0.4 ms vs ~60 us
// of traffic at T=8192, H=4096 with 32 rows per block, one row at a time).
template <int NV>
__global__ void __launch_bounds__(kRowThreads) rmsnorm_bwd_kernel(
    const bf16* __restrict__ dy, const float* __restrict__ x, const float* __restrict__ rstd,
    const float* __restrict__ gain, const float* __restrict__ dres, int T, int H, float* __restrict__ dx,
    bf16* __restrict__ dx_bf16, float* __restrict__ dgain_part) {
    static_assert(kRowThreads / 32 <= 16, "block_sum2 holds 16 warp partials per value");
    __shared__ float red[34];
    float4 acc[NV], g[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        const int c = (j * kRowThreads + threadIdx.x) * 4;
        g[j] = c < H ? *reinterpret_cast<const float4*>(gain + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const int r0 = blockIdx.x * kBwdRows;
    const int r1 = min(T, r0 + kBwdRows);
    constexpr int kQ = NV <= 4 ? 2 : 1;   // rows per step (register budget: no spills at NV 8/16)
    for (int row = r0; row < r1; row += kQ) {
        const bool two = kQ == 2 && row + 1 < r1;
        float4 xv[kQ][NV], dv[kQ][NV], rv[kQ][NV];
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            const size_t o = (size_t)(row + q) * H;
            const bool on = q == 0 || two;
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                const int c = (j * kRowThreads + threadIdx.x) * 4;
                const bool in = on && c < H;
                dv[q][j] = in ? ld_bf16x4(dy + o + c) : z4;
                xv[q][j] = in ? *reinterpret_cast<const float4*>(x + o + c) : z4;
                rv[q][j] = (in && dres != nullptr) ? *reinterpret_cast<const float4*>(dres + o + c) : z4;
            }
        }
        const float ra = rstd[row];
        const float rb = two ? rstd[row + 1] : 0.f;
        float dot[2] = {0.f, 0.f};
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            const float r = q == 0 ? ra : rb;
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                const float4 d = dv[q][j];
                const float4 xx = xv[q][j];
                const float4 gg = make_float4(d.x * g[j].x, d.y * g[j].y, d.z * g[j].z, d.w * g[j].w);
                dot[q] += gg.x * xx.x + gg.y * xx.y + gg.z * xx.z + gg.w * xx.w;
                acc[j].x += d.x * xx.x * r;
                acc[j].y += d.y * xx.y * r;
                acc[j].z += d.z * xx.z * r;
                acc[j].w += d.w * xx.w * r;
                dv[q][j] = gg;
            }
        }
        const float2 dots = kQ == 2 ? block_sum2(dot[0], dot[1], red) : make_float2(block_sum(dot[0], red), 0.f);
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            if (q == 1 && !two) break;
            const float r = q == 0 ? ra : rb;
            const float k3 = r * r * r / (float)H * (q == 0 ? dots.x : dots.y);
            const size_t o = (size_t)(row + q) * H;
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                const int c = (j * kRowThreads + threadIdx.x) * 4;
                if (c < H) {
                    const float4 gg = dv[q][j], xx = xv[q][j], d = rv[q][j];
                    float4 v = make_float4(r * gg.x - k3 * xx.x, r * gg.y - k3 * xx.y, r * gg.z - k3 * xx.z,
                                           r * gg.w - k3 * xx.w);
                    if (dres != nullptr) { v.x += d.x; v.y += d.y; v.z += d.z; v.w += d.w; }
                    if (dx != nullptr) *reinterpret_cast<float4*>(dx + o + c) = v;
                    if (dx_bf16 != nullptr) st_bf16x4(dx_bf16 + o + c, v);
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = (j * kRowThreads + threadIdx.x) * 4;
        if (c < H) *reinterpret_cast<float4*>(dgain_part + (size_t)blockIdx.x * H + c) = acc[j];
    }
}

// Pipelined variant for the model shapes (H % 8 == 0): one block per SM
// walks a contiguous run of rows; each row's dy, x and residual gradient
// arrive in shared memory by three 1-D bulk async copies, kRmsStages rows
// ahead of the row being reduced, so the loads are not bounded by register
// space (the register kernel above holds two rows per block in flight and
// reaches ~1.9 TB/s at T=8192, H=4096).  Same arithmetic as rmsnorm_bwd_kernel
// per row; dgain partials per block.
constexpr int kRmsStages = 4;
constexpr int kRmsSmemMax = 200 * 1024;

template <int NV>
__global__ void __launch_bounds__(kRowThreads, 1) rmsnorm_bwd_ring_kernel(
    const bf16* __restrict__ dy, const float* __restrict__ x, const float* __restrict__ rstd,
    const float* __restrict__ gain, const float* __restrict__ dres, int T, int H, int rows_per_block, int stages,
    float* __restrict__ dx, bf16* __restrict__ dx_bf16, float* __restrict__ dgain_part) {
    extern __shared__ __align__(128) uint8_t rsm[];
    __shared__ float red[34];
    __shared__ __align__(8) uint64_t bar[kRmsStages];
    const size_t stage_bytes = (size_t)H * (2 + 4 + (dres != nullptr ? 4 : 0));
    const int r0 = blockIdx.x * rows_per_block;
    const int r1 = min(T, r0 + rows_per_block);
    auto issue = [&](int row, int st) {   // thread 0: the three row copies into stage st
        uint8_t* b = rsm + st * stage_bytes;
        const uint32_t bytes = (uint32_t)stage_bytes;
        ptx::mbar_arrive_expect_tx(&bar[st], bytes);
        ptx::bulk_load_1d(b, dy + (size_t)row * H, H * 2, &bar[st]);
        ptx::bulk_load_1d(b + H * 2, x + (size_t)row * H, H * 4, &bar[st]);
        if (dres != nullptr) ptx::bulk_load_1d(b + H * 6, dres + (size_t)row * H, H * 4, &bar[st]);
    };
    if (threadIdx.x == 0) {
        for (int i = 0; i < stages; ++i) ptx::mbar_init(&bar[i], 1);
        ptx::fence_mbar_init();
        for (int i = 0; i < stages && r0 + i < r1; ++i) issue(r0 + i, i);
    }
    float4 acc[NV], g[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        const int c = (j * kRowThreads + threadIdx.x) * 4;
        g[j] = c < H ? *reinterpret_cast<const float4*>(gain + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    int st = 0;
    uint32_t ph = 0;
    float r_next = r0 < r1 ? rstd[r0] : 0.f;   // one row ahead: its load latency is not on the row's path
    for (int row = r0; row < r1; ++row) {
        const float r = r_next;
        if (row + 1 < r1) r_next = rstd[row + 1];
        ptx::mbar_wait(&bar[st], ph);
        const uint8_t* b = rsm + st * stage_bytes;
        const bf16* sdy = reinterpret_cast<const bf16*>(b);
        const float* sx = reinterpret_cast<const float*>(b + H * 2);
        const float* sr = reinterpret_cast<const float*>(b + H * 6);
        float4 xv[NV], gv[NV], rv[NV];
        float dot = 0.f;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const int c = (j * kRowThreads + threadIdx.x) * 4;
            if (c < H) {
                const float4 d = ld_bf16x4(sdy + c);
                xv[j] = *reinterpret_cast<const float4*>(sx + c);
                rv[j] = dres != nullptr ? *reinterpret_cast<const float4*>(sr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
                gv[j] = make_float4(d.x * g[j].x, d.y * g[j].y, d.z * g[j].z, d.w * g[j].w);
                dot += gv[j].x * xv[j].x + gv[j].y * xv[j].y + gv[j].z * xv[j].z + gv[j].w * xv[j].w;
                acc[j].x += d.x * xv[j].x * r;
                acc[j].y += d.y * xv[j].y * r;
                acc[j].z += d.z * xv[j].z * r;
                acc[j].w += d.w * xv[j].w * r;
            }
        }
        dot = block_sum(dot, red);   // its barriers also mean every thread is done with stage st
        if (threadIdx.x == 0 && row + stages < r1) issue(row + stages, st);
        const float k3 = r * r * r / (float)H * dot;
        const size_t o = (size_t)row * H;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const int c = (j * kRowThreads + threadIdx.x) * 4;
            if (c < H) {
                float4 v = make_float4(r * gv[j].x - k3 * xv[j].x, r * gv[j].y - k3 * xv[j].y,
                                       r * gv[j].z - k3 * xv[j].z, r * gv[j].w - k3 * xv[j].w);
                v.x += rv[j].x; v.y += rv[j].y; v.z += rv[j].z; v.w += rv[j].w;
                if (dx != nullptr) *reinterpret_cast<float4*>(dx + o + c) = v;
                if (dx_bf16 != nullptr) st_bf16x4(dx_bf16 + o + c, v);
            }
        }
        if (++st == stages) { st = 0; ph ^= 1; }
    }
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = (j * kRowThreads + threadIdx.x) * 4;
        if (c < H) *reinterpret_cast<float4*>(dgain_part + (size_t)blockIdx.x * H + c) = acc[j];
    }
}

// Column sums of part[nrows, H] in a fixed order: a block owns 32 columns;
// its 8 row lanes sum rows y, y+8, ... (coalesced 128-byte rows), then lane 0
// adds the 8 partials in order.
constexpr int kRedCols = 32, kRedLanes = 8;

__global__ void __launch_bounds__(kRedCols * kRedLanes) reduce_rows_kernel(const float* __restrict__ part, int nrows,
                                                                           int H, float* __restrict__ out) {
    __shared__ float sm[kRedLanes][kRedCols];
    const int cx = threadIdx.x % kRedCols, y = threadIdx.x / kRedCols;
    const int c = blockIdx.x * kRedCols + cx;
    float s = 0.f;
    if (c < H)
        for (int i = y; i < nrows; i += kRedLanes) s += part[(size_t)i * H + c];
    sm[y][cx] = s;
    __syncthreads();
    if (y == 0 && c < H) {
        float t = sm[0][cx];
#pragma unroll
        for (int k = 1; k < kRedLanes; ++k) t += sm[k][cx];
        out[c] = t;
    }
}

// ---------------------------------------------------------------------------
// Embedding (tensor.py:324-337): gather rows; the backward scatter-add runs
// per distinct token id over a stable (host-sorted) token order, so each
// table row's gradient is the token-order sum np.add.at produces, without
// float atomics.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kRowThreads) embedding_fwd_kernel(const float* __restrict__ table,
                                                                    const int64_t* __restrict__ ids, int H, int V,
                                                                    float* __restrict__ out, int* __restrict__ err) {
    const size_t t = blockIdx.x;
    const int64_t id = ids[t];
    if (id < 0 || id >= V) {
        if (threadIdx.x == 0) atomicExch(err, 1);
        return;
    }
    const float* src = table + (size_t)id * H;
    for (int c = threadIdx.x * 4; c < H; c += kRowThreads * 4)
        *reinterpret_cast<float4*>(out + t * H + c) = *reinterpret_cast<const float4*>(src + c);
}

__global__ void __launch_bounds__(kRowThreads) embedding_bwd_kernel(const float* __restrict__ g,
                                                                    const int* __restrict__ order,
                                                                    const int* __restrict__ seg_start,
                                                                    const int* __restrict__ seg_id, int H,
                                                                    float* __restrict__ grad) {
    const int s = blockIdx.x;
    const int i0 = seg_start[s], i1 = seg_start[s + 1];
    float* dst = grad + (size_t)seg_id[s] * H;
    for (int c = threadIdx.x * 4; c < H; c += kRowThreads * 4) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int i = i0; i < i1; ++i) {
            const float4 v = *reinterpret_cast<const float4*>(g + (size_t)order[i] * H + c);
            a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
        }
        *reinterpret_cast<float4*>(dst + c) = a;
    }
}

// Same scatter-add from a device-sorted token order, no host round trip:
// position i starts a segment iff sid[i] != sid[i-1]; that block sums the
// segment's rows in order.  Used by the data-parallel embedding backward over
// the all-gathered tokens of every rank.
__global__ void __launch_bounds__(kRowThreads) embedding_bwd_sorted_kernel(const float* __restrict__ g,
                                                                           const int64_t* __restrict__ order,
                                                                           const int64_t* __restrict__ sid, int n,
                                                                           int H, float* __restrict__ grad) {
    const int i0 = blockIdx.x;
    const int64_t id = sid[i0];
    if (i0 > 0 && sid[i0 - 1] == id) return;
    int i1 = i0 + 1;
    while (i1 < n && sid[i1] == id) ++i1;
    float* dst = grad + (size_t)id * H;
    for (int c = threadIdx.x * 4; c < H; c += kRowThreads * 4) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int i = i0; i < i1; ++i) {
            const float4 v = *reinterpret_cast<const float4*>(g + (size_t)order[i] * H + c);
            a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
        }
        *reinterpret_cast<float4*>(dst + c) = a;
    }
}

// ---------------------------------------------------------------------------
// Cross entropy (tensor.py:340-364): per row m = max, z = sum exp(x - m),
// lse = log z + m, nll = lse - x[target]; loss = mean nll, evaluated as
// (m - x_t) + log1p(z - 1) so near-zero losses are not rounded to 0.
// Backward writes (softmax - onehot) * dloss / T in bf16.  One block per row;
// two passes over the row (the second hits L2).
// ---------------------------------------------------------------------------
// 2^x on the SFU (ex2.approx: ~2 ulp; -inf -> 0, +inf -> +inf; results below 2^-126 flush to 0)
__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));   // .ftz: one MUFU.EX2, no denormal fix-up
    return y;
}

__device__ __forceinline__ void load8(const bf16* p, float* f) { unpack8(*reinterpret_cast<const uint4*>(p), f); }

__global__ void __launch_bounds__(kRowThreads) ce_fwd_kernel(const bf16* __restrict__ logits,
                                                             const int64_t* __restrict__ targets, int V,
                                                             float* __restrict__ nll, float* __restrict__ lse,
                                                             int* __restrict__ err) {
    __shared__ float red[33];
    const size_t row = blockIdx.x;
    const bf16* xr = logits + row * V;
    const bool vec = (V & 7) == 0;
    // One pass (the row is read once): each thread keeps a running maximum m
    // and s = sum of exp(f - m) over its elements except one occurrence of m,
    // rescaled when the maximum moves.  The block then forms
    //   z - 1 = sum_t s_t * [m_t == M] + (s_t + 1) e^{m_t - M} * [m_t < M] + (holders - 1)
    // (holders: threads whose maximum is the row maximum M), which keeps the
    // max's exact 1.0 apart so confident rows keep their tiny loss:
    // nll = (M - x_t) + log1p(z - 1).
    float m = -INFINITY, sacc = 0.f;
    auto upd = [&](float f) {
        if (f > m) {
            sacc = (sacc + 1.f) * expf(m - f);   // the old maximum now counts; first element: 0
            m = f;
        } else if (f > -INFINITY || f != f) {   // -inf contributes 0; NaN propagates
            sacc += expf(f - m);
        }
    };
    if (vec) {
        // 8 logits per step: one max-compare for the group, then exp2 (MUFU) of
        // each (f - m) * log2(e); the group's first maximum is left out when it
        // becomes the running maximum.  ~5 instructions per logit instead of
        // ~20 (the kernel was issue-bound at ~0.45 of HBM with expf per element).
        constexpr float kL2e = 1.4426950408889634f;
        constexpr int kU = 4;   // 16-byte loads in flight per thread
        for (int c0 = threadIdx.x * 8; c0 < V; c0 += kU * kRowThreads * 8) {
          uint4 raw[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
              const int c = c0 + u * kRowThreads * 8;
              raw[u] = c < V ? *reinterpret_cast<const uint4*>(xr + c) : make_uint4(0xFF80FF80u, 0xFF80FF80u,
                                                                                     0xFF80FF80u, 0xFF80FF80u);
          }
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            float f[8];
            unpack8(raw[u], f);   // past the row end: bf16 -inf, contributes nothing
            float m8 = f[0];
#pragma unroll
            for (int i = 1; i < 8; ++i) m8 = fmaxf(m8, f[i]);
            // NaN logits propagate through ex2 into the sum; fmaxf skips them, so
            // only an all-NaN group seen before any other logit needs a case
            if (m8 > m) {
                const float mb = m8 * kL2e;
                float t = (m > -INFINITY) ? (sacc + 1.f) * ex2f(fmaf(m, kL2e, -mb)) : sacc;   // 0 or NaN
                bool skipped = false;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const bool skip = !skipped && f[i] == m8;
                    skipped |= skip;
                    t += skip ? 0.f : ex2f(fmaf(f[i], kL2e, -mb));
                }
                sacc = t;
                m = m8;
            } else if (m > -INFINITY) {
                const float mb = m * kL2e;
#pragma unroll
                for (int i = 0; i < 8; ++i) sacc += ex2f(fmaf(f[i], kL2e, -mb));
            } else if (m8 != m8) {
                sacc = m8;
            }
          }
        }
    } else {
        for (int c = threadIdx.x; c < V; c += kRowThreads) upd(bf2f(xr[c]));
    }
    const float mrow = block_max(m, red);
    const bool holder = (m == mrow) && m > -INFINITY;
    float z1 = block_sum(holder ? sacc : (m > -INFINITY ? (sacc + 1.f) * expf(m - mrow) : 0.f), red);
    const float holders = block_sum(holder ? 1.f : 0.f, red);
    z1 += holders - 1.f;
    m = mrow;
    if (threadIdx.x == 0) {
        const int64_t t = targets[row];
        const float lp = log1pf(z1);
        lse[row] = m + lp;
        if (t < 0 || t >= V) {
            atomicExch(err, 1);
            nll[row] = 0.f;
        } else {
            nll[row] = (m - bf2f(xr[t])) + lp;
        }
    }
}

__global__ void __launch_bounds__(1024) mean_kernel(const float* __restrict__ v, int n, float* __restrict__ out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) out[0] = (float)(s / n);
    }
}

__global__ void __launch_bounds__(kRowThreads) ce_bwd_kernel(const bf16* __restrict__ logits,
                                                             const int64_t* __restrict__ targets,
                                                             const float* __restrict__ lse,
                                                             const float* __restrict__ dloss, int T, int V,
                                                             bf16* __restrict__ dlogits) {
    const size_t row = blockIdx.x;
    const bf16* xr = logits + row * V;
    bf16* dr = dlogits + row * V;
    const float l = lse[row];
    const float scale = dloss[0] / (float)T;
    const int64_t t = targets[row];
    if ((V & 7) == 0) {
        for (int c = threadIdx.x * 8; c < V; c += kRowThreads * 8) {
            float f[8];
            load8(xr + c, f);
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = (expf(f[i] - l) - (c + i == t ? 1.f : 0.f)) * scale;
            *reinterpret_cast<uint4*>(dr + c) = pack8(f);
        }
    } else {
        for (int c = threadIdx.x; c < V; c += kRowThreads)
            dr[c] = __float2bfloat16_rn((expf(bf2f(xr[c]) - l) - (c == t ? 1.f : 0.f)) * scale);
    }
}

// ---------------------------------------------------------------------------
// Optimizer step over a list of tensors (train.py:146-179), one launch for
// the whole model.  Adam follows numpy's float32 evaluation order exactly:
//   m = m*b1 + (1-b1)*g;  v = v*b2 + ((1-b2)*g)*g
//   p = p - (lr * (m/bc1)) / (sqrt(v/bc2) + eps)
// with every constant rounded to float32 and no contraction into FMA, so a
// step is bit-identical to the reference's on the same gradients.  The bf16
// compute copy (`shadow`) is refreshed in the same pass.
// ---------------------------------------------------------------------------
constexpr int kOptChunk = 8192;

template <typename G>
__device__ __forceinline__ float load_g(const void* g, long long i) {
    if constexpr (sizeof(G) == 4) return reinterpret_cast<const float*>(g)[i];
    else return __bfloat162float(reinterpret_cast<const bf16*>(g)[i]);
}

struct OptScalars {
    float lr, b1, c1, b2, c2, eps, bc1, bc2, momentum;
};

__device__ __forceinline__ float adam_elem(float& p, float& m, float& v, float g, const OptScalars& s) {
    m = __fadd_rn(__fmul_rn(m, s.b1), __fmul_rn(s.c1, g));
    v = __fadd_rn(__fmul_rn(v, s.b2), __fmul_rn(__fmul_rn(s.c2, g), g));
    const float mh = __fdiv_rn(m, s.bc1);
    const float vh = __fdiv_rn(v, s.bc2);
    p = __fsub_rn(p, __fdiv_rn(__fmul_rn(s.lr, mh), __fadd_rn(__fsqrt_rn(vh), s.eps)));
    return p;
}

__device__ __forceinline__ float sgd_elem(float& p, float& buf, float g, const OptScalars& s) {
    buf = __fadd_rn(__fmul_rn(buf, s.momentum), g);
    p = __fsub_rn(p, __fmul_rn(s.lr, buf));
    return p;
}

// 4 consecutive elements per thread: 16-byte loads, the update, 16-byte stores
// (a 2-group unroll measured slower: 25-27 ms vs 22.4 ms for 3.95 B params).
struct OptVec {
    float g[4];
    float4 p, m, v;
};

template <int kKind>
__device__ __forceinline__ void opt_load4(const b200moe_opt_tensor& d, long long i, OptVec& o) {
    if (d.grad_bf16) {
        const float4 t = ld_bf16x4(reinterpret_cast<const bf16*>(d.grad) + i);
        o.g[0] = t.x; o.g[1] = t.y; o.g[2] = t.z; o.g[3] = t.w;
    } else {
        const float4 t = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(d.grad) + i);
        o.g[0] = t.x; o.g[1] = t.y; o.g[2] = t.z; o.g[3] = t.w;
    }
    o.p = *reinterpret_cast<const float4*>(d.param + i);
    o.m = *reinterpret_cast<const float4*>(d.m + i);
    if constexpr (kKind == B200MOE_OPT_ADAM) o.v = *reinterpret_cast<const float4*>(d.v + i);
}

template <int kKind>
__device__ __forceinline__ void opt_store4(const b200moe_opt_tensor& d, long long i, OptVec& o, const OptScalars& s) {
    float* pp = &o.p.x;
    float* mp = &o.m.x;
    if constexpr (kKind == B200MOE_OPT_ADAM) {
        float* vp = &o.v.x;
#pragma unroll
        for (int j = 0; j < 4; ++j) adam_elem(pp[j], mp[j], vp[j], o.g[j], s);
        *reinterpret_cast<float4*>(d.v + i) = o.v;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) sgd_elem(pp[j], mp[j], o.g[j], s);
    }
    *reinterpret_cast<float4*>(d.m + i) = o.m;
    *reinterpret_cast<float4*>(d.param + i) = o.p;
    if (d.shadow != nullptr) st_bf16x4(reinterpret_cast<bf16*>(d.shadow) + i, o.p);
}

template <int kKind>
// 6 resident blocks per SM (40 registers): the loads are latency-bound, so
// occupancy is in-flight bytes -- 0.89 of HBM vs 0.74 at the default 58
// registers (tools/opt_bench.py, 2 B parameters); 8 blocks spill.
__global__ void __launch_bounds__(256, 6) optimizer_kernel(const b200moe_opt_tensor* __restrict__ list,
                                                        const int* __restrict__ chunk_tensor,
                                                        const long long* __restrict__ chunk_off, int n_chunks,
                                                        OptScalars s) {
    for (int ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
        const b200moe_opt_tensor d = list[chunk_tensor[ch]];
        const long long i0 = chunk_off[ch];
        const long long i1 = min(d.n, i0 + (long long)kOptChunk);
        // Vector body: 4 elements per thread (all buffers are 16-byte aligned
        // torch allocations and chunks start at multiples of kOptChunk).
        const long long iv = i0 + ((i1 - i0) & ~3LL);
        for (long long i = i0 + 4 * threadIdx.x; i < iv; i += 4 * blockDim.x) {
            OptVec a;
            opt_load4<kKind>(d, i, a);
            opt_store4<kKind>(d, i, a, s);
        }
        for (long long i = iv + threadIdx.x; i < i1; i += blockDim.x) {
            const float g = d.grad_bf16 ? load_g<bf16>(d.grad, i) : load_g<float>(d.grad, i);
            float p = d.param[i];
            if constexpr (kKind == B200MOE_OPT_ADAM) {
                adam_elem(p, d.m[i], d.v[i], g, s);
            } else {
                sgd_elem(p, d.m[i], g, s);
            }
            d.param[i] = p;
            if (d.shadow != nullptr) reinterpret_cast<bf16*>(d.shadow)[i] = __float2bfloat16_rn(p);
        }
    }
}

}  // namespace b200moe

using namespace b200moe;

extern "C" {

int b200moe_rmsnorm_fwd(const float* x, const void* delta, const float* gain, int T, int H, float eps, float* x_out,
                        void* y, float* rstd, cudaStream_t stream) {
    B200_CHECK_ARG(T >= 0 && H >= 4 && H % 4 == 0, B200MOE_ERR_SHAPE, "rmsnorm: hidden %d must be a multiple of 4", H);
    B200_CHECK_ARG(delta == nullptr || x_out != nullptr, B200MOE_ERR_CONFIG, "rmsnorm: residual add needs x_out");
    if (T == 0) return B200MOE_OK;
    rmsnorm_fwd_kernel<<<T, kRowThreads, 0, stream>>>(x, (const bf16*)delta, gain, H, eps, x_out, (bf16*)y, rstd);
    B200_CHECK_LAUNCH("rmsnorm_fwd");
    return B200MOE_OK;
}

int b200moe_rmsnorm_bwd(const void* dy, const float* x, const float* rstd, const float* gain, const float* dres, int T,
                        int H, float* dx, void* dx_bf16, float* dgain, float* workspace, cudaStream_t stream) {
    B200_CHECK_ARG(T >= 1 && H >= 4 && H % 4 == 0 && H <= 16 * 1024, B200MOE_ERR_SHAPE,
                   "rmsnorm_bwd: hidden %d must be a multiple of 4 and <= 16384", H);
    const int nv = ceil_div(H, kRowThreads * 4);
    const size_t stage_bytes = (size_t)H * (2 + 4 + (dres != nullptr ? 4 : 0));
    const int stages = (int)(kRmsSmemMax / stage_bytes) < kRmsStages ? (int)(kRmsSmemMax / stage_bytes) : kRmsStages;
    const bool aligned = ((reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(x) |
                           reinterpret_cast<uintptr_t>(dres)) & 15) == 0;   // bulk copies need 16-byte addresses
    // the register kernel's vector accesses: 8-byte bf16 quads, 16-byte fp32 quads
    B200_CHECK_ARG(((reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(dx_bf16)) & 7) == 0 &&
                       ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dres) |
                         reinterpret_cast<uintptr_t>(dx)) & 15) == 0,
                   B200MOE_ERR_SHAPE, "rmsnorm_bwd: misaligned buffer (bf16 rows need 8, fp32 rows 16 bytes)");
    if (H % 8 == 0 && nv <= 4 && stages >= 2 && aligned) {
        // one wave: rows split evenly over the SMs, at least kBwdRows per block (workspace contract)
        const int rpb = max(kBwdRows, ceil_div(T, kNumSMs));
        const int nbr = ceil_div(T, rpb);
        const size_t smem = stages * stage_bytes;
#define B200_RMS_RING(NV)                                                                                         \
    do {                                                                                                          \
        auto kern = rmsnorm_bwd_ring_kernel<NV>;                                                                  \
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kRmsSmemMax);                     \
        kern<<<nbr, kRowThreads, smem, stream>>>((const bf16*)dy, x, rstd, gain, dres, T, H, rpb, stages, dx,     \
                                                 (bf16*)dx_bf16, workspace);                                      \
    } while (0)
        if (nv <= 1) B200_RMS_RING(1);
        else if (nv <= 2) B200_RMS_RING(2);
        else B200_RMS_RING(4);
#undef B200_RMS_RING
        reduce_rows_kernel<<<ceil_div(H, kRedCols), kRedCols * kRedLanes, 0, stream>>>(workspace, nbr, H, dgain);
        B200_CHECK_LAUNCH("rmsnorm_bwd");
        return B200MOE_OK;
    }
    const int nb = ceil_div(T, kBwdRows);
#define B200_RMS_BWD(NV)                                                                                         \
    rmsnorm_bwd_kernel<NV><<<nb, kRowThreads, 0, stream>>>((const bf16*)dy, x, rstd, gain, dres, T, H, dx,       \
                                                           (bf16*)dx_bf16, workspace)
    if (nv <= 1) B200_RMS_BWD(1);
    else if (nv <= 2) B200_RMS_BWD(2);
    else if (nv <= 4) B200_RMS_BWD(4);
    else if (nv <= 8) B200_RMS_BWD(8);
    else B200_RMS_BWD(16);
#undef B200_RMS_BWD
    reduce_rows_kernel<<<ceil_div(H, kRedCols), kRedCols * kRedLanes, 0, stream>>>(workspace, nb, H, dgain);
    B200_CHECK_LAUNCH("rmsnorm_bwd");
    return B200MOE_OK;
}

int b200moe_embedding_fwd(const float* table, const int64_t* ids, int T, int H, int V, float* out, int* err_flag,
                          cudaStream_t stream) {
    B200_CHECK_ARG(H >= 4 && H % 4 == 0 && V >= 1, B200MOE_ERR_SHAPE, "embedding: bad table [%d, %d]", V, H);
    if (T == 0) return B200MOE_OK;
    embedding_fwd_kernel<<<T, kRowThreads, 0, stream>>>(table, ids, H, V, out, err_flag);
    B200_CHECK_LAUNCH("embedding_fwd");
    return B200MOE_OK;
}

int b200moe_embedding_bwd(const float* g, const int* order, const int* seg_start, const int* seg_id, int n_seg, int H,
                          float* grad, cudaStream_t stream) {
    B200_CHECK_ARG(H >= 4 && H % 4 == 0, B200MOE_ERR_SHAPE, "embedding_bwd: hidden %d must be a multiple of 4", H);
    if (n_seg == 0) return B200MOE_OK;
    embedding_bwd_kernel<<<n_seg, kRowThreads, 0, stream>>>(g, order, seg_start, seg_id, H, grad);
    B200_CHECK_LAUNCH("embedding_bwd");
    return B200MOE_OK;
}

int b200moe_embedding_bwd_sorted(const float* g, const int64_t* order, const int64_t* sorted_ids, int n, int H,
                                 float* grad, cudaStream_t stream) {
    B200_CHECK_ARG(H >= 4 && H % 4 == 0, B200MOE_ERR_SHAPE, "embedding_bwd: hidden %d must be a multiple of 4", H);
    if (n == 0) return B200MOE_OK;
    embedding_bwd_sorted_kernel<<<n, kRowThreads, 0, stream>>>(g, order, sorted_ids, n, H, grad);
    B200_CHECK_LAUNCH("embedding_bwd_sorted");
    return B200MOE_OK;
}

int b200moe_cross_entropy_fwd(const void* logits, const int64_t* targets, int T, int V, float* nll, float* lse,
                              float* loss, int* err_flag, cudaStream_t stream) {
    B200_CHECK_ARG(T >= 1 && V >= 1, B200MOE_ERR_SHAPE, "cross_entropy: bad logits [%d, %d]", T, V);
    ce_fwd_kernel<<<T, kRowThreads, 0, stream>>>((const bf16*)logits, targets, V, nll, lse, err_flag);
    mean_kernel<<<1, 1024, 0, stream>>>(nll, T, loss);
    B200_CHECK_LAUNCH("cross_entropy_fwd");
    return B200MOE_OK;
}

int b200moe_cross_entropy_bwd(const void* logits, const int64_t* targets, const float* lse, const float* dloss, int T,
                              int V, void* dlogits, cudaStream_t stream) {
    B200_CHECK_ARG(T >= 1 && V >= 1, B200MOE_ERR_SHAPE, "cross_entropy_bwd: bad logits [%d, %d]", T, V);
    ce_bwd_kernel<<<T, kRowThreads, 0, stream>>>((const bf16*)logits, targets, lse, dloss, T, V, (bf16*)dlogits);
    B200_CHECK_LAUNCH("cross_entropy_bwd");
    return B200MOE_OK;
}

int b200moe_optimizer_chunk(void) { return kOptChunk; }

int b200moe_optimizer_step(const b200moe_opt_tensor* tensors, const int* chunk_tensor, const long long* chunk_off,
                           int n_chunks, int kind, float lr, float beta1, float one_minus_beta1, float beta2,
                           float one_minus_beta2, float eps, float bias_corr1, float bias_corr2, float momentum,
                           cudaStream_t stream) {
    B200_CHECK_ARG(kind == B200MOE_OPT_ADAM || kind == B200MOE_OPT_SGD, B200MOE_ERR_CONFIG,
                   "optimizer kind %d unknown", kind);
    if (n_chunks == 0) return B200MOE_OK;
    const int grid = n_chunks < kNumSMs * 16 ? n_chunks : kNumSMs * 16;
    const OptScalars s{lr, beta1, one_minus_beta1, beta2, one_minus_beta2, eps, bias_corr1, bias_corr2, momentum};
    if (kind == B200MOE_OPT_ADAM)
        optimizer_kernel<B200MOE_OPT_ADAM><<<grid, 256, 0, stream>>>(tensors, chunk_tensor, chunk_off, n_chunks, s);
    else
        optimizer_kernel<B200MOE_OPT_SGD><<<grid, 256, 0, stream>>>(tensors, chunk_tensor, chunk_off, n_chunks, s);
    B200_CHECK_LAUNCH("optimizer_step");
    return B200MOE_OK;
}

}  // extern "C"
