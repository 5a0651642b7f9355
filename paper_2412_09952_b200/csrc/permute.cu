// Token permute (K2), weighted combine (K5) and combine backward (K6), local
// or fused with the expert-parallel exchange over NVLink peer memory.
//
// Reference: moefold/moe.py:272-282 (per expert: take_rows, ffn, multiply by the
// gate column, put_rows, add in expert order) and the backward closures
// tensor.py:185 (mul), :389 (put_rows), :375 (take_rows).  Every kernel is a
// warp per token with 128-bit loads/stores; the per-token sum over its kept
// experts runs in ascending expert order (deterministic, no atomics).
//
// Row addressing: expert e's rows live in buffer bufs[e / e_per_rank] at row
// seg_base[e] + slot_rank[t, e].  Single GPU: one local buffer.  Expert
// parallel (kPeer): bufs[d] is rank d's symmetric-memory buffer mapped into this
// process, so the permute writes each token straight into its expert owner's
// receive buffer and the combine reads expert outputs straight from the owner:
// the all-to-all happens inside these kernels, overlapped with their own
// loads and arithmetic, with no staging copies.
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "common.cuh"

namespace b200moe {

constexpr int kPermThreads = 256;  // 8 warps
#ifndef B200_COMBINE_MINB
#define B200_COMBINE_MINB 1   // min resident blocks per SM for combine / combine-backward (A/B knob)
#endif
constexpr int kVecPerLane = 8;     // uint4 per lane per pass (4 KB per warp pass)

struct Rows {
    __nv_bfloat16* local;   // single-GPU buffer (or nullptr)
    const uint64_t* bufs;   // per-rank buffer bases (device array) when kPeer
    int e_per_rank;

    template <bool kPeer>
    __device__ __forceinline__ __nv_bfloat16* base(int e) const {
        if constexpr (kPeer) return reinterpret_cast<__nv_bfloat16*>(bufs[e / e_per_rank]);
        else return local;
    }
};

// Kept experts of token t (ascending) -> rows; returns the count.
__device__ __forceinline__ int token_rows(const int32_t* __restrict__ slot_rank, const int32_t* __restrict__ seg_base,
                                          int t, int E, int* rows, int* experts) {
    const int lane = threadIdx.x & 31;
    int r = -1;
    if (lane < E) {
        const int rk = slot_rank[(size_t)t * E + lane];
        if (rk >= 0) r = seg_base[lane] + rk;
    }
    const unsigned m = __ballot_sync(0xffffffffu, r >= 0);
    int n = 0;
    unsigned mm = m;
    while (mm) {
        const int e = __ffs(mm) - 1;
        mm &= mm - 1;
        rows[n] = __shfl_sync(0xffffffffu, r, e);
        experts[n] = e;
        ++n;
    }
    return n;
}

// Zero rows [seg_base[e]+counts[e], seg_base[e]+round_up(counts[e],128)) of buf
// (up to 127 rows = 1 MB at H=4096, over NVLink in the expert-parallel
// kernels): kPadParts blocks per expert, each a slice.  The pad blocks are the
// grid's FIRST blocks, so they run alongside the token blocks instead of
// forming a tail of E single blocks after them.
constexpr int kPadParts = 4;
__device__ __forceinline__ void zero_pad_rows(__nv_bfloat16* buf, const int32_t* seg_base, const int32_t* counts,
                                              int e, int part, int H) {
    const int c = counts[e];
    const size_t r0 = (size_t)seg_base[e] + c;
    const size_t r1 = (size_t)seg_base[e] + round_up(c, kSegPad);
    const size_t nvec = (r1 - r0) * (H / 8);
    uint4* p = reinterpret_cast<uint4*>(buf + r0 * H);
    const uint4 zero = make_uint4(0, 0, 0, 0);
    for (size_t i = threadIdx.x + (size_t)part * blockDim.x; i < nvec; i += (size_t)kPadParts * blockDim.x) p[i] = zero;
}

template <bool kPeer>
__global__ void __launch_bounds__(kPermThreads)
permute_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ slot_rank,
               const int32_t* __restrict__ seg_base, const int32_t* __restrict__ counts, int T, int H, int E,
               int token_blocks, Rows out, const uint64_t* __restrict__ count_bufs, int rank) {
    if ((int)blockIdx.x < E * kPadParts) {
        const int e = blockIdx.x / kPadParts, part = blockIdx.x % kPadParts;
        zero_pad_rows(out.base<kPeer>(e), seg_base, counts, e, part, H);
        if (kPeer && part == 0 && threadIdx.x == 0) {  // publish this rank's count into the owner's receive table
            const int el = e % out.e_per_rank;
            reinterpret_cast<int32_t*>(count_bufs[e / out.e_per_rank])[rank * out.e_per_rank + el] = counts[e];
        }
        return;
    }
    const int lane = threadIdx.x & 31;
    const int t = ((int)blockIdx.x - E * kPadParts) * (kPermThreads / 32) + (threadIdx.x >> 5);
    if (t >= T) return;
    int rows[32], experts[32];
    const int n = token_rows(slot_rank, seg_base, t, E, rows, experts);
    if (n == 0) return;
    const int nvec = H / 8;
    const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)t * H);
    for (int base = 0; base < nvec; base += 32 * kVecPerLane) {
        uint4 v[kVecPerLane];
#pragma unroll
        for (int i = 0; i < kVecPerLane; ++i) {
            const int j = base + i * 32 + lane;
            if (j < nvec) v[i] = ld_nc_v4(src + j);
        }
        for (int r = 0; r < n; ++r) {
            uint4* dst = reinterpret_cast<uint4*>(out.base<kPeer>(experts[r]) + (size_t)rows[r] * H);
#pragma unroll
            for (int i = 0; i < kVecPerLane; ++i) {
                const int j = base + i * 32 + lane;
                if (j < nvec) dst[j] = v[i];
            }
        }
    }
}

// og (optional): the gathered expert rows, og[(t * og_k + j) * H] = token t's
// j-th kept row (ascending expert), written while they pass through registers
// so that the backward reads them locally instead of over NVLink again.
template <bool kPeer>
__global__ void __launch_bounds__(kPermThreads, B200_COMBINE_MINB)
combine_kernel(Rows o, const float* __restrict__ gates, const int32_t* __restrict__ slot_rank,
               const int32_t* __restrict__ seg_base, int T, int H, int E, __nv_bfloat16* __restrict__ y,
               __nv_bfloat16* __restrict__ og, int og_k) {
    const int lane = threadIdx.x & 31;
    const int t = blockIdx.x * (kPermThreads / 32) + (threadIdx.x >> 5);
    if (t >= T) return;
    int rows[32], experts[32];
    const int n = token_rows(slot_rank, seg_base, t, E, rows, experts);
    float g[32];
    for (int r = 0; r < n; ++r) g[r] = gates[(size_t)t * E + experts[r]];
    const int nvec = H / 8;
    uint4* dst = reinterpret_cast<uint4*>(y + (size_t)t * H);
    if (n <= 1) {   // zero or one kept slot: y = 0 or g * o, the row's loads all in flight
        const uint4* s0 = n ? reinterpret_cast<const uint4*>(o.base<kPeer>(experts[0]) + (size_t)rows[0] * H) : nullptr;
        uint4* m0 = (og && n) ? reinterpret_cast<uint4*>(og + (size_t)t * og_k * H) : nullptr;
        const float g0 = n ? g[0] : 0.f;
        for (int base = 0; base < nvec; base += 32 * 8) {
            uint4 v0[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int j = base + i * 32 + lane;
                v0[i] = make_uint4(0, 0, 0, 0);
                if (n && j < nvec) v0[i] = kPeer ? s0[j] : ld_nc_v4(s0 + j);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int j = base + i * 32 + lane;
                if (j < nvec) {
                    if (m0) m0[j] = v0[i];
                    float f0[8], a[8];
                    unpack8(v0[i], f0);
#pragma unroll
                    for (int c = 0; c < 8; ++c) a[c] = n ? fmaf(g0, f0[c], 0.f) : 0.f;
                    dst[j] = pack8(a);
                }
            }
        }
        return;
    }
    if (n == 2) {
        // top-2 tokens (the common case): both expert rows' loads are issued
        // before any arithmetic, 8 x 16 B in flight per lane -- over NVLink the
        // latency-bound single-row loop reached only ~0.6 of the link
        const uint4* s0 = reinterpret_cast<const uint4*>(o.base<kPeer>(experts[0]) + (size_t)rows[0] * H);
        const uint4* s1 = reinterpret_cast<const uint4*>(o.base<kPeer>(experts[1]) + (size_t)rows[1] * H);
        uint4* m0 = og ? reinterpret_cast<uint4*>(og + (size_t)t * og_k * H) : nullptr;
        uint4* m1 = og ? m0 + nvec : nullptr;
        const float g0 = g[0], g1 = g[1];
        for (int base = 0; base < nvec; base += 32 * 4) {
            uint4 v0[4], v1[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = base + i * 32 + lane;
                if (j < nvec) {
                    v0[i] = kPeer ? s0[j] : ld_nc_v4(s0 + j);
                    v1[i] = kPeer ? s1[j] : ld_nc_v4(s1 + j);
                }
            }
            if (m0) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int j = base + i * 32 + lane;
                    if (j < nvec) {
                        m0[j] = v0[i];
                        m1[j] = v1[i];
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = base + i * 32 + lane;
                if (j < nvec) {
                    float f0[8], f1[8], a[8];
                    unpack8(v0[i], f0);
                    unpack8(v1[i], f1);
#pragma unroll
                    for (int c = 0; c < 8; ++c) a[c] = fmaf(g1, f1[c], fmaf(g0, f0[c], 0.f));
                    dst[j] = pack8(a);
                }
            }
        }
        return;
    }
    for (int base = 0; base < nvec; base += 32 * 4) {
        float acc[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[i][c] = 0.f;
        for (int r = 0; r < n; ++r) {
            const uint4* src = reinterpret_cast<const uint4*>(o.base<kPeer>(experts[r]) + (size_t)rows[r] * H);
            uint4 v[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = base + i * 32 + lane;
                if (j < nvec) v[i] = kPeer ? src[j] : ld_nc_v4(src + j);
            }
            if (og) {
                uint4* m = reinterpret_cast<uint4*>(og + ((size_t)t * og_k + r) * H);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int j = base + i * 32 + lane;
                    if (j < nvec) m[j] = v[i];
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                float f[8];
                unpack8(v[i], f);
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[i][c] = fmaf(g[r], f[c], acc[i][c]);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int j = base + i * 32 + lane;
            if (j < nvec) dst[j] = pack8(acc[i]);
        }
    }
}

// og (optional): the forward's gathered rows (combine_kernel): read locally
// instead of from the owners' buffers.
template <bool kPeer>
__global__ void __launch_bounds__(kPermThreads, B200_COMBINE_MINB)
combine_bwd_kernel(const __nv_bfloat16* __restrict__ dy, Rows o, const float* __restrict__ gates,
                   const int32_t* __restrict__ slot_rank, const int32_t* __restrict__ seg_base,
                   const int32_t* __restrict__ counts, int T, int H, int E, int token_blocks, Rows dout,
                   float* __restrict__ dg, const __nv_bfloat16* __restrict__ og, int og_k) {
    if ((int)blockIdx.x < E * kPadParts) {
        const int e = blockIdx.x / kPadParts;
        zero_pad_rows(dout.base<kPeer>(e), seg_base, counts, e, blockIdx.x % kPadParts, H);
        return;
    }
    const int lane = threadIdx.x & 31;
    const int t = ((int)blockIdx.x - E * kPadParts) * (kPermThreads / 32) + (threadIdx.x >> 5);
    if (t >= T) return;
    int rows[32], experts[32];
    const int n = token_rows(slot_rank, seg_base, t, E, rows, experts);
    float g[32], dot[32];
    for (int r = 0; r < n; ++r) {
        g[r] = gates[(size_t)t * E + experts[r]];
        dot[r] = 0.f;
    }
    const int nvec = H / 8;
    const uint4* src = reinterpret_cast<const uint4*>(dy + (size_t)t * H);
    if (n <= 1) {
        // a token with no kept slot only zeroes its dg row (its dy is not read);
        // one kept slot: dy and the expert row's loads in flight together
        float* dgt = dg + (size_t)t * E;
        if (lane < E) dgt[lane] = 0.f;
        __syncwarp();
        if (n == 0) return;
        const bool mir = og != nullptr;
        const uint4* os0 = mir ? reinterpret_cast<const uint4*>(og + (size_t)t * og_k * H)
                               : reinterpret_cast<const uint4*>(o.base<kPeer>(experts[0]) + (size_t)rows[0] * H);
        uint4* ds0 = reinterpret_cast<uint4*>(dout.base<kPeer>(experts[0]) + (size_t)rows[0] * H);
        const float g0 = g[0];
        float s0 = 0.f;
        for (int base = 0; base < nvec; base += 32 * 4) {
            uint4 dv[4], v0[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = base + i * 32 + lane;
                if (j < nvec) {
                    dv[i] = ld_nc_v4(src + j);
                    v0[i] = (kPeer && !mir) ? os0[j] : ld_nc_v4(os0 + j);
                }
            }
            float p0 = 0.f;   // the general path's per-chunk fma chain (bit-identical dg)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = base + i * 32 + lane;
                if (j < nvec) {
                    float d[8], f[8], w[8];
                    unpack8(dv[i], d);
                    unpack8(v0[i], f);
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        p0 = fmaf(d[c], f[c], p0);
                        w[c] = g0 * d[c];
                    }
                    ds0[j] = pack8(w);
                }
            }
            s0 += p0;
        }
        const float a0 = warp_sum(s0);
        if (lane == 0) dgt[experts[0]] = a0;
        return;
    }
    if (n == 2) {
        // top-2 tokens: dy and both expert rows' loads in flight together
        // (12 x 16 B per lane) before the dot products and the two stores
        const bool mir = og != nullptr;
        const uint4* os0 = mir ? reinterpret_cast<const uint4*>(og + (size_t)t * og_k * H)
                               : reinterpret_cast<const uint4*>(o.base<kPeer>(experts[0]) + (size_t)rows[0] * H);
        const uint4* os1 = mir ? os0 + nvec
                               : reinterpret_cast<const uint4*>(o.base<kPeer>(experts[1]) + (size_t)rows[1] * H);
        uint4* ds0 = reinterpret_cast<uint4*>(dout.base<kPeer>(experts[0]) + (size_t)rows[0] * H);
        uint4* ds1 = reinterpret_cast<uint4*>(dout.base<kPeer>(experts[1]) + (size_t)rows[1] * H);
        const float g0 = g[0], g1 = g[1];
        float s0 = 0.f, s1 = 0.f;
        for (int base = 0; base < nvec; base += 32 * 4) {
            uint4 dv[4], v0[4], v1[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = base + i * 32 + lane;
                if (j < nvec) {
                    dv[i] = ld_nc_v4(src + j);
                    v0[i] = (kPeer && !mir) ? os0[j] : ld_nc_v4(os0 + j);
                    v1[i] = (kPeer && !mir) ? os1[j] : ld_nc_v4(os1 + j);
                }
            }
            // per-chunk fma chains in the general path's order (bit-identical dg)
            float p0 = 0.f, p1 = 0.f;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = base + i * 32 + lane;
                if (j < nvec) {
                    float d[8], f[8], w[8];
                    unpack8(dv[i], d);
                    unpack8(v0[i], f);
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        p0 = fmaf(d[c], f[c], p0);
                        w[c] = g0 * d[c];
                    }
                    ds0[j] = pack8(w);
                    unpack8(v1[i], f);
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        p1 = fmaf(d[c], f[c], p1);
                        w[c] = g1 * d[c];
                    }
                    ds1[j] = pack8(w);
                }
            }
            s0 += p0;
            s1 += p1;
        }
        float* dgt = dg + (size_t)t * E;
        if (lane < E) dgt[lane] = 0.f;
        __syncwarp();
        const float a0 = warp_sum(s0), a1 = warp_sum(s1);
        if (lane == 0) {
            dgt[experts[0]] = a0;
            dgt[experts[1]] = a1;
        }
        return;
    }
    for (int base = 0; base < nvec; base += 32 * 4) {
        float d[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int j = base + i * 32 + lane;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (j < nvec) v = ld_nc_v4(src + j);
            unpack8(v, d[i]);
        }
        for (int r = 0; r < n; ++r) {
            const uint4* os = og ? reinterpret_cast<const uint4*>(og + ((size_t)t * og_k + r) * H)
                                 : reinterpret_cast<const uint4*>(o.base<kPeer>(experts[r]) + (size_t)rows[r] * H);
            uint4* ds = reinterpret_cast<uint4*>(dout.base<kPeer>(experts[r]) + (size_t)rows[r] * H);
            float s = 0.f;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = base + i * 32 + lane;
                if (j < nvec) {
                    float f[8], w[8];
                    unpack8((kPeer && !og) ? os[j] : ld_nc_v4(os + j), f);
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        s = fmaf(d[i][c], f[c], s);
                        w[c] = g[r] * d[i][c];
                    }
                    ds[j] = pack8(w);
                }
            }
            dot[r] += s;
        }
    }
    float* dgt = dg + (size_t)t * E;
    if (lane < E) dgt[lane] = 0.f;
    __syncwarp();
    for (int r = 0; r < n; ++r) {
        const float s = warp_sum(dot[r]);
        if (lane == 0) dgt[experts[r]] = s;
    }
}

}  // namespace b200moe

using namespace b200moe;

namespace {
int check_perm(int T, int H, int E) {
    B200_CHECK_ARG(T >= 1, B200MOE_ERR_CONFIG, "tokens_per_batch must be >= 1, got %d", T);
    B200_CHECK_ARG(E >= 1 && E <= 32, B200MOE_ERR_CONFIG, "n_experts %d outside [1,32]", E);
    B200_CHECK_ARG(H % 8 == 0, B200MOE_ERR_SHAPE, "hidden must be a multiple of 8, got %d", H);
    return B200MOE_OK;
}
int check_peer(int E, int e_per_rank) {
    B200_CHECK_ARG(e_per_rank >= 1 && E % e_per_rank == 0, B200MOE_ERR_CONFIG,
                   "n_experts (%d) not divisible by experts per rank (%d)", E, e_per_rank);
    return B200MOE_OK;
}
Rows local_rows(void* p, int E) { return Rows{(__nv_bfloat16*)p, nullptr, E}; }
Rows peer_rows(const uint64_t* bufs, int epr) { return Rows{nullptr, bufs, epr}; }
}  // namespace

extern "C" {

int b200moe_permute(const void* x, const int32_t* slot_rank, const int32_t* seg_base, const int32_t* counts, int T,
                    int H, int E, void* xp, cudaStream_t stream) {
    int rc = check_perm(T, H, E);
    if (rc) return rc;
    const int tb = ceil_div(T, kPermThreads / 32);
    permute_kernel<false><<<tb + E * kPadParts, kPermThreads, 0, stream>>>((const __nv_bfloat16*)x, slot_rank, seg_base, counts,
                                                                T, H, E, tb, local_rows(xp, E), nullptr, 0);
    B200_CHECK_LAUNCH("permute");
    return B200MOE_OK;
}

int b200moe_permute_peer(const void* x, const int32_t* slot_rank, const int32_t* seg_base, const int32_t* counts,
                         int T, int H, int E, int e_per_rank, int rank, const uint64_t* xp_bufs,
                         const uint64_t* count_bufs, cudaStream_t stream) {
    int rc = check_perm(T, H, E);
    if (rc) return rc;
    if ((rc = check_peer(E, e_per_rank))) return rc;
    const int tb = ceil_div(T, kPermThreads / 32);
    permute_kernel<true><<<tb + E * kPadParts, kPermThreads, 0, stream>>>((const __nv_bfloat16*)x, slot_rank, seg_base, counts,
                                                               T, H, E, tb, peer_rows(xp_bufs, e_per_rank),
                                                               count_bufs, rank);
    B200_CHECK_LAUNCH("permute_peer");
    return B200MOE_OK;
}

int b200moe_combine(const void* o, const float* gates, const int32_t* slot_rank, const int32_t* seg_base, int T,
                    int H, int E, void* y, cudaStream_t stream) {
    int rc = check_perm(T, H, E);
    if (rc) return rc;
    const int tb = ceil_div(T, kPermThreads / 32);
    combine_kernel<false><<<tb, kPermThreads, 0, stream>>>(local_rows((void*)o, E), gates, slot_rank, seg_base, T, H,
                                                            E, (__nv_bfloat16*)y, nullptr, 0);
    B200_CHECK_LAUNCH("combine");
    return B200MOE_OK;
}

int b200moe_combine_peer(const uint64_t* o_bufs, int e_per_rank, const float* gates, const int32_t* slot_rank,
                         const int32_t* seg_base, int T, int H, int E, void* y, void* og, int og_k,
                         cudaStream_t stream) {
    int rc = check_perm(T, H, E);
    if (rc) return rc;
    if ((rc = check_peer(E, e_per_rank))) return rc;
    B200_CHECK_ARG(og == nullptr || (og_k >= 1 && og_k <= E), B200MOE_ERR_CONFIG, "og_k %d outside [1, %d]", og_k, E);
    const int tb = ceil_div(T, kPermThreads / 32);
    combine_kernel<true><<<tb, kPermThreads, 0, stream>>>(peer_rows(o_bufs, e_per_rank), gates, slot_rank, seg_base,
                                                           T, H, E, (__nv_bfloat16*)y, (__nv_bfloat16*)og, og_k);
    B200_CHECK_LAUNCH("combine_peer");
    return B200MOE_OK;
}

int b200moe_combine_bwd(const void* dy, const void* o, const float* gates, const int32_t* slot_rank,
                        const int32_t* seg_base, const int32_t* counts, int T, int H, int E, void* dout, float* dg,
                        cudaStream_t stream) {
    int rc = check_perm(T, H, E);
    if (rc) return rc;
    const int tb = ceil_div(T, kPermThreads / 32);
    combine_bwd_kernel<false><<<tb + E * kPadParts, kPermThreads, 0, stream>>>((const __nv_bfloat16*)dy, local_rows((void*)o, E),
                                                                    gates, slot_rank, seg_base, counts, T, H, E, tb,
                                                                    local_rows(dout, E), dg, nullptr, 0);
    B200_CHECK_LAUNCH("combine_bwd");
    return B200MOE_OK;
}

int b200moe_combine_bwd_peer(const void* dy, const uint64_t* o_bufs, const float* gates, const int32_t* slot_rank,
                             const int32_t* seg_base, const int32_t* counts, int T, int H, int E, int e_per_rank,
                             const uint64_t* dout_bufs, float* dg, const void* og, int og_k, cudaStream_t stream) {
    int rc = check_perm(T, H, E);
    if (rc) return rc;
    if ((rc = check_peer(E, e_per_rank))) return rc;
    B200_CHECK_ARG(og == nullptr || (og_k >= 1 && og_k <= E), B200MOE_ERR_CONFIG, "og_k %d outside [1, %d]", og_k, E);
    const int tb = ceil_div(T, kPermThreads / 32);
    combine_bwd_kernel<true><<<tb + E * kPadParts, kPermThreads, 0, stream>>>(
        (const __nv_bfloat16*)dy, peer_rows(o_bufs, e_per_rank), gates, slot_rank, seg_base, counts, T, H, E, tb,
        peer_rows(dout_bufs, e_per_rank), dg, (const __nv_bfloat16*)og, og_k);
    B200_CHECK_LAUNCH("combine_bwd_peer");
    return B200MOE_OK;
}

}  // extern "C"
