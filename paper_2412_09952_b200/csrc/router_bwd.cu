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
//
// Two kernels: a per-token pass (dh, dn and the compact list of the token's
// kept rows), then a bandwidth pass over [T, H] with 16-byte loads (8 hidden
// units per lane per chunk) that gathers the expert rows and adds the router
// term from an L1-resident swizzled copy of W.
#include <algorithm>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <math.h>

#include "common.cuh"
#include "ptx.cuh"

namespace b200moe {

// W [H, E] fp32 -> float4 blocks: index ((j * (EP/4) + e4) * (H/J) + hb), h = hb*J + j,
// so lane-consecutive hb are address-consecutive (conflict-free, coalesced).
template <int EP, int J>
__global__ void swizzle_w_j(const float* __restrict__ w, int H, int E, float4* __restrict__ out) {
    const int HB = H / J;
    const int n = HB * J * (EP / 4);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int hb = i % HB;
        const int rest = i / HB;
        const int e4 = rest % (EP / 4);
        const int j = rest / (EP / 4);
        const int h = hb * J + j;
        float v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int e = e4 * 4 + c;
            v[c] = (e < E) ? w[(size_t)h * E + e] : 0.f;
        }
        out[i] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

// ---- pass 1: one thread per token
// Row handles: row index in the owner's buffer, with the owner rank in bits
// 26..30 (expert parallel: owner = e / e_per_rank; single GPU: owner 0).
constexpr int kRowBits = 26;

template <int EP, int KM>
__global__ void __launch_bounds__(256)
router_dh_kernel(const int32_t* __restrict__ slot_rank, const int32_t* __restrict__ seg_base,
                 const float* __restrict__ dg, const float* __restrict__ dgx, int64_t sx_t, int64_t sx_e,
                 const float* __restrict__ gates, const float* __restrict__ probs, const float* __restrict__ z,
                 const float* __restrict__ noise_act, int T, int E, int router_type, float* __restrict__ dh_out,
                 float* __restrict__ dn_out, int32_t* __restrict__ rows_out, int e_per_rank) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    float p[EP], g[EP];
    float dot = 0.f;
    int nrow = 0;
    int rows[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) rows[j] = -1;
#pragma unroll
    for (int e = 0; e < EP; ++e) {
        p[e] = 0.f;
        g[e] = 0.f;
        if (e < E) {
            const size_t i = (size_t)t * E + e;
            float gt = dg[i];
            if (dgx) gt += dgx[(int64_t)t * sx_t + (int64_t)e * sx_e];
            const float gv = gates[i];
            const float pv = (router_type == B200MOE_ROUTER_MIXTRAL) ? gv : probs[i];
            const bool topk = gv > 0.f;  // top-k and not underflowed (underflowed entries contribute 0)
            const float geff = (router_type == B200MOE_ROUTER_MIXTRAL) ? (pv > 0.f ? gt : 0.f) : (topk ? gt : 0.f);
            p[e] = pv;
            g[e] = geff;
            dot = fmaf(pv, geff, dot);
            const int rk = slot_rank ? slot_rank[i] : -1;   // null: gate backward only (no expert rows)
            if (rk >= 0 && nrow < KM) {
#pragma unroll
                for (int j = 0; j < KM; ++j)
                    if (j == nrow) rows[j] = ((e / e_per_rank) << kRowBits) | (seg_base[e] + rk);
                ++nrow;
            }
        }
    }
#pragma unroll
    for (int e = 0; e < EP; ++e) {
        if (e < E) {
            const size_t i = (size_t)t * E + e;
            float dhv = p[e] * (g[e] - dot);
            if (router_type == B200MOE_ROUTER_MIXTRAL && !(p[e] > 0.f)) dhv = 0.f;
            dh_out[i] = dhv;
            if (dn_out) {
                const float an = noise_act[i];
                dn_out[i] = dhv * z[i] * (1.0f / (1.0f + expf(-an)));
            }
        }
    }
    if (rows_out) {
#pragma unroll
        for (int j = 0; j < KM; ++j) rows_out[(size_t)t * KM + j] = rows[j];
    }
}

// dn = dh * z * sigmoid(a_n) for the standalone router-logits backward
// (tensor.py:220-227 softplus' times the constant draw z, moe.py:149).
__global__ void router_dn_kernel(const float* __restrict__ dh, const float* __restrict__ z,
                                 const float* __restrict__ noise_act, size_t n, float* __restrict__ dn) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dn[i] = dh[i] * z[i] * (1.0f / (1.0f + expf(-noise_act[i])));
}

// ---- pass 2: warp per TT tokens, lane owns 8 hidden units per 256-wide chunk
constexpr int kDxThreads = 256;
// 32/EP tokens per warp (4 at E=8).  Two tokens per warp cut registers from 128
// to 80 but measured slower in the bench (0.062 -> 0.088 ms: W traffic doubles);
// W_g in shared memory (bulk copy) with 2 tokens per warp, 16 warps per block
// and a one-chunk prefetch of the dxp rows measured 45.4 vs 42.9 us (ncu); the
// dxp rows through a 3-stage cp.async ring (96 KB per block) 56.0 us -- the
// ring evicts the 128 KB W_g table from L1.
__host__ __device__ constexpr int dx_tokens_per_warp(int ep) { return 32 / ep; }

// Inputs of the softmax' step when it is fused into the dx kernel (the
// per-token pass of router_dh_kernel done by the warp that owns the token).
struct DhIn {
    const int32_t* slot_rank;
    const int32_t* seg_base;
    const float* dg;
    const float* dgx;
    int64_t sx_t, sx_e;
    const float* gates;
    const float* probs;
    const float* z;
    const float* noise_act;
    int router_type;
    int e_per_rank;
};

#ifndef B200_DX_MIN_BLOCKS
#define B200_DX_MIN_BLOCKS 2
#endif
template <int EP, int KM, bool kNoise, bool kFused = false>
__global__ void __launch_bounds__(kDxThreads, B200_DX_MIN_BLOCKS)
router_dx_kernel(const __nv_bfloat16* __restrict__ dxp_local, const uint64_t* __restrict__ dxp_bufs,
                 const int32_t* __restrict__ rows_in,
                 float* __restrict__ dh, float* __restrict__ dn, const float4* __restrict__ wsw,
                 const float4* __restrict__ wnsw, int T, int H, int E, __nv_bfloat16* __restrict__ dx,
                 const DhIn din) {
    constexpr int TT = dx_tokens_per_warp(EP);
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (kDxThreads / 32) + (threadIdx.x >> 5);
    const int t0 = gw * TT;
    if (t0 >= T) return;
    const int HB = H / 8;
    const int t_l = t0 + lane / EP, e_l = lane % EP;              // this lane's (token, expert)
    const bool live = lane < TT * EP && t_l < T && e_l < E;
    int rr[TT][KM];
    float v = 0.f, w = 0.f;
    if constexpr (kFused) {
        // softmax' of this lane's entry, bit-identical to router_dh_kernel: the
        // row dot product is the same sequential fmaf chain over e, evaluated by
        // every lane of the token's EP-lane group from shuffled values
        const size_t i = (size_t)t_l * E + e_l;
        float gt = 0.f, pv = 0.f, geff = 0.f;
        int rk = -1;
        if (live) {
            gt = din.dg[i];
            if (din.dgx) gt += din.dgx[(int64_t)t_l * din.sx_t + (int64_t)e_l * din.sx_e];
            const float gv = din.gates[i];
            pv = (din.router_type == B200MOE_ROUTER_MIXTRAL) ? gv : din.probs[i];
            const bool topk = gv > 0.f;
            geff = (din.router_type == B200MOE_ROUTER_MIXTRAL) ? (pv > 0.f ? gt : 0.f) : (topk ? gt : 0.f);
            rk = din.slot_rank[i];
        }
        const int gbase = (lane / EP) * EP;
        float dot = 0.f;
#pragma unroll
        for (int e = 0; e < EP; ++e) {
            const float pe = __shfl_sync(0xffffffffu, pv, gbase + e);
            const float ge = __shfl_sync(0xffffffffu, geff, gbase + e);
            if (e < E) dot = fmaf(pe, ge, dot);
        }
        float dhv = pv * (geff - dot);
        if (din.router_type == B200MOE_ROUTER_MIXTRAL && !(pv > 0.f)) dhv = 0.f;
        v = live ? dhv : 0.f;
        if (live) dh[i] = dhv;
        if constexpr (kNoise) {
            if (live) {
                w = dhv * din.z[i] * (1.0f / (1.0f + expf(-din.noise_act[i])));
                dn[i] = w;
            }
        }
        // the token's kept rows in ascending expert order (row handles as in router_dh_kernel)
        const int handle = rk >= 0 ? (((e_l / din.e_per_rank) << kRowBits) | (din.seg_base[e_l] + rk)) : -1;
        const unsigned kept = __ballot_sync(0xffffffffu, rk >= 0);
        const unsigned gmask = (EP == 32) ? 0xffffffffu : (((1u << EP) - 1u) << gbase);
        const int pos = __popc(kept & gmask & ((1u << lane) - 1u));   // rank among the group's kept lanes
#pragma unroll
        for (int j = 0; j < KM; ++j) {
            const unsigned m = __ballot_sync(0xffffffffu, rk >= 0 && pos == j);
#pragma unroll
            for (int tt = 0; tt < TT; ++tt) {
                const unsigned gm = (EP == 32) ? 0xffffffffu : (((1u << EP) - 1u) << (tt * EP));
                const unsigned mm = m & gm;
                const int src = mm ? (__ffs(mm) - 1) : 0;
                const int hv = __shfl_sync(0xffffffffu, handle, src);
                rr[tt][j] = mm ? hv : -1;
            }
        }
    } else {
        v = live ? dh[(size_t)t_l * E + e_l] : 0.f;
        w = (kNoise && live) ? dn[(size_t)t_l * E + e_l] : 0.f;
#pragma unroll
        for (int tt = 0; tt < TT; ++tt)
#pragma unroll
            for (int j = 0; j < KM; ++j)
                rr[tt][j] = (rows_in && t0 + tt < T) ? rows_in[(size_t)(t0 + tt) * KM + j] : -1;
    }
    // (token, expert) values broadcast to every lane
    float dhall[TT * EP], dnall[TT * EP];
#pragma unroll
    for (int i = 0; i < TT * EP; ++i) {
        dhall[i] = __shfl_sync(0xffffffffu, v, i);
        if constexpr (kNoise) dnall[i] = __shfl_sync(0xffffffffu, w, i);
    }

    for (int hb = lane; hb < HB; hb += 32) {
        float acc[TT][8];
        uint4 ld[TT][KM];
#pragma unroll
        for (int tt = 0; tt < TT; ++tt)
#pragma unroll
            for (int j = 0; j < KM; ++j)
                if (rr[tt][j] >= 0) {
                    const int h = rr[tt][j];
                    const size_t row = (size_t)(h & ((1 << kRowBits) - 1));
                    if (dxp_bufs) {  // expert parallel: the owner's buffer, over NVLink
                        const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(dxp_bufs[h >> kRowBits]);
                        ld[tt][j] = *reinterpret_cast<const uint4*>(src + row * H + hb * 8);
                    } else {
                        ld[tt][j] = ld_nc_v4(dxp_local + row * H + hb * 8);
                    }
                }
#pragma unroll
        for (int tt = 0; tt < TT; ++tt)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[tt][c] = 0.f;
        // expert-path rows, ascending expert order
#pragma unroll
        for (int tt = 0; tt < TT; ++tt)
#pragma unroll
            for (int j = 0; j < KM; ++j)
                if (rr[tt][j] >= 0) {
                    float f[8];
                    unpack8(ld[tt][j], f);
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc[tt][c] += f[c];
                }
        // router path
#pragma unroll
        for (int jh = 0; jh < 8; ++jh) {
#pragma unroll
            for (int e4 = 0; e4 < EP / 4; ++e4) {
                const float4 w = __ldg(&wsw[(jh * (EP / 4) + e4) * HB + hb]);
                if constexpr (TT % 2 == 0) {   // token pairs in one FFMA2 each, same fmaf order per token
#pragma unroll
                    for (int tt = 0; tt < TT; tt += 2) {
                        const float* d0 = dhall + tt * EP + e4 * 4;
                        const float* d1 = d0 + EP;
                        float2 a2 = make_float2(acc[tt][jh], acc[tt + 1][jh]);
                        ffma2(a2, make_float2(d0[0], d1[0]), make_float2(w.x, w.x));
                        ffma2(a2, make_float2(d0[1], d1[1]), make_float2(w.y, w.y));
                        ffma2(a2, make_float2(d0[2], d1[2]), make_float2(w.z, w.z));
                        ffma2(a2, make_float2(d0[3], d1[3]), make_float2(w.w, w.w));
                        acc[tt][jh] = a2.x;
                        acc[tt + 1][jh] = a2.y;
                    }
                } else {
#pragma unroll
                    for (int tt = 0; tt < TT; ++tt) {
                        const float* d = dhall + tt * EP + e4 * 4;
                        float a = acc[tt][jh];
                        a = fmaf(d[0], w.x, a);
                        a = fmaf(d[1], w.y, a);
                        a = fmaf(d[2], w.z, a);
                        a = fmaf(d[3], w.w, a);
                        acc[tt][jh] = a;
                    }
                }
                if constexpr (kNoise) {
                    const float4 wn = __ldg(&wnsw[(jh * (EP / 4) + e4) * HB + hb]);
#pragma unroll
                    for (int tt = 0; tt < TT; ++tt) {
                        const float* d = dnall + tt * EP + e4 * 4;
                        float a = acc[tt][jh];
                        a = fmaf(d[0], wn.x, a);
                        a = fmaf(d[1], wn.y, a);
                        a = fmaf(d[2], wn.z, a);
                        a = fmaf(d[3], wn.w, a);
                        acc[tt][jh] = a;
                    }
                }
            }
        }
#pragma unroll
        for (int tt = 0; tt < TT; ++tt)
            if (t0 + tt < T) st_v4(dx + (size_t)(t0 + tt) * H + hb * 8, pack8(acc[tt]));
    }
}

// dW[h, e] = sum_t x[t, h] * d[t, e]: per (H/1024 block, 128-token chunk) partials,
// then a fixed-order reduction over chunks (64-token chunks measured slower:
// the doubled partial traffic outweighs the occupancy gain).
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
#pragma unroll 8
    for (int tt = 0; tt < tn; ++tt) {
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(x + (size_t)(t0 + tt) * H + h0));
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

// E <= 8, TMA ring: a block owns 256 hidden units x kRgTok tokens.  A producer
// thread streams the block's x tile into a kRgStages-deep shared-memory ring,
// one 2-D TMA box (256 hidden x 32 tokens, 16 KB) per stage (32 separate 1-D
// row copies per stage were request-rate bound: 41 us vs 38 us with the
// prologue fixed), so ~64 KB per block are in flight without registers;
// 8 consumer warps take 4 rows of each 32-row stage, accumulate 8 hidden x EP
// experts per lane in registers, and hand the slot back.  One cross-warp
// reduction per block (through the drained ring), fixed order: deterministic.
#ifndef B200_RG_TOK
#define B200_RG_TOK 512
#endif
#ifndef B200_RG_ROWS
#define B200_RG_ROWS 32
#endif
#ifndef B200_RG_STAGES
#define B200_RG_STAGES 4
#endif
constexpr int kRgTok = B200_RG_TOK;
constexpr int kRgStageRows = B200_RG_ROWS;
constexpr int kRgStages = B200_RG_STAGES;
constexpr int kRgStageBytes = kRgStageRows * 256 * 2;   // 16 KB
constexpr int kRgConsumers = 8;

template <int EP>
__global__ void __launch_bounds__((kRgConsumers + 1) * 32, 2)
router_wgrad_ring(const __grid_constant__ CUtensorMap xmap, const float* __restrict__ d, int T, int H, int E,
                  float* __restrict__ part, float* __restrict__ out, int32_t* __restrict__ tickets) {
    extern __shared__ __align__(128) uint8_t sm_raw[];
    __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(sm_raw);
    float* ds = reinterpret_cast<float*>(sm_raw + kRgStages * kRgStageBytes);       // [kRgTok][EP]
    uint64_t* full = reinterpret_cast<uint64_t*>(ds + kRgTok * EP);
    uint64_t* empty = full + kRgStages;
    uint64_t* dsbar = empty + kRgStages;
    const int chunk = blockIdx.y;
    const int t0 = chunk * kRgTok;
    const int h0 = blockIdx.x * 256;
    const int hw = min(256, H - h0);                       // hidden units of this block (multiple of 8)
    const int ntok = min(kRgTok, T - t0);
    const int nst = ceil_div(ntok, kRgStageRows);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // the block's dh rows: one bulk copy when they are contiguous in the [T, EP]
    // layout (E == EP), else an unrolled gather (a dependent load loop here
    // was the kernel's main stall)
    const bool dh_bulk = (E == EP) && ((ntok * E * 4) % 16 == 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kRgStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], kRgConsumers);
        }
        ptx::mbar_init(dsbar, 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (dh_bulk) {
        if (threadIdx.x == 0) {
            ptx::mbar_arrive_expect_tx(dsbar, (uint32_t)(ntok * E * 4));
            ptx::bulk_load_1d(ds, d + (size_t)t0 * E, (uint32_t)(ntok * E * 4), dsbar);
        }
    } else {
        constexpr int kPer = (kRgTok * EP + (kRgConsumers + 1) * 32 - 1) / ((kRgConsumers + 1) * 32);
        float v[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int i = threadIdx.x + u * blockDim.x;
            const int tt = i / EP, e = i % EP, t = t0 + tt;
            v[u] = (i < kRgTok * EP && t < T && e < E) ? d[(size_t)t * E + e] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int i = threadIdx.x + u * blockDim.x;
            if (i < kRgTok * EP) ds[i] = v[u];
        }
        __syncthreads();
    }
    if (warp == kRgConsumers) {            // producer: one 2-D TMA box (256 hidden x 32 tokens) per stage
        if (lane == 0) {
            for (int st = 0; st < nst; ++st) {
                const int slot = st % kRgStages;
                if (st >= kRgStages) ptx::mbar_wait(&empty[slot], ((st / kRgStages) - 1) & 1);
                ptx::mbar_arrive_expect_tx(&full[slot], (uint32_t)kRgStageBytes);   // OOB rows arrive as zeros
                ptx::tma_load_2d(&xmap, &full[slot], ring + (size_t)slot * kRgStageRows * 256, h0,
                                 t0 + st * kRgStageRows);
            }
        }
    } else {                               // consumers
        float acc[8][EP];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int e = 0; e < EP; ++e) acc[j][e] = 0.f;
        const bool hok = lane * 8 < hw;
        if (dh_bulk) ptx::mbar_wait(dsbar, 0);
        for (int st = 0; st < nst; ++st) {
            const int slot = st % kRgStages;
            ptx::mbar_wait(&full[slot], (st / kRgStages) & 1);
            const int rows = min(kRgStageRows, ntok - st * kRgStageRows);
            const __nv_bfloat16* base = ring + (size_t)slot * kRgStageRows * 256;
#pragma unroll
            for (int i = 0; i < kRgStageRows / kRgConsumers; ++i) {
                const int r = warp * (kRgStageRows / kRgConsumers) + i;
                if (r < rows && hok) {
                    float xv[8];
                    unpack8(*reinterpret_cast<const uint4*>(base + r * 256 + lane * 8), xv);
                    const float* dr = ds + (st * kRgStageRows + r) * EP;
#pragma unroll
                    for (int e = 0; e < EP; ++e) {
                        const float dv = dr[e];
#pragma unroll
                        for (int j = 0; j < 8; j += 2) {   // (acc[j][e], acc[j+1][e]) in one FFMA2
                            float2 a2 = make_float2(acc[j][e], acc[j + 1][e]);
                            ffma2(a2, make_float2(xv[j], xv[j + 1]), make_float2(dv, dv));
                            acc[j][e] = a2.x;
                            acc[j + 1][e] = a2.y;
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&empty[slot]);
        }
        __syncthreads();                    // (A) every consumer is done with the ring
        float* rw = reinterpret_cast<float*>(sm_raw) + (size_t)warp * 256 * EP;   // [(j*EP+e)*32 + lane]
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int e = 0; e < EP; ++e) rw[(j * EP + e) * 32 + lane] = acc[j][e];
    }
    if (warp == kRgConsumers) __syncthreads();   // matches (A)
    __syncthreads();
    const float* red = reinterpret_cast<const float*>(sm_raw);
    float* p = part + (size_t)chunk * H * E;
    for (int i = threadIdx.x; i < 256 * EP; i += blockDim.x) {
        const int l = i % 32, je = i / 32;
        const int j = je / EP, e = je % EP;
        const int hh = l * 8 + j;
        float sum = 0.f;
#pragma unroll
        for (int w = 0; w < kRgConsumers; ++w) sum += red[(size_t)w * 256 * EP + i];
        if (e < E && hh < hw) p[(size_t)(h0 + hh) * E + e] = sum;
    }
    if (tickets == nullptr) return;        // reduce_partials follows
    // the last chunk block of this hidden block sums the chunks' partials in
    // chunk order (same order as reduce_partials) and resets its ticket
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&tickets[blockIdx.x], 1) == (int)gridDim.y - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int nch = gridDim.y;
    for (int i = threadIdx.x; i < hw * E; i += blockDim.x) {
        const size_t o = (size_t)h0 * E + i;
        float sum = 0.f;
        int c = 0;
        for (; c + 8 <= nch; c += 8) {
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = __ldcg(part + (size_t)(c + j) * H * E + o);
#pragma unroll
            for (int j = 0; j < 8; ++j) sum += v[j];
        }
        for (; c < nch; ++c) sum += __ldcg(part + (size_t)c * H * E + o);
        out[o] = sum;
    }
    if (threadIdx.x == 0) tickets[blockIdx.x] = 0;
}

// Router weight gradients on tcgen05 (E <= 8): dW[h, e] = sum_t x[t, h] dh[t, e]
// (and dW_noise from dn) as one MN-major GEMM per CTA: M = 128 hidden units
// (TMEM lanes), N = 64 split columns, K = a chunk of kRwTok tokens.  The fp32
// dh / dn are split into three bf16 parts hi + mid + lo (each the bf16
// rounding of the remainder, together within 2^-24 of the value) written by
// the producer warp straight into the swizzled B tile -- columns [0, 24) dh,
// [32, 56) dn, the rest zero -- while x arrives by TMA (two 64-hidden boxes
// per 64-token stage); x is bf16, so every product is exact and the MMA
// accumulates in fp32.  The epilogue adds the parts smallest first; per-chunk
// partials are summed in chunk order by the last CTA of each hidden block
// (tickets), so the result is deterministic.  x is read once for both
// matrices.
#ifndef B200_RW_TOK
#define B200_RW_TOK 1024
#endif
#ifndef B200_RW_STAGES
#define B200_RW_STAGES 3
#endif
constexpr int kRwTok = B200_RW_TOK;
constexpr int kRwStages = B200_RW_STAGES;
constexpr int kRwABytes = 2 * 64 * 64 * 2;   // two 64-hidden x 64-token boxes (SWIZZLE_128B)
constexpr int kRwBBytes = 64 * 64 * 2;       // 64 tokens x 64 split columns
constexpr int kRwStageBytes = kRwABytes + kRwBBytes;
constexpr int kRwSmem = kRwStages * kRwStageBytes + 1024 + 256;

__device__ __forceinline__ void rw_split3(float v, __nv_bfloat16& hi, __nv_bfloat16& mid, __nv_bfloat16& lo) {
    hi = __float2bfloat16_rn(v);
    const float r1 = v - __bfloat162float(hi);
    mid = __float2bfloat16_rn(r1);
    lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
}

// element (row k, column n) of a [64 x 64] bf16 SWIZZLE_128B tile
__device__ __forceinline__ int sw128_off(int k, int n) {
    return k * 128 + ((((n * 2) >> 4) ^ (k & 7)) << 4) + ((n * 2) & 15);
}

template <bool kNoise>
__global__ void __launch_bounds__(128, 1)
router_wgrad_tc_kernel(const __grid_constant__ CUtensorMap xmap, const float* __restrict__ dh,
                       const float* __restrict__ dn, int T, int H, int E, float* __restrict__ part,
                       float* __restrict__ out_g, float* __restrict__ out_n, int32_t* __restrict__ tickets) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRwStages * kRwStageBytes);
    uint64_t* empty = full + kRwStages;
    uint64_t* done = empty + kRwStages;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
    __shared__ bool last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int h0 = blockIdx.x * 128;
    const int chunk = blockIdx.y;
    const int t0 = chunk * kRwTok;
    const int ntok = min(kRwTok, T - t0);
    const int nkb = (ntok + 63) / 64;
    // zero every stage's B tile once: the producer rewrites only the split columns
    for (int i = threadIdx.x; i < kRwStages * kRwBBytes / 16; i += blockDim.x) {
        const int st = i / (kRwBBytes / 16), j = i % (kRwBBytes / 16);
        reinterpret_cast<uint4*>(smem + st * kRwStageBytes + kRwABytes)[j] = make_uint4(0, 0, 0, 0);
    }
    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&xmap);
        for (int s = 0; s < kRwStages; ++s) {
            ptx::mbar_init(&full[s], 2);     // the x TMA (with its bytes) + the split-B writers
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(done, 1);
        ptx::fence_mbar_init();
    }
    ptx::fence_proxy_async();   // the zeroed tiles, before the MMAs read them
    if (warp == 1) ptx::tmem_alloc<1>(tslot, 64);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == 0) {                        // x producer: two TMA boxes per stage
        if (lane == 0) {
            for (int kb = 0; kb < nkb; ++kb) {
                const int st = kb % kRwStages;
                if (kb >= kRwStages) ptx::mbar_wait(&empty[st], ((kb / kRwStages) - 1) & 1);
                uint8_t* a = smem + st * kRwStageBytes;
                ptx::mbar_arrive_expect_tx(&full[st], kRwABytes);   // tokens beyond T arrive as zeros
                ptx::tma_load_2d(&xmap, &full[st], a, h0, t0 + kb * 64);
                ptx::tma_load_2d(&xmap, &full[st], a + kRwABytes / 2, h0 + 64, t0 + kb * 64);
            }
        }
    } else if (warp >= 2) {                 // split-B producers: one token row per thread (64 threads)
        const int tt = threadIdx.x - 64;
        for (int kb = 0; kb < nkb; ++kb) {
            const int st = kb % kRwStages;
            if (kb >= kRwStages) ptx::mbar_wait(&empty[st], ((kb / kRwStages) - 1) & 1);
            uint8_t* b = smem + st * kRwStageBytes + kRwABytes;
            const int t = t0 + kb * 64 + tt;
            const bool ok = tt < ntok - kb * 64;
            float g[8], q[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                g[e] = (ok && e < E) ? dh[(size_t)t * E + e] : 0.f;
                if constexpr (kNoise) q[e] = (ok && e < E) ? dn[(size_t)t * E + e] : 0.f;
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                __nv_bfloat16 hi, mid, lo;
                rw_split3(g[e], hi, mid, lo);
                *reinterpret_cast<__nv_bfloat16*>(b + sw128_off(tt, e)) = hi;
                *reinterpret_cast<__nv_bfloat16*>(b + sw128_off(tt, 8 + e)) = mid;
                *reinterpret_cast<__nv_bfloat16*>(b + sw128_off(tt, 16 + e)) = lo;
                if constexpr (kNoise) {
                    rw_split3(q[e], hi, mid, lo);
                    *reinterpret_cast<__nv_bfloat16*>(b + sw128_off(tt, 32 + e)) = hi;
                    *reinterpret_cast<__nv_bfloat16*>(b + sw128_off(tt, 40 + e)) = mid;
                    *reinterpret_cast<__nv_bfloat16*>(b + sw128_off(tt, 48 + e)) = lo;
                }
            }
            ptx::fence_proxy_async();
            asm volatile("bar.sync 1, 64;" ::: "memory");    // all 64 rows of the tile written
            if (tt == 0) ptx::mbar_arrive(&full[st]);
        }
    } else if (warp == 1 && lane == 0) {    // MMA issuer
        constexpr uint32_t idesc = ptx::make_idesc_bf16(128, 64, true, true);
        for (int kb = 0; kb < nkb; ++kb) {
            const int st = kb % kRwStages;
            ptx::mbar_wait(&full[st], (kb / kRwStages) & 1);
            ptx::tc_fence_after();
            const uint32_t a = ptx::smem_u32(smem + st * kRwStageBytes);
            const uint32_t b = a + kRwABytes;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                ptx::mma_bf16<1>(tmem, ptx::make_sdesc(a + kk * 2048, 8192, 1024),
                                 ptx::make_sdesc(b + kk * 2048, 8192, 1024), idesc, (kb | kk) != 0);
            ptx::mma_commit<1>(&empty[st], 1);
        }
        ptx::mma_commit<1>(done, 1);
    }
    // ---- epilogue: thread i owns hidden unit h0 + i (TMEM lane i)
    ptx::mbar_wait(done, 0);
    ptx::tc_fence_after();
    uint32_t d[64];
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
    ptx::tmem_ld_32x32b_x32(lane_addr, d);
    if constexpr (kNoise) ptx::tmem_ld_32x32b_x32(lane_addr + 32, d + 32);
    ptx::tmem_ld_wait();
    const int h = h0 + threadIdx.x;
    float* pg = part + (size_t)chunk * (kNoise ? 2 : 1) * H * E;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        if (e < E && h < H) {
            pg[(size_t)h * E + e] = (__uint_as_float(d[16 + e]) + __uint_as_float(d[8 + e])) + __uint_as_float(d[e]);
            if constexpr (kNoise)
                pg[(size_t)H * E + (size_t)h * E + e] =
                    (__uint_as_float(d[48 + e]) + __uint_as_float(d[40 + e])) + __uint_as_float(d[32 + e]);
        }
    }
    ptx::tc_fence_before();
    __threadfence();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<1>(tmem, 64);
    }
    if (threadIdx.x == 0) last = atomicAdd(&tickets[blockIdx.x], 1) == (int)gridDim.y - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // the last chunk CTA of this hidden block: chunk-ordered sums of the partials
    const int nch = gridDim.y;
    const size_t stride = (size_t)(kNoise ? 2 : 1) * H * E;
    for (int m = 0; m < (kNoise ? 2 : 1); ++m) {
        float* out = m == 0 ? out_g : out_n;
        for (int i = threadIdx.x; i < 128 * E; i += blockDim.x) {
            const int hh = h0 + i / E, e = i % E;
            if (hh >= H) continue;
            const size_t o = (size_t)m * H * E + (size_t)hh * E + e;
            float sum = 0.f;
            for (int c = 0; c < nch; ++c) sum += __ldcg(part + (size_t)c * stride + o);
            out[(size_t)hh * E + e] = sum;
        }
    }
    if (threadIdx.x == 0) tickets[blockIdx.x] = 0;
}

__global__ void reduce_partials(const float* __restrict__ part, int nchunks, size_t n, float* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float s = 0.f;
        int c = 0;
        for (; c + 8 <= nchunks; c += 8) {  // 8 independent loads in flight, summed in chunk order
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = __ldg(&part[(size_t)(c + j) * n + i]);
#pragma unroll
            for (int j = 0; j < 8; ++j) s += v[j];
        }
        for (; c < nchunks; ++c) s += part[(size_t)c * n + i];
        out[i] = s;
    }
}

// Loss only, from a precomputed importance vector (the dispatch kernel's
// per-expert sum of the same gates): mean, population variance, var / mean^2.
__global__ void importance_loss_kernel(const float* __restrict__ imp, int E, float* __restrict__ loss,
                                       int32_t* __restrict__ err_flag) {
    if (threadIdx.x != 0) return;
    importance_cv2(imp, E, loss, err_flag);
}

// Importance penalty forward: one block of 1024 threads; thread i sums the
// rows i, i+1024, ... (fixed order), then a fixed-order block reduction per
// expert; mean, population variance, loss = var / mean^2 (tensor.py:509-514).
__global__ void __launch_bounds__(1024)
importance_fwd_kernel(const float* __restrict__ g, int T, int E, float* __restrict__ imp, float* __restrict__ loss,
                      int32_t* __restrict__ err_flag) {
    __shared__ float part[32][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int e0 = 0; e0 < E; e0 += 32) {
        float s[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) s[i] = 0.f;
        for (int t = threadIdx.x; t < T; t += blockDim.x) {
            const float* row = g + (size_t)t * E + e0;
#pragma unroll
            for (int i = 0; i < 32; ++i)
                if (e0 + i < E) s[i] += row[i];
        }
        // warp reduce each of the (up to 32) expert sums, lane i keeps expert i
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            float v = warp_sum(s[i]);
            if (lane == i) part[warp][i] = v;
        }
        __syncthreads();
        if (warp == 0 && e0 + lane < E) {
            float r = 0.f;
            for (int w = 0; w < 32; ++w) r += part[w][lane];
            imp[e0 + lane] = r;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        float mean = 0.f;
        for (int e = 0; e < E; ++e) mean += ((volatile float*)imp)[e];
        mean /= (float)E;
        float var = 0.f;
        for (int e = 0; e < E; ++e) {
            const float dd = ((volatile float*)imp)[e] - mean;
            var += dd * dd;
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
template <int EP, int KM>
int router_bwd_impl(const void* dxp, const uint64_t* dxp_bufs, int e_per_rank, const int32_t* slot_rank,
                    const int32_t* seg_base, const float* dg,
                    const float* dgx, int64_t sx_t, int64_t sx_e, const float* gates, const float* probs,
                    const float* w_g, const float* w_noise, const float* z, const float* noise_act,
                    const float* wg_swz, const float* wn_swz, int T, int H,
                    int E, int router_type, void* dx, float* dh, float* dn, float* workspace, cudaStream_t stream) {
    // workspace: swizzled W_g [H*EP], W_noise [H*EP], rows [T*KM] (int32).  The
    // router forward leaves the same swizzled tables in its workspace; when
    // they are passed in (wg_swz / wn_swz) the swizzle launches are skipped.
    float4* wsw = reinterpret_cast<float4*>(workspace);
    float4* wnsw = reinterpret_cast<float4*>(workspace + (size_t)H * EP);
    int32_t* rows = reinterpret_cast<int32_t*>(workspace + (size_t)2 * H * EP);
    const bool noise = z != nullptr;
    if (wg_swz) wsw = reinterpret_cast<float4*>(const_cast<float*>(wg_swz));
    else swizzle_w_j<EP, 8><<<64, 256, 0, stream>>>(w_g, H, E, wsw);
    if (noise) {
        if (wn_swz) wnsw = reinterpret_cast<float4*>(const_cast<float*>(wn_swz));
        else swizzle_w_j<EP, 8><<<64, 256, 0, stream>>>(w_noise, H, E, wnsw);
    }
    (void)rows;
    // softmax' + kept-row lists fused into the dx pass (one launch: each warp
    // derives its tokens' dh / dn rows before streaming their dxp rows)
    const DhIn din{slot_rank, seg_base, dg, dgx, sx_t, sx_e, gates, probs, z, noise_act, router_type, e_per_rank};
    constexpr int TT = dx_tokens_per_warp(EP);
    const int grid = ceil_div(ceil_div(T, TT), kDxThreads / 32);
    if (noise)
        router_dx_kernel<EP, KM, true, true><<<grid, kDxThreads, 0, stream>>>(
            (const __nv_bfloat16*)dxp, dxp_bufs, nullptr, dh, dn, wsw, wnsw, T, H, E, (__nv_bfloat16*)dx, din);
    else
        router_dx_kernel<EP, KM, false, true><<<grid, kDxThreads, 0, stream>>>(
            (const __nv_bfloat16*)dxp, dxp_bufs, nullptr, dh, nullptr, wsw, wnsw, T, H, E, (__nv_bfloat16*)dx, din);
    B200_CHECK_LAUNCH("router_bwd");
    return B200MOE_OK;
}

template <int EP>
int router_bwd_k(int k, const void* dxp, const uint64_t* dxp_bufs, int e_per_rank, const int32_t* slot_rank,
                 const int32_t* seg_base, const float* dg,
                 const float* dgx, int64_t sx_t, int64_t sx_e, const float* gates, const float* probs,
                 const float* w_g, const float* w_noise, const float* z, const float* noise_act, const float* wg_swz,
                 const float* wn_swz, int T, int H, int E,
                 int router_type, void* dx, float* dh, float* dn, float* workspace, cudaStream_t stream) {
#define CALL(KM) router_bwd_impl<EP, KM>(dxp, dxp_bufs, e_per_rank, slot_rank, seg_base, dg, dgx, sx_t, sx_e, gates, \
                                         probs, w_g, w_noise, z, noise_act, wg_swz, wn_swz, T, H, E, router_type, dx, \
                                         dh, dn, workspace, stream)
    if (k <= 2) return CALL(2);
    if (k <= 4 || EP == 4) return CALL((EP < 4 ? EP : 4));
    return CALL(EP);
#undef CALL
}

template <int EP>
int wgrad_impl(const void* x, const float* d, int T, int H, int E, float* out, float* part, cudaStream_t stream,
               int32_t* tickets = nullptr) {
    int nch = ceil_div(T, kWgTok);
    if constexpr (EP <= 8) {
        nch = ceil_div(T, kRgTok);
        const size_t sh = (size_t)kRgStages * kRgStageBytes + (size_t)kRgTok * EP * sizeof(float) +
                          (2 * kRgStages + 1) * sizeof(uint64_t);
        static_assert((size_t)kRgConsumers * 256 * 8 * sizeof(float) <= (size_t)kRgStages * kRgStageBytes,
                      "the drained ring holds the cross-warp reduction");
        CUtensorMap xmap;
        const int rc = make_tmap_bf16_2d(&xmap, x, (uint64_t)H, (uint64_t)T, (uint64_t)H, 256, kRgStageRows);
        if (rc) return rc;
        auto kern = router_wgrad_ring<EP>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh);
        dim3 grid(ceil_div(H, 256), nch);
        kern<<<grid, (kRgConsumers + 1) * 32, sh, stream>>>(xmap, d, T, H, E, part, out, tickets);
        if (tickets) {
            B200_CHECK_LAUNCH("router_wgrad");
            return B200MOE_OK;
        }
    } else {
        dim3 grid(ceil_div(H, 1024), nch);
        router_wgrad_partial<EP><<<grid, 256, 0, stream>>>((const __nv_bfloat16*)x, d, T, H, E, part);
    }
    const size_t n = (size_t)H * E;
    reduce_partials<<<(int)((n + 255) / 256), 256, 0, stream>>>(part, nch, n, out);
    B200_CHECK_LAUNCH("router_wgrad");
    return B200MOE_OK;
}
}  // namespace

namespace {
template <int EP>
int router_logits_bwd_impl(const void* x, const float* dh, const float* w_g, const float* w_noise, const float* z,
                           const float* noise_act, int T, int H, int E, void* dx, float* dw_g, float* dw_noise,
                           float* dn, float* workspace, cudaStream_t stream) {
    float4* wsw = reinterpret_cast<float4*>(workspace);
    float4* wnsw = reinterpret_cast<float4*>(workspace + (size_t)H * EP);
    float* part = workspace + (size_t)2 * H * EP;
    const bool noise = z != nullptr;
    if (noise) {
        const size_t n = (size_t)T * E;
        router_dn_kernel<<<(int)std::min<size_t>((n + 255) / 256, 4 * kNumSMs), 256, 0, stream>>>(dh, z, noise_act,
                                                                                                  n, dn);
    }
    if (dx) {
        swizzle_w_j<EP, 8><<<64, 256, 0, stream>>>(w_g, H, E, wsw);
        if (noise) swizzle_w_j<EP, 8><<<64, 256, 0, stream>>>(w_noise, H, E, wnsw);
        constexpr int TT = dx_tokens_per_warp(EP);
        const int grid = ceil_div(ceil_div(T, TT), kDxThreads / 32);
        const DhIn none{};
        if (noise)
            router_dx_kernel<EP, 1, true><<<grid, kDxThreads, 0, stream>>>(nullptr, nullptr, nullptr,
                                                                            const_cast<float*>(dh), dn, wsw, wnsw, T,
                                                                            H, E, (__nv_bfloat16*)dx, none);
        else
            router_dx_kernel<EP, 1, false><<<grid, kDxThreads, 0, stream>>>(nullptr, nullptr, nullptr,
                                                                             const_cast<float*>(dh), dn, wsw, wnsw, T,
                                                                             H, E, (__nv_bfloat16*)dx, none);
    }
    if (dw_g) {
        int rc = wgrad_impl<EP>(x, dh, T, H, E, dw_g, part, stream);
        if (rc) return rc;
    }
    if (noise && dw_noise) return wgrad_impl<EP>(x, dn, T, H, E, dw_noise, part, stream);
    B200_CHECK_LAUNCH("router_logits_bwd");
    return B200MOE_OK;
}
}  // namespace

extern "C" {

static int router_bwd_any(const void* dxp, const uint64_t* dxp_bufs, int e_per_rank, const int32_t* slot_rank,
                          const int32_t* seg_base, const float* dg, const float* dgates_ext, int64_t dgates_stride_t,
                          int64_t dgates_stride_e, const float* gates, const float* probs, const float* w_g,
                          const float* w_noise, const float* z, const float* noise_act, const float* wg_swz,
                          const float* wn_swz, int T, int H, int E, int k,
                          int router_type, void* dx, float* dh, float* dn, float* workspace, cudaStream_t stream) {
    B200_CHECK_ARG(T >= 1 && E >= 1 && E <= 32, B200MOE_ERR_CONFIG, "bad T/E (%d, %d)", T, E);
    B200_CHECK_ARG(k >= 1 && k <= E, B200MOE_ERR_CONFIG, "top-k out of range: k=%d, n=%d", k, E);
    B200_CHECK_ARG(H % 8 == 0, B200MOE_ERR_SHAPE, "hidden must be a multiple of 8");
    B200_CHECK_ARG(router_type != B200MOE_ROUTER_ST || probs != nullptr, B200MOE_ERR_CONFIG, "st needs probs");
    B200_CHECK_ARG(z == nullptr || (w_noise && noise_act && dn), B200MOE_ERR_CONFIG, "noise args missing");
    B200_CHECK_ARG(e_per_rank >= 1 && E % e_per_rank == 0 && E / e_per_rank <= 32, B200MOE_ERR_CONFIG,
                   "experts per rank %d does not divide %d", e_per_rank, E);
#define CALL(EP) router_bwd_k<EP>(k, dxp, dxp_bufs, e_per_rank, slot_rank, seg_base, dg, dgates_ext,              \
                                  dgates_stride_t, dgates_stride_e, gates, probs, w_g, w_noise, z, noise_act, wg_swz, \
                                  wn_swz, T, H, E, router_type, dx, dh, dn, workspace, stream)
    if (E <= 4) return CALL(4);
    if (E <= 8) return CALL(8);
    if (E <= 16) return CALL(16);
    return CALL(32);
#undef CALL
}

int b200moe_router_bwd(const void* dxp, const int32_t* slot_rank, const int32_t* seg_base, const float* dg,
                       const float* dgates_ext, int64_t dgates_stride_t, int64_t dgates_stride_e, const float* gates,
                       const float* probs, const float* w_g, const float* w_noise, const float* z,
                       const float* noise_act, const float* wg_swz, const float* wn_swz, int T, int H, int E, int k,
                       int router_type, void* dx, float* dh, float* dn, float* workspace, cudaStream_t stream) {
    return router_bwd_any(dxp, nullptr, E, slot_rank, seg_base, dg, dgates_ext, dgates_stride_t, dgates_stride_e,
                          gates, probs, w_g, w_noise, z, noise_act, wg_swz, wn_swz, T, H, E, k, router_type, dx, dh,
                          dn, workspace, stream);
}

int b200moe_router_bwd_peer(const uint64_t* dxp_bufs, int e_per_rank, const int32_t* slot_rank,
                            const int32_t* seg_base, const float* dg, const float* dgates_ext,
                            int64_t dgates_stride_t, int64_t dgates_stride_e, const float* gates, const float* probs,
                            const float* w_g, const float* w_noise, const float* z, const float* noise_act,
                            const float* wg_swz, const float* wn_swz, int T,
                            int H, int E, int k, int router_type, void* dx, float* dh, float* dn, float* workspace,
                            cudaStream_t stream) {
    B200_CHECK_ARG(dxp_bufs != nullptr, B200MOE_ERR_CONFIG, "peer buffers required");
    return router_bwd_any(nullptr, dxp_bufs, e_per_rank, slot_rank, seg_base, dg, dgates_ext, dgates_stride_t,
                          dgates_stride_e, gates, probs, w_g, w_noise, z, noise_act, wg_swz, wn_swz, T, H, E, k,
                          router_type, dx, dh, dn, workspace, stream);
}

int b200moe_router_wgrad(const void* x, const float* dh, const float* dn, int T, int H, int E, float* dw_g,
                         float* dw_noise, float* workspace, int32_t* tickets, cudaStream_t stream) {
    B200_CHECK_ARG(T >= 1 && E >= 1 && E <= 32, B200MOE_ERR_CONFIG, "bad T/E (%d, %d)", T, E);
    B200_CHECK_ARG(H % 4 == 0, B200MOE_ERR_SHAPE, "hidden must be a multiple of 4");
#ifndef B200_RWGRAD_TC
#define B200_RWGRAD_TC 1
#endif
    // tensor-core path: E <= 8, whole 128-hidden blocks, partials within the workspace bound
    const int nch = ceil_div(T, kRwTok);
    if (B200_RWGRAD_TC && tickets && E <= 8 && H % 128 == 0 &&
        (size_t)nch * (dn ? 2 : 1) * H * E <= (size_t)ceil_div(T, 64) * H * E) {
        CUtensorMap xmap;
        const int rc = make_tmap_bf16_2d(&xmap, x, (uint64_t)H, (uint64_t)T, (uint64_t)H, 64, 64, true);
        if (rc) return rc;
        dim3 grid(H / 128, nch);
        if (dn) {
            auto kern = router_wgrad_tc_kernel<true>;
            static std::atomic<uint64_t> attr{0};
            if (cudaError_t ae = ensure_smem_attr(kern, kRwSmem, attr); ae != cudaSuccess) {
                set_error("router_wgrad_tc smem attribute: %s", cudaGetErrorString(ae));
                return B200MOE_ERR_CUDA;
            }
            kern<<<grid, 128, kRwSmem, stream>>>(xmap, dh, dn, T, H, E, workspace, dw_g, dw_noise, tickets);
        } else {
            auto kern = router_wgrad_tc_kernel<false>;
            static std::atomic<uint64_t> attr{0};
            if (cudaError_t ae = ensure_smem_attr(kern, kRwSmem, attr); ae != cudaSuccess) {
                set_error("router_wgrad_tc smem attribute: %s", cudaGetErrorString(ae));
                return B200MOE_ERR_CUDA;
            }
            kern<<<grid, 128, kRwSmem, stream>>>(xmap, dh, nullptr, T, H, E, workspace, dw_g, nullptr, tickets);
        }
        B200_CHECK_LAUNCH("router_wgrad");
        return B200MOE_OK;
    }
#define CALL(EP, D, O) wgrad_impl<EP>(x, D, T, H, E, O, workspace, stream, tickets)
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

int b200moe_gate_bwd(const float* dgates, const float* gates, const float* probs, int T, int E, int router_type,
                     float* dh, cudaStream_t stream) {
    B200_CHECK_ARG(T >= 1 && E >= 1 && E <= 32, B200MOE_ERR_CONFIG, "bad T/E (%d, %d)", T, E);
    B200_CHECK_ARG(router_type != B200MOE_ROUTER_ST || probs != nullptr, B200MOE_ERR_CONFIG, "st needs probs");
#define CALL(EP) router_dh_kernel<EP, 1><<<ceil_div(T, 256), 256, 0, stream>>>(                                 \
        nullptr, nullptr, dgates, nullptr, 0, 0, gates, probs, nullptr, nullptr, T, E, router_type, dh, nullptr, \
        nullptr, 1)
    if (E <= 4) CALL(4);
    else if (E <= 8) CALL(8);
    else if (E <= 16) CALL(16);
    else CALL(32);
#undef CALL
    B200_CHECK_LAUNCH("gate_bwd");
    return B200MOE_OK;
}


int b200moe_router_logits_bwd(const void* x, const float* dh, const float* w_g, const float* w_noise, const float* z,
                              const float* noise_act, int T, int H, int E, void* dx, float* dw_g, float* dw_noise,
                              float* dn, float* workspace, cudaStream_t stream) {
    B200_CHECK_ARG(T >= 1 && E >= 1 && E <= 32, B200MOE_ERR_CONFIG, "bad T/E (%d, %d)", T, E);
    B200_CHECK_ARG(H >= 8 && H % 8 == 0, B200MOE_ERR_SHAPE, "hidden must be a multiple of 8, got %d", H);
    B200_CHECK_ARG(z == nullptr || (w_noise && noise_act && dn), B200MOE_ERR_CONFIG, "noise args missing");
#define CALL(EP) router_logits_bwd_impl<EP>(x, dh, w_g, w_noise, z, noise_act, T, H, E, dx, dw_g, dw_noise, dn, \
                                            workspace, stream)
    if (E <= 4) return CALL(4);
    if (E <= 8) return CALL(8);
    if (E <= 16) return CALL(16);
    return CALL(32);
#undef CALL
}

int b200moe_importance_fwd(const float* gates, int T, int E, float* imp, float* loss, int32_t* err_flag,
                           cudaStream_t stream) {
    B200_CHECK_ARG(T >= 1 && E >= 1, B200MOE_ERR_SHAPE, "importance penalty needs a [T, E] gate matrix");
    importance_fwd_kernel<<<1, 1024, 0, stream>>>(gates, T, E, imp, loss, err_flag);
    B200_CHECK_LAUNCH("importance_fwd");
    return B200MOE_OK;
}

int b200moe_importance_loss(const float* imp, int E, float* loss, int32_t* err_flag, cudaStream_t stream) {
    B200_CHECK_ARG(E >= 1, B200MOE_ERR_SHAPE, "E >= 1");
    importance_loss_kernel<<<1, 32, 0, stream>>>(imp, E, loss, err_flag);
    B200_CHECK_LAUNCH("importance_loss");
    return B200MOE_OK;
}

int b200moe_importance_bwd(const float* imp, const float* gscale, int E, float* dimp, cudaStream_t stream) {
    B200_CHECK_ARG(E >= 1, B200MOE_ERR_SHAPE, "E >= 1");
    importance_bwd_kernel<<<1, 32, 0, stream>>>(imp, gscale, E, dimp);
    B200_CHECK_LAUNCH("importance_bwd");
    return B200MOE_OK;
}

}  // extern "C"
