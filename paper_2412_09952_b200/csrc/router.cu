// Router forward (K1), gating from logits, and capacity dispatch (K1b).
//
// Reference semantics (moefold):
//   logits   moe.py:136-149   h = x.W_g (+ z * softplus(x.W_noise))
//   top-k    moe.py:152-162   stable argsort(-h): ties -> lowest index, NaN last
//   mixtral  moe.py:171-173   softmax over the kept k (tensor.py:267-297)
//   st       moe.py:176-186   softmax over all E, times the logit top-k mask
//   dispatch moe.py:206-240   slot iff gate > 0; capacity by token position or
//                             by gate (stable, position breaks ties)
// The gate arithmetic reproduces numpy float32 bit-for-bit: numpy's exp
// (npexp.cuh), its pairwise row sum, IEEE division, no FTZ.
#include <atomic>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <math.h>

#include "common.cuh"
#include "ptx.cuh"
#include "npexp.cuh"

namespace b200moe {

constexpr int kMaxE = 32;

// ---------------------------------------------------------------- gating core
// numpy's pairwise sum of a contiguous row of n <= 128 float32 values
// (numpy/_core/src/umath/loops_utils.h.src pairwise_sum).
template <int EP>
__device__ __forceinline__ float np_rowsum(const float (&v)[EP], int n) {
    if (n < 8) {
        float r = 0.0f;
#pragma unroll
        for (int i = 0; i < EP; ++i)
            if (i < n) r = __fadd_rn(r, v[i]);
        return r;
    }
    float r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = (j < EP) ? v[j % EP] : 0.f;
    int full = n - (n % 8);
#pragma unroll
    for (int i = 8; i < EP; i += 8) {
        if (i < full) {
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], v[(i + j) % EP]);
        }
    }
    float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                          __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
#pragma unroll
    for (int i = 8; i < EP; ++i)
        if (i >= full && i < n) res = __fadd_rn(res, v[i]);
    return res;
}

// Compute gates (and st probs) of one token from its E logits. Returns false on
// a GateError row (no finite kept entry).
template <int EP>
__device__ __forceinline__ bool gate_row(const float (&h)[EP], int E, int k, int router_type, float (&g)[EP],
                                         float (&p)[EP], uint32_t* sel_out = nullptr) {
    // ---- stable top-k on -h (NaN last)
    uint32_t sel = 0;
    for (int it = 0; it < k; ++it) {
        int best = -1;
        float bv = 0.f;
#pragma unroll
        for (int e = 0; e < EP; ++e) {
            if (e >= E || (sel >> e) & 1u) continue;
            const float v = h[e];
            if (best < 0) { best = e; bv = v; continue; }
            const bool bnan = (bv != bv), vnan = (v != v);
            if ((bnan && !vnan) || (!bnan && !vnan && v > bv)) { best = e; bv = v; }
        }
        sel |= 1u << best;
    }
    if (sel_out) *sel_out = sel;
    // ---- softmax keep mask
    uint32_t keep = 0;
#pragma unroll
    for (int e = 0; e < EP; ++e) {
        if (e >= E) continue;
        const bool fin = isfinite(h[e]);
        if (router_type == B200MOE_ROUTER_MIXTRAL) { if (fin && ((sel >> e) & 1u)) keep |= 1u << e; }
        else if (fin) keep |= 1u << e;
    }
    if (keep == 0) {
#pragma unroll
        for (int e = 0; e < EP; ++e) { g[e] = 0.f; p[e] = 0.f; }
        return false;
    }
    float mx = -INFINITY;
#pragma unroll
    for (int e = 0; e < EP; ++e)
        if ((keep >> e) & 1u) mx = fmaxf(mx, h[e]);
    float ev[EP];
#pragma unroll
    for (int e = 0; e < EP; ++e) ev[e] = ((keep >> e) & 1u) ? np_expf(__fsub_rn(h[e], mx)) : 0.0f;
    const float den = np_rowsum<EP>(ev, E);
#pragma unroll
    for (int e = 0; e < EP; ++e) {
        const float pe = __fdiv_rn(ev[e], den);
        p[e] = pe;
        if (router_type == B200MOE_ROUTER_MIXTRAL) g[e] = pe;
        else g[e] = __fmul_rn(pe, ((sel >> e) & 1u) ? 1.0f : 0.0f);
    }
    return true;
}

// ---------------------------------------------------------------- K1
// Swizzle W [H, E] (fp32) into float4 blocks laid out so that lane-consecutive
// 8-wide h-blocks are address-consecutive: index ((j * (EP/4) + e4) * (H/8) + hb),
// h = hb*8 + j.
template <int EP>
__global__ void swizzle_w_kernel(const float* __restrict__ w, int H, int E, float4* __restrict__ out) {
    const int n = (H / 8) * 8 * (EP / 4);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int hb = i % (H / 8);
        const int rest = i / (H / 8);
        const int e4 = rest % (EP / 4);
        const int j = rest / (EP / 4);
        const int h = hb * 8 + j;
        float v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int e = e4 * 4 + c;
            v[c] = (e < E) ? w[(size_t)h * E + e] : 0.f;
        }
        out[i] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

// Butterfly reduce-scatter: 32 values per lane -> lane l holds the warp sum of value l.
__device__ __forceinline__ float reduce_scatter32(float (&v)[32]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 16, n = 32; o >= 1; o >>= 1, n >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < n / 2; ++i) {
            const float send = upper ? v[i] : v[i + n / 2];
            const float keep = upper ? v[i + n / 2] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}

constexpr int kRouterThreads = 512;

template <int EP, bool kNoise, bool kSmemW>
__global__ void __launch_bounds__(kRouterThreads, 1)
router_fwd_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ w_g, float4* __restrict__ wsw,
                  const float4* __restrict__ wnsw,
                  const float* __restrict__ z, int T, int H, int E, int k, int router_type,
                  float* __restrict__ logits, float* __restrict__ gates, float* __restrict__ probs,
                  float* __restrict__ noise_act, int32_t* __restrict__ err_flag) {
    constexpr int TT = 32 / EP;  // tokens per warp iteration
    extern __shared__ float4 smem_w[];
    const int nvec = H * EP / 4;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    const int HB = H / 8;
    const int tfirst = (blockIdx.x * (blockDim.x >> 5) + warp) * TT;
    // first x chunk in flight before the W staging below
    uint4 cur[TT];
#pragma unroll
    for (int tt = 0; tt < TT; ++tt)
        cur[tt] = (lane < HB && tfirst + tt < T) ? ld_nc_v4(x + (size_t)(tfirst + tt) * H + lane * 8)
                                                 : make_uint4(0, 0, 0, 0);
    const float4* W = wsw;
    if constexpr (kSmemW) {
        // Every block swizzles W_g [H, E] straight into shared memory (no
        // separate swizzle launch): all loads of a thread are issued before any
        // store, and each block also writes its 1/gridDim slice of the table to
        // `wsw`, where the router backward reuses it.
        constexpr int kPer = 8;
        const int nb = gridDim.x;
        const int s0 = (int)((long long)nvec * blockIdx.x / nb), s1 = (int)((long long)nvec * (blockIdx.x + 1) / nb);
        for (int i0 = threadIdx.x; i0 < nvec; i0 += kPer * blockDim.x) {
            float4 v[kPer];
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int i = i0 + u * blockDim.x;
                v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (i < nvec) {
                    const int hb = i % HB, rest = i / HB, e4 = rest % (EP / 4), j = rest / (EP / 4);
                    const float* src = w_g + (size_t)(hb * 8 + j) * E + e4 * 4;
                    if (E % 4 == 0) v[u] = __ldg(reinterpret_cast<const float4*>(src));
                    else {
                        float t[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) t[c] = (e4 * 4 + c < E) ? __ldg(src + c) : 0.f;
                        v[u] = make_float4(t[0], t[1], t[2], t[3]);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int i = i0 + u * blockDim.x;
                if (i < nvec) {
                    smem_w[i] = v[u];
                    if (i >= s0 && i < s1) wsw[i] = v[u];
                }
            }
        }
        __syncthreads();
        W = smem_w;
    }

    for (int t0 = tfirst; t0 < T; t0 += nwarps * TT) {
        float acc[32], accn[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) { acc[i] = 0.f; accn[i] = 0.f; }
        // software-pipelined: the next chunk's 16-byte loads are in flight while
        // the current chunk is multiplied
        if (t0 != tfirst) {
#pragma unroll
            for (int tt = 0; tt < TT; ++tt)
                cur[tt] = (lane < HB && t0 + tt < T) ? ld_nc_v4(x + (size_t)(t0 + tt) * H + lane * 8)
                                                     : make_uint4(0, 0, 0, 0);
        }
        for (int hb = lane; hb < HB; hb += 32) {
            uint4 nxt[TT];
            const int hn = hb + 32;
#pragma unroll
            for (int tt = 0; tt < TT; ++tt)
                nxt[tt] = (hn < HB && t0 + tt < T) ? ld_nc_v4(x + (size_t)(t0 + tt) * H + hn * 8)
                                                   : make_uint4(0, 0, 0, 0);
            float xv[TT][8];
#pragma unroll
            for (int tt = 0; tt < TT; ++tt) unpack8(cur[tt], xv[tt]);
#pragma unroll
            for (int tt = 0; tt < TT; ++tt) cur[tt] = nxt[tt];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
#pragma unroll
                for (int e4 = 0; e4 < EP / 4; ++e4) {
                    const float4 w = W[(j * (EP / 4) + e4) * HB + hb];
#pragma unroll
                    for (int tt = 0; tt < TT; ++tt) {   // two FFMA2 per (token, 4 experts): same fmaf order
                        float* a = acc + tt * EP + e4 * 4;
                        const float2 xx = make_float2(xv[tt][j], xv[tt][j]);
                        float2 lo = make_float2(a[0], a[1]), hi = make_float2(a[2], a[3]);
                        ffma2(lo, xx, make_float2(w.x, w.y));
                        ffma2(hi, xx, make_float2(w.z, w.w));
                        a[0] = lo.x; a[1] = lo.y; a[2] = hi.x; a[3] = hi.y;
                    }
                    if constexpr (kNoise) {
                        const float4 wn = __ldg(&wnsw[(j * (EP / 4) + e4) * HB + hb]);
#pragma unroll
                        for (int tt = 0; tt < TT; ++tt) {
                            float* a = accn + tt * EP + e4 * 4;
                            const float2 xx = make_float2(xv[tt][j], xv[tt][j]);
                            float2 lo = make_float2(a[0], a[1]), hi = make_float2(a[2], a[3]);
                            ffma2(lo, xx, make_float2(wn.x, wn.y));
                            ffma2(hi, xx, make_float2(wn.z, wn.w));
                            a[0] = lo.x; a[1] = lo.y; a[2] = hi.x; a[3] = hi.y;
                        }
                    }
                }
            }
        }
        // lane l now owns value l: token t0 + l / EP, expert l % EP
        float hv = reduce_scatter32(acc);
        const int tt_mine = lane / EP;
        const int e_mine = lane % EP;
        const int t_mine = t0 + tt_mine;
        const bool live = (t_mine < T) && (e_mine < E);
        if constexpr (kNoise) {
            const float an = reduce_scatter32(accn);
            if (live) {
                const float zz = z[(size_t)t_mine * E + e_mine];
                const float sp = fmaxf(an, 0.f) + log1pf(expf(-fabsf(an)));
                hv = hv + zz * sp;
                noise_act[(size_t)t_mine * E + e_mine] = an;
            }
        }
        if (live) logits[(size_t)t_mine * E + e_mine] = hv;
        // gather this token's row inside its EP-lane group
        float row[EP];
        const int gbase = tt_mine * EP;
#pragma unroll
        for (int e = 0; e < EP; ++e) row[e] = __shfl_sync(0xffffffffu, hv, gbase + e);
        float g[EP], p[EP];
        const bool ok = gate_row<EP>(row, E, k, router_type, g, p);
        if (live) {
            float ge = 0.f, pe = 0.f;
#pragma unroll
            for (int e = 0; e < EP; ++e)
                if (e == e_mine) { ge = g[e]; pe = p[e]; }
            gates[(size_t)t_mine * E + e_mine] = ge;
            if (probs) probs[(size_t)t_mine * E + e_mine] = pe;
            if (!ok && e_mine == 0 && err_flag) atomicExch(err_flag, 1);
        }
    }
}

// ---------------------------------------------------------------- K1 on tcgen05
// The router GEMV h = x . W_g (+ x . W_noise) on the tensor cores.  W (fp32)
// is split into three bf16 parts, W = W_hi + W_mid + W_lo, each the bf16
// rounding of what the previous parts leave (together within 2^-24 of W); x
// is bf16, so every product x * W_s is exact and the MMA accumulates in fp32.
// B = [W_hi | W_mid | W_lo (| noise parts)]^T is stacked along N, so a CTA's
// accumulator row t holds x_t . W_s[:, e] in column s*EP + e; the epilogue adds
// the parts smallest first and runs the gating of K1 on its token.  A CTA owns
// 128 tokens: x streams through an 8-deep TMA ring (SWIZZLE_128B, 64 hidden per
// stage), one thread issues 4 MMAs (K = 16) per stage, and the 128 threads of
// the epilogue each own one token (TMEM lane).  The CUDA-core K1 above stays
// for E > 16 (N would exceed the TMEM budget of this layout).
template <int EP, bool kNoise, int CS = 2>
struct RtcCfg {
    static constexpr int NB = ((3 * EP + 15) / 16) * 16;   // B rows per matrix (3 splits, padded)
    static constexpr int N = kNoise ? 2 * NB : NB;
    // cluster of CS CTAs per 128-token tile, CTA r streaming the r-th hidden
    // slice; with 4 the ring is halved so two CTAs share an SM (256 CTAs on 148
    // SMs at T = 8192 instead of 128), and must still hold the 3 peers' partials
    static constexpr int kStages = CS == 2 ? 8 : 4;
    static constexpr int kABytes = 128 * 64 * 2;         // 16 KB of x per stage
    static constexpr int kBBytes = N * 64 * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kTmemCols = N <= 32 ? 32 : (N <= 64 ? 64 : 128);
    static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
    static_assert((CS - 1) * N * 128 * 4 <= kStages * kStageBytes, "the drained ring holds the peers' partials");
};

// W_g / W_noise [H, E] fp32 -> the bf16 split table B [N, H] (row s*EP + e of
// matrix block m: part s of column e; unused rows zero) and the swizzled fp32
// tables the router backward reads (same layout as swizzle_w_kernel).
template <int EP, bool kNoise>
__global__ void router_wsplit_kernel(const float* __restrict__ w_g, const float* __restrict__ w_n, int H, int E,
                                     __nv_bfloat16* __restrict__ bsplit, float4* __restrict__ wsw,
                                     float4* __restrict__ wnsw) {
    using C = RtcCfg<EP, kNoise>;
    const int HB = H / 8;
    for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x) {
#pragma unroll
        for (int m = 0; m < (kNoise ? 2 : 1); ++m) {
            const float* w = m == 0 ? w_g : w_n;
            float v[EP];
#pragma unroll
            for (int e = 0; e < EP; ++e) v[e] = (e < E) ? w[(size_t)h * E + e] : 0.f;
            __nv_bfloat16* b = bsplit + (size_t)m * C::NB * H;
#pragma unroll
            for (int e = 0; e < EP; ++e) {
                const __nv_bfloat16 hi = __float2bfloat16_rn(v[e]);
                const float r1 = v[e] - __bfloat162float(hi);
                const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
                const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
                b[(size_t)e * H + h] = hi;
                b[(size_t)(EP + e) * H + h] = mid;
                b[(size_t)(2 * EP + e) * H + h] = lo;
            }
            for (int r = 3 * EP; r < C::NB; ++r) b[(size_t)r * H + h] = __float2bfloat16_rn(0.f);
            float4* sw = m == 0 ? wsw : wnsw;
            const int hb = h / 8, j = h % 8;
#pragma unroll
            for (int e4 = 0; e4 < EP / 4; ++e4)
                sw[(j * (EP / 4) + e4) * HB + hb] = make_float4(v[4 * e4], v[4 * e4 + 1], v[4 * e4 + 2], v[4 * e4 + 3]);
        }
    }
}

template <int EP, bool kNoise, int CS>
__global__ void __launch_bounds__(128, 1)
router_fwd_tc_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap bmap,
                     const float* __restrict__ z, int T, int H, int E, int k, int router_type,
                     float* __restrict__ logits, float* __restrict__ gates, float* __restrict__ probs,
                     float* __restrict__ noise_act, int32_t* __restrict__ err_flag) {
    using C = RtcCfg<EP, kNoise, CS>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
    uint64_t* empty = full + C::kStages;
    uint64_t* done = empty + C::kStages;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // a cluster of CS CTAs shares one 128-token tile: CTA r accumulates the
    // hidden slice r (CS times the SMs streaming x), then CTAs 1..CS-1 hand
    // their partial sums to CTA 0 through distributed shared memory
    const uint32_t crank = ptx::cluster_ctarank();
    const int t0 = (int)ptx::cluster_id_x() * 128;
    const int nkb_all = H / 64;
    const int per = nkb_all / CS;
    const int kb0 = (int)crank * per;
    const int nkb = (int)crank == CS - 1 ? nkb_all - per * (CS - 1) : per;
    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&xmap);
        ptx::prefetch_tmap(&bmap);
        for (int s = 0; s < C::kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(done, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc<1>(tslot, C::kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == 0 && lane == 0) {            // TMA producer: x tile + split-B tile per stage
        for (int kb = 0; kb < nkb; ++kb) {
            const int st = kb % C::kStages;
            if (kb >= C::kStages) ptx::mbar_wait(&empty[st], ((kb / C::kStages) - 1) & 1);
            uint8_t* a = smem + st * C::kStageBytes;
            ptx::mbar_arrive_expect_tx(&full[st], C::kStageBytes);   // rows beyond T arrive as zeros
            ptx::tma_load_2d(&xmap, &full[st], a, (kb0 + kb) * 64, t0);
            ptx::tma_load_2d(&bmap, &full[st], a + C::kABytes, (kb0 + kb) * 64, 0);
        }
    } else if (warp == 1 && lane == 0) {     // MMA issuer
        constexpr uint32_t idesc = ptx::make_idesc_bf16(128, C::N, false, false);
        for (int kb = 0; kb < nkb; ++kb) {
            const int st = kb % C::kStages;
            ptx::mbar_wait(&full[st], (kb / C::kStages) & 1);
            ptx::tc_fence_after();
            const uint32_t a = ptx::smem_u32(smem + st * C::kStageBytes);
            const uint32_t b = a + C::kABytes;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                ptx::mma_bf16<1>(tmem, ptx::make_sdesc(a + kk * 32, 16, 1024), ptx::make_sdesc(b + kk * 32, 16, 1024),
                                 idesc, (kb | kk) != 0);
            ptx::mma_commit<1>(&empty[st], 1);
        }
        ptx::mma_commit<1>(done, 1);
    }
    // ---- epilogue: thread i owns token t0 + i (TMEM lane i)
    ptx::mbar_wait(done, 0);
    ptx::tc_fence_after();
    constexpr int kLoads = (C::N + 31) / 32;
    uint32_t d[kLoads * 32];
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll
    for (int c = 0; c < kLoads; ++c) ptx::tmem_ld_32x32b_x32(lane_addr + c * 32, d + c * 32);
    ptx::tmem_ld_wait();
    // cross-CTA reduction over the hidden slices: every ring is drained
    // (barrier 1), CTA r > 0 stores its partials into CTA 0's ring memory
    // (block r - 1, [column][row] floats, conflict-free), barrier 2, CTA 0
    // adds them in rank order
    float* red = reinterpret_cast<float*>(smem);
    ptx::cluster_sync();
    if (crank != 0) {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(ptx::smem_u32(red)));
        remote += (crank - 1) * (uint32_t)(C::N * 128 * 4);
#pragma unroll
        for (int c = 0; c < C::N; ++c)
            asm volatile("st.shared::cluster.f32 [%0], %1;" :: "r"(remote + (uint32_t)(c * 128 + threadIdx.x) * 4u),
                         "f"(__uint_as_float(d[c])) : "memory");
    }
    ptx::cluster_sync();
    if (crank != 0) {
        ptx::tc_fence_before();
        __syncthreads();
        if (warp == 1) {
            ptx::tc_fence_after();
            ptx::tmem_dealloc<1>(tmem, C::kTmemCols);
        }
        return;
    }
#pragma unroll
    for (int r = 0; r < CS - 1; ++r)
#pragma unroll
        for (int c = 0; c < C::N; ++c)
            d[c] = __float_as_uint(__uint_as_float(d[c]) + red[(r * C::N + c) * 128 + threadIdx.x]);
    const int t = t0 + threadIdx.x;
    float row[EP];
#pragma unroll
    for (int e = 0; e < EP; ++e) {
        float hv = (__uint_as_float(d[2 * EP + e]) + __uint_as_float(d[EP + e])) + __uint_as_float(d[e]);
        if constexpr (kNoise) {
            const int o = C::NB;
            const float an = (__uint_as_float(d[o + 2 * EP + e]) + __uint_as_float(d[o + EP + e])) +
                             __uint_as_float(d[o + e]);
            if (t < T && e < E) {
                const float zz = z[(size_t)t * E + e];
                const float sp = fmaxf(an, 0.f) + log1pf(expf(-fabsf(an)));
                hv = hv + zz * sp;
                noise_act[(size_t)t * E + e] = an;
            }
        }
        row[e] = hv;
        if (t < T && e < E) logits[(size_t)t * E + e] = hv;
    }
    if (t < T) {
        float g[EP], p[EP];
        const bool ok = gate_row<EP>(row, E, k, router_type, g, p);
#pragma unroll
        for (int e = 0; e < EP; ++e) {
            if (e < E) {
                gates[(size_t)t * E + e] = g[e];
                if (probs) probs[(size_t)t * E + e] = p[e];
            }
        }
        if (!ok && err_flag) atomicExch(err_flag, 1);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<1>(tmem, C::kTmemCols);
    }
}

template <int EP>
__global__ void gate_from_logits_kernel(const float* __restrict__ logits, int T, int E, int k, int router_type,
                                        float* __restrict__ gates, float* __restrict__ probs,
                                        uint8_t* __restrict__ topk, int32_t* __restrict__ err_flag) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
        float h[EP], g[EP], p[EP];
#pragma unroll
        for (int e = 0; e < EP; ++e) h[e] = (e < E) ? logits[(size_t)t * E + e] : 0.f;
        uint32_t sel = 0;
        const bool ok = gate_row<EP>(h, E, k, router_type, g, p, &sel);
        if (!ok) atomicExch(err_flag, 1);
#pragma unroll
        for (int e = 0; e < EP; ++e) {
            if (e < E) {
                gates[(size_t)t * E + e] = g[e];
                if (probs) probs[(size_t)t * E + e] = p[e];
                if (topk) topk[(size_t)t * E + e] = (sel >> e) & 1u;
            }
        }
    }
}

// ---------------------------------------------------------------- K1b dispatch
constexpr int kDispThreads = 1024;
constexpr int kDispItems = 8;  // tokens per thread per chunk

// Block-wide exclusive scan of one int per thread; returns the prefix and
// writes the block total to *total.
__device__ __forceinline__ int block_excl_scan(int v, int* sm, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n;
    }
    __syncthreads();
    if (lane == 31) sm[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = (lane < nw) ? sm[lane] : 0;
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int n = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += n;
        }
        if (lane < nw) sm[lane] = wi - w;
        if (lane == 31) sm[32] = wi;
    }
    __syncthreads();
    const int res = sm[warp] + incl - v;
    *total = sm[32];
    return res;
}

__device__ __forceinline__ float block_sum_f(float v, float* sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sm[warp] = v;
    __syncthreads();
    float r = 0.f;
    if (warp == 0) {
        r = (lane < nw) ? sm[lane] : 0.f;
        r = warp_sum(r);
        if (lane == 0) sm[0] = r;
    }
    __syncthreads();
    r = sm[0];
    return r;
}

__global__ void __launch_bounds__(kDispThreads)
dispatch_kernel(const float* __restrict__ gates, int T, int E, int capacity, int policy, int layout, int seg_stride,
                int32_t* __restrict__ slot_rank, int32_t* __restrict__ counts, int32_t* __restrict__ seg_base,
                float* __restrict__ gate_mass, float* __restrict__ importance, int64_t* __restrict__ stats,
                int32_t* __restrict__ ws) {
    __shared__ int sm_i[40];
    __shared__ float sm_f[40];
    __shared__ int hist[256];
    __shared__ int sel_info[4];
    __shared__ bool am_last;
    const int e = blockIdx.x;
    const int chunk = kDispThreads * kDispItems;
    const bool dropless = capacity < 0;

    int nslots = 0, kept_total = 0;
    float imp = 0.f, mass = 0.f;
    if (T <= chunk && (dropless || policy == B200MOE_POLICY_POSITION)) {
        // ---- one chunk, position policy: a kept slot's rank is its slot index, so one scan
        // gives counts, ranks and the capacity cut (same per-thread and block summation
        // order for importance and gate mass as the general path below)
        float gv[kDispItems];
        int c = 0;
#pragma unroll
        for (int i = 0; i < kDispItems; ++i) {
            const int t = threadIdx.x * kDispItems + i;
            gv[i] = (t < T) ? gates[(size_t)t * E + e] : 0.f;
            imp += (t < T) ? gv[i] : 0.f;
            c += gv[i] > 0.f;
        }
        int sp = block_excl_scan(c, sm_i, &nslots);
#pragma unroll
        for (int i = 0; i < kDispItems; ++i) {
            const int t = threadIdx.x * kDispItems + i;
            int r = -1;
            if (gv[i] > 0.f) {
                if (dropless || sp < capacity) { r = sp; mass += gv[i]; }
                ++sp;
            }
            if (t < T) slot_rank[(size_t)t * E + e] = r;
        }
        kept_total = dropless ? nslots : min(nslots, capacity);
        imp = block_sum_f(imp, sm_f);
        mass = block_sum_f(mass, sm_f);
    } else {
    // ---- pass 1: slot count and importance
    for (int base = 0; base < T; base += chunk) {
        int c = 0;
        for (int i = 0; i < kDispItems; ++i) {
            const int t = base + threadIdx.x * kDispItems + i;
            if (t < T) {
                const float g = gates[(size_t)t * E + e];
                imp += g;
                c += (g > 0.f);
            }
        }
        int tot;
        block_excl_scan(c, sm_i, &tot);
        nslots += tot;
    }
    imp = block_sum_f(imp, sm_f);

    // ---- score policy with overflow: radix-select the capacity-th largest gate
    const bool select = (policy == B200MOE_POLICY_SCORE) && !dropless && nslots > capacity;
    uint32_t thr = 0;
    int need_ties = 0;
    if (select) {
        uint32_t prefix = 0, pmask = 0;
        int remaining = capacity;  // how many of the matching keys we still take
        for (int shift = 24; shift >= 0; shift -= 8) {
            for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
            __syncthreads();
            for (int t = threadIdx.x; t < T; t += blockDim.x) {
                const float g = gates[(size_t)t * E + e];
                if (g > 0.f) {
                    const uint32_t key = __float_as_uint(g);
                    if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int cum = 0, d = 255;
                for (; d > 0; --d) {
                    if (cum + hist[d] >= remaining) break;
                    cum += hist[d];
                }
                sel_info[0] = d;
                sel_info[1] = remaining - cum;
            }
            __syncthreads();
            prefix |= (uint32_t)sel_info[0] << shift;
            pmask |= 255u << shift;
            remaining = sel_info[1];
            __syncthreads();
        }
        thr = prefix;
        need_ties = remaining;  // number of keys == thr to keep (in token order)
    }

    // ---- pass 2: kept flags and ranks in token order
    int ties_seen = 0, slots_seen = 0;
    for (int base = 0; base < T; base += chunk) {
        float gv[kDispItems];
        int nslot = 0, ntie = 0;
        for (int i = 0; i < kDispItems; ++i) {
            const int t = base + threadIdx.x * kDispItems + i;
            gv[i] = (t < T) ? gates[(size_t)t * E + e] : 0.f;
            nslot += gv[i] > 0.f;
            ntie += (select && gv[i] > 0.f && __float_as_uint(gv[i]) == thr);
        }
        int tot_slot, tot_tie;
        const int slot_pre = block_excl_scan(nslot, sm_i, &tot_slot) + slots_seen;
        int tie_pre = 0;
        if (select) tie_pre = block_excl_scan(ntie, sm_i, &tot_tie) + ties_seen;
        // decide kept per item
        int kflags = 0, nk = 0;
        int sp = slot_pre, tp = tie_pre;
        for (int i = 0; i < kDispItems; ++i) {
            bool kept = false;
            if (gv[i] > 0.f) {
                if (dropless) kept = true;
                else if (!select) kept = sp < capacity;
                else {
                    const uint32_t key = __float_as_uint(gv[i]);
                    if (key > thr) kept = true;
                    else if (key == thr) { kept = tp < need_ties; ++tp; }
                }
                ++sp;
            }
            if (kept) { kflags |= 1 << i; ++nk; mass += gv[i]; }
        }
        int tot_kept;
        int kp = block_excl_scan(nk, sm_i, &tot_kept) + kept_total;
        for (int i = 0; i < kDispItems; ++i) {
            const int t = base + threadIdx.x * kDispItems + i;
            if (t < T) slot_rank[(size_t)t * E + e] = ((kflags >> i) & 1) ? kp++ : -1;
        }
        kept_total += tot_kept;
        slots_seen += tot_slot;
        if (select) ties_seen += tot_tie;
    }
    mass = block_sum_f(mass, sm_f);
    }

    if (threadIdx.x == 0) {
        counts[e] = kept_total;
        gate_mass[e] = mass;
        importance[e] = imp;
        ws[8 + e] = nslots;
        __threadfence();
        const int ticket = atomicAdd(&ws[0], 1);
        am_last = (ticket == (int)gridDim.x - 1);
    }
    __syncthreads();
    if (am_last) {   // GateError rows (all gates zero) over the whole batch, for stats[2]
        bool zero = false;
        for (int t = threadIdx.x; t < T; t += blockDim.x) {
            bool z = true;
            for (int i = 0; i < E; ++i) z &= !(gates[(size_t)t * E + i] > 0.f);
            zero |= z;
        }
        zero = __syncthreads_or(zero);
        if (threadIdx.x == 0) stats[2] = zero ? 1 : 0;
    }
    if (am_last && threadIdx.x == 0) {
        __threadfence();
        int acc = 0;
        long long dropped = 0, total = 0;
        for (int i = 0; i < E; ++i) {
            const int c = ((volatile int32_t*)counts)[i];
            const int s = ((volatile int32_t*)ws)[8 + i];
            seg_base[i] = (layout == B200MOE_LAYOUT_FIXED) ? i * seg_stride : acc;
            acc += round_up(c, kSegPad);
            dropped += s - c;
            total += s;
        }
        stats[0] = dropped;
        stats[1] = total;
        ws[0] = 0;  // reset the ticket for the next launch
    }
}

__global__ void importance_loss_kernel_fwd(const float* __restrict__ imp, int E, float* __restrict__ loss,
                                           int32_t* __restrict__ err_flag) {
    if (threadIdx.x == 0) importance_cv2(imp, E, loss, err_flag);
}

// ---------------------------------------------------------------- K1b fast path
// Position policy (and dropless): a kept slot's rank is its index among the
// expert's slots in token order, so capacity needs only a prefix count over
// tokens.  One CTA per 256-token tile (tile ids taken from an atomic counter,
// so tiles start in order): each thread holds one token's row of gates
// (coalesced), a block scan gives in-tile slot ranks for all experts at once
// (four 16-bit counters per 64-bit word), and a decoupled look-back over the
// tiles' published per-expert aggregates / inclusive prefixes gives the
// cross-tile offset.  Per-tile sums of gates (importance) and kept gates
// (gate mass) are reduced in fixed tile order by the last CTA, which also
// writes counts, seg_base, drop stats and the importance (CV^2) loss.
// Workspace (int32 words, zero-initialised once): [0] ticket, [1] tile counter,
// [2] epoch, [8..8+40) per-expert slot totals, then status words (uint64,
// [tile][EP]) and per-tile partial sums (float2, [tile][EP]).
#ifndef B200_SCAN_TILE
#define B200_SCAN_TILE 256
#endif
constexpr int kScanTile = B200_SCAN_TILE;
constexpr int kWsStatus = 64;   // int32 offset of the status words (8-byte aligned)

__host__ __device__ constexpr size_t dispatch_ws_words(int T) {
    return (size_t)kWsStatus + (size_t)((T + kScanTile - 1) / kScanTile) * kMaxE * 4;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

template <int EP>
__global__ void __launch_bounds__(kScanTile)
dispatch_scan_kernel(const float* __restrict__ gates, int T, int E, int capacity, int layout, int seg_stride,
                     int32_t* __restrict__ slot_rank, int32_t* __restrict__ counts, int32_t* __restrict__ seg_base,
                     float* __restrict__ gate_mass, float* __restrict__ importance, int64_t* __restrict__ stats,
                     float* __restrict__ imp_loss, int32_t* __restrict__ imp_err, int32_t* __restrict__ ws) {
    constexpr int NW = EP / 4;                      // 64-bit words of four 16-bit counters
    constexpr int kWarps = kScanTile / 32;
    __shared__ unsigned long long wsum[kWarps][NW];
    __shared__ int excl_sh[EP];
    __shared__ float red_sh[2][kWarps][EP];
    __shared__ int tile_sh;
    __shared__ bool last_sh;
    const int ntiles = (T + kScanTile - 1) / kScanTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long* status = reinterpret_cast<unsigned long long*>(ws + kWsStatus);
    float2* part = reinterpret_cast<float2*>(status + (size_t)ntiles * EP);
    if (threadIdx.x == 0) tile_sh = atomicAdd(&ws[1], 1);
    __syncthreads();
    const int tile = tile_sh;
    const unsigned epoch = ((volatile unsigned*)ws)[2];
    const int t = tile * kScanTile + threadIdx.x;
    const bool dropless = capacity < 0;

    // ---- this token's gates (E contiguous floats) and slot flags
    float g[EP];
#pragma unroll
    for (int e = 0; e < EP; ++e) g[e] = 0.f;
    if (t < T) {
        if (E == EP) {
#pragma unroll
            for (int q = 0; q < EP / 4; ++q) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(gates + (size_t)t * E) + q);
                g[4 * q] = v.x; g[4 * q + 1] = v.y; g[4 * q + 2] = v.z; g[4 * q + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int e = 0; e < EP; ++e) g[e] = (e < E) ? __ldg(gates + (size_t)t * E + e) : 0.f;
        }
    }
    unsigned long long f[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        f[w] = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) f[w] |= (unsigned long long)(g[4 * w + c] > 0.f) << (16 * c);
    }
    // ---- block exclusive scan of the packed counters
    unsigned long long inc[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        inc[w] = f[w];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long n = __shfl_up_sync(0xffffffffu, inc[w], o);
            if (lane >= o) inc[w] += n;
        }
        if (lane == 31) wsum[warp][w] = inc[w];
    }
    __syncthreads();
    unsigned long long pre[NW], tot[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        pre[w] = 0;
        tot[w] = 0;
        for (int i = 0; i < kWarps; ++i) {
            if (i < warp) pre[w] += wsum[i][w];
            tot[w] += wsum[i][w];
        }
        pre[w] += inc[w] - f[w];
    }
    // ---- decoupled look-back (flag 1 = aggregate, 2 = inclusive prefix).  Every
    // expert's aggregate is published first; then warp w looks back for experts
    // w, w + 8, ...: lane l polls tile (base - l), so a window of 32
    // predecessors costs one round trip, and the nearest inclusive prefix in the
    // window ends the walk.
    const unsigned long long tag = (unsigned long long)epoch << 34;
    if (threadIdx.x < E) {
        const int e = threadIdx.x;
        const unsigned long long agg = (tot[e >> 2] >> (16 * (e & 3))) & 0xFFFFull;
        st_release_u64(status + (size_t)tile * EP + e, tag | ((tile == 0 ? 2ull : 1ull) << 32) | agg);
    }
    for (int e = warp; e < E; e += kWarps) {
        const unsigned long long agg = (tot[e >> 2] >> (16 * (e & 3))) & 0xFFFFull;
        long long excl = 0;
        int base = tile - 1;
        while (base >= 0) {
            const int j = base - lane;
            unsigned long long v = 0;
            if (j >= 0) {
                do {
                    v = ld_acquire_u64(status + (size_t)j * EP + e);
                } while ((v >> 34) != (unsigned long long)epoch || ((v >> 32) & 3ull) == 0);
            }
            const unsigned pmask = __ballot_sync(0xffffffffu, j >= 0 && ((v >> 32) & 3ull) == 2);
            const int stop = pmask ? (__ffs(pmask) - 1) : 31;            // nearest inclusive prefix
            long long val = (j >= 0 && lane <= stop) ? (long long)(v & 0xFFFFFFFFull) : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
            excl += val;
            if (pmask) break;
            base -= 32;
        }
        if (lane == 0) {
            if (tile > 0)
                st_release_u64(status + (size_t)tile * EP + e, tag | (2ull << 32) | (unsigned long long)(excl + agg));
            excl_sh[e] = (int)excl;
            if (tile == ntiles - 1) ws[8 + e] = (int)(excl + (long long)agg);   // total slots of expert e
        }
    }
    __syncthreads();
    // a token row whose gates are all zero is a GateError row (the router found
    // no finite kept logit, tensor.py:283-284): every valid row has a positive
    // top-1 gate.  OR-ed into ws[3], reported in stats[2] by the last CTA.
    {
        bool zero_row = (t < T);
#pragma unroll
        for (int e = 0; e < EP; ++e) zero_row &= !(g[e] > 0.f);
        if (__syncthreads_or(zero_row) && threadIdx.x == 0) atomicOr(&ws[3], 1);
    }
    // ---- ranks, kept flags, per-thread sums
    float imp_e[EP], mass_e[EP];
#pragma unroll
    for (int e = 0; e < EP; ++e) {
        const int r = excl_sh[e < E ? e : 0] + (int)((pre[e >> 2] >> (16 * (e & 3))) & 0xFFFFull);
        const bool slot = g[e] > 0.f;
        const bool kept = slot && (dropless || r < capacity);
        if (t < T && e < E) slot_rank[(size_t)t * E + e] = kept ? r : -1;
        imp_e[e] = g[e];
        mass_e[e] = kept ? g[e] : 0.f;
    }
    // fixed-order block sums: warp butterflies, then warps in order (thread e < E)
#pragma unroll
    for (int e = 0; e < EP; ++e) {
        const float a = warp_sum(imp_e[e]), b = warp_sum(mass_e[e]);
        if (lane == 0) { red_sh[0][warp][e] = a; red_sh[1][warp][e] = b; }
    }
    __syncthreads();
    if (threadIdx.x < E) {
        const int e = threadIdx.x;
        float a = 0.f, b = 0.f;
        for (int i = 0; i < kWarps; ++i) { a += red_sh[0][i][e]; b += red_sh[1][i][e]; }
        part[(size_t)tile * EP + e] = make_float2(a, b);
    }
    // ---- last CTA: fixed-order reduction over tiles, counts, stats, seg_base, loss
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last_sh = (atomicAdd(&ws[0], 1) == ntiles - 1);
    __syncthreads();
    if (!last_sh) return;
    __threadfence();
    // warp w reduces experts w, w + 8, ...: lane l sums tiles l, l + 32, ...
    // (L2 loads, all in flight together), then a butterfly -- a fixed order
    for (int e = warp; e < E; e += kWarps) {
        float a = 0.f, b = 0.f;
        for (int j = lane; j < ntiles; j += 32) {
            const float2 v = __ldcg(part + (size_t)j * EP + e);
            a += v.x;
            b += v.y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
        }
        if (lane == 0) {
            importance[e] = a;
            gate_mass[e] = b;
            const int tot_e = __ldcg(ws + 8 + e);
            counts[e] = dropless ? tot_e : min(tot_e, capacity);
        }
    }
    __syncthreads();
    __threadfence();
    if (threadIdx.x == 0) {
        int acc = 0;
        long long dropped = 0, total = 0;
        for (int i = 0; i < E; ++i) {
            const int c = ((volatile int32_t*)counts)[i];
            const int s = ((volatile int32_t*)ws)[8 + i];
            seg_base[i] = (layout == B200MOE_LAYOUT_FIXED) ? i * seg_stride : acc;
            acc += round_up(c, kSegPad);
            dropped += s - c;
            total += s;
        }
        stats[0] = dropped;
        stats[1] = total;
        stats[2] = ((volatile int32_t*)ws)[3];
        if (imp_loss) importance_cv2(importance, E, imp_loss, imp_err);
        ws[0] = 0;          // ticket
        ws[1] = 0;          // tile counter
        ws[3] = 0;          // error flag
        ws[2] = (int)((epoch + 1) & 0x3FFFFFFFu);
    }
}

}  // namespace b200moe

using namespace b200moe;

namespace {
// Diagnostics (A/B against the CUDA-core K1): thread-local, product default off.
thread_local int g_router_fma = 0;

#ifndef B200_RTC_CS4
#define B200_RTC_CS4 1
#endif
template <int EP, bool kNoise, int CS>
int router_fwd_tc_launch(const CUtensorMap& xmap, const CUtensorMap& bmap, const float* z, int T, int H, int E, int k,
                         int router_type, float* logits, float* gates, float* probs, float* noise_act,
                         int32_t* err_flag, cudaStream_t stream) {
    using C = RtcCfg<EP, kNoise, CS>;
    auto kern = router_fwd_tc_kernel<EP, kNoise, CS>;
    static std::atomic<uint64_t> attr{0};
    if (cudaError_t ae = ensure_smem_attr(kern, C::kSmem, attr); ae != cudaSuccess) {
        set_error("router_fwd_tc smem attribute: %s", cudaGetErrorString(ae));
        return B200MOE_ERR_CUDA;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS * ceil_div(T, 128));
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = stream;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeClusterDimension;
    la[0].val.clusterDim.x = CS;
    la[0].val.clusterDim.y = 1;
    la[0].val.clusterDim.z = 1;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    cudaError_t le = cudaLaunchKernelEx(&cfg, kern, xmap, bmap, z, T, H, E, k, router_type, logits, gates, probs,
                                        noise_act, err_flag);
    if (le != cudaSuccess) {
        set_error("router_fwd_tc launch: %s", cudaGetErrorString(le));
        return B200MOE_ERR_CUDA;
    }
    return B200MOE_OK;
}

template <int EP, bool kNoise>
int router_fwd_tc(const void* x, const float* w_g, const float* w_noise, const float* z, int T, int H, int E, int k,
                  int router_type, float* logits, float* gates, float* probs, float* noise_act, float* workspace,
                  int32_t* err_flag, cudaStream_t stream) {
    using C = RtcCfg<EP, kNoise>;
    float4* wsw = reinterpret_cast<float4*>(workspace);
    float4* wnsw = reinterpret_cast<float4*>(workspace + (size_t)H * EP);
    __nv_bfloat16* bsplit = reinterpret_cast<__nv_bfloat16*>(workspace + (size_t)2 * H * EP);
    router_wsplit_kernel<EP, kNoise><<<ceil_div(H, 256), 256, 0, stream>>>(w_g, w_noise, H, E, bsplit, wsw, wnsw);
    CUtensorMap xmap, bmap;
    int rc = make_tmap_bf16_2d(&xmap, x, (uint64_t)H, (uint64_t)T, (uint64_t)H, 64, 128, true);
    if (rc) return rc;
    rc = make_tmap_bf16_2d(&bmap, bsplit, (uint64_t)H, (uint64_t)C::N, (uint64_t)H, 64, C::N, true);
    if (rc) return rc;
    // four hidden slices per tile (no noise: the peers' partials fit the halved ring)
    if constexpr (!kNoise && B200_RTC_CS4) {
        if (H % 256 == 0)
            return router_fwd_tc_launch<EP, kNoise, 4>(xmap, bmap, z, T, H, E, k, router_type, logits, gates, probs,
                                                       noise_act, err_flag, stream);
    }
    return router_fwd_tc_launch<EP, kNoise, 2>(xmap, bmap, z, T, H, E, k, router_type, logits, gates, probs,
                                               noise_act, err_flag, stream);
}

template <int EP>
int router_fwd_impl(const void* x, const float* w_g, const float* w_noise, const float* z, int T, int H, int E,
                    int k, int router_type, float* logits, float* gates, float* probs, float* noise_act,
                    float* workspace, int32_t* err_flag, cudaStream_t stream) {
    if constexpr (EP <= 16) {   // tensor-core path (H a multiple of 128: two full-width hidden halves)
        if (H % 128 == 0 && !g_router_fma) {
            if (z != nullptr)
                return router_fwd_tc<EP, true>(x, w_g, w_noise, z, T, H, E, k, router_type, logits, gates, probs,
                                               noise_act, workspace, err_flag, stream);
            return router_fwd_tc<EP, false>(x, w_g, w_noise, z, T, H, E, k, router_type, logits, gates, probs,
                                            noise_act, workspace, err_flag, stream);
        }
    }
    float4* wsw = reinterpret_cast<float4*>(workspace);
    float4* wnsw = reinterpret_cast<float4*>(workspace + (size_t)H * EP);
    const size_t wbytes = (size_t)H * EP * sizeof(float);
    const bool smem_w = wbytes <= 160 * 1024;   // else the kernel reads the table from L2
    if (!smem_w) swizzle_w_kernel<EP><<<64, 256, 0, stream>>>(w_g, H, E, wsw);
    const bool noise = z != nullptr;
    if (noise) swizzle_w_kernel<EP><<<64, 256, 0, stream>>>(w_noise, H, E, wnsw);
    constexpr int TT = 32 / EP;
    const int warps_needed = ceil_div(T, TT);
    int grid = ceil_div(warps_needed, kRouterThreads / 32);
    if (grid > kNumSMs) grid = kNumSMs;
    if (grid < 1) grid = 1;
#define LAUNCH(NZ, SM)                                                                                        \
    do {                                                                                                      \
        auto kern = router_fwd_kernel<EP, NZ, SM>;                                                            \
        const size_t sh = SM ? wbytes : 0;                                                                    \
        if (SM) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh);             \
        kern<<<grid, kRouterThreads, sh, stream>>>((const __nv_bfloat16*)x, w_g, wsw, wnsw, z, T, H, E, k,    \
                                                   router_type, logits, gates, probs, noise_act, err_flag);   \
    } while (0)
    if (noise) {
        if (smem_w) LAUNCH(true, true); else LAUNCH(true, false);
    } else {
        if (smem_w) LAUNCH(false, true); else LAUNCH(false, false);
    }
#undef LAUNCH
    B200_CHECK_LAUNCH("router_fwd");
    return B200MOE_OK;
}

template <int EP>
int gate_impl(const float* logits, int T, int E, int k, int router_type, float* gates, float* probs,
              uint8_t* topk, int32_t* err_flag, cudaStream_t stream) {
    int grid = ceil_div(T, 256);
    if (grid > 4 * kNumSMs) grid = 4 * kNumSMs;
    if (grid < 1) grid = 1;
    gate_from_logits_kernel<EP><<<grid, 256, 0, stream>>>(logits, T, E, k, router_type, gates, probs, topk,
                                                           err_flag);
    B200_CHECK_LAUNCH("gate_from_logits");
    return B200MOE_OK;
}

int check_router_args(int T, int H, int E, int k, int router_type) {
    B200_CHECK_ARG(T >= 1, B200MOE_ERR_CONFIG, "tokens_per_batch must be >= 1, got %d", T);
    B200_CHECK_ARG(E >= 1 && E <= kMaxE, B200MOE_ERR_CONFIG, "n_experts must be in [1, %d], got %d", kMaxE, E);
    B200_CHECK_ARG(k >= 1 && k <= E, B200MOE_ERR_CONFIG, "top-k out of range: k=%d, n=%d", k, E);
    B200_CHECK_ARG(router_type == B200MOE_ROUTER_MIXTRAL || router_type == B200MOE_ROUTER_ST, B200MOE_ERR_CONFIG,
                   "router_type %d", router_type);
    B200_CHECK_ARG(H >= 8 && H % 8 == 0, B200MOE_ERR_SHAPE, "hidden must be a multiple of 8, got %d", H);
    return B200MOE_OK;
}
}  // namespace

extern "C" {

int b200moe_router_fwd(const void* x, const float* w_g, const float* w_noise, const float* z, int T, int H, int E,
                       int k, int router_type, float* logits, float* gates, float* probs, float* noise_act,
                       float* workspace, int32_t* err_flag, cudaStream_t stream) {
    int rc = check_router_args(T, H, E, k, router_type);
    if (rc) return rc;
    B200_CHECK_ARG(z == nullptr || (w_noise != nullptr && noise_act != nullptr), B200MOE_ERR_CONFIG,
                   "noise needs w_noise and noise_act");
    if (E <= 4) return router_fwd_impl<4>(x, w_g, w_noise, z, T, H, E, k, router_type, logits, gates, probs, noise_act, workspace, err_flag, stream);
    if (E <= 8) return router_fwd_impl<8>(x, w_g, w_noise, z, T, H, E, k, router_type, logits, gates, probs, noise_act, workspace, err_flag, stream);
    if (E <= 16) return router_fwd_impl<16>(x, w_g, w_noise, z, T, H, E, k, router_type, logits, gates, probs, noise_act, workspace, err_flag, stream);
    return router_fwd_impl<32>(x, w_g, w_noise, z, T, H, E, k, router_type, logits, gates, probs, noise_act, workspace, err_flag, stream);
}

size_t b200moe_router_workspace_floats(int H, int E) {
    const int EP = E <= 4 ? 4 : E <= 8 ? 8 : E <= 16 ? 16 : 32;
    const int NB = ((3 * EP + 15) / 16) * 16;
    return (size_t)2 * H * EP + (size_t)NB * H;   // swizzled W_g, W_noise (fp32) + split table (2 x NB x H bf16)
}

int b200moe_router_set_fma(int on) {
    g_router_fma = on;
    return B200MOE_OK;
}

int b200moe_gate_from_logits(const float* logits, int T, int E, int k, int router_type, float* gates, float* probs,
                             uint8_t* topk_mask, int32_t* err_flag, cudaStream_t stream) {
    int rc = check_router_args(T, 8, E, k, router_type);
    if (rc) return rc;
    if (E <= 4) return gate_impl<4>(logits, T, E, k, router_type, gates, probs, topk_mask, err_flag, stream);
    if (E <= 8) return gate_impl<8>(logits, T, E, k, router_type, gates, probs, topk_mask, err_flag, stream);
    if (E <= 16) return gate_impl<16>(logits, T, E, k, router_type, gates, probs, topk_mask, err_flag, stream);
    return gate_impl<32>(logits, T, E, k, router_type, gates, probs, topk_mask, err_flag, stream);
}

size_t b200moe_dispatch_workspace_words(int T) { return dispatch_ws_words(T < 1 ? 1 : T); }

int b200moe_dispatch(const float* gates, int T, int E, int capacity, int policy, int layout, int seg_stride,
                     int32_t* slot_rank, int32_t* counts, int32_t* seg_base, float* gate_mass, float* importance,
                     int64_t* stats, float* importance_loss, int32_t* importance_err, int32_t* workspace,
                     cudaStream_t stream) {
    B200_CHECK_ARG(T >= 1, B200MOE_ERR_CONFIG, "tokens_per_batch must be >= 1, got %d", T);
    B200_CHECK_ARG(E >= 1 && E <= kMaxE, B200MOE_ERR_CONFIG, "n_experts %d", E);
    B200_CHECK_ARG(policy == B200MOE_POLICY_POSITION || policy == B200MOE_POLICY_SCORE, B200MOE_ERR_CONFIG,
                   "drop_policy must be one of ('position', 'score')");
    B200_CHECK_ARG(layout == B200MOE_LAYOUT_COMPACT || (layout == B200MOE_LAYOUT_FIXED && seg_stride % kSegPad == 0),
                   B200MOE_ERR_CONFIG, "fixed layout needs a segment stride multiple of %d", kSegPad);
    if (policy == B200MOE_POLICY_POSITION || capacity < 0) {
        const int ntiles = ceil_div(T, kScanTile);
#define SCAN(EP) dispatch_scan_kernel<EP><<<ntiles, kScanTile, 0, stream>>>(                                     \
        gates, T, E, capacity, layout, seg_stride, slot_rank, counts, seg_base, gate_mass, importance, stats,     \
        importance_loss, importance_err, workspace)
        if (E <= 4) SCAN(4);
        else if (E <= 8) SCAN(8);
        else if (E <= 16) SCAN(16);
        else SCAN(32);
#undef SCAN
        B200_CHECK_LAUNCH("dispatch");
        return B200MOE_OK;
    }
    // score policy with a capacity: per-expert radix select (one CTA per expert)
    dispatch_kernel<<<E, kDispThreads, 0, stream>>>(gates, T, E, capacity, B200MOE_POLICY_SCORE, layout, seg_stride,
                                                    slot_rank, counts, seg_base, gate_mass, importance, stats,
                                                    workspace);
    if (importance_loss) importance_loss_kernel_fwd<<<1, 32, 0, stream>>>(importance, E, importance_loss,
                                                                          importance_err);
    B200_CHECK_LAUNCH("dispatch");
    return B200MOE_OK;
}

}  // extern "C"
