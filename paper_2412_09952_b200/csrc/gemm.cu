// Grouped expert GEMMs on tcgen05 / TMEM / TMA (sm_100a).
//
// One persistent, warp-specialised kernel template serves every GEMM of the
// E8T2 layer (reference: moefold/moe.py:131-133 ffn_forward and the matmul
// backward closures of moefold/tensor.py:192-207, 210-217):
//
//   FWD1   [a|b] = xp . [W1;W3]^T       epilogue: a, b, h = silu(a)*b   (bf16)
//   FWD2   o     = h . W2^T             epilogue: o                      (bf16)
//   BWD2   dm    = do . W2              epilogue: da, db (SwiGLU')        (bf16)
//   BWD1   dxp   = da . W1 + db . W3                                      (bf16)
//   WGRAD  dW1 = da^T xp, dW3 = db^T xp, dW2 = do^T h   (K = expert rows) (bf16)
//
// Activation rows live in expert *segments* (SegTable): segment s holds
// count[s] valid rows starting at base[s], zero-padded to a multiple of 128.
// Expert weights are stored K-major for the forward pass:
//   W1, W3: [E_local, F, H]    W2: [E_local, H, F]
// and read MN-major (transpose bit in the instruction descriptor) by the
// backward GEMMs, so no weight is ever transposed in memory.
//
// Tiling: a CTA pair (cta_group::2, cluster of 2) computes a 256 x 256 fp32
// tile in TMEM (each CTA: its 128 rows x 256 columns), K stepped by 64 with a
// 6-deep TMA -> smem ring (SWIZZLE_128B).  TMEM holds two accumulators
// (2 x 256 columns) so the epilogue of tile i overlaps the mainloop of i+1.
// kCtaGroup == 1 is the single-SM variant (128 x 256 tile, 4 stages).
//
// Warp roles (192 threads): w0 TMA producer, w1 MMA issuer (leader CTA),
// w2..w5 epilogue (TMEM lane quarter = warp % 4).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdio.h>

#include "common.cuh"
#include "ptx.cuh"

namespace b200moe {

enum GemmMode : int { kFwd1 = 0, kFwd2 = 1, kBwd2 = 2, kBwd1 = 3, kWgrad = 4 };

constexpr int kBK = 64;            // K per pipeline stage (128 B of bf16 = one swizzle row)
constexpr int kBN = 256;           // accumulator columns per tile
constexpr int kRowsPerCta = 128;   // M rows per CTA
constexpr int kMaxSeg = 64;
constexpr int kNumThreads = 192;

struct TmaSet {
    CUtensorMap m[5];
};

struct GemmArgs {
    const int* seg_base;
    const int* seg_count;
    const int* seg_expert;
    int nseg;
    int H, F, E_local;
    __nv_bfloat16* out0;
    __nv_bfloat16* out1;
    __nv_bfloat16* out2;
    const __nv_bfloat16* in0;
    const __nv_bfloat16* in1;
};

template <int kCG>
struct Cfg {
    static constexpr int kStages = (kCG == 2) ? 6 : 4;
    static constexpr int kBRows = kBN / kCG;                    // B rows (N) held per CTA
    static constexpr int kABytes = kRowsPerCta * kBK * 2;       // 16 KB
    static constexpr int kBBytes = kBRows * kBK * 2;            // 16 KB (cg2) / 32 KB (cg1)
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kTileM = kRowsPerCta * kCG;
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/ + 4 * (kMaxSeg + 2);
};

// ------------------------------------------------------------------ tile map
struct TileInfo {
    int seg;      // row-tiled modes: segment; wgrad: expert
    int sub;      // wgrad sub-problem: 0 = dW1, 1 = dW3, 2 = dW2
    int m_tile;   // row tile within the segment / output-row tile
    int n_tile;
};

template <int kMode, int kCG>
struct Sched {
    int total;
    int n_tiles;
    const int* prefix;  // smem: prefix[s] = first tile of segment/expert s

    __device__ TileInfo decode(int t, const GemmArgs& a) const {
        TileInfo ti;
        int s = 0;
        while (prefix[s + 1] <= t) ++s;
        int r = t - prefix[s];
        ti.seg = s;
        if constexpr (kMode == kWgrad) {
            const int tiles_w13 = (a.F / Cfg<kCG>::kTileM) * (a.H / kBN);
            if (r < 2 * tiles_w13) {
                ti.sub = r / tiles_w13;
                r -= ti.sub * tiles_w13;
                const int nt = a.H / kBN;
                ti.m_tile = r / nt;
                ti.n_tile = r % nt;
            } else {
                ti.sub = 2;
                r -= 2 * tiles_w13;
                const int nt = a.F / kBN;
                ti.m_tile = r / nt;
                ti.n_tile = r % nt;
            }
        } else {
            const int mt = (prefix[s + 1] - prefix[s]) / n_tiles;
            ti.sub = 0;
            ti.n_tile = r / mt;
            ti.m_tile = r % mt;
        }
        return ti;
    }
};

template <int kMode>
__device__ __forceinline__ int mode_n_tiles(const GemmArgs& a) {
    if constexpr (kMode == kFwd1) return a.F / 128;
    if constexpr (kMode == kFwd2) return a.H / 256;
    if constexpr (kMode == kBwd2) return a.F / 256;
    if constexpr (kMode == kBwd1) return a.H / 256;
    return 0;
}

template <int kMode>
__device__ __forceinline__ int mode_k_blocks(const GemmArgs& a) {
    if constexpr (kMode == kFwd1 || kMode == kBwd2) return a.H / kBK;
    if constexpr (kMode == kFwd2) return a.F / kBK;
    if constexpr (kMode == kBwd1) return 2 * a.F / kBK;
    return 0;
}

// K blocks of expert e in WGRAD: sum over its segments of ceil(count/64).
__device__ __forceinline__ int wgrad_k_blocks(const GemmArgs& a, int e) {
    int kb = 0;
    for (int s = 0; s < a.nseg; ++s)
        if (a.seg_expert[s] == e) kb += ceil_div(a.seg_count[s], kBK);
    return kb;
}

// ------------------------------------------------------------------ loads
template <bool kMN>
__device__ __forceinline__ void load_operand(const CUtensorMap* m, uint64_t* bar, uint8_t* dst, int mn0, int k0,
                                             int n_mn, bool cg2) {
    if constexpr (!kMN) {
        for (int i = 0; i < n_mn / 128; ++i) {
            if (cg2) ptx::tma_load_2d_cg2(m, bar, dst + i * 16384, k0, mn0 + i * 128);
            else ptx::tma_load_2d(m, bar, dst + i * 16384, k0, mn0 + i * 128);
        }
    } else {
        for (int i = 0; i < n_mn / 64; ++i) {
            if (cg2) ptx::tma_load_2d_cg2(m, bar, dst + i * 8192, mn0 + i * 64, k0);
            else ptx::tma_load_2d(m, bar, dst + i * 8192, mn0 + i * 64, k0);
        }
    }
}

template <int kMode>
struct Majors;
template <> struct Majors<kFwd1>  { static constexpr bool a = false, b = false; };
template <> struct Majors<kFwd2>  { static constexpr bool a = false, b = false; };
template <> struct Majors<kBwd2>  { static constexpr bool a = false, b = true; };
template <> struct Majors<kBwd1>  { static constexpr bool a = false, b = true; };
template <> struct Majors<kWgrad> { static constexpr bool a = true, b = true; };

// Issue the TMA loads of k-block `kb` of tile `ti` into stage buffers.
template <int kMode, int kCG>
__device__ __forceinline__ void produce_kblock(const TmaSet& tm, const GemmArgs& a, const TileInfo& ti, int kb,
                                               int row0_seg, uint32_t rank, uint64_t* bar, uint8_t* sA,
                                               uint8_t* sB) {
    using C = Cfg<kCG>;
    const bool cg2 = (kCG == 2);
    if constexpr (kMode == kFwd1) {
        const int e = a.seg_expert[ti.seg];
        const int rowA = a.seg_base[ti.seg] + ti.m_tile * C::kTileM + rank * kRowsPerCta;
        load_operand<false>(&tm.m[0], bar, sA, rowA, kb * kBK, 128, cg2);
        const int frow = e * a.F + ti.n_tile * 128;
        if constexpr (kCG == 2) {
            load_operand<false>(&tm.m[rank == 0 ? 1 : 2], bar, sB, frow, kb * kBK, 128, true);
        } else {
            load_operand<false>(&tm.m[1], bar, sB, frow, kb * kBK, 128, false);
            load_operand<false>(&tm.m[2], bar, sB + 16384, frow, kb * kBK, 128, false);
        }
    } else if constexpr (kMode == kFwd2) {
        const int e = a.seg_expert[ti.seg];
        const int rowA = a.seg_base[ti.seg] + ti.m_tile * C::kTileM + rank * kRowsPerCta;
        load_operand<false>(&tm.m[0], bar, sA, rowA, kb * kBK, 128, cg2);
        const int nrow = e * a.H + ti.n_tile * kBN + rank * C::kBRows;
        load_operand<false>(&tm.m[1], bar, sB, nrow, kb * kBK, C::kBRows, cg2);
    } else if constexpr (kMode == kBwd2) {
        const int e = a.seg_expert[ti.seg];
        const int rowA = a.seg_base[ti.seg] + ti.m_tile * C::kTileM + rank * kRowsPerCta;
        load_operand<false>(&tm.m[0], bar, sA, rowA, kb * kBK, 128, cg2);
        const int ncol = ti.n_tile * kBN + rank * C::kBRows;  // f
        load_operand<true>(&tm.m[1], bar, sB, ncol, e * a.H + kb * kBK, C::kBRows, cg2);
    } else if constexpr (kMode == kBwd1) {
        const int e = a.seg_expert[ti.seg];
        const int rowA = a.seg_base[ti.seg] + ti.m_tile * C::kTileM + rank * kRowsPerCta;
        const int kF = a.F / kBK;
        const bool second = kb >= kF;
        const int kk = second ? kb - kF : kb;
        load_operand<false>(&tm.m[second ? 1 : 0], bar, sA, rowA, kk * kBK, 128, cg2);
        const int ncol = ti.n_tile * kBN + rank * C::kBRows;  // h
        load_operand<true>(&tm.m[second ? 3 : 2], bar, sB, ncol, e * a.F + kk * kBK, C::kBRows, cg2);
    } else {  // WGRAD: kb is the absolute row of this k-block
        const int m0 = ti.m_tile * C::kTileM + rank * kRowsPerCta;
        const int n0 = ti.n_tile * kBN + rank * C::kBRows;
        const int amap = ti.sub == 0 ? 2 : (ti.sub == 1 ? 4 : 0);
        const int bmap = ti.sub == 2 ? 1 : 3;
        load_operand<true>(&tm.m[amap], bar, sA, m0, kb, 128, cg2);
        load_operand<true>(&tm.m[bmap], bar, sB, n0, kb, C::kBRows, cg2);
    }
    (void)row0_seg;
}

// ------------------------------------------------------------------ epilogues
__device__ __forceinline__ void store32(__nv_bfloat16* dst, const float* v) {
    uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i] = pack8(v + 8 * i);
}

__device__ __forceinline__ void load32(const __nv_bfloat16* src, float* v) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
#pragma unroll
    for (int i = 0; i < 4; ++i) unpack8(s[i], v + 8 * i);
}

__device__ __forceinline__ float sigmoidf_(float x) { return 1.0f / (1.0f + __expf(-x)); }

template <int kMode, int kCG>
__device__ __forceinline__ void epilogue_tile(const GemmArgs& a, const TileInfo& ti, uint32_t tmem_acc, int q,
                                              int lane, uint32_t rank, bool k_empty) {
    using C = Cfg<kCG>;
    uint32_t r0[32], r1[32];
    float v0[32], v1[32], v2[32];
    const uint32_t lane_addr = tmem_acc + ((uint32_t)(q * 32) << 16);
    if constexpr (kMode == kWgrad) {
        const int e = ti.seg;
        const int row = ti.m_tile * C::kTileM + rank * kRowsPerCta + q * 32 + lane;  // output row
        int ncols;
        __nv_bfloat16* out;
        if (ti.sub == 2) { ncols = a.F; out = a.out1 + ((size_t)e * a.H + row) * a.F; }
        else { ncols = a.H; out = (ti.sub == 0 ? a.out0 : a.out2) + ((size_t)e * a.F + row) * a.H; }
        out += ti.n_tile * kBN;
        (void)ncols;
        for (int c = 0; c < kBN; c += 32) {
            if (!k_empty) {
                ptx::tmem_ld_32x32b_x32(lane_addr + c, r0);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) v0[i] = __uint_as_float(r0[i]);
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) v0[i] = 0.f;
            }
            store32(out + c, v0);
        }
        return;
    } else {
        const int cnt = a.seg_count[ti.seg];
        const int rel = ti.m_tile * C::kTileM + rank * kRowsPerCta + q * 32;  // first row of this warp
        const int limit = round_up(cnt, kSegPad);
        if (rel >= limit) return;  // whole warp outside the padded segment (warp-uniform)
        const bool valid = (rel + lane) < limit;
        const size_t row = (size_t)a.seg_base[ti.seg] + rel + lane;
        if constexpr (kMode == kFwd1) {
            const size_t off = row * a.F + ti.n_tile * 128;
            for (int c = 0; c < 128; c += 32) {
                ptx::tmem_ld_32x32b_x32(lane_addr + c, r0);
                ptx::tmem_ld_32x32b_x32(lane_addr + 128 + c, r1);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const float av = __uint_as_float(r0[i]);
                    const float bv = __uint_as_float(r1[i]);
                    v0[i] = av;
                    v1[i] = bv;
                    v2[i] = av * sigmoidf_(av) * bv;
                }
                if (valid) {
                    store32(a.out0 + off + c, v0);
                    store32(a.out1 + off + c, v1);
                    store32(a.out2 + off + c, v2);
                }
            }
        } else if constexpr (kMode == kFwd2 || kMode == kBwd1) {
            const size_t off = row * a.H + ti.n_tile * kBN;
            for (int c = 0; c < kBN; c += 32) {
                ptx::tmem_ld_32x32b_x32(lane_addr + c, r0);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) v0[i] = __uint_as_float(r0[i]);
                if (valid) store32(a.out0 + off + c, v0);
            }
        } else {  // kBwd2: SwiGLU backward from the stored pre-activations
            const size_t off = row * a.F + ti.n_tile * kBN;
            for (int c = 0; c < kBN; c += 32) {
                ptx::tmem_ld_32x32b_x32(lane_addr + c, r0);
                if (valid) {
                    load32(a.in0 + off + c, v0);  // a
                    load32(a.in1 + off + c, v1);  // b
                }
                ptx::tmem_ld_wait();
                if (valid) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const float dm = __uint_as_float(r0[i]);
                        const float av = v0[i], bv = v1[i];
                        const float sg = sigmoidf_(av);
                        const float da = dm * bv * (sg * (1.0f + av * (1.0f - sg)));
                        const float db = dm * (av * sg);
                        v0[i] = da;
                        v1[i] = db;
                    }
                    store32(a.out0 + off + c, v0);
                    store32(a.out1 + off + c, v1);
                }
            }
        }
    }
    (void)v2;
    (void)r1;
}

// ------------------------------------------------------------------ kernel
template <int kMode, int kCG>
__global__ void __launch_bounds__(kNumThreads, 1) moe_gemm_kernel(const __grid_constant__ TmaSet tm, GemmArgs a) {
    using C = Cfg<kCG>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stages = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
    uint64_t* empty = full + C::kStages;
    uint64_t* tfull = empty + C::kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int* prefix = reinterpret_cast<int*>(tmem_base_slot + 1);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t rank = (kCG == 2) ? ptx::cluster_ctarank() : 0;
    const int cid = (kCG == 2) ? (int)ptx::cluster_id_x() : (int)blockIdx.x;
    const int ncl = (kCG == 2) ? (int)ptx::nclusters_x() : (int)gridDim.x;

    // ---- tile table (identical in every CTA)
    if (threadIdx.x == 0) {
        int acc = 0;
        prefix[0] = 0;
        if constexpr (kMode == kWgrad) {
            const int per_e = 2 * (a.F / C::kTileM) * (a.H / kBN) + (a.H / C::kTileM) * (a.F / kBN);
            for (int e = 0; e < a.E_local; ++e) {
                acc += per_e;
                prefix[e + 1] = acc;
            }
        } else {
            const int nt = mode_n_tiles<kMode>(a);
            for (int s = 0; s < a.nseg; ++s) {
                acc += ceil_div(a.seg_count[s], C::kTileM) * nt;
                prefix[s + 1] = acc;
            }
        }
    }
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < 5; ++i) ptx::prefetch_tmap(&tm.m[i]);
        for (int s = 0; s < C::kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], kCG * 4);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc<kCG>(tmem_base_slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    if constexpr (kCG == 2) ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_base_slot;

    Sched<kMode, kCG> sched;
    sched.prefix = prefix;
    sched.n_tiles = mode_n_tiles<kMode>(a);
    sched.total = prefix[(kMode == kWgrad) ? a.E_local : a.nseg];

    if (warp == 0) {
        // ================= TMA producer
        if (ptx::elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cid; t < sched.total; t += ncl) {
                const TileInfo ti = sched.decode(t, a);
                if constexpr (kMode == kWgrad) {
                    for (int s = 0; s < a.nseg; ++s) {
                        if (a.seg_expert[s] != ti.seg) continue;
                        const int nkb = ceil_div(a.seg_count[s], kBK);
                        for (int kb = 0; kb < nkb; ++kb) {
                            ptx::mbar_wait(&empty[stage], phase ^ 1);
                            if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes * kCG);
                            uint8_t* sA = stages + stage * C::kStageBytes;
                            produce_kblock<kMode, kCG>(tm, a, ti, a.seg_base[s] + kb * kBK, 0, rank, &full[stage],
                                                       sA, sA + C::kABytes);
                            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
                        }
                    }
                } else {
                    const int nkb = mode_k_blocks<kMode>(a);
                    for (int kb = 0; kb < nkb; ++kb) {
                        ptx::mbar_wait(&empty[stage], phase ^ 1);
                        if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes * kCG);
                        uint8_t* sA = stages + stage * C::kStageBytes;
                        produce_kblock<kMode, kCG>(tm, a, ti, kb, 0, rank, &full[stage], sA, sA + C::kABytes);
                        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer (leader CTA of the pair)
        if (rank == 0) {
            constexpr uint32_t idesc = ptx::make_idesc_bf16(kRowsPerCta * kCG, kBN, Majors<kMode>::a, Majors<kMode>::b);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = cid; t < sched.total; t += ncl) {
                const TileInfo ti = sched.decode(t, a);
                const int nkb = (kMode == kWgrad) ? wgrad_k_blocks(a, ti.seg) : mode_k_blocks<kMode>(a);
                ptx::mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t dtm = tmem_base + acc * kBN;
                for (int kb = 0; kb < nkb; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        const uint32_t aaddr = ptx::smem_u32(stages + stage * C::kStageBytes);
                        const uint32_t baddr = aaddr + C::kABytes;
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k) {
                            const uint64_t ad = Majors<kMode>::a ? ptx::make_sdesc(aaddr + k * 2048, 8192, 1024)
                                                                 : ptx::make_sdesc(aaddr + k * 32, 16, 1024);
                            const uint64_t bd = Majors<kMode>::b ? ptx::make_sdesc(baddr + k * 2048, 8192, 1024)
                                                                 : ptx::make_sdesc(baddr + k * 32, 16, 1024);
                            ptx::mma_bf16<kCG>(dtm, ad, bd, idesc, (kb | k) != 0);
                        }
                        ptx::mma_commit<kCG>(&empty[stage], 0x3);
                    }
                    __syncwarp();
                    if (++stage == C::kStages) { stage = 0; phase ^= 1; }
                }
                if (ptx::elect_one()) ptx::mma_commit<kCG>(&tfull[acc], 0x3);
                __syncwarp();
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {
        // ================= epilogue (warps 2..5)
        const int q = warp % 4;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = cid; t < sched.total; t += ncl) {
            const TileInfo ti = sched.decode(t, a);
            const bool k_empty = (kMode == kWgrad) ? (wgrad_k_blocks(a, ti.seg) == 0) : false;
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            epilogue_tile<kMode, kCG>(a, ti, tmem_base + acc * kBN, q, lane, rank, k_empty);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(&tempty[acc], 0);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if constexpr (kCG == 2) ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<kCG>(tmem_base, 512);
    }
}

// ================================================================== host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 2-D bf16 tensor [outer, inner] (inner contiguous, row pitch `ld` elements).
// K-major operands use box {64, 128}; MN-major operands box {64, 64}.
static int make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, bool mn_major) {
    EncodeTiledFn enc = get_encode();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return B200MOE_ERR_CUDA;
    }
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld * 2};
    cuuint32_t box[2] = {64, mn_major ? 64u : 128u};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d) inner=%llu outer=%llu ld=%llu", (int)r,
                  (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)ld);
        return B200MOE_ERR_CUDA;
    }
    return B200MOE_OK;
}

static int g_cta_group = 2;  // 2 = CTA-pair kernels (default), 1 = single-SM kernels
static int g_max_ctas = kNumSMs;

template <int kMode, int kCG>
static int launch(const TmaSet& tm, const GemmArgs& a, cudaStream_t s) {
    using C = Cfg<kCG>;
    auto kern = moe_gemm_kernel<kMode, kCG>;
    static bool attr_done = false;
    if (!attr_done) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
        attr_done = true;
    }
    cudaLaunchConfig_t cfg = {};
    int grid = g_max_ctas - (g_max_ctas % kCG);
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kNumThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tm, a);
    if (e != cudaSuccess) {
        set_error("moe_gemm_kernel<%d,%d> launch: %s", kMode, kCG, cudaGetErrorString(e));
        return B200MOE_ERR_CUDA;
    }
    return B200MOE_OK;
}

template <int kMode>
static int dispatch_launch(const TmaSet& tm, const GemmArgs& a, cudaStream_t s) {
    return g_cta_group == 2 ? launch<kMode, 2>(tm, a, s) : launch<kMode, 1>(tm, a, s);
}

static int check_common(int nseg, int H, int F, int E_local) {
    B200_CHECK_ARG(nseg >= 1 && nseg <= kMaxSeg, B200MOE_ERR_CONFIG, "nseg %d outside [1,%d]", nseg, kMaxSeg);
    B200_CHECK_ARG(E_local >= 1 && E_local <= kMaxSeg, B200MOE_ERR_CONFIG, "E_local %d outside [1,%d]", E_local,
                   kMaxSeg);
    B200_CHECK_ARG(H % 256 == 0 && F % 256 == 0, B200MOE_ERR_SHAPE,
                   "grouped GEMM needs hidden and ffn multiples of 256 (got H=%d F=%d)", H, F);
    return B200MOE_OK;
}

#define B200_TRY(x)                 \
    do {                            \
        int _rc = (x);              \
        if (_rc != B200MOE_OK) return _rc; \
    } while (0)

}  // namespace b200moe

using namespace b200moe;

extern "C" {

int b200moe_gemm_set_cta_group(int cg) {
    B200_CHECK_ARG(cg == 1 || cg == 2, B200MOE_ERR_CONFIG, "cta group must be 1 or 2");
    g_cta_group = cg;
    return B200MOE_OK;
}

int b200moe_gemm_set_max_ctas(int n) {
    B200_CHECK_ARG(n >= 2 && n <= 4096, B200MOE_ERR_CONFIG, "max ctas %d", n);
    g_max_ctas = n;
    return B200MOE_OK;
}

int b200moe_expert_fwd1(const void* xp, const void* w1, const void* w3, const int* seg_base, const int* seg_count,
                        const int* seg_expert, int nseg, int rows, int H, int F, int E_local, void* a_out,
                        void* b_out, void* h_out, cudaStream_t stream) {
    B200_TRY(check_common(nseg, H, F, E_local));
    TmaSet tm = {};
    B200_TRY(make_map(&tm.m[0], xp, H, rows, H, false));
    B200_TRY(make_map(&tm.m[1], w1, H, (uint64_t)E_local * F, H, false));
    B200_TRY(make_map(&tm.m[2], w3, H, (uint64_t)E_local * F, H, false));
    tm.m[3] = tm.m[0];
    tm.m[4] = tm.m[0];
    GemmArgs a = {seg_base, seg_count, seg_expert, nseg, H, F, E_local,
                  (__nv_bfloat16*)a_out, (__nv_bfloat16*)b_out, (__nv_bfloat16*)h_out, nullptr, nullptr};
    return dispatch_launch<kFwd1>(tm, a, stream);
}

int b200moe_expert_fwd2(const void* h, const void* w2, const int* seg_base, const int* seg_count,
                        const int* seg_expert, int nseg, int rows, int H, int F, int E_local, void* o_out,
                        cudaStream_t stream) {
    B200_TRY(check_common(nseg, H, F, E_local));
    TmaSet tm = {};
    B200_TRY(make_map(&tm.m[0], h, F, rows, F, false));
    B200_TRY(make_map(&tm.m[1], w2, F, (uint64_t)E_local * H, F, false));
    tm.m[2] = tm.m[3] = tm.m[4] = tm.m[0];
    GemmArgs a = {seg_base, seg_count, seg_expert, nseg, H, F, E_local,
                  (__nv_bfloat16*)o_out, nullptr, nullptr, nullptr, nullptr};
    return dispatch_launch<kFwd2>(tm, a, stream);
}

int b200moe_expert_bwd2(const void* dout, const void* w2, const void* a_pre, const void* b_pre, const int* seg_base,
                        const int* seg_count, const int* seg_expert, int nseg, int rows, int H, int F, int E_local,
                        void* da_out, void* db_out, cudaStream_t stream) {
    B200_TRY(check_common(nseg, H, F, E_local));
    TmaSet tm = {};
    B200_TRY(make_map(&tm.m[0], dout, H, rows, H, false));
    B200_TRY(make_map(&tm.m[1], w2, F, (uint64_t)E_local * H, F, true));
    tm.m[2] = tm.m[3] = tm.m[4] = tm.m[0];
    GemmArgs a = {seg_base, seg_count, seg_expert, nseg, H, F, E_local,
                  (__nv_bfloat16*)da_out, (__nv_bfloat16*)db_out, nullptr,
                  (const __nv_bfloat16*)a_pre, (const __nv_bfloat16*)b_pre};
    return dispatch_launch<kBwd2>(tm, a, stream);
}

int b200moe_expert_bwd1(const void* da, const void* db, const void* w1, const void* w3, const int* seg_base,
                        const int* seg_count, const int* seg_expert, int nseg, int rows, int H, int F, int E_local,
                        void* dxp_out, cudaStream_t stream) {
    B200_TRY(check_common(nseg, H, F, E_local));
    TmaSet tm = {};
    B200_TRY(make_map(&tm.m[0], da, F, rows, F, false));
    B200_TRY(make_map(&tm.m[1], db, F, rows, F, false));
    B200_TRY(make_map(&tm.m[2], w1, H, (uint64_t)E_local * F, H, true));
    B200_TRY(make_map(&tm.m[3], w3, H, (uint64_t)E_local * F, H, true));
    tm.m[4] = tm.m[0];
    GemmArgs a = {seg_base, seg_count, seg_expert, nseg, H, F, E_local,
                  (__nv_bfloat16*)dxp_out, nullptr, nullptr, nullptr, nullptr};
    return dispatch_launch<kBwd1>(tm, a, stream);
}

int b200moe_expert_wgrad(const void* xp, const void* h, const void* dout, const void* da, const void* db,
                         const int* seg_base, const int* seg_count, const int* seg_expert, int nseg, int rows, int H,
                         int F, int E_local, void* dw1, void* dw2, void* dw3, cudaStream_t stream) {
    B200_TRY(check_common(nseg, H, F, E_local));
    TmaSet tm = {};
    B200_TRY(make_map(&tm.m[0], dout, H, rows, H, true));
    B200_TRY(make_map(&tm.m[1], h, F, rows, F, true));
    B200_TRY(make_map(&tm.m[2], da, F, rows, F, true));
    B200_TRY(make_map(&tm.m[3], xp, H, rows, H, true));
    B200_TRY(make_map(&tm.m[4], db, F, rows, F, true));
    GemmArgs a = {seg_base, seg_count, seg_expert, nseg, H, F, E_local,
                  (__nv_bfloat16*)dw1, (__nv_bfloat16*)dw2, (__nv_bfloat16*)dw3, nullptr, nullptr};
    return dispatch_launch<kWgrad>(tm, a, stream);
}

}  // extern "C"
