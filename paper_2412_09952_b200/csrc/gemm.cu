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
// Warp roles (320 threads): w0 TMA producer, w1 MMA issuer (leader CTA),
// w2..w9 epilogue (TMEM lane quarter = warp % 4, column half = (warp-2)/4).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "ptx.cuh"

namespace b200moe {

enum GemmMode : int { kFwd1 = 0, kFwd2 = 1, kBwd2 = 2, kBwd1 = 3, kWgrad = 4, kWgradW = 5, kWgradAcc = 6 };

// kWgradAcc: WGRAD that adds into the existing bf16 gradients (gradient
// accumulation over micro-batches).  Same tiles and mainloop as kWgrad; the
// epilogue streams each 32 x 32 chunk of the old gradient into shared memory by
// TMA (one chunk ahead, the first before the accumulator wait) and adds it in
// fp32 before the single rounding to bf16.
template <int kMode>
__host__ __device__ constexpr bool is_wgrad1() { return kMode == kWgrad || kMode == kWgradAcc; }

// kWgradW ("wide" WGRAD, CTA pairs only, opt-in -- see b200moe_expert_wgrad
// for the measurement): each tile is two 256 x 256
// accumulators that share one operand, so a k-block loads three 16 KB operand
// pieces per CTA instead of four:
//   sub 0: dW1 and dW3 tiles at the same (f, h) share the xp columns,
//   sub 2: two adjacent dW2 tiles (f and f + 256) share the do columns.
// With K = the expert's rows (1024 at the bench shape) WGRAD is bound by L2 ->
// SM operand bandwidth, not by the tensor pipe, and this cuts its operand
// traffic by 25%.  Both accumulators fill all 512 TMEM columns; instead of a
// double buffer, the MMA issuer starts the next tile on slot 0 as soon as the
// epilogue has drained it and catches slot 1 up a few k-blocks later.

constexpr int kBK = 64;            // K per pipeline stage (128 B of bf16 = one swizzle row)
constexpr int kBN = 256;           // accumulator columns per tile
constexpr int kRowsPerCta = 128;   // M rows per CTA
constexpr int kMaxSeg = 64;
constexpr int kNumEpiWarps = 8;
constexpr bool kWideStores = false;  // see Geo::kWide
constexpr bool kLsuStores = true;    // see emit32
constexpr int kNumThreads = 64 + 32 * kNumEpiWarps;   // producer, MMA, 8 epilogue warps

constexpr int kMaxPeers = 8;   // expert-parallel ranks an epilogue can push rows to

struct TmaSet {
    CUtensorMap m[5];   // operand loads (SWIZZLE_128B)
    CUtensorMap st[3];  // epilogue stores: 32 x 32 bf16 boxes (SWIZZLE_64B)
    CUtensorMap stp[kMaxPeers];  // FWD2 / BWD1 with peer output: every rank's receive plane (peer_El > 0)
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
    int debug;  // bit 0: skip wgrad epilogue stores (diagnostics only)
    int wgrad_subs;  // WGRAD sub-problems to compute: bit 0 dW1, bit 1 dW3, bit 2 dW2 (0 = all)
    int dense;       // BWD1 as a plain dense GEMM: one (A, B) pair, K = F (0 = the two-pair expert BWD1)
    int wgrad_mfast; // WGRAD raster: output-row tiles fastest (dense wgrad with many more column tiles than row
                     // tiles and a long K: concurrent tiles then share the column block of dy in L2)
    // FWD2 / BWD1 fused with the expert-parallel return exchange (peer_El > 0): segment s = (src, el) =
    // (s / peer_El, s % peer_El) of this owner rank; its output rows go straight into rank src's receive
    // plane (tm.stp[src], peer-mapped over NVLink) at row (peer_rank * peer_El + el) * peer_cap + r,
    // i.e. where the source's own dispatch layout (expert-major, peer_cap rows each) expects them
    int peer_El, peer_rank, peer_cap;
};

__host__ __device__ __forceinline__ int wgrad_mask(const GemmArgs& a) { return a.wgrad_subs ? a.wgrad_subs : 7; }

template <int kCG>
struct Cfg {
    static constexpr int kStages = (kCG == 2) ? 6 : 4;
    static constexpr int kBRows = kBN / kCG;                    // B rows (N) held per CTA
    static constexpr int kABytes = kRowsPerCta * kBK * 2;       // 16 KB
    static constexpr int kBBytes = kBRows * kBK * 2;            // 16 KB (cg2) / 32 KB (cg1)
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kTileM = kRowsPerCta * kCG;
};

// Per-(mode, cta-group) shared-memory plan: operand ring + per-epilogue-warp
// staging (store ring of 2 x 2 KB; BWD2 on CTA pairs adds a TMA load ring of
// 2 x (a, b) 2 KB chunks and trades two operand stages for it).
template <int kMode, int kCG>
struct Geo {
#ifndef B200_BWD2_TMA_EPI
#define B200_BWD2_TMA_EPI 1
#endif
    static constexpr bool kTmaEpiLoads = B200_BWD2_TMA_EPI && (kMode == kBwd2) && (kCG == 2);
    // BWD2's a/b load ring: one (a, b) buffer pair per epilogue warp, refilled right after the
    // chunk is taken (the epilogue has slack: it waits on the accumulator a third of the time),
    // which frees shared memory for a 5th operand stage.
#ifndef B200_BWD2_LOAD_BUFS
#define B200_BWD2_LOAD_BUFS 1
#endif
    static constexpr int kEpiLoadBufs = B200_BWD2_LOAD_BUFS;
    // In place: the a/b load buffers double as the da/db store staging (same
    // 32 x 32 SWIZZLE_64B box), 4 KB per epilogue warp instead of 8, which buys
    // a 6th operand stage; a chunk's loads are issued once the previous
    // chunk's stores have read the buffers.
#ifndef B200_BWD2_INPLACE
#define B200_BWD2_INPLACE 1
#endif
    static constexpr bool kInPlace = kTmaEpiLoads && B200_BWD2_INPLACE;
    // Store-ring depth per epilogue warp (4 buffers + 5 stages measured no
    // better than 2 + 6 for WGRAD on B200).
    static constexpr int kRing = 2;
    // Wide stores: 32 x 64 bf16 boxes (128-byte rows, SWIZZLE_128B) halve the
    // TMA row requests of the plain-store epilogues, but cost one operand stage
    // of shared memory.  Measured on B200: WGRAD 2.12-2.27 ms -> 2.33-2.42 ms
    // (its operand loads are latency-bound, in-flight bytes matter more), BWD1
    // and FWD2 within noise -- so disabled; kept for the next tile-shape study.
    static constexpr bool kWide = kWideStores && (kCG == 2) && (kMode == kFwd2 || kMode == kBwd1 || kMode == kWgrad);
    static constexpr int kStoreBytes = kWide ? 4096 : 2048;
    static constexpr bool kPairAcc = (kMode == kWgradW);   // two accumulators sharing one operand
    static constexpr bool kAccLoads = (kMode == kWgradAcc);  // old-gradient TMA load ring (2 x 2 KB per warp)
    static constexpr int kStageBytes = kPairAcc ? 3 * 16384 : Cfg<kCG>::kStageBytes;
    static constexpr int kStages = kPairAcc ? 4 : (kAccLoads ? (kCG == 2 ? 5 : 3)
                                                             : (kTmaEpiLoads ? (kInPlace ? 6 : (kEpiLoadBufs == 1 ? 5 : 4))
                                                                             : (kWide ? 5 : Cfg<kCG>::kStages)));
    static constexpr int kEpiWarpBytes = kInPlace ? 2 * 2048
                                                  : (kTmaEpiLoads ? kEpiLoadBufs * 2 * 2048 : 0) +
                                                        (kAccLoads ? 2 * 2048 : 0) + kRing * kStoreBytes;
    static constexpr int kSmemBytes = kStages * kStageBytes + kNumEpiWarps * kEpiWarpBytes +
                                      1024 /*align*/ + 512 /*barriers*/ + 4 * (kMaxSeg + 2) +
                                      3 * 4 * kMaxSeg /*segment table*/;
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
        if constexpr (kMode == kWgradW) {
            const int tiles_w13 = (a.F / 256) * (a.H / 256);   // (dW1, dW3) pairs
            if (r < tiles_w13) {
                ti.sub = 0;
                ti.m_tile = r / (a.H / 256);
                ti.n_tile = r % (a.H / 256);
            } else {                                            // dW2 column pairs
                ti.sub = 2;
                r -= tiles_w13;
                ti.m_tile = r / (a.F / 512);
                ti.n_tile = r % (a.F / 512);
            }
        } else if constexpr (is_wgrad1<kMode>()) {
            const int tiles_w13 = (a.F / Cfg<kCG>::kTileM) * (a.H / kBN);
            const int tiles_w2 = (a.H / Cfg<kCG>::kTileM) * (a.F / kBN);
            const int mask = wgrad_mask(a);
            ti.sub = 0;
#pragma unroll
            for (int sb = 0; sb < 3; ++sb) {          // enabled sub-problems in order dW1, dW3, dW2
                if (!((mask >> sb) & 1)) continue;
                const int n = sb < 2 ? tiles_w13 : tiles_w2;
                ti.sub = sb;
                if (r < n) break;
                r -= n;
            }
            const int nt = (ti.sub == 2 ? a.F : a.H) / kBN;
            if (a.wgrad_mfast) {
                const int mt = (ti.sub == 2 ? a.H : a.F) / Cfg<kCG>::kTileM;
                ti.n_tile = r / mt;
                ti.m_tile = r % mt;
            } else {
                ti.m_tile = r / nt;
                ti.n_tile = r % nt;
            }
        } else {
            const int mt = (prefix[s + 1] - prefix[s]) / n_tiles;
            ti.sub = 0;
            if (a.debug & 16) {  // experiment: n fastest
                ti.m_tile = r / n_tiles;
                ti.n_tile = r % n_tiles;
            } else {             // m fastest: concurrent clusters share weight tiles in L2
                ti.n_tile = r / mt;
                ti.m_tile = r % mt;
            }
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
    if constexpr (kMode == kBwd1) return (a.dense ? 1 : 2) * a.F / kBK;
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
template <> struct Majors<kWgradW> { static constexpr bool a = true, b = true; };
template <> struct Majors<kWgradAcc> { static constexpr bool a = true, b = true; };

// kWgradW k-block (absolute row kb) into the three 16 KB pieces of a stage:
//   sub 0: s0 = da[:, f], s1 = db[:, f], s2 = xp[:, h]   (MMA0: s0 x s2, MMA1: s1 x s2)
//   sub 2: s0 = do[:, h], s1 = h[:, f],  s2 = h[:, f+256] (MMA0: s0 x s1, MMA1: s0 x s2)
__device__ __forceinline__ void produce_wide(const TmaSet& tm, const TileInfo& ti, int kb, uint32_t rank,
                                             uint64_t* bar, uint8_t* st) {
    const int m0 = ti.m_tile * 256 + rank * kRowsPerCta;
    if (ti.sub == 0) {
        const int n0 = ti.n_tile * 256 + rank * 128;
        load_operand<true>(&tm.m[2], bar, st, m0, kb, 128, true);
        load_operand<true>(&tm.m[4], bar, st + 16384, m0, kb, 128, true);
        load_operand<true>(&tm.m[3], bar, st + 32768, n0, kb, 128, true);
    } else {
        const int f0 = ti.n_tile * 512 + rank * 128;
        load_operand<true>(&tm.m[0], bar, st, m0, kb, 128, true);
        load_operand<true>(&tm.m[1], bar, st + 16384, f0, kb, 128, true);
        load_operand<true>(&tm.m[1], bar, st + 32768, f0 + 256, kb, 128, true);
    }
}

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
// Each epilogue warp owns a ring of kRing x 2 KB staging buffers in shared
// memory.  A 32-row x 32-column bf16 chunk is written row-per-lane into the
// SWIZZLE_64B layout (16-byte chunk j of row r lives at chunk j ^ ((r >> 1) & 3):
// conflict-free) and shipped with one TMA bulk tensor store, so global writes
// are full, coalesced lines instead of 32 scattered 16-byte pieces.
constexpr int kStageBufBytes = 2048;

struct EpiRing {
    uint8_t* base;  // this warp's buffers
    int idx;
};

template <int kRing>
__device__ __forceinline__ void stage_store(EpiRing& ring, const CUtensorMap* m, const float* v, int lane, int col,
                                            int row0, bool evict_first = false) {
    uint8_t* buf = ring.base + ring.idx * kStageBufBytes;
    if (lane == 0) ptx::bulk_wait_read<kRing - 1>();  // the store that last used this buffer has read it
    __syncwarp();
    uint4* rowp = reinterpret_cast<uint4*>(buf + lane * 64);
    const int sw = (lane >> 1) & 3;
#pragma unroll
    for (int j = 0; j < 4; ++j) rowp[j ^ sw] = pack8(v + 8 * j);
    ptx::fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
        if (evict_first) ptx::tma_store_2d_hint(m, buf, col, row0, ptx::policy_evict_first());
        else ptx::tma_store_2d(m, buf, col, row0);
        ptx::bulk_commit();
    }
    ring.idx = (ring.idx + 1 == kRing) ? 0 : ring.idx + 1;
}

// Same 32 x 32 chunk, written back through the LSU instead of TMA: after the
// row-per-lane swizzled smem write, each lane re-reads (row i*8 + lane/4,
// 16-byte chunk lane%4) so every st.global instruction writes eight complete
// 64-byte row segments.  Keeps the TMA engine free for operand loads.
__device__ __forceinline__ void stage_store_lsu(uint8_t* buf, __nv_bfloat16* gdst, size_t ld, const float* v,
                                                int lane, bool stream) {
    uint4* rowp = reinterpret_cast<uint4*>(buf + lane * 64);
    const int sw = (lane >> 1) & 3;
    __syncwarp();  // previous chunk's readers are done with buf
#pragma unroll
    for (int j = 0; j < 4; ++j) rowp[j ^ sw] = pack8(v + 8 * j);
    __syncwarp();
    const int cj = lane & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = i * 8 + (lane >> 2);
        const uint4 val = *reinterpret_cast<const uint4*>(buf + r * 64 + ((cj ^ ((r >> 1) & 3)) << 4));
        if (stream) ptx::st_cs_v4(gdst + (size_t)r * ld + cj * 8, val);
        else *reinterpret_cast<uint4*>(gdst + (size_t)r * ld + cj * 8) = val;
    }
}

// Epilogue store of one 32x32 chunk: LSU write-back or TMA bulk store.  A/B on
// one B200 (interleaved runs): LSU is faster for WGRAD (2.10 vs 2.17-2.42 ms),
// slower for BWD1 (+6%) and neutral for FWD1/BWD2, so only WGRAD uses it
// (kLsuStores); debug bits 4 / 8 force TMA / LSU for experiments.
// GemmArgs.debug bit 2 (4) forces TMA stores, bit 3 (8) forces LSU stores.
// Streaming (evict-first) stores for outputs nobody reads soon: WGRAD's weight
// gradients always (bit 10 = 1024 turns it off for A/B runs; layer step, 5
// interleaved runs of 40 steps each: 6.968 vs 7.017 ms mean), other LSU stores
// with bit 7 (128); `evict_first` asks the same of TMA stores (FWD1's a/b with
// bit 11 = 2048: 6.975 ms, no gain).
template <int kRing, bool kLsuDefault = false>
__device__ __forceinline__ void emit32(EpiRing& ring, const CUtensorMap* m, __nv_bfloat16* gbase, size_t ld,
                                       const float* v, int lane, int col, int row0, int debug,
                                       bool evict_first = false) {
    const bool lsu = (debug & 4) ? false : ((debug & 8) ? true : kLsuDefault);
    const bool stream = kLsuDefault ? !(debug & 1024) : ((debug & 128) || evict_first);
    if (lsu) stage_store_lsu(ring.base, gbase + (size_t)row0 * ld + col, ld, v, lane, stream);
    else stage_store<kRing>(ring, m, v, lane, col, row0, evict_first);
}

// 32 rows x 64 columns (128-byte rows, SWIZZLE_128B: chunk j of row r at j ^ (r & 7)).
template <int kRing>
__device__ __forceinline__ void stage_store64(EpiRing& ring, const CUtensorMap* m, const float* v, int lane, int col,
                                              int row0) {
    uint8_t* buf = ring.base + ring.idx * 4096;
    if (lane == 0) ptx::bulk_wait_read<kRing - 1>();
    __syncwarp();
    uint4* rowp = reinterpret_cast<uint4*>(buf + lane * 128);
    const int sw = lane & 7;
#pragma unroll
    for (int j = 0; j < 8; ++j) rowp[j ^ sw] = pack8(v + 8 * j);
    ptx::fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
        ptx::tma_store_2d(m, buf, col, row0);
        ptx::bulk_commit();
    }
    ring.idx = (ring.idx + 1 == kRing) ? 0 : ring.idx + 1;
}

// BWD2 load ring: two buffers, each holding a 32x32 chunk of the stored `a`
// and `b` pre-activations (2 KB each, SWIZZLE_64B), filled by TMA and tracked
// by one mbarrier per buffer.
struct EpiLoads {
    uint8_t* base;     // 2 x (a 2 KB, b 2 KB)
    uint64_t* bar;     // 2 mbarriers
    int idx;           // next buffer to fill
    uint32_t phases;   // bit i = parity of bar[i]'s next completion
};

__device__ __forceinline__ void epi_load_issue(EpiLoads& ld, const CUtensorMap* ma, const CUtensorMap* mb, int col,
                                               int row0, int lane) {
    if (lane == 0) {
        uint8_t* buf = ld.base + ld.idx * 2 * kStageBufBytes;
        ptx::mbar_arrive_expect_tx(&ld.bar[ld.idx], 2 * kStageBufBytes);
        ptx::tma_load_2d(ma, &ld.bar[ld.idx], buf, col, row0);
        ptx::tma_load_2d(mb, &ld.bar[ld.idx], buf + kStageBufBytes, col, row0);
    }
    ld.idx ^= 1;
}

// Wait for buffer `i`, then unpack this lane's row of a and b.
__device__ __forceinline__ void epi_load_take(EpiLoads& ld, int i, int lane, float* av, float* bv) {
    ptx::mbar_wait(&ld.bar[i], (ld.phases >> i) & 1u);
    ld.phases ^= 1u << i;
    const uint8_t* buf = ld.base + i * 2 * kStageBufBytes;
    const uint4* ra = reinterpret_cast<const uint4*>(buf + lane * 64);
    const uint4* rb = reinterpret_cast<const uint4*>(buf + kStageBufBytes + lane * 64);
    const int sw = (lane >> 1) & 3;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        unpack8(ra[j ^ sw], av + 8 * j);
        unpack8(rb[j ^ sw], bv + 8 * j);
    }
    __syncwarp();  // every lane has read buffer i before it can be refilled
}

// Single-box variant (kWgradAcc): buffer i of the ring holds one 32 x 32 chunk.
__device__ __forceinline__ void epi_load1_issue(EpiLoads& ld, const CUtensorMap* m, int col, int row0, int lane) {
    if (lane == 0) {
        ptx::mbar_arrive_expect_tx(&ld.bar[ld.idx], kStageBufBytes);
        ptx::tma_load_2d(m, &ld.bar[ld.idx], ld.base + ld.idx * kStageBufBytes, col, row0);
    }
    ld.idx ^= 1;
}

__device__ __forceinline__ void epi_load1_take(EpiLoads& ld, int i, int lane, float* v) {
    ptx::mbar_wait(&ld.bar[i], (ld.phases >> i) & 1u);
    ld.phases ^= 1u << i;
    const uint4* r = reinterpret_cast<const uint4*>(ld.base + i * kStageBufBytes + lane * 64);
    const int sw = (lane >> 1) & 3;
#pragma unroll
    for (int j = 0; j < 4; ++j) unpack8(r[j ^ sw], v + 8 * j);
    __syncwarp();  // every lane has read buffer i before it can be refilled
}

__device__ __forceinline__ float sigmoidf_(float x) { return 1.0f / (1.0f + __expf(-x)); }

// One epilogue warp: TMEM lane quarter q (rows q*32..q*32+31 of this CTA's
// 128) and column half `half` of the 256-column accumulator.  Waits on the
// accumulator itself (tfull) so that loads which do not depend on it (the
// stored pre-activations in BWD2) are issued before the wait.  Segment rows
// are padded to 128, so a warp's 32 rows are either all inside the padded
// segment or all outside it.
template <int kMode, int kCG>
__device__ __forceinline__ void epilogue_tile(const TmaSet& tm, const GemmArgs& a, const TileInfo& ti,
                                              uint32_t tmem_acc, int q, int half, int lane, uint32_t rank,
                                              bool k_empty, uint64_t* tfull, uint32_t tphase, EpiRing& ring,
                                              EpiLoads& ld) {
    using C = Cfg<kCG>;
    constexpr int kRing = Geo<kMode, kCG>::kRing;
    uint32_t r0[32], r1[32];
    float v0[32], v1[32], v2[32];
    const uint32_t lane_addr = tmem_acc + ((uint32_t)(q * 32) << 16);
    if constexpr (is_wgrad1<kMode>()) {
        const int e = ti.seg;
        const int orow = ti.m_tile * C::kTileM + rank * kRowsPerCta + q * 32;  // first output row of the warp
        const int smap = ti.sub == 0 ? 0 : (ti.sub == 1 ? 2 : 1);            // dW1, dW3, dW2
        const int grow = (ti.sub == 2 ? e * a.H : e * a.F) + orow;
        const int col0 = ti.n_tile * kBN;
        if constexpr (kMode == kWgradAcc) {
            __nv_bfloat16* const obase = ti.sub == 2 ? a.out1 : (ti.sub == 0 ? a.out0 : a.out2);
            const size_t old_ld = ti.sub == 2 ? a.F : a.H;
            const CUtensorMap* om = &tm.st[smap];
            const int c0 = col0 + half * 128;
            epi_load1_issue(ld, om, c0, grow, lane);   // chunk 0 of the old gradient, before the accumulator wait
            ptx::mbar_wait(tfull, tphase);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int cc = 0; cc < 4; ++cc) {
                const int cur = ld.idx ^ 1;   // buffer holding chunk cc
                if (cc + 1 < 4) epi_load1_issue(ld, om, c0 + (cc + 1) * 32, grow, lane);
                if (!k_empty) ptx::tmem_ld_32x32b_x32(lane_addr + half * 128 + cc * 32, r0);
                epi_load1_take(ld, cur, lane, v1);
                if (!k_empty) {
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) v0[i] = __uint_as_float(r0[i]) + v1[i];
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v0[i] = v1[i];
                }
                emit32<kRing, kLsuStores>(ring, om, obase, old_ld, v0, lane, c0 + cc * 32, grow, a.debug);
            }
            return;
        }
        ptx::mbar_wait(tfull, tphase);
        ptx::tc_fence_after();
        if constexpr (Geo<kMode, kCG>::kWide) {
            float w[64];
            for (int c = half * 128; c < half * 128 + 128; c += 64) {
                if (!k_empty) {
                    ptx::tmem_ld_32x32b_x32(lane_addr + c, r0);
                    ptx::tmem_ld_32x32b_x32(lane_addr + c + 32, r1);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        w[i] = __uint_as_float(r0[i]);
                        w[32 + i] = __uint_as_float(r1[i]);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 64; ++i) w[i] = 0.f;
                }
                if (!(a.debug & 1)) stage_store64<kRing>(ring, &tm.st[smap], w, lane, col0 + c, grow);
            }
        } else {
            __nv_bfloat16* const obase = ti.sub == 2 ? a.out1 : (ti.sub == 0 ? a.out0 : a.out2);
            for (int c = half * 128; c < half * 128 + 128; c += 32) {
                if (!k_empty) {
                    ptx::tmem_ld_32x32b_x32(lane_addr + c, r0);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) v0[i] = __uint_as_float(r0[i]);
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v0[i] = 0.f;
                }
                if (!(a.debug & 1)) {
                    __nv_bfloat16* base = obase;
                    emit32<kRing, kLsuStores>(ring, &tm.st[smap], base, ti.sub == 2 ? a.F : a.H, v0, lane,
                                              col0 + c, grow, a.debug);
                }
            }
        }
        return;
    } else {
        const int cnt = a.seg_count[ti.seg];
        const int rel = ti.m_tile * C::kTileM + rank * kRowsPerCta + q * 32;  // first row of this warp
        const int limit = round_up(cnt, kSegPad);
        const bool live = rel < limit;                                        // warp-uniform
        const int row0 = a.seg_base[ti.seg] + rel;
        if constexpr (Geo<kMode, kCG>::kTmaEpiLoads) {
            // SwiGLU backward with the stored pre-activations (a, b) streamed by
            // TMA one 32-column chunk ahead; chunk 0 is requested before the
            // accumulator wait.
            // experiment switches: debug & 32 skips the a/b loads, & 64 the stores
            const bool no_ld = a.debug & 32, no_st = a.debug & 64;
            const int col0 = ti.n_tile * kBN + half * 128;
            if constexpr (Geo<kMode, kCG>::kInPlace) {
                // buffers: a chunk at ld.base (then da), b chunk at +2 KB (then db)
                uint8_t* const abuf = ld.base;
                uint8_t* const bbuf = ld.base + kStageBufBytes;
                auto issue = [&](int col) {
                    if (lane == 0) ptx::bulk_wait_read<0>();   // the previous chunk's stores have read the buffers
                    __syncwarp();
                    ld.idx = 0;
                    epi_load_issue(ld, &tm.m[2], &tm.m[3], col, row0, lane);
                };
                if (live) issue(col0);
                ptx::mbar_wait(tfull, tphase);
                ptx::tc_fence_after();
                if (!live) return;
#pragma unroll 1
                for (int cc = 0; cc < 4; ++cc) {
                    const int c = cc * 32;
                    ptx::tmem_ld_32x32b_x32(lane_addr + half * 128 + c, r0);
                    epi_load_take(ld, 0, lane, v0, v1);
                    ptx::tmem_ld_wait();
                    if (a.out2) {
                        // h = silu(a) * b rebuilt from the stored (bf16) a, b for a caller
                        // that dropped the forward's h (WGRAD's dW2 operand): 64 contiguous
                        // bytes of this lane's row, straight from registers
#pragma unroll
                        for (int i = 0; i < 32; ++i) v2[i] = v0[i] * sigmoidf_(v0[i]) * v1[i];
                        uint4* hp = reinterpret_cast<uint4*>(a.out2 + (size_t)(row0 + lane) * a.F + col0 + c);
#pragma unroll
                        for (int j = 0; j < 4; ++j) hp[j] = pack8(v2 + 8 * j);
                    }
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const float dm = __uint_as_float(r0[i]);
                        const float av = v0[i], bv = v1[i];
                        const float sg = sigmoidf_(av);
                        v0[i] = dm * bv * (sg * (1.0f + av * (1.0f - sg)));
                        v1[i] = dm * (av * sg);
                    }
                    uint4* ra = reinterpret_cast<uint4*>(abuf + lane * 64);
                    uint4* rb = reinterpret_cast<uint4*>(bbuf + lane * 64);
                    const int sw = (lane >> 1) & 3;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        ra[j ^ sw] = pack8(v0 + 8 * j);
                        rb[j ^ sw] = pack8(v1 + 8 * j);
                    }
                    ptx::fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::tma_store_2d(&tm.st[0], abuf, col0 + c, row0);
                        ptx::tma_store_2d(&tm.st[1], bbuf, col0 + c, row0);
                        ptx::bulk_commit();
                    }
                    if (cc + 1 < 4) issue(col0 + c + 32);
                }
                return;
            }
            if (live && !no_ld) {
                if (Geo<kMode, kCG>::kEpiLoadBufs == 1) ld.idx = 0;
                epi_load_issue(ld, &tm.m[2], &tm.m[3], col0, row0, lane);
            }
            ptx::mbar_wait(tfull, tphase);
            ptx::tc_fence_after();
            if (!live) return;
            constexpr bool kOneBuf = Geo<kMode, kCG>::kEpiLoadBufs == 1;
#pragma unroll 1
            for (int cc = 0; cc < 4; ++cc) {
                const int c = cc * 32;
                const int cur = kOneBuf ? 0 : (ld.idx ^ 1);  // buffer holding chunk cc
                if (!kOneBuf && cc + 1 < 4 && !no_ld)
                    epi_load_issue(ld, &tm.m[2], &tm.m[3], col0 + c + 32, row0, lane);
                ptx::tmem_ld_32x32b_x32(lane_addr + half * 128 + c, r0);
                if (!no_ld) {
                    epi_load_take(ld, cur, lane, v0, v1);
                    if (kOneBuf && cc + 1 < 4) {   // refill the (now read) buffer with the next chunk
                        ld.idx = 0;
                        epi_load_issue(ld, &tm.m[2], &tm.m[3], col0 + c + 32, row0, lane);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) { v0[i] = 0.5f; v1[i] = 0.25f; }
                }
                ptx::tmem_ld_wait();
                if (a.out2) {   // h = silu(a) * b for a caller that dropped the forward's h
#pragma unroll
                    for (int i = 0; i < 32; ++i) v2[i] = v0[i] * sigmoidf_(v0[i]) * v1[i];
                    uint4* hp = reinterpret_cast<uint4*>(a.out2 + (size_t)(row0 + lane) * a.F + col0 + c);
#pragma unroll
                    for (int j = 0; j < 4; ++j) hp[j] = pack8(v2 + 8 * j);
                }
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const float dm = __uint_as_float(r0[i]);
                    const float av = v0[i], bv = v1[i];
                    const float sg = sigmoidf_(av);
                    v0[i] = dm * bv * (sg * (1.0f + av * (1.0f - sg)));
                    v1[i] = dm * (av * sg);
                }
                if (no_st) continue;
                emit32<kRing>(ring, &tm.st[0], a.out0, a.F, v0, lane, col0 + c, row0, a.debug);
                emit32<kRing>(ring, &tm.st[1], a.out1, a.F, v1, lane, col0 + c, row0, a.debug);
            }
            return;
        } else if constexpr (kMode == kBwd2) {
            // SwiGLU backward: prefetch the stored pre-activations (a, b) one
            // 32-column chunk ahead; the first chunk is in flight before the
            // accumulator wait.
            const int col0 = ti.n_tile * kBN + half * 128;
            const size_t off = (size_t)(row0 + lane) * a.F + col0;
            uint4 pa[2][4], pb[2][4];
            if (live) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    pa[0][i] = ld_nc_v4(a.in0 + off + 8 * i);
                    pb[0][i] = ld_nc_v4(a.in1 + off + 8 * i);
                }
            }
            ptx::mbar_wait(tfull, tphase);
            ptx::tc_fence_after();
            if (!live) return;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const int c = cc * 32;
                const int cur = cc & 1;
                if (cc + 1 < 4) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        pa[cur ^ 1][i] = ld_nc_v4(a.in0 + off + c + 32 + 8 * i);
                        pb[cur ^ 1][i] = ld_nc_v4(a.in1 + off + c + 32 + 8 * i);
                    }
                }
                ptx::tmem_ld_32x32b_x32(lane_addr + half * 128 + c, r0);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    unpack8(pa[cur][i], v0 + 8 * i);
                    unpack8(pb[cur][i], v1 + 8 * i);
                }
                if (a.out2) {   // h = silu(a) * b for a caller that dropped the forward's h
#pragma unroll
                    for (int i = 0; i < 32; ++i) v2[i] = v0[i] * sigmoidf_(v0[i]) * v1[i];
                    uint4* hp = reinterpret_cast<uint4*>(a.out2 + (size_t)(row0 + lane) * a.F + col0 + c);
#pragma unroll
                    for (int j = 0; j < 4; ++j) hp[j] = pack8(v2 + 8 * j);
                }
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const float dm = __uint_as_float(r0[i]);
                    const float av = v0[i], bv = v1[i];
                    const float sg = sigmoidf_(av);
                    v0[i] = dm * bv * (sg * (1.0f + av * (1.0f - sg)));
                    v1[i] = dm * (av * sg);
                }
                emit32<kRing>(ring, &tm.st[0], a.out0, a.F, v0, lane, col0 + c, row0, a.debug);
                emit32<kRing>(ring, &tm.st[1], a.out1, a.F, v1, lane, col0 + c, row0, a.debug);
            }
            return;
        }
        ptx::mbar_wait(tfull, tphase);
        ptx::tc_fence_after();
        if (!live) return;
        if constexpr (kMode == kFwd1) {
            const int col0 = ti.n_tile * 128;
            for (int c = half * 64; c < half * 64 + 64; c += 32) {
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
                // a, b are read again only by BWD2 (after FWD2, combine and the loss); h by FWD2 next
                const bool ef = a.debug & 2048;
                emit32<kRing>(ring, &tm.st[0], a.out0, a.F, v0, lane, col0 + c, row0, a.debug, ef);
                emit32<kRing>(ring, &tm.st[1], a.out1, a.F, v1, lane, col0 + c, row0, a.debug, ef);
                emit32<kRing>(ring, &tm.st[2], a.out2, a.F, v2, lane, col0 + c, row0, a.debug);
            }
        } else if constexpr (Geo<kMode, kCG>::kWide) {  // kFwd2 / kBwd1, 64-column stores
            const int col0 = ti.n_tile * kBN;
            float w[64];
            for (int c = half * 128; c < half * 128 + 128; c += 64) {
                ptx::tmem_ld_32x32b_x32(lane_addr + c, r0);
                ptx::tmem_ld_32x32b_x32(lane_addr + c + 32, r1);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    w[i] = __uint_as_float(r0[i]);
                    w[32 + i] = __uint_as_float(r1[i]);
                }
                stage_store64<kRing>(ring, &tm.st[0], w, lane, col0 + c, row0, a.debug);
            }
        } else {  // kFwd2 / kBwd1: plain bf16 store
            const int col0 = ti.n_tile * kBN;
            const CUtensorMap* smap = &tm.st[0];
            int orow = row0;
            int dbg = a.debug;
            if (a.peer_El) {   // straight into the source rank's receive plane over NVLink (TMA store)
                smap = &tm.stp[ti.seg / a.peer_El];
                orow = (a.peer_rank * a.peer_El + ti.seg % a.peer_El) * a.peer_cap + rel;
                dbg &= ~8;     // never the local LSU write-back
            }
            for (int c = half * 128; c < half * 128 + 128; c += 32) {
                ptx::tmem_ld_32x32b_x32(lane_addr + c, r0);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) v0[i] = __uint_as_float(r0[i]);
                emit32<kRing>(ring, smap, a.out0, a.H, v0, lane, col0 + c, orow, dbg);
            }
        }
    }
    (void)v2;
    (void)r1;
}

// kWgradW epilogue.  Per slot: read the warp's 32 rows x 128 columns from
// TMEM into registers (as packed bf16), release the slot, then write them out;
// the MMA issuer, which starts the next tile on slot 0 as soon as it is
// released, only waits for the TMEM reads, not for the global stores.  Each
// warp owns TMEM lane quarter q and a 128-column half of each 256-column slot.
// An expert without rows (k_empty) writes zeros.
__device__ __forceinline__ void tmem_take64(uint32_t taddr, uint32_t* pk) {
    uint32_t r0[32], r1[32];
    ptx::tmem_ld_32x32b_x32(taddr, r0);
    ptx::tmem_ld_32x32b_x32(taddr + 32, r1);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        pk[i] = pack2(__uint_as_float(r0[2 * i]), __uint_as_float(r0[2 * i + 1]));
        pk[16 + i] = pack2(__uint_as_float(r1[2 * i]), __uint_as_float(r1[2 * i + 1]));
    }
}

// 32 x 32 chunk of packed bf16 (16 words per lane = its row) through the
// swizzled staging buffer to global memory (same pattern as stage_store_lsu).
__device__ __forceinline__ void store_packed_lsu(uint8_t* buf, __nv_bfloat16* gdst, size_t ld, const uint32_t* p,
                                                 int lane, bool stream) {
    uint4* rowp = reinterpret_cast<uint4*>(buf + lane * 64);
    const int sw = (lane >> 1) & 3;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 4; ++j) rowp[j ^ sw] = make_uint4(p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3]);
    __syncwarp();
    const int cj = lane & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = i * 8 + (lane >> 2);
        const uint4 val = *reinterpret_cast<const uint4*>(buf + r * 64 + ((cj ^ ((r >> 1) & 3)) << 4));
        if (stream) ptx::st_cs_v4(gdst + (size_t)r * ld + cj * 8, val);
        else *reinterpret_cast<uint4*>(gdst + (size_t)r * ld + cj * 8) = val;
    }
}

__device__ __forceinline__ void epilogue_wide(const GemmArgs& a, const TileInfo& ti, uint32_t tmem_base, int q,
                                              int half, int lane, uint32_t rank, bool k_empty, uint64_t* tfull,
                                              uint64_t* tempty, uint32_t tphase, uint8_t* buf) {
    uint32_t pk[64];
    const int e = ti.seg;
    const int orow = ti.m_tile * 256 + rank * kRowsPerCta + q * 32;
    const uint32_t lane_addr = tmem_base + ((uint32_t)(q * 32) << 16) + half * 128;
#pragma unroll 1
    for (int slot = 0; slot < 2; ++slot) {
        __nv_bfloat16* dst;
        size_t ld;
        if (ti.sub == 0) {   // slot 0: dW1, slot 1: dW3 (same rows and columns)
            dst = (slot == 0 ? a.out0 : a.out2) + (size_t)(e * a.F + orow) * a.H + ti.n_tile * 256 + half * 128;
            ld = a.H;
        } else {             // dW2 columns f and f + 256
            dst = a.out1 + (size_t)(e * a.H + orow) * a.F + ti.n_tile * 512 + slot * 256 + half * 128;
            ld = a.F;
        }
        ptx::mbar_wait(&tfull[slot], tphase);
        ptx::tc_fence_after();
        if (!k_empty) {
            tmem_take64(lane_addr + slot * 256, pk);
            tmem_take64(lane_addr + slot * 256 + 64, pk + 32);
        } else {
#pragma unroll
            for (int i = 0; i < 64; ++i) pk[i] = 0u;
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(&tempty[slot], 0);
        if (!(a.debug & 1)) {
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) store_packed_lsu(buf, dst + cc * 32, ld, pk + 16 * cc, lane, !(a.debug & 1024));
        }
    }
}

// kWgradW MMA issuer (one thread of the leader CTA).  Per k-block it issues
// the slot-0 MMAs, then the slot-1 MMAs.  At the start of a tile slot 1 may
// still be draining the previous tile, so up to kStages - 1 k-blocks of slot-0
// MMAs run ahead (their stages stay held) and slot 1 catches up once the
// epilogue releases it.  tfull[0] is committed after the last slot-0 MMA so the
// epilogue starts on slot 0 while the last slot-1 MMAs still run.
template <int kStages, class S>
__device__ __forceinline__ void mma_wide(const GemmArgs& a, const S& sched, uint8_t* stages, uint64_t* full,
                                         uint64_t* empty, uint64_t* tfull, uint64_t* tempty, uint32_t tmem_base,
                                         int cid, int ncl) {
    constexpr int kSB = 3 * 16384;
    constexpr int kLag = kStages - 1;
    constexpr uint32_t idesc = ptx::make_idesc_bf16(256, kBN, true, true);
    auto issue = [&](uint32_t dtm, uint32_t aaddr, uint32_t baddr, int kb) {
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)
            ptx::mma_bf16<2>(dtm, ptx::make_sdesc(aaddr + k * 2048, 8192, 1024),
                             ptx::make_sdesc(baddr + k * 2048, 8192, 1024), idesc, (kb | k) != 0);
    };
    int stage = 0;
    uint32_t phase = 0, tph = 0;
    for (int t = cid; t < sched.total; t += ncl) {
        const TileInfo ti = sched.decode(t, a);
        const int nkb = wgrad_k_blocks(a, ti.seg);
        const uint32_t a0 = 0, b0 = ti.sub == 0 ? 32768 : 16384;   // MMA0 operands within a stage
        const uint32_t a1 = ti.sub == 0 ? 16384 : 0, b1 = 32768;   // MMA1 operands
        ptx::mbar_wait_cluster(&tempty[0], tph ^ 1);
        ptx::tc_fence_after();
        bool s1 = false;
        int pend0 = 0, pkb0 = 0, npend = 0;   // k-blocks whose slot-1 MMAs are still to issue
        for (int kb = 0; kb < nkb; ++kb) {
            ptx::mbar_wait(&full[stage], phase);
            ptx::tc_fence_after();
            const uint32_t sb = ptx::smem_u32(stages + stage * kSB);
            issue(tmem_base, sb + a0, sb + b0, kb);
            if (kb == nkb - 1) ptx::mma_commit<2>(&tfull[0], 0x3);
            if (npend == 0) { pend0 = stage; pkb0 = kb; }
            ++npend;
            if (!s1) {
                if (npend >= kLag || kb == nkb - 1) {
                    ptx::mbar_wait_cluster(&tempty[1], tph ^ 1);
                    s1 = true;
                } else {
                    s1 = ptx::mbar_try_wait_cluster(&tempty[1], tph ^ 1);
                }
                if (s1) ptx::tc_fence_after();
            }
            if (s1) {
                for (int i = 0; i < npend; ++i) {
                    const int st = (pend0 + i) % kStages;
                    const uint32_t pb = ptx::smem_u32(stages + st * kSB);
                    issue(tmem_base + kBN, pb + a1, pb + b1, pkb0 + i);
                    ptx::mma_commit<2>(&empty[st], 0x3);
                }
                npend = 0;
            }
            if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (nkb == 0) {   // expert without rows: the epilogue writes zeros
            ptx::mbar_wait_cluster(&tempty[1], tph ^ 1);
            ptx::mma_commit<2>(&tfull[0], 0x3);
        }
        ptx::mma_commit<2>(&tfull[1], 0x3);
        tph ^= 1;
    }
}

// ------------------------------------------------------------------ kernel
template <int kMode, int kCG>
__global__ void __launch_bounds__(kNumThreads, 1) moe_gemm_kernel(const __grid_constant__ TmaSet tm, GemmArgs a_in) {
    using C = Cfg<kCG>;
    using G = Geo<kMode, kCG>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stages = smem;
    uint8_t* staging = smem + G::kStages * G::kStageBytes;  // per-epilogue-warp rings
    uint64_t* full = reinterpret_cast<uint64_t*>(staging + kNumEpiWarps * G::kEpiWarpBytes);
    uint64_t* empty = full + G::kStages;
    uint64_t* tfull = empty + G::kStages;
    uint64_t* tempty = tfull + 2;
    uint64_t* ldbar = tempty + 2;  // 2 per epilogue warp (BWD2 TMA load ring)
    uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(ldbar + 2 * kNumEpiWarps);
    int* prefix = reinterpret_cast<int*>(tmem_base_slot + 1);
    // The segment table (base, count, expert; nseg <= 64) is read by every
    // role at every tile: keep a shared-memory copy so no tile start waits on a
    // global load.
    int* segtab = prefix + kMaxSeg + 2;
    for (int i = threadIdx.x; i < a_in.nseg; i += blockDim.x) {
        segtab[i] = a_in.seg_base[i];
        segtab[kMaxSeg + i] = a_in.seg_count[i];
        segtab[2 * kMaxSeg + i] = a_in.seg_expert[i];
    }
    __syncthreads();
    GemmArgs a = a_in;
    a.seg_base = segtab;
    a.seg_count = segtab + kMaxSeg;
    a.seg_expert = segtab + 2 * kMaxSeg;

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t rank = (kCG == 2) ? ptx::cluster_ctarank() : 0;
    const int cid = (kCG == 2) ? (int)ptx::cluster_id_x() : (int)blockIdx.x;
    const int ncl = (kCG == 2) ? (int)ptx::nclusters_x() : (int)gridDim.x;

    // ---- tile table (identical in every CTA)
    if (threadIdx.x == 0) {
        int acc = 0;
        prefix[0] = 0;
        if constexpr (kMode == kWgradW) {
            const int per_e = (a.F / 256) * (a.H / 256) + (a.H / 256) * (a.F / 512);
            for (int e = 0; e < a.E_local; ++e) {
                acc += per_e;
                prefix[e + 1] = acc;
            }
        } else if constexpr (is_wgrad1<kMode>()) {
            const int mask = wgrad_mask(a);
            const int per_e = (((mask & 1) != 0) + ((mask & 2) != 0)) * (a.F / C::kTileM) * (a.H / kBN) +
                              ((mask & 4) != 0) * (a.H / C::kTileM) * (a.F / kBN);
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
        for (int i = 0; i < 3; ++i) ptx::prefetch_tmap(&tm.st[i]);
        for (int s = 0; s < G::kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], kCG * kNumEpiWarps);
        }
        for (int i = 0; i < 2 * kNumEpiWarps; ++i) ptx::mbar_init(&ldbar[i], 1);
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
    constexpr bool kW = (is_wgrad1<kMode>() || kMode == kWgradW);
    sched.total = prefix[kW ? a.E_local : a.nseg];

    if (warp == 0) {
        // ================= TMA producer
        if (ptx::elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cid; t < sched.total; t += ncl) {
                const TileInfo ti = sched.decode(t, a);
                if constexpr (kW) {
                    for (int s = 0; s < a.nseg; ++s) {
                        if (a.seg_expert[s] != ti.seg) continue;
                        const int nkb = ceil_div(a.seg_count[s], kBK);
                        for (int kb = 0; kb < nkb; ++kb) {
                            ptx::mbar_wait(&empty[stage], phase ^ 1);
                            if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], G::kStageBytes * kCG);
                            uint8_t* sA = stages + stage * G::kStageBytes;
                            if constexpr (kMode == kWgradW)
                                produce_wide(tm, ti, a.seg_base[s] + kb * kBK, rank, &full[stage], sA);
                            else
                                produce_kblock<kMode, kCG>(tm, a, ti, a.seg_base[s] + kb * kBK, 0, rank,
                                                           &full[stage], sA, sA + C::kABytes);
                            if (++stage == G::kStages) { stage = 0; phase ^= 1; }
                        }
                    }
                } else {
                    const int nkb = mode_k_blocks<kMode>(a);
                    for (int kb = 0; kb < nkb; ++kb) {
                        ptx::mbar_wait(&empty[stage], phase ^ 1);
                        if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], G::kStageBytes * kCG);
                        uint8_t* sA = stages + stage * G::kStageBytes;
                        produce_kblock<kMode, kCG>(tm, a, ti, kb, 0, rank, &full[stage], sA, sA + C::kABytes);
                        if (++stage == G::kStages) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer (leader CTA of the pair)
        if constexpr (kMode == kWgradW) {
            if (rank == 0 && lane == 0)
                mma_wide<G::kStages>(a, sched, stages, full, empty, tfull, tempty, tmem_base, cid, ncl);
        } else if (rank == 0) {
            constexpr uint32_t idesc = ptx::make_idesc_bf16(kRowsPerCta * kCG, kBN, Majors<kMode>::a, Majors<kMode>::b);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = cid; t < sched.total; t += ncl) {
                const TileInfo ti = sched.decode(t, a);
                const int nkb = is_wgrad1<kMode>() ? wgrad_k_blocks(a, ti.seg) : mode_k_blocks<kMode>(a);
                ptx::mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t dtm = tmem_base + acc * kBN;
                for (int kb = 0; kb < nkb; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        const uint32_t aaddr = ptx::smem_u32(stages + stage * G::kStageBytes);
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
                    if (++stage == G::kStages) { stage = 0; phase ^= 1; }
                }
                if (ptx::elect_one()) ptx::mma_commit<kCG>(&tfull[acc], 0x3);
                __syncwarp();
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {
        // ================= epilogue (warps 2..9): lane quarter warp%4, column half
        const int q = warp % 4;
        const int half = (warp - 2) / 4;
        int acc = 0;
        uint32_t acc_phase = 0;
        EpiRing ring{staging + (warp - 2) * G::kEpiWarpBytes, 0};
        EpiLoads ld{staging + (warp - 2) * G::kEpiWarpBytes + (G::kInPlace ? 0 : G::kRing * G::kStoreBytes),
                    ldbar + 2 * (warp - 2), 0, 0};
        if constexpr (kMode == kWgradW) {
            uint32_t tphase = 0;
            for (int t = cid; t < sched.total; t += ncl) {
                const TileInfo ti = sched.decode(t, a);
                const bool k_empty = wgrad_k_blocks(a, ti.seg) == 0;
                epilogue_wide(a, ti, tmem_base, q, half, lane, rank, k_empty, tfull, tempty, tphase, ring.base);
                tphase ^= 1;
            }
        } else
        for (int t = cid; t < sched.total; t += ncl) {
            const TileInfo ti = sched.decode(t, a);
            const bool k_empty = is_wgrad1<kMode>() ? (wgrad_k_blocks(a, ti.seg) == 0) : false;
            epilogue_tile<kMode, kCG>(tm, a, ti, tmem_base + acc * kBN, q, half, lane, rank, k_empty, &tfull[acc],
                                      acc_phase, ring, ld);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(&tempty[acc], 0);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (lane == 0) ptx::bulk_wait<0>();  // all stores of this warp complete
        __syncwarp();
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
static int make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, bool mn_major,
                    bool ptr_is_store_target = false, bool wide = false) {
    EncodeTiledFn enc = get_encode();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return B200MOE_ERR_CUDA;
    }
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld * 2};
    cuuint32_t box[2] = {64, mn_major ? 64u : 128u};
    cuuint32_t estr[2] = {1, 1};
    CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B;
    if (ptr_is_store_target) {  // epilogue map: 32 x 32 boxes (64-byte swizzle) or 32 x 64 (128-byte)
        box[0] = wide ? 64 : 32;
        box[1] = 32;
        sw = wide ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    }
    auto encode = [&] {
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUresult r = encode();
    if (r == CUDA_ERROR_INVALID_CONTEXT && bind_current_context()) r = encode();
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d) inner=%llu outer=%llu ld=%llu", (int)r,
                  (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)ld);
        return B200MOE_ERR_CUDA;
    }
    return B200MOE_OK;
}

// Diagnostics knobs (tests and A/B tools only; the product path never sets
// them).  Thread-local, so concurrent callers on other threads always get the
// defaults: CTA pairs, one persistent CTA per SM, no debug flags.
static thread_local int g_cta_group = 2;  // 2 = CTA-pair kernels (default), 1 = single-SM kernels
static thread_local int g_max_ctas = kNumSMs;
static thread_local int g_debug = 0;

template <int kMode, int kCG>
static int launch(const TmaSet& tm, const GemmArgs& a, cudaStream_t s, int grid_ctas = 0) {
    using G = Geo<kMode, kCG>;
    static_assert(G::kSmemBytes <= 227 * 1024, "shared memory plan exceeds 227 KB");
    auto kern = moe_gemm_kernel<kMode, kCG>;
    static std::atomic<uint64_t> attr_done{0};
    if (cudaError_t ae = ensure_smem_attr(kern, G::kSmemBytes, attr_done); ae != cudaSuccess) {
        set_error("moe_gemm_kernel<%d,%d> smem attribute: %s", kMode, kCG, cudaGetErrorString(ae));
        return B200MOE_ERR_CUDA;
    }
    cudaLaunchConfig_t cfg = {};
    // persistent grid: one CTA per SM, or `grid_ctas` (a per-call request, e.g.
    // to co-run two GEMMs on disjoint halves of the chip), or the diagnostics knob
    const int want = grid_ctas > 0 ? (grid_ctas < g_max_ctas ? grid_ctas : g_max_ctas) : g_max_ctas;
    int grid = want - (want % kCG);
    if (grid < kCG) grid = kCG;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kNumThreads);
    cfg.dynamicSmemBytes = G::kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    GemmArgs args = a;
    args.debug = g_debug;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tm, args);
    if (e != cudaSuccess) {
        set_error("moe_gemm_kernel<%d,%d> launch: %s", kMode, kCG, cudaGetErrorString(e));
        return B200MOE_ERR_CUDA;
    }
    return B200MOE_OK;
}

template <int kMode>
static int dispatch_launch(const TmaSet& tm, const GemmArgs& a, cudaStream_t s, int grid_ctas = 0) {
    return g_cta_group == 2 ? launch<kMode, 2>(tm, a, s, grid_ctas) : launch<kMode, 1>(tm, a, s, grid_ctas);
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

int b200moe_gemm_set_debug(int flags) {
    g_debug = flags;
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
    B200_TRY(make_map(&tm.st[0], a_out, F, rows, F, false, true));
    B200_TRY(make_map(&tm.st[1], b_out, F, rows, F, false, true));
    B200_TRY(make_map(&tm.st[2], h_out, F, rows, F, false, true));
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
    B200_TRY(make_map(&tm.st[0], o_out, H, rows, H, false, true, kWideStores && g_cta_group == 2));
    tm.st[1] = tm.st[2] = tm.st[0];
    GemmArgs a = {seg_base, seg_count, seg_expert, nseg, H, F, E_local,
                  (__nv_bfloat16*)o_out, nullptr, nullptr, nullptr, nullptr};
    return dispatch_launch<kFwd2>(tm, a, stream);
}

// Receive-plane store maps of every rank (host array of device base pointers,
// each plane dst_rows x H bf16) for the peer-output FWD2 / BWD1.
static int peer_maps(TmaSet& tm, const uint64_t* dst_host, int world, int H, int dst_rows) {
    B200_CHECK_ARG(world >= 1 && world <= kMaxPeers, B200MOE_ERR_CONFIG, "world %d outside [1, %d]", world, kMaxPeers);
    for (int r = 0; r < world; ++r) B200_TRY(make_map(&tm.stp[r], (const void*)dst_host[r], H, dst_rows, H, false, true));
    return B200MOE_OK;
}

int b200moe_expert_fwd2_peer(const void* h, const void* w2, const int* seg_base, const int* seg_count,
                             const int* seg_expert, int nseg, int rows, int H, int F, int E_local,
                             const uint64_t* dst_host, int world, int rank, int cap_pad, int dst_rows,
                             cudaStream_t stream) {
    B200_TRY(check_common(nseg, H, F, E_local));
    B200_CHECK_ARG(nseg == world * E_local && rank >= 0 && rank < world && cap_pad % 128 == 0 &&
                       (int64_t)world * E_local * cap_pad <= dst_rows, B200MOE_ERR_CONFIG,
                   "peer FWD2: nseg %d, world %d, E_local %d, rank %d, cap_pad %d, dst_rows %d", nseg, world, E_local,
                   rank, cap_pad, dst_rows);
    TmaSet tm = {};
    B200_TRY(make_map(&tm.m[0], h, F, rows, F, false));
    B200_TRY(make_map(&tm.m[1], w2, F, (uint64_t)E_local * H, F, false));
    tm.m[2] = tm.m[3] = tm.m[4] = tm.m[0];
    B200_TRY(peer_maps(tm, dst_host, world, H, dst_rows));
    tm.st[0] = tm.st[1] = tm.st[2] = tm.stp[rank];
    GemmArgs a = {seg_base, seg_count, seg_expert, nseg, H, F, E_local, nullptr, nullptr, nullptr, nullptr, nullptr};
    a.peer_El = E_local;
    a.peer_rank = rank;
    a.peer_cap = cap_pad;
    return dispatch_launch<kFwd2>(tm, a, stream);
}

int b200moe_expert_bwd1_peer(const void* da, const void* db, const void* w1, const void* w3, const int* seg_base,
                             const int* seg_count, const int* seg_expert, int nseg, int rows, int H, int F,
                             int E_local, const uint64_t* dst_host, int world, int rank, int cap_pad, int dst_rows,
                             cudaStream_t stream) {
    B200_TRY(check_common(nseg, H, F, E_local));
    B200_CHECK_ARG(nseg == world * E_local && rank >= 0 && rank < world && cap_pad % 128 == 0 &&
                       (int64_t)world * E_local * cap_pad <= dst_rows, B200MOE_ERR_CONFIG,
                   "peer BWD1: nseg %d, world %d, E_local %d, rank %d, cap_pad %d, dst_rows %d", nseg, world, E_local,
                   rank, cap_pad, dst_rows);
    TmaSet tm = {};
    B200_TRY(make_map(&tm.m[0], da, F, rows, F, false));
    B200_TRY(make_map(&tm.m[1], db, F, rows, F, false));
    B200_TRY(make_map(&tm.m[2], w1, H, (uint64_t)E_local * F, H, true));
    B200_TRY(make_map(&tm.m[3], w3, H, (uint64_t)E_local * F, H, true));
    tm.m[4] = tm.m[0];
    B200_TRY(peer_maps(tm, dst_host, world, H, dst_rows));
    tm.st[0] = tm.st[1] = tm.st[2] = tm.stp[rank];
    GemmArgs a = {seg_base, seg_count, seg_expert, nseg, H, F, E_local, nullptr, nullptr, nullptr, nullptr, nullptr};
    a.peer_El = E_local;
    a.peer_rank = rank;
    a.peer_cap = cap_pad;
    return dispatch_launch<kBwd1>(tm, a, stream);
}

int b200moe_expert_bwd2(const void* dout, const void* w2, const void* a_pre, const void* b_pre, const int* seg_base,
                        const int* seg_count, const int* seg_expert, int nseg, int rows, int H, int F, int E_local,
                        void* da_out, void* db_out, cudaStream_t stream) {
    return b200moe_expert_bwd2_ex(dout, w2, a_pre, b_pre, seg_base, seg_count, seg_expert, nseg, rows, H, F, E_local,
                                  da_out, db_out, 0, stream);
}

int b200moe_expert_bwd2_ex(const void* dout, const void* w2, const void* a_pre, const void* b_pre,
                           const int* seg_base, const int* seg_count, const int* seg_expert, int nseg, int rows,
                           int H, int F, int E_local, void* da_out, void* db_out, int grid_ctas,
                           cudaStream_t stream) {
    return b200moe_expert_bwd2_h(dout, w2, a_pre, b_pre, seg_base, seg_count, seg_expert, nseg, rows, H, F, E_local,
                                 da_out, db_out, nullptr, grid_ctas, stream);
}

int b200moe_expert_bwd2_h(const void* dout, const void* w2, const void* a_pre, const void* b_pre,
                          const int* seg_base, const int* seg_count, const int* seg_expert, int nseg, int rows,
                          int H, int F, int E_local, void* da_out, void* db_out, void* h_out, int grid_ctas,
                          cudaStream_t stream) {
    B200_TRY(check_common(nseg, H, F, E_local));
    TmaSet tm = {};
    B200_TRY(make_map(&tm.m[0], dout, H, rows, H, false));
    B200_TRY(make_map(&tm.m[1], w2, F, (uint64_t)E_local * H, F, true));
    B200_TRY(make_map(&tm.m[2], a_pre, F, rows, F, false, true));  // epilogue loads: 32 x 32 boxes
    B200_TRY(make_map(&tm.m[3], b_pre, F, rows, F, false, true));
    tm.m[4] = tm.m[0];
    B200_TRY(make_map(&tm.st[0], da_out, F, rows, F, false, true));
    B200_TRY(make_map(&tm.st[1], db_out, F, rows, F, false, true));
    tm.st[2] = tm.st[0];
    GemmArgs a = {seg_base, seg_count, seg_expert, nseg, H, F, E_local,
                  (__nv_bfloat16*)da_out, (__nv_bfloat16*)db_out, (__nv_bfloat16*)h_out,
                  (const __nv_bfloat16*)a_pre, (const __nv_bfloat16*)b_pre};
    return dispatch_launch<kBwd2>(tm, a, stream, grid_ctas);
}

int b200moe_expert_bwd1(const void* da, const void* db, const void* w1, const void* w3, const int* seg_base,
                        const int* seg_count, const int* seg_expert, int nseg, int rows, int H, int F, int E_local,
                        void* dxp_out, cudaStream_t stream) {
    return b200moe_expert_bwd1_ex(da, db, w1, w3, seg_base, seg_count, seg_expert, nseg, rows, H, F, E_local, dxp_out,
                                  0, stream);
}

int b200moe_expert_bwd1_ex(const void* da, const void* db, const void* w1, const void* w3, const int* seg_base,
                           const int* seg_count, const int* seg_expert, int nseg, int rows, int H, int F, int E_local,
                           void* dxp_out, int grid_ctas, cudaStream_t stream) {
    B200_TRY(check_common(nseg, H, F, E_local));
    TmaSet tm = {};
    B200_TRY(make_map(&tm.m[0], da, F, rows, F, false));
    B200_TRY(make_map(&tm.m[1], db, F, rows, F, false));
    B200_TRY(make_map(&tm.m[2], w1, H, (uint64_t)E_local * F, H, true));
    B200_TRY(make_map(&tm.m[3], w3, H, (uint64_t)E_local * F, H, true));
    tm.m[4] = tm.m[0];
    B200_TRY(make_map(&tm.st[0], dxp_out, H, rows, H, false, true, kWideStores && g_cta_group == 2));
    tm.st[1] = tm.st[2] = tm.st[0];
    GemmArgs a = {seg_base, seg_count, seg_expert, nseg, H, F, E_local,
                  (__nv_bfloat16*)dxp_out, nullptr, nullptr, nullptr, nullptr};
    return dispatch_launch<kBwd1>(tm, a, stream, grid_ctas);
}

int b200moe_expert_wgrad(const void* xp, const void* h, const void* dout, const void* da, const void* db,
                         const int* seg_base, const int* seg_count, const int* seg_expert, int nseg, int rows, int H,
                         int F, int E_local, void* dw1, void* dw2, void* dw3, cudaStream_t stream) {
    return b200moe_expert_wgrad_acc(xp, h, dout, da, db, seg_base, seg_count, seg_expert, nseg, rows, H, F, E_local,
                                    dw1, dw2, dw3, 0, stream);
}

int b200moe_expert_wgrad_acc(const void* xp, const void* h, const void* dout, const void* da, const void* db,
                             const int* seg_base, const int* seg_count, const int* seg_expert, int nseg, int rows,
                             int H, int F, int E_local, void* dw1, void* dw2, void* dw3, int accumulate,
                             cudaStream_t stream) {
    return b200moe_expert_wgrad_ex(xp, h, dout, da, db, seg_base, seg_count, seg_expert, nseg, rows, H, F, E_local,
                                   dw1, dw2, dw3, accumulate, 7, 0, stream);
}

int b200moe_expert_wgrad_ex(const void* xp, const void* h, const void* dout, const void* da, const void* db,
                            const int* seg_base, const int* seg_count, const int* seg_expert, int nseg, int rows,
                            int H, int F, int E_local, void* dw1, void* dw2, void* dw3, int accumulate, int subs,
                            int grid_ctas, cudaStream_t stream) {
    B200_CHECK_ARG(subs >= 1 && subs <= 7, B200MOE_ERR_CONFIG, "wgrad sub-problem mask %d outside [1, 7]", subs);
    B200_TRY(check_common(nseg, H, F, E_local));
    TmaSet tm = {};
    B200_TRY(make_map(&tm.m[0], dout, H, rows, H, true));
    B200_TRY(make_map(&tm.m[1], h, F, rows, F, true));
    B200_TRY(make_map(&tm.m[2], da, F, rows, F, true));
    B200_TRY(make_map(&tm.m[3], xp, H, rows, H, true));
    B200_TRY(make_map(&tm.m[4], db, F, rows, F, true));
    const bool wide = kWideStores && g_cta_group == 2;
    B200_TRY(make_map(&tm.st[0], dw1, H, (uint64_t)E_local * F, H, false, true, wide));
    B200_TRY(make_map(&tm.st[1], dw2, F, (uint64_t)E_local * H, F, false, true, wide));
    B200_TRY(make_map(&tm.st[2], dw3, H, (uint64_t)E_local * F, H, false, true, wide));
    GemmArgs a = {seg_base, seg_count, seg_expert, nseg, H, F, E_local,
                  (__nv_bfloat16*)dw1, (__nv_bfloat16*)dw2, (__nv_bfloat16*)dw3, nullptr, nullptr};
    a.wgrad_subs = subs;
    if (accumulate) return dispatch_launch<kWgradAcc>(tm, a, stream, grid_ctas);   // adds into the existing gradients
    // Wide tiles (shared-operand accumulator pairs) are opt-in (GemmArgs.debug
    // bit 8 = 256, CTA pairs, F % 512 == 0): bit-identical and 25% less operand
    // traffic, but measured inside the layer step WGRAD takes 2.36-2.41 ms vs
    // 2.27-2.32 ms with the double-buffered one-accumulator tiles (standalone:
    // 2.10 ms both; 1.77 vs 1.82 ms without the weight-gradient stores).
    if (g_cta_group == 2 && F % 512 == 0 && (g_debug & 256) && subs == 7) return launch<kWgradW, 2>(tm, a, stream);
    return dispatch_launch<kWgrad>(tm, a, stream, grid_ctas);
}

// ------------------------------------------------------------------ dense
// Plain GEMMs of the transformer step around the MoE layer (qkv / wo / lm-head
// projections, reference model.py:135-169 through tensor.py:192-207 matmul),
// on the same kernel template with one segment: weights in the reference
// [in, out] layout, w [K, N] row-major.
//   fwd    y[M,N]  = x[M,K] . w          BWD1 mainloop, one pair (A K-major, B MN-major)
//   dgrad  dx[M,K] = dy[M,N] . w^T       FWD2 mainloop (B = w rows, K-major)
//   wgrad  dw[K,N] = x^T . dy            WGRAD, dW1 sub-problem only (A, B MN-major)
// seg_* : device segment table of one segment {base 0, count M, expert 0}.
static int check_dense(int M, int K, int N) {
    B200_CHECK_ARG(M >= 1 && K % 256 == 0 && N % 256 == 0 && K > 0 && N > 0, B200MOE_ERR_SHAPE,
                   "dense GEMM needs K and N multiples of 256 (M=%d K=%d N=%d)", M, K, N);
    return B200MOE_OK;
}

int b200moe_dense_fwd(const void* x, const void* w, const int* seg_base, const int* seg_count, const int* seg_expert,
                      int M, int K, int N, int ldx, int ldw, int ldy, void* y, int grid_ctas, cudaStream_t stream) {
    B200_TRY(check_dense(M, K, N));
    TmaSet tm = {};
    B200_TRY(make_map(&tm.m[0], x, K, M, ldx, false));
    B200_TRY(make_map(&tm.m[2], w, N, K, ldw, true));
    tm.m[1] = tm.m[0];
    tm.m[3] = tm.m[2];
    tm.m[4] = tm.m[0];
    B200_TRY(make_map(&tm.st[0], y, N, M, ldy, false, true));
    tm.st[1] = tm.st[2] = tm.st[0];
    GemmArgs a = {seg_base, seg_count, seg_expert, 1, N, K, 1, (__nv_bfloat16*)y, nullptr, nullptr, nullptr, nullptr};
    a.dense = 1;
    return dispatch_launch<kBwd1>(tm, a, stream, grid_ctas);
}

int b200moe_dense_dgrad(const void* dy, const void* w, const int* seg_base, const int* seg_count,
                        const int* seg_expert, int M, int K, int N, int lddy, int ldw, int lddx, void* dx,
                        int grid_ctas, cudaStream_t stream) {
    B200_TRY(check_dense(M, K, N));
    TmaSet tm = {};
    B200_TRY(make_map(&tm.m[0], dy, N, M, lddy, false));
    B200_TRY(make_map(&tm.m[1], w, N, K, ldw, false));
    tm.m[2] = tm.m[3] = tm.m[4] = tm.m[0];
    B200_TRY(make_map(&tm.st[0], dx, K, M, lddx, false, true));
    tm.st[1] = tm.st[2] = tm.st[0];
    GemmArgs a = {seg_base, seg_count, seg_expert, 1, K, N, 1, (__nv_bfloat16*)dx, nullptr, nullptr, nullptr,
                  nullptr};
    return dispatch_launch<kFwd2>(tm, a, stream, grid_ctas);
}

int b200moe_dense_wgrad(const void* x, const void* dy, const int* seg_base, const int* seg_count,
                        const int* seg_expert, int M, int K, int N, int ldx, int lddy, int lddw, void* dw,
                        int grid_ctas, cudaStream_t stream) {
    B200_TRY(check_dense(M, K, N));
    B200_CHECK_ARG(lddw == N, B200MOE_ERR_SHAPE, "dense wgrad writes a contiguous [K, N] gradient (ld %d != N %d)",
                   lddw, N);
    TmaSet tm = {};
    B200_TRY(make_map(&tm.m[2], x, K, M, ldx, true));      // "da": output rows = K
    B200_TRY(make_map(&tm.m[3], dy, N, M, lddy, true));    // "xp": output columns = N
    tm.m[0] = tm.m[1] = tm.m[4] = tm.m[2];
    B200_TRY(make_map(&tm.st[0], dw, N, K, lddw, false, true));
    tm.st[1] = tm.st[2] = tm.st[0];
    GemmArgs a = {seg_base, seg_count, seg_expert, 1, N, K, 1, (__nv_bfloat16*)dw, nullptr, nullptr, nullptr,
                  nullptr};
    a.wgrad_subs = 1;
    a.wgrad_mfast = (N / 256) > (K / 256);   // e.g. the lm-head: 16 row tiles x 501 column tiles, K = tokens
    return dispatch_launch<kWgrad>(tm, a, stream, grid_ctas);
}

}  // extern "C"
