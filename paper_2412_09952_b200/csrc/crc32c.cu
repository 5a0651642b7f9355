// CRC32C (Castagnoli) of device buffers, for the reference checkpoint format
// (moefold/checkpoint.py:40-78: crc32c of every tensor payload, check value
// crc32c("123456789") = 0xE3069283).  SURVEY 8(f) row 3.
//
// A CRC without init/xorout ("raw") is linear over GF(2):
//   raw(A || B) = shift(raw(A), |B|) ^ raw(B)
// where shift(c, L) runs the register over L zero bytes (a 32x32 bit matrix).
// Leading zero bytes leave a raw CRC of 0 unchanged, so the buffer is treated
// as front-padded with zeros to a whole number of equal per-warp ranges, and
// the standard init 0xFFFFFFFF is folded in by inverting the first 4 bytes.
//
//   crc_warp_kernel  each warp owns a contiguous range and walks it in 4 KB
//                    steps of four 1 KB rows (the next step's loads in flight
//                    while the current one is hashed); lane j takes bytes
//                    [32j, 32j+32) of each row (two 16-byte loads; the warp's
//                    loads cover each row completely).  A lane's four 32-byte
//                    pieces are independent slicing-by-4 chains (tables
//                    replicated 32x in shared memory: replica `lane` lives in
//                    bank `lane`, so the data-dependent lookups never conflict);
//                    the lane folds them and its running value with
//                    table-driven shifts (A = shift(A, 4 KB) ^ XOR_q
//                    shift(p_q, (3-q) rows)), the warp folds its lanes with
//                    shift((31-j)*32), shifts the range CRC into place with the
//                    binary decomposition of its distance to the end, and
//                    atomicXor folds the warps (XOR commutes: the result is
//                    deterministic).
//   crc_finish       one thread runs the (<16 byte) tail and the final xor.
// HBM-bound by design: every byte is read once, in 8 KB coalesced runs.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "common.cuh"

namespace b200moe {

constexpr uint32_t kPoly = 0x82F63B78u;   // reflected Castagnoli polynomial
constexpr int kCrcThreads = 512;
constexpr int kCrcWarps = kCrcThreads / 32;
constexpr int kReps = 32;                 // table replicas (one per bank)
constexpr int kPiece = 32;                // bytes per lane per row (two 16-byte loads; the warp reads 1 KB rows)
constexpr int kVec = kPiece / 16;
constexpr int kRow = 32 * kPiece;         // 1 KB per warp row
constexpr int kChains = 4;                // rows per step: independent chains (ILP)
constexpr int kStep = kChains * kRow;     // 4 KB per warp step
// 32-byte pieces halve the step-fold shift-table lookups per byte (those tables
// are not bank-replicated, so their data-dependent reads conflict): 16-byte
// pieces x 8 chains measured 2.96 TB/s.
// T[4][256][kReps] | S[kChains][4][256] (shift by kStep, then kChains-1 .. 1 rows) | L[32][33] | P[40][32]
constexpr size_t kCrcSmem = (size_t)((4 * 256 * kReps + kChains * 4 * 256 + 32 * 33 + 40 * 32 + 3) / 4 * 4) * 4;

__host__ __device__ inline uint32_t mat_apply(const uint32_t* m, uint32_t c, int stride = 1) {
    uint32_t r = 0;
    for (int j = 0; j < 32; ++j) r ^= m[j * stride] & (0u - ((c >> j) & 1u));
    return r;
}

__device__ __forceinline__ uint32_t crc_word(const uint32_t* __restrict__ T, uint32_t c, uint32_t w, int lane) {
    c ^= w;
    return T[(3 * 256 + (c & 0xFF)) * kReps + lane] ^ T[(2 * 256 + ((c >> 8) & 0xFF)) * kReps + lane] ^
           T[(1 * 256 + ((c >> 16) & 0xFF)) * kReps + lane] ^ T[(0 * 256 + (c >> 24)) * kReps + lane];
}

// Fixed tables, built once into the caller's workspace by crc_init_kernel:
// slicing tables replicated per bank, the step / row shift tables and the
// lane-fold matrices (row stride 33: conflict-free), laid out exactly as the
// kernel's shared memory so each block copies them with 16-byte loads.
constexpr int kPowBits = 40;           // P[b] = shift by kStep << b bytes
constexpr int kTabWords = 4 * 256 * kReps + kChains * 4 * 256 + 32 * 33 + kPowBits * 32;
constexpr int kTabWordsPadded = (kTabWords + 3) / 4 * 4;
constexpr long long kWsTables = 256;   // byte offset of the tables in the workspace (after the accumulator)

struct FixedMats {
    uint32_t step[kChains][32];      // shift by kStep, then by kChains-1 .. 1 rows
    uint32_t lane[32 * 32];          // lane[j] = shift by (31 - j) * kPiece bytes
    uint32_t pow[kPowBits][32];      // pow[b] = shift by kStep << b bytes
};

__global__ void crc_init_kernel(const __grid_constant__ FixedMats mats, uint32_t* __restrict__ tab) {
    uint32_t* T = tab;
    uint32_t* S = T + 4 * 256 * kReps;
    uint32_t* L = S + kChains * 4 * 256;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 256; i += gridDim.x * blockDim.x) {
        uint32_t t[4];
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
        t[0] = c;
        for (int k = 1; k < 4; ++k) {
            uint32_t q = t[k - 1] & 0xFF;
            for (int b = 0; b < 8; ++b) q = (q & 1) ? (q >> 1) ^ kPoly : q >> 1;
            t[k] = q ^ (t[k - 1] >> 8);
        }
        for (int k = 0; k < 4; ++k) {
            for (int r = 0; r < kReps; ++r) T[(k * 256 + i) * kReps + r] = t[k];
            for (int sh = 0; sh < kChains; ++sh)
                S[(sh * 4 + k) * 256 + i] = mat_apply(mats.step[sh], (uint32_t)i << (8 * k));
        }
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 32 * 32; i += gridDim.x * blockDim.x)
        L[(i / 32) * 33 + i % 32] = mats.lane[i];
    uint32_t* P = L + 32 * 33;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kPowBits * 32; i += gridDim.x * blockDim.x)
        P[i] = mats.pow[i / 32][i % 32];
}

__global__ void __launch_bounds__(kCrcThreads) crc_warp_kernel(const uint8_t* __restrict__ data, long long pad,
                                                               long long range_bytes, long long nranges,
                                                               const uint4* __restrict__ tab,
                                                               uint32_t* __restrict__ acc) {
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* T = sm;                               // slicing tables, replicated
    uint32_t* S = T + 4 * 256 * kReps;              // shift tables: S[s][k][b] = step[s](b << 8k)
    uint32_t* L = S + kChains * 4 * 256;            // lane fold matrices, row stride 33 (conflict-free)
    uint32_t* P = L + 32 * 33;                      // P[b] = shift by kStep << b
    for (int i = threadIdx.x; i < kTabWordsPadded / 4; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = tab[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long gw = (long long)blockIdx.x * kCrcWarps + (threadIdx.x >> 5);
    const long long nw = (long long)gridDim.x * kCrcWarps;
    for (long long r = gw; r < nranges; r += nw) {
        uint32_t A = 0;
        const long long base = r * range_bytes + (long long)lane * kPiece;   // logical offset of row 0, step 0
        auto ld = [&](long long lo) -> uint4 {
            if (lo < pad) return make_uint4(0, 0, 0, 0);
            uint4 v = __ldg(reinterpret_cast<const uint4*>(data + (lo - pad)));
            if (lo == pad) v.x ^= 0xFFFFFFFFu;
            return v;
        };
        uint4 v[kChains][kVec];    // chain q = this lane's kPiece bytes of row q of the step
#pragma unroll
        for (int q = 0; q < kChains; ++q)
#pragma unroll
            for (int u = 0; u < kVec; ++u) v[q][u] = ld(base + (long long)q * kRow + 16 * u);
        for (long long st = 0; st < range_bytes; st += kStep) {
            uint4 nx[kChains][kVec];   // next step, in flight while this one is hashed
            const bool more = st + kStep < range_bytes;
#pragma unroll
            for (int q = 0; q < kChains; ++q)
#pragma unroll
                for (int u = 0; u < kVec; ++u)
                    nx[q][u] = more ? ld(base + st + kStep + (long long)q * kRow + 16 * u) : make_uint4(0, 0, 0, 0);
            uint32_t c[kChains];
#pragma unroll
            for (int q = 0; q < kChains; ++q) c[q] = crc_word(T, 0u, v[q][0].x, lane);
#pragma unroll
            for (int u = 0; u < kVec; ++u) {
                if (u > 0) {
#pragma unroll
                    for (int q = 0; q < kChains; ++q) c[q] = crc_word(T, c[q], v[q][u].x, lane);
                }
#pragma unroll
                for (int q = 0; q < kChains; ++q) c[q] = crc_word(T, c[q], v[q][u].y, lane);
#pragma unroll
                for (int q = 0; q < kChains; ++q) c[q] = crc_word(T, c[q], v[q][u].z, lane);
#pragma unroll
                for (int q = 0; q < kChains; ++q) c[q] = crc_word(T, c[q], v[q][u].w, lane);
            }
            // step = XOR_q shift(c_q, kChains-1-q rows);  A = shift(A, kStep) ^ step
            uint32_t x = c[kChains - 1];
#pragma unroll
            for (int q = 0; q < kChains - 1; ++q) {
                const uint32_t* Sq = S + (q + 1) * 1024;
                x ^= Sq[c[q] & 0xFF] ^ Sq[256 + ((c[q] >> 8) & 0xFF)] ^ Sq[512 + ((c[q] >> 16) & 0xFF)] ^
                     Sq[768 + (c[q] >> 24)];
            }
            A = S[A & 0xFF] ^ S[256 + ((A >> 8) & 0xFF)] ^ S[512 + ((A >> 16) & 0xFF)] ^ S[768 + (A >> 24)] ^ x;
#pragma unroll
            for (int q = 0; q < kChains; ++q)
#pragma unroll
                for (int u = 0; u < kVec; ++u) v[q][u] = nx[q][u];
        }
        uint32_t w = mat_apply(L + lane * 33, A);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w ^= __shfl_xor_sync(0xffffffffu, w, o);
        if (lane == 0) {
            // distance to the end in kStep units, applied bit by bit
            const unsigned long long d = (unsigned long long)(nranges - 1 - r) * (unsigned long long)(range_bytes / kStep);
            for (int b = 0; b < kPowBits && (d >> b); ++b)
                if ((d >> b) & 1ull) w = mat_apply(P + b * 32, w);
            if (w != 0) atomicXor(acc, w);
        }
    }
}

__global__ void crc_finish_kernel(uint32_t* __restrict__ acc, const uint8_t* __restrict__ tail, int tail_len,
                                  int have_body, uint32_t* __restrict__ out) {
    __shared__ uint32_t T0[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
        T0[i] = c;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    uint32_t c = have_body ? acc[0] : 0xFFFFFFFFu;
    acc[0] = 0;   // ready for the next (stream-ordered) call on this workspace
    for (int i = 0; i < tail_len; ++i) c = T0[(c ^ tail[i]) & 0xFF] ^ (c >> 8);
    out[0] = c ^ 0xFFFFFFFFu;
}

// ---- host: shift matrices -------------------------------------------------
static void mat_mul(const uint32_t* a, const uint32_t* b, uint32_t* r) {   // r = a * b (apply b, then a)
    uint32_t t[32];
    for (int j = 0; j < 32; ++j) t[j] = mat_apply(a, b[j]);
    memcpy(r, t, sizeof(t));
}

// m = shift by `bytes` zero bytes
static void mat_shift(long long bytes, uint32_t* m) {
    uint32_t base[32];
    for (int j = 0; j < 32; ++j) {   // one zero byte
        uint32_t c = 1u << j;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
        base[j] = c;
        m[j] = 1u << j;
    }
    while (bytes > 0) {
        if (bytes & 1) mat_mul(base, m, m);
        mat_mul(base, base, base);
        bytes >>= 1;
    }
}

}  // namespace b200moe

using namespace b200moe;

extern "C" {

// workspace: [0, 4) the XOR accumulator, [256, ...) the fixed tables
long long b200moe_crc32c_workspace_bytes(void) { return kWsTables + (long long)kTabWordsPadded * 4; }

int b200moe_crc32c_init(void* workspace, cudaStream_t stream) {
    FixedMats f;
    uint32_t piece[32];
    mat_shift(kStep, f.step[0]);
    for (int q = 0; q < kChains - 1; ++q) mat_shift((long long)kRow * (kChains - 1 - q), f.step[q + 1]);
    mat_shift(kPiece, piece);
    mat_shift(0, f.lane + 31 * 32);
    for (int j = 30; j >= 0; --j) mat_mul(piece, f.lane + (j + 1) * 32, f.lane + j * 32);
    memcpy(f.pow[0], f.step[0], sizeof(f.pow[0]));
    for (int b = 1; b < kPowBits; ++b) mat_mul(f.pow[b - 1], f.pow[b - 1], f.pow[b]);
    cudaMemsetAsync(workspace, 0, 4, stream);
    crc_init_kernel<<<8, 256, 0, stream>>>(f, (uint32_t*)((char*)workspace + kWsTables));
    B200_CHECK_LAUNCH("crc32c_init");
    return B200MOE_OK;
}

int b200moe_crc32c(const void* data, long long nbytes, unsigned int* out, void* workspace, cudaStream_t stream) {
    B200_CHECK_ARG(nbytes >= 0, B200MOE_ERR_SHAPE, "crc32c: negative length");
    B200_CHECK_ARG(nbytes == 0 || ((uintptr_t)data & 15) == 0, B200MOE_ERR_CONFIG,
                   "crc32c: buffer must be 16-byte aligned");
    static std::atomic<uint64_t> attr{0};
    if (cudaError_t ae = ensure_smem_attr(crc_warp_kernel, (int)kCrcSmem, attr); ae != cudaSuccess) {
        set_error("crc32c smem attribute: %s", cudaGetErrorString(ae));
        return B200MOE_ERR_CUDA;
    }
    const long long body = nbytes & ~15LL;
    const int tail_len = (int)(nbytes - body);
    uint32_t* acc = (uint32_t*)workspace;
    if (body > 0) {
        // one range per warp of a full-chip grid, whole kStep steps
        const long long warps = (long long)kNumSMs * kCrcWarps;
        const long long steps = (body + kStep - 1) / kStep;
        const long long range = (steps + warps - 1) / warps * kStep;
        const long long nranges = (body + range - 1) / range;
        const long long blocks = (nranges + kCrcWarps - 1) / kCrcWarps;
        crc_warp_kernel<<<(int)(blocks < kNumSMs ? blocks : kNumSMs), kCrcThreads, kCrcSmem, stream>>>(
            (const uint8_t*)data, nranges * range - body, range, nranges,
            (const uint4*)((const char*)workspace + kWsTables), acc);
    }
    crc_finish_kernel<<<1, 256, 0, stream>>>(acc, (const uint8_t*)data + body, tail_len, body > 0 ? 1 : 0, out);
    B200_CHECK_LAUNCH("crc32c");
    return B200MOE_OK;
}

}  // extern "C"
