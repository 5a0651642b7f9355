// CRC32C (Castagnoli) of device buffers, for the reference checkpoint format
// (moefold/checkpoint.py:40-78: crc32c of every tensor payload, check value
// crc32c("123456789") = 0xE3069283).  SURVEY 8(f) row 3.
//
// A CRC without init/xorout ("raw") is linear over GF(2), and
// raw(A || B) = shift(raw(A), |B|) ^ raw(B), where shift(c, L) runs the
// register over L zero bytes -- a fixed 32x32 bit matrix per L.  Leading zero
// bytes leave a raw CRC of 0 unchanged, so the buffer is treated as if
// front-padded with zeros to a whole number of equal blocks, and the standard
// init 0xFFFFFFFF is folded in by inverting the first 4 data bytes.
//
//   crc_blocks  grid of blocks, each owning a contiguous run of 16 KB tiles.
//               A tile is loaded coalesced into shared memory (segment stride
//               17 words: conflict-free), each of the 256 threads computes the
//               raw CRC of its 64-byte segment (slicing-by-4 tables in shared
//               memory), a 8-level tree of shift matrices folds the 256
//               segment CRCs into the tile CRC, and the block folds its tiles.
//   crc_finish  one thread folds the block CRCs, runs the (<16 byte) tail
//               byte-wise and applies the final xor.
// HBM-bound: every byte is read once.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "common.cuh"

namespace b200moe {

constexpr uint32_t kPoly = 0x82F63B78u;   // reflected Castagnoli polynomial
constexpr int kCrcThreads = 256;
constexpr int kSegBytes = 64;
constexpr int kTileBytes = kCrcThreads * kSegBytes;   // 16 KB
constexpr int kSegWords = kSegBytes / 4;
constexpr int kSegStride = kSegWords + 1;             // 17 words: conflict-free
constexpr int kMaxCrcBlocks = kNumSMs * 8;
constexpr int kLevels = 8;                            // log2(kCrcThreads)

// Shift matrices: lvl[l] = shift by kSegBytes << l bytes, tile = shift by
// kTileBytes, block = shift by one block's bytes.  Column j = image of bit j.
struct CrcMats {
    uint32_t lvl[kLevels][32];
    uint32_t tile[32];
    uint32_t block[32];
};

__host__ __device__ inline uint32_t mat_apply(const uint32_t* m, uint32_t c) {
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) r ^= m[j] & (0u - ((c >> j) & 1u));
    return r;
}

__device__ __forceinline__ void build_tables(uint32_t (*T)[256]) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
        T[0][i] = c;
    }
    __syncthreads();
    for (int t = 1; t < 4; ++t) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) T[t][i] = T[0][T[t - 1][i] & 0xFF] ^ (T[t - 1][i] >> 8);
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kCrcThreads) crc_blocks_kernel(const uint8_t* __restrict__ data, long long body,
                                                                 long long pad, int tiles_per_block,
                                                                 const CrcMats mats, uint32_t* __restrict__ out) {
    __shared__ uint32_t T[4][256];
    __shared__ uint32_t seg[kCrcThreads * kSegStride];
    __shared__ uint32_t part[kCrcThreads];
    __shared__ uint32_t M[kLevels][32];
    build_tables(T);
    for (int i = threadIdx.x; i < kLevels * 32; i += blockDim.x) M[i / 32][i % 32] = mats.lvl[i / 32][i % 32];
    uint32_t acc = 0;
    const long long blk0 = (long long)blockIdx.x * tiles_per_block * kTileBytes;   // logical (padded) offset
    for (int tile = 0; tile < tiles_per_block; ++tile) {
        const long long t0 = blk0 + (long long)tile * kTileBytes;
        // coalesced load of the tile; logical bytes before `pad` are zeros
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int q = threadIdx.x + k * kCrcThreads;   // uint4 index inside the tile
            const long long lo = t0 + 16LL * q;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (lo >= pad) {
                v = *reinterpret_cast<const uint4*>(data + (lo - pad));
                if (lo == pad) v.x ^= 0xFFFFFFFFu;         // init 0xFFFFFFFF == invert the first 4 bytes
            }
            const int s = q >> 2, w = (q & 3) * 4;
            uint32_t* dst = seg + s * kSegStride + w;
            dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w;
        }
        __syncthreads();
        // raw CRC of this thread's 64-byte segment
        uint32_t c = 0;
        const uint32_t* src = seg + threadIdx.x * kSegStride;
#pragma unroll
        for (int j = 0; j < kSegWords; ++j) {
            c ^= src[j];
            c = T[3][c & 0xFF] ^ T[2][(c >> 8) & 0xFF] ^ T[1][(c >> 16) & 0xFF] ^ T[0][c >> 24];
        }
        // tree fold: left partner is shifted past the right one's bytes
        part[threadIdx.x] = c;
#pragma unroll
        for (int l = 0; l < kLevels; ++l) {
            __syncthreads();
            const int stride = 1 << l;
            uint32_t nv = 0;
            const bool active = (threadIdx.x & ((stride << 1) - 1)) == 0;
            if (active) nv = mat_apply(M[l], part[threadIdx.x]) ^ part[threadIdx.x + stride];
            __syncthreads();
            if (active) part[threadIdx.x] = nv;
        }
        if (threadIdx.x == 0) acc = mat_apply(mats.tile, acc) ^ part[0];
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

__global__ void crc_finish_kernel(const uint32_t* __restrict__ blk, int nblocks, const CrcMats mats,
                                  const uint8_t* __restrict__ tail, int tail_len, int have_body,
                                  uint32_t* __restrict__ out) {
    __shared__ uint32_t T0[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
        T0[i] = c;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    uint32_t c = 0xFFFFFFFFu;
    if (have_body) {
        c = 0;
        for (int b = 0; b < nblocks; ++b) c = mat_apply(mats.block, c) ^ blk[b];
    }
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
    uint32_t base[32], id[32];
    for (int j = 0; j < 32; ++j) {   // one zero byte
        uint32_t c = 1u << j;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
        base[j] = c;
        id[j] = 1u << j;
    }
    memcpy(m, id, sizeof(id));
    while (bytes > 0) {
        if (bytes & 1) mat_mul(base, m, m);
        mat_mul(base, base, base);
        bytes >>= 1;
    }
}

}  // namespace b200moe

using namespace b200moe;

extern "C" {

long long b200moe_crc32c_workspace_bytes(void) { return (long long)kMaxCrcBlocks * 4; }

int b200moe_crc32c(const void* data, long long nbytes, unsigned int* out, void* workspace, cudaStream_t stream) {
    B200_CHECK_ARG(nbytes >= 0, B200MOE_ERR_SHAPE, "crc32c: negative length");
    B200_CHECK_ARG(nbytes == 0 || ((uintptr_t)data & 15) == 0, B200MOE_ERR_CONFIG,
                   "crc32c: buffer must be 16-byte aligned");
    const long long body = nbytes & ~15LL;
    const int tail_len = (int)(nbytes - body);
    const long long tiles = (body + kTileBytes - 1) / kTileBytes;
    int tpb = 1, nblocks = 0;
    if (tiles > 0) {
        tpb = (int)((tiles + kMaxCrcBlocks - 1) / kMaxCrcBlocks);
        nblocks = (int)((tiles + tpb - 1) / tpb);
    }
    const long long padded = (long long)nblocks * tpb * kTileBytes;
    CrcMats mats;   // a few microseconds of host GF(2) algebra per call
    for (int l = 0; l < kLevels; ++l) mat_shift((long long)kSegBytes << l, mats.lvl[l]);
    mat_shift(kTileBytes, mats.tile);
    mat_shift((long long)tpb * kTileBytes, mats.block);
    if (nblocks > 0)
        crc_blocks_kernel<<<nblocks, kCrcThreads, 0, stream>>>((const uint8_t*)data, body, padded - body, tpb, mats,
                                                               (uint32_t*)workspace);
    crc_finish_kernel<<<1, 256, 0, stream>>>((const uint32_t*)workspace, nblocks, mats,
                                             (const uint8_t*)data + body, tail_len, body > 0 ? 1 : 0, out);
    B200_CHECK_LAUNCH("crc32c");
    return B200MOE_OK;
}

}  // extern "C"
