// NVLink peer-memory probe (one process, 2 GPUs): what an SM kernel can move
// to / from a peer GPU's memory, with both GPUs doing it at the same time (the
// expert-parallel exchange pattern at EP2: each link direction carries one
// GPU's stores plus the other GPU's load responses).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/p2p_probe.cu -o /tmp/p2p_probe
//   /tmp/p2p_probe            -> one line per variant: GB/s per direction
//
// Variants (each moves `bytes` per GPU, rows of 8 KB = one bf16 token row at H=4096):
//   ce       cudaMemcpyPeerAsync (copy engines)
//   st16     warp per row, 16-byte loads local, 16-byte stores to the peer
//   ld16     warp per row, 16-byte loads from the peer, stores local
//   ld16x2   ld16 with two rows in flight per warp
//   bulk_st  CTA: cp.async.bulk global->smem (local), smem->global (peer)
//   bulk_ld  CTA: cp.async.bulk global (peer)->smem, smem->global (local)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int kRowBytes = 8192;

__global__ void copy_rows(const uint4* __restrict__ src, uint4* __restrict__ dst, int rows) {
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    constexpr int V = kRowBytes / 16;   // 512 uint4 per row
    for (int r = w; r < rows; r += nw) {
        const uint4* s = src + (size_t)r * V;
        uint4* d = dst + (size_t)r * V;
        uint4 v[V / 32];
#pragma unroll
        for (int i = 0; i < V / 32; ++i) v[i] = s[i * 32 + lane];
#pragma unroll
        for (int i = 0; i < V / 32; ++i) d[i * 32 + lane] = v[i];
    }
}

__global__ void copy_rows2(const uint4* __restrict__ src, uint4* __restrict__ dst, int rows) {
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    constexpr int V = kRowBytes / 16;
    for (int r = 2 * w; r < rows; r += 2 * nw) {
        const bool two = r + 1 < rows;
        uint4 v[V / 32], u[V / 32];
#pragma unroll
        for (int i = 0; i < V / 32; ++i) {
            v[i] = src[(size_t)r * V + i * 32 + lane];
            if (two) u[i] = src[(size_t)(r + 1) * V + i * 32 + lane];
        }
#pragma unroll
        for (int i = 0; i < V / 32; ++i) {
            dst[(size_t)r * V + i * 32 + lane] = v[i];
            if (two) dst[(size_t)(r + 1) * V + i * 32 + lane] = u[i];
        }
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// One CTA streams rows through a ring of kSlots smem buffers: bulk load (with
// an mbarrier per slot), then bulk store; a slot is reused after its store has
// read it.  One elected thread drives everything.
template <int kSlots>
__global__ void bulk_rows(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int rows) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[kSlots];
    if (threadIdx.x != 0) return;
    for (int i = 0; i < kSlots; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint32_t phase = 0;
    int issued = 0;
    const int first = blockIdx.x, step = gridDim.x;
    // prologue: fill the ring
    int r_load = first;
    for (int s = 0; s < kSlots && r_load < rows; ++s, r_load += step, ++issued) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[s])), "r"(kRowBytes));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(smem_u32(sm + s * kRowBytes)), "l"(src + (size_t)r_load * kRowBytes), "r"(kRowBytes),
                        "r"(smem_u32(&bar[s])) : "memory");
    }
    int slot = 0;
    for (int r = first; r < rows; r += step) {
        // wait for the load of this slot
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                     :: "r"(smem_u32(&bar[slot])), "r"((phase >> slot) & 1u) : "memory");
        phase ^= 1u << slot;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     :: "l"(dst + (size_t)r * kRowBytes), "r"(smem_u32(sm + slot * kRowBytes)), "r"(kRowBytes) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (r_load < rows) {
            // reuse the oldest slot once its store has read it: allow kSlots-1 pending
            asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(0) : "memory");
            const int s = slot;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[s])), "r"(kRowBytes));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         :: "r"(smem_u32(sm + s * kRowBytes)), "l"(src + (size_t)r_load * kRowBytes), "r"(kRowBytes),
                            "r"(smem_u32(&bar[s])) : "memory");
            r_load += step;
        }
        slot = (slot + 1 == kSlots) ? 0 : slot + 1;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    (void)issued;
}

struct Side {
    uint8_t* local;   // this GPU's source / destination
    uint8_t* peer;    // buffer on the other GPU
    cudaStream_t s;
    cudaEvent_t e0, e1;
};

int main() {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (n < 2) { printf("need 2 GPUs\n"); return 0; }
    const size_t bytes = (size_t)256 << 20;
    const int rows = (int)(bytes / kRowBytes);
    Side sd[2];
    uint8_t *bufA[2], *bufB[2];
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceEnablePeerAccess(1 - d, 0));
        CK(cudaMalloc(&bufA[d], bytes));
        CK(cudaMalloc(&bufB[d], bytes));
        CK(cudaMemset(bufA[d], d + 1, bytes));
        CK(cudaStreamCreateWithFlags(&sd[d].s, cudaStreamNonBlocking));
        CK(cudaEventCreate(&sd[d].e0));
        CK(cudaEventCreate(&sd[d].e1));
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
        CK(cudaFuncSetAttribute(bulk_rows<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kRowBytes));
        CK(cudaFuncSetAttribute(bulk_rows<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * kRowBytes));
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char* names[] = {"ce", "st16", "ld16", "ld16x2", "bulk_st4", "bulk_st8", "bulk_ld4", "bulk_ld8"};
    for (int bidir = 1; bidir >= 0; --bidir)
    for (int v = 0; v < 8; ++v) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
            const int nd = bidir ? 2 : 1;
            for (int d = 0; d < nd; ++d) {
                CK(cudaSetDevice(d));
                const int p = 1 - d;
                cudaStream_t s = sd[d].s;
                CK(cudaEventRecord(sd[d].e0, s));
                const bool store_side = (v == 1 || v == 4 || v == 5);
                // store variants: local A -> peer B; load variants: peer A -> local B
                const uint8_t* src = store_side ? bufA[d] : bufA[p];
                uint8_t* dst = store_side ? bufB[p] : bufB[d];
                switch (v) {
                    case 0: CK(cudaMemcpyPeerAsync(bufB[p], p, bufA[d], d, bytes, s)); break;
                    case 1: case 2: copy_rows<<<sms * 4, 256, 0, s>>>((const uint4*)src, (uint4*)dst, rows); break;
                    case 3: copy_rows2<<<sms * 2, 256, 0, s>>>((const uint4*)src, (uint4*)dst, rows); break;
                    case 4: case 6: bulk_rows<4><<<sms * 6, 32, 4 * kRowBytes, s>>>(src, dst, rows); break;
                    case 5: case 7: bulk_rows<8><<<sms * 3, 32, 8 * kRowBytes, s>>>(src, dst, rows); break;
                }
                CK(cudaGetLastError());
                CK(cudaEventRecord(sd[d].e1, s));
            }
            float worst = 0.f;
            for (int d = 0; d < nd; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaEventSynchronize(sd[d].e1));
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, sd[d].e0, sd[d].e1));
                worst = ms > worst ? ms : worst;
            }
            if (rep > 0 && worst < best) best = worst;
        }
        printf("{\"variant\": \"%s\", \"bidirectional\": %s, \"MiB\": %zu, \"ms\": %.4f, \"GBps_per_direction\": %.1f}\n",
               names[v], bidir ? "true" : "false", bytes >> 20, best, bytes / (best * 1e-3) / 1e9);
    }
    return 0;
}
