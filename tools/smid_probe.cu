// Records %smid of every CTA of a 148-CTA cluster-of-2 launch (placement probe).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(2, 1, 1) probe(int* out) {
    unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
}
int main() {
    int* d; cudaMalloc(&d, 148 * sizeof(int));
    probe<<<148, 32>>>(d);
    int h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int i = 0; i < 148; ++i) printf("%d%c", h[i], i % 16 == 15 ? '\n' : ' ');
    printf("\n");
    return 0;
}
