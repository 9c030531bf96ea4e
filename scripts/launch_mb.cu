// launch_mb.cu -- fixed cost of a persistent 148-CTA launch: dynamic smem size,
// TMEM alloc/dealloc, cluster size (event-timed, 200 back-to-back launches).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <bool TMEM>
__global__ void __launch_bounds__(352, 1) k(int* out) {
    extern __shared__ uint8_t sm[];
    __shared__ uint32_t tb;
    if (TMEM && (threadIdx.x >> 5) == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if (threadIdx.x == 0) sm[0] = 1;
    __syncthreads();
    if (TMEM && (threadIdx.x >> 5) == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
    if (threadIdx.x == 0 && sm[0] == 7) out[0] = 1;
}
template <class K>
void run(const char* name, K kern, size_t smem) {
    int* d; cudaMalloc(&d, 4);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int i = 0; i < 10; ++i) kern<<<148, 352, smem>>>(d);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < 200; ++i) kern<<<148, 352, smem>>>(d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s smem %6zu: %.2f us/launch (%s)\n", name, smem, ms * 1e3 / 200, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    run("plain", k<false>, 1024);
    run("plain", k<false>, 166 * 1024);
    run("tmem alloc 512", k<true>, 1024);
    run("tmem alloc 512", k<true>, 166 * 1024);
    return 0;
}
