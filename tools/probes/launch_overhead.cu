// Launch-overhead probe: per-launch time of empty kernels with the qgemm
// launch configuration (148 CTAs x 512 threads), adding 200 KB dynamic smem,
// TMEM alloc/dealloc (512 cols), and a __grid_constant__ 128-B parameter.
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

struct Big { unsigned long long v[16]; };

__global__ void __launch_bounds__(512, 1) k_empty(int* p) { if (p && threadIdx.x == 9999) *p = 1; }
__global__ void __launch_bounds__(512, 1) k_smem(int* p) {
    extern __shared__ int s[];
    if (threadIdx.x == 0) s[0] = 1;
    __syncthreads();
    if (p && s[0] == 7) *p = 1;
}
__global__ void __launch_bounds__(512, 1) k_tmem(int* p) {
    extern __shared__ unsigned int s2[];
    if ((threadIdx.x >> 5) == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((unsigned)__cvta_generic_to_shared(s2)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    unsigned t = s2[0];
    __syncthreads();
    if ((threadIdx.x >> 5) == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
    if (p && t == 12345) *p = 1;
}
__global__ void __launch_bounds__(512, 1) k_param(const __grid_constant__ Big b, int* p) {
    extern __shared__ int s[];
    if (threadIdx.x == 0) s[0] = (int)b.v[3];
    __syncthreads();
    if (p && s[0] == 77) *p = 1;
}

template <class F>
float timeit(F launch, int n) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 5; ++i) launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < n; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms * 1000.f / n;
}

int main() {
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_param, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    Big b{};
    printf("empty 148x512, no smem      : %.2f us\n", timeit([&] { k_empty<<<148, 512>>>(nullptr); }, 200));
    printf("148x512 + 200KB dyn smem     : %.2f us\n", timeit([&] { k_smem<<<148, 512, smem>>>(nullptr); }, 200));
    printf("148x512 + 200KB + TMEM 512   : %.2f us\n", timeit([&] { k_tmem<<<148, 512, smem>>>(nullptr); }, 200));
    printf("148x512 + 200KB + 128B param : %.2f us\n", timeit([&] { k_param<<<148, 512, smem>>>(b, nullptr); }, 200));
    printf("148x512 + 1KB dyn smem       : %.2f us\n", timeit([&] { k_smem<<<148, 512, 1024>>>(nullptr); }, 200));
    printf("alternating 200KB / 1KB smem : %.2f us (pair)\n", timeit([&] { k_smem<<<148, 512, smem>>>(nullptr); k_empty<<<148, 128>>>(nullptr); }, 200));
    cudaError_t e = cudaGetLastError();
    printf("err: %s\n", cudaGetErrorString(e));
    return 0;
}
