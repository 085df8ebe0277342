// Floor of a step measured the way bench.py measures it: L2 flushed by a 256 MiB memset, then
// event -> one kernel -> event.  Empty 1024-thread kernel with 0 / 227 KB dynamic shared memory,
// one CTA and 148 CTAs (cooperative), to separate launch + carveout cost from the step's work.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty(int* p) { extern __shared__ int s[]; if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0]; }
int main() {
    void* flush; cudaMalloc(&flush, 256 << 20);
    cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int cfg = 0; cfg < 6; cfg++) {
        int smem = (cfg & 1) ? 232448 : 0, grid = (cfg & 2) ? 148 : 1;
        bool coop = cfg >= 4;
        float tot = 0; int n = 50;
        for (int i = 0; i < n + 5; i++) {
            cudaMemsetAsync(flush, i, 256 << 20);
            cudaEventRecord(a);
            if (coop) { int* p = nullptr; void* args[] = {&p}; cudaLaunchCooperativeKernel((void*)k_empty, dim3(148), dim3(1024), args, smem, 0); }
            else k_empty<<<grid, 1024, smem>>>(nullptr);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (i >= 5) tot += ms;
        }
        printf("grid %3d smem %6d coop %d: %.2f us\n", coop ? 148 : grid, smem, coop, 1e3 * tot / n);
    }
    return 0;
}
