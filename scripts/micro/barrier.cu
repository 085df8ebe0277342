// Microbenchmark: grid-wide barrier latency on B200, one 1024-thread CTA per SM
// (the fused step kernel's shape).  Variants:
//   0 tree   : 16 group counters (acq_rel atom), root counter, release flag, acquire poll
//   1 flat   : red.release.gpu.add on one monotonic counter, ld.acquire poll until value*G
//   2 flat+ns: as 1 with __nanosleep(20) between polls
//   3 flat-atom: atom.add.acq_rel (returned value used to skip the poll for the last arriver)
// Reports microseconds per barrier (1000 back-to-back barriers, CUDA events).
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>

constexpr uint32_t kGroups = 16;

__device__ __forceinline__ void bar_tree(uint32_t* bar, uint32_t G, uint32_t value) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t g = blockIdx.x % kGroups;
        const uint32_t gsize = G / kGroups + (g < G % kGroups ? 1u : 0u);
        const uint32_t ng = G < kGroups ? G : kGroups;
        uint32_t* gc = bar + 32u * (1u + g);
        uint32_t* root = bar + 32u * (1u + kGroups);
        uint32_t old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(gc) : "memory");
        if (old == gsize - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(gc) : "memory");
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(root) : "memory");
            if (old == ng - 1) {
                asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(root) : "memory");
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar), "r"(value) : "memory");
            }
        }
        uint32_t cur;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
        } while ((int)(cur - value) < 0);
    }
    __syncthreads();
}

template <int SLEEP>
__device__ __forceinline__ void bar_flat(uint32_t* bar, uint32_t G, uint32_t value) {
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t* cnt = bar + 32u * 20u;
        const uint32_t target = value * G;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        uint32_t cur;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(cnt) : "memory");
            if ((int)(cur - target) >= 0) break;
            if (SLEEP) __nanosleep(SLEEP);
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void bar_flat_atom(uint32_t* bar, uint32_t G, uint32_t value) {
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t* cnt = bar + 32u * 21u;
        const uint32_t target = value * G;
        uint32_t old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
        if (old + 1u != target) {
            uint32_t cur;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(cnt) : "memory");
            } while ((int)(cur - target) < 0);
        }
    }
    __syncthreads();
}

template <int V>
__global__ void __launch_bounds__(1024, 1) k(uint32_t* bar, int iters, uint32_t base, uint32_t* sink) {
    extern __shared__ uint32_t big[];  // force one CTA per SM, like the fused kernel
    uint32_t acc = 0;
    for (int i = 0; i < iters; i++) {
        const uint32_t v = base + (uint32_t)i + 1u;
        if (V == 0) bar_tree(bar, gridDim.x, v);
        else if (V == 1) bar_flat<0>(bar, gridDim.x, v);
        else if (V == 2) bar_flat<20>(bar, gridDim.x, v);
        else bar_flat_atom(bar, gridDim.x, v);
        acc += big[threadIdx.x];
    }
    if (acc == 0xdeadbeef) sink[0] = acc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *bar, *sink;
    cudaMalloc(&bar, 32 * 4 * 32);
    cudaMalloc(&sink, 4);
    cudaMemset(bar, 0, 32 * 4 * 32);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const size_t smem = 200 * 1024;
    void* fns[] = {(void*)k<0>, (void*)k<1>, (void*)k<2>, (void*)k<3>};
    const char* names[] = {"tree (16 groups)", "flat red+poll", "flat red+poll+nanosleep20", "flat atom"};
    uint32_t base[4] = {0, 0, 0, 0};
    for (int v = 0; v < 4; v++) cudaFuncSetAttribute(fns[v], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 3; rep++) {
        for (int v = 0; v < 4; v++) {
            int iters = 1000;
            void* args[] = {&bar, &iters, &base[v], &sink};
            cudaMemset(bar, 0, 32 * 4 * 32);
            base[v] = 0;
            cudaLaunchCooperativeKernel(fns[v], dim3(sms), dim3(1024), args, smem, 0);  // warm
            cudaDeviceSynchronize();
            base[v] = 1000;
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel(fns[v], dim3(sms), dim3(1024), args, smem, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("%-28s %7.3f us/barrier  (%s)\n", names[v], ms * 1000.0f / iters,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
