// Microbenchmark: host cost of launching the step kernel's shape (148 x 1024 threads, ~200 KB
// dynamic shared memory) -- cooperative vs plain launch, small vs 2.5 KB parameter block,
// and a CUDA graph relaunch with updated kernel-node parameters.  Prints the host time of
// the launch call (median of 2000, GPU idle between launches).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

struct Big { unsigned char b[2560]; };

__global__ void __launch_bounds__(1024, 1) k_small(int x, int* out) { if (x == 12345 && threadIdx.x == 0) out[0] = x; }
__global__ void __launch_bounds__(1024, 1) k_big(int x, int* out, const __grid_constant__ Big big) {
    if (x == 12345 && threadIdx.x == 0) out[0] = big.b[x & 1023];
}

template <class F>
double med(F f) {
    std::vector<double> t;
    for (int i = 0; i < 2000; i++) {
        cudaDeviceSynchronize();
        auto a = std::chrono::steady_clock::now();
        f(i);
        auto b = std::chrono::steady_clock::now();
        t.push_back(std::chrono::duration<double, std::micro>(b - a).count());
    }
    cudaDeviceSynchronize();
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int* out;
    cudaMalloc(&out, 4);
    const size_t smem = 200 * 1024;
    cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    static Big big{};
    int x = 0;
    void* a_small[] = {&x, &out};
    void* a_big[] = {&x, &out, &big};
    printf("plain  small params: %6.2f us\n", med([&](int i) { x = i; cudaLaunchKernel((void*)k_small, dim3(sms), dim3(1024), a_small, smem, s); }));
    printf("coop   small params: %6.2f us\n", med([&](int i) { x = i; cudaLaunchCooperativeKernel((void*)k_small, dim3(sms), dim3(1024), a_small, smem, s); }));
    printf("plain  2.5KB params: %6.2f us\n", med([&](int i) { x = i; cudaLaunchKernel((void*)k_big, dim3(sms), dim3(1024), a_big, smem, s); }));
    printf("coop   2.5KB params: %6.2f us\n", med([&](int i) { x = i; cudaLaunchCooperativeKernel((void*)k_big, dim3(sms), dim3(1024), a_big, smem, s); }));
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeCooperative;
    attr.val.cooperative = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = smem; cfg.stream = s;
    cfg.attrs = &attr; cfg.numAttrs = 1;
    printf("coop   2.5KB, legacy stream 0: %6.2f us\n", med([&](int i) { x = i; cudaLaunchCooperativeKernel((void*)k_big, dim3(sms), dim3(1024), a_big, smem, 0); }));
    printf("exC    2.5KB params: %6.2f us\n", med([&](int i) { x = i; cudaLaunchKernelExC(&cfg, (void*)k_big, a_big); }));
    // graph: one cooperative kernel node, parameters updated per launch
    cudaGraph_t g;
    cudaGraphCreate(&g, 0);
    cudaKernelNodeParams kp = {};
    kp.func = (void*)k_big; kp.gridDim = dim3(sms); kp.blockDim = dim3(1024); kp.sharedMemBytes = smem;
    kp.kernelParams = a_big;
    cudaGraphNode_t n;
    cudaGraphAddKernelNode(&n, g, nullptr, 0, &kp);
    cudaKernelNodeAttrValue v;
    v.cooperative = 1;
    cudaGraphKernelNodeSetAttribute(n, cudaKernelNodeAttributeCooperative, &v);
    cudaGraphExec_t ge;
    cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
    printf("graph instantiate: %s\n", cudaGetErrorString(e));
    printf("graph  relaunch   : %6.2f us\n", med([&](int) { cudaGraphLaunch(ge, s); }));
    printf("graph  set+launch : %6.2f us\n", med([&](int i) { x = i; cudaGraphExecKernelNodeSetParams(ge, n, &kp); cudaGraphLaunch(ge, s); }));
    printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
