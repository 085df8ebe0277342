// kernels_merge.cu -- the merge kernel of the NCCL / loopback exchange (the peer-memory
// transport merges inside the fused step kernel instead).  See merge_dev.cuh.
#include <algorithm>

#include "merge_dev.cuh"

namespace lamps {

namespace {

__global__ void __launch_bounds__(kMT) k_merge(Bufs b, Cost c, StepArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ AdmitSmem adm;
    __shared__ uint32_t nv[32];
    __shared__ unsigned long long hsum[2];
    merge_admit_cta(b, c, a, b.xrecv, smem_raw, adm, nv, hsum);
}

// large exchanges: the merged order by rank, grid-wide (merge_dev.cuh), then one CTA cuts
__global__ void __launch_bounds__(1024) k_merge_count(Bufs b, uint32_t W, uint32_t K) {
    merge_count(b.xrecv, W, K, b.xcnt);
}
__global__ void __launch_bounds__(1024) k_merge_place(Bufs b, uint32_t W, uint32_t K) {
    merge_place(b.xrecv, W, K, b.xcnt, b.xorder);
}
__global__ void __launch_bounds__(kMT) k_merge_cut(Bufs b, Cost c, StepArgs a) {
    __shared__ AdmitSmem adm;
    __shared__ uint32_t nv[32];
    __shared__ unsigned long long hsum[2];
    merge_cut_from_order(b, c, a, b.xrecv, b.xorder, adm, nv, hsum);
}

}  // namespace

bool merge_is_large(uint32_t world, uint32_t K) { return merge_smem_bytes(world, K) > kMergeSmemMax; }

cudaError_t launch_merge(const Bufs& b, const Cost& c, const StepArgs& a, cudaStream_t s) {
    if (merge_is_large(a.world, a.max_batch)) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const uint64_t R = (uint64_t)a.world * a.max_batch;
        const uint32_t gc = (uint32_t)std::min<uint64_t>((R * a.world + 1023) / 1024, (uint64_t)sms * 2);
        const uint32_t gp = (uint32_t)std::min<uint64_t>((R + 1023) / 1024, (uint64_t)sms);
        k_merge_count<<<gc, 1024, 0, s>>>(b, a.world, a.max_batch);
        k_merge_place<<<gp, 1024, 0, s>>>(b, a.world, a.max_batch);
        k_merge_cut<<<1, kMT, 0, s>>>(b, c, a);
        return cudaGetLastError();
    }
    const size_t smem = merge_smem_bytes(a.world, a.max_batch);
    cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_merge<<<1, kMT, smem, s>>>(b, c, a);
    return cudaGetLastError();
}

}  // namespace lamps
