// kernels_merge.cu -- the merge kernel of the NCCL / loopback exchange (the peer-memory
// transport merges inside the fused step kernel instead).  See merge_dev.cuh.
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

}  // namespace

cudaError_t launch_merge(const Bufs& b, const Cost& c, const StepArgs& a, cudaStream_t s) {
    const size_t smem = merge_smem_bytes(a.world, a.max_batch);
    cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_merge<<<1, kMT, smem, s>>>(b, c, a);
    return cudaGetLastError();
}

}  // namespace lamps
