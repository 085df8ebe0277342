// kernels_sort.cu -- A4: LSD radix sort of the unique 64-bit keys, ascending
// (= ranked order, Alg.1).  sm_100a.
//
// One persistent cooperative launch does every pass.  The grid is exactly the
// set of CTAs that can be resident (one 1024-thread CTA per SM), so the whole
// key set is processed by a single wave and CTAs can synchronise:
//
//   per pass (8-bit digit, only digit positions whose bits vary -- from the
//   per-block key OR/AND that K1 produced):
//     A  each CTA loads its tile(s) (warp-striped, 8 keys/thread) and ranks
//        every key among the same-digit keys of its warp with a stable warp
//        multisplit (__match_any_sync); per-digit counts of its keys go to
//        global memory
//     -- grid barrier --
//     B  each CTA reads the counts of the CTAs before it (its global per-digit
//        offsets) and of all CTAs (digit totals -> digit bases)
//     C  keys are staged digit-sorted in shared memory and written to their
//        final positions in coalesced runs
//     -- grid barrier --
//
// This replaces the per-tile decoupled look-back of a classic onesweep pass:
// measured on B200 (profiles/r01/ncu_v0_lookback.txt) the look-back over ~450
// concurrently started tiles serialised (25 us per pass); with one resident
// wave a grid-synchronous exchange of per-CTA counts is shorter and exact.
#include "sort_dev.cuh"

namespace lamps {

namespace {

__global__ void __launch_bounds__(kSortThreads, 1) k_sort(Bufs b, StepArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortSmem& sm = *reinterpret_cast<SortSmem*>(smem_raw);
    const uint32_t n = __ldcg(&b.ctl->n_elig);
    uint32_t bar = a.step * kBarPerStep;
    const uint32_t np = lsd_sort_global(b, n, b.kmask, b.score_grid, sm, bar);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        b.ctl->n_passes = np;
        b.ctl->final_buf = np & 1u;
    }
}

}  // namespace

int sort_blocks_per_sm() {
    int nb = 0;
    cudaFuncSetAttribute(k_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SortSmem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sort, kSortThreads, sizeof(SortSmem));
    return nb;
}

cudaError_t launch_sort(const Bufs& b, const Cost& c, const StepArgs& a, cudaStream_t s) {
    (void)c;
    Bufs bb = b;
    StepArgs aa = a;
    void* args[] = {&bb, &aa};
    return cudaLaunchCooperativeKernel((const void*)k_sort, dim3(b.sort_grid), dim3(kSortThreads), args,
                                       sizeof(SortSmem), s);
}

}  // namespace lamps
