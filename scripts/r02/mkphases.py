"""Phase line ranges of kernels_fused.cu (for ncu_phase.py) from marker strings in the source:
each phase starts at the first line containing its marker (after the previous phase's start)."""
import sys
src = open(sys.argv[1]).read().split("\n")
marks = [("tables", "__device__ __forceinline__ uint32_t bucket_t("),
         ("L.local_lsd", "__device__ __forceinline__ uint64_t* local_lsd("),
         ("L.refine", "__device__ __forceinline__ bool refine_groups("),
         ("L.range_sort_old", "__device__ __forceinline__ void local_sort("),
         ("L.rs_loop", "__device__ __forceinline__ unsigned long long key_code("),
         ("L.small_sort", "constexpr uint32_t kSmallSort"),
         ("L.head_sparse", "__device__ __forceinline__ bool head_sparse_sort("),
         ("P.prologue", "__global__ void __launch_bounds__(kFT, 1) k_fused("),
         ("S.score_loop", "uint32_t pinned = 0, nmine = 0;"),
         ("S.reduce", 'asm volatile("cp.async.wait_all;" ::: "memory");  // table, splitters'),
         ("X.cold", "if (a.cold) {\n"),
         ("R.search", "uint32_t* const kr = reinterpret_cast<uint32_t*>(sm.s.cnt);"),
         ("R.offsets", "    TRACE(4);"),
         ("R.place", "    TRACE(5);"),
         ("R.store", "    TRACE(12);"),
         ("L.prep", "    TRACE(7);"),
         ("L.dispatch", "    // ---------------- L: sort the key ranges"),
         ("L.fallback", "    } else if (fallback) {"),
         ("A.admit", "    TRACE(8);"),
         ("end", "}  // namespace\n")]
text = "\n".join(src)
pos = 0
starts = []
for nm, m in marks:
    i = text.find(m.rstrip("\n"), pos)
    if i < 0:
        continue
    ln = text.count("\n", 0, i) + 1
    starts.append((nm, ln))
    pos = i + 1
for (nm, a), (_, b) in zip(starts, starts[1:]):
    print(f"{nm:16s} kernels_fused.cu {a} {b - 1}")
print("S.arith          lamps_dev.cuh 1 300\nS.apply          step_dev.cuh 1 78\nscans            step_dev.cuh 79 198\n"
      "S.strategy_score step_dev.cuh 199 344\nA.admit_cta      step_dev.cuh 345 600\nsort_dev         sort_dev.cuh 1 400")
