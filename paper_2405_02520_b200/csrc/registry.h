// Kernel registry filled by the generated instantiation files (codegen.py).
#pragma once
#include <atomic>

namespace tfft {

// Kernels this library has launched (process-wide): tfft_launch_count(),
// the bench's `gpu_launches` claim.
inline std::atomic<long long> g_launches{0};
inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

struct SingleEntry {
    int logn;
    int variant;     // index into codegen.SINGLE_CANDIDATES[prec][logn]
    int chosen;      // 1 for the tuned default
    int e;           // elements per thread
    int threads;     // CTA size
    int smem;        // dynamic shared memory bytes
    int tps;         // threads per signal
    int stage;       // load strategy (STAGE template argument; 5 needs a tensor map)
    const void* fn[4];  // ABFT off / Wang / table / thread-level (last two only on the chosen variant)
    const void* fix;    // fix_single_kernel of this config (chosen variant only), see fix.cuh
    int fix_threads;    // its CTA size: max(TPS, 32)
    int fix_smem;       // its dynamic shared memory (exchange slices)
};

struct SingleTable {
    const SingleEntry* entries;
    const int* count;
};

extern const SingleTable kSingleTables_fp32[];
extern const SingleTable kSingleTables_fp64[];
extern const int kSingleParts;

}  // namespace tfft
