// Kernel registry filled by the generated instantiation files (codegen.py).
#pragma once

namespace tfft {

struct SingleEntry {
    int logn;
    int e;           // elements per thread
    int threads;     // CTA size
    int smem;        // dynamic shared memory bytes
    int tps;         // threads per signal
    const void* fn[3];  // ABFT off / Wang / table
};

extern const SingleEntry kSingle_fp32[];
extern const int kSingleCount_fp32;
extern const SingleEntry kSingle_fp64[];
extern const int kSingleCount_fp64;

}  // namespace tfft
