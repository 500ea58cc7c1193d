// N-point transform split across a 2-CTA thread-block cluster (sm_100a):
// CTA rank h computes the N/2-point FFT of the decimation-in-frequency half
//   y_0[j] = x[j] + x[j + N/2],   y_1[j] = (x[j] - x[j + N/2]) w_N^j,
// whose outputs are X[2k + h]. Both CTAs receive the whole signal by TMA
// multicast (each issues one half, delivered to both), so each half-FFT's
// input is formed in registers without any exchange; the outputs are
// re-partitioned through distributed shared memory (each CTA sends the
// partner the k range it stores) so every CTA writes one contiguous half of
// X as 16-byte (X[2k], X[2k+1]) pairs. Two CTAs of ~113 KB smem and 8 warps
// each share an SM: twice the warps of the single-CTA N = 8192 kernel, and
// its three CTA-wide exchanges become two CTA-local ones plus one
// cluster exchange.
#pragma once
#include "single.cuh"

namespace tfft {

__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// whole-cluster barrier (every thread of both CTAs, warp-converged)
__device__ __forceinline__ void cl_sync() {
    __syncwarp();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the partner CTA's shared-window address of a local shared address
__device__ __forceinline__ unsigned cl_map(unsigned local, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
__device__ __forceinline__ void cl_store(unsigned addr, float2 v) {
    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void cl_store(unsigned addr, double2 v) {
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}
// bulk global -> shared copy delivered to every CTA in `mask` (same offset,
// completing on the same-offset mbarrier of each)
__device__ __forceinline__ void bulk_g2s_mc(unsigned dst, const void* src, unsigned bytes, unsigned bar,
                                            unsigned short mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
        "%4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "h"(mask)
        : "memory");
}

template <class T, int N, int E, int PS, int ABFT, int THREADS, int MINB, int STAGE, class Radices>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, MINB)
fft_cluster_kernel(const __grid_constant__ SingleArgs<T> a) {
    constexpr int NH = N / 2;           // points per CTA
    constexpr bool NO_MC = (STAGE & 128) != 0;   // experiment: each CTA loads the whole signal itself
    constexpr bool NO_DS = (STAGE & 256) != 0;   // experiment: no DSMEM exchange (interleaved stores)
    constexpr int TPS = NH / E;
    static_assert(TPS == THREADS, "one half-signal per CTA");
    static_assert(E % 2 == 0, "E must split into the two output ranges");
    using Eng = Engine<T, NH, E, Radices>;
    constexpr int SL = SmemLen<NH, PS>::v;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    C<T>* xin = reinterpret_cast<C<T>*>(smem_raw);  // the whole signal (multicast)
    C<T>* ex = xin + N;                              // exchange slice of the half FFT
    C<T>* xo = ex + SL;                              // partner's values for my output range
    __shared__ unsigned long long in_bar;
    const unsigned rank = cluster_rank();
    const int t = threadIdx.x;
    const long long ncl = gridDim.x / 2, cid = blockIdx.x / 2;
    const unsigned bar_s = smem_u32(&in_bar), xin_s = smem_u32(xin);
    constexpr unsigned HALF_BYTES = (unsigned)(NH * sizeof(C<T>));
    auto issue = [&](long long sig) {  // thread 0: my half of signal `sig`, to both CTAs
        if constexpr (NO_MC) {
            bulk_g2s_s(xin_s, a.in + sig * N, 2 * HALF_BYTES, bar_s);
        } else {
            bulk_g2s_mc(xin_s + rank * HALF_BYTES, a.in + sig * N + rank * NH, HALF_BYTES, bar_s,
                        (unsigned short)3);
        }
    };
    if (t == 0) {
        mbar_init(&in_bar, 1);
    }
    __syncthreads();
    cl_sync();  // both barriers initialised
    if (t == 0 && cid < a.batch) mbar_expect_tx_s(bar_s, 2 * HALF_BYTES);
    cl_sync();  // both armed before either issues
    if (t == 0 && cid < a.batch) issue(cid);
    const unsigned xo_remote = cl_map(smem_u32(xo), rank ^ 1u);
    // w_N^j for j = t + m TPS: base w_N^t times the E constants w_E^m
    const C<T> wt = __ldg(a.tw + N + t);
    unsigned it = 0;
    for (long long sig = cid; sig < a.batch; sig += ncl, ++it) {
        mbar_wait_s(bar_s, it & 1);
        C<T> v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const C<T> x0 = xin[t + m * TPS], x1 = xin[t + m * TPS + NH];
            if (rank == 0) {
                v[m] = cadd<T>(x0, x1);
            } else {
                // w_N^(t + m TPS) = w_N^t w_2E^m (TPS = N / 2E); w_2E^m = unit64(m 32/E) conjugated
                constexpr int K64 = 32 / E;
                const Oct o = unit64(m * K64);
                v[m] = cmul<T>(cmul<T>(csub<T>(x0, x1), wt), mk<T>((T)o.c, (T)-o.s));
            }
        }
        // done reading xin: arm the next phase, then let the partner (and me) refill it
        const bool more = sig + ncl < a.batch;
        if (t == 0 && more) mbar_expect_tx_s(bar_s, 2 * HALF_BYTES);
        cl_sync();  // both CTAs have their signal in registers: refill both buffers
        if (t == 0 && more) issue(sig + ncl);
        {
            const SliceMem<T, TPS, PS> mem{ex};
            Eng::run(v, mem, t, a.tw);
        }
        if constexpr (NO_DS) {
            C<T>* dst = a.out + sig * N;
#pragma unroll
            for (int m = 0; m < E; ++m) __stcs(dst + 2 * (t + m * TPS) + rank, v[m]);
            continue;
        }
        // v[m] = Y_h[k], k = t + m TPS; CTA 0 stores X[0, N/2) (k < N/4), CTA 1 the rest
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const bool mine = (m < E / 2) == (rank == 0);
            if (!mine) {
                const int kk = t + (m % (E / 2)) * TPS;  // index within the partner's range
                cl_store(xo_remote + (unsigned)(kk * sizeof(C<T>)), v[m]);
            }
        }
        cl_sync();
        C<T>* dst = a.out + sig * N;
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const bool mine = (m < E / 2) == (rank == 0);
            if (mine) {
                const int k = t + m * TPS;
                const C<T> other = xo[t + (m % (E / 2)) * TPS];
                const C<T> e0 = rank == 0 ? v[m] : other, e1 = rank == 0 ? other : v[m];
                if constexpr (sizeof(T) == 4) {
                    __stcs(reinterpret_cast<float4*>(dst) + k, make_float4(e0.x, e0.y, e1.x, e1.y));
                } else {
                    __stcs(dst + 2 * k, e0);
                    __stcs(dst + 2 * k + 1, e1);
                }
            }
        }
    }
    // the partner may still read my xo / multicast into me: leave together
    cl_sync();
}

}  // namespace tfft
