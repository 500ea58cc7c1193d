// Block-level Stockham engine: one L-point transform held by TPS = L/E
// threads, E complex values per thread in registers.
//
// Pass p (radix R, span Ns = product of earlier radices) treats every thread's
// E values as E/R radix-R butterflies j = t + q*TPS whose inputs are the
// elements j + r*L/R. Thread t therefore always holds elements
// t + m*TPS (m = q + r*E/R) at the start of a pass, so the first load and the
// last store are unit-stride across threads (coalesced), and the output comes
// out in natural order with no bit-reversal (autosort). Between passes the
// results are scattered to padded shared memory at
//     o = (j / Ns) * Ns * R + (j % Ns) + r * Ns
// and re-gathered at t + m*TPS. This replaces the reference's per-stage
// radix-2 loop (kernels/_stockham.pyx:16-43) with radix-R macro butterflies
// and smem exchanges.
//
// The shared-memory placement is a policy (`Mem`): one signal per smem slice
// (single-kernel path) or U transforms interleaved element-major so that the
// U lanes of a row hit consecutive banks (multi-pass tiles).
#pragma once
#include "common.cuh"

namespace tfft {

template <int... Rs> struct RList {};

template <class L> struct RProd;
template <> struct RProd<RList<>> { static constexpr int v = 1; };
template <int R, int... Rs> struct RProd<RList<R, Rs...>> { static constexpr int v = R * RProd<RList<Rs...>>::v; };

template <class L> struct RCount;
template <int... Rs> struct RCount<RList<Rs...>> { static constexpr int v = sizeof...(Rs); };

// One padding element every 2^PS elements.
template <int PS>
__device__ __forceinline__ int padidx(int i) {
    if constexpr (PS == 0) return i; else return i + (i >> PS);
}
template <int L, int PS>
struct SmemLen { static constexpr int v = (PS == 0) ? L : L + (L >> PS) + 1; };

// ---- smem policies
// Signal-contiguous slice; signals never span warps when TPS <= 32.
template <class T, int TPS, int PS>
struct SliceMem {
    C<T>* base;
    __device__ __forceinline__ void put(int i, C<T> v) const { base[padidx<PS>(i)] = v; }
    __device__ __forceinline__ C<T> get(int i) const { return base[padidx<PS>(i)]; }
    __device__ __forceinline__ void sync() const {
        if constexpr (TPS <= 32) __syncwarp(); else __syncthreads();
    }
    __device__ __forceinline__ void after_last_exchange() const {}
};
// U transforms interleaved: element i of transform u at pad(i)*U + u.
template <class T, int U, int PS>
struct TileMem {
    C<T>* base;
    int u;
    __device__ __forceinline__ void put(int i, C<T> v) const { base[padidx<PS>(i) * U + u] = v; }
    __device__ __forceinline__ C<T> get(int i) const { return base[padidx<PS>(i) * U + u]; }
    __device__ __forceinline__ void sync() const { __syncthreads(); }
    __device__ __forceinline__ void after_last_exchange() const {}
};

template <class T, int L, int E, class Radices>
struct Engine {
    static constexpr int TPS = L / E;
    static_assert(RProd<Radices>::v == L, "radices must multiply to L");
    static_assert(E <= L && L % E == 0, "bad E");

    // tw: multi-resolution root table, tw[M + k] = w_M^k for every power of
    // two M <= L and k < M (2L entries, see twiddle_table_size()).
    template <class Mem>
    static __device__ __forceinline__ void run(C<T> (&v)[E], const Mem& mem, int t,
                                               const C<T>* __restrict__ tw) {
        passes<1>(v, mem, t, tw, Radices{});
    }

  private:
    // Pass twiddles w^r (r = 1..R-1, w = w_M^k, M = Ns*R): two contiguous
    // lookups (w and w^Q, lanes read consecutive k) and binary powering for
    // the rest, so a butterfly costs 2 loads instead of R-1 scattered ones
    // (which made L1TEX the bottleneck) at <= ~3 ulp of extra error.
    template <int Ns, int R, int SUB>
    static __device__ __forceinline__ void twiddle(C<T> (&v)[E], int q, int k,
                                                   const C<T>* __restrict__ tw) {
        constexpr int M = Ns * R;
        constexpr int Q = R <= 4 ? R : (R == 8 ? 4 : (R == 16 ? 4 : 8));
        C<T> p[Q];  // p[b] = w^b, b < Q
        p[1] = __ldg(tw + M + k);
#pragma unroll
        for (int b = 2; b < Q; ++b) p[b] = cmul<T>(p[b / 2], p[b - b / 2]);
        if constexpr (Q == R) {
#pragma unroll
            for (int r = 1; r < R; ++r) v[q + r * SUB] = cmul<T>(v[q + r * SUB], p[r]);
        } else {
            constexpr int A = R / Q;
            C<T> g[A];  // g[a] = w^(Q a)
            g[1] = __ldg(tw + M / Q + k);
#pragma unroll
            for (int a = 2; a < A; ++a) g[a] = cmul<T>(g[a / 2], g[a - a / 2]);
#pragma unroll
            for (int r = 1; r < R; ++r) {
                const int a = r / Q, b = r % Q;
                C<T> w;
                if (a == 0) w = p[b];
                else if (b == 0) w = g[a];
                else w = cmul<T>(g[a], p[b]);
                v[q + r * SUB] = cmul<T>(v[q + r * SUB], w);
            }
        }
    }

    template <int Ns, class Mem, int R, int... Rest>
    static __device__ __forceinline__ void passes(C<T> (&v)[E], const Mem& mem, int t,
                                                  const C<T>* __restrict__ tw,
                                                  RList<R, Rest...>) {
        static_assert(E % R == 0, "radix must divide elements per thread");
        constexpr int SUB = E / R;
#pragma unroll
        for (int q = 0; q < SUB; ++q) {
            const int j = t + q * TPS;
            if constexpr (Ns > 1) twiddle<Ns, R, SUB>(v, q, j & (Ns - 1), tw);  // w_{Ns R}^{(j mod Ns) r}
            C<T> a[R];
#pragma unroll
            for (int r = 0; r < R; ++r) a[r] = v[q + r * SUB];
            Dft<T, R>::run(a);
#pragma unroll
            for (int r = 0; r < R; ++r) v[q + r * SUB] = a[r];
        }
        if constexpr (sizeof...(Rest) > 0) {
#pragma unroll
            for (int q = 0; q < SUB; ++q) {
                const int j = t + q * TPS;
                const int base = (j / Ns) * Ns * R + (j & (Ns - 1));
#pragma unroll
                for (int r = 0; r < R; ++r) mem.put(base + r * Ns, v[q + r * SUB]);
            }
            mem.sync();
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = mem.get(t + m * TPS);
            mem.sync();
            if constexpr (sizeof...(Rest) == 1) mem.after_last_exchange();
            passes<Ns * R>(v, mem, t, tw, RList<Rest...>{});
        }
    }
    template <int Ns, class Mem>
    static __device__ __forceinline__ void passes(C<T> (&)[E], const Mem&, int, const C<T>* __restrict__,
                                                  RList<>) {}
};

}  // namespace tfft
