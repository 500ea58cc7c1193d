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
#include "wang_etw.cuh"

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
    static constexpr int kPS = PS;
    static constexpr bool kShuffle = false;
    C<T>* base;
    // p = padidx<PS>(i): the engine computes padded indices (mostly per-thread
    // base + compile-time offset), the policy maps them to an address
    __device__ __forceinline__ void putp(int p, C<T> v) const { base[p] = v; }
    __device__ __forceinline__ C<T> getp(int p) const { return base[p]; }
    __device__ __forceinline__ void sync() const {
        if constexpr (TPS <= 32) __syncwarp(); else __syncthreads();
    }
    // after the re-gather: the buffer may be rewritten by the next exchange
    __device__ __forceinline__ void release() const { sync(); }
    __device__ __forceinline__ void after_last_exchange() const {}
};
// SliceMem whose radix-E -> radix-E exchange (the full transpose of a
// two-pass signal with E = TPS = R) runs on warp shuffles instead (the
// paper's warp-level stage); any other exchange still goes through smem.
template <class T, int TPS, int PS>
struct ShflSliceMem : SliceMem<T, TPS, PS> {
    static constexpr bool kShuffle = true;
};

// In-warp transpose of an E x E block (lanes t of one signal x registers):
// log2 E rounds, each swapping one lane-index bit with the same register-
// index bit: per register pair one 64-bit xor shuffle and the selects around
// it. Afterwards lane t holds what lane m held in register t, in register m.
template <class T, int E>
__device__ __forceinline__ void shfl_transpose(C<T> (&v)[E], int t) {
#pragma unroll
    for (int mask = 1; mask < E; mask <<= 1) {
        const bool hi = (t & mask) != 0;
#pragma unroll
        for (int r0 = 0; r0 < E; ++r0) {
            if (r0 & mask) continue;
            const int r1 = r0 | mask;
            const C<T> send = hi ? v[r0] : v[r1];
            C<T> recv;
            recv.x = __shfl_xor_sync(0xffffffffu, send.x, mask);
            recv.y = __shfl_xor_sync(0xffffffffu, send.y, mask);
            v[r0] = hi ? recv : v[r0];
            v[r1] = hi ? v[r1] : recv;
        }
    }
}

// Two alternating exchange regions (ping-pong): exchange k puts into and gets
// from region `cur`, then switches, so the next exchange never writes what a
// slower thread may still be reading and the trailing barrier of every
// exchange disappears (one CTA barrier per exchange instead of two). The
// region of exchange k + 2 is protected by the barrier of exchange k + 1.
// `cur` persists across tiles (the alternation continues), and `hook` runs
// once, right after the first barrier of the tile (every thread has its
// input in registers by then: the prefetch buffer may be refilled).
template <class T, int TPS, int PS, class Hook>
struct PingPongMem {
    C<T>* r0;
    C<T>* r1;
    C<T>** cur;
    Hook hook;
    mutable bool first = true;
    static constexpr int kPS = PS;
    static constexpr bool kShuffle = false;
    __device__ __forceinline__ void putp(int p, C<T> v) const { (*cur)[p] = v; }
    __device__ __forceinline__ C<T> getp(int p) const { return (*cur)[p]; }
    __device__ __forceinline__ void sync() const {
        __syncthreads();
        if (first) hook();
        first = false;
    }
    __device__ __forceinline__ void release() const { *cur = (*cur == r0) ? r1 : r0; }
    __device__ __forceinline__ void after_last_exchange() const {}
};
// U transforms interleaved: element i of transform u at pad(i)*U + u.
template <class T, int U, int PS>
struct TileMem {
    static constexpr int kPS = PS;
    static constexpr bool kShuffle = false;
    C<T>* base;
    int u;
    __device__ __forceinline__ void putp(int p, C<T> v) const { base[p * U + u] = v; }
    __device__ __forceinline__ C<T> getp(int p) const { return base[p * U + u]; }
    __device__ __forceinline__ void sync() const { __syncthreads(); }
    __device__ __forceinline__ void release() const { sync(); }
    __device__ __forceinline__ void after_last_exchange() const {}
};

// Per-tile check policy of the engine: `pre` sees a radix tile before its
// DFT, `post` after it. NoCheck compiles away; TileCheck is the thread-level
// two-sided ABFT of the paper's scheme comparison (each thread verifies the
// radix-R DFTs it computes with the Wang encoding: c_in = a . e^T W_R before,
// c_out = A . e after), keeping the worst squared relative discrepancy.
struct NoCheck {
    template <int R, class T> __device__ __forceinline__ C<T> pre(const C<T>*) { return C<T>{}; }
    template <int R, class T> __device__ __forceinline__ void post(const C<T>*, C<T>) const {}
};
template <class T>
struct TileCheck {
    // max |c_in - c_out|^2 / max(|c_in|, abs_floor, TILE_FLOOR * l1_tile)^2.
    // A radix tile's checksums carry rounding noise ~eps * sum|a|, so the
    // relative test needs a tile-scale floor (1e-2 fp32, 1e-6 fp64: noise /
    // floor stays ~1e-4 / 1e-9 below the default deltas).
    static constexpr T TILE_FLOOR = sizeof(T) == 4 ? T(1e-2) : T(1e-6);
    T worst = T(0);
    T floor2 = T(0);
    T tile_l1 = T(0);
    template <int R, class U> __device__ __forceinline__ C<T> pre(const C<T>* a) {
        C<T> c = mk<T>(T(0), T(0));
        C<T> l = mk<T>(T(0), T(0));
#pragma unroll
        for (int r = 0; r < R; ++r) {
            c = cmac<T>(c, a[r], mk<T>((T)wang_etw_re(R, r), (T)wang_etw_im(R, r)));
            l = cadd<T>(l, cabs2<T>(a[r]));
        }
        tile_l1 = fmul(TILE_FLOOR, fadd(l.x, l.y));
        return c;
    }
    template <int R, class U> __device__ __forceinline__ void post(const C<T>* A, C<T> cin) {
        C<T> acc[3] = {mk<T>(T(0), T(0)), mk<T>(T(0), T(0)), mk<T>(T(0), T(0))};
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k % 3] = cadd<T>(acc[k % 3], A[k]);
        constexpr T hr = T(-0.5), hi = T(0.8660254037844386467637232);
        C<T> cout = acc[0];
        if (R > 1) cout = cadd<T>(cout, cmul<T>(acc[1], mk<T>(hr, -hi)));
        if (R > 2) cout = cadd<T>(cout, cmul<T>(acc[2], mk<T>(hr, hi)));
        const T dx = fsub(cin.x, cout.x), dy = fsub(cin.y, cout.y);
        const T raw2 = ffma(dx, dx, fmul(dy, dy));
        const T fl = tile_l1;
        const T den2 = nanmax<T>(nanmax<T>(ffma(cin.x, cin.x, fmul(cin.y, cin.y)), floor2), fmul(fl, fl));
        const T q = raw2 / den2;
        worst = (q != q) ? T(INFINITY) : (q > worst ? q : worst);
    }
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
        NoCheck chk;
        passes<1>(v, mem, t, tw, chk, Radices{});
    }
    template <class Mem, class Check>
    static __device__ __forceinline__ void run(C<T> (&v)[E], const Mem& mem, int t,
                                               const C<T>* __restrict__ tw, Check& chk) {
        passes<1>(v, mem, t, tw, chk, Radices{});
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

    template <int Ns, class Mem, class Check, int R, int... Rest>
    static __device__ __forceinline__ void passes(C<T> (&v)[E], const Mem& mem, int t,
                                                  const C<T>* __restrict__ tw, Check& chk,
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
            const C<T> ci = chk.template pre<R, T>(a);
            Dft<T, R>::run(a);
            chk.template post<R, T>(a, ci);
#pragma unroll
            for (int r = 0; r < R; ++r) v[q + r * SUB] = a[r];
        }
        if constexpr (sizeof...(Rest) > 0 && Mem::kShuffle && Ns == 1 && R == E && TPS == E) {
            shfl_transpose<T, E>(v, t);  // warp-level stage: no shared memory, no barrier
            passes<Ns * R>(v, mem, t, tw, chk, RList<Rest...>{});
        } else if constexpr (sizeof...(Rest) > 0) {
            // padded indices: one per-thread base and compile-time offsets
            // whenever the stride is a multiple of the padding period (then
            // pad(b + k) = pad(b) + pad(k) exactly), else per element
            constexpr int PS = Mem::kPS;
            constexpr bool PUT_LIN = PS == 0 || (Ns % (1 << PS)) == 0;
            constexpr bool GET_LIN = PS == 0 || (TPS % (1 << PS)) == 0;
#pragma unroll
            for (int q = 0; q < SUB; ++q) {
                const unsigned j = (unsigned)t + q * TPS;
                const unsigned base = (j / Ns) * Ns * R + (j & (Ns - 1));
                if constexpr (PUT_LIN) {
                    const int pb = (int)(base + (PS ? base >> PS : 0u));
#pragma unroll
                    for (int r = 0; r < R; ++r) mem.putp(pb + r * (Ns + (PS ? Ns >> PS : 0)), v[q + r * SUB]);
                } else {
#pragma unroll
                    for (int r = 0; r < R; ++r) mem.putp(padidx<PS>((int)base + r * Ns), v[q + r * SUB]);
                }
            }
            mem.sync();
            if constexpr (GET_LIN) {
                const int pt = (int)((unsigned)t + (PS ? (unsigned)t >> PS : 0u));
#pragma unroll
                for (int m = 0; m < E; ++m) v[m] = mem.getp(pt + m * (TPS + (PS ? TPS >> PS : 0)));
            } else {
#pragma unroll
                for (int m = 0; m < E; ++m) v[m] = mem.getp(padidx<PS>(t + m * TPS));
            }
            mem.release();
            if constexpr (sizeof...(Rest) == 1) mem.after_last_exchange();
            passes<Ns * R>(v, mem, t, tw, chk, RList<Rest...>{});
        }
    }
    template <int Ns, class Mem, class Check>
    static __device__ __forceinline__ void passes(C<T> (&)[E], const Mem&, int, const C<T>* __restrict__,
                                                  Check&, RList<>) {}
};

}  // namespace tfft
