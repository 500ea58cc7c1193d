// Single-kernel fault-tolerant FFT for N <= 2^13 (one reference "stage",
// reference planner.py:20-23), with two-sided ABFT fused into its only memory
// pass:
//   load   : x -> registers; left-side input checksum c_in = x . (e^T W) and the
//            l1 mass are accumulated from the pristine values (reference
//            abft/pipeline.py:72-85, protected.py:105-109);
//   compute: Stockham passes in registers + padded smem (engine.cuh);
//   store  : y -> HBM; output checksum c_out = y . e (Wang weights folded
//            into three residue-class sums), per-signal relative discrepancy
//            and the flag decision (pipeline.py:104-135) are computed while the
//            results are stored. Only flagged signals and the running max are
//            written — no per-signal HBM traffic on the fault-free path.
// The cross-batch (right-side) combination s0 = sum_b x_b is rebuilt from the
// preserved input only for flagged groups ("s0").
#pragma once
#include <cuda.h>  // CUtensorMap (STAGE 5 tile loads)

#include "engine.cuh"

namespace tfft {

enum { AT_NONE = 0, AT_INPUT = 1, AT_PRESCALE = 2, AT_OUTPUT = 3 };

// Cost-attribution builds only (tools/ablate.py): drop parts of the fused
// ABFT to time them. 1: cross-thread reduction, 2: c_in MACs, 4: l1 bound,
// 8: c_out class sums. Never set in the product build.
#ifndef TFFT_ABLATE
#define TFFT_ABLATE 0
#endif
#ifndef TFFT_EW_HOIST
#define TFFT_EW_HOIST 1
#endif
#ifndef TFFT_DEFER_MIN
#define TFFT_DEFER_MIN 128  // signals of >= this many threads use the smem partial pipeline
#endif
#ifndef TFFT_ONE_LOOP_ALL
#define TFFT_ONE_LOOP_ALL 0  // experiment builds: every config with the single runtime tile loop
#endif
#ifndef TFFT_EW_SMEM
#define TFFT_EW_SMEM 1
#endif
// ABFT_THREAD: the paper's thread-level scheme (scheme comparison only):
// every radix tile is verified by its thread (engine TileCheck) instead of
// the per-signal threadblock checksums.
enum { ABFT_OFF = 0, ABFT_WANG = 1, ABFT_TABLE = 2, ABFT_THREAD = 3 };

// One flagged (or recheck) signal: global index and relative discrepancy
// (double for both precisions). The records follow the counters in one
// device block, so one copy brings back the counters and the first records.
struct FlagRec {
    long long sig;
    double rel;
};

// One group of a correction pass: its first signal and the flagged one
// (global indices); ok = 1 once corrected and verified.
struct FixJob {
    long long first;
    long long flagged;
    int ok;
    int pad;
};

// Append one flag: a record while the list has room, else a bit in the
// overflow mask (the host recomputes those signals' rel exactly). The record
// list is bounded (kMaxFlagRecords), so a degenerate batch with millions of
// flags costs batch/8 bytes of mask instead of 16 B per signal.
__device__ __forceinline__ void record_flag(FlagRec* rec, long long cap, unsigned* ovf, long long slot,
                                            long long sig, double rel) {
    if (slot < cap) rec[slot] = FlagRec{sig, rel};
    else atomicOr(ovf + (sig >> 5), 1u << (sig & 31));
}

template <class T> struct KeyT;
template <> struct KeyT<float>  { using type = unsigned int; };
template <> struct KeyT<double> { using type = unsigned long long; };

// One fault per run of a batched fault campaign (f_table[r] applies to the
// f_div signals of run r; signal is run-relative). pos: element (single
// kernel) or tile unit (multi-pass), idx: element within the unit; where uses
// the launch codes of the kernel (AT_NONE = no fault in this run / pass).
struct FaultRec {
    long long pos;
    int idx, signal, where, comp, bit, pad;
};

// 2-D tensor TMA (SASS UTMALDG) of one box into shared memory
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_2d_s(unsigned dst, const CUtensorMap* map, int c0, int c1, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(dst), "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

template <class T>
struct alignas(64) SingleArgs {
    CUtensorMap tmap;       // STAGE 5: (batch x N) rows, box S x (N + pad) (OOB pad columns zero-filled)
    const C<T>* in;
    C<T>* out;
    long long batch;        // signals in this launch
    long long sig_base;     // global index of signal 0 (for reports)
    const C<T>* tw;         // w_N^k, k < N
    const C<T>* etw;        // input-side checksum row (e^T W or e^T W^-1), plan dtype
    const C<T>* values;     // encoding weights (ABFT_TABLE only)
    T delta, abs_floor, floor_coef;
    int inverse;            // conjugate-direction transform
    int scale_inv;          // multiply by 1/N (fft_execute inverse; tile_fft never)
    // results
    int* flag_count;
    FlagRec* flag_rec;
    long long flag_cap;
    unsigned* flag_ovf;     // bitmask (global signal index) of flags past flag_cap
    typename KeyT<T>::type* max_key;
    T* rel_out;             // optional per-signal relative discrepancy
    // one device-side fault (reference fault_lab/bits.py:56-77 semantics)
    long long f_signal, f_elem;
    int f_where, f_comp, f_bit;
    const FaultRec* f_table;  // batched campaign: one fault per f_div signals (overrides f_*)
    long long f_div;
};


// Detection decision of one signal from its reduced checksums (reference
// pipeline.py:104-121): rel = |c_in - c_out| / max(|c_in|, max(abs_floor,
// FLOOR_COEF * sum|x|)), flag when rel > delta, non-finite -> inf.
// The kernels carry l1b = sum(|re| + |im|), an upper bound of sum|x| within a
// factor sqrt(2) that costs one packed add per element instead of a hypot.
// Whenever the floor cannot matter (|c_in| >= FLOOR_COEF * l1b) or is exactly
// abs_floor, the decision and rel are the reference's; otherwise (tiny
// |c_in|, rare) the signal is sent back for an exact recheck (recheck_kernel).
// A squared screen (no sqrt/div) clears the common case; anything near delta,
// non-finite or out of range takes the exact arithmetic.
#ifndef TFFT_BATCH_DECIDE
#define TFFT_BATCH_DECIDE 1
#endif

template <class T>
__device__ __forceinline__ void abft_decide(T r0, T r1, T r2, T r3, T l1b, T delta, T abs_floor, T coef,
                                            bool want_rel, T& rel, T& rel2, bool& flagged, bool& recheck) {
    flagged = false;
    recheck = false;
    rel = T(0);
    rel2 = T(0);
    const T dx = fsub(r0, r2), dy = fsub(r1, r3);
    const T raw2 = ffma(dx, dx, fmul(dy, dy));
    const T cin2 = ffma(r0, r0, fmul(r1, r1));
    const T fb = fmul(coef, l1b);
    const T flb = nanmax<T>(abs_floor, fb);
    const bool floor_free = cin2 >= fmul(flb, flb);  // false for NaN
    const bool abs_floor_exact = l1b == l1b && !(fb > abs_floor);
    if (!floor_free && !abs_floor_exact) {
        recheck = true;
        return;
    }
    const T fl = floor_free ? T(0) : abs_floor;  // the exact floor term that can still matter
    const T den2 = floor_free ? cin2 : nanmax<T>(cin2, fmul(fl, fl));
    const T d2 = fmul(delta, delta);
    // screen by multiplication (no division on the common path); fp32 keeps
    // den2 <= 2^126 so the approximate reciprocal below stays normal
    constexpr T DEN_MAX = sizeof(T) == 4 ? T(8.5070592e37) : std::numeric_limits<T>::max();
    const bool in_range = den2 >= std::numeric_limits<T>::min() && den2 <= DEN_MAX &&
                          raw2 <= std::numeric_limits<T>::max();
    if (in_range && raw2 < fmul(fmul(T(0.81), d2), den2)) {
        // q = raw2 / den2 only feeds the running max and rel_out (decisions
        // come from the exact path below): fp32 uses the approximate reciprocal
        T q;
        if constexpr (sizeof(T) == 4) {
            float r;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(den2));
            q = raw2 * r;
        } else {
            q = raw2 / den2;
        }
        rel2 = q;
        if (want_rel) rel = sqrt(q);
    } else {
        const T cin = cabs<T>(mk<T>(r0, r1));
        const T den = floor_free ? cin : nanmax<T>(cin, fl);
        rel = cabs<T>(mk<T>(dx, dy)) / den;
        if (!isfinite(rel)) rel = T(INFINITY);
        flagged = rel > delta;
        rel2 = T(0);  // the caller keeps exact rel values un-squared
    }
}

// Sum K values over the TPS consecutive threads of one signal (deterministic
// tree). For TPS > 32 the per-warp partials go through `scratch` (K slots per
// warp of the CTA) with a single barrier; only thread t == 0 of the signal
// gets the totals. The scratch is next written only after the following
// tile's Stockham barriers, so no trailing barrier is needed.
template <int TPS, int K, class T>
__device__ __forceinline__ void sig_sum(T (&val)[K], T* scratch, int t) {
    constexpr int W = TPS < 32 ? TPS : 32;
#pragma unroll
    for (int off = W / 2; off >= 1; off >>= 1) {
#pragma unroll
        for (int i = 0; i < K; ++i) val[i] = fadd(val[i], shfl_xor(val[i], off));
    }
    if constexpr (TPS > 32) {
        const int warp = threadIdx.x >> 5;
        if ((threadIdx.x & 31) == 0) {
#pragma unroll
            for (int i = 0; i < K; ++i) scratch[warp * K + i] = val[i];
        }
        __syncthreads();
        if (t == 0) {
#pragma unroll
            for (int i = 0; i < K; ++i) {
                T s = scratch[warp * K + i];
#pragma unroll
                for (int w = 1; w < TPS / 32; ++w) s = fadd(s, scratch[(warp + w) * K + i]);
                val[i] = s;
            }
        }
    }
}

// TPS > 32: warp-level partial sums of K values, written by lane 0 of each
// warp to `slot` (K per warp) with no barrier; the cross-warp sum and the
// decision are deferred until after the next tile's first barrier.
template <int K, class T>
__device__ __forceinline__ void warp_partials(T (&val)[K], T* slot) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
#pragma unroll
        for (int i = 0; i < K; ++i) val[i] = fadd(val[i], shfl_xor(val[i], off));
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int i = 0; i < K; ++i) slot[(threadIdx.x >> 5) * K + i] = val[i];
    }
}

// Smem slice length of one signal: the Stockham exchange buffer and/or the
// staging buffer of coalesced I/O (stride N+1 keeps per-thread rows off the
// same banks).
template <int N, int PS, bool MULTIPASS, bool STAGE, bool INPLACE = false>
struct SliceLen {
    static constexpr int ex = MULTIPASS ? SmemLen<N, PS>::v : 0;
    static constexpr int st = STAGE ? N + 1 : (INPLACE ? N : 0);
    static constexpr int v = ex > st ? ex : st;
};

// Engine memory policy of the in-place prefetch (STAGE 4): the padded
// exchange slices, plus a hook the engine calls once the last exchange has
// been read back, when the buffer is free to receive the next tile.
template <class T, int TPS, int PS, class Hook>
struct SliceMemHook : SliceMem<T, TPS, PS> {
    Hook hook;
    __device__ __forceinline__ void after_last_exchange() const { hook(); }
};

// CTA-cooperative, fully coalesced vector copies between HBM and the staging
// slices (used when a signal is too short for per-thread coalescing).
template <class T, int N, int S, int SL, int THREADS>
__device__ __forceinline__ void stage_in(const C<T>* __restrict__ src, long long valid, C<T>* sm_all) {
    if constexpr (sizeof(T) == 4) {
        const float4* s4 = reinterpret_cast<const float4*>(src);
        for (int i = threadIdx.x; i < S * N / 2; i += THREADS) {
            const int e = 2 * i;
            if (e < valid) {
                const float4 q = __ldcs(s4 + i);
                const int sg = e / N, p = e % N;
                sm_all[sg * SL + p] = make_float2(q.x, q.y);
                sm_all[sg * SL + p + 1] = make_float2(q.z, q.w);
            }
        }
    } else {
        for (int e = threadIdx.x; e < S * N; e += THREADS) {
            if (e < valid) sm_all[(e / N) * SL + e % N] = __ldcs(src + e);
        }
    }
}
template <class T, int N, int S, int SL, int THREADS>
__device__ __forceinline__ void stage_out(C<T>* __restrict__ dst, long long valid, const C<T>* sm_all) {
    if constexpr (sizeof(T) == 4) {
        float4* d4 = reinterpret_cast<float4*>(dst);
        for (int i = threadIdx.x; i < S * N / 2; i += THREADS) {
            const int e = 2 * i;
            if (e < valid) {
                const int sg = e / N, p = e % N;
                const float2 u = sm_all[sg * SL + p], w = sm_all[sg * SL + p + 1];
                __stcs(d4 + i, make_float4(u.x, u.y, w.x, w.y));
            }
        }
    } else {
        for (int e = threadIdx.x; e < S * N; e += THREADS) {
            if (e < valid) __stcs(dst + e, sm_all[(e / N) * SL + e % N]);
        }
    }
}

template <bool B>
struct BoolC {
    static constexpr bool value = B;
};
template <int I>
struct IntC {
    static constexpr int value = I;
};

template <class T, int N, int E, int PS, int ABFT, int THREADS, int MINB, int STAGE_CODE, class Radices>
__global__ void __launch_bounds__(THREADS, MINB)
fft_single_kernel(const __grid_constant__ SingleArgs<T> a) {
    // STAGE_CODE = load strategy (below) | 8: the e^T W row read from shared
    // memory every tile even for short signals (frees the registers the
    // compiler would otherwise pin it in across tiles: occupancy)
    constexpr int STAGE = STAGE_CODE & 7;
    constexpr bool EW_SM_ALL = (STAGE_CODE & 8) != 0;
    constexpr bool SHFL = (STAGE_CODE & 16) != 0;  // warp-shuffle transpose stage (E = TPS = radix)
    // | 32: the e^T W row in DYNAMIC shared memory behind the ABFT scratch,
    // for any N (the static copy below is capped at 16 KB); for kernels whose
    // occupancy registers, not shared memory, set (fp32 N = 4096 / 8192)
    constexpr bool EWB = (STAGE_CODE & 32) != 0;
    // | 64: ONE tile loop with the direction and the fault injection decided
    // at run time (fewer registers: the occupancy of some short-signal configs)
    constexpr bool ONE_LOOP = (STAGE_CODE & 64) != 0 || TFFT_ONE_LOOP_ALL;
    using Eng = Engine<T, N, E, Radices>;
    constexpr int TPS = N / E;
    constexpr int S = THREADS / TPS;  // signals per CTA
    static_assert(S >= 1 && S * TPS == THREADS, "CTA must hold whole signals");
    static_assert(!STAGE || N >= 2, "staging needs N >= 2");
    // STAGE: 0 direct coalesced loads, 1 CTA-staged vector I/O (short
    // signals), 2 TMA bulk prefetch of the next tile into smem (cp.async.bulk
    // + mbarrier) while the current tile computes.
    // 3: both — TMA prefetch of the next contiguous chunk, then an on-chip
    // reshuffle into the padded staging slices (short signals).
    // 4: in-place TMA prefetch — the next tile lands in the exchange buffer
    // itself (linear layout) once the last exchange of the current tile has
    // been read, so prefetching costs no extra shared memory (two CTAs/SM at
    // N = 8192).
    // 6: like 2 (TMA bulk prefetch of the next tile into its own buffer), with
    // two ping-pong exchange regions (PingPongMem): one CTA barrier per
    // exchange instead of two, and the refill issued right after the tile's
    // first exchange barrier (multi-warp signals only).
    // 5: one 2-D tensor TMA per tile whose box is 4 (complex64) / 2
    // (complex128) elements WIDER than a signal: the out-of-bounds columns are
    // zero-filled, so signals land at a padded stride and the t + m*TPS reads
    // of one warp's signals fall on different banks (a linear chunk puts them
    // all on the same banks: 8-way conflicts at N = 32).
    constexpr bool STG = STAGE == 1 || STAGE == 3;
    constexpr bool PF = STAGE == 2 || STAGE == 3 || STAGE == 5 || STAGE == 6;
    constexpr bool PP = STAGE == 6;
    constexpr bool PFI = STAGE == 4;
    constexpr bool PFR = STAGE == 5;
    constexpr int SLP = PFR ? N + 32 / (int)sizeof(C<T>) : N;  // prefetch slot stride (elements)
    static_assert(!PFR || (SLP * (int)sizeof(C<T>) / 4 <= 256 && S <= 256), "tensor-TMA box limits");
    static_assert(!PFI || TPS > 32, "in-place prefetch needs CTA-wide exchange barriers");
    static_assert(!PP || (TPS > 32 && RCount<Radices>::v > 1), "ping-pong exchanges need CTA-wide exchanges");
    constexpr bool MULTIPASS = RCount<Radices>::v > 1;
    constexpr int SL = SliceLen<N, PS, MULTIPASS, STG, PFI>::v;
    constexpr int NW = THREADS / 32 > 0 ? THREADS / 32 : 1;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    C<T>* ib = reinterpret_cast<C<T>*>(smem_raw);  // prefetch buffer (PF)
    C<T>* sm_all = ib + (PF ? S * SLP : 0);
    T* red = reinterpret_cast<T*>(sm_all + (PP ? 2 : 1) * S * SL);  // 5 partial sums per warp
    // ABFT scratch size in T (codegen.single_configs `red`), rounded to 16 bytes
    constexpr int RED_T = (10 * (THREADS / 32 + 1) + (TPS >= 64 ? 10 * THREADS + 10 * S : 0) + 3) / 4 * 4;
    __shared__ typename KeyT<T>::type cta_max;
    __shared__ unsigned long long in_bar;

    const int sl = threadIdx.x / TPS;
    const int t = threadIdx.x % TPS;
    C<T>* sm = sm_all + sl * SL;
    C<T>* pp_cur = sm;  // PP: the exchange region of the next exchange (alternates across tiles)
    T my_max = T(0);   // max rel^2 of screen-decided signals
    T my_maxr = T(0);  // max rel of exactly decided signals (rel^2 would overflow at rel > ~1e19 in fp32)
    if (threadIdx.x == 0) cta_max = 0;

    const long long tiles = (a.batch + S - 1) / S;
    C<T>* const pf_dst = PFI ? sm_all : ib;
    const unsigned pf_dst_s = smem_u32(pf_dst), in_bar_s = smem_u32(&in_bar);  // once, outside the tile loop
    auto prefetch = [&](long long tl) {  // thread 0 only (PFR: threads 0..S-1, one row each)
        const long long nsig = (a.batch - tl * S) < S ? (a.batch - tl * S) : S;
        if constexpr (PFR) {  // the full box arrives, OOB rows / columns as zeros
            (void)nsig;
            mbar_expect_tx_s(in_bar_s, (unsigned)(S * SLP * sizeof(C<T>)));
            tma_load_2d_s(pf_dst_s, &a.tmap, 0, (int)(tl * S), in_bar_s);
        } else {
            const unsigned bytes = (unsigned)(nsig * N * sizeof(C<T>));
            mbar_expect_tx_s(in_bar_s, bytes);
            bulk_g2s_s(pf_dst_s, a.in + tl * S * N, bytes, in_bar_s);
        }
    };
    constexpr int ISSUE = 1;  // the thread that issues (and arrives on) each prefetch
    if constexpr (PF || PFI) {
        if (threadIdx.x == 0) mbar_init(&in_bar, ISSUE);
        __syncthreads();
        if (threadIdx.x < ISSUE && blockIdx.x < tiles) prefetch(blockIdx.x);
    }
    // Detection decision of one signal from its five reduced sums and the
    // warp-aggregated append of flagged / recheck signals (rare). Every lane
    // of the warp calls it (ballot); only `owner` lanes decide.
    auto decide_signal = [&](const T (&sums)[5], long long bsig, bool owner) {
        bool flagged = false, recheck = false;
        T rel = T(0);
        if (owner) {
            T rel2;
            abft_decide<T>(sums[0], sums[1], sums[2], sums[3], sums[4], a.delta, a.abs_floor, a.floor_coef,
                           a.rel_out != nullptr, rel, rel2, flagged, recheck);
            if (recheck) {
                rel = T(-1);  // sentinel: the host recomputes it exactly
            } else {
                my_max = my_max > rel2 ? my_max : rel2;  // squared screen value; sqrt once per CTA
                my_maxr = my_maxr > rel ? my_maxr : rel;  // exact path (rel2 = 0 there: no overflow)
            }
            if (a.rel_out) a.rel_out[bsig] = rel;
            flagged = flagged || recheck;
        }
        const unsigned ball = __ballot_sync(0xffffffffu, flagged);
        if (ball) {
            const int lane = threadIdx.x & 31;
            int base = 0;
            if (lane == __ffs(ball) - 1) base = atomicAdd(a.flag_count, __popc(ball));
            base = __shfl_sync(0xffffffffu, base, __ffs(ball) - 1);
            if (flagged) {
                const long long slot = base + __popc(ball & ((1u << lane) - 1u));
                record_flag(a.flag_rec, a.flag_cap, a.flag_ovf, slot, a.sig_base + bsig, (double)rel);
            }
        }
    };
    // TPS > 32: the cross-thread sums run as a two-tile pipeline through the
    // barriers the next tiles already have (no extra barrier, few shuffles):
    //   end of tile i     : every thread stores its 5 partials (part[par]);
    //   tile i+1 (stage 1): the signal's warps reduce them, warp w taking sums
    //                       w, w + TPS/32, ... (strided LDS + 5 shuffles), and
    //                       store the totals (tot[par]);
    //   tile i+2 (stage 2): thread t == 0 decides tile i.
    // Summation order is fixed (deterministic rel values).
    // 32 < TPS < 128 (two or three warps per signal): one-tile deferral — the
    // warps shuffle their sums fully, lanes 0 store them (parity-buffered), and
    // thread t == 0 adds the few warp totals after the next tile's barrier.
    constexpr bool TB = ABFT == ABFT_WANG || ABFT == ABFT_TABLE;  // threadblock-level checksums
    constexpr bool DEFER1 = TB && TPS > 32 && TPS < TFFT_DEFER_MIN;
    constexpr bool DEFER = TB && TPS >= TFFT_DEFER_MIN && TPS > 32;
    bool pend = false, pend_live = false;
    long long pend_b = 0;
    unsigned pend_par = 0;
    auto finish_pending = [&]() {
        T sums[5] = {T(0), T(0), T(0), T(0), T(0)};
        const bool owner = t == 0 && pend_live;
        if (owner) {
            const T* pr = red + (size_t)pend_par * NW * 5;
            const int warp = threadIdx.x >> 5;
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                T sacc = pr[warp * 5 + i];
#pragma unroll
                for (int w = 1; w < (TPS > 32 ? TPS / 32 : 1); ++w) sacc = fadd(sacc, pr[(warp + w) * 5 + i]);
                sums[i] = sacc;
            }
        }
        decide_signal(sums, pend_b, owner);
        pend = false;
    };
    // 2 <= TPS <= 32: batched decisions (one decision pass per TPS tiles)
    constexpr bool BATCHD = TB && TPS >= 2 && TPS <= 32 && TFFT_BATCH_DECIDE;
    T keep[5] = {T(0), T(0), T(0), T(0), T(0)};
    long long keep_b = 0;
    bool keep_v = false;
    constexpr int NWS = TPS > 32 ? TPS / 32 : 1;  // warps per signal
    constexpr int PPS = TPS;                         // stored partials per sum per signal
    T* const part = red;                             // [2][S][5][PPS]
    T* const tot = red + 2 * S * 5 * PPS;            // [2][S][5]
    bool p1 = false, p1_live = false, p2 = false, p2_live = false;
    long long p1_b = 0, p2_b = 0;
    unsigned p1_par = 0, p2_par = 0;
    auto stage_reduce = [&]() {  // tile held in p1 -> totals; moves it to p2
        const int ws = t >> 5, lane = threadIdx.x & 31;
        const T* pp = part + ((size_t)p1_par * S + sl) * 5 * PPS;
#pragma unroll
        for (int i0 = 0; i0 < 5; i0 += NWS) {
            const int i = i0 + ws;
            if (i < 5) {  // warp-uniform
                T acc = lane < PPS ? pp[i * PPS + lane] : T(0);
#pragma unroll
                for (int k = 1; k < (PPS + 31) / 32; ++k) acc = fadd(acc, pp[i * PPS + k * 32 + lane]);
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) acc = fadd(acc, shfl_xor(acc, off));
                if (lane == 0) tot[((size_t)p1_par * S + sl) * 5 + i] = acc;
            }
        }
        p2 = true;
        p2_live = p1_live;
        p2_b = p1_b;
        p2_par = p1_par;
        p1 = false;
    };
    auto stage_decide = [&]() {  // tile held in p2
        T sums[5] = {T(0), T(0), T(0), T(0), T(0)};
        const bool owner = t == 0 && p2_live;
        if (owner) {
#pragma unroll
            for (int i = 0; i < 5; ++i) sums[i] = tot[((size_t)p2_par * S + sl) * 5 + i];
        }
        decide_signal(sums, p2_b, owner);
        p2 = false;
    };
    // The e^T W row (<= 16 KB, signals of >= 2 warps) staged in shared memory once per CTA: the
    // per-tile reads are then LDS instead of L1-hit LDGs (fp32 N = 2048:
    // 0.512 -> 0.491 ms; at 32 KB the lost occupancy costs more than it saves)
    // (not with the ping-pong regions, whose dynamic smem already sets the occupancy)
    constexpr bool EWS = TFFT_EW_SMEM && TB &&
                         (EWB || ((TPS >= 64 || EW_SM_ALL) && N * (int)sizeof(C<T>) <= 16384 && !PP));
    __shared__ C<T> etw_st[EWS && !EWB ? N : 1];
    C<T>* const etw_sm = EWB ? reinterpret_cast<C<T>*>(red + RED_T) : etw_st;
    if constexpr (EWS) {
        for (int i = threadIdx.x; i < N; i += THREADS) etw_sm[i] = a.etw[i];
        __syncthreads();
    }
    // the persistent tile loop, instantiated for the fault-free forward and
    // inverse transforms and once for fault injection (runtime direction):
    // the inverse's re/im swaps and the injection selects would otherwise cost
    // predicated moves on every element of every tile
    auto tile_loop = [&](auto dir_c, auto flt_c) {
    constexpr int DIR = decltype(dir_c)::value;  // 0 forward, 1 inverse, 2 a.inverse
    constexpr bool FLT = decltype(flt_c)::value;
    const bool INV = DIR == 2 ? a.inverse != 0 : DIR == 1;
    unsigned iter = 0;
    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++iter) {
        const long long b = tile * S + sl;
        const bool live = b < a.batch;
        const C<T>* src = a.in + b * N;
        C<T>* dst = a.out + b * N;
        const long long valid = (a.batch - tile * S) * N;  // elements of this CTA chunk in range

        // input-side ABFT row e^T W at this thread's positions (the same for
        // every tile: L1 hits), requested before the tile data is waited for
        C<T> ew[TB ? E : 1];
        if constexpr (TB && TFFT_EW_HOIST) {
#pragma unroll
            for (int m = 0; m < E; ++m) ew[m] = EWS ? etw_sm[t + m * TPS] : __ldg(a.etw + t + m * TPS);
        }
        C<T> v[E];
        if constexpr (PF && STG) {
            mbar_wait_s(in_bar_s, iter & 1);
            // contiguous chunk -> padded slices (16-byte reads, 8-byte writes)
            for (int e = threadIdx.x * (16 / (int)sizeof(C<T>)); e < S * N; e += THREADS * (16 / (int)sizeof(C<T>))) {
                if constexpr (sizeof(T) == 4) {
                    const float4 q = reinterpret_cast<const float4*>(ib)[e / 2];
                    sm_all[(e / N) * SL + e % N] = make_float2(q.x, q.y);
                    sm_all[(e / N) * SL + e % N + 1] = make_float2(q.z, q.w);
                } else {
                    sm_all[(e / N) * SL + e % N] = ib[e];
                }
            }
            __syncthreads();  // chunk consumed: refill the buffer
            if (threadIdx.x == 0 && tile + gridDim.x < tiles) {
                fence_proxy_async();
                prefetch(tile + gridDim.x);
            }
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = live ? sm[t + m * TPS] : mk<T>(T(0), T(0));
            __syncthreads();
        } else if constexpr (PFI) {
            mbar_wait_s(in_bar_s, iter & 1);
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = live ? sm_all[sl * N + t + m * TPS] : mk<T>(T(0), T(0));
            __syncthreads();  // linear tile consumed; the exchanges below reuse the buffer
            if constexpr (!MULTIPASS) {
                if (threadIdx.x == 0 && tile + gridDim.x < tiles) {
                    fence_proxy_async();
                    prefetch(tile + gridDim.x);
                }
            }
        } else if constexpr (PP) {
            mbar_wait_s(in_bar_s, iter & 1);
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = live ? ib[sl * SLP + t + m * TPS] : mk<T>(T(0), T(0));
            // refilled after the first exchange barrier (PingPongMem hook)
        } else if constexpr (PF) {
            mbar_wait_s(in_bar_s, iter & 1);
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = live ? ib[sl * SLP + t + m * TPS] : mk<T>(T(0), T(0));
            __syncthreads();  // everyone has the tile in registers: refill the buffer
            if (threadIdx.x < ISSUE && tile + gridDim.x < tiles) {
                fence_proxy_async();
                prefetch(tile + gridDim.x);
            }
        } else if constexpr (STG) {
            stage_in<T, N, S, SL, THREADS>(a.in + tile * S * N, valid, sm_all);
            __syncthreads();
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = live ? sm[t + m * TPS] : mk<T>(T(0), T(0));
            __syncthreads();
        } else if (live) {
#pragma unroll
            for (int m = 0; m < E; ++m) {
                if constexpr (TPS >= 4) v[m] = __ldcs(src + t + m * TPS);
                else v[m] = src[t + m * TPS];
            }
        } else {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = mk<T>(T(0), T(0));
        }

        // ---- left-side input checksum on the pristine values
        // KA independent partial sums per quantity (short dependency chains
        // the scheduler can interleave with the first radix pass), combined
        // pairwise in a fixed order
        constexpr int KA = E >= 16 ? 4 : (E >= 4 ? 2 : 1);
        C<T> cin = mk<T>(T(0), T(0));
        C<T> l1p = mk<T>(T(0), T(0));  // (sum |re|, sum |im|): the l1 upper bound
        if constexpr (TB) {
            C<T> ca[KA], la[KA];
#pragma unroll
            for (int k = 0; k < KA; ++k) ca[k] = la[k] = mk<T>(T(0), T(0));
#pragma unroll
            for (int m = 0; m < E; ++m) {
                if constexpr (!TFFT_EW_HOIST) ew[m] = EWS ? etw_sm[t + m * TPS] : __ldg(a.etw + t + m * TPS);
                if constexpr (!(TFFT_ABLATE & 2)) ca[m % KA] = cmac<T>(ca[m % KA], v[m], ew[m]);
                if constexpr (!(TFFT_ABLATE & 4)) la[m % KA] = cadd<T>(la[m % KA], cabs2<T>(v[m]));
            }
#pragma unroll
            for (int w = KA / 2; w >= 1; w /= 2) {
#pragma unroll
                for (int k = 0; k < w; ++k) {
                    ca[k] = cadd<T>(ca[k], ca[k + w]);
                    la[k] = cadd<T>(la[k], la[k + w]);
                }
            }
            cin = ca[0];
            l1p = la[0];
        }
        int fw = a.f_where, fc = a.f_comp, fb = a.f_bit;
        long long fs = a.f_signal, fe = a.f_elem;
        if (FLT && a.f_table != nullptr && live) {  // batched campaign (never on the product path)
            const long long g = a.sig_base + b, r = g / a.f_div;
            const FaultRec fr = a.f_table[r];
            fw = fr.where; fc = fr.comp; fb = fr.bit;
            fs = r * a.f_div + fr.signal; fe = fr.pos;
        }
        const bool fault_here = FLT && fw != AT_NONE && live && (a.sig_base + b) == fs && (int)(fe % TPS) == t;
        const int fm = (int)(fe / TPS);
        if (fault_here && fw == AT_INPUT) {
#pragma unroll
            for (int m = 0; m < E; ++m) if (m == fm) flip_component<T>(v[m], fc, fb);
        }

        // ---- transform (inverse = swap(FFT(swap(x))) — conjugate symmetry)
        if (INV) {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = swapri<T>(v[m]);
        }
        // thread-level scheme: each thread verifies its radix tiles
        TileCheck<T> tchk;
        tchk.floor2 = fmul(a.abs_floor, a.abs_floor);
        if constexpr (PP) {
            auto refill = [&]() {
                if (threadIdx.x < ISSUE && tile + gridDim.x < tiles) {
                    fence_proxy_async();
                    prefetch(tile + gridDim.x);
                }
            };
            const PingPongMem<T, TPS, PS, decltype(refill)> mem{sm, sm + S * SL, &pp_cur, refill};
            if constexpr (ABFT == ABFT_THREAD) Eng::run(v, mem, t, a.tw, tchk);
            else Eng::run(v, mem, t, a.tw);
        } else if constexpr (PFI && MULTIPASS) {
            // refill the buffer as soon as the last exchange has been read
            auto refill = [&]() {
                if (threadIdx.x == 0 && tile + gridDim.x < tiles) {
                    fence_proxy_async();
                    prefetch(tile + gridDim.x);
                }
            };
            const SliceMemHook<T, TPS, PS, decltype(refill)> mem{{sm}, refill};
            if constexpr (ABFT == ABFT_THREAD) Eng::run(v, mem, t, a.tw, tchk);
            else Eng::run(v, mem, t, a.tw);
        } else if constexpr (SHFL) {
            const ShflSliceMem<T, TPS, PS> mem{{sm}};
            if constexpr (ABFT == ABFT_THREAD) Eng::run(v, mem, t, a.tw, tchk);
            else Eng::run(v, mem, t, a.tw);
        } else {
            const SliceMem<T, TPS, PS> mem{sm};
            if constexpr (ABFT == ABFT_THREAD) Eng::run(v, mem, t, a.tw, tchk);
            else Eng::run(v, mem, t, a.tw);
        }
        if (INV) {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = swapri<T>(v[m]);
        }
        if constexpr (DEFER) {  // the exchanges above contain barriers
            if (p2) stage_decide();
            if (p1) stage_reduce();
        }
        if constexpr (DEFER1) {
            if (pend) finish_pending();
        }
        if (fault_here && fw == AT_PRESCALE) {
#pragma unroll
            for (int m = 0; m < E; ++m) if (m == fm) flip_component<T>(v[m], fc, fb);
        }
        if (DIR != 0 && a.scale_inv) {  // the forward loop runs only unscaled
            const T s = T(1) / T(N);  // exact power of two
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = cscale<T>(v[m], s);
        }
        if (fault_here && fw == AT_OUTPUT) {
#pragma unroll
            for (int m = 0; m < E; ++m) if (m == fm) flip_component<T>(v[m], fc, fb);
        }

        // ---- store + output checksum
        if constexpr (STG) {
#pragma unroll
            for (int m = 0; m < E; ++m) sm[t + m * TPS] = v[m];
            __syncthreads();
            stage_out<T, N, S, SL, THREADS>(a.out + tile * S * N, valid, sm_all);
            __syncthreads();
        } else if (live) {
#pragma unroll
            for (int m = 0; m < E; ++m) {
                if constexpr (TPS >= 4) __stcs(dst + t + m * TPS, v[m]);
                else dst[t + m * TPS] = v[m];
            }
        }
        if constexpr (ABFT == ABFT_THREAD) {
            // worst tile of the signal (max over its threads), one decision
            T w = tchk.worst;
            constexpr int W = TPS < 32 ? TPS : 32;
#pragma unroll
            for (int off = W / 2; off >= 1; off >>= 1) {
                const T o = shfl_xor(w, off);
                w = (o != o || o > w) ? o : w;
            }
            if constexpr (TPS > 32) {
                if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
                __syncthreads();
                if (t == 0) {
                    for (int k = 1; k < TPS / 32; ++k) {
                        const T o = red[(threadIdx.x >> 5) + k];
                        w = (o != o || o > w) ? o : w;
                    }
                }
                __syncthreads();
            }
            bool flagged = false;
            T rel = T(0);
            if (t == 0 && live) {
                rel = (w != w) ? T(INFINITY) : sqrt(w);
                if (!isfinite(rel)) rel = T(INFINITY);
                flagged = rel > a.delta;
                my_maxr = my_maxr > rel ? my_maxr : rel;
                if (a.rel_out) a.rel_out[b] = rel;
            }
            const unsigned ball = __ballot_sync(0xffffffffu, flagged);
            if (ball) {
                const int lane = threadIdx.x & 31;
                int base = 0;
                if (lane == __ffs(ball) - 1) base = atomicAdd(a.flag_count, __popc(ball));
                base = __shfl_sync(0xffffffffu, base, __ffs(ball) - 1);
                if (flagged) {
                    const long long slot = base + __popc(ball & ((1u << lane) - 1u));
                    record_flag(a.flag_rec, a.flag_cap, a.flag_ovf, slot, a.sig_base + b, (double)rel);
                }
            }
        }
        if constexpr (TB) {
            C<T> cout = mk<T>(T(0), T(0));
            if constexpr (ABFT == ABFT_WANG) {
                // e_k = w3^(k mod 3): sum per residue class, then 3 weights.
                // six partial sums for long rows (m mod 6 keeps the class m mod 3)
                constexpr int K6 = E >= 16 ? 6 : 3;
                C<T> acc[K6];
#pragma unroll
                for (int k = 0; k < K6; ++k) acc[k] = mk<T>(T(0), T(0));
#pragma unroll
                for (int m = 0; m < E; ++m)
                    if constexpr (!(TFFT_ABLATE & 8)) acc[m % K6] = cadd<T>(acc[m % K6], v[m]);
                if constexpr (K6 == 6) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) acc[k] = cadd<T>(acc[k], acc[k + 3]);
                }
                constexpr int tau = TPS % 3;  // 1 or 2 (TPS is a power of two)
                const int t0 = t % 3;
                constexpr T hr = T(-0.5), hi = T(0.8660254037844386467637232);
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    if (c >= E) break;
                    const int cls = (t0 + c * tau) % 3;
                    const T wy = cls == 0 ? T(0) : (cls == 1 ? -hi : hi);
                    const T wx = cls == 0 ? T(1) : hr;
                    cout = cadd<T>(cout, cmul<T>(acc[c], mk<T>(wx, wy)));
                }
            } else {
#pragma unroll
                for (int m = 0; m < E; ++m) {
                    const C<T> e = __ldg(a.values + t + m * TPS);
                    cout = cadd<T>(cout, cmul<T>(v[m], e));
                }
            }
            T sums[5] = {cin.x, cin.y, cout.x, cout.y, fadd(l1p.x, l1p.y)};
            if constexpr (DEFER) {
                T* pp = part + ((size_t)(iter & 1) * S + sl) * 5 * PPS + t;
#pragma unroll
                for (int i = 0; i < 5; ++i) pp[i * PPS] = sums[i];
                p1 = !(TFFT_ABLATE & 1);
                p1_live = live;
                p1_b = b;
                p1_par = iter & 1;
            } else if constexpr (DEFER1) {
                if constexpr (!(TFFT_ABLATE & 1)) warp_partials<5>(sums, red + (size_t)(iter & 1) * NW * 5);
                pend = true;
                pend_live = live;
                pend_b = b;
                pend_par = iter & 1;
            } else if constexpr (BATCHD) {
                // every lane of the signal holds the totals after the xor tree;
                // lane t keeps tile (iter mod TPS), and every TPS tiles all lanes
                // decide their kept signal at once (TPS x fewer decision passes)
                if constexpr (!(TFFT_ABLATE & 1)) sig_sum<TPS>(sums, red, t);
                if ((int)(iter & (TPS - 1)) == t) {
#pragma unroll
                    for (int i = 0; i < 5; ++i) keep[i] = sums[i];
                    keep_b = b;
                    keep_v = live;
                }
                if ((int)(iter & (TPS - 1)) == TPS - 1) {
                    decide_signal(keep, keep_b, keep_v);
                    keep_v = false;
                }
            } else {
                if constexpr (!(TFFT_ABLATE & 1)) sig_sum<TPS>(sums, red, t);
                decide_signal(sums, b, t == 0 && live);
            }
        }
    }
    };
    if (ONE_LOOP || a.f_where != AT_NONE || a.f_table != nullptr || (a.scale_inv && !a.inverse))
        tile_loop(IntC<2>{}, BoolC<true>{});
    else if (a.inverse) tile_loop(IntC<1>{}, BoolC<false>{});
    else tile_loop(IntC<0>{}, BoolC<false>{});
    if constexpr (DEFER1) {
        if (pend) {
            __syncthreads();
            finish_pending();
        }
    }
    if constexpr (BATCHD) decide_signal(keep, keep_b, keep_v);  // the last partial batch
    if constexpr (DEFER) {  // drain the pipeline (uniform across the CTA)
        if (p1 || p2) {
            __syncthreads();
            if (p2) stage_decide();
            if (p1) {
                stage_reduce();
                __syncthreads();
                stage_decide();
            }
        }
    }
    if constexpr (ABFT != ABFT_OFF) {
        // one atomic per CTA for the running max discrepancy
        const T mr = sqrt(my_max);
        typename KeyT<T>::type k = order_key(my_maxr > mr ? my_maxr : mr);
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            typename KeyT<T>::type o = __shfl_xor_sync(0xffffffffu, k, off);
            k = o > k ? o : k;
        }
        __syncthreads();
        if ((threadIdx.x & 31) == 0 && k) atomicMax(&cta_max, k);
        __syncthreads();
        if (threadIdx.x == 0 && cta_max) atomicMax(a.max_key, cta_max);
    }
    (void)NW;
}

}  // namespace tfft
