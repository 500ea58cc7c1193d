// Multi-launch tiled FFT for N > 2^13 (reference stages 2-3,
// fft_core/execute.py:82-106 and planner.py:82-97), with the ABFT checksums
// carried across launches as per-tile partial sums.
//
// Every launch is one "pass" = one reference stage: a batch of L-point
// transforms (L = stage dim) addressed through
//     in (u, j) = hi*in_hi  + lo*in_lo  + j*in_j       u = hi*lo_count + lo
//     out(u, k) = hi*out_hi + lo*out_lo + k*out_k
// A CTA owns U consecutive transforms u (a "tile") of one signal, lanes run
// along u, so every global row segment is U*sizeof(complex) contiguous bytes.
//   kind 0 (first stage): strided columns c of the (d0 x rest) view, post
//          twiddle w_N^{c k}; stores back in place (no transpose copy — the
//          reference's ascontiguousarray transposes disappear into the
//          address maps); accumulates c_in = x.(e^T W) and the l1 mass per
//          tile from the pristine input;
//   kind 1 (3-stage middle): columns c2 inside each k0 block, twiddle
//          w_{d1 d2}^{c2 k};
//   kind 2 (last stage): contiguous rows staged through shared memory,
//          stores an (N1 x N3) plane per CTA — consecutive k0 lanes write
//          consecutive output addresses f = k0 + d0*(k1 + d1*k) — and
//          accumulates c_out = y.e per tile.
// A finalize kernel reduces the tile partials per signal in a fixed order and
// takes the detection decision (reference abft/pipeline.py:104-135).
#pragma once
#include <cuda.h>  // CUtensorMap (TMA descriptor; encoded on the host per launch)

#include "single.cuh"

namespace tfft {

enum { KIND_FIRST = 0, KIND_MID = 1, KIND_LAST = 2 };

template <class T>
struct alignas(64) PassArgs {
    CUtensorMap tmap;                 // PF >= 3: strided input rows as a 3-D tensor
    CUtensorMap tmap_etw;             // PF == 4, first pass with ABFT: the e^T W row, same geometry
    const C<T>* in;
    C<T>* out;
    long long batch, sig_base, n;
    long long lo_count, in_hi, in_lo, in_j, out_hi, out_lo, out_k;
    long long tiles_per_sig;          // units / U
    const C<T>* twL;                  // w_L^k, k < L
    const C<T>* ptw_lo;               // post twiddle w_M^e = hi[e >> s] * lo[e & mask]
    const C<T>* ptw_hi;
    int ptw_shift;
    long long ptw_mask, M;            // M - 1 == mask for e reduction
    const C<T>* etw;                  // kind 0 ABFT row
    const C<T>* values;               // kind 2 table encoding
    T* part;                          // tile partials (3 or 2 T per tile)
    int inverse, scale_inv;
    T scale;
    long long f_signal, f_unit;
    int f_idx, f_where, f_comp, f_bit;  // f_where: 1 after load, 2 store pre-scale, 3 post-scale
    const FaultRec* f_table;          // batched campaign: this pass's fault per f_div signals
    long long f_div;
};

// element-granular async global->shared copy (SASS LDGSTS)
template <int BYTES>
__device__ __forceinline__ void cp_async(void* dst, const void* src) {
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(BYTES)
                     : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// PF = 1: the CTA prefetches tile i+1 into the second half of a ping-pong
// smem buffer with cp.async while tile i is transformed (the engine's
// exchanges run in tile i's half), so HBM latency overlaps compute even at
// one or two CTAs per SM.
// 3-D tensor TMA load (SASS UTMALDG) of one box into shared memory
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

#ifndef TFFT_ETW_CF
#define TFFT_ETW_CF 1  // Wang first pass: closed-form e^T W in registers (0: the n-element table)
#endif

// Closed form of the Wang input-side row (checked against the
// table path in tests/test_gpu_etw.py):
//   etw[n]     = (A / 2) (1 - i cot(pi k_n / (3N))),  k_n = (N + 3n) mod 3N,
//   etw_inv[n] = (A / 2N)(1 - i cot(pi k_n / (3N))),  k_n = (N - 3n) mod 3N,
// A = 1 - w3^N, k reduced to (-1.5N, 1.5N] (cot has period pi). In the first
// pass element (column lo, row j) has n = lo + j N/L, i.e. angle
// alpha_lo +- j pi / L: one exactly reduced cot per column and tile
// (sincospi in double, by U threads, shared through smem), a per-launch smem
// table of cot(j pi / L), and the addition formula
// cot(a + b) = (cot a cot b - 1) / (cot a + cot b) per element. The formula
// loses accuracy only near the pole of the sum; elements within 1/256 rad of
// it (|k| < 3N / (256 pi), integer test) use the Laurent series of cot at 0
// on the exactly reduced angle. Nothing is read from HBM.
template <class T>
__device__ __forceinline__ T fast_rcp(T d);
template <>
__device__ __forceinline__ float fast_rcp<float>(float d) { return __fdividef(1.0f, d); }
template <>
__device__ __forceinline__ double fast_rcp<double>(double d) {
    double r = (double)__fdividef(1.0f, (float)d);  // |d| in [4e-3, 1e8]: a normal float
    double e = __fma_rn(-d, r, 1.0);
    r = __fma_rn(r, e, r);
    e = __fma_rn(-d, r, 1.0);
    return __fma_rn(r, e, r);  // two Newton steps: ~1e-16 relative
}
// k of column lo (exact, in (-1.5N, 1.5N]) and cot(pi k / 3N)
template <class T>
__device__ __forceinline__ void wang_col_base(long long lo, int N, bool inv, int& k, T& c) {
    const int N3 = 3 * N, H = N3 / 2;
    int kk = inv ? N - 3 * (int)lo : N + 3 * (int)lo;  // lo < N: one wrap at most
    if (kk > H) kk -= N3;
    else if (kk <= -H) kk += N3;
    double sb, cb;
    sincospi((double)kk / (double)N3, &sb, &cb);
    k = kk;
    c = (T)(cb / sb);  // k != 0: N is not a multiple of 3
}
// Laurent series of cot at 0: for the one element per thread that lies within
// 1/256 rad of the pole (|k| < 3N / (256 pi))
template <class T>
__device__ __forceinline__ T cot_near_pole(int k, int N3) {
    const T d = (T)k * (T)(3.14159265358979323846 / (double)N3);
    const T d2 = d * d;
    return fast_rcp<T>(d) - d * (T(1) / T(3) + d2 * (T(1) / T(45) + d2 * (T(2) / T(945))));
}

// Engine memory policy of a pass tile: [L][U] rows of stride RS, lane u.
template <class T, int RS>
struct RowMem {
    static constexpr int kPS = 0;
    static constexpr bool kShuffle = false;
    C<T>* base;
    int u;
    __device__ __forceinline__ void putp(int i, C<T> v) const { base[i * RS + u] = v; }
    __device__ __forceinline__ C<T> getp(int i) const { return base[i * RS + u]; }
    __device__ __forceinline__ void sync() const { __syncthreads(); }
    __device__ __forceinline__ void release() const { __syncthreads(); }
    __device__ __forceinline__ void after_last_exchange() const {}
};

template <class T, int L, int E, int U, int P, int KIND, int ABFT, int MINB, int PF, class Radices>
__global__ void __launch_bounds__(U * (L / E), MINB)
fft_pass_kernel(const __grid_constant__ PassArgs<T> a) {
    constexpr int TPS = L / E;
    constexpr int THREADS = U * TPS;
    constexpr int RS = U + P;  // smem row stride (elements) of the [L][U] tile
    // PF = 2: per-row TMA bulk copies (cp.async.bulk, one instruction per row
    // segment, no per-element issue work) into a dense staging layout, two
    // buffers on two mbarriers. Rows of the last kind land at a padded stride.
    // PF = 3: like 2, but the strided kinds load whole [U x 256] boxes with one
    // tensor-TMA instruction each (thread 0), the last kind keeps bulk rows.
    // PF = 4: like 3, and the first pass with ABFT also brings its e^T W tile
    // with tensor TMA (same box geometry, batch 1) into a parallel buffer
    // instead of one L2 round trip of per-element loads.
    constexpr bool BULK = PF == 2 || PF == 3 || PF == 4;
    constexpr bool TENSOR = (PF == 3 || PF == 4) && KIND != KIND_LAST;
    constexpr bool CF = KIND == KIND_FIRST && ABFT == ABFT_WANG && TFFT_ETW_CF;  // closed-form row
    constexpr bool ETW_TMA = PF == 4 && KIND == KIND_FIRST && ABFT != ABFT_OFF && !CF;
    constexpr int BOXR = L < 256 ? L : 256;
    constexpr int SU = sizeof(T) == 4 ? L + 2 : L + 1;  // 16-byte aligned padded row
    // buffer size rounded to 16 elements so the second buffer stays 128-byte
    // aligned (tensor-TMA destination requirement)
    constexpr int BUFE = ((BULK ? (L * RS > U * SU ? L * RS : U * SU) : L * RS) + 15) / 16 * 16;
    constexpr int ISSUERS = KIND == KIND_LAST ? U : (TENSOR ? 1 : (L < THREADS ? L : THREADS));
    using Eng = Engine<T, L, E, Radices>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int ETWE = PF == 4 ? (L * U + 15) / 16 * 16 : 0;  // e^T W tile (elements)
    C<T>* tile = reinterpret_cast<C<T>*>(smem_raw);
    C<T>* etile = tile + (PF ? 2 : 1) * BUFE;                   // 2 x ETWE
    T* red = reinterpret_cast<T*>(etile + 2 * ETWE);
    __shared__ unsigned long long bbar[2];
    // closed-form row: cot(+-j pi / L) per launch, column bases per tile (parity buffered)
    __shared__ T cf_cj[CF ? L : 1];
    __shared__ T cf_cc[CF ? 2 * U : 1];
    __shared__ int cf_kc[CF ? 2 * U : 1];

    const int u = threadIdx.x % U;
    const int t = threadIdx.x / U;
    const long long total = a.batch * a.tiles_per_sig;

    using Mem = RowMem<T, RS>;

    // Tile order. The first pass with ABFT walks tile-position-major (all
    // signals' tile i, then tile i+1, ...) so concurrent CTAs read the same
    // e^T W slice: the input-side table (n elements, up to 512 MB) is then
    // fetched from HBM about once per launch instead of once per signal.
    constexpr bool POS_MAJOR = KIND == KIND_FIRST && ABFT != ABFT_OFF;
    auto tile_of = [&](long long tx, long long& bb, long long& ts) {
        if constexpr (POS_MAJOR) {
            ts = tx / a.batch;
            bb = tx - ts * a.batch;
        } else {
            bb = tx / a.tiles_per_sig;
            ts = tx - bb * a.tiles_per_sig;
        }
    };
    // async copy of tile `tx` into `buf` as [j][u] rows of stride RS
    auto issue = [&](long long tx, C<T>* buf) {
        long long bb, ts;
        tile_of(tx, bb, ts);
        const long long v0 = ts * U;
        const long long h0 = v0 / a.lo_count, l0 = v0 - h0 * a.lo_count;
        const C<T>* sb = a.in + bb * a.n + h0 * a.in_hi + l0 * a.in_lo;
        if constexpr (KIND == KIND_LAST) {  // U contiguous rows of L: j fastest
            for (int f = threadIdx.x; f < U * L; f += THREADS) {
                const int r = f / L, j = f % L;
                cp_async<sizeof(C<T>)>(buf + j * RS + r, sb + (long long)r * a.in_lo + j);
            }
        } else {  // L strided rows of U contiguous elements: u fastest
            for (int f = threadIdx.x; f < U * L; f += THREADS) {
                const int r = f % U, j = f / U;
                cp_async<sizeof(C<T>)>(buf + j * RS + r, sb + r * a.in_lo + (long long)j * a.in_j);
            }
        }
    };
    // bulk variant: the ISSUERS threads each arrive with their byte count
    auto issue_bulk = [&](long long tx, C<T>* buf, C<T>* ebuf, unsigned long long* bar) {
        if (threadIdx.x >= ISSUERS) return;
        long long bb, ts;
        tile_of(tx, bb, ts);
        const long long v0 = ts * U;
        const long long h0 = v0 / a.lo_count, l0 = v0 - h0 * a.lo_count;
        const C<T>* sb = a.in + bb * a.n + h0 * a.in_hi + l0 * a.in_lo;
        fence_proxy_async();
        if constexpr (TENSOR) {  // boxes of [U contiguous x BOXR strided rows]
            constexpr int CW = sizeof(C<T>) / 4;  // 32-bit words per element
            mbar_expect_tx(bar, (ETW_TMA ? 2 : 1) * L * U * sizeof(C<T>));
            const int c2 = KIND == KIND_FIRST ? (int)bb : (int)(bb * (a.n / a.in_hi) + h0);
#pragma unroll
            for (int k = 0; k < L / BOXR; ++k)
                tma_load_3d(buf + k * BOXR * U, &a.tmap, (int)(l0 * CW), k * BOXR, c2, bar);
            if constexpr (ETW_TMA) {
#pragma unroll
                for (int k = 0; k < L / BOXR; ++k)
                    tma_load_3d(ebuf + k * BOXR * U, &a.tmap_etw, (int)(l0 * CW), k * BOXR, 0, bar);
            }
        } else if constexpr (KIND == KIND_LAST) {  // row u: L contiguous elements
            const unsigned bytes = L * sizeof(C<T>);
            mbar_expect_tx(bar, bytes);
            bulk_g2s(buf + threadIdx.x * SU, sb + (long long)threadIdx.x * a.in_lo, bytes, bar);
        } else {  // rows j: U contiguous elements each, dense [j][U]
            constexpr int RPI = L / ISSUERS;
            mbar_expect_tx(bar, RPI * U * sizeof(C<T>));
#pragma unroll
            for (int k = 0; k < RPI; ++k) {
                const int j = threadIdx.x + k * ISSUERS;
                bulk_g2s(buf + j * U, sb + (long long)j * a.in_j, U * sizeof(C<T>), bar);
            }
        }
    };
    if constexpr (BULK) {
        if (threadIdx.x == 0) {
            mbar_init(&bbar[0], ISSUERS);
            mbar_init(&bbar[1], ISSUERS);
        }
        __syncthreads();
        if (blockIdx.x < total) issue_bulk(blockIdx.x, tile, etile, &bbar[0]);
    } else if constexpr (PF) {
        if (blockIdx.x < total) issue(blockIdx.x, tile);
        cp_async_commit();
    }

    const unsigned bbar_s = smem_u32(&bbar[0]);  // shared-window address, converted once
    // closed-form row: column bases of tile tx (threads u < U, i.e. t == 0)
    const int cf_n = (int)a.n;
    const int cf_kap = (int)((double)(3 * cf_n) * (1.0 / (256.0 * 3.14159265358979323846))) + 1;
    auto cf_col_base = [&](long long tx, unsigned par) {
        long long bb, ts;
        tile_of(tx, bb, ts);
        int k;
        T c;
        wang_col_base<T>(ts * U + threadIdx.x, cf_n, a.inverse != 0, k, c);
        cf_kc[par * U + threadIdx.x] = k;
        cf_cc[par * U + threadIdx.x] = c;
    };
    if constexpr (CF) {
        const double sg = a.inverse ? -1.0 : 1.0;
        for (int j = threadIdx.x; j < L; j += THREADS) {
            double sj, cj;
            sincospi((double)j / (double)L, &sj, &cj);
            cf_cj[j] = j ? (T)(sg * cj / sj) : T(0);
        }
        if (threadIdx.x < U && blockIdx.x < total) cf_col_base(blockIdx.x, 0);
        __syncthreads();
    }
    // the tile loop, instantiated per direction and once for fault injection
    // (as in single.cuh): no per-element predicated swaps / injection selects
    auto tile_loop = [&](auto dir_c, auto flt_c) {
    constexpr int DIR = decltype(dir_c)::value;  // 0 forward, 1 inverse, 2 a.inverse
    constexpr bool FLT = decltype(flt_c)::value;
    const bool INV = DIR == 2 ? a.inverse != 0 : DIR == 1;
    unsigned it = 0;
    for (long long tix = blockIdx.x; tix < total; tix += gridDim.x, ++it) {
        C<T>* cur = (PF && (it & 1)) ? tile + BUFE : tile;
        const Mem mem{cur, u};
        long long b, tsig;
        tile_of(tix, b, tsig);
        const long long u0 = tsig * U;               // first unit of the tile
        const long long uu = u0 + u;
        const long long hi = uu / a.lo_count, lo = uu - hi * a.lo_count;
        const C<T>* src = a.in + b * a.n;
        C<T>* dst = a.out + b * a.n;
        const long long ibase = hi * a.in_hi + lo * a.in_lo;
        const long long obase = hi * a.out_hi + lo * a.out_lo;
        int fw = a.f_where, fc = a.f_comp, fb = a.f_bit, fi = a.f_idx;
        long long fs = a.f_signal, fu = a.f_unit;
        if (FLT && a.f_table != nullptr) {  // batched campaign (never on the product path)
            const long long g = a.sig_base + b, r = g / a.f_div;
            const FaultRec fr = a.f_table[r];
            fw = fr.where; fc = fr.comp; fb = fr.bit; fi = fr.idx;
            fs = r * a.f_div + fr.signal; fu = fr.pos;
        }
        const bool fsig = FLT && fw != 0 && (a.sig_base + b) == fs && uu == fu && (fi % TPS) == t;
        const int fm = fi / TPS;

        // input-side ABFT row e^T W for this tile, requested before the tile
        // data is waited for so its latency overlaps (one batch of
        // independent loads, not one round trip per element)
        C<T> ew[(KIND == KIND_FIRST && ABFT != ABFT_OFF && !CF) ? E : 1];
        T ct[CF ? E : 1];
        if constexpr (CF) {
            const unsigned par = it & 1;
            const T cc = cf_cc[par * U + u];
            // this thread's rows j = t + m TPS are pi/E apart in angle: at most
            // one of them (m*) can lie within 1/256 rad of the pole; find it with
            // integer arithmetic and patch it after the addition formula
            const int N3 = 3 * cf_n, H = N3 / 2;
            const int dk = (INV ? -3 : 3) * (int)a.in_j;  // +-3 N / L per row
            int kt = cf_kc[par * U + u] + dk * t;
            if (kt > H) kt -= N3;
            else if (kt <= -H) kt += N3;
            const int dm = dk * TPS;  // +-3N / E per element
            int ms = (int)llrint(-(double)kt / (double)dm);
            ms = ((ms % E) + E) % E;
            int km = kt + dm * ms;
            if (km > H) km -= N3;
            else if (km <= -H) km += N3;
            const bool pole = km < cf_kap && km > -cf_kap && (t + ms * TPS) != 0;
            const T cp = pole ? cot_near_pole<T>(km, N3) : T(0);
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int j = t + m * TPS;
                const T cj = cf_cj[j];
                T cm = (cc * cj - T(1)) * fast_rcp<T>(cc + cj);
                if (m == 0) cm = t == 0 ? cc : cm;
                ct[m] = (pole && m == ms) ? cp : cm;
            }
            // the next tile's column bases (its readers run after this tile's trailing barrier)
            if (threadIdx.x < U && tix + gridDim.x < total) cf_col_base(tix + gridDim.x, par ^ 1u);
        } else if constexpr (KIND == KIND_FIRST && ABFT != ABFT_OFF && !ETW_TMA) {
            const C<T>* ep = a.etw + ibase + (long long)t * a.in_j;
            const long long es = (long long)TPS * a.in_j;
#pragma unroll
            for (int m = 0; m < E; ++m) {
                if constexpr (TFFT_ABLATE & 16) ew[m] = mk<T>(T(1), T(0));  // cost attribution only
                else ew[m] = __ldg(ep + m * es);
            }
        }
        C<T> v[E];
        if constexpr (BULK) {
            if (tix + gridDim.x < total)
                issue_bulk(tix + gridDim.x, (it & 1) ? tile : tile + BUFE, (it & 1) ? etile : etile + ETWE,
                           &bbar[(it + 1) & 1]);
            mbar_wait_s(bbar_s + 8u * (it & 1), (it >> 1) & 1);
            if constexpr (KIND == KIND_LAST) {
#pragma unroll
                for (int m = 0; m < E; ++m) v[m] = cur[u * SU + t + m * TPS];
            } else {
#pragma unroll
                for (int m = 0; m < E; ++m) v[m] = cur[(t + m * TPS) * U + u];
            }
            if constexpr (ETW_TMA) {
                const C<T>* ecur = (it & 1) ? etile + ETWE : etile;
#pragma unroll
                for (int m = 0; m < E; ++m) ew[m] = ecur[(t + m * TPS) * U + u];
            }
            __syncthreads();
        } else if constexpr (PF) {
            if (tix + gridDim.x < total) issue(tix + gridDim.x, (it & 1) ? tile : tile + BUFE);
            cp_async_commit();
            cp_async_wait<1>();  // this tile's group has landed
            __syncthreads();
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = cur[(t + m * TPS) * RS + u];
            __syncthreads();
        } else if constexpr (KIND == KIND_LAST) {
            // rows are contiguous: stage the U x L tile through smem with
            // j-fastest (fully coalesced) loads.
            const long long hi0 = u0 / a.lo_count, lo0 = u0 - hi0 * a.lo_count;
            const long long rbase0 = hi0 * a.in_hi + lo0 * a.in_lo;
#pragma unroll 4
            for (int f = threadIdx.x; f < U * L; f += THREADS) {
                const int r = f / L, j = f % L;
                tile[j * RS + r] = __ldcs(src + rbase0 + (long long)r * a.in_lo + j);
            }
            __syncthreads();
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = tile[(t + m * TPS) * RS + u];
            __syncthreads();
        } else {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = __ldcs(src + ibase + (long long)(t + m * TPS) * a.in_j);
        }

        if constexpr (KIND == KIND_FIRST && ABFT != ABFT_OFF) {
            // KA independent partial sums (short chains), combined pairwise
            constexpr int KA = E >= 16 ? 4 : (E >= 4 ? 2 : 1);
            C<T> ca[KA], la[KA];  // la: l1 upper bound sum(|re| + |im|), see abft_decide
#pragma unroll
            for (int k = 0; k < KA; ++k) ca[k] = la[k] = mk<T>(T(0), T(0));
            C<T> sa[CF ? KA : 1];  // closed form: ca = sum x, sa = sum x cot
            if constexpr (CF) {
#pragma unroll
                for (int k = 0; k < KA; ++k) sa[k] = mk<T>(T(0), T(0));
            }
#pragma unroll
            for (int m = 0; m < E; ++m) {
                if constexpr (CF) {
                    ca[m % KA] = cadd<T>(ca[m % KA], v[m]);
                    sa[m % KA] = mk<T>(ffma(v[m].x, ct[m], sa[m % KA].x), ffma(v[m].y, ct[m], sa[m % KA].y));
                } else {
                    ca[m % KA] = cmac<T>(ca[m % KA], v[m], ew[m]);
                }
                la[m % KA] = cadd<T>(la[m % KA], cabs2<T>(v[m]));
            }
#pragma unroll
            for (int w = KA / 2; w >= 1; w /= 2) {
#pragma unroll
                for (int k = 0; k < w; ++k) {
                    ca[k] = cadd<T>(ca[k], ca[k + w]);
                    la[k] = cadd<T>(la[k], la[k + w]);
                    if constexpr (CF) sa[k] = cadd<T>(sa[k], sa[k + w]);
                }
            }
            C<T> cin = ca[0];
            if constexpr (CF) {
                // x . etw = (A / 2)(S0 - i S1), S0 = sum x, S1 = sum x cot; A = 1 - w3^N
                // = (1.5, +-sqrt(3)/2) for N = 1 / 2 (mod 3); inverse: also / N
                const T hs = T(0.8660254037844386467637232) * ((a.n % 3 == 1) ? T(1) : T(-1));
                const T g = INV ? T(0.5) / T(a.n) : T(0.5);
                const C<T> u = mk<T>(fadd(ca[0].x, sa[0].y), fsub(ca[0].y, sa[0].x));
                cin = cmul<T>(u, mk<T>(T(1.5) * g, hs * g));
            }
            const C<T> l1p = la[0];
            T s[3] = {cin.x, cin.y, fadd(l1p.x, l1p.y)};
            warp_partials<3>(s, red);  // summed by thread 0 after the tile's trailing barrier
        }
        if (fsig && fw == 1) {
#pragma unroll
            for (int m = 0; m < E; ++m) if (m == fm) flip_component<T>(v[m], fc, fb);
        }

        if (INV) {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = swapri<T>(v[m]);
        }
        Eng::run(v, mem, t, a.twL);
        if constexpr (KIND != KIND_LAST) {
            // post twiddle w_M^{c k} with c = lo (column), k = t + m*TPS:
            // base w^{c t} and step w^{c TPS} from the two-level table (4
            // loads per thread), powers of the step by binary splitting.
            const long long lmask = (1ll << a.ptw_shift) - 1;
            const long long e0 = (lo * (long long)t) & a.ptw_mask;
            const long long es = (lo * (long long)TPS) & a.ptw_mask;
            const C<T> base = cmul<T>(__ldg(a.ptw_hi + (e0 >> a.ptw_shift)), __ldg(a.ptw_lo + (e0 & lmask)));
            C<T> st[E];
            st[0] = mk<T>(T(1), T(0));
            if constexpr (E > 1) st[1] = cmul<T>(__ldg(a.ptw_hi + (es >> a.ptw_shift)), __ldg(a.ptw_lo + (es & lmask)));
#pragma unroll
            for (int m = 2; m < E; ++m) st[m] = cmul<T>(st[m / 2], st[m - m / 2]);
            v[0] = cmul<T>(v[0], base);
#pragma unroll
            for (int m = 1; m < E; ++m) v[m] = cmul<T>(v[m], cmul<T>(base, st[m]));
        }
        if (INV) {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = swapri<T>(v[m]);
        }
        if (fsig && fw == 2) {
#pragma unroll
            for (int m = 0; m < E; ++m) if (m == fm) flip_component<T>(v[m], fc, fb);
        }
        if constexpr (KIND == KIND_LAST) {
            if (DIR != 0 && a.scale_inv) {  // the forward loop runs only unscaled
#pragma unroll
                for (int m = 0; m < E; ++m) v[m] = cscale<T>(v[m], a.scale);
            }
            if (fsig && fw == 3) {
#pragma unroll
                for (int m = 0; m < E; ++m) if (m == fm) flip_component<T>(v[m], fc, fb);
            }
        }
#pragma unroll
        for (int m = 0; m < E; ++m) __stcs(dst + obase + (long long)(t + m * TPS) * a.out_k, v[m]);

        if constexpr (KIND == KIND_LAST && ABFT != ABFT_OFF) {
            C<T> cout = mk<T>(T(0), T(0));
            if constexpr (ABFT == ABFT_TABLE) {
#pragma unroll
                for (int m = 0; m < E; ++m)
                    cout = cadd<T>(cout, cmul<T>(v[m], __ldg(a.values + obase + (long long)(t + m * TPS) * a.out_k)));
            } else {
                // Wang weights w3^(f mod 3) of output index f = obase + (t + m TPS) out_k:
                // class(m) = (c0 + m*sc) mod 3 with one 64-bit residue per tile, so
                // elements are summed per class (one packed add each) and weighted
                // three times at the end
                const int c0 = (int)((obase + (long long)t * a.out_k) % 3);
                const int sc = (int)(((long long)TPS * a.out_k) % 3);
                C<T> acc[3] = {mk<T>(T(0), T(0)), mk<T>(T(0), T(0)), mk<T>(T(0), T(0))};
                if (sc == 1) {
#pragma unroll
                    for (int m = 0; m < E; ++m) acc[m % 3] = cadd<T>(acc[m % 3], v[m]);
                } else if (sc == 2) {
#pragma unroll
                    for (int m = 0; m < E; ++m) acc[(2 * m) % 3] = cadd<T>(acc[(2 * m) % 3], v[m]);
                } else {
#pragma unroll
                    for (int m = 0; m < E; ++m) acc[0] = cadd<T>(acc[0], v[m]);
                }
                const T hr = T(-0.5), hq = T(0.8660254037844386467637232);
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                    const int cls = (c0 + r) % 3;  // acc[r] holds class (c0 + r) mod 3
                    const C<T> w = cls == 0 ? mk<T>(T(1), T(0)) : (cls == 1 ? mk<T>(hr, -hq) : mk<T>(hr, hq));
                    cout = cadd<T>(cout, cmul<T>(acc[r], w));
                }
            }
            T s[2] = {cout.x, cout.y};
            warp_partials<2>(s, red);
        }
        __syncthreads();  // smem tile reused by the next iteration; warp partials visible
        if constexpr (ABFT != ABFT_OFF && KIND != KIND_MID) {
            // the tile's checksum partial (3 values in, 2 out), fixed warp order;
            // `red` is rewritten only after the next tile's barriers
            constexpr int K = KIND == KIND_FIRST ? 3 : 2;
            if (threadIdx.x == 0) {
                T* p = a.part + (b * a.tiles_per_sig + tsig) * K;
#pragma unroll
                for (int i = 0; i < K; ++i) {
                    T acc = red[i];
                    for (int w = 1; w < THREADS / 32; ++w) acc = fadd(acc, red[w * K + i]);
                    p[i] = acc;
                }
            }
        }
    }
    };
    if (TFFT_ONE_LOOP_ALL || a.f_where != 0 || a.f_table != nullptr || (a.scale_inv && !a.inverse))
        tile_loop(IntC<2>{}, BoolC<true>{});
    else if (a.inverse) tile_loop(IntC<1>{}, BoolC<false>{});
    else tile_loop(IntC<0>{}, BoolC<false>{});
}

// Per-signal reduction of the tile partials and the detection decision.
template <class T>
struct FinalArgs {
    long long batch, sig_base;
    const T* part_in;  long long tiles_in;
    const T* part_out; long long tiles_out;
    T delta, abs_floor, floor_coef;
    int* flag_count;
    FlagRec* flag_rec;
    long long flag_cap;
    unsigned* flag_ovf;
    typename KeyT<T>::type* max_key;
    T* rel_out;  // optional per-signal relative discrepancy
};

template <class T>
__global__ void __launch_bounds__(256) abft_finalize_kernel(const FinalArgs<T> a) {
    __shared__ typename KeyT<T>::type cta_max;
    if (threadIdx.x == 0) cta_max = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x / 32);
    T my_max = T(0);
    for (long long b = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); b < a.batch; b += warps) {
        T ci_x = 0, ci_y = 0, l1 = 0, co_x = 0, co_y = 0;
        for (long long i = lane; i < a.tiles_in; i += 32) {
            const T* p = a.part_in + (b * a.tiles_in + i) * 3;
            ci_x = fadd(ci_x, p[0]); ci_y = fadd(ci_y, p[1]); l1 = fadd(l1, p[2]);
        }
        for (long long i = lane; i < a.tiles_out; i += 32) {
            const T* p = a.part_out + (b * a.tiles_out + i) * 2;
            co_x = fadd(co_x, p[0]); co_y = fadd(co_y, p[1]);
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            ci_x = fadd(ci_x, shfl_xor(ci_x, off)); ci_y = fadd(ci_y, shfl_xor(ci_y, off));
            l1 = fadd(l1, shfl_xor(l1, off));
            co_x = fadd(co_x, shfl_xor(co_x, off)); co_y = fadd(co_y, shfl_xor(co_y, off));
        }
        if (lane == 0) {
            T rel, rel2;
            bool flagged, recheck;
            abft_decide<T>(ci_x, ci_y, co_x, co_y, l1, a.delta, a.abs_floor, a.floor_coef, true, rel, rel2,
                           flagged, recheck);
            if (recheck) rel = T(-1);  // sentinel: the host recomputes it exactly
            else my_max = my_max > rel ? my_max : rel;
            if (a.rel_out) a.rel_out[b] = rel;
            if (flagged || recheck) {
                const int slot = atomicAdd(a.flag_count, 1);
                record_flag(a.flag_rec, a.flag_cap, a.flag_ovf, slot, a.sig_base + b, (double)rel);
            }
        }
    }
    if (lane == 0 && my_max > T(0)) atomicMax(&cta_max, order_key(my_max));
    __syncthreads();
    if (threadIdx.x == 0 && cta_max) atomicMax(a.max_key, cta_max);
}

// Same decision with a whole CTA per signal, for few signals with many tiles
// (2^23..2^25: 2-8 signals x 8k-130k tiles, where a warp per signal
// serialised on load latency for ~0.1 ms). Four independent accumulator sets
// per thread keep loads in flight; fixed combination order (deterministic).
template <class T>
__global__ void __launch_bounds__(256) abft_finalize_cta_kernel(const FinalArgs<T> a) {
    __shared__ T sh[8][5];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T my_max = T(0);
    for (long long b = blockIdx.x; b < a.batch; b += gridDim.x) {
        T acc[4][5];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int k = 0; k < 5; ++k) acc[u][k] = T(0);
        const T* pin = a.part_in + b * a.tiles_in * 3;
        long long i = threadIdx.x;
        for (; i + 3 * 256 < a.tiles_in; i += 4 * 256) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const T* p = pin + (i + u * 256) * 3;
                acc[u][0] = fadd(acc[u][0], p[0]); acc[u][1] = fadd(acc[u][1], p[1]); acc[u][2] = fadd(acc[u][2], p[2]);
            }
        }
        for (; i < a.tiles_in; i += 256) {
            const T* p = pin + i * 3;
            acc[0][0] = fadd(acc[0][0], p[0]); acc[0][1] = fadd(acc[0][1], p[1]); acc[0][2] = fadd(acc[0][2], p[2]);
        }
        const T* pout = a.part_out + b * a.tiles_out * 2;
        i = threadIdx.x;
        for (; i + 3 * 256 < a.tiles_out; i += 4 * 256) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const T* p = pout + (i + u * 256) * 2;
                acc[u][3] = fadd(acc[u][3], p[0]); acc[u][4] = fadd(acc[u][4], p[1]);
            }
        }
        for (; i < a.tiles_out; i += 256) {
            const T* p = pout + i * 2;
            acc[0][3] = fadd(acc[0][3], p[0]); acc[0][4] = fadd(acc[0][4], p[1]);
        }
        T v[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            v[k] = fadd(fadd(acc[0][k], acc[1][k]), fadd(acc[2][k], acc[3][k]));
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) v[k] = fadd(v[k], shfl_xor(v[k], off));
        }
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < 5; ++k) sh[warp][k] = v[k];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            T t5[5];
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                t5[k] = sh[0][k];
                for (int w = 1; w < 8; ++w) t5[k] = fadd(t5[k], sh[w][k]);
            }
            T rel, rel2;
            bool flagged, recheck;
            abft_decide<T>(t5[0], t5[1], t5[3], t5[4], t5[2], a.delta, a.abs_floor, a.floor_coef, true, rel, rel2,
                           flagged, recheck);
            if (recheck) rel = T(-1);
            else my_max = my_max > rel ? my_max : rel;
            if (a.rel_out) a.rel_out[b] = rel;
            if (flagged || recheck) {
                const int slot = atomicAdd(a.flag_count, 1);
                record_flag(a.flag_rec, a.flag_cap, a.flag_ovf, slot, a.sig_base + b, (double)rel);
            }
        }
        __syncthreads();  // sh reused by the next signal
    }
    if (threadIdx.x == 0 && my_max > T(0)) atomicMax(a.max_key, order_key(my_max));
}

// ------------------------------------------------------------------ host
struct PassEntry {
    int logl;
    int variant;  // index into codegen.PASS_CANDIDATES[prec][logl]
    int pf;       // 0 direct, 1 cp.async, 2 bulk rows, 3 tensor TMA (needs a tensor map)
    int e, u, p, threads, smem;
    const void* fn[3][3];  // [kind][abft]
};
extern const PassEntry kPass_fp32[];
extern const int kPassCount_fp32;
extern const PassEntry kPass_fp64[];
extern const int kPassCount_fp64;
extern const int kPassChoice_fp32[12][3];  // tuned variant per (log2 L, kind)
extern const int kPassChoice_fp64[12][3];
// runtime override for tuning (-1 = tuned choice)
int pass_tune_select(int prec, int logl, int kind, int variant);
int pass_tune_variants(int prec, int logl);

struct MultiPlan {
    int prec = 0;
    int nst = 0;
    long long n = 0;
    long long d[3] = {0, 0, 0};
    int num_sms = 148;
    void* twL[3] = {nullptr, nullptr, nullptr};        // w_{d_k}^i tables
    void* ptw_lo[2] = {nullptr, nullptr};              // post twiddles per non-last stage
    void* ptw_hi[2] = {nullptr, nullptr};
    int ptw_shift[2] = {0, 0};
    void* ws = nullptr;                                // intermediate batch buffer
    size_t ws_bytes = 0;
    void* part = nullptr;                              // ABFT partials
    size_t part_bytes = 0;
    void* ftab = nullptr;                              // campaign fault tables (one per pass)
    size_t ftab_bytes = 0;
};

// One fault per run of a batched campaign, in multi-pass launch codes
// (where 1 input / 2 stage / 3 output; signal run-relative).
struct HostFault {
    long long signal, elem;
    int where, stage, comp, bit;
};

struct MultiLaunch {
    const void* in;
    void* out;
    long long batch, sig_base;
    int inverse, scale_inv, abft;
    const void* etw;
    const void* values;
    double delta, abs_floor;
    long long f_signal, f_elem;
    int f_where, f_stage, f_comp, f_bit;
    int* flag_count;
    FlagRec* flag_rec;
    long long flag_cap;
    unsigned* flag_ovf;
    unsigned long long* max_key;
    int only_stage;  // -1: whole transform; k: just stage k, in -> out
    const HostFault* faults;  // batched campaign: nfaults runs of f_div signals
    long long nfaults, f_div;
    void* rel_out;            // optional per-signal relative discrepancy (plan dtype)
};

int multi_plan_init(MultiPlan& mp, long long n, int prec, int nst, const int64_t* dims, int num_sms);
int multi_launch(MultiPlan& mp, const MultiLaunch& m, cudaStream_t st);
// Only stage `k` (no ABFT, no scaling): in -> out in the pass layout.
int multi_launch_stage(MultiPlan& mp, int k, const void* in, void* out, long long batch, int inverse,
                       cudaStream_t st);
void multi_plan_free(MultiPlan& mp);
const char* multi_last_error();

}  // namespace tfft
