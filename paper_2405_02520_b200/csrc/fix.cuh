// Device-side online correction for the single-kernel sizes (N <= 2^13):
// the reference's correct_group (abft/pipeline.py:164-192) and the
// ONE_SIDED recompute (abft/protected.py:142-147) for every flagged group,
// in ONE launch queued right behind the fused transform — no host round trip
// between detection and correction.
//
// Job source:
//   * plan mode (jobs == nullptr): every CTA reads the detection block the
//     fused kernel just wrote (flag count + records), sorts the <= kFixCap
//     records by signal and groups them exactly like the host's decide()
//     (protected.py:127-136: one flag in a group -> a correction job, more ->
//     unrecoverable). More flags than kFixCap, or an l1-floor recheck sentinel,
//     set `fallback` and the host takes over (rare);
//   * list mode: the host passes the jobs (host-streaming / file paths).
// CTA j corrects job j with the SAME engine configuration as the fused
// kernel (identical W s0 to the unprotected transform of s0):
//   s0 = sum_b x_b (sequential in b), W s0 by the Stockham engine,
//   y_f = W s0 - sum_{b != f} y_b, re-verified with the exact detection
//   arithmetic (pipeline.py:104-121), committed only when it passes.
// ONE_SIDED: y_f = W x_f, committed (recompute_count += 1).
#pragma once
#include "single.cuh"

namespace tfft {

constexpr int kFixCap = 64;  // records / jobs handled on the device per call

// Verdicts of the device correction, read back with the detection summary.
struct FixHead {
    int ran;        // the device pass ran (plan mode)
    int fallback;   // 1: the host must decide / correct this call
    int njobs;
    int pad;
};
struct FixRes {
    long long group, signal;
    int ok, pad;
};

template <class T>
struct FixArgs {
    const C<T>* in;
    C<T>* out;
    long long batch, bs;
    const C<T>* tw;
    const C<T>* etw;
    const C<T>* values;      // table encodings; nullptr = Wang weights
    T delta, abs_floor, floor_coef;
    int inverse, scale_inv, one_sided;
    const int* flag_count;   // plan mode
    const FlagRec* flag_rec;
    const FixJob* jobs;      // list mode (nullptr: plan mode)
    int njobs;
    FixHead* head;           // plan mode verdicts
    FixRes* res;             // [kFixCap] plan mode
    FixJob* jobs_out;        // list mode verdicts (ok), may alias `jobs`
};

template <class T, int N, int E, int PS, int THREADS, class Radices>
__global__ void __launch_bounds__(THREADS)
fix_single_kernel(const __grid_constant__ FixArgs<T> a) {
    using Eng = Engine<T, N, E, Radices>;
    constexpr int TPS = N / E;
    constexpr bool MULTIPASS = RCount<Radices>::v > 1;
    constexpr int SL = MULTIPASS ? SmemLen<N, PS>::v : 1;
    extern __shared__ __align__(128) unsigned char fix_smem[];
    C<T>* xbuf = reinterpret_cast<C<T>*>(fix_smem);  // (THREADS / TPS) slices of SL
    __shared__ T scratch[(THREADS / 32 + 1) * 5];
    __shared__ long long s_sig[kFixCap];
    __shared__ long long j_first[kFixCap], j_flag[kFixCap];
    __shared__ int s_njobs, s_ok;

    // ---- the job list
    int njobs;
    if (a.jobs == nullptr) {
        if (threadIdx.x == 0) {
            const int cnt = *a.flag_count;
            int fb = cnt > kFixCap;
            int nj = 0;
            if (!fb && cnt > 0) {
                for (int i = 0; i < cnt; ++i) {
                    const FlagRec r = a.flag_rec[i];
                    if (r.rel < 0) fb = 1;  // l1-floor recheck: exact host arithmetic
                    const long long sg = r.sig;
                    int k = i;  // insertion sort by signal (<= kFixCap records)
                    while (k > 0 && s_sig[k - 1] > sg) {
                        s_sig[k] = s_sig[k - 1];
                        --k;
                    }
                    s_sig[k] = sg;
                }
                for (int i = 0; !fb && i < cnt;) {  // group decisions, as the host's decide()
                    const long long g = s_sig[i] / a.bs;
                    int j = i;
                    while (j < cnt && s_sig[j] / a.bs == g) ++j;
                    if (j - i == 1) {
                        j_first[nj] = g * a.bs;
                        j_flag[nj] = s_sig[i];
                        ++nj;
                    }
                    i = j;
                }
            }
            s_njobs = fb ? 0 : nj;
            if (blockIdx.x == 0) *a.head = FixHead{1, fb, fb ? 0 : nj, 0};
        }
        __syncthreads();
        njobs = s_njobs;
    } else {
        njobs = a.njobs;
    }

    const int sl = threadIdx.x / TPS;
    const int t = threadIdx.x % TPS;
    const bool live = sl == 0;  // only slice 0 carries the job (short signals fill a warp)
    for (int j = blockIdx.x; j < njobs; j += gridDim.x) {
        const long long first = a.jobs ? a.jobs[j].first : j_first[j];
        const long long fsig = a.jobs ? a.jobs[j].flagged : j_flag[j];
        const C<T>* xf = a.in + fsig * N;
        // ---- s0 (two-sided) or x_f (one-sided) at this thread's positions;
        // b outer / m inner: E independent loads per round trip (the sum
        // stays sequential in b, as the host path's)
        C<T> v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[m] = mk<T>(T(0), T(0));
        if (live) {
            const C<T>* xg = a.one_sided ? xf : a.in + first * N;
            const long long nb = a.one_sided ? 1 : a.bs;
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = xg[t + m * TPS];
#pragma unroll 4
            for (long long b = 1; b < nb; ++b) {
#pragma unroll
                for (int m = 0; m < E; ++m) v[m] = cadd<T>(v[m], xg[b * N + t + m * TPS]);
            }
        }
        if (a.inverse) {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = swapri<T>(v[m]);
        }
        {
            const SliceMem<T, TPS, PS> mem{xbuf + (MULTIPASS ? sl * SL : 0)};
            Eng::run(v, mem, t, a.tw);
        }
        if (a.inverse) {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = swapri<T>(v[m]);
        }
        if (a.scale_inv) {
            const T sc = T(1) / T(N);
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = cscale<T>(v[m], sc);
        }
        C<T>* dst = a.out + fsig * N;
        int ok = 1;
        if (!a.one_sided) {
            // ---- rebuild y_f = W s0 - sum_{b != f} y_b and its checksums
            C<T> cin = mk<T>(T(0), T(0)), cout = mk<T>(T(0), T(0));
            T l1 = T(0);
            const T hr = T(-0.5), hi = T(0.8660254037844386467637232);
            if (live) {
                C<T> others[E];
                bool firstb = true;
#pragma unroll 4
                for (long long b = 0; b < a.bs; ++b) {  // loads of 4 signals in flight
                    const long long sg = first + b;
                    C<T> y[E];
#pragma unroll
                    for (int m = 0; m < E; ++m) y[m] = a.out[sg * N + t + m * TPS];
                    if (sg != fsig) {
#pragma unroll
                        for (int m = 0; m < E; ++m) others[m] = firstb ? y[m] : cadd<T>(others[m], y[m]);
                        firstb = false;
                    }
                }
                if (firstb) {
#pragma unroll
                    for (int m = 0; m < E; ++m) others[m] = mk<T>(T(0), T(0));
                }
#pragma unroll
                for (int m = 0; m < E; ++m) {
                    const long long k = t + m * TPS;
                    const C<T> f = csub<T>(v[m], others[m]);
                    v[m] = f;
                    C<T> e;
                    if (a.values) e = a.values[k];
                    else {
                        const int cls = (int)(k % 3);
                        e = cls == 0 ? mk<T>(T(1), T(0)) : (cls == 1 ? mk<T>(hr, -hi) : mk<T>(hr, hi));
                    }
                    cout = cadd<T>(cout, cmul<T>(f, e));
                    const C<T> x = xf[k];
                    cin = cadd<T>(cin, cmul<T>(x, a.etw[k]));
                    l1 = fadd(l1, cabs<T>(x));
                }
            }
            T sums[5] = {cin.x, cin.y, cout.x, cout.y, l1};
            sig_sum<TPS>(sums, scratch, t);
            if (threadIdx.x == 0) {  // fix_decide_kernel's exact decision (pipeline.py:104-121)
                const C<T> raw = mk<T>(fsub(sums[0], sums[2]), fsub(sums[1], sums[3]));
                const T fl = nanmax<T>(a.abs_floor, fmul(a.floor_coef, sums[4]));
                const T den = nanmax<T>(cabs<T>(mk<T>(sums[0], sums[1])), fl);
                T r = cabs<T>(raw) / den;
                if (!isfinite(r)) r = T(INFINITY);
                s_ok = !(r > a.delta);
            }
            __syncthreads();
            ok = s_ok;
        }
        if (ok && live) {
#pragma unroll
            for (int m = 0; m < E; ++m) dst[t + m * TPS] = v[m];
        }
        if (threadIdx.x == 0) {
            if (a.jobs == nullptr) a.res[j] = FixRes{first / a.bs, fsig, ok, 0};
            else a.jobs_out[j].ok = ok;
        }
        __syncthreads();  // scratch / xbuf / s_ok reused by the next job
    }
}

}  // namespace tfft
