// Small kernels off the fault-free hot path: the API-level encode / detect
// entry points (reference abft/pipeline.py:72-135), the online correction of a
// flagged group (pipeline.py:164-192) and device-side bit flips
// (fault_lab/bits.py:48-53).
#pragma once
#include "single.cuh"

namespace tfft {

constexpr int AUX_THREADS = 512;

template <class T>
__device__ __forceinline__ T block_sum(T v, T* sh) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = fadd(v, shfl_xor(v, off));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    T s = T(0);
    if (threadIdx.x == 0) {
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s = fadd(s, sh[w]);
    }
    return s;  // valid in thread 0
}

// One CTA per signal: c[b] = x_b . row (row may be null -> skipped),
// l1[b] = sum |x_b| (hypot, like numpy's abs).
template <class T>
__global__ void __launch_bounds__(AUX_THREADS)
dot_l1_kernel(const C<T>* __restrict__ x, long long n, const C<T>* __restrict__ row,
              C<T>* __restrict__ c, T* __restrict__ l1) {
    __shared__ T sh[AUX_THREADS / 32];
    const C<T>* xb = x + (long long)blockIdx.x * n;
    C<T> acc = mk<T>(T(0), T(0));
    T l = T(0);
    for (long long k = threadIdx.x; k < n; k += blockDim.x) {
        const C<T> v = xb[k];
        if (row) acc = cadd<T>(acc, cmul<T>(v, row[k]));
        l = fadd(l, cabs<T>(v));
    }
    T sx = block_sum(acc.x, sh);
    T sy = block_sum(acc.y, sh);
    T sl = block_sum(l, sh);
    if (threadIdx.x == 0) {
        if (c) c[blockIdx.x] = mk<T>(sx, sy);
        if (l1) l1[blockIdx.x] = sl;
    }
}

// Exact detection of signals the fused kernels could not decide from their
// l1 upper bound (|c_in| below FLOOR_COEF * sum(|re|+|im|), so the floor may
// matter): one CTA per listed signal recomputes c_in = x.etw, c_out = y.e and
// sum|x| (IEEE hypot) and the reference's rel (pipeline.py:104-121).
template <class T>
__global__ void __launch_bounds__(AUX_THREADS)
recheck_kernel(const C<T>* __restrict__ in, const C<T>* __restrict__ out, long long n,
               const long long* __restrict__ sigs, const C<T>* __restrict__ etw,
               const C<T>* __restrict__ values, T abs_floor, T floor_coef, double* __restrict__ rel) {
    __shared__ T sh[AUX_THREADS / 32];
    const long long sg = sigs[blockIdx.x];
    const C<T>* x = in + sg * n;
    const C<T>* y = out + sg * n;
    C<T> cin = mk<T>(T(0), T(0)), cout = mk<T>(T(0), T(0));
    T l1 = T(0);
    const T hr = T(-0.5), hi = T(0.8660254037844386467637232);
    for (long long k = threadIdx.x; k < n; k += blockDim.x) {
        C<T> e;
        if (values) e = values[k];
        else {
            const int cls = (int)(k % 3);
            e = cls == 0 ? mk<T>(T(1), T(0)) : (cls == 1 ? mk<T>(hr, -hi) : mk<T>(hr, hi));
        }
        cout = cadd<T>(cout, cmul<T>(y[k], e));
        cin = cadd<T>(cin, cmul<T>(x[k], etw[k]));
        l1 = fadd(l1, cabs<T>(x[k]));
    }
    T a0 = block_sum(cin.x, sh), a1 = block_sum(cin.y, sh);
    T a2 = block_sum(cout.x, sh), a3 = block_sum(cout.y, sh);
    T a4 = block_sum(l1, sh);
    if (threadIdx.x == 0) {
        const C<T> raw = mk<T>(fsub(a0, a2), fsub(a1, a3));
        const T fl = nanmax<T>(abs_floor, fmul(floor_coef, a4));
        const T den = nanmax<T>(cabs<T>(mk<T>(a0, a1)), fl);
        T r = cabs<T>(raw) / den;
        if (!isfinite(r)) r = T(INFINITY);
        rel[blockIdx.x] = (double)r;
    }
}

// s0[k] = sum_b x_b[k] (sequential in b, like numpy's axis-0 sum),
// s1[k] = sum_b (b+1) x_b[k] in complex128 (the reference promotes through
// its float64 weights, pipeline.py:79-82).
template <class T>
__global__ void group_sums_kernel(const C<T>* __restrict__ xg, long long bs, long long n,
                                  C<T>* __restrict__ s0, double2* __restrict__ s1) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x) {
        C<T> a = xg[k];
        double2 w = make_double2((double)a.x, (double)a.y);
        for (long long b = 1; b < bs; ++b) {
            const C<T> v = xg[b * n + k];
            a = cadd<T>(a, v);
            w.x = __dadd_rn(w.x, __dmul_rn((double)(b + 1), (double)v.x));
            w.y = __dadd_rn(w.y, __dmul_rn((double)(b + 1), (double)v.y));
        }
        if (s0) s0[k] = a;
        if (s1) s1[k] = w;
    }
}

// Relative discrepancy per signal of a group (pipeline.py:104-135); one CTA
// per signal. values == null -> Wang weights.
template <class T>
__global__ void __launch_bounds__(AUX_THREADS)
detect_kernel(const C<T>* __restrict__ y, long long n, const C<T>* __restrict__ values,
              const C<T>* __restrict__ c_in, const T* __restrict__ x_l1, T abs_floor,
              T floor_coef, T* __restrict__ rel, C<T>* __restrict__ raw_out) {
    __shared__ T sh[AUX_THREADS / 32];
    const C<T>* yb = y + (long long)blockIdx.x * n;
    C<T> acc = mk<T>(T(0), T(0));
    const T hr = T(-0.5), hi = T(0.8660254037844386467637232);
    for (long long k = threadIdx.x; k < n; k += blockDim.x) {
        C<T> e;
        if (values) e = values[k];
        else {
            const int cls = (int)(k % 3);
            e = cls == 0 ? mk<T>(T(1), T(0)) : (cls == 1 ? mk<T>(hr, -hi) : mk<T>(hr, hi));
        }
        acc = cadd<T>(acc, cmul<T>(yb[k], e));
    }
    T sx = block_sum(acc.x, sh);
    T sy = block_sum(acc.y, sh);
    if (threadIdx.x == 0) {
        const C<T> ci = c_in[blockIdx.x];
        const C<T> raw = mk<T>(fsub(ci.x, sx), fsub(ci.y, sy));
        const T fl = nanmax<T>(abs_floor, fmul(floor_coef, x_l1[blockIdx.x]));
        const T den = nanmax<T>(cabs<T>(ci), fl);
        T r = cabs<T>(raw) / den;
        if (!isfinite(r)) r = T(INFINITY);
        rel[blockIdx.x] = r;
        if (raw_out) raw_out[blockIdx.x] = raw;
    }
}

struct FixJob {
    long long first;     // global index of the group's first signal
    long long flagged;   // global index of the flagged signal
    int ok;              // out: 1 = corrected and verified
    int pad;
};

// Online correction of K flagged groups, one CTA per group:
//   fixed = W s0 - sum_{b != f} y_b  (pipeline.py:180-185),
//   then re-verify the rebuilt signal against its input-side checksum and
//   commit it into `out` only if it passes (protected.py:156-162).
// ws0: K transformed group sums; scratch: K x n staging.
template <class T>
__global__ void __launch_bounds__(AUX_THREADS)
fix_groups_kernel(const C<T>* __restrict__ in, C<T>* __restrict__ out, long long n, long long bs,
                  const C<T>* __restrict__ ws0, C<T>* __restrict__ scratch,
                  const C<T>* __restrict__ etw, const C<T>* __restrict__ values, T delta,
                  T abs_floor, T floor_coef, FixJob* jobs) {
    __shared__ T sh[AUX_THREADS / 32];
    __shared__ int verdict;
    FixJob job = jobs[blockIdx.x];
    const C<T>* w = ws0 + (long long)blockIdx.x * n;
    C<T>* fx = scratch + (long long)blockIdx.x * n;
    const C<T>* xf = in + job.flagged * n;
    C<T> cin = mk<T>(T(0), T(0)), cout = mk<T>(T(0), T(0));
    T l1 = T(0);
    const T hr = T(-0.5), hi = T(0.8660254037844386467637232);
    for (long long k = threadIdx.x; k < n; k += blockDim.x) {
        C<T> others = mk<T>(T(0), T(0));
        bool first = true;
        for (long long b = 0; b < bs; ++b) {
            const long long s = job.first + b;
            if (s == job.flagged) continue;
            const C<T> v = out[s * n + k];
            others = first ? v : cadd<T>(others, v);
            first = false;
        }
        const C<T> f = csub<T>(w[k], others);
        fx[k] = f;
        C<T> e;
        if (values) e = values[k];
        else {
            const int cls = (int)(k % 3);
            e = cls == 0 ? mk<T>(T(1), T(0)) : (cls == 1 ? mk<T>(hr, -hi) : mk<T>(hr, hi));
        }
        cout = cadd<T>(cout, cmul<T>(f, e));
        const C<T> x = xf[k];
        cin = cadd<T>(cin, cmul<T>(x, etw[k]));
        l1 = fadd(l1, cabs<T>(x));
    }
    T a0 = block_sum(cin.x, sh), a1 = block_sum(cin.y, sh);
    T a2 = block_sum(cout.x, sh), a3 = block_sum(cout.y, sh);
    T a4 = block_sum(l1, sh);
    if (threadIdx.x == 0) {
        const C<T> raw = mk<T>(fsub(a0, a2), fsub(a1, a3));
        const T fl = nanmax<T>(abs_floor, fmul(floor_coef, a4));
        const T den = nanmax<T>(cabs<T>(mk<T>(a0, a1)), fl);
        T r = cabs<T>(raw) / den;
        if (!isfinite(r)) r = T(INFINITY);
        verdict = !(r > delta);
        jobs[blockIdx.x].ok = verdict;
    }
    __syncthreads();
    if (verdict) {
        C<T>* dst = out + job.flagged * n;
        for (long long k = threadIdx.x; k < n; k += blockDim.x) dst[k] = fx[k];
    }
}

// out = y_f = ws0 - sum_{b != f} y_b for one signal (tfft_correct_signal).
template <class T>
__global__ void rebuild_kernel(const C<T>* __restrict__ ws0, const C<T>* __restrict__ yg,
                               long long bs, long long n, long long f, C<T>* __restrict__ fixed) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x) {
        C<T> others = mk<T>(T(0), T(0));
        bool first = true;
        for (long long b = 0; b < bs; ++b) {
            if (b == f) continue;
            const C<T> v = yg[b * n + k];
            others = first ? v : cadd<T>(others, v);
            first = false;
        }
        fixed[k] = csub<T>(ws0[k], others);
    }
}

template <class T>
__global__ void scale_kernel(C<T>* buf, long long count, T s) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x)
        buf[i] = cscale<T>(buf[i], s);
}

__global__ void flip_word_kernel(void* buf, long long word, int bit, int bytes) {
    if (bytes == 4) {
        unsigned int* p = reinterpret_cast<unsigned int*>(buf) + word;
        *p ^= (1u << bit);
    } else {
        unsigned long long* p = reinterpret_cast<unsigned long long*>(buf) + word;
        *p ^= (1ull << bit);
    }
}

}  // namespace tfft
