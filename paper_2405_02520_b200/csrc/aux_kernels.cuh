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
#pragma unroll 8
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


// s0 of K flagged groups in one launch (grid.y = group): s0[k] = sum over
// the group's bs signals, sequential in b like group_sums_kernel.
template <class T>
__global__ void group_sums_jobs_kernel(const C<T>* __restrict__ in, long long bs, long long n,
                                       const FixJob* __restrict__ jobs, C<T>* __restrict__ s0) {
    const C<T>* xg = in + jobs[blockIdx.y].first * n;
    C<T>* dst = s0 + (long long)blockIdx.y * n;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x) {
        C<T> a = xg[k];
#pragma unroll 8
        for (long long b = 1; b < bs; ++b) a = cadd<T>(a, xg[b * n + k]);  // 8 loads in flight, sum in order
        dst[k] = a;
    }
}

// The same correction split over many CTAs per group (grid.x chunks of the
// n points, grid.y groups) for long signals: phase 1 rebuilds its chunk into
// `scratch` and writes the chunk's (c_in, c_out, l1) partials; phase 2 (one
// CTA per group) sums them in chunk order and decides; phase 3 commits the
// verified groups chunk by chunk.
constexpr int FIX_CHUNK = 512;  // points per CTA in phase 1 / 3 (2 per thread: latency, not bandwidth)
template <class T>
__global__ void __launch_bounds__(256)
fix_rebuild_kernel(const C<T>* __restrict__ in, const C<T>* __restrict__ out, long long n, long long bs,
                   const C<T>* __restrict__ ws0, C<T>* __restrict__ scratch, const C<T>* __restrict__ etw,
                   const C<T>* __restrict__ values, const FixJob* __restrict__ jobs, T* __restrict__ part) {
    __shared__ T sh[8][5];
    const FixJob job = jobs[blockIdx.y];
    const C<T>* w = ws0 + (long long)blockIdx.y * n;
    C<T>* fx = scratch + (long long)blockIdx.y * n;
    const C<T>* xf = in + job.flagged * n;
    const long long k0 = (long long)blockIdx.x * FIX_CHUNK;
    const long long k1 = k0 + FIX_CHUNK < n ? k0 + FIX_CHUNK : n;
    C<T> cin = mk<T>(T(0), T(0)), cout = mk<T>(T(0), T(0));
    T l1 = T(0);
    const T hr = T(-0.5), hi = T(0.8660254037844386467637232);
    for (long long k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        C<T> others = mk<T>(T(0), T(0));
        bool first = true;
#pragma unroll 8
        for (long long b = 0; b < bs; ++b) {  // unconditional loads (8 in flight), sum in order
            const long long sg = job.first + b;
            const C<T> v = out[sg * n + k];
            if (sg != job.flagged) {
                others = first ? v : cadd<T>(others, v);
                first = false;
            }
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
    T v[5] = {cin.x, cin.y, cout.x, cout.y, l1};
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) v[i] = fadd(v[i], shfl_xor(v[i], off));
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int i = 0; i < 5; ++i) sh[threadIdx.x >> 5][i] = v[i];
    }
    __syncthreads();
    if (threadIdx.x < 5) {
        T acc = sh[0][threadIdx.x];
        for (int wv = 1; wv < 8; ++wv) acc = fadd(acc, sh[wv][threadIdx.x]);
        part[((long long)blockIdx.y * gridDim.x + blockIdx.x) * 5 + threadIdx.x] = acc;
    }
}

template <class T>
__global__ void __launch_bounds__(256) fix_decide_kernel(long long chunks, const T* __restrict__ part, T delta,
                                                         T abs_floor, T floor_coef, FixJob* jobs) {
    // fixed-order parallel sum of the chunk partials: thread t takes chunks
    // t, t + 256, ... in order, then a fixed tree (deterministic)
    __shared__ T sh[256][5];
    T a[5] = {T(0), T(0), T(0), T(0), T(0)};
    for (long long c = threadIdx.x; c < chunks; c += blockDim.x)
#pragma unroll
        for (int i = 0; i < 5; ++i) a[i] = fadd(a[i], part[((long long)blockIdx.x * chunks + c) * 5 + i]);
#pragma unroll
    for (int i = 0; i < 5; ++i) sh[threadIdx.x][i] = a[i];
    __syncthreads();
    for (int w = blockDim.x / 2; w >= 1; w /= 2) {
        if ((int)threadIdx.x < w) {
#pragma unroll
            for (int i = 0; i < 5; ++i) sh[threadIdx.x][i] = fadd(sh[threadIdx.x][i], sh[threadIdx.x + w][i]);
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
#pragma unroll
    for (int i = 0; i < 5; ++i) a[i] = sh[0][i];
    const C<T> raw = mk<T>(fsub(a[0], a[2]), fsub(a[1], a[3]));
    const T fl = nanmax<T>(abs_floor, fmul(floor_coef, a[4]));
    const T den = nanmax<T>(cabs<T>(mk<T>(a[0], a[1])), fl);
    T r = cabs<T>(raw) / den;
    if (!isfinite(r)) r = T(INFINITY);
    jobs[blockIdx.x].ok = !(r > delta);
}

template <class T>
__global__ void fix_commit_kernel(C<T>* __restrict__ out, long long n, const C<T>* __restrict__ scratch,
                                  const FixJob* __restrict__ jobs) {
    const FixJob job = jobs[blockIdx.y];
    if (!job.ok) return;
    const long long k0 = (long long)blockIdx.x * FIX_CHUNK;
    const long long k1 = k0 + FIX_CHUNK < n ? k0 + FIX_CHUNK : n;
    const C<T>* fx = scratch + (long long)blockIdx.y * n;
    C<T>* dst = out + job.flagged * n;
    for (long long k = k0 + threadIdx.x; k < k1; k += blockDim.x) dst[k] = fx[k];
}

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


// ---------------------------------------------------------------- element level
// Element-level two-sided check of one r x B tile (reference abft/element.py:
// 33-92), complex128 like the reference. Tile layout: row-major (r, B), column
// j is one signal's r-point slice.

// y[:, j] = DFT_r(x[:, j]); row_in[j] = etw_row . x[:, j]; xe[i] = x[i, :] . vals_col
__global__ void element_encode_kernel(int r, long long B, const double2* __restrict__ x,
                                      const double2* __restrict__ etw_row, const double2* __restrict__ vals_col,
                                      double2* __restrict__ y, double2* __restrict__ row_in,
                                      double2* __restrict__ xe) {
    __shared__ double2 root[32];
    if (threadIdx.x < r) {
        double s, c;
        sincospi(-2.0 * threadIdx.x / r, &s, &c);  // w_r^m, exactly rounded
        root[threadIdx.x] = make_double2(c, s);
    }
    __syncthreads();
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < B; j += stride) {
        double2 ri = make_double2(0.0, 0.0);
        for (int i = 0; i < r; ++i) ri = cadd<double>(ri, cmul<double>(etw_row[i], x[i * B + j]));
        row_in[j] = ri;
        for (int k = 0; k < r; ++k) {
            double2 acc = make_double2(0.0, 0.0);
            for (int i = 0; i < r; ++i) acc = cadd<double>(acc, cmul<double>(x[i * B + j], root[(i * k) % r]));
            y[k * B + j] = acc;
        }
    }
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < r; i += stride) {
        double2 acc = make_double2(0.0, 0.0);
        for (long long j = 0; j < B; ++j) acc = cadd<double>(acc, cmul<double>(x[i * B + j], vals_col[j]));
        xe[i] = acc;
    }
}

__device__ __forceinline__ double2 cdiv_d(double2 a, double2 b) {
    const double d = b.x * b.x + b.y * b.y;
    return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
__device__ __forceinline__ bool cfinite(double2 z) { return isfinite(z.x) && isfinite(z.y); }

// Row side locates the column (signal), column side the row; one CTA.
// result[0]: 0 clean, 1 corrected, 2 several columns flagged, 3 row/column
// disagreements inconsistent; result[1..2] = (row, col) when corrected.
__global__ void __launch_bounds__(AUX_THREADS)
element_verify_kernel(int r, long long B, double2* __restrict__ y, const double2* __restrict__ row_in,
                      const double2* __restrict__ xe, const double2* __restrict__ vals_row,
                      const double2* __restrict__ vals_col, double delta, double abs_floor,
                      double* __restrict__ rel, int* __restrict__ result) {
    __shared__ int nflag, col;
    __shared__ double2 d_row_j, dcol[32], wxe[32];
    if (threadIdx.x == 0) { nflag = 0; col = -1; }
    __syncthreads();
    for (long long j = threadIdx.x; j < B; j += blockDim.x) {
        double2 c = make_double2(0.0, 0.0);
        bool fin = true;
        for (int i = 0; i < r; ++i) {
            const double2 v = y[i * B + j];
            fin = fin && cfinite(v);
            c = cadd<double>(c, cmul<double>(vals_row[i], v));
        }
        const double2 d = make_double2(row_in[j].x - c.x, row_in[j].y - c.y);
        const double den = fmax(hypot(row_in[j].x, row_in[j].y), abs_floor);
        double q = hypot(d.x, d.y) / (den > 0 ? den : 1.0);
        if (!fin || !isfinite(q)) q = INFINITY;
        rel[j] = q;
        if (q > delta) {
            atomicAdd(&nflag, 1);
            atomicMax(&col, (int)j);
            d_row_j = d;  // meaningful when exactly one column is flagged
        }
    }
    __syncthreads();
    if (nflag == 0 || nflag > 1) {
        if (threadIdx.x == 0) result[0] = nflag == 0 ? 0 : 2;
        return;
    }
    const int j = col;
    // column side: d_col = DFT_r(xe) - y @ vals_col
    if (threadIdx.x < r) {
        const int i = threadIdx.x;
        double2 w = make_double2(0.0, 0.0);
        for (int m = 0; m < r; ++m) {
            double s, c;
            sincospi(-2.0 * ((m * i) % r) / r, &s, &c);
            w = cadd<double>(w, cmul<double>(xe[m], make_double2(c, s)));
        }
        wxe[i] = w;
        double2 acc = make_double2(0.0, 0.0);
        for (long long b = 0; b < B; ++b) acc = cadd<double>(acc, cmul<double>(y[i * B + b], vals_col[b]));
        dcol[i] = make_double2(w.x - acc.x, w.y - acc.y);
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    int bi = 0;
    double best = -1.0;
    for (int i = 0; i < r; ++i) {  // first maximal |d_col|, non-finite counts as inf
        const double a = cfinite(dcol[i]) ? hypot(dcol[i].x, dcol[i].y) : INFINITY;
        if (a > best) { best = a; bi = i; }
    }
    const double2 fix = cdiv_d(dcol[bi], vals_col[j]);
    const double2 eps_col = make_double2(-fix.x, -fix.y);
    const double2 er = cdiv_d(d_row_j, vals_row[bi]);
    const double2 eps_row = make_double2(-er.x, -er.y);
    if (cfinite(eps_col) && cfinite(eps_row)) {
        const double gap = hypot(eps_row.x - eps_col.x, eps_row.y - eps_col.y);
        if (gap > delta * fmax(hypot(eps_col.x, eps_col.y), abs_floor)) {
            result[0] = 3;
            return;
        }
    }
    double2& t = y[bi * B + j];
    if (cfinite(t)) {
        t = make_double2(t.x + fix.x, t.y + fix.y);
    } else {
        double2 others = make_double2(0.0, 0.0);
        for (long long b = 0; b < B; ++b)
            if (b != j) others = cadd<double>(others, cmul<double>(y[bi * B + b], vals_col[b]));
        t = cdiv_d(make_double2(wxe[bi].x - others.x, wxe[bi].y - others.y), vals_col[j]);
    }
    result[0] = 1;
    result[1] = bi;
    result[2] = j;
}

// Direct O(n^2) DFT in complex128 for dft_reference (reference
// fft_core/reference.py:12-39): y_j = scale * sum_k x_k w^(j k mod n) for ANY
// length n, w^m from an exactly rounded table. Deliberately shares nothing
// with the FFT kernels (it is the independent check of the transform path).
// Grid (ceil(n / 256), batch); the CTA stages 256 inputs at a time in smem.
__global__ void __launch_bounds__(256)
dft_direct_kernel(const double2* __restrict__ x, double2* __restrict__ y, long long n,
                  const double2* __restrict__ w, double scale) {
    __shared__ double2 xs[256];
    const long long j = (long long)blockIdx.x * 256 + threadIdx.x;
    const double2* xb = x + (long long)blockIdx.y * n;
    double ax = 0.0, ay = 0.0;
    for (long long k0 = 0; k0 < n; k0 += 256) {
        __syncthreads();
        if (k0 + threadIdx.x < n) xs[threadIdx.x] = xb[k0 + threadIdx.x];
        __syncthreads();
        if (j < n) {
            long long e = (j % n) * (k0 % n) % n;  // (j k) mod n, advanced by j per step
            const int cnt = (int)(n - k0 < 256 ? n - k0 : 256);
            for (int t = 0; t < cnt; ++t) {
                const double2 wv = __ldg(w + e);
                const double2 xv = xs[t];
                ax = fma(xv.x, wv.x, fma(-xv.y, wv.y, ax));
                ay = fma(xv.x, wv.y, fma(xv.y, wv.x, ay));
                e += j;
                if (e >= n) e -= n;
            }
        }
    }
    if (j < n) y[(long long)blockIdx.y * n + j] = make_double2(ax * scale, ay * scale);
}

}  // namespace tfft
