// Shared device building blocks for the B200 (sm_100a) fault-tolerant FFT.
//
// * complex arithmetic with explicit fma/rn intrinsics, so every instantiation
//   (ABFT on/off, fault injection on/off) rounds identically — the reference's
//   "protected output is bitwise equal to unprotected output" contract
//   (reference tests/test_abft.py:265-273) holds by construction;
// * compile-time twiddle constants w_R^m for R <= 64 (thread-level macro FFTs
//   with twiddles baked in as immediates);
// * in-register natural-order DFTs of size 2..64 built by template recursion.
#pragma once
#include <cstdint>
#include <limits>
#include <cuda_runtime.h>

namespace tfft {

template <class T> struct cx;
template <> struct cx<float>  { using type = float2; };
template <> struct cx<double> { using type = double2; };
template <class T> using C = typename cx<T>::type;

template <class T> __device__ __forceinline__ T fmul(T a, T b);
template <> __device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ double fmul(double a, double b) { return __dmul_rn(a, b); }
template <class T> __device__ __forceinline__ T ffma(T a, T b, T c);
template <> __device__ __forceinline__ float ffma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
template <> __device__ __forceinline__ double ffma(double a, double b, double c) { return __fma_rn(a, b, c); }
template <class T> __device__ __forceinline__ T fadd(T a, T b);
template <> __device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double fadd(double a, double b) { return __dadd_rn(a, b); }
template <class T> __device__ __forceinline__ T fsub(T a, T b);
template <> __device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
template <> __device__ __forceinline__ double fsub(double a, double b) { return __dsub_rn(a, b); }

template <class T> __device__ __forceinline__ C<T> mk(T x, T y) { C<T> r; r.x = x; r.y = y; return r; }
template <class T> __device__ __forceinline__ C<T> cadd(C<T> a, C<T> b) { return mk<T>(fadd(a.x, b.x), fadd(a.y, b.y)); }
template <class T> __device__ __forceinline__ C<T> csub(C<T> a, C<T> b) { return mk<T>(fsub(a.x, b.x), fsub(a.y, b.y)); }
// (a.x + i a.y)(b.x + i b.y), two roundings per component, fixed order.
template <class T> __device__ __forceinline__ C<T> cmul(C<T> a, C<T> b) {
    return mk<T>(ffma(a.x, b.x, -fmul(a.y, b.y)), ffma(a.x, b.y, fmul(a.y, b.x)));
}
// a * conj(b)
template <class T> __device__ __forceinline__ C<T> cmulc(C<T> a, C<T> b) {
    return mk<T>(ffma(a.x, b.x, fmul(a.y, b.y)), ffma(a.y, b.x, -fmul(a.x, b.y)));
}
template <class T> __device__ __forceinline__ C<T> swapri(C<T> a) { return mk<T>(a.y, a.x); }
template <class T> __device__ __forceinline__ C<T> cscale(C<T> a, T s) { return mk<T>(fmul(a.x, s), fmul(a.y, s)); }

// ---- fp32: Blackwell packed f32x2 arithmetic (SASS FADD2/FMUL2/FFMA2).
// A complex64 value is one 64-bit register pair, so complex add/sub is one
// instruction and a multiply by a twiddle two (plus operand swizzles that
// ptxas folds into the instruction). Every lane is still one IEEE rn op, and
// the rounding sequence of each component is fixed, so all instantiations
// stay bitwise consistent.
namespace f2 {
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float x, float y) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
    return r;
}
__device__ __forceinline__ float2 up(u64 r) {
    float2 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
__device__ __forceinline__ u64 add(u64 a, u64 b) {
    u64 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 sub(u64 a, u64 b) {
    u64 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 mul(u64 a, u64 b) {
    u64 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 fma(u64 a, u64 b, u64 c) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
}  // namespace f2

template <> __device__ __forceinline__ float2 cadd<float>(float2 a, float2 b) {
    return f2::up(f2::add(f2::pk(a.x, a.y), f2::pk(b.x, b.y)));
}
template <> __device__ __forceinline__ float2 csub<float>(float2 a, float2 b) {
    return f2::up(f2::sub(f2::pk(a.x, a.y), f2::pk(b.x, b.y)));
}
// (ax wx - ay wy, ay wx + ax wy) = (a.x,a.y)*wx + (a.y,a.x)*(-wy, wy)
template <> __device__ __forceinline__ float2 cmul<float>(float2 a, float2 w) {
    return f2::up(f2::fma(f2::pk(a.x, a.y), f2::pk(w.x, w.x),
                          f2::mul(f2::pk(a.y, a.x), f2::pk(-w.y, w.y))));
}
// a * conj(w) = (ax wx + ay wy, ay wx - ax wy)
template <> __device__ __forceinline__ float2 cmulc<float>(float2 a, float2 w) {
    return f2::up(f2::fma(f2::pk(a.x, a.y), f2::pk(w.x, w.x),
                          f2::mul(f2::pk(a.y, a.x), f2::pk(w.y, -w.y))));
}
template <> __device__ __forceinline__ float2 cscale<float>(float2 a, float s) {
    return f2::up(f2::mul(f2::pk(a.x, a.y), f2::pk(s, s)));
}

// a + (-i) b = (a.x + b.y, a.y - b.x) and a - (-i) b, one packed FMA each.
template <class T> __device__ __forceinline__ C<T> add_mi(C<T> a, C<T> b) {
    return mk<T>(fadd(a.x, b.y), fsub(a.y, b.x));
}
template <class T> __device__ __forceinline__ C<T> sub_mi(C<T> a, C<T> b) {
    return mk<T>(fsub(a.x, b.y), fadd(a.y, b.x));
}
template <> __device__ __forceinline__ float2 add_mi<float>(float2 a, float2 b) {
    return f2::up(f2::fma(f2::pk(b.y, b.x), f2::pk(1.0f, -1.0f), f2::pk(a.x, a.y)));
}
template <> __device__ __forceinline__ float2 sub_mi<float>(float2 a, float2 b) {
    return f2::up(f2::fma(f2::pk(b.y, b.x), f2::pk(-1.0f, 1.0f), f2::pk(a.x, a.y)));
}
// acc + v * e  (ABFT dot-product step)
template <class T> __device__ __forceinline__ C<T> cmac(C<T> acc, C<T> v, C<T> e) {
    return mk<T>(ffma(v.x, e.x, ffma(-v.y, e.y, acc.x)), ffma(v.x, e.y, ffma(v.y, e.x, acc.y)));
}
template <> __device__ __forceinline__ float2 cmac<float>(float2 acc, float2 v, float2 e) {
    const f2::u64 t = f2::fma(f2::pk(v.y, v.x), f2::pk(-e.y, e.y), f2::pk(acc.x, acc.y));
    return f2::up(f2::fma(f2::pk(v.x, v.y), f2::pk(e.x, e.x), t));
}

// ---------------------------------------------------------------- constants
// First octant of the 64th roots of unity: (cos, sin)(2*pi*k/64), k = 0..8.
struct Oct { double c, s; };
__host__ __device__ constexpr Oct oct_base(int k) {
    return k == 0 ? Oct{1.0, 0.0}
         : k == 1 ? Oct{0.995184726672196886244837, 0.09801714032956060199419556}
         : k == 2 ? Oct{0.9807852804032304491261822, 0.1950903220161282678482849}
         : k == 3 ? Oct{0.9569403357322088649357979, 0.2902846772544623676361924}
         : k == 4 ? Oct{0.9238795325112867561281832, 0.38268343236508977172846}
         : k == 5 ? Oct{0.8819212643483550297127569, 0.4713967368259976485563876}
         : k == 6 ? Oct{0.8314696123025452370787884, 0.5555702330196022247428308}
         : k == 7 ? Oct{0.7730104533627369608109066, 0.6343932841636454982151716}
         :          Oct{0.7071067811865475244008444, 0.7071067811865475244008444};
}
// (cos, sin)(2*pi*k/64) for any k in [0, 64) by octant symmetry (exact).
__host__ __device__ constexpr Oct unit64(int k) {
    return k <= 8  ? oct_base(k)
         : k <= 16 ? Oct{oct_base(16 - k).s, oct_base(16 - k).c}
         : k <= 32 ? Oct{-unit64(32 - k).c, unit64(32 - k).s}
         :           Oct{unit64(64 - k).c, -unit64(64 - k).s};
}

// z * w_R^M with w_R = exp(-2*pi*i/R); special angles avoid multiplications.
template <class T, int R, int M>
__device__ __forceinline__ C<T> mul_w(C<T> z) {
    constexpr int m = ((M % R) + R) % R;
    if constexpr (m == 0) {
        return z;
    } else if constexpr (4 * m == R) {          // -i
        return mk<T>(z.y, -z.x);
    } else if constexpr (2 * m == R) {          // -1
        return mk<T>(-z.x, -z.y);
    } else if constexpr (4 * m == 3 * R) {      // +i
        return mk<T>(-z.y, z.x);
    } else if constexpr (8 * m == R) {          // (1 - i)/sqrt2
        constexpr T h = T(0.7071067811865475244008444);
        if constexpr (sizeof(T) == 4)
            return f2::up(f2::mul(f2::fma(f2::pk(z.x, z.x), f2::pk(1.f, -1.f), f2::pk(z.y, z.y)),
                                  f2::pk(h, h)));
        else
            return mk<T>(fmul(fadd(z.x, z.y), h), fmul(fsub(z.y, z.x), h));
    } else if constexpr (8 * m == 3 * R) {      // (-1 - i)/sqrt2
        constexpr T h = T(0.7071067811865475244008444);
        if constexpr (sizeof(T) == 4)
            return f2::up(f2::mul(f2::fma(f2::pk(z.x, z.x), f2::pk(-1.f, 1.f), f2::pk(z.y, z.y)),
                                  f2::pk(h, -h)));
        else
            return mk<T>(fmul(fsub(z.y, z.x), h), -fmul(fadd(z.x, z.y), h));
    } else if constexpr (8 * m == 5 * R) {      // (-1 + i)/sqrt2
        constexpr T h = T(0.7071067811865475244008444);
        if constexpr (sizeof(T) == 4)
            return f2::up(f2::mul(f2::fma(f2::pk(z.y, z.y), f2::pk(1.f, -1.f), f2::pk(z.x, z.x)),
                                  f2::pk(-h, h)));
        else
            return mk<T>(-fmul(fadd(z.x, z.y), h), fmul(fsub(z.x, z.y), h));
    } else if constexpr (8 * m == 7 * R) {      // (1 + i)/sqrt2
        constexpr T h = T(0.7071067811865475244008444);
        if constexpr (sizeof(T) == 4)
            return f2::up(f2::mul(f2::fma(f2::pk(z.y, z.y), f2::pk(-1.f, 1.f), f2::pk(z.x, z.x)),
                                  f2::pk(h, h)));
        else
            return mk<T>(fmul(fsub(z.x, z.y), h), fmul(fadd(z.x, z.y), h));
    } else {
        static_assert(64 % R == 0, "compile-time twiddles limited to R <= 64");
        constexpr Oct u = unit64(m * (64 / R));
        return cmul<T>(z, mk<T>(T(u.c), T(-u.s)));
    }
}

// ------------------------------------------------------ in-register DFTs
// a[k] <- sum_n a[n] w_R^{nk}; indices are compile-time so everything lives
// in registers. Split R = R1*R2 (decimation in time): R2-point DFTs over the
// stride-R1 subsequences, twiddle w_R^{n1 k2}, R1-point DFTs across.
template <class T, int R> struct Dft;

template <class T> struct Dft<T, 1> {
    static __device__ __forceinline__ void run(C<T>*) {}
};
template <class T> struct Dft<T, 2> {
    static __device__ __forceinline__ void run(C<T>* a) {
        C<T> s = cadd<T>(a[0], a[1]);
        a[1] = csub<T>(a[0], a[1]);
        a[0] = s;
    }
};
template <class T> struct Dft<T, 4> {
    static __device__ __forceinline__ void run(C<T>* a) {
        C<T> t0 = cadd<T>(a[0], a[2]), t1 = csub<T>(a[0], a[2]);
        C<T> t2 = cadd<T>(a[1], a[3]), d = csub<T>(a[1], a[3]);
        a[0] = cadd<T>(t0, t2);
        a[2] = csub<T>(t0, t2);
        a[1] = add_mi<T>(t1, d);  // t1 + (a1 - a3)(-i)
        a[3] = sub_mi<T>(t1, d);
    }
};

template <class T, int R1, int R2, int N1>
struct TwRow {  // apply w_R^{n1 k2} for k2 = 0..R2-1 on row n1
    template <int K2>
    static __device__ __forceinline__ void go(C<T> (&b)[R1 * R2]) {
        if constexpr (K2 < R2) {
            b[N1 * R2 + K2] = mul_w<T, R1 * R2, N1 * K2>(b[N1 * R2 + K2]);
            go<K2 + 1>(b);
        }
    }
};

template <class T, int R>
struct Dft {
    static constexpr int R1 = (R >= 16) ? 4 : 2;
    static constexpr int R2 = R / R1;
    static __device__ __forceinline__ void run(C<T>* a) {
        C<T> b[R];
        // b[n1*R2 + k2] = DFT_R2 over n2 of a[n1 + R1*n2]
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1) {
            C<T> s[R2];
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) s[n2] = a[n1 + R1 * n2];
            Dft<T, R2>::run(s);
#pragma unroll
            for (int k2 = 0; k2 < R2; ++k2) b[n1 * R2 + k2] = s[k2];
        }
        twid<1>(b);
        // X[k2 + R2*k1] = DFT_R1 over n1 of b[n1*R2 + k2]
#pragma unroll
        for (int k2 = 0; k2 < R2; ++k2) {
            C<T> s[R1];
#pragma unroll
            for (int n1 = 0; n1 < R1; ++n1) s[n1] = b[n1 * R2 + k2];
            Dft<T, R1>::run(s);
#pragma unroll
            for (int k1 = 0; k1 < R1; ++k1) a[k2 + R2 * k1] = s[k1];
        }
    }
    template <int N1>
    static __device__ __forceinline__ void twid(C<T> (&b)[R]) {
        if constexpr (N1 < R1) {
            TwRow<T, R1, R2, N1>::template go<0>(b);
            twid<N1 + 1>(b);
        }
    }
};

// ------------------------------------------------------------- bit flips
template <class T> __device__ __forceinline__ T flip_bit(T v, int bit);
template <> __device__ __forceinline__ float flip_bit(float v, int bit) {
    return __uint_as_float(__float_as_uint(v) ^ (1u << bit));
}
template <> __device__ __forceinline__ double flip_bit(double v, int bit) {
    return __longlong_as_double(__double_as_longlong(v) ^ (1ll << bit));
}
template <class T> __device__ __forceinline__ void flip_component(C<T>& z, int comp, int bit) {
    if (comp == 0) z.x = flip_bit<T>(z.x, bit); else z.y = flip_bit<T>(z.y, bit);
}

// ------------------------------------------------------------ misc
template <class T> __device__ __forceinline__ T cabs(C<T> z);
template <> __device__ __forceinline__ float cabs(float2 z) { return hypotf(z.x, z.y); }
template <> __device__ __forceinline__ double cabs(double2 z) { return hypot(z.x, z.y); }

// cheap magnitude for the l1 floor (only ever used as a floor, reference
// abft/pipeline.py:100-101): fp32 via the SFU sqrt, fp64 in full precision.
__device__ __forceinline__ float mag_fast(float2 z) {
    float s = ffma(z.x, z.x, fmul(z.y, z.y));
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(s));
    return r;
}
template <class T> __device__ __forceinline__ T nanmax(T a, T b) {
    return (a != a) ? a : ((b != b) ? b : (a > b ? a : b));
}

// (|re|, |im|): per-element term of the l1 upper bound sum(|re| + |im|)
template <class T> __device__ __forceinline__ C<T> cabs2(C<T> z) { return mk<T>(fabs(z.x), fabs(z.y)); }

// |z| for the l1 mass, which only feeds the detection floor
// (FLOOR_COEF * sum|x|, pipeline.py:100-101): s * rsqrt.approx(s) (MUFU.RSQ64H,
// ~1e-7 relative) instead of the IEEE sqrt's DFMA Newton chain. The floor
// decides only when |c_in| < 1e-12 * sum|x|; at that relative accuracy no
// decision moves.
__device__ __forceinline__ double mag_fast(double2 z) {
    const double s = ffma(z.x, z.x, fmul(z.y, z.y));
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
    return s > 0.0 ? (s < 1e300 ? s * r : sqrt(s)) : s;
}

// Order-preserving key for non-negative floating values (NaN mapped to +inf
// by the caller) — lets max_rel be reduced with integer atomicMax.
__device__ __forceinline__ unsigned int order_key(float v) { return __float_as_uint(v); }
__device__ __forceinline__ unsigned long long order_key(double v) {
    return (unsigned long long)__double_as_longlong(v);
}

template <class T> __device__ __forceinline__ T shfl_xor(T v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

// ------------------------------------------------ TMA bulk copies + mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy (TMA, SASS UBLKCP) completing on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// the same with shared-window addresses computed once per kernel (the
// generic -> shared conversion reads SR_CgaCtaId, a long-latency S2R, and
// was being redone inside the tile loop)
__device__ __forceinline__ void mbar_expect_tx_s(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s_s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
// order this thread's (barrier-synchronised) generic smem accesses before
// subsequent async-proxy (TMA) writes to the same buffer
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace tfft
