/*
 * ORACLE — test infrastructure only. Never linked into the product path.
 *
 * Plain-C restatement of the reference's compiled butterfly kernel
 * (`pkg/src/fftshield/kernels/_stockham.pyx:16-65`, function `_steps` and its
 * wrapper `tile_fft`): a radix-2 Stockham autosort applied independently to
 * each row of a (T, L) complex matrix, ping-ponging between two buffers, with
 * no 1/L scaling and conjugated factors on the inverse path.
 *
 * The arithmetic is written with C99 `_Complex` types, which is what Cython
 * emits for `float complex` / `double complex` when CYTHON_CCOMPLEX is on
 * (checked in the generated `_stockham.c`), so with the same gcc flags the
 * results are bit-identical to the reference extension.
 *
 * Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
 * `--impl reference` leg may load this library.
 */
#include <complex.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>

#define DEFINE_STEPS(NAME, CT)                                                   \
static void NAME(CT *a, CT *b, int64_t t_count, int64_t length,                  \
                 const CT *base, int inverse, CT **result)                      \
{                                                                               \
    /* _stockham.pyx:18-43 — m halves, s doubles, one radix-2 step per round */ \
    int64_t m = length / 2, s = 1;                                              \
    CT *x = a, *y = b, *tmp;                                                    \
    while (m >= 1) {                                                            \
        int64_t stride = length / (2 * s);                                      \
        for (int64_t t = 0; t < t_count; ++t) {                                 \
            CT *xr = x + t * length, *yr = y + t * length;                      \
            for (int64_t p = 0; p < m; ++p) {                                   \
                for (int64_t q = 0; q < s; ++q) {                               \
                    CT w = base[q * stride];                                    \
                    if (inverse) w = conj(w);                                   \
                    CT lo = xr[q + s * p];                                      \
                    CT hi = xr[q + s * (p + m)] * w;                            \
                    yr[q + s * 2 * p] = lo + hi;                                \
                    yr[q + s * (2 * p + 1)] = lo - hi;                          \
                }                                                               \
            }                                                                   \
        }                                                                       \
        tmp = x; x = y; y = tmp;                                                \
        m /= 2; s *= 2;                                                         \
    }                                                                           \
    *result = x;                                                                \
}

DEFINE_STEPS(steps_c64, float _Complex)
DEFINE_STEPS(steps_c128, double _Complex)

/* tile_fft (_stockham.pyx:46-65): out-of-place, `in` is never written.
 * dtype: 8 = complex64, 16 = complex128. Returns 0 ok, 1 bad argument. */
int oracle_tile_fft(const void *in, void *out, int64_t t_count, int64_t length,
                    const void *base, int inverse, int dtype)
{
    if (t_count < 0 || length < 1 || (length & (length - 1))) return 1;
    size_t bytes = (size_t)t_count * (size_t)length * (size_t)dtype;
    if (length == 1) { memcpy(out, in, bytes); return 0; }
    void *scratch = malloc(bytes ? bytes : 1);
    if (!scratch) return 1;
    memcpy(out, in, bytes);
    if (dtype == 8) {
        float _Complex *res;
        steps_c64((float _Complex *)out, (float _Complex *)scratch, t_count,
                  length, (const float _Complex *)base, inverse, &res);
        if (res != out) memcpy(out, res, bytes);
    } else if (dtype == 16) {
        double _Complex *res;
        steps_c128((double _Complex *)out, (double _Complex *)scratch, t_count,
                   length, (const double _Complex *)base, inverse, &res);
        if (res != out) memcpy(out, res, bytes);
    } else {
        free(scratch);
        return 1;
    }
    free(scratch);
    return 0;
}
