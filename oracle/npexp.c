/*
 * ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product library.
 *
 * Scalar C restatement of numpy's float32 `np.exp` as dispatched on x86-64
 * hosts with AVX512F (numpy 2.x, `loops_exponent_log.dispatch.c.src`, the
 * AVX512F `simd_exp_f32` kernel): Cody-Waite range reduction by ln2,
 * a degree-5 / degree-2 rational approximation, then scaling by 2^q.
 *
 * Why it exists: the reference gates (`moefold/tensor.py:288`,
 * `np.exp(safe - row_max)`) are computed by numpy's float32 exp, which is
 * NOT correctly rounded (it differs from glibc expf in ~1/3 of inputs).
 * The B200 router kernel must reproduce those gate bits, so the device code
 * ports this algorithm; this file is the host-side checker that the port is
 * pinned against `np.exp` itself (tests/test_oracle.py) and against the
 * golden gates generated from the reference (tests/golden/).
 *
 * Compile WITHOUT contraction and WITHOUT fast-math:
 *     gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC npexp.c -lm
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

float npexp_f32(float x) {
    const float xmax = 88.72283935546875f;
    const float xmin = -103.97208404541015625f;
    const int is_nan = (x != x);
    const int is_hi = (x >= xmax);
    const int is_lo = (x <= xmin);
    if (is_nan || is_hi || is_lo) x = 0.0f;

    /* rint(x * log2e) via the 1.5*2^23 magic constant: three separately
     * rounded float ops (must not be fused). */
    volatile float t = x * 1.442695040888963407359924681001892137f;
    volatile float u = t + 0x1.8p23f;
    float q = u - 0x1.8p23f;

    float r = fmaf(q, -6.93145752e-1f, x);
    r = fmaf(q, -1.42860677e-6f, r);
    r = fmaf(q, 0.0f, r);

    float num = fmaf(5.082762527590693718096e-04f, r, 6.757896990527504603057e-03f);
    num = fmaf(num, r, 5.114512081637298353406e-02f);
    num = fmaf(num, r, 2.473615434895520810817e-01f);
    num = fmaf(num, r, 7.257664613233124478488e-01f);
    num = fmaf(num, r, 9.999999999980870924916e-01f);

    float den = fmaf(2.159509375685829852307e-02f, r, -2.742335390411667452936e-01f);
    den = fmaf(den, r, 1.0f);

    float y = ldexpf(num / den, (int)q);
    if (is_nan) y = NAN;
    if (is_hi) y = INFINITY;
    if (is_lo) y = 0.0f;
    return y;
}

void npexp_f32_array(const float* x, float* y, size_t n) {
    for (size_t i = 0; i < n; ++i) y[i] = npexp_f32(x[i]);
}

/* Exhaustive sweep helper: count mismatches of the port against a caller
 * supplied table over the float32 bit patterns [lo_bits, hi_bits). */
size_t npexp_f32_count_mismatch(const float* x, const float* ref, size_t n) {
    size_t bad = 0;
    for (size_t i = 0; i < n; ++i) {
        float y = npexp_f32(x[i]);
        uint32_t a, b;
        __builtin_memcpy(&a, &y, 4);
        __builtin_memcpy(&b, &ref[i], 4);
        if (a != b) ++bad;
    }
    return bad;
}
