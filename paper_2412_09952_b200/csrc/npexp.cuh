// numpy's float32 exp (AVX512F `simd_exp_f32`), ported op for op so that the
// device gates reproduce the reference's numpy gates bit-for-bit
// (moefold/tensor.py:288 `np.exp(safe - row_max)`).  Host twin and its
// exhaustive check: oracle/npexp.c, tests/test_oracle.py.
//
// Every rounding step is explicit (__f*_rn): the magic-constant rint must not
// be contracted into an FMA, the rational uses true FMAs, the division is IEEE
// and the final scaling by 2^q rounds once (denormal results included).  This
// file must not be compiled with --use_fast_math / -ftz=true.
#pragma once

namespace b200moe {

__device__ __forceinline__ float np_expf(float x) {
    const float xmax = 88.72283935546875f;
    const float xmin = -103.97208404541015625f;
    const bool is_nan = (x != x);
    const bool is_hi = (x >= xmax);
    const bool is_lo = (x <= xmin);
    if (is_nan || is_hi || is_lo) x = 0.0f;

    const float t = __fmul_rn(x, 1.442695040888963407359924681001892137f);
    const float u = __fadd_rn(t, 12582912.0f);  // 0x1.8p23
    const float q = __fsub_rn(u, 12582912.0f);

    float r = __fmaf_rn(q, -6.93145752e-1f, x);
    r = __fmaf_rn(q, -1.42860677e-6f, r);
    r = __fmaf_rn(q, 0.0f, r);

    float num = __fmaf_rn(5.082762527590693718096e-04f, r, 6.757896990527504603057e-03f);
    num = __fmaf_rn(num, r, 5.114512081637298353406e-02f);
    num = __fmaf_rn(num, r, 2.473615434895520810817e-01f);
    num = __fmaf_rn(num, r, 7.257664613233124478488e-01f);
    num = __fmaf_rn(num, r, 9.999999999980870924916e-01f);

    float den = __fmaf_rn(2.159509375685829852307e-02f, r, -2.742335390411667452936e-01f);
    den = __fmaf_rn(den, r, 1.0f);

    const float quot = __fdiv_rn(num, den);
    const int qi = (int)q;
    float y;
    if (qi > 127) {
        y = __fmul_rn(__fmul_rn(quot, 2.0f), __int_as_float((qi - 1 + 127) << 23));
    } else if (qi >= -126) {
        y = __fmul_rn(quot, __int_as_float((qi + 127) << 23));
    } else {
        // exact pre-scale into the normal range, then one rounding into denormals
        y = __fmul_rn(__fmul_rn(quot, __int_as_float((qi + 64 + 127) << 23)), __int_as_float((127 - 64) << 23));
    }
    if (is_nan) y = __int_as_float(0x7fc00000);
    if (is_hi) y = __int_as_float(0x7f800000);
    if (is_lo) y = 0.0f;
    return y;
}

}  // namespace b200moe
