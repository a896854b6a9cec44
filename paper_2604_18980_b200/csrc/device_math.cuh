// device_math.cuh -- bit-exact float semantics of the reference CPU path on
// sm_100a.
//
// The reference objects are compiled for baseline x86-64 (SSE2, no FMA) and
// call glibc libm.  This translation unit family is
// compiled with --fmad=false, -prec-div=true, -prec-sqrt=true and no
// -ftz, so plain C++ expressions below round exactly like SSE scalar code.
// What remains are
//   * std::min/max/clamp semantics (libstdc++: max(a,b)= a<b?b:a, ...);
//   * x86 cvttss2si for static_cast<int>(float) out of range (-> INT_MIN);
//   * glibc's logf / expf (table + polynomial algorithms of glibc 2.39,
//     IFUNC variants on x86-64).  They are re-evaluated here with the same
//     double-precision steps; tests/test_gpu_parity.py
//     (test_device_logf_matches_host_glibc, test_device_expf_matches_host_glibc)
//     pins them against the host libm on the GPU box.
#pragma once
#include <cstdint>

namespace agsx {

// ---- libstdc++ std::min / std::max / std::clamp ----------------------
__host__ __device__ __forceinline__ float smax(float a, float b) { return a < b ? b : a; }
__host__ __device__ __forceinline__ float smin(float a, float b) { return b < a ? b : a; }
__host__ __device__ __forceinline__ float sclamp(float v, float lo, float hi) {
    return smin(smax(v, lo), hi);
}
__host__ __device__ __forceinline__ double sclampd(double v, double lo, double hi) {
    const double m = v < lo ? lo : v;
    return hi < m ? hi : m;
}
__host__ __device__ __forceinline__ int imax(int a, int b) { return a < b ? b : a; }
__host__ __device__ __forceinline__ int imin(int a, int b) { return b < a ? b : a; }

// x86-64 cvttss2si: NaN / out of range -> INT_MIN (0x80000000).
__host__ __device__ __forceinline__ int f2i_x86(float v) {
    if (!(v > -2147483904.0f && v < 2147483648.0f)) return INT32_MIN;
    return static_cast<int>(v);
}

// ---- glibc logf (sysdeps/ieee754/flt-32/e_logf.c algorithm) -----------
// 16-entry table {1/c, log(c)} and degree-3 polynomial in r = z/c - 1.
struct LogfTab {
    double invc, logc;
};
__device__ __constant__ static const LogfTab kLogfTab[16] = {
    {0x1.661ec79f8f3bep+0, -0x1.57bf7808caadep-2}, {0x1.571ed4aaf883dp+0, -0x1.2bef0a7c06ddbp-2},
    {0x1.49539f0f010b0p+0, -0x1.01eae7f513a67p-2}, {0x1.3c995b0b80385p+0, -0x1.b31d8a68224e9p-3},
    {0x1.30d190c8864a5p+0, -0x1.6574f0ac07758p-3}, {0x1.25e227b0b8ea0p+0, -0x1.1aa2bc79c8100p-3},
    {0x1.1bb4a4a1a343fp+0, -0x1.a4e76ce8c0e5ep-4}, {0x1.12358f08ae5bap+0, -0x1.1973c5a611cccp-4},
    {0x1.0953f419900a7p+0, -0x1.252f438e10c1ep-5}, {0x1.0000000000000p+0, 0x0p+0},
    {0x1.e608cfd9a47acp-1, 0x1.aa5aa5df25984p-5}, {0x1.ca4b31f026aa0p-1, 0x1.c5e53aa362eb4p-4},
    {0x1.b2036576afce6p-1, 0x1.526e57720db08p-3}, {0x1.9c2d163a1aa2dp-1, 0x1.bc2860d224770p-3},
    {0x1.886e6037841edp-1, 0x1.1058bc8a07ee1p-2}, {0x1.767dcf5534862p-1, 0x1.4043057b6ee09p-2},
};

__device__ __forceinline__ float glibc_logf(float x) {
    uint32_t ix = __float_as_uint(x);
    if (ix == 0x3f800000u) return 0.0f;
    if (ix - 0x00800000u >= 0x7f800000u - 0x00800000u) {
        // x < 0x1p-126, inf or nan
        if (ix * 2u == 0u) return __int_as_float(0xff800000);  // log(+-0) = -inf
        if (ix == 0x7f800000u) return x;                        // log(inf) = inf
        if ((ix & 0x80000000u) || ix * 2u >= 0xff000000u) return __int_as_float(0x7fc00000);
        ix = __float_as_uint(x * 0x1p23f);  // subnormal: normalise
        ix -= 23u << 23;
    }
    const uint32_t tmp = ix - 0x3f330000u;
    const int i = (tmp >> 19) % 16;
    const int k = static_cast<int32_t>(tmp) >> 23;
    const uint32_t iz = ix - (tmp & 0xff800000u);
    const double invc = kLogfTab[i].invc, logc = kLogfTab[i].logc;
    const double z = static_cast<double>(__uint_as_float(iz));
    const double r = z * invc - 1.0;
    const double y0 = logc + static_cast<double>(k) * 0x1.62e42fefa39efp-1;
    const double r2 = r * r;
    double y = 0x1.5575b0be00b6ap-2 * r + -0x1.ffffef20a4123p-2;
    y = -0x1.00ea348b88334p-2 * r2 + y;
    y = y * r2 + (y0 + r);
    return static_cast<float>(y);
}

// ---- glibc expf (sysdeps/ieee754/flt-32/e_expf.c algorithm) ------------
// exp(x) = 2^(k/32) * 2^(r/32); table entries bits(2^(i/32)) - (i << 47),
// (the table of glibc 2.39's __exp2f_data; SURVEY.md Appendix A gives its
// libm offset and how to regenerate it from correctly rounded 2^(i/32)).
__device__ __constant__ static const uint64_t kExp2fTab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull,
};

__device__ __forceinline__ float glibc_expf(float x) {
    const uint32_t abstop = (__float_as_uint(x) >> 20) & 0x7ffu;
    if (abstop >= 0x42bu) {  // top12(88.0f): |x| >= 88 or nan
        if (__float_as_uint(x) == 0xff800000u) return 0.0f;
        if (abstop >= 0x7f8u) return x + x;
        if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);
        if (x < -0x1.9fe368p6f) return 0.0f;
    }
    const double xd = static_cast<double>(x);
    // glibc is built with FMA on x86-64 (IFUNC variant): r = fma(InvLn2N, x, -kd) etc.;
    // pinned against the host libm on every float in [-20, -0] (the decision
    // domain [ln tau, 0] and beyond) plus 3M samples over [-110, 88]
    // (test_device_expf_matches_host_glibc).
    double kd = fma(0x1.71547652b82fep+5, xd, 0x1.8p+52);
    const uint64_t ki = static_cast<uint64_t>(__double_as_longlong(kd));
    kd -= 0x1.8p+52;
    const double r = fma(0x1.71547652b82fep+5, xd, -kd);
    const uint64_t t = kExp2fTab[ki % 32] + (ki << 47);
    const double s = __longlong_as_double(static_cast<long long>(t));
    const double zz = fma(0x1.c6af84b912394p-20, r, 0x1.ebfce50fac4f3p-13);
    const double r2 = r * r;
    double y = fma(0x1.62e42ff0c52d6p-6, r, 1.0);
    y = fma(zz, r2, y);
    y = y * s;
    return static_cast<float>(y);
}

// Hardware 2^x (MUFU.EX2).
__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Hardware log2 (MUFU.LG2).
__device__ __forceinline__ float fast_log2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Hardware exp2 (MUFU.EX2), flush-to-zero for tiny results.
__device__ __forceinline__ float fast_exp(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * 1.4426950408889634f));
    return y;
}

}  // namespace agsx
