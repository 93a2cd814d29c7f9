// tt_noise.cuh — device implementation of docs/tt-normal-v1.md (Philox4x32-10 +
// fixed-arithmetic Box-Muller). Written independently of oracle/tt_oracle.c; both
// follow the spec document. Every floating-point step is an explicit round-to-
// nearest intrinsic so nvcc cannot contract or reorder it (bit-exact by spec).
#pragma once
#include <stdint.h>

namespace tt {

struct u32x4 {
    uint32_t a, b, c, d;
};

// Philox4x32-10 (Salmon et al., SC'11): 10 rounds, key bumped between rounds.
__device__ __forceinline__ u32x4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                               uint32_t k1) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint32_t lo0 = 0xD2511F53u * c0;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return {c0, c1, c2, c3};
}

// spec §2 "Radius": rho = sqrt(-2 ln u), u = ((a >> 8) + 1) 2^-24
__device__ __forceinline__ float normal_radius(uint32_t a) {
    const uint32_t A = (a >> 8) + 1u;
    const int e = 31 - __clz(A);
    // m = A * 2^-e, exact: A < 2^25 converts exactly, and 2^-e is a power of two
    float m = __fmul_rn(__uint2float_rn(A), __int_as_float((127 - e) << 23));
    int E = e - 24;
    if (m > 0x1.6a09e6p+0f) {
        m = __fmul_rn(m, 0.5f);
        E += 1;
    }
    const float f = __fsub_rn(m, 1.0f);
    float q = -0x1.321a4cp-4f;
    q = __fmaf_rn(q, f, 0x1.068b2ap-3f);
    q = __fmaf_rn(q, f, -0x1.0f9b0cp-3f);
    q = __fmaf_rn(q, f, 0x1.22bf86p-3f);
    q = __fmaf_rn(q, f, -0x1.5424e0p-3f);
    q = __fmaf_rn(q, f, 0x1.999fc2p-3f);
    q = __fmaf_rn(q, f, -0x1.000422p-2f);
    q = __fmaf_rn(q, f, 0x1.555558p-2f);
    q = __fmaf_rn(q, f, -0x1.fffff8p-2f);
    const float r = __fmaf_rn(__fmul_rn(f, f), q, f);
    const float Ef = __int2float_rn(E);
    const float lnu = __fmaf_rn(Ef, 0x1.62e430p-1f, __fmaf_rn(Ef, -0x1.05c610p-29f, r));
    const float v = __fmaf_rn(-2.0f, lnu, 0.0f);
    return __fsqrt_rn(v);
}

// spec §2 "Angle": (cos, sin) of pi/2 (q4 + phi)
__device__ __forceinline__ void normal_angle(uint32_t b, float& ct, float& st) {
    const uint32_t j = b >> 8;
    const uint32_t q4 = j >> 22;
    const float phi = __fmul_rn(__uint2float_rn(j & 0x3FFFFFu), 0x1p-22f);
    const bool swap = phi > 0.5f;
    const float x = swap ? __fsub_rn(1.0f, phi) : phi;
    const float x2 = __fmul_rn(x, x);
    float ps = 0x1.4bdc50p-13f;
    ps = __fmaf_rn(ps, x2, -0x1.32caf6p-8f);
    ps = __fmaf_rn(ps, x2, 0x1.466bbcp-4f);
    ps = __fmaf_rn(ps, x2, -0x1.4abbcep-1f);
    ps = __fmaf_rn(ps, x2, 0x1.921fb6p+0f);
    float s = __fmul_rn(x, ps);
    float pc = 0x1.d9f0a8p-11f;
    pc = __fmaf_rn(pc, x2, -0x1.55c63cp-6f);
    pc = __fmaf_rn(pc, x2, 0x1.03c1dep-2f);
    pc = __fmaf_rn(pc, x2, -0x1.3bd3ccp+0f);
    pc = __fmaf_rn(pc, x2, 0x1.000000p+0f);
    float c = pc;
    if (swap) {
        const float t = s;
        s = c;
        c = t;
    }
    // quadrant rotation: exact negations / swaps
    const float cs = (q4 & 1u) ? s : c;   // |cos theta|
    const float sn = (q4 & 1u) ? c : s;   // |sin theta|
    ct = (q4 == 1u || q4 == 2u) ? -cs : cs;
    st = (q4 >= 2u) ? -sn : sn;
}

// spec §2 output + §3 scaling: one complex noise sample from a word pair
__device__ __forceinline__ float2 noise_from_words(uint32_t a, uint32_t b, float sc) {
    const float rho = normal_radius(a);
    float ct, st;
    normal_angle(b, ct, st);
    return make_float2(__fmul_rn(__fmul_rn(rho, ct), sc), __fmul_rn(__fmul_rn(rho, st), sc));
}

}  // namespace tt
