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

// Two samples at once, (a0, b0) and (a1, b1): the same operation sequence as
// noise_from_words on each, with the floating-point steps packed into FFMA2 / FMUL2 /
// FADD2 (per component exactly __fmaf_rn / __fmul_rn / __fadd_rn, so the results are
// bit-identical) to halve their issue slots. ptxas contracts an FMUL2 that feeds an
// FADD2 into one FFMA2 even with .rn; the two such pairs here (m - 1 and 1 - phi) have
// exact products (scaling by a power of two), so the contraction does not change them.
__device__ __forceinline__ void noise_from_words2(uint32_t a0, uint32_t b0, uint32_t a1, uint32_t b1, float sc,
                                                  float2& w0, float2& w1) {
    // radius: rho = sqrt(-2 ln u), u = ((a >> 8) + 1) 2^-24
    const uint32_t A0 = (a0 >> 8) + 1u, A1 = (a1 >> 8) + 1u;
    const int e0 = 31 - __clz(A0), e1 = 31 - __clz(A1);
    float2 m = __fmul2_rn(make_float2(__uint2float_rn(A0), __uint2float_rn(A1)),
                          make_float2(__int_as_float((127 - e0) << 23), __int_as_float((127 - e1) << 23)));
    const bool h0 = m.x > 0x1.6a09e6p+0f, h1 = m.y > 0x1.6a09e6p+0f;
    const float2 mh = __fmul2_rn(m, make_float2(0.5f, 0.5f));
    m = make_float2(h0 ? mh.x : m.x, h1 ? mh.y : m.y);
    const int E0 = e0 - 24 + (h0 ? 1 : 0), E1 = e1 - 24 + (h1 ? 1 : 0);
    const float2 f = __fadd2_rn(m, make_float2(-1.0f, -1.0f));  // fsub_rn(m, 1) == fadd_rn(m, -1)
    auto c2 = [](float c) { return make_float2(c, c); };
    float2 q = c2(-0x1.321a4cp-4f);
    q = __ffma2_rn(q, f, c2(0x1.068b2ap-3f));
    q = __ffma2_rn(q, f, c2(-0x1.0f9b0cp-3f));
    q = __ffma2_rn(q, f, c2(0x1.22bf86p-3f));
    q = __ffma2_rn(q, f, c2(-0x1.5424e0p-3f));
    q = __ffma2_rn(q, f, c2(0x1.999fc2p-3f));
    q = __ffma2_rn(q, f, c2(-0x1.000422p-2f));
    q = __ffma2_rn(q, f, c2(0x1.555558p-2f));
    q = __ffma2_rn(q, f, c2(-0x1.fffff8p-2f));
    const float2 r = __ffma2_rn(__fmul2_rn(f, f), q, f);
    const float2 Ef = make_float2(__int2float_rn(E0), __int2float_rn(E1));
    const float2 lnu = __ffma2_rn(Ef, c2(0x1.62e430p-1f), __ffma2_rn(Ef, c2(-0x1.05c610p-29f), r));
    const float2 v = __ffma2_rn(c2(-2.0f), lnu, c2(0.0f));
    const float rho0 = __fsqrt_rn(v.x), rho1 = __fsqrt_rn(v.y);
    // angle: (cos, sin) of pi/2 (q4 + phi)
    const uint32_t j0 = b0 >> 8, j1 = b1 >> 8;
    const uint32_t q40 = j0 >> 22, q41 = j1 >> 22;
    const float2 phi = __fmul2_rn(make_float2(__uint2float_rn(j0 & 0x3FFFFFu), __uint2float_rn(j1 & 0x3FFFFFu)),
                                  c2(0x1p-22f));
    const bool s0 = phi.x > 0.5f, s1 = phi.y > 0.5f;
    const float2 om = __fadd2_rn(c2(1.0f), make_float2(-phi.x, -phi.y));  // fsub_rn(1, phi)
    const float2 x = make_float2(s0 ? om.x : phi.x, s1 ? om.y : phi.y);
    const float2 x2 = __fmul2_rn(x, x);
    float2 ps = c2(0x1.4bdc50p-13f);
    ps = __ffma2_rn(ps, x2, c2(-0x1.32caf6p-8f));
    ps = __ffma2_rn(ps, x2, c2(0x1.466bbcp-4f));
    ps = __ffma2_rn(ps, x2, c2(-0x1.4abbcep-1f));
    ps = __ffma2_rn(ps, x2, c2(0x1.921fb6p+0f));
    const float2 sn2 = __fmul2_rn(x, ps);
    float2 pc = c2(0x1.d9f0a8p-11f);
    pc = __ffma2_rn(pc, x2, c2(-0x1.55c63cp-6f));
    pc = __ffma2_rn(pc, x2, c2(0x1.03c1dep-2f));
    pc = __ffma2_rn(pc, x2, c2(-0x1.3bd3ccp+0f));
    pc = __ffma2_rn(pc, x2, c2(0x1.000000p+0f));
    auto rot = [](bool swap, uint32_t q4, float s, float c, float& ct, float& st) {
        if (swap) {
            const float t = s;
            s = c;
            c = t;
        }
        const float cs = (q4 & 1u) ? s : c;
        const float sn = (q4 & 1u) ? c : s;
        ct = (q4 == 1u || q4 == 2u) ? -cs : cs;
        st = (q4 >= 2u) ? -sn : sn;
    };
    float ct0, st0, ct1, st1;
    rot(s0, q40, sn2.x, pc.x, ct0, st0);
    rot(s1, q41, sn2.y, pc.y, ct1, st1);
    w0 = __fmul2_rn(__fmul2_rn(make_float2(rho0, rho0), make_float2(ct0, st0)), c2(sc));
    w1 = __fmul2_rn(__fmul2_rn(make_float2(rho1, rho1), make_float2(ct1, st1)), c2(sc));
}

}  // namespace tt
