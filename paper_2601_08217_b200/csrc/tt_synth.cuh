// tt_synth.cuh — NEXT f3: on-GPU channel-state synthesis (§IV: "3GPP
// statistical channels based on standardized PDPs ... time variation synthesized via a
// Jakes-based Doppler model"; traces are taps "onto a fixed delay grid"). DESIGN.md R21:
//
//   a_p(k) = M^-1/2 sum_m exp(j 2 pi (nu cos(theta_{p,m}) k + phi_{p,m}))
//   theta_{p,m} = 2 pi (m + u_p) / M,   g_p(k) = sqrt(w_p) a_p(k),
//   taps 2p, 2p+1 at delays floor(tau_p), floor(tau_p) + 1 get (1 - f) g_p, f g_p.
//
// with u_p, phi_{p,m} uniform draws from Philox4x32-10 (counter (m, p, c_g, 0x5EEDF3),
// key = seed; phi from word 0, u_p from word 1 of the m = 0 block). Written
// independently of oracle/tt_oracle.c from the same definition.
//
// Two kernels: a per-(channel, path, sinusoid) table of (Doppler frequency in cycles
// per snapshot, phase in revolutions) in double, then one thread per (channel, path,
// block of 32 snapshots) summing the M sinusoids. The block's starting phase
// nu cos(theta) k + phi is formed in double (one DFMA) and reduced to [0, 1)
// revolutions before a float sincospi, so long runs (k ~ 10^6) keep full accuracy.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tt_noise.cuh"

namespace tt {

__device__ __forceinline__ double unit_u24(uint32_t w) { return static_cast<double>(w >> 8) * (1.0 / 16777216.0); }

// tab[(c P + p) M + m] = (nu cos theta_{p,m}, phi_{p,m})
__global__ void tt_synth_table_kernel(int32_t C, int32_t P, int32_t M, double nu, uint32_t key0, uint32_t key1,
                                      int64_t c_offset, double2* __restrict__ tab) {
    const int64_t tot = static_cast<int64_t>(C) * P * M;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < tot;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t m = static_cast<int32_t>(e % M);
        const int64_t cp = e / M;
        const int32_t p = static_cast<int32_t>(cp % P);
        const int32_t c = static_cast<int32_t>(cp / P);
        const uint32_t cg = static_cast<uint32_t>(c_offset + c);
        const u32x4 r0 = philox4x32_10(0u, static_cast<uint32_t>(p), cg, 0x5EEDF3u, key0, key1);
        const u32x4 rm = philox4x32_10(static_cast<uint32_t>(m), static_cast<uint32_t>(p), cg, 0x5EEDF3u, key0, key1);
        const double up = unit_u24(r0.b);
        // cos(2 pi (m + u_p) / M) = cospi(2 (m + u_p) / M)
        const double f = nu * cospi(2.0 * (static_cast<double>(m) + up) / static_cast<double>(M));
        tab[e] = make_double2(f, unit_u24(rm.a));
    }
}

// gains [C][K][2P][2]: snapshots k0 + k of every path, split onto its two grid bins.
// One thread per (channel, path, block of 32 snapshots): each sinusoid's phasor is
// evaluated exactly (double phase reduction, float sincospi) at the block start and then
// advanced by its per-snapshot rotation exp(j 2 pi f) in float (32 complex multiplies),
// so the sum of M sinusoids over the block costs ~8 flops per term instead of a
// sincospi; the drift over 32 steps stays ~1e-6 relative.
constexpr int kSynthBlock = 32;
__global__ void __launch_bounds__(128) tt_synth_gain_kernel(int32_t C, int32_t P, int32_t M,
                                                            const double2* __restrict__ tab,
                                                            const float* __restrict__ tau,
                                                            const float* __restrict__ pw, int64_t k0, int64_t K,
                                                            float2* __restrict__ gains) {
    const int64_t nb = (K + kSynthBlock - 1) / kSynthBlock;
    const int64_t tot = static_cast<int64_t>(C) * P * nb;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < tot;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t p = static_cast<int32_t>(e % P);
        const int64_t cb = e / P;
        const int64_t b = cb % nb;
        const int32_t c = static_cast<int32_t>(cb / nb);
        const double2* t = tab + (static_cast<int64_t>(c) * P + p) * M;
        const double kb = static_cast<double>(k0 + b * kSynthBlock);
        float ar[kSynthBlock], ai[kSynthBlock];
#pragma unroll
        for (int i = 0; i < kSynthBlock; ++i) ar[i] = ai[i] = 0.f;
        for (int32_t m = 0; m < M; ++m) {
            const double2 fp = __ldg(t + m);
            double r = fma(fp.x, kb, fp.y);
            r -= floor(r);  // revolutions in [0, 1)
            float zs, zc, ws, wc;
            sincospif(2.0f * static_cast<float>(r), &zs, &zc);
            sincospif(static_cast<float>(2.0 * fp.x), &ws, &wc);
#pragma unroll
            for (int i = 0; i < kSynthBlock; ++i) {
                ar[i] += zc;
                ai[i] += zs;
                const float nc = __fmaf_rn(zc, wc, -zs * ws);
                zs = __fmaf_rn(zc, ws, zs * wc);
                zc = nc;
            }
        }
        const float tp = __ldg(tau + static_cast<int64_t>(c) * P + p);
        const float fr = tp - floorf(tp);
        const float amp = static_cast<float>(sqrt(static_cast<double>(__ldg(pw + static_cast<int64_t>(c) * P + p)) /
                                                  static_cast<double>(M)));
#pragma unroll
        for (int i = 0; i < kSynthBlock; ++i) {
            const int64_t k = b * kSynthBlock + i;
            if (k < K) {
                const float gr = amp * ar[i], gi = amp * ai[i];
                float2* row = gains + (static_cast<int64_t>(c) * K + k) * 2 * P;
                row[2 * p] = make_float2((1.f - fr) * gr, (1.f - fr) * gi);
                row[2 * p + 1] = make_float2(fr * gr, fr * gi);
            }
        }
    }
}

}  // namespace tt
