/*
 * tt_oracle.c — THE ORACLE. Test infrastructure only.
 *
 * A plain, slow, obviously-correct CPU implementation of what the Tiny-Twin hot
 * path computes (arXiv 2601.08217). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library. The
 * product path (paper_2601_08217_b200/) never links, imports or executes it, and
 * this file includes nothing from the product path.
 *
 * Citations: "P:<line>" = /root/reference/PAPER.md line; "S:<line>" = SPEC.md line;
 * "NS" = BASELINE.json north_star; "R<k>" = reading k in DESIGN.md §3.
 *
 * What it computes (the plain definition, NS formula; §III-B "y_u(t) =
 * x(t) * h_u(t) ... linear convolution"; §III-B time-varying multi-tap CIR
 * traces; §IV discrete complex taps on a fixed delay grid over time):
 *
 *   for channel c, global sample n >= 0 of the channel's stream:
 *     x_c[m] = 0 for m < 0                       (zero delay line at start, R4)
 *     k = floor(n / S), j = n - k S, alpha = j / S           (R2)
 *     h_{c,l}[n] = g_{c,l,k} + alpha (g_{c,l,k+1} - g_{c,l,k})  (output-time index, R1)
 *     y_c[n] = sum_l h_{c,l}[n] x_c[n - d_{c,l}] + w_c[n]
 *
 * in double precision (float32 inputs promoted exactly), with w_c[n] the float32
 * noise sample of docs/tt-normal-v1.md added in double. There is no streaming
 * state: any output is computed from the stored input stream directly.
 *
 * Parity pins (tests/test_oracle_*.py, -m "not gpu"):
 *   philox      : cuRAND host Philox4x32-10 generator + Random123 known-answer vector
 *   normal pair : exhaustive 2^24-input accuracy vs double libm; moment statistics
 *   convolve    : identity (L=1,d=0,g=1), pure delay, scalar fading piecewise-linear
 *                 closed form, unit-impulse time-index convention, numpy.convolve for
 *                 time-invariant taps, pure-Python brute force, linearity, streaming
 *                 window independence, received-power closed form.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math -shared -fPIC (no
 * contraction, so float steps of tt-normal-v1 round exactly as specified).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TTO_OK 0
#define TTO_EINVAL -1
#define TTO_EXMISSING -2
#define TTO_ESNAPMISSING -3

/* ---------------------------------------------------------------------------
 * Philox4x32-10 (Salmon et al., SC'11), docs/tt-normal-v1.md §1.
 * ------------------------------------------------------------------------- */
static void mulhilo32(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo) {
    uint64_t p = (uint64_t)a * (uint64_t)b;
    *hi = (uint32_t)(p >> 32);
    *lo = (uint32_t)p;
}

void tto_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo32(0xD2511F53u, c0, &hi0, &lo0);
        mulhilo32(0xCD9E8D57u, c2, &hi1, &lo1);
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ---------------------------------------------------------------------------
 * tt-normal-v1 (docs/tt-normal-v1.md §2), step by step in the document's order.
 * ------------------------------------------------------------------------- */
static const float LNQ[9] = {
    -0x1.fffff8p-2f, 0x1.555558p-2f, -0x1.000422p-2f, 0x1.999fc2p-3f, -0x1.5424e0p-3f,
    0x1.22bf86p-3f, -0x1.0f9b0cp-3f, 0x1.068b2ap-3f, -0x1.321a4cp-4f};
static const float LN2_HI = 0x1.62e430p-1f;
static const float LN2_LO = -0x1.05c610p-29f;
static const float SQRT2F = 0x1.6a09e6p+0f;
static const float SINP[5] = {0x1.921fb6p+0f, -0x1.4abbcep-1f, 0x1.466bbcp-4f, -0x1.32caf6p-8f,
                              0x1.4bdc50p-13f};
static const float COSP[5] = {0x1.000000p+0f, -0x1.3bd3ccp+0f, 0x1.03c1dep-2f, -0x1.55c63cp-6f,
                              0x1.d9f0a8p-11f};

/* radius rho = sqrt(-2 ln u), u = ((a >> 8) + 1) 2^-24 */
float tto_radius(uint32_t a) {
    uint32_t A = (a >> 8) + 1u;                 /* step 1 */
    int e = 31;                                 /* step 2: e = 31 - clz(A) */
    while (!(A & (1u << e))) --e;
    float m = ldexpf((float)A, -e);             /* exact */
    int E = e - 24;
    if (m > SQRT2F) { m = m * 0.5f; E = E + 1; } /* step 3 */
    float f = m - 1.0f;                         /* step 4 */
    float q = LNQ[8];                           /* step 5 */
    for (int i = 7; i >= 0; --i) q = fmaf(q, f, LNQ[i]);
    float ff = f * f;                           /* step 6 */
    float r = fmaf(ff, q, f);
    float Ef = (float)E;                        /* step 7 */
    float lnu = fmaf(Ef, LN2_HI, fmaf(Ef, LN2_LO, r));
    float v = fmaf(-2.0f, lnu, 0.0f);           /* step 8 */
    return sqrtf(v);
}

/* (cos theta, sin theta), theta = pi/2 (q4 + phi) */
void tto_angle(uint32_t b, float* cos_t, float* sin_t) {
    uint32_t j = b >> 8;                        /* step 1 */
    uint32_t q4 = j >> 22;
    float phi = ldexpf((float)(j & 0x3FFFFFu), -22);
    float x;                                    /* step 2 */
    int swap;
    if (phi > 0.5f) { x = 1.0f - phi; swap = 1; } else { x = phi; swap = 0; }
    float x2 = x * x;                           /* step 3 */
    float ps = SINP[4];                         /* step 4 */
    for (int i = 3; i >= 0; --i) ps = fmaf(ps, x2, SINP[i]);
    float s = x * ps;
    float pc = COSP[4];                         /* step 5 */
    for (int i = 3; i >= 0; --i) pc = fmaf(pc, x2, COSP[i]);
    float c = pc;
    if (swap) { float t = s; s = c; c = t; }    /* step 6 */
    float ct, st;                               /* step 7 */
    switch (q4) {
        case 0: ct = c; st = s; break;
        case 1: ct = -s; st = c; break;
        case 2: ct = -c; st = -s; break;
        default: ct = s; st = -c; break;
    }
    *cos_t = ct;
    *sin_t = st;
}

void tto_normal_pair(uint32_t a, uint32_t b, float z[2]) {
    float rho = tto_radius(a);
    float ct, st;
    tto_angle(b, &ct, &st);
    z[0] = rho * ct;
    z[1] = rho * st;
}

/* docs/tt-normal-v1.md §3 */
float tto_noise_scale(float sigma) { return (float)((double)sigma * 0x1.6a09e667f3bcdp-1); }

void tto_noise_sample(uint64_t seed, int64_t c_global, int64_t n, float sc, float w[2]) {
    uint64_t m = (uint64_t)n >> 1;
    uint32_t ctr[4] = {(uint32_t)m, (uint32_t)(m >> 32), (uint32_t)(uint64_t)c_global, 0u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t r[4];
    tto_philox4x32_10(ctr, key, r);
    float z[2];
    if ((n & 1) == 0) tto_normal_pair(r[0], r[1], z);
    else tto_normal_pair(r[2], r[3], z);
    w[0] = z[0] * sc;
    w[1] = z[1] * sc;
}

/* Batch helpers for the exhaustive accuracy pins (radius over all A in [1, 2^24],
 * angle over all j in [0, 2^24)). */
void tto_radius_all(float* out /* [2^24] */) {
#pragma omp parallel for schedule(static)
    for (int64_t A = 1; A <= (1 << 24); ++A) out[A - 1] = tto_radius((uint32_t)((A - 1) << 8));
}
void tto_angle_all(float* out /* [2^24][2] = (cos, sin) */) {
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < (1 << 24); ++j) tto_angle((uint32_t)(j << 8), &out[2 * j], &out[2 * j + 1]);
}
void tto_noise_block(uint64_t seed, int64_t c_global, int64_t n0, int64_t N, float sigma,
                     float* w /* [N][2] */) {
    float sc = tto_noise_scale(sigma);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i) tto_noise_sample(seed, c_global, n0 + i, sc, &w[2 * i]);
}

/* ---------------------------------------------------------------------------
 * NEXT f2: sparse top-n taps (§III-C "convolution is performed only with the
 * top-n dominant taps at each time step"). DESIGN.md reading R20: the time
 * step is the snapshot interval; interval k uses the n taps of largest |g_{l,k}| (its
 * opening snapshot); "dominant" is compared on m_l = |g_{l,k}|^2 computed in float32
 * as fl(fl(re*re) + fl(im*im)) (the decision is taken in the kernel's precision); ties
 * go to the smaller delay, then the smaller tap index ("ties broken toward
 * smaller bin index"). sel[l] = 1 iff fewer than n taps precede l in that order.
 * ------------------------------------------------------------------------- */
void tto_select_top_n(int32_t L, const int32_t* d, const float* g_row /* [L][2] */, int32_t n,
                      uint8_t* sel /* [L] */) {
    for (int32_t l = 0; l < L; ++l) {
        float ml = g_row[2 * l] * g_row[2 * l] + g_row[2 * l + 1] * g_row[2 * l + 1];
        int32_t rank = 0;
        for (int32_t i = 0; i < L; ++i) {
            float mi = g_row[2 * i] * g_row[2 * i] + g_row[2 * i + 1] * g_row[2 * i + 1];
            int before = mi > ml || (mi == ml && (d[i] < d[l] || (d[i] == d[l] && i < l)));
            rank += before;
        }
        sel[l] = (uint8_t)(rank < n);
    }
}

/* ---------------------------------------------------------------------------
 * The convolution (NS formula). One output sample.
 * top_n in [1, L) restricts the sum to the taps tto_select_top_n picks for the
 * output's interval (f2); top_n <= 0 or >= L is the dense sum.
 * ------------------------------------------------------------------------- */
static int one_output(int32_t L, const int32_t* d /* [L] */, int32_t S,
                      const float* g /* [K][L][2] */, int64_t k0, int64_t K,
                      const float* x /* [Nx][2] */, int64_t x0, int64_t Nx,
                      int64_t n, float sc, uint64_t seed, int64_t c_global, int32_t top_n, double out[2]) {
    int64_t k = n / S;                     /* n >= 0: floor */
    int64_t j = n - k * S;
    double alpha = (double)j / (double)S;
    int64_t i0 = k - k0;
    if (i0 < 0 || i0 + 1 >= K) return TTO_ESNAPMISSING;
    uint8_t sel_buf[4096];
    const int sparse = top_n > 0 && top_n < L;
    if (sparse) {
        if (L > 4096) return TTO_EINVAL;
        tto_select_top_n(L, d, g + i0 * L * 2, top_n, sel_buf);
    }
    double yr = 0.0, yi = 0.0;
    for (int32_t l = 0; l < L; ++l) {
        if (sparse && !sel_buf[l]) continue;
        double g0r = g[(i0 * L + l) * 2], g0i = g[(i0 * L + l) * 2 + 1];
        double g1r = g[((i0 + 1) * L + l) * 2], g1i = g[((i0 + 1) * L + l) * 2 + 1];
        double hr = g0r + alpha * (g1r - g0r);
        double hi = g0i + alpha * (g1i - g0i);
        int64_t m = n - d[l];
        double xr = 0.0, xi = 0.0;
        if (m >= 0) {
            if (m < x0 || m >= x0 + Nx) return TTO_EXMISSING;
            xr = x[(m - x0) * 2];
            xi = x[(m - x0) * 2 + 1];
        }
        yr += hr * xr - hi * xi;
        yi += hr * xi + hi * xr;
    }
    if (sc != 0.0f) {
        float w[2];
        tto_noise_sample(seed, c_global, n, sc, w);
        yr += (double)w[0];
        yi += (double)w[1];
    }
    out[0] = yr;
    out[1] = yi;
    return TTO_OK;
}

static int check_common(int32_t C, int32_t L, const int32_t* delays, int32_t S, float sigma) {
    if (C <= 0 || L <= 0 || S <= 0 || !delays || !(sigma >= 0.0f) || isinf(sigma)) return TTO_EINVAL;
    for (int64_t i = 0; i < (int64_t)C * L; ++i)
        if (delays[i] < 0) return TTO_EINVAL;
    return TTO_OK;
}

/* Block form: outputs n0 .. n0+N-1 of every channel.
 *   delays [C][L]; gains [C][K][L][2] = snapshots k0 .. k0+K-1;
 *   x [C][Nx][2] = stream samples x0 .. x0+Nx-1; y [C][N][2] (double). */
int tto_convolve_topn(int32_t C, int32_t L, const int32_t* delays, int32_t S, const float* gains,
                      int64_t k0, int64_t K, const float* x, int64_t x0, int64_t Nx, int64_t n0,
                      int64_t N, float sigma, uint64_t seed, int64_t c_offset, int32_t top_n, double* y) {
    int st = check_common(C, L, delays, S, sigma);
    if (st) return st;
    if (n0 < 0 || N < 0 || K < 0 || Nx < 0 || x0 < 0) return TTO_EINVAL;
    float sc = sigma > 0.0f ? tto_noise_scale(sigma) : 0.0f;
    const int64_t B = 4096; /* time blocks, only to spread work over cores */
    int64_t nb = (N + B - 1) / B;
    int err = TTO_OK;
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
    for (int32_t c = 0; c < C; ++c) {
        for (int64_t b = 0; b < nb; ++b) {
            for (int64_t i = b * B; i < N && i < (b + 1) * B; ++i) {
                int r = one_output(L, delays + (int64_t)c * L, S, gains + (int64_t)c * K * L * 2, k0, K,
                                   x + (int64_t)c * Nx * 2, x0, Nx, n0 + i, sc, seed, c_offset + c, top_n,
                                   y + ((int64_t)c * N + i) * 2);
                if (r) {
#pragma omp atomic write
                    err = r;
                }
            }
        }
    }
    return err;
}

int tto_convolve(int32_t C, int32_t L, const int32_t* delays, int32_t S, const float* gains,
                 int64_t k0, int64_t K, const float* x, int64_t x0, int64_t Nx, int64_t n0,
                 int64_t N, float sigma, uint64_t seed, int64_t c_offset, double* y) {
    return tto_convolve_topn(C, L, delays, S, gains, k0, K, x, x0, Nx, n0, N, sigma, seed, c_offset, 0, y);
}

/* Point form: outputs at (cs[p], ns[p]), p < P; same input layouts; y [P][2]. */
int tto_convolve_points(int32_t C, int32_t L, const int32_t* delays, int32_t S, const float* gains,
                        int64_t k0, int64_t K, const float* x, int64_t x0, int64_t Nx,
                        const int32_t* cs, const int64_t* ns, int64_t P, float sigma, uint64_t seed,
                        int64_t c_offset, double* y) {
    int st = check_common(C, L, delays, S, sigma);
    if (st) return st;
    float sc = sigma > 0.0f ? tto_noise_scale(sigma) : 0.0f;
    int err = TTO_OK;
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < P; ++p) {
        int32_t c = cs[p];
        int r;
        if (c < 0 || c >= C || ns[p] < 0) r = TTO_EINVAL;
        else
            r = one_output(L, delays + (int64_t)c * L, S, gains + (int64_t)c * K * L * 2, k0, K,
                           x + (int64_t)c * Nx * 2, x0, Nx, ns[p], sc, seed, c_offset + c, 0, y + p * 2);
        if (r) {
#pragma omp atomic write
            err = r;
        }
    }
    return err;
}

/* ---------------------------------------------------------------------------
 * NEXT f3: channel-state synthesis (§IV: traces are "discrete complex tap
 * values over time" resampled "onto a fixed delay grid"; 3GPP PDPs with "time variation
 * synthesized via a Jakes-based Doppler model"). DESIGN.md reading R21, step by step:
 *   path p of channel c: fractional delay tau_p >= 0 (samples), power w_p;
 *   random numbers: Philox4x32-10 key (seed lo, seed hi),
 *     u_p      = U(word 1 of Philox(ctr = (0, p, c_g, 0x5EEDF3)))   angle offset
 *     phi_{p,m}= U(word 0 of Philox(ctr = (m, p, c_g, 0x5EEDF3)))   phase (revolutions)
 *     U(w) = (w >> 8) 2^-24 in [0, 1);
 *   theta_{p,m} = 2 pi (m + u_p) / M (M arrival angles, Clarke sum of sinusoids);
 *   nu = f_D S / f_s: Doppler in cycles per snapshot period;
 *   a_p(k) = M^-1/2 sum_m exp(j 2 pi (nu cos(theta_{p,m}) k + phi_{p,m}))
 *   g_p(k) = sqrt(w_p) a_p(k);
 *   two-bin split onto the integer grid: b = floor(tau_p), f = tau_p - b,
 *     tap 2p at delay b gets (1 - f) g_p(k), tap 2p+1 at delay b + 1 gets f g_p(k).
 * Everything in double; outputs rounded to float32 once.
 * ------------------------------------------------------------------------- */
static double u01(uint32_t w) { return (double)(w >> 8) * (1.0 / 16777216.0); }

void tto_synth_jakes(int32_t C, int32_t P, const float* tau /* [C][P] */, const float* pw /* [C][P] */,
                     int32_t M, double nu, uint64_t seed, int64_t c_offset, int64_t k0, int64_t K,
                     int32_t* delays /* [C][2P] */, float* gains /* [C][K][2P][2] */) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    const double PI = 3.14159265358979323846;
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t c = 0; c < C; ++c) {
        const uint32_t cg = (uint32_t)(c_offset + c);
        for (int32_t p = 0; p < P; ++p) {
            const double t = tau[c * P + p];
            const double b = floor(t), f = t - b;
            delays[(int64_t)c * 2 * P + 2 * p] = (int32_t)b;
            delays[(int64_t)c * 2 * P + 2 * p + 1] = (int32_t)b + 1;
            uint32_t ctr[4] = {0u, (uint32_t)p, cg, 0x5EEDF3u}, r[4];
            tto_philox4x32_10(ctr, key, r);
            const double up = u01(r[1]);
            const double amp = sqrt((double)pw[c * P + p] / (double)M);
            for (int64_t k = 0; k < K; ++k) {
                double ar = 0.0, ai = 0.0;
                for (int32_t m = 0; m < M; ++m) {
                    uint32_t cm[4] = {(uint32_t)m, (uint32_t)p, cg, 0x5EEDF3u}, rm[4];
                    tto_philox4x32_10(cm, key, rm);
                    const double phi = u01(rm[0]);
                    const double th = 2.0 * PI * ((double)m + up) / (double)M;
                    const double ph = 2.0 * PI * (nu * cos(th) * (double)(k0 + k) + phi);
                    ar += cos(ph);
                    ai += sin(ph);
                }
                const double gr = amp * ar, gi = amp * ai;
                float* row = gains + (((int64_t)c * K + k) * 2 * P) * 2;
                row[4 * p] = (float)((1.0 - f) * gr);
                row[4 * p + 1] = (float)((1.0 - f) * gi);
                row[4 * p + 2] = (float)(f * gr);
                row[4 * p + 3] = (float)(f * gi);
            }
        }
    }
}
