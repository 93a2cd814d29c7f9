/* c_api_demo.c: the Tiny-Twin channel library used from plain C through its C ABI
 * (include/tt_channel.h), with host buffers only: no CUDA headers, no Python.
 *
 * It streams NCALLS slot calls of C channels through tt_channel_apply_host, the
 * delay line carried between calls, and writes inputs and outputs to a binary file
 * that tests/test_c_api_demo.py checks against the oracle:
 *   int32 C, L, S, N_total, K;  uint64 seed;  float sigma;
 *   int32 delays[C][L];  float gains[C][K][L][2];  float x[C][N_total][2];  float y[C][N_total][2]
 *
 *   gcc -O2 -I include examples/c_api_demo.c -L paper_2601_08217_b200 -ltt \
 *       -Wl,-rpath,'$ORIGIN/../paper_2601_08217_b200' -o examples/c_api_demo
 *   examples/c_api_demo out.bin
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "tt_channel.h"

enum { C = 6, L = 5, S = 64, NCALL = 3000, NCALLS = 4 };

/* a small deterministic generator for the demo's inputs (not the library's noise) */
static uint64_t lcg_state = 0x9E3779B97F4A7C15ull;
static float uniform_pm1(void) {
    lcg_state = lcg_state * 6364136223846793005ull + 1442695040888963407ull;
    return (float)((double)(lcg_state >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0);
}

static int check(tt_status s, const char* what) {
    if (s != TT_OK) {
        fprintf(stderr, "%s failed: %s (%s)\n", what, tt_status_string(s), tt_last_error());
        return 1;
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 2) {
        fprintf(stderr, "usage: %s out.bin\n", argv[0]);
        return 2;
    }
    const int32_t N = NCALL * NCALLS;
    const int32_t K = (N - 1) / S + 2; /* snapshots 0 .. K-1 cover every interval */
    const uint64_t seed = 20260108217ull;
    const float sigma = 0.05f;
    int32_t delays[C][L];
    for (int c = 0; c < C; ++c)
        for (int l = 0; l < L; ++l) delays[c][l] = l * 7 + c; /* distinct, up to 34 samples */
    float* gains = malloc(sizeof(float) * C * K * L * 2);
    float* x = malloc(sizeof(float) * C * N * 2);
    float* y = malloc(sizeof(float) * C * N * 2);
    float* xs = malloc(sizeof(float) * C * NCALL * 2); /* one call's input, [C][n][2] */
    float* ys = malloc(sizeof(float) * C * NCALL * 2);
    if (!gains || !x || !y || !xs || !ys) return 3;
    for (size_t i = 0; i < (size_t)C * K * L * 2; ++i) gains[i] = 0.5f * uniform_pm1();
    for (size_t i = 0; i < (size_t)C * N * 2; ++i) x[i] = uniform_pm1();

    printf("libtt ABI %d\n", tt_abi_version());
    tt_channel_t h = NULL;
    if (check(tt_channel_create(&h, C, L, &delays[0][0], S, seed, K, 0), "tt_channel_create")) return 1;
    /* host-memory snapshots: the library stages them to the device */
    if (check(tt_channel_load_snapshots(h, gains, 0, K, NULL), "tt_channel_load_snapshots")) return 1;
    for (int k = 0; k < NCALLS; ++k) {
        for (int c = 0; c < C; ++c)
            memcpy(xs + (size_t)c * NCALL * 2, x + ((size_t)c * N + (size_t)k * NCALL) * 2, sizeof(float) * NCALL * 2);
        /* host buffers in and out; the output is complete once the stream (here the
         * default one) reaches this point */
        if (check(tt_channel_apply_host(h, xs, ys, NCALL, sigma, NULL), "tt_channel_apply_host")) return 1;
        if (check(tt_channel_synchronize(h, NULL), "tt_channel_synchronize")) return 1;
        for (int c = 0; c < C; ++c)
            memcpy(y + ((size_t)c * N + (size_t)k * NCALL) * 2, ys + (size_t)c * NCALL * 2, sizeof(float) * NCALL * 2);
        tt_channel_info info;
        if (check(tt_channel_get_info(h, &info), "tt_channel_get_info")) return 1;
        if (info.t != (int64_t)(k + 1) * NCALL) {
            fprintf(stderr, "stream position %lld after call %d\n", (long long)info.t, k);
            return 1;
        }
    }
    if (check(tt_channel_destroy(h), "tt_channel_destroy")) return 1;

    FILE* f = fopen(argv[1], "wb");
    if (!f) return 4;
    const int32_t hdr[5] = {C, L, S, N, K};
    fwrite(hdr, sizeof(hdr), 1, f);
    fwrite(&seed, sizeof(seed), 1, f);
    fwrite(&sigma, sizeof(sigma), 1, f);
    fwrite(delays, sizeof(delays), 1, f);
    fwrite(gains, sizeof(float), (size_t)C * K * L * 2, f);
    fwrite(x, sizeof(float), (size_t)C * N * 2, f);
    fwrite(y, sizeof(float), (size_t)C * N * 2, f);
    fclose(f);
    printf("wrote %s: %d channels x %d samples in %d calls\n", argv[1], C, N, NCALLS);
    return 0;
}
