/*
 * tt_channel.h — C ABI of the B200-native Tiny-Twin channel convolution
 * (arXiv 2601.08217). This is the boundary of the hot path: the Python binding
 * (paper_2601_08217_b200/_lib.py), the tests and bench.py call exactly these
 * functions; every arithmetic step runs in the library's sm_100a kernels.
 *
 * Citations: "P:<n>" = PAPER.md line n; "S:<n>" = SPEC.md line n; "NS" =
 * BASELINE.json north_star; "R<k>" = reading k of the paper in DESIGN.md §3.
 *
 * What one handle computes (NS formula; §III-B "y_u(t) = x(t) * h_u(t)
 * ... the convolution operator * denotes linear convolution and varies
 * independently for each receiver"; §III-B "time-varying CIR traces ...
 * per-UE linear filtering"; §IV "discrete complex tap values over time ...
 * on a fixed delay grid"):
 *
 *   for every channel c of the handle and every global sample n of its stream
 *   (n counts from create/reset across all apply calls):
 *     k = floor(n / S), alpha = (n - k S) / S
 *     h_{c,l}[n] = g_{c,l,k} + alpha (g_{c,l,k+1} - g_{c,l,k})       (R1, R2)
 *     y_c[n] = sum_l h_{c,l}[n] x_c[n - d_{c,l}] + w_c[n],  x_c[m] = 0 for m < 0 (R4)
 *
 * with w_c[n] the AWGN of docs/tt-normal-v1.md keyed by (seed, channel_offset + c,
 * n). Arithmetic is float32 (FMA); taps are summed in ascending-delay order (ties
 * by tap index), so a channel's outputs are bit-identical for any split of its
 * stream into apply calls, any channel grouping and any GPU count.
 *
 * Data layout (all row-major, interleaved complex float32 = (re, im) pairs):
 *   delays  int32 [C][L]                  (host)
 *   gains   float [C][count][L][2]        (host or device)
 *   in/out  float [C][n_samples][2]       (device for tt_channel_apply,
 *                                           host for tt_channel_apply_host)
 * "UE" in this API means one directional channel stream: a UE's DL and UL are
 * two channels (c = 2u + dir), as in P:330's UE-localised DL+UL convolution.
 *
 * Errors: every call returns a tt_status and never aborts or prints; the
 * thread-local message of the last failure is tt_last_error(). A failed call
 * leaves the handle unchanged (apply: t is not advanced).
 * Threading: a handle is not thread-safe; calls on one handle must be
 * stream-ordered (use one stream per handle, or order them yourself).
 */
#ifndef TT_CHANNEL_H
#define TT_CHANNEL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TT_ABI_VERSION 2
#define TT_MAX_DELAY 4096  /* delays are integers in [0, TT_MAX_DELAY] (R5) */
#define TT_MAX_TAPS 4096

typedef struct tt_channel_s* tt_channel_t; /* opaque; owned by the library */
typedef void* tt_stream_t;                 /* a cudaStream_t (NULL = legacy default stream) */

typedef enum {
    TT_OK = 0,
    TT_ERR_INVALID_ARG = 1,      /* bad size, pointer, delay, period or sigma */
    TT_ERR_OUT_OF_MEMORY = 2,    /* a device or pinned allocation failed */
    TT_ERR_CUDA = 3,             /* a CUDA runtime call or launch failed (see tt_last_error) */
    TT_ERR_SNAPSHOT_MISSING = 4, /* apply needs a snapshot index that is not resident */
    TT_ERR_UNSUPPORTED = 5       /* e.g. no sm_100 device */
} tt_status;

typedef struct {
    int32_t num_ue;            /* C: channel streams in this handle */
    int32_t num_taps;          /* L */
    int32_t snapshot_period;   /* S */
    int32_t history;           /* H: delay-line samples kept per channel = max delay rounded up to 16, + 16 */
    int32_t max_delay;         /* max over all d_{c,l} */
    int32_t device;            /* CUDA device the handle is bound to */
    int64_t t;                 /* global index of the next sample to be applied */
    int64_t snapshot_capacity; /* ring slots per channel */
    int64_t resident_lo;       /* resident snapshot indices are [resident_lo, resident_hi) */
    int64_t resident_hi;
    int64_t channel_offset;    /* global id of channel 0 (noise key) */
    uint64_t seed;             /* noise key */
    int64_t device_bytes;      /* device memory owned by the handle */
    int32_t outputs_per_thread; /* outputs per thread of the selected kernel (0 = generic kernel) */
    int32_t launches_per_apply; /* kernel launches one tt_channel_apply enqueues */
    int32_t kernel;             /* TT_KERNEL_* the plan selected */
    int32_t top_n;              /* NEXT f2 taps per interval (0 = dense) */
    int32_t device_clock;       /* 1 in device-clock mode (tt_channel_set_device_clock); t is then stale */
} tt_channel_info;

/* kernels a plan can select (all compute the same per-output operation sequence, so
 * their outputs are bit-identical; the environment variable TT_KERNEL=dw|rw|tiled|generic
 * read at create restricts the choice) */
#define TT_KERNEL_GENERIC 0 /* one thread per output, operands from global memory */
#define TT_KERNEL_TILED 1   /* TMA-staged tiles, lane-strided outputs, x from shared memory */
#define TT_KERNEL_RW 2      /* register-window kernel: 16 consecutive outputs per thread */
#define TT_KERNEL_DW 3      /* dense-window kernel (opt-in, TT_KERNEL=dw): 16 consecutive outputs
                               per thread from two 16-sample x blocks in registers, window and
                               outputs moved by 2-D TMA tensor copies (128-B swizzle); calls whose
                               start or length is not a multiple of 16 run the tiled kernel */

/* Create a handle for C = num_ue channels with L = num_taps taps each.
 *   delays: host int32 [C][L], each in [0, TT_MAX_DELAY]; duplicates allowed (the
 *     taps add, R6). The library copies them.
 *   snapshot_period: S >= 1 samples between gain snapshots (P:411's trace time step,
 *     R2); snapshot k is the gain at global sample k S.
 *   seed: noise key (docs/tt-normal-v1.md).
 *   snapshot_capacity: snapshot slots per channel kept on the device (>= 2); a ring.
 *   channel_offset: global id of this handle's channel 0 (so a sharded run keys
 *     noise by global channel, NS "keyed by (seed, UE, sample)").
 * Binds to the current CUDA device. Allocates: the ring C x capacity x L x 16 B (each
 * slot holds (g_k, g_{k+1} - g_k) per tap, taps sorted by delay), the
 * delay-line history 2 x C x H x 8 B, and small per-channel tables; zeroes the
 * history (R4) and sets t = 0.
 * Errors: INVALID_ARG (out == NULL, C <= 0, L <= 0 or > TT_MAX_TAPS, delays == NULL,
 *   a delay outside [0, TT_MAX_DELAY], S <= 0, capacity < 2, channel_offset < 0),
 *   UNSUPPORTED (current device is not compute capability 10.x), OUT_OF_MEMORY, CUDA. */
tt_status tt_channel_create(tt_channel_t* out, int32_t num_ue, int32_t num_taps, const int32_t* delays,
                            int32_t snapshot_period, uint64_t seed, int64_t snapshot_capacity,
                            int64_t channel_offset);

/* Load gain snapshots first_index .. first_index+count-1 of every channel
 * ("read time-varying CIR traces"; "discrete complex tap values over
 * time") into the ring. gains: float [C][count][L][2], host or device memory (the
 * library detects which); the copy is enqueued on `stream` and the source must stay
 * valid until it completes there. A host source is staged through one device buffer
 * owned by the handle; loads on different streams are ordered on that buffer (a
 * load waits for the previous load's kernel to have read it). If the new block is contiguous with the resident
 * range the range grows (older snapshots fall out once capacity is exceeded);
 * otherwise the resident range is replaced by the new block. A block that starts
 * inside the resident range may also end inside it (a reload of snapshots already
 * resident): the snapshots after it stay resident and the interpolation across the
 * block's both ends uses the new values (the differences to the resident neighbours
 * first-1 and first+count are recomputed).
 * Errors: INVALID_ARG (NULL handle/gains, first_index < 0, count <= 0,
 *   count > capacity), CUDA. */
tt_status tt_channel_load_snapshots(tt_channel_t h, const float* gains, int64_t first_index, int64_t count,
                                    tt_stream_t stream);

/* Apply the channel to the next n_samples samples of every channel's stream:
 * in/out: device float [C][n_samples][2]; in and out must not overlap. One kernel
 * launch on `stream`; no synchronisation, no allocation. Carries the delay line:
 * y of this call uses the last H input samples of the previous calls (zeros at
 * stream start), "ConvState ... carried tail". noise_sigma: complex
 * standard deviation of the AWGN (E|w|^2 = sigma^2); 0 = no noise (R8).
 * Needs snapshots floor(t/S) .. floor((t+n_samples-1)/S)+1 resident (R3).
 * On success t += n_samples.
 * Errors: INVALID_ARG (NULL handle/in/out, n_samples <= 0, in == out, sigma < 0 or
 *   not finite), SNAPSHOT_MISSING, CUDA (launch failure). */
tt_status tt_channel_apply(tt_channel_t h, const float* in, float* out, int64_t n_samples, float noise_sigma,
                           tt_stream_t stream);

/* NEXT f2 (§III-C "convolution is performed only with the top-n dominant taps at
 * each time step"): from now on each snapshot interval k sums only its top_n taps of
 * largest |g_{l,k}|^2 (float32 fl(re*re) + fl(im*im); ties to the smaller delay, then
 * the smaller tap index), in ascending-delay order, interpolated as usual (DESIGN.md
 * R20). top_n = 0 or >= L restores the dense sum (the default). Selection happens when
 * snapshots are loaded; this call also (re)selects every resident snapshot. Allocates
 * the compacted ring (C x capacity x top_n x 20 B). Synchronises the device.
 * Errors: INVALID_ARG (NULL handle, top_n < 0), OUT_OF_MEMORY, CUDA. */
tt_status tt_channel_set_top_n(tt_channel_t h, int32_t top_n);

/* NEXT f4 (§V: each UE "receive[s] and sum[s] signals from all neighboring gNB"
 * sources): let several channels ("links") read the same input stream. After this call
 * channel c reads row rows[c] of the `in` buffer of every apply call, which is then
 * float [num_rows][n_samples][2]; each link keeps its own delay line, gains and noise.
 * rows = NULL restores the identity (row c, num_rows = C). rows is host memory, copied.
 * Errors: INVALID_ARG (NULL handle, num_rows <= 0, a row outside [0, num_rows)), CUDA. */
tt_status tt_channel_set_input_map(tt_channel_t h, const int32_t* rows, int32_t num_rows);

#define TT_AGG_CHUNK 8 /* channels per partial sum of tt_channel_apply_aggregate */

/* NEXT f1 ("the gNB ... applies convolution independently for each UE ...
 * and only then aggregates them"; P:330 UE-localised convolution) and f4: apply the
 * channels and sum them in groups of group_size consecutive channels:
 *   agg[g][n] = sum_{c = g G}^{(g+1) G - 1} y_c[n]
 * where y_c is exactly what tt_channel_apply computes for channel c (noise included).
 * The sum is float32 in a fixed order (so it is bit-identical for any call split):
 * chunks of TT_AGG_CHUNK consecutive channels are summed in channel order, then the
 * chunk sums in chunk order. agg: device float [C / G][n_samples][2]. out: device
 * float [C][n_samples][2] for the per-channel outputs, or NULL (not stored). The input
 * map (tt_channel_set_input_map) applies. May allocate device scratch for the chunk
 * sums on first use or growth (like tt_channel_apply_host's staging); to capture it in
 * a CUDA graph, make one call of the same shape before the capture so no allocation
 * happens inside it.
 * Errors: as tt_channel_apply, plus INVALID_ARG (agg NULL, G <= 0, C % G != 0),
 * OUT_OF_MEMORY. */
tt_status tt_channel_apply_aggregate(tt_channel_t h, const float* in, float* out, float* agg, int32_t group_size,
                                     int64_t n_samples, float noise_sigma, tt_stream_t stream);

/* NEXT f3 (§IV: traces of "discrete complex tap values over time" on "a fixed
 * delay grid", 3GPP PDPs "with time variation synthesized via a Jakes-based Doppler
 * model"): synthesise gain snapshots first_index .. first_index+count-1 on the GPU, in
 * the layout tt_channel_load_snapshots takes (R21):
 *   path p of channel c: delay tau = path_delay[c][p] samples (fractional allowed, in
 *   [0, TT_MAX_DELAY - 1]), power w = path_power[c][p]; Jakes/Clarke sum of M =
 *   num_sinusoids sinusoids with arrival angles 2 pi (m + u_p) / M and Philox-drawn
 *   phases (key seed, counter (m, p, channel_offset + c, 0x5EEDF3)); Doppler nu =
 *   f_D S / f_s cycles per snapshot (0 <= nu < 0.5);
 *   the path's gain is split onto grid taps 2p, 2p+1 at delays floor(tau), floor(tau)+1
 *   with weights (1 - frac, frac) (so the handle has L = 2 num_paths taps).
 * path_delay, path_power: host float [C][P]. delays_out: host int32 [C][2P] receives
 * the grid delays (may be NULL). gains_out: device float [C][count][2P][2]. Enqueued on
 * `stream` (path_delay / path_power are copied before returning); uses a per-device
 * scratch the library keeps and grows on demand (not thread-safe across devices' calls
 * beyond an internal lock).
 * Errors: INVALID_ARG (NULL inputs, sizes, nu outside [0, 0.5), delays or powers out of
 * range), OUT_OF_MEMORY, CUDA. */
tt_status tt_synth_jakes(const float* path_delay, const float* path_power, int32_t num_ue, int32_t num_paths,
                         int32_t num_sinusoids, double nu, uint64_t seed, int64_t channel_offset, int64_t first_index,
                         int64_t count, int32_t* delays_out, float* gains_out, tt_stream_t stream);

/* Same as tt_channel_apply but `in` and `out` are HOST memory (pinned for full
 * overlap; pageable works but copies synchronously). The library pipelines
 * host->device copies, the kernel and device->host copies over channel chunks on
 * internal streams ordered after / before `stream`; out is complete when `stream`
 * reaches this point. Lazily allocates device staging (3 chunk buffers) on first use
 * or growth. Errors: as tt_channel_apply, plus OUT_OF_MEMORY, UNSUPPORTED (an input
 * map is set: use tt_channel_apply with device buffers). */
tt_status tt_channel_apply_host(tt_channel_t h, const float* in, float* out, int64_t n_samples, float noise_sigma,
                                tt_stream_t stream);

/* t = 0 and zero delay-line history; the resident snapshot range is kept. No device
 * work: calls at t = 0 read the delay line from a zero buffer (`stream` is used only in
 * device-clock mode, where the device clock is reset stream-ordered on it).
 * Errors: INVALID_ARG, CUDA. */
tt_status tt_channel_reset(tt_channel_t h, tt_stream_t stream);

/* Device-clock mode, for slot loops captured into a CUDA graph (SURVEY §7.3 item 6:
 * "allow CUDA-Graph capture of slot loops").
 *
 * A kernel launch bakes its arguments, so a captured tt_channel_apply would replay the
 * same stream position t and the same delay-line half. In device-clock mode the
 * position and the history parity live in device memory instead. Each apply's kernel
 * reads them after the previous grid has completed (programmatic dependent launch
 * wait), and the last CTA to finish advances them by n_samples. A graph of K slot calls
 * therefore replays the next K slots every time.
 *
 * enable = 1: stream-ordered on `stream`, copies the handle's (t, parity) to the device.
 *   Requires the tiled kernel plan (else UNSUPPORTED) and t % A == 0, where A = 32R of
 *   the plan (256 for the default tile). While enabled:
 *   - tt_channel_apply and tt_channel_apply_aggregate need n_samples % A == 0 (else
 *     UNSUPPORTED), so every call stays on the aligned fast path;
 *   - snapshot residency is not checked per call: the caller keeps the ring loaded for
 *     every slot a graph will replay;
 *   - tt_channel_apply_host and tt_channel_set_top_n return UNSUPPORTED;
 *   - tt_channel_get_info reports device_clock = 1 and a stale t;
 *   - tt_channel_reset also resets the device clock.
 * enable = 0: synchronises `stream` and reads the device clock back into the handle's
 *   t and parity (host-side validation resumes).
 * Calling with the current mode is a no-op. Errors: INVALID_ARG, UNSUPPORTED, CUDA. */
tt_status tt_channel_set_device_clock(tt_channel_t h, int32_t enable, tt_stream_t stream);

/* Block the calling host thread until all work enqueued on `stream` (NULL = the legacy
 * default stream) has completed, on the handle's device: lets C callers of the
 * host-buffer path read their output without the CUDA runtime. Errors: INVALID_ARG, CUDA. */
tt_status tt_channel_synchronize(tt_channel_t h, tt_stream_t stream);

/* Fill *info. Errors: INVALID_ARG. */
tt_status tt_channel_get_info(tt_channel_t h, tt_channel_info* info);

/* Synchronise the handle's device, free everything the handle owns. NULL is OK. */
tt_status tt_channel_destroy(tt_channel_t h);

/* Thread-local message describing the last failed call on this thread ("" if none). */
const char* tt_last_error(void);

/* Static name of a status code. */
const char* tt_status_string(tt_status s);

/* TT_ABI_VERSION the library was built with. */
int32_t tt_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TT_CHANNEL_H */
