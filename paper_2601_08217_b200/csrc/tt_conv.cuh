// tt_conv.cuh — the sm_100a kernels of the Tiny-Twin channel convolution
// (arXiv 2601.08217; NS formula, §III-B, §IV).
//
//   y_c[n] = sum_l (g_{c,l,k} + alpha (g_{c,l,k+1} - g_{c,l,k})) x_c[n - d_{c,l}] + w_c[n]
//
// Design:
//  * data layout in HBM: the snapshot ring holds, per channel and snapshot k, one
//    float4 (g_k, g_{k+1} - g_k) per tap, taps sorted by delay — written once by
//    tt_load_kernel when snapshots are loaded — so a tile's coefficients are a
//    contiguous, directly stageable block;
//  * persistent, warp-specialised CTAs (one per SM): a producer warp walks the CTA's
//    (channel, tile) work items and stages everything a tile reads — the input window
//    x[i0 - H, i0 + T) (H = max-delay halo; the part before the call start comes from
//    the carried delay line), the coefficient rows of the intervals it touches, and
//    the channel's tap offsets H - d — into a ring of shared-memory stages with 1-D TMA
//    bulk copies (cp.async.bulk ... mbarrier::complete_tx); 16 consumer warps wait on
//    the stage's `full` mbarrier, compute, and release it on its `empty` mbarrier.
//    There is no CTA-wide barrier in the steady state;
//  * a tile is T = 16 warps x 32 lanes x R outputs of one channel; lane j of consumer
//    warp w owns outputs w*32R + r*32 + j, so every x read is a conflict-free 256-B
//    warp access and the warp's 32R outputs normally sit in one snapshot interval,
//    making the coefficient read a broadcast;
//  * taps run in groups of four with the next group's offsets prefetched; per tap the R
//    gains h = fma(alpha, dg, g) are formed first (FFMA2), then two packed FMAs per
//    output into split accumulators A += h_re x, B += h_im x; y = (A.re - B.im, A.im + B.re);
//  * optional AWGN (docs/tt-normal-v1.md) fused in the epilogue, one Philox call per
//    sample pair shared by neighbouring lanes via a shuffle, the Gaussian transform of
//    two samples packed into FFMA2/FMUL2/FADD2;
//  * the consumer warps of a channel's last tile write the new delay-line history from
//    the staged window into the other half of a ping-pong buffer;
//  * a ROBUST variant (chosen per call by the host) handles calls that do not start on
//    a 32R-aligned sample (a short lead-in tile) and input rows 8 B off a 16-B boundary
//    (a per-tile window shift), and can run on the device clock (stream position in
//    device memory, advanced by the last CTA) for CUDA-graph capture.
//
// Every output's operation sequence depends only on (channel, global n) — never on
// the tile, path or launch shape — so results are bit-identical across partitions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tt_noise.cuh"

namespace tt {

constexpr int kConsumerWarps = 16;                   // default tile shape: 16 consumer warps
constexpr int kThreads = (kConsumerWarps + 1) * 32;  // + 1 producer warp
constexpr int kMaxStages = 4;
#ifndef TT_V
#define TT_V 0  // kernel variant hook for A/B builds (tools/build_variants.sh); 0 = the product
#endif
// The noise add stays two scalar __fadd_rn: ptxas contracts an FMUL2 feeding an FADD2
// into one FFMA2 even with .rn (checked in SASS), which would fuse the noise scaling
// w = (rho (cos, sin)) sc into the add and change the rounding.
__device__ __forceinline__ float2 add_noise(float2 a, float2 w) {
    return make_float2(__fadd_rn(a.x, w.x), __fadd_rn(a.y, w.y));
}
// y = A + i B for A = sum h.re x, B = sum h.im x: (A.x - B.y, A.y + B.x) as one FFMA2
// with exact +-1 products, per component the rounding of __fsub_rn / __fadd_rn.
__device__ __forceinline__ float2 combine(float2 a, float2 b) {
    return __ffma2_rn(make_float2(b.y, b.x), make_float2(-1.f, 1.f), a);
}

// Stream position kept in device memory (tt_channel_set_device_clock): the kernel
// reads t and the history parity at its start and its last CTA advances them, so a
// captured CUDA graph of slot calls replays correctly.
struct DevClock {
    int64_t t;      // global index of the next call's first sample
    int32_t par;    // history buffer holding the current delay line
    uint32_t done;  // CTAs of the running call that have finished (last one advances)
};

struct ConvParams {
    const float2* x;        // [rows][n]: row of channel c = in_row ? in_row[c] : c - c_lo
    float2* y;              // [C_launch][n] per-channel outputs, or nullptr (aggregate only)
    const int32_t* in_row;  // [C] input row per channel (NEXT f4: links share a gNB stream), or nullptr
    float2* agg;            // group sums [groups][n] (nchunks == 1) or partials [groups][nchunks][n]; or nullptr
    int32_t group;          // G channels summed per group (1 = no aggregation)
    int32_t chunk;          // KC channels per chunk (partial sum in one CTA, in channel order)
    int32_t nchunks;        // ceil(G / KC)
    int64_t total_super;    // groups * nchunks * tiles_per_ch work items
    const float2* hist_rd;  // [C][H]  last H samples of the stream so far
    float2* hist_wr;        // [C][H]  written with the new history
    const float4* ring;     // [C][cap][L] (g_k, g_{k+1} - g_k), taps sorted by delay
    const int32_t* xoff;    // [C][L4] window offset H - d_j of sorted tap j (pads: 0)
    const int32_t* xoff_rows;  // NEXT f2 sparse: [C][cap][L4] offsets of each interval's selected
                               // taps (then `ring` holds [C][cap][L] compacted rows, L = top-n); or nullptr
    int64_t n;              // samples per channel in this call
    int64_t t;              // global index of the call's first sample
    int64_t cap;            // ring slots per channel
    int64_t chan_offset;    // global id of channel 0 (noise key)
    int64_t total_tiles;    // (c_hi - c_lo) * tiles_per_ch (channel tiles)
    int64_t t_div;          // t / S
    int32_t t_mod;          // t % S
    int32_t c_lo;           // first channel of this launch
    int32_t tiles_per_ch;
    int32_t lead;           // outputs in a short first tile that aligns the others (0 = none)
    int32_t L, L4, H, S;
    int32_t nk_max;         // max snapshot intervals a tile touches
    int32_t stages;         // shared-memory pipeline depth (<= kMaxStages)
    uint32_t key0, key1;    // noise key
    float noise_sc;         // sigma / sqrt(2) as float; 0 = no noise
    int32_t s_shift;        // log2(S) if S is a power of two, else -1
    float inv_S;            // 1/S (exact when S is a power of two)
    DevClock* clk;          // device clock (ROBUST variant only), or nullptr: t/history from above
    float2* hist_base;      // [2][C][H] history ping-pong (device-clock mode picks the half)
    const float2* hist_zero;  // [C][H] zeros, the delay line at t = 0
    int64_t hist_half;      // C * H
};

// ---------------------------------------------------------------------------------
// PTX helpers: mbarrier + 1-D TMA bulk copy (global -> shared)
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t a = smem_u32(bar);
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// A global -> shared copy of `bytes` (a multiple of 8) split into a TMA body that is
// 16-B aligned at both ends and at most one 8-B element before / after it; a copy whose
// ends cannot both be aligned is all plain (8-B loads).
struct Piece {
    const unsigned char* src;
    unsigned char* dst;
    uint32_t bytes;
    uint32_t head, body;  // plain bytes before the body (0 or 8), TMA body bytes
};
__device__ __forceinline__ Piece make_piece(void* dst, const void* src, uint32_t bytes) {
    Piece pc{static_cast<const unsigned char*>(src), static_cast<unsigned char*>(dst), bytes, 0u, 0u};
    if (bytes == 0) return pc;
    const uintptr_t sa = reinterpret_cast<uintptr_t>(src);
    if (((sa ^ smem_u32(dst)) & 15u) != 0) return pc;
    pc.head = (sa & 15u) ? 8u : 0u;
    const uint32_t body = (bytes - pc.head) & ~15u;
    pc.body = body >= 16u ? body : 0u;
    if (pc.body == 0) pc.head = 0;
    return pc;
}
// plain part of a piece, spread over the producer warp's lanes
__device__ __forceinline__ void piece_plain(const Piece& pc, int lane) {
    if (pc.body == 0) {
        for (uint32_t o = 8u * lane; o < pc.bytes; o += 256u)
            *reinterpret_cast<float2*>(pc.dst + o) = __ldg(reinterpret_cast<const float2*>(pc.src + o));
    } else {
        if (lane == 0 && pc.head) *reinterpret_cast<float2*>(pc.dst) = __ldg(reinterpret_cast<const float2*>(pc.src));
        const uint32_t tail = pc.head + pc.body;
        if (lane == 1 && tail < pc.bytes)
            *reinterpret_cast<float2*>(pc.dst + tail) = __ldg(reinterpret_cast<const float2*>(pc.src + tail));
    }
}
__device__ __forceinline__ void piece_tma(const Piece& pc, uint64_t* bar) {
    if (pc.body) tma_load_1d(pc.dst + pc.head, pc.src + pc.head, pc.body, bar);
}

struct TileInfo {
    int32_t c;      // channel (absolute)
    int64_t i0;     // first output (call-local)
    int32_t Tt;     // outputs in this tile
    uint32_t kq;    // first snapshot interval, relative to the call's (t / S)
    int32_t nk;     // intervals touched
    int32_t j0;     // (t + i0) - kb*S
};

// 32-bit index math only: w < 2^31 tiles, i0 < 2^31 samples per call; the global
// start t enters through the host-precomputed t / S and t % S.
__host__ __device__ constexpr int ilog2_c(int v) { return v <= 1 ? 0 : 1 + ilog2_c(v / 2); }

__device__ __forceinline__ uint32_t div_S(const ConvParams& p, uint32_t v) {
    return p.s_shift >= 0 ? (v >> p.s_shift) : v / static_cast<uint32_t>(p.S);
}

// A work item ("super tile"): tile tl of the KC-channel chunk q of group g. Without
// aggregation (G = 1) it is exactly one channel tile.
struct SuperInfo {
    int32_t g, q, tl;
    int32_t c_first;  // absolute channel of the chunk's first member
    int32_t kcount;   // channels in the chunk
};
// 32-bit index math (the host keeps total_super < 2^31)
__device__ __forceinline__ SuperInfo super_info(const ConvParams& p, int64_t su64) {
    SuperInfo si;
    const uint32_t su = static_cast<uint32_t>(su64);
    const uint32_t rest = su / static_cast<uint32_t>(p.tiles_per_ch);
    si.tl = static_cast<int32_t>(su - rest * static_cast<uint32_t>(p.tiles_per_ch));
    if (p.nchunks == 1) {
        si.g = static_cast<int32_t>(rest);
        si.q = 0;
    } else {
        si.g = static_cast<int32_t>(rest / static_cast<uint32_t>(p.nchunks));
        si.q = static_cast<int32_t>(rest - static_cast<uint32_t>(si.g) * static_cast<uint32_t>(p.nchunks));
    }
    si.c_first = p.c_lo + si.g * p.group + si.q * p.chunk;
    const int32_t left = p.group - si.q * p.chunk;
    si.kcount = left < p.chunk ? left : p.chunk;
    return si;
}

// (channel, tile) of the work items blockIdx.x, blockIdx.x + gridDim.x, ... of the plain
// variant, advanced without a division per item
struct TileWalk {
    uint32_t cl, tl, dcl, dtl, tpc;
    __device__ __forceinline__ explicit TileWalk(uint32_t tiles_per_ch)
        : cl(blockIdx.x / tiles_per_ch),
          tl(blockIdx.x % tiles_per_ch),
          dcl(gridDim.x / tiles_per_ch),
          dtl(gridDim.x % tiles_per_ch),
          tpc(tiles_per_ch) {}
    __device__ __forceinline__ void next() {
        tl += dtl;
        cl += dcl;
        if (tl >= tpc) {
            tl -= tpc;
            ++cl;
        }
    }
};

template <int R, int CW, bool ROBUST>
__device__ __forceinline__ TileInfo tile_info(const ConvParams& p, int32_t c, int32_t tl) {
    constexpr int T = CW * 32 * R;
    TileInfo ti;
    ti.c = c;
    // with a lead-in (p.lead > 0) tile 0 is [0, lead) and tile tl >= 1 starts at
    // lead + (tl - 1) T, a multiple of 32R in global samples: every warp then starts on a
    // 32R-aligned sample (one snapshot interval per warp, paired noise) whatever the
    // call lengths so far
    if constexpr (ROBUST) {
        const int64_t base = static_cast<int64_t>(tl) * T - (p.lead ? T - p.lead : 0);
        ti.i0 = base < 0 ? 0 : base;
        const int64_t end = base + T < p.n ? base + T : p.n;
        ti.Tt = static_cast<int32_t>(end - ti.i0);
    } else {
        ti.i0 = static_cast<int64_t>(tl) * T;
        const int64_t rem = p.n - ti.i0;
        ti.Tt = rem < T ? static_cast<int32_t>(rem) : T;
    }
    const uint32_t u0 = static_cast<uint32_t>(p.t_mod) + static_cast<uint32_t>(ti.i0);  // (t + i0) - (t / S) S
    const uint32_t q0 = div_S(p, u0);
    ti.kq = q0;
    ti.j0 = static_cast<int32_t>(u0 - q0 * static_cast<uint32_t>(p.S));
    ti.nk = static_cast<int32_t>(div_S(p, static_cast<uint32_t>(ti.j0 + ti.Tt - 1))) + 1;
    return ti;
}

// One pipeline stage in shared memory: input window (H + T float2), coefficient rows
// (nk_max x L float4), tap offsets (L4 int32). Every region is a multiple of 16 B.
struct Stage {
    int32_t* meta;  // [0]: window shift (0 or 1 float2) chosen by the producer for this tile
    float2* win;
    float4* coef;
    int32_t* xo;
};

// Producer warp: stage tile `w` and arm `full` (plain parts first, then the barrier,
// then the TMA bodies).
template <int R, bool ROBUST>
__device__ __forceinline__ void produce_tile(const ConvParams& p, const TileInfo& ti, const Stage& st, uint64_t* full,
                                             int lane) {
    const int32_t H = p.H;
    const int64_t lo = ti.i0 - H;
    const int64_t hi = ti.i0 + ti.Tt;
    // A: delay-line history, call-local [lo, min(0, hi)) -> history index H + local
    const int64_t nA = lo < 0 ? ((hi < 0 ? hi : 0) - lo) : 0;
    // B: this call's input, call-local [max(lo, 0), hi)
    const int64_t bl = lo < 0 ? 0 : lo;
    const int64_t row = p.in_row ? static_cast<int64_t>(__ldg(p.in_row + ti.c)) : static_cast<int64_t>(ti.c - p.c_lo);
    const float2* xsrc = p.x + row * p.n + bl;
    // the window starts one float2 later when the input row is 8 B off a 16-B boundary
    // (odd call lengths), so that the large x piece stays a TMA copy (src and dst must
    // agree mod 16); bl - lo is even, st.win is 16-B aligned
    const int32_t wsh = ROBUST ? static_cast<int32_t>((reinterpret_cast<uintptr_t>(xsrc) >> 3) & 1u) : 0;
    float2* const win = st.win + wsh;
    const Piece a = make_piece(win, p.hist_rd + static_cast<int64_t>(ti.c) * H + (H + lo),
                               static_cast<uint32_t>(nA) * 8u);
    const Piece bx = make_piece(win + (bl - lo), xsrc, static_cast<uint32_t>(hi - bl) * 8u);
    // C, D: coefficient rows kb .. kb + nk - 1, wrapping at the ring's capacity
    const int64_t s0 = (p.t_div + ti.kq) % p.cap;
    const int32_t r1 = static_cast<int32_t>((p.cap - s0) < ti.nk ? (p.cap - s0) : ti.nk);
    const float4* ringc = p.ring + static_cast<int64_t>(ti.c) * p.cap * p.L;
    const uint32_t rowb = static_cast<uint32_t>(p.L) * 16u;
    const Piece c1 = make_piece(st.coef, ringc + s0 * p.L, static_cast<uint32_t>(r1) * rowb);
    const Piece c2 = make_piece(st.coef + static_cast<int64_t>(r1) * p.L, ringc,
                                static_cast<uint32_t>(ti.nk - r1) * rowb);
    // E, F: tap offsets — the channel's row, or (sparse) one row per staged interval
    Piece e, f;
    const uint32_t xrowb = static_cast<uint32_t>(p.L4) * 4u;
    if (p.xoff_rows) {
        const int32_t* xr = p.xoff_rows + static_cast<int64_t>(ti.c) * p.cap * p.L4;
        e = make_piece(st.xo, xr + s0 * p.L4, static_cast<uint32_t>(r1) * xrowb);
        f = make_piece(st.xo + static_cast<int64_t>(r1) * p.L4, xr, static_cast<uint32_t>(ti.nk - r1) * xrowb);
    } else {
        e = make_piece(st.xo, p.xoff + static_cast<int64_t>(ti.c) * p.L4, xrowb);
        f = make_piece(st.xo, p.xoff, 0u);
    }
    piece_plain(a, lane);
    piece_plain(bx, lane);
    piece_plain(c1, lane);
    piece_plain(c2, lane);
    piece_plain(e, lane);
    piece_plain(f, lane);
    if (ROBUST && lane == 0) *st.meta = wsh;
    __syncwarp();  // the lanes' plain stores happen-before lane 0's release (arrive)
    if (lane == 0) {
        mbar_arrive_expect_tx(full, a.body + bx.body + c1.body + c2.body + e.body + f.body);
        piece_tma(a, full);
        piece_tma(bx, full);
        piece_tma(c1, full);
        piece_tma(c2, full);
        piece_tma(e, full);
        piece_tma(f, full);
    }
}

// One tap for the R outputs this lane owns (rows RS outputs apart): gains first, then
// the packed MACs.
template <int R, int RS = 32>
__device__ __forceinline__ void mac_tap(const float4 q, const float2* __restrict__ xp, const float (&alpha)[R],
                                        float2 (&A)[R], float2 (&B)[R]) {
    float2 xv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) xv[r] = xp[r * RS];
    const float2 g = make_float2(q.x, q.y);
    const float2 dg = make_float2(q.z, q.w);
    float2 h[R];
#pragma unroll
    for (int r = 0; r < R; ++r) h[r] = __ffma2_rn(make_float2(alpha[r], alpha[r]), dg, g);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        A[r] = __ffma2_rn(make_float2(h[r].x, h[r].x), xv[r], A[r]);
        B[r] = __ffma2_rn(make_float2(h[r].y, h[r].y), xv[r], B[r]);
    }
}

// One tap when the warp's R rows (32 outputs each) fall into NG consecutive snapshot
// intervals of R/NG rows each (rows aligned to interval starts): NG broadcast gain
// reads per tap instead of one per row.
template <int R, int NG>
__device__ __forceinline__ void mac_tap_grouped(const float4* __restrict__ cf, int32_t L, int32_t j,
                                                const float2* const (&xp)[NG], const float (&alpha)[R],
                                                float2 (&A)[R], float2 (&B)[R]) {
    constexpr int RPG = R / NG;
    float4 q[NG];
#pragma unroll
    for (int g = 0; g < NG; ++g) q[g] = cf[g * L + j];
    float2 xv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) xv[r] = xp[r / RPG][r * 32];
    float2 h[R];
#pragma unroll
    for (int r = 0; r < R; ++r)
        h[r] = __ffma2_rn(make_float2(alpha[r], alpha[r]), make_float2(q[r / RPG].z, q[r / RPG].w),
                          make_float2(q[r / RPG].x, q[r / RPG].y));
#pragma unroll
    for (int r = 0; r < R; ++r) {
        A[r] = __ffma2_rn(make_float2(h[r].x, h[r].x), xv[r], A[r]);
        B[r] = __ffma2_rn(make_float2(h[r].y, h[r].y), xv[r], B[r]);
    }
}

// ROWS: (sparse) each interval has its own tap offsets row; else all share row 0
template <int R, int NG, bool ROWS>
__device__ __forceinline__ void taps_grouped(const ConvParams& p, const float4* cf, const int32_t* xo,
                                             const float2* xb, const float (&alpha)[R], float2 (&A)[R],
                                             float2 (&B)[R]) {
#pragma unroll 2
    for (int32_t j = 0; j < p.L; ++j) {
        const float2* xp[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) xp[g] = xb + (ROWS ? xo[g * p.L4 + j] : xo[j]);
        mac_tap_grouped<R, NG>(cf, p.L, j, xp, alpha, A, B);
    }
}
template <int R, int NG>
__device__ __forceinline__ void taps_grouped_rt(const ConvParams& p, const float4* cf, const int32_t* xo,
                                                const float2* xb, const float (&alpha)[R], float2 (&A)[R],
                                                float2 (&B)[R]) {
    if (p.xoff_rows) taps_grouped<R, NG, true>(p, cf, xo, xb, alpha, A, B);
    else taps_grouped<R, NG, false>(p, cf, xo, xb, alpha, A, B);
}

// Consumer warp of the non-split kernel instances: the 32R outputs of warp `cw` in tile
// `ti`, lane j owning cw 32R + j + 32 r. GEN: the general variant (group sums, sparse
// per-interval offsets); the plain variant compiles none of it. (consume_body<RS = 32>
// computes the same; this copy keeps the code of the instances that never split —
// c2-c4 — as measured, ptxas schedules the templated form 0.4-1 % slower.)
template <int R, int CW, bool NOISE, bool GEN>
__device__ __forceinline__ void consume_tile_plain(const ConvParams& p, const TileInfo& ti, const Stage& st, int cw,
                                             int lane, bool first, float2* aggdst) {
    const int32_t obase = cw * 32 * R + lane;
    if (cw * 32 * R < ti.Tt) {
        // per-output interpolation weight alpha = j / S (a multiply when S is a power of
        // two: then j * (1/S) is exact and equals the correctly rounded quotient)
        float alpha[R];
        int32_t kk[R];
        // outputs past a tail tile's end are computed but never stored; their coefficient
        // row is clamped into the staged block
        if (p.s_shift >= 0) {
            const uint32_t sh = static_cast<uint32_t>(p.s_shift), mask = static_cast<uint32_t>(p.S) - 1u;
            const float inv_S = p.inv_S;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t jj = static_cast<uint32_t>(ti.j0 + obase + r * 32);
                kk[r] = min(static_cast<int32_t>(jj >> sh), ti.nk - 1);
                alpha[r] = __fmul_rn(__uint2float_rn(jj & mask), inv_S);
            }
        } else {
            const float Sf = __int2float_rn(p.S);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t jj = static_cast<uint32_t>(ti.j0 + obase + r * 32);
                const uint32_t k = jj / static_cast<uint32_t>(p.S);
                kk[r] = min(static_cast<int32_t>(k), ti.nk - 1);
                alpha[r] = __fdiv_rn(__uint2float_rn(jj - k * static_cast<uint32_t>(p.S)), Sf);
            }
        }
        float2 A[R], B[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            A[r] = make_float2(0.f, 0.f);
            B[r] = make_float2(0.f, 0.f);
        }
        const float2* xb = st.win + obase;
        // warp-uniform: are all 32R outputs of this warp in one snapshot interval?
        const uint32_t wj0 = static_cast<uint32_t>(ti.j0 + cw * 32 * R);
        const uint32_t kw0 = div_S(p, wj0);
        const uint32_t kw1 = div_S(p, wj0 + 32 * R - 1);
        // tap offsets of interval kk: one row per interval when sparse, else the channel's
        const int32_t xo_row = (GEN && p.xoff_rows) ? p.L4 : 0;
        if (kw0 == kw1) {
            const float4* cf = st.coef + static_cast<int64_t>(kw0) * p.L;
            const int32_t* xo = st.xo + kw0 * xo_row;
            const int4* xo4 = reinterpret_cast<const int4*>(xo);
            int32_t j = 0;
            int4 o4 = xo4[0];
            for (; j + 4 <= p.L; j += 4) {
                const int4 o = o4;
                o4 = xo4[(j >> 2) + 1];  // next group's offsets (L4 >= L + 1 keeps this in range)
                const float4 q0 = cf[j], q1 = cf[j + 1], q2 = cf[j + 2], q3 = cf[j + 3];
                mac_tap<R>(q0, xb + o.x, alpha, A, B);
                mac_tap<R>(q1, xb + o.y, alpha, A, B);
                mac_tap<R>(q2, xb + o.z, alpha, A, B);
                mac_tap<R>(q3, xb + o.w, alpha, A, B);
            }
            for (; j < p.L; ++j) mac_tap<R>(cf[j], xb + xo[j], alpha, A, B);
        } else if ((R & (R - 1)) == 0 && p.s_shift >= 5 && p.s_shift <= ilog2_c(32 * R) &&
                   (wj0 & (p.S - 1)) == 0 && ((32 * R) >> p.s_shift) <= 4 &&
                   static_cast<int32_t>(kw0) + ((32 * R) >> p.s_shift) <= ti.nk) {  // (tail tiles: rows staged)
            // the warp starts on an interval boundary and spans NG = 32R / S (2 or 4) whole intervals
            const float4* cf = st.coef + static_cast<int64_t>(kw0) * p.L;
            const int32_t* xo = st.xo + kw0 * xo_row;
            if constexpr (GEN) {
                if (((32 * R) >> p.s_shift) == 2) taps_grouped_rt<R, (R >= 2 ? 2 : 1)>(p, cf, xo, xb, alpha, A, B);
                else taps_grouped_rt<R, (R >= 4 ? 4 : 1)>(p, cf, xo, xb, alpha, A, B);
            } else {
                if (((32 * R) >> p.s_shift) == 2) taps_grouped<R, (R >= 2 ? 2 : 1), false>(p, cf, xo, xb, alpha, A, B);
                else taps_grouped<R, (R >= 4 ? 4 : 1), false>(p, cf, xo, xb, alpha, A, B);
            }
        } else {
            for (int32_t j = 0; j < p.L; ++j) {
                const float2* xp = xb + st.xo[j];  // dense: one offset row
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float4 q = st.coef[kk[r] * p.L + j];
                    const float2 xv = (GEN && xo_row) ? xb[st.xo[kk[r] * xo_row + j] + r * 32] : xp[r * 32];
                    const float2 h =
                        __ffma2_rn(make_float2(alpha[r], alpha[r]), make_float2(q.z, q.w), make_float2(q.x, q.y));
                    A[r] = __ffma2_rn(make_float2(h.x, h.x), xv, A[r]);
                    B[r] = __ffma2_rn(make_float2(h.y, h.y), xv, B[r]);
                }
            }
        }

        // epilogue: combine, add noise, store
        float2 out[R];
#pragma unroll
        for (int r = 0; r < R; ++r) out[r] = combine(A[r], B[r]);
        if constexpr (NOISE) {
            const int64_t nb = p.t + ti.i0 + obase;  // global sample of row 0
            const uint32_t cg = static_cast<uint32_t>(p.chan_offset + ti.c);
            const bool even_base = ((p.t + ti.i0) & 1) == 0;  // CTA-uniform
            if (even_base && (R % 2 == 0)) {
                const bool ev = (lane & 1) == 0;
#pragma unroll
                for (int r = 0; r < R; r += 2) {
                    // even lane: pair of its row-r sample; odd lane: pair of its row-(r+1) sample
                    const uint64_t m = static_cast<uint64_t>(nb + (ev ? r : r + 1) * 32) >> 1;
                    const u32x4 q = philox4x32_10(static_cast<uint32_t>(m), static_cast<uint32_t>(m >> 32), cg, 0u,
                                                  p.key0, p.key1);
                    const uint32_t s0 = ev ? q.c : q.a, s1 = ev ? q.d : q.b;
                    const uint32_t v0 = __shfl_xor_sync(0xffffffffu, s0, 1);
                    const uint32_t v1 = __shfl_xor_sync(0xffffffffu, s1, 1);
                    // select the words first so each lane runs the transform once per sample
                    float2 wa, wb;
                    noise_from_words2(ev ? q.a : v0, ev ? q.b : v1, ev ? v0 : q.c, ev ? v1 : q.d, p.noise_sc, wa,
                                      wb);
                    out[r] = add_noise(out[r], wa);
                    out[r + 1] = add_noise(out[r + 1], wb);
                }
            } else if constexpr (R % 2 == 0) {
                // odd tile base: every lane draws its own pair per row (rows two at a time)
#pragma unroll
                for (int r = 0; r < R; r += 2) {
                    const int64_t n0 = nb + r * 32, n1 = n0 + 32;
                    const uint64_t m0 = static_cast<uint64_t>(n0) >> 1, m1 = static_cast<uint64_t>(n1) >> 1;
                    const u32x4 q0 = philox4x32_10(static_cast<uint32_t>(m0), static_cast<uint32_t>(m0 >> 32), cg, 0u,
                                                   p.key0, p.key1);
                    const u32x4 q1 = philox4x32_10(static_cast<uint32_t>(m1), static_cast<uint32_t>(m1 >> 32), cg, 0u,
                                                   p.key0, p.key1);
                    const bool odd = (n0 & 1) != 0;  // rows are 32 apart: same parity
                    float2 w0, w1;
                    noise_from_words2(odd ? q0.c : q0.a, odd ? q0.d : q0.b, odd ? q1.c : q1.a, odd ? q1.d : q1.b,
                                      p.noise_sc, w0, w1);
                    out[r] = add_noise(out[r], w0);
                    out[r + 1] = add_noise(out[r + 1], w1);
                }
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int64_t n = nb + r * 32;
                    const uint64_t m = static_cast<uint64_t>(n) >> 1;
                    const u32x4 q = philox4x32_10(static_cast<uint32_t>(m), static_cast<uint32_t>(m >> 32), cg, 0u,
                                                  p.key0, p.key1);
                    const bool odd = (n & 1) != 0;
                    const float2 wv = noise_from_words(odd ? q.c : q.a, odd ? q.d : q.b, p.noise_sc);
                    out[r] = add_noise(out[r], wv);
                }
            }
        }
        if (p.y) {
            float2* yc = p.y + static_cast<int64_t>(ti.c - p.c_lo) * p.n + ti.i0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int32_t o = obase + r * 32;
                if (o < ti.Tt) yc[o] = out[r];
            }
        }
        if (GEN && aggdst) {
            // running chunk sum in channel order, kept in the destination row itself (each
            // element is read back only by the thread that wrote it): s = y_first, s += y_k
            if (first) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int32_t o = obase + r * 32;
                    if (o < ti.Tt) aggdst[o] = out[r];
                }
            } else {
                // all R reads first (independent loads in flight), then the sums
                float2 v[R];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int32_t o = obase + r * 32;
                    v[r] = o < ti.Tt ? aggdst[o] : make_float2(0.f, 0.f);
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int32_t o = obase + r * 32;
                    if (o < ti.Tt) aggdst[o] = make_float2(__fadd_rn(v[r].x, out[r].x), __fadd_rn(v[r].y, out[r].y));
                }
            }
        }
    }
    // the tile that ends the call writes the new delay-line history (ping-pong); the
    // window index of call-local sample n - H + i is Tt + i
    if (ti.i0 + ti.Tt == p.n) {
        float2* hw = p.hist_wr + static_cast<int64_t>(ti.c) * p.H;
        for (int32_t i = cw * 32 + lane; i < p.H; i += CW * 32) hw[i] = st.win[ti.Tt + i];
    }
}

// Consumer warp: the 32R outputs of warp `cw` in tile `ti`. GEN: the general variant
// (group sums, sparse per-interval offsets); the plain variant compiles none of it.
//
// Lane layout. RS = 32: lane j owns outputs cw 32R + j + 32 r (r < R), so a row is one
// contiguous 256-B warp access. RS = 16 ("split warp", used when the snapshot period is
// S = 16R and the warp starts on an interval boundary, e.g. BASELINE c5: S = 128, R = 8):
// half-warp g = j / 16 owns the S outputs of interval kw0 + g, lane j owning
// cw 32R + g S + (j mod 16) + 16 r. Every half-warp then sits in one interval, so a tap
// reads one gain row per lane (the two half-warps' rows in one LDS.128) and the int4
// tap-offset prefetch of the one-interval path, instead of the grouped path's two gain
// rows plus a scalar offset per tap; each half-warp's row is a contiguous 128-B access
// (one wavefront), so the x reads stay conflict-free. Per output the operation sequence
// is unchanged.
template <int R, int CW, bool NOISE, bool GEN, int RS>
__device__ __forceinline__ void consume_body(const ConvParams& p, const TileInfo& ti, const Stage& st, int cw,
                                             int lane, bool first, float2* aggdst) {
    const int32_t obase = RS == 32 ? cw * 32 * R + lane : cw * 32 * R + (lane >> 4) * (16 * R) + (lane & 15);
    {
        // per-output interpolation weight alpha = j / S (a multiply when S is a power of
        // two: then j * (1/S) is exact and equals the correctly rounded quotient)
        float alpha[R];
        int32_t kk[R];
        // outputs past a tail tile's end are computed but never stored; their coefficient
        // row is clamped into the staged block
        if (p.s_shift >= 0) {
            const uint32_t sh = static_cast<uint32_t>(p.s_shift), mask = static_cast<uint32_t>(p.S) - 1u;
            const float inv_S = p.inv_S;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t jj = static_cast<uint32_t>(ti.j0 + obase + r * RS);
                kk[r] = min(static_cast<int32_t>(jj >> sh), ti.nk - 1);
                alpha[r] = __fmul_rn(__uint2float_rn(jj & mask), inv_S);
            }
        } else {
            const float Sf = __int2float_rn(p.S);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t jj = static_cast<uint32_t>(ti.j0 + obase + r * RS);
                const uint32_t k = jj / static_cast<uint32_t>(p.S);
                kk[r] = min(static_cast<int32_t>(k), ti.nk - 1);
                alpha[r] = __fdiv_rn(__uint2float_rn(jj - k * static_cast<uint32_t>(p.S)), Sf);
            }
        }
        float2 A[R], B[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            A[r] = make_float2(0.f, 0.f);
            B[r] = make_float2(0.f, 0.f);
        }
        const float2* xb = st.win + obase;
        // warp-uniform: are all 32R outputs of this warp in one snapshot interval?
        const uint32_t wj0 = static_cast<uint32_t>(ti.j0 + cw * 32 * R);
        const uint32_t kw0 = div_S(p, wj0);
        const uint32_t kw1 = div_S(p, wj0 + 32 * R - 1);
        // tap offsets of interval kk: one row per interval when sparse, else the channel's
        const int32_t xo_row = (GEN && p.xoff_rows) ? p.L4 : 0;
        if (RS == 16 || kw0 == kw1) {
            // one interval per lane: this lane's gain row (split warp: its half-warp's
            // interval, clamped into the staged rows for outputs past a tail tile's end)
            const int32_t kl = RS == 16 ? min(static_cast<int32_t>(kw0) + (lane >> 4), ti.nk - 1)
                                        : static_cast<int32_t>(kw0);
            const float4* cf = st.coef + static_cast<int64_t>(kl) * p.L;
            const int32_t* xo = st.xo + kl * xo_row;
            const int4* xo4 = reinterpret_cast<const int4*>(xo);
            int32_t j = 0;
            int4 o4 = xo4[0];
            for (; j + 4 <= p.L; j += 4) {
                const int4 o = o4;
                o4 = xo4[(j >> 2) + 1];  // next group's offsets (L4 >= L + 1 keeps this in range)
                const float4 q0 = cf[j], q1 = cf[j + 1], q2 = cf[j + 2], q3 = cf[j + 3];
                mac_tap<R, RS>(q0, xb + o.x, alpha, A, B);
                mac_tap<R, RS>(q1, xb + o.y, alpha, A, B);
                mac_tap<R, RS>(q2, xb + o.z, alpha, A, B);
                mac_tap<R, RS>(q3, xb + o.w, alpha, A, B);
            }
            for (; j < p.L; ++j) mac_tap<R, RS>(cf[j], xb + xo[j], alpha, A, B);
        } else if ((R & (R - 1)) == 0 && p.s_shift >= 5 && p.s_shift <= ilog2_c(32 * R) &&
                   (wj0 & (p.S - 1)) == 0 && ((32 * R) >> p.s_shift) <= 4 &&
                   static_cast<int32_t>(kw0) + ((32 * R) >> p.s_shift) <= ti.nk) {  // (tail tiles: rows staged)
            // the warp starts on an interval boundary and spans NG = 32R / S (2 or 4) whole intervals
            const float4* cf = st.coef + static_cast<int64_t>(kw0) * p.L;
            const int32_t* xo = st.xo + kw0 * xo_row;
            if constexpr (GEN) {
                if (((32 * R) >> p.s_shift) == 2) taps_grouped_rt<R, (R >= 2 ? 2 : 1)>(p, cf, xo, xb, alpha, A, B);
                else taps_grouped_rt<R, (R >= 4 ? 4 : 1)>(p, cf, xo, xb, alpha, A, B);
            } else {
                if (((32 * R) >> p.s_shift) == 2) taps_grouped<R, (R >= 2 ? 2 : 1), false>(p, cf, xo, xb, alpha, A, B);
                else taps_grouped<R, (R >= 4 ? 4 : 1), false>(p, cf, xo, xb, alpha, A, B);
            }
        } else {
            for (int32_t j = 0; j < p.L; ++j) {
                const float2* xp = xb + st.xo[j];  // dense: one offset row
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float4 q = st.coef[kk[r] * p.L + j];
                    const float2 xv = (GEN && xo_row) ? xb[st.xo[kk[r] * xo_row + j] + r * RS] : xp[r * RS];
                    const float2 h =
                        __ffma2_rn(make_float2(alpha[r], alpha[r]), make_float2(q.z, q.w), make_float2(q.x, q.y));
                    A[r] = __ffma2_rn(make_float2(h.x, h.x), xv, A[r]);
                    B[r] = __ffma2_rn(make_float2(h.y, h.y), xv, B[r]);
                }
            }
        }

        // epilogue: combine, add noise, store
        float2 out[R];
#pragma unroll
        for (int r = 0; r < R; ++r) out[r] = combine(A[r], B[r]);
        if constexpr (NOISE) {
            const int64_t nb = p.t + ti.i0 + obase;  // global sample of row 0
            const uint32_t cg = static_cast<uint32_t>(p.chan_offset + ti.c);
            const bool even_base = ((p.t + ti.i0) & 1) == 0;  // CTA-uniform
            if (even_base && (R % 2 == 0)) {
                const bool ev = (lane & 1) == 0;
#pragma unroll
                for (int r = 0; r < R; r += 2) {
                    // even lane: pair of its row-r sample; odd lane: pair of its row-(r+1) sample
                    const uint64_t m = static_cast<uint64_t>(nb + (ev ? r : r + 1) * RS) >> 1;
                    const u32x4 q = philox4x32_10(static_cast<uint32_t>(m), static_cast<uint32_t>(m >> 32), cg, 0u,
                                                  p.key0, p.key1);
                    const uint32_t s0 = ev ? q.c : q.a, s1 = ev ? q.d : q.b;
                    const uint32_t v0 = __shfl_xor_sync(0xffffffffu, s0, 1);
                    const uint32_t v1 = __shfl_xor_sync(0xffffffffu, s1, 1);
                    // select the words first so each lane runs the transform once per sample
                    float2 wa, wb;
                    noise_from_words2(ev ? q.a : v0, ev ? q.b : v1, ev ? v0 : q.c, ev ? v1 : q.d, p.noise_sc, wa,
                                      wb);
                    out[r] = add_noise(out[r], wa);
                    out[r + 1] = add_noise(out[r + 1], wb);
                }
            } else if constexpr (R % 2 == 0) {
                // odd tile base: every lane draws its own pair per row (rows two at a time)
#pragma unroll
                for (int r = 0; r < R; r += 2) {
                    const int64_t n0 = nb + r * RS, n1 = n0 + RS;
                    const uint64_t m0 = static_cast<uint64_t>(n0) >> 1, m1 = static_cast<uint64_t>(n1) >> 1;
                    const u32x4 q0 = philox4x32_10(static_cast<uint32_t>(m0), static_cast<uint32_t>(m0 >> 32), cg, 0u,
                                                   p.key0, p.key1);
                    const u32x4 q1 = philox4x32_10(static_cast<uint32_t>(m1), static_cast<uint32_t>(m1 >> 32), cg, 0u,
                                                   p.key0, p.key1);
                    const bool odd = (n0 & 1) != 0;  // rows are RS (even) apart: same parity
                    float2 w0, w1;
                    noise_from_words2(odd ? q0.c : q0.a, odd ? q0.d : q0.b, odd ? q1.c : q1.a, odd ? q1.d : q1.b,
                                      p.noise_sc, w0, w1);
                    out[r] = add_noise(out[r], w0);
                    out[r + 1] = add_noise(out[r + 1], w1);
                }
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int64_t n = nb + r * RS;
                    const uint64_t m = static_cast<uint64_t>(n) >> 1;
                    const u32x4 q = philox4x32_10(static_cast<uint32_t>(m), static_cast<uint32_t>(m >> 32), cg, 0u,
                                                  p.key0, p.key1);
                    const bool odd = (n & 1) != 0;
                    const float2 wv = noise_from_words(odd ? q.c : q.a, odd ? q.d : q.b, p.noise_sc);
                    out[r] = add_noise(out[r], wv);
                }
            }
        }
        if (p.y) {
            float2* yc = p.y + static_cast<int64_t>(ti.c - p.c_lo) * p.n + ti.i0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int32_t o = obase + r * RS;
                if (o < ti.Tt) yc[o] = out[r];
            }
        }
        if (GEN && aggdst) {
            // running chunk sum in channel order, kept in the destination row itself (each
            // element is read back only by the thread that wrote it): s = y_first, s += y_k
            if (first) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int32_t o = obase + r * RS;
                    if (o < ti.Tt) aggdst[o] = out[r];
                }
            } else {
                // all R reads first (independent loads in flight), then the sums
                float2 v[R];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int32_t o = obase + r * RS;
                    v[r] = o < ti.Tt ? aggdst[o] : make_float2(0.f, 0.f);
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int32_t o = obase + r * RS;
                    if (o < ti.Tt) aggdst[o] = make_float2(__fadd_rn(v[r].x, out[r].x), __fadd_rn(v[r].y, out[r].y));
                }
            }
        }
    }
}

// SPLIT: a kernel instance launched only when S = 16R (the host checks); its warps that
// start on an interval boundary take the split-warp layout. Other instances run
// consume_tile_plain.
template <int R, int CW, bool NOISE, bool GEN, bool SPLIT>
__device__ __forceinline__ void consume_tile(const ConvParams& p, const TileInfo& ti, const Stage& st, int cw,
                                             int lane, bool first, float2* aggdst) {
    if constexpr (!SPLIT) {
        consume_tile_plain<R, CW, NOISE, GEN>(p, ti, st, cw, lane, first, aggdst);
    } else {
        if (cw * 32 * R < ti.Tt) {
            const uint32_t wj0 = static_cast<uint32_t>(ti.j0 + cw * 32 * R);
            if ((wj0 & static_cast<uint32_t>(16 * R - 1)) == 0)  // S = 16R
                consume_body<R, CW, NOISE, GEN, 16>(p, ti, st, cw, lane, first, aggdst);
            else
                consume_body<R, CW, NOISE, GEN, 32>(p, ti, st, cw, lane, first, aggdst);
        }
        // the tile that ends the call writes the new delay-line history (ping-pong); the
        // window index of call-local sample n - H + i is Tt + i
        if (ti.i0 + ti.Tt == p.n) {
            float2* hw = p.hist_wr + static_cast<int64_t>(ti.c) * p.H;
            for (int32_t i = cw * 32 + lane; i < p.H; i += CW * 32) hw[i] = st.win[ti.Tt + i];
        }
    }
}

// CW consumer warps + 1 producer warp; tile T = CW x 32 x R outputs of one channel
template <int R, int CW, bool NOISE, bool GEN, bool ROBUST, bool SPLIT>
// (shapes with <= 8 consumer warps and R <= 8 run two CTAs per SM: independent CTAs drift apart, so
// one CTA's noise epilogue can overlap the other's tap loop; measured slower, opt-in)
__device__ __forceinline__ void conv_body(const ConvParams& p) {
    constexpr int T = CW * 32 * R;
    extern __shared__ __align__(128) unsigned char smem[];
    // layout: [full kMaxStages x 8 B | empty kMaxStages x 8 B | pad to 128][stage 0][stage 1]...
    //   stage = [win (H+T) float2][coef nk_max x L float4][xo (sparse: nk_max x) L4 int32]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kMaxStages;
    // ROBUST: meta + window with one float2 of shift room; else the window alone
    const int64_t WB = ROBUST ? 16 + static_cast<int64_t>(p.H + T + 2) * 8 : static_cast<int64_t>(p.H + T) * 8;
    const int64_t CB = static_cast<int64_t>(p.nk_max) * p.L * 16;
    const int64_t SB = WB + CB + static_cast<int64_t>(p.xoff_rows ? p.nk_max : 1) * p.L4 * 4;
    auto stage = [&](int s) {
        unsigned char* base = smem + 128 + s * SB;
        Stage st;
        st.meta = reinterpret_cast<int32_t*>(base);
        st.win = reinterpret_cast<float2*>(base + (ROBUST ? 16 : 0));
        st.coef = reinterpret_cast<float4*>(base + WB);
        st.xo = reinterpret_cast<int32_t*>(base + WB + CB);
        return st;
    };
    // consumer view of a full stage: the window as the producer placed it
    auto shifted = [](Stage st) {
        if constexpr (ROBUST) st.win += *st.meta;
        return st;
    };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    // programmatic dependent launch: the next call's grid may be scheduled now (its CTAs
    // take over SMs as ours exit); and nothing here touches global memory before the
    // previous grid on the stream has completed (history, gain ring, y reuse)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp == CW) {
        // producer: run ahead of the consumers by up to `stages` tiles
        // stage s and its use count kk, advanced incrementally (no runtime division)
        int s = 0, kk = 0;
        auto next = [&] {
            if (++s == p.stages) {
                s = 0;
                ++kk;
            }
        };
        if (!GEN || p.agg == nullptr) {
            // one channel tile per work item: w -> (channel, tile)
            TileWalk tw(static_cast<uint32_t>(p.tiles_per_ch));
            for (int64_t w = blockIdx.x; w < p.total_tiles; w += gridDim.x, next(), tw.next()) {
                if (kk > 0) mbar_wait(&empty[s], (kk - 1) & 1);
                produce_tile<R, ROBUST>(p, tile_info<R, CW, ROBUST>(p, p.c_lo + static_cast<int32_t>(tw.cl), static_cast<int32_t>(tw.tl)),
                                stage(s), &full[s], lane);
            }
        } else {
            for (int64_t su = blockIdx.x; su < p.total_super; su += gridDim.x) {
                const SuperInfo si = super_info(p, su);
                for (int32_t k = 0; k < si.kcount; ++k, next()) {
                    if (kk > 0) mbar_wait(&empty[s], (kk - 1) & 1);
                    produce_tile<R, ROBUST>(p, tile_info<R, CW, ROBUST>(p, si.c_first + k, si.tl), stage(s), &full[s], lane);
                }
            }
        }
    } else {
        int s = 0;
        uint32_t ph = 0;  // parity of the stage's current use
        auto next = [&] {
            if (++s == p.stages) {
                s = 0;
                ph ^= 1u;
            }
        };
        if (!GEN || p.agg == nullptr) {
            TileWalk tw(static_cast<uint32_t>(p.tiles_per_ch));
            for (int64_t w = blockIdx.x; w < p.total_tiles; w += gridDim.x, next(), tw.next()) {
                mbar_wait(&full[s], ph);
                const TileInfo ti =
                    tile_info<R, CW, ROBUST>(p, p.c_lo + static_cast<int32_t>(tw.cl), static_cast<int32_t>(tw.tl));
                consume_tile<R, CW, NOISE, GEN, SPLIT>(p, ti, shifted(stage(s)), warp, lane, true, nullptr);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
        } else {
            for (int64_t su = blockIdx.x; su < p.total_super; su += gridDim.x) {
                const SuperInfo si = super_info(p, su);
                for (int32_t k = 0; k < si.kcount; ++k, next()) {
                    mbar_wait(&full[s], ph);
                    const TileInfo ti = tile_info<R, CW, ROBUST>(p, si.c_first + k, si.tl);
                    // the chunk's sum goes straight into the group row, or into its partial row
                    float2* aggdst =
                        p.agg ? p.agg + (static_cast<int64_t>(si.g) * p.nchunks + si.q) * p.n + ti.i0 : nullptr;
                    consume_tile<R, CW, NOISE, true, SPLIT>(p, ti, shifted(stage(s)), warp, lane, k == 0, aggdst);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s]);
                }
            }
        }
    }
}

// The tiled kernel. The ROBUST variant can run on the device clock: it waits for the
// previous grid (PDL) before reading it, and the last CTA to finish advances it.
template <int R, int CW, bool NOISE, bool GEN, bool ROBUST, bool SPLIT = false>
__global__ void __launch_bounds__((CW + 1) * 32, (CW <= 8 && R <= 8 ? 2 : 1)) tt_conv_kernel(const ConvParams p) {
    if constexpr (ROBUST) {
        ConvParams q = p;
        int64_t t = 0;
        int32_t par = 0;
        if (p.clk) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            t = *reinterpret_cast<volatile int64_t*>(&p.clk->t);
            par = *reinterpret_cast<volatile int32_t*>(&p.clk->par);
            q.t = t;
            q.t_div = p.s_shift >= 0 ? (t >> p.s_shift) : t / p.S;
            q.t_mod = static_cast<int32_t>(t - q.t_div * p.S);
            q.hist_rd = t == 0 ? p.hist_zero : p.hist_base + par * p.hist_half;
            q.hist_wr = p.hist_base + (par ^ 1) * p.hist_half;
        }
        conv_body<R, CW, NOISE, GEN, ROBUST, SPLIT>(q);
        if (p.clk) {
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                if (atomicAdd(&p.clk->done, 1u) == gridDim.x - 1) {
                    p.clk->t = t + p.n;
                    p.clk->par = p.H > 0 ? (par ^ 1) : par;
                    p.clk->done = 0u;
                    __threadfence();
                }
            }
        }
    } else {
        conv_body<R, CW, NOISE, GEN, ROBUST, SPLIT>(p);
    }
}


// Generic path: one thread per output, operands straight from global memory. Used
// when the tiled kernel's shared-memory plan does not fit (very long filters with very
// short snapshot periods). Same per-output operation sequence => bit-identical.
template <bool NOISE>
__global__ void __launch_bounds__(256) tt_conv_generic_kernel(const ConvParams p) {
    const int64_t nch = p.total_tiles / p.tiles_per_ch;
    const int64_t N = nch * p.n;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < N;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t cl = e / p.n;
        const int64_t i = e - cl * p.n;
        const int32_t c = p.c_lo + static_cast<int32_t>(cl);
        const int64_t n = p.t + i;
        const int64_t k = n / p.S;
        const int32_t jj = static_cast<int32_t>(n - k * p.S);
        const float alpha = __fdiv_rn(__uint2float_rn(static_cast<uint32_t>(jj)), __int2float_rn(p.S));
        const int64_t rowi = static_cast<int64_t>(c) * p.cap + (k % p.cap);
        const float4* cr = p.ring + rowi * p.L;
        const float2* xc = p.x + (p.in_row ? static_cast<int64_t>(__ldg(p.in_row + c)) : cl) * p.n;
        const float2* hc = p.hist_rd + static_cast<int64_t>(c) * p.H;
        const int32_t* xo = p.xoff_rows ? p.xoff_rows + rowi * p.L4 : p.xoff + static_cast<int64_t>(c) * p.L4;
        float2 A = make_float2(0.f, 0.f), Bv = make_float2(0.f, 0.f);
        for (int32_t j = 0; j < p.L; ++j) {
            const float4 q = __ldg(cr + j);
            const int64_t m = i - (p.H - __ldg(xo + j));
            const float2 xv = m >= 0 ? __ldg(xc + m) : __ldg(hc + (p.H + m));
            const float2 h = __ffma2_rn(make_float2(alpha, alpha), make_float2(q.z, q.w), make_float2(q.x, q.y));
            A = __ffma2_rn(make_float2(h.x, h.x), xv, A);
            Bv = __ffma2_rn(make_float2(h.y, h.y), xv, Bv);
        }
        float2 o = make_float2(__fsub_rn(A.x, Bv.y), __fadd_rn(A.y, Bv.x));
        if constexpr (NOISE) {
            const uint64_t mm = static_cast<uint64_t>(n) >> 1;
            const u32x4 q = philox4x32_10(static_cast<uint32_t>(mm), static_cast<uint32_t>(mm >> 32),
                                          static_cast<uint32_t>(p.chan_offset + c), 0u, p.key0, p.key1);
            const bool odd = (n & 1) != 0;
            const float2 wv = noise_from_words(odd ? q.c : q.a, odd ? q.d : q.b, p.noise_sc);
            o = make_float2(__fadd_rn(o.x, wv.x), __fadd_rn(o.y, wv.y));
        }
        p.y[cl * p.n + i] = o;
    }
}

// History update for the generic path (the tiled kernel fuses it): the new history is
// the last H samples of (old history ++ x).
// device clock := (t, par) (tt_channel_set_device_clock, reset)
__global__ void tt_set_clock_kernel(DevClock* clk, int64_t t, int32_t par) {
    clk->t = t;
    clk->par = par;
    clk->done = 0u;
}

__global__ void tt_history_kernel(const ConvParams p, int32_t nch) {
    const int64_t tot = static_cast<int64_t>(nch) * p.H;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < tot;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t cl = e / p.H;
        const int32_t i = static_cast<int32_t>(e - cl * p.H);
        const int32_t c = p.c_lo + static_cast<int32_t>(cl);
        const int64_t m = p.n - p.H + i;  // call-local index of the sample
        const int64_t row = p.in_row ? static_cast<int64_t>(__ldg(p.in_row + c)) : cl;
        p.hist_wr[static_cast<int64_t>(c) * p.H + i] =
            m >= 0 ? p.x[row * p.n + m] : p.hist_rd[static_cast<int64_t>(c) * p.H + (p.H + m)];
    }
}

// Group sums (NEXT f1 UL aggregation, f4 multi-gNB):
//   agg[g][i] = sum_q P_q[i],  P_q = y_{c_q} + y_{c_q + 1} + ... (chunk q of KC channels)
// each sum taken left to right in float32 — the order the tiled kernel's fused chunk
// sums use, so both paths give identical bits. from_partials: src holds the chunk sums
// P [groups][nchunks][n] (tiled kernel); else src holds per-channel outputs [C][n].
__global__ void tt_group_sum_kernel(const float2* __restrict__ src, float2* __restrict__ agg, int64_t n,
                                    int32_t groups, int32_t G, int32_t KC, int32_t nchunks, int32_t from_partials) {
    const int64_t tot = static_cast<int64_t>(groups) * n;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < tot;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t g = e / n, i = e - g * n;
        float2 s = make_float2(0.f, 0.f);
        for (int32_t q = 0; q < nchunks; ++q) {
            float2 pq;
            if (from_partials) {
                pq = __ldg(src + (g * nchunks + q) * n + i);
            } else {
                const int64_t c0 = g * G + static_cast<int64_t>(q) * KC;
                const int32_t kc = (G - q * KC) < KC ? (G - q * KC) : KC;
                pq = __ldg(src + c0 * n + i);
                for (int32_t k = 1; k < kc; ++k) {
                    const float2 v = __ldg(src + (c0 + k) * n + i);
                    pq = make_float2(__fadd_rn(pq.x, v.x), __fadd_rn(pq.y, v.y));
                }
            }
            s = q == 0 ? pq : make_float2(__fadd_rn(s.x, pq.x), __fadd_rn(s.y, pq.y));
        }
        agg[e] = s;
    }
}

// NEXT f2 selection + compaction ("top-n dominant taps at each time step";
// DESIGN.md R20): for each staged snapshot row (c, k) of the dense ring, keep the n taps
// of largest m_j = fl(fl(g.re g.re) + fl(g.im g.im)) — ties to the smaller sorted index j
// (= smaller delay, then smaller original index) — and write them, in ascending delay
// order, with their (g, dg) and window offsets into the sparse ring. One warp per row:
// the row's magnitudes go to shared memory, each lane ranks its taps against all L,
// and a ballot prefix count gives each selected tap its compacted slot.
__global__ void tt_select_kernel(const float4* __restrict__ ring, float4* __restrict__ sring,
                                 int32_t* __restrict__ soff, const int32_t* __restrict__ xoff, int32_t C, int64_t cap,
                                 int32_t L, int32_t L4, int32_t n, int32_t n4, int64_t k_first, int64_t rows) {
    extern __shared__ float mags[];  // [warps per block][L]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* m = mags + warp * L;
    const int64_t nrow = static_cast<int64_t>(C) * rows;
    for (int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp; row < nrow;
         row += static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5)) {
        const int64_t c = row / rows;
        const int64_t slot = (k_first + (row - c * rows)) % cap;
        const float4* src = ring + (c * cap + slot) * L;
        for (int32_t j = lane; j < L; j += 32) {
            const float4 q = src[j];
            m[j] = __fadd_rn(__fmul_rn(q.x, q.x), __fmul_rn(q.y, q.y));
        }
        __syncwarp();
        float4* dst = sring + (c * cap + slot) * n;
        int32_t* od = soff + (c * cap + slot) * n4;
        int32_t base = 0;  // selected taps before this 32-tap chunk
        for (int32_t j0 = 0; j0 < L; j0 += 32) {
            const int32_t j = j0 + lane;
            bool sel = false;
            if (j < L) {
                const float mj = m[j];
                int32_t rank = 0;
                for (int32_t i = 0; i < L; ++i) {
                    const float mi = m[i];
                    rank += (mi > mj || (mi == mj && i < j)) ? 1 : 0;
                }
                sel = rank < n;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, sel);
            if (sel) {
                const int32_t pos = base + __popc(bal & ((1u << lane) - 1u));
                dst[pos] = src[j];
                od[pos] = __ldg(xoff + c * L4 + j);
            }
            base += __popc(bal);
        }
        __syncwarp();
    }
}

// Snapshot loader (P:309 / P:411 trace ingestion): writes snapshots first .. first +
// count - 1 of every channel into the ring as (g_k, g_{k+1} - g_k) in sorted-tap order.
// src: device float2 [C][count][L] in the caller's (original) tap order; perm [C][L]:
// original index of sorted tap j. The difference of the last new snapshot is completed
// by the next contiguous load; `fix_prev` completes snapshot first - 1's difference;
// `fix_next` (a block reloaded inside the resident range, so snapshot first + count
// stays resident) completes the last new snapshot's difference against the ring's copy
// of snapshot first + count.
__global__ void tt_load_kernel(const float2* __restrict__ src, int64_t count, int64_t first, float4* ring, int64_t cap,
                               const int32_t* __restrict__ perm, int32_t C, int32_t L, int32_t fix_prev,
                               int32_t fix_next) {
    const int64_t tot = static_cast<int64_t>(C) * count * L;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < tot;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t j = static_cast<int32_t>(e % L);
        const int64_t ci = e / L;
        const int64_t i = ci % count;
        const int64_t c = ci / count;
        const int32_t o = __ldg(perm + c * L + j);
        const float2 g = __ldg(src + (c * count + i) * L + o);
        float4 v = make_float4(g.x, g.y, 0.f, 0.f);
        const int64_t k = first + i;
        if (i + 1 < count) {
            const float2 g1 = __ldg(src + (c * count + i + 1) * L + o);
            v.z = __fsub_rn(g1.x, g.x);
            v.w = __fsub_rn(g1.y, g.y);
        } else if (fix_next) {
            // snapshot k + 1 is resident and not rewritten by this load (count < cap)
            const float4 nx = ring[(c * cap + (k + 1) % cap) * L + j];
            v.z = __fsub_rn(nx.x, g.x);
            v.w = __fsub_rn(nx.y, g.y);
        }
        ring[(c * cap + k % cap) * L + j] = v;
        if (i == 0 && fix_prev) {
            float4* pv = ring + (c * cap + (k - 1) % cap) * L + j;
            pv->z = __fsub_rn(g.x, pv->x);
            pv->w = __fsub_rn(g.y, pv->y);
        }
    }
}

}  // namespace tt
