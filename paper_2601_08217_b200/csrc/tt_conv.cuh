// tt_conv.cuh — the sm_100a kernels of the Tiny-Twin channel convolution
// (arXiv 2601.08217; NS formula, §III-B, §IV).
//
//   y_c[n] = sum_l (g_{c,l,k} + alpha (g_{c,l,k+1} - g_{c,l,k})) x_c[n - d_{c,l}] + w_c[n]
//
// Design:
//  * persistent CTAs (grid = SMs x resident CTAs) walk a flat list of (channel, tile)
//    work items; a tile is T = 256 R consecutive outputs of one channel;
//  * each tile's input window x[i0 - H, i0 + T) (H = max-delay halo) and its raw gain
//    snapshots are staged into shared memory by 1-D TMA bulk copies
//    (cp.async.bulk ... mbarrier::complete_tx) into a double buffer, so the next
//    tile's bytes are in flight while this tile computes; the halo before the call
//    start comes from the carried delay-line history;
//  * the snapshot pair of every interval the tile touches becomes a table of
//    (g_k, g_{k+1} - g_k) float4 in tap order sorted by delay;
//  * lane-interleaved outputs: lane j of warp w owns outputs w*32R + r*32 + j, so every
//    x read is a conflict-free 256-B warp access; the warp's 32R outputs normally sit
//    in one snapshot interval, making the coefficient read a broadcast;
//  * per output-tap: h = fma(alpha, dg, g) then two packed FMAs (FFMA2, sm_100) into
//    split accumulators A += h_re x, B += h_im x; y = (A.re - B.im, A.im + B.re);
//  * optional AWGN (docs/tt-normal-v1.md) fused in the epilogue, one Philox call per
//    sample pair shared by neighbouring lanes via a shuffle;
//  * the CTA that owns a channel's last tile writes the new delay-line history from
//    its staged window into the other half of a ping-pong buffer.
//
// Every output's operation sequence depends only on (channel, global n) — never on
// the tile, path or launch shape — so results are bit-identical across partitions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tt_noise.cuh"

namespace tt {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct ConvParams {
    const float2* x;        // [C_launch][n]: row 0 = channel c_lo
    float2* y;              // [C_launch][n]
    const float2* hist_rd;  // [C][H]  last H samples of the stream so far
    float2* hist_wr;        // [C][H]  written with the new history
    const float2* ring;     // [C][cap][Lp] raw gain snapshots, original tap order
    const int32_t* dsort;   // [C][L] delays sorted ascending
    const int32_t* perm;    // [C][L] original tap index of each sorted position
    int64_t n;              // samples per channel in this call
    int64_t t;              // global index of the call's first sample
    int64_t cap;            // ring slots per channel
    int64_t chan_offset;    // global id of channel 0 (noise key)
    int64_t total_tiles;    // (c_hi - c_lo) * tiles_per_ch
    int32_t c_lo;           // first channel of this launch
    int32_t tiles_per_ch;
    int32_t L, Lp, H, S;
    int32_t nk_max;         // max snapshot intervals a tile touches
    uint32_t key0, key1;    // noise key
    float noise_sc;         // sigma / sqrt(2) as float; 0 = no noise
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

// Stage `count` float2 from global `src` to shared `dst`. Thread 0 issues one TMA bulk
// copy for the 16-B aligned body; the other elements (misaligned head / odd tail, or
// everything when src and dst disagree mod 16 B) are copied by plain loads spread over
// the CTA. Returns (to thread 0) the TMA bytes it issued. Plain stores become visible
// at the CTA's next __syncthreads; TMA bytes at the mbarrier.
__device__ __forceinline__ uint32_t stage_copy(float2* dst, const float2* src, int32_t count, uint64_t* bar,
                                               bool issue) {
    if (count <= 0) return 0;
    int32_t head = 0, body = 0;
    const uintptr_t sa = reinterpret_cast<uintptr_t>(src), da = smem_u32(dst);
    if (((sa ^ da) & 15u) == 0) {
        head = (sa & 15u) ? 1 : 0;
        body = (count - head) & ~1;
        if (body < 2) body = 0;
    }
    if (body > 0 && issue) tma_load_1d(dst + head, src + head, static_cast<uint32_t>(body) * 8u, bar);
    for (int32_t i = threadIdx.x; i < count; i += kThreads) {
        if (i >= head && i < head + body) continue;
        dst[i] = __ldg(src + i);
    }
    return static_cast<uint32_t>(body) * 8u;
}

struct TileInfo {
    int32_t c;      // channel (absolute)
    int64_t i0;     // first output (call-local)
    int32_t Tt;     // outputs in this tile
    int64_t kb;     // first snapshot interval
    int32_t nk;     // intervals touched
    int32_t j0;     // (t + i0) - kb*S
};

template <int R>
__device__ __forceinline__ TileInfo tile_info(const ConvParams& p, int64_t w) {
    constexpr int T = kThreads * R;
    TileInfo ti;
    const int64_t cl = w / p.tiles_per_ch;
    const int64_t tl = w - cl * p.tiles_per_ch;
    ti.c = p.c_lo + static_cast<int32_t>(cl);
    ti.i0 = tl * T;
    const int64_t rem = p.n - ti.i0;
    ti.Tt = rem < T ? static_cast<int32_t>(rem) : T;
    const int64_t g0 = p.t + ti.i0;
    ti.kb = g0 / p.S;
    ti.j0 = static_cast<int32_t>(g0 - ti.kb * p.S);
    ti.nk = static_cast<int32_t>((g0 + ti.Tt - 1) / p.S - ti.kb) + 1;
    return ti;
}

// Issue the staging of tile `w` into buffer b: window [i0 - H, i0 + Tt) and raw snapshot
// rows kb .. kb + nk. All threads call it (plain-load remainders are cooperative).
template <int R>
__device__ __forceinline__ void issue_tile(const ConvParams& p, int64_t w, float2* win, float2* raw, uint64_t* bar) {
    const TileInfo ti = tile_info<R>(p, w);
    const bool lead = threadIdx.x == 0;
    uint32_t tx = 0;
    // Thread 0 must announce the byte count before any copy can complete, so it
    // first computes the TMA bytes of every piece (issue = false pass is pure math).
    // To keep it simple and exact, thread 0 arms the barrier with the total it will
    // issue below; stage_copy's decision is deterministic.
    const int32_t H = p.H;
    const int64_t lo = ti.i0 - H;
    const int64_t hi = ti.i0 + ti.Tt;
    // piece A: history part, local [lo, min(0, hi)) -> hist index H + local
    const int32_t nA = lo < 0 ? static_cast<int32_t>((hi < 0 ? hi : 0) - lo) : 0;
    const float2* srcA = p.hist_rd + static_cast<int64_t>(ti.c) * H + (H + lo);
    // piece B: input part, local [max(lo, 0), hi)
    const int64_t bl = lo < 0 ? 0 : lo;
    const int32_t nB = static_cast<int32_t>(hi - bl);
    const float2* srcB = p.x + static_cast<int64_t>(ti.c - p.c_lo) * p.n + bl;
    float2* dstB = win + (bl - lo);
    // snapshot rows kb .. kb + nk (nk + 1 rows) from the ring, wrapping at cap
    const int32_t rows = ti.nk + 1;
    const int64_t s0 = ti.kb % p.cap;
    const int32_t r1 = static_cast<int32_t>((p.cap - s0) < rows ? (p.cap - s0) : rows);
    const float2* ringc = p.ring + static_cast<int64_t>(ti.c) * p.cap * p.Lp;
    auto body_bytes = [](const float2* src, const float2* dst, int32_t count) -> uint32_t {
        if (count <= 0) return 0;
        const uintptr_t sa = reinterpret_cast<uintptr_t>(src);
        const uint32_t da = smem_u32(dst);
        if (((sa ^ da) & 15u) != 0) return 0;
        const int32_t head = (sa & 15u) ? 1 : 0;
        int32_t body = (count - head) & ~1;
        return body < 2 ? 0u : static_cast<uint32_t>(body) * 8u;
    };
    if (lead) {
        tx = body_bytes(srcA, win, nA) + body_bytes(srcB, dstB, nB) +
             body_bytes(ringc + s0 * p.Lp, raw, r1 * p.Lp) +
             body_bytes(ringc, raw + static_cast<int64_t>(r1) * p.Lp, (rows - r1) * p.Lp);
        mbar_arrive_expect_tx(bar, tx);
    }
    stage_copy(win, srcA, nA, bar, lead);
    stage_copy(dstB, srcB, nB, bar, lead);
    stage_copy(raw, ringc + s0 * p.Lp, r1 * p.Lp, bar, lead);
    stage_copy(raw + static_cast<int64_t>(r1) * p.Lp, ringc, (rows - r1) * p.Lp, bar, lead);
}

// One tap of the output-tap loop for the R outputs a lane owns (rows r of its warp).
template <int R>
__device__ __forceinline__ void mac_tap(const float4 q, const float2* __restrict__ xp, const float (&alpha)[R],
                                        float2 (&A)[R], float2 (&B)[R]) {
    const float2 g = make_float2(q.x, q.y);
    const float2 dg = make_float2(q.z, q.w);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const float2 xv = xp[r * 32];
        const float2 h = __ffma2_rn(make_float2(alpha[r], alpha[r]), dg, g);
        A[r] = __ffma2_rn(make_float2(h.x, h.x), xv, A[r]);
        B[r] = __ffma2_rn(make_float2(h.y, h.y), xv, B[r]);
    }
}

template <int R, bool NOISE>
__global__ void __launch_bounds__(kThreads, 2) tt_conv_kernel(const ConvParams p) {
    constexpr int T = kThreads * R;
    extern __shared__ __align__(128) unsigned char smem[];
    // layout: [bar 2 x 8 B][pad to 128][win 2 x (H+T) float2][raw 2 x RAW float2][coef nk_max x L float4][dl L int]
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    const int32_t W = p.H + T;
    const int32_t RAW = (p.nk_max + 1) * p.Lp;
    float2* win0 = reinterpret_cast<float2*>(smem + 128);
    float2* raw0 = win0 + 2 * W;
    float4* coef = reinterpret_cast<float4*>(raw0 + 2 * RAW);
    int32_t* dl = reinterpret_cast<int32_t*>(coef + static_cast<int64_t>(p.nk_max) * p.L);

    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t phase = 0u;  // bit b = parity of buffer b's next completion
    int b = 0;
    int64_t w = blockIdx.x;
    if (w < p.total_tiles) issue_tile<R>(p, w, win0, raw0, &bar[0]);

    for (; w < p.total_tiles; w += gridDim.x, b ^= 1) {
        const int64_t wn = w + gridDim.x;
        if (wn < p.total_tiles) issue_tile<R>(p, wn, win0 + (b ^ 1) * W, raw0 + (b ^ 1) * RAW, &bar[b ^ 1]);
        const TileInfo ti = tile_info<R>(p, w);
        float2* win = win0 + b * W;
        const float2* raw = raw0 + b * RAW;
        mbar_wait(&bar[b], (phase >> b) & 1u);
        phase ^= 1u << b;
        __syncthreads();  // plain-load remainders of this buffer are visible

        // coefficient table in sorted-tap order: coef[kk][j] = (g_k, g_{k+1} - g_k)
        {
            const int32_t* permc = p.perm + static_cast<int64_t>(ti.c) * p.L;
            const int32_t* dc = p.dsort + static_cast<int64_t>(ti.c) * p.L;
            const int32_t tot = ti.nk * p.L;
            for (int32_t e = threadIdx.x; e < tot; e += kThreads) {
                const int32_t kk = e / p.L, j = e - kk * p.L;
                const int32_t src = __ldg(permc + j);
                const float2 g0 = raw[kk * p.Lp + src];
                const float2 g1 = raw[(kk + 1) * p.Lp + src];
                coef[e] = make_float4(g0.x, g0.y, __fsub_rn(g1.x, g0.x), __fsub_rn(g1.y, g0.y));
            }
            for (int32_t j = threadIdx.x; j < p.L; j += kThreads) dl[j] = __ldg(dc + j);
        }
        __syncthreads();

        // per-output interpolation weight alpha = j / S and interval index
        const int32_t obase = warp * 32 * R + lane;
        float alpha[R];
        int32_t kk[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t jj = static_cast<uint32_t>(ti.j0 + obase + r * 32);
            const uint32_t k = jj / static_cast<uint32_t>(p.S);
            // outputs past a tail tile's end are computed but never stored; keep their
            // coefficient row inside the table
            kk[r] = min(static_cast<int32_t>(k), ti.nk - 1);
            alpha[r] = __fdiv_rn(__uint2float_rn(jj - k * static_cast<uint32_t>(p.S)), __int2float_rn(p.S));
        }
        float2 A[R], B[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            A[r] = make_float2(0.f, 0.f);
            B[r] = make_float2(0.f, 0.f);
        }
        const float2* xb = win + p.H + obase;
        // warp-uniform: are all 32R outputs of this warp in one snapshot interval?
        const uint32_t wj0 = static_cast<uint32_t>(ti.j0 + warp * 32 * R);
        const bool uniform = (wj0 / static_cast<uint32_t>(p.S)) ==
                             ((wj0 + 32 * R - 1) / static_cast<uint32_t>(p.S));
        if (warp * 32 * R >= ti.Tt) {
            // whole warp past the tail: nothing to compute
        } else if (uniform) {
            const float4* cf = coef + static_cast<int64_t>(wj0 / static_cast<uint32_t>(p.S)) * p.L;
#pragma unroll 2
            for (int32_t j = 0; j < p.L; ++j) mac_tap<R>(cf[j], xb - dl[j], alpha, A, B);
        } else {
            for (int32_t j = 0; j < p.L; ++j) {
                const float2* xp = xb - dl[j];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float4 q = coef[kk[r] * p.L + j];
                    const float2 xv = xp[r * 32];
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
        for (int r = 0; r < R; ++r) out[r] = make_float2(__fsub_rn(A[r].x, B[r].y), __fadd_rn(A[r].y, B[r].x));
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
                    const float2 wa = ev ? noise_from_words(q.a, q.b, p.noise_sc) : noise_from_words(v0, v1, p.noise_sc);
                    const float2 wb = ev ? noise_from_words(v0, v1, p.noise_sc) : noise_from_words(q.c, q.d, p.noise_sc);
                    out[r] = make_float2(__fadd_rn(out[r].x, wa.x), __fadd_rn(out[r].y, wa.y));
                    out[r + 1] = make_float2(__fadd_rn(out[r + 1].x, wb.x), __fadd_rn(out[r + 1].y, wb.y));
                }
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int64_t n = nb + r * 32;
                    const uint64_t m = static_cast<uint64_t>(n) >> 1;
                    const u32x4 q = philox4x32_10(static_cast<uint32_t>(m), static_cast<uint32_t>(m >> 32), cg, 0u,
                                                  p.key0, p.key1);
                    const float2 wv = (n & 1) ? noise_from_words(q.c, q.d, p.noise_sc)
                                              : noise_from_words(q.a, q.b, p.noise_sc);
                    out[r] = make_float2(__fadd_rn(out[r].x, wv.x), __fadd_rn(out[r].y, wv.y));
                }
            }
        }
        float2* yc = p.y + static_cast<int64_t>(ti.c - p.c_lo) * p.n + ti.i0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int32_t o = obase + r * 32;
            if (o < ti.Tt) yc[o] = out[r];
        }
        // the tile that ends the call writes the new delay-line history (ping-pong)
        if (ti.i0 + ti.Tt == p.n) {
            float2* hw = p.hist_wr + static_cast<int64_t>(ti.c) * p.H;
            const int32_t off = ti.Tt;  // window index of local sample n - H is (n - H) - (i0 - H) = Tt
            for (int32_t i = threadIdx.x; i < p.H; i += kThreads) hw[i] = win[off + i];
        }
        __syncthreads();  // buffer b, coef and dl are free for reuse
    }
}

// Generic path: one thread per output, operands straight from global memory. Used
// when the tiled kernel's shared-memory plan does not fit (very long filters with very
// short snapshot periods). Same per-output operation sequence => bit-identical.
template <bool NOISE>
__global__ void __launch_bounds__(kThreads) tt_conv_generic_kernel(const ConvParams p) {
    const int64_t nch = p.total_tiles / p.tiles_per_ch;
    const int64_t N = nch * p.n;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; e < N;
         e += static_cast<int64_t>(gridDim.x) * kThreads) {
        const int64_t cl = e / p.n;
        const int64_t i = e - cl * p.n;
        const int32_t c = p.c_lo + static_cast<int32_t>(cl);
        const int64_t n = p.t + i;
        const int64_t k = n / p.S;
        const int32_t jj = static_cast<int32_t>(n - k * p.S);
        const float alpha = __fdiv_rn(__uint2float_rn(static_cast<uint32_t>(jj)), __int2float_rn(p.S));
        const float2* g0r = p.ring + (static_cast<int64_t>(c) * p.cap + (k % p.cap)) * p.Lp;
        const float2* g1r = p.ring + (static_cast<int64_t>(c) * p.cap + ((k + 1) % p.cap)) * p.Lp;
        const float2* xc = p.x + cl * p.n;
        const float2* hc = p.hist_rd + static_cast<int64_t>(c) * p.H;
        float2 A = make_float2(0.f, 0.f), Bv = make_float2(0.f, 0.f);
        for (int32_t j = 0; j < p.L; ++j) {
            const int32_t src = __ldg(p.perm + static_cast<int64_t>(c) * p.L + j);
            const int32_t d = __ldg(p.dsort + static_cast<int64_t>(c) * p.L + j);
            const float2 g0 = __ldg(g0r + src), g1 = __ldg(g1r + src);
            const float2 dg = make_float2(__fsub_rn(g1.x, g0.x), __fsub_rn(g1.y, g0.y));
            const int64_t m = i - d;
            const float2 xv = m >= 0 ? __ldg(xc + m) : __ldg(hc + (p.H + m));
            const float2 h = __ffma2_rn(make_float2(alpha, alpha), dg, g0);
            A = __ffma2_rn(make_float2(h.x, h.x), xv, A);
            Bv = __ffma2_rn(make_float2(h.y, h.y), xv, Bv);
        }
        float2 o = make_float2(__fsub_rn(A.x, Bv.y), __fadd_rn(A.y, Bv.x));
        if constexpr (NOISE) {
            const uint64_t mm = static_cast<uint64_t>(n) >> 1;
            const u32x4 q = philox4x32_10(static_cast<uint32_t>(mm), static_cast<uint32_t>(mm >> 32),
                                          static_cast<uint32_t>(p.chan_offset + c), 0u, p.key0, p.key1);
            const float2 wv = (n & 1) ? noise_from_words(q.c, q.d, p.noise_sc) : noise_from_words(q.a, q.b, p.noise_sc);
            o = make_float2(__fadd_rn(o.x, wv.x), __fadd_rn(o.y, wv.y));
        }
        p.y[cl * p.n + i] = o;
    }
}

// History update for the generic path (the tiled kernel fuses it): the new history is
// the last H samples of (old history ++ x).
__global__ void tt_history_kernel(const ConvParams p, int32_t nch) {
    const int64_t tot = static_cast<int64_t>(nch) * p.H;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < tot;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t cl = e / p.H;
        const int32_t i = static_cast<int32_t>(e - cl * p.H);
        const int32_t c = p.c_lo + static_cast<int32_t>(cl);
        const int64_t m = p.n - p.H + i;  // call-local index of the sample
        p.hist_wr[static_cast<int64_t>(c) * p.H + i] =
            m >= 0 ? p.x[cl * p.n + m] : p.hist_rd[static_cast<int64_t>(c) * p.H + (p.H + m)];
    }
}

}  // namespace tt
