// tt_conv_dw.cuh — the dense-window ("dw") convolution kernel for sm_100a: the fast path
// of tt_channel_apply when the taps are DENSE in delay (mean gap between sorted delays
// well below 16 samples, e.g. BASELINE c5: L taps in [0, 4L]). Same per-output arithmetic
// as tt_conv.cuh (NS formula; §III-B, §IV), so the outputs are
// bit-identical to the tiled and generic kernels':
//
//   h = fma(alpha_n, g_{k+1} - g_k, g_k),  A += h.re * x,  B += h.im * x  (taps ascending
//   by delay),  y = (A.re - B.im, A.im + B.re) + w.
//
// Why. The tiled kernel reads one 8-B x operand from shared memory per
// output-tap, so it is bound by shared-memory bandwidth (128 B/clk/SM). Here each thread
// owns R = 16 CONSECUTIVE outputs and keeps two aligned 16-sample blocks of x in
// registers: the block holding x[n0 - d .. n0 - d + 15]'s high part (HI) and the one
// before it (LO). A tap at delay d = 16 q + f reads its 16 operands from registers at the
// static offset f (a warp-uniform switch over f and the blocks' register parity). Taps
// are sorted by delay, so q only grows: when it grows by 1 the old LO becomes HI and one
// new block is read; a thread reads about (D + 32) / (16 L) samples per output-tap
// instead of 1 (c5: 0.26-0.38), and the kernel becomes FMA-bound.
//
// Layout. The window x[n0 - Hw, n0 + T) is staged by 2-D TMA tensor copies with the
// 128-B swizzle: window row rho (16 samples, 128 B) keeps its 16-B chunk i at chunk
// i ^ (rho & 7), so the 8 lanes of a quarter-warp reading aligned chunk i of 8 different
// rows hit 8 different bank groups: every block read is a conflict-free LDS.128. The
// part of the window before the call start comes from the carried delay line (a second
// tensor map over the history buffer). Outputs go through a per-warp swizzled staging
// tile and a 2-D TMA tensor store (rows past the call end are clipped by the map).
//
// Pipeline: persistent CTAs (one per SM), CW consumer warps + 1 producer warp, a ring of
// shared-memory stages with full/empty mbarriers (as tt_conv.cuh).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "tt_conv.cuh"
#include "tt_noise.cuh"

namespace tt {
namespace dw {

constexpr int R = 16;           // consecutive outputs per thread
constexpr int kRowBytes = 128;  // one window row = 16 complex samples
constexpr int kXBoxRows = 32;   // x / y tensor-map box: 32 rows (4 KB)
constexpr int kHBoxRows = 8;    // history tensor-map box: 8 rows (1 KB)
constexpr int kMaxStages = 4;

struct Params {
    const float4* ring;     // [C][cap][L] (g_k, g_{k+1} - g_k), taps sorted by delay
    const int32_t* tab;     // [C][L4] per sorted tap: f | dq class << 4 | q << 8 (d = 16 q + f)
    float2* hist_wr;        // [C][H] receives the new delay line
    int64_t n;              // samples per channel in this call (multiple of 16)
    int64_t t;              // global index of the call's first sample (multiple of 16)
    int64_t cap;            // ring slots per channel
    int64_t chan_offset;    // global id of channel 0 (noise key)
    int64_t t_div;          // t / S
    int64_t total_tiles;
    int32_t t_mod;          // t % S
    int32_t c_lo;           // first channel of this launch
    int32_t tiles_per_ch;
    int32_t L, L4, H, Hw, S;  // Hw = H rounded up to 128: window rows before n0 (multiple of 8)
    int32_t s_shift;        // log2(S) if S is a power of two, else -1
    float inv_S;
    int32_t nk_max;         // gain rows staged per tile
    int32_t stages;
    int32_t win_rows;       // window rows allocated per stage (multiple of kXBoxRows)
    int32_t hist_row0;      // history-map row of window row 0 when n0 = 0: (H - Hw) / 16
    int32_t stage_bytes;    // bytes per stage (multiple of 1024)
    int32_t coef_off, tab_off;  // byte offsets of the gain rows / tap table in a stage
    uint32_t key0, key1;    // noise key
    float noise_sc;         // sigma / sqrt(2); 0 = no noise
};

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Window row rho (16 samples) into X: chunk i (samples 2i, 2i+1) sits at chunk i ^ (rho & 7)
// of the row (TMA 128-B swizzle; the window base is 1024-B aligned).
// (Plain C++ loads through a shared-space pointer: the compiler schedules them freely
// but never across the mbarrier waits, which clobber memory.)
__device__ __forceinline__ void load_block(float2 (&X)[R], const unsigned char* win, int32_t rho) {
    const uint32_t a = (static_cast<uint32_t>(rho) * kRowBytes) | ((static_cast<uint32_t>(rho) & 7u) << 4);
#pragma unroll
    for (int i = 0; i < R / 2; ++i) {
        const float4 v = *reinterpret_cast<const float4*>(win + (a ^ (static_cast<uint32_t>(i) << 4)));
        X[2 * i] = make_float2(v.x, v.y);
        X[2 * i + 1] = make_float2(v.z, v.w);
    }
}

// One tap at in-block offset F with HI in P (PAR = 0) or Q (PAR = 1): operand r is
// HI[r - F] (r >= F) or LO[16 + r - F] (r < F). Same operation sequence per output as
// mac_tap in tt_conv.cuh.
template <int F, int PAR>
__device__ __forceinline__ void tap_case(const float4 q, const float (&alpha)[R], const float2 (&P)[R],
                                         const float2 (&Q)[R], float2 (&A)[R], float2 (&B)[R]) {
    const float2 g = make_float2(q.x, q.y);
    const float2 dg = make_float2(q.z, q.w);
    // all gains first (independent FFMA2s), then the MACs: no RAW stall on a shared temp
    float2 h[R];
#pragma unroll
    for (int r = 0; r < R; ++r) h[r] = __ffma2_rn(make_float2(alpha[r], alpha[r]), dg, g);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const float2 xv = r >= F ? (PAR ? Q[r - F] : P[r - F]) : (PAR ? P[R + r - F] : Q[R + r - F]);
        A[r] = __ffma2_rn(make_float2(h[r].x, h[r].x), xv, A[r]);
        B[r] = __ffma2_rn(make_float2(h[r].y, h[r].y), xv, B[r]);
    }
}

// Per-tap dispatch: a warp-uniform switch over (f, parity) (ptxas lowers it to a
// compare-and-branch tree; see DESIGN.md §5.5 for what that costs).
__device__ __forceinline__ void tap_dispatch(int sel, const float4 q, const float (&alpha)[R], const float2 (&P)[R],
                                             const float2 (&Q)[R], float2 (&A)[R], float2 (&B)[R]) {
#define TT_DW_CASE(F)                                    \
    case F: tap_case<F, 0>(q, alpha, P, Q, A, B); break; \
    case 16 + F: tap_case<F, 1>(q, alpha, P, Q, A, B); break;
    switch (sel) {
        TT_DW_CASE(0) TT_DW_CASE(1) TT_DW_CASE(2) TT_DW_CASE(3) TT_DW_CASE(4) TT_DW_CASE(5) TT_DW_CASE(6)
        TT_DW_CASE(7) TT_DW_CASE(8) TT_DW_CASE(9) TT_DW_CASE(10) TT_DW_CASE(11) TT_DW_CASE(12) TT_DW_CASE(13)
        TT_DW_CASE(14) TT_DW_CASE(15)
        default: __builtin_unreachable();
    }
#undef TT_DW_CASE
}

__device__ __forceinline__ uint32_t divS(const Params& p, uint32_t v) {
    return p.s_shift >= 0 ? (v >> p.s_shift) : v / static_cast<uint32_t>(p.S);
}

// The (channel, tile) walk of tt_conv.cuh's plain variant.
template <int CW, bool NOISE>
__global__ void __launch_bounds__((CW + 1) * 32, 1)
    tt_conv_dw_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmy,
                      const __grid_constant__ CUtensorMap tmh, const Params p) {
    constexpr int T = CW * 32 * R;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // [full kMaxStages x 8 | empty kMaxStages x 8 | pad to 1024][stage 0]...[stage S-1][staging CW x 4 KB]
    // (aligned by pointer arithmetic on smem_raw, so the compiler keeps the shared state space)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kMaxStages;
    unsigned char* stage0 = smem + 1024;
    unsigned char* staging = stage0 + static_cast<size_t>(p.stages) * p.stage_bytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp == CW) {
        // ---- producer: stage window, gain rows and tap table of each work item ----------
        int s = 0, kk = 0;
        TileWalk tw(static_cast<uint32_t>(p.tiles_per_ch));
        for (int64_t w = blockIdx.x; w < p.total_tiles; w += gridDim.x, tw.next()) {
            if (kk > 0) mbar_wait(&empty[s], (kk - 1) & 1);
            unsigned char* st = stage0 + static_cast<size_t>(s) * p.stage_bytes;
            const int32_t cl = static_cast<int32_t>(tw.cl), c = p.c_lo + cl;
            const int64_t n0 = static_cast<int64_t>(tw.tl) * T;
            const int32_t Tt = static_cast<int32_t>(p.n - n0 < T ? p.n - n0 : T);
            const uint32_t u0 = static_cast<uint32_t>(p.t_mod) + static_cast<uint32_t>(n0);
            const uint32_t kq = divS(p, u0);
            const int32_t nk = static_cast<int32_t>(divS(p, u0 + static_cast<uint32_t>(Tt) - 1u) - kq) + 1;
            // window boxes: history rows (first tile only), then x rows
            const int32_t hrows = n0 == 0 ? p.Hw / 16 : 0;               // multiple of 8
            const int32_t xrow_first = static_cast<int32_t>((n0 - p.Hw) / 16) + hrows;  // x row of window row hrows
            const int32_t xrows = (p.Hw + T) / 16 - hrows;
            const int32_t nhb = hrows / kHBoxRows, nxb = (xrows + kXBoxRows - 1) / kXBoxRows;
            // gain rows kb .. kb + nk - 1 (ring wraps at cap), tap table row
            const int64_t s0 = (p.t_div + kq) % p.cap;
            const int32_t r1 = static_cast<int32_t>((p.cap - s0) < nk ? (p.cap - s0) : nk);
            const uint32_t rowb = static_cast<uint32_t>(p.L) * 16u;
            const float4* ringc = p.ring + static_cast<int64_t>(c) * p.cap * p.L;
            const uint32_t bytes = static_cast<uint32_t>(nhb) * kHBoxRows * kRowBytes +
                                   static_cast<uint32_t>(nxb) * kXBoxRows * kRowBytes + static_cast<uint32_t>(nk) * rowb +
                                   static_cast<uint32_t>(p.L4) * 4u;
            if (lane == 0) mbar_arrive_expect_tx(&full[s], bytes);
            __syncwarp();
            for (int b = lane; b < nhb + nxb + 3; b += 32) {
                if (b < nhb) {
                    tma_load_3d(st + b * kHBoxRows * kRowBytes, &tmh, 0, p.hist_row0 + b * kHBoxRows, c, &full[s]);
                } else if (b < nhb + nxb) {
                    const int xb = b - nhb;
                    tma_load_3d(st + (hrows + xb * kXBoxRows) * kRowBytes, &tmx, 0, xrow_first + xb * kXBoxRows, cl,
                                &full[s]);
                } else if (b == nhb + nxb) {
                    tma_load_1d(st + p.coef_off, ringc + s0 * p.L, static_cast<uint32_t>(r1) * rowb, &full[s]);
                } else if (b == nhb + nxb + 1) {
                    if (nk > r1)
                        tma_load_1d(st + p.coef_off + static_cast<size_t>(r1) * rowb, ringc,
                                    static_cast<uint32_t>(nk - r1) * rowb, &full[s]);
                } else {
                    tma_load_1d(st + p.tab_off, p.tab + static_cast<int64_t>(c) * p.L4, static_cast<uint32_t>(p.L4) * 4u,
                                &full[s]);
                }
            }
            if (++s == p.stages) {
                s = 0;
                ++kk;
            }
        }
        return;
    }

    // ---- consumers -------------------------------------------------------------------
    const int tid = warp * 32 + lane;
    unsigned char* stg = staging + warp * (32 * kRowBytes);  // this warp's 32-row output tile (1024-aligned)
    int s = 0;
    uint32_t ph = 0;
    TileWalk tw(static_cast<uint32_t>(p.tiles_per_ch));
    for (int64_t w = blockIdx.x; w < p.total_tiles; w += gridDim.x, tw.next()) {
        mbar_wait(&full[s], ph);
        unsigned char* st = stage0 + static_cast<size_t>(s) * p.stage_bytes;
        const unsigned char* win = st;
        const int32_t cl = static_cast<int32_t>(tw.cl), c = p.c_lo + cl;
        const int64_t n0 = static_cast<int64_t>(tw.tl) * T;
        const int64_t nf = n0 + static_cast<int64_t>(tid) * R;  // this thread's first output (call-local)
        if (n0 + static_cast<int64_t>(warp) * 32 * R < p.n) {
            // interpolation weights: the thread's 16 outputs sit in one snapshot interval
            const uint32_t u0 = static_cast<uint32_t>(p.t_mod) + static_cast<uint32_t>(n0);
            const uint32_t uf = static_cast<uint32_t>(p.t_mod) + static_cast<uint32_t>(nf);
            const uint32_t kf = divS(p, uf);
            const uint32_t j0 = uf - kf * static_cast<uint32_t>(p.S);
            float alpha[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                alpha[r] = p.s_shift >= 0 ? __fmul_rn(__uint2float_rn(j0 + r), p.inv_S)
                                          : __fdiv_rn(__uint2float_rn(j0 + r), __int2float_rn(p.S));
            }
            const float4* cf = reinterpret_cast<const float4*>(st + p.coef_off) + (kf - divS(p, u0)) * p.L;
            const int32_t* tb = reinterpret_cast<const int32_t*>(st + p.tab_off);
            float2 P[R], Q[R], A[R], B[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                A[r] = make_float2(0.f, 0.f);
                B[r] = make_float2(0.f, 0.f);
            }
            const int32_t base_rho = tid + p.Hw / 16;
            int par = 0;
            int32_t e = tb[0];
            float4 q = cf[0];
            for (int32_t j = 0; j < p.L; ++j) {
                const int32_t en = tb[j + 1];
                const float4 qn = cf[j + 1];
                const int32_t rho_hi = base_rho - (e >> 8);
                const int dqc = (e >> 4) & 3;
                if (dqc == 2) {
                    if (par) {
                        load_block(Q, win, rho_hi);
                        load_block(P, win, rho_hi - 1);
                    } else {
                        load_block(P, win, rho_hi);
                        load_block(Q, win, rho_hi - 1);
                    }
                } else if (dqc == 1) {
                    if (par) load_block(Q, win, rho_hi - 1);
                    else load_block(P, win, rho_hi - 1);
                    par ^= 1;
                }
                tap_dispatch((e & 15) + 16 * par, q, alpha, P, Q, A, B);
                e = en;
                q = qn;
            }
            // epilogue: combine, noise, stage (swizzled), TMA store of the warp's 32 rows
            float2 out[R];
#pragma unroll
            for (int r = 0; r < R; ++r) out[r] = make_float2(__fsub_rn(A[r].x, B[r].y), __fadd_rn(A[r].y, B[r].x));
            if constexpr (NOISE) {
                const uint32_t cg = static_cast<uint32_t>(p.chan_offset + c);
                const int64_t gf = p.t + nf;  // even (multiple of 16)
#pragma unroll
                for (int r = 0; r < R; r += 4) {
                    const uint64_t m0 = static_cast<uint64_t>(gf + r) >> 1, m1 = m0 + 1;
                    const u32x4 z0 = philox4x32_10(static_cast<uint32_t>(m0), static_cast<uint32_t>(m0 >> 32), cg, 0u,
                                                   p.key0, p.key1);
                    const u32x4 z1 = philox4x32_10(static_cast<uint32_t>(m1), static_cast<uint32_t>(m1 >> 32), cg, 0u,
                                                   p.key0, p.key1);
                    float2 w0, w1, w2, w3;
                    noise_from_words2(z0.a, z0.b, z0.c, z0.d, p.noise_sc, w0, w1);
                    noise_from_words2(z1.a, z1.b, z1.c, z1.d, p.noise_sc, w2, w3);
                    out[r] = make_float2(__fadd_rn(out[r].x, w0.x), __fadd_rn(out[r].y, w0.y));
                    out[r + 1] = make_float2(__fadd_rn(out[r + 1].x, w1.x), __fadd_rn(out[r + 1].y, w1.y));
                    out[r + 2] = make_float2(__fadd_rn(out[r + 2].x, w2.x), __fadd_rn(out[r + 2].y, w2.y));
                    out[r + 3] = make_float2(__fadd_rn(out[r + 3].x, w3.x), __fadd_rn(out[r + 3].y, w3.y));
                }
            }
            // the previous tile's store must have finished reading the staging tile
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
            const uint32_t sw = (static_cast<uint32_t>(lane) & 7u) << 4;
            unsigned char* row = stg + lane * kRowBytes;
#pragma unroll
            for (int i = 0; i < R / 2; ++i)
                *reinterpret_cast<float4*>(row + ((static_cast<uint32_t>(i) << 4) ^ sw)) =
                    make_float4(out[2 * i].x, out[2 * i].y, out[2 * i + 1].x, out[2 * i + 1].y);
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                tma_store_3d(&tmy, stg, 0, static_cast<int32_t>((n0 + static_cast<int64_t>(warp) * 32 * R) / 16), cl);
                bulk_commit();
            }
        }
        // the tile that ends the call writes the new delay line from the staged window:
        // call-local sample n - H + i is window row (n - H + i - n0 + Hw) / 16
        if (n0 + T >= p.n) {
            float2* hw = p.hist_wr + static_cast<int64_t>(c) * p.H;
            const int32_t v0 = static_cast<int32_t>(p.n - p.H - n0 + p.Hw);
            for (int32_t i = tid; i < p.H; i += CW * 32) {
                const int32_t v = v0 + i;
                const int32_t rho = v >> 4, k = v & 15;
                const uint32_t a = static_cast<uint32_t>(rho) * kRowBytes +
                                   ((((static_cast<uint32_t>(k) >> 1) ^ (static_cast<uint32_t>(rho) & 7u)) << 4) |
                                    ((static_cast<uint32_t>(k) & 1u) << 3));
                hw[i] = *reinterpret_cast<const float2*>(win + a);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == p.stages) {
            s = 0;
            ph ^= 1u;
        }
    }
    if (lane == 0) bulk_wait0();  // outstanding output stores complete before the CTA exits
}

}  // namespace dw
}  // namespace tt
