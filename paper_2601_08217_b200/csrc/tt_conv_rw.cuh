// tt_conv_rw.cuh — the register-window convolution kernel (sm_100a), the fast path of
// tt_channel_apply for snapshot periods S that are multiples of 16 (every BASELINE
// config). Same per-output arithmetic as tt_conv.cuh (NS formula; §III-B,
// P:309, §IV), so its outputs are bit-identical to the other kernels':
//
//   h = fma(alpha_n, g_{k+1} - g_k, g_k),  A += h.re * x,  B += h.im * x  (taps ascending
//   by delay),  y = (A.re - B.im, A.im + B.re) + w.
//
// Why a register window. With one 8-B shared-memory read per output-tap
// the kernel is bound by shared-memory bandwidth (128 B/clk/SM -> 16 output-taps/clk/SM,
// below the 21 the FMA pipe allows at 6 lanes per output-tap). Here each thread owns
// R = 16 CONSECUTIVE outputs and keeps the 16 x samples x[n0 - d_j + r] of the current tap
// in registers. Taps are sorted by delay, so moving to the next tap (delay gap s) shifts
// the window by s: the thread keeps 16 - s samples and reads only s fresh ones. The
// window rotates through the registers instead of moving (see tap_rot), so the kept
// samples cost nothing; every lane of the CTA works on the same channel, so the
// rotation switch is warp-uniform. At c4 (48 taps in [0, 1024]) that is ~0.7 shared-memory reads per
// output-tap instead of 1.
//
// Shared-memory layout ("doubled blocks"). Lane spans are 16 samples apart; a plain
// linear window would put all 16 lanes of a half-warp on the same bank. The window is
// stored as blocks of 33 8-B slots: block k holds window samples 16k .. 16k+31 (its own 16
// and the next block's 16) plus one pad slot. Thread t's fresh run for a tap with window
// offset o is block (o >> 4) + t, slots (o & 15) + r, r < s <= 16 — always inside one
// block, so the address is (thread base) + (per-tap uniform offset) + 8r with compile-
// time r, and the 33-slot (odd) stride makes every half-warp access conflict-free. TMA
// cannot write an odd 8-B stride (16-B granularity), so the window is filled with
// 8-byte cp.async (LDGSTS) copies whose completion arrives on an mbarrier.
//
// Pipeline. Persistent CTAs (one per SM) of 8 symmetric warps walk (channel, tile)
// items, tile = 8 x 32 x 16 = 4096 outputs. Two window stages: while the warps compute
// tile i from one stage, each warp has already issued its 1/8 share of tile i+1's
// copies into the other (full mbarrier: 256 cp.async arrivals; empty mbarrier: 8 warp
// arrivals). The same copies stage the tile's gain rows (16-B cp.async) and the
// channel's tap table next to the window, so the tap loop reads only shared memory.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tt_noise.cuh"

namespace tt {
namespace rw {

constexpr int R = 16;                       // outputs per thread
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int T = kThreads * R;             // outputs per tile
constexpr int kSlots = 33;                  // 8-B slots per doubled block (32 samples + pad)
constexpr int kBlockBytes = kSlots * 8;

struct Params {
    const float2* x;        // [C_launch][n]: row 0 = channel c_lo
    float2* y;              // [C_launch][n]
    const float2* hist_rd;  // [C][H]  last H samples of the stream so far
    float2* hist_wr;        // [C][H]  receives the new delay line
    const float4* ring;     // [C][cap][L] (g_k, g_{k+1} - g_k), taps sorted by delay (+1 float4 pad)
    const int2* tab;        // [C][L + 1] per sorted tap: (window byte offset, fresh samples s)
    int64_t n;              // samples per channel in this call
    int64_t t;              // global index of the call's first sample
    int64_t cap;            // ring slots per channel
    int64_t chan_offset;    // global id of channel 0 (noise key)
    int64_t total_tiles;
    int32_t c_lo;           // first channel of this launch
    int32_t tiles_per_ch;
    int32_t L, H, Hp, S;    // H = history length = Hp + 16; window = Hp + T samples
    int32_t a;              // t mod 16: the first tile starts at call-local -a (16-aligned)
    int32_t nb;             // doubled blocks per stage = (Hp + T) / 16
    int32_t s_shift;        // log2(S) if S is a power of two, else -1
    float inv_S;
    uint32_t key0, key1;    // noise key
    float noise_sc;         // sigma / sqrt(2); 0 = no noise
    int32_t vec_store;      // 1: every 16-output span starts 16-B aligned in y (n, a even)
    int32_t rows;           // gain rows a tile touches (<= (T - 1) / S + 2)
    int32_t row_stride;     // bytes per staged gain row: 16 L + 16 (the pad spreads rows over banks)
    int32_t wbytes;         // window bytes per stage (nb x 264, rounded up to 16)
    int32_t sbytes;         // stage bytes: window | gain rows | tap table
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t a = smem_addr(bar);
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}
// 8-byte async copy global -> shared; src_bytes = 0 zero-fills the destination
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
// this thread's prior cp.async copies arrive on `bar` when complete (no pending-count bump)
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// Issue this warp's share of the copies that fill `win` with tile w's window:
// window sample q (0 <= q < Hp + T) is call-local v = v0 - Hp + q; it comes from the
// carried history (v < 0), this call's input (v < n), or is zero (v >= n). It is
// written to slot (q & 15) of block q >> 4 and to slot 16 + (q & 15) of block (q >> 4) - 1.
__device__ __forceinline__ void fill_window(const Params& p, int64_t w, unsigned char* win, int warp, int lane) {
    const int32_t cl = static_cast<int32_t>(w / p.tiles_per_ch);
    const int32_t tl = static_cast<int32_t>(w - static_cast<int64_t>(cl) * p.tiles_per_ch);
    const int32_t c = p.c_lo + cl;
    const int64_t vbase = static_cast<int64_t>(tl) * T - p.a - p.Hp;  // call-local sample of q = 0
    const float2* xr = p.x + static_cast<int64_t>(cl) * p.n;
    const float2* hr = p.hist_rd + static_cast<int64_t>(c) * p.H + p.H;  // hr[v] for -H <= v < 0
    const uint32_t wb = smem_addr(win);
    const int32_t nq = p.Hp + T;
    const int tid = warp * 32 + lane;
    // the tile's gain rows (16-B copies, ring slots wrap at cap) and the channel's tap table
    {
        const int64_t n0 = p.t + static_cast<int64_t>(tl) * T - p.a;  // global, 16-aligned, >= 0
        const int64_t k0 = p.s_shift >= 0 ? (n0 >> p.s_shift) : n0 / p.S;
        const uint32_t cb = wb + p.wbytes;
        const int32_t tot = p.rows * p.L;
        for (int32_t i = tid; i < tot; i += kThreads) {
            const int32_t r = i / p.L, jj = i - r * p.L;
            const int64_t slot = (k0 + r) % p.cap;
            const float4* src = p.ring + (static_cast<int64_t>(c) * p.cap + slot) * p.L + jj;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(cb + r * p.row_stride + jj * 16), "l"(src)
                         : "memory");
        }
        const uint32_t tbs = cb + p.rows * p.row_stride;
        const int2* tsrc = p.tab + static_cast<int64_t>(c) * (p.L + 1);
        for (int32_t i = tid; i <= p.L; i += kThreads) cp_async8(tbs + i * 8, tsrc + i, 8);
    }
    for (int32_t q = warp * 32 + lane; q < nq; q += kThreads) {
        const int64_t v = vbase + q;
        const float2* src;
        uint32_t sz = 8;
        if (v < 0) {
            src = hr + v;
        } else if (v < p.n) {
            src = xr + v;
        } else {
            src = xr;
            sz = 0;
        }
        const uint32_t k = static_cast<uint32_t>(q) >> 4, o = static_cast<uint32_t>(q) & 15u;
        const uint32_t d0 = wb + k * kBlockBytes + o * 8u;
        cp_async8(d0, src, sz);
        if (k > 0) cp_async8(d0 - kBlockBytes + 128u, src, sz);  // slot 16 + o of block k - 1
    }
}

// One tap on a ROTATING register window: window sample r (x[n0 - d + r]) lives in
// register (RHO + r) & 15. Advancing to a tap whose delay is s larger moves the window
// s samples earlier, which is just RHO' = RHO - s (mod 16): the 16 - s kept samples stay
// where they are and the s fresh ones (r < s) overwrite the evicted registers. So there
// are no register moves; the price is one copy of this body per rotation, selected by a
// warp-uniform switch, and 16 predicated loads (r < s) per tap.
template <int RHO>
__device__ __forceinline__ void tap_rot(int s, const float2* __restrict__ src, float2 (&xw)[R],
                                        const float2 (&h)[R], float2 (&A)[R], float2 (&B)[R]) {
#pragma unroll
    for (int r = 0; r < R; ++r)
        if (r < s) xw[(RHO + r) & (R - 1)] = src[r];
#pragma unroll
    for (int r = R - 1; r >= 0; --r) {
        const float2 xv = xw[(RHO + r) & (R - 1)];
        A[r] = __ffma2_rn(make_float2(h[r].x, h[r].x), xv, A[r]);
        B[r] = __ffma2_rn(make_float2(h[r].y, h[r].y), xv, B[r]);
    }
}

__device__ __forceinline__ void tap(int rho, int s, const float2* __restrict__ src, float2 (&xw)[R],
                                    const float2 (&h)[R], float2 (&A)[R], float2 (&B)[R]) {
    switch (rho) {
        case 0: tap_rot<0>(s, src, xw, h, A, B); break;
        case 1: tap_rot<1>(s, src, xw, h, A, B); break;
        case 2: tap_rot<2>(s, src, xw, h, A, B); break;
        case 3: tap_rot<3>(s, src, xw, h, A, B); break;
        case 4: tap_rot<4>(s, src, xw, h, A, B); break;
        case 5: tap_rot<5>(s, src, xw, h, A, B); break;
        case 6: tap_rot<6>(s, src, xw, h, A, B); break;
        case 7: tap_rot<7>(s, src, xw, h, A, B); break;
        case 8: tap_rot<8>(s, src, xw, h, A, B); break;
        case 9: tap_rot<9>(s, src, xw, h, A, B); break;
        case 10: tap_rot<10>(s, src, xw, h, A, B); break;
        case 11: tap_rot<11>(s, src, xw, h, A, B); break;
        case 12: tap_rot<12>(s, src, xw, h, A, B); break;
        case 13: tap_rot<13>(s, src, xw, h, A, B); break;
        case 14: tap_rot<14>(s, src, xw, h, A, B); break;
        case 15: tap_rot<15>(s, src, xw, h, A, B); break;
        default: __builtin_unreachable();
    }
}

template <bool NOISE>
__device__ __forceinline__ void compute_tile(const Params& p, int64_t w, const unsigned char* win, int tid) {
    const int32_t cl = static_cast<int32_t>(w / p.tiles_per_ch);
    const int32_t tl = static_cast<int32_t>(w - static_cast<int64_t>(cl) * p.tiles_per_ch);
    const int32_t c = p.c_lo + cl;
    const int64_t v_first = static_cast<int64_t>(tl) * T - p.a + static_cast<int64_t>(tid) * R;  // call-local
    if (v_first >= p.n) return;  // whole span past the end of the call (tail tile)
    const int64_t n_first = p.t + v_first;                                                       // global, % 16 == 0
    int64_t k;
    int32_t j0;
    if (p.s_shift >= 0) {
        k = n_first >> p.s_shift;
        j0 = static_cast<int32_t>(n_first & (p.S - 1));
    } else {
        k = n_first / p.S;
        j0 = static_cast<int32_t>(n_first - k * p.S);
    }
    float alpha[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const float jf = __int2float_rn(j0 + r);
        alpha[r] = p.s_shift >= 0 ? __fmul_rn(jf, p.inv_S) : __fdiv_rn(jf, __int2float_rn(p.S));
    }
    // staged gain row of this thread's interval, and the staged tap table
    const int64_t n_tile = p.t + static_cast<int64_t>(tl) * T - p.a;
    const int64_t k_tile = p.s_shift >= 0 ? (n_tile >> p.s_shift) : n_tile / p.S;
    const float4* cf = reinterpret_cast<const float4*>(win + p.wbytes + (k - k_tile) * p.row_stride);
    const int2* tb = reinterpret_cast<const int2*>(win + p.wbytes + p.rows * p.row_stride);
    const unsigned char* wt = win + tid * kBlockBytes;  // this thread's block base

    float2 xw[R], A[R], B[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        xw[r] = make_float2(0.f, 0.f);
        A[r] = make_float2(0.f, 0.f);
        B[r] = make_float2(0.f, 0.f);
    }
    int2 e = tb[0];
    float4 q = cf[0];
    int rho = 0;
#pragma unroll 2
    for (int32_t j = 0; j < p.L; ++j) {
        const int2 en = tb[j + 1];   // the table has L + 1 entries
        const float4 qn = cf[j + 1];  // row pad: one float4 past the row's last tap
        const float2 g = make_float2(q.x, q.y);
        const float2 dg = make_float2(q.z, q.w);
        float2 h[R];
#pragma unroll
        for (int r = 0; r < R; ++r) h[r] = __ffma2_rn(make_float2(alpha[r], alpha[r]), dg, g);
        rho = (rho - e.y) & (R - 1);  // e.y = fresh samples s (16 for the first tap)
        tap(rho, e.y, reinterpret_cast<const float2*>(wt + e.x), xw, h, A, B);
        e = en;
        q = qn;
    }

    float2 out[R];
#pragma unroll
    for (int r = 0; r < R; ++r) out[r] = make_float2(__fsub_rn(A[r].x, B[r].y), __fadd_rn(A[r].y, B[r].x));
    if constexpr (NOISE) {
        const uint32_t cg = static_cast<uint32_t>(p.chan_offset + c);
#pragma unroll
        for (int r = 0; r < R; r += 2) {
            const uint64_t m = static_cast<uint64_t>(n_first + r) >> 1;  // n_first + r is even
            const u32x4 z = philox4x32_10(static_cast<uint32_t>(m), static_cast<uint32_t>(m >> 32), cg, 0u, p.key0,
                                          p.key1);
            const float2 wa = noise_from_words(z.a, z.b, p.noise_sc);
            const float2 wb = noise_from_words(z.c, z.d, p.noise_sc);
            out[r] = make_float2(__fadd_rn(out[r].x, wa.x), __fadd_rn(out[r].y, wa.y));
            out[r + 1] = make_float2(__fadd_rn(out[r + 1].x, wb.x), __fadd_rn(out[r + 1].y, wb.y));
        }
    }
    float2* yr = p.y + static_cast<int64_t>(cl) * p.n + v_first;
    if (p.vec_store && v_first >= 0 && v_first + R <= p.n) {
        float4* y4 = reinterpret_cast<float4*>(yr);
#pragma unroll
        for (int r = 0; r < R; r += 2) y4[r >> 1] = make_float4(out[r].x, out[r].y, out[r + 1].x, out[r + 1].y);
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t v = v_first + r;
            if (v >= 0 && v < p.n) yr[r] = out[r];
        }
    }
}

// the tile that ends a channel's call writes the new delay line (the last H samples of
// old history ++ x) from global memory into the other ping-pong buffer
__device__ __forceinline__ void write_history(const Params& p, int32_t cl, int tid) {
    const int32_t c = p.c_lo + cl;
    const float2* xr = p.x + static_cast<int64_t>(cl) * p.n;
    const float2* hr = p.hist_rd + static_cast<int64_t>(c) * p.H;
    float2* hw = p.hist_wr + static_cast<int64_t>(c) * p.H;
    for (int32_t i = tid; i < p.H; i += kThreads) {
        const int64_t m = p.n - p.H + i;
        hw[i] = m >= 0 ? __ldg(xr + m) : __ldg(hr + (p.H + m));
    }
}

template <bool NOISE>
__global__ void __launch_bounds__(kThreads, 1) tt_conv_rw_kernel(const Params p) {
    extern __shared__ __align__(128) unsigned char smem[];
    // [full 2 x 8 B | empty 2 x 8 B | pad to 128][stage 0 window][stage 1 window]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + 2;
    const int32_t SB = p.sbytes;
    unsigned char* win0 = smem + 128;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&full[s], kThreads);
            mbar_init(&empty[s], kWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    int64_t w = blockIdx.x;
    if (w < p.total_tiles) {
        fill_window(p, w, win0, warp, lane);
        cp_async_arrive(&full[0]);
    }
    for (int it = 0; w < p.total_tiles; w += gridDim.x, ++it) {
        const int s = it & 1;
        const int64_t wn = w + gridDim.x;
        if (wn < p.total_tiles) {
            // the other stage last held tile it - 1: wait until every warp released it
            if (it > 0) mbar_wait(&empty[s ^ 1], ((it - 1) >> 1) & 1);
            fill_window(p, wn, win0 + (s ^ 1) * SB, warp, lane);
            cp_async_arrive(&full[s ^ 1]);
        }
        mbar_wait(&full[s], (it >> 1) & 1);
        compute_tile<NOISE>(p, w, win0 + s * SB, tid);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        const int32_t cl = static_cast<int32_t>(w / p.tiles_per_ch);
        const int32_t tl = static_cast<int32_t>(w - static_cast<int64_t>(cl) * p.tiles_per_ch);
        if (tl == p.tiles_per_ch - 1) write_history(p, cl, tid);
    }
}

}  // namespace rw
}  // namespace tt
