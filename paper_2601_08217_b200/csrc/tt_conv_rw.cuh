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

// R = 16 (8 warps; namespace tt::rw) and R = 8 (16 warps; namespace tt::rw8): the
// smaller window reuses less but keeps 4 warps per SMSP for latency hiding
#define TT_RW_NS rw
#define TT_RW_R 16
#include "tt_conv_rw_body.inc"
#undef TT_RW_NS
#undef TT_RW_R
#define TT_RW_NS rw8
#define TT_RW_R 8
#include "tt_conv_rw_body.inc"
#undef TT_RW_NS
#undef TT_RW_R
