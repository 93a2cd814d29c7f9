// tt_channel.cu — host side of the C ABI in include/tt_channel.h: handle ownership,
// validation, snapshot ring residency, the delay-line ping-pong, launch planning,
// and the pipelined host-buffer path. Every arithmetic step of the channel runs in
// the kernels of tt_conv.cuh; nothing here touches sample values.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <vector>

#include "tt_channel.h"
#include "tt_conv.cuh"
#include "tt_conv_dw.cuh"
#include "tt_conv_rw.cuh"
#include "tt_synth.cuh"

namespace {

thread_local char g_err[512] = "";

tt_status fail(tt_status s, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return s;
}

tt_status cuda_fail(cudaError_t e, const char* what) {
    cudaGetLastError();  // clear a sticky-free error so later calls are not poisoned
    if (e == cudaErrorMemoryAllocation) return fail(TT_ERR_OUT_OF_MEMORY, "%s: %s", what, cudaGetErrorString(e));
    return fail(TT_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define TT_CUDA(call, what)                         \
    do {                                            \
        cudaError_t e__ = (call);                   \
        if (e__ != cudaSuccess) return cuda_fail(e__, what); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess) ok = (prev == dev) || (cudaSetDevice(dev) == cudaSuccess);
    }
    ~DeviceGuard() {
        if (ok && prev >= 0) cudaSetDevice(prev);
    }
};

// Launch plan of one handle. kind: TT_KERNEL_GENERIC / TILED / RW. The tiled kernel has
// one plan per noise flag (they may differ in R if the variants' budgets ever differ).
struct TiledPlan {
    int R = 0;           // outputs per consumer thread (0: does not fit -> generic kernel)
    int CW = 16;         // consumer warps (tile T = CW x 32 x R)
    int ctas = 1;        // resident CTAs per SM (2 for shapes with <= 8 consumer warps and R <= 8)
    int stages = 2;      // shared-memory pipeline depth (2..4)
    size_t smem = 0;     // dynamic shared memory bytes
    int nk_max = 0;      // gain rows staged per tile
};
// dense-window kernel (tt_conv_dw.cuh; opt-in, TT_KERNEL=dw)
struct DwPlan {
    int CW = 0;            // consumer warps (0: not planned)
    int stages = 0;
    int nk_max = 0;        // gain rows staged per tile
    int win_rows = 0;      // window rows per stage
    int stage_bytes = 0;   // multiple of 1024
    int coef_off = 0, tab_off = 0;
    size_t smem = 0;       // dynamic shared memory (incl. alignment slack)
};
struct Plan {
    int kind = TT_KERNEL_GENERIC;
    DwPlan dw;
    TiledPlan tiled[2];  // [noise]
    // register-window kernel (opt-in: TT_KERNEL=rw)
    int rw_R = 0, rw_wbytes = 0, rw_rows = 0, rw_row_stride = 0, rw_sbytes = 0;
    size_t rw_smem = 0;
};

constexpr size_t kSmemBudget = 227 * 1024;  // one CTA per SM

// must match tt_conv_kernel's layout: 128 B of barriers + `stages` x [meta | win | coef | xo]
// (L = taps per gain row: top-n when sparse, whose offsets come one row per interval)
size_t smem_bytes(int R, int CW, int stages, int H, int L, int L4, int S, bool noise, bool xo_rows, int* nk_out) {
    const int T = CW * 32 * R;
    const int nk = (T - 1) / S + 2;  // worst-case intervals touched by a tile
    *nk_out = nk;
    const size_t st = 16 + (static_cast<size_t>(H) + T + 2) * 8 + static_cast<size_t>(nk) * L * 16 +
                      static_cast<size_t>(xo_rows ? nk : 1) * L4 * 4;
    (void)noise;  // the noise variant needs no extra shared memory (fused epilogue)
    return 128 + static_cast<size_t>(stages) * st;
}

// device scratch of tt_synth_jakes (one per device, reused across calls)
struct SynthScratch {
    unsigned char* buf = nullptr;
    size_t bytes = 0;
    cudaEvent_t done = nullptr;
};

}  // namespace

struct tt_channel_s {
    int dev = 0;
    int num_sms = 148;
    int C = 0, L = 0, L4 = 0, S = 0, H = 0, maxD = 0;
    uint64_t seed = 0;
    int64_t cap = 0, chan_off = 0;
    int64_t t = 0;
    int p = 0;  // history buffer holding the current delay line
    int64_t res_lo = 0, res_hi = 0;
    float4* ring = nullptr;    // [C][cap][L] (g_k, g_{k+1} - g_k), taps sorted by delay
    float2* hist = nullptr;    // [2][C][H] delay-line ping-pong
    float2* hist_zero = nullptr;  // [C][H] zeros: the delay line at t = 0 (reset needs no device work)
    int32_t* perm = nullptr;   // [C][L] original tap index of sorted tap j
    int32_t* xoff = nullptr;   // [C][L4] window offset H - d_j of sorted tap j
    int2* tab = nullptr;       // [C][L + 1] register-window table: (window byte offset, fresh samples)
    int32_t* dwtab = nullptr;  // [C][L4] dense-window tap table: f | dq class << 4 | q << 8 (d = 16 q + f)
    CUtensorMap dw_hist[3];    // history tensor maps: [0], [1] ping-pong halves, [2] the zero buffer
    std::vector<int32_t> sorted_d;  // [C][L] delays in sorted-tap order (host; rebuilds the rw table)
    int32_t* in_row = nullptr;  // [C] input row per channel (NEXT f4), nullptr = identity
    tt::DevClock* dclk = nullptr;  // device clock (stream position for graph-captured slot loops)
    bool dclock = false;           // tt_channel_set_device_clock: kernels run on dclk
    bool force_robust = false;  // TT_ROBUST=1: the robust tiled variant for every call (tests)
    bool pdl = true;            // launch the tiled kernel with programmatic dependent launch (TT_PDL=0: off)
    int32_t top_n = 0;          // NEXT f2: taps kept per interval (0 = dense)
    int32_t n4 = 0;             // sparse offsets row stride (>= top_n + 1, multiple of 4)
    float4* sring = nullptr;    // [C][cap][top_n] (+1) compacted rows of the selected taps
    int32_t* soff = nullptr;    // [C][cap][n4] window offsets of the selected taps
    int32_t in_rows = 0;        // rows of `in` when in_row is set
    float2* agg_scratch = nullptr;  // chunk sums / per-channel outputs for tt_channel_apply_aggregate
    size_t agg_scratch_elems = 0;
    float2* load_stage = nullptr;  // device staging for host-memory snapshot sources
    size_t load_stage_elems = 0;
    cudaEvent_t ev_load = nullptr;  // the last loader kernel that read load_stage
    size_t dev_bytes = 0;
    Plan plan;
    // host-buffer path
    static constexpr int kHostBufs = 4;  // (in + out) chunk buffers in flight
    float2* stage = nullptr;  // kHostBufs x (in + out) chunk buffers
    size_t stage_elems = 0;   // float2 per in (or out) chunk buffer
    cudaStream_t cs_h2d[2] = {}, cs_d2h[2] = {};  // two copy streams per direction
    cudaEvent_t ev_h2d[kHostBufs] = {}, ev_k[kHostBufs] = {}, ev_free[kHostBufs] = {}, ev_start = nullptr;
    cudaEvent_t ev_done[2] = {};
};

namespace {

// The attribute is per kernel function for the whole process, not per handle: it is
// set to the shape's full budget (never to one handle's size), so creating a handle
// with a smaller plan can never lower the cap of handles already alive.
template <int R, int CW, bool NOISE>
cudaError_t prepare_kernel(size_t budget) {
    const int sm = static_cast<int>(budget);
    for (cudaError_t e : {cudaFuncSetAttribute(tt::tt_conv_kernel<R, CW, NOISE, false, false>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
                          cudaFuncSetAttribute(tt::tt_conv_kernel<R, CW, NOISE, true, false>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
                          cudaFuncSetAttribute(tt::tt_conv_kernel<R, CW, NOISE, false, true>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
                          cudaFuncSetAttribute(tt::tt_conv_kernel<R, CW, NOISE, true, true>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, sm)})
        if (e != cudaSuccess) return e;
    if constexpr (R == 8 && CW == 16) {  // split-warp instances (S = 16R = 128), plain and robust
        for (cudaError_t e : {cudaFuncSetAttribute(tt::tt_conv_kernel<R, CW, NOISE, false, false, true>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
                              cudaFuncSetAttribute(tt::tt_conv_kernel<R, CW, NOISE, true, false, true>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
                              cudaFuncSetAttribute(tt::tt_conv_kernel<R, CW, NOISE, false, true, true>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
                              cudaFuncSetAttribute(tt::tt_conv_kernel<R, CW, NOISE, true, true, true>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, sm)})
            if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// tile shapes (R outputs per thread, CW consumer warps), in order of preference
struct Shape {
    int R, CW;
};
constexpr Shape kShapes[] = {{8, 16}, {16, 8}, {8, 8}, {4, 16}, {2, 16}};

template <bool NOISE>
cudaError_t prepare_tiled(tt_channel_s* h) {
    TiledPlan& tp = h->plan.tiled[NOISE ? 1 : 0];
    // deepest pipeline (<= 4 stages) that fits: streaming configs with short filters are
    // bound by HBM latency x bytes in flight, so they want more tiles in flight
    const char* fs = getenv("TT_STAGES");
    const int max_stages = fs ? std::max(2, std::min(tt::kMaxStages, atoi(fs))) : tt::kMaxStages;
    const bool sparse = h->top_n > 0;
    const int Lr = sparse ? h->top_n : h->L, L4r = sparse ? h->n4 : h->L4;
    // TT_TILE=RxCW (experiments) restricts the shape
    int fR = 0, fCW = 0;
    if (const char* ft = getenv("TT_TILE")) sscanf(ft, "%dx%d", &fR, &fCW);
    // the first shape that fits with >= 2 stages; (16, 8) only when forced (measured
    // slower at the BASELINE configs)
    for (const Shape& sh : kShapes) {
        if (fR ? (sh.R != fR || sh.CW != fCW) : (sh.CW != 16)) continue;
        int nk = 0;
        const int ctas = (sh.CW <= 8 && sh.R <= 8) ? 2 : 1;  // must match the kernel's launch bounds
        const size_t budget = ctas == 1 ? kSmemBudget : 112 * 1024;  // 2 CTAs share 228 KB
        if (smem_bytes(sh.R, sh.CW, 2, h->H, Lr, L4r, h->S, NOISE, sparse, &nk) > budget) continue;
        int stages = max_stages;
        while (stages > 2 && smem_bytes(sh.R, sh.CW, stages, h->H, Lr, L4r, h->S, NOISE, sparse, &nk) > budget)
            --stages;
        tp.ctas = ctas;
        tp.R = sh.R;
        tp.CW = sh.CW;
        tp.stages = stages;
        tp.smem = smem_bytes(sh.R, sh.CW, stages, h->H, Lr, L4r, h->S, NOISE, sparse, &nk);
        tp.nk_max = nk;
        break;
    }
    const size_t budget = tp.ctas == 1 ? kSmemBudget : 112 * 1024;
    switch (tp.R * 100 + tp.CW) {
        case 816: return prepare_kernel<8, 16, NOISE>(budget);
        case 1608: return prepare_kernel<16, 8, NOISE>(budget);
        case 808: return prepare_kernel<8, 8, NOISE>(budget);
        case 416: return prepare_kernel<4, 16, NOISE>(budget);
        case 216: return prepare_kernel<2, 16, NOISE>(budget);
        default: return cudaSuccess;  // generic kernel
    }
}

// RW-namespace of the register-window kernel with R outputs per thread
template <int R> struct RwNs;
template <> struct RwNs<16> {
    using Params = tt::rw::Params;
    static constexpr int T = tt::rw::T, kBlockBytes = tt::rw::kBlockBytes, kThreads = tt::rw::kThreads;
    template <bool NOISE> static constexpr auto kernel() { return tt::rw::tt_conv_rw_kernel<NOISE>; }
};
template <> struct RwNs<8> {
    using Params = tt::rw8::Params;
    static constexpr int T = tt::rw8::T, kBlockBytes = tt::rw8::kBlockBytes, kThreads = tt::rw8::kThreads;
    template <bool NOISE> static constexpr auto kernel() { return tt::rw8::tt_conv_rw_kernel<NOISE>; }
};

// plan + tap table of the register-window kernel: per sorted tap, the byte offset of
// its window in a thread's doubled block ((o / R) blocks + (o % R) slots, o = Hp - d)
// and the number of fresh samples min(d_j - d_{j-1}, R) (R for the first tap)
template <int R>
cudaError_t prepare_rw(tt_channel_s* h) {
    using NS = RwNs<R>;
    const int Hp = h->H - 16;
    const int nb = (Hp + NS::T) / R;
    const size_t wbytes = (static_cast<size_t>(nb) * NS::kBlockBytes + 15) & ~size_t(15);
    const size_t rows = (NS::T - 1) / h->S + 2;
    const size_t row_stride = static_cast<size_t>(h->L) * 16 + 16;
    const size_t tbytes = (static_cast<size_t>(h->L + 1) * 8 + 15) & ~size_t(15);
    const size_t sbytes = wbytes + rows * row_stride + tbytes;
    const size_t sm = 128 + 2 * sbytes;
    if (sm > kSmemBudget) return cudaSuccess;  // does not fit: tiled kernel
    std::vector<int2> tb(static_cast<size_t>(h->C) * (h->L + 1), int2{0, 0});
    for (int c = 0; c < h->C; ++c) {
        const int32_t* dc = h->sorted_d.data() + static_cast<size_t>(c) * h->L;
        for (int j = 0; j < h->L; ++j) {
            const int o = Hp - dc[j];
            const int gap = j == 0 ? R : std::min(R, dc[j] - dc[j - 1]);
            tb[static_cast<size_t>(c) * (h->L + 1) + j] = int2{(o / R) * NS::kBlockBytes + (o % R) * 8, gap};
        }
    }
    cudaError_t e;
    if ((e = cudaMemcpy(h->tab, tb.data(), tb.size() * sizeof(int2), cudaMemcpyHostToDevice)) != cudaSuccess) return e;
    // process-wide attribute: the full budget, not this handle's size (see prepare_kernel)
    if ((e = cudaFuncSetAttribute(NS::template kernel<false>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSmemBudget))) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(NS::template kernel<true>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSmemBudget))) != cudaSuccess)
        return e;
    h->plan.rw_R = R;
    h->plan.rw_wbytes = static_cast<int>(wbytes);
    h->plan.rw_rows = static_cast<int>(rows);
    h->plan.rw_row_stride = static_cast<int>(row_stride);
    h->plan.rw_sbytes = static_cast<int>(sbytes);
    h->plan.rw_smem = sm;
    return cudaSuccess;
}

// launch the register-window kernel with R outputs per thread
template <int R>
void launch_rw(tt_channel_s* h, const tt::ConvParams& p, const float2* x, float2* y, int32_t c_lo, int nch, int64_t n,
               bool noise, cudaStream_t st) {
    using NS = RwNs<R>;
    typename NS::Params q{};
    q.x = x;
    q.y = y;
    q.hist_rd = p.hist_rd;
    q.hist_wr = p.hist_wr;
    q.ring = h->ring;
    q.tab = h->tab;
    q.n = n;
    q.t = h->t;
    q.cap = h->cap;
    q.chan_offset = h->chan_off;
    q.c_lo = c_lo;
    q.L = h->L;
    q.H = h->H;
    q.Hp = h->H - 16;
    q.S = h->S;
    q.a = static_cast<int32_t>(h->t & (R - 1));
    q.nb = (q.Hp + NS::T) / R;
    q.s_shift = p.s_shift;
    q.inv_S = p.inv_S;
    q.key0 = p.key0;
    q.key1 = p.key1;
    q.noise_sc = p.noise_sc;
    q.vec_store = ((n & 1) == 0 && (q.a & 1) == 0) ? 1 : 0;
    q.rows = h->plan.rw_rows;
    q.row_stride = h->plan.rw_row_stride;
    q.wbytes = h->plan.rw_wbytes;
    q.sbytes = h->plan.rw_sbytes;
    q.tiles_per_ch = static_cast<int32_t>((n + q.a + NS::T - 1) / NS::T);
    q.total_tiles = static_cast<int64_t>(nch) * q.tiles_per_ch;
    const int64_t grid = std::min<int64_t>(q.total_tiles, static_cast<int64_t>(h->num_sms));
    if (noise)
        NS::template kernel<true>()<<<static_cast<unsigned>(grid), NS::kThreads, h->plan.rw_smem, st>>>(q);
    else
        NS::template kernel<false>()<<<static_cast<unsigned>(grid), NS::kThreads, h->plan.rw_smem, st>>>(q);
}

// ---- 2-D/3-D TMA tensor maps (dense-window kernel) ---------------------------------
// cuTensorMapEncodeTiled comes from the driver through the runtime's entry-point query,
// so libtt.so has no link-time dependency on libcuda (it loads on hosts without a GPU).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(f);
        else
            cudaGetLastError();
    });
    return fn;
}

// A [planes][rows][16 complex samples] view of float2 rows (one row = 128 B), boxes of
// box_rows rows of one plane, 128-B swizzle in shared memory, zero fill out of bounds.
bool encode_rows(CUtensorMap* m, const void* base, uint64_t rows, uint64_t planes, uint32_t box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || rows == 0 || planes == 0) return false;
    const cuuint64_t dims[3] = {32, rows, planes};
    const cuuint64_t strides[2] = {128, rows * 128};
    const cuuint32_t box[3] = {32, box_rows, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int CW, bool NOISE>
cudaError_t prepare_dw_kernel() {
    return cudaFuncSetAttribute(tt::dw::tt_conv_dw_kernel<CW, NOISE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmemBudget));  // process-wide: the full budget
}

// Dense-window plan (tt_conv_dw.cuh; opt-in with TT_KERNEL=dw). A thread reads about
// (D + 32) / (16 L) x samples per output-tap from shared memory instead of 1.
cudaError_t prepare_dw(tt_channel_s* h) {
    DwPlan& dp = h->plan.dw;
    dp = DwPlan{};
    if (h->top_n > 0 || h->S % 16 != 0 || h->H % 16 != 0) return cudaSuccess;
    if (!encode_fn()) return cudaSuccess;
    const int Hw = (h->H + 127) & ~127;
    // consumer warps: 7 (+ the producer = 8 warps, 2 per SMSP: up to 255 registers per
    // thread, no spills; 8 + 1 warps cap the kernel at 168 and spill); TT_DW_WARPS=8|4 for
    // experiments; 4 when the stage does not fit
    int first_cw = 7;
    if (const char* fw = getenv("TT_DW_WARPS"))
        if (*fw) first_cw = atoi(fw);
    for (int CW : {first_cw, 4}) {
        if (CW != 8 && CW != 7 && CW != 4) continue;
        const int T = CW * 32 * tt::dw::R;
        if (Hw > T) continue;
        const int nk = (T - 1) / h->S + 2;
        const int win_rows = (((Hw + T) / 16) + tt::dw::kXBoxRows - 1) / tt::dw::kXBoxRows * tt::dw::kXBoxRows;
        const size_t win_b = static_cast<size_t>(win_rows) * tt::dw::kRowBytes;
        const size_t coef_b = (static_cast<size_t>(nk) * h->L * 16 + 16 + 15) & ~size_t(15);
        const size_t tab_b = static_cast<size_t>(h->L4) * 4;
        const size_t stage = (win_b + coef_b + tab_b + 1023) & ~size_t(1023);
        const size_t fixed = 1024 + 1024 + static_cast<size_t>(CW) * 32 * tt::dw::kRowBytes;
        int stages = tt::dw::kMaxStages;
        while (stages >= 2 && fixed + stages * stage > kSmemBudget) --stages;
        if (stages < 2) continue;
        if (stage > (size_t(1) << 30)) continue;
        dp.CW = CW;
        dp.stages = stages;
        dp.nk_max = nk;
        dp.win_rows = win_rows;
        dp.stage_bytes = static_cast<int>(stage);
        dp.coef_off = static_cast<int>(win_b);
        dp.tab_off = static_cast<int>(win_b + coef_b);
        dp.smem = fixed + stages * stage;
        break;
    }
    if (!dp.CW) return cudaSuccess;
    const size_t hs = static_cast<size_t>(h->C) * h->H;
    if (!encode_rows(&h->dw_hist[0], h->hist, h->H / 16, h->C, tt::dw::kHBoxRows) ||
        !encode_rows(&h->dw_hist[1], h->hist + hs, h->H / 16, h->C, tt::dw::kHBoxRows) ||
        !encode_rows(&h->dw_hist[2], h->hist_zero, h->H / 16, h->C, tt::dw::kHBoxRows)) {
        dp = DwPlan{};
        return cudaSuccess;
    }
    cudaError_t e;
    if (dp.CW == 8) {
        if ((e = prepare_dw_kernel<8, false>()) != cudaSuccess || (e = prepare_dw_kernel<8, true>()) != cudaSuccess)
            return e;
    } else if (dp.CW == 7) {
        if ((e = prepare_dw_kernel<7, false>()) != cudaSuccess || (e = prepare_dw_kernel<7, true>()) != cudaSuccess)
            return e;
    } else {
        if ((e = prepare_dw_kernel<4, false>()) != cudaSuccess || (e = prepare_dw_kernel<4, true>()) != cudaSuccess)
            return e;
    }
    return cudaSuccess;
}

cudaError_t prepare_plan(tt_channel_s* h) {
    h->plan = Plan{};
    // TT_KERNEL=rw|tiled|generic selects the kernel (all are bit-identical; default tiled)
    const char* force = getenv("TT_KERNEL");
    const bool want_rw = force && !strcmp(force, "rw");
    const bool want_generic = force && !strcmp(force, "generic");
    if (want_generic) return cudaSuccess;
    // dense-window kernel: opt-in (TT_KERNEL=dw), wherever it fits. It reads ~3x fewer
    // x operands from shared memory than the tiled kernel on dense delays, but measured
    // slower on every BASELINE shape (per-tap dispatch)
    const bool want_dw = force && !strcmp(force, "dw");
    if (want_dw) {
        cudaError_t e = prepare_dw(h);
        if (e != cudaSuccess) return e;
    }
    // register-window kernel (R = 16 or 8 consecutive outputs per thread): needs
    // R-aligned snapshot intervals and two window stages of (Hp + T) / R doubled blocks
    const bool want_rw8 = force && !strcmp(force, "rw8");
    if ((want_rw || want_rw8) && h->S % 16 == 0) {
        cudaError_t e = want_rw8 ? prepare_rw<tt::rw8::R>(h) : prepare_rw<tt::rw::R>(h);
        if (e != cudaSuccess) return e;
    }
    // tiled plans (also behind the rw kernel: aggregation and input maps use them)
    cudaError_t e;
    if ((e = prepare_tiled<false>(h)) != cudaSuccess) return e;
    if ((e = prepare_tiled<true>(h)) != cudaSuccess) return e;
    if (h->plan.rw_smem) h->plan.kind = TT_KERNEL_RW;
    else if (h->plan.dw.CW && h->plan.tiled[0].R != 0 && h->plan.tiled[1].R != 0) h->plan.kind = TT_KERNEL_DW;
    else if (h->plan.tiled[0].R != 0 || h->plan.tiled[1].R != 0) h->plan.kind = TT_KERNEL_TILED;
    return cudaSuccess;
}

// Enqueue the convolution of channels [c_lo, c_hi) for this call (no state change).
// Group-sum request of one launch (tt_channel_apply_aggregate): per-channel outputs go
// to y (may be nullptr), group sums of G channels to agg, via `scratch` when needed.
struct AggReq {
    float2* agg = nullptr;
    int32_t G = 1;
    float2* scratch = nullptr;
};

tt_status launch(tt_channel_s* h, const float2* x, float2* y, int32_t c_lo, int32_t c_hi, int64_t n, float sigma,
                 cudaStream_t st, const AggReq& ar = AggReq{}) {
    tt::ConvParams p{};
    p.x = x;
    p.y = y;
    p.in_row = h->in_row;
    p.group = 1;
    p.chunk = 1;
    p.nchunks = 1;
    const int32_t ngroups = ar.agg ? (c_hi - c_lo) / ar.G : 0;
    const int32_t KC = ar.agg ? std::min<int32_t>(ar.G, TT_AGG_CHUNK) : 1;
    const int32_t nchunks = ar.agg ? (ar.G + KC - 1) / KC : 1;
    const size_t hs = static_cast<size_t>(h->C) * h->H;
    // at t = 0 the delay line is zero by definition: read the zero buffer, so a
    // reset needs no device work
    p.hist_rd = h->t == 0 ? h->hist_zero : h->hist + h->p * hs;
    p.hist_wr = h->hist + (1 - h->p) * hs;
    p.hist_base = h->hist;
    p.hist_zero = h->hist_zero;
    p.hist_half = static_cast<int64_t>(hs);
    const bool sparse = h->top_n > 0;
    p.ring = sparse ? h->sring : h->ring;
    p.xoff = h->xoff;
    p.xoff_rows = sparse ? h->soff : nullptr;
    p.n = n;
    p.t = h->t;
    p.cap = h->cap;
    p.chan_offset = h->chan_off;
    p.c_lo = c_lo;
    p.L = sparse ? h->top_n : h->L;
    p.L4 = sparse ? h->n4 : h->L4;
    p.H = h->H;
    p.S = h->S;
    p.key0 = static_cast<uint32_t>(h->seed);
    p.key1 = static_cast<uint32_t>(h->seed >> 32);
    // docs/tt-normal-v1.md §3: sigma / sqrt(2) rounded once in double, then to float
    p.noise_sc = static_cast<float>(static_cast<double>(sigma) * 0x1.6a09e667f3bcdp-1);
    p.s_shift = -1;
    if ((h->S & (h->S - 1)) == 0) {
        p.s_shift = 0;
        while ((1 << p.s_shift) < h->S) ++p.s_shift;
    }
    p.inv_S = static_cast<float>(1.0 / h->S);
    p.t_div = h->t / h->S;
    p.t_mod = static_cast<int32_t>(h->t % h->S);
    const bool noise = sigma > 0.0f;
    const int nch = c_hi - c_lo;
    // dense-window kernel: plain calls whose start and length are multiples of 16 (each
    // thread's 16 outputs then sit in one snapshot interval, and x / y rows are whole
    // 16-sample TMA rows) on 16-B aligned buffers
    const bool dw_call = h->plan.kind == TT_KERNEL_DW && !ar.agg && !h->in_row && !sparse && !h->dclock &&
                         !h->force_robust && h->t % 16 == 0 && n % 16 == 0 &&
                         (reinterpret_cast<uintptr_t>(x) & 15u) == 0 && (reinterpret_cast<uintptr_t>(y) & 15u) == 0 &&
                         y != nullptr;
    if (dw_call) {
        const DwPlan& dp = h->plan.dw;
        const int T = dp.CW * 32 * tt::dw::R;
        tt::dw::Params q{};
        q.ring = h->ring;
        q.tab = h->dwtab;
        q.hist_wr = p.hist_wr;
        q.n = n;
        q.t = h->t;
        q.cap = h->cap;
        q.chan_offset = h->chan_off;
        q.t_div = p.t_div;
        q.t_mod = p.t_mod;
        q.c_lo = c_lo;
        q.tiles_per_ch = static_cast<int32_t>((n + T - 1) / T);
        q.total_tiles = static_cast<int64_t>(nch) * q.tiles_per_ch;
        q.L = h->L;
        q.L4 = h->L4;
        q.H = h->H;
        q.Hw = (h->H + 127) & ~127;
        q.S = h->S;
        q.s_shift = p.s_shift;
        q.inv_S = p.inv_S;
        q.nk_max = dp.nk_max;
        q.stages = dp.stages;
        q.win_rows = dp.win_rows;
        q.hist_row0 = (h->H - q.Hw) / 16;
        q.stage_bytes = dp.stage_bytes;
        q.coef_off = dp.coef_off;
        q.tab_off = dp.tab_off;
        q.key0 = p.key0;
        q.key1 = p.key1;
        q.noise_sc = p.noise_sc;
        if (q.total_tiles >= (int64_t(1) << 31)) return fail(TT_ERR_INVALID_ARG, "call too large");
        CUtensorMap tmx, tmy;
        if (!encode_rows(&tmx, x, static_cast<uint64_t>(n / 16), static_cast<uint64_t>(nch), tt::dw::kXBoxRows) ||
            !encode_rows(&tmy, y, static_cast<uint64_t>(n / 16), static_cast<uint64_t>(nch), tt::dw::kXBoxRows))
            return fail(TT_ERR_CUDA, "cuTensorMapEncodeTiled failed for the input / output buffers");
        const CUtensorMap& tmh = h->t == 0 ? h->dw_hist[2] : h->dw_hist[h->p];
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
        cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>(q.total_tiles, h->num_sms)));
        cfg.blockDim = dim3((dp.CW + 1) * 32);
        cfg.dynamicSmemBytes = dp.smem;
        cfg.stream = st;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (dp.CW == 8) {
            if (noise) cudaLaunchKernelEx(&cfg, tt::dw::tt_conv_dw_kernel<8, true>, tmx, tmy, tmh, q);
            else cudaLaunchKernelEx(&cfg, tt::dw::tt_conv_dw_kernel<8, false>, tmx, tmy, tmh, q);
        } else if (dp.CW == 7) {
            if (noise) cudaLaunchKernelEx(&cfg, tt::dw::tt_conv_dw_kernel<7, true>, tmx, tmy, tmh, q);
            else cudaLaunchKernelEx(&cfg, tt::dw::tt_conv_dw_kernel<7, false>, tmx, tmy, tmh, q);
        } else {
            if (noise) cudaLaunchKernelEx(&cfg, tt::dw::tt_conv_dw_kernel<4, true>, tmx, tmy, tmh, q);
            else cudaLaunchKernelEx(&cfg, tt::dw::tt_conv_dw_kernel<4, false>, tmx, tmy, tmh, q);
        }
    } else if (h->plan.kind == TT_KERNEL_RW && !ar.agg && !h->in_row && !sparse) {
        if (h->plan.rw_R == 8) launch_rw<8>(h, p, x, y, c_lo, nch, n, noise, st);
        else launch_rw<16>(h, p, x, y, c_lo, nch, n, noise, st);
    } else if (h->plan.tiled[noise ? 1 : 0].R != 0 &&
               (h->plan.kind == TT_KERNEL_TILED || h->plan.kind == TT_KERNEL_DW || ar.agg || h->in_row || sparse)) {
        const TiledPlan& tp = h->plan.tiled[noise ? 1 : 0];
        const int T = tp.CW * 32 * tp.R;
        // a short lead-in tile when the call does not start on a 32R-aligned global
        // sample (call lengths not a multiple of it), so the other tiles' warps keep the
        // one-interval fast path and the paired noise draw
        const int64_t A = 32 * tp.R;
        p.lead = h->dclock ? 0 : static_cast<int32_t>((A - h->t % A) % A);  // device clock: aligned by contract
        if (p.lead >= n) p.lead = 0;
        p.tiles_per_ch = static_cast<int32_t>(p.lead ? 1 + (n - p.lead + T - 1) / T : (n + T - 1) / T);
        // the robust kernel variant (lead-in tile, window shift for input rows 8 B off a
        // 16-B boundary) only when the call needs it; aligned calls run the plain schedule
        const bool robust = h->dclock || h->force_robust || p.lead != 0 ||
                            (reinterpret_cast<uintptr_t>(x) & 15u) != 0 || (n & 1) != 0;
        if (h->dclock) p.clk = h->dclk;
        p.total_tiles = static_cast<int64_t>(nch) * p.tiles_per_ch;
        if (ar.agg) {
            // fused chunk sums: straight into agg when a group is one chunk, else into
            // scratch partials [groups][nchunks][n] reduced below in chunk order
            p.group = ar.G;
            p.chunk = KC;
            p.nchunks = nchunks;
            p.agg = nchunks > 1 ? ar.scratch : ar.agg;
            p.total_super = static_cast<int64_t>(ngroups) * nchunks * p.tiles_per_ch;
        } else {
            p.total_super = p.total_tiles;
        }
        p.nk_max = tp.nk_max;
        p.stages = tp.stages;
        if (p.total_super >= (int64_t(1) << 31) || p.total_tiles >= (int64_t(1) << 31))
            return fail(TT_ERR_INVALID_ARG, "call too large: %lld work items", (long long)p.total_super);
        const int64_t grid = std::min<int64_t>(p.total_super, static_cast<int64_t>(h->num_sms) * tp.ctas);
        const dim3 g(static_cast<unsigned>(grid)), b((tp.CW + 1) * 32);
        const size_t sm = tp.smem;
        // the general variant only when a group sum or sparse offsets are in play
        const bool gen = ar.agg || sparse;
        // programmatic dependent launch (PDL): back-to-back slot calls overlap the next
        // grid's launch and CTA set-up with this one's tail (the kernel waits on
        // griddepcontrol.wait before touching global memory)
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
        cfg.gridDim = g;
        cfg.blockDim = b;
        cfg.dynamicSmemBytes = sm;
        cfg.stream = st;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
#define TT_LAUNCH_R(RR, CC, RB)                                                                 \
    do {                                                                                        \
        if (noise) {                                                                            \
            if (gen) cudaLaunchKernelEx(&cfg, tt::tt_conv_kernel<RR, CC, true, true, RB>, p);   \
            else cudaLaunchKernelEx(&cfg, tt::tt_conv_kernel<RR, CC, true, false, RB>, p);      \
        } else {                                                                                \
            if (gen) cudaLaunchKernelEx(&cfg, tt::tt_conv_kernel<RR, CC, false, true, RB>, p);  \
            else cudaLaunchKernelEx(&cfg, tt::tt_conv_kernel<RR, CC, false, false, RB>, p);     \
        }                                                                                       \
    } while (0)
#define TT_LAUNCH(RR, CC)                         \
    do {                                          \
        if (robust) TT_LAUNCH_R(RR, CC, true);    \
        else TT_LAUNCH_R(RR, CC, false);          \
    } while (0)
        // split-warp instances (tt_conv.cuh consume_body): S = 16R; in the robust variant
        // the tiles after the lead-in start on the 32R grid, so their warps split too
        const bool split = tp.R == 8 && tp.CW == 16 && h->S == 16 * tp.R;
#define TT_LAUNCH_SPLIT(RB)                                                                          \
    do {                                                                                             \
        if (noise) {                                                                                 \
            if (gen) cudaLaunchKernelEx(&cfg, tt::tt_conv_kernel<8, 16, true, true, RB, true>, p);   \
            else cudaLaunchKernelEx(&cfg, tt::tt_conv_kernel<8, 16, true, false, RB, true>, p);      \
        } else {                                                                                     \
            if (gen) cudaLaunchKernelEx(&cfg, tt::tt_conv_kernel<8, 16, false, true, RB, true>, p);  \
            else cudaLaunchKernelEx(&cfg, tt::tt_conv_kernel<8, 16, false, false, RB, true>, p);     \
        }                                                                                            \
    } while (0)
        switch (tp.R * 100 + tp.CW) {
            case 816:
                if (split && robust) TT_LAUNCH_SPLIT(true);
                else if (split) TT_LAUNCH_SPLIT(false);
                else TT_LAUNCH(8, 16);
                break;
            case 1608: TT_LAUNCH(16, 8); break;
            case 808: TT_LAUNCH(8, 8); break;
            case 416: TT_LAUNCH(4, 16); break;
            default: TT_LAUNCH(2, 16); break;
        }
#undef TT_LAUNCH
#undef TT_LAUNCH_R
#undef TT_LAUNCH_SPLIT
        if (ar.agg && nchunks > 1) {
            const int64_t tot = static_cast<int64_t>(ngroups) * n;
            const int64_t gg = std::min<int64_t>((tot + 255) / 256, int64_t(h->num_sms) * 8);
            tt::tt_group_sum_kernel<<<static_cast<unsigned>(gg), 256, 0, st>>>(ar.scratch, ar.agg, n, ngroups, ar.G, KC,
                                                                                nchunks, 1);
        }
    } else {
        if (ar.agg && !y) p.y = y = ar.scratch;  // per-channel outputs are needed for the sums
        p.tiles_per_ch = 1;
        p.total_tiles = nch;
        const int64_t N = static_cast<int64_t>(nch) * n;
        const int64_t grid = std::min<int64_t>((N + 255) / 256, int64_t(h->num_sms) * 8);
        if (noise)
            tt::tt_conv_generic_kernel<true><<<static_cast<unsigned>(grid), 256, 0, st>>>(p);
        else
            tt::tt_conv_generic_kernel<false><<<static_cast<unsigned>(grid), 256, 0, st>>>(p);
        if (h->H > 0) {
            const int64_t tot = static_cast<int64_t>(nch) * h->H;
            const int64_t hg = std::min<int64_t>((tot + 255) / 256, int64_t(h->num_sms) * 8);
            tt::tt_history_kernel<<<static_cast<unsigned>(hg), 256, 0, st>>>(p, nch);
        }
        if (ar.agg) {
            const int64_t tot = static_cast<int64_t>(ngroups) * n;
            const int64_t gg = std::min<int64_t>((tot + 255) / 256, int64_t(h->num_sms) * 8);
            tt::tt_group_sum_kernel<<<static_cast<unsigned>(gg), 256, 0, st>>>(y, ar.agg, n, ngroups, ar.G, KC,
                                                                                nchunks, 0);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    return TT_OK;
}

// alignment the device-clock mode keeps every call start on (32R of the tiled plans)
int64_t clock_grid(const tt_channel_s* h) {
    return 32 * std::max(h->plan.tiled[0].R, h->plan.tiled[1].R);
}

tt_status check_apply(tt_channel_s* h, const void* in, const void* out, int64_t n, float sigma) {
    if (!h) return fail(TT_ERR_INVALID_ARG, "NULL handle");
    if (!in || !out) return fail(TT_ERR_INVALID_ARG, "NULL in/out");
    if (n <= 0) return fail(TT_ERR_INVALID_ARG, "n_samples must be > 0 (got %lld)", (long long)n);
    if (n > (int64_t(1) << 30)) return fail(TT_ERR_INVALID_ARG, "n_samples must be <= 2^30 per call (got %lld)", (long long)n);
    if (in == out) return fail(TT_ERR_INVALID_ARG, "in and out must not overlap");
    if (!(sigma >= 0.0f) || !std::isfinite(sigma)) return fail(TT_ERR_INVALID_ARG, "noise_sigma must be finite and >= 0");
    if (h->dclock) {
        // the stream position lives on the device: calls must keep it on the 32R grid,
        // and snapshot residency is the caller's contract (not checked per call)
        const int64_t A = clock_grid(h);
        if (n % A != 0)
            return fail(TT_ERR_UNSUPPORTED, "device-clock mode needs n_samples %% %lld == 0 (got %lld)", (long long)A,
                        (long long)n);
        return TT_OK;
    }
    const int64_t k_lo = h->t / h->S;
    const int64_t k_hi = (h->t + n - 1) / h->S + 1;
    if (h->res_hi <= h->res_lo || k_lo < h->res_lo || k_hi >= h->res_hi)
        return fail(TT_ERR_SNAPSHOT_MISSING, "apply needs snapshots [%lld, %lld] but [%lld, %lld) are resident",
                    (long long)k_lo, (long long)k_hi, (long long)h->res_lo, (long long)h->res_hi);
    return TT_OK;
}

void free_all(tt_channel_s* h) {
    cudaFree(h->ring);
    cudaFree(h->hist);
    cudaFree(h->hist_zero);
    cudaFree(h->perm);
    cudaFree(h->xoff);
    cudaFree(h->tab);
    cudaFree(h->dwtab);
    cudaFree(h->dclk);
    cudaFree(h->in_row);
    cudaFree(h->sring);
    cudaFree(h->soff);
    cudaFree(h->agg_scratch);
    cudaFree(h->load_stage);
    cudaFree(h->stage);
    for (int i = 0; i < tt_channel_s::kHostBufs; ++i) {
        if (h->ev_h2d[i]) cudaEventDestroy(h->ev_h2d[i]);
        if (h->ev_k[i]) cudaEventDestroy(h->ev_k[i]);
        if (h->ev_free[i]) cudaEventDestroy(h->ev_free[i]);
    }
    if (h->ev_start) cudaEventDestroy(h->ev_start);
    if (h->ev_load) cudaEventDestroy(h->ev_load);
    for (int i = 0; i < 2; ++i) {
        if (h->ev_done[i]) cudaEventDestroy(h->ev_done[i]);
        if (h->cs_h2d[i]) cudaStreamDestroy(h->cs_h2d[i]);
        if (h->cs_d2h[i]) cudaStreamDestroy(h->cs_d2h[i]);
    }
}

}  // namespace

extern "C" {

int32_t tt_abi_version(void) { return TT_ABI_VERSION; }

const char* tt_last_error(void) { return g_err; }

const char* tt_status_string(tt_status s) {
    switch (s) {
        case TT_OK: return "TT_OK";
        case TT_ERR_INVALID_ARG: return "TT_ERR_INVALID_ARG";
        case TT_ERR_OUT_OF_MEMORY: return "TT_ERR_OUT_OF_MEMORY";
        case TT_ERR_CUDA: return "TT_ERR_CUDA";
        case TT_ERR_SNAPSHOT_MISSING: return "TT_ERR_SNAPSHOT_MISSING";
        case TT_ERR_UNSUPPORTED: return "TT_ERR_UNSUPPORTED";
    }
    return "TT_ERR_UNKNOWN";
}

tt_status tt_channel_create(tt_channel_t* out, int32_t num_ue, int32_t num_taps, const int32_t* delays,
                            int32_t snapshot_period, uint64_t seed, int64_t snapshot_capacity,
                            int64_t channel_offset) {
    if (!out) return fail(TT_ERR_INVALID_ARG, "NULL out");
    *out = nullptr;
    if (num_ue <= 0) return fail(TT_ERR_INVALID_ARG, "num_ue must be > 0");
    if (num_taps <= 0 || num_taps > TT_MAX_TAPS) return fail(TT_ERR_INVALID_ARG, "num_taps must be in [1, %d]", TT_MAX_TAPS);
    if (!delays) return fail(TT_ERR_INVALID_ARG, "NULL delays");
    if (snapshot_period <= 0) return fail(TT_ERR_INVALID_ARG, "snapshot_period must be > 0");
    if (snapshot_capacity < 2) return fail(TT_ERR_INVALID_ARG, "snapshot_capacity must be >= 2");
    if (channel_offset < 0) return fail(TT_ERR_INVALID_ARG, "channel_offset must be >= 0");
    const int64_t CL = static_cast<int64_t>(num_ue) * num_taps;
    int maxD = 0;
    for (int64_t i = 0; i < CL; ++i) {
        if (delays[i] < 0 || delays[i] > TT_MAX_DELAY)
            return fail(TT_ERR_INVALID_ARG, "delay[%lld] = %d outside [0, %d]", (long long)i, delays[i], TT_MAX_DELAY);
        maxD = std::max(maxD, static_cast<int>(delays[i]));
    }
    int dev = 0;
    TT_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    cudaDeviceProp prop;
    TT_CUDA(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
    if (prop.major != 10) return fail(TT_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a", dev, prop.major, prop.minor);

    tt_channel_s* h = new (std::nothrow) tt_channel_s();
    if (!h) return fail(TT_ERR_OUT_OF_MEMORY, "host allocation");
    h->dev = dev;
    h->num_sms = prop.multiProcessorCount;
    h->C = num_ue;
    h->L = num_taps;
    h->L4 = (num_taps + 1 + 3) & ~3;  // >= L + 1: room for the kernel's next-group prefetch
    h->S = snapshot_period;
    h->maxD = maxD;
    h->H = ((maxD + 15) & ~15) + 16;  // >= D + 16: a 16-aligned window start reaches back <= 15 more
    h->seed = seed;
    h->cap = snapshot_capacity;
    h->chan_off = channel_offset;
    if (const char* fp = getenv("TT_PDL")) h->pdl = atoi(fp) != 0;
    if (const char* fr = getenv("TT_ROBUST")) h->force_robust = atoi(fr) != 0;

    // per channel: taps sorted by delay (stable: ties keep tap index order); perm[c][j]
    // is the original index of sorted tap j, xoff[c][j] its window offset H - d
    std::vector<int32_t> pm(static_cast<size_t>(CL)), xo(static_cast<size_t>(num_ue) * h->L4, 0);
    // (the register-window table is built by its plan, prepare_rw)
    const size_t tb_elems = static_cast<size_t>(num_ue) * (num_taps + 1);
    h->sorted_d.assign(static_cast<size_t>(CL), 0);
    for (int c = 0; c < num_ue; ++c) {
        int32_t* pc = pm.data() + static_cast<size_t>(c) * num_taps;
        std::iota(pc, pc + num_taps, 0);
        const int32_t* dc = delays + static_cast<int64_t>(c) * num_taps;
        std::stable_sort(pc, pc + num_taps, [dc](int32_t a, int32_t b) { return dc[a] < dc[b]; });
        for (int j = 0; j < num_taps; ++j) xo[static_cast<size_t>(c) * h->L4 + j] = h->H - dc[pc[j]];
        for (int j = 0; j < num_taps; ++j) h->sorted_d[static_cast<size_t>(c) * num_taps + j] = dc[pc[j]];
    }
    auto bail = [&](tt_status s) {
        free_all(h);
        delete h;
        return s;
    };
    cudaError_t e;
    // + one float4: the kernels prefetch one tap ahead
    const size_t ring_b = (static_cast<size_t>(num_ue) * snapshot_capacity * num_taps + 1) * sizeof(float4);
    const size_t tb_b = tb_elems * sizeof(int2);
    const size_t hist_b = 2 * static_cast<size_t>(num_ue) * h->H * sizeof(float2);
    const size_t pm_b = pm.size() * sizeof(int32_t), xo_b = xo.size() * sizeof(int32_t);
    if ((e = cudaMalloc(&h->ring, ring_b)) != cudaSuccess) return bail(cuda_fail(e, "cudaMalloc(snapshot ring)"));
    if (hist_b && (e = cudaMalloc(&h->hist, hist_b)) != cudaSuccess) return bail(cuda_fail(e, "cudaMalloc(history)"));
    if (hist_b && (e = cudaMalloc(&h->hist_zero, hist_b / 2)) != cudaSuccess)
        return bail(cuda_fail(e, "cudaMalloc(zero history)"));
    if ((e = cudaMalloc(&h->perm, pm_b)) != cudaSuccess) return bail(cuda_fail(e, "cudaMalloc(perm)"));
    if ((e = cudaMalloc(&h->xoff, xo_b)) != cudaSuccess) return bail(cuda_fail(e, "cudaMalloc(xoff)"));
    if ((e = cudaMalloc(&h->tab, tb_b)) != cudaSuccess) return bail(cuda_fail(e, "cudaMalloc(tab)"));
    {
        // dense-window tap table: per sorted tap, d = 16 q + f and the block step from the
        // previous tap (0, 1, or 2 = jump / first tap: read both blocks)
        std::vector<int32_t> dt(static_cast<size_t>(num_ue) * h->L4, -1);  // pads: -1 ends a block scan
        for (int c = 0; c < num_ue; ++c) {
            const int32_t* dc = h->sorted_d.data() + static_cast<size_t>(c) * num_taps;
            for (int j = 0; j < num_taps; ++j) {
                const int32_t q = dc[j] >> 4, f = dc[j] & 15;
                const int32_t dq = j == 0 ? 2 : std::min(2, q - (dc[j - 1] >> 4));
                dt[static_cast<size_t>(c) * h->L4 + j] = f | (dq << 4) | (q << 8);
            }
        }
        const size_t dt_b = dt.size() * sizeof(int32_t);
        if ((e = cudaMalloc(&h->dwtab, dt_b)) != cudaSuccess) return bail(cuda_fail(e, "cudaMalloc(dw table)"));
        if ((e = cudaMemcpy(h->dwtab, dt.data(), dt_b, cudaMemcpyHostToDevice)) != cudaSuccess)
            return bail(cuda_fail(e, "copy dw table"));
        h->dev_bytes += dt_b;
    }
    if ((e = cudaMalloc(&h->dclk, sizeof(tt::DevClock))) != cudaSuccess) return bail(cuda_fail(e, "cudaMalloc(clock)"));
    if ((e = cudaMemset(h->dclk, 0, sizeof(tt::DevClock))) != cudaSuccess) return bail(cuda_fail(e, "zero clock"));
    h->dev_bytes += ring_b + hist_b + hist_b / 2 + pm_b + xo_b + tb_b;
    if ((e = cudaMemset(h->tab, 0, tb_b)) != cudaSuccess) return bail(cuda_fail(e, "zero tab"));
    if ((e = cudaMemcpy(h->perm, pm.data(), pm_b, cudaMemcpyHostToDevice)) != cudaSuccess) return bail(cuda_fail(e, "copy perm"));
    if ((e = cudaMemcpy(h->xoff, xo.data(), xo_b, cudaMemcpyHostToDevice)) != cudaSuccess) return bail(cuda_fail(e, "copy xoff"));
    if (hist_b && (e = cudaMemset(h->hist, 0, hist_b)) != cudaSuccess) return bail(cuda_fail(e, "zero history"));
    if (hist_b && (e = cudaMemset(h->hist_zero, 0, hist_b / 2)) != cudaSuccess)
        return bail(cuda_fail(e, "zero history"));
    // the ring is zeroed so a never-loaded slot can never inject NaN into a CTA's
    // table (apply refuses non-resident ranges anyway)
    if ((e = cudaMemset(h->ring, 0, ring_b)) != cudaSuccess) return bail(cuda_fail(e, "zero ring"));
    if ((e = prepare_plan(h)) != cudaSuccess) return bail(cuda_fail(e, "kernel setup"));
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return bail(cuda_fail(e, "create sync"));
    *out = h;
    return TT_OK;
}

namespace {
// NEXT f2: (re)select the top-n taps of dense ring rows [k_first, k_first + rows)
tt_status select_rows(tt_channel_s* h, int64_t k_first, int64_t rows, cudaStream_t st) {
    if (h->top_n <= 0 || rows <= 0) return TT_OK;
    const int warps = 4;
    const size_t sm = static_cast<size_t>(warps) * h->L * sizeof(float);
    const int64_t nrow = static_cast<int64_t>(h->C) * rows;
    const int64_t grid = std::min<int64_t>((nrow + warps - 1) / warps, int64_t(h->num_sms) * 16);
    tt::tt_select_kernel<<<static_cast<unsigned>(std::max<int64_t>(grid, 1)), warps * 32, sm, st>>>(
        h->ring, h->sring, h->soff, h->xoff, h->C, h->cap, h->L, h->L4, h->top_n, h->n4, k_first, rows);
    TT_CUDA(cudaGetLastError(), "top-n selection launch");
    return TT_OK;
}
}  // namespace

tt_status tt_channel_load_snapshots(tt_channel_t h, const float* gains, int64_t first_index, int64_t count,
                                    tt_stream_t stream) {
    if (!h) return fail(TT_ERR_INVALID_ARG, "NULL handle");
    if (!gains) return fail(TT_ERR_INVALID_ARG, "NULL gains");
    if (first_index < 0 || count <= 0) return fail(TT_ERR_INVALID_ARG, "need first_index >= 0 and count > 0");
    if (count > h->cap) return fail(TT_ERR_INVALID_ARG, "count %lld exceeds snapshot_capacity %lld", (long long)count, (long long)h->cap);
    DeviceGuard dg(h->dev);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the loader kernel reads device memory; a host source goes through device staging
    cudaPointerAttributes attr{};
    cudaError_t pe = cudaPointerGetAttributes(&attr, gains);
    if (pe != cudaSuccess) cudaGetLastError();
    const bool on_device = pe == cudaSuccess && (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged);
    const size_t elems = static_cast<size_t>(h->C) * count * h->L;
    const float2* src = reinterpret_cast<const float2*>(gains);
    if (!on_device) {
        // the staging buffer is shared by every load of the handle: a load on another
        // stream waits for the previous loader kernel to have read it
        if (!h->ev_load) TT_CUDA(cudaEventCreateWithFlags(&h->ev_load, cudaEventDisableTiming), "event create");
        if (elems > h->load_stage_elems) {
            TT_CUDA(cudaEventSynchronize(h->ev_load), "staging drain");
            cudaFree(h->load_stage);
            h->load_stage = nullptr;
            h->load_stage_elems = 0;
            TT_CUDA(cudaMalloc(&h->load_stage, elems * sizeof(float2)), "cudaMalloc(snapshot staging)");
            h->load_stage_elems = elems;
        } else {
            TT_CUDA(cudaStreamWaitEvent(st, h->ev_load, 0), "stream wait");
        }
        TT_CUDA(cudaMemcpyAsync(h->load_stage, gains, elems * sizeof(float2), cudaMemcpyHostToDevice, st), "snapshot H2D");
        src = h->load_stage;
    }
    // snapshot first - 1 gets its difference now if it is resident and stays resident
    const int fix_prev = (h->res_hi > h->res_lo && first_index - 1 >= h->res_lo && first_index - 1 < h->res_hi &&
                          count <= h->cap - 1)
                             ? 1
                             : 0;
    // a block reloaded inside the resident range (it ends before res_hi): snapshot
    // first + count stays resident, so the block's last difference is completed against
    // it now (else that row would keep dg = 0 while intervals through it stay accepted)
    const int64_t hi_new = first_index + count;
    const int fix_next = (h->res_hi > h->res_lo && first_index >= h->res_lo && first_index <= h->res_hi &&
                          hi_new < h->res_hi && count <= h->cap - 1)
                             ? 1
                             : 0;
    const int64_t grid = std::min<int64_t>((static_cast<int64_t>(elems) + 255) / 256, int64_t(h->num_sms) * 16);
    tt::tt_load_kernel<<<static_cast<unsigned>(std::max<int64_t>(grid, 1)), 256, 0, st>>>(
        src, count, first_index, h->ring, h->cap, h->perm, h->C, h->L, fix_prev, fix_next);
    TT_CUDA(cudaGetLastError(), "snapshot loader launch");
    if (!on_device) TT_CUDA(cudaEventRecord(h->ev_load, st), "event record");
    {
        // sparse rows follow the dense rows they are selected from (the previous row's
        // difference was just completed by fix_prev)
        tt_status ss = select_rows(h, first_index - fix_prev, count + fix_prev, st);
        if (ss != TT_OK) return ss;
    }
    const int64_t lo = first_index, hi = first_index + count;
    if (h->res_hi > h->res_lo && lo >= h->res_lo && lo <= h->res_hi) {
        h->res_hi = std::max(h->res_hi, hi);
        h->res_lo = std::max(h->res_lo, h->res_hi - h->cap);
    } else {
        h->res_lo = lo;
        h->res_hi = hi;
    }
    return TT_OK;
}

tt_status tt_channel_apply(tt_channel_t h, const float* in, float* out, int64_t n_samples, float noise_sigma,
                           tt_stream_t stream) {
    tt_status s = check_apply(h, in, out, n_samples, noise_sigma);
    if (s != TT_OK) return s;
    DeviceGuard dg(h->dev);
    s = launch(h, reinterpret_cast<const float2*>(in), reinterpret_cast<float2*>(out), 0, h->C, n_samples,
               noise_sigma, static_cast<cudaStream_t>(stream));
    if (s != TT_OK) return s;
    if (!h->dclock) {
        h->t += n_samples;
        if (h->H > 0) h->p ^= 1;
    }
    return TT_OK;
}

tt_status tt_channel_apply_host(tt_channel_t h, const float* in, float* out, int64_t n_samples, float noise_sigma,
                                tt_stream_t stream) {
    if (h && h->dclock) return fail(TT_ERR_UNSUPPORTED, "apply_host in device-clock mode: use tt_channel_apply");
    tt_status s = check_apply(h, in, out, n_samples, noise_sigma);
    if (s != TT_OK) return s;
    if (h->in_row) return fail(TT_ERR_UNSUPPORTED, "apply_host with an input map: use tt_channel_apply");
    DeviceGuard dg(h->dev);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // chunk of channels per pipeline stage: ~16 MiB of input (short pipeline fill, PCIe
    // duplex kept busy), at least one channel
    const int64_t per_ch = n_samples;
    const char* fc = getenv("TT_HOST_CHUNK_MB");  // experiments
    const int64_t chunk_b = (fc ? std::max<int64_t>(1, atoll(fc)) : int64_t(16)) << 20;
    int64_t cc = std::max<int64_t>(1, chunk_b / (per_ch * 8));
    cc = std::min<int64_t>(cc, h->C);
    const size_t need = static_cast<size_t>(cc * per_ch);
    constexpr int NB = tt_channel_s::kHostBufs;
    if (need > h->stage_elems) {
        if (h->stage) {
            TT_CUDA(cudaStreamSynchronize(h->cs_d2h[0]), "staging drain");
            TT_CUDA(cudaStreamSynchronize(h->cs_d2h[1]), "staging drain");
            cudaFree(h->stage);
            h->stage = nullptr;
            h->stage_elems = 0;
        }
        TT_CUDA(cudaMalloc(&h->stage, need * 2 * NB * sizeof(float2)), "cudaMalloc(host-path staging)");
        h->stage_elems = need;
        if (!h->cs_h2d[0]) {
            for (int k = 0; k < 2; ++k) {
                TT_CUDA(cudaStreamCreateWithFlags(&h->cs_h2d[k], cudaStreamNonBlocking), "stream create");
                TT_CUDA(cudaStreamCreateWithFlags(&h->cs_d2h[k], cudaStreamNonBlocking), "stream create");
                TT_CUDA(cudaEventCreateWithFlags(&h->ev_done[k], cudaEventDisableTiming), "event create");
            }
            for (int i = 0; i < NB; ++i) {
                TT_CUDA(cudaEventCreateWithFlags(&h->ev_h2d[i], cudaEventDisableTiming), "event create");
                TT_CUDA(cudaEventCreateWithFlags(&h->ev_k[i], cudaEventDisableTiming), "event create");
                TT_CUDA(cudaEventCreateWithFlags(&h->ev_free[i], cudaEventDisableTiming), "event create");
                TT_CUDA(cudaEventRecord(h->ev_free[i], h->cs_d2h[i & 1]), "event record");
            }
            TT_CUDA(cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming), "event create");
        }
    }
    // the copy streams start after everything already enqueued on `stream`; chunk i uses
    // buffer i % NB and the copy streams of parity i % 2 (two DMA queues per direction
    // keep the PCIe link busier in both directions)
    TT_CUDA(cudaEventRecord(h->ev_start, st), "event record");
    for (int k = 0; k < 2; ++k) TT_CUDA(cudaStreamWaitEvent(h->cs_h2d[k], h->ev_start, 0), "stream wait");
    const float2* hin = reinterpret_cast<const float2*>(in);
    float2* hout = reinterpret_cast<float2*>(out);
    int i = 0;
    for (int64_t c0 = 0; c0 < h->C; c0 += cc, ++i) {
        const int b = i % NB, q = i & 1;
        const int64_t c1 = std::min<int64_t>(h->C, c0 + cc);
        const size_t bytes = static_cast<size_t>((c1 - c0) * per_ch) * sizeof(float2);
        float2* din = h->stage + static_cast<size_t>(b) * 2 * need;
        float2* dout = din + need;
        TT_CUDA(cudaStreamWaitEvent(h->cs_h2d[q], h->ev_free[b], 0), "stream wait");
        TT_CUDA(cudaMemcpyAsync(din, hin + c0 * per_ch, bytes, cudaMemcpyHostToDevice, h->cs_h2d[q]), "H2D");
        TT_CUDA(cudaEventRecord(h->ev_h2d[b], h->cs_h2d[q]), "event record");
        TT_CUDA(cudaStreamWaitEvent(st, h->ev_h2d[b], 0), "stream wait");
        s = launch(h, din, dout, static_cast<int32_t>(c0), static_cast<int32_t>(c1), n_samples, noise_sigma, st);
        if (s != TT_OK) return s;
        TT_CUDA(cudaEventRecord(h->ev_k[b], st), "event record");
        TT_CUDA(cudaStreamWaitEvent(h->cs_d2h[q], h->ev_k[b], 0), "stream wait");
        TT_CUDA(cudaMemcpyAsync(hout + c0 * per_ch, dout, bytes, cudaMemcpyDeviceToHost, h->cs_d2h[q]), "D2H");
        TT_CUDA(cudaEventRecord(h->ev_free[b], h->cs_d2h[q]), "event record");
    }
    // `stream` reaches this point only when every D2H has landed
    for (int k = 0; k < 2; ++k) {
        TT_CUDA(cudaEventRecord(h->ev_done[k], h->cs_d2h[k]), "event record");
        TT_CUDA(cudaStreamWaitEvent(st, h->ev_done[k], 0), "stream wait");
    }
    h->t += n_samples;
    if (h->H > 0) h->p ^= 1;
    return TT_OK;
}

tt_status tt_channel_set_top_n(tt_channel_t h, int32_t top_n) {
    if (!h) return fail(TT_ERR_INVALID_ARG, "NULL handle");
    if (h->dclock) return fail(TT_ERR_UNSUPPORTED, "set_top_n in device-clock mode (it may change the plan)");
    if (top_n < 0) return fail(TT_ERR_INVALID_ARG, "top_n must be >= 0");
    DeviceGuard dg(h->dev);
    const int32_t n = (top_n == 0 || top_n >= h->L) ? 0 : top_n;
    if (n == h->top_n) return TT_OK;
    TT_CUDA(cudaDeviceSynchronize(), "top-n drain");
    // back to the dense state first; any failure below leaves the handle dense with a
    // dense plan (the plan always matches top_n: a sparse plan stages L = top_n wide
    // coefficient rows and would overrun shared memory on a dense apply)
    auto to_dense = [h]() {
        cudaFree(h->sring);
        cudaFree(h->soff);
        h->sring = nullptr;
        h->soff = nullptr;
        h->top_n = 0;
        h->n4 = 0;
    };
    auto fail_dense = [h, &to_dense](cudaError_t e, const char* what) {
        to_dense();
        const tt_status s = cuda_fail(e, what);
        const cudaError_t pe = prepare_plan(h);
        if (pe != cudaSuccess) cudaGetLastError();
        return s;
    };
    to_dense();
    cudaError_t e = cudaSuccess;
    if (n > 0) {
        const int32_t n4 = (n + 1 + 3) & ~3;
        const size_t ring_b = (static_cast<size_t>(h->C) * h->cap * n + 1) * sizeof(float4);
        const size_t off_b = static_cast<size_t>(h->C) * h->cap * n4 * sizeof(int32_t);
        if ((e = cudaMalloc(&h->sring, ring_b)) != cudaSuccess) return fail_dense(e, "cudaMalloc(sparse ring)");
        if ((e = cudaMalloc(&h->soff, off_b)) != cudaSuccess) return fail_dense(e, "cudaMalloc(sparse offsets)");
        if ((e = cudaMemset(h->sring, 0, ring_b)) != cudaSuccess) return fail_dense(e, "zero ring");
        if ((e = cudaMemset(h->soff, 0, off_b)) != cudaSuccess) return fail_dense(e, "zero offsets");
        // process-wide attribute: the largest any handle can need (4 warps x TT_MAX_TAPS
        // magnitudes), so a later handle with fewer taps never lowers it
        if (h->L * sizeof(float) * 4 > 48 * 1024 &&
            (e = cudaFuncSetAttribute(tt::tt_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(TT_MAX_TAPS * sizeof(float) * 4))) != cudaSuccess)
            return fail_dense(e, "selection smem");
        h->top_n = n;
        h->n4 = n4;
    }
    e = prepare_plan(h);
    if (e != cudaSuccess && h->top_n > 0) return fail_dense(e, "plan");
    if (e != cudaSuccess) return cuda_fail(e, "plan");
    if (h->top_n > 0 && h->res_hi > h->res_lo) {
        tt_status s = select_rows(h, h->res_lo, h->res_hi - h->res_lo, nullptr);
        if (s != TT_OK) return s;
    }
    TT_CUDA(cudaDeviceSynchronize(), "top-n selection");
    return TT_OK;
}

tt_status tt_channel_set_input_map(tt_channel_t h, const int32_t* rows, int32_t num_rows) {
    if (!h) return fail(TT_ERR_INVALID_ARG, "NULL handle");
    DeviceGuard dg(h->dev);
    if (!rows) {
        if (h->in_row) {
            TT_CUDA(cudaDeviceSynchronize(), "input map drain");
            cudaFree(h->in_row);  // the map owns only its row table, never the sparse ring
        }
        h->in_row = nullptr;
        h->in_rows = 0;
        return TT_OK;
    }
    if (num_rows <= 0) return fail(TT_ERR_INVALID_ARG, "num_rows must be > 0");
    for (int32_t c = 0; c < h->C; ++c)
        if (rows[c] < 0 || rows[c] >= num_rows)
            return fail(TT_ERR_INVALID_ARG, "rows[%d] = %d outside [0, %d)", c, rows[c], num_rows);
    if (!h->in_row) TT_CUDA(cudaMalloc(&h->in_row, static_cast<size_t>(h->C) * sizeof(int32_t)), "cudaMalloc(input map)");
    else TT_CUDA(cudaDeviceSynchronize(), "input map drain");
    TT_CUDA(cudaMemcpy(h->in_row, rows, static_cast<size_t>(h->C) * sizeof(int32_t), cudaMemcpyHostToDevice),
            "copy input map");
    h->in_rows = num_rows;
    return TT_OK;
}

tt_status tt_channel_apply_aggregate(tt_channel_t h, const float* in, float* out, float* agg, int32_t group_size,
                                     int64_t n_samples, float noise_sigma, tt_stream_t stream) {
    tt_status s = check_apply(h, in, agg, n_samples, noise_sigma);
    if (s != TT_OK) return s;
    if (group_size <= 0 || h->C % group_size != 0)
        return fail(TT_ERR_INVALID_ARG, "group_size %d must divide the %d channels", group_size, h->C);
    if (out == in) return fail(TT_ERR_INVALID_ARG, "in and out must not overlap");
    DeviceGuard dg(h->dev);
    AggReq ar;
    ar.agg = reinterpret_cast<float2*>(agg);
    ar.G = group_size;
    const int32_t KC = std::min<int32_t>(group_size, TT_AGG_CHUNK);
    const int32_t nchunks = (group_size + KC - 1) / KC;
    const bool tiled = h->plan.tiled[noise_sigma > 0.0f ? 1 : 0].R != 0;
    // scratch: chunk sums (tiled, > 1 chunk) or per-channel outputs (generic, out == NULL)
    size_t need = 0;
    if (tiled && nchunks > 1) need = static_cast<size_t>(h->C / group_size) * nchunks * n_samples;
    if (!tiled && !out) need = static_cast<size_t>(h->C) * n_samples;
    if (need > h->agg_scratch_elems) {
        if (h->agg_scratch) {
            TT_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "scratch drain");
            cudaFree(h->agg_scratch);
            h->agg_scratch = nullptr;
            h->agg_scratch_elems = 0;
        }
        TT_CUDA(cudaMalloc(&h->agg_scratch, need * sizeof(float2)), "cudaMalloc(aggregate scratch)");
        h->agg_scratch_elems = need;
    }
    ar.scratch = h->agg_scratch;
    s = launch(h, reinterpret_cast<const float2*>(in), reinterpret_cast<float2*>(out), 0, h->C, n_samples,
               noise_sigma, static_cast<cudaStream_t>(stream), ar);
    if (s != TT_OK) return s;
    if (!h->dclock) {
        h->t += n_samples;
        if (h->H > 0) h->p ^= 1;
    }
    return TT_OK;
}

tt_status tt_synth_jakes(const float* path_delay, const float* path_power, int32_t num_ue, int32_t num_paths,
                         int32_t num_sinusoids, double nu, uint64_t seed, int64_t channel_offset, int64_t first_index,
                         int64_t count, int32_t* delays_out, float* gains_out, tt_stream_t stream) {
    if (!path_delay || !path_power || !gains_out) return fail(TT_ERR_INVALID_ARG, "NULL path_delay/path_power/gains_out");
    if (num_ue <= 0 || num_paths <= 0 || num_sinusoids <= 0 || count <= 0 || first_index < 0 || channel_offset < 0)
        return fail(TT_ERR_INVALID_ARG, "need num_ue, num_paths, num_sinusoids, count > 0 and first_index, "
                                        "channel_offset >= 0");
    if (!(nu >= 0.0) || !(nu < 0.5)) return fail(TT_ERR_INVALID_ARG, "nu = f_D S / f_s must be in [0, 0.5) (Nyquist)");
    const int64_t CP = static_cast<int64_t>(num_ue) * num_paths;
    if (2 * static_cast<int64_t>(num_paths) > TT_MAX_TAPS) return fail(TT_ERR_INVALID_ARG, "2 num_paths > TT_MAX_TAPS");
    for (int64_t i = 0; i < CP; ++i) {
        if (!(path_delay[i] >= 0.0f) || !(path_delay[i] + 1.0f <= static_cast<float>(TT_MAX_DELAY)) ||
            !(path_power[i] >= 0.0f) || !std::isfinite(path_power[i]))
            return fail(TT_ERR_INVALID_ARG, "path %lld: delay must be in [0, %d - 1], power finite and >= 0",
                        (long long)i, TT_MAX_DELAY);
        if (delays_out) {
            const int32_t b = static_cast<int32_t>(floorf(path_delay[i]));
            const int64_t c = i / num_paths, p = i % num_paths;
            delays_out[c * 2 * num_paths + 2 * p] = b;
            delays_out[c * 2 * num_paths + 2 * p + 1] = b + 1;
        }
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int dev = 0, sms = 148;
    TT_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    // per-device scratch (path table, delays, powers), kept across calls and grown on
    // demand; calls on one device are serialised by the lock and by `stream` ordering
    // (the next call's copies are ordered after this call's kernels via the event)
    static std::mutex mu;
    static std::map<int, SynthScratch> scratch;
    std::lock_guard<std::mutex> lk(mu);
    SynthScratch& sc = scratch[dev];
    const size_t need = static_cast<size_t>(CP) * (2 * sizeof(float) + num_sinusoids * sizeof(double2)) + 256;
    if (need > sc.bytes) {
        if (sc.buf) {
            TT_CUDA(cudaDeviceSynchronize(), "synthesis scratch drain");
            cudaFree(sc.buf);
            sc.buf = nullptr;
            sc.bytes = 0;
        }
        TT_CUDA(cudaMalloc(&sc.buf, need), "cudaMalloc(synthesis scratch)");
        sc.bytes = need;
    }
    if (!sc.done) TT_CUDA(cudaEventCreateWithFlags(&sc.done, cudaEventDisableTiming), "event create");
    TT_CUDA(cudaStreamWaitEvent(st, sc.done, 0), "stream wait");  // previous users of the scratch
    double2* tab = reinterpret_cast<double2*>(sc.buf);
    float* dtau = reinterpret_cast<float*>(sc.buf + static_cast<size_t>(CP) * num_sinusoids * sizeof(double2));
    float* dpw = dtau + CP;
    cudaError_t e;
    if ((e = cudaMemcpyAsync(dtau, path_delay, CP * sizeof(float), cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dpw, path_power, CP * sizeof(float), cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return cuda_fail(e, "copy paths");
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tt = CP * num_sinusoids;
    tt::tt_synth_table_kernel<<<static_cast<unsigned>(std::min<int64_t>((tt + 255) / 256, int64_t(sms) * 16)), 256, 0,
                                st>>>(num_ue, num_paths, num_sinusoids, nu, static_cast<uint32_t>(seed),
                                      static_cast<uint32_t>(seed >> 32), channel_offset, tab);
    const int64_t tg = CP * ((count + tt::kSynthBlock - 1) / tt::kSynthBlock);
    tt::tt_synth_gain_kernel<<<static_cast<unsigned>(std::min<int64_t>((tg + 127) / 128, int64_t(sms) * 32)), 128, 0,
                               st>>>(num_ue, num_paths, num_sinusoids, tab, dtau, dpw, first_index, count,
                                     reinterpret_cast<float2*>(gains_out));
    TT_CUDA(cudaGetLastError(), "synthesis launch");
    TT_CUDA(cudaEventRecord(sc.done, st), "event record");
    return TT_OK;
}

tt_status tt_channel_reset(tt_channel_t h, tt_stream_t stream) {
    if (!h) return fail(TT_ERR_INVALID_ARG, "NULL handle");
    DeviceGuard dg(h->dev);
    // no device work for the delay line: calls at t = 0 read the zero buffer
    h->t = 0;
    h->p = 0;
    if (h->dclock) {
        tt::tt_set_clock_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(h->dclk, 0, 0);
        TT_CUDA(cudaGetLastError(), "reset clock");
    }
    return TT_OK;
}

tt_status tt_channel_set_device_clock(tt_channel_t h, int32_t enable, tt_stream_t stream) {
    if (!h) return fail(TT_ERR_INVALID_ARG, "NULL handle");
    DeviceGuard dg(h->dev);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (enable && !h->dclock) {
        if ((h->plan.kind != TT_KERNEL_TILED && h->plan.kind != TT_KERNEL_DW) || h->plan.tiled[0].R == 0 ||
            h->plan.tiled[1].R == 0)
            return fail(TT_ERR_UNSUPPORTED, "device-clock mode needs the tiled kernel for this handle's shape");
        const int64_t A = clock_grid(h);
        if (h->t % A != 0)
            return fail(TT_ERR_UNSUPPORTED, "device-clock mode must start at t %% %lld == 0 (t = %lld)", (long long)A,
                        (long long)h->t);
        tt::tt_set_clock_kernel<<<1, 1, 0, st>>>(h->dclk, h->t, h->p);
        TT_CUDA(cudaGetLastError(), "set clock");
        h->dclock = true;
    } else if (!enable && h->dclock) {
        tt::DevClock c{};
        TT_CUDA(cudaStreamSynchronize(st), "clock sync");
        TT_CUDA(cudaMemcpy(&c, h->dclk, sizeof(c), cudaMemcpyDeviceToHost), "read clock");
        h->t = c.t;
        h->p = c.par;
        h->dclock = false;
    }
    return TT_OK;
}

tt_status tt_channel_synchronize(tt_channel_t h, tt_stream_t stream) {
    if (!h) return fail(TT_ERR_INVALID_ARG, "NULL handle");
    DeviceGuard dg(h->dev);
    TT_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "stream synchronize");
    return TT_OK;
}

tt_status tt_channel_get_info(tt_channel_t h, tt_channel_info* info) {
    if (!h || !info) return fail(TT_ERR_INVALID_ARG, "NULL handle or info");
    info->num_ue = h->C;
    info->num_taps = h->L;
    info->snapshot_period = h->S;
    info->history = h->H;
    info->max_delay = h->maxD;
    info->device = h->dev;
    info->t = h->t;
    info->snapshot_capacity = h->cap;
    info->resident_lo = h->res_lo;
    info->resident_hi = h->res_hi;
    info->channel_offset = h->chan_off;
    info->seed = h->seed;
    info->device_bytes = static_cast<int64_t>(h->dev_bytes + h->stage_elems * 2 * tt_channel_s::kHostBufs * sizeof(float2) +
                                              h->load_stage_elems * sizeof(float2) +
                                              h->agg_scratch_elems * sizeof(float2));
    info->kernel = h->plan.kind;
    info->top_n = h->top_n;
    info->device_clock = h->dclock ? 1 : 0;
    info->outputs_per_thread = h->plan.kind == TT_KERNEL_RW    ? h->plan.rw_R
                               : h->plan.kind == TT_KERNEL_DW    ? tt::dw::R
                               : h->plan.kind == TT_KERNEL_TILED ? h->plan.tiled[1].R
                                                                 : 0;
    info->launches_per_apply = h->plan.kind == TT_KERNEL_GENERIC ? 2 : 1;
    return TT_OK;
}

tt_status tt_channel_destroy(tt_channel_t h) {
    if (!h) return TT_OK;
    DeviceGuard dg(h->dev);
    cudaDeviceSynchronize();
    free_all(h);
    delete h;
    return TT_OK;
}

}  // extern "C"
