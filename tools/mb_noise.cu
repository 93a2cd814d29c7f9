// mb_noise.cu — throughput of the tiled kernel's noise epilogue alone (tt_conv.cuh,
// consume_tile_plain, even tile base): per lane 8 rows 32 apart, one Philox4x32-10 call
// per row pair shared by a lane pair through two shuffles, the packed tt-normal-v1
// transform of two samples, y = acc + w. W warps per CTA, one CTA per SM; samples per
// SM-clock (clock64 spans, median over CTAs). Variants (template V):
//   0: the product's epilogue;
//   1: the four row pairs' Philox calls issued before any transform (more independent chains);
//   2: as 0, with combine + noise add as packed FFMA2/FADD2 (acc.re - B.im via a (-1, 1) multiply).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_noise tools/mb_noise.cu && ./mb_noise
#include <cuda_runtime.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#include "../paper_2601_08217_b200/csrc/tt_noise.cuh"

constexpr int ITERS = 256;

template <int W, int V, int R = 8>
__global__ void __launch_bounds__(W * 32, 1) k_noise(float* out, long long* cyc, float sc) {
    const int lane = threadIdx.x & 31;
    const bool ev = (lane & 1) == 0;
    float2 A[R], B[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        A[r] = make_float2(1e-3f * (threadIdx.x + r), 2e-3f * r);
        B[r] = make_float2(-1e-3f * r, 3e-3f * threadIdx.x);
    }
    float2 acc = make_float2(0.f, 0.f);
    const uint32_t cg = blockIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
        const int64_t nb = static_cast<int64_t>(it) * 8192 + (threadIdx.x >> 5) * 256 + lane;  // even base
        float2 o[R];
        if constexpr (V == 2) {
#pragma unroll
            for (int r = 0; r < R; ++r)
                o[r] = __ffma2_rn(make_float2(B[r].y, B[r].x), make_float2(-1.f, 1.f), A[r]);
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) o[r] = make_float2(__fsub_rn(A[r].x, B[r].y), __fadd_rn(A[r].y, B[r].x));
        }
        if constexpr (V == 1) {
            tt::u32x4 q[R / 2];
#pragma unroll
            for (int r = 0; r < R; r += 2) {
                const uint64_t m = static_cast<uint64_t>(nb + (ev ? r : r + 1) * 32) >> 1;
                q[r / 2] = tt::philox4x32_10(static_cast<uint32_t>(m), static_cast<uint32_t>(m >> 32), cg, 0u, 0x1234u,
                                             0x5678u);
            }
#pragma unroll
            for (int r = 0; r < R; r += 2) {
                const tt::u32x4 qq = q[r / 2];
                const uint32_t s0 = ev ? qq.c : qq.a, s1 = ev ? qq.d : qq.b;
                const uint32_t v0 = __shfl_xor_sync(0xffffffffu, s0, 1);
                const uint32_t v1 = __shfl_xor_sync(0xffffffffu, s1, 1);
                float2 wa, wb;
                tt::noise_from_words2(ev ? qq.a : v0, ev ? qq.b : v1, ev ? v0 : qq.c, ev ? v1 : qq.d, sc, wa, wb);
                o[r] = make_float2(__fadd_rn(o[r].x, wa.x), __fadd_rn(o[r].y, wa.y));
                o[r + 1] = make_float2(__fadd_rn(o[r + 1].x, wb.x), __fadd_rn(o[r + 1].y, wb.y));
            }
        } else {
#pragma unroll
            for (int r = 0; r < R; r += 2) {
                const uint64_t m = static_cast<uint64_t>(nb + (ev ? r : r + 1) * 32) >> 1;
                const tt::u32x4 qq = tt::philox4x32_10(static_cast<uint32_t>(m), static_cast<uint32_t>(m >> 32), cg, 0u,
                                                       0x1234u, 0x5678u);
                const uint32_t s0 = ev ? qq.c : qq.a, s1 = ev ? qq.d : qq.b;
                const uint32_t v0 = __shfl_xor_sync(0xffffffffu, s0, 1);
                const uint32_t v1 = __shfl_xor_sync(0xffffffffu, s1, 1);
                float2 wa, wb;
                tt::noise_from_words2(ev ? qq.a : v0, ev ? qq.b : v1, ev ? v0 : qq.c, ev ? v1 : qq.d, sc, wa, wb);
                if constexpr (V == 2) {
                    o[r] = __fadd2_rn(o[r], wa);
                    o[r + 1] = __fadd2_rn(o[r + 1], wb);
                } else {
                    o[r] = make_float2(__fadd_rn(o[r].x, wa.x), __fadd_rn(o[r].y, wa.y));
                    o[r + 1] = make_float2(__fadd_rn(o[r + 1].x, wb.x), __fadd_rn(o[r + 1].y, wb.y));
                }
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            acc.x += o[r].x;
            acc.y += o[r].y;
        }
    }
    __syncthreads();
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int W, int V, int R = 8>
void run(float* out, long long* cyc, int sms, bool first) {
    auto k = k_noise<W, V, R>;
    const int smem = 200 * 1024;  // one CTA per SM
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int i = 0; i < 2; ++i) k<<<sms, W * 32, smem>>>(out, cyc, 0.2236f);
    cudaDeviceSynchronize();
    std::vector<long long> h(sms);
    cudaMemcpy(h.data(), cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    std::sort(h.begin(), h.end());
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k);
    printf("%s{\"warps\": %d, \"variant\": %d, \"rows\": %d, \"regs\": %d, \"samples_per_clk_per_sm\": %.3f}",
           first ? "" : ",\n", W, V, R, fa.numRegs, (double)W * 32 * R * ITERS / h[sms / 2]);
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    const int sms = prop.multiProcessorCount;
    float* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(float) * sms * 1024);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    printf("[\n");
    run<4, 0>(out, cyc, sms, true);
    run<8, 0>(out, cyc, sms, false);
    run<16, 0>(out, cyc, sms, false);
    run<16, 1>(out, cyc, sms, false);
    run<16, 2>(out, cyc, sms, false);
    run<32, 0>(out, cyc, sms, false);
    run<8, 0, 16>(out, cyc, sms, false);
    run<8, 1, 16>(out, cyc, sms, false);
    run<8, 1>(out, cyc, sms, false);
    run<12, 1, 16>(out, cyc, sms, false);
    printf("\n]\n");
    return 0;
}
