// microbench.cu — B200 (sm_100a) microbenchmarks that decide the kernel design
// (SURVEY.md §7.1 step 0): FP32 lane throughput of scalar FFMA vs packed FFMA2,
// shared-memory LDS.64 bandwidth, and the per-output-tap cost of the convolution's
// inner loop with operands from registers vs from shared memory.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
//   ./microbench > gpurun_out/microbench.json
//
// Rates are per SM per SM-clock, from in-kernel clock64() spans (median over CTAs).
#include <cuda_runtime.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e = (x);                                                      \
        if (e != cudaSuccess) {                                                   \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            return 1;                                                             \
        }                                                                         \
    } while (0)

constexpr int ITERS = 4096;

__global__ void k_ffma(float* out, long long* cyc, float a, float b) {
    float c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3f + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = __fmaf_rn(c[i], a, b);
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma2(float* out, long long* cyc, float a, float b) {
    float2 c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    const float2 aa = make_float2(a, a * 0.5f), bb = make_float2(b, b * 2.f);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = __ffma2_rn(c[i], aa, bb);
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i].x + c[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// the convolution MAC body, operands from registers: 8 outputs x 1 tap per iteration
__global__ void k_mac_reg(float* out, long long* cyc, float4 q) {
    float2 A[8], B[8], x[8];
    float al[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        A[r] = B[r] = make_float2(0, 0);
        x[r] = make_float2(threadIdx.x * 1e-3f + r, r * 0.25f);
        al[r] = r * (1.f / 8);
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS / 4; ++it) {
        const float2 g = make_float2(q.x + it, q.y), dg = make_float2(q.z, q.w);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const float2 h = __ffma2_rn(make_float2(al[r], al[r]), dg, g);
            A[r] = __ffma2_rn(make_float2(h.x, h.x), x[r], A[r]);
            B[r] = __ffma2_rn(make_float2(h.y, h.y), x[r], B[r]);
        }
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) s += A[r].x + A[r].y + B[r].x + B[r].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}


// MAC-body variants (operands in registers). MODE 0: per output h/A/B FFMA2 (kernel v1);
// 1: all h first (FFMA2) then A/B FFMA2; 2: all h first (scalar) then 4 scalar FFMA in
// reuse-friendly order; 3: scalar with 2 chained accumulators; 4: h FFMA2 first, MAC scalar.
template <int MODE>
__global__ void k_mac_var(float* out, long long* cyc, float4 q, const float* init) {
    float2 A[8], B[8], x[8];
    float al[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        A[r] = B[r] = make_float2(0, 0);
        x[r] = make_float2(init[threadIdx.x + r], init[threadIdx.x + r + 8]);
        al[r] = init[threadIdx.x + r + 16];
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS / 4; ++it) {
        const float2 g = make_float2(q.x + it, q.y - it), dg = make_float2(q.z, q.w);
        if (MODE == 0) {
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const float2 h = __ffma2_rn(make_float2(al[r], al[r]), dg, g);
                A[r] = __ffma2_rn(make_float2(h.x, h.x), x[r], A[r]);
                B[r] = __ffma2_rn(make_float2(h.y, h.y), x[r], B[r]);
            }
        } else if (MODE == 1 || MODE == 4) {
            float2 h[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) h[r] = __ffma2_rn(make_float2(al[r], al[r]), dg, g);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                if (MODE == 1) {
                    A[r] = __ffma2_rn(make_float2(h[r].x, h[r].x), x[r], A[r]);
                    B[r] = __ffma2_rn(make_float2(h[r].y, h[r].y), x[r], B[r]);
                } else {
                    A[r].x = __fmaf_rn(h[r].x, x[r].x, A[r].x);
                    B[r].x = __fmaf_rn(h[r].y, x[r].x, B[r].x);
                    B[r].y = __fmaf_rn(h[r].y, x[r].y, B[r].y);
                    A[r].y = __fmaf_rn(h[r].x, x[r].y, A[r].y);
                }
            }
        } else if (MODE == 2) {
            float hr[8], hi[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) hr[r] = __fmaf_rn(al[r], dg.x, g.x);
#pragma unroll
            for (int r = 0; r < 8; ++r) hi[r] = __fmaf_rn(al[r], dg.y, g.y);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                A[r].x = __fmaf_rn(hr[r], x[r].x, A[r].x);
                B[r].x = __fmaf_rn(hi[r], x[r].x, B[r].x);
                B[r].y = __fmaf_rn(hi[r], x[r].y, B[r].y);
                A[r].y = __fmaf_rn(hr[r], x[r].y, A[r].y);
            }
        } else {
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const float hr = __fmaf_rn(al[r], dg.x, g.x), hi = __fmaf_rn(al[r], dg.y, g.y);
                A[r].x = __fmaf_rn(hr, x[r].x, A[r].x);
                A[r].x = __fmaf_rn(-hi, x[r].y, A[r].x);
                A[r].y = __fmaf_rn(hr, x[r].y, A[r].y);
                A[r].y = __fmaf_rn(hi, x[r].x, A[r].y);
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) s += A[r].x + A[r].y + B[r].x + B[r].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// the kernel's real inner loop: x from shared memory (lane-interleaved, conflict-free)
__global__ void k_mac_smem(float* out, long long* cyc, const int* dl, int L) {
    __shared__ float2 xs[2048 + 2048];
    __shared__ float4 cf[64];
    __shared__ int sd[64];
    for (int i = threadIdx.x; i < 2048 + 2048; i += blockDim.x) xs[i] = make_float2(i * 1e-3f, 1.f - i * 1e-4f);
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        cf[i] = make_float4(i * 0.1f, 0.2f, 0.01f, -0.02f);
        sd[i] = dl[i];
    }
    float2 A[8], B[8];
    float al[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        A[r] = B[r] = make_float2(0, 0);
        al[r] = r * (1.f / 8);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float2* xb = xs + 2048 + warp * 256 + lane;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < 16; ++it) {
#pragma unroll 2
        for (int j = 0; j < L; ++j) {
            const float4 q = cf[j];
            const float2* xp = xb - sd[j];
            const float2 g = make_float2(q.x, q.y), dg = make_float2(q.z, q.w);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const float2 xv = xp[r * 32];
                const float2 h = __ffma2_rn(make_float2(al[r], al[r]), dg, g);
                A[r] = __ffma2_rn(make_float2(h.x, h.x), xv, A[r]);
                B[r] = __ffma2_rn(make_float2(h.y, h.y), xv, B[r]);
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) s += A[r].x + A[r].y + B[r].x + B[r].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_lds64(float* out, long long* cyc) {
    __shared__ float2 xs[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) xs[i] = make_float2(i, -i);
    __syncthreads();
    float2 acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) acc[r] = make_float2(0, 0);
    long long t0 = clock64();
    for (int it = 0; it < ITERS / 8; ++it) {
        const int base = ((it * 97) & 15) * 256 + threadIdx.x;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const float2 v = xs[(base + r * 256) & 4095];
            acc[r].x += v.x;
            acc[r].y += v.y;
        }
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) s += acc[r].x + acc[r].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

static double median(std::vector<long long> v) {
    std::sort(v.begin(), v.end());
    return (double)v[v.size() / 2];
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_per_sm\": %zu, \"hbm_bytes\": %zu",
           prop.name, sms, prop.l2CacheSize, prop.sharedMemPerMultiprocessor, prop.totalGlobalMem);
    const int threads = 256;
    float* out;
    long long* cyc;
    const int maxb = sms * 8;
    CK(cudaMalloc(&out, sizeof(float) * maxb * threads));
    CK(cudaMalloc(&cyc, sizeof(long long) * maxb));
    int* dl;
    std::vector<int> hd(64);
    for (int i = 0; i < 64; ++i) hd[i] = (i * 1021) % 1024 / 2;  // arbitrary delays < 2048
    std::sort(hd.begin(), hd.end());
    CK(cudaMalloc(&dl, 64 * sizeof(int)));
    CK(cudaMemcpy(dl, hd.data(), 64 * sizeof(int), cudaMemcpyHostToDevice));
    std::vector<long long> h(maxb);
    float* initp;
    {
        std::vector<float> hi(1024);
        for (int i = 0; i < 1024; ++i) hi[i] = 0.001f * (i % 97) - 0.03f;
        CK(cudaMalloc(&initp, 1024 * sizeof(float)));
        CK(cudaMemcpy(initp, hi.data(), 1024 * sizeof(float), cudaMemcpyHostToDevice));
    }
    for (int per_sm : {1, 2, 3}) {
        const int blocks = sms * per_sm;
        // warm-up + measure each kernel
        auto run = [&](const char* name, double ops_per_thread, auto launch) -> int {
            launch(blocks);
            CK(cudaDeviceSynchronize());
            launch(blocks);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(h.data(), cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost));
            std::vector<long long> v(h.begin(), h.begin() + blocks);
            const double c = median(v);
            printf(", \"%s_per_sm%d\": %.3f", name, per_sm, ops_per_thread * threads * per_sm / c);
            return 0;
        };
        run("ffma_lanes_per_clk", 8.0 * ITERS, [&](int b) { k_ffma<<<b, threads>>>(out, cyc, 0.999f, 1e-3f); });
        run("ffma2_lanes_per_clk", 16.0 * ITERS, [&](int b) { k_ffma2<<<b, threads>>>(out, cyc, 0.999f, 1e-3f); });
        run("mac_reg_outtaps_per_clk", 8.0 * (ITERS / 4),
            [&](int b) { k_mac_reg<<<b, threads>>>(out, cyc, make_float4(1, 2, 3, 4)); });
        run("mac_v0_outtaps_per_clk", 8.0 * (ITERS / 4), [&](int b) { k_mac_var<0><<<b, threads>>>(out, cyc, make_float4(1, 2, 3, 4), initp); });
        run("mac_v1_outtaps_per_clk", 8.0 * (ITERS / 4), [&](int b) { k_mac_var<1><<<b, threads>>>(out, cyc, make_float4(1, 2, 3, 4), initp); });
        run("mac_v2_outtaps_per_clk", 8.0 * (ITERS / 4), [&](int b) { k_mac_var<2><<<b, threads>>>(out, cyc, make_float4(1, 2, 3, 4), initp); });
        run("mac_v3_outtaps_per_clk", 8.0 * (ITERS / 4), [&](int b) { k_mac_var<3><<<b, threads>>>(out, cyc, make_float4(1, 2, 3, 4), initp); });
        run("mac_v4_outtaps_per_clk", 8.0 * (ITERS / 4), [&](int b) { k_mac_var<4><<<b, threads>>>(out, cyc, make_float4(1, 2, 3, 4), initp); });
        run("mac_smem_L48_outtaps_per_clk", 8.0 * 16 * 48, [&](int b) { k_mac_smem<<<b, threads>>>(out, cyc, dl, 48); });
        run("lds64_bytes_per_clk", 8.0 * 8 * (ITERS / 8), [&](int b) { k_lds64<<<b, threads>>>(out, cyc); });
    }
    printf("}\n");
    return 0;
}
